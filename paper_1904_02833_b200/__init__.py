"""B200-native implicit compliant-constraint step for the arXiv:1904.02833
soft-snake simulator (drop-in for the `softsnake` package's hot path).

Public names mirror softsnake/__init__.py:13-36 for the stepping path:
scene construction, Simulator.step(), state readback. The step itself runs
in hand-written sm_100a CUDA (paper_1904_02833_b200/lib/libsoftsnake_b200.so)
behind the C ABI in include/softsnake_b200.h; there is no CPU fallback.
"""
from .model import (GaitParams, SnakeModel, build_bend_fixture, build_snake,
                    gait_commands, heading_yaw)
from .scene import SceneConfig
from .simulator import BatchedSimulator, Simulator, SolverConfig, StepStats
from .structures import (PSI_TO_PA, AttachmentConstraint, AttachmentSet,
                         ChannelBank, DistanceConstraint, DistanceSet,
                         HingeJoint, HingeSet, ParticleSet, PneumaticChannel,
                         RigidBody, StrainLaw, SystemState, TetraElement,
                         TetraSet, WheelCollider, center_of_mass,
                         kinetic_energy, route_antagonistic, update_pressure)

__version__ = "0.1.0"

__all__ = [
    "AttachmentConstraint", "AttachmentSet", "BatchedSimulator", "ChannelBank",
    "DistanceConstraint", "DistanceSet", "GaitParams", "HingeJoint", "HingeSet",
    "ParticleSet", "PneumaticChannel", "PSI_TO_PA", "RigidBody", "SceneConfig",
    "Simulator", "SnakeModel", "SolverConfig", "StepStats", "StrainLaw",
    "SystemState", "TetraElement", "TetraSet", "WheelCollider",
    "build_bend_fixture", "build_snake", "center_of_mass", "gait_commands",
    "heading_yaw", "kinetic_energy", "route_antagonistic", "update_pressure",
    "__version__",
]
