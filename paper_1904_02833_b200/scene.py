"""Scene description (drop-in for softsnake/scene.py:16-189).

A table of (section, key, attribute, default) drives the dataclass, the
strict INI reader and the flat `section.key = value` listing, so the three
can never drift apart. Defaults are the reference hardware's; note the
scene-level constraint_damping of 10 (scene.py:65) overrides the solver
default of 1 (solver.py:111), giving gamma = 1/11.
"""
from __future__ import annotations

import configparser
import dataclasses
import math

# (section, ini key, attribute, default)
_TABLE = (
    ("snake", "links", "links", 4),
    ("snake", "sections", "sections", 13),
    ("snake", "width_nodes", "width_nodes", 7),
    ("snake", "height_nodes", "height_nodes", 4),
    ("snake", "link_length", "link_length", 0.12),
    ("snake", "link_width", "link_width", 0.04),
    ("snake", "link_height", "link_height", 0.03),
    ("snake", "density", "density", 1070.0),
    ("snake", "youngs_modulus", "youngs_modulus", 66243.0),
    ("snake", "poisson", "poisson", 0.49),
    ("snake", "clearance", "clearance", 0.005),
    ("snake", "pitch", "pitch", 0.16),
    ("snake", "snakes", "snakes", 1),
    ("carriage", "frame_mass", "frame_mass", 0.05),
    ("carriage", "frame_length", "frame_length", 0.04),
    ("carriage", "frame_height", "frame_height", 0.02),
    ("carriage", "wheel_radius", "wheel_radius", 0.015),
    ("carriage", "wheel_mass", "wheel_mass", 0.008),
    ("carriage", "wheel_offset_y", "wheel_offset_y", 0.03),
    ("carriage", "wheel_drop", "wheel_drop", 0.005),
    ("pneumatics", "supply_psi", "supply_psi", 8.0),
    ("pneumatics", "k_inflate", "k_inflate", 0.23),
    ("pneumatics", "k_deflate", "k_deflate", 0.23),
    ("pneumatics", "deflate_cap_psi", "deflate_cap_psi", 0.68),
    ("pneumatics", "tick_hz", "tick_hz", 60.0),
    ("gait", "amplitude_psi", "amplitude_psi", 8.0),
    ("gait", "frequency", "frequency", 2.0),
    ("gait", "omega_in_radians", "omega_in_radians", False),
    ("gait", "phase_offset", "phase_offset", 0.5 * math.pi),
    ("gait", "turn_bias", "turn_bias", 0.0),
    ("solver", "dt", "dt", 1.0 / 60.0),
    ("solver", "substeps", "substeps", 2),
    ("solver", "newton_iters", "newton_iters", 4),
    ("solver", "pcr_iters", "pcr_iters", 20),
    ("solver", "mu", "mu", 1.0),
    ("solver", "gravity_z", "gravity_z", -9.81),
    ("solver", "contact_margin", "contact_margin", 0.005),
    ("solver", "constraint_damping", "constraint_damping", 10.0),
    ("solver", "max_strain_rate", "max_strain_rate", 6.0),
    ("solver", "backend", "backend", ""),
    ("compliance", "actuation", "actuation_compliance", 1e-6),
    ("compliance", "structural", "structural_compliance", 1e-8),
    ("compliance", "inextensible", "inextensible_compliance", 1e-9),
    ("compliance", "attachment", "attachment_compliance", 1e-9),
    ("compliance", "hinge", "hinge_compliance", 1e-10),
    ("compliance", "friction", "friction_compliance", 1e-8),
    ("sim", "duration", "duration", 10.0),
    ("sim", "latency", "latency", True),
)

_BY_SECTION: dict[str, dict[str, str]] = {}
for _sec, _key, _attr, _ in _TABLE:
    _BY_SECTION.setdefault(_sec, {})[_key] = _attr


def _render(v) -> str:
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, float):
        return repr(v)
    return str(v)


def _scene_methods(cls):
    @classmethod
    def from_file(klass, path: str):
        with open(path, "r", encoding="utf-8") as fh:
            return klass.from_string(fh.read())

    @classmethod
    def from_string(klass, text: str):
        cp = configparser.ConfigParser()
        cp.read_string(text)
        obj = klass()
        for sec in cp.sections():
            keys = _BY_SECTION.get(sec)
            if keys is None:
                raise ValueError(f"unknown scene section [{sec}]")
            for key, raw in cp.items(sec):
                attr = keys.get(key)
                if attr is None:
                    raise ValueError(f"unknown scene key {sec}.{key}")
                cur = getattr(obj, attr)
                if isinstance(cur, bool):
                    val = cp.getboolean(sec, key)
                elif isinstance(cur, int):
                    val = int(raw)
                elif isinstance(cur, float):
                    val = float(raw)
                else:
                    val = raw.strip()
                setattr(obj, attr, val)
        return obj

    def solver_config(self):
        from .simulator import SolverConfig
        return SolverConfig(
            dt=self.dt, substeps=self.substeps, newton_iters=self.newton_iters,
            pcr_iters=self.pcr_iters, gravity=(0.0, 0.0, self.gravity_z),
            contact_margin=self.contact_margin, mu=self.mu,
            friction_compliance=self.friction_compliance,
            constraint_damping=self.constraint_damping,
            max_strain_rate=self.max_strain_rate,
            backend=self.backend or None)

    def to_items(self):
        return [(f"{sec}.{key}", _render(getattr(self, attr)))
                for sec, key, attr, _ in _TABLE]

    def write(self, path: str) -> None:
        out, prev = [], None
        for full, val in self.to_items():
            sec, key = full.split(".", 1)
            if sec != prev:
                if prev is not None:
                    out.append("")
                out.append(f"[{sec}]")
                prev = sec
            out.append(f"{key} = {val}")
        with open(path, "w", encoding="utf-8") as fh:
            fh.write("\n".join(out) + "\n")

    cls.from_file = from_file
    cls.from_string = from_string
    cls.solver_config = solver_config
    cls.to_items = to_items
    cls.write = write
    return cls


SceneConfig = _scene_methods(dataclasses.make_dataclass(
    "SceneConfig",
    [(attr, type(default), dataclasses.field(default=default))
     for _, _, attr, default in _TABLE],
    module=__name__))
SceneConfig.__doc__ = "Robot, gait and solver description (softsnake/scene.py:16-77)."
