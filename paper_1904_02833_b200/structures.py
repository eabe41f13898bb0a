"""Host-side scene containers (construction only; no step math here).

These mirror the reference's constructor-facing types so a scene built
for the reference can be built the same way here:
  ParticleSet / RigidBody / SystemState        softsnake/state.py:59-168
  Distance/Tetra/Attachment/Hinge sets         softsnake/constraints.py:43-356
  WheelCollider                                softsnake/contact.py:35-41
  StrainLaw / PneumaticChannel / ChannelBank   softsnake/pneumatics.py:32-116
The Simulator accepts these or the reference's own objects (duck typing on
the array attributes). Array dtypes and shapes follow the reference
(float64 / int32, C-contiguous).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

PSI_TO_PA = 6894.76
KIND_STRUCTURAL, KIND_ACTUATION, KIND_INEXTENSIBLE = 0, 1, 2


# ----------------------------------------------------------------- rigid math
def quat_normalize(q) -> np.ndarray:
    q = np.asarray(q, np.float64)
    n = float(np.linalg.norm(q))
    return np.array([1.0, 0.0, 0.0, 0.0]) if n < 1e-12 else q / n


def quat_mul(a, b) -> np.ndarray:
    aw, ax, ay, az = a
    bw, bx, by, bz = b
    return np.array([aw * bw - ax * bx - ay * by - az * bz,
                     aw * bx + ax * bw + ay * bz - az * by,
                     aw * by - ax * bz + ay * bw + az * bx,
                     aw * bz + ax * by - ay * bx + az * bw])


def quat_from_axis_angle(axis, angle) -> np.ndarray:
    axis = np.asarray(axis, np.float64)
    n = float(np.linalg.norm(axis))
    if n < 1e-12:
        return np.array([1.0, 0.0, 0.0, 0.0])
    return np.concatenate([[np.cos(0.5 * angle)], np.sin(0.5 * angle) * axis / n])


def rotation_matrix(q) -> np.ndarray:
    w, x, y, z = quat_normalize(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


# ------------------------------------------------------------------- state
@dataclass
class ParticleSet:
    positions: np.ndarray
    velocities: np.ndarray
    inv_mass: np.ndarray

    @classmethod
    def create(cls, positions, masses) -> "ParticleSet":
        x = np.array(positions, np.float64).reshape(-1, 3)
        m = np.asarray(masses, np.float64)
        safe = np.where(m > 0, m, 1.0)
        return cls(x, np.zeros_like(x), np.where(m > 0, 1.0 / safe, 0.0))

    @property
    def count(self) -> int:
        return int(self.positions.shape[0])


@dataclass
class RigidBody:
    position: np.ndarray
    orientation: np.ndarray
    linear_velocity: np.ndarray
    angular_velocity: np.ndarray
    mass: float
    inertia: np.ndarray

    @classmethod
    def create(cls, position, mass, inertia, orientation=(1, 0, 0, 0)) -> "RigidBody":
        return cls(np.array(position, np.float64),
                   quat_normalize(np.array(orientation, np.float64)),
                   np.zeros(3), np.zeros(3), float(mass),
                   np.array(inertia, np.float64).reshape(3, 3))


@dataclass
class SystemState:
    particles: ParticleSet
    body_pos: np.ndarray
    body_quat: np.ndarray
    body_lin_vel: np.ndarray
    body_ang_vel: np.ndarray
    body_mass: np.ndarray
    body_inertia: np.ndarray
    time: float = 0.0

    @classmethod
    def create(cls, particles: ParticleSet, bodies: list) -> "SystemState":
        nb = len(bodies)
        st = cls(particles, np.zeros((nb, 3)), np.zeros((nb, 4)), np.zeros((nb, 3)),
                 np.zeros((nb, 3)), np.zeros(nb), np.zeros((nb, 3, 3)))
        for i, b in enumerate(bodies):
            st.body_pos[i] = b.position
            st.body_quat[i] = quat_normalize(b.orientation)
            st.body_lin_vel[i] = b.linear_velocity
            st.body_ang_vel[i] = b.angular_velocity
            st.body_mass[i] = b.mass
            st.body_inertia[i] = b.inertia
        return st

    @property
    def num_particles(self) -> int:
        return self.particles.count

    @property
    def num_bodies(self) -> int:
        return int(self.body_pos.shape[0])

    @property
    def num_dof(self) -> int:
        return 3 * self.num_particles + 6 * self.num_bodies

    def get_velocities(self) -> np.ndarray:
        tail = np.concatenate([self.body_lin_vel, self.body_ang_vel], axis=1).ravel()
        return np.concatenate([self.particles.velocities.ravel(), tail])

    def set_velocities(self, u: np.ndarray) -> None:
        n3 = 3 * self.num_particles
        self.particles.velocities[:] = u[:n3].reshape(-1, 3)
        tail = u[n3:].reshape(-1, 6)
        self.body_lin_vel[:] = tail[:, :3]
        self.body_ang_vel[:] = tail[:, 3:]

    def copy(self) -> "SystemState":
        p = ParticleSet(self.particles.positions.copy(), self.particles.velocities.copy(),
                        self.particles.inv_mass.copy())
        return SystemState(p, self.body_pos.copy(), self.body_quat.copy(),
                           self.body_lin_vel.copy(), self.body_ang_vel.copy(),
                           self.body_mass.copy(), self.body_inertia.copy(), self.time)


def kinetic_energy(state) -> float:
    """state.py:271-282 (host readback helper)."""
    p = state.particles
    live = p.inv_mass > 0
    v = p.velocities[live]
    ke = 0.5 * float(np.sum((1.0 / p.inv_mass[live]) * np.einsum("ij,ij->i", v, v)))
    for b in range(state.body_pos.shape[0]):
        R = rotation_matrix(state.body_quat[b])
        iw = R @ state.body_inertia[b] @ R.T
        lv, av = state.body_lin_vel[b], state.body_ang_vel[b]
        ke += 0.5 * state.body_mass[b] * float(lv @ lv) + 0.5 * float(av @ iw @ av)
    return ke


def center_of_mass(state) -> np.ndarray:
    """state.py:285-292 (host readback helper)."""
    p = state.particles
    live = p.inv_mass > 0
    m = 1.0 / p.inv_mass[live]
    tot = float(np.sum(m)) + float(np.sum(state.body_mass))
    com = (m[:, None] * p.positions[live]).sum(axis=0)
    com += (state.body_mass[:, None] * state.body_pos).sum(axis=0)
    return com / tot


# ------------------------------------------------------------- constraints
def tetra_compliance(rest_volume: float, youngs_modulus: float, poisson: float) -> np.ndarray:
    """Voigt [xx yy zz yz xz xy] isotropic block (constraints.py:26-40)."""
    c = 1.0 / (rest_volume * youngs_modulus)
    nu = poisson
    E = np.zeros((6, 6))
    E[:3, :3] = c * np.array([[1.0, -nu, -nu], [-nu, 1.0, -nu], [-nu, -nu, 1.0]])
    E[3, 3] = E[4, 4] = E[5, 5] = c * (1.0 + nu)
    return E


@dataclass
class DistanceConstraint:
    i: int
    j: int
    rest_length: float
    compliance: float
    kind: int = KIND_STRUCTURAL
    channel: int = -1


@dataclass
class DistanceSet:
    pairs: np.ndarray
    rest: np.ndarray
    compliance: np.ndarray
    kind: np.ndarray
    channel: np.ndarray
    scale: np.ndarray
    dirs: np.ndarray

    @classmethod
    def from_constraints(cls, cs) -> "DistanceSet":
        n = len(cs)
        dirs = np.zeros((n, 3))
        dirs[:, 0] = 1.0
        return cls(np.array([(c.i, c.j) for c in cs], np.int32).reshape(n, 2),
                   np.array([c.rest_length for c in cs], np.float64),
                   np.array([c.compliance for c in cs], np.float64),
                   np.array([c.kind for c in cs], np.int32),
                   np.array([c.channel for c in cs], np.int32),
                   np.ones(n), dirs)

    @property
    def count(self) -> int:
        return int(self.pairs.shape[0])


@dataclass
class TetraElement:
    particles: np.ndarray
    rest_inv: np.ndarray
    rest_volume: float
    compliance: np.ndarray

    @classmethod
    def from_positions(cls, ids, rest_positions, youngs_modulus, poisson) -> "TetraElement":
        x = np.asarray(rest_positions, np.float64)
        D = np.stack([x[1] - x[0], x[2] - x[0], x[3] - x[0]], axis=1)
        det = float(np.linalg.det(D))
        if abs(det) < 1e-18:
            raise ValueError("degenerate rest tetrahedron")
        vol = abs(det) / 6.0
        return cls(np.asarray(ids, np.int64), np.linalg.inv(D), vol,
                   tetra_compliance(vol, youngs_modulus, poisson))


@dataclass
class TetraSet:
    tets: np.ndarray
    rest_inv: np.ndarray
    rest_volume: np.ndarray
    compliance: np.ndarray
    quats: np.ndarray
    inverted_count: int = 0

    @classmethod
    def from_elements(cls, els) -> "TetraSet":
        n = len(els)
        q = np.zeros((n, 4))
        q[:, 0] = 1.0
        return cls(np.array([e.particles for e in els], np.int32).reshape(n, 4),
                   np.array([e.rest_inv for e in els]).reshape(n, 3, 3),
                   np.array([e.rest_volume for e in els], np.float64),
                   np.array([e.compliance for e in els]).reshape(n, 6, 6), q)

    @property
    def count(self) -> int:
        return int(self.tets.shape[0])


@dataclass
class AttachmentConstraint:
    particle: int
    body: int
    local_anchor: np.ndarray
    compliance: float


@dataclass
class AttachmentSet:
    particle: np.ndarray
    body: np.ndarray
    local_anchor: np.ndarray
    compliance: np.ndarray

    @classmethod
    def from_constraints(cls, cs) -> "AttachmentSet":
        n = len(cs)
        return cls(np.array([c.particle for c in cs], np.int32).reshape(n),
                   np.array([c.body for c in cs], np.int32).reshape(n),
                   np.array([c.local_anchor for c in cs], np.float64).reshape(n, 3),
                   np.array([c.compliance for c in cs], np.float64).reshape(n))

    @property
    def count(self) -> int:
        return int(self.particle.shape[0])


@dataclass
class HingeJoint:
    body_a: int
    body_b: int
    anchor_a: np.ndarray
    anchor_b: np.ndarray
    axis_a: np.ndarray
    axis_b: np.ndarray
    compliance: float


def _perp_unit(v: np.ndarray) -> np.ndarray:
    """constraints.py:276-279"""
    ref = np.array([0.0, 0.0, 1.0]) if abs(v[2]) <= 0.9 else np.array([1.0, 0.0, 0.0])
    t = ref - (ref @ v) * v
    return t / np.linalg.norm(t)


@dataclass
class HingeSet:
    body_a: np.ndarray
    body_b: np.ndarray
    anchor_a: np.ndarray
    anchor_b: np.ndarray
    axis_a: np.ndarray
    axis_b: np.ndarray
    tan1_b: np.ndarray
    tan2_b: np.ndarray
    compliance: np.ndarray

    @classmethod
    def from_joints(cls, js) -> "HingeSet":
        n = len(js)
        unit = lambda v: np.asarray(v, np.float64) / np.linalg.norm(v)  # noqa: E731
        axb = np.array([unit(j.axis_b) for j in js]).reshape(n, 3)
        t1 = np.array([_perp_unit(a) for a in axb]).reshape(n, 3)
        return cls(np.array([j.body_a for j in js], np.int32).reshape(n),
                   np.array([j.body_b for j in js], np.int32).reshape(n),
                   np.array([j.anchor_a for j in js], np.float64).reshape(n, 3),
                   np.array([j.anchor_b for j in js], np.float64).reshape(n, 3),
                   np.array([unit(j.axis_a) for j in js]).reshape(n, 3),
                   axb, t1, np.cross(axb, t1),
                   np.array([j.compliance for j in js], np.float64).reshape(n))

    @property
    def count(self) -> int:
        return int(self.body_a.shape[0])


@dataclass
class WheelCollider:
    body: int
    radius: float
    axis_local: np.ndarray


# -------------------------------------------------------------- pneumatics
def update_pressure(p: float, target: float, k_i: float = 0.23, k_d: float = 0.23,
                    cap: float = 0.68, p_s: float = 8.0) -> float:
    """One 60 Hz valve tick in psi (pneumatics.py:62-72); host mirror of the
    device kernel for API completeness."""
    if target > p:
        g = (target - p) / p_s
        return min(p + p_s * g * g * k_i, target)
    if target < p:
        return max(0.0, p - min(p * k_d, cap))
    return p


def route_antagonistic(command: float) -> tuple[float, float]:
    """Signed link command -> (left, right) targets (pneumatics.py:75-85)."""
    if command > 0.0:
        return 0.0, command
    if command < 0.0:
        return -command, 0.0
    return 0.0, 0.0


@dataclass
class StrainLaw:
    youngs_modulus_pa: float

    def strain_pa(self, p_pa):
        return 1.0 + p_pa / self.youngs_modulus_pa

    def strain(self, p_psi):
        return self.strain_pa(p_psi * PSI_TO_PA)


@dataclass
class PneumaticChannel:
    pressure: float = 0.0
    k_inflate: float = 0.23
    k_deflate: float = 0.23
    deflate_cap: float = 0.68
    supply: float = 8.0

    def tick(self, target: float) -> float:
        self.pressure = update_pressure(self.pressure, target, self.k_inflate,
                                        self.k_deflate, self.deflate_cap, self.supply)
        return self.pressure


@dataclass
class ChannelBank:
    """Chamber pressures, index 2i = left, 2i+1 = right (pneumatics.py:88-116).
    On a Simulator the authoritative copy lives on the device; `pressures`
    is refreshed on readback."""
    pressures: np.ndarray
    k_inflate: float = 0.23
    k_deflate: float = 0.23
    deflate_cap: float = 0.68
    supply: float = 8.0

    @classmethod
    def create(cls, n_links: int, **kw) -> "ChannelBank":
        return cls(np.zeros(2 * n_links), **kw)

    def tick(self, commands, latency: bool = True) -> np.ndarray:
        for i, a in enumerate(np.asarray(commands, np.float64)):
            left, right = route_antagonistic(float(a))
            if latency:
                args = (self.k_inflate, self.k_deflate, self.deflate_cap, self.supply)
                self.pressures[2 * i] = update_pressure(self.pressures[2 * i], left, *args)
                self.pressures[2 * i + 1] = update_pressure(self.pressures[2 * i + 1], right, *args)
            else:
                self.pressures[2 * i], self.pressures[2 * i + 1] = left, right
        return self.pressures
