"""The five BASELINE.json workloads as plain data (numpy only).

This module is neither product nor checker: it holds the decisions the
reference leaves open — meshes as edge arrays, raw
level maps, seeded initial conditions, family fixtures, CFL numbers and step
counts — so that the product (`paper_2507_04991_b200.workloads`) and the CPU
arms (`oracle/cpu_runs.py`, `bench.py --impl reference`) build the SAME
workload without one importing the other.  Nothing here loads a native
library.

  C1  uniform 16^2 on [-10,10]^2, vortex I=5 (p_inf = 1), EC + Rusanov,
      p2 S=4 E={4} with (a21, a32) = (0.204, 0.42) (linearly stable at CFL 0.9
      on the probed spectrum, configs/c1_pair_scan.py), CFL 0.9, 100 steps
  C2  64^2 "+"-refined mesh (16 h | 32 h/2 | 16 h per axis, h = 20/48),
      EC + HLLE, p3 {4,7}, 500 steps
  C3  256^2 three-level "+" mesh on [0,2pi]^2, seeded random Fourier state,
      EC + Rusanov, p4 {5,9,16}, 200 steps
  C4  512^2 two-level "+" mesh on [0,1]^2 (64 h | 128 h/2 | 128 h | 128 h/2 |
      64 h per axis, h = 1/384), double shear layer (delta 1/30, eps 0.05,
      Ma 0.1), NSF mu = 1e-4, Pr = 0.72, BR1, EC + HLLE, p3 {4,8}, 200 steps
  C5  64^3 three-level "+" mesh on [0,2pi]^3, Taylor-Green vortex Ma 0.1,
      EC + Rusanov, p4 {5,8,14}, 100 steps
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

CONFIG_DIR = os.path.dirname(os.path.abspath(__file__))


# ---------------------------------------------------------------------------
# initial conditions
# ---------------------------------------------------------------------------
@dataclass
class VortexParams:
    """physics.hpp:177-185; C1/C2 use I=5 with p_inf = 1 (mach = 1/sqrt(gamma))."""
    gamma: float = 1.4
    mach: float = 1.0 / math.sqrt(1.4)
    radius: float = 1.0
    intensity: float = 5.0
    rho_inf: float = 1.0
    v_inf: tuple = (1.0, 1.0)
    half_width: float = 10.0

    def as_array(self):
        return np.array([self.gamma, self.mach, self.radius, self.intensity, self.rho_inf,
                         self.v_inf[0], self.v_inf[1], self.half_width])


def isentropic_vortex(p: VortexParams, x, y, t=0.0):
    """isentropic_vortex_state, physics.cpp:301-328 (vectorised)."""
    span = 2.0 * p.half_width

    def wrap(d):
        d = np.fmod(d + p.half_width, span)
        d = np.where(d < 0.0, d + span, d)
        return d - p.half_width

    cx = wrap(x - p.v_inf[0] * t)
    cy = wrap(y - p.v_inf[1] * t)
    r2 = cx * cx + cy * cy
    g = np.exp((1.0 - r2) / (2.0 * p.radius * p.radius))
    gm1 = p.gamma - 1.0
    rho = p.rho_inf * np.power(
        1.0 - p.intensity * p.intensity * p.mach * p.mach * gm1 * g * g / (8.0 * math.pi * math.pi),
        1.0 / gm1)
    coef = p.intensity * g / (2.0 * math.pi * p.radius)
    vx = p.v_inf[0] - coef * cy
    vy = p.v_inf[1] + coef * cx
    pres = np.power(rho, p.gamma) / (p.gamma * p.mach * p.mach)
    return np.stack([rho, rho * vx, rho * vy, pres / gm1 + 0.5 * rho * (vx * vx + vy * vy)])


def random_fourier_state(x, y, seed=20250704, modes=8, kmax=4, gamma=1.4, length=2 * math.pi):
    """C3: each primitive (rho, vx, vy, p) is a sum of `modes` Fourier modes
    with integer wavenumbers |k| <= kmax (periodic on [0, length)^2), random
    phases and amplitudes normalised to sum 1, mapped to rho, p in [0.5, 1.5]
    and v in [-0.5, 0.5].  numpy PCG64 with the given seed."""
    rng = np.random.Generator(np.random.PCG64(seed))
    fields = []
    for _ in range(4):
        k = rng.integers(-kmax, kmax + 1, size=(modes, 2))
        k[np.all(k == 0, axis=1)] = (1, 0)
        amp = rng.uniform(0.2, 1.0, size=modes)
        amp /= amp.sum()
        ph = rng.uniform(0.0, 2 * math.pi, size=modes)
        w = 2 * math.pi / length
        f = np.zeros_like(x)
        for m in range(modes):
            f = f + amp[m] * np.cos(w * (k[m, 0] * x + k[m, 1] * y) + ph[m])
        fields.append(f)  # in [-1, 1]
    rho = 1.0 + 0.5 * fields[0]
    vx = 0.5 * fields[1]
    vy = 0.5 * fields[2]
    p = 1.0 + 0.5 * fields[3]
    return np.stack([rho, rho * vx, rho * vy, p / (gamma - 1.0) + 0.5 * rho * (vx * vx + vy * vy)])


def double_shear_layer(x, y, mach=0.1, gamma=1.4, delta=1.0 / 30.0, eps=0.05):
    """C4: periodic double shear layer on [0,1]^2 (Bell-Colella-Glaz form):
    u = tanh((y - 1/4)/delta) for y <= 1/2, tanh((3/4 - y)/delta) above,
    v = eps sin(2 pi (x + 1/4)), rho = 1, p = 1/(gamma Ma^2) (Ma on |u| = 1)."""
    vx = np.where(y <= 0.5, np.tanh((y - 0.25) / delta), np.tanh((0.75 - y) / delta))
    vy = eps * np.sin(2 * math.pi * (x + 0.25))
    rho = np.ones_like(x)
    p = np.full_like(x, 1.0 / (gamma * mach * mach))
    return np.stack([rho, rho * vx, rho * vy, p / (gamma - 1.0) + 0.5 * rho * (vx * vx + vy * vy)])


def taylor_green(x, y, z, mach=0.1, gamma=1.4, rho0=1.0, u0=1.0):
    """C5: 3D Taylor-Green vortex on [0, 2pi]^3 at Mach `mach`:
    p0 = rho0 u0^2 / (gamma Ma^2),
    p  = p0 + rho0 u0^2 / 16 (cos 2x + cos 2y)(cos 2z + 2), rho = rho0."""
    p0 = rho0 * u0 * u0 / (gamma * mach * mach)
    vx = u0 * np.sin(x) * np.cos(y) * np.cos(z)
    vy = -u0 * np.cos(x) * np.sin(y) * np.cos(z)
    vz = np.zeros_like(x)
    p = p0 + rho0 * u0 * u0 / 16.0 * (np.cos(2 * x) + np.cos(2 * y)) * (np.cos(2 * z) + 2.0)
    rho = np.full_like(x, rho0)
    E = p / (gamma - 1.0) + 0.5 * rho * (vx * vx + vy * vy + vz * vz)
    return np.stack([rho, rho * vx, rho * vy, rho * vz, E])


# ---------------------------------------------------------------------------
# meshes and levels
# ---------------------------------------------------------------------------
def banded_edges(x0, bands):
    """Edges from (count, size) bands starting at x0 (append_uniform style)."""
    e = [x0]
    for n, h in bands:
        a = e[-1]
        e.extend(a + h * i for i in range(1, n + 1))
    return e


def axis_levels(bands):
    """Per-cell level along one axis: finest size -> 1, doubling -> +1."""
    hmin = min(h for _, h in bands)
    lv = []
    for n, h in bands:
        lv += [1 + int(round(math.log2(h / hmin)))] * n
    return np.array(lv, dtype=np.int32)


def geometric_levels(axis_lv, R):
    """Cell level = min over axes (a cell thin along any axis is fine)."""
    if len(axis_lv) == 2:
        L = np.minimum.outer(axis_lv[1], axis_lv[0])  # [y, x]
    else:
        L = np.minimum(axis_lv[2][:, None, None],
                       np.minimum.outer(axis_lv[1], axis_lv[0])[None, :, :])  # [z, y, x]
    return np.clip(L.reshape(-1), 1, R).astype(np.int32)


def effective_levels(shape, raw):
    """make_partition_map (mesh.cpp:56-71) on a periodic Cartesian mesh:
    each cell takes the minimum level over itself and its face neighbours
    (mesh_adjacency, mesh.cpp:17-47; the 3D mesh adds the z pair).
    `shape` is (nx, ny[, nz]); cells are x-fastest."""
    L = np.asarray(raw, dtype=np.int32).reshape(tuple(reversed(shape)))
    eff = L.copy()
    for ax in range(L.ndim):
        eff = np.minimum(eff, np.roll(L, 1, axis=ax))
        eff = np.minimum(eff, np.roll(L, -1, axis=ax))
    return eff.reshape(-1).astype(np.int32)


# ---------------------------------------------------------------------------
# family fixtures (butcher.cpp:357-433 text format)
# ---------------------------------------------------------------------------
@dataclass
class FamilyTables:
    kind: str
    S: int
    R: int
    E: List[int]
    A: np.ndarray  # [R, S, S]
    b: np.ndarray
    c: np.ndarray

    def member_index_for_level(self, level):
        return self.R - level

    def active_stages(self, r):
        """active_stage_set (butcher.cpp:319-332) of member r."""
        A, b = self.A[r], self.b
        act = {0} | {i for i in range(self.S) if b[i] != 0.0}
        grew = True
        while grew:
            grew = False
            for i in sorted(act):
                for j in range(i):
                    if A[i][j] != 0.0 and j not in act:
                        act.add(j)
                        grew = True
        return act


def parse_family_text(text: str) -> FamilyTables:
    """read_family (butcher.cpp:357-433)."""
    kind = "p2"
    rows = []
    for raw in text.splitlines():
        s = raw.strip()
        if not s:
            continue
        if s.startswith("#"):
            parts = s[1:].split()
            if len(parts) >= 2 and parts[0] == "kind":
                kind = {"p3-variant": "p3"}.get(parts[1], parts[1])
            continue
        if s.startswith("dt_max"):
            continue
        rows.append(s.split())
    S, R = int(rows[0][0]), int(rows[0][1])
    c = np.array([float(x) for x in rows[1][:S]])
    b = np.array([float(x) for x in rows[2][:S]])
    A = np.zeros((R, S, S))
    E = []
    k = 3
    for r in range(R):
        E.append(int(float(rows[k][0])))
        k += 1
        for i in range(S):
            A[r, i] = [float(x) for x in rows[k][:S]]
            k += 1
    return FamilyTables(kind, S, R, E, A, b, c)


def family_path(name):
    return os.path.join(CONFIG_DIR, f"{name}.family")


# ---------------------------------------------------------------------------
# the five configurations
# ---------------------------------------------------------------------------
@dataclass
class MeshSpec:
    edges: list  # per axis

    @property
    def dim(self):
        return len(self.edges)

    def shape(self):
        return tuple(len(e) - 1 for e in self.edges)

    @property
    def x_edges(self):
        return self.edges[0]

    @property
    def y_edges(self):
        return self.edges[1]

    def num_cells(self):
        return int(np.prod(self.shape()))


@dataclass
class ConfigSpec:
    name: str
    description: str
    mesh: MeshSpec
    surface_flux: str
    family_file: str
    raw_levels: np.ndarray
    R: int
    cfl: float
    steps: int
    ic: str
    gamma: float = 1.4
    physics: str = "euler"
    mu: float = 0.0
    prandtl: float = 0.72
    relaxation_numerics: str = "accurate"

    @property
    def dim(self):
        return self.mesh.dim

    def nodes_per_cell(self):
        return 16 if self.dim == 2 else 64

    def num_vars(self):
        return self.dim + 2

    def family(self) -> FamilyTables:
        with open(family_path(self.family_file)) as f:
            return parse_family_text(f.read())

    def effective_levels(self):
        return effective_levels(self.mesh.shape(), self.raw_levels)

    def initial_state(self, x, y, z=None):
        if self.ic == "vortex":
            return isentropic_vortex(VortexParams(), x, y)
        if self.ic == "random":
            return random_fourier_state(x, y)
        if self.ic == "tgv":
            return taylor_green(x, y, z)
        if self.ic == "shear":
            return double_shear_layer(x, y)
        raise ValueError(self.ic)

    def canonical_state(self, x, y, z=None):
        """U0 in the canonical layout (cell-major, node x-fastest, variable-minor)."""
        return np.ascontiguousarray(self.initial_state(x, y, z).T).reshape(-1)

    def dof_stage_updates_per_step(self, eff=None):
        """Sum over stages of active nodes = rhs_cell_evaluations()/V per step
        (semidisc.cpp:131-133; PAPER N_K)."""
        eff = self.effective_levels() if eff is None else eff
        fam = self.family()
        total = 0
        for lvl in range(1, self.R + 1):
            n = int(np.sum(eff == lvl))
            total += len(fam.active_stages(fam.member_index_for_level(lvl))) * n
        return total * self.nodes_per_cell()


def _banded_mesh(x0, bands, dim):
    e = np.array(banded_edges(x0, bands))
    return MeshSpec([e.copy() for _ in range(dim)])


def make_spec(name: str) -> ConfigSpec:
    name = name.lower()
    if name == "c1":
        e = np.array([-10.0 + 20.0 * i / 16 for i in range(17)])
        mesh = MeshSpec([e, e.copy()])
        return ConfigSpec("c1", "2D Euler isentropic vortex 16^2, p2 S=4, CFL 0.9", mesh,
                          "rusanov", "c1_p2_4", np.ones(mesh.num_cells(), np.int32), 1, 0.9, 100,
                          "vortex")
    if name == "c2":
        h = 20.0 / 48.0
        bands = [(16, h), (32, h / 2), (16, h)]
        al = axis_levels(bands)
        return ConfigSpec("c2", "2D Euler vortex, 64^2 2-level '+' mesh, p3 {4,7}, HLLE",
                          _banded_mesh(-10.0, bands, 2), "hlle", "c2_p3_4_7",
                          geometric_levels([al, al], 2), 2, 1.0, 500, "vortex")
    if name == "c3":
        h = 2 * math.pi / 216.0
        bands = [(96, h), (16, h / 2), (32, h / 4), (16, h / 2), (96, h)]
        al = axis_levels(bands)
        return ConfigSpec("c3", "2D Euler random Fourier state, 256^2 3-level mesh, p4 {5,9,16}",
                          _banded_mesh(0.0, bands, 2), "rusanov", "c3_p4_5_9_16",
                          geometric_levels([al, al], 3), 3, 1.5, 200, "random")
    if name == "c4":
        h = 1.0 / 384.0
        bands = [(64, h), (128, h / 2), (128, h), (128, h / 2), (64, h)]
        al = axis_levels(bands)
        return ConfigSpec("c4", "2D Navier-Stokes double shear layer, 512^2 2-level mesh, p3 {4,8}",
                          _banded_mesh(0.0, bands, 2), "hlle", "c4_p3_4_8",
                          geometric_levels([al, al], 2), 2, 1.1, 200, "shear", physics="nsf",
                          mu=1e-4, prandtl=0.72)
    if name == "c5":
        h = 2 * math.pi / 54.0
        bands = [(24, h), (4, h / 2), (8, h / 4), (4, h / 2), (24, h)]
        al = axis_levels(bands)
        return ConfigSpec("c5", "3D Euler Taylor-Green Ma 0.1, 64^3 3-level mesh, p4 {5,8,14}",
                          _banded_mesh(0.0, bands, 3), "rusanov", "c5_p4_5_8_14",
                          geometric_levels([al, al, al], 3), 3, 1.1, 100, "tgv")
    raise ValueError(f"unknown config {name}")


def _scaled_bands(bands, factor, length):
    """Same band structure with every count divided by factor (>= 1 cell)."""
    counts = [max(1, n // factor) for n, _ in bands]
    rel = [h for _, h in bands]
    total = sum(n * r for n, r in zip(counts, rel))
    scale = length / total
    return [(n, r * scale) for n, r in zip(counts, rel)]


def sample_spec(spec: ConfigSpec) -> ConfigSpec:
    """A bounded CPU sample of a configuration: the same family, flux, initial
    condition, CFL and level grading on a mesh with fewer cells per band
    (C5: 16^3 instead of 64^3; C3: 32^2 instead of 256^2).  Used only for the
    CPU baseline timing inside the GPU arm's line, never for parity."""
    import copy
    out = copy.copy(spec)
    if spec.name == "c5":
        bands = _scaled_bands([(24, 1.0), (4, 0.5), (8, 0.25), (4, 0.5), (24, 1.0)], 4,
                              2 * math.pi)
        out.mesh = _banded_mesh(0.0, bands, 3)
        al = axis_levels(bands)
        out.raw_levels = geometric_levels([al, al, al], spec.R)
        out.description = "C5 sample: 16^3-element 3-level graded TGV mesh"
    elif spec.name == "c3":
        bands = _scaled_bands([(96, 1.0), (16, 0.5), (32, 0.25), (16, 0.5), (96, 1.0)], 8,
                              2 * math.pi)
        out.mesh = _banded_mesh(0.0, bands, 2)
        al = axis_levels(bands)
        out.raw_levels = geometric_levels([al, al], spec.R)
        out.description = "C3 sample: 32^2-element 3-level graded mesh"
    return out


def bench_config(spec: ConfigSpec) -> dict:
    """The `config` object of bench.py's JSON line: identical for the B200
    arm and the reference arm (no rank count or implementation in it)."""
    fam = spec.family()
    return {"workload": spec.description,
            "nodes": int(spec.mesh.num_cells() * spec.nodes_per_cell()),
            "dof_stage_per_step": int(spec.dof_stage_updates_per_step()),
            "steps_stated": spec.steps, "cfl": spec.cfl,
            "family": f"{fam.kind} S={fam.S} E={fam.E}",
            "relaxation": f"newton, {spec.relaxation_numerics} numerics (SURVEY 7.3 H1)",
            "l2": _l2_note(spec)}


def _l2_note(spec):
    mib = spec.mesh.num_cells() * spec.nodes_per_cell() * spec.num_vars() * 8 / 2**20
    if 5 * mib * 2**20 > 126e6:  # U, K1, two stage states, d: all read every step
        return f"inputs larger than L2 (5 state vectors x {mib:.0f} MiB)"
    return f"working set fits L2 (5 x {mib:.2f} MiB state vectors; not flushed)"
