"""Synthetic workloads of BASELINE.json's five configurations (host side).

No dataset is involved: every input is generated here from seeded, documented
formulas (initial conditions, meshes, level maps) or loaded from the frozen
family fixtures under configs/.  Decisions the reference leaves open (SURVEY.md
Appendix A) are fixed here and recorded in DESIGN.md:

  C1  uniform 16^2 on [-10,10]^2, vortex I=5 (p_inf = 1), EC + Rusanov,
      p2 S=4 E={4} with (a21, a32) = (0.2, 0.35), CFL 0.9, 100 steps
  C2  64^2 "+"-refined mesh (16 h | 32 h/2 | 16 h per axis, h = 20/48),
      EC + HLLE, p3 {4,7}, 500 steps
  C3  256^2 three-level "+" mesh on [0,2pi]^2, seeded random Fourier state,
      EC + Rusanov, p4 {5,9,16}, 200 steps
  C4  512^2 two-level "+" mesh on [0,1]^2 (64 h | 128 h/2 | 128 h | 128 h/2 |
      64 h per axis, h = 1/384), double shear layer (delta 1/30, eps 0.05,
      Ma 0.1), NSF mu = 1e-4, Pr = 0.72, BR1, EC + HLLE, p3 {4,8}, 200 steps
  C5  64^3 three-level "+" mesh on [0,2pi]^3, Taylor-Green vortex Ma 0.1,
      EC + Rusanov, p4 {5,8,14}, 100 steps
Free coefficients of the C2-C5 families come from configs/make_families.py
(model-spectrum stability optimisation; member CFL limits in DESIGN.md); the
CFL numbers are ~75 % of each family's model limit (C2 1.37, C3 2.03,
C5 1.45).
Levels are assigned geometrically (finest cell size along any axis -> level
1), then widened by make_partition_map's neighbour rule (mesh.cpp:56-71).
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import perrk as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONFIG_DIR = os.path.join(ROOT, "configs")


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


# ---------------------------------------------------------------------------
# configurations
# ---------------------------------------------------------------------------
@dataclass
class Config:
    name: str
    description: str
    mesh: object
    surface_flux: str
    family: P.PartitionFamily
    raw_levels: np.ndarray
    cfl: float
    steps: int
    ic: str
    gamma: float = 1.4
    relaxation: Optional[P.RelaxationConfig] = field(
        default_factory=lambda: P.RelaxationConfig(numerics="accurate"))
    physics: str = "euler"
    mu: float = 0.0
    prandtl: float = 0.72

    @property
    def dim(self):
        return self.mesh.dim

    def spec(self, device=0):
        return P.SemidiscretizationSpec(self.mesh, 3, self.gamma, self.physics, self.mu,
                                        self.prandtl, self.surface_flux, "flux_differencing", "ec",
                                        device)

    def partition_map(self):
        return P.make_partition_map(self.mesh, self.raw_levels, self.family.R)

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

    def nodes_per_cell(self):
        return 16 if self.dim == 2 else 64


def family_path(name):
    return os.path.join(CONFIG_DIR, f"{name}.family")


def load_config_family(name):
    return P.load_family(family_path(name))


def c1_family():
    return P.build_perk2(4, [4], [[0.2, 0.35]])


def make_config(name: str, family=None, cfl=None, steps=None) -> Config:
    name = name.lower()
    if name == "c1":
        mesh = P.build_uniform_mesh2d(10.0, 16)
        fam = family or c1_family()
        return Config("c1", "2D Euler isentropic vortex 16^2, p2 S=4, CFL 0.9", mesh, "rusanov",
                      fam, np.ones(mesh.num_cells(), np.int32), cfl or 0.9, steps or 100,
                      "vortex")
    if name == "c2":
        h = 20.0 / 48.0
        bands = [(16, h), (32, h / 2), (16, h)]
        e = banded_edges(-10.0, bands)
        mesh = P.Mesh2DRect(e, list(e))
        al = axis_levels(bands)
        fam = family or load_config_family("c2_p3_4_7")
        return Config("c2", "2D Euler vortex, 64^2 2-level '+' mesh, p3 {4,7}, HLLE", mesh,
                      "hlle", fam, geometric_levels([al, al], fam.R), cfl or 1.0, steps or 500,
                      "vortex")
    if name == "c3":
        h = 2 * math.pi / 216.0
        bands = [(96, h), (16, h / 2), (32, h / 4), (16, h / 2), (96, h)]
        e = banded_edges(0.0, bands)
        mesh = P.Mesh2DRect(e, list(e))
        al = axis_levels(bands)
        fam = family or load_config_family("c3_p4_5_9_16")
        return Config("c3", "2D Euler random Fourier state, 256^2 3-level mesh, p4 {5,9,16}",
                      mesh, "rusanov", fam, geometric_levels([al, al], fam.R), cfl or 1.5,
                      steps or 200, "random")
    if name == "c4":
        h = 1.0 / 384.0
        bands = [(64, h), (128, h / 2), (128, h), (128, h / 2), (64, h)]
        e = banded_edges(0.0, bands)
        mesh = P.Mesh2DRect(e, list(e))
        al = axis_levels(bands)
        fam = family or load_config_family("c4_p3_4_8")
        return Config("c4", "2D Navier-Stokes double shear layer, 512^2 2-level mesh, p3 {4,8}",
                      mesh, "hlle", fam, geometric_levels([al, al], fam.R), cfl or 1.1,
                      steps or 200, "shear", physics="nsf", mu=1e-4, prandtl=0.72)
    if name == "c5":
        h = 2 * math.pi / 54.0
        bands = [(24, h), (4, h / 2), (8, h / 4), (4, h / 2), (24, h)]
        e = banded_edges(0.0, bands)
        mesh = P.Mesh3DRect(e, list(e), list(e))
        al = axis_levels(bands)
        fam = family or load_config_family("c5_p4_5_8_14")
        return Config("c5", "3D Euler Taylor-Green Ma 0.1, 64^3 3-level mesh, p4 {5,8,14}",
                      mesh, "rusanov", fam, geometric_levels([al, al, al], fam.R), cfl or 1.1,
                      steps or 100, "tgv")
    raise ValueError(f"unknown config {name}")


def _scaled_bands(bands, factor, length):
    """Same band structure with every count divided by factor (>= 1 cell)."""
    counts = [max(1, n // factor) for n, _ in bands]
    rel = [h for _, h in bands]
    total = sum(n * r for n, r in zip(counts, rel))
    scale = length / total
    return [(n, r * scale) for n, r in zip(counts, rel)]


def sample_config(cfg: Config) -> Config:
    """A bounded CPU sample of a configuration: the same family, flux, initial
    condition, CFL and level grading on a mesh with fewer cells per band
    (C5: 16^3 instead of 64^3; C3: 32^2 instead of 256^2).  Used only for the
    CPU baseline timing, never for parity."""
    import copy
    out = copy.copy(cfg)
    if cfg.name == "c5":
        bands = _scaled_bands([(24, 1.0), (4, 0.5), (8, 0.25), (4, 0.5), (24, 1.0)], 4,
                              2 * math.pi)
        e = banded_edges(0.0, bands)
        out.mesh = P.Mesh3DRect(e, list(e), list(e))
        al = axis_levels(bands)
        out.raw_levels = geometric_levels([al, al, al], cfg.family.R)
        out.description = "C5 sample: 16^3-element 3-level graded TGV mesh"
    elif cfg.name == "c3":
        bands = _scaled_bands([(96, 1.0), (16, 0.5), (32, 0.25), (16, 0.5), (96, 1.0)], 8,
                              2 * math.pi)
        e = banded_edges(0.0, bands)
        out.mesh = P.Mesh2DRect(e, list(e))
        al = axis_levels(bands)
        out.raw_levels = geometric_levels([al, al], cfg.family.R)
        out.description = "C3 sample: 32^2-element 3-level graded mesh"
    return out


class ConfigRun:
    """A configuration instantiated on one device: semidiscretization,
    partition map, initial state.  With world > 1 the context owns the
    rank's cells (perrk_comm_init) of a per-level balanced partition
    ("levels", the default: every stage balanced) or of work-balanced
    last-axis slabs ("slabs": least halo)."""

    def __init__(self, cfg: Config, device=0, rank=0, world=1, comm=None, partition="levels"):
        self.cfg = cfg
        self.rank, self.world = rank, world
        self.partition = partition
        self.semi = P.Semidiscretization(cfg.spec(device))
        self.pmap = cfg.partition_map()
        if world > 1:
            self.owner = make_owner(cfg, self.pmap, world, partition)
            P.init_partition(self.semi, rank, world, self.owner)

    def initial_state(self):
        s = self.semi
        return initial_state_for(self.cfg, (s.node_x(), s.node_y(),
                                            s.node_z() if self.cfg.dim == 3 else None))

    def dof_stage_updates_per_step(self):
        """This rank's share (all ranks when world == 1)."""
        return dof_stage_updates_per_step(self.cfg.family, self.local_pmap(),
                                          self.cfg.nodes_per_cell())

    def halo_traces(self):
        """Face traces all ranks exchange per stage."""
        return int(sum(P.halo_plan(self.cfg.mesh, self.owner, r)["send"].shape[0]
                       for r in range(self.world)))

    def local_pmap(self):
        return self.pmap if self.world == 1 else P.local_pmap(self.semi, self.pmap)

    def total_nodes(self):
        return self.cfg.mesh.num_cells() * self.cfg.nodes_per_cell()


def make_owner(cfg: Config, pmap, world, partition="levels"):
    """Global ownership map (cell -> rank) of a decomposition over `world` ranks."""
    if partition == "levels":
        return P.partition_levels(cfg.mesh, pmap, world)
    if partition == "slabs":
        return P.partition_slabs(cfg.mesh, world,
                                 P.cell_work(pmap, cfg.family, cfg.nodes_per_cell()))
    raise ValueError(f"unknown partition {partition!r}")


def initial_state_for(cfg: Config, semi_or_coords):
    """U0 in the canonical layout from node coordinates (x, y[, z])."""
    x, y, z = semi_or_coords
    vals = cfg.initial_state(x, y, z)
    return np.ascontiguousarray(vals.T).reshape(-1)


def dof_stage_updates_per_step(family: P.PartitionFamily, pmap: P.PartitionMap, npc: int):
    """Sum over stages of active nodes = rhs_cell_evaluations()/V per step
    (semidisc.cpp:131-133; PAPER N_K)."""
    counts = pmap.cells_per_level()
    total = 0
    for lvl, n in enumerate(counts, start=1):
        total += len(family.active_sets[family.member_index_for_level(lvl)]) * n
    return total * npc
