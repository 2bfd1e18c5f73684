"""Synthetic workloads of BASELINE.json's five configurations (host side).

The workload definitions themselves (meshes as edge arrays, raw level maps,
seeded initial conditions, family fixtures, CFL numbers, step counts) live in
`configs/spec.py`, which is plain numpy and shared with the CPU arms; this
module instantiates them on the product's types (Mesh2DRect/Mesh3DRect,
PartitionFamily, the native make_partition_map).  Decisions the reference
leaves open are recorded in configs/spec.py and
DESIGN.md.
"""
from __future__ import annotations

import importlib.util
import math
import os
import sys
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import perrk as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONFIG_DIR = os.path.join(ROOT, "configs")


def _load_spec_module():
    name = "perrk_config_spec"
    if name in sys.modules:
        return sys.modules[name]
    s = importlib.util.spec_from_file_location(name, os.path.join(CONFIG_DIR, "spec.py"))
    m = importlib.util.module_from_spec(s)
    sys.modules[name] = m
    s.loader.exec_module(m)
    return m


S = _load_spec_module()
VortexParams = S.VortexParams
isentropic_vortex = S.isentropic_vortex
random_fourier_state = S.random_fourier_state
double_shear_layer = S.double_shear_layer
taylor_green = S.taylor_green
banded_edges = S.banded_edges
axis_levels = S.axis_levels
geometric_levels = S.geometric_levels


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
    spec_: object = None

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
        return self.spec_.initial_state(x, y, z)

    def nodes_per_cell(self):
        return 16 if self.dim == 2 else 64


def family_path(name):
    return os.path.join(CONFIG_DIR, f"{name}.family")


def load_config_family(name):
    return P.load_family(family_path(name))


def c1_family():
    """C1's p2 S = 4 member: (a21, a32) = (0.204, 0.42), linearly stable at
    CFL 0.9 on C1's probed spectrum (max |P| = 1.000000, 1.000003 at 5% above;
    configs/c1_pair_scan.py).  The survey's (0.2, 0.35) reached 1.60."""
    return P.build_perk2(4, [4], [[0.204, 0.42]])


def _mesh(ms):
    e = [list(map(float, x)) for x in ms.edges]
    return P.Mesh2DRect(*e) if ms.dim == 2 else P.Mesh3DRect(*e)


def from_spec(sp, family=None, cfl=None, steps=None) -> Config:
    fam = family or (c1_family() if sp.name == "c1" else load_config_family(sp.family_file))
    return Config(sp.name, sp.description, _mesh(sp.mesh), sp.surface_flux, fam,
                  np.asarray(sp.raw_levels, np.int32), cfl or sp.cfl, steps or sp.steps, sp.ic,
                  gamma=sp.gamma, physics=sp.physics, mu=sp.mu, prandtl=sp.prandtl, spec_=sp)


def make_config(name: str, family=None, cfl=None, steps=None) -> Config:
    return from_spec(S.make_spec(name), family, cfl, steps)


def sample_config(cfg: Config) -> Config:
    """The bounded CPU sample of configs/spec.py (sample_spec) on product types."""
    return from_spec(S.sample_spec(cfg.spec_), family=cfg.family, cfl=cfg.cfl, steps=cfg.steps)


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
