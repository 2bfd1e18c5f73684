"""TEST INFRASTRUCTURE — the BASELINE workloads on the CPU checkers.

Builds a configuration of `configs/spec.py` on the oracle restatement
(`Orc`, oracle/_build/liboracle.so) or, for the 2D Euler configs, on the
unmodified reference (`Ref`, oracle/_ref/libperrk_ref.so), WITHOUT the
product package: meshes, level maps (make_partition_map restated in
configs/spec.py, mesh.cpp:56-71), families (text fixtures, butcher.cpp:357-433)
and initial conditions all come from configs/spec.py.

Used by tests/ (long-run parity fixtures), and by bench.py's CPU legs
(cpu_baseline and `--impl reference`).  Never by the product.
"""
import importlib.util
import math
import os
import sys
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
if HERE not in sys.path:
    sys.path.insert(0, HERE)
import oracle as O  # noqa: E402


def load_spec_module():
    name = "perrk_config_spec"
    if name in sys.modules:
        return sys.modules[name]
    s = importlib.util.spec_from_file_location(name, os.path.join(ROOT, "configs", "spec.py"))
    m = importlib.util.module_from_spec(s)
    sys.modules[name] = m
    s.loader.exec_module(m)
    return m


S = load_spec_module()


@dataclass
class RelaxCfg:
    """RelaxationConfig defaults (relax.hpp:16-24) + the numerics selector."""
    method: str = "newton"
    max_iter: int = 5
    residual_tol: float = 1e-14
    step_tol: float = 1e-15
    bracket_min: float = 0.8
    bracket_max: float = 1.2
    seed_from_previous: bool = True
    numerics: str = "accurate"


class FamilyArgs:
    """The attribute set oracle._Base._fam reads (S, R, kind, E, A, b, c)."""

    def __init__(self, ft):
        self.kind, self.S, self.R = ft.kind, ft.S, ft.R
        self.E, self.A, self.b, self.c = ft.E, ft.A, ft.b, ft.c


class CpuConfig:
    """One configuration on a CPU checker.  kind 'orc' (restatement, every
    config) or 'ref' (the unmodified reference: 2D Euler only)."""

    def __init__(self, spec, threads=1, kind="orc"):
        self.spec = spec
        kw = dict(surface_flux=spec.surface_flux, threads=threads, gamma=spec.gamma)
        if kind == "orc":
            if spec.physics == "nsf":
                kw.update(viscous=True, mu=spec.mu, prandtl=spec.prandtl)
            self.chk = O.Orc(spec.mesh, **kw)
        else:
            if spec.physics != "euler" or spec.dim != 2:
                raise ValueError("the reference has 2D Euler only")
            self.chk = O.Ref(spec.mesh, **kw)
            self.chk.set_threads(threads)
        self.kind = kind
        self.family = FamilyArgs(spec.family())
        self.eff = spec.effective_levels()
        self.relax = RelaxCfg(numerics=spec.relaxation_numerics if kind == "orc" else "reference")

    def initial_state(self):
        x, y, z, _ = self.chk.node_coords()
        return self.spec.canonical_state(x, y, z)

    def run(self, U, steps, t=0.0, records=True):
        """run() loop body (stepper.cpp:144-188) for exactly `steps` steps, in
        place on U; returns (t, taken, log[steps, 6+V], seconds)."""
        return self.chk.run_steps(U, t, steps, self.family, self.eff, self.relax, False,
                                  self.spec.cfl, records=records)

    def total_entropy(self, U):
        return self.chk.total_entropy(U)

    def total_entropy_acc(self, U):
        return self.chk.total_entropy_acc(U)

    def dof_stage_updates_per_step(self):
        return self.spec.dof_stage_updates_per_step(self.eff)


def sample_indices(n_nodes, count, seed=12345):
    """Seeded node sample (sorted, without replacement) for the committed
    long-run fixtures."""
    rng = np.random.Generator(np.random.PCG64(seed))
    count = min(count, n_nodes)
    return np.sort(rng.choice(n_nodes, size=count, replace=False)).astype(np.int64)
