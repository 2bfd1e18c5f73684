"""GPU parity of the 2D Navier-Stokes-Fourier + BR1 path (BASELINE config C4)
against the oracle's 2D NSF extension (pinned on the reference's 1D NSF by
tests/test_oracle.py::test_orc_nsf2d_reduces_to_reference_nsf1d).
Tolerances as tests/test_gpu_parity.py."""
import numpy as np
import pytest

import oracle as O
from helpers import max_rel, mesh2d, rel_err, smooth_state
from paper_2507_04991_b200 import perrk as P
from paper_2507_04991_b200 import workloads as W

pytestmark = pytest.mark.gpu

MU = 2e-2


def _pair(mesh, surface="hlle", mu=MU):
    spec = P.SemidiscretizationSpec(mesh, physics="nsf", mu=mu, prandtl=0.72,
                                    surface_flux=surface)
    return P.Semidiscretization(spec), O.Orc(mesh, surface_flux=surface, viscous=True, mu=mu,
                                             prandtl=0.72)


@pytest.mark.parametrize("surface", ["rusanov", "hlle", "ec"])
def test_nsf_rhs_vs_oracle(surface):
    mesh = mesh2d(9, 7, seed=81)
    semi, orc = _pair(mesh, surface)
    U = smooth_state((semi.node_x(), semi.node_y()), 2, seed=13)
    assert max_rel(semi.rhs(0.0, U), orc.rhs(0.0, U)) < 1e-12


def test_br1_gradients_vs_oracle():
    mesh = mesh2d(8, 6, seed=82)
    semi, orc = _pair(mesh)
    U = smooth_state((semi.node_x(), semi.node_y()), 2, seed=14)
    g, go = semi.br1_gradients(0.0, U), orc.br1_gradients(0.0, U)
    assert max_rel(g, go) < 1e-12


def test_nsf_masked_rhs_vs_oracle():
    mesh = mesh2d(8, 8, seed=83)
    semi, orc = _pair(mesh)
    U = smooth_state((semi.node_x(), semi.node_y()), 2, seed=15)
    rng = np.random.default_rng(6)
    for _ in range(3):
        mask = rng.integers(0, 2, semi.num_cells()).astype(np.int8)
        g, r = semi.rhs_masked(0.0, U, mask), orc.rhs_masked(0.0, U, mask)
        assert max_rel(g, r) < 1e-12
        assert np.all(g.reshape(semi.num_cells(), -1)[mask == 0] == 0.0)


def test_nsf_mu0_equals_euler():
    """test_dg.cpp:242-267 in 2D: mu = 0 gives the inviscid RHS."""
    mesh = mesh2d(6, 6, seed=84)
    semi, _ = _pair(mesh, mu=0.0)
    eul = P.Semidiscretization(P.SemidiscretizationSpec(mesh, surface_flux="hlle"))
    U = smooth_state((semi.node_x(), semi.node_y()), 2, seed=16)
    assert max_rel(semi.rhs(0.0, U), eul.rhs(0.0, U)) < 1e-14


def test_nsf_multilevel_relaxed_steps_vs_oracle():
    mesh = mesh2d(10, 8, seed=85)
    fam = W.load_config_family("c4_p3_4_8")
    pm = P.make_partition_map(mesh, np.random.default_rng(8).integers(1, 3, mesh.num_cells()), 2)
    semi, orc = _pair(mesh)
    U0 = smooth_state((semi.node_x(), semi.node_y()), 2, seed=17, amp=0.2)
    dt = 0.3 * orc.compute_dt(U0, False, 1.0)
    rx = P.RelaxationConfig(numerics="accurate")
    Ug, Uo = U0.copy(), U0.copy()
    tg = to = 0.0
    for _ in range(5):
        tg, rg = P.perk_step(Ug, tg, dt, fam, pm, semi, P.PerkStepOptions(relaxation=rx))
        to, ro = orc.perk_step(Uo, to, dt, fam, pm.effective_level, rx)
        assert abs(rg.gamma - ro.gamma) < 1e-12
        assert abs(rg.delta_h - ro.delta_h) < 1e-12
    assert rel_err(Ug, Uo, 4) < 1e-11
    semi.reset_evaluation_counter()
    P.perk_step(Ug, tg, dt, fam, pm, semi, P.PerkStepOptions(relaxation=rx))
    assert semi.rhs_cell_evaluations() == W.dof_stage_updates_per_step(fam, pm, 16) * 4


def test_c4_initial_rhs_vs_oracle_small():
    """C4's double shear layer on a reduced mesh of the same grading."""
    e = W.banded_edges(0.0, [(4, 1 / 24), (8, 1 / 48), (8, 1 / 24), (8, 1 / 48), (4, 1 / 24)])
    mesh = P.Mesh2DRect(e, list(e))
    semi, orc = _pair(mesh, "hlle", mu=1e-4)
    U = np.ascontiguousarray(W.double_shear_layer(semi.node_x(), semi.node_y()).T).reshape(-1)
    # at Ma 0.1 the RHS (~1e-2) is a difference of flux-differencing terms
    # ~ |U| (2/h) max|D_lm| ~ 5e4: FP64 parity is relative to that flux scale
    flux_scale = np.abs(U).max() * 2.0 / min(np.diff(e)) * 3.0
    assert np.abs(semi.rhs(0.0, U) - orc.rhs(0.0, U)).max() < 1e-14 * flux_scale
