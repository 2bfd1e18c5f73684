"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Oracles: `Ref` is the unmodified reference library (dim 2), `Orc` the C
restatement (dim 2 and 3, accurate relaxation numerics).  Tolerances:
  RHS / reductions   1e-12 relative to the field's max (FP64 statistical
                     parity: CUDA libdevice log/sqrt vs glibc, FMA contraction,
                     log a - log b in the EC flux)
  states after N steps  1e-11 relative L2 per conserved variable (north_star)
  gamma sequence, dH    1e-12 absolute (north_star), against the oracle with the
                        same relaxation numerics
"""
import math

import numpy as np
import pytest

import oracle as O
from helpers import max_rel, mesh2d, mesh3d, rel_err, smooth_state
from paper_2507_04991_b200 import perrk as P
from paper_2507_04991_b200 import workloads as W

pytestmark = pytest.mark.gpu

SURFACES = ["rusanov", "hlle", "hllc", "ec", "central"]


def c1_setup():
    cfg = W.make_config("c1")
    semi = P.Semidiscretization(cfg.spec())
    U0 = W.initial_state_for(cfg, (semi.node_x(), semi.node_y(), None))
    return cfg, semi, U0


# --------------------------------------------------------------------------- RHS
def test_rhs_c1_initial_condition_vs_reference():
    cfg, semi, U0 = c1_setup()
    ref = O.Ref(cfg.mesh, surface_flux="rusanov")
    r_ref = ref.rhs(0.0, U0)
    r_gpu = semi.rhs(0.0, U0)
    assert max_rel(r_gpu, r_ref) < 1e-12


@pytest.mark.parametrize("surface", SURFACES)
def test_rhs_2d_random_state_all_surface_fluxes(surface):
    mesh = mesh2d(9, 7, seed=3)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh, surface_flux=surface))
    U = smooth_state((semi.node_x(), semi.node_y()), 2, seed=11)
    ref = O.Ref(mesh, surface_flux=surface)
    assert max_rel(semi.rhs(0.0, U), ref.rhs(0.0, U)) < 1e-12


VOLUMES = [("weak", "ec"), ("flux_differencing", "central")]


@pytest.mark.parametrize("mode,vflux", VOLUMES)
@pytest.mark.parametrize("surface", SURFACES)
def test_rhs_2d_volume_variants_vs_reference(mode, vflux, surface):
    """Weak form (semidisc.cpp:429-445) and central flux differencing on the
    device (the SIMPLE stage kernels)."""
    mesh = mesh2d(9, 7, seed=13)
    kw = dict(surface_flux=surface, volume_mode=mode, volume_flux=vflux)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh, **kw))
    U = smooth_state((semi.node_x(), semi.node_y()), 2, seed=17)
    ref = O.Ref(mesh, **kw)
    assert max_rel(semi.rhs(0.0, U), ref.rhs(0.0, U)) < 1e-12
    mask = np.random.default_rng(6).integers(0, 2, semi.num_cells()).astype(np.int8)
    assert max_rel(semi.rhs_masked(0.0, U, mask), ref.rhs_masked(0.0, U, mask)) < 1e-12


@pytest.mark.parametrize("mode,vflux", VOLUMES)
@pytest.mark.parametrize("surface", ["rusanov", "hlle", "ec"])
def test_rhs_3d_volume_variants_vs_oracle(mode, vflux, surface):
    mesh = mesh3d(4, 3, 5, seed=19)
    kw = dict(surface_flux=surface, volume_mode=mode, volume_flux=vflux)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh, **kw))
    U = smooth_state((semi.node_x(), semi.node_y(), semi.node_z()), 3, seed=23)
    orc = O.Orc(mesh, **kw)
    assert max_rel(semi.rhs(0.0, U), orc.rhs(0.0, U)) < 1e-12


@pytest.mark.parametrize("mode,vflux", VOLUMES)
def test_multilevel_steps_volume_variants_vs_reference(mode, vflux):
    """Unrelaxed multirate steps against the reference; relaxed steps (accurate
    numerics) against the oracle for the gamma sequence."""
    mesh = mesh2d(8, 8, seed=29)
    fam = P.build_perk3_variant(7, [4, 7], [[0.3], [0.2, 0.25, 0.3, 0.35]])
    rng = np.random.default_rng(8)
    pm = P.make_partition_map(mesh, rng.integers(1, 3, mesh.num_cells()), 2)
    kw = dict(surface_flux="hlle", volume_mode=mode, volume_flux=vflux)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh, **kw))
    ref, orc = O.Ref(mesh, **kw), O.Orc(mesh, **kw)
    U0 = smooth_state((semi.node_x(), semi.node_y()), 2, seed=31, amp=0.2)
    dt = 0.3 * ref.compute_dt(U0, False, 1.0)
    Ug, Ur = U0.copy(), U0.copy()
    for _ in range(5):
        P.perk_step(Ug, 0.0, dt, fam, pm, semi, P.PerkStepOptions())
        ref.perk_step(Ur, 0.0, dt, fam, pm.effective_level)
    assert rel_err(Ug, Ur, 4) < 1e-12
    rx = P.RelaxationConfig(numerics="accurate")
    Ug, Uo = U0.copy(), U0.copy()
    tg = to = 0.0
    for _ in range(5):
        tg, rg = P.perk_step(Ug, tg, dt, fam, pm, semi, P.PerkStepOptions(relaxation=rx))
        to, ro = orc.perk_step(Uo, to, dt, fam, pm.effective_level, rx)
        assert abs(rg.gamma - ro.gamma) < 1e-12 and rg.fell_back == bool(ro.fell_back)
    assert rel_err(Ug, Uo, 4) < 1e-11


def test_volume_variant_argument_errors():
    mesh = mesh2d(4, 4)
    with pytest.raises(P.Error):
        P.Semidiscretization(P.SemidiscretizationSpec(mesh, volume_mode="flux_differencing",
                                                      volume_flux="rusanov"))


def test_rhs_masked_matches_reference_and_zero_fill():
    mesh = mesh2d(8, 8, seed=5)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh, surface_flux="hlle"))
    U = smooth_state((semi.node_x(), semi.node_y()), 2, seed=2)
    ref = O.Ref(mesh, surface_flux="hlle")
    rng = np.random.default_rng(4)
    for _ in range(3):
        mask = rng.integers(0, 2, semi.num_cells()).astype(np.int8)
        g = semi.rhs_masked(0.0, U, mask)
        r = ref.rhs_masked(0.0, U, mask)
        assert max_rel(g, r) < 1e-12
        cellwise = g.reshape(semi.num_cells(), -1)
        assert np.all(cellwise[mask == 0] == 0.0)


def test_partition_restricted_union_equals_full():
    """test_dg.cpp:302-346 on the device: disjoint supports, union = full."""
    mesh = mesh2d(10, 6, seed=8)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh))
    U = smooth_state((semi.node_x(), semi.node_y()), 2, seed=9)
    levels = np.random.default_rng(1).integers(1, 3, semi.num_cells())
    pm = P.make_partition_map(mesh, levels, 2)
    full = semi.rhs(0.0, U)
    r1 = semi.rhs_partition_restricted(0.0, U, pm, 1)
    r2 = semi.rhs_partition_restricted(0.0, U, pm, 2)
    assert np.all((r1 == 0.0) | (r2 == 0.0))
    assert np.array_equal(r1 + r2, full)


def test_free_stream_and_entropy_conservation():
    """test_dg.cpp:84-102 and :157-172 on the device (EC surface flux)."""
    mesh = P.Mesh2DRect(*[W.banded_edges(-10, [(4, 3.0), (4, 2.0)])] * 2)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh, surface_flux="ec"))
    n = semi.num_nodes()
    U = np.tile([1.0, 1.0, 1.0, 12.16], n)
    assert np.abs(semi.rhs(0.0, U)).max() < 1e-11
    U = W.isentropic_vortex(W.VortexParams(mach=0.4, radius=1.5, intensity=13.5),
                            semi.node_x(), semi.node_y())
    U = np.ascontiguousarray(U.T).reshape(-1)
    assert abs(semi.entropy_inner_product(U, semi.rhs(0.0, U))) < 1e-11


def test_conservation_of_quadrature_totals():
    mesh = mesh2d(8, 8, seed=12)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh, surface_flux="hllc"))
    U = smooth_state((semi.node_x(), semi.node_y()), 2, seed=3)
    assert np.abs(semi.integral_per_variable(semi.rhs(0.0, U))).max() < 5e-12


# --------------------------------------------------------------------------- reductions
def test_reductions_vs_reference():
    mesh = mesh2d(12, 10, seed=21)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh))
    ref = O.Ref(mesh)
    U = smooth_state((semi.node_x(), semi.node_y()), 2, seed=5)
    K = smooth_state((semi.node_x(), semi.node_y()), 2, seed=6)
    assert abs(semi.total_entropy(U) - ref.total_entropy(U)) < 1e-12 * abs(ref.total_entropy(U))
    ip_ref = ref.entropy_inner_product(U, K)
    assert abs(semi.entropy_inner_product(U, K) - ip_ref) < 1e-12 * max(1.0, abs(ip_ref))
    assert np.allclose(semi.integral_per_variable(U), ref.integral_per_variable(U), rtol=1e-13)
    nu_g, nu_r = semi.characteristic_speed(U), ref.characteristic_speed(U)
    assert max_rel(nu_g, nu_r) < 1e-14
    ok, bad = semi.admissible(U)
    assert ok and bad == -1
    Ub = U.copy()
    Ub[(37 * semi.nodes_per_cell() + 3) * 4 + 0] = -1.0
    Ub[(55 * semi.nodes_per_cell() + 1) * 4 + 3] = 0.0
    assert semi.admissible(Ub) == ref.admissible(Ub) == (False, 37)


# --------------------------------------------------------------------------- stepping
def test_perk_step_c1_reference_numerics():
    cfg, semi, U0 = c1_setup()
    ref = O.Ref(cfg.mesh)
    dt = ref.compute_dt(U0, False, 0.9)
    opts = P.PerkStepOptions(relaxation=P.RelaxationConfig())
    Ug = U0.copy()
    tg, rg = P.perk_step(Ug, 0.0, dt, cfg.family, cfg.partition_map(), semi, opts)
    Ur = U0.copy()
    tr, rr = ref.perk_step(Ur, 0.0, dt, cfg.family, cfg.partition_map().effective_level,
                           P.RelaxationConfig())
    assert rel_err(Ug, Ur, 4) < 1e-13
    assert abs(rg.gamma - rr.gamma) < 1e-12
    assert abs(rg.delta_h - rr.delta_h) < 1e-12
    assert rg.fell_back == bool(rr.fell_back)
    assert abs(tg - tr) < 1e-12 * dt  # t advances by gamma dt


def _run_c1(semi, cfg, U0, numerics, steps=100):
    semi.upload(U0)
    run_cfg = P.IntegratorConfig(tf=1e9, time=P.TimeControl(fixed=False, ramp=P.CflRamp(0.9, 0.9)),
                                 relaxation=P.RelaxationConfig(numerics=numerics))
    t, taken, aborted, recs = P.advance(semi, cfg.family, cfg.partition_map(), run_cfg, 0.0, steps)
    assert taken == steps and not aborted
    return semi.download(), recs


def test_c1_100_steps_vs_oracle_accurate_relaxation():
    """BASELINE C1: 100 relaxed P-ERRK steps at CFL 0.9 — state 1e-11 rel L2
    per variable, gamma sequence and H within 1e-12 of the oracle."""
    cfg, semi, U0 = c1_setup()
    Ug, recs = _run_c1(semi, cfg, U0, "accurate")
    orc = O.Orc(cfg.mesh)
    Uo = U0.copy()
    _, taken, log, _ = orc.run_steps(Uo, 0.0, 100, cfg.family, cfg.partition_map().effective_level,
                                     P.RelaxationConfig(numerics="accurate"), False, 0.9)
    assert taken == 100
    assert rel_err(Ug, Uo, 4) < 1e-11
    gam = np.array([r.gamma for r in recs])
    assert np.abs(gam - log[:, 2]).max() < 1e-12
    H = np.array([r.entropy for r in recs])
    assert np.abs(H - log[:, 4]).max() < 1e-12
    assert np.abs(np.array([r.t for r in recs]) - log[:, 0]).max() < 1e-11


def test_c1_100_steps_vs_unmodified_reference():
    cfg, semi, U0 = c1_setup()
    Ug, recs = _run_c1(semi, cfg, U0, "reference")
    ref = O.Ref(cfg.mesh)
    Ur = U0.copy()
    _, taken, log, _ = ref.run_steps(Ur, 0.0, 100, cfg.family, cfg.partition_map().effective_level,
                                     P.RelaxationConfig(), False, 0.9)
    assert taken == 100
    assert rel_err(Ug, Ur, 4) < 1e-11
    assert np.abs(np.array([r.gamma for r in recs]) - log[:, 2]).max() < 1e-12
    assert sum(r.fell_back for r in recs) == int(log[:, 5].sum())


def _multilevel(mesh, R, seed):
    rng = np.random.default_rng(seed)
    return P.make_partition_map(mesh, rng.integers(1, R + 1, mesh.num_cells()), R)


@pytest.mark.parametrize("kind", ["p3", "p4"])
def test_multilevel_steps_2d_vs_reference(kind):
    """Multirate stage loop (active cell lists, per-level rows, neighbour
    traces formed with the neighbour's row) against the reference."""
    mesh = mesh2d(10, 8, seed=31)
    if kind == "p3":
        fam = P.build_perk3_variant(7, [4, 7], [[0.3], [0.2, 0.25, 0.3, 0.35]])
    else:
        fam = P.build_perk4(14, [5, 8, 14], [[], [0.5] * 3, [0.7] * 9])
    pm = _multilevel(mesh, fam.R, 3)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh, surface_flux="hlle"))
    ref = O.Ref(mesh, surface_flux="hlle")
    U0 = smooth_state((semi.node_x(), semi.node_y()), 2, seed=17, amp=0.2)
    dt = 0.3 * ref.compute_dt(U0, False, 1.0)
    Ug, Ur = U0.copy(), U0.copy()
    for _ in range(5):
        P.perk_step(Ug, 0.0, dt, fam, pm, semi, P.PerkStepOptions())
        ref.perk_step(Ur, 0.0, dt, fam, pm.effective_level)
    assert rel_err(Ug, Ur, 4) < 1e-12
    semi.reset_evaluation_counter()
    P.perk_step(Ug, 0.0, dt, fam, pm, semi, P.PerkStepOptions())
    assert semi.rhs_cell_evaluations() == W.dof_stage_updates_per_step(fam, pm, 16) * 4


def test_multilevel_relaxed_accurate_vs_oracle():
    mesh = mesh2d(10, 8, seed=41)
    fam = P.build_perk4(14, [5, 8, 14], [[], [0.5] * 3, [0.7] * 9])
    pm = _multilevel(mesh, fam.R, 5)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh))
    orc = O.Orc(mesh)
    U0 = smooth_state((semi.node_x(), semi.node_y()), 2, seed=19, amp=0.3)
    dt = 0.3 * orc.compute_dt(U0, False, 1.0)
    rx = P.RelaxationConfig(numerics="accurate")
    Ug, Uo = U0.copy(), U0.copy()
    tg = to = 0.0
    for _ in range(5):
        tg, rg = P.perk_step(Ug, tg, dt, fam, pm, semi, P.PerkStepOptions(relaxation=rx))
        to, ro = orc.perk_step(Uo, to, dt, fam, pm.effective_level, rx)
        assert abs(rg.gamma - ro.gamma) < 1e-12
        assert abs(rg.delta_h - ro.delta_h) < 1e-12
        assert not rg.fell_back and not ro.fell_back
    assert rel_err(Ug, Uo, 4) < 1e-11


def test_positivity_abort_leaves_state_untouched():
    cfg, semi, U0 = c1_setup()
    ref = O.Ref(cfg.mesh)
    Ub = U0.copy()
    Ub[(77 * 16 + 5) * 4 + 0] = -0.5
    Ug, Ur = Ub.copy(), Ub.copy()
    tg, rg = P.perk_step(Ug, 1.0, 0.01, cfg.family, cfg.partition_map(), semi, P.PerkStepOptions())
    tr, rr = ref.perk_step(Ur, 1.0, 0.01, cfg.family, cfg.partition_map().effective_level)
    assert rg.aborted and rr.aborted
    assert (rg.bad_cell, rg.bad_stage) == (rr.bad_cell, rr.bad_stage) == (77, 0)
    assert np.array_equal(Ug, Ub) and tg == 1.0


# --------------------------------------------------------------------------- 3D
def test_rhs_3d_vs_oracle():
    mesh = mesh3d(5, 4, 3, seed=51)
    for surface in ["rusanov", "hlle", "ec"]:
        semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh, surface_flux=surface))
        orc = O.Orc(mesh, surface_flux=surface)
        U = smooth_state((semi.node_x(), semi.node_y(), semi.node_z()), 3, seed=23)
        assert max_rel(semi.rhs(0.0, U), orc.rhs(0.0, U)) < 1e-12


def test_3d_multilevel_relaxed_vs_oracle():
    mesh = mesh3d(4, 5, 4, seed=61)
    fam = P.build_perk4(14, [5, 8, 14], [[], [0.5] * 3, [0.7] * 9])
    pm = _multilevel(mesh, 3, 7)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh))
    orc = O.Orc(mesh)
    U0 = smooth_state((semi.node_x(), semi.node_y(), semi.node_z()), 3, seed=29, amp=0.25)
    dt = 0.3 * orc.compute_dt(U0, False, 1.0)
    rx = P.RelaxationConfig(numerics="accurate")
    Ug, Uo = U0.copy(), U0.copy()
    for _ in range(3):
        _, rg = P.perk_step(Ug, 0.0, dt, fam, pm, semi, P.PerkStepOptions(relaxation=rx))
        _, ro = orc.perk_step(Uo, 0.0, dt, fam, pm.effective_level, rx)
        assert abs(rg.gamma - ro.gamma) < 1e-12
    assert rel_err(Ug, Uo, 5) < 1e-11


def test_tgv_initial_rhs_3d_vs_oracle():
    mesh = P.build_uniform_mesh3d(0.0, 2 * math.pi, 4)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh))
    orc = O.Orc(mesh)
    U = np.ascontiguousarray(W.taylor_green(semi.node_x(), semi.node_y(), semi.node_z()).T).reshape(-1)
    assert max_rel(semi.rhs(0.0, U), orc.rhs(0.0, U)) < 1e-12


def test_cpp_adapter_drop_in_parity():
    """The reference's own perk_step vs perrk_b200::perk_step at identical C++
    call sites (tests/cpp/adapter_parity.cpp, built against the unmodified
    reference in oracle/_ref)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(O.REF_LIB), "adapter_parity")
    if not os.path.exists(exe):
        pytest.skip("adapter_parity not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("method", ["bisection", "secant"])
def test_bisection_secant_relaxation_vs_reference(method):
    """relax.cpp:105-148 on the device: the same residual sequence as the
    unmodified reference (reference numerics, C1 vortex; a bracket around 1)."""
    cfg, semi, U0 = c1_setup()
    ref = O.Ref(cfg.mesh)
    dt = ref.compute_dt(U0, False, 0.9)
    rx = P.RelaxationConfig(method=method, max_iter=30, bracket_min=0.9, bracket_max=1.1,
                            residual_tol=1e-14, step_tol=1e-12)
    Ug, Ur = U0.copy(), U0.copy()
    tg = tr = 0.0
    for _ in range(5):
        tg, rg = P.perk_step(Ug, tg, dt, cfg.family, cfg.partition_map(), semi,
                             P.PerkStepOptions(relaxation=rx))
        tr, rr = ref.perk_step(Ur, tr, dt, cfg.family, cfg.partition_map().effective_level, rx)
        assert rg.fell_back == bool(rr.fell_back)
        # the stop test |r| <= residual_tol (relax.cpp:105-148) sits at the
        # residual's rounding noise here (|r| ~ 9e-15 against 1e-14), so an
        # ulp-level difference of the RHS may stop one iteration earlier or
        # later; the root itself must agree to 1e-12
        early = rg if rg.iterations < rr.iterations else rr  # the side that stopped first
        near_tol = abs(early.residual) >= 0.1 * rx.residual_tol
        assert abs(rg.iterations - rr.iterations) <= (1 if near_tol else 0)
        assert abs(rg.gamma - rr.gamma) < 1e-12
    assert rel_err(Ug, Ur, 4) < 1e-12


@pytest.mark.parametrize("method", ["bisection", "secant"])
def test_bisection_secant_accurate_vs_oracle(method):
    mesh = mesh2d(10, 8, seed=91)
    fam = P.build_perk4(14, [5, 8, 14], [[], [0.5] * 3, [0.7] * 9])
    pm = _multilevel(mesh, fam.R, 9)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh))
    orc = O.Orc(mesh)
    U0 = smooth_state((semi.node_x(), semi.node_y()), 2, seed=23, amp=0.3)
    dt = 0.3 * orc.compute_dt(U0, False, 1.0)
    rx = P.RelaxationConfig(method=method, numerics="accurate", max_iter=40, bracket_min=0.95,
                            bracket_max=1.05, residual_tol=1e-15, step_tol=1e-13)
    Ug, Uo = U0.copy(), U0.copy()
    for _ in range(3):
        _, rg = P.perk_step(Ug, 0.0, dt, fam, pm, semi, P.PerkStepOptions(relaxation=rx))
        _, ro = orc.perk_step(Uo, 0.0, dt, fam, pm.effective_level, rx)
        assert rg.fell_back == bool(ro.fell_back)
        assert abs(rg.gamma - ro.gamma) < 1e-12
    assert rel_err(Ug, Uo, 4) < 1e-11


def test_cfl_ramp_on_device_matches_stepwise_compute_dt():
    """CflRamp (stepper.cpp:13-15) evaluated in begin_step equals compute_dt
    with the ramp evaluated on the host, step by step (gamma seed carried as
    run() does, stepper.cpp:153,170)."""
    cfg, semi, U0 = c1_setup()
    ramp = P.CflRamp(0.3, 0.9, 0.5)
    ic = P.IntegratorConfig(t0=0.1, tf=1e9, time=P.TimeControl(False, 0.0, ramp),
                            relaxation=P.RelaxationConfig(numerics="accurate"))
    semi.upload(U0)
    t, taken, aborted, recs = P.advance(semi, cfg.family, cfg.partition_map(), ic, 0.1, 12)
    assert taken == 12 and not aborted
    Uh = U0.copy()
    th, seed = 0.1, 1.0
    for r in recs:
        dt = P.compute_dt(Uh, semi, ic, th)
        assert abs(dt - r.dt) <= 1e-13 * dt
        th, res = P.perk_step(Uh, th, dt, cfg.family, cfg.partition_map(), semi,
                              P.PerkStepOptions(relaxation=ic.relaxation, gamma_seed=seed))
        seed = 1.0 if res.fell_back else res.gamma
    dts = [r.dt for r in recs]
    assert dts[-1] > 1.5 * dts[0]  # the ramp raises the step


def test_error_norms_vortex_vs_reference():
    """error_norms (stepper.cpp:195-265) on the device against the reference,
    for the C1 vortex at t = 0 and after 20 device steps."""
    cfg, semi, U0 = c1_setup()
    ref = O.Ref(cfg.mesh)
    vp = W.VortexParams()
    l1, li = semi.error_norms_vortex(U0, vp, 0.0)
    r1, ri = ref.error_norms_vortex(U0, vp.as_array(), 0.0)
    assert np.allclose(l1, r1, rtol=1e-11, atol=1e-16) and np.allclose(li, ri, rtol=1e-11, atol=1e-16)
    Ug, recs = _run_c1(semi, cfg, U0, "accurate", steps=20)
    t = recs[-1].t
    l1, li = semi.error_norms_vortex(Ug, vp, t)
    r1, ri = ref.error_norms_vortex(Ug, vp.as_array(), t)
    assert np.allclose(l1, r1, rtol=1e-11) and np.allclose(li, ri, rtol=1e-11)
    assert l1.max() < 1e-2  # the vortex is resolved: small discretisation error


def test_snapshot_csv_matches_reference_writer(tmp_path):
    cfg, semi, U0 = c1_setup()
    ref = O.Ref(cfg.mesh)
    ours, theirs = tmp_path / "ours.csv", tmp_path / "ref.csv"
    P.write_snapshot_csv(semi, U0, str(ours))
    assert ref.L.ref_write_snapshot(ref.h, O.dp(U0), str(theirs).encode()) == 0
    assert ours.read_bytes() == theirs.read_bytes()


def _mixed_state_3d(semi, seed=5):
    """A 3D state with smooth cells (rho, beta within 0.5 % per cell: the
    warp-per-cell kernel's series-only path) and rough ones (a strong
    Gaussian bump: the per-pair logarithm branch), with the cell split checked."""
    x, y, z = semi.node_x(), semi.node_y(), semi.node_z()
    rng = np.random.default_rng(seed)
    c = rng.uniform(-0.5, 0.5, 3)
    bump = np.exp(-((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2) / 0.08)
    rho = 1.0 + 0.002 * np.sin(math.pi * x) + 0.8 * bump
    v = [0.1 * np.cos(math.pi * y), 0.1 * np.sin(math.pi * z), 0.05 + 0.3 * bump]
    p = 1.0 + 0.002 * np.cos(math.pi * z) + 0.5 * bump
    U = np.stack([rho] + [rho * vv for vv in v] + [p / 0.4 + 0.5 * rho * sum(vv * vv for vv in v)])
    r = rho.reshape(-1, 64)
    ratio = r.max(axis=1) / r.min(axis=1)
    assert (ratio < 1.01).sum() > 0 and (ratio > 1.05).sum() > 0
    return np.ascontiguousarray(U.T).reshape(-1)


@pytest.mark.parametrize("surface", ["rusanov", "central"])
def test_w3_kernel_mixed_smooth_rough_cells_vs_oracle(surface):
    """The 3D warp-per-cell stage kernel (dg_stage3w.cuh) on cells that take
    its series-only path and cells that take the logarithm branch, full and
    masked (active-list) RHS against the oracle."""
    mesh = mesh3d(6, 5, 4, seed=71)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh, surface_flux=surface))
    orc = O.Orc(mesh, surface_flux=surface)
    U = _mixed_state_3d(semi)
    assert max_rel(semi.rhs(0.0, U), orc.rhs(0.0, U)) < 1e-12
    mask = np.random.default_rng(8).integers(0, 2, semi.num_cells()).astype(np.int8)
    assert max_rel(semi.rhs_masked(0.0, U, mask), orc.rhs_masked(0.0, U, mask)) < 1e-12


def test_w3_kernel_multilevel_relaxed_mixed_vs_oracle():
    mesh = mesh3d(5, 4, 4, seed=73)
    fam = P.build_perk4(14, [5, 8, 14], [[], [0.5] * 3, [0.7] * 9])
    pm = _multilevel(mesh, 3, 9)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh))
    orc = O.Orc(mesh)
    U0 = _mixed_state_3d(semi, seed=6)
    dt = 0.3 * orc.compute_dt(U0, False, 1.0)
    rx = P.RelaxationConfig(numerics="accurate")
    Ug, Uo = U0.copy(), U0.copy()
    for _ in range(2):
        _, rg = P.perk_step(Ug, 0.0, dt, fam, pm, semi, P.PerkStepOptions(relaxation=rx))
        _, ro = orc.perk_step(Uo, 0.0, dt, fam, pm.effective_level, rx)
        assert abs(rg.gamma - ro.gamma) < 1e-12
    assert rel_err(Ug, Uo, 5) < 1e-11
