"""CPU: pin the oracle before trusting it.

The C restatement (oracle/perrk_oracle.c, `Orc`) is checked against
  * the reference's own known-answer and property tests (SURVEY.md 8c —
    the reference has no golden files; its pins are analytic values and
    invariants), restated here against both libraries:
      logmean            test_physics.cpp:42-61
      GLL k=3            test_basis.cpp:9-68
      flux consistency / EC symmetry / Tadmor   test_physics.cpp:121-187
      free stream, EC <w, rhs>, conservation     test_dg.cpp:62-200
      partition union                           test_dg.cpp:302-346
      H quadrature, relaxation roots            test_relax.cpp:63-248
  * the unmodified reference library itself (oracle/_ref, `Ref`), for the 2D
    RHS, reductions and P-ERRK steps: bit for bit where the restatement keeps
    the reference's operation order (both built -ffp-contract=off);
  * the committed golden fixtures under tests/golden/ (made from `Ref` by
    tests/golden/make_golden.py), so the pins hold where /root/reference is
    absent.
3D and 2D Navier-Stokes are oracle extensions (no reference counterpart);
they are pinned by reduction to the 2D reference (z-constant data) and by
the same invariants.
"""
import math
import os

import numpy as np
import pytest

import oracle as O
from conftest import HAS_REF_LIB
from helpers import mesh2d, mesh3d, smooth_state
from paper_2507_04991_b200 import perrk as P
from paper_2507_04991_b200 import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
need_ref = pytest.mark.skipif(not HAS_REF_LIB, reason="oracle/_ref not built")
_D = O.C.POINTER(O.C.c_double)


def libs():
    out = [("orc", O.orc_lib())]
    if HAS_REF_LIB:
        out.append(("ref", O.ref_lib()))
    return out


# --------------------------------------------------------------------------- pointwise
@pytest.mark.parametrize("name,L", libs())
def test_logmean_known_answers(name, L):
    lm = L.ref_logmean if name == "ref" else L.orc_logmean
    for a in (0.3, 1.0, 7.5):
        assert lm(a, a) == a
    assert abs(lm(1.0, math.e) - (math.e - 1.0)) < 1e-14
    rng = np.random.default_rng(5)
    for _ in range(1000):
        a, b = rng.uniform(0.1, 10.0, 2)
        m = lm(a, b)
        assert min(a, b) - 1e-14 <= m <= max(a, b) + 1e-14
        d = b - a
        if abs(d) > 1e-8:
            assert abs(m - d / math.log1p(d / a)) < 1e-13 * max(a, b)


@pytest.mark.parametrize("name,L", libs())
def test_gll_k3(name, L):
    x, w, D = np.zeros(4), np.zeros(4), np.zeros(16)
    (L.ref_gll if name == "ref" else L.orc_gll)(3, O.dp(x), O.dp(w), O.dp(D))
    s5 = 1.0 / math.sqrt(5.0)
    assert np.allclose(x, [-1, -s5, s5, 1], atol=1e-15)
    assert np.allclose(w, [1 / 6, 5 / 6, 5 / 6, 1 / 6], atol=1e-15)
    D = D.reshape(4, 4)
    Q = np.diag(w) @ D
    B = np.zeros((4, 4))
    B[0, 0], B[-1, -1] = -1.0, 1.0
    assert np.abs(Q + Q.T - B).max() < 1e-13          # SBP
    assert np.abs(D @ x ** 3 - 3 * x ** 2).max() < 1e-12  # exact to degree 3


def _random_state(rng, dim, gamma=1.4):
    rho = rng.uniform(0.5, 2.0)
    v = rng.uniform(-1.0, 1.0, dim)
    p = rng.uniform(0.5, 2.0)
    return np.array([rho, *(rho * v), p / (gamma - 1) + 0.5 * rho * v @ v])


@pytest.mark.parametrize("name,L", libs())
@pytest.mark.parametrize("dim", [2, 3])
def test_fluxes_consistency_symmetry_tadmor(name, L, dim):
    if name == "ref" and dim == 3:
        pytest.skip("the reference is 2D")
    nf = L.ref_numerical_flux if name == "ref" else L.orc_numerical_flux
    pe = L.ref_physics_eval if name == "ref" else L.orc_physics_eval
    rng = np.random.default_rng(7 + dim)
    V = dim + 2
    for _ in range(500):
        ul, ur = _random_state(rng, dim), _random_state(rng, dim)
        d = int(rng.integers(0, dim))
        f, w, lam = np.zeros(V), np.zeros(V), np.zeros(1)
        s = O.C.c_double()
        pe(dim, 1.4, O.dp(ul), d, O.dp(f), O.dp(w), O.C.byref(s), O.dp(lam))
        for tag in (0, 2, 3, 4, 5):
            fs = np.zeros(V)
            assert nf(dim, 1.4, tag, O.dp(ul), O.dp(ul), d, O.dp(fs)) == 0
            assert np.abs(fs - f).max() < 1e-14 * max(1.0, np.abs(f).max())
        fa, fb = np.zeros(V), np.zeros(V)
        nf(dim, 1.4, 5, O.dp(ul), O.dp(ur), d, O.dp(fa))
        nf(dim, 1.4, 5, O.dp(ur), O.dp(ul), d, O.dp(fb))
        assert np.abs(fa - fb).max() < 1e-13 * max(1.0, np.abs(fa).max())
        # Tadmor (test_physics.cpp:20-38): <w_R - w_L, f*> = Psi_R - Psi_L with
        # the flux potential Psi = <w, f(u)> - s v_d
        def potential(u):
            f_, w_, lam_ = np.zeros(V), np.zeros(V), np.zeros(1)
            s_ = O.C.c_double()
            pe(dim, 1.4, O.dp(u), d, O.dp(f_), O.dp(w_), O.C.byref(s_), O.dp(lam_))
            return w_ @ f_ - s_.value * u[1 + d] / u[0], w_
        pr, wr = potential(ur)
        pl, wl = potential(ul)
        psi = pr - pl
        assert abs((wr - wl) @ fa - psi) < 1e-11


def test_entropy_difference_matches_plain_difference():
    L = O.orc_lib()
    rng = np.random.default_rng(3)
    for dim in (2, 3):
        V = dim + 2
        for _ in range(200):
            u = _random_state(rng, dim)
            du = 1e-3 * rng.standard_normal(V) * np.abs(u)
            f, w, lam = np.zeros(V), np.zeros(V), np.zeros(1)
            s0, s1 = O.C.c_double(), O.C.c_double()
            L.orc_physics_eval(dim, 1.4, O.dp(u), 0, O.dp(f), O.dp(w), O.C.byref(s0), O.dp(lam))
            u1 = u + du
            L.orc_physics_eval(dim, 1.4, O.dp(u1), 0, O.dp(f), O.dp(w), O.C.byref(s1), O.dp(lam))
            ds = L.orc_entropy_difference(dim, 1.4, O.dp(u), O.dp(du))
            assert abs(ds - (s1.value - s0.value)) < 1e-12 * max(1.0, abs(s0.value))


# --------------------------------------------------------------------------- semidiscretization
def _orc_state(orc, seed=7, amp=0.3):
    x, y, z, _ = orc.node_coords()
    return smooth_state((x, y, z) if orc.dim == 3 else (x, y), orc.dim, seed=seed, amp=amp)


@need_ref
@pytest.mark.parametrize("surface", ["rusanov", "hlle", "hllc", "ec", "central"])
def test_orc_rhs_bitwise_equals_reference_2d(surface):
    mesh = mesh2d(7, 6, seed=2)
    orc, ref = O.Orc(mesh, surface_flux=surface), O.Ref(mesh, surface_flux=surface)
    U = _orc_state(orc, seed=4)
    assert np.array_equal(orc.rhs(0.0, U), ref.rhs(0.0, U))
    mask = np.random.default_rng(1).integers(0, 2, orc.ncells).astype(np.int8)
    assert np.array_equal(orc.rhs_masked(0.0, U, mask), ref.rhs_masked(0.0, U, mask))


@need_ref
@pytest.mark.parametrize("mode,vflux", [("weak", "ec"), ("flux_differencing", "central")])
@pytest.mark.parametrize("surface", ["rusanov", "hllc", "central"])
def test_orc_volume_variants_bitwise_equal_reference_2d(mode, vflux, surface):
    """Weak form (semidisc.cpp:429-445) and central flux differencing."""
    mesh = mesh2d(6, 5, seed=12)
    kw = dict(surface_flux=surface, volume_mode=mode, volume_flux=vflux)
    orc, ref = O.Orc(mesh, **kw), O.Ref(mesh, **kw)
    U = _orc_state(orc, seed=14)
    assert np.array_equal(orc.rhs(0.0, U), ref.rhs(0.0, U))


def test_orc_volume_variants_agree_on_smooth_data_3d():
    """The three volume forms are consistent discretisations of the same
    divergence: on a smooth state they agree to the discretisation error,
    and on the free stream all vanish."""
    mesh = mesh3d(3, 3, 3, seed=15)
    outs = []
    for mode, vflux in (("flux_differencing", "ec"), ("flux_differencing", "central"),
                        ("weak", "ec")):
        orc = O.Orc(mesh, surface_flux="rusanov", volume_mode=mode, volume_flux=vflux)
        n = orc.ndofs // orc.V
        Uf = np.tile([1.0, 0.5, -0.25, 0.125, 3.0], n)
        assert np.abs(orc.rhs(0.0, Uf)).max() < 1e-12
        outs.append(orc.rhs(0.0, _orc_state(orc, 16, amp=0.05)))
    scale = np.abs(outs[0]).max()
    for o in outs[1:]:
        assert np.abs(o - outs[0]).max() < 0.2 * scale


@need_ref
def test_orc_reductions_equal_reference_2d():
    mesh = mesh2d(8, 5, seed=9)
    orc, ref = O.Orc(mesh), O.Ref(mesh)
    U, K = _orc_state(orc, 1), _orc_state(orc, 2)
    assert orc.total_entropy(U) == ref.total_entropy(U)
    assert orc.entropy_inner_product(U, K) == ref.entropy_inner_product(U, K)
    assert np.array_equal(orc.integral_per_variable(U), ref.integral_per_variable(U))
    assert np.array_equal(orc.characteristic_speed(U), ref.characteristic_speed(U))
    assert orc.compute_dt(U, False, 0.7) == ref.compute_dt(U, False, 0.7)


@need_ref
@pytest.mark.parametrize("kind", ["p2", "p3", "p4"])
def test_orc_perk_steps_equal_reference_2d(kind):
    mesh = mesh2d(6, 6, seed=13)
    fam = {"p2": lambda: P.build_perk2(4, [4], [[0.2, 0.35]]),
           "p3": lambda: P.build_perk3_variant(7, [4, 7], [[0.3], [0.2, 0.25, 0.3, 0.35]]),
           "p4": lambda: P.build_perk4(14, [5, 8, 14], [[], [0.5] * 3, [0.7] * 9])}[kind]()
    rng = np.random.default_rng(2)
    pm = P.make_partition_map(mesh, rng.integers(1, fam.R + 1, mesh.num_cells()), fam.R)
    orc, ref = O.Orc(mesh, surface_flux="hlle"), O.Ref(mesh, surface_flux="hlle")
    U0 = _orc_state(orc, 3, amp=0.2)
    dt = 0.3 * ref.compute_dt(U0, False, 1.0)
    Uo, Ur = U0.copy(), U0.copy()
    rx = P.RelaxationConfig()
    to = tr = 0.0
    for _ in range(4):
        to, ro = orc.perk_step(Uo, to, dt, fam, pm.effective_level, rx)
        tr, rr = ref.perk_step(Ur, tr, dt, fam, pm.effective_level, rx)
        assert ro.gamma == rr.gamma and ro.iterations == rr.iterations
        assert ro.fell_back == rr.fell_back and ro.delta_h == rr.delta_h
    assert np.array_equal(Uo, Ur) and to == tr
    assert orc.rhs_cell_evaluations() == ref.rhs_cell_evaluations()


def test_free_stream_ec_and_conservation_orc():
    for dim, mesh in ((2, mesh2d(6, 5, seed=3)), (3, mesh3d(4, 3, 3, seed=4))):
        orc = O.Orc(mesh, surface_flux="ec")
        n = orc.ndofs // orc.V
        U = np.tile([1.0, 1.0, -0.5] + ([0.25] if dim == 3 else []) + [4.0], n)
        assert np.abs(orc.rhs(0.0, U)).max() < 1e-11
        U = _orc_state(orc, 5)
        r = orc.rhs(0.0, U)
        assert abs(orc.entropy_inner_product(U, r)) < 1e-11
        assert np.abs(orc.integral_per_variable(r)).max() < 5e-12


def test_partition_union_orc_3d():
    mesh = mesh3d(4, 4, 3, seed=8)
    orc = O.Orc(mesh)
    U = _orc_state(orc, 6)
    full = orc.rhs(0.0, U)
    lv = np.random.default_rng(3).integers(1, 3, orc.ncells)
    r1 = orc.rhs_masked(0.0, U, (lv == 1).astype(np.int8))
    r2 = orc.rhs_masked(0.0, U, (lv == 2).astype(np.int8))
    assert np.all((r1 == 0) | (r2 == 0))
    assert np.array_equal(r1 + r2, full)


def _embed_2d(U2, axes, n_other):
    """2D state [J][I][iy][ix][4] -> 3D [K][J3][I3][iz][iy][ix][5] on the
    axis pair `axes` (2D x -> axes[0], 2D y -> axes[1]), constant along the
    third axis (n_other cells), zero velocity along it."""
    J, I = U2.shape[:2]
    a, b = axes
    other = 3 - a - b
    # 3D [cell z][cell y][cell x][iz][iy][ix]; place (cell, node) axes of the pair
    cells = [None, None, None]  # per 3D axis: ("J"|"I"|"other")
    cells[a], cells[b], cells[other] = "I", "J", "O"
    sizes = {"I": I, "J": J, "O": n_other}
    shape = (sizes[cells[2]], sizes[cells[1]], sizes[cells[0]], 4, 4, 4)
    U3 = np.zeros(shape + (5,))
    # index grids of the 3D array
    kz, ky, kx, iz, iy, ix = np.indices(shape)
    cidx = {0: kx, 1: ky, 2: kz}
    nidx = {0: ix, 1: iy, 2: iz}
    src = U2[cidx[b], cidx[a], nidx[b], nidx[a]]  # [..., 4]
    U3[..., 0] = src[..., 0]
    U3[..., 1 + a] = src[..., 1]
    U3[..., 1 + b] = src[..., 2]
    U3[..., 4] = src[..., 3]
    return U3, (cidx, nidx)


@need_ref
@pytest.mark.parametrize("axes", [(0, 1), (0, 2), (1, 2), (2, 0)])
def test_3d_reduces_to_reference_2d_on_each_axis_pair(axes):
    """Oracle extension pin (semidisc.cpp:446-556 extended to 3D): 2D data on
    the axis pair `axes`, constant along the third axis with zero velocity
    there, gives the 2D reference RHS on that pair and a zero RHS for the
    third momentum.  The (x,z), (y,z) and (z,x) pairs carry real z-line and
    z-face terms (the (x,y) pair alone would leave them identically zero)."""
    m2 = mesh2d(5, 4, seed=21)
    ref = O.Ref(m2)
    edges = [None, None, None]
    a, b = axes
    edges[a], edges[b] = list(m2.x_edges), list(m2.y_edges)
    other = 3 - a - b
    edges[other] = [0.0, 0.7, 1.5, 2.0]
    orc3 = O.Orc(P.Mesh3DRect(*edges))
    x2, y2, _, _ = ref.node_coords()
    U2 = smooth_state((x2, y2), 2, seed=8)
    J, I = m2.ny(), m2.nx()
    U2g = U2.reshape(J, I, 4, 4, 4)
    U3, (cidx, nidx) = _embed_2d(U2g, axes, 3)
    r3 = orc3.rhs(0.0, U3.reshape(-1)).reshape(U3.shape)
    r2 = ref.rhs(0.0, U2).reshape(J, I, 4, 4, 4)
    r2e = r2[cidx[b], cidx[a], nidx[b], nidx[a]]
    scale = np.abs(r2).max()
    for v, v3 in ((0, 0), (1, 1 + a), (2, 1 + b), (3, 4)):
        assert np.abs(r3[..., v3] - r2e[..., v]).max() < 1e-12 * scale, (axes, v)
    assert np.abs(r3[..., 1 + other]).max() < 1e-12 * scale


# --------------------------------------------------------------------------- relaxation
@need_ref
def test_relaxation_reference_numerics_equal_reference():
    cfg = W.make_config("c1")
    orc, ref = O.Orc(cfg.mesh), O.Ref(cfg.mesh)
    x, y, _, _ = ref.node_coords()
    U0 = W.initial_state_for(cfg, (x, y, None))
    eff = cfg.partition_map().effective_level
    Uo, Ur = U0.copy(), U0.copy()
    _, no, lo, _ = orc.run_steps(Uo, 0.0, 20, cfg.family, eff, P.RelaxationConfig(), False, 0.9)
    _, nr, lr, _ = ref.run_steps(Ur, 0.0, 20, cfg.family, eff, P.RelaxationConfig(), False, 0.9)
    assert no == nr == 20
    assert np.array_equal(lo[:, :lr.shape[1]], lr) and np.array_equal(Uo, Ur)


def test_accurate_relaxation_is_order_insensitive():
    """H1: the accurate numerics make gamma insensitive to 1e-16 input
    perturbations."""
    mesh = mesh2d(16, 16, seed=3)
    orc = O.Orc(mesh)
    U0 = _orc_state(orc, 12, amp=0.4)
    fam = P.build_perk2(4, [4], [[0.2, 0.35]])
    eff = np.ones(orc.ncells, np.int32)
    rx = P.RelaxationConfig(numerics="accurate")
    Ua = U0.copy()
    Ub = U0 * (1.0 + 1e-16 * np.random.default_rng(1).standard_normal(U0.size))
    _, na, la, _ = orc.run_steps(Ua, 0.0, 10, fam, eff, rx, False, 0.45)
    _, nb, lb, _ = orc.run_steps(Ub, 0.0, 10, fam, eff, rx, False, 0.45)
    assert na == nb == 10
    assert np.abs(la[:, 2] - lb[:, 2]).max() < 1e-13
    assert la[:, 5].sum() == 0  # never falls back


# --------------------------------------------------------------------------- golden fixtures
def _golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated")
    return np.load(path)


def test_golden_rhs_c1_and_random():
    g = _golden("rhs_2d.npz")
    cfg = W.make_config("c1")
    orc = O.Orc(cfg.mesh)
    assert np.array_equal(orc.rhs(0.0, g["U_c1"]), g["rhs_c1"])
    m = P.Mesh2DRect(g["xe"], g["ye"])
    for surface in ("rusanov", "hlle", "hllc", "ec", "central"):
        o = O.Orc(m, surface_flux=surface)
        assert np.array_equal(o.rhs(0.0, g["U_rand"]), g[f"rhs_rand_{surface}"])


def test_golden_c1_run_reference_relaxation():
    g = _golden("c1_run.npz")
    cfg = W.make_config("c1")
    orc = O.Orc(cfg.mesh)
    U = g["U0"].copy()
    n = int(g["steps"])
    _, taken, log, _ = orc.run_steps(U, 0.0, n, cfg.family, cfg.partition_map().effective_level,
                                     P.RelaxationConfig(), False, 0.9)
    assert taken == n
    assert np.array_equal(log[:, :g["log"].shape[1]], g["log"])
    assert np.array_equal(U, g["U"])


def test_golden_family_text_roundtrip():
    g = _golden("families.npz")
    for key in ("p2", "p3", "p4"):
        fam = P.family_from_text(str(g[f"text_{key}"]))
        assert np.array_equal(fam.A, g[f"A_{key}"])
        assert np.array_equal(fam.b, g[f"b_{key}"])
        assert np.array_equal(fam.c, g[f"c_{key}"])


# --------------------------------------------------------------------------- the reference's own suites
REF_TESTS = ["test_basis", "test_butcher", "test_dg", "test_mesh", "test_physics", "test_relax"]


@pytest.mark.parametrize("name", REF_TESTS)
def test_reference_own_suite_passes(name):
    """The reference's Eigen-free doctest suites (proj/tests), compiled against
    oracle/_ref through oracle/doctest_shim, pass: the checker library is
    the reference as its authors test it."""
    import subprocess
    exe = os.path.join(os.path.dirname(O.REF_LIB), name)
    if not os.path.exists(exe):
        pytest.skip("reference test binaries not built (make -C oracle ref-tests)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "failed: 0" in r.stdout


@need_ref
@pytest.mark.parametrize("surface", ["rusanov", "hlle"])
def test_orc_nsf2d_reduces_to_reference_nsf1d(surface):
    """Oracle extension pin (2D NSF + BR1): on y-independent data with v = 0
    the 2D RHS equals the reference's own 1D NSF + BR1 RHS (NSFPhysics,
    semidisc.cpp:245-395) in (rho, m_x, E), with a zero y-momentum RHS."""
    xe = nonuniform = np.cumsum(np.r_[0.0, np.random.default_rng(4).uniform(0.5, 1.5, 9)])
    xe = list(xe / xe[-1] * 2.0 - 1.0)
    ref = O.RefNSF1D(xe, mu=2e-2, surface_flux=surface)
    x1 = ref.node_coords()
    rho = 1.0 + 0.2 * np.sin(np.pi * x1)
    vx = 0.3 * np.cos(np.pi * x1)
    p = 1.0 + 0.25 * np.sin(2 * np.pi * x1 + 0.3)
    U1 = np.stack([rho, rho * vx, p / 0.4 + 0.5 * rho * vx * vx]).T.reshape(-1)
    r1 = ref.rhs(0.0, U1).reshape(-1, 4, 3)            # [cell][node][var]
    m2 = P.Mesh2DRect(xe, [0.0, 0.5, 1.2, 2.0])
    orc = O.Orc(m2, surface_flux=surface, viscous=True, mu=2e-2, prandtl=0.72)
    nx, ny = 9, 3
    u1 = U1.reshape(nx, 4, 3)
    U2 = np.zeros((ny, nx, 4, 4, 4))                   # [cj][ci][iy][ix][v]
    for v, v2 in ((0, 0), (1, 1), (2, 3)):
        U2[..., v2] = u1[None, :, None, :, v]
    r2 = orc.rhs(0.0, U2.reshape(-1)).reshape(U2.shape)
    scale = np.abs(r1).max()
    for v, v2 in ((0, 0), (1, 1), (2, 3)):
        assert np.abs(r2[..., v2] - r1.reshape(nx, 4, 3)[None, :, None, :, v]).max() < 1e-12 * scale
    assert np.abs(r2[..., 2]).max() < 1e-12 * scale


@need_ref
def test_step_log_csv_matches_reference_writer(tmp_path):
    """write_step_log_csv (stepper.cpp:267-301): the same file bytes."""
    import types
    rng = np.random.default_rng(2)
    log = [P.StepRecord(k + 1, *rng.standard_normal(3), int(rng.integers(0, 5)),
                        float(rng.standard_normal()), rng.standard_normal(4), bool(k % 2))
           for k in range(7)]
    semi = types.SimpleNamespace(num_vars=lambda: 4, dim=lambda: 2)
    ours = tmp_path / "ours.csv"
    P.write_step_log_csv(log, semi, str(ours))
    ref = O.Ref(mesh2d(3, 3, seed=1))
    rows = np.array([[r.step, r.t, r.dt, r.gamma, r.newton_iters, r.entropy, float(r.fell_back),
                      *r.invariants] for r in log])
    theirs = tmp_path / "ref.csv"
    assert ref.L.ref_write_step_log(ref.h, len(log), O.dp(np.ascontiguousarray(rows)),
                                    str(theirs).encode()) == 0
    assert ours.read_bytes() == theirs.read_bytes()


# --------------------------------------------------------------------------- update matrix
@need_ref
@pytest.mark.parametrize("surface", ["upwind", "central"])
def test_reference_update_matrix_properties(surface):
    """The reference's assemble_update_matrix loop (analysis.cpp:11-32 via
    ref_shim.cpp) is the oracle for perrk_update_matrix.  Pins: linearity
    (D u = perk_step(u)), constants preserved (row sums 1), and for the upwind
    surface flux at a stable dt a spectral radius <= 1."""
    mesh = P.build_two_level_advection_mesh()
    ref = O.RefAdvection(mesh, [1.0], surface_flux=surface)
    fam = P.build_perk3_variant(7, [4, 7], [[0.3], [0.2, 0.25, 0.3, 0.35]])
    pm = P.make_partition_map(mesh, [2] * 6 + [1] * 8 + [2] * 6, 2)
    dt = 0.05
    D = ref.update_matrix(fam, pm.effective_level, dt, 1.0)
    x = np.asarray(mesh.edges[0])
    u = np.sin(np.linspace(0, 2 * np.pi, ref.ndofs, endpoint=False)) + 0.3
    v = u.copy()
    ref.perk_step(v, 0.0, dt, fam, pm.effective_level, None, gamma_override=1.0)
    assert np.abs(D @ u - v).max() < 1e-13
    assert np.abs(D.sum(axis=1) - 1.0).max() < 1e-13
    mn, mx, dev = P.monotonicity_metrics(D)
    assert dev < 1e-13 and mn < mx
    if surface == "upwind":
        assert P.spectral_radius(D) <= 1.0 + 1e-12
    assert x.size == 21
