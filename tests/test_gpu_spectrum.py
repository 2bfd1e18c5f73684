"""GPU: spectrum probing for family design: the
device RHS's Jacobian by central differences, compressed by cell colouring,
against the reference's own procedure (specopt.cpp:18-35, dense column by
column) on the unmodified reference RHS."""
import numpy as np
import pytest

import oracle as O
from helpers import mesh2d, mesh3d, smooth_state
from paper_2507_04991_b200 import perrk as P
from paper_2507_04991_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _ref_jacobian(ref, U, eps=1e-7):
    M = U.size
    J = np.zeros((M, M))
    u = U.copy()
    for j in range(M):
        h = eps * (1.0 + abs(U[j]))
        u[j] = U[j] + h
        fp = ref.rhs(0.0, u)
        u[j] = U[j] - h
        fm = ref.rhs(0.0, u)
        u[j] = U[j]
        J[:, j] = (fp - fm) / (2.0 * h)
    return J


def test_colored_device_jacobian_vs_reference_probe():
    mesh = mesh2d(6, 6, seed=101)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh, surface_flux="hlle"))
    U = smooth_state((semi.node_x(), semi.node_y()), 2, seed=5, amp=0.2)
    Jg = P.probe_jacobian(semi, U)                  # 2 x 4 colours x 64 RHS pairs
    Jr = _ref_jacobian(O.Ref(mesh, surface_flux="hlle"), U)
    scale = np.abs(Jr).max()
    assert np.abs(Jg - Jr).max() < 1e-6 * scale    # central differences at eps 1e-7
    eg = P.clean_spectrum(np.linalg.eigvals(Jg))
    er = P.clean_spectrum(np.linalg.eigvals(Jr))
    assert abs(np.abs(eg).max() - np.abs(er).max()) < 1e-6 * np.abs(er).max()
    assert abs(eg.real.min() - er.real.min()) < 1e-6 * np.abs(er).max()
    assert abs(np.abs(eg.imag).max() - np.abs(er.imag).max()) < 1e-6 * np.abs(er).max()


def test_probed_spectrum_supports_the_c1_family_at_its_cfl():
    """The probed C1 spectrum with the C1 family: |P(dt lambda)| ~ 1 at the
    CFL step the config uses (the isentropic vortex runs 100 steps stably)."""
    cfg = W.make_config("c1")
    mesh = P.build_uniform_mesh2d(10.0, 6)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh))
    U = np.ascontiguousarray(W.isentropic_vortex(W.VortexParams(), semi.node_x(),
                                                 semi.node_y()).T).reshape(-1)
    eigs = P.probe_spectrum(semi, U)
    dt = P.compute_dt(U, semi, P.IntegratorConfig(time=P.TimeControl(False, 0.0,
                                                                      P.CflRamp(0.9, 0.9))), 0.0)
    margin = P.stability_margin(cfg.family, eigs, dt)
    assert margin[0] < 1.0 + 1e-2


def _single_column(semi, U, j, eps):
    """specopt.cpp:25-32 for one column, through the device RHS."""
    h = eps * (1.0 + abs(U[j]))
    up, um = U.copy(), U.copy()
    up[j] = U[j] + h
    um[j] = U[j] - h
    return (semi.rhs(0.0, up) - semi.rhs(0.0, um)) / (2.0 * h)


def _nsf(mesh):
    return P.Semidiscretization(P.SemidiscretizationSpec(mesh, physics="nsf", mu=2e-2,
                                                         prandtl=0.72, surface_flux="hlle"))


@pytest.mark.parametrize("case", ["2d", "3d", "nsf"])
def test_device_probe_equals_single_column_probes_bitwise(case):
    """perrk_probe_jacobian (include/perrk_b200.h): each coloured column equals
    the reference's one-column-at-a-time probe on the same RHS bit for bit,
    and the colour count is independent of the column count."""
    if case == "3d":
        from helpers import mesh3d
        semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh3d(3, 2, 2, seed=9)))
        U = smooth_state((semi.node_x(), semi.node_y(), semi.node_z()), 3, seed=6, amp=0.2)
    else:
        mesh = mesh2d(7, 6, seed=8)
        semi = _nsf(mesh) if case == "nsf" else \
            P.Semidiscretization(P.SemidiscretizationSpec(mesh, surface_flux="hlle"))
        U = smooth_state((semi.node_x(), semi.node_y()), 2, seed=6, amp=0.2)
    eps = 1e-6
    J, ncol = semi.probe_jacobian(U, 0.0, eps, return_colours=True)
    assert J.shape == (U.size, U.size)
    assert ncol < semi.num_cells() or case == "3d"
    cols = np.random.default_rng(3).choice(U.size, 12, replace=False)
    for j in cols:
        assert np.array_equal(J[:, j], _single_column(semi, U, j, eps)), j
    # same matrix as the host-driven coloured probe
    assert np.array_equal(J, P.probe_jacobian(semi, U, 0.0, eps, device=False))


def test_device_probe_guard():
    mesh = mesh2d(10, 9, seed=2)  # 90 cells x 64 DOFs > 5000
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh))
    U = smooth_state((semi.node_x(), semi.node_y()), 2, seed=1)
    with pytest.raises(P.Error):
        semi.probe_jacobian(U)


def _envelope(e):
    e = np.asarray(e)
    return np.array([np.abs(e).max(), e.real.min(), np.abs(e.imag).max()])


@pytest.mark.parametrize("surface", ["rusanov", "hlle"])
def test_krylov_full_space_equals_dense_probe(surface):
    """perrk_krylov_hessenberg (matrix-free Arnoldi on the RHS's central-
    difference JVP) run to the full space (m = M) on a
    small mesh: its Ritz values are the probed Jacobian's eigenvalues, so the
    spectral envelope (max |lambda|, min Re lambda, max |Im lambda|) equals
    the dense probe's (specopt.cpp:18-35 procedure) to 1e-6."""
    mesh = mesh2d(3, 3, seed=41)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh, surface_flux=surface))
    U = smooth_state((semi.node_x(), semi.node_y()), 2, seed=9, amp=0.2)
    M = U.size
    dense = P.probe_spectrum(semi, U)
    ritz = P.krylov_spectrum(semi, U, m=M)
    ed, ek = _envelope(dense), _envelope(ritz)
    assert np.abs(ek - ed).max() < 1e-6 * ed[0], (ek, ed)


def test_krylov_masked_is_the_level_block():
    """cell_mask restricts the operator to the flagged cells: the Ritz values
    of the full masked space are the eigenvalues of the dense Jacobian's
    block on those cells' DOFs."""
    mesh = mesh2d(4, 3, seed=43)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh, surface_flux="rusanov"))
    U = smooth_state((semi.node_x(), semi.node_y()), 2, seed=10, amp=0.2)
    mask = np.zeros(mesh.num_cells(), np.int8)
    mask[[0, 1, 5, 6, 10]] = 1
    J = P.probe_jacobian(semi, U)
    stride = 16 * 4
    idx = np.concatenate([np.arange(c * stride, (c + 1) * stride) for c in np.nonzero(mask)[0]])
    ed = _envelope(P.clean_spectrum(np.linalg.eigvals(J[np.ix_(idx, idx)])))
    ek = _envelope(P.krylov_spectrum(semi, U, m=idx.size, cell_mask=mask))
    assert np.abs(ek - ed).max() < 1e-6 * ed[0], (ek, ed)


def test_krylov_envelope_3d_partial_space():
    """A partial Krylov space (m << M) on a 3D mesh: the Ritz spectral radius
    approaches the dense probe's as m grows (Arnoldi resolves the extreme
    eigenvalues first); checked on a 3D mesh the dense probe can still take
    (M = 2560).  Ritz values of a non-normal operator lie in its field of
    values, so they may slightly overshoot the spectrum."""
    mesh = mesh3d(2, 2, 2, seed=44)
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh, surface_flux="rusanov"))
    U = smooth_state((semi.node_x(), semi.node_y(), semi.node_z()), 3, seed=11, amp=0.2)
    rho_dense = np.abs(P.probe_spectrum(semi, U)).max()
    r = [np.abs(P.krylov_spectrum(semi, U, m=m)).max() for m in (60, 200)]
    print({"rho_dense": rho_dense, "ritz_rho_m60": r[0], "ritz_rho_m200": r[1]})
    # measured: 1.5e-7 (m = 60) and 2.8e-7 (m = 200) relative, the
    # central-difference noise of the two probes
    for x in r:
        assert abs(x - rho_dense) < 1e-5 * rho_dense
