"""GPU: the batched update matrix of one linear-advection P-ERK step
(perrk_update_matrix, csrc/dg_advection.cuh) against the reference's
assemble_update_matrix loop (analysis.cpp:11-32: perk_step of every unit
vector with relaxation off and gamma fixed, run through ref_shim.cpp).

Tolerance: entries are O(1); S x 1e-13 absolute for an S-stage family (FP64
statistical parity: FMA contraction and the accumulation order of volume and
face terms differ from the reference's loops, and each stage multiplies the
rounding by up to |dt J D| ~ 4 at the larger dt).  At sizes where the reference loop is slow the
size-independent properties are checked instead: linearity against the
reference's perk_step on a smooth vector, row sums 1 (constants preserved)."""
import numpy as np
import pytest

import oracle as O
from helpers import nonuniform_edges
from paper_2507_04991_b200 import perrk as P

pytestmark = pytest.mark.gpu

FAMILIES = {
    "p2": lambda: P.build_perk2(4, [4], [[0.2, 0.35]]),
    "p3": lambda: P.build_perk3_variant(7, [4, 7], [[0.3], [0.2, 0.25, 0.3, 0.35]]),
    "p4": lambda: P.build_perk4(14, [5, 8, 14], [[], [0.5] * 3, [0.7] * 9]),
}


def _levels_1d(mesh, R):
    h = np.diff(mesh.edges[0])
    raw = np.where(h < h.max(), 1, R).astype(np.int32)
    return P.make_partition_map(mesh, raw, R)


@pytest.mark.parametrize("kind", ["p2", "p3", "p4"])
@pytest.mark.parametrize("surface", ["upwind", "central", "rusanov", "ec"])
def test_update_matrix_1d_two_level_vs_reference(kind, surface):
    mesh = P.build_two_level_advection_mesh()
    fam = FAMILIES[kind]()
    pm = _levels_1d(mesh, fam.R)
    spec = P.AdvectionSpec(mesh, [1.0], surface_flux=surface)
    ref = O.RefAdvection(mesh, [1.0], surface_flux=surface)
    for dt, gamma in ((0.05, 1.0), (0.08, 0.97)):
        um = P.assemble_update_matrix(fam, pm, spec, dt, gamma)
        Dr = ref.update_matrix(fam, pm.effective_level, dt, gamma)
        assert um.D.shape == Dr.shape == (80, 80)
        assert np.abs(um.D - Dr).max() < fam.S * 1e-13


@pytest.mark.parametrize("mode,vflux", [("weak", "ec"), ("flux_differencing", "central"),
                                        ("flux_differencing", "ec")])
@pytest.mark.parametrize("velocity", [[1.0, 0.5], [-0.7, 1.3]])
def test_update_matrix_2d_vs_reference(mode, vflux, velocity):
    mesh = P.Mesh2DRect(nonuniform_edges(4, -1.0, 1.0, 3), nonuniform_edges(3, -1.0, 1.0, 4))
    fam = FAMILIES["p3"]()
    rng = np.random.default_rng(2)
    pm = P.make_partition_map(mesh, rng.integers(1, 3, mesh.num_cells()), 2)
    kw = dict(surface_flux="upwind", volume_mode=mode, volume_flux=vflux)
    um = P.assemble_update_matrix(fam, pm, P.AdvectionSpec(mesh, velocity, **kw), 0.01, 1.0)
    Dr = O.RefAdvection(mesh, velocity, **kw).update_matrix(fam, pm.effective_level, 0.01, 1.0)
    assert np.abs(um.D - Dr).max() < fam.S * 1e-13


def test_update_matrix_1d_weak_form_vs_reference():
    mesh = P.Mesh1D(nonuniform_edges(9, -2.0, 2.0, 7))
    fam = FAMILIES["p4"]()
    pm = P.make_partition_map(mesh, np.random.default_rng(4).integers(1, 4, 9), 3)
    kw = dict(surface_flux="upwind", volume_mode="weak")
    um = P.assemble_update_matrix(fam, pm, P.AdvectionSpec(mesh, [-1.5], **kw), 0.02, 1.0)
    Dr = O.RefAdvection(mesh, [-1.5], **kw).update_matrix(fam, pm.effective_level, 0.02, 1.0)
    assert np.abs(um.D - Dr).max() < fam.S * 1e-13


def test_update_matrix_2d_large_properties():
    """M = 9216 (24^2 cells): linearity against the reference's perk_step on a
    smooth vector, constants preserved, stable spectrum proxy (max |entry|)."""
    mesh = P.build_uniform_mesh2d(1.0, 24)
    fam = FAMILIES["p3"]()
    x = np.arange(24)
    raw = np.where((np.abs(x[None, :] - 11.5) < 6) | (np.abs(x[:, None] - 11.5) < 6), 1, 2)
    pm = P.make_partition_map(mesh, raw.reshape(-1), 2)
    spec = P.AdvectionSpec(mesh, [1.0, 0.5])
    um = P.assemble_update_matrix(fam, pm, spec, 0.004, 1.0)
    M = spec.num_dofs()
    assert um.D.shape == (M, M)
    ref = O.RefAdvection(mesh, [1.0, 0.5])
    u = np.cos(np.linspace(0, 6 * np.pi, M)) + 0.1 * np.sin(np.linspace(0, 40, M))
    v = u.copy()
    ref.perk_step(v, 0.0, 0.004, fam, pm.effective_level, None, gamma_override=1.0)
    assert np.abs(um.D @ u - v).max() < 1e-12
    assert np.abs(um.D.sum(axis=1) - 1.0).max() < 1e-12
