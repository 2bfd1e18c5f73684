"""GPU: the element-slab decomposition's device path on ONE GPU.

perrk_loopback_group makes n contexts on one device ranks 0..n-1 of a slab
decomposition sharing one stream: per stage every rank packs its boundary
traces, the halo and the reduction gathers are stream-ordered device copies
(the data movement NcclExchange does with ncclSend/Recv and ncclAllGather),
and every kernel of the multi-rank path runs (ghost traces in the stage
kernel, stash/combine reductions, global positivity codes).  The
concatenated slabs must reproduce the single-context run.  Tolerance: the
reductions are regrouped by slab, so 1e-13 relative (not bitwise)."""
import numpy as np
import pytest

from helpers import mesh2d, mesh3d, rel_err, smooth_state
from paper_2507_04991_b200 import perrk as P

pytestmark = pytest.mark.gpu


def _run(semis, fam, pm, U0, steps, cfl, relax, cuts=None):
    for s in semis:
        s._use_family(fam, pm)
    rc = P.IntegratorConfig(tf=1e30, time=P.TimeControl(False, 0.0, P.CflRamp(cfl, cfl)),
                            relaxation=relax)
    npc, V = semis[0].nodes_per_cell(), semis[0].num_vars()
    lc = semis[0].global_num_cells() // semis[0].spec.mesh.shape()[-1]
    cells = U0.reshape(-1, npc, V)
    for s in semis:
        b, e = s.slab_range()
        s.upload(np.ascontiguousarray(cells[b * lc:e * lc]).reshape(-1))
    t, taken, aborted, recs = P.advance(semis[0], fam, pm, rc, 0.0, steps)
    assert taken == steps and not aborted
    U = np.concatenate([s.download() for s in semis])
    return U, recs


@pytest.mark.parametrize("dim,nranks", [(2, 2), (2, 3), (3, 2), (3, 4)])
def test_loopback_slabs_reproduce_single_domain(dim, nranks):
    if dim == 2:
        mesh = mesh2d(10, 12, seed=71)
        fam = P.build_perk3_variant(7, [4, 7], [[0.3], [0.2, 0.25, 0.3, 0.35]])
        coords = lambda s: (s.node_x(), s.node_y())
    else:
        mesh = mesh3d(5, 4, 8, seed=72)
        fam = P.build_perk4(14, [5, 8, 14], [[], [0.5] * 3, [0.7] * 9])
        coords = lambda s: (s.node_x(), s.node_y(), s.node_z())
    rng = np.random.default_rng(5)
    pm = P.make_partition_map(mesh, rng.integers(1, fam.R + 1, mesh.num_cells()), fam.R)
    spec = P.SemidiscretizationSpec(mesh, surface_flux="hlle")
    one = P.Semidiscretization(spec)
    U0 = smooth_state(coords(one), dim, seed=31, amp=0.25)
    relax = P.RelaxationConfig(numerics="accurate")
    U1, r1 = _run([one], fam, pm, U0, 6, 0.3, relax)
    semis = [P.Semidiscretization(spec) for _ in range(nranks)]
    P.loopback_group(semis)
    # the slab geometry is the global geometry's layers
    gx = one.node_x().reshape(-1, one.nodes_per_cell())
    lc = mesh.num_cells() // mesh.shape()[-1]
    for s in semis:
        b, e = s.slab_range()
        assert np.array_equal(s.node_x(), gx[b * lc:e * lc].reshape(-1))
    Un, rn = _run(semis, fam, pm, U0, 6, 0.3, relax)
    assert rel_err(Un, U1, dim + 2) < 1e-13
    g1 = np.array([r.gamma for r in r1])
    gn = np.array([r.gamma for r in rn])
    assert np.abs(g1 - gn).max() < 1e-13
    assert np.abs(np.array([r.entropy for r in r1]) - np.array([r.entropy for r in rn])).max() \
        < 1e-13 * max(1.0, abs(r1[0].entropy))
    assert abs(rn[-1].t - r1[-1].t) < 1e-14


def test_loopback_slab_positivity_reports_global_cell():
    mesh = mesh3d(4, 4, 6, seed=73)
    fam = P.build_perk2(4, [4], [[0.2, 0.35]])
    pm = P.make_partition_map(mesh, np.ones(mesh.num_cells(), np.int32), 1)
    spec = P.SemidiscretizationSpec(mesh)
    one = P.Semidiscretization(spec)
    U0 = smooth_state((one.node_x(), one.node_y(), one.node_z()), 3, seed=2, amp=0.2)
    bad = 4 * 4 * 4 + 5  # a cell in layer 4 (rank 1 of 2)
    U0.reshape(-1, 64, 5)[bad, 7, 0] = -1.0
    semis = [P.Semidiscretization(spec) for _ in range(2)]
    P.loopback_group(semis)
    lc = 16
    for s in semis:
        s._use_family(fam, pm)
        b, e = s.slab_range()
        s.upload(np.ascontiguousarray(U0.reshape(-1, 64, 5)[b * lc:e * lc]).reshape(-1))
    t, res = P.perk_step_resident(0.0, 0.01, fam, pm, semis[0], P.PerkStepOptions())
    assert res.aborted and res.bad_cell == bad and res.bad_stage == 0
    Ud = np.concatenate([s.download() for s in semis])
    assert np.array_equal(Ud, U0)  # untouched on abort
