"""GPU: the element partition's device path on ONE GPU.

perrk_loopback_group makes n contexts on one device ranks 0..n-1 of a
partition (uniform slabs, per-level balanced, or scattered cells) sharing one
stream: per stage every rank packs its boundary
traces, the halo and the reduction gathers are stream-ordered device copies
(the data movement NcclExchange does with ncclSend/Recv and ncclAllGather),
and every kernel of the multi-rank path runs (ghost traces in the stage
kernel, stash/combine reductions, global positivity codes).  The
ranks' cells, scattered back by their global ids, must reproduce the
single-context run.  Tolerance: the reductions are regrouped by rank, so
1e-13 relative (not bitwise)."""
import numpy as np
import pytest

from helpers import mesh2d, mesh3d, rel_err, smooth_state
from paper_2507_04991_b200 import perrk as P

pytestmark = pytest.mark.gpu


def _scatter(semis, U0):
    npc, V = semis[0].nodes_per_cell(), semis[0].num_vars()
    cells = U0.reshape(-1, npc, V)
    for s in semis:
        s.upload(np.ascontiguousarray(cells[s.local_cells()]).reshape(-1))


def _gather(semis, like):
    npc, V = semis[0].nodes_per_cell(), semis[0].num_vars()
    out = np.full(like.size, np.nan).reshape(-1, npc, V)
    for s in semis:
        out[s.local_cells()] = s.download().reshape(-1, npc, V)
    return out.reshape(-1)


def _run(semis, fam, pm, U0, steps, cfl, relax):
    for s in semis:
        s._use_family(fam, pm)
    rc = P.IntegratorConfig(tf=1e30, time=P.TimeControl(False, 0.0, P.CflRamp(cfl, cfl)),
                            relaxation=relax)
    _scatter(semis, U0)
    t, taken, aborted, recs = P.advance(semis[0], fam, pm, rc, 0.0, steps)
    assert taken == steps and not aborted
    return _gather(semis, U0), recs


def _owner(kind, mesh, pm, nranks):
    if kind == "slabs":
        return None
    if kind == "levels":
        return P.partition_levels(mesh, pm, nranks)
    rng = np.random.default_rng(17)
    own = rng.integers(0, nranks, mesh.num_cells()).astype(np.int32)
    own[:nranks] = np.arange(nranks)
    return own


@pytest.mark.parametrize("dim,nranks,kind", [(2, 2, "slabs"), (2, 3, "slabs"), (3, 2, "slabs"),
                                             (3, 4, "slabs"), (2, 3, "levels"), (3, 4, "levels"),
                                             (2, 2, "scattered"), (3, 3, "scattered")])
def test_loopback_partition_reproduces_single_domain(dim, nranks, kind):
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
    owner = _owner(kind, mesh, pm, nranks)
    P.loopback_group(semis, owner)
    # every rank's geometry is the global geometry of its cells
    gx = one.node_x().reshape(-1, one.nodes_per_cell())
    gz = (one.node_z() if dim == 3 else one.node_y()).reshape(-1, one.nodes_per_cell())
    seen = np.zeros(mesh.num_cells(), int)
    for r, s in enumerate(semis):
        g = s.local_cells()
        seen[g] += 1
        if owner is not None:
            assert np.array_equal(g, np.flatnonzero(owner == r))
        assert np.array_equal(s.node_x(), gx[g].reshape(-1))
        assert np.array_equal(s.node_z() if dim == 3 else s.node_y(), gz[g].reshape(-1))
    assert np.all(seen == 1)
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
    for s in semis:
        s._use_family(fam, pm)
    _scatter(semis, U0)
    t, res = P.perk_step_resident(0.0, 0.01, fam, pm, semis[0], P.PerkStepOptions())
    assert res.aborted and res.bad_cell == bad and res.bad_stage == 0
    assert np.array_equal(_gather(semis, U0), U0)  # untouched on abort
