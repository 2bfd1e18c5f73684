"""CPU, world_size 2 over gloo: the host-side logic of the element-slab
decomposition, with the library's own host helpers.

  * layer cuts: contiguous, covering, balanced by DOF-stage work;
  * the halo pattern of perrk_comm_init (send top -> rank above as its
    ghost_lo, send bottom -> rank below as its ghost_hi, periodic ring; with
    2 ranks both go to the same peer and are matched in order) delivers to
    each rank exactly the neighbour face traces the stage kernel reads in the
    single-domain (periodic) run;
  * the reduction combine (double-double partials summed in rank order)
    reproduces the single-domain sums.
The device side of the same path runs on one GPU through perrk_loopback_group
(tests/test_gpu_slab.py)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_04991_b200 import perrk as P
from paper_2507_04991_b200 import workloads as W


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def two_sum(a, b):
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def dd_add(x, y):
    s, e = two_sum(x[0], y[0])
    e = e + (x[1] + y[1])
    hi = s + e
    return hi, e - (hi - s)


def _worker(rank, world, port, dim, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    try:
        V, npc = dim + 2, (16 if dim == 2 else 64)
        n = (5, 4, 6) if dim == 3 else (7, 6)
        ncells = int(np.prod(n))
        rng = np.random.default_rng(11)
        Ug = rng.standard_normal(ncells * npc * V)          # the global state, every rank
        cuts = P.slab_cuts(n[-1], world)
        b, e = int(cuts[rank]), int(cuts[rank + 1])
        lc = ncells // n[-1]
        cells = Ug.reshape(ncells, npc, V)
        mine = cells[b * lc:e * lc]
        bot, top = P.slab_trace_nodes(dim, 0), P.slab_trace_nodes(dim, 1)
        send_lo = np.ascontiguousarray(mine[:lc][:, bot, :])     # [face cell][pt][V]
        send_hi = np.ascontiguousarray(mine[-lc:][:, top, :])
        up, dn = (rank + 1) % world, (rank - 1) % world
        ghost_lo, ghost_hi = np.empty_like(send_lo), np.empty_like(send_hi)
        t = lambda a: torch.from_numpy(a)
        # the grouped order of NcclExchange::halo
        reqs = [dist.isend(t(send_hi), up), dist.irecv(t(ghost_lo), dn),
                dist.isend(t(send_lo), dn), dist.irecv(t(ghost_hi), up)]
        for r in reqs:
            r.wait()
        # what the single-domain stage kernel reads across those faces
        below = (b - 1) % n[-1]
        above = e % n[-1]
        want_lo = cells[below * lc:(below + 1) * lc][:, top, :]
        want_hi = cells[above * lc:(above + 1) * lc][:, bot, :]
        ok_halo = np.array_equal(ghost_lo, want_lo) and np.array_equal(ghost_hi, want_hi)
        # rank-ordered double-double combine of per-rank partials
        w = rng.uniform(0.1, 1.0, ncells * npc)
        vals = rng.standard_normal(ncells * npc) * 1e3
        part = (0.0, 0.0)
        for x in (w * vals).reshape(ncells, npc)[b * lc:e * lc].ravel():
            part = dd_add(part, (x, 0.0))
        allp = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allp, torch.tensor(part, dtype=torch.float64))
        tot = (0.0, 0.0)
        for p in allp:
            tot = dd_add(tot, (float(p[0]), float(p[1])))
        exact = float(np.sum((w * vals).astype(np.longdouble)))
        q.put((rank, ok_halo, abs(tot[0] + tot[1] - exact) / abs(exact), (b, e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dim", [2, 3])
def test_slab_halo_and_reductions_gloo_world2(dim):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, dim, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [True, True]
    assert max(r[2] for r in res) < 1e-15
    assert res[0][3][0] == 0 and res[0][3][1] == res[1][3][0]


def test_slab_cuts_balance_the_c5_work():
    cfg = W.make_config("c5")
    pm = cfg.partition_map()
    work = P.layer_work(cfg.mesh, pm, cfg.family, 64)
    assert work.size == 64 and abs(work.sum() - W.dof_stage_updates_per_step(cfg.family, pm, 64)) < 1
    for nr in (1, 2, 4, 8):
        cuts = P.slab_cuts(64, nr, work)
        assert cuts[0] == 0 and cuts[-1] == 64 and np.all(np.diff(cuts) >= 1)
        loads = [work[cuts[r]:cuts[r + 1]].sum() for r in range(nr)]
        assert max(loads) / (work.sum() / nr) < 1.0 + 2.0 * work.max() * nr / work.sum()
    uni = P.slab_cuts(10, 3)
    assert list(uni) == [0, 3, 7, 10] or list(uni) == [0, 3, 6, 10] or list(uni) == [0, 4, 7, 10]
