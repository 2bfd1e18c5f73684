"""CPU, world_size 2 and 3 over gloo: the host-side logic of the element
partition, with the library's own host helpers.

  * ownership maps: slabs cover the mesh in contiguous layers balanced by
    DOF-stage work; the per-level partition gives every rank an equal share
    of every level (every P-ERK stage balanced);
  * the halo plan of perrk_comm_init (perrk_halo_plan: per-peer ghost slots and
    send lists, both ordered by the sender's (cell, face)) delivers to each
    rank, through point-to-point messages to its peers, exactly the
    neighbour face traces the stage kernel reads in the single-domain
    (periodic) run, for slab, per-level and scattered ownership;
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


def _neighbour(n, g, f):
    co = [g % n[0], (g // n[0]) % n[1], g // (n[0] * n[1])]
    d, side = f >> 1, f & 1
    co[d] = (co[d] + (1 if side else -1)) % n[d]
    return co[0] + n[0] * (co[1] + n[1] * co[2])


def _owner(kind, mesh, world, rng):
    if kind == "slabs":
        return P.partition_slabs(mesh, world)
    if kind == "levels":
        lv = rng.integers(1, 4, mesh.num_cells()).astype(np.int32)
        return P.partition_levels(mesh, P.PartitionMap(3, lv, lv), world)
    own = rng.integers(0, world, mesh.num_cells()).astype(np.int32)
    own[:world] = np.arange(world)
    return own


def _worker(rank, world, port, dim, kind, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    try:
        V, npc = dim + 2, (16 if dim == 2 else 64)
        n = (5, 4, 6) if dim == 3 else (7, 6)
        mesh = P.Mesh3DRect(*[np.linspace(0, 1, k + 1) for k in n]) if dim == 3 else \
            P.Mesh2DRect(*[np.linspace(0, 1, k + 1) for k in n])
        n3 = list(n) + [1] * (3 - dim)
        ncells = int(np.prod(n))
        rng = np.random.default_rng(11)
        Ug = rng.standard_normal(ncells * npc * V)          # the global state, every rank
        owner = _owner(kind, mesh, world, rng)               # same seed: same map on every rank
        h = P.halo_plan(mesh, owner, rank)
        cells = Ug.reshape(ncells, npc, V)
        mine = cells[h["gid"]]
        assert np.array_equal(h["gid"], np.flatnonzero(owner == rank))
        faces = [P.face_nodes(dim, f) for f in range(2 * dim)]
        # pack (pack_traces_kernel) and exchange per peer (NcclExchange::sendrecv)
        sendbuf = np.stack([mine[c][faces[f]] for c, f in h["send"]]) if len(h["send"]) else \
            np.zeros((0, len(faces[0]), V))
        ghost = np.zeros((len(h["ghost_gid"]), len(faces[0]), V))
        t = lambda a: torch.from_numpy(a)
        reqs, recv = [], []
        for k, p in enumerate(h["peers"]):
            so, se = h["send_off"][k], h["send_off"][k + 1]
            ro, re = h["recv_off"][k], h["recv_off"][k + 1]
            reqs.append(dist.isend(t(np.ascontiguousarray(sendbuf[so:se])), int(p)))
            buf = np.zeros((re - ro, len(faces[0]), V))
            reqs.append(dist.irecv(t(buf), int(p)))
            recv.append((ro, re, buf))
        for r in reqs:
            r.wait()
        for ro, re, buf in recv:
            ghost[ro:re] = buf
        # what the single-domain stage kernel reads across every face
        ok_halo = True
        nf = 2 * dim
        for li, g in enumerate(h["gid"]):
            for f in range(nf):
                ng = _neighbour(n3, int(g), f)
                want = cells[ng][faces[f ^ 1]]
                k = int(h["nbr"][li * nf + f])
                if k >= 0:
                    ok_halo &= int(h["gid"][k]) == ng
                else:
                    ok_halo &= int(h["ghost_gid"][-1 - k]) == ng and \
                        np.array_equal(ghost[-1 - k], want)
        # rank-ordered double-double combine of per-rank partials
        w = rng.uniform(0.1, 1.0, ncells * npc)
        vals = rng.standard_normal(ncells * npc) * 1e3
        part = (0.0, 0.0)
        for x in (w * vals).reshape(ncells, npc)[h["gid"]].ravel():
            part = dd_add(part, (x, 0.0))
        allp = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allp, torch.tensor(part, dtype=torch.float64))
        tot = (0.0, 0.0)
        for p in allp:
            tot = dd_add(tot, (float(p[0]), float(p[1])))
        exact = float(np.sum((w * vals).astype(np.longdouble)))
        q.put((rank, bool(ok_halo), abs(tot[0] + tot[1] - exact) / abs(exact), len(h["ghost_gid"])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dim,world,kind", [(2, 2, "slabs"), (3, 2, "slabs"), (2, 3, "levels"),
                                            (3, 2, "levels"), (2, 3, "scattered"),
                                            (3, 3, "scattered")])
def test_halo_plan_and_reductions_gloo(dim, world, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dim, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [True] * world
    assert max(r[2] for r in res) < 1e-15
    assert all(r[3] > 0 for r in res)


def test_partitions_balance_the_c5_work():
    cfg = W.make_config("c5")
    pm = cfg.partition_map()
    npc = cfg.nodes_per_cell()
    work = P.cell_work(pm, cfg.family, npc)
    assert abs(work.sum() - W.dof_stage_updates_per_step(cfg.family, pm, npc)) < 1
    lv = np.asarray(pm.effective_level)
    for nr in (1, 2, 4, 8):
        own = P.partition_slabs(cfg.mesh, nr, work)
        layers = own.reshape(64, -1)
        assert np.all(layers == layers[:, :1]) and np.all(np.diff(layers[:, 0]) >= 0)
        loads = np.bincount(own, weights=work, minlength=nr)
        assert loads.max() <= work.sum() / nr + work.reshape(64, -1).sum(axis=1).max()
        own = P.partition_levels(cfg.mesh, pm, nr)
        for l in range(1, pm.R + 1):
            c = np.bincount(own[lv == l], minlength=nr)
            assert c.max() - c.min() <= 1
    assert list(np.unique(P.partition_slabs(P.Mesh2DRect(np.linspace(0, 1, 4),
                                                         np.linspace(0, 1, 11)), 3)
                          .reshape(10, 3)[:, 0], return_counts=True)[1]) in ([3, 4, 3], [4, 3, 3],
                                                                              [3, 3, 4])
