"""GPU: traversal order of the 3D cell lists (host.cpp brick_order,
PERRK_BRICK=B).  The order only permutes the persistent warps' work and the
order of the delta-H partial sums, so a brick-ordered run must agree with
the natural-order run to rounding: states to 1e-13, gamma to 1e-13, the same
DOF-stage count.  The C5 16^3 sample has three levels, so the per-stage
active lists are proper sublists."""
import numpy as np
import pytest

from paper_2507_04991_b200 import perrk as P
from paper_2507_04991_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _run(cfg, steps, brick, monkeypatch):
    monkeypatch.setenv("PERRK_BRICK", str(brick))
    semi = P.Semidiscretization(cfg.spec())
    U = W.initial_state_for(cfg, (semi.node_x(), semi.node_y(), semi.node_z()))
    semi.upload(U)
    rc = P.IntegratorConfig(tf=1e9, time=P.TimeControl(fixed=False, ramp=P.CflRamp(cfg.cfl, cfg.cfl)),
                            relaxation=P.RelaxationConfig(numerics="accurate"))
    t, taken, aborted, recs = P.advance(semi, cfg.family, cfg.partition_map(), rc, 0.0, steps)
    assert taken == steps and not aborted
    return semi.download(), recs, semi.rhs_cell_evaluations()


@pytest.mark.parametrize("brick", [2, 4, 8])
def test_brick_order_matches_natural_order(brick, monkeypatch):
    cfg = W.sample_config(W.make_config("c5"))
    U0, r0, n0 = _run(cfg, 3, 0, monkeypatch)
    U1, r1, n1 = _run(cfg, 3, brick, monkeypatch)
    assert n0 == n1
    V = 5
    a, b = U0.reshape(-1, V), U1.reshape(-1, V)
    scale = np.linalg.norm(a, axis=0).max()  # (the z-momentum of the TGV starts at zero)
    for v in range(V):
        assert np.linalg.norm(a[:, v] - b[:, v]) / scale < 1e-13, (brick, v)
    for x, y in zip(r0, r1):
        assert abs(x.gamma - y.gamma) < 1e-13
        assert x.dt == y.dt
