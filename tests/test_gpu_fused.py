"""GPU: perrk_advance's fused relaxation (relax_spec_kernel: Newton pass 2
fused with a speculative out-of-place final update, host.cpp enqueue_step)
against the unfused chain of relax_pass_kernel + update_kernel.

The speculation is accepted only when Newton finishes at the gamma the pass
evaluated, so the two chains must agree bitwise: state, step records, time.
C1's first steps start from gamma_seed = 1 far from the root (pass 2 does not
converge there: the speculation is rejected and the ordinary passes and
update take over); later steps accept it.  Odd and even step counts and a
chunked run() exercise the buffer alternation (c->U / c->Ualt)."""
import numpy as np
import pytest

from paper_2507_04991_b200 import perrk as P
from paper_2507_04991_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _advance(cfg, U0, coords_of, chunks, fused, monkeypatch):
    monkeypatch.setenv("PERRK_NO_FUSED_RELAX", "0" if fused else "1")
    semi = P.Semidiscretization(cfg.spec())
    U = U0(semi)
    semi.upload(U)
    rc = P.IntegratorConfig(tf=1e9, time=P.TimeControl(fixed=False, ramp=P.CflRamp(cfg.cfl, cfg.cfl)),
                            relaxation=P.RelaxationConfig(numerics="accurate"))
    t, recs = 0.0, []
    for n in chunks:
        t, taken, aborted, r = P.advance(semi, cfg.family, cfg.partition_map(), rc, t, n)
        assert taken == n and not aborted
        recs += r
    return semi.download(), recs, t


def _compare(cfg, U0, chunks, monkeypatch):
    Uf, rf, tf = _advance(cfg, U0, None, chunks, True, monkeypatch)
    Uu, ru, tu = _advance(cfg, U0, None, chunks, False, monkeypatch)
    assert np.array_equal(Uf, Uu)
    assert tf == tu
    for a, b in zip(rf, ru):
        assert (a.t, a.dt, a.gamma, a.newton_iters, a.entropy, a.fell_back) == \
               (b.t, b.dt, b.gamma, b.newton_iters, b.entropy, b.fell_back)
        assert list(a.invariants) == list(b.invariants)
    return rf


@pytest.mark.parametrize("chunks", [[7], [8], [3, 4, 5]])
def test_fused_relaxation_bitwise_c1(chunks, monkeypatch):
    cfg = W.make_config("c1")
    U0 = lambda semi: W.initial_state_for(cfg, (semi.node_x(), semi.node_y(), None))
    recs = _compare(cfg, U0, chunks, monkeypatch)
    # the first step needs more than two Newton passes (speculation rejected)
    assert recs[0].newton_iters > 2


@pytest.mark.parametrize("chunks", [[5], [2, 3]])
def test_fused_relaxation_bitwise_tgv_sample(chunks, monkeypatch):
    cfg = W.sample_config(W.make_config("c5"))
    U0 = lambda semi: W.initial_state_for(cfg, (semi.node_x(), semi.node_y(), semi.node_z()))
    recs = _compare(cfg, U0, chunks, monkeypatch)
    # steps 1-2 start far from the root (speculation rejected), later steps
    # finish at pass 2 (accepted: the update came from relax_spec_kernel)
    iters = [r.newton_iters for r in recs]
    assert iters[0] > 2 and 2 in iters


def test_anchored_relaxation_fused_vs_oracle(monkeypatch):
    """Anchored relaxation (h_ref = H(U_0), stepper.cpp:154-156) through
    perrk_advance: fused and unfused chains bitwise equal, and 40 C1 steps
    against the oracle restatement (state 1e-11 rel L2 per variable, gamma and
    H within 1e-12)."""
    import oracle as O
    from helpers import rel_err
    cfg = W.make_config("c1")
    out = {}
    for fused in (True, False):
        monkeypatch.setenv("PERRK_NO_FUSED_RELAX", "0" if fused else "1")
        semi = P.Semidiscretization(cfg.spec())
        U0 = W.initial_state_for(cfg, (semi.node_x(), semi.node_y(), None))
        semi.upload(U0)
        rc = P.IntegratorConfig(tf=1e9, time=P.TimeControl(fixed=False, ramp=P.CflRamp(0.9, 0.9)),
                                relaxation=P.RelaxationConfig(numerics="accurate"), anchor="initial")
        t, taken, aborted, recs = P.advance(semi, cfg.family, cfg.partition_map(), rc, 0.0, 40)
        assert taken == 40 and not aborted
        out[fused] = (semi.download(), recs)
    (Uf, rf), (Uu, ru) = out[True], out[False]
    assert np.array_equal(Uf, Uu)
    assert [r.gamma for r in rf] == [r.gamma for r in ru]
    orc = O.Orc(cfg.mesh)
    Uo = U0.copy()
    _, taken, log, _ = orc.run_steps(Uo, 0.0, 40, cfg.family, cfg.partition_map().effective_level,
                                     P.RelaxationConfig(numerics="accurate"), False, 0.9, anchor=True)
    assert taken == 40
    assert rel_err(Uf, Uo, 4) < 1e-11
    assert np.abs(np.array([r.gamma for r in rf]) - log[:, 2]).max() < 1e-12
    assert np.abs(np.array([r.entropy for r in rf]) - log[:, 4]).max() < 1e-12


@pytest.mark.parametrize("numerics,anchor", [("accurate", "initial"), ("reference", "step"),
                                             ("reference", "initial"), ("accurate", "step")])
def test_chunked_run_is_one_run(numerics, anchor):
    """run() in chunks (perrk.run -> several perrk_advance calls) is ONE run:
    the gamma seed and the anchor H(U_0) carry across the chunks
    (stepper.cpp:151,153,170), so run(chunk=7) equals one advance call of the
    same steps bit for bit (state, gamma, Newton iterations, H)."""
    cfg = W.make_config("c1")
    relax = P.RelaxationConfig(numerics=numerics)
    steps = 30
    semi = P.Semidiscretization(cfg.spec())
    U0 = W.initial_state_for(cfg, (semi.node_x(), semi.node_y(), None))
    semi.upload(U0)
    rc = P.IntegratorConfig(tf=1e9, time=P.TimeControl(fixed=False, ramp=P.CflRamp(0.9, 0.9)),
                            relaxation=relax, anchor=anchor)
    _, taken, _, one = P.advance(semi, cfg.family, cfg.partition_map(), rc, 0.0, steps)
    assert taken == steps
    U_one = semi.download()
    # run() stops at tf: put tf just past the one-call run's final time
    rc2 = P.IntegratorConfig(tf=one[-1].t, time=rc.time, relaxation=relax, anchor=anchor)
    res = P.run(rc2, cfg.family, cfg.partition_map(), semi, U0, chunk=7)
    assert len(res.log) == steps
    assert np.array_equal(res.U, U_one)
    assert [r.gamma for r in res.log] == [r.gamma for r in one]
    assert [r.newton_iters for r in res.log] == [r.newton_iters for r in one]
    assert [r.entropy for r in res.log] == [r.entropy for r in one]
    assert [r.delta_h for r in res.log] == [r.delta_h for r in one]


def test_relaxation_methods_alternate_on_one_context():
    """The captured step graph is keyed by the relaxation method (bisection
    and secant capture more passes than Newton): Newton, bisection, secant,
    Newton again on ONE context, nsteps > 1 each, equal to fresh contexts."""
    cfg = W.make_config("c1")
    rc_of = lambda m: P.IntegratorConfig(
        tf=1e9, time=P.TimeControl(fixed=False, ramp=P.CflRamp(0.9, 0.9)),
        relaxation=P.RelaxationConfig(method=m, numerics="reference"))
    shared = P.Semidiscretization(cfg.spec())
    U0 = W.initial_state_for(cfg, (shared.node_x(), shared.node_y(), None))
    for m in ["newton", "bisection", "secant", "newton"]:
        shared.upload(U0)
        _, n1, _, r1 = P.advance(shared, cfg.family, cfg.partition_map(), rc_of(m), 0.0, 4)
        fresh = P.Semidiscretization(cfg.spec())
        fresh.upload(U0)
        _, n2, _, r2 = P.advance(fresh, cfg.family, cfg.partition_map(), rc_of(m), 0.0, 4)
        assert n1 == n2 == 4
        assert np.array_equal(shared.download(), fresh.download()), m
        assert [r.gamma for r in r1] == [r.gamma for r in r2], m
        assert [(r.newton_iters, r.fell_back) for r in r1] == \
               [(r.newton_iters, r.fell_back) for r in r2], m
