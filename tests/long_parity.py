"""Long-run parity: the B200 path against the CPU oracle at each BASELINE
config's STATED step count (north_star gate: state within 1e-11 relative L2
per conserved variable, the relaxation gamma sequence and the entropy change
within 1e-12).

The oracle side is precomputed by tests/golden/make_long_parity.py (the
restatement oracle/perrk_oracle.c with the accurate relaxation numerics, the
numerics the configs run with; stepper.cpp:144-188, relax.cpp:51-104) and
committed as tests/golden/long_<cfg>.npz: the full step log (t, dt, gamma,
iterations, H, fell_back, invariants, delta_h, compensated H) and the final
state at a seeded sample of 32768 nodes.  Where the full oracle state is
present (baseline/_ref/parity/ or parity_full/<cfg>_U.npy, written by the
same script; git-ignored), the state metrics are ALSO computed over every
node.

Metrics (all reported; `gate` lists the north_star ones):
  state_rel[v]      ||U_gpu[:,v] - U_orc[:,v]|| / ||U_orc[:,v]||, literal,
                    per conserved variable (sample, and full when present)
  state_rel_mom[v]  the same with the momentum components measured against
                    the momentum field's norm (rotation invariant)
  gamma             max_n |gamma_gpu - gamma_orc|
  delta_h           max_n |delta_h_gpu - delta_h_orc| (PerkStepResult::delta_h)
  dH_total          max_n |(H_n - H_0)_gpu - (H_n - H_0)_orc|, compensated sums
  t                 max_n |t_gpu - t_orc| / max(1, t_end)
  fell_back         fallback counts on both sides

usage (GPU box): python tests/long_parity.py c1 c2 c3 c4 c5 [--json out.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, os.path.join(ROOT, "oracle"), HERE):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(HERE, "golden")
# full oracle final states: baseline/_ref/parity travels to the GPU box
# (git-ignored; C2-C4, <= 128 MiB each), parity_full/ stays here (C5's 640 MiB
# exceeds the box snapshot limit)
FULL_DIRS = [os.path.join(ROOT, "baseline", "_ref", "parity"), os.path.join(ROOT, "parity_full")]
TOL_STATE = 1e-11
TOL_GAMMA = 1e-12
TOL_DH = 1e-12


def fixture_path(name):
    return os.path.join(GOLDEN, f"long_{name}.npz")


def have_fixture(name):
    return os.path.exists(fixture_path(name))


def _rel(a, b, mom=False):
    V = b.shape[1]
    out = []
    nm = np.linalg.norm(b[:, 1:V - 1]) if mom else None
    for v in range(V):
        den = nm if (mom and 0 < v < V - 1) else np.linalg.norm(b[:, v])
        out.append(float(np.linalg.norm(a[:, v] - b[:, v]) / max(den, 1e-300)))
    return out


def compare(name, device=0):
    """Run config `name` on the GPU for the fixture's step count; return the
    metrics dict."""
    from paper_2507_04991_b200 import perrk as P
    from paper_2507_04991_b200 import workloads as W

    fx = np.load(fixture_path(name))
    steps = int(fx["steps"])
    log = fx["log"]
    ref = name.endswith("ref")  # against the unmodified reference (its numerics)
    cfg = W.make_config(name[:-3] if ref else name, steps=steps)
    if ref:
        cfg.relaxation = P.RelaxationConfig(numerics="reference")
    semi = P.Semidiscretization(cfg.spec(device))
    coords = (semi.node_x(), semi.node_y(), semi.node_z() if cfg.dim == 3 else None)
    U0 = W.initial_state_for(cfg, coords)
    V = semi.num_vars()
    semi.upload(U0)
    H0 = semi.total_entropy(U0)
    rc = P.IntegratorConfig(tf=1e30, time=P.TimeControl(False, 0.0, P.CflRamp(cfg.cfl, cfg.cfl)),
                            relaxation=cfg.relaxation)
    w0 = time.time()
    t, taken, aborted, recs = P.advance(semi, cfg.family, cfg.partition_map(), rc, 0.0, steps)
    gpu_s = time.time() - w0
    assert taken == steps and not aborted, (name, taken, aborted)
    U = semi.download().reshape(-1, V)
    g = np.array([r.gamma for r in recs])
    tt = np.array([r.t for r in recs])
    H = np.array([r.entropy for r in recs])
    dh = np.array([r.delta_h for r in recs])
    fb = sum(int(r.fell_back) for r in recs)
    idx = fx["idx"]
    hcol, h0o = (4, float(fx["H0"])) if ref else (7 + V, float(fx["H0_acc"]))
    m = {
        "config": name, "steps": steps, "nodes": int(U.shape[0]), "V": V,
        "gpu_seconds": gpu_s, "oracle_seconds": float(fx["seconds"]),
        "oracle_threads": int(fx["threads"]),
        "gamma": float(np.abs(g - log[:, 2]).max()),
        "gamma_range": [float(g.min()), float(g.max())],
        "t": float(np.abs(tt - log[:, 0]).max() / max(1.0, abs(log[-1, 0]))),
        # the reference's log has no delta_h / compensated H: its own naive H
        "delta_h": float(np.abs(dh - log[:, 6 + V]).max()) if not ref else None,
        "delta_h_scale": float(np.abs(log[:, 6 + V]).max()) if not ref else None,
        "dH_total": float(np.abs((H - H0) - (log[:, hcol] - h0o)).max()),
        "dH_total_scale": float(np.abs(log[:, hcol] - h0o).max()),
        "H0": float(H0), "H0_oracle": h0o,
        "iters_gpu": [int(r.newton_iters) for r in recs][:8],
        "iters_mismatch_steps": int(np.sum(np.array([r.newton_iters for r in recs]) != log[:, 3])),
        "gamma_argmax_step": int(np.argmax(np.abs(g - log[:, 2]))) + 1,
        "gamma_minus_1_at_argmax": float(log[int(np.argmax(np.abs(g - log[:, 2]))), 2] - 1.0),
        "gamma_rel_err_of_gamma_minus_1": float(
            np.abs(g - log[:, 2]).max() / max(np.abs(log[:, 2] - 1.0).max(), 1e-300)),
        "fell_back_gpu": fb, "fell_back_oracle": int(log[:, 5].sum()),
        "sample_nodes": int(idx.size),
        "state_rel_sample": _rel(U[idx], fx["sample"]),
        "state_rel_mom_sample": _rel(U[idx], fx["sample"], mom=True),
    }
    full = next((p for p in (os.path.join(d, f"{name}_U.npy") for d in FULL_DIRS)
                 if os.path.exists(p)), None)
    if full:
        Uo = np.load(full).reshape(-1, V)
        m["state_rel_full"] = _rel(U, Uo)
        m["state_rel_mom_full"] = _rel(U, Uo, mom=True)
        m["state_max_abs_full"] = float(np.abs(U - Uo).max())
    st = m.get("state_rel_full", m["state_rel_sample"])
    m["gate"] = {
        "state_1e-11_per_variable": max(st) <= TOL_STATE,
        "gamma_1e-12": m["gamma"] <= TOL_GAMMA,
        "delta_h_1e-12": ref or m["delta_h"] <= TOL_DH,
        "dH_total_1e-12": m["dH_total"] <= TOL_DH,
    }
    return m


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    out = []
    for name in args.configs:
        if not have_fixture(name):
            print(f"{name}: no fixture", flush=True)
            continue
        m = compare(name)
        out.append(m)
        print(json.dumps(m), flush=True)
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
