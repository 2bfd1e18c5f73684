"""Generate the long-run parity fixtures: each BASELINE config advanced by the
CPU oracle restatement (oracle/_build/liboracle.so, accurate relaxation
numerics — the numerics the product runs the configs with) for its STATED
step count (C2 500, C3 200, C4 200, C5 100), and C1 (100 steps) also on the
unmodified reference (oracle/_ref, reference numerics).

Writes, per config:
  tests/golden/long_<cfg>.npz   (committed; small)
      log      [steps, 8+V]  t, dt, gamma, iters, H, fell_back, invariants[V],
               delta_h (PerkStepResult::delta_h), H_acc (compensated H)
               (the reference run, c1ref, has the first 6+V columns)
      H0, H0_acc  initial total entropy (naive / compensated sum)
      idx      seeded node sample (oracle/cpu_runs.sample_indices)
      sample   [len(idx), V]  final state at the sampled nodes
      norms    [V]  ||U_final[:, v]||_2 over ALL nodes
      seconds  oracle wall time, threads
  baseline/_ref/parity/<cfg>_U.npy   (git-ignored; travels to the GPU box)
      the full final state, for the full-field comparison in
      tests/long_parity.py (C5's 640 MiB exceeds the GPU box's 512 MiB
      snapshot limit: C5 is compared on the committed node sample only)

The oracle's threading only splits the per-cell volume pass (parallel_cells,
semidisc.cpp:75-89); faces, stage formation and every reduction are serial
and fixed-order, so the outputs do not depend on the thread count.

usage: python tests/golden/make_long_parity.py c2 [c3 c4 c5 c1ref] [--threads N]
"""
import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import cpu_runs as CR  # noqa: E402

SAMPLE = 32768


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--steps", type=int, default=None, help="override (testing only)")
    ap.add_argument("--out", default=HERE)
    args = ap.parse_args()
    full_dir = os.path.join(ROOT, "baseline", "_ref", "parity")
    os.makedirs(full_dir, exist_ok=True)
    for name in args.configs:
        ref = name.endswith("ref")
        spec = CR.S.make_spec(name[:-3] if ref else name)
        run = CR.CpuConfig(spec, threads=args.threads, kind="ref" if ref else "orc")
        U = run.initial_state()
        H0 = run.total_entropy(U)
        H0_acc = run.total_entropy_acc(U) if not ref else H0
        steps = args.steps or spec.steps
        t0 = time.time()
        t, taken, log, secs = run.run(U, steps)
        assert taken == steps, (name, taken)
        V = spec.num_vars()
        Uv = U.reshape(-1, V)
        idx = CR.sample_indices(Uv.shape[0], SAMPLE)
        tag = name if args.steps is None else f"{name}_{steps}"
        np.savez_compressed(os.path.join(args.out, f"long_{tag}.npz"), log=log, H0=H0, H0_acc=H0_acc, idx=idx,
                            sample=Uv[idx], norms=np.linalg.norm(Uv, axis=0), steps=steps,
                            seconds=secs, threads=args.threads)
        np.save(os.path.join(full_dir, f"{tag}_U.npy"), U)
        print(f"{tag}: {steps} steps, t={t:.6g}, {secs:.1f} s ({time.time() - t0:.1f} s wall), "
              f"gamma [{log[:, 2].min():.15g}, {log[:, 2].max():.15g}], "
              f"fell_back {int(log[:, 5].sum())}, H {H0:.15g} -> {log[-1, 4]:.15g}", flush=True)


if __name__ == "__main__":
    main()
