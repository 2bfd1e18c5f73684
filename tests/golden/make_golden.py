"""Generate the golden fixtures of tests/test_oracle.py from the UNMODIFIED
reference library (oracle/_ref/libperrk_ref.so, built from /root/reference
by oracle/Makefile).  Run here, where /root/reference exists:

    make -C oracle ref && python tests/golden/make_golden.py

Fixtures (small, committed):
  rhs_2d.npz     reference RHS of the C1 initial state (16^2 vortex, EC +
                 Rusanov) and of a seeded smooth state on a 7x6 non-uniform
                 mesh for every surface flux
  c1_run.npz     30 reference P-ERRK steps of C1 (CFL 0.9, reference Newton
                 relaxation): per-step log (t, dt, gamma, iters, H, fell_back,
                 invariants) and the final state
  families.npz   reference-built p2/p3/p4 families (A, b, c) and their
                 family_to_text output (butcher.cpp:334-355)
"""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

import oracle as O  # noqa: E402
from helpers import mesh2d, smooth_state  # noqa: E402
from paper_2507_04991_b200 import perrk as P  # noqa: E402
from paper_2507_04991_b200 import workloads as W  # noqa: E402


def main():
    cfg = W.make_config("c1")
    ref = O.Ref(cfg.mesh)
    x, y, _, _ = ref.node_coords()
    U_c1 = W.initial_state_for(cfg, (x, y, None))
    out = {"U_c1": U_c1, "rhs_c1": ref.rhs(0.0, U_c1)}
    m = mesh2d(7, 6, seed=2)
    out["xe"], out["ye"] = np.array(m.x_edges), np.array(m.y_edges)
    r0 = O.Ref(m)
    x, y, _, _ = r0.node_coords()
    U = smooth_state((x, y), 2, seed=4)
    out["U_rand"] = U
    for s in ("rusanov", "hlle", "hllc", "ec", "central"):
        out[f"rhs_rand_{s}"] = O.Ref(m, surface_flux=s).rhs(0.0, U)
    np.savez_compressed(os.path.join(HERE, "rhs_2d.npz"), **out)

    U = U_c1.copy()
    steps = 30
    _, taken, log, _ = ref.run_steps(U, 0.0, steps, cfg.family,
                                     cfg.partition_map().effective_level,
                                     P.RelaxationConfig(), False, 0.9)
    assert taken == steps
    np.savez_compressed(os.path.join(HERE, "c1_run.npz"), U0=U_c1, U=U, log=log, steps=steps)

    L = O.ref_lib()
    fams = {"p2": (0, 4, [4], [0.2, 0.35]),
            "p3": (1, 7, [4, 7], [0.3, 0.2, 0.25, 0.3, 0.35]),
            "p4": (3, 14, [5, 8, 14], [0.5] * 3 + [0.7] * 9)}
    out = {}
    for key, (kind, S, E, free) in fams.items():
        R = len(E)
        Ea = np.array(E, np.int32)
        fr = np.array(free, float)
        A, b, c = np.zeros((R, S, S)), np.zeros(S), np.zeros(S)
        act = np.zeros((R, S), np.int32)
        assert L.ref_family_build(kind, S, R, O.ip(Ea), O.dp(fr), 1.0, O.dp(A), O.dp(b), O.dp(c),
                                  O.ip(act)) == 0
        rf = O.RefFamily(S, R, kind, O.ip(Ea), O.dp(A), O.dp(b), O.dp(c))
        buf = C.create_string_buffer(1 << 16)
        assert L.ref_family_to_text(C.byref(rf), buf, len(buf)) == 0
        out[f"A_{key}"], out[f"b_{key}"], out[f"c_{key}"] = A, b, c
        out[f"act_{key}"] = act
        out[f"text_{key}"] = np.array(buf.value.decode())
    np.savez_compressed(os.path.join(HERE, "families.npz"), **out)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
