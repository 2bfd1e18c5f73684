"""Check the frozen C1-C5 families on the REAL configuration meshes (GPU),
with the matrix-free Krylov spectrum estimate (perrk_krylov_hessenberg,
SURVEY.md 8f item 1) in place of the dense probe, which the reference guards
to M <= 5000 unknowns (specopt.cpp:18-35) and check_families.py therefore
runs on small proxy meshes.

For each configuration: the full mesh, its initial state, its effective
level map, and the CFL step dt = CFL / nu_max of its first step.  For each
level r the Jacobian restricted to the level's cells (the operator member r
integrates; cell_mask) is probed by m Arnoldi steps on the central-
difference JVP, and member r's stability polynomial (butcher.cpp stability
function) is evaluated on dt times the Ritz values: max |P_r(dt lambda)|
<= 1 is stable.  The Ritz values resolve the spectral envelope (the extreme
eigenvalues the step size is limited by); on small meshes they match the
dense probe's to 1e-6 (tests/test_gpu_spectrum.py).

    python configs/check_families_krylov.py [c1 ... c5] > configs/family_check_krylov.txt
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_04991_b200 import perrk as P  # noqa: E402
from paper_2507_04991_b200 import workloads as W  # noqa: E402

M_KRYLOV = {"c1": 120, "c2": 80, "c3": 60, "c4": 60, "c5": 40}


def main(names):
    for name in names:
        cfg = W.make_config(name)
        semi = P.Semidiscretization(cfg.spec())
        coords = (semi.node_x(), semi.node_y(), semi.node_z() if cfg.dim == 3 else None)
        U = W.initial_state_for(cfg, coords)
        ic = P.IntegratorConfig(time=P.TimeControl(False, 0.0, P.CflRamp(cfg.cfl, cfg.cfl)))
        dt = P.compute_dt(U, semi, ic, 0.0)
        pm = cfg.partition_map()
        fam = cfg.family
        m = M_KRYLOV[name]
        out = []
        t0 = time.time()
        for level in range(1, fam.R + 1):
            mask = (pm.effective_level == level).astype(np.int8)
            if not mask.any():
                continue
            ritz = P.krylov_spectrum(semi, U, m=m, cell_mask=mask)
            r = fam.member_index_for_level(level)
            one = P.PartitionFamily(fam.kind, fam.S, 1, [fam.E[r]], fam.A[r:r + 1], fam.b, fam.c)
            marg = P.stability_margin(one, ritz, dt)[0]
            out.append(f"L{level}(E={fam.E[r]}, {int(mask.sum())} cells): rho={np.abs(ritz).max():.5g} "
                       f"min Re={ritz.real.min():.5g} max|P|={marg:.6f}")
        print(f"{name}: M={semi.num_dofs()} m={m} dt={dt:.5g} CFL={cfg.cfl} E={fam.E} "
              f"[{time.time() - t0:.1f} s] " + "; ".join(out), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"])
