"""Check the frozen C2-C5 families against PROBED spectra (GPU).

For each configuration: a small uniform periodic mesh at the finest spacing
of the configuration's grading, the configuration's initial state, the
device RHS's Jacobian by colour-compressed central differences
(perrk.probe_jacobian, the reference's probe_jacobian procedure,
specopt.cpp:18-35), its eigenvalues, and the configuration's CFL step
dt = CFL / nu_max.  A cell of level r has spacing 2^(r-1) h_min, so member r
is checked on the spectrum scaled by 2^-(r-1).  Prints max |P_r(dt lambda)|
per member (<= 1: stable).  Run on a GPU box:

    python configs/check_families.py > configs/family_check.txt
"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_04991_b200 import perrk as P  # noqa: E402
from paper_2507_04991_b200 import workloads as W  # noqa: E402

CASES = {  # config: (cells per axis of the probe mesh, finest spacing, domain origin)
    "c1": (6, 20.0 / 16, -10.0),
    "c2": (6, 20.0 / 96, -10.0),
    "c3": (6, 2 * math.pi / 864, 0.0),
    "c4": (6, 1.0 / 768, 0.0),
    "c5": (3, 2 * math.pi / 216, 0.0),
}


def main():
    for name, (n, h, x0) in CASES.items():
        cfg = W.make_config(name)
        e = [x0 + h * i for i in range(n + 1)]
        mesh = P.Mesh2DRect(e, list(e)) if cfg.dim == 2 else P.Mesh3DRect(e, list(e), list(e))
        spec = P.SemidiscretizationSpec(mesh, physics=cfg.physics, mu=cfg.mu,
                                        prandtl=cfg.prandtl, surface_flux=cfg.surface_flux)
        semi = P.Semidiscretization(spec)
        coords = (semi.node_x(), semi.node_y(), semi.node_z() if cfg.dim == 3 else None)
        U = W.initial_state_for(cfg, coords)
        eigs = P.probe_spectrum(semi, U)
        ic = P.IntegratorConfig(time=P.TimeControl(False, 0.0, P.CflRamp(cfg.cfl, cfg.cfl)))
        dt = P.compute_dt(U, semi, ic, 0.0)
        fam = cfg.family
        margins = []
        for r in range(fam.R):
            level = fam.R - r
            one = P.PartitionFamily(fam.kind, fam.S, 1, [fam.E[r]], fam.A[r:r + 1], fam.b, fam.c)
            margins.append(P.stability_margin(one, eigs / 2 ** (level - 1), dt)[0])
        print(f"{name}: M={semi.num_dofs()} rho(J)={np.abs(eigs).max():.4g} dt={dt:.4g} "
              f"CFL={cfg.cfl} E={fam.E} max|P(dt lambda)| per member="
              + ", ".join(f"{m:.6f}" for m in margins))


if __name__ == "__main__":
    main()
