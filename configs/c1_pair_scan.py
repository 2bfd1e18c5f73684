"""C1's free coefficients: is there an (a21, a32) pair of the p2 S = 4 member
(butcher.cpp:51-105, constraints a21 <= 1/3, a32 <= 1/2 of :89-104) that is
linearly stable at C1's CFL 0.9 on the probed spectrum?  (VERDICT round 1,
item 9.)

The spectrum is the union of the dense central-difference probe
(specopt.cpp:18-35 procedure, perrk.probe_spectrum on the device) of the C1
vortex state on a 6 x 6 periodic proxy mesh at C1's spacing (h = 20/16;
check_families.py) and the Ritz values of 400 matrix-free Arnoldi steps on
the real 16 x 16 mesh (perrk.krylov_spectrum), each scaled by its first-step
dt.  The scan evaluates max |P(dt lambda)| over a
grid of the feasible box and reports the best pair, alongside the
survey-verified default (0.2, 0.35) and the spectrum's extent.

    python configs/c1_pair_scan.py          (GPU box: probes, then scans)
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_04991_b200 import perrk as P  # noqa: E402
from paper_2507_04991_b200 import workloads as W  # noqa: E402


def poly(a21, a32):
    fam = P.build_perk2(4, [4], [[a21, a32]])
    A, b = fam.A[0], fam.b
    # P(z) = 1 + z b^T (I - z A)^-1 1, coefficients b^T A^(k-1) 1
    one = np.ones(4)
    c = [1.0]
    v = one.copy()
    for _ in range(4):
        c.append(float(b @ v))
        v = A @ v
    return np.array(c)  # ascending powers


def margin(coef, z):
    return float(np.abs(np.polyval(coef[::-1], z)).max())


def main():
    cfg = W.make_config("c1")
    ic = P.IntegratorConfig(time=P.TimeControl(False, 0.0, P.CflRamp(cfg.cfl, cfg.cfl)))
    # (1) the dense probe on the 6 x 6 proxy at C1's spacing (check_families.py)
    h = 20.0 / 16
    e = [-10.0 + h * i for i in range(7)]
    mesh = P.Mesh2DRect(e, list(e))
    semi = P.Semidiscretization(P.SemidiscretizationSpec(mesh, surface_flux=cfg.surface_flux))
    U = W.initial_state_for(cfg, (semi.node_x(), semi.node_y(), None))
    zs = [P.compute_dt(U, semi, ic, 0.0) * P.probe_spectrum(semi, U)]
    # (2) Ritz values of the real 16 x 16 C1 mesh (matrix-free Arnoldi, m = 400)
    semi = P.Semidiscretization(cfg.spec())
    U = W.initial_state_for(cfg, (semi.node_x(), semi.node_y(), None))
    dt = P.compute_dt(U, semi, ic, 0.0)
    zs.append(dt * P.krylov_spectrum(semi, U, m=400))
    for what, z in zip(("proxy dense probe", "real mesh Krylov m=400"), zs):
        print(f"C1 {what}: {z.size} values, max|z|={np.abs(z).max():.4f} "
              f"max|Im z|={np.abs(z.imag).max():.4f} min Re z={z.real.min():.4f}")
    z = np.concatenate(zs)
    base = margin(poly(0.2, 0.35), z)
    print(f"survey pair (0.2, 0.35): max|P| = {base:.6f}")
    best = (None, 1e300)
    for a21 in np.linspace(0.005, 1.0 / 3.0, 67):
        for a32 in np.linspace(0.005, 0.5, 100):
            try:
                mg = margin(poly(a21, a32), z)
            except Exception:
                continue
            if mg < best[1]:
                best = ((float(a21), float(a32)), mg)
    print(f"best pair on the feasible box {best[0]}: max|P| = {best[1]:.6f}")
    # refine: the pair with the largest CFL headroom, max|P| at 5% above C1's dt
    from scipy.optimize import minimize
    zc = 1.05 * z

    def obj(x):
        a21, a32 = x
        if not (0.0 < a21 <= 1.0 / 3.0 and 0.0 < a32 <= 0.5):
            return 10.0
        return margin(poly(a21, a32), zc)

    r = minimize(obj, best[0], method="Nelder-Mead", options={"xatol": 1e-6, "fatol": 1e-9})
    a21, a32 = (float(v) for v in r.x)
    print(f"refined pair ({a21:.6f}, {a32:.6f}): max|P| = {margin(poly(a21, a32), z):.6f} at "
          f"CFL 0.9, {margin(poly(a21, a32), zc):.6f} at 1.05 x 0.9")
    np.savez(os.path.join(os.environ.get("OUT", "."), "c1_spectrum.npz"), z=z)


if __name__ == "__main__":
    main()
