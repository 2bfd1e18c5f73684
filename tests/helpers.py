"""Shared fixtures for the parity tests: meshes, seeded states, families."""
import math

import numpy as np

from paper_2507_04991_b200 import perrk as P
from paper_2507_04991_b200 import workloads as W


def nonuniform_edges(n, lo, hi, seed):
    rng = np.random.default_rng(seed)
    w = rng.uniform(0.6, 1.4, n)
    e = np.concatenate([[0.0], np.cumsum(w)])
    return (lo + (hi - lo) * e / e[-1]).tolist()


def mesh2d(nx, ny, seed=1):
    return P.Mesh2DRect(nonuniform_edges(nx, -1.0, 1.0, seed), nonuniform_edges(ny, -1.0, 1.0, seed + 1))


def mesh3d(nx, ny, nz, seed=1):
    return P.Mesh3DRect(nonuniform_edges(nx, -1.0, 1.0, seed), nonuniform_edges(ny, -1.0, 1.0, seed + 1),
                        nonuniform_edges(nz, -1.0, 1.0, seed + 2))


def smooth_state(coords, dim, seed=7, amp=0.3, gamma=1.4):
    """Seeded smooth periodic-ish state with O(1) entropy: rho, p in
    [1-amp, 1+amp], |v| <= amp."""
    rng = np.random.default_rng(seed)
    x = coords[:dim]
    fields = []
    for _ in range(dim + 2):
        k = rng.integers(1, 3, size=dim)
        ph = rng.uniform(0, 2 * math.pi, size=dim)
        f = np.ones_like(x[0])
        for d in range(dim):
            f = f * np.cos(math.pi * k[d] * x[d] + ph[d])
        fields.append(f)
    rho = 1.0 + amp * fields[0]
    v = [amp * fields[1 + d] for d in range(dim)]
    p = 1.0 + amp * fields[dim + 1]
    kin = 0.5 * rho * sum(vv * vv for vv in v)
    U = np.stack([rho] + [rho * vv for vv in v] + [p / (gamma - 1.0) + kin])
    return np.ascontiguousarray(U.T).reshape(-1)


def rel_err(a, b, V):
    """max over variables of ||a_v - b_v||_2 / ||b_v||_2 (||b_v|| floored at 1e-300)."""
    a = a.reshape(-1, V)
    b = b.reshape(-1, V)
    out = 0.0
    for v in range(V):
        nb = np.linalg.norm(b[:, v])
        d = np.linalg.norm(a[:, v] - b[:, v])
        out = max(out, d / max(nb, 1e-300) if nb > 1e-12 else d)
    return out


def max_rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))
