"""GPU: the reference's SPEC.md acceptance criteria that fall on the hot path,
re-hosted on the B200 path.

Criterion 4 ("linear invariants"): randomized p = 4 family
assignment on the 16x16 uniform vortex run, 5000 fixed steps: per-variable
conservation errors <= 1e-11 absolute for both P-ERK (no relaxation) and
P-ERRK (relaxation on).  The family is the C3 p4 {5,9,16} fixture; each cell
draws its level at random (seeded), widened by make_partition_map
(mesh.cpp:56-71).  The invariants are the StepRecord quadratures of every
step (stepper.cpp:179-180), compared with the initial state's.

Criterion 10 ("multirate cost accounting"): on criterion 1's
weak-blast setup, N_RHS of the multirate family against its standalone E = S
member at equal dt.  The blast mesh (build_blast_mesh, mesh.cpp:139-149) is
1D, which the B200 path does not run; it is extruded here to 2D with four
coarse (h = 1) cells in y and a y-independent weak-blast state
(physics.cpp:330-338), so the x-speeds set the levels exactly as in 1D
(assign_levels on characteristic_speed, then make_partition_map).  The device
counter (rhs_cell_evaluations, semidisc.cpp:133) must equal
steps * sum_cells |active set of the cell's member| * nodes * V for both runs.

The SPEC bound is N_RHS(multirate) <= 0.65 N_RHS(standalone).  On this mesh
the ratio is fixed by the level counts alone.  assign_levels (mesh.cpp:73-95,
ceil of log2(nu_max / nu)) puts the h = 1/16 band on level 3 (its nu is
1/2.38 of the fine band's) except the column touching the fine band, and the
neighbour widening adds one fine-level column each side: 34 / 2 / 28 columns
on levels 1 / 2 / 3, so N_multi / N_solo = (34 E_S + 2 E_mid + 28 E_min) /
(64 S) = 0.694 ({3,5,9}), 0.683 ({4,7,13}) and 0.694 ({6,10,18}), whatever
code counts it.  The test checks the measured ratios against that formula and
below 1; the SPEC's 0.65 is not reachable on the reference's own blast mesh
(DESIGN.md section 7).
"""
import json
import math

import numpy as np
import pytest

from paper_2507_04991_b200 import perrk as P
from paper_2507_04991_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _vortex_semi():
    mesh = P.build_uniform_mesh2d(10.0, 16)
    spec = P.SemidiscretizationSpec(mesh, 3, 1.4, "euler", 0.0, 0.72, "rusanov",
                                    "flux_differencing", "ec", 0)
    semi = P.Semidiscretization(spec)
    U0 = W.isentropic_vortex(W.VortexParams(), semi.node_x(), semi.node_y())
    return mesh, semi, np.ascontiguousarray(U0.T).reshape(-1)


@pytest.mark.parametrize("relaxed", [False, True])
def test_criterion4_linear_invariants_randomized_p4(relaxed):
    mesh, semi, U0 = _vortex_semi()
    fam = W.load_config_family("c3_p4_5_9_16")
    raw = np.random.Generator(np.random.PCG64(4)).integers(1, 4, mesh.num_cells()).astype(np.int32)
    pm = P.make_partition_map(mesh, raw, 3)
    assert min(pm.cells_per_level()) > 0
    inv0 = semi.integral_per_variable(U0)
    nu = semi.characteristic_speed(U0).max()
    dt = 0.3 / nu  # fixed step, inside the E = 5 member's stability range
    rc = P.IntegratorConfig(tf=1e30, time=P.TimeControl(fixed=True, dt=dt),
                            relaxation=P.RelaxationConfig(numerics="accurate") if relaxed else None)
    semi.upload(U0)
    steps = 5000
    t, taken, aborted, recs = P.advance(semi, fam, pm, rc, 0.0, steps)
    assert taken == steps and not aborted
    inv = np.array([r.invariants[:4] for r in recs])
    err = np.abs(inv - inv0).max(axis=0)
    print(json.dumps({"criterion": 4, "relaxed": relaxed, "steps": steps, "t_end": t,
                      "max_abs_conservation_error": err.tolist(),
                      "gamma_range": [min(r.gamma for r in recs), max(r.gamma for r in recs)]}))
    assert np.all(err <= 1e-11), err


def _blast_semi():
    x_edges = [-2.0]
    for a, b, n in ((-2.0, -1.0, 8), (-1.0, -0.5, 8), (-0.5, 0.5, 32), (0.5, 1.0, 8), (1.0, 2.0, 8)):
        x_edges += [a + (b - a) * i / n for i in range(1, n + 1)]  # append_uniform (mesh.cpp:137-141)
    mesh = P.Mesh2DRect(x_edges, [-2.0, -1.0, 0.0, 1.0, 2.0])
    spec = P.SemidiscretizationSpec(mesh, 3, 1.4, "euler", 0.0, 0.72, "ec",
                                    "flux_differencing", "ec", 0)
    semi = P.Semidiscretization(spec)
    x = semi.node_x()
    inner = np.abs(x) <= 0.5
    rho = np.where(inner, 1.1691, 1.0)
    v = np.where(inner, 0.1882 * np.sign(x), 0.0)
    p = np.where(inner, 1.245, 1.0)
    U = np.stack([rho, rho * v, np.zeros_like(x), p / 0.4 + 0.5 * rho * v * v])
    return mesh, semi, np.ascontiguousarray(U.T).reshape(-1)


def _count(semi, U0, fam, pm, dt, steps):
    semi.upload(U0)
    semi.reset_evaluation_counter()
    rc = P.IntegratorConfig(tf=1e30, time=P.TimeControl(fixed=True, dt=dt),
                            relaxation=P.RelaxationConfig(numerics="accurate"))
    _, taken, aborted, _ = P.advance(semi, fam, pm, rc, 0.0, steps)
    assert taken == steps and not aborted
    return semi.rhs_cell_evaluations()


@pytest.mark.parametrize("name,E", [("blast_p2_3_5_9", [3, 5, 9]),
                                    ("blast_p3_4_7_13", [4, 7, 13]),
                                    ("blast_p4_6_10_18", [6, 10, 18])])
def test_criterion10_multirate_rhs_count(name, E):
    mesh, semi, U0 = _blast_semi()
    fam = W.load_config_family(name)
    assert fam.E == E
    nu = semi.characteristic_speed(U0)
    pm = P.make_partition_map(mesh, P.assign_levels(nu, 3), 3)
    counts = pm.cells_per_level()
    # the x-speeds set the levels, as on the 1D blast mesh: 34 / 2 / 28
    # columns of four cells
    assert counts == [34 * 4, 2 * 4, 28 * 4], counts
    # the standalone E = S member at the same dt
    S = fam.S
    top = fam.member_index_for_level(1)
    solo = P.PartitionFamily(fam.kind, S, 1, [S], fam.A[top:top + 1].copy(), fam.b, fam.c,
                             [fam.active_sets[top]])
    dt = 0.5 / nu.max()
    steps = 10
    npc_v = 16 * 4
    n_multi = _count(semi, U0, fam, pm, dt, steps)
    n_solo = _count(semi, U0, solo, P.uniform_map(semi), dt, steps)
    expect_multi = steps * npc_v * sum(
        len(fam.active_sets[fam.member_index_for_level(l)]) * n for l, n in enumerate(counts, 1))
    assert n_multi == expect_multi
    assert n_solo == steps * npc_v * S * mesh.num_cells()
    ratio = n_multi / n_solo
    formula = sum(e * n for e, n in zip(reversed(E), counts)) / (S * sum(counts))
    print(json.dumps({"criterion": 10, "family": name, "levels": counts, "n_rhs_multirate": n_multi,
                      "n_rhs_standalone": n_solo, "ratio": ratio, "spec_bound": 0.65}))
    assert math.isclose(ratio, formula, rel_tol=1e-15)
    assert ratio < 1.0
