"""CPU: configs/spec.py (the workloads as plain data, shared by the product
and the CPU arms) agrees with the product's host layer: level maps against
the native make_partition_map (mesh.cpp:56-71), families against the
product's parser and family builder (butcher.cpp), DOF-stage counts, and the
oracle-side CpuConfig builds the same mesh, levels and initial state without
importing the product."""
import subprocess
import sys

import numpy as np
import pytest

import cpu_runs as CR
from paper_2507_04991_b200 import perrk as P
from paper_2507_04991_b200 import workloads as W

NAMES = ["c1", "c2", "c3", "c4", "c5"]


@pytest.mark.parametrize("name", NAMES)
def test_spec_matches_product(name):
    cfg = W.make_config(name)
    sp = CR.S.make_spec(name)
    pm = cfg.partition_map()
    assert np.array_equal(pm.effective_level, sp.effective_levels())
    ft = sp.family()
    assert ft.E == list(cfg.family.E)
    assert np.array_equal(ft.A, cfg.family.A) and np.array_equal(ft.b, cfg.family.b)
    assert np.array_equal(ft.c, cfg.family.c)
    assert [ft.active_stages(r) for r in range(ft.R)] == list(cfg.family.active_sets)
    assert sp.dof_stage_updates_per_step() == \
        W.dof_stage_updates_per_step(cfg.family, pm, cfg.nodes_per_cell())
    for a, b in zip(sp.mesh.edges, cfg.mesh.edges):
        assert np.array_equal(a, b)


def test_c1_family_fixture_is_build_perk2():
    """configs/c1_p2_4.family is build_perk2(4, {4}, {{0.204, 0.42}}) (butcher.cpp:24-105)."""
    ft = CR.S.make_spec("c1").family()
    fam = P.build_perk2(4, [4], [[0.204, 0.42]])
    assert np.array_equal(ft.A, fam.A) and np.array_equal(ft.b, fam.b)
    assert np.array_equal(ft.c, fam.c)


@pytest.mark.parametrize("name", ["c1", "c5"])
def test_cpu_config_initial_state(name):
    """The oracle-side build gives the same nodes and U0 as the product's."""
    sp = CR.S.make_spec(name) if name != "c5" else CR.S.sample_spec(CR.S.make_spec("c5"))
    run = CR.CpuConfig(sp, threads=2)
    cfg = W.make_config(name) if name != "c5" else W.sample_config(W.make_config("c5"))
    x, y, z, _ = run.chk.node_coords()
    U0 = run.initial_state()
    assert np.array_equal(U0, W.initial_state_for(cfg, (x, y, z)))
    assert run.dof_stage_updates_per_step() == \
        W.dof_stage_updates_per_step(cfg.family, cfg.partition_map(), cfg.nodes_per_cell())


def test_reference_arm_does_not_load_the_product():
    """bench.py --impl reference runs the oracle port only (no
    paper_2507_04991_b200 import, no libperrk_b200.so mapping)."""
    code = (
        "import sys, runpy; sys.argv=['bench.py','--impl','reference','--config','c1',"
        "'--steps','2','--warmup','1']; runpy.run_path('bench.py', run_name='__main__');"
        "assert not any(m.startswith('paper_2507') for m in sys.modules), 'product imported';"
        "maps=open('/proc/self/maps').read(); assert 'libperrk_b200' not in maps, 'product .so'")
    r = subprocess.run([sys.executable, "-c", code], cwd=CR.ROOT, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr
    import json
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["config"] == CR.S.bench_config(CR.S.make_spec("c1"))


def test_bench_gpus_n_fails_loudly_without_the_gpus():
    """bench.py --gpus N without a launcher re-executes under torchrun with N
    ranks; with fewer than N visible GPUs it exits 2 (never one silent rank)."""
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1", "--warmup", "0"],
                       cwd=CR.ROOT, capture_output=True, text=True, timeout=300,
                       env={**__import__("os").environ, "CUDA_VISIBLE_DEVICES": ""})
    assert r.returncode == 2, (r.returncode, r.stderr)
    assert "needs 2 visible GPUs" in r.stderr
