"""CPU: the C-ABI library loads, exports every symbol include/perrk_b200.h
declares, and its host-side helpers (no device work) match the reference:
  perrk_family_build        butcher.cpp:51-247 (build_perk2/3/4)
  perrk_assign_levels       mesh.cpp:73-95
  perrk_make_partition_map  mesh.cpp:56-71
plus the error contract (status codes + perrk_last_error instead of the
reference's perrk::Error throws, common.hpp:15-23).
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
from conftest import HAS_GPU, HAS_REF_LIB, ROOT
from paper_2507_04991_b200 import capi
from paper_2507_04991_b200 import perrk as P
from paper_2507_04991_b200 import workloads as W

need_ref = pytest.mark.skipif(not HAS_REF_LIB, reason="oracle/_ref not built")


def header_symbols():
    src = open(os.path.join(ROOT, "include", "perrk_b200.h")).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(perrk_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    L = capi.lib()
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(capi.EXPORTED)
    assert L.perrk_abi_version() == 2


def test_library_is_cuda_code():
    """The product library carries sm_100a device code (no CPU fallback)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", capi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(HAS_GPU, reason="checks the no-device error path")
def test_create_without_device_fails_loudly():
    with pytest.raises(P.Error) as e:
        P.Semidiscretization(P.SemidiscretizationSpec(P.build_uniform_mesh2d(1.0, 2)))
    assert e.value.code in (capi.PERRK_ECUDA, capi.PERRK_EINVAL)


def test_error_contract():
    L = capi.lib()
    assert L.perrk_create(None, None) == capi.PERRK_EINVAL
    assert b"null" in L.perrk_last_error()
    with pytest.raises(P.Error, match="E must be strictly increasing"):
        P.build_perk2(4, [4, 3], [[0.2, 0.3], [0.1]])
    with pytest.raises(P.Error, match="negative first-column"):
        P.build_perk2(4, [4], [[0.9, 0.35]])
    with pytest.raises(P.Error, match="speeds must be positive"):
        P.assign_levels([1.0, 0.0], 2)


@need_ref
@pytest.mark.parametrize("kind,S,E,free", [
    ("p2", 4, [4], [[0.2, 0.35]]),
    ("p2", 6, [3, 6], [[0.1], [0.1, 0.2, 0.3, 0.4]]),
    ("p3", 7, [4, 7], [[0.3], [0.2, 0.25, 0.3, 0.35]]),
    ("p3-original", 8, [4, 8], [[0.3], [0.2, 0.25, 0.3, 0.35, 0.1]]),
    ("p4", 14, [5, 8, 14], [[], [0.5] * 3, [0.7] * 9]),
    ("p4", 16, [5, 9, 16], [[], [0.4] * 4, [0.6] * 11]),
])
def test_family_build_bitwise_vs_reference(kind, S, E, free):
    fam = P.build_family(kind, S, E, free)
    R = len(E)
    Ea = np.array(E, np.int32)
    fr = np.array([x for f in free for x in f] or [0.0])
    A, b, c = np.zeros((R, S, S)), np.zeros(S), np.zeros(S)
    act = np.zeros((R, S), np.int32)
    assert O.ref_lib().ref_family_build(O.KIND[kind], S, R, O.ip(Ea), O.dp(fr), 1.0, O.dp(A),
                                        O.dp(b), O.dp(c), O.ip(act)) == 0
    assert np.array_equal(fam.A, A) and np.array_equal(fam.b, b) and np.array_equal(fam.c, c)
    for r in range(R):
        assert fam.active_sets[r] == set(np.nonzero(act[r])[0].tolist())
        assert len(fam.active_sets[r]) == E[r]


def test_family_text_roundtrip_and_fixtures():
    fam = P.build_perk4(14, [5, 8, 14], [[], [0.5] * 3, [0.7] * 9])
    back = P.family_from_text(P.family_to_text(fam))
    assert np.array_equal(back.A, fam.A) and back.E == fam.E and back.kind == "p4"
    for name in ("c2_p3_4_7", "c3_p4_5_9_16", "c4_p3_4_8", "c5_p4_5_8_14"):
        f = W.load_config_family(name)
        rebuilt = P.build_family(f.kind, f.S, f.E, [
            [f.A[r, i, i - 1] for i in range(f.S - f.E[r] + 2,
                                              f.S - {"p2": 0, "p3": 1, "p4": 3}[f.kind])]
            for r in range(f.R)])
        assert np.allclose(rebuilt.A, f.A, atol=1e-15, rtol=1e-15)
        for r in range(f.R):
            assert len(f.active_sets[r]) == f.E[r]


@need_ref
def test_assign_levels_and_partition_map_vs_reference():
    rng = np.random.default_rng(3)
    nu = rng.uniform(0.1, 8.0, 300)
    for R in (1, 2, 3, 4):
        got = P.assign_levels(nu, R)
        want = np.zeros(nu.size, np.int32)
        assert O.ref_lib().ref_assign_levels(O.dp(nu), nu.size, R, O.ip(want)) == 0
        assert np.array_equal(got, want)
    mesh = P.Mesh2DRect(W.banded_edges(0, [(5, 1.0), (4, 0.5)]), W.banded_edges(0, [(7, 1.0)]))
    ref = O.Ref(mesh)
    for R in (2, 3):
        lv = rng.integers(1, R + 1, mesh.num_cells()).astype(np.int32)
        got = P.make_partition_map(mesh, lv, R).effective_level
        want = np.zeros_like(lv)
        assert O.ref_lib().ref_make_partition_map(ref.h, O.ip(lv), R, O.ip(want)) == 0
        assert np.array_equal(got, want)


def test_dof_stage_count_matches_active_sets():
    cfg = W.make_config("c5")
    pm = cfg.partition_map()
    counts = pm.cells_per_level()
    assert sum(counts) == 64 ** 3 and all(c > 0 for c in counts)
    per_step = W.dof_stage_updates_per_step(cfg.family, pm, 64)
    manual = sum(len(cfg.family.active_sets[cfg.family.member_index_for_level(lv)]) * n * 64
                 for lv, n in enumerate(counts, start=1))
    assert per_step == manual
    assert 5 * 64 ** 4 <= per_step <= 14 * 64 ** 4


def test_cpp_adapter_fails_loudly_without_device():
    """include/perrk_b200.hpp compiled against the reference headers/objects
    (oracle/_ref/adapter_parity): with no CUDA device the drop-in throws
    perrk::Error instead of falling back to the CPU."""
    import subprocess
    exe = os.path.join(ROOT, "oracle", "_ref", "adapter_parity")
    if not os.path.exists(exe):
        pytest.skip("adapter_parity not built (make -C oracle adapter)")
    if HAS_GPU:
        pytest.skip("device present: covered by the gpu parity test")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 3, r.stdout + r.stderr


def test_update_matrix_size_query_and_flux_errors_without_device():
    """perrk_update_matrix (analysis.cpp:11-32): D = NULL queries M; HLLE/HLLC
    are rejected for advection as in the reference (physics.cpp:73-78)."""
    mesh = P.build_two_level_advection_mesh()
    assert mesh.num_cells() == 20
    assert np.allclose(np.diff(mesh.edges[0])[:6], 0.5) and np.allclose(np.diff(mesh.edges[0])[6:14], 0.25)
    spec = P.AdvectionSpec(mesh, [1.0])
    d, keep = P._adv_desc(spec)
    M = C.c_int64()
    assert capi.lib().perrk_update_matrix(C.byref(d), None, None, 0.1, 1.0, None, C.byref(M)) == 0
    assert M.value == 80 == spec.num_dofs()
    for bad in ("hlle", "hllc"):
        d, keep = P._adv_desc(P.AdvectionSpec(mesh, [1.0], surface_flux=bad))
        rc = capi.lib().perrk_update_matrix(C.byref(d), None, None, 0.1, 1.0, None, C.byref(M))
        assert rc == capi.PERRK_EINVAL and b"not available" in capi.lib().perrk_last_error()
    d, keep = P._adv_desc(P.AdvectionSpec(mesh, [1.0], volume_flux="rusanov"))
    assert capi.lib().perrk_update_matrix(C.byref(d), None, None, 0.1, 1.0, None,
                                          C.byref(M)) == capi.PERRK_EINVAL
    with pytest.raises(P.Error):
        P._adv_desc(P.AdvectionSpec(mesh, [1.0, 2.0]))
    pm = P.make_partition_map(mesh, [2] * 6 + [1] * 8 + [2] * 6, 2)
    assert list(pm.effective_level) == [2] * 5 + [1] * 10 + [2] * 5
