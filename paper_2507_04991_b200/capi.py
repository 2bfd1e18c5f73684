"""ctypes declarations of the C-ABI in include/perrk_b200.h.

This is the binding a maintainer of a Python host would add; INTEGRATION.md
shows it beside the C++ one.  Loading fails loudly when the CUDA library is
missing: there is no CPU fallback.
"""
import ctypes as C
import os

from . import build as _build

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libperrk_b200.so")

FLUX = {"central": 0, "upwind": 1, "godunov": 1, "rusanov": 2, "llf": 2, "hlle": 3,
        "hll": 3, "hllc": 4, "ec": 5, "ranocha": 5}
FAMILY = {"p2": 0, "p3": 1, "p3-variant": 1, "p3-original": 2, "p4": 3}

PERRK_OK, PERRK_EINVAL, PERRK_ECUDA, PERRK_EUNSUP, PERRK_ENUMERIC, PERRK_ECOMM = 0, -1, -2, -3, -4, -5


class SemiDesc(C.Structure):
    _fields_ = [("dim", C.c_int), ("n", C.c_int * 3), ("edges", C.POINTER(C.c_double) * 3),
                ("polydeg", C.c_int), ("physics", C.c_int), ("gamma", C.c_double),
                ("mu", C.c_double), ("prandtl", C.c_double), ("surface_flux", C.c_int),
                ("volume_mode", C.c_int), ("volume_flux", C.c_int), ("device", C.c_int)]


class FamilyDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("S", C.c_int), ("R", C.c_int), ("E", C.POINTER(C.c_int)),
                ("A", C.POINTER(C.c_double)), ("b", C.POINTER(C.c_double)),
                ("c", C.POINTER(C.c_double))]


class AdvectionDesc(C.Structure):
    _fields_ = [("dim", C.c_int), ("n", C.c_int * 2), ("edges", C.POINTER(C.c_double) * 2),
                ("velocity", C.c_double * 2), ("surface_flux", C.c_int),
                ("volume_mode", C.c_int), ("volume_flux", C.c_int), ("device", C.c_int)]


class RelaxCfg(C.Structure):
    _fields_ = [("method", C.c_int), ("max_iter", C.c_int), ("residual_tol", C.c_double),
                ("step_tol", C.c_double), ("bracket_min", C.c_double),
                ("bracket_max", C.c_double), ("seed_from_previous", C.c_int),
                ("numerics", C.c_int)]


class StepOpts(C.Structure):
    _fields_ = [("relax_enabled", C.c_int), ("relax", RelaxCfg), ("gamma_override", C.c_double),
                ("gamma_seed", C.c_double), ("h_ref", C.c_double), ("idt", C.c_int)]


class StepResult(C.Structure):
    _fields_ = [("gamma", C.c_double), ("iterations", C.c_int), ("residual", C.c_double),
                ("fell_back", C.c_int), ("delta_h", C.c_double), ("aborted", C.c_int),
                ("bad_cell", C.c_int), ("bad_stage", C.c_int)]


class RunCfg(C.Structure):
    _fields_ = [("fixed_dt", C.c_int), ("dt_or_cfl", C.c_double), ("tf", C.c_double),
                ("relax_enabled", C.c_int), ("relax", RelaxCfg), ("anchor_initial", C.c_int),
                ("idt", C.c_int), ("records", C.c_int), ("cfl0", C.c_double),
                ("t_ramp", C.c_double), ("t0", C.c_double), ("carry", C.c_int),
                ("gamma_seed", C.c_double), ("h_anchor", C.c_double)]


class StepRecord(C.Structure):
    _fields_ = [("t", C.c_double), ("dt", C.c_double), ("gamma", C.c_double),
                ("newton_iters", C.c_int), ("fell_back", C.c_int), ("entropy", C.c_double),
                ("invariants", C.c_double * 5), ("delta_h", C.c_double)]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)
_PROTOS = {
    "perrk_last_error": (C.c_char_p, []),
    "perrk_abi_version": (C.c_int, []),
    "perrk_create": (C.c_int, [C.POINTER(SemiDesc), C.POINTER(_P)]),
    "perrk_destroy": (C.c_int, [_P]),
    "perrk_sizes": (C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                              C.POINTER(C.c_int64), _I, _I]),
    "perrk_node_geometry": (C.c_int, [_P, _D, _D, _D, _D]),
    "perrk_set_family": (C.c_int, [_P, C.POINTER(FamilyDesc), _I]),
    "perrk_upload_state": (C.c_int, [_P, _D, C.c_size_t]),
    "perrk_download_state": (C.c_int, [_P, _D, C.c_size_t]),
    "perrk_state_device_ptr": (C.c_int, [_P, C.POINTER(_D)]),
    "perrk_sync": (C.c_int, [_P]),
    "perrk_rhs_masked": (C.c_int, [_P, C.c_double, _D, _D, C.c_char_p]),
    "perrk_probe_jacobian": (C.c_int, [_P, _D, C.c_double, C.c_double, _D, _I]),
    "perrk_br1_gradients": (C.c_int, [_P, C.c_double, _D, _D]),
    "perrk_total_entropy": (C.c_int, [_P, _D, _D]),
    "perrk_entropy_inner_product": (C.c_int, [_P, _D, _D, _D]),
    "perrk_integral_per_variable": (C.c_int, [_P, _D, _D]),
    "perrk_admissible": (C.c_int, [_P, _D, _I, _I]),
    "perrk_characteristic_speed": (C.c_int, [_P, _D, _D]),
    "perrk_compute_dt": (C.c_int, [_P, _D, C.c_int, C.c_double, C.c_double, C.c_double, _D]),
    "perrk_perk_step": (C.c_int, [_P, _D, _D, C.c_double, C.POINTER(StepOpts),
                                  C.POINTER(StepResult)]),
    "perrk_perk_step_resident": (C.c_int, [_P, _D, C.c_double, C.POINTER(StepOpts),
                                           C.POINTER(StepResult)]),
    "perrk_advance": (C.c_int, [_P, C.POINTER(RunCfg), _D, C.c_int, C.POINTER(StepRecord),
                                _I, _I]),
    "perrk_krylov_hessenberg": (C.c_int, [_P, _D, C.c_double, C.c_double, C.c_int, C.c_char_p,
                                          _D, _I]),
    "perrk_error_norms": (C.c_int, [_P, _D, C.c_int, _D, C.c_double, _D, _D]),
    "perrk_rhs_cell_evaluations": (C.c_int, [_P, C.POINTER(C.c_uint64)]),
    "perrk_reset_counter": (C.c_int, [_P]),
    "perrk_family_build": (C.c_int, [C.c_int, C.c_int, C.c_int, _I, _D, C.c_double, _D, _D, _D,
                                     _I]),
    "perrk_assign_levels": (C.c_int, [_D, C.c_int64, C.c_int, _I]),
    "perrk_make_partition_map": (C.c_int, [C.c_int, _I, _I, C.c_int, _I]),
    "perrk_set_stream": (C.c_int, [_P, C.c_void_p]),
    "perrk_profile": (C.c_int, [_P, C.c_int]),
    "perrk_profile_read": (C.c_int, [_P, _D, C.POINTER(C.c_int64), _D]),
    "perrk_launch_count": (C.c_int, [_P, C.POINTER(C.c_int64)]),
    "perrk_step_traffic": (C.c_int, [_P, _D, _D, _D]),
    "perrk_fp64_peak": (C.c_int, [C.c_int, _D]),
    "perrk_update_matrix": (C.c_int, [C.POINTER(AdvectionDesc), C.POINTER(FamilyDesc), _I,
                                      C.c_double, C.c_double, _D, C.POINTER(C.c_int64)]),
    "perrk_nccl_id": (C.c_int, [C.c_void_p]),
    "perrk_comm_init": (C.c_int, [_P, C.c_void_p, C.c_int, C.c_int, _I]),
    "perrk_local_cells": (C.c_int, [_P, _I, C.POINTER(C.c_int64)]),
    "perrk_loopback_group": (C.c_int, [C.POINTER(_P), C.c_int, _I]),
    "perrk_partition_slabs": (C.c_int, [C.c_int, _I, _D, C.c_int, _I]),
    "perrk_partition_levels": (C.c_int, [C.c_int, _I, _I, C.c_int, C.c_int, _I]),
    "perrk_halo_plan": (C.c_int, [C.c_int, _I, _I, C.c_int, C.POINTER(C.c_int64), _I, _I,
                                  C.POINTER(C.c_int64), _I, C.POINTER(C.c_int64),
                                  C.POINTER(C.c_int64), _I]),
    "perrk_face_nodes": (C.c_int, [C.c_int, C.c_int, _I]),
}
EXPORTED = tuple(_PROTOS)

_lib = None


class PerrkError(RuntimeError):
    """Mirrors perrk::Error (common.hpp:15-18); .code holds the C status."""

    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def lib():
    """Load libperrk_b200.so (building it first if sources are newer)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH) or _build._stale():
            _build.build()
        if not os.path.exists(LIB_PATH):
            raise ImportError("libperrk_b200.so is missing and could not be built")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _PROTOS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc):
    if rc != PERRK_OK:
        raise PerrkError(rc, lib().perrk_last_error().decode())
    return rc
