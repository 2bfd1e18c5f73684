"""TEST INFRASTRUCTURE — ctypes wrappers of the CPU checkers.

  Ref  -> oracle/_ref/libperrk_ref.so : the unmodified reference library
          (dim 2 only), through oracle/ref_shim.cpp
  Orc  -> oracle/_build/liboracle.so  : the C restatement (perrk_oracle.c),
          dim 2 and 3, accurate relaxation numerics, 2D NSF/BR1 extension

Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline
leg import this module.  Both expose the same small interface so tests can
run either against the GPU path.
"""
import ctypes as C
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libperrk_ref.so")
ORC_LIB = os.path.join(HERE, "_build", "liboracle.so")
FLUX = {"central": 0, "upwind": 1, "rusanov": 2, "hlle": 3, "hll": 3, "hllc": 4, "ec": 5}
KIND = {"p2": 0, "p3": 1, "p3-original": 2, "p4": 3}

_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)


def dp(a):
    return a.ctypes.data_as(_D)


def ip(a):
    return a.ctypes.data_as(_I)


def build():
    """Compile the oracle (and, where /root/reference exists, the reference)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


class Family(C.Structure):  # shared layout of ref_family / orc_family (+kind for ref)
    pass


class RefFamily(C.Structure):
    _fields_ = [("S", C.c_int), ("R", C.c_int), ("kind", C.c_int), ("E", _I), ("A", _D),
                ("b", _D), ("c", _D)]


class OrcFamily(C.Structure):
    _fields_ = [("S", C.c_int), ("R", C.c_int), ("E", _I), ("A", _D), ("b", _D), ("c", _D)]


class RefRelax(C.Structure):
    _fields_ = [("method", C.c_int), ("max_iter", C.c_int), ("residual_tol", C.c_double),
                ("step_tol", C.c_double), ("bracket_min", C.c_double),
                ("bracket_max", C.c_double), ("seed_from_previous", C.c_int)]


class OrcRelax(C.Structure):
    _fields_ = RefRelax._fields_ + [("numerics", C.c_int)]


class StepResult(C.Structure):
    _fields_ = [("gamma", C.c_double), ("iterations", C.c_int), ("residual", C.c_double),
                ("fell_back", C.c_int), ("delta_h", C.c_double), ("aborted", C.c_int),
                ("bad_cell", C.c_int), ("bad_stage", C.c_int)]


class OrcSpec(C.Structure):
    _fields_ = [("dim", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
                ("xe", _D), ("ye", _D), ("ze", _D), ("k", C.c_int), ("gamma", C.c_double),
                ("viscous", C.c_int), ("mu", C.c_double), ("prandtl", C.c_double),
                ("surface_flux", C.c_int), ("volume_mode", C.c_int), ("volume_flux", C.c_int),
                ("threads", C.c_int)]


def _load(path, protos):
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
    L = C.CDLL(path)
    for name, (res, args) in protos.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


_ref = None
_orc = None


def ref_lib():
    global _ref
    if _ref is None:
        _ref = _load(REF_LIB, {
            "ref_last_error": (C.c_char_p, []),
            "ref_create": (C.c_void_p, [C.c_int, _D, C.c_int, _D, C.c_int, C.c_int, C.c_int,
                                        C.c_double, _D, C.c_int, C.c_int, C.c_int]),
            "ref_destroy": (None, [C.c_void_p]),
            "ref_create_nsf1d": (C.c_void_p, [_D, C.c_int, C.c_int, C.c_double, C.c_double,
                                              C.c_double, C.c_int, C.c_int, C.c_int]),
            "ref_num_dofs": (C.c_int, [C.c_void_p]),
            "ref_num_cells": (C.c_int, [C.c_void_p]),
            "ref_set_threads": (None, [C.c_void_p, C.c_int]),
            "ref_rhs_cell_evaluations": (C.c_ulonglong, [C.c_void_p]),
            "ref_reset_counter": (None, [C.c_void_p]),
            "ref_node_coords": (None, [C.c_void_p, _D, _D, _D]),
            "ref_rhs_masked": (C.c_int, [C.c_void_p, C.c_double, _D, _D, C.c_char_p]),
            "ref_total_entropy": (C.c_double, [C.c_void_p, _D]),
            "ref_entropy_inner_product": (C.c_double, [C.c_void_p, _D, _D]),
            "ref_integral_per_variable": (None, [C.c_void_p, _D, _D]),
            "ref_admissible": (C.c_int, [C.c_void_p, _D, _I]),
            "ref_characteristic_speed": (C.c_int, [C.c_void_p, _D, _D]),
            "ref_project_vortex": (C.c_int, [C.c_void_p, _D, C.c_double, _D]),
            "ref_gll": (None, [C.c_int, _D, _D, _D]),
            "ref_error_norms_vortex": (C.c_int, [C.c_void_p, _D, _D, C.c_double, _D, _D]),
            "ref_write_step_log": (C.c_int, [C.c_void_p, C.c_int, _D, C.c_char_p]),
            "ref_write_snapshot": (C.c_int, [C.c_void_p, _D, C.c_char_p]),
            "ref_logmean": (C.c_double, [C.c_double, C.c_double]),
            "ref_numerical_flux": (C.c_int, [C.c_int, C.c_double, C.c_int, _D, _D, C.c_int, _D]),
            "ref_physics_eval": (C.c_int, [C.c_int, C.c_double, _D, C.c_int, _D, _D, _D, _D]),
            "ref_family_build": (C.c_int, [C.c_int, C.c_int, C.c_int, _I, _D, C.c_double, _D,
                                           _D, _D, _I]),
            "ref_family_to_text": (C.c_int, [C.POINTER(RefFamily), C.c_char_p, C.c_int]),
            "ref_assign_levels": (C.c_int, [_D, C.c_int, C.c_int, _I]),
            "ref_make_partition_map": (C.c_int, [C.c_void_p, _I, C.c_int, _I]),
            "ref_update_matrix": (C.c_int, [C.c_void_p, C.POINTER(RefFamily), _I, C.c_double,
                                            C.c_double, _D]),
            "ref_perk_step": (C.c_int, [C.c_void_p, _D, _D, C.c_double, C.POINTER(RefFamily),
                                        _I, C.POINTER(RefRelax), C.c_double, C.c_double,
                                        C.c_int, C.c_double, C.POINTER(StepResult)]),
            "ref_compute_dt": (C.c_double, [C.c_void_p, _D, C.c_int, C.c_double, C.c_double,
                                            C.c_double]),
            "ref_run_steps": (C.c_int, [C.c_void_p, _D, _D, C.c_int, C.POINTER(RefFamily), _I,
                                        C.POINTER(RefRelax), C.c_int, C.c_double, C.c_int,
                                        C.c_int, _D, _D]),
        })
    return _ref


def orc_lib():
    global _orc
    if _orc is None:
        _orc = _load(ORC_LIB, {
            "orc_last_error": (C.c_char_p, []),
            "orc_create": (C.c_void_p, [C.POINTER(OrcSpec)]),
            "orc_destroy": (None, [C.c_void_p]),
            "orc_num_dofs": (C.c_int64, [C.c_void_p]),
            "orc_num_cells": (C.c_int64, [C.c_void_p]),
            "orc_num_vars": (C.c_int, [C.c_void_p]),
            "orc_set_threads": (None, [C.c_void_p, C.c_int]),
            "orc_rhs_cell_evaluations": (C.c_uint64, [C.c_void_p]),
            "orc_reset_counter": (None, [C.c_void_p]),
            "orc_node_coords": (None, [C.c_void_p, _D, _D, _D, _D]),
            "orc_rhs_masked": (C.c_int, [C.c_void_p, C.c_double, _D, _D, C.c_char_p]),
            "orc_br1_gradients": (C.c_int, [C.c_void_p, C.c_double, _D, _D]),
            "orc_total_entropy": (C.c_double, [C.c_void_p, _D]),
            "orc_total_entropy_acc": (C.c_double, [C.c_void_p, _D]),
            "orc_entropy_inner_product": (C.c_double, [C.c_void_p, _D, _D]),
            "orc_integral_per_variable": (None, [C.c_void_p, _D, _D]),
            "orc_admissible": (C.c_int, [C.c_void_p, _D, _I]),
            "orc_characteristic_speed": (None, [C.c_void_p, _D, _D]),
            "orc_compute_dt": (C.c_double, [C.c_void_p, _D, C.c_int, C.c_double, C.c_double,
                                            C.c_double]),
            "orc_perk_step": (C.c_int, [C.c_void_p, _D, _D, C.c_double, C.POINTER(OrcFamily), _I,
                                        C.POINTER(OrcRelax), C.c_double, C.c_double, C.c_int,
                                        C.c_double, C.POINTER(StepResult)]),
            "orc_run_steps": (C.c_int, [C.c_void_p, _D, _D, C.c_int, C.POINTER(OrcFamily), _I,
                                        C.POINTER(OrcRelax), C.c_int, C.c_double, C.c_int,
                                        C.c_int, _D, _D]),
            "orc_gll": (None, [C.c_int, _D, _D, _D]),
            "orc_logmean": (C.c_double, [C.c_double, C.c_double]),
            "orc_numerical_flux": (C.c_int, [C.c_int, C.c_double, C.c_int, _D, _D, C.c_int, _D]),
            "orc_physics_eval": (None, [C.c_int, C.c_double, _D, C.c_int, _D, _D, _D, _D]),
            "orc_entropy_difference": (C.c_double, [C.c_int, C.c_double, _D, _D]),
        })
    return _orc


class _Base:
    """Common interface of Ref / Orc (host numpy arrays)."""

    def _fam(self, fam):
        self._keep = (np.ascontiguousarray(fam.E, dtype=np.int32),
                      np.ascontiguousarray(fam.A, dtype=np.float64),
                      np.ascontiguousarray(fam.b, dtype=np.float64),
                      np.ascontiguousarray(fam.c, dtype=np.float64))
        E, A, b, c = self._keep
        if self.kind == "ref":
            return RefFamily(fam.S, fam.R, KIND[fam.kind], ip(E), dp(A), dp(b), dp(c))
        return OrcFamily(fam.S, fam.R, ip(E), dp(A), dp(b), dp(c))

    def _relax(self, relax):
        if relax is None:
            return None
        m = {"newton": 0, "bisection": 1, "secant": 2}[relax.method]
        base = (m, relax.max_iter, relax.residual_tol, relax.step_tol, relax.bracket_min,
                relax.bracket_max, int(relax.seed_from_previous))
        if self.kind == "ref":
            if relax.numerics != "reference":
                raise ValueError("the reference only has its own relaxation numerics")
            return RefRelax(*base)
        return OrcRelax(*base, {"reference": 0, "accurate": 1}[relax.numerics])

    def rhs(self, t, U):
        return self.rhs_masked(t, U, None)

    def perk_step(self, U, t, dt, fam, eff, relax=None, gamma_seed=1.0, h_ref=math.nan, idt=False,
                  gamma_override=1.0):
        """Advances U (float64, in place); returns (t, StepResult)."""
        f = self._fam(fam)
        eff = np.ascontiguousarray(eff, dtype=np.int32)
        rx = self._relax(relax)
        tt = C.c_double(t)
        res = StepResult()
        fn = self.L.ref_perk_step if self.kind == "ref" else self.L.orc_perk_step
        rc = fn(self.h, dp(U), C.byref(tt), dt, C.byref(f), ip(eff),
                C.byref(rx) if rx is not None else None, gamma_seed, h_ref, int(idt),
                gamma_override, C.byref(res))
        self._check(rc)
        return tt.value, res

    def run_steps(self, U, t, nsteps, fam, eff, relax=None, fixed=False, dt_or_cfl=0.5,
                  anchor=False, records=True):
        """run() loop for exactly nsteps steps; returns (t, taken, log, seconds), log rows
        [t, dt, gamma, iters, H, fell_back, invariants[V]] (+ [delta_h, H_acc] for Orc)."""
        f = self._fam(fam)
        eff = np.ascontiguousarray(eff, dtype=np.int32)
        rx = self._relax(relax)
        tt = C.c_double(t)
        cols = 6 + self.V + (2 if self.kind == "orc" else 0)  # orc adds delta_h, H_acc
        log = np.zeros((max(nsteps, 1), cols))
        secs = C.c_double()
        fn = self.L.ref_run_steps if self.kind == "ref" else self.L.orc_run_steps
        taken = fn(self.h, dp(U), C.byref(tt), nsteps, C.byref(f), ip(eff),
                   C.byref(rx) if rx is not None else None, int(fixed), dt_or_cfl, int(anchor),
                   int(records), dp(log), C.byref(secs))
        if taken < 0:
            self._check(1)
        return tt.value, taken, log[:taken], secs.value


class Ref(_Base):
    kind = "ref"

    def __init__(self, mesh, gamma=1.4, surface_flux="rusanov", volume_flux="ec",
                 volume_mode="flux_differencing", k=3, threads=1):
        self.L = ref_lib()
        if mesh.dim != 2:
            raise ValueError("the reference is 1D/2D only")
        xe = np.ascontiguousarray(mesh.x_edges, dtype=np.float64)
        ye = np.ascontiguousarray(mesh.y_edges, dtype=np.float64)
        self.h = self.L.ref_create(2, dp(xe), xe.size, dp(ye), ye.size, k, 0, gamma, None,
                                   FLUX[surface_flux], int(volume_mode == "flux_differencing"),
                                   FLUX[volume_flux])
        if not self.h:
            raise RuntimeError(self.L.ref_last_error().decode())
        self.V = 4
        self.ndofs = self.L.ref_num_dofs(self.h)
        self.ncells = self.L.ref_num_cells(self.h)
        self.L.ref_set_threads(self.h, threads)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_destroy(self.h)
            self.h = None

    def _check(self, rc):
        if rc:
            raise RuntimeError(self.L.ref_last_error().decode())

    def set_threads(self, n):
        self.L.ref_set_threads(self.h, n)

    def node_coords(self):
        n = self.ndofs // self.V
        x, y, m = np.zeros(n), np.zeros(n), np.zeros(n)
        self.L.ref_node_coords(self.h, dp(x), dp(y), dp(m))
        return x, y, None, m

    def rhs_masked(self, t, U, mask):
        U = np.ascontiguousarray(U, dtype=np.float64)
        out = np.empty_like(U)
        mb = None if mask is None else np.ascontiguousarray(mask, dtype=np.int8).tobytes()
        self._check(self.L.ref_rhs_masked(self.h, t, dp(U), dp(out), mb))
        return out

    def total_entropy(self, U):
        return self.L.ref_total_entropy(self.h, dp(np.ascontiguousarray(U)))

    def entropy_inner_product(self, U, K):
        return self.L.ref_entropy_inner_product(self.h, dp(np.ascontiguousarray(U)),
                                                dp(np.ascontiguousarray(K)))

    def integral_per_variable(self, U):
        out = np.zeros(self.V)
        self.L.ref_integral_per_variable(self.h, dp(np.ascontiguousarray(U)), dp(out))
        return out

    def admissible(self, U):
        bad = C.c_int(-1)
        ok = self.L.ref_admissible(self.h, dp(np.ascontiguousarray(U)), C.byref(bad))
        return bool(ok), bad.value

    def characteristic_speed(self, U):
        nu = np.zeros(self.ncells)
        self._check(self.L.ref_characteristic_speed(self.h, dp(np.ascontiguousarray(U)), dp(nu)))
        return nu

    def compute_dt(self, U, fixed, dt_or_cfl, t=0.0, tf=1e300):
        return self.L.ref_compute_dt(self.h, dp(np.ascontiguousarray(U)), int(fixed), dt_or_cfl,
                                     t, tf)

    def rhs_cell_evaluations(self):
        return self.L.ref_rhs_cell_evaluations(self.h)

    def error_norms_vortex(self, U, params, t):
        pv = np.ascontiguousarray(params, dtype=np.float64)
        l1, li = np.zeros(4), np.zeros(4)
        self._check(self.L.ref_error_norms_vortex(self.h, dp(np.ascontiguousarray(U)), dp(pv), t,
                                                  dp(l1), dp(li)))
        return l1, li


class RefAdvection(Ref):
    """The reference on AdvectionPhysics (physics.hpp:54-85), periodic 1D
    (Mesh1D) or 2D meshes: RHS, perk_step and the update matrix
    (analysis.cpp:11-32, looped in ref_shim.cpp)."""

    def __init__(self, mesh, velocity, surface_flux="upwind", volume_flux="ec",
                 volume_mode="flux_differencing", k=3, threads=1):
        self.L = ref_lib()
        xe = np.ascontiguousarray(mesh.edges[0], dtype=np.float64)
        ye = np.ascontiguousarray(mesh.edges[1] if mesh.dim == 2 else [0.0, 1.0],
                                  dtype=np.float64)
        vel = np.ascontiguousarray(velocity, dtype=np.float64)
        self.h = self.L.ref_create(mesh.dim, dp(xe), xe.size, dp(ye), ye.size, k, 1, 1.4,
                                   dp(vel), FLUX[surface_flux],
                                   int(volume_mode == "flux_differencing"), FLUX[volume_flux])
        if not self.h:
            raise RuntimeError(self.L.ref_last_error().decode())
        self.V = 1
        self.ndofs = self.L.ref_num_dofs(self.h)
        self.ncells = self.L.ref_num_cells(self.h)
        self.L.ref_set_threads(self.h, threads)

    def update_matrix(self, fam, eff, dt, gamma):
        """D (M x M) of one step, D[:, j] = perk_step(e_j)."""
        f = self._fam(fam)
        eff = np.ascontiguousarray(eff, dtype=np.int32)
        M = self.ndofs
        D = np.zeros(M * M)
        self._check(self.L.ref_update_matrix(self.h, C.byref(f), ip(eff), dt, gamma, dp(D)))
        return D.reshape(M, M).T  # column-major -> D[i, j]


class RefNSF1D:
    """The reference's own 1D NSF + BR1 semidiscretization (the oracle's 2D
    NSF extension reduces to it on y-independent data with v = 0)."""

    def __init__(self, x_edges, gamma=1.4, mu=1e-2, prandtl=0.72, surface_flux="rusanov",
                 volume_flux="ec"):
        self.L = ref_lib()
        xe = np.ascontiguousarray(x_edges, dtype=np.float64)
        self.h = self.L.ref_create_nsf1d(dp(xe), xe.size, 3, gamma, mu, prandtl,
                                         FLUX[surface_flux], 1, FLUX[volume_flux])
        if not self.h:
            raise RuntimeError(self.L.ref_last_error().decode())
        self.V = 3
        self.ndofs = self.L.ref_num_dofs(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_destroy(self.h)
            self.h = None

    def node_coords(self):
        n = self.ndofs // self.V
        x, y, m = np.zeros(n), np.zeros(n), np.zeros(n)
        self.L.ref_node_coords(self.h, dp(x), dp(y), dp(m))
        return x

    def rhs(self, t, U):
        U = np.ascontiguousarray(U, dtype=np.float64)
        out = np.empty_like(U)
        if self.L.ref_rhs_masked(self.h, t, dp(U), dp(out), None):
            raise RuntimeError(self.L.ref_last_error().decode())
        return out


class Orc(_Base):
    kind = "orc"

    def __init__(self, mesh, gamma=1.4, surface_flux="rusanov", volume_flux="ec",
                 volume_mode="flux_differencing", k=3, threads=1, viscous=False, mu=0.0,
                 prandtl=0.72):
        self.L = orc_lib()
        self._edges = [np.ascontiguousarray(e, dtype=np.float64) for e in mesh.edges]
        s = OrcSpec()
        s.dim = mesh.dim
        s.nx = self._edges[0].size - 1
        s.ny = self._edges[1].size - 1
        s.nz = self._edges[2].size - 1 if mesh.dim == 3 else 1
        s.xe = dp(self._edges[0])
        s.ye = dp(self._edges[1])
        s.ze = dp(self._edges[2]) if mesh.dim == 3 else None
        s.k = k
        s.gamma = gamma
        s.viscous = int(viscous)
        s.mu = mu
        s.prandtl = prandtl
        s.surface_flux = FLUX[surface_flux]
        s.volume_mode = int(volume_mode == "flux_differencing")
        s.volume_flux = FLUX[volume_flux]
        s.threads = threads
        self.h = self.L.orc_create(C.byref(s))
        if not self.h:
            raise RuntimeError(self.L.orc_last_error().decode())
        self.dim = mesh.dim
        self.V = self.L.orc_num_vars(self.h)
        self.ndofs = self.L.orc_num_dofs(self.h)
        self.ncells = self.L.orc_num_cells(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.orc_destroy(self.h)
            self.h = None

    def _check(self, rc):
        if rc:
            raise RuntimeError(self.L.orc_last_error().decode())

    def set_threads(self, n):
        self.L.orc_set_threads(self.h, n)

    def node_coords(self):
        n = self.ndofs // self.V
        x, y, z, m = np.zeros(n), np.zeros(n), np.zeros(n), np.zeros(n)
        self.L.orc_node_coords(self.h, dp(x), dp(y), dp(z), dp(m))
        return x, y, (z if self.dim == 3 else None), m

    def rhs_masked(self, t, U, mask):
        U = np.ascontiguousarray(U, dtype=np.float64)
        out = np.empty_like(U)
        mb = None if mask is None else np.ascontiguousarray(mask, dtype=np.int8).tobytes()
        self._check(self.L.orc_rhs_masked(self.h, t, dp(U), dp(out), mb))
        return out

    def br1_gradients(self, t, U):
        U = np.ascontiguousarray(U, dtype=np.float64)
        g = np.zeros(2 * U.size)
        self._check(self.L.orc_br1_gradients(self.h, t, dp(U), dp(g)))
        return g.reshape(2, -1)

    def total_entropy(self, U):
        return self.L.orc_total_entropy(self.h, dp(np.ascontiguousarray(U)))

    def total_entropy_acc(self, U):
        """total_entropy as a compensated sum (accurate numerics)."""
        return self.L.orc_total_entropy_acc(self.h, dp(np.ascontiguousarray(U)))

    def entropy_inner_product(self, U, K):
        return self.L.orc_entropy_inner_product(self.h, dp(np.ascontiguousarray(U)),
                                                dp(np.ascontiguousarray(K)))

    def integral_per_variable(self, U):
        out = np.zeros(self.V)
        self.L.orc_integral_per_variable(self.h, dp(np.ascontiguousarray(U)), dp(out))
        return out

    def admissible(self, U):
        bad = C.c_int(-1)
        ok = self.L.orc_admissible(self.h, dp(np.ascontiguousarray(U)), C.byref(bad))
        return bool(ok), bad.value

    def characteristic_speed(self, U):
        nu = np.zeros(self.ncells)
        self.L.orc_characteristic_speed(self.h, dp(np.ascontiguousarray(U)), dp(nu))
        return nu

    def compute_dt(self, U, fixed, dt_or_cfl, t=0.0, tf=1e300):
        return self.L.orc_compute_dt(self.h, dp(np.ascontiguousarray(U)), int(fixed), dt_or_cfl,
                                     t, tf)

    def rhs_cell_evaluations(self):
        return self.L.orc_rhs_cell_evaluations(self.h)
