"""Python mirror of the reference's solver/integrator API for the hot path.

Names, argument meanings and error behaviour follow the reference's C++ API
(proj/core/include/perrk/*.hpp), so parity tests read like the reference's
own tests.  All compute runs in libperrk_b200.so on the GPU through the C-ABI
(include/perrk_b200.h); this module only marshals arguments.

Reference interfaces mirrored here:
  Mesh2DRect / build_uniform_mesh2d / build_vortex_mesh   mesh.hpp:22-83
  Mesh3DRect                                               (3D extension)
  SemidiscretizationSpec / Semidiscretization              semidisc.hpp:24-113
  PartitionFamily + build_perk2/3/4, family text I/O       butcher.hpp:36-125
  PartitionMap / make_partition_map / assign_levels        mesh.hpp:44-76
  RelaxationConfig / PerkStepOptions / PerkStepResult      relax.hpp:16-31, stepper.hpp:54-68
  perk_step / compute_dt / run                             stepper.hpp:72-99
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import capi
from .capi import check, lib

Error = capi.PerrkError


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------
# meshes (mesh.hpp:22-33 plus the 3D extension), periodic rectilinear
# ---------------------------------------------------------------------------
@dataclass
class Mesh1D:
    """Periodic 1D mesh (mesh.hpp:13-20); only the advection update-matrix
    engine (perrk_update_matrix) runs 1D."""
    x_edges: Sequence[float]
    periodic: bool = True

    @property
    def dim(self):
        return 1

    @property
    def edges(self):
        return [np.asarray(self.x_edges, float)]

    def num_cells(self):
        return len(self.x_edges) - 1

    def shape(self):
        return (self.num_cells(),)


def build_uniform_mesh1d(x0, x1, n, periodic=True):
    return Mesh1D(_uniform_edges(x0, x1, n), periodic)


def build_two_level_advection_mesh():
    """mesh.cpp:151-159: [-4, 4], h = 1/2 outside [-1, 1], 1/4 inside."""
    e = [-4.0]
    for a, b, n in ((-4.0, -1.0, 6), (-1.0, 1.0, 8), (1.0, 4.0, 6)):
        e += _uniform_edges(a, b, n)[1:]
    return Mesh1D(e, True)


@dataclass
class Mesh2DRect:
    x_edges: Sequence[float]
    y_edges: Sequence[float]

    @property
    def dim(self):
        return 2

    @property
    def edges(self):
        return [np.asarray(self.x_edges, float), np.asarray(self.y_edges, float)]

    def nx(self):
        return len(self.x_edges) - 1

    def ny(self):
        return len(self.y_edges) - 1

    def num_cells(self):
        return self.nx() * self.ny()

    def shape(self):
        return (self.nx(), self.ny())


@dataclass
class Mesh3DRect:
    x_edges: Sequence[float]
    y_edges: Sequence[float]
    z_edges: Sequence[float]

    @property
    def dim(self):
        return 3

    @property
    def edges(self):
        return [np.asarray(e, float) for e in (self.x_edges, self.y_edges, self.z_edges)]

    def num_cells(self):
        return (len(self.x_edges) - 1) * (len(self.y_edges) - 1) * (len(self.z_edges) - 1)

    def shape(self):
        return tuple(len(e) - 1 for e in (self.x_edges, self.y_edges, self.z_edges))


def _uniform_edges(a, b, n):
    # append_uniform (mesh.cpp:137-141): from + (to - from) * i / n
    return [a] + [a + (b - a) * i / n for i in range(1, n + 1)]


def build_uniform_mesh2d(half_width, n):
    e = _uniform_edges(-half_width, half_width, n)
    return Mesh2DRect(e, list(e))


def build_uniform_mesh3d(lo, hi, n):
    e = _uniform_edges(lo, hi, n)
    return Mesh3DRect(e, list(e), list(e))


def mesh_num_cells(mesh):
    return mesh.num_cells()


# ---------------------------------------------------------------------------
# semidiscretization
# ---------------------------------------------------------------------------
@dataclass
class SemidiscretizationSpec:
    mesh: object
    polydeg: int = 3
    gamma: float = 1.4
    physics: str = "euler"          # "euler" | "nsf"
    mu: float = 0.0
    prandtl: float = 0.72
    surface_flux: str = "rusanov"
    volume_mode: str = "flux_differencing"
    volume_flux: str = "ec"
    device: int = 0


class Semidiscretization:
    """GPU-resident Semidiscretization (semidisc.hpp:40-113)."""

    def __init__(self, spec: SemidiscretizationSpec):
        self.spec = spec
        mesh = spec.mesh
        self._edges = [_f64(e) for e in mesh.edges]
        d = capi.SemiDesc()
        d.dim = mesh.dim
        for a, e in enumerate(self._edges):
            d.n[a] = len(e) - 1
            d.edges[a] = _dp(e)
        d.polydeg = spec.polydeg
        d.physics = {"euler": 0, "nsf": 1}[spec.physics]
        d.gamma = spec.gamma
        d.mu = spec.mu
        d.prandtl = spec.prandtl
        d.surface_flux = capi.FLUX[spec.surface_flux]
        d.volume_mode = {"weak": 0, "flux_differencing": 1}[spec.volume_mode]
        d.volume_flux = capi.FLUX[spec.volume_flux]
        d.device = spec.device
        h = C.c_void_p()
        check(lib().perrk_create(C.byref(d), C.byref(h)))
        self._h = h
        dofs, nodes, cells = C.c_int64(), C.c_int64(), C.c_int64()
        v, npc = C.c_int(), C.c_int()
        check(lib().perrk_sizes(h, C.byref(dofs), C.byref(nodes), C.byref(cells), C.byref(v),
                                C.byref(npc)))
        self._n = (dofs.value, nodes.value, cells.value, v.value, npc.value)
        self._family_key = None
        self._geom = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().perrk_destroy(h)
            self._h = None

    # sizes (semidisc.hpp:44-49)
    def num_dofs(self):
        return self._n[0]

    def num_nodes(self):
        return self._n[1]

    def num_cells(self):
        return self._n[2]

    def num_vars(self):
        return self._n[3]

    def nodes_per_cell(self):
        return self._n[4]

    def dim(self):
        return self.spec.mesh.dim

    def mesh(self):
        return self.spec.mesh

    def _geometry(self):
        if self._geom is None:
            n = self.num_nodes()
            x, y, z, m = (np.zeros(n) for _ in range(4))
            check(lib().perrk_node_geometry(self._h, _dp(x), _dp(y), _dp(z), _dp(m)))
            self._geom = (x, y, z, m)
        return self._geom

    def node_x(self):
        return self._geometry()[0]

    def node_y(self):
        return self._geometry()[1]

    def node_z(self):
        return self._geometry()[2]

    def node_measure(self):
        return self._geometry()[3]

    def _state(self, U):
        U = _f64(U)
        if U.size != self.num_dofs():
            raise Error(capi.PERRK_EINVAL, "state size mismatch")
        return U

    # RHS (semidisc.cpp:121-147)
    def rhs(self, t, U):
        return self.rhs_masked(t, U, None)

    def rhs_masked(self, t, U, mask):
        U = self._state(U)
        out = np.empty_like(U)
        mb = None
        if mask is not None:
            m = np.ascontiguousarray(mask, dtype=np.int8)
            if m.size != self.num_cells():
                raise Error(capi.PERRK_EINVAL, "mask size mismatch")
            mb = m.tobytes()
        check(lib().perrk_rhs_masked(self._h, float(t), _dp(U), _dp(out), mb))
        return out

    def probe_jacobian(self, base, t=0.0, epsilon=1e-6, return_colours=False):
        """probe_jacobian (specopt.cpp:18-35): dense central-difference
        Jacobian of the RHS, M x M with J[i, j] = d rhs_i / d u_j, guarded to
        M <= 5000.  Probed on the device in cell colours (include/perrk_b200.h)."""
        U = self._state(base)
        M = U.size
        if M > 5000:
            raise Error(capi.PERRK_EINVAL, "dense Jacobian probing guarded to M <= 5000")
        Jc = np.empty(M * M)
        ncol = C.c_int(0)
        check(lib().perrk_probe_jacobian(self._h, _dp(U), float(t), float(epsilon), _dp(Jc),
                                         C.byref(ncol)))
        J = Jc.reshape(M, M).T  # column-major storage
        return (J, ncol.value) if return_colours else J

    def krylov_hessenberg(self, base=None, m=60, t=0.0, epsilon=1e-6, cell_mask=None):
        """Matrix-free spectrum estimation (
        perrk_krylov_hessenberg): m Arnoldi steps on the central-difference
        Jacobian-vector product of the RHS at `base` (None: the resident
        state), on the device.  cell_mask (per cell, nonzero = on) restricts
        the operator to those cells.  Returns the (m_done + 1) x m_done
        Hessenberg matrix."""
        Up = None if base is None else _dp(self._state(base))
        H = np.zeros((m + 1) * m)
        done = C.c_int(0)
        mb = None
        if cell_mask is not None:
            mk = np.ascontiguousarray(cell_mask, dtype=np.int8)
            if mk.size != self.num_cells():
                raise Error(capi.PERRK_EINVAL, "cell mask size must equal the cell count")
            mb = mk.tobytes()
        check(lib().perrk_krylov_hessenberg(self._h, Up, float(t), float(epsilon), int(m), mb,
                                            _dp(H), C.byref(done)))
        k = done.value
        return H.reshape(m, m + 1).T[: k + 1, :k]

    def br1_gradients(self, t, U):
        """BR1 auxiliary gradients (semidisc.hpp:75), NSF physics: [dim][dofs]."""
        U = self._state(U)
        g = np.empty(2 * U.size)
        check(lib().perrk_br1_gradients(self._h, float(t), _dp(U), _dp(g)))
        return g.reshape(2, -1)

    def error_norms_vortex(self, U, params, t):
        """error_norms (stepper.cpp:195-265) against the isentropic vortex
        (physics.cpp:301-328); params: workloads.VortexParams.  U None: the
        resident state.  Returns (l1[V], linf[V])."""
        pv = _f64(params.as_array())
        l1, li = np.zeros(4), np.zeros(4)
        Up = None if U is None else _dp(self._state(U))
        check(lib().perrk_error_norms(self._h, Up, 0, _dp(pv), float(t), _dp(l1), _dp(li)))
        return l1, li

    def rhs_partition_restricted(self, t, U, pmap, level):
        mask = (np.asarray(pmap.effective_level) == level).astype(np.int8)
        return self.rhs_masked(t, U, mask)

    # reductions (semidisc.cpp:561-607)
    def total_entropy(self, U):
        out = C.c_double()
        check(lib().perrk_total_entropy(self._h, _dp(self._state(U)), C.byref(out)))
        return out.value

    def entropy_inner_product(self, U, K):
        out = C.c_double()
        check(lib().perrk_entropy_inner_product(self._h, _dp(self._state(U)), _dp(self._state(K)),
                                                C.byref(out)))
        return out.value

    def integral_per_variable(self, U):
        out = np.zeros(5)
        check(lib().perrk_integral_per_variable(self._h, _dp(self._state(U)), _dp(out)))
        return out[: self.num_vars()]

    def admissible(self, U):
        ok, bad = C.c_int(), C.c_int()
        check(lib().perrk_admissible(self._h, _dp(self._state(U)), C.byref(ok), C.byref(bad)))
        return bool(ok.value), bad.value

    def characteristic_speed(self, U):
        nu = np.zeros(self.num_cells())
        check(lib().perrk_characteristic_speed(self._h, _dp(self._state(U)), _dp(nu)))
        return nu

    def project(self, fn: Callable):
        """semidisc.cpp:588-594 on the host: fn(x, y[, z]) -> (V, n) array."""
        x, y, z, _ = self._geometry()
        args = (x, y) if self.dim() == 2 else (x, y, z)
        vals = np.asarray(fn(*args), dtype=np.float64)
        return np.ascontiguousarray(vals.T).reshape(-1)

    def rhs_cell_evaluations(self):
        out = C.c_uint64()
        check(lib().perrk_rhs_cell_evaluations(self._h, C.byref(out)))
        return out.value

    def reset_evaluation_counter(self):
        check(lib().perrk_reset_counter(self._h))

    # resident state
    def upload(self, U):
        U = self._state(U)
        check(lib().perrk_upload_state(self._h, _dp(U), U.size))

    def download(self, out=None):
        out = np.empty(self.num_dofs()) if out is None else out
        check(lib().perrk_download_state(self._h, _dp(out), out.size))
        return out

    def device_state_ptr(self):
        p = C.POINTER(C.c_double)()
        check(lib().perrk_state_device_ptr(self._h, C.byref(p)))
        return C.cast(p, C.c_void_p).value

    def sync(self):
        check(lib().perrk_sync(self._h))

    # element partition (perrk_comm_init, include/perrk_b200.h)
    def _refresh_sizes(self):
        dofs, nodes, cells = C.c_int64(), C.c_int64(), C.c_int64()
        v, npc = C.c_int(), C.c_int()
        check(lib().perrk_sizes(self._h, C.byref(dofs), C.byref(nodes), C.byref(cells), C.byref(v),
                                C.byref(npc)))
        self._n = (dofs.value, nodes.value, cells.value, v.value, npc.value)
        self._geom = None
        self._family_key = None
        self._cells = None

    def comm_init(self, nccl_id: bytes, rank: int, nranks: int, owner=None):
        """Own the cells `owner` (global cell -> rank; None: uniform last-axis
        slabs) gives `rank` (one process per GPU)."""
        ow = None if owner is None else np.ascontiguousarray(owner, dtype=np.int32)
        buf = C.create_string_buffer(bytes(nccl_id), 128)
        check(lib().perrk_comm_init(self._h, buf, int(rank), int(nranks),
                                    None if ow is None else _ip(ow)))
        self._refresh_sizes()

    def local_cells(self):
        """Global ids of this context's cells (ascending; the local cell order)."""
        if getattr(self, "_cells", None) is None:
            n = C.c_int64()
            check(lib().perrk_local_cells(self._h, None, C.byref(n)))
            out = np.zeros(n.value, dtype=np.int32)
            check(lib().perrk_local_cells(self._h, _ip(out), C.byref(n)))
            self._cells = out
        return self._cells

    def global_num_cells(self):
        return self.spec.mesh.num_cells()

    # instrumentation (perrk_set_stream / perrk_profile*, include/perrk_b200.h)
    def set_stream(self, cuda_stream):
        """Order this context's work on a caller CUDA stream (int handle, 0/None:
        back to a private stream)."""
        check(lib().perrk_set_stream(self._h, C.c_void_p(cuda_stream or None)))

    def profile(self, enable=True):
        check(lib().perrk_profile(self._h, int(enable)))

    def profile_read(self):
        """(stage-kernel ms, stage launches, stage compulsory bytes) since profile(True)."""
        ms, n, b = C.c_double(), C.c_int64(), C.c_double()
        check(lib().perrk_profile_read(self._h, C.byref(ms), C.byref(n), C.byref(b)))
        return ms.value, n.value, b.value

    def launch_count(self):
        n = C.c_int64()
        check(lib().perrk_launch_count(self._h, C.byref(n)))
        return n.value

    def step_traffic(self, family, pmap):
        """Compulsory HBM bytes: (stage launches of one step, one relaxation
        pass, final update)."""
        self._use_family(family, pmap)
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        check(lib().perrk_step_traffic(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def _use_family(self, family, pmap):
        key = (id(family), id(pmap), family.version, pmap.version)
        if key == self._family_key:
            return
        E = np.ascontiguousarray(family.E, dtype=np.int32)
        A = _f64(family.A)
        b, c = _f64(family.b), _f64(family.c)
        eff = np.ascontiguousarray(pmap.effective_level, dtype=np.int32)
        if eff.size != self.global_num_cells():
            raise Error(capi.PERRK_EINVAL, "partition map does not match semidiscretization")
        fd = capi.FamilyDesc(capi.FAMILY[family.kind], family.S, family.R, _ip(E), _dp(A), _dp(b),
                             _dp(c))
        check(lib().perrk_set_family(self._h, C.byref(fd), _ip(eff)))
        self._family_key = key


def nccl_id() -> bytes:
    """A fresh ncclUniqueId (128 bytes) for perrk_comm_init."""
    buf = C.create_string_buffer(128)
    check(lib().perrk_nccl_id(buf))
    return buf.raw


def _shape3(mesh):
    sh = list(mesh.shape()) + [1]
    return np.ascontiguousarray(sh[:3], dtype=np.int32), len(mesh.shape())


def cell_work(pmap, family, npc):
    """DOF-stage work per cell of one step (active stages x nodes)."""
    E = np.array([len(family.active_sets[family.member_index_for_level(l)])
                  for l in range(1, family.R + 1)], dtype=np.float64)
    return E[np.asarray(pmap.effective_level) - 1] * npc


def partition_slabs(mesh, nranks, work=None):
    """Ownership map: contiguous last-axis layers balanced by per-cell work."""
    n, dim = _shape3(mesh)
    owner = np.zeros(mesh.num_cells(), dtype=np.int32)
    w = None if work is None else _f64(work)
    check(lib().perrk_partition_slabs(dim, _ip(n), None if w is None else _dp(w), int(nranks),
                                      _ip(owner)))
    return owner


def partition_levels(mesh, pmap, nranks):
    """Ownership map: 1/nranks of every level per rank (balanced stages)."""
    n, dim = _shape3(mesh)
    owner = np.zeros(mesh.num_cells(), dtype=np.int32)
    lv = np.ascontiguousarray(pmap.effective_level, dtype=np.int32)
    check(lib().perrk_partition_levels(dim, _ip(n), _ip(lv), int(pmap.R), int(nranks),
                                       _ip(owner)))
    return owner


def halo_plan(mesh, owner, rank):
    """The halo plan perrk_comm_init builds for `rank` (dict of arrays)."""
    n, dim = _shape3(mesh)
    ow = np.ascontiguousarray(owner, dtype=np.int32)
    cnt = np.zeros(4, dtype=np.int64)
    i64 = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))
    check(lib().perrk_halo_plan(dim, _ip(n), _ip(ow), int(rank), i64(cnt), None, None, None, None,
                                None, None, None))
    nl, ng, ns, npe = (int(x) for x in cnt)
    h = dict(gid=np.zeros(nl, np.int32), nbr=np.zeros(nl * 2 * dim, np.int32),
             ghost_gid=np.zeros(max(ng, 1), np.int64), peers=np.zeros(max(npe, 1), np.int32),
             recv_off=np.zeros(npe + 1, np.int64), send_off=np.zeros(npe + 1, np.int64),
             send=np.zeros(max(2 * ns, 1), np.int32))
    check(lib().perrk_halo_plan(dim, _ip(n), _ip(ow), int(rank), i64(cnt), _ip(h["gid"]),
                                _ip(h["nbr"]), i64(h["ghost_gid"]), _ip(h["peers"]),
                                i64(h["recv_off"]), i64(h["send_off"]), _ip(h["send"])))
    h["ghost_gid"], h["peers"], h["send"] = h["ghost_gid"][:ng], h["peers"][:npe], h["send"][:2 * ns]
    h["send"] = h["send"].reshape(-1, 2)
    return h


def face_nodes(dim, face):
    """Cell-local node indices of face `face` (2 d + side), exchange point order."""
    out = np.zeros(16 if dim == 3 else 4, dtype=np.int32)
    check(lib().perrk_face_nodes(int(dim), int(face), _ip(out)))
    return out


def local_pmap(semi, pmap):
    """The rank's part of a global partition map (for work accounting)."""
    g = semi.local_cells()
    eff = np.asarray(pmap.effective_level)[g]
    raw = np.asarray(pmap.raw_level)[g]
    return PartitionMap(pmap.R, raw.copy(), eff.copy())


def init_partition(semi, rank, nranks, owner=None):
    """Decompose `semi` over torch.distributed ranks (NCCL id broadcast from
    rank 0 over the default process group)."""
    import torch
    import torch.distributed as dist
    ident = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        ident = torch.frombuffer(bytearray(nccl_id()), dtype=torch.uint8).clone()
    if dist.get_backend() == "nccl":
        ident = ident.cuda()
    dist.broadcast(ident, 0)
    semi.comm_init(bytes(ident.cpu().numpy().tobytes()), rank, nranks, owner)


def loopback_group(semis, owner=None):
    """Ranks 0..n-1 of a partition as contexts on one device (test harness of
    the multi-rank logic; stepping any member steps all)."""
    arr = (C.c_void_p * len(semis))(*[s._h.value if isinstance(s._h, C.c_void_p) else s._h
                                       for s in semis])
    ow = None if owner is None else np.ascontiguousarray(owner, dtype=np.int32)
    check(lib().perrk_loopback_group(arr, len(semis), None if ow is None else _ip(ow)))
    for s in semis:
        s._refresh_sizes()
        s._group = semis


def fp64_peak(device=0):
    """Measured FP64 DFMA throughput of the device, GFLOP/s."""
    out = C.c_double()
    check(lib().perrk_fp64_peak(int(device), C.byref(out)))
    return out.value


# ---------------------------------------------------------------------------
# P-ERK families (butcher.hpp:36-125)
# ---------------------------------------------------------------------------
_FREE = {"p2": lambda E: E - 2, "p3": lambda E: E - 3, "p3-original": lambda E: E - 3,
         "p4": lambda E: E - 5}


@dataclass
class PartitionFamily:
    kind: str
    S: int
    R: int
    E: List[int]
    A: np.ndarray        # [R, S, S]
    b: np.ndarray
    c: np.ndarray
    active_sets: List[set] = field(default_factory=list)
    dt_max: List[float] = field(default_factory=list)
    version: int = 0

    @property
    def order(self):
        return {"p2": 2, "p3": 3, "p3-original": 3, "p4": 4}[self.kind]

    def member_index_for_level(self, level):
        return self.R - level

    def member_for_level(self, level):
        return self.A[self.member_index_for_level(level)]


def free_coefficient_count(kind, E):
    return _FREE[kind](E)


def build_family(kind, S, E_list, free_subdiagonals, c_Sminus3=1.0):
    kind = {"p3-variant": "p3"}.get(kind, kind)
    R = len(E_list)
    if len(free_subdiagonals) != R:
        raise Error(capi.PERRK_EINVAL, "inconsistent member count")
    for E, fr in zip(E_list, free_subdiagonals):
        if E >= 0 and len(fr) != _FREE[kind](E):
            raise Error(capi.PERRK_EINVAL, "inconsistent free coefficient count")
    E = np.ascontiguousarray(E_list, dtype=np.int32)
    flat = _f64([x for fr in free_subdiagonals for x in fr] or [0.0])
    A = np.zeros((R, S, S))
    b, c = np.zeros(S), np.zeros(S)
    act = np.zeros((R, S), dtype=np.int32)
    check(lib().perrk_family_build(capi.FAMILY[kind], S, R, _ip(E), _dp(flat), float(c_Sminus3),
                                   _dp(A), _dp(b), _dp(c), _ip(act)))
    sets = [set(np.nonzero(act[r])[0].tolist()) for r in range(R)]
    return PartitionFamily(kind, S, R, list(map(int, E_list)), A, b, c, sets)


def build_perk2(S, E_list, free):
    return build_family("p2", S, E_list, free)


def build_perk3_variant(S, E_list, free):
    return build_family("p3", S, E_list, free)


def build_perk3_original(S, E_list, free):
    return build_family("p3-original", S, E_list, free)


def build_perk4(S, E_list, free, c_Sminus3=1.0):
    return build_family("p4", S, E_list, free, c_Sminus3)


def active_stage_set(A, b):
    """butcher.cpp:319-332 (host)."""
    S = len(b)
    act = {0} | {i for i in range(S) if b[i] != 0.0}
    grew = True
    while grew:
        grew = False
        for i in sorted(act):
            for j in range(i):
                if A[i][j] != 0.0 and j not in act:
                    act.add(j)
                    grew = True
    return act


def _fmt17(v):
    return "%.17g" % v


def family_to_text(fam: PartitionFamily) -> str:
    """Plain-text family format of butcher.cpp:334-355."""
    lines = [f"{fam.S} {fam.R}", f"# kind {fam.kind}",
             " ".join(_fmt17(x) for x in fam.c), " ".join(_fmt17(x) for x in fam.b)]
    for r in range(fam.R):
        lines.append(str(fam.E[r]))
        for i in range(fam.S):
            lines.append(" ".join(_fmt17(x) for x in fam.A[r, i]))
    if fam.dt_max:
        lines.append("dt_max " + " ".join(_fmt17(x) for x in fam.dt_max))
    return "\n".join(lines) + "\n"


def family_from_text(text: str) -> PartitionFamily:
    """butcher.cpp:357-433."""
    kind = "p2"
    rows = []
    dt_max = []
    for raw in text.splitlines():
        s = raw.strip()
        if not s:
            continue
        if s.startswith("#"):
            parts = s[1:].split()
            if len(parts) >= 2 and parts[0] == "kind":
                kind = {"p3-variant": "p3"}.get(parts[1], parts[1])
            continue
        if s.startswith("dt_max"):
            dt_max = [float(x) for x in s.split()[1:]]
            continue
        rows.append(s.split())
    if not rows:
        raise Error(capi.PERRK_EINVAL, "empty family file")
    S, R = int(rows[0][0]), int(rows[0][1])
    c = np.array([float(x) for x in rows[1][:S]])
    b = np.array([float(x) for x in rows[2][:S]])
    A = np.zeros((R, S, S))
    E = []
    k = 3
    for r in range(R):
        E.append(int(float(rows[k][0])))
        k += 1
        for i in range(S):
            A[r, i] = [float(x) for x in rows[k][:S]]
            k += 1
    sets = [active_stage_set(A[r], b) for r in range(R)]
    return PartitionFamily(kind, S, R, E, A, b, c, sets, dt_max)


def load_family(path):
    with open(path) as f:
        return family_from_text(f.read())


def save_family(fam, path):
    with open(path, "w") as f:
        f.write(family_to_text(fam))


# ---------------------------------------------------------------------------
# partition map (mesh.hpp:44-76)
# ---------------------------------------------------------------------------
@dataclass
class PartitionMap:
    R: int
    raw_level: np.ndarray
    effective_level: np.ndarray
    version: int = 0

    def cells_per_level(self):
        return [int(np.sum(self.effective_level == r)) for r in range(1, self.R + 1)]


def make_partition_map(mesh, levels, R):
    levels = np.ascontiguousarray(levels, dtype=np.int32)
    if levels.size != mesh.num_cells():
        raise Error(capi.PERRK_EINVAL, "level list does not match mesh")
    n = np.ascontiguousarray(list(mesh.shape()) + [1] * (3 - mesh.dim), dtype=np.int32)
    eff = np.zeros_like(levels)
    check(lib().perrk_make_partition_map(mesh.dim, _ip(n), _ip(levels), int(R), _ip(eff)))
    return PartitionMap(int(R), levels.copy(), eff)


def assign_levels(nu, R):
    nu = _f64(nu)
    out = np.zeros(nu.size, dtype=np.int32)
    check(lib().perrk_assign_levels(_dp(nu), nu.size, int(R), _ip(out)))
    return out


def uniform_map(semi, level=1, R=1):
    lv = np.full(semi.num_cells(), level, dtype=np.int32)
    return PartitionMap(R, lv.copy(), lv)


# ---------------------------------------------------------------------------
# integrator (relax.hpp, stepper.hpp)
# ---------------------------------------------------------------------------
@dataclass
class RelaxationConfig:
    method: str = "newton"
    max_iter: int = 5
    residual_tol: float = 1e-14
    step_tol: float = 1e-15
    bracket_min: float = 0.8
    bracket_max: float = 1.2
    seed_from_previous: bool = True
    numerics: str = "reference"     # "reference" (relax.cpp) | "accurate"

    def to_c(self):
        return capi.RelaxCfg({"newton": 0, "bisection": 1, "secant": 2}[self.method],
                             self.max_iter, self.residual_tol, self.step_tol, self.bracket_min,
                             self.bracket_max, int(self.seed_from_previous),
                             {"reference": 0, "accurate": 1}[self.numerics])


@dataclass
class PerkStepOptions:
    relaxation: Optional[RelaxationConfig] = None
    gamma_override: float = 1.0
    gamma_seed: float = 1.0
    h_ref: float = math.nan
    idt: bool = False

    def to_c(self):
        o = capi.StepOpts()
        o.relax_enabled = int(self.relaxation is not None)
        if self.relaxation is not None:
            o.relax = self.relaxation.to_c()
        o.gamma_override = self.gamma_override
        o.gamma_seed = self.gamma_seed
        o.h_ref = self.h_ref
        o.idt = int(self.idt)
        return o


@dataclass
class PerkStepResult:
    gamma: float
    iterations: int
    residual: float
    fell_back: bool
    delta_h: float
    aborted: bool
    bad_cell: int
    bad_stage: int


def _result(r):
    return PerkStepResult(r.gamma, r.iterations, r.residual, bool(r.fell_back), r.delta_h,
                          bool(r.aborted), r.bad_cell, r.bad_stage)


def perk_step(U, t, dt, family, pmap, semi, opts=None):
    """stepper.cpp:17-114.  U (numpy, host) is advanced in place; returns
    (t_new, PerkStepResult).  On a positivity abort U and t are untouched."""
    opts = opts or PerkStepOptions()
    if U.dtype != np.float64 or not U.flags.c_contiguous:
        raise Error(capi.PERRK_EINVAL, "U must be a contiguous float64 array")
    semi._use_family(family, pmap)
    tt = C.c_double(t)
    res = capi.StepResult()
    o = opts.to_c()
    check(lib().perrk_perk_step(semi._h, _dp(U), C.byref(tt), float(dt), C.byref(o),
                                C.byref(res)))
    return tt.value, _result(res)


def perk_step_resident(t, dt, family, pmap, semi, opts=None):
    """perk_step on the state already resident on the device (semi.upload)."""
    opts = opts or PerkStepOptions()
    semi._use_family(family, pmap)
    tt = C.c_double(t)
    res = capi.StepResult()
    o = opts.to_c()
    check(lib().perrk_perk_step_resident(semi._h, C.byref(tt), float(dt), C.byref(o),
                                         C.byref(res)))
    return tt.value, _result(res)


@dataclass
class CflRamp:
    cfl0: float = 0.5
    cfl_max: float = 0.5
    t_ramp: float = 1.0


@dataclass
class TimeControl:
    fixed: bool = True
    dt: float = 0.0
    ramp: CflRamp = field(default_factory=CflRamp)


@dataclass
class IntegratorConfig:
    t0: float = 0.0
    tf: float = 1.0
    time: TimeControl = field(default_factory=TimeControl)
    relaxation: Optional[RelaxationConfig] = None
    anchor: str = "step"          # "step" | "initial"
    idt: bool = False
    max_steps: int = 10_000_000


def cfl_at(ramp: CflRamp, s):
    """CflRamp::operator() (stepper.cpp:13-15)."""
    if ramp.cfl0 == ramp.cfl_max:
        return ramp.cfl_max
    return min(ramp.cfl_max, ramp.cfl0 + (ramp.cfl_max - ramp.cfl0) * s / ramp.t_ramp)


def compute_dt(U, semi, config: IntegratorConfig, t):
    """stepper.cpp:116-127."""
    r = config.time.ramp
    val = config.time.dt if config.time.fixed else cfl_at(r, t - config.t0)
    out = C.c_double()
    check(lib().perrk_compute_dt(semi._h, _dp(semi._state(U)), int(config.time.fixed), float(val),
                                 float(t), float(config.tf), C.byref(out)))
    return out.value


@dataclass
class StepRecord:
    step: int
    t: float
    dt: float
    gamma: float
    newton_iters: int
    entropy: float
    invariants: np.ndarray
    fell_back: bool
    delta_h: float = 0.0  # PerkStepResult::delta_h of the step (stepper.hpp:62-68)


@dataclass
class RunResult:
    U: np.ndarray
    log: List[StepRecord]
    final_time: float
    aborted: bool
    n_rhs: int
    initial_entropy: float


def _run_cfg(config: IntegratorConfig, records=True, carry=None):
    r = config.time.ramp
    rc = capi.RunCfg()
    rc.cfl0 = r.cfl0
    rc.t_ramp = r.t_ramp
    rc.t0 = config.t0
    rc.fixed_dt = int(config.time.fixed)
    rc.dt_or_cfl = config.time.dt if config.time.fixed else r.cfl_max
    rc.tf = config.tf
    rc.relax_enabled = int(config.relaxation is not None)
    if config.relaxation is not None:
        rc.relax = config.relaxation.to_c()
    rc.anchor_initial = int(config.anchor == "initial")
    rc.idt = int(config.idt)
    rc.records = int(records)
    if carry is not None:  # continue a run: (next gamma seed, anchor H(U_0))
        rc.carry = 1
        rc.gamma_seed, rc.h_anchor = carry
    return rc


def advance(semi, family, pmap, config: IntegratorConfig, t, nsteps, records=True, carry=None):
    """Up to nsteps steps of run()'s loop on the resident state, on the
    device (one host sync at the end).  Returns (t, steps, aborted, records).
    `carry` = (gamma_seed, h_anchor) continues a run started by an earlier
    call (perrk_run_cfg.carry)."""
    semi._use_family(family, pmap)
    rc = _run_cfg(config, records, carry)
    log = (capi.StepRecord * max(nsteps, 1))()
    tt = C.c_double(t)
    taken, ab = C.c_int(), C.c_int()
    check(lib().perrk_advance(semi._h, C.byref(rc), C.byref(tt), int(nsteps),
                              log if records else None, C.byref(taken), C.byref(ab)))
    return tt.value, taken.value, bool(ab.value), list(log)[: taken.value] if records else []


def _record(step, r, V):
    return StepRecord(step, r.t, r.dt, r.gamma, r.newton_iters, r.entropy,
                      np.array(r.invariants[:V]), bool(r.fell_back), r.delta_h)


def run(config: IntegratorConfig, family, pmap, semi, U0, chunk=64):
    """stepper.cpp:129-193: integrate from t0 to tf on the device."""
    U0 = semi._state(U0)
    h0 = semi.total_entropy(U0)
    semi.reset_evaluation_counter()
    semi.upload(U0)
    t = config.t0
    log: List[StepRecord] = []
    aborted = False
    t_eps = 1e-12 * max(1.0, abs(config.tf))
    carry = None  # the chunks are ONE run: gamma seed and anchor carry over
    while t < config.tf - t_eps and not aborted:
        if len(log) >= config.max_steps:
            raise Error(capi.PERRK_EINVAL, "step limit exceeded")
        n = min(chunk, config.max_steps - len(log))
        t, taken, aborted, recs = advance(semi, family, pmap, config, t, n, True, carry)
        for r in recs:
            log.append(_record(len(log) + 1, r, semi.num_vars()))
        if log:
            last = log[-1]
            carry = (1.0 if last.fell_back else last.gamma, h0)
        if taken == 0 and not aborted:
            break
    return RunResult(semi.download(), log, t, aborted, semi.rhs_cell_evaluations(), h0)


def run_steps(config: IntegratorConfig, family, pmap, semi, U0, nsteps, out=None, chunk=None):
    """run() (stepper.cpp:129-193) for exactly nsteps steps (the reference's
    run has no step-count mode): U0 (host) -> device once, the
    steps resident, the final state -> `out` (host).  The step log comes back
    to the host every `chunk` steps (None: once at the end; 1: every step's
    StepRecord is on the host before the next step is issued, as run()'s
    on_step callback sees it, stepper.cpp:182); gamma seed and anchor carry
    across the chunks."""
    U0 = semi._state(U0)
    h0 = semi.total_entropy(U0) if (chunk and config.relaxation is not None
                                    and config.anchor == "initial") else float("nan")
    semi.upload(U0)
    chunk = chunk or max(nsteps, 1)
    t, log, aborted, carry = config.t0, [], False, None
    while len(log) < nsteps and not aborted:
        n = min(chunk, nsteps - len(log))
        t, taken, aborted, recs = advance(semi, family, pmap, config, t, n, True, carry)
        for r in recs:
            log.append(_record(len(log) + 1, r, semi.num_vars()))
        if not recs:
            break
        carry = (1.0 if log[-1].fell_back else log[-1].gamma, h0)
    U = semi.download(out)
    return RunResult(U, log, t, aborted, semi.rhs_cell_evaluations(), float("nan"))


# ---------------------------------------------------------------------------
# spectrum probing for family design (reference:
# probe_jacobian / eigenvalues_dense / clean_spectrum, specopt.cpp:18-60)
# ---------------------------------------------------------------------------
def _color_period(n, radius):
    """Smallest period k >= 2 radius + 1 dividing n (periodic wrap keeps the
    colouring proper), else n (no compression along that axis)."""
    for k in range(2 * radius + 1, n + 1):
        if n % k == 0:
            return k
    return n


def probe_jacobian(semi, U, t=0.0, epsilon=1e-6, colored=True, device=True):
    """Dense Jacobian of the device RHS by central differences, column j with
    h_j = epsilon (1 + |U_j|) as specopt.cpp:18-35.  With `colored`, the
    columns of cells that are far enough apart are probed in one RHS pair
    (compressed Jacobian): a cell's RHS depends on its face neighbours (BR1:
    on their neighbours too), so cells whose footprints do not overlap share
    an evaluation; 2 x colours x (nodes per cell x V) RHS calls instead of
    2 M.  With `device` (and M <= 5000) the whole probe runs inside the
    library (perrk_probe_jacobian): perturbation, RHS pairs and the column
    scatter stay on the GPU, one M x M copy back."""
    U = semi._state(U)
    M, npc, V = U.size, semi.nodes_per_cell(), semi.num_vars()
    if colored and device and M <= 5000:
        return semi.probe_jacobian(U, t, epsilon)
    if M > 5000 and not colored:
        raise Error(capi.PERRK_EINVAL, "dense Jacobian probing guarded to M <= 5000")
    shape = semi.spec.mesh.shape()
    dim = len(shape)
    cells = np.arange(semi.num_cells())
    coords = [cells % shape[0], (cells // shape[0]) % shape[1]]
    if dim == 3:
        coords.append(cells // (shape[0] * shape[1]))
    radius = 2 if semi.spec.physics == "nsf" else 1
    if colored:
        periods = [_color_period(n, radius) for n in shape]
    else:
        periods = list(shape)
    color = np.zeros(cells.size, dtype=np.int64)
    mult = 1
    for a in range(dim):
        color += (coords[a] % periods[a]) * mult
        mult *= periods[a]
    ncolors = mult
    # footprint rows of each cell: itself and its neighbours within `radius`
    def footprint(c):
        out = set()
        base = [coords[a][c] for a in range(dim)]
        rng = range(-radius, radius + 1)
        offs = [(dx, dy) for dx in rng for dy in rng] if dim == 2 else \
               [(dx, dy, dz) for dx in rng for dy in rng for dz in rng]
        for o in offs:
            if sum(abs(x) > 0 for x in o) > 1 and radius == 1:
                continue  # face neighbours only for the inviscid footprint
            q = [(base[a] + o[a]) % shape[a] for a in range(dim)]
            cid = q[0] + shape[0] * (q[1] + (shape[1] * q[2] if dim == 3 else 0))
            out.add(int(cid))
        return sorted(out)
    J = np.zeros((M, M))
    for col in range(ncolors):
        members = cells[color == col]
        if members.size == 0:
            continue
        feet = {int(c): footprint(int(c)) for c in members}
        for q in range(npc * V):
            idx = members * npc * V + q
            h = epsilon * (1.0 + np.abs(U[idx]))
            up, um = U.copy(), U.copy()
            up[idx] += h
            um[idx] -= h
            diff = semi.rhs(t, up) - semi.rhs(t, um)
            for c, hc in zip(members, h):
                rows = np.concatenate([np.arange(f * npc * V, (f + 1) * npc * V) for f in feet[int(c)]])
                J[rows, c * npc * V + q] = diff[rows] / (2.0 * hc)
    return J


def clean_spectrum(eigs, relative_tol=1e-10):
    """specopt.cpp:48-54: clip tiny positive real parts and imaginary parts."""
    eigs = np.array(eigs, dtype=complex)
    rho = np.abs(eigs).max()
    re, im = eigs.real.copy(), eigs.imag.copy()
    re[(re > 0.0) & (re <= relative_tol * rho)] = 0.0
    im[np.abs(im) <= 1e-14 * rho] = 0.0
    return re + 1j * im


def probe_spectrum(semi, U, t=0.0, colored=True, epsilon=1e-6):
    """probe_spectrum (specopt.cpp:56-60) on the device RHS."""
    return clean_spectrum(np.linalg.eigvals(probe_jacobian(semi, U, t, epsilon=epsilon,
                                                           colored=colored)))


def krylov_spectrum(semi, U=None, m=60, t=0.0, epsilon=1e-6, cell_mask=None):
    """Ritz values of m matrix-free Arnoldi steps (Semidiscretization.
    krylov_hessenberg): the spectral envelope of the RHS Jacobian (largest
    |lambda|, the extreme real and imaginary parts) on meshes of any size,
    where probe_spectrum's dense M x M probe is guarded to M <= 5000."""
    H = semi.krylov_hessenberg(U, m, t, epsilon, cell_mask)
    k = H.shape[1]
    return clean_spectrum(np.linalg.eigvals(H[:k, :k]))


def stability_margin(family, eigs, dt):
    """max |P_r(dt lambda)| over the spectrum for every member r (P from the
    tableau, butcher.cpp stability_function): <= 1 means stable at dt."""
    out = []
    for r in range(family.R):
        A, b = family.A[r], family.b
        S = family.S
        z = dt * np.asarray(eigs, dtype=complex)
        k = np.zeros((S, z.size), dtype=complex)
        for i in range(S):
            acc = np.zeros(z.size, dtype=complex)
            for j in range(i):
                if A[i, j] != 0.0:
                    acc += A[i, j] * k[j]
            k[i] = 1.0 + z * acc
        R_ = 1.0 + z * sum(b[i] * k[i] for i in range(S) if b[i] != 0.0)
        out.append(float(np.abs(R_).max()))
    return out


# ---------------------------------------------------------------------------
# CSV writers (write_step_log_csv, stepper.cpp:267-301; write_snapshot_csv,
# semidisc.cpp:609-632): the reference's headers and %.17g formatting
# ---------------------------------------------------------------------------
def write_step_log_csv(log, semi, path):
    V = semi.num_vars()
    names = ["mass", "momentum_x", "momentum_y", "momentum_z"][: semi.dim() + 1] + ["energy"]
    with open(path, "w") as f:
        f.write("step,t,dt,gamma,newton_iters,H," + ",".join(names[:V]) + ",fell_back\n")
        for r in log:
            vals = [r.t, r.dt, r.gamma]
            f.write(f"{r.step}," + ",".join("%.17g" % v for v in vals) + f",{r.newton_iters},"
                    + "%.17g" % r.entropy + "," + ",".join("%.17g" % v for v in r.invariants[:V])
                    + f",{1 if r.fell_back else 0}\n")


def write_snapshot_csv(semi, U, path):
    V = semi.num_vars()
    # EulerPhysics::variable_name (physics.cpp:90-95), z extended
    names = ["rho", "rho_v_x", "rho_v_y", "rho_v_z"][: semi.dim() + 1] + ["rho_e"]
    x, y, z = semi.node_x(), semi.node_y(), semi.node_z()
    U = np.asarray(U).reshape(-1, V)
    with open(path, "w") as f:
        f.write("x,y" + (",z" if semi.dim() == 3 else "") + "," + ",".join(names[:V]) + "\n")
        for n in range(U.shape[0]):
            cols = [x[n], y[n]] + ([z[n]] if semi.dim() == 3 else []) + list(U[n])
            f.write(",".join("%.17g" % v for v in cols) + "\n")


# ---------------------------------------------------------------------------
# linear advection: the update matrix of one step (analysis.hpp / analysis.cpp)
# ---------------------------------------------------------------------------
@dataclass
class AdvectionSpec:
    """SemidiscretizationSpec with AdvectionPhysics(velocity) (physics.hpp:54-85)
    on a periodic Mesh1D or Mesh2DRect."""
    mesh: object
    velocity: Sequence[float]
    polydeg: int = 3
    surface_flux: str = "upwind"
    volume_mode: str = "flux_differencing"
    volume_flux: str = "ec"
    device: int = 0

    def num_dofs(self):
        return self.mesh.num_cells() * (self.polydeg + 1) ** self.mesh.dim


@dataclass
class UpdateMatrix:
    gamma: float
    dt: float
    D: np.ndarray


def _adv_desc(spec):
    if spec.polydeg != 3:
        raise Error(capi.PERRK_EUNSUP, "the device path is built for polydeg 3")
    if not getattr(spec.mesh, "periodic", True):
        raise Error(capi.PERRK_EUNSUP, "the update-matrix engine runs periodic meshes")
    d = capi.AdvectionDesc()
    d.dim = spec.mesh.dim
    keep = [_f64(e) for e in spec.mesh.edges]
    for a, e in enumerate(keep):
        d.n[a] = len(e) - 1
        d.edges[a] = _dp(e)
    vel = list(spec.velocity)
    if len(vel) != spec.mesh.dim:
        raise Error(capi.PERRK_EINVAL, "physics/mesh dimension mismatch")
    for a, v in enumerate(vel):
        d.velocity[a] = float(v)
    d.surface_flux = capi.FLUX[spec.surface_flux]
    d.volume_mode = {"weak": 0, "flux_differencing": 1}[spec.volume_mode]
    d.volume_flux = capi.FLUX[spec.volume_flux]
    d.device = spec.device
    return d, keep


def assemble_update_matrix(family, pmap, spec, dt, gamma=1.0):
    """analysis::assemble_update_matrix (analysis.cpp:11-32) on the device:
    D[:, j] = perk_step(e_j) with relaxation off and gamma fixed, all columns
    batched (perrk_update_matrix)."""
    d, keep = _adv_desc(spec)
    E = np.ascontiguousarray(family.E, dtype=np.int32)
    A = _f64(family.A)
    b, c = _f64(family.b), _f64(family.c)
    eff = np.ascontiguousarray(pmap.effective_level, dtype=np.int32)
    if eff.size != spec.mesh.num_cells():
        raise Error(capi.PERRK_EINVAL, "partition map does not match mesh")
    fd = capi.FamilyDesc(capi.FAMILY[family.kind], family.S, family.R, _ip(E), _dp(A), _dp(b),
                         _dp(c))
    M = C.c_int64()
    check(lib().perrk_update_matrix(C.byref(d), C.byref(fd), _ip(eff), float(dt), float(gamma),
                                    None, C.byref(M)))
    out = np.zeros(M.value * M.value)
    check(lib().perrk_update_matrix(C.byref(d), C.byref(fd), _ip(eff), float(dt), float(gamma),
                                    _dp(out), C.byref(M)))
    return UpdateMatrix(gamma, dt, out.reshape(M.value, M.value).T)  # column-major storage


def monotonicity_metrics(D):
    """analysis.cpp:34-40: (min entry, max entry, max |row sum - 1|)."""
    D = np.asarray(D)
    return float(D.min()), float(D.max()), float(np.abs(D.sum(axis=1) - 1.0).max())


def spectral_radius(D):
    """analysis.cpp:42-47 (eigenvalues on the host)."""
    return float(np.abs(np.linalg.eigvals(np.asarray(D))).max())


def save_matrix(D, path):
    """analysis.cpp:49-60: rows of %.17g separated by single spaces."""
    with open(path, "w") as fh:
        for row in np.asarray(D):
            fh.write(" ".join("%.17g" % v for v in row) + "\n")
