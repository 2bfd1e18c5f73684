// Stage kernel, 2D Euler with the EC volume flux and the Rusanov / central
// surface flux: one warp per FOUR cells, two LGL nodes per lane, no block
// barriers — the 2D counterpart of stage3w_kernel (dg_stage3w.cuh).
//
// Same work per active cell as stage_kernel (dg_stage.cuh; reference
// semidisc.cpp:409-557 via rhs_masked :126-138, stepper.cpp:52-92 around it):
// stage-state formation, flux-differencing volume term with the Ranocha EC
// flux, surface flux + strong-form lift + endpoint diagonal term, b-stage
// epilogue and the next stage's formed state.
//
// Mapping.  Lane l serves cell slot cs = l >> 3 of the warp's four cells and
// owns nodes A = s and B = s + 8 of that cell (s = l & 7, node n = ix + 4 iy:
// A has iy = s >> 2 in {0, 1}, B has iy + 2).  Then
//   * x-lines lie in groups of four lanes, once for the A row and once for
//     the B row: each node evaluates its pair (j, j+1 mod 4) and receives
//     (j-1, j) by shuffle; the distance-2 pairs of the two rows are split
//     between the lanes (j < 2: the A pair, j >= 2: the B pair) and exchanged
//     with a lane^2 shuffle;
//   * y-lines pair lane l with lane l^4: the distance-2 pair (A, B) is inside
//     the lane, and each node's (j, j+1 mod 4) pair goes to the partner lane
//     by a lane^4 shuffle.
// So every lane evaluates exactly 6 EC fluxes (3 per node, each pair of the
// cell once) and 2 face points (16 per cell, one direction per round).
#pragma once

namespace perrk {
namespace dev {

#ifndef PERRK_W2_FLAT
// 1: as stage3w_kernel's PERRK_W3_HOIST / PERRK_W3_FLAT: neighbour ids and formed
// flags read once, branch-free trace staging, a warp-uniform pre-pass for
// neighbours formed from the first column, the two surface rounds as one
// straight-line block, y-face terms added by the owning lane, branch-free x gather
#define PERRK_W2_FLAT 1
#endif

#ifndef PERRK_W2_RSQ
#define PERRK_W2_RSQ 0  // 1: beta and c from one reciprocal square root (no gain on C3; see PERRK_SURF_RSQ)
#endif

#ifndef PERRK_W2_COAL
#define PERRK_W2_COAL 0  // 1: epilogue blocks through the slice and bulk stores (the round-2 session-1 form)
#endif

struct W2 {
  static constexpr int V = 4, NPC = 16, FP = 4, CPW = 4, WPB = 8, T = 32 * WPB;
  static constexpr int NQ = CPW * NPC;  // nodes per warp (64)
  // primitives: four arrays of 16-byte pairs over the warp's 64 nodes,
  // (rho, beta), (vx, vy), (p, E), (c, -); node n of cell slot cs at entry
  // 16 cs + (n ^ ((n >> 3) & 1)), which keeps every access pattern of the
  // kernel (own nodes, x/y partners, distance-2 pairs, the face nodes of both
  // surface rounds) on eight distinct 16-byte bank groups per quarter-warp
  static constexpr int SM_PR = 8 * NQ;
  // face slots: 5 doubles per slot (V = 4 and one padding double), slot
  // 24 cs + 8 d + 4 side + pt: with the 40-byte stride a cell's eight lanes
  // take eight distinct bank pairs, and the 24-slot cell pitch puts the other
  // cell of the half-warp on the complementary eight (8-byte accesses are
  // conflict free)
  static constexpr int FS = 5;
  static constexpr int SM_FS = (24 * (CPW - 1) + 16) * FS;
  // epilogue blocks: per array and cell slot, 64 doubles at a 72-double pitch
  // (the pad puts the half-warp's two cells on disjoint banks)
  static constexpr int EPITCH = 72;
  static constexpr int SM_WARP = SM_PR + SM_FS;
  static_assert(SM_WARP >= 3 * CPW * EPITCH, "the epilogue stages U, K1 and d in the slice");
  static constexpr int SM_TOTAL = WPB * SM_WARP;  // doubles per block
};

__device__ __forceinline__ int w2_sw(int cs, int n) { return 16 * cs + (n ^ ((n >> 3) & 1)); }

__device__ __forceinline__ int w2_fs(int cs, int d, int side, int pt) {
  return (24 * cs + 8 * d + 4 * side + pt) * W2::FS;
}

struct W2Prim {
  double rho, beta, v[2], p;
};

__device__ __forceinline__ W2Prim w2_load(const double* pr, int q) {
  const double2* b = reinterpret_cast<const double2*>(pr) + q;
  const double2 a = b[0], c = b[W2::NQ], e = b[2 * W2::NQ];
  W2Prim r;
  r.rho = a.x;
  r.beta = a.y;
  r.v[0] = c.x;
  r.v[1] = c.y;
  r.p = e.x;
  return r;
}

template <int D, bool SM>
__device__ __forceinline__ void w2_ec(const Phys& ph, const double* pr, int p, int q, double* f) {
  const W2Prim L = w2_load(pr, p), R = w2_load(pr, q);
  ec2<2, SM>(ph, D, L.rho, L.v, L.p, L.beta, R.rho, R.v, R.p, R.beta, f);
}

// x-lines: each node's (j, j+1 mod 4) pair, the received (j-1, j), and the
// distance-2 pairs split between the rows (as w3_inplane with D = 0)
template <bool SM>
__device__ __forceinline__ void w2_x(const Phys& ph, const double* pr, int lane, int cs, int s,
                                     double J2, double* KA, double* KB) {
  constexpr int V = W2::V;
  const int j = s & 3;
  const int kn = (j + 1) & 3, kp = (j + 3) & 3;
  const double cn = J2 * c_D[j * N1 + kn], cp = J2 * c_D[j * N1 + kp], c2 = J2 * c_D[j * N1 + (j ^ 2)];
  const int src = lane + (kp - j);
  const int nA = s, nB = s + 8;
  double f[V];
  w2_ec<0, SM>(ph, pr, w2_sw(cs, nA), w2_sw(cs, nA + (kn - j)), f);
#pragma unroll
  for (int v = 0; v < V; ++v) {
    KA[v] = fma(-cn, f[v], KA[v]);
    KA[v] = fma(-cp, __shfl_sync(0xffffffffu, f[v], src), KA[v]);
  }
  w2_ec<0, SM>(ph, pr, w2_sw(cs, nB), w2_sw(cs, nB + (kn - j)), f);
#pragma unroll
  for (int v = 0; v < V; ++v) {
    KB[v] = fma(-cn, f[v], KB[v]);
    KB[v] = fma(-cp, __shfl_sync(0xffffffffu, f[v], src), KB[v]);
  }
  const bool lo = j < 2;
  const int own = lo ? nA : nB;
  w2_ec<0, SM>(ph, pr, w2_sw(cs, own), w2_sw(cs, own ^ 2), f);
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double r = __shfl_xor_sync(0xffffffffu, f[v], 2);
    KA[v] = fma(-c2, lo ? f[v] : r, KA[v]);
    KB[v] = fma(-c2, lo ? r : f[v], KB[v]);
  }
}

// y-lines: lane l holds iy = yA and yA + 2, lane l^4 the other two (as w3_z)
template <bool SM>
__device__ __forceinline__ void w2_y(const Phys& ph, const double* pr, int lane, int cs, int s,
                                     double J2, double* KA, double* KB) {
  constexpr int V = W2::V;
  const int yA = s >> 2, yB = yA + 2;
  const int nA = s, nB = s + 8;
  double f[V];
  w2_ec<1, SM>(ph, pr, w2_sw(cs, nA), w2_sw(cs, nB), f);  // distance 2 inside the lane
  const double cab = J2 * c_D[yA * N1 + yB], cba = J2 * c_D[yB * N1 + yA];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    KA[v] = fma(-cab, f[v], KA[v]);
    KB[v] = fma(-cba, f[v], KB[v]);
  }
  // the partner lane l^4 holds the nodes of the other two rows:
  // yA = 0: A(0)-A'(1), B(2)-B'(3);  yA = 1: A(1)-B'(2), B(3)-A'(0)
  const int ps = s ^ 4;
  const int pA = yA ? ps + 8 : ps, pB = yA ? ps : ps + 8;
  const double cnA = J2 * c_D[yA * N1 + ((yA + 1) & 3)], cnB = J2 * c_D[yB * N1 + ((yB + 1) & 3)];
  const double cpA = J2 * c_D[yA * N1 + ((yA + 3) & 3)], cpB = J2 * c_D[yB * N1 + ((yB + 3) & 3)];
  double g[V];
  w2_ec<1, SM>(ph, pr, w2_sw(cs, nA), w2_sw(cs, pA), f);
  w2_ec<1, SM>(ph, pr, w2_sw(cs, nB), w2_sw(cs, pB), g);
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double rA = __shfl_xor_sync(0xffffffffu, f[v], 4);
    const double rB = __shfl_xor_sync(0xffffffffu, g[v], 4);
    KA[v] = fma(-cnA, f[v], KA[v]);
    KB[v] = fma(-cnB, g[v], KB[v]);
    KA[v] = fma(-cpA, yA ? rA : rB, KA[v]);
    KB[v] = fma(-cpB, yA ? rB : rA, KB[v]);
  }
  (void)lane;
}

// node of cell face (d, side) at face point pt
__device__ __forceinline__ int w2_face_node(int d, int side, int pt) {
  return d == 0 ? 3 * side + 4 * pt : pt + 12 * side;
}

template <int SURF>
__global__ void __launch_bounds__(W2::T, 2)
    stage2w_kernel(StageArgs a, MeshDev m, Phys ph, StepState* st, double* partials,
                   unsigned* counter) {
  using S = W2;
  constexpr int V = S::V, N = S::NPC, CPW = S::CPW;
  extern __shared__ double smem[];
  __shared__ double s_red[2 * 2 * S::WPB];
  __shared__ CellRec s_rec[S::WPB][2][CPW];  // descriptors, prefetched one group ahead
  if (st->aborted || st->finished) return;  // uniform across the grid
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int cs = lane >> 3, s = lane & 7;
  const int ix = s & 3, yA = s >> 2, yB = yA + 2;
  const int side = s >> 2, pt = s & 3;  // surface rounds: this lane's face point
  double* pr = smem + wib * S::SM_WARP;
  double* fs = pr + S::SM_PR;
  constexpr int RECQ = static_cast<int>(sizeof(CellRec) / 16);  // 16-byte pieces per record
  auto cell_at = [&](int sl) { return sl < a.n ? (a.list ? a.list[sl] : sl) : -1; };
  // the group's four descriptors into buffer b (lanes 0 .. 4 RECQ - 1)
  auto fetch_rec = [&](int b, int g0) {
    if (lane < CPW * RECQ) {
      const int c = cell_at(g0 + lane / RECQ);
      if (c >= 0)
        cp_async16(reinterpret_cast<char*>(&s_rec[wib][b][lane / RECQ]) + 16 * (lane % RECQ),
                   reinterpret_cast<const char*>(m.rec + c) + 16 * (lane % RECQ));
    }
    cp_async_commit();
  };
  const double dt = st->dt;
  const double sqrt_gamma = sqrt(ph.gamma);
  dd acc_dh = dd_zero(), acc_h = dd_zero();
  unsigned long long dmax_bits = 0;
  const int nw = gridDim.x * S::WPB;
  int g0 = (blockIdx.x * S::WPB + wib) * CPW;  // first list slot of the warp's group
  int rb = 0;
  fetch_rec(0, g0);

  while (g0 < a.n) {
    const int cell = cell_at(g0 + cs);  // -1: padding lanes (tail group)
    const bool live = cell >= 0;
    const int ng0 = g0 + nw * CPW;
    if (PERRK_ST_L2PF && s == 0) {  // the next group's state arrays to L2
      const int ncell = cell_at(ng0 + cs);
      if (ncell >= 0) {
        constexpr unsigned kBytes = N * V * sizeof(double);
        const size_t off = static_cast<size_t>(ncell) * N * V;
        if (a.form) l2_prefetch(a.Us + off, kBytes);
        if (!a.form || a.write_next) l2_prefetch(a.U + off, kBytes);
        if (a.write_next && a.form) l2_prefetch(a.K1 + off, kBytes);
        if (a.d_mode == 2) l2_prefetch(a.d + off, kBytes);
      }
    }
    cp_async_wait<0>();
    if (s == 0) bulk_wait_read();  // this cell slot's previous blocks left the slice
    __syncwarp();
    const CellRec* rp = &s_rec[wib][rb][cs];
    const unsigned long long lv =
        live ? static_cast<unsigned long long>(*reinterpret_cast<const long long*>(rp->lev)) : 0;
    const int lev = static_cast<int>(lv & 0xff);
    const double J2x = live ? rp->J2[0] : 0.0, J2y = live ? rp->J2[1] : 0.0;
    // ---- own nodes A, B (device layout: variable v of node n at cbase + v N + n)
    const size_t cbase = static_cast<size_t>(live ? cell : 0) * N * V;
    double uA[V] = {1.0, 0.0, 0.0, 2.5}, uB[V] = {1.0, 0.0, 0.0, 2.5};  // padding: rest state
    if (live) {
      const size_t gA = cbase + s, gB = gA + 8;
      if (!a.form) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          uA[v] = __ldg(a.U + gA + v * N);
          uB[v] = __ldg(a.U + gB + v * N);
        }
      } else if (a.formed[lev]) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          uA[v] = __ldg(a.Us + gA + v * N);
          uB[v] = __ldg(a.Us + gB + v * N);
        }
      } else {
        const double a1 = dt * a.a1[lev];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          uA[v] = fma(a1, __ldg(a.K1 + gA + v * N), __ldg(a.U + gA + v * N));
          uB[v] = fma(a1, __ldg(a.K1 + gB + v * N), __ldg(a.U + gB + v * N));
        }
      }
    }
    // ---- neighbour face traces -> the face slots (cp.async), one direction
    // per round: round d, face 2 d + side, point pt ----------------------------
#if PERRK_W2_FLAT
    int nb2[2];
    unsigned unf = 0;  // bit d: the neighbour on (d, side) is formed from U and K1 in the pre-pass
#pragma unroll
    for (int d = 0; d < 2; ++d) nb2[d] = live ? rp->nb[2 * d + side] : 0;
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      const int l2 = static_cast<int>((lv >> (8 * (1 + 2 * d + side))) & 0xff);
      if (live && a.form && nb2[d] >= 0 && !a.formed[l2]) unf |= 1u << d;
    }
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      // branch free (padding lanes copy a trace of cell 0: unused)
      double* dst = fs + w2_fs(cs, d, side, pt);
      const int nbc = nb2[d];
      const bool gh = nbc < 0;
      const double* src =
          gh ? m.ghost + (static_cast<size_t>(-1 - nbc) * S::FP + pt) * V
             : ((a.form && !((unf >> d) & 1u)) ? a.Us : a.U) + static_cast<size_t>(nbc) * N * V +
                   w2_face_node(d, 1 - side, pt);
      const int vs = gh ? 1 : N;
#pragma unroll
      for (int v = 0; v < V; ++v) cp_async8(dst + v, src + v * vs);
    }
#else
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      double* dst = fs + w2_fs(cs, d, side, pt);
      if (!live) continue;
      const int nbc = rp->nb[2 * d + side];
      if (nbc < 0) {
        const double* g = m.ghost + (static_cast<size_t>(-1 - nbc) * S::FP + pt) * V;
#pragma unroll
        for (int v = 0; v < V; ++v) cp_async8(dst + v, g + v);
      } else {
        const size_t gi = static_cast<size_t>(nbc) * N * V + w2_face_node(d, 1 - side, pt);
        const int l2 = static_cast<int>((lv >> (8 * (1 + 2 * d + side))) & 0xff);
        if (!a.form) {
#pragma unroll
          for (int v = 0; v < V; ++v) cp_async8(dst + v, a.U + gi + v * N);
        } else if (a.formed[l2]) {
#pragma unroll
          for (int v = 0; v < V; ++v) cp_async8(dst + v, a.Us + gi + v * N);
        }  // else: formed from U and K1 in the surface phase
      }
    }
#endif
    cp_async_commit();
    fetch_rec(rb ^ 1, ng0);  // the next group's descriptors
    // ---- primitives of A and B -> the slice; per-warp smoothness range -------
    bool okAB = true;
    unsigned hr_lo = 0xffffffffu, hr_hi = 0u, hb_lo = 0xffffffffu, hb_hi = 0u;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int n = s + 8 * h;
      double ir;
      const Prim<2> q = prim_of<2>(ph, h ? uB : uA, ir);
      okAB = okAB & prim_ok<2>(q);
      // (Rusanov) beta = rho / p and c = sqrt(gamma p / rho) from one reciprocal
      // square root y of x = p / rho: beta = y^2, c = sqrt(gamma) x y (as stage3w_kernel)
      double be, cs_ = 0.0;
      if (SURF == 2 && PERRK_W2_RSQ) {
        const double x = q.p * ir;
        const double y = frsqrt(x);
        be = y * y;
        cs_ = sqrt_gamma * (x * y);
      } else {
        be = q.rho * frcp(q.p);
        if (SURF == 2) cs_ = fsqrt(ph.gamma * q.p * ir);
      }
      double2* dst = reinterpret_cast<double2*>(pr) + w2_sw(cs, n);
      dst[0] = make_double2(q.rho, be);
      dst[S::NQ] = make_double2(q.v[0], q.v[1]);
      dst[2 * S::NQ] = make_double2(q.p, q.E);
      dst[3 * S::NQ] = make_double2(cs_, 0.0);
      if (live) {
        const unsigned hr = static_cast<unsigned>(__double2hiint(q.rho));
        const unsigned hb = static_cast<unsigned>(__double2hiint(be));
        hr_lo = min(hr_lo, hr);
        hr_hi = max(hr_hi, hr);
        hb_lo = min(hb_lo, hb);
        hb_hi = max(hb_hi, hb);
      }
    }
    if (live && !okAB) report_bad(st, a.stage, a.ncells, m.gid ? m.gid[cell] : cell);
    bool smooth;  // every pair of the warp's cells below logmean's series threshold
    {
      hr_lo = __reduce_min_sync(0xffffffffu, hr_lo);
      hr_hi = __reduce_max_sync(0xffffffffu, hr_hi);
      hb_lo = __reduce_min_sync(0xffffffffu, hb_lo);
      hb_hi = __reduce_max_sync(0xffffffffu, hb_hi);
      auto ratio_ok = [](unsigned lo, unsigned hi) {
        if (hi >= 0x7ff00000u || lo < 0x00100000u) return false;
        return __hiloint2double(static_cast<int>(hi + 1), 0) <
               1.0198 * __hiloint2double(static_cast<int>(lo), 0);
      };
      smooth = ratio_ok(hr_lo, hr_hi) && ratio_ok(hb_lo, hb_hi);
    }
    __syncwarp();

    // ---- flux-differencing volume terms (semidisc.cpp:455-464) --------------
    double KA[V], KB[V];
#pragma unroll
    for (int v = 0; v < V; ++v) KA[v] = KB[v] = 0.0;
    if (smooth) {
      w2_x<true>(ph, pr, lane, cs, s, J2x, KA, KB);
      w2_y<true>(ph, pr, lane, cs, s, J2y, KA, KB);
    } else {
      w2_x<false>(ph, pr, lane, cs, s, J2x, KA, KB);
      w2_y<false>(ph, pr, lane, cs, s, J2y, KA, KB);
    }

    // ---- surface flux + lift + endpoint diagonal at the lane's two face
    // points (semidisc.cpp:489-556, :450-454) ----------------------------------
    cp_async_wait<1>();  // the traces (the next descriptors may fly on)
    __syncwarp();
#if PERRK_W2_FLAT
    if (__any_sync(0xffffffffu, unf != 0u)) {  // a level's first active stage
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        if ((unf >> d) & 1u) {
          const int l2 = static_cast<int>((lv >> (8 * (1 + 2 * d + side))) & 0xff);
          const size_t gi = static_cast<size_t>(nb2[d]) * N * V + w2_face_node(d, 1 - side, pt);
          const double b1 = dt * a.a1[l2];
          double* sl = fs + w2_fs(cs, d, side, pt);  // the lane's own slot: the U trace
          double un[V];
#pragma unroll
          for (int v = 0; v < V; ++v) un[v] = fma(b1, __ldg(a.K1 + gi + v * N), sl[v]);
#pragma unroll
          for (int v = 0; v < V; ++v) sl[v] = un[v];
        }
      }
    }
    unsigned badf = 0;
    const double lift2[2] = {live ? rp->lift[0] : 0.0, live ? rp->lift[1] : 0.0};
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      double* slotp = fs + w2_fs(cs, d, side, pt);
      double un[V];
#pragma unroll
      for (int v = 0; v < V; ++v) un[v] = slotp[v];
      const double J2 = d == 0 ? J2x : J2y;
      const int j = side ? N1 - 1 : 0;
      double o4[V];
      const double2* on = reinterpret_cast<const double2*>(pr) + w2_sw(cs, w2_face_node(d, side, pt));
      const double2 o0 = on[0], o1 = on[S::NQ], o2 = on[2 * S::NQ], o3 = on[3 * S::NQ];
      const double vo[2] = {o1.x, o1.y};
      const bool ok = rus_lift_v<2, SURF>(ph, o0.x, vo, o2.x, o2.y, o3.x, un, d, side,
                                          J2 * c_D[j * N1 + j], side ? -lift2[d] : lift2[d],
                                          false, o4);
      if (!ok) badf |= 1u << d;
      if (d == 1) {
        // y faces: face point (1, side, pt) of lane (side, pt) belongs to the
        // lane's own node (A on side 0, B on side 1)
        const double mA = side ? 0.0 : 1.0, mB = side ? 1.0 : 0.0;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          KA[v] = fma(mA, o4[v], KA[v]);
          KB[v] = fma(mB, o4[v], KB[v]);
        }
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v) slotp[v] = o4[v];
      }
    }
    if (live && badf) {
      const int nbc = (badf & 1u) ? nb2[0] : nb2[1];
      report_bad(st, a.stage, a.ncells,
                 nbc < 0 ? m.ghost_gid[-1 - nbc] : (m.gid ? m.gid[nbc] : nbc));
    }
    __syncwarp();
    {  // x faces (pt = iy): every lane reads a written slot, nodes off the face weigh it with 0
      const double mx = (ix == 0 || ix == N1 - 1) ? 1.0 : 0.0;
      const int sd = ix ? 1 : 0;
      const double* cA = fs + w2_fs(cs, 0, sd, yA);
      const double* cB = fs + w2_fs(cs, 0, sd, yB);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        KA[v] = fma(mx, cA[v], KA[v]);
        KB[v] = fma(mx, cB[v], KB[v]);
      }
    }
#else
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      double* slotp = fs + w2_fs(cs, d, side, pt);
      if (!live) continue;
      const int nbc = rp->nb[2 * d + side];
      double un[V];
      if (nbc >= 0 && a.form) {
        const int l2 = static_cast<int>((lv >> (8 * (1 + 2 * d + side))) & 0xff);
        if (a.formed[l2]) {
#pragma unroll
          for (int v = 0; v < V; ++v) un[v] = slotp[v];
        } else {
          const size_t gi = static_cast<size_t>(nbc) * N * V + w2_face_node(d, 1 - side, pt);
          const double b1 = dt * a.a1[l2];
#pragma unroll
          for (int v = 0; v < V; ++v)
            un[v] = fma(b1, __ldg(a.K1 + gi + v * N), __ldg(a.U + gi + v * N));
        }
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v) un[v] = slotp[v];
      }
      const double J2 = d == 0 ? J2x : J2y;
      const double lift = rp->lift[d];
      const int j = side ? N1 - 1 : 0;
      double o4[V];
      const double2* on = reinterpret_cast<const double2*>(pr) + w2_sw(cs, w2_face_node(d, side, pt));
      const double2 o0 = on[0], o1 = on[S::NQ], o2 = on[2 * S::NQ], o3 = on[3 * S::NQ];
      const double vo[2] = {o1.x, o1.y};
      const bool ok = rus_lift_v<2, SURF>(ph, o0.x, vo, o2.x, o2.y, o3.x, un, d, side,
                                          J2 * c_D[j * N1 + j], side ? -lift : lift, false, o4);
      if (!ok)
        report_bad(st, a.stage, a.ncells,
                   nbc < 0 ? m.ghost_gid[-1 - nbc] : (m.gid ? m.gid[nbc] : nbc));
#pragma unroll
      for (int v = 0; v < V; ++v) slotp[v] = o4[v];
    }
    __syncwarp();
    // gather: node A / B on face (d, side) takes the term of face point
    // (d, side, pt(node, d))
    {
      if (ix == 0 || ix == N1 - 1) {  // x faces: pt = iy
        const int sd = ix ? 1 : 0;
        const double* cA = fs + w2_fs(cs, 0, sd, yA);
        const double* cB = fs + w2_fs(cs, 0, sd, yB);
#pragma unroll
        for (int v = 0; v < V; ++v) {
          KA[v] += cA[v];
          KB[v] += cB[v];
        }
      }
      if (yA == 0) {  // y faces: A on side 0 (iy = 0), B on side 1 (iy = 3) when yA = 1
        const double* c = fs + w2_fs(cs, 1, 0, ix);
#pragma unroll
        for (int v = 0; v < V; ++v) KA[v] += c[v];
      } else {
        const double* c = fs + w2_fs(cs, 1, 1, ix);
#pragma unroll
        for (int v = 0; v < V; ++v) KB[v] += c[v];
      }
    }
#endif

    // ---- epilogue (stepper.cpp:52-55, 60-72, 89-92) ---------------------------
    if ((a.want_dh || a.want_h) && live) {
      const double meas = rp->meas;
      auto node = [&](int n, const double* K, int iy) {
        const W2Prim q = w2_load(pr, w2_sw(cs, n));
        const double be = q.beta;
        const double s_therm = -(flog_core(be) + ph.gm1 * flog_core(q.rho));  // admissible here
        const double om = meas * c_w[ix] * c_w[iy];
        if (a.want_dh) {
          double v2 = 0.0, dot = 0.0;
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            v2 = fma(q.v[i], q.v[i], v2);
            dot = fma(ph.gm1 * be * q.v[i], K[1 + i], dot);
          }
          dot = fma(ph.gamma - s_therm - 0.5 * ph.gm1 * be * v2, K[0], dot);
          dot = fma(-ph.gm1 * be, K[V - 1], dot);
          acc_dh = dd_add_prod(acc_dh, om, dot);
        }
        if (a.want_h) acc_h = dd_add_prod(acc_h, om, -q.rho * s_therm);
      };
      node(s, KA, yA);
      node(s + 8, KB, yB);
    }
    const double an = dt * a.a1n[lev], pn = dt * a.apn[lev];
#if !PERRK_W2_COAL
    // Direct epilogue: in the device layout variable v of node n lies at
    // cbase + v N + n, so the eight lanes of a cell read and write 64
    // contiguous bytes per access (as stage3w_kernel's direct epilogue).
    if (live) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double* K = h ? KB : KA;
        const size_t g = cbase + s + 8 * h;
        if (a.write_k) {
#pragma unroll
          for (int v = 0; v < V; ++v) a.Kout[g + v * N] = K[v];
        }
        double x[V], y[V];
        if (a.write_next) {
#pragma unroll
          for (int v = 0; v < V; ++v) x[v] = __ldg(a.U + g + v * N);
          if (a.form) {
#pragma unroll
            for (int v = 0; v < V; ++v) y[v] = __ldg(a.K1 + g + v * N);
#pragma unroll
            for (int v = 0; v < V; ++v) a.Usn[g + v * N] = x[v] + fma(an, y[v], pn * K[v]);
          } else {
#pragma unroll
            for (int v = 0; v < V; ++v) a.Usn[g + v * N] = fma(an, K[v], x[v]);
          }
        }
        if (a.d_mode) {
          if (a.d_mode == 2) {
#pragma unroll
            for (int v = 0; v < V; ++v) x[v] = fma(a.b, K[v], a.d[g + v * N]);
          } else {
#pragma unroll
            for (int v = 0; v < V; ++v) x[v] = a.b * K[v];
          }
#pragma unroll
          for (int v = 0; v < V; ++v) {
            a.d[g + v * N] = x[v];
            const unsigned long long bits =
                static_cast<unsigned long long>(__double_as_longlong(x[v])) & 0x7fffffffffffffffULL;
            if (a.want_dmax) dmax_bits = bits > dmax_bits ? bits : dmax_bits;
          }
        }
      }
    }
#else
    // Epilogue through the slice (dead after the gather and the dH terms): the
    // cells' U, K1 and d blocks (512 contiguous bytes each) arrive by 16-byte
    // cp.async, the results leave as bulk copies, per cell slot.
    //   slice: U [cs EPITCH] | K1 / K_0 [4 EPITCH + ...] | d [8 EPITCH + ...]
    {
      constexpr int EP = S::EPITCH;
      double* eu = pr + cs * EP;
      double* ek = pr + (CPW + cs) * EP;
      double* ed = pr + (2 * CPW + cs) * EP;
      __syncwarp();
      if (live) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // 64 doubles = 32 pieces of 16 B over the cell's 8 lanes
          const int q = 2 * (s + 8 * k);
          if (a.write_next) cp_async16(eu + q, a.U + cbase + q);
          if (a.write_next && a.form) cp_async16(ek + q, a.K1 + cbase + q);
          if (a.d_mode == 2) cp_async16(ed + q, a.d + cbase + q);
        }
      }
      cp_async_commit();
      cp_async_wait<0>();
      __syncwarp();
      if (live) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double* K = h ? KB : KA;
          const int o = s + 8 * h;  // variable v of this node at o + v N
          if (a.write_k) {
#pragma unroll
            for (int v = 0; v < V; ++v) ek[o + v * N] = K[v];
          }
          if (a.write_next) {
            double x[V];
            if (a.form) {
#pragma unroll
              for (int v = 0; v < V; ++v) x[v] = eu[o + v * N] + fma(an, ek[o + v * N], pn * K[v]);
            } else {
#pragma unroll
              for (int v = 0; v < V; ++v) x[v] = fma(an, K[v], eu[o + v * N]);
            }
#pragma unroll
            for (int v = 0; v < V; ++v) eu[o + v * N] = x[v];
          }
          if (a.d_mode) {
#pragma unroll
            for (int v = 0; v < V; ++v) {
              const double x = a.d_mode == 2 ? fma(a.b, K[v], ed[o + v * N]) : a.b * K[v];
              ed[o + v * N] = x;
              const unsigned long long bits =
                  static_cast<unsigned long long>(__double_as_longlong(x)) & 0x7fffffffffffffffULL;
              if (a.want_dmax) dmax_bits = bits > dmax_bits ? bits : dmax_bits;
            }
          }
        }
      }
      bulk_store_fence();
      __syncwarp();
      if (live && s == 0) {
        constexpr unsigned kBytes = N * V * sizeof(double);
        if (a.write_next) bulk_store(a.Usn + cbase, eu, kBytes);
        if (a.write_k) bulk_store(a.Kout + cbase, ek, kBytes);
        if (a.d_mode) bulk_store(a.d + cbase, ed, kBytes);
      }
    }
#endif
    __syncwarp();  // the slice is rewritten by the next group
    g0 = ng0;
    rb ^= 1;
  }

  if (s == 0) bulk_wait_all();
  // ---- grid epilogue (as stage3w_kernel) ------------------------------------
  if (a.want_dmax) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o = __shfl_down_sync(0xffffffffu, dmax_bits, off);
      dmax_bits = o > dmax_bits ? o : dmax_bits;
    }
    if (lane == 0) {
      if (dmax_bits >= 0x7ff0000000000000ULL) st->d_nonfinite = 1;
      else atomicMax(&st->dmax_bits, dmax_bits);
    }
  }
  dd v[2] = {acc_dh, acc_h}, tot[2];
  if (a.want_dh || a.want_h) block_reduce_dd<2>(v, s_red);
  if (grid_reduce_dd<2>(v, partials, counter, s_red, tot) && threadIdx.x == 0) {
    if (a.want_dh) {
      const dd inc = dd_mul_d(tot[0], dt * a.b);
      const dd cur = {st->dh_hi, st->dh_lo};
      const dd nw2 = dd_add(cur, inc);
      st->dh_hi = nw2.hi;
      st->dh_lo = nw2.lo;
    }
    if (a.want_h) {
      st->h_hi = tot[1].hi;
      st->h_lo = tot[1].lo;
    }
    if (st->bad_code != kNoBad) st->aborted = 1;
  }
}

}  // namespace dev
}  // namespace perrk
