// Stage kernel (v2): one P-ERK stage over the stage's active cell list.
//
// Reference work it replaces, per active cell (semidisc.cpp:409-557 via
// rhs_masked :126-138, plus stepper.cpp:60-92 around it):
//   * stage-state formation U_i = U + dt (a_i1 K1 + a_i,i-1 K_{i-1}) with the
//     cell's member row (stepper.cpp:60-72), for the cell and for the face
//     traces of its neighbours (neighbour's own row);
//   * flux-differencing volume term with the Ranocha EC two-point flux
//     (semidisc.cpp:446-485, physics.cpp:157-179), diagonal via the
//     physical flux at the LGL endpoints;
//   * surface numerical flux + strong-form LGL lift (semidisc.cpp:489-556);
//   * b-stage epilogue d (+)= b K, dH += dt b <w(U_i), K_i> (stepper.cpp:52-55,
//     89-92) and the admissibility scan of every state it evaluates
//     (semidisc.cpp:596-607; SURVEY.md 7.3 H9 option (a)).
//
// Mapping (B200, FP64 pipe bound): a block of 128 threads owns CPB cells
// (3D: 8, 2D: 32), i.e. exactly one LGL line per thread per direction.  All
// warps run the same code in lock-step phases:
//   A   coalesced load + formation of the cells' stage states, per-node
//       primitives (rho, v, p, E, log rho, beta = rho/p, log beta) to smem;
//   per direction d:
//     B_d  neighbour face traces of the two d-faces (formed, checked);
//     L_d  one line task per thread: 6 symmetric EC pairs, 2 endpoint
//          diagonal fluxes and the 2 endpoint surface fluxes + lift,
//          accumulated into the cell's K tile (each node lies on exactly
//          one d-line, so the phase is conflict free);
//   E   per node epilogue (entropy products) and coalesced stores of K / d.
// Divisions are reciprocal-multiplies (MUFU seed + 2 Newton steps); the
// logarithmic means reuse the per-node logarithms, and the series branch of
// logmean (physics.cpp:30-38) is kept with the reference's threshold.
#pragma once

#include <type_traits>

// resident stage blocks per SM the register allocation targets (64 threads each)
#ifndef PERRK_STAGE_MINB
#define PERRK_STAGE_MINB 10
#endif

namespace perrk {
namespace dev {

// cp.async.bulk.prefetch.L2 (sm_90+): bytes a multiple of 16, 16-byte aligned
#ifndef PERRK_SURF_RSQ
#define PERRK_SURF_RSQ 0  // 1: the neighbour trace's sound speed as z rsqrt(z); rejected: the anchored C1 run misses the 1e-12 gamma gate (1.2e-12)
#endif

#ifndef PERRK_ST_L2PF
#define PERRK_ST_L2PF 0  // 1: the 2D / block-per-cell stage kernels prefetch the next group's blocks to L2
#endif

__device__ __forceinline__ void l2_prefetch(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <int DIM>
struct StageGeo {
  static constexpr int V = DIM + 2;
  static constexpr int NPC = DIM == 2 ? 16 : 64;  // nodes per cell
  static constexpr int FP = DIM == 2 ? 4 : 16;    // points per face
  static constexpr int NFP = 2 * DIM * FP;        // face points per cell
  static constexpr int T = 64;                    // threads per block
  static constexpr int CPB = T / NPC;             // cells per block (one node per thread)
  static constexpr int NPR = DIM + 5;             // primitives per node (see slots)
  // shared memory (doubles)
  static constexpr int SM_PR = NPR * T;           // primitives, SoA [slot][cell*NPC+node]
  static constexpr int SM_NB = CPB * NFP * V;     // neighbour traces [cell][face][pt][var]
  static constexpr int SM_TOTAL = SM_PR + SM_NB;
  // BR1 (2D NSF): own viscous fluxes [2][T][V] and neighbour face values [CPB][NFP][V]
  static constexpr int SM_VISC = 2 * T * V + CPB * NFP * V;
  static constexpr int SM_ZF = DIM == 3 ? T * V : 0;  // published z-pair fluxes
  static constexpr int SM_PF = DIM * CPB * FP * 2 * V;  // distance-2 pair fluxes
};

// primitive slots: rho, v[DIM], p, E, beta = rho / p, sound speed (the last
// only for the Rusanov surface flux)
template <int DIM>
struct Slot {
  static constexpr int RHO = 0, V0 = 1, P = DIM + 1, E = DIM + 2, BETA = DIM + 3, C = DIM + 4;
};

// a state in the primitive form the fluxes use
template <int DIM>
struct Prim {
  double rho, v[DIM], p, E;
};

template <int DIM>
__device__ __forceinline__ Prim<DIM> prim_of(const Phys& ph, const double* u, double& ir) {
  Prim<DIM> q;
  q.rho = u[0];
  ir = frcp(u[0]);
  double kin = 0.0;
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    q.v[d] = u[1 + d] * ir;
    kin = fma(u[1 + d], q.v[d], kin);
  }
  q.E = u[DIM + 1];
  q.p = ph.gm1 * (q.E - 0.5 * kin);
  return q;
}

template <int DIM>
__device__ __forceinline__ Prim<DIM> prim_of(const Phys& ph, const double* u) {
  Prim<DIM> q;
  q.rho = u[0];
  const double ir = frcp(u[0]);
  double kin = 0.0;
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    q.v[d] = u[1 + d] * ir;
    kin = fma(u[1 + d], q.v[d], kin);
  }
  q.E = u[DIM + 1];
  q.p = ph.gm1 * (q.E - 0.5 * kin);
  return q;
}

template <int DIM>
__device__ __forceinline__ bool prim_ok(const Prim<DIM>& q) {
  bool ok = (q.rho > 0.0) & (q.p > 0.0) & static_cast<bool>(isfinite(q.E));
#pragma unroll
  for (int d = 0; d < DIM; ++d) ok = ok & static_cast<bool>(isfinite(q.v[d]));
  return ok;
}

template <int DIM>
__device__ __forceinline__ double pick(const double (&v)[DIM], int d) {
  if (DIM == 2) return d == 0 ? v[0] : v[1];
  return d == 0 ? v[0] : (d == 1 ? v[1] : v[DIM - 1]);
}

// physical flux in direction d (physics.cpp:108-116)
template <int DIM>
__device__ __forceinline__ void pflux(const Prim<DIM>& q, int d, double* f) {
  const double vd = pick<DIM>(q.v, d);
  const double m = q.rho * vd;
  f[0] = m;
#pragma unroll
  for (int i = 0; i < DIM; ++i) f[1 + i] = m * q.v[i] + (i == d ? q.p : 0.0);
  f[DIM + 1] = (q.E + q.p) * vd;
}

// logmean (physics.cpp:30-38).  Below the reference's threshold
// u = ((a-b)/(a+b))^2 < 1e-4 the reference evaluates
// 0.5 (a+b) / (1 + u/3 + u^2/5 + u^3/7); here the reciprocal of that
// polynomial is taken as its series 1 - u/3 - 4u^2/45 - 44u^3/945 (the two
// differ by O(u^4) < 1e-17 relative), so the branch needs no division and u
// only to ~1e-12 relative (one Newton step on the reciprocal seed).  Above
// it: (a - b) / (log a - log b), the logarithms evaluated in that branch only:
// on smooth data (every pair of a TGV cell) no logarithm is taken at all.
// series coefficients and threshold in the constant bank: DFMA takes them as
// c[][] operands (a literal double would be rebuilt in registers every use)
__constant__ double c_lm[8] = {-11.0 / 1890.0, -1.0 / 90.0, -1.0 / 24.0, 0.125,
                               1.0 / 7.0,      1.0 / 5.0,   1.0 / 3.0,   1e-4};

// logarithm branch of lmeans (physics.cpp:37), out of line: the hot code
// stays compact (one copy instead of one per inlined flux) and it runs only
// for warps with a pair above the series threshold
__device__ __noinline__ double2 lmeans_log(double rl, double rr, double bl, double br, double k2,
                                           bool rough1, bool rough2, double lq, double ib) {
  if (rough1) lq = 0.25 * ((rl - rr) * frcp(flog(rl) - flog(rr)));
  if (rough2) ib = 0.5 * k2 * ((flog(bl) - flog(br)) * frcp(bl - br));
  return make_double2(lq, ib);
}

// Both logarithmic means of one EC pair: lq = logmean(rl, rr) / 4 and
// ib = k / logmean(bl, br) (k2 = 2 k).  The series (the factors folded into
// its coefficients) is evaluated unconditionally; a warp vote sends the warp
// to the logarithm branch only if one of its lanes has a pair above the
// threshold, and there each lane keeps the reference's choice per value.
// SMOOTH: the caller guarantees every pair is below the threshold (w3 kernel's
// per-cell range test), so the series is taken without the vote and branch
// and consecutive fluxes schedule as one straight-line block.
template <bool SMOOTH = false>
__device__ __forceinline__ void lmeans(double rl, double rr, double bl, double br, double k2,
                                       double& lq, double& ib) {
  const double s1 = rl + rr, d1 = rl - rr;
  double r1;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r1) : "d"(s1));
  r1 = fma(r1, fma(-s1, r1, 1.0), r1);
  const double f1 = d1 * r1, u1 = f1 * f1;
  lq = s1 * fma(u1, fma(u1, fma(u1, c_lm[0], c_lm[1]), c_lm[2]), c_lm[3]);
  const double s2 = bl + br, d2 = bl - br;
  const double rs = frcp(s2);
  const double f2 = d2 * rs, u2 = f2 * f2;
  ib = fma(u2, fma(u2, fma(u2, c_lm[4], c_lm[5]), c_lm[6]), 1.0) * (k2 * rs);
  if (SMOOTH) return;
  const bool rough1 = !(u1 < c_lm[7]), rough2 = !(u2 < c_lm[7]);
  if (__any_sync(__activemask(), rough1 || rough2)) {
    const double2 r = lmeans_log(rl, rr, bl, br, k2, rough1, rough2, lq, ib);
    lq = r.x;
    ib = r.y;
  }
}

// Ranocha EC flux (physics.cpp:157-179) from primitives and beta = rho / p:
// with sigma = v_l + v_r, t = logmean(rho) sigma_d / 4,
//   f_rho = 2 t,  f_m,i = t sigma_i + delta_id (p_l + p_r) / 2,
//   f_E = f_rho (v_l.v_r / 2 + 1 / ((gamma - 1) logmean(beta))) + (p_l v_r,d + p_r v_l,d) / 2
// HP: pl and pr arrive halved (p / 2, as the warp kernels store them), which
// folds the two 1/2 factors of the pressure terms into the stored value
template <int DIM, bool SMOOTH = false, bool HP = false>
__device__ __forceinline__ void ec2(const Phys& ph, int d, double rl, const double (&vl)[DIM],
                                    double pl, double bl, double rr, const double (&vr)[DIM],
                                    double pr, double br, double* f) {
  double lq, ib;
  lmeans<SMOOTH>(rl, rr, bl, br, 2.0 * ph.inv_gm1, lq, ib);
  double sg[DIM], vlvr = 0.0;
#pragma unroll
  for (int i = 0; i < DIM; ++i) {
    sg[i] = vl[i] + vr[i];
    vlvr = fma(vl[i], vr[i], vlvr);
  }
  const double t = lq * pick<DIM>(sg, d);
  const double fr = t + t;
  f[0] = fr;
  const double pavg = HP ? pl + pr : 0.5 * (pl + pr);
#pragma unroll
  for (int i = 0; i < DIM; ++i) f[1 + i] = i == d ? fma(t, sg[i], pavg) : t * sg[i];
  const double pv = fma(pl, pick<DIM>(vr, d), pr * pick<DIM>(vl, d));
  f[DIM + 1] = fma(fr, fma(0.5, vlvr, ib), HP ? pv : 0.5 * pv);
}

// Roe-average wave speed estimates (physics.cpp:181-203)
template <int DIM>
__device__ __forceinline__ void wse(const Phys& ph, const Prim<DIM>& l, const Prim<DIM>& r, int d,
                                    double& sl, double& sr) {
  // fsqrt (~1 ulp, no slow path) on the admissible states' positive arguments
  const double cl = fsqrt(ph.gamma * l.p * frcp(l.rho)), cr = fsqrt(ph.gamma * r.p * frcp(r.rho));
  const double sql = fsqrt(l.rho), sqr = fsqrt(r.rho);
  const double iw = frcp(sql + sqr);
  const double hl = (l.E + l.p) * frcp(l.rho), hr = (r.E + r.p) * frcp(r.rho);
  double v2 = 0.0, vd = 0.0;
#pragma unroll
  for (int i = 0; i < DIM; ++i) {
    const double vroe = (sql * l.v[i] + sqr * r.v[i]) * iw;
    v2 = fma(vroe, vroe, v2);
    if (i == d) vd = vroe;
  }
  const double hroe = (sql * hl + sqr * hr) * iw;
  const double c2roe = ph.gm1 * (hroe - 0.5 * v2);
  const double croe = c2roe > 0.0 ? fsqrt(c2roe) : 0.0;
  sl = fmin(pick<DIM>(l.v, d) - cl, vd - croe);
  sr = fmax(pick<DIM>(r.v, d) + cr, vd + croe);
}

template <int DIM>
__device__ __forceinline__ void cons_of(const Prim<DIM>& q, double* u) {
  u[0] = q.rho;
#pragma unroll
  for (int i = 0; i < DIM; ++i) u[1 + i] = q.rho * q.v[i];
  u[DIM + 1] = q.E;
}

// surface numerical flux f*(l, r) in direction d (physics.cpp:40-65,181-258)
template <int DIM, int SURF>
__device__ __forceinline__ void sflux(const Phys& ph, const Prim<DIM>& l, const Prim<DIM>& r,
                                      int d, double* f) {
  constexpr int V = DIM + 2;
  if constexpr (SURF == 5) {
    const double bl = l.rho * frcp(l.p), br = r.rho * frcp(r.p);
    ec2<DIM>(ph, d, l.rho, l.v, l.p, bl, r.rho, r.v, r.p, br, f);
    return;
  }
  double fl[V], fr[V];
  pflux<DIM>(l, d, fl);
  pflux<DIM>(r, d, fr);
  if constexpr (SURF == 0) {
#pragma unroll
    for (int v = 0; v < V; ++v) f[v] = 0.5 * (fl[v] + fr[v]);
  } else if constexpr (SURF == 2) {
    const double lam = fmax(fabs(pick<DIM>(l.v, d)) + fsqrt(ph.gamma * l.p * frcp(l.rho)),
                            fabs(pick<DIM>(r.v, d)) + fsqrt(ph.gamma * r.p * frcp(r.rho)));
    double ul[V], ur[V];
    cons_of<DIM>(l, ul);
    cons_of<DIM>(r, ur);
#pragma unroll
    for (int v = 0; v < V; ++v) f[v] = 0.5 * (fl[v] + fr[v]) - 0.5 * lam * (ur[v] - ul[v]);
  } else if constexpr (SURF == 3) {
    double sl, sr;
    wse<DIM>(ph, l, r, d, sl, sr);
    if (sl >= 0.0) {
#pragma unroll
      for (int v = 0; v < V; ++v) f[v] = fl[v];
    } else if (sr <= 0.0) {
#pragma unroll
      for (int v = 0; v < V; ++v) f[v] = fr[v];
    } else {
      double ul[V], ur[V];
      cons_of<DIM>(l, ul);
      cons_of<DIM>(r, ur);
      const double inv = frcp(sr - sl);
#pragma unroll
      for (int v = 0; v < V; ++v) f[v] = (sr * fl[v] - sl * fr[v] + sl * sr * (ur[v] - ul[v])) * inv;
    }
  } else {  // SURF == 4: HLLC
    double sl, sr;
    wse<DIM>(ph, l, r, d, sl, sr);
    if (sl >= 0.0) {
#pragma unroll
      for (int v = 0; v < V; ++v) f[v] = fl[v];
    } else if (sr <= 0.0) {
#pragma unroll
      for (int v = 0; v < V; ++v) f[v] = fr[v];
    } else {
      const double vl = pick<DIM>(l.v, d), vr = pick<DIM>(r.v, d);
      const double s_star = fdiv(r.p - l.p + l.rho * vl * (sl - vl) - r.rho * vr * (sr - vr),
                                 l.rho * (sl - vl) - r.rho * (sr - vr));
      const bool left = s_star >= 0.0;
      const Prim<DIM>& k = left ? l : r;
      const double sk = left ? sl : sr, vk = left ? vl : vr;
      const double* fk = left ? fl : fr;
      const double factor = fdiv(k.rho * (sk - vk), sk - s_star);
      double uk[V], us[V];
      cons_of<DIM>(k, uk);
      us[0] = factor;
#pragma unroll
      for (int i = 0; i < DIM; ++i) us[1 + i] = factor * (i == d ? s_star : k.v[i]);
      us[DIM + 1] = factor * (k.E * frcp(k.rho) +
                              (s_star - vk) * (s_star + fdiv(k.p, k.rho * (sk - vk))));
#pragma unroll
      for (int v = 0; v < V; ++v) f[v] = fk[v] + sk * (us[v] - uk[v]);
    }
  }
}

// a[d] for a runtime direction d without a local-memory array
template <int DIM, typename A>
__device__ __forceinline__ double pick_rt(const A& a, int off, int d) {
  if (DIM == 2) return d == 0 ? a[off] : a[off + 1];
  return d == 0 ? a[off] : (d == 1 ? a[off + 1] : a[off + 2]);
}

// Rusanov (physics.cpp:52-59) or central (:46-50) surface flux at one face
// point, runtime direction d, returned as the lifted contribution to the own
// trace node (semidisc.cpp:489-556 strong form; weak form: the lift of f*
// alone) plus the endpoint diagonal term -2J D_jj f(u_o) (:450-454).  With o
// the own trace and n the neighbour's,
//   f* - f(u_o) = 1/2 (f_n - f_o) + s 1/2 lam (u_n - u_o),
// s = +1 when the own node is the right state (side 0) and -1 when it is the
// left one (side 1), lam = max(|v_o,d| + c_o, |v_n,d| + c_n).  One code copy
// for all faces (runtime d, side) keeps the kernel's instruction footprint
// small.  Own primitives (and sound speed) come from shared memory; the
// neighbour's conservative trace from registers.  Returns admissibility of
// the neighbour's trace.
template <int DIM, int SURF>
__device__ __forceinline__ bool rus_lift_v(const Phys& ph, double ro, const double (&vo)[DIM],
                                           double po, double Eo, double co,
                                           const double (&un)[DIM + 2], int d, int side,
                                           double cll, double sg, bool weak, double* out) {
  constexpr int V = DIM + 2;
  const double rn = un[0], En = un[V - 1];
  const double irn = frcp(rn);
  double vn[DIM], kin = 0.0;
#pragma unroll
  for (int i = 0; i < DIM; ++i) {
    vn[i] = un[1 + i] * irn;
    kin = fma(un[1 + i], vn[i], kin);
  }
  const double pn = ph.gm1 * (En - 0.5 * kin);
  // (no short-circuit: the tests stay straight-line code)
  bool ok = (rn > 0.0) & (pn > 0.0) & static_cast<bool>(isfinite(En));
#pragma unroll
  for (int i = 0; i < DIM; ++i) ok = ok & static_cast<bool>(isfinite(vn[i]));
  const double vod = pick_rt<DIM>(vo, 0, d), vnd = pick_rt<DIM>(vn, 0, d);
  const double mnd = pick_rt<DIM>(un, 1, d), mod = ro * vod;
  double fo[V], g[V];
  fo[0] = mod;
  g[0] = 0.5 * (mnd - mod);
#pragma unroll
  for (int i = 0; i < DIM; ++i) {
    fo[1 + i] = fma(mod, vo[i], i == d ? po : 0.0);
    g[1 + i] = 0.5 * (fma(mnd, vn[i], i == d ? pn : 0.0) - fo[1 + i]);
  }
  fo[V - 1] = (Eo + po) * vod;
  g[V - 1] = 0.5 * ((En + pn) * vnd - fo[V - 1]);
  if constexpr (SURF == 2) {
    // sqrt(z) = z rsqrt(z), without fsqrt's last correction step (~1.5 ulp)
    const double zn = ph.gamma * pn * irn;
    const double lam = fmax(fabs(vod) + co, fabs(vnd) + (PERRK_SURF_RSQ ? zn * frsqrt(zn) : fsqrt(zn)));
    const double hl = side ? -0.5 * lam : 0.5 * lam;
    g[0] = fma(hl, rn - ro, g[0]);
#pragma unroll
    for (int i = 0; i < DIM; ++i) g[1 + i] = fma(hl, un[1 + i] - ro * vo[i], g[1 + i]);
    g[V - 1] = fma(hl, En - Eo, g[V - 1]);
  }
  if (weak) {
#pragma unroll
    for (int v = 0; v < V; ++v) out[v] = sg * (g[v] + fo[v]);
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v) out[v] = fma(sg, g[v], -cll * fo[v]);
  }
  return ok;
}

// rus_lift_v with the own trace's primitives from the block-per-cell
// kernel's shared-memory slots
template <int DIM, int SURF>
__device__ __forceinline__ bool rus_lift(const Phys& ph, const double* pr, int oq,
                                         const double (&un)[DIM + 2], int d, int side,
                                         double cll, double sg, bool weak, double* out) {
  using S = Slot<DIM>;
  constexpr int T = StageGeo<DIM>::T;
  double vo[DIM];
#pragma unroll
  for (int i = 0; i < DIM; ++i) vo[i] = pr[(S::V0 + i) * T + oq];
  return rus_lift_v<DIM, SURF>(ph, pr[S::RHO * T + oq], vo, pr[S::P * T + oq], pr[S::E * T + oq],
                               SURF == 2 ? pr[S::C * T + oq] : 0.0, un, d, side, cll, sg, weak,
                               out);
}

template <int DIM>
__device__ __forceinline__ int line_base(int d, int t1, int t2) {
  if (DIM == 2) return d == 0 ? N1 * t1 : t1;
  return d == 0 ? N1 * t1 + N1 * N1 * t2 : (d == 1 ? t1 + N1 * N1 * t2 : t1 + N1 * t2);
}

__device__ __forceinline__ int line_stride(int d) { return d == 0 ? 1 : (d == 1 ? N1 : N1 * N1); }

__device__ __forceinline__ int pick_int3(const int (&a)[3], int i) {
  return i == 0 ? a[0] : (i == 1 ? a[1] : a[2]);
}

// Flux-differencing volume term of one node along direction D (compile-time,
// so velocity components, strides and flux slots resolve statically).
template <int DIM, int D>
__device__ __forceinline__ void volume_terms(const Phys& ph, const double* pr, int tid,
                                             const int (&il)[3], double J2, const Prim<DIM>& own,
                                             double be, const double* cf, double* K,
                                             double* zf = nullptr) {
  using G = StageGeo<DIM>;
  using S = Slot<DIM>;
  constexpr int V = G::V, T = G::T;
  constexpr int stride = D == 0 ? 1 : (D == 1 ? N1 : N1 * N1);
  const int j = il[D];
  // ---- volume: the three partners on this node's D-line (semidisc.cpp:455-464).
  // Lines along x and y lie inside a warp (node = ix + 4 iy + 16 iz), so each
  // symmetric pair is evaluated once: lane j computes f(j, j+1 mod 4) and
  // receives f(j-1, j) from its neighbour by shuffle; the distance-2 pair is
  // evaluated by both ends.  Along z the lines cross warps: every lane
  // evaluates its three pairs.  The EC flux is symmetric in its arguments up
  // to the order of commutative operations.
  auto ec_with = [&](int k, double* f) {
    const int qk = tid + (k - j) * stride;
    double vk[DIM];
#pragma unroll
    for (int i = 0; i < DIM; ++i) vk[i] = pr[(S::V0 + i) * T + qk];
    ec2<DIM>(ph, D, own.rho, own.v, own.p, be, pr[S::RHO * T + qk], vk, pr[S::P * T + qk],
             pr[S::BETA * T + qk], f);
  };
  // the distance-2 pair (j, j+2) is evaluated once per pair by dist2_pairs
  // and gathered after the block's next barrier (dist2_gather)
  const int kn = (j + 1) & (N1 - 1);
  double f1[V];
  ec_with(kn, f1);
  const double cn = J2 * cf[(3 * D) * T + tid];
#pragma unroll
  for (int v = 0; v < V; ++v) K[v] = fma(-cn, f1[v], K[v]);
  if constexpr (D < 2) {
    const int kp = (j + N1 - 1) & (N1 - 1);
    const int src = (threadIdx.x & 31) + (kp - j) * stride;
    const double cp = J2 * cf[(3 * D + 1) * T + tid];
#pragma unroll
    for (int v = 0; v < V; ++v) K[v] = fma(-cp, __shfl_sync(0xffffffffu, f1[v], src), K[v]);
  } else {
    // z-lines cross warps: f(j, j+1) is published in shared memory and the
    // partner's f(j-1, j) is picked up after the block's next barrier (zf_gather)
#pragma unroll
    for (int v = 0; v < V; ++v) zf[tid * V + v] = f1[v];
  }
}

// Distance-2 pairs (0,2) and (1,3) of every LGL line, each evaluated once:
// pair p = ((d * CPB + cell) * FP + line) * 2 + lower end; a warp's 32 pairs
// share the direction, so the flux kernel is selected per warp.
template <int DIM>
__device__ __forceinline__ void dist2_pairs(const Phys& ph, const double* pr, double* pf, int tid) {
  using G = StageGeo<DIM>;
  using S = Slot<DIM>;
  constexpr int V = G::V, T = G::T, FP = G::FP, CPB = G::CPB, NPC = G::NPC;
  constexpr int NP = DIM * CPB * FP * 2;
#pragma unroll
  for (int r = 0; r < (NP + T - 1) / T; ++r) {
    // a partial last round goes to the upper warp: the surface phase's
    // partial round (96 face points on 64 threads in 3D) runs on the lower one
    const int p = (r ? tid ^ 32 : tid) + r * T;
    if (p >= NP) break;
    const int d = p / (CPB * FP * 2), rem = p % (CPB * FP * 2);
    const int c2 = rem / (FP * 2), li = (rem / 2) % FP, which = rem & 1;
    const int lo = c2 * NPC + line_base<DIM>(d, li % N1, li / N1) + which * line_stride(d);
    const int hi = lo + 2 * line_stride(d);
    double vl[DIM], vr[DIM];
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
      vl[i] = pr[(S::V0 + i) * T + lo];
      vr[i] = pr[(S::V0 + i) * T + hi];
    }
    double f[V];
    auto run = [&](auto dc) {
      constexpr int Dd = decltype(dc)::value;
      ec2<DIM>(ph, Dd, pr[S::RHO * T + lo], vl, pr[S::P * T + lo], pr[S::BETA * T + lo],
               pr[S::RHO * T + hi], vr, pr[S::P * T + hi], pr[S::BETA * T + hi], f);
    };
    if (d == 0)
      run(std::integral_constant<int, 0>{});
    else if (d == 1)
      run(std::integral_constant<int, 1>{});
    else
      run(std::integral_constant<int, DIM - 1>{});
#pragma unroll
    for (int v = 0; v < V; ++v) pf[p * V + v] = f[v];
  }
}

// per-thread constants of the volume and gather phases, set once per launch
// (kernel prologue) so the group loop reads them with fixed-offset shared
// loads instead of re-deriving node indices: [3 d + 0/1/2][T] the SBP
// coefficients D_{j,j+1}, D_{j,j-1}, D_{j,j^2} of the node's d-line, and
// integer offsets (in doubles) of the node's distance-2 pair flux per d, of
// its z-partner's published pair flux, and of its face slots per d (-1: the
// node is not on a d-face).
template <int DIM>
struct ThreadTab {
  static constexpr int NCF = 3 * DIM;
  static constexpr int I_D2 = 0, I_ZF = DIM, I_FACE = DIM + 1, NI = 2 * DIM + 1;
};

template <int DIM>
__device__ __forceinline__ void thread_tab_init(double* cf, int* ti, int tid, int cs,
                                                const int (&il)[3]) {
  using G = StageGeo<DIM>;
  using TT = ThreadTab<DIM>;
  constexpr int V = G::V, FP = G::FP, CPB = G::CPB, T = G::T, NFP = G::NFP;
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    const int j = il[d];
    cf[(3 * d + 0) * T + tid] = c_D[j * N1 + ((j + 1) & (N1 - 1))];
    cf[(3 * d + 1) * T + tid] = c_D[j * N1 + ((j + N1 - 1) & (N1 - 1))];
    cf[(3 * d + 2) * T + tid] = c_D[j * N1 + (j ^ 2)];
    const int li = d == 0 ? il[1] + N1 * il[2] : (d == 1 ? il[0] + N1 * il[2] : il[0] + N1 * il[1]);
    ti[(TT::I_D2 + d) * T + tid] = (((d * CPB + cs) * FP + li) * 2 + (j & 1)) * V;
    ti[(TT::I_FACE + d) * T + tid] =
        (j == 0 || j == N1 - 1) ? ((cs * NFP + (2 * d + (j ? 1 : 0)) * FP) + li) * V : -1;
  }
  const int jz = il[2], kz = (jz + N1 - 1) & (N1 - 1);
  ti[TT::I_ZF * T + tid] = (tid + (kz - jz) * N1 * N1) * V;
}

template <int DIM>
__device__ __forceinline__ void dist2_gather(const double* pf, const double* cf, const int* ti,
                                             int tid, const double* J2, double* K) {
  using G = StageGeo<DIM>;
  constexpr int V = G::V, T = G::T;
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    const double c2 = J2[d] * cf[(3 * d + 2) * T + tid];
    const double* f = pf + ti[(ThreadTab<DIM>::I_D2 + d) * T + tid];
#pragma unroll
    for (int v = 0; v < V; ++v) K[v] = fma(-c2, f[v], K[v]);
  }
}

// the z-partner's published pair flux f(j-1, j) (after a block barrier)
template <int DIM>
__device__ __forceinline__ void zf_gather(const double* zf, const double* cf, const int* ti,
                                          int tid, double J2, double* K) {
  constexpr int V = DIM + 2, T = StageGeo<DIM>::T;
  const double cp = J2 * cf[(3 * 2 + 1) * T + tid];
  const double* f = zf + ti[ThreadTab<DIM>::I_ZF * T + tid];
#pragma unroll
  for (int v = 0; v < V; ++v) K[v] = fma(-cp, f[v], K[v]);
}

// Volume term without the EC flux (SIMPLE kernels), along direction D:
//   weak form (semidisc.cpp:429-445):  K += J sum_m D_mj w_m / w_j f(u_m);
//   flux differencing with the central two-point flux 1/2 (f_j + f_m)
//   (semidisc.cpp:446-485 with FluxTag::central): K -= 2 J sum_{m != j} D_jm f*,
//   the diagonal -2 J D_jj f(u_j) being added by the surface phase as for EC.
// The physical fluxes of the line's nodes come from the primitives in smem.
template <int DIM, int D>
__device__ __forceinline__ void simple_volume(const double* pr, int tid, const int (&il)[3],
                                              double J2, const Prim<DIM>& own, bool weak,
                                              double* K) {
  using G = StageGeo<DIM>;
  using S = Slot<DIM>;
  constexpr int V = G::V, T = G::T;
  constexpr int stride = D == 0 ? 1 : (D == 1 ? N1 : N1 * N1);
  const int j = il[D];
  double fj[V];
  pflux<DIM>(own, D, fj);
#pragma unroll
  for (int m = 0; m < N1; ++m) {
    double f[V];
    if (m == j) {
#pragma unroll
      for (int v = 0; v < V; ++v) f[v] = fj[v];
    } else {
      const int q = tid + (m - j) * stride;
      Prim<DIM> pm;
      pm.rho = pr[S::RHO * T + q];
#pragma unroll
      for (int i = 0; i < DIM; ++i) pm.v[i] = pr[(S::V0 + i) * T + q];
      pm.p = pr[S::P * T + q];
      pm.E = pr[S::E * T + q];
      pflux<DIM>(pm, D, f);
    }
    if (weak) {
      const double coef = 0.5 * J2 * c_D[m * N1 + j] * c_w[m] / c_w[j];
#pragma unroll
      for (int v = 0; v < V; ++v) K[v] = fma(coef, f[v], K[v]);
    } else if (m != j) {
      const double coef = J2 * c_D[j * N1 + m];
#pragma unroll
      for (int v = 0; v < V; ++v) K[v] = fma(-coef, 0.5 * (fj[v] + f[v]), K[v]);
    }
  }
}

template <int DIM, int SURF, bool VISC, bool SIMPLE>
__global__ void __launch_bounds__(StageGeo<DIM>::T, (VISC || SURF >= 3) ? 8 : PERRK_STAGE_MINB)
    stage_kernel(StageArgs a, MeshDev m, Phys ph, StepState* st, double* partials,
                 unsigned* counter) {
  using G = StageGeo<DIM>;
  using S = Slot<DIM>;
  constexpr int V = G::V, NPC = G::NPC, FP = G::FP, NFP = G::NFP, CPB = G::CPB, T = G::T;
  constexpr int NQ = (CPB * NFP + T - 1) / T;  // face points per thread
  extern __shared__ double smem[];
  double* pr = smem;            // [NPR][T] per-node primitives
  double* sf = pr + G::SM_PR;   // [CPB][NFP][V] surface + diagonal terms per face point
  double* zf = sf + G::SM_NB;   // 3D: published z-pair fluxes [T][V]
  double* pf = zf + G::SM_ZF;   // distance-2 pair fluxes [DIM*CPB*FP*2][V]
  double* vg = pf + G::SM_PF;   // VISC: own G [2][T][V], then neighbour G_d [CPB][NFP][V]
  double* vn = vg + 2 * T * V;
  // group descriptors, double-buffered: the next group's are written while
  // the current one computes
  __shared__ int s_cell_[2][CPB];
  __shared__ double s_ca1_[2][CPB];
  __shared__ signed char s_cform_[2][CPB];
  __shared__ int s_lev_[2][CPB];
  __shared__ double s_J2_[2][CPB][DIM], s_lift_[2][CPB][DIM];
  __shared__ double s_meas_[2][CPB];  // h_x h_y (h_z) / 2^DIM of the cell
  __shared__ int s_nbc_[2][CPB][2 * DIM];        // local neighbour, or -1 - face cell (ghost)
  __shared__ double s_na1_[2][CPB][2 * DIM];
  __shared__ signed char s_nform_[2][CPB][2 * DIM];
  __shared__ double s_red[2 * 2 * (T / 32)];

  __shared__ double s_cf[ThreadTab<DIM>::NCF * T];
  __shared__ int s_ti[ThreadTab<DIM>::NI * T];

  if (st->aborted || st->finished) return;  // uniform across the grid
  const int tid = threadIdx.x;
  const double dt = st->dt;
  const int cs = tid / NPC, l = tid % NPC;
  const int il[3] = {l % N1, (l / N1) % N1, l / (N1 * N1)};  // node position per axis
  thread_tab_init<DIM>(s_cf, s_ti, tid, cs, il);
  dd acc_dh = dd_zero(), acc_h = dd_zero();
  // max |d| as the bit pattern of |d| (non-negative doubles order like their
  // bits; a NaN or inf lands at or above the infinity pattern)
  unsigned long long dmax_bits = 0;
  const int ngroups = (a.n + CPB - 1) / CPB;

  // descriptor of one group (threads < CPB, one cell each) into buffer b
  // group descriptor of one cell into buffer b from its static record
  // (host.cpp build_cell_records: neighbours, geometry, levels; 6 vector loads)
  auto describe = [&](int b, int t, int cell) {
      s_cell_[b][t] = cell;
      if (cell < 0) return;
      const int4* ri = reinterpret_cast<const int4*>(m.rec + cell);
      const double2* rd = reinterpret_cast<const double2*>(m.rec + cell);
      const int4 n0 = __ldg(ri), n1 = __ldg(ri + 1);
      const double2 j01 = __ldg(rd + 2), j2l0 = __ldg(rd + 3), l12 = __ldg(rd + 4),
                    ml = __ldg(rd + 5);
      const unsigned long long lv = static_cast<unsigned long long>(__double_as_longlong(ml.y));
      const int lev = static_cast<int>(lv & 0xff);
      s_ca1_[b][t] = dt * a.a1[lev];
      s_cform_[b][t] = a.formed[lev];
      s_lev_[b][t] = lev;
      s_meas_[b][t] = ml.x;
      const double J2[3] = {j01.x, j01.y, j2l0.x}, lift[3] = {j2l0.y, l12.x, l12.y};
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        s_J2_[b][t][d] = J2[d];
        s_lift_[b][t][d] = lift[d];
      }
      const int nb[6] = {n0.x, n0.y, n0.z, n0.w, n1.x, n1.y};
#pragma unroll
      for (int f = 0; f < 2 * DIM; ++f) {  // face neighbours (local or ghost slot), rows
        const int nbc = nb[f];
        s_nbc_[b][t][f] = nbc;
        if (nbc < 0) {  // trace formed and sent by the neighbour's owner
          s_na1_[b][t][f] = 0.0;
          s_nform_[b][t][f] = 1;
        } else {
          const int l2 = static_cast<int>((lv >> (8 * (1 + f))) & 0xff);
          s_na1_[b][t][f] = dt * a.a1[l2];
          s_nform_[b][t][f] = a.formed[l2];
        }
      }
  };

  // first group's descriptors; afterwards each group describes the next one
  // while it computes (list -> cell -> level chains resolve off the critical path)
  if (tid < CPB) {
    const int slot = blockIdx.x * CPB + tid;
    describe(0, tid, slot < a.n ? (a.list ? a.list[slot] : slot) : -1);
  }
  __syncthreads();
  int buf = 0;
  for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x, buf ^= 1) {
    auto& s_cell = s_cell_[buf];
    auto& s_ca1 = s_ca1_[buf];
    auto& s_cform = s_cform_[buf];
    auto& s_lev = s_lev_[buf];
    auto& s_meas = s_meas_[buf];
    auto& s_J2 = s_J2_[buf];
    auto& s_lift = s_lift_[buf];
    auto& s_nbc = s_nbc_[buf];
    auto& s_na1 = s_na1_[buf];
    auto& s_nform = s_nform_[buf];
    // the last CPB threads fetch and describe the next group
    const int dt_t = tid - (T - CPB);
    int nx_cell = -1;
    if (dt_t >= 0) {
      const int slot = (grp + gridDim.x) * CPB + dt_t;
      nx_cell = slot < a.n ? (a.list ? a.list[slot] : slot) : -1;
    }
    const int cell = s_cell[cs];
    // the next group's own cells go to L2 now (bulk prefetch, contiguous
    // NPC*V doubles per array), so its loads hit L2 instead of HBM
    if (PERRK_ST_L2PF && dt_t >= 0 && nx_cell >= 0) {
      constexpr unsigned kBytes = NPC * V * sizeof(double);
      const size_t off = static_cast<size_t>(nx_cell) * NPC * V;
      if (a.form) l2_prefetch(a.Us + off, kBytes);
      if (!a.form || a.write_next) l2_prefetch(a.U + off, kBytes);  // stage 0 state / epilogue
      if (a.write_next && a.form) l2_prefetch(a.K1 + off, kBytes);  // epilogue formation
      if (a.d_mode == 2) l2_prefetch(a.d + off, kBytes);              // d read-modify-write
    }
    // ---- load: own node (coalesced: consecutive threads, consecutive nodes),
    // formed with the cell's member row (stepper.cpp:60-72) ------------------
    Prim<DIM> own;
    own.rho = 1.0;  // padding lanes (tail group) compute on a dummy state
    own.p = 1.0;
    own.E = 2.5;
#pragma unroll
    for (int i = 0; i < DIM; ++i) own.v[i] = 0.0;
    double be = 1.0;
    if (cell >= 0) {
      // device layout (sidx): variable v at gi + v NPC
      const size_t gi = static_cast<size_t>(cell) * NPC * V + l;
      double u[V];
      // U_i: from the previous stage's epilogue, or formed here from the first
      // column (cells that were inactive at i-1, whose a_{i,i-1} = 0)
      if (!a.form) {
#pragma unroll
        for (int v = 0; v < V; ++v) u[v] = __ldg(a.U + gi + v * NPC);
      } else if (s_cform[cs]) {
#pragma unroll
        for (int v = 0; v < V; ++v) u[v] = __ldg(a.Us + gi + v * NPC);
      } else {
        const double a1 = s_ca1[cs];
#pragma unroll
        for (int v = 0; v < V; ++v)
          u[v] = fma(a1, __ldg(a.K1 + gi + v * NPC), __ldg(a.U + gi + v * NPC));
      }
      double ir;
      own = prim_of<DIM>(ph, u, ir);
      if (!prim_ok<DIM>(own)) report_bad(st, a.stage, a.ncells, m.gid ? m.gid[cell] : cell);
      if constexpr (SURF == 2) pr[S::C * T + tid] = fsqrt(ph.gamma * own.p * ir);
      be = own.rho * frcp(own.p);
      pr[S::RHO * T + tid] = own.rho;
#pragma unroll
      for (int i = 0; i < DIM; ++i) pr[(S::V0 + i) * T + tid] = own.v[i];
      pr[S::P * T + tid] = own.p;
      pr[S::E * T + tid] = own.E;
      pr[S::BETA * T + tid] = be;
    }
    // ---- this thread's face points: the neighbour's trace, formed with the
    // neighbour's row (or received from the neighbouring slab), kept in
    // registers across the barrier --------------------------------------------
    double nbu[NQ][V];
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      const int q = tid + k * T;
      if (q >= CPB * NFP) break;
      const int c2 = q / NFP, r = q % NFP, f = r / FP, pt = r % FP;
      const int d = f >> 1, side = f & 1;
      if (s_cell[c2] < 0) continue;
      const int nbc = s_nbc[c2][f];
      if (nbc < 0) {
        const double* g = m.ghost + (static_cast<size_t>(-1 - nbc) * FP + pt) * V;
#pragma unroll
        for (int v = 0; v < V; ++v) nbu[k][v] = g[v];
        continue;
      }
      // the neighbour's node on the shared face: far end of the same line
      const int node =
          line_base<DIM>(d, pt % N1, pt / N1) + (side ? 0 : N1 - 1) * line_stride(d);
      const size_t gi = static_cast<size_t>(nbc) * NPC * V + node;
      if (!a.form) {
#pragma unroll
        for (int v = 0; v < V; ++v) nbu[k][v] = __ldg(a.U + gi + v * NPC);
      } else if (s_nform[c2][f]) {
#pragma unroll
        for (int v = 0; v < V; ++v) nbu[k][v] = __ldg(a.Us + gi + v * NPC);
      } else {
        const double b1 = s_na1[c2][f];
#pragma unroll
        for (int v = 0; v < V; ++v)
          nbu[k][v] = fma(b1, __ldg(a.K1 + gi + v * NPC), __ldg(a.U + gi + v * NPC));
      }
    }
    if constexpr (VISC) {  // BR1 viscous fluxes from grad_kernel (2D)
      const size_t nd = static_cast<size_t>(a.ndofs);
      if (cell >= 0) {
        const size_t gi = static_cast<size_t>(cell) * NPC * V + l;
#pragma unroll
        for (int v = 0; v < V; ++v) {  // [dir][V][T]: conflict-free 8-byte accesses
          vg[v * T + tid] = a.G[gi + v * NPC];
          vg[(V + v) * T + tid] = a.G[nd + gi + v * NPC];
        }
      }
      for (int q = tid; q < CPB * NFP; q += T) {
        const int c2 = q / NFP, r = q % NFP, f = r / FP, pt = r % FP;
        if (s_cell[c2] < 0) continue;
        const int d = f >> 1, side = f & 1;
        const int node =
            line_base<DIM>(d, pt % N1, pt / N1) + (side ? 0 : N1 - 1) * line_stride(d);
        const size_t gi = static_cast<size_t>(s_nbc[c2][f]) * NPC * V + node + d * nd;
#pragma unroll
        for (int v = 0; v < V; ++v) vn[v * (CPB * NFP) + q] = a.G[gi + v * NPC];  // [V][face pt]
      }
    }
    __syncthreads();

    // ---- surface flux + strong-form lift and the endpoint diagonal term, one
    // face point per thread (semidisc.cpp:489-556, diagonal :450-454) ----------
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      const int q = tid + k * T;
      if (q >= CPB * NFP) break;
      const int c2 = q / NFP, r = q % NFP, f = r / FP, pt = r % FP;
      const int d = f >> 1, side = f & 1;
      if (s_cell[c2] < 0) continue;
      const int own_q = c2 * NPC + line_base<DIM>(d, pt % N1, pt / N1) +
                        (side ? N1 - 1 : 0) * line_stride(d);
      if constexpr (SURF == 0 || SURF == 2) {
        const double J2 = s_J2[c2][d], lift = s_lift[c2][d];
        const int j = side ? N1 - 1 : 0;
        double o5[V];
        const bool ok = rus_lift<DIM, SURF>(ph, pr, own_q, nbu[k], d, side, J2 * c_D[j * N1 + j],
                                            side ? -lift : lift, SIMPLE && a.weak, o5);
        if (!ok) {
          const int nb = s_nbc[c2][f];  // global id of the neighbour, only on failure
          report_bad(st, a.stage, a.ncells,
                     nb < 0 ? m.ghost_gid[-1 - nb] : (m.gid ? m.gid[nb] : nb));
        }
#pragma unroll
        for (int v = 0; v < V; ++v) sf[q * V + v] = o5[v];
        continue;
      }
      Prim<DIM> o;
      o.rho = pr[S::RHO * T + own_q];
#pragma unroll
      for (int i = 0; i < DIM; ++i) o.v[i] = pr[(S::V0 + i) * T + own_q];
      o.p = pr[S::P * T + own_q];
      o.E = pr[S::E * T + own_q];
      const Prim<DIM> nbp = prim_of<DIM>(ph, nbu[k]);
      if (!prim_ok<DIM>(nbp)) {
        const int nb = s_nbc[c2][f];  // global id of the neighbour, only on failure
        report_bad(st, a.stage, a.ncells,
                   nb < 0 ? m.ghost_gid[-1 - nb] : (m.gid ? m.gid[nb] : nb));
      }
      double fs[V], fo[V];
      const double J2 = s_J2[c2][d], lift = s_lift[c2][d];
      const int j = side ? N1 - 1 : 0;
      const double cll = J2 * c_D[j * N1 + j];
      const double sg = side ? -lift : lift;
      // compile-time direction for the flux kernels
      if (d == 0) {
        pflux<DIM>(o, 0, fo);
        if (side) sflux<DIM, SURF>(ph, o, nbp, 0, fs); else sflux<DIM, SURF>(ph, nbp, o, 0, fs);
      } else if (d == 1) {
        pflux<DIM>(o, 1, fo);
        if (side) sflux<DIM, SURF>(ph, o, nbp, 1, fs); else sflux<DIM, SURF>(ph, nbp, o, 1, fs);
      } else {
        pflux<DIM>(o, DIM - 1, fo);
        if (side) sflux<DIM, SURF>(ph, o, nbp, DIM - 1, fs);
        else sflux<DIM, SURF>(ph, nbp, o, DIM - 1, fs);
      }
      if (SIMPLE && a.weak) {  // weak form: the lift of f* alone (semidisc.cpp:505,548)
#pragma unroll
        for (int v = 0; v < V; ++v) sf[q * V + v] = sg * fs[v];
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v) sf[q * V + v] = fma(sg, fs[v] - fo[v], -cll * fo[v]);
      }
    }

    // ---- flux-differencing volume terms (every lane: the in-warp pair
    // exchange needs the whole warp; padding lanes are discarded) ------------
    double K[V];
#pragma unroll
    for (int v = 0; v < V; ++v) K[v] = 0.0;
    if constexpr (SIMPLE) {
      simple_volume<DIM, 0>(pr, tid, il, s_J2[cs][0], own, a.weak, K);
      simple_volume<DIM, 1>(pr, tid, il, s_J2[cs][1], own, a.weak, K);
      if constexpr (DIM == 3) simple_volume<DIM, DIM - 1>(pr, tid, il, s_J2[cs][DIM - 1], own, a.weak, K);
    } else {
      volume_terms<DIM, 0>(ph, pr, tid, il, s_J2[cs][0], own, be, s_cf, K);
      volume_terms<DIM, 1>(ph, pr, tid, il, s_J2[cs][1], own, be, s_cf, K);
      if constexpr (DIM == 3)
        volume_terms<DIM, DIM - 1>(ph, pr, tid, il, s_J2[cs][DIM - 1], own, be, s_cf, K, zf);
      dist2_pairs<DIM>(ph, pr, pf, tid);
    }
    if (dt_t >= 0) describe(buf ^ 1, dt_t, nx_cell);  // the next group, off the critical path
    __syncthreads();  // surface terms of every face point visible

    if constexpr (!SIMPLE) {
      if constexpr (DIM == 3) zf_gather<DIM>(zf, s_cf, s_ti, tid, s_J2[cs][DIM - 1], K);
      dist2_gather<DIM>(pf, s_cf, s_ti, tid, s_J2[cs], K);
    }
    if (cell >= 0) {
      // gather the node's face contributions (one per direction it ends)
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        const int off = s_ti[(ThreadTab<DIM>::I_FACE + d) * T + tid];
        if (off >= 0) {
          const double* c = sf + off;
#pragma unroll
          for (int v = 0; v < V; ++v) K[v] += c[v];
        }
      }
      if constexpr (VISC) {
        // weak-form divergence of the viscous flux with the central interface
        // flux (add_viscous_1d, semidisc.cpp:341-394, per direction)
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          const int stride = d == 0 ? 1 : N1;
          const int j = il[d];
          const double jac = 0.5 * s_J2[cs][d];
#pragma unroll
          for (int k = 0; k < N1; ++k) {
            const double coef = jac * c_Dw[k * N1 + j];
            const double* gk = vg + d * V * T + tid + (k - j) * stride;
#pragma unroll
            for (int v = 0; v < V; ++v) K[v] -= coef * gk[v * T];
          }
          if (j == 0 || j == N1 - 1) {
            const int e = j == 0 ? 0 : 1;
            const int pt = d == 0 ? il[1] : il[0];
            const double* gn = vn + (cs * 2 * DIM + 2 * d + e) * FP + pt;
            const double* go = vg + d * V * T + tid;
            const double coef = s_lift[cs][d];
#pragma unroll
            for (int v = 0; v < V; ++v) {
              const double gs = 0.5 * (e ? go[v * T] + gn[v * CPB * NFP]
                                         : gn[v * CPB * NFP] + go[v * T]);
              K[v] += (e ? coef : -coef) * gs;
            }
          }
        }
      }

      // ---- epilogue: entropy products, K and d stores (coalesced) -------------
      if (a.want_dh || a.want_h) {
        // log(p / rho^gamma) = -(log beta + (gamma - 1) log rho)
        const double s_therm = -(flog(be) + ph.gm1 * flog(own.rho));
        // node_measure (semidisc.cpp:67) with the cell factor from the descriptor
        const double om = DIM == 2 ? s_meas[cs] * c_w[il[0]] * c_w[il[1]]
                                   : s_meas[cs] * c_w[il[0]] * c_w[il[1]] * c_w[il[2]];
        if (a.want_dh) {
          double v2 = 0.0, dot = 0.0;
#pragma unroll
          for (int i = 0; i < DIM; ++i) {
            v2 = fma(own.v[i], own.v[i], v2);
            dot = fma(ph.gm1 * be * own.v[i], K[1 + i], dot);
          }
          dot = fma(ph.gamma - s_therm - 0.5 * ph.gm1 * be * v2, K[0], dot);
          dot = fma(-ph.gm1 * be, K[DIM + 1], dot);
          acc_dh = dd_add_prod(acc_dh, om, dot);
        }
        if (a.want_h) acc_h = dd_add_prod(acc_h, om, -own.rho * s_therm);
      }
      const size_t gi = static_cast<size_t>(cell) * NPC * V + l;  // variable v at gi + v NPC
      if (a.write_k)
#pragma unroll
        for (int v = 0; v < V; ++v) a.Kout[gi + v * NPC] = K[v];
      if (a.write_next) {
        // U_{i+1} = U + dt (a_{i+1,1} K1 + a_{i+1,i} K_i) with the cell's row
        // (stepper.cpp:60-72, one stage ahead); at stage 0, K1 = K_0 = K
        // (all loads of a batch before its stores: the compiler cannot tell
        // that Usn / d do not alias U / K1 and would serialise the pairs)
        const int lev = s_lev[cs];
        const double an = dt * a.a1n[lev], pn = dt * a.apn[lev];
        double x[V], y[V];
#pragma unroll
        for (int v = 0; v < V; ++v) x[v] = __ldg(a.U + gi + v * NPC);
        if (!a.form) {
#pragma unroll
          for (int v = 0; v < V; ++v) a.Usn[gi + v * NPC] = fma(an, K[v], x[v]);
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v) y[v] = __ldg(a.K1 + gi + v * NPC);
#pragma unroll
          for (int v = 0; v < V; ++v) a.Usn[gi + v * NPC] = x[v] + fma(an, y[v], pn * K[v]);
        }
      }
      if (a.d_mode) {
        double dn5[V];
#pragma unroll
        for (int v = 0; v < V; ++v)
          dn5[v] = a.d_mode == 1 ? a.b * K[v] : fma(a.b, K[v], a.d[gi + v * NPC]);
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const double dn = dn5[v];
          a.d[gi + v * NPC] = dn;
          if (a.want_dmax) {
            const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(dn)) &
                                         0x7fffffffffffffffULL;
            dmax_bits = b > dmax_bits ? b : dmax_bits;
          }
        }
      }
    }
    __syncthreads();  // smem of this group consumed; next descriptors visible
  }

  // ---- grid epilogue --------------------------------------------------------
  if (a.want_dmax) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o = __shfl_down_sync(0xffffffffu, dmax_bits, off);
      dmax_bits = o > dmax_bits ? o : dmax_bits;
    }
    if ((tid & 31) == 0) {
      if (dmax_bits >= 0x7ff0000000000000ULL) st->d_nonfinite = 1;
      else atomicMax(&st->dmax_bits, dmax_bits);
    }
  }
  dd v[2] = {acc_dh, acc_h}, tot[2];
  if (a.want_dh || a.want_h) block_reduce_dd<2>(v, s_red);
  if (grid_reduce_dd<2>(v, partials, counter, s_red, tot) && tid == 0) {
    if (a.want_dh) {
      const dd inc = dd_mul_d(tot[0], dt * a.b);
      const dd cur = {st->dh_hi, st->dh_lo};
      const dd nw = dd_add(cur, inc);
      st->dh_hi = nw.hi;
      st->dh_lo = nw.lo;
    }
    if (a.want_h) {
      st->h_hi = tot[1].hi;
      st->h_lo = tot[1].lo;
    }
    if (st->bad_code != kNoBad) st->aborted = 1;
  }
}

// Domain decomposition: the formed stage traces a neighbouring rank reads
// (stepper.cpp:60-72 restricted to those face nodes).  send: [entry] =
// (local cell, face) in peer order; out: [entry][FP][V], points in the
// (t1 + 4 t2) order of the face (line_base), so the receiver indexes them as
// its own face points.
template <int DIM>
__global__ void __launch_bounds__(256)
    pack_traces_kernel(StageArgs a, MeshDev m, StepState* st, const int* send, int nsend,
                       double* out) {
  using G = StageGeo<DIM>;
  constexpr int V = G::V, NPC = G::NPC, FP = G::FP;
  if (st->aborted || st->finished) return;
  const double dt = st->dt;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nsend * FP; q += gridDim.x * blockDim.x) {
    const int e = q / FP, pt = q % FP;
    const int cell = send[2 * e], f = send[2 * e + 1];
    const int d = f >> 1, side = f & 1;
    const int node = line_base<DIM>(d, pt % N1, pt / N1) + (side ? N1 - 1 : 0) * line_stride(d);
    const size_t gi = static_cast<size_t>(cell) * NPC * V + node;  // device layout (sidx)
    double u[V];
    const int lev = m.level[cell];
    if (!a.form) {
#pragma unroll
      for (int v = 0; v < V; ++v) u[v] = __ldg(a.U + gi + v * NPC);
    } else if (a.formed[lev]) {
#pragma unroll
      for (int v = 0; v < V; ++v) u[v] = __ldg(a.Us + gi + v * NPC);
    } else {
      const double b1 = dt * a.a1[lev];
#pragma unroll
      for (int v = 0; v < V; ++v)
        u[v] = fma(b1, __ldg(a.K1 + gi + v * NPC), __ldg(a.U + gi + v * NPC));
    }
    double* o = out + (static_cast<size_t>(e) * FP + pt) * V;
#pragma unroll
    for (int v = 0; v < V; ++v) o[v] = u[v];
  }
}

}  // namespace dev
}  // namespace perrk
