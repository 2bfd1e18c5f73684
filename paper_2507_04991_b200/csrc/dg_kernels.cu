// sm_100a FP64 kernels of the P-ERRK / EC-DGSEM hot path.
//
//   stage_kernel   one P-ERK stage over the stage's active cell list: forms
//                  the stage state on the fly (stepper.cpp:60-72) for the cell
//                  and the face traces of its neighbours, then evaluates the
//                  flux-differencing volume term (semidisc.cpp:446-485) and
//                  the surface flux + LGL lift (semidisc.cpp:489-556) in one
//                  pass, and fuses the b-stage epilogue (d += b K, dH += dt b
//                  <w,K>, stepper.cpp:52-55,89-92) and the admissibility scan
//                  (semidisc.cpp:596-607).
//   relax_pass     one Newton iteration of solve_relaxation (relax.cpp:79-104
//                  or the accurate H1 variant): r and r' at the same gamma in
//                  one fused pass, the scalar update done by the last block.
//   update_kernel  U += gamma dt d (stepper.cpp:107-113) fused with the next
//                  step's CFL speed (mesh.cpp:97-129), the StepRecord H and
//                  invariants (stepper.cpp:179-180) and the clock advance.
//   begin_step     compute_dt (stepper.cpp:116-127) and per-step resets.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdio>

#include "dg_device.cuh"
#include "dg_launch.hpp"

namespace perrk {
namespace dev {

__constant__ double c_D[N1 * N1];  // SBP derivative matrix, row-major D[l][m]
__constant__ double c_w[N1];       // LGL weights
__constant__ double c_Dw[N1 * N1];  // weak-form transpose coefficients D[k][j] w[k] / w[j]

constexpr long long kNoBad = LLONG_MAX;

// select from a 3-array with a runtime index without spilling the array
template <class T>
__device__ __forceinline__ T pick3(const T (&a)[3], int i) {
  return i == 0 ? a[0] : (i == 1 ? a[1] : a[2]);
}

__device__ __forceinline__ void cell_coords(const MeshDev& m, int cell, int& ci, int& cj, int& ck) {
  if (m.gid) cell = m.gid[cell];  // a local cell of a decomposed context
  ci = cell % m.nc[0];
  const int r = cell / m.nc[0];
  cj = r % m.nc[1];
  ck = r / m.nc[1];
}

// local node index of the point (t1, t2) of a line/face family of
// direction dir at position idx along dir
template <int DIM>
__device__ __forceinline__ int line_node(int dir, int idx, int t1, int t2) {
  if (dir == 0) return idx + N1 * (t1 + N1 * t2);
  if (dir == 1) return t1 + N1 * (idx + N1 * t2);
  return t1 + N1 * (t2 + N1 * idx);
}

template <int DIM>
__device__ __forceinline__ double node_measure(const MeshDev& m, int ci, int cj, int ck, int l) {
  const int ix = l % N1, iy = (l / N1) % N1, iz = l / (N1 * N1);
  if (DIM == 2) return 0.25 * m.h[0][ci] * m.h[1][cj] * c_w[ix] * c_w[iy];
  return 0.125 * m.h[0][ci] * m.h[1][cj] * m.h[2][ck] * c_w[ix] * c_w[iy] * c_w[iz];
}

// the same measure from the cell's static record (host.cpp build_cell_records:
// meas = (h_x/2)(h_y/2)(h_z/2), bitwise 0.125 h_x h_y h_z), no index division
template <int DIM>
__device__ __forceinline__ double node_measure_rec(const MeshDev& m, int cell, int l) {
  const int ix = l % N1, iy = (l / N1) % N1, iz = l / (N1 * N1);
  const double meas = __ldg(&m.rec[cell].meas);
  if (DIM == 2) return meas * c_w[ix] * c_w[iy];
  return meas * c_w[ix] * c_w[iy] * c_w[iz];
}

__device__ __forceinline__ void report_bad(StepState* st, int stage, long long ncells, long long cell) {
  atomicMin(&st->bad_code, static_cast<long long>(stage) * ncells + cell);
}

}  // namespace dev
}  // namespace perrk

#include "dg_stage.cuh"
#include "dg_stage3w.cuh"
#include "dg_stage2w.cuh"
#include "dg_visc.cuh"
#include "dg_advection.cuh"
#include "dg_krylov.cuh"

namespace perrk {
namespace dev {

// ---------------------------------------------------------------------------
// per-step control
// ---------------------------------------------------------------------------

__global__ void begin_step_kernel(StepState* st) {
  if (st->aborted || st->finished) return;
  if (st->run_mode && !(st->t < st->tf - st->t_eps)) {
    st->finished = 1;
    return;
  }
  double dt;
  if (st->dt_mode == 0) {
    dt = st->dt_given;
  } else if (st->dt_mode == 1) {
    dt = fmin(st->dt_or_cfl, st->tf - st->t);
  } else {
    const double numax = 4.0 * __longlong_as_double(static_cast<long long>(st->numax_bits));
    if (!(numax > 0.0)) {
      st->error = 2;  // "vanishing characteristic speed"
      st->finished = 1;
      return;
    }
    // CflRamp::operator() (stepper.cpp:13-15) at t - t0
    const double cfl = st->t_ramp > 0.0
                           ? fmin(st->dt_or_cfl, st->cfl0 + (st->dt_or_cfl - st->cfl0) *
                                                                (st->t - st->t0) / st->t_ramp)
                           : st->dt_or_cfl;
    dt = cfl / numax;
    st->numax_bits = 0ull;  // re-accumulated by this step's update kernel
  }
  st->dt = dt;
  st->dh_hi = st->dh_lo = 0.0;
  st->dmax_bits = 0ull;
  st->d_nonfinite = 0;
  st->gamma = st->method == 1 ? st->bracket_min
                              : (st->seed_from_previous ? st->gamma_seed : 1.0);
  st->residual = 0.0;
  st->pending_step = st->prev_step = 0.0;
  st->iters = 0;
  st->pass = 0;
  st->fell_back = 0;
  st->relax_done = st->relax_enabled ? 0 : 1;
  st->spec_done = 0;
  st->numax_spec_bits = 0ull;
}

// ---------------------------------------------------------------------------
// relaxation: one Newton iteration per launch
// ---------------------------------------------------------------------------

__device__ void relax_fallback(StepState* st, int iters, double res) {
  st->gamma = 1.0;
  st->iters = iters;
  st->residual = res;
  st->fell_back = 1;
  st->relax_done = 1;
}

// Scalar Newton logic, executed by one thread after the fused reduction of
// A = sum w Ds (accurate) or sum w s(T) (reference) and B = sum w <w(T), d>.
__device__ void relax_newton_update(StepState* st, dd A, dd B) {
  const double dt = st->dt;
  const dd dh = {st->dh_hi, st->dh_lo};
  const double gamma = st->gamma;
  double r, dr;
  if (st->numerics == 1) {
    // r = offset + sum w Ds - gamma dH ; r' = dt <w(T),d> - dH
    dd rr = A;
    if (!isnan(st->h_ref))  // anchored: + (H(U_n) - h_ref)
      rr = dd_add(rr, dd_add(dd{st->h_hi, st->h_lo}, dd{-st->h_ref, 0.0}));
    rr = dd_add(rr, dd_mul_d(dh, -gamma));
    r = rr.hi + rr.lo;
    const dd d2 = dd_add(dd_mul_d(B, dt), dd{-dh.hi, -dh.lo});
    dr = d2.hi + d2.lo;
    const int it = st->pass + 1;
    st->iters = it;
    st->residual = r;
    if (dr == 0.0 || !isfinite(dr) || !isfinite(r)) return relax_fallback(st, it, r);
    const double step = r / dr;
    // after the first step (always take >= 1), a
    // correction below 1e-13 gamma is under the residual's noise floor: the
    // current iterate is the root and is kept, not moved by the noise (which
    // also lets relax_spec_kernel's update at this gamma stand)
    if (it >= 2 && fabs(step) <= 1e-13 * gamma && gamma > 0.0) {
      st->relax_done = 1;
      return;
    }
    const double g2 = gamma - step;
    if (!isfinite(g2) || !(g2 > 0.0)) return relax_fallback(st, it, r);
    st->gamma = g2;
    if (fabs(step) <= 1e-13 * g2 ||
        (it >= 2 && fabs(step) < 1e-10 * g2 && fabs(step) > 0.5 * fabs(st->prev_step))) {
      st->relax_done = 1;
      return;
    }
    if (it >= st->max_iter) {
      // out of iterations: a last correction inside the noise band (1e-10
      // gamma) is converged; anything larger has not, and falls back to
      // gamma = 1 as the reference does (relax.cpp:104)
      if (fabs(step) <= 1e-10 * g2)
        st->relax_done = 1;
      else
        relax_fallback(st, it, r);
      return;
    }
    st->prev_step = step;
    st->pass = it;
    return;
  }
  // reference numerics: relax.cpp:79-104 verbatim on the fused pass values
  const double H = A.hi + A.lo;
  const double dhv = dh.hi + dh.lo;
  const double h_ref = isnan(st->h_ref) ? st->h_hi + st->h_lo : st->h_ref;
  r = H - h_ref - gamma * dhv;
  dr = dt * (B.hi + B.lo) - dhv;
  const int pass = st->pass;
  if (pass > 0) {
    if (fabs(r) <= st->residual_tol || fabs(st->pending_step) <= st->step_tol) {
      st->residual = r;
      st->iters = pass;
      st->relax_done = 1;
      if (!(gamma > 0.0)) relax_fallback(st, pass, r);
      return;
    }
    if (pass >= st->max_iter) return relax_fallback(st, st->max_iter, r);
  } else if (fabs(r) <= st->residual_tol) {
    st->residual = r;
    st->iters = 0;
    st->relax_done = 1;
    if (!(gamma > 0.0)) relax_fallback(st, 0, r);
    return;
  }
  const int it = pass + 1;
  if (dr == 0.0 || !isfinite(dr)) return relax_fallback(st, it, r);
  const double step = r / dr;
  const double g2 = gamma - step;
  if (!isfinite(g2)) return relax_fallback(st, it, r);
  st->gamma = g2;
  st->pending_step = step;
  st->iters = it;
  st->residual = r;
  st->pass = it;
}

// Bisection (relax.cpp:105-127) and secant (relax.cpp:128-148) on the device:
// each launch evaluates the residual at st->gamma; this single-thread step
// consumes it and sets the next evaluation point, or finishes.
__device__ double relax_residual(const StepState* st, dd A) {
  const dd dh = {st->dh_hi, st->dh_lo};
  const double gamma = st->gamma;
  if (st->numerics == 1) {
    dd rr = A;
    if (!isnan(st->h_ref)) rr = dd_add(rr, dd_add(dd{st->h_hi, st->h_lo}, dd{-st->h_ref, 0.0}));
    rr = dd_add(rr, dd_mul_d(dh, -gamma));
    return rr.hi + rr.lo;
  }
  const double h_ref = isnan(st->h_ref) ? st->h_hi + st->h_lo : st->h_ref;
  return (A.hi + A.lo) - h_ref - gamma * (dh.hi + dh.lo);
}

__device__ void relax_done_at(StepState* st, double g, int iters, double r) {
  st->gamma = g;
  st->iters = iters;
  st->residual = r;
  st->relax_done = 1;
  if (!(g > 0.0)) relax_fallback(st, iters, r);
}

__device__ void relax_update(StepState* st, dd A, dd B) {
  if (st->method == 0) return relax_newton_update(st, A, B);
  const double r = relax_residual(st, A);
  const int pass = st->pass;
  st->pass = pass + 1;
  if (st->method == 1) {  // bisection
    if (pass == 0) {  // r(lo)
      st->lo = st->bracket_min;
      st->hi = st->bracket_max;
      st->rlo = r;
      st->gamma = st->hi;
      return;
    }
    if (pass == 1) {  // r(hi): a sign change is required
      if (signbit(st->rlo) == signbit(r)) return relax_fallback(st, 0, st->rlo);
      st->gamma = 0.5 * (st->lo + st->hi);
      return;
    }
    const int it = pass - 1;  // r(mid), iteration it
    const double mid = st->gamma;
    st->iters = it;
    if (fabs(r) <= st->residual_tol || (st->hi - st->lo) <= st->step_tol)
      return relax_done_at(st, mid, it, r);
    if (signbit(r) == signbit(st->rlo)) {
      st->lo = mid;
      st->rlo = r;
    } else {
      st->hi = mid;
    }
    if (it >= st->max_iter) {  // the reference re-tests with the halved bracket
      if ((st->hi - st->lo) <= st->step_tol) return relax_done_at(st, mid, it, r);
      return relax_fallback(st, it, r);
    }
    st->gamma = 0.5 * (st->lo + st->hi);
    return;
  }
  // secant
  if (pass == 0) {  // r(g0)
    st->g0 = st->gamma;
    st->r0 = r;
    st->gamma = st->g0 - 1e-6;
    return;
  }
  if (pass >= 2) {  // r(g1) of iteration pass-1: converged?
    const int it = pass - 1;
    if (fabs(r) <= st->residual_tol || fabs(st->gamma - st->g0) <= st->step_tol)
      return relax_done_at(st, st->gamma, it, r);
    if (it >= st->max_iter) return relax_fallback(st, st->max_iter, r);
  }
  // next secant point from (g0, r0), (g1, r1)
  const int it = pass;  // iteration about to be taken
  const double g1 = st->gamma, r1 = r;
  if (r1 == st->r0) return relax_fallback(st, it, r1);
  const double g2 = g1 - r1 * (g1 - st->g0) / (r1 - st->r0);
  if (!isfinite(g2)) return relax_fallback(st, it, r1);
  st->g0 = g1;
  st->r0 = r1;
  st->gamma = g2;
  st->iters = it;
}

#ifndef PERRK_RELAX_DIRECT
// 1: the relaxation / update kernels read U and d with direct coalesced loads
// (one 256-byte warp access per variable in the device layout); 0: the
// blocks are staged through shared memory by cp.async first
#define PERRK_RELAX_DIRECT 1
#endif
#ifndef PERRK_RELAX_MINB
#define PERRK_RELAX_MINB 3  // resident 256-thread blocks per SM the relaxation kernels are compiled for
#endif
#ifndef PERRK_RELAX_PF
// 1 (direct loads): the next block's U and d are loaded into registers before
// the current block's terms are evaluated (twice the bytes in flight per warp;
// the per-lane order of the sums, and so every bit of the result, is unchanged).
// Measured (profiles/r02_ab.txt, pass 11): slower, 318 -> 387 us (pass) and
// 551 -> 710 us (fused pass 2) at 3 blocks per SM (spills), 376 / 620 us at 2:
// these kernels run the FP64 pipe at 55% (two logarithms per node), they are
// not waiting for memory
#define PERRK_RELAX_PF 0
#endif

// One warp's 32-node block k of two state arrays (U and d) into shared
// memory by coalesced 16-byte cp.async, one commit group per call (empty past
// the end).  In the device layout (sidx) a block's variable v is 32 (3D) or
// two runs of 16 (2D) contiguous doubles; the staging area is [v][32], read
// by lane with conflict-free 8-byte loads (s[v * 32 + lane]).
template <int DIM>
__device__ __forceinline__ void stage_pair(const double* A, const double* B, long long nnodes,
                                           long long nblk, long long k, double* sa, double* sb,
                                           int lane) {
  constexpr int V = DIM + 2;
  if (k < nblk) {
    const long long n0 = k * 32;
    // this lane's piece p (nodes n0 + 2p, n0 + 2p + 1: one cell, NPC is even)
    // of variables v = (lane >> 4) + 2 r
    const int p = lane & 15;
    const long long n = n0 + 2 * p;
    if (n < nnodes) {
      const long long g = sidx_n<DIM>(n, lane >> 4);  // + 2 r NPC per round
#pragma unroll
      for (int r = 0; r < (V + 1) / 2; ++r) {
        const int v = (lane >> 4) + 2 * r;
        if (v < V) {
          cp_async16(sa + v * 32 + 2 * p, A + g + 2 * r * Geo<DIM>::NPC);
          cp_async16(sb + v * 32 + 2 * p, B + g + 2 * r * Geo<DIM>::NPC);
        }
      }
    }
  }
  cp_async_commit();
}

// node n's U and d: from the warp's staged block, or straight from global
// memory (PERRK_RELAX_DIRECT: coalesced in the device layout)
template <int DIM>
__device__ __forceinline__ void load_pair(const double* __restrict__ A,
                                          const double* __restrict__ B, long long n,
                                          const double* sa, const double* sb, int lane,
                                          double* ua, double* ub) {
  constexpr int V = DIM + 2;
  if (PERRK_RELAX_DIRECT) {
    const long long g = sidx_n<DIM>(n, 0);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      ua[v] = __ldg(A + g + v * Geo<DIM>::NPC);
      ub[v] = __ldg(B + g + v * Geo<DIM>::NPC);
    }
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      ua[v] = sa[32 * v + lane];
      ub[v] = sb[32 * v + lane];
    }
  }
}

// One relaxation pass.  Each warp walks blocks of 32 consecutive nodes: the
// block's U and d (32 V doubles each, contiguous) arrive by coalesced 16-byte
// cp.async into a double-buffered per-warp staging area one block ahead, and
// each lane reads its node with 8-byte loads (40- / 32-byte stride: conflict
// free).  The previous layout (a thread's own node straight from global
// memory, stride V doubles) cost 5x the L1 wavefronts per byte.
template <int DIM>
__global__ void __launch_bounds__(256, PERRK_RELAX_MINB)
    relax_pass_kernel(const double* __restrict__ U, const double* __restrict__ d, MeshDev m,
                      Phys ph, StepState* st, double* partials, unsigned* counter, long long nnodes) {
  constexpr int V = DIM + 2, NPC = Geo<DIM>::NPC, BLK = 32 * V;  // doubles per block and array
  __shared__ double s_red[2 * 2 * 8];
  __shared__ __align__(16) double s_stage[8][2][2][BLK];  // [warp][buffer][U, d][block]
  if (st->aborted || st->finished || st->relax_done) return;
  const double dmax = __longlong_as_double(static_cast<long long>(st->dmax_bits));
  if (st->d_nonfinite || dmax == 0.0) {
    // relax.cpp:56-63 — handled once, by block 0
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (st->d_nonfinite) {
        st->error = 1;
        st->aborted = 1;  // stop the step; the host reports the error
      }
      st->gamma = 1.0;
      st->iters = 0;
      st->residual = 0.0;
      st->relax_done = 1;
    }
    return;
  }
  const double gamma = st->gamma;
  const double gdt = gamma * st->dt;
  const int numerics = st->numerics;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long nblk = (nnodes + 31) / 32;
  const long long stride = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  auto stage = [&](long long k, int b) {
    if (!PERRK_RELAX_DIRECT)
      stage_pair<DIM>(U, d, nnodes, nblk, k, s_stage[wib][b][0], s_stage[wib][b][1], lane);
  };
  ksum A = ks_zero(), B = ks_zero();
  long long k = blockIdx.x * static_cast<long long>(blockDim.x >> 5) + wib;
  int b = 0;
  stage(k, 0);
  constexpr bool kPf = PERRK_RELAX_DIRECT && PERRK_RELAX_PF;
  double un[V], dn[V];
#pragma unroll
  for (int v = 0; v < V; ++v) un[v] = dn[v] = 0.0;
  auto prefetch = [&](long long kk) {
    const long long nn = kk * 32 + lane;
    if (kPf && kk < nblk && nn < nnodes) load_pair<DIM>(U, d, nn, nullptr, nullptr, lane, un, dn);
  };
  prefetch(k);
  for (; k < nblk; k += stride, b ^= 1) {
    stage(k + stride, b ^ 1);
    if (!PERRK_RELAX_DIRECT) cp_async_wait<1>();
    __syncwarp();
    const long long n = k * 32 + lane;
    double u[V], dv[V];
    if (kPf) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        u[v] = un[v];
        dv[v] = dn[v];
      }
      prefetch(k + stride);
    }
    if (n < nnodes) {
      const int cell = static_cast<int>(n / NPC), l = static_cast<int>(n % NPC);
      const double om = node_measure_rec<DIM>(m, cell, l);
      if (!kPf) load_pair<DIM>(U, d, n, s_stage[wib][b][0], s_stage[wib][b][1], lane, u, dv);
      if (numerics == 1) {
        double du[V], ra, rb;
        // rounded products (never contracted into later sums): the same bits
        // in relax_spec_kernel
#pragma unroll
        for (int v = 0; v < V; ++v) du[v] = __dmul_rn(gdt, dv[v]);
        relax_terms<DIM>(ph, u, du, dv, trial_state<DIM>(ph, u, du), ra, rb);
        ks_add_prod(A, om, ra);
        ks_add_prod(B, om, rb);
      } else {  // the reference's residual / derivative on the rounded trial state
        double T[V];
#pragma unroll
        for (int v = 0; v < V; ++v) T[v] = u[v] + gdt * dv[v];
        ks_add_prod(A, om, entropy<DIM>(ph, T));
        ks_add_prod(B, om, entropy_dot<DIM>(ph, T, dv));
      }
    }
    __syncwarp();  // buffer b is restaged two blocks on
  }
  cp_async_wait<0>();
  dd v[2] = {ks_dd(A), ks_dd(B)}, tot[2];
  block_reduce_dd<2>(v, s_red);
  if (grid_reduce_dd<2>(v, partials, counter, s_red, tot) && threadIdx.x == 0) {
    if (st->slab) {  // gathered over ranks, then combine_kernel(COMBINE_RELAX)
      st->red_local[R_A_HI] = tot[0].hi;
      st->red_local[R_A_LO] = tot[0].lo;
      st->red_local[R_B_HI] = tot[1].hi;
      st->red_local[R_B_LO] = tot[1].lo;
    } else {
      relax_update(st, tot[0], tot[1]);
    }
  }
}

// ---------------------------------------------------------------------------
// final update, CFL speed, step record
// ---------------------------------------------------------------------------

// the update's per-node terms of the new state u: the next step's CFL speed
// (mesh.cpp:97-129 takes |v_dir| + c per direction; 1/h_dir = jac_dir / 2
// exactly, one pressure / sound speed per node) and the StepRecord H and
// invariants (stepper.cpp:179-180)
// per-thread accumulators kept in shared memory, thread-interleaved (no bank
// conflicts), to hold relax_spec_kernel's registers for three blocks per SM
struct KsShared {
  ksum* base;  // &arr[0][threadIdx.x] of a [rows][blockDim] array
  int stride;  // blockDim.x
  __device__ __forceinline__ ksum& operator[](int r) const { return base[r * stride]; }
};

// max_dir lambda_dir / h_dir of one node (mesh.cpp:97-129 divided by k+1):
// the ONE expression of the CFL speed, used by the update kernels (the next
// step's speed) and numax_kernel (the first step's), so a run split over
// several perrk_advance calls takes the same dt as one call
template <int DIM>
__device__ __forceinline__ double node_speed_over_h(const MeshDev& m, const Phys& ph,
                                                    const double* u, int cell) {
  const double ir = frcp(u[0]);
  double m2 = 0.0;
#pragma unroll
  for (int dir = 0; dir < DIM; ++dir) m2 = fma(u[1 + dir], u[1 + dir], m2);
  const double p = ph.gm1 * (u[DIM + 1] - 0.5 * m2 * ir);
  const double c = fsqrt(ph.gamma * p * ir);
  double best = 0.0;
#pragma unroll
  for (int dir = 0; dir < DIM; ++dir)
    best = fmax(best, (fabs(u[1 + dir]) * ir + c) * (0.25 * __ldg(&m.rec[cell].J2[dir])));
  return best;
}

template <int DIM, class Acc>
__device__ __forceinline__ void update_node_terms(const MeshDev& m, const Phys& ph, const double* u,
                                                  long long n, int want_nu, int want_record,
                                                  double s_new, double& numax, Acc acc) {
  constexpr int V = DIM + 2, NPC = Geo<DIM>::NPC;
  const int cell = static_cast<int>(n / NPC), l = static_cast<int>(n % NPC);
  if (want_nu) numax = fmax(numax, node_speed_over_h<DIM>(m, ph, u, cell));
  if (want_record) {
    const double om = node_measure_rec<DIM>(m, cell, l);
    ks_add_prod(acc[0], om, s_new);
#pragma unroll
    for (int v = 0; v < V; ++v) ks_add_prod(acc[1 + v], om, u[v]);
  }
}

// StepRecord entropy of the new state u + du, s = -rho log(p / rho^gamma)
// (physics.cpp:130-132), from the trial state's logarithms
__device__ __forceinline__ double trial_entropy(const Phys& ph, const Trial& t) {
  return -t.rho_t * (t.lp_t - ph.gamma * t.lr_t);
}

// the update's last-block step: clock advance (stepper.cpp:107-113), the
// StepRecord row, the next gamma seed
__device__ void finish_step(StepState* st, double gamma, const dd* tot, int V, int want_record,
                            double* records) {
  const double dt = st->dt;
  if (st->relax_enabled && !st->idt)
    st->t += gamma * dt;
  else
    st->t += dt;
  if (want_record && records) {
    double* row = records + static_cast<size_t>(st->steps_taken) * REC_COLS;
    row[0] = st->t;
    row[1] = dt;
    row[2] = gamma;
    row[3] = st->iters;
    row[4] = st->fell_back;
    row[5] = tot[0].hi + tot[0].lo;
    for (int v = 0; v < V; ++v) row[6 + v] = tot[1 + v].hi + tot[1 + v].lo;
    row[11] = st->dh_hi + st->dh_lo;
  }
  st->gamma_seed = st->fell_back ? 1.0 : gamma;
  st->steps_taken += 1;
}

// U_out = U_in + gamma dt d (in place when U_out == U_in; out of place after
// a relax_spec_kernel, which has already done it when its speculation held).
// Same node walk as the relaxation passes (warp blocks of 32 nodes staged by
// coalesced cp.async, launched on relax_pass_kernel's grid), so the StepRecord
// sums come out bitwise the same as relax_spec_kernel's.
template <int DIM>
__global__ void __launch_bounds__(256, 3)
    update_kernel(double* Uout, const double* Uin, const double* __restrict__ d, MeshDev m,
                  Phys ph, StepState* st, double* partials, unsigned* counter, long long nnodes,
                  int want_nu, int want_record, double* records) {
  constexpr int V = DIM + 2, BLK = 32 * V;
  __shared__ double s_red[2 * 6 * 8];
  __shared__ __align__(16) double s_stage[8][2][2][BLK];  // [warp][buffer][U, d][block]
  if (st->aborted || st->finished || st->spec_done) return;
  const double gamma = st->relax_enabled ? st->gamma : st->gamma_override;
  const double scale = gamma * st->dt;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long nblk = (nnodes + 31) / 32;
  const long long stride = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  double numax = 0.0;
  ksum acc[6];
#pragma unroll
  for (int r = 0; r < 6; ++r) acc[r] = ks_zero();
  long long k = blockIdx.x * static_cast<long long>(blockDim.x >> 5) + wib;
  int b = 0;
  if (!PERRK_RELAX_DIRECT)
    stage_pair<DIM>(Uin, d, nnodes, nblk, k, s_stage[wib][0][0], s_stage[wib][0][1], lane);
  for (; k < nblk; k += stride, b ^= 1) {
    if (!PERRK_RELAX_DIRECT) {
      stage_pair<DIM>(Uin, d, nnodes, nblk, k + stride, s_stage[wib][b ^ 1][0],
                      s_stage[wib][b ^ 1][1], lane);
      cp_async_wait<1>();
    }
    __syncwarp();
    const long long n = k * 32 + lane;
    if (n < nnodes) {
      double u0[V], u[V], du[V], dv[V];
      const long long gb = sidx_n<DIM>(n, 0);
      load_pair<DIM>(Uin, d, n, s_stage[wib][b][0], s_stage[wib][b][1], lane, u0, dv);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        u[v] = fma(scale, dv[v], u0[v]);
        du[v] = __dmul_rn(scale, dv[v]);
        Uout[gb + v * Geo<DIM>::NPC] = u[v];
      }
      const double s_new = want_record ? trial_entropy(ph, trial_state<DIM>(ph, u0, du)) : 0.0;
      if (want_nu || want_record)
        update_node_terms<DIM>(m, ph, u, n, want_nu, want_record, s_new, numax, acc);
    }
    __syncwarp();
  }
  cp_async_wait<0>();
  if (want_nu) {
    numax = warp_max(numax);
    if (lane == 0) atomic_max_pos(&st->numax_bits, numax);
  }
  dd tot[6], accd[6];
#pragma unroll
  for (int r = 0; r < 6; ++r) accd[r] = ks_dd(acc[r]);
  if (want_record) block_reduce_dd<6>(accd, s_red);
  if (grid_reduce_dd<6>(accd, partials, counter, s_red, tot) && threadIdx.x == 0) {
    if (st->slab) {  // gathered over ranks, then combine_kernel(COMBINE_UPDATE)
      for (int r = 0; r < 6; ++r) {
        st->red_local[R_REC0 + 2 * r] = tot[r].hi;
        st->red_local[R_REC0 + 2 * r + 1] = tot[r].lo;
      }
      return;
    }
    finish_step(st, gamma, tot, V, want_record, records);
  }
}

// Newton pass 2 of the accurate relaxation fused with a speculative final
// update.  Pass 1 has produced gamma_1; Newton from the previous step's gamma
// converges in that one step (the next correction is ~1e-22, below half an
// ulp of gamma), so this pass evaluates r(gamma_1), r'(gamma_1) (exactly as
// relax_pass_kernel) and, from the same U and d, the state U + gamma_1 dt d
// into U_out with the update's CFL speed and StepRecord terms (exactly as
// update_kernel).  Its last block runs the Newton logic; if that finishes at
// gamma_1 itself, the speculation is the update and the step is completed
// here (spec_done: update_kernel returns at once).  Otherwise the remaining
// passes and update_kernel proceed from the untouched U_in.  One full read of
// U and d per step is saved (SURVEY.md 7.3 H1 numerics only).
template <int DIM>
__global__ void __launch_bounds__(256, PERRK_RELAX_MINB)
    relax_spec_kernel(const double* __restrict__ U, const double* __restrict__ d,
                      double* __restrict__ Uout, MeshDev m, Phys ph, StepState* st,
                      double* partials, unsigned* counter, long long nnodes, int want_nu,
                      int want_record, double* records) {
  constexpr int V = DIM + 2, BLK = 32 * V;
  __shared__ double s_red[2 * 8 * 8];
  // dynamic shared memory (66.5 KB: over the 48 KB static limit):
  // [warp][buffer][U, d][block] staging, then the six per-thread record sums
  extern __shared__ __align__(16) double spec_smem[];
  auto s_stage = reinterpret_cast<double(*)[2][2][BLK]>(spec_smem);
  if (st->aborted || st->finished || st->relax_done) return;
  const double dmax = __longlong_as_double(static_cast<long long>(st->dmax_bits));
  if (st->d_nonfinite || dmax == 0.0) return;  // handled by pass 1
  const double gamma = st->gamma;
  const double gdt = gamma * st->dt;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long nblk = (nnodes + 31) / 32;
  const long long stride = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  auto stage = [&](long long k, int b) {
    if (!PERRK_RELAX_DIRECT)
      stage_pair<DIM>(U, d, nnodes, nblk, k, s_stage[wib][b][0], s_stage[wib][b][1], lane);
  };
  ksum acc[2];  // A, B in registers; the update's six record sums in shared memory
  acc[0] = acc[1] = ks_zero();
  ksum* s_acc = reinterpret_cast<ksum*>(spec_smem + (PERRK_RELAX_DIRECT ? 0 : 8 * 2 * 2 * BLK));
  const KsShared racc{s_acc + threadIdx.x, static_cast<int>(blockDim.x)};
#pragma unroll
  for (int r = 0; r < 6; ++r) racc[r] = ks_zero();
  double numax = 0.0;
  long long k = blockIdx.x * static_cast<long long>(blockDim.x >> 5) + wib;
  int b = 0;
  stage(k, 0);
  constexpr bool kPf = PERRK_RELAX_DIRECT && PERRK_RELAX_PF;
  double un[V], dn[V];
#pragma unroll
  for (int v = 0; v < V; ++v) un[v] = dn[v] = 0.0;
  auto prefetch = [&](long long kk) {
    const long long nn = kk * 32 + lane;
    if (kPf && kk < nblk && nn < nnodes) load_pair<DIM>(U, d, nn, nullptr, nullptr, lane, un, dn);
  };
  prefetch(k);
  for (; k < nblk; k += stride, b ^= 1) {
    stage(k + stride, b ^ 1);
    if (!PERRK_RELAX_DIRECT) cp_async_wait<1>();
    __syncwarp();
    const long long n = k * 32 + lane;
    double u[V], dv[V];
    if (kPf) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        u[v] = un[v];
        dv[v] = dn[v];
      }
      prefetch(k + stride);
    }
    if (n < nnodes) {
      double du[V], T[V], ra, rb;
      const long long gb = sidx_n<DIM>(n, 0);
      if (!kPf) load_pair<DIM>(U, d, n, s_stage[wib][b][0], s_stage[wib][b][1], lane, u, dv);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        du[v] = __dmul_rn(gdt, dv[v]);
        T[v] = fma(gdt, dv[v], u[v]);  // update_kernel's U + (gamma dt) d
      }
      const double om = node_measure_rec<DIM>(m, static_cast<int>(n / Geo<DIM>::NPC),
                                              static_cast<int>(n % Geo<DIM>::NPC));
      const Trial tr = trial_state<DIM>(ph, u, du);
      relax_terms<DIM>(ph, u, du, dv, tr, ra, rb);
      ks_add_prod(acc[0], om, ra);
      ks_add_prod(acc[1], om, rb);
#pragma unroll
      for (int v = 0; v < V; ++v) Uout[gb + v * Geo<DIM>::NPC] = T[v];
      if (want_nu || want_record)
        update_node_terms<DIM>(m, ph, T, n, want_nu, want_record, trial_entropy(ph, tr), numax,
                               racc);
    }
    __syncwarp();
  }
  cp_async_wait<0>();
  if (want_nu) {
    numax = warp_max(numax);
    if (lane == 0) atomic_max_pos(&st->numax_spec_bits, numax);
  }
  dd tot[8], accd[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) accd[r] = ks_dd(r < 2 ? acc[r] : racc[r - 2]);
  block_reduce_dd<8>(accd, s_red);
  if (grid_reduce_dd<8>(accd, partials, counter, s_red, tot) && threadIdx.x == 0) {
    relax_update(st, tot[0], tot[1]);
    if (st->relax_done && !st->fell_back && st->gamma == gamma) {
      st->spec_done = 1;
      if (want_nu) st->numax_bits = st->numax_spec_bits;
      finish_step(st, gamma, tot + 2, V, want_record, records);
    }
  }
}

// max over nodes of lambda_dir / h_dir (the max of characteristic_speed,
// mesh.cpp:97-129, divided by k+1) into st->numax_bits
template <int DIM>
__global__ void __launch_bounds__(256)
    numax_kernel(const double* __restrict__ U, MeshDev m, Phys ph, StepState* st,
                 long long nnodes) {
  constexpr int V = DIM + 2, NPC = Geo<DIM>::NPC;
  double best = 0.0;
  for (long long n = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; n < nnodes;
       n += static_cast<long long>(gridDim.x) * blockDim.x) {
    double u[V];
#pragma unroll
    for (int v = 0; v < V; ++v) u[v] = __ldg(U + sidx_n<DIM>(n, v));
    best = fmax(best, node_speed_over_h<DIM>(m, ph, u, static_cast<int>(n / NPC)));
  }
  best = warp_max(best);
  if ((threadIdx.x & 31) == 0) atomic_max_pos(&st->numax_bits, best);
}

// per-cell nu = (k+1) max_dir(max_nodes lambda_dir / h_dir), mesh.cpp:97-129
template <int DIM>
__global__ void nu_cell_kernel(const double* __restrict__ U, MeshDev m, Phys ph, double* nu,
                               long long ncells) {
  constexpr int V = DIM + 2, NPC = Geo<DIM>::NPC;
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < ncells;
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    double r[3] = {0.0, 0.0, 0.0};
    for (int l = 0; l < NPC; ++l) {
      double u[V];
#pragma unroll
      for (int v = 0; v < V; ++v) u[v] = U[sidx<DIM>(c, l, v)];
      const double p = pressure<DIM>(ph, u);
#pragma unroll
      for (int dir = 0; dir < DIM; ++dir) r[dir] = fmax(r[dir], max_wave_speed<DIM>(ph, u, p, dir));
    }
    int ci, cj, ck;
    cell_coords(m, static_cast<int>(c), ci, cj, ck);
    const int cc[3] = {ci, cj, ck};
    double best = r[0] / m.h[0][cc[0]];
#pragma unroll
    for (int dir = 1; dir < DIM; ++dir) best = fmax(best, r[dir] / m.h[dir][cc[dir]]);
    nu[c] = 4.0 * best;
  }
}

// ---------------------------------------------------------------------------
// reductions behind the reference's Semidiscretization queries
// ---------------------------------------------------------------------------

// mode 0: H = sum w s(U); 1: sum w <w(U), K>; 2: sum w U_v (V values)
template <int DIM>
__global__ void __launch_bounds__(256)
    quad_kernel(const double* __restrict__ U, const double* __restrict__ K, MeshDev m, Phys ph,
                int mode, double* partials, unsigned* counter, double* out, long long nnodes) {
  constexpr int V = DIM + 2, NPC = Geo<DIM>::NPC;
  __shared__ double s_red[2 * 5 * 8];
  dd acc[5];
#pragma unroll
  for (int r = 0; r < 5; ++r) acc[r] = dd_zero();
  for (long long n = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; n < nnodes;
       n += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int cell = static_cast<int>(n / NPC), l = static_cast<int>(n % NPC);
    int ci, cj, ck;
    cell_coords(m, cell, ci, cj, ck);
    const double om = node_measure<DIM>(m, ci, cj, ck, l);
    double u[V];
#pragma unroll
    for (int v = 0; v < V; ++v) u[v] = __ldg(U + sidx_n<DIM>(n, v));
    if (mode == 0) {
      acc[0] = dd_add_prod(acc[0], om, entropy<DIM>(ph, u));
    } else if (mode == 1) {
      double k[V];
#pragma unroll
      for (int v = 0; v < V; ++v) k[v] = __ldg(K + sidx_n<DIM>(n, v));
      acc[0] = dd_add_prod(acc[0], om, entropy_dot<DIM>(ph, u, k));
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v] = dd_add_prod(acc[v], om, u[v]);
    }
  }
  dd tot[5];
  block_reduce_dd<5>(acc, s_red);
  if (grid_reduce_dd<5>(acc, partials, counter, s_red, tot) && threadIdx.x == 0)
    for (int r = 0; r < 5; ++r) out[r] = tot[r].hi + tot[r].lo;
}

template <int DIM>
__global__ void admissible_kernel(const double* __restrict__ U, Phys ph, int* first_bad,
                                  long long nnodes) {
  constexpr int V = DIM + 2, NPC = Geo<DIM>::NPC;
  for (long long n = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; n < nnodes;
       n += static_cast<long long>(gridDim.x) * blockDim.x) {
    double u[V];
#pragma unroll
    for (int v = 0; v < V; ++v) u[v] = U[sidx_n<DIM>(n, v)];
    if (!admissible<DIM>(ph, u)) atomicMin(first_bad, static_cast<int>(n / NPC));
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

template <int DIM, bool VISC>
static size_t stage_smem() {
  return sizeof(double) *
         (StageGeo<DIM>::SM_TOTAL + StageGeo<DIM>::SM_ZF + StageGeo<DIM>::SM_PF +
          (VISC ? StageGeo<DIM>::SM_VISC : 0));
}

// function attributes are per device: the launch helpers configure each
// kernel once per device ordinal
constexpr int MAX_DEVICES = 64;
static int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev >= 0 && dev < MAX_DEVICES ? dev : 0;
}

template <int DIM, int SURF, bool VISC, bool SIMPLE>
static void configure_stage() {
  static bool configured[MAX_DEVICES] = {};
  const int dev = current_device();
  if (!configured[dev]) {
    cudaFuncSetAttribute(stage_kernel<DIM, SURF, VISC, SIMPLE>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(stage_smem<DIM, VISC>()));
    configured[dev] = true;
  }
}

template <int DIM, int SURF, bool SIMPLE>
static int stage_occ_t() {
  configure_stage<DIM, SURF, false, SIMPLE>();
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, stage_kernel<DIM, SURF, false, SIMPLE>,
                                                StageGeo<DIM>::T, stage_smem<DIM, false>());
  return n;
}

template <int DIM, int SURF, bool VISC, bool SIMPLE>
static cudaError_t launch_stage_t(const StageArgs& a, const MeshDev& m, const Phys& ph,
                                  StepState* st, double* partials, unsigned* counter, int grid,
                                  cudaStream_t s) {
  using G = StageGeo<DIM>;
  configure_stage<DIM, SURF, VISC, SIMPLE>();
  const int groups = (a.n + G::CPB - 1) / G::CPB;
  const int g = groups < grid ? groups : grid;
  if (g <= 0) return cudaSuccess;
  stage_kernel<DIM, SURF, VISC, SIMPLE><<<g, G::T, stage_smem<DIM, VISC>(), s>>>(
      a, m, ph, st, partials, counter);
  return cudaGetLastError();
}

template <int DIM, bool VISC, bool SIMPLE>
static cudaError_t launch_stage_d(int surf, const StageArgs& a, const MeshDev& m, const Phys& ph,
                                  StepState* st, double* partials, unsigned* counter, int grid,
                                  cudaStream_t s) {
  switch (surf) {
    case 0: return launch_stage_t<DIM, 0, VISC, SIMPLE>(a, m, ph, st, partials, counter, grid, s);
    case 2: return launch_stage_t<DIM, 2, VISC, SIMPLE>(a, m, ph, st, partials, counter, grid, s);
    case 3: return launch_stage_t<DIM, 3, VISC, SIMPLE>(a, m, ph, st, partials, counter, grid, s);
    case 4: return launch_stage_t<DIM, 4, VISC, SIMPLE>(a, m, ph, st, partials, counter, grid, s);
    case 5: return launch_stage_t<DIM, 5, VISC, SIMPLE>(a, m, ph, st, partials, counter, grid, s);
  }
  return cudaErrorInvalidValue;
}

// FP64 peak probe: 8 independent DFMA chains per thread (the FP64 pipe's
// latency is hidden by chains x resident warps); one store keeps it live.
__global__ void __launch_bounds__(256) dfma_probe_kernel(double* out, int iters, double a,
                                                         double b) {
  double x[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) x[q] = threadIdx.x * 1e-3 + q;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = fma(x[q], a, b);
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += x[q];
  if (s == 12345.678) out[0] = s;
}

// ---------------------------------------------------------------------------
// slab decomposition: reduction points (stash local -> gather -> combine)
// ---------------------------------------------------------------------------
enum { COMBINE_STAGES = 0, COMBINE_RELAX = 1, COMBINE_UPDATE = 2, COMBINE_NUMAX = 3 };

// copy this rank's partials kept in StepState fields into red_local
__global__ void stash_kernel(StepState* st, int mode) {
  double* r = st->red_local;
  if (mode == COMBINE_STAGES) {
    r[R_DH_HI] = st->dh_hi;
    r[R_DH_LO] = st->dh_lo;
    r[R_H_HI] = st->h_hi;
    r[R_H_LO] = st->h_lo;
    r[R_DMAX] = __longlong_as_double(static_cast<long long>(st->dmax_bits));
    r[R_DBAD] = st->d_nonfinite;
    r[R_BAD] = static_cast<double>(st->bad_code == kNoBad ? -1 : st->bad_code);
  }
  r[R_NUMAX] = __longlong_as_double(static_cast<long long>(st->numax_bits));
}

// all[nranks][NRED]: sums in rank order (double-double), maxima, minima;
// then the scalar logic that the single-GPU kernels run in their last block
__global__ void combine_kernel(StepState* st, const double* all, int nranks, int mode) {
  auto sum = [&](int hi, int lo) {
    dd acc = dd_zero();
    for (int q = 0; q < nranks; ++q) acc = dd_add(acc, dd{all[q * NRED + hi], all[q * NRED + lo]});
    return acc;
  };
  auto vmax = [&](int k) {
    double v = all[k];
    for (int q = 1; q < nranks; ++q) v = fmax(v, all[q * NRED + k]);
    return v;
  };
  if (mode == COMBINE_NUMAX || mode == COMBINE_UPDATE) {
    const double nu = vmax(R_NUMAX);
    st->numax_bits = static_cast<unsigned long long>(__double_as_longlong(nu));
  }
  if (mode == COMBINE_STAGES) {
    const dd dh = sum(R_DH_HI, R_DH_LO), h = sum(R_H_HI, R_H_LO);
    st->dh_hi = dh.hi;
    st->dh_lo = dh.lo;
    st->h_hi = h.hi;
    st->h_lo = h.lo;
    st->dmax_bits = static_cast<unsigned long long>(__double_as_longlong(vmax(R_DMAX)));
    st->d_nonfinite = vmax(R_DBAD) > 0.0 ? 1 : 0;
    long long bad = kNoBad;
    for (int q = 0; q < nranks; ++q) {
      const double b = all[q * NRED + R_BAD];
      if (b >= 0.0 && static_cast<long long>(b) < bad) bad = static_cast<long long>(b);
    }
    st->bad_code = bad;
    st->aborted = bad != kNoBad ? 1 : st->aborted;
  } else if (mode == COMBINE_RELAX) {
    if (st->aborted || st->finished || st->relax_done) return;
    relax_update(st, sum(R_A_HI, R_A_LO), sum(R_B_HI, R_B_LO));
  } else if (mode == COMBINE_UPDATE) {
    if (st->aborted || st->finished) return;
    const double gamma = st->relax_enabled ? st->gamma : st->gamma_override;
    const double dt = st->dt;
    st->t += (st->relax_enabled && !st->idt) ? gamma * dt : dt;
    st->gamma_seed = st->fell_back ? 1.0 : gamma;
    st->steps_taken += 1;
  }
}

// StepRecord row from the gathered partials (COMBINE_UPDATE), written by the
// host-side sequencing right after combine_kernel
__global__ void record_kernel(StepState* st, const double* all, int nranks, int V, double* records) {
  if (st->aborted || st->finished || !records) return;
  double* row = records + static_cast<size_t>(st->steps_taken - 1) * REC_COLS;
  row[11] = st->dh_hi + st->dh_lo;
  row[0] = st->t;
  row[1] = st->dt;
  row[2] = st->relax_enabled ? st->gamma : st->gamma_override;
  row[3] = st->iters;
  row[4] = st->fell_back;
  for (int r = 0; r < 1 + V; ++r) {
    dd acc = dd_zero();
    for (int q = 0; q < nranks; ++q)
      acc = dd_add(acc, dd{all[q * NRED + R_REC0 + 2 * r], all[q * NRED + R_REC0 + 2 * r + 1]});
    row[5 + r] = acc.hi + acc.lo;
  }
}

// ---------------------------------------------------------------------------
// error_norms (stepper.cpp:195-265), 2D, isentropic-vortex exact solution
// (isentropic_vortex_state, physics.cpp:301-328): the DG solution
// interpolated to the degree-2k GLL points of each cell, L1 (quadrature, later
// divided by the domain measure) and Linf of the pointwise difference.
// fine: [nf nodes][nf weights][nf x 4 interpolation matrix]
// ---------------------------------------------------------------------------
__device__ void vortex_state(const double* p, double x, double y, double t, double* u) {
  const double gamma = p[0], mach = p[1], radius = p[2], intensity = p[3], rho_inf = p[4];
  const double vix = p[5], viy = p[6], hw = p[7];
  auto wrap = [&](double d) {
    const double span = 2.0 * hw;
    d = fmod(d + hw, span);
    if (d < 0.0) d += span;
    return d - hw;
  };
  const double cx = wrap(x - vix * t), cy = wrap(y - viy * t);
  const double r2 = cx * cx + cy * cy;
  const double g = exp((1.0 - r2) / (2.0 * radius * radius));
  const double gm1 = gamma - 1.0;
  const double rho = rho_inf * pow(1.0 - intensity * intensity * mach * mach * gm1 * g * g /
                                             (8.0 * M_PI * M_PI),
                                   1.0 / gm1);
  const double coef = intensity * g / (2.0 * M_PI * radius);
  const double vx = vix - coef * cy, vy = viy + coef * cx;
  const double pres = pow(rho, gamma) / (gamma * mach * mach);
  u[0] = rho;
  u[1] = rho * vx;
  u[2] = rho * vy;
  u[3] = pres / gm1 + 0.5 * rho * (vx * vx + vy * vy);
}

__global__ void __launch_bounds__(256)
    error_norms_kernel(const double* __restrict__ U, MeshDev m, const double* x0,
                       const double* y0, const double* fine, int nf, const double* vp, double t,
                       double* partials, unsigned* counter, double* out, unsigned long long* linf,
                       long long npts) {
  constexpr int V = 4;
  __shared__ double s_red[2 * 4 * 8];
  dd acc[4];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = dd_zero();
  double mx[V] = {0.0, 0.0, 0.0, 0.0};
  const double* fx = fine;
  const double* fw = fine + nf;
  const double* L = fine + 2 * nf;
  for (long long n = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; n < npts;
       n += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int cell = static_cast<int>(n / (nf * nf)), q = static_cast<int>(n % (nf * nf));
    const int qx = q / nf, qy = q % nf;
    const int ci = cell % m.nc[0], cj = cell / m.nc[0];
    const double hx = m.h[0][ci], hy = m.h[1][cj];
    double val[V] = {0.0, 0.0, 0.0, 0.0};
    // interpolate along x per original row, then along y (stepper.cpp:231-251)
#pragma unroll
    for (int iy = 0; iy < N1; ++iy) {
      double row[V] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int l = 0; l < N1; ++l)
#pragma unroll
        for (int v = 0; v < V; ++v)
          row[v] += L[qx * N1 + l] * __ldg(U + sidx<2>(cell, l + N1 * iy, v));
#pragma unroll
      for (int v = 0; v < V; ++v) val[v] += L[qy * N1 + iy] * row[v];
    }
    const double x = x0[ci] + 0.5 * hx * (fx[qx] + 1.0);
    const double y = y0[cj] + 0.5 * hy * (fx[qy] + 1.0);
    double ue[V];
    vortex_state(vp, x, y, t, ue);
    const double w = 0.25 * hx * hy * fw[qx] * fw[qy];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const double diff = fabs(val[v] - ue[v]);
      acc[v] = dd_add_prod(acc[v], w, diff);
      mx[v] = fmax(mx[v], diff);
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double w = warp_max(mx[v]);
    if ((threadIdx.x & 31) == 0) atomic_max_pos(&linf[v], w);
  }
  dd tot[4];
  block_reduce_dd<4>(acc, s_red);
  if (grid_reduce_dd<4>(acc, partials, counter, s_red, tot) && threadIdx.x == 0)
    for (int v = 0; v < V; ++v) out[v] = tot[v].hi + tot[v].lo;
}

}  // namespace dev

using namespace dev;

cudaError_t launch_error_norms(const double* U, const MeshDev& m, const double* x0,
                               const double* y0, const double* fine, int nf, const double* vp,
                               double t, double* partials, unsigned* counter, double* out,
                               unsigned long long* linf, long long ncells, int grid,
                               cudaStream_t s) {
  error_norms_kernel<<<grid, 256, 0, s>>>(U, m, x0, y0, fine, nf, vp, t, partials, counter, out,
                                          linf, ncells * nf * nf);
  return cudaGetLastError();
}

cudaError_t launch_pack_traces(int dim, const StageArgs& a, const MeshDev& m, StepState* st,
                               const int* send, int nsend, double* out, cudaStream_t s) {
  if (nsend <= 0) return cudaSuccess;
  const int fp = dim == 3 ? 16 : 4;
  const int grid = (nsend * fp + 255) / 256;
  if (dim == 2)
    pack_traces_kernel<2><<<grid, 256, 0, s>>>(a, m, st, send, nsend, out);
  else
    pack_traces_kernel<3><<<grid, 256, 0, s>>>(a, m, st, send, nsend, out);
  return cudaGetLastError();
}

cudaError_t launch_stash(StepState* st, int mode, cudaStream_t s) {
  stash_kernel<<<1, 1, 0, s>>>(st, mode);
  return cudaGetLastError();
}

cudaError_t launch_combine(StepState* st, const double* all, int nranks, int mode, int V,
                           double* records, cudaStream_t s) {
  combine_kernel<<<1, 1, 0, s>>>(st, all, nranks, mode);
  if (mode == COMBINE_UPDATE && records) record_kernel<<<1, 1, 0, s>>>(st, all, nranks, V, records);
  return cudaGetLastError();
}

double measure_fp64_peak() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out = nullptr;
  cudaMalloc(&out, sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, iters = 4096;
  dfma_probe_kernel<<<blocks, 256>>>(out, iters, 0.999999, 1e-7);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_probe_kernel<<<blocks, 256>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  const double flops = 2.0 * 8.0 * iters * static_cast<double>(blocks) * 256.0;
  return flops / (best * 1e-3) / 1e9;
}

cudaError_t upload_basis(const double* D, const double* w) {
  cudaError_t e = cudaMemcpyToSymbol(c_D, D, sizeof(double) * N1 * N1);
  if (e != cudaSuccess) return e;
  double Dw[N1 * N1];
  for (int k = 0; k < N1; ++k)
    for (int j = 0; j < N1; ++j) Dw[k * N1 + j] = D[k * N1 + j] * w[k] / w[j];
  e = cudaMemcpyToSymbol(c_Dw, Dw, sizeof(double) * N1 * N1);
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(c_w, w, sizeof(double) * N1);
}

size_t stage_smem_bytes(int dim) {
  return dim == 2 ? sizeof(double) * StageGeo<2>::SM_TOTAL : sizeof(double) * StageGeo<3>::SM_TOTAL;
}

template <int DIM, bool SIMPLE>
static int stage_occ_d(int surf) {
  switch (surf) {
    case 0: return stage_occ_t<DIM, 0, SIMPLE>();
    case 2: return stage_occ_t<DIM, 2, SIMPLE>();
    case 3: return stage_occ_t<DIM, 3, SIMPLE>();
    case 4: return stage_occ_t<DIM, 4, SIMPLE>();
    case 5: return stage_occ_t<DIM, 5, SIMPLE>();
  }
  return 1;
}

// 3D EC volume with the Rusanov or central surface flux runs the warp-per-cell
// kernel (dg_stage3w.cuh); every other variant the block-per-cell one
static bool use_w3(int dim, int surf, int vol, bool visc) {
#ifdef PERRK_NO_W3
  (void)dim; (void)surf; (void)vol; (void)visc;
  return false;
#else
  return dim == 3 && vol == VOL_EC && !visc && (surf == 0 || surf == 2);
#endif
}

template <int SURF, int FORM = -1, int NEXT = -1, int DM = -1>
static void configure_w3() {
  static bool configured[MAX_DEVICES] = {};
  const int dev = current_device();
  if (!configured[dev]) {
    cudaFuncSetAttribute(stage3w_kernel<SURF, FORM, NEXT, DM>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(double) * W3::SM_TOTAL));
    configured[dev] = true;
  }
}

template <int SURF>
static int w3_occ() {
  configure_w3<SURF>();
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, stage3w_kernel<SURF>, W3::T,
                                                sizeof(double) * W3::SM_TOTAL);
  return n;
}

template <int SURF, int FORM = -1, int NEXT = -1, int DM = -1>
static cudaError_t launch_w3_k(const StageArgs& a, const MeshDev& m, const Phys& ph,
                               StepState* st, double* partials, unsigned* counter, int g,
                               cudaStream_t s) {
  configure_w3<SURF, FORM, NEXT, DM>();
  stage3w_kernel<SURF, FORM, NEXT, DM><<<g, W3::T, sizeof(double) * W3::SM_TOTAL, s>>>(
      a, m, ph, st, partials, counter);
  return cudaGetLastError();
}

#ifndef PERRK_W3_SPECIALIZE
#define PERRK_W3_SPECIALIZE 1  // compile-time stage kinds (stage3w_kernel FORM / NEXT / DM)
#endif

template <int SURF>
static cudaError_t launch_w3(const StageArgs& a, const MeshDev& m, const Phys& ph, StepState* st,
                             double* partials, unsigned* counter, int grid, cudaStream_t s) {
  const int blocks = (a.n + W3::WPB - 1) / W3::WPB;
  const int g = blocks < grid ? blocks : grid;
  if (g <= 0) return cudaSuccess;
  if constexpr (PERRK_W3_SPECIALIZE && SURF == 2) {
    // the stage kinds of the p4 families: stage 0, interior stages, the first
    // and the last b-stage (host.cpp build_plan)
    const int key = a.form * 100 + a.write_next * 10 + a.d_mode;
    switch (key) {
      case 10: return launch_w3_k<SURF, 0, 1, 0>(a, m, ph, st, partials, counter, g, s);
      case 110: return launch_w3_k<SURF, 1, 1, 0>(a, m, ph, st, partials, counter, g, s);
      case 111: return launch_w3_k<SURF, 1, 1, 1>(a, m, ph, st, partials, counter, g, s);
      case 102: return launch_w3_k<SURF, 1, 0, 2>(a, m, ph, st, partials, counter, g, s);
      default: break;
    }
  }
  return launch_w3_k<SURF>(a, m, ph, st, partials, counter, g, s);
}

// 2D EC volume with the Rusanov or central surface flux: the warp-per-four-
// cells kernel (dg_stage2w.cuh)
static bool use_w2(int dim, int surf, int vol, bool visc) {
#if defined(PERRK_NO_W2)
  (void)dim; (void)surf; (void)vol; (void)visc;
  return false;
#else
  return dim == 2 && vol == VOL_EC && !visc && (surf == 0 || surf == 2);
#endif
}

template <int SURF>
static void configure_w2() {
  static bool configured[MAX_DEVICES] = {};
  const int dev = current_device();
  if (!configured[dev]) {
    cudaFuncSetAttribute(stage2w_kernel<SURF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(double) * W2::SM_TOTAL));
    configured[dev] = true;
  }
}

template <int SURF>
static int w2_occ() {
  configure_w2<SURF>();
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, stage2w_kernel<SURF>, W2::T,
                                                sizeof(double) * W2::SM_TOTAL);
  return n;
}

template <int SURF>
static cudaError_t launch_w2(const StageArgs& a, const MeshDev& m, const Phys& ph, StepState* st,
                             double* partials, unsigned* counter, int grid, cudaStream_t s) {
  configure_w2<SURF>();
  const int warps = (a.n + W2::CPW - 1) / W2::CPW;
  const int blocks = (warps + W2::WPB - 1) / W2::WPB;
  const int g = blocks < grid ? blocks : grid;
  if (g <= 0) return cudaSuccess;
  stage2w_kernel<SURF><<<g, W2::T, sizeof(double) * W2::SM_TOTAL, s>>>(a, m, ph, st, partials,
                                                                       counter);
  return cudaGetLastError();
}

int stage_blocks_per_sm(int dim, int surf, int vol) {
  if (use_w3(dim, surf, vol, false)) return surf == 2 ? w3_occ<2>() : w3_occ<0>();
  if (use_w2(dim, surf, vol, false)) return surf == 2 ? w2_occ<2>() : w2_occ<0>();
  const bool simple = vol != VOL_EC;
  if (dim == 2) return simple ? stage_occ_d<2, true>(surf) : stage_occ_d<2, false>(surf);
  return simple ? stage_occ_d<3, true>(surf) : stage_occ_d<3, false>(surf);
}

int stage_cells_per_block(int dim) { return dim == 2 ? StageGeo<2>::CPB : StageGeo<3>::CPB; }

cudaError_t launch_stage(int dim, int surf, int vol, const StageArgs& a0, const MeshDev& m,
                         const Phys& ph, StepState* st, double* partials, unsigned* counter,
                         int grid, cudaStream_t s) {
  StageArgs a = a0;
  a.weak = vol == VOL_WEAK;
  if (a.G) {  // BR1 (2D Navier-Stokes) runs with the EC volume flux only
    if (dim != 2 || vol != VOL_EC) return cudaErrorInvalidValue;
    return launch_stage_d<2, true, false>(surf, a, m, ph, st, partials, counter, grid, s);
  }
  if (use_w3(dim, surf, vol, false))
    return surf == 2 ? launch_w3<2>(a, m, ph, st, partials, counter, grid, s)
                     : launch_w3<0>(a, m, ph, st, partials, counter, grid, s);
  if (use_w2(dim, surf, vol, false))
    return surf == 2 ? launch_w2<2>(a, m, ph, st, partials, counter, grid, s)
                     : launch_w2<0>(a, m, ph, st, partials, counter, grid, s);
  if (vol == VOL_EC)
    return dim == 2 ? launch_stage_d<2, false, false>(surf, a, m, ph, st, partials, counter, grid, s)
                    : launch_stage_d<3, false, false>(surf, a, m, ph, st, partials, counter, grid, s);
  return dim == 2 ? launch_stage_d<2, false, true>(surf, a, m, ph, st, partials, counter, grid, s)
                  : launch_stage_d<3, false, true>(surf, a, m, ph, st, partials, counter, grid, s);
}

cudaError_t launch_adv_stage(const AdvArgs& a, int grid, cudaStream_t s) {
  adv_stage_kernel<<<grid, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_adv_final(const double* d, long long M, long long col0, int ncols, double scale,
                             double* D, int grid, cudaStream_t s) {
  adv_final_kernel<<<grid, 256, 0, s>>>(d, M, col0, ncols, scale, D);
  return cudaGetLastError();
}

template <typename K>
static int resident_grid(K kernel, int threads, int cap);

cudaError_t launch_grad(const StageArgs& a, const MeshDev& m, const Phys& ph, StepState* st,
                        double* out, long long ndofs, int mode, int grid, cudaStream_t s) {
  // its own resident capacity (per device), not the stage kernel's grid
  static int resident[MAX_DEVICES] = {};
  const int dev = current_device();
  if (!resident[dev]) resident[dev] = resident_grid(grad_kernel, 128, 1 << 30);
  (void)grid;
  const int groups = (a.n + 7) / 8;
  const int g = groups < resident[dev] ? groups : resident[dev];
  if (g <= 0) return cudaSuccess;
  grad_kernel<<<g, 128, 0, s>>>(a, m, ph, st, out, ndofs, mode);
  return cudaGetLastError();
}

cudaError_t launch_begin_step(StepState* st, cudaStream_t s) {
  begin_step_kernel<<<1, 1, 0, s>>>(st);
  return cudaGetLastError();
}

// grid of a grid-stride node kernel: the resident capacity (one wave, so no
// block waits for a second wave), at most the caller's grid; a function of the
// device only, so the fixed-order reductions stay reproducible
template <typename K>
static int resident_grid(K kernel, int threads, int cap) {
  int dev = 0, sms = 148, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, 0);
  const int g = sms * (occ > 0 ? occ : 1);
  return g < cap ? g : cap;
}

// One grid for relax_pass_kernel, relax_spec_kernel and update_kernel: the
// three walk the nodes in the same warp-block order, so their sums agree bit
// for bit (the fused and unfused relaxation chains give the same step).  It
// is relax_pass_kernel's resident grid; relax_spec_kernel (128 registers)
// holds two of its three blocks per SM at once.  Measured: sizing all three to
// relax_spec_kernel's residency costs the passes more than the spec kernel's
// tail (-4%), and capping relax_spec_kernel at 80 registers spills (neutral).
// Cached per device ordinal (contexts on different devices get their own
// residency), capped by the caller's grid on every call.

template <int DIM>
static int relax_grid(int cap) {
  static int resident[MAX_DEVICES] = {};
  const int dev = current_device();
  if (!resident[dev]) resident[dev] = resident_grid(relax_pass_kernel<DIM>, 256, 1 << 30);
  return resident[dev] < cap ? resident[dev] : cap;
}

cudaError_t launch_relax_pass(int dim, const double* U, const double* d, const MeshDev& m,
                              const Phys& ph, StepState* st, double* partials, unsigned* counter,
                              long long nnodes, int grid, cudaStream_t s) {
  if (dim == 2) {
    const int g = relax_grid<2>(grid);
    relax_pass_kernel<2><<<g, 256, 0, s>>>(U, d, m, ph, st, partials, counter, nnodes);
  } else {
    const int g = relax_grid<3>(grid);
    relax_pass_kernel<3><<<g, 256, 0, s>>>(U, d, m, ph, st, partials, counter, nnodes);
  }
  return cudaGetLastError();
}

cudaError_t launch_update(int dim, double* Uout, const double* Uin, const double* d,
                          const MeshDev& m, const Phys& ph, StepState* st, double* partials,
                          unsigned* counter, long long nnodes, int want_nu, int want_record,
                          double* records, int grid, cudaStream_t s) {
  // relax_pass_kernel's grid: the node walk (and record sums) of relax_spec_kernel
  if (dim == 2) {
    const int g = relax_grid<2>(grid);
    update_kernel<2><<<g, 256, 0, s>>>(Uout, Uin, d, m, ph, st, partials, counter, nnodes,
                                       want_nu, want_record, records);
  } else {
    const int g = relax_grid<3>(grid);
    update_kernel<3><<<g, 256, 0, s>>>(Uout, Uin, d, m, ph, st, partials, counter, nnodes,
                                       want_nu, want_record, records);
  }
  return cudaGetLastError();
}

template <int DIM>
static size_t spec_smem_bytes() {  // [staging] + the six [256] record sums
  return (PERRK_RELAX_DIRECT ? 0 : sizeof(double) * 8 * 2 * 2 * 32 * (DIM + 2)) +
         sizeof(ksum) * 6 * 256;
}

template <int DIM>
static void configure_spec() {  // a function attribute is per device
  static bool done[MAX_DEVICES] = {};
  const int dev = current_device();
  if (!done[dev]) {
    cudaFuncSetAttribute(relax_spec_kernel<DIM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(spec_smem_bytes<DIM>()));
    done[dev] = true;
  }
}

cudaError_t launch_relax_spec(int dim, const double* U, const double* d, double* Uout,
                              const MeshDev& m, const Phys& ph, StepState* st, double* partials,
                              unsigned* counter, long long nnodes, int want_nu, int want_record,
                              double* records, int grid, cudaStream_t s) {
  // the grid of relax_pass_kernel: the same nodes per warp, so the same
  // summation order of r and r' (bitwise the unfused pass)
  if (dim == 2) {
    configure_spec<2>();
    const int g = relax_grid<2>(grid);
    relax_spec_kernel<2><<<g, 256, spec_smem_bytes<2>(), s>>>(U, d, Uout, m, ph, st, partials,
                                                              counter, nnodes, want_nu,
                                                              want_record, records);
  } else {
    configure_spec<3>();
    const int g = relax_grid<3>(grid);
    relax_spec_kernel<3><<<g, 256, spec_smem_bytes<3>(), s>>>(U, d, Uout, m, ph, st, partials,
                                                              counter, nnodes, want_nu,
                                                              want_record, records);
  }
  return cudaGetLastError();
}

cudaError_t launch_numax(int dim, const double* U, const MeshDev& m, const Phys& ph,
                         StepState* st, long long nnodes, int grid, cudaStream_t s) {
  if (dim == 2)
    numax_kernel<2><<<grid, 256, 0, s>>>(U, m, ph, st, nnodes);
  else
    numax_kernel<3><<<grid, 256, 0, s>>>(U, m, ph, st, nnodes);
  return cudaGetLastError();
}

cudaError_t launch_nu_cell(int dim, const double* U, const MeshDev& m, const Phys& ph, double* nu,
                           long long ncells, cudaStream_t s) {
  const int grid = static_cast<int>((ncells + 255) / 256);
  if (dim == 2)
    nu_cell_kernel<2><<<grid, 256, 0, s>>>(U, m, ph, nu, ncells);
  else
    nu_cell_kernel<3><<<grid, 256, 0, s>>>(U, m, ph, nu, ncells);
  return cudaGetLastError();
}

cudaError_t launch_quad(int dim, const double* U, const double* K, const MeshDev& m,
                        const Phys& ph, int mode, double* partials, unsigned* counter, double* out,
                        long long nnodes, int grid, cudaStream_t s) {
  if (dim == 2)
    quad_kernel<2><<<grid, 256, 0, s>>>(U, K, m, ph, mode, partials, counter, out, nnodes);
  else
    quad_kernel<3><<<grid, 256, 0, s>>>(U, K, m, ph, mode, partials, counter, out, nnodes);
  return cudaGetLastError();
}

cudaError_t launch_admissible(int dim, const double* U, const Phys& ph, int* first_bad,
                              long long nnodes, int grid, cudaStream_t s) {
  if (dim == 2)
    admissible_kernel<2><<<grid, 256, 0, s>>>(U, ph, first_bad, nnodes);
  else
    admissible_kernel<3><<<grid, 256, 0, s>>>(U, ph, first_bad, nnodes);
  return cudaGetLastError();
}

// ---- dense Jacobian probe (specopt.cpp:18-35) --------------------------------
// One colour of the probe perturbs local DOF l of every cell in `cells`; the
// colouring (host) keeps their dependency stencils disjoint, so each RHS row
// sees at most one perturbed input and equals the single-column probe bit for
// bit.  h, the u +/- h values and (fp - fm) / (2h) follow specopt.cpp:25-32.
__global__ void probe_set_kernel(double* up, double* um, const double* base, const double* h,
                                 const int* cells, int n, long long stride, int l, int on) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const long long j = static_cast<long long>(cells[q]) * stride + l;
  up[j] = on ? base[j] + h[j] : base[j];
  um[j] = on ? base[j] - h[j] : base[j];
}

// canonical index of device-layout entry i (sidx): a cell's local offset
// v NPC + node is node V + v in the reference's layout
__device__ __forceinline__ long long canonical_of(long long i, long long stride, int npc) {
  const long long c = i / stride;
  const int o = static_cast<int>(i - c * stride);
  const int V = static_cast<int>(stride / npc);
  return c * stride + static_cast<long long>(o % npc) * V + o / npc;
}

__global__ void probe_scatter_kernel(double* J, const double* fp, const double* fm,
                                     const double* h, const int* owner, long long M,
                                     long long stride, int l, int npc) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < M;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int p = owner[i / stride];
    if (p < 0) continue;
    const long long j = static_cast<long long>(p) * stride + l;  // device layout
    // J in the reference's (canonical) column-major order
    J[canonical_of(j, stride, npc) * M + canonical_of(i, stride, npc)] =
        (fp[i] - fm[i]) / (2.0 * h[j]);
  }
}

cudaError_t launch_probe_set(double* up, double* um, const double* base, const double* h,
                             const int* cells, int n, long long stride, int l, int on,
                             cudaStream_t s) {
  if (n > 0) probe_set_kernel<<<(n + 127) / 128, 128, 0, s>>>(up, um, base, h, cells, n, stride, l, on);
  return cudaGetLastError();
}

cudaError_t launch_probe_scatter(double* J, const double* fp, const double* fm, const double* h,
                                 const int* owner, long long M, long long stride, int l, int npc,
                                 int grid, cudaStream_t s) {
  probe_scatter_kernel<<<grid, 256, 0, s>>>(J, fp, fm, h, owner, M, stride, l, npc);
  return cudaGetLastError();
}

// ---- canonical <-> device layout (sidx), at upload / download ----------------
// Writes are coalesced; each thread's read stays inside its cell's block
// (2.5 KB in 3D), which L1 holds.
__global__ void layout_kernel(double* dst, const double* src, long long ncells, int npc, int V,
                              int to_device) {
  const long long stride = static_cast<long long>(npc) * V, n = ncells * stride;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long c = i / stride;
    const int o = static_cast<int>(i - c * stride);
    // to_device: i is (v, node) with o = v npc + node; else (node, v), o = node V + v
    const int other = to_device ? (o % npc) * V + o / npc : (o % V) * npc + o / V;
    dst[i] = src[c * stride + other];
  }
}

cudaError_t launch_layout(double* dst, const double* src, long long ncells, int npc, int V,
                          int to_device, int grid, cudaStream_t s) {
  layout_kernel<<<grid, 256, 0, s>>>(dst, src, ncells, npc, V, to_device);
  return cudaGetLastError();
}

// ---- matrix-free spectrum estimation (dg_krylov.cuh) -------------------------
cudaError_t launch_krylov_perturb(double* up, double* um, const double* u, const double* v,
                                  double h, long long n, int grid, cudaStream_t s) {
  krylov_perturb_kernel<<<grid, 256, 0, s>>>(up, um, u, v, h, n);
  return cudaGetLastError();
}

cudaError_t launch_krylov_fd(double* w, const double* fp, const double* fm, double inv2h,
                             const unsigned char* cmask, long long stride, long long n, int grid,
                             cudaStream_t s) {
  krylov_fd_kernel<<<grid, 256, 0, s>>>(w, fp, fm, inv2h, cmask, stride, n);
  return cudaGetLastError();
}

cudaError_t launch_krylov_seed(double* v, const unsigned char* cmask, long long stride,
                               long long n, unsigned long long seed, int grid, cudaStream_t s) {
  krylov_seed_kernel<<<grid, 256, 0, s>>>(v, cmask, stride, n, seed);
  return cudaGetLastError();
}

cudaError_t launch_krylov_dots(const double* Vb, long long ld, int k, const double* w,
                               double* partials, int nblocks, double* out, long long n,
                               cudaStream_t s) {
  krylov_dots_kernel<<<dim3(nblocks, k), 256, 0, s>>>(Vb, ld, w, partials, n);
  krylov_dots_finish_kernel<<<(k + 127) / 128, 128, 0, s>>>(partials, nblocks, k, out);
  return cudaGetLastError();
}

cudaError_t launch_krylov_project(double* w, const double* Vb, long long ld, const double* c,
                                  int k, long long n, int grid, cudaStream_t s) {
  krylov_project_kernel<<<grid, 256, 0, s>>>(w, Vb, ld, c, k, n);
  return cudaGetLastError();
}

cudaError_t launch_krylov_scale(double* dst, const double* src, double sc, long long n, int grid,
                                cudaStream_t s) {
  krylov_scale_kernel<<<grid, 256, 0, s>>>(dst, src, sc, n);
  return cudaGetLastError();
}

}  // namespace perrk
