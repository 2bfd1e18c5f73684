// BR1 viscous terms of the 2D compressible Navier-Stokes-Fourier equations
// (oracle extension of the reference's 1D path, semidisc.cpp:245-395 and
// physics.cpp:260-273; the 2D restatement is oracle/perrk_oracle.c
// gradients_2d / add_viscous_2d / viscous_flux_2d).
//
//   grad_kernel   per stage, over the stage's gradient cells (active cells and
//                 their face neighbours, semidisc.cpp:254-263): strong-form
//                 gradient of the formed stage state, D u along each LGL line
//                 plus the central interface lift (1/2 (u_L + u_R) - u) at the
//                 line ends, then the viscous flux G_d(u, grad u) per node
//                 (stored, [dir][node][var]) or the raw gradients (br1_gradients).
//   stage kernel  (VISC) adds the weak-form divergence of G with the central
//                 interface flux 1/2 (G_L + G_R) (semidisc.cpp:321-395).
#pragma once

namespace perrk {
namespace dev {

// NSFPhysics::viscous_flux (physics.cpp:260-273) in 2D: Stokes stress with
// lambda = -2/3 mu, Fourier heat flux q = -kappa grad T, T = p / rho.
// g: d/dx then d/dy of the conserved variables.
__device__ __forceinline__ void visc_flux2(const Phys& ph, const double* u, const double* gx,
                                           const double* gy, double* fx, double* fy) {
  // one reciprocal of rho (frcp: full double precision) instead of eight
  // IEEE divisions
  const double rho = u[0], ir = frcp(rho);
  const double vx = u[1] * ir, vy = u[2] * ir;
  const double vx_x = (gx[1] - vx * gx[0]) * ir, vy_x = (gx[2] - vy * gx[0]) * ir;
  const double vx_y = (gy[1] - vx * gy[0]) * ir, vy_y = (gy[2] - vy * gy[0]) * ir;
  const double e = u[3] * ir * ir;
  const double t_x = ph.gm1 * (gx[3] * ir - e * gx[0] - (vx * vx_x + vy * vy_x));
  const double t_y = ph.gm1 * (gy[3] * ir - e * gy[0] - (vx * vx_y + vy * vy_y));
  const double tau_xx = ph.mu * (4.0 / 3.0 * vx_x - 2.0 / 3.0 * vy_y);
  const double tau_yy = ph.mu * (4.0 / 3.0 * vy_y - 2.0 / 3.0 * vx_x);
  const double tau_xy = ph.mu * (vx_y + vy_x);
  fx[0] = 0.0;
  fx[1] = tau_xx;
  fx[2] = tau_xy;
  fx[3] = vx * tau_xx + vy * tau_xy + ph.kappa * t_x;
  fy[0] = 0.0;
  fy[1] = tau_xy;
  fy[2] = tau_yy;
  fy[3] = vx * tau_xy + vy * tau_yy + ph.kappa * t_y;
}

// out: mode 0 -> viscous flux G [2][nodes][V]; mode 1 -> gradients [2][nodes][V]
// (both in the device layout).  Per group of eight cells the descriptors come
// from the static cell records (host.cpp build_cell_records: neighbours,
// levels, 4/h, lift; no dependent level loads), and the stage state and the
// neighbour traces sit in shared memory variable-major ([V][node]: the
// 8-byte accesses of a warp are conflict free).
#ifndef PERRK_GRAD_MINB
#define PERRK_GRAD_MINB 10  // resident 128-thread blocks per SM grad_kernel is compiled for (48 registers, no spills)
#endif

__global__ void __launch_bounds__(128, PERRK_GRAD_MINB)
    grad_kernel(StageArgs a, MeshDev m, Phys ph, StepState* st, double* out, long long ndofs,
                int mode) {
  constexpr int DIM = 2, V = 4, NPC = 16, FP = 4, NFP = 4 * FP, T = 128, CPB = T / NPC;
  __shared__ double su[V][T];             // formed stage state
  __shared__ double sn[V][CPB * NFP];     // neighbour traces [cell][face][pt]
  if (st->aborted || st->finished) return;
  const int tid = threadIdx.x;
  const int cs = tid / NPC, l = tid % NPC;
  const int il[2] = {l % N1, l / N1};
  const double dt = st->dt;
  const int ngroups = (a.n + CPB - 1) / CPB;
  // thread tid also fetches one neighbour trace point of its own cell:
  // item q = tid = (cs, face f, point pt), CPB * NFP = T
  static_assert(CPB * NFP == T, "one trace point per thread");
  const int f = (tid % NFP) / FP, pt = tid % FP;
  const int fd = f >> 1, fside = f & 1;
  const int fnode = (fd == 0 ? N1 * pt : pt) + (fside ? 0 : N1 - 1) * (fd == 0 ? 1 : N1);
  for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    // every thread reads its cell's descriptor itself (the 16 threads of a
    // cell load the same words: broadcast), so no thread waits on a
    // descriptor stage and its barrier
    const int slot = grp * CPB + cs;
    const int cell = slot < a.n ? (a.list ? a.list[slot] : slot) : -1;
    double jac[2] = {0.0, 0.0}, lift[2] = {0.0, 0.0};
    __syncthreads();  // su / sn of the previous group are read
    if (cell >= 0) {
      const CellRec* r = m.rec + cell;  // the whole mesh is local (no slabs)
      const int lev = r->lev[0], l2 = r->lev[1 + f], nbc = r->nb[f];
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        jac[d] = 0.5 * r->J2[d];  // 2 / h (J2 = 2 (2 / h): exact)
        lift[d] = r->lift[d];
      }
      const bool cform = a.formed[lev] != 0, nform = a.formed[l2] != 0;
      const double ca1 = dt * a.a1[lev], na1 = dt * a.a1[l2];
      const size_t gi = static_cast<size_t>(cell) * NPC * V + l;  // device layout (sidx)
      const size_t gn = static_cast<size_t>(nbc) * NPC * V + fnode;
      double uo_[V], un_[V];
      if (!a.form) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          uo_[v] = __ldg(a.U + gi + v * NPC);
          un_[v] = __ldg(a.U + gn + v * NPC);
        }
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          uo_[v] = cform ? __ldg(a.Us + gi + v * NPC)
                         : fma(ca1, __ldg(a.K1 + gi + v * NPC), __ldg(a.U + gi + v * NPC));
          un_[v] = nform ? __ldg(a.Us + gn + v * NPC)
                         : fma(na1, __ldg(a.K1 + gn + v * NPC), __ldg(a.U + gn + v * NPC));
        }
      }
#pragma unroll
      for (int v = 0; v < V; ++v) {
        su[v][tid] = uo_[v];
        sn[v][tid] = un_[v];
      }
    }
    __syncthreads();
    if (cell < 0) continue;
    double uo[V];
#pragma unroll
    for (int v = 0; v < V; ++v) uo[v] = su[v][tid];
    double g[2][V];
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      const int stride = d == 0 ? 1 : N1;
      const int j = il[d];
      const double jacd = jac[d];
#pragma unroll
      for (int v = 0; v < V; ++v) g[d][v] = 0.0;
      // strong-form derivative along the line (gradients_1d, semidisc.cpp:266-281)
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        const double coef = jacd * c_D[j * N1 + k];
        const int tk = tid + (k - j) * stride;
#pragma unroll
        for (int v = 0; v < V; ++v) g[d][v] += coef * su[v][tk];
      }
      // central interface lift (semidisc.cpp:283-318)
      if (j == 0 || j == N1 - 1) {
        const int e = j == 0 ? 0 : 1;
        const int pt = d == 0 ? il[1] : il[0];
        const int qn = (cs * 4 + 2 * d + e) * FP + pt;
        const double coef = lift[d];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const double un = sn[v][qn];
          const double ustar = 0.5 * (e ? uo[v] + un : un + uo[v]);
          g[d][v] += (e ? coef : -coef) * (ustar - uo[v]);
        }
      }
    }
    const size_t gi = static_cast<size_t>(cell) * NPC * V + l;  // variable v at gi + v NPC
    if (mode == 1) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        out[gi + v * NPC] = g[0][v];
        out[ndofs + gi + v * NPC] = g[1][v];
      }
    } else {
      double fx[V], fy[V];
      visc_flux2(ph, uo, g[0], g[1], fx, fy);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        out[gi + v * NPC] = fx[v];
        out[ndofs + gi + v * NPC] = fy[v];
      }
    }
  }
}

}  // namespace dev
}  // namespace perrk
