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
#define PERRK_GRAD_MINB 12  // resident 128-thread blocks per SM grad_kernel is compiled for (40 registers, no spills; A/B: 114 -> 104 us)
#endif

__global__ void __launch_bounds__(128, PERRK_GRAD_MINB)
    grad_kernel(StageArgs a, MeshDev m, Phys ph, StepState* st, double* out, long long ndofs,
                int mode) {
  constexpr int DIM = 2, V = 4, NPC = 16, FP = 4, NFP = 4 * FP, T = 128, CPB = T / NPC;
  __shared__ double su[V][T];             // formed stage state
  __shared__ double sn[V][CPB * NFP];     // neighbour traces [cell][face][pt]
  __shared__ int s_cell[CPB], s_nbc[CPB][4];
  __shared__ double s_ca1[CPB], s_na1[CPB][4], s_jac[CPB][2], s_lift[CPB][2];
  __shared__ signed char s_cform[CPB], s_nform[CPB][4];
  if (st->aborted || st->finished) return;
  const int tid = threadIdx.x;
  const int cs = tid / NPC, l = tid % NPC;
  const int il[2] = {l % N1, l / N1};
  const double dt = st->dt;
  const int ngroups = (a.n + CPB - 1) / CPB;
  for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    __syncthreads();
    if (tid < CPB) {
      const int slot = grp * CPB + tid;
      const int cell = slot < a.n ? (a.list ? a.list[slot] : slot) : -1;
      s_cell[tid] = cell;
      if (cell >= 0) {
        const CellRec* r = m.rec + cell;
        const int lev = r->lev[0];
        s_ca1[tid] = dt * a.a1[lev];
        s_cform[tid] = a.formed[lev];
#pragma unroll
        for (int f = 0; f < 4; ++f) {  // face 2 d + side; the whole mesh is local (no slabs)
          const int l2 = r->lev[1 + f];
          s_nbc[tid][f] = r->nb[f];
          s_na1[tid][f] = dt * a.a1[l2];
          s_nform[tid][f] = a.formed[l2];
        }
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          s_jac[tid][d] = 0.5 * r->J2[d];  // 2 / h (J2 = 2 (2 / h): exact)
          s_lift[tid][d] = r->lift[d];
        }
      }
    }
    __syncthreads();
    const int cell = s_cell[cs];
    if (cell >= 0) {
      const size_t gi = static_cast<size_t>(cell) * NPC * V + l;  // device layout (sidx)
#pragma unroll
      for (int v = 0; v < V; ++v) {
        double u;
        const size_t g = gi + v * NPC;
        if (!a.form) u = __ldg(a.U + g);
        else if (s_cform[cs]) u = __ldg(a.Us + g);
        else u = fma(s_ca1[cs], __ldg(a.K1 + g), __ldg(a.U + g));
        su[v][tid] = u;
      }
    }
    for (int q = tid; q < CPB * NFP; q += T) {
      const int c2 = q / NFP, r = q % NFP, f = r / FP, pt = r % FP;
      if (s_cell[c2] < 0) continue;
      const int d = f >> 1, side = f & 1;
      const int nbc = s_nbc[c2][f];
      const int node = (d == 0 ? N1 * pt : pt) + (side ? 0 : N1 - 1) * (d == 0 ? 1 : N1);
      const size_t gi = static_cast<size_t>(nbc) * NPC * V + node;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        double u;
        const size_t g = gi + v * NPC;
        if (!a.form) u = __ldg(a.U + g);
        else if (s_nform[c2][f]) u = __ldg(a.Us + g);
        else u = fma(s_na1[c2][f], __ldg(a.K1 + g), __ldg(a.U + g));
        sn[v][q] = u;
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
      const double jac = s_jac[cs][d];
#pragma unroll
      for (int v = 0; v < V; ++v) g[d][v] = 0.0;
      // strong-form derivative along the line (gradients_1d, semidisc.cpp:266-281)
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        const double coef = jac * c_D[j * N1 + k];
        const int tk = tid + (k - j) * stride;
#pragma unroll
        for (int v = 0; v < V; ++v) g[d][v] += coef * su[v][tk];
      }
      // central interface lift (semidisc.cpp:283-318)
      if (j == 0 || j == N1 - 1) {
        const int e = j == 0 ? 0 : 1;
        const int pt = d == 0 ? il[1] : il[0];
        const int qn = (cs * 4 + 2 * d + e) * FP + pt;
        const double coef = s_lift[cs][d];
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
