// Batched linear-advection P-ERK step: the update matrix of one step
// (analysis::assemble_update_matrix, analysis.cpp:11-32).
//
// The reference assembles D column by column: for every unit vector e_j it
// runs perk_step (stepper.cpp:17-114) with relaxation off and gamma fixed
// (gamma_override) on AdvectionPhysics (physics.hpp:54-85), 1D or 2D, and
// stores the stepped vector as column j.  Here a chunk of B columns advances
// together, one launch per stage:
//
//   adv_stage_kernel  one thread per (column, node of an active cell): forms
//                     the stage state of the node's line partners and face
//                     neighbours on the fly from the column's unit vector
//                     (never stored: U = e_j), K1 and K_{i-1}
//                     (stepper.cpp:60-72), evaluates the DGSEM RHS of the node
//                     (semidisc.cpp:153-243 in 1D, :409-557 in 2D; weak or
//                     flux-differencing volume, surface flux + LGL lift) and
//                     accumulates d += b_i K_i (stepper.cpp:89-92);
//   adv_final_kernel  D(:, j) = e_j + gamma dt d_j (stepper.cpp:108-109),
//                     written column-major (Eigen's layout of UpdateMatrix::D).
//
// Buffers per chunk: K1, two K_{i-1}/K_i ping-pong buffers and d, each
// B x M doubles, column-major like D.  Work per stage is B x (active nodes),
// embarrassingly parallel; the kernel is HBM-bound (3 reads of K-type data per
// line partner hit L1/L2 within the column's cell).
#pragma once

namespace perrk {
namespace dev {

// AdvArgs: dg_launch.hpp

// numerical_flux (physics.cpp:40-65) with AdvectionPhysics (physics.cpp:80-88)
__device__ __forceinline__ double adv_flux(int tag, double a, double ul, double ur) {
  switch (tag) {
    case 0:  // central: 1/2 (f(ul) + f(ur))
      return 0.5 * (a * ul + a * ur);
    case 1:  // upwind
      return 0.5 * a * (ul + ur) - 0.5 * fabs(a) * (ur - ul);
    case 2: {  // rusanov: max_wave_speed = |a| on both sides
      const double lam = fabs(a);
      return 0.5 * (a * ul + a * ur) - 0.5 * lam * (ur - ul);
    }
    default:  // 5, ec: central for s = u^2
      return 0.5 * a * (ul + ur);
  }
}

__device__ __forceinline__ double adv_formed(const AdvArgs& A, long long col, long long g, int npc) {
  const double u = (g == A.col0 + col) ? 1.0 : 0.0;  // the column's unit vector U = e_j
  if (A.stage == 0) return u;
  const int lev = A.level[g / npc];
  const double a1 = A.a1[lev], ap = A.ap[lev];
  const size_t k = static_cast<size_t>(col) * A.M + g;
  if (ap != 0.0) return u + A.dt * (a1 * A.K1[k] + ap * A.Kp[k]);
  return u + A.dt * a1 * A.K1[k];
}

__global__ void __launch_bounds__(256) adv_stage_kernel(AdvArgs A) {
  const int npc = A.dim == 1 ? N1 : N1 * N1;
  const long long per_col = static_cast<long long>(A.nlist) * npc;
  const long long total = per_col * A.ncols;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long col = q / per_col;
    const long long r = q % per_col;
    const int slot = static_cast<int>(r / npc), l = static_cast<int>(r % npc);
    const int cell = A.list ? A.list[slot] : slot;
    const int co[2] = {cell % A.nc[0], cell / A.nc[0]};
    const int il[2] = {l % N1, l / N1};
    const long long g0 = static_cast<long long>(cell) * npc;
    const double uj = adv_formed(A, col, g0 + l, npc);
    const double w0 = c_w[0];
    double K = 0.0;
    for (int d = 0; d < A.dim; ++d) {
      const double h = A.h[d][co[d]];
      const double J = 2.0 / h;
      const double a = A.a[d];
      const int j = il[d], stride = d == 0 ? 1 : N1;
      const int base = l - j * stride;
      if (A.weak) {  // (1/w_j) sum_m D_mj w_m f_m (semidisc.cpp:172-181, :427-441)
        for (int m = 0; m < N1; ++m) {
          const double um = m == j ? uj : adv_formed(A, col, g0 + base + m * stride, npc);
          K += J * c_D[m * N1 + j] * c_w[m] / c_w[j] * (a * um);
        }
      } else {  // flux differencing (semidisc.cpp:183-198, :446-485)
        const double djj = c_D[j * N1 + j];
        if (djj != 0.0) K -= J * 2.0 * djj * (a * uj);
        for (int m = 0; m < N1; ++m) {
          if (m == j) continue;
          const double um = adv_formed(A, col, g0 + base + m * stride, npc);
          const double fv = m > j ? adv_flux(A.volume_flux, a, uj, um)
                                  : adv_flux(A.volume_flux, a, um, uj);
          K -= J * 2.0 * c_D[j * N1 + m] * fv;
        }
      }
      // faces (periodic wrap): the lift onto this node's trace
      // (semidisc.cpp:207-234 in 1D, :489-556 in 2D)
      if (j == 0 || j == N1 - 1) {
        const int side = j == N1 - 1;
        int c2[2] = {co[0], co[1]};
        const int nd = A.nc[d];
        c2[d] = side ? (c2[d] + 1 == nd ? 0 : c2[d] + 1) : (c2[d] == 0 ? nd - 1 : c2[d] - 1);
        const int nbc = c2[0] + A.nc[0] * c2[1];
        const int nl = side ? l - (N1 - 1) * stride : l + (N1 - 1) * stride;
        const double un = adv_formed(A, col, static_cast<long long>(nbc) * npc + nl, npc);
        const double coef = 2.0 / (h * w0);
        const double fstar = side ? adv_flux(A.surface, a, uj, un) : adv_flux(A.surface, a, un, uj);
        const double term = A.weak ? fstar : fstar - a * uj;
        K += side ? -coef * term : coef * term;
      }
    }
    const size_t k = static_cast<size_t>(col) * A.M + g0 + l;
    A.Kout[k] = K;
    if (A.b != 0.0) A.d[k] += A.b * K;
  }
}

__global__ void __launch_bounds__(256) adv_final_kernel(const double* d, long long M, long long col0,
                                                         int ncols, double scale, double* D) {
  const long long total = M * ncols;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long col = q / M, g = q % M;
    const double u = (g == col0 + col) ? 1.0 : 0.0;
    D[q] = u + scale * d[q];
  }
}

}  // namespace dev
}  // namespace perrk
