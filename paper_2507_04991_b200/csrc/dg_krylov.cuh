// Matrix-free spectrum estimation: the device side of
// perrk_krylov_hessenberg.  Arnoldi on the central-difference Jacobian-vector
// product of the full RHS,
//   J v = (rhs(u + h v) - rhs(u - h v)) / (2 h),
// the product the reference's dense probe (specopt.cpp:18-35) takes one unit
// vector at a time; here along Krylov vectors, so the mesh size is not bounded
// by an M x M matrix.  Vector kernels only: the RHS evaluations are the stage
// kernels (rhs_full_device in host.cpp).
#pragma once

namespace perrk {
namespace dev {

// up = u + h v, um = u - h v
__global__ void krylov_perturb_kernel(double* up, double* um, const double* u, const double* v,
                                      double h, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double a = u[i], b = h * v[i];
    up[i] = a + b;
    um[i] = a - b;
  }
}

// w = (fp - fm) / (2h), zero outside the flagged cells (stride = nodes * V)
__global__ void krylov_fd_kernel(double* w, const double* fp, const double* fm, double inv2h,
                                 const unsigned char* cmask, long long stride, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const bool on = !cmask || cmask[i / stride];
    w[i] = on ? (fp[i] - fm[i]) * inv2h : 0.0;
  }
}

// deterministic start vector: a hashed uniform value in [-1, 1) per entry
// (splitmix64 of the index and the seed), zero outside the flagged cells
__global__ void krylov_seed_kernel(double* v, const unsigned char* cmask, long long stride,
                                   long long n, unsigned long long seed) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    unsigned long long z = seed + 0x9E3779B97F4A7C15ULL * static_cast<unsigned long long>(i + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    const double r = static_cast<double>(z >> 11) * (1.0 / 9007199254740992.0);  // [0, 1)
    v[i] = (!cmask || cmask[i / stride]) ? 2.0 * r - 1.0 : 0.0;
  }
}

// partials[j * gridDim.x + b] = block b's part of <V_j, w>, j = blockIdx.y
// (double-double per thread, fixed order: reproducible)
__global__ void __launch_bounds__(256) krylov_dots_kernel(const double* Vb, long long ld,
                                                          const double* w, double* partials,
                                                          long long n) {
  const int j = blockIdx.y;
  const double* vj = Vb + static_cast<long long>(j) * ld;
  dd acc = dd_zero();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    acc = dd_add_prod(acc, vj[i], w[i]);
  __shared__ double s[2 * 8];
  dd v[1] = {acc};
  block_reduce_dd<1>(v, s);
  if (threadIdx.x == 0) {
    partials[2 * (static_cast<long long>(j) * gridDim.x + blockIdx.x)] = v[0].hi;
    partials[2 * (static_cast<long long>(j) * gridDim.x + blockIdx.x) + 1] = v[0].lo;
  }
}

// out[j] = sum over blocks of partials (one thread per j, fixed order)
__global__ void krylov_dots_finish_kernel(const double* partials, int nblocks, int k,
                                          double* out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  dd acc = dd_zero();
  for (int b = 0; b < nblocks; ++b)
    acc = dd_add(acc, dd{partials[2 * (static_cast<long long>(j) * nblocks + b)],
                         partials[2 * (static_cast<long long>(j) * nblocks + b) + 1]});
  out[j] = acc.hi + acc.lo;
}

// w -= sum_j c_j V_j (classical Gram-Schmidt sweep), c on the device
__global__ void krylov_project_kernel(double* w, const double* Vb, long long ld, const double* c,
                                      int k, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    double x = w[i];
    for (int j = 0; j < k; ++j) x = fma(-c[j], Vb[static_cast<long long>(j) * ld + i], x);
    w[i] = x;
  }
}

__global__ void krylov_scale_kernel(double* dst, const double* src, double s, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[i] = s * src[i];
}

}  // namespace dev
}  // namespace perrk
