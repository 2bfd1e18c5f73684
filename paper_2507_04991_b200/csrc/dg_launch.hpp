// Host-visible launch interface of the device kernels (dg_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include "dg_device.cuh"

namespace perrk {

// Arguments of one stage launch (one P-ERK stage i over its active cells).
struct StageArgs {
  const double* U;       // U_n
  const double* K1;      // K_1 (stage 0 RHS)
  const double* Us;      // formed stage state U_i (cells of levels with formed[lev])
  double* Usn;           // U_{i+1} of the processed cells (write_next)
  double* Kout;          // K_i (written when write_k: stage 0 -> K1, rhs queries)
  double* d;             // update direction
  const int* list;       // active cells of the stage (nullptr: all cells 0..n-1)
  int n;                 // number of cells processed
  double a1[dev::MAXR + 1];   // a_{i,1} by level: fallback formation U + dt a1 K1
  double a1n[dev::MAXR + 1];  // a_{i+1,1} by level (epilogue formation of U_{i+1})
  double apn[dev::MAXR + 1];  // a_{i+1,i} by level
  signed char formed[dev::MAXR + 1];  // U_i of this level's cells is in Us (active at i-1)
  int form;              // 0: the stage state is U_n (stage 0, RHS queries)
  int write_next;        // U_{i+1} = U + dt (a_{i+1,1} K1 + a_{i+1,i} K_i) for processed cells
  int write_k;
  int d_mode;            // 0 none, 1 d = b K, 2 d += b K
  double b;
  int want_dh;           // dH += dt b <w(U_i), K_i>
  int want_h;            // H(U_n) (stage 0)
  int want_dmax;         // max |d| (last b-stage)
  int stage;
  long long ncells;      // GLOBAL cells (positivity codes are stage * ncells + global cell)
  const double* G;       // BR1 viscous fluxes [2][ndofs] (nullptr: inviscid)
  long long ndofs;
  int weak;              // volume: set by launch_stage from its vol argument
};

// one stage of the batched advection update-matrix step (dg_advection.cuh)
struct AdvArgs {
  int dim;          // 1 or 2
  int nc[2];        // cells per axis
  const double* h[2];  // cell sizes per axis
  const int8_t* level;  // effective level per cell
  double a[2];      // advection velocity
  int surface;      // PERRK_FLUX_* (central, upwind, rusanov, ec)
  int volume_flux;  // flux differencing: central or ec (both 1/2 a (ul + ur) up to rounding)
  int weak;         // weak-form volume integral
  long long M;      // dofs per column
  long long col0;   // first column of the chunk
  int ncols;        // columns in the chunk
  const double* K1;
  const double* Kp;  // K_{i-1}
  double* Kout;      // K_i (stage 0: K1)
  double* d;
  double dt;
  int stage;
  double a1[dev::MAXR + 1], ap[dev::MAXR + 1];  // by level: a_{i,1}, a_{i,i-1} (0 at i = 1)
  double b;                           // b_i
  const int* list;                    // active cells (nullptr: all)
  int nlist;
};

// volume integral of the stage kernel (SemidiscretizationSpec::volume_mode/_flux)
enum { VOL_WEAK = 0, VOL_CENTRAL = 1, VOL_EC = 2 };

double measure_fp64_peak();  // GFLOP/s on the current device (DFMA loop)
cudaError_t upload_basis(const double* D, const double* w);
size_t stage_smem_bytes(int dim);
int stage_cells_per_block(int dim);
int stage_blocks_per_sm(int dim, int surf, int vol);  // resident stage blocks per SM

cudaError_t launch_stage(int dim, int surf, int vol, const StageArgs& a, const dev::MeshDev& m,
                         const dev::Phys& ph, dev::StepState* st, double* partials,
                         unsigned* counter, int grid, cudaStream_t s);
cudaError_t launch_adv_stage(const AdvArgs& a, int grid, cudaStream_t s);
cudaError_t launch_adv_final(const double* d, long long M, long long col0, int ncols, double scale,
                             double* D, int grid, cudaStream_t s);
cudaError_t launch_grad(const StageArgs& a, const dev::MeshDev& m, const dev::Phys& ph,
                        dev::StepState* st, double* out, long long ndofs, int mode, int grid,
                        cudaStream_t s);
cudaError_t launch_begin_step(dev::StepState* st, cudaStream_t s);
cudaError_t launch_relax_pass(int dim, const double* U, const double* d, const dev::MeshDev& m,
                              const dev::Phys& ph, dev::StepState* st, double* partials,
                              unsigned* counter, long long nnodes, int grid, cudaStream_t s);
cudaError_t launch_update(int dim, double* Uout, const double* Uin, const double* d,
                          const dev::MeshDev& m, const dev::Phys& ph, dev::StepState* st,
                          double* partials, unsigned* counter, long long nnodes, int want_nu,
                          int want_record, double* records, int grid, cudaStream_t s);
cudaError_t launch_relax_spec(int dim, const double* U, const double* d, double* Uout,
                              const dev::MeshDev& m, const dev::Phys& ph, dev::StepState* st,
                              double* partials, unsigned* counter, long long nnodes, int want_nu,
                              int want_record, double* records, int grid, cudaStream_t s);
cudaError_t launch_numax(int dim, const double* U, const dev::MeshDev& m, const dev::Phys& ph,
                         dev::StepState* st, long long nnodes, int grid, cudaStream_t s);
cudaError_t launch_nu_cell(int dim, const double* U, const dev::MeshDev& m, const dev::Phys& ph,
                           double* nu, long long ncells, cudaStream_t s);
cudaError_t launch_quad(int dim, const double* U, const double* K, const dev::MeshDev& m,
                        const dev::Phys& ph, int mode, double* partials, unsigned* counter,
                        double* out, long long nnodes, int grid, cudaStream_t s);
cudaError_t launch_error_norms(const double* U, const dev::MeshDev& m, const double* x0,
                               const double* y0, const double* fine, int nf, const double* vp,
                               double t, double* partials, unsigned* counter, double* out,
                               unsigned long long* linf, long long ncells, int grid,
                               cudaStream_t s);

// element-slab decomposition
enum { RED_STAGES = 0, RED_RELAX = 1, RED_UPDATE = 2, RED_NUMAX = 3 };
cudaError_t launch_pack_traces(int dim, const StageArgs& a, const dev::MeshDev& m,
                               dev::StepState* st, const int* send, int nsend, double* out,
                               cudaStream_t s);
cudaError_t launch_stash(dev::StepState* st, int mode, cudaStream_t s);
cudaError_t launch_combine(dev::StepState* st, const double* all, int nranks, int mode, int V,
                           double* records, cudaStream_t s);
cudaError_t launch_probe_set(double* up, double* um, const double* base, const double* h,
                             const int* cells, int n, long long stride, int l, int on,
                             cudaStream_t s);
cudaError_t launch_probe_scatter(double* J, const double* fp, const double* fm, const double* h,
                                 const int* owner, long long M, long long stride, int l, int npc,
                                 int grid, cudaStream_t s);
// canonical (reference) <-> device (sidx) layout of ncells cell blocks
cudaError_t launch_layout(double* dst, const double* src, long long ncells, int npc, int V,
                          int to_device, int grid, cudaStream_t s);
// matrix-free spectrum estimation (dg_krylov.cuh)
cudaError_t launch_krylov_perturb(double* up, double* um, const double* u, const double* v,
                                  double h, long long n, int grid, cudaStream_t s);
cudaError_t launch_krylov_fd(double* w, const double* fp, const double* fm, double inv2h,
                             const unsigned char* cmask, long long stride, long long n, int grid,
                             cudaStream_t s);
cudaError_t launch_krylov_seed(double* v, const unsigned char* cmask, long long stride,
                               long long n, unsigned long long seed, int grid, cudaStream_t s);
cudaError_t launch_krylov_dots(const double* Vb, long long ld, int k, const double* w,
                               double* partials, int nblocks, double* out, long long n,
                               cudaStream_t s);
cudaError_t launch_krylov_project(double* w, const double* Vb, long long ld, const double* c,
                                  int k, long long n, int grid, cudaStream_t s);
cudaError_t launch_krylov_scale(double* dst, const double* src, double sc, long long n, int grid,
                                cudaStream_t s);
cudaError_t launch_admissible(int dim, const double* U, const dev::Phys& ph, int* first_bad,
                              long long nnodes, int grid, cudaStream_t s);

}  // namespace perrk
