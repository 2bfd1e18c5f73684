/* perrk_b200 — C-ABI of the B200-native P-ERRK / EC-DGSEM hot path.
 *
 * This is the drop-in boundary.  The reference (arxiv/paper_2507_04991, a
 * C++20 CPU library under proj/core) has no FFI; its hot path sits behind the
 * C++ API listed per entry point below.  Every function here replaces one of
 * those calls with plain pointers and sizes (no C++ or torch types), returns
 * 0 on success and a negative PERRK_E* code on failure (the reference throws
 * perrk::Error, common.hpp:15-23), and leaves a message for perrk_last_error().
 *
 * State layout (host and device) is the reference's canonical one
 * (common.hpp:11-13, semidisc.hpp:37-39): cell-major (cells x-fastest, then y,
 * then z), node-major within a cell (LGL node x-fastest), variable-minor.
 *
 * Threading: one host thread per context (the reference's
 * Semidiscretization is not thread-safe either, semidisc.hpp:112).  All work
 * of a context is ordered on its own CUDA stream; the *_resident / advance
 * calls are asynchronous until perrk_sync().
 */
#ifndef PERRK_B200_H
#define PERRK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PERRK_B200_ABI_VERSION 2

/* status codes */
#define PERRK_OK 0
#define PERRK_EINVAL -1    /* precondition violated (reference: PERRK_REQUIRE throws) */
#define PERRK_ECUDA -2     /* CUDA runtime / device error */
#define PERRK_EUNSUP -3    /* option not implemented on the device path */
#define PERRK_ENUMERIC -4  /* inadmissible state / non-finite direction (reference throws) */
#define PERRK_ECOMM -5     /* NCCL error */

/* numerical flux ids: order of FluxTag, physics.hpp:14 */
#define PERRK_FLUX_CENTRAL 0
#define PERRK_FLUX_UPWIND 1
#define PERRK_FLUX_RUSANOV 2
#define PERRK_FLUX_HLLE 3
#define PERRK_FLUX_HLLC 4
#define PERRK_FLUX_EC 5

/* family kinds: order of FamilyKind, butcher.hpp:28 */
#define PERRK_FAMILY_P2 0
#define PERRK_FAMILY_P3_VARIANT 1
#define PERRK_FAMILY_P3_ORIGINAL 2
#define PERRK_FAMILY_P4 3

typedef struct perrk_ctx perrk_ctx;

/* Replaces SemidiscretizationSpec (semidisc.hpp:24-35) for the periodic
 * rectilinear Euler / Navier-Stokes-Fourier cases of the hot path.
 * dim 2 matches Mesh2DRect (mesh.hpp:22-33); dim 3 is the Mesh3DRect
 * extension the configs need. */
typedef struct {
  int dim;                   /* 2 or 3 */
  int n[3];                  /* cells per axis; n[2] ignored for dim 2 */
  const double* edges[3];    /* n[a]+1 strictly increasing edges per axis */
  int polydeg;               /* only 3 on the device path */
  int physics;               /* 0 Euler (EulerPhysics), 1 NSF with BR1 (dim 2) */
  double gamma;              /* ratio of specific heats (> 1) */
  double mu, prandtl;        /* NSF only */
  int surface_flux;          /* PERRK_FLUX_* */
  int volume_mode;           /* 1 flux differencing, 0 weak form (semidisc.cpp:429-445) */
  int volume_flux;           /* flux differencing: PERRK_FLUX_EC or PERRK_FLUX_CENTRAL
                                (NSF: EC only) */
  int device;                /* CUDA device ordinal */
} perrk_semi_desc;

/* Replaces PartitionFamily (butcher.hpp:36-51): R members sharing b and c,
 * stored with E ascending; member r integrates cells of level R - r
 * (member_index_for_level, butcher.hpp:47). */
typedef struct {
  int kind;                  /* PERRK_FAMILY_* (order bookkeeping only) */
  int S, R;
  const int* E;              /* [R] */
  const double* A;           /* [R][S][S] row-major */
  const double* b;           /* [S] */
  const double* c;           /* [S] */
} perrk_family_desc;

/* Replaces RelaxationConfig (relax.hpp:16-24).  numerics selects the root
 * residual: 0 = the reference's form r = H(U+g dt d) - h_ref - g dH with its
 * stopping rule (relax.cpp:79-104); 1 = the accurate form:
 * compensated reductions, per-node cancellation-free entropy differences,
 * Newton stop on |dg| <= 1e-13 g or stagnation.  Methods: Newton
 * (relax.cpp:51-104), bisection and secant (relax.cpp:105-148). */
typedef struct {
  int method;                /* 0 newton, 1 bisection, 2 secant */
  int max_iter;
  double residual_tol, step_tol, bracket_min, bracket_max;
  int seed_from_previous;
  int numerics;
} perrk_relax_cfg;

/* Replaces PerkStepOptions (stepper.hpp:54-60). */
typedef struct {
  int relax_enabled;         /* 0: opts.relaxation == nullptr */
  perrk_relax_cfg relax;
  double gamma_override;     /* used when relaxation is off */
  double gamma_seed;
  double h_ref;              /* NaN: H(U_n) (step mode) */
  int idt;
} perrk_step_opts;

/* Replaces PerkStepResult + RelaxationOutcome (stepper.hpp:62-68, relax.hpp:26-31). */
typedef struct {
  double gamma;
  int iterations;
  double residual;
  int fell_back;
  double delta_h;
  int aborted, bad_cell, bad_stage;
} perrk_step_result;

/* Replaces IntegratorConfig/TimeControl/CflRamp for the loop of run()
 * (stepper.hpp:13-41).  CFL mode: dt = cfl(t - t0) / nu_max with the ramp
 * cfl(s) = min(cfl_max, cfl0 + (cfl_max - cfl0) s / t_ramp) (stepper.cpp:13-15);
 * dt_or_cfl is cfl_max, and cfl0 == cfl_max (or t_ramp <= 0) is constant. */
typedef struct {
  int fixed_dt;              /* 1: dt fixed (truncated to tf), 0: CFL */
  double dt_or_cfl;          /* fixed dt, or cfl_max */
  double tf;                 /* stop when t >= tf - 1e-12 max(1,|tf|) */
  int relax_enabled;
  perrk_relax_cfg relax;
  int anchor_initial;        /* EntropyAnchor::initial: h_ref = H(U_0) */
  int idt;
  int records;               /* fill the per-step log */
  double cfl0, t_ramp, t0;   /* CflRamp and IntegratorConfig::t0 */
  /* continuing one run() over several perrk_advance calls (stepper.cpp:
   * 144-188 keeps gamma_seed and h0 across the whole loop): carry == 0 starts
   * a run (seed 1, anchor H of the resident state); carry == 1 continues one
   * with the previous call's next seed (fell_back ? 1 : gamma of its last
   * step, stepper.cpp:170) and the run's anchor H(U_0) (stepper.cpp:151) */
  int carry;
  double gamma_seed;
  double h_anchor;
} perrk_run_cfg;

/* One row of the step log; replaces StepRecord (stepper.hpp:43-52). */
typedef struct {
  double t, dt, gamma;
  int newton_iters;
  int fell_back;
  double entropy;
  double invariants[5];
  double delta_h;            /* PerkStepResult::delta_h of the step (stepper.hpp:62-68) */
} perrk_step_record;

/* ---- errors / version -------------------------------------------------- */
const char* perrk_last_error(void);
int perrk_abi_version(void);

/* ---- context: Semidiscretization(spec) (semidisc.cpp:15-73) ------------ */
int perrk_create(const perrk_semi_desc* desc, perrk_ctx** out);
int perrk_destroy(perrk_ctx* ctx);
/* num_dofs/num_nodes/num_cells/num_vars/nodes_per_cell (semidisc.hpp:44-49) */
int perrk_sizes(const perrk_ctx* ctx, int64_t* dofs, int64_t* nodes, int64_t* cells, int* vars,
                int* nodes_per_cell);
/* node_x/node_y/node_measure (semidisc.hpp:56-60); any pointer may be NULL */
int perrk_node_geometry(const perrk_ctx* ctx, double* x, double* y, double* z, double* measure);

/* ---- partition family + level map (perk_step's family/map arguments) --- */
/* effective_level: per cell, 1..R (PartitionMap::effective_level,
 * mesh.hpp:48-54).  Builds the per-stage active cell lists on the device. */
int perrk_set_family(perrk_ctx* ctx, const perrk_family_desc* fam, const int* effective_level);

/* ---- resident state (the product path keeps U in HBM between steps) --- */
int perrk_upload_state(perrk_ctx* ctx, const double* U, size_t n);
int perrk_download_state(perrk_ctx* ctx, double* U, size_t n);
/* device pointer of the resident state (for zero-copy interop); valid until
 * the next perrk_advance, which alternates the state between two buffers when
 * it fuses the relaxation with the update (relax_spec_kernel).  The resident
 * state is in the DEVICE layout, cell-blocked SoA: entry (cell c, node l,
 * variable v) at (c V + v) nodes_per_cell + l.  Host buffers of every other
 * entry point use the reference's canonical layout ((c nodes_per_cell + l) V
 * + v, common.hpp:11-13); upload / download transpose between the two. */
int perrk_state_device_ptr(perrk_ctx* ctx, double** dptr);
int perrk_sync(perrk_ctx* ctx);

/* ---- RHS: Semidiscretization::rhs / rhs_masked (semidisc.cpp:121-138) ---
 * Host buffers.  mask == NULL evaluates every cell.  Cells not flagged in the
 * mask get a zero RHS, as the reference's zero fill (semidisc.cpp:130). */
int perrk_rhs_masked(perrk_ctx* ctx, double t, const double* U, double* out, const char* mask);
/* BR1 auxiliary gradients (semidisc.hpp:75), NSF only: grads[dim][dofs] */
int perrk_br1_gradients(perrk_ctx* ctx, double t, const double* U, double* grads);

/* ---- reductions (semidisc.cpp:561-607, mesh.cpp:97-129) ----------------
 * U == NULL reads the resident state.  Sums are compensated (double-double)
 * and fixed-order, so results are bitwise reproducible run to run. */
int perrk_total_entropy(perrk_ctx* ctx, const double* U, double* out);
int perrk_entropy_inner_product(perrk_ctx* ctx, const double* U, const double* K, double* out);
int perrk_integral_per_variable(perrk_ctx* ctx, const double* U, double* out);
int perrk_admissible(perrk_ctx* ctx, const double* U, int* ok, int* first_bad_cell);
int perrk_characteristic_speed(perrk_ctx* ctx, const double* U, double* nu);
/* compute_dt (stepper.cpp:116-127) with a constant CFL ramp */
int perrk_compute_dt(perrk_ctx* ctx, const double* U, int fixed, double dt_or_cfl, double t,
                     double tf, double* dt);

/* ---- time stepping ------------------------------------------------------
 * perk_step (stepper.cpp:17-114): host U and t updated in place, untouched
 * on a positivity abort. */
int perrk_perk_step(perrk_ctx* ctx, double* U, double* t, double dt, const perrk_step_opts* opts,
                    perrk_step_result* res);
/* the same on the resident state (no host copies) */
int perrk_perk_step_resident(perrk_ctx* ctx, double* t, double dt, const perrk_step_opts* opts,
                             perrk_step_result* res);
/* run() loop body (stepper.cpp:144-188) for up to nsteps steps on the
 * resident state, entirely on the device: compute_dt, perk_step with the
 * gamma-seed carry, StepRecord.  Asynchronous; log (nsteps rows, may be
 * NULL) and *t / *steps_taken / *aborted are valid after perrk_sync(). */
int perrk_advance(perrk_ctx* ctx, const perrk_run_cfg* cfg, double* t, int nsteps,
                  perrk_step_record* log, int* steps_taken, int* aborted);

/* Matrix-free spectrum estimation: the dense probe of
 * specopt.cpp:18-35 needs an M x M Jacobian (guarded to M <= 5000); this
 * runs m steps of Arnoldi (classical Gram-Schmidt applied twice) on the
 * central-difference Jacobian-vector product of the full RHS at `base`
 * (host, NULL: the resident state),
 *   J v = (rhs(u + h v) - rhs(u - h v)) / (2 h),  h = epsilon (1 + max|u|),
 * |v|_2 = 1, entirely on the device; the Krylov basis needs (m + 1) M
 * doubles of device memory.  cell_mask (NULL: every cell) restricts the
 * operator to the flagged cells (v and J v zero elsewhere): a level's own
 * block of the Jacobian.  H receives the (m + 1) x m upper Hessenberg
 * matrix, column-major; the eigenvalues of its leading m_done x m_done block
 * are the Ritz values (m_done < m: an invariant subspace was found, and those
 * Ritz values are eigenvalues of the probed operator). */
int perrk_krylov_hessenberg(perrk_ctx* ctx, const double* base, double t, double epsilon, int m,
                            const char* cell_mask, double* H, int* m_done);

/* probe_jacobian (specopt.cpp:18-35; declared specopt.hpp:25-26, default
 * epsilon 1e-6): dense central-difference Jacobian of the full RHS at `base`,
 * column j stepped by epsilon*(1+|base_j|), guarded to M <= 5000.  J is the
 * M x M matrix in column-major order (Eigen's MatrixXd storage):
 * J[j*M + i] = (rhs_i(u + h_j e_j) - rhs_i(u - h_j e_j)) / (2 h_j).  The
 * columns are probed in colours: one local DOF of a distance-2 independent
 * set of cells per RHS pair, so 2 * n_colours * nodes*V RHS evaluations
 * replace the reference's 2M, and each entry equals the single-column probe
 * bit for bit.  n_colours (may be NULL) receives the number of cell colours. */
int perrk_probe_jacobian(perrk_ctx* ctx, const double* base, double t, double epsilon, double* J,
                         int* n_colours);

/* error_norms (stepper.cpp:195-265): L1 (domain-normalised) and Linf of the
 * DG solution interpolated to the degree-2k GLL points against an exact
 * solution; exact = 0: the 2D isentropic vortex (isentropic_vortex_state,
 * physics.cpp:301-328) with params = {gamma, mach, radius, intensity,
 * rho_inf, v_inf_x, v_inf_y, half_width} at time t.  U == NULL: resident. */
int perrk_error_norms(perrk_ctx* ctx, const double* U, int exact, const double* params, double t,
                      double* l1, double* linf);

/* scalar RHS evaluation counter (semidisc.hpp:81-82): n_active*nodes*V per
 * evaluated stage */
int perrk_rhs_cell_evaluations(const perrk_ctx* ctx, uint64_t* out);
int perrk_reset_counter(perrk_ctx* ctx);

/* ---- host-side helpers of the same library (no device work) -------------
 * build_family (butcher.cpp:237-247): free_flat holds the members' free
 * subdiagonals back to back in E order.  A: [R][S][S], active: [R][S]. */
int perrk_family_build(int kind, int S, int R, const int* E, const double* free_flat,
                       double c_sm3, double* A, double* b, double* c, int* active);
/* assign_levels (mesh.cpp:73-95) */
int perrk_assign_levels(const double* nu, int64_t n, int R, int* levels);
/* make_partition_map (mesh.cpp:56-71) on a periodic rectilinear mesh, dim 1-3 */
int perrk_make_partition_map(int dim, const int* ncells, const int* levels, int R, int* effective);

/* ---- instrumentation (bench.py / profiling; no reference counterpart) ---
 * set_stream: order the context's work on a caller stream (e.g. torch's
 * current stream, so CUDA events recorded there bracket it); NULL restores a
 * private stream.  profile: start (1, resets) / stop (0) recording an event
 * pair around every stage-kernel launch; profile_read returns their summed
 * device time, count and compulsory bytes.  launch_count: kernels launched
 * by the context so far.  step_traffic: compulsory HBM bytes of one step's
 * stage launches, of one relaxation pass and of the final update.
 * fp64_peak: DFMA-loop FP64 throughput of the device (GFLOP/s). */
int perrk_set_stream(perrk_ctx* ctx, void* cuda_stream);
int perrk_profile(perrk_ctx* ctx, int enable);
int perrk_profile_read(perrk_ctx* ctx, double* stage_ms, int64_t* stage_launches,
                       double* stage_bytes);
int perrk_launch_count(const perrk_ctx* ctx, int64_t* launches);
int perrk_step_traffic(const perrk_ctx* ctx, double* stage_bytes, double* pass_bytes,
                       double* update_bytes);
int perrk_fp64_peak(int device, double* gflops);

/* ---- linear advection: the update matrix of one step --------------------
 * Replaces analysis::assemble_update_matrix (analysis.cpp:11-32): for every
 * unit vector e_j, perk_step (stepper.cpp:17-114) with relaxation off and
 * gamma fixed, on AdvectionPhysics (physics.hpp:54-85) over a periodic 1D
 * mesh (Mesh1D) or a periodic 2D rectilinear mesh.  All M = cells * 4^dim
 * columns advance together on the device, in column chunks sized to free
 * memory.  D is written column-major: D(i, j) = D[j * M + i] (Eigen's layout
 * of UpdateMatrix::D).  HLLE/HLLC surface fluxes are rejected as in the
 * reference (physics.cpp:73-78). */
typedef struct {
  int dim;                   /* 1 or 2 */
  int n[2];                  /* cells per axis */
  const double* edges[2];    /* n[a]+1 strictly increasing edges per axis */
  double velocity[2];        /* AdvectionPhysics velocity */
  int surface_flux;          /* PERRK_FLUX_CENTRAL / _UPWIND / _RUSANOV / _EC */
  int volume_mode;           /* 1 flux differencing, 0 weak form */
  int volume_flux;           /* flux differencing: PERRK_FLUX_CENTRAL or _EC */
  int device;
} perrk_advection_desc;
/* M: out, number of dofs (D has M*M entries); D may be NULL to query M. */
int perrk_update_matrix(const perrk_advection_desc* desc, const perrk_family_desc* fam,
                        const int* effective_level, double dt, double gamma, double* D,
                        int64_t* M);

/* ---- multi-GPU: element partition ------------------------
 * No reference counterpart (the reference is single-process).  Every global
 * cell is owned by one rank (one process per GPU); `owner` is the global
 * ownership map (global cell id -> rank, the reference's cell order; NULL:
 * uniform slabs of last-axis cell layers).  Per stage each rank packs the
 * formed stage traces of its faces that border another rank and exchanges
 * them with those peers (grouped ncclSend/ncclRecv on a comm stream while the
 * interior cells run); the reductions (dH, the Newton residual/derivative,
 * max |d|, the CFL speed, H and invariants) are per-rank double-double
 * partials all-gathered and summed in rank order.
 *
 * nccl_id: the 128-byte ncclUniqueId from perrk_nccl_id on rank 0 (broadcast
 * by the caller, e.g. through torch.distributed).  Call before
 * perrk_set_family; afterwards upload/download/geometry refer to the rank's
 * cells in ascending global id (perrk_local_cells), while perrk_set_family
 * still takes the GLOBAL effective-level array and positivity reports carry
 * global cell ids.  nranks == 1 is a no-op. */
int perrk_nccl_id(void* nccl_id_out);
int perrk_comm_init(perrk_ctx* ctx, const void* nccl_id, int rank, int nranks,
                    const int* owner);
/* the context's cells (global ids, ascending); gids may be NULL to query n */
int perrk_local_cells(const perrk_ctx* ctx, int* gids, int64_t* n);
/* Test harness for the multi-rank logic on ONE device: the n contexts (same
 * global mesh) become ranks 0..n-1 of a group sharing one stream; the halo
 * and the gathers are stream-ordered device copies.  perrk_advance /
 * perrk_perk_step_resident / perrk_compute_dt(U = NULL) on any member then
 * step every member. */
int perrk_loopback_group(perrk_ctx** ctxs, int n, const int* owner);
/* Host helpers (no device work).
 * perrk_partition_slabs: contiguous last-axis layers balanced by per-cell
 *   work (NULL: uniform).
 * perrk_partition_levels: every level's cells cut into nranks equal runs in
 *   global order, so each rank holds 1/nranks of every level and every P-ERK
 *   stage is balanced (the stage loop synchronises ranks once per stage).
 * perrk_halo_plan: the plan perrk_comm_init builds for `rank`.  counts[4] =
 *   {local cells, ghost traces, sent traces, peers}; any array may be NULL
 *   (call once with NULLs for the sizes).  gid[local]; nbr[local*2dim + f] =
 *   local neighbour or -1-ghost slot; ghost_gid[slot] = the neighbour's
 *   global id; peers ascending; a peer k's ghost slots are
 *   [recv_off[k], recv_off[k+1]) and the traces we send it are the
 *   (local cell, face) pairs send[2 j], send[2 j + 1] for j in
 *   [send_off[k], send_off[k+1]).  Both sides order a peer's traces by the
 *   sender's (global cell, face).
 * perrk_face_nodes: cell-local node index of trace point pt of face f
 *   (2 d + side), the point order of the exchanged traces. */
int perrk_partition_slabs(int dim, const int* n, const double* cell_work, int nranks, int* owner);
int perrk_partition_levels(int dim, const int* n, const int* level, int nlevels, int nranks,
                           int* owner);
int perrk_halo_plan(int dim, const int* n, const int* owner, int rank, int64_t* counts, int* gid,
                    int* nbr, int64_t* ghost_gid, int* peers, int64_t* recv_off,
                    int64_t* send_off, int* send);
int perrk_face_nodes(int dim, int face, int* nodes);

#ifdef __cplusplus
}
#endif
#endif
