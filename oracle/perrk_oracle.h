/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * CPU restatement ("oracle") of the reference's hot path, in plain C.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference leg
 * may load it, and only as the checker.  The product path
 * (paper_2507_04991_b200/) never links or calls it.
 *
 * What it restates (reference file:line in each function's comment):
 *   - GLL basis                      proj/core/src/basis.cpp:35-84
 *   - Euler physics + fluxes         proj/core/src/physics.cpp:30-258
 *   - DGSEM RHS (weak / flux diff.)  proj/core/src/semidisc.cpp:409-557
 *   - reductions                     proj/core/src/semidisc.cpp:561-607
 *   - characteristic speed           proj/core/src/mesh.cpp:97-129
 *   - perk_step / compute_dt         proj/core/src/stepper.cpp:17-127
 *   - solve_relaxation               proj/core/src/relax.cpp:51-151
 * Extensions the reference does not contain (labelled "oracle extension"):
 *   - dim = 3 (Mesh3DRect, 5 variables, z line family and z faces), built
 *     by the reference's own tensor-product structure;
 *   - 2D compressible Navier-Stokes-Fourier with BR1 lifting, the 2D analogue
 *     of semidisc.cpp:245-395 and physics.cpp:260-273;
 *   - "accurate" relaxation numerics: compensated
 *     sums, per-node cancellation-free entropy differences, step-based Newton
 *     stop.  numerics = 0 reproduces relax.cpp exactly.
 *
 * Parity pin: for dim = 2 the restatement performs the reference's floating
 * point operations in the reference's order (the reference is built with
 * -ffp-contract=off, and so is this file), so against oracle/_ref it is
 * expected to agree bit for bit; tests/test_oracle.py checks that.
 */
#ifndef PERRK_ORACLE_H
#define PERRK_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_CENTRAL = 0, ORC_UPWIND = 1, ORC_RUSANOV = 2, ORC_HLLE = 3, ORC_HLLC = 4, ORC_EC = 5 };

typedef struct orc_semi orc_semi;

typedef struct {
  int dim;                    /* 2 or 3 */
  int nx, ny, nz;             /* cells per axis (nz ignored for dim 2) */
  const double *xe, *ye, *ze; /* nx+1, ny+1, nz+1 edges; periodic */
  int k;                      /* polynomial degree */
  double gamma;
  int viscous;                /* 2D only: NSF + BR1 */
  double mu, prandtl;
  int surface_flux;
  int volume_mode;            /* 0 weak, 1 flux differencing */
  int volume_flux;
  int threads;                /* volume-loop threads, as Semidiscretization::set_threads */
} orc_spec;

typedef struct {
  int S, R;
  const int* E;      /* R, ascending; member r <-> level R - r */
  const double* A;   /* R*S*S row-major */
  const double* b;   /* S */
  const double* c;   /* S */
} orc_family;

typedef struct {
  int method;        /* 0 newton, 1 bisection, 2 secant */
  int max_iter;
  double residual_tol, step_tol, bracket_min, bracket_max;
  int seed_from_previous;
  int numerics;      /* 0 reference (relax.cpp), 1 accurate (H1) */
} orc_relax;

typedef struct {
  double gamma;
  int iterations;
  double residual;
  int fell_back;
  double delta_h;
  int aborted, bad_cell, bad_stage;
} orc_step_result;

const char* orc_last_error(void);

orc_semi* orc_create(const orc_spec* spec);
void orc_destroy(orc_semi* s);
int64_t orc_num_dofs(const orc_semi* s);
int64_t orc_num_cells(const orc_semi* s);
int orc_num_vars(const orc_semi* s);
int orc_nodes_per_cell(const orc_semi* s);
void orc_set_threads(orc_semi* s, int threads);
uint64_t orc_rhs_cell_evaluations(const orc_semi* s);
void orc_reset_counter(orc_semi* s);
void orc_node_coords(const orc_semi* s, double* x, double* y, double* z, double* measure);

int orc_rhs_masked(orc_semi* s, double t, const double* U, double* out, const char* mask);
int orc_br1_gradients(orc_semi* s, double t, const double* U, double* grads);

double orc_total_entropy(const orc_semi* s, const double* U);
/* the same as a compensated (Kahan-Babuska) sum, for the accurate numerics */
double orc_total_entropy_acc(const orc_semi* s, const double* U);
double orc_entropy_inner_product(const orc_semi* s, const double* U, const double* K);
void orc_integral_per_variable(const orc_semi* s, const double* U, double* out);
int orc_admissible(const orc_semi* s, const double* U, int* first_bad_cell);
void orc_characteristic_speed(const orc_semi* s, const double* U, double* nu);
double orc_compute_dt(const orc_semi* s, const double* U, int fixed, double dt_or_cfl, double t,
                      double tf);

int orc_perk_step(orc_semi* s, double* U, double* t, double dt, const orc_family* fam,
                  const int* eff_level, const orc_relax* relax, double gamma_seed, double h_ref,
                  int idt, double gamma_override, orc_step_result* out);
int orc_run_steps(orc_semi* s, double* U, double* t, int nsteps, const orc_family* fam,
                  const int* eff_level, const orc_relax* relax, int fixed, double dt_or_cfl,
                  int anchor, int records, double* log, double* seconds);

/* pointwise pins */
void orc_gll(int k, double* nodes, double* weights, double* D);
double orc_logmean(double a, double b);
int orc_numerical_flux(int dim, double gamma, int tag, const double* ul, const double* ur, int dir,
                       double* f);
void orc_physics_eval(int dim, double gamma, const double* u, int dir, double* f, double* w,
                      double* s, double* lam);
double orc_entropy_difference(int dim, double gamma, const double* u, const double* delta);

#ifdef __cplusplus
}
#endif
#endif
