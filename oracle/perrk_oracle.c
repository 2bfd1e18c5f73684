/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.  See perrk_oracle.h for scope.
 *
 * Plain-C restatement of the reference hot path.  Each function names the
 * reference lines it follows.  Expressions keep the reference's evaluation
 * order (left-to-right, no contraction) so that dim=2 results can be checked
 * bit for bit against the compiled reference (oracle/_ref).
 */
#define _GNU_SOURCE
#include "perrk_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define MAXV 5
#define MAXN1 16

static __thread char g_err[256];

static void set_err(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}

const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------ */
/* GLL basis — basis.cpp:8-84                                                */
/* ------------------------------------------------------------------------ */

static void legendre_and_derivative(int k, double x, double* p, double* dp) {
  double pm1 = 1.0, pm0 = x;
  if (k == 0) {
    *p = 1.0;
    *dp = 0.0;
    return;
  }
  for (int n = 1; n < k; ++n) {
    const double pn = ((2.0 * n + 1.0) * x * pm0 - n * pm1) / (n + 1.0);
    pm1 = pm0;
    pm0 = pn;
  }
  *p = pm0;
  *dp = k * (pm1 - x * pm0) / (1.0 - x * x);
}

static double legendre(int k, double x) {
  double p, dp;
  if (fabs(x) == 1.0) return (x > 0 || k % 2 == 0) ? 1.0 : -1.0;
  legendre_and_derivative(k, x, &p, &dp);
  return p;
}

void orc_gll(int k, double* nodes, double* weights, double* D) {
  const int n = k + 1;
  for (int i = 0; i < n; ++i) nodes[i] = 0.0;
  nodes[0] = -1.0;
  nodes[k] = 1.0;
  for (int i = 1; i < k; ++i) {
    double x = -cos(M_PI * i / k);
    for (int iter = 0; iter < 100; ++iter) {
      double p, dp;
      legendre_and_derivative(k, x, &p, &dp);
      const double ddp = (2.0 * x * dp - k * (k + 1.0) * p) / (1.0 - x * x);
      const double step = dp / ddp;
      x -= step;
      if (fabs(step) < 1e-15) break;
    }
    nodes[i] = x;
  }
  for (int i = 0; i < n / 2; ++i) {
    const double v = 0.5 * (nodes[n - 1 - i] - nodes[i]);
    nodes[i] = -v;
    nodes[n - 1 - i] = v;
  }
  if (n % 2 == 1) nodes[n / 2] = 0.0;
  double pk[MAXN1];
  for (int i = 0; i < n; ++i) {
    pk[i] = legendre(k, nodes[i]);
    weights[i] = 2.0 / (k * (k + 1.0) * pk[i] * pk[i]);
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      D[i * n + j] = (i == j) ? 0.0 : pk[i] / (pk[j] * (nodes[i] - nodes[j]));
  D[0] = -k * (k + 1.0) / 4.0;
  D[n * n - 1] = k * (k + 1.0) / 4.0;
}

/* ------------------------------------------------------------------------ */
/* Euler physics — physics.cpp:30-258 (dim generalised to 3: oracle ext.)    */
/* ------------------------------------------------------------------------ */

typedef struct {
  int dim, V;
  double gamma;
  double mu, prandtl;
} phys_t;

/* physics.cpp:30-38 */
double orc_logmean(double a, double b) {
  const double f = (a - b) / (a + b);
  const double u = f * f;
  if (u < 1e-4) return 0.5 * (a + b) / (1.0 + u / 3.0 + u * u / 5.0 + u * u * u / 7.0);
  return (a - b) / log(a / b);
}

/* physics.cpp:97-102 */
static double pressure(const phys_t* P, const double* u) {
  double kinetic = 0.0;
  for (int d = 0; d < P->dim; ++d) kinetic += u[1 + d] * u[1 + d];
  kinetic /= (2.0 * u[0]);
  return (P->gamma - 1.0) * (u[P->dim + 1] - kinetic);
}

/* physics.cpp:104-106 */
static double sound_speed(const phys_t* P, const double* u) {
  return sqrt(P->gamma * pressure(P, u) / u[0]);
}

/* physics.cpp:108-116 */
static void flux(const phys_t* P, const double* u, int dir, double* f) {
  const double rho = u[0];
  const double p = pressure(P, u);
  const double vdir = u[1 + dir] / rho;
  f[0] = u[1 + dir];
  for (int d = 0; d < P->dim; ++d) f[1 + d] = u[1 + d] * vdir;
  f[1 + dir] += p;
  f[P->dim + 1] = (u[P->dim + 1] + p) * vdir;
}

/* physics.cpp:118-120 */
static double max_wave_speed(const phys_t* P, const double* u, int dir) {
  return fabs(u[1 + dir] / u[0]) + sound_speed(P, u);
}

/* physics.cpp:122-128 */
static int admissible(const phys_t* P, const double* u) {
  if (!(u[0] > 0.0)) return 0;
  if (!(pressure(P, u) > 0.0)) return 0;
  for (int v = 0; v < P->V; ++v)
    if (!isfinite(u[v])) return 0;
  return 1;
}

/* physics.cpp:130-132 */
static double entropy(const phys_t* P, const double* u) {
  return -u[0] * log(pressure(P, u) / pow(u[0], P->gamma));
}

/* physics.cpp:134-146 */
static void entropy_variables(const phys_t* P, const double* u, double* w) {
  const double g = P->gamma;
  const double rho = u[0];
  const double p = pressure(P, u);
  const double s_therm = log(p / pow(rho, g));
  double v2 = 0.0;
  for (int d = 0; d < P->dim; ++d) {
    const double vd = u[1 + d] / rho;
    v2 += vd * vd;
    w[1 + d] = (g - 1.0) * rho * vd / p;
  }
  w[0] = g - s_therm - (g - 1.0) * rho * v2 / (2.0 * p);
  w[P->dim + 1] = -(g - 1.0) * rho / p;
}

/* physics.cpp:157-179 (v arrays widened to 3 components) */
static void ec_flux(const phys_t* P, const double* ul, const double* ur, int dir, double* f) {
  const int dim = P->dim;
  const double rho_l = ul[0], rho_r = ur[0];
  const double p_l = pressure(P, ul), p_r = pressure(P, ur);
  const double rho_log = orc_logmean(rho_l, rho_r);
  const double inv_rho_p_log = orc_logmean(rho_l / p_l, rho_r / p_r);
  double v_l[3] = {0, 0, 0}, v_r[3] = {0, 0, 0}, v_avg[3] = {0, 0, 0};
  double vl_vr = 0.0;
  for (int d = 0; d < dim; ++d) {
    v_l[d] = ul[1 + d] / rho_l;
    v_r[d] = ur[1 + d] / rho_r;
    v_avg[d] = 0.5 * (v_l[d] + v_r[d]);
    vl_vr += v_l[d] * v_r[d];
  }
  const double p_avg = 0.5 * (p_l + p_r);
  const double f_rho = rho_log * v_avg[dir];
  f[0] = f_rho;
  for (int d = 0; d < dim; ++d) f[1 + d] = f_rho * v_avg[d];
  f[1 + dir] += p_avg;
  f[dim + 1] = f_rho * (0.5 * vl_vr + 1.0 / ((P->gamma - 1.0) * inv_rho_p_log)) +
               0.5 * (p_l * v_r[dir] + p_r * v_l[dir]);
}

/* physics.cpp:181-203 */
static void wave_speed_estimates(const phys_t* P, const double* ul, const double* ur, int dir,
                                 double* sl, double* sr) {
  const int dim = P->dim;
  const double rho_l = ul[0], rho_r = ur[0];
  const double vl = ul[1 + dir] / rho_l, vr = ur[1 + dir] / rho_r;
  const double cl = sound_speed(P, ul), cr = sound_speed(P, ur);
  const double sql = sqrt(rho_l), sqr = sqrt(rho_r);
  const double p_l = pressure(P, ul), p_r = pressure(P, ur);
  const double hl = (ul[dim + 1] + p_l) / rho_l;
  const double hr = (ur[dim + 1] + p_r) / rho_r;
  double v_roe2 = 0.0, v_roe_dir = 0.0;
  for (int d = 0; d < dim; ++d) {
    const double vroe = (sql * ul[1 + d] / rho_l + sqr * ur[1 + d] / rho_r) / (sql + sqr);
    v_roe2 += vroe * vroe;
    if (d == dir) v_roe_dir = vroe;
  }
  const double h_roe = (sql * hl + sqr * hr) / (sql + sqr);
  const double arg = (P->gamma - 1.0) * (h_roe - 0.5 * v_roe2);
  const double c_roe = sqrt(arg < 0.0 ? 0.0 : arg); /* std::max(0.0, arg) */
  const double a = vl - cl, b = v_roe_dir - c_roe;
  *sl = (b < a) ? b : a; /* std::min */
  const double c = vr + cr, e = v_roe_dir + c_roe;
  *sr = (c < e) ? e : c; /* std::max */
}

/* physics.cpp:205-220 */
static void hlle_flux(const phys_t* P, const double* ul, const double* ur, int dir, double* f) {
  double sl, sr, fl[MAXV], fr[MAXV];
  wave_speed_estimates(P, ul, ur, dir, &sl, &sr);
  flux(P, ul, dir, fl);
  flux(P, ur, dir, fr);
  if (sl >= 0.0) {
    memcpy(f, fl, sizeof(double) * P->V);
  } else if (sr <= 0.0) {
    memcpy(f, fr, sizeof(double) * P->V);
  } else {
    for (int v = 0; v < P->V; ++v)
      f[v] = (sr * fl[v] - sl * fr[v] + sl * sr * (ur[v] - ul[v])) / (sr - sl);
  }
}

/* physics.cpp:222-258 */
static void hllc_flux(const phys_t* P, const double* ul, const double* ur, int dir, double* f) {
  const int dim = P->dim, V = P->V;
  double sl, sr, fk[MAXV], ustar[MAXV];
  wave_speed_estimates(P, ul, ur, dir, &sl, &sr);
  if (sl >= 0.0) {
    flux(P, ul, dir, f);
    return;
  }
  if (sr <= 0.0) {
    flux(P, ur, dir, f);
    return;
  }
  const double rho_l = ul[0], rho_r = ur[0];
  const double vl = ul[1 + dir] / rho_l, vr = ur[1 + dir] / rho_r;
  const double p_l = pressure(P, ul), p_r = pressure(P, ur);
  const double s_star = (p_r - p_l + rho_l * vl * (sl - vl) - rho_r * vr * (sr - vr)) /
                        (rho_l * (sl - vl) - rho_r * (sr - vr));
  const int left = s_star >= 0.0;
  const double* uk = left ? ul : ur;
  const double sk = left ? sl : sr;
  const double vk = left ? vl : vr;
  const double pk = left ? p_l : p_r;
  const double rho_k = uk[0];
  const double factor = rho_k * (sk - vk) / (sk - s_star);
  ustar[0] = factor;
  for (int d = 0; d < dim; ++d) ustar[1 + d] = factor * (d == dir ? s_star : uk[1 + d] / rho_k);
  ustar[dim + 1] =
      factor * (uk[dim + 1] / rho_k + (s_star - vk) * (s_star + pk / (rho_k * (sk - vk))));
  flux(P, uk, dir, fk);
  for (int v = 0; v < V; ++v) f[v] = fk[v] + sk * (ustar[v] - uk[v]);
}

/* physics.cpp:40-65 — returns 0 on success, -1 on inadmissible input (the
 * reference throws perrk::Error there). */
static int numerical_flux(const phys_t* P, int tag, const double* ul, const double* ur, int dir,
                          double* f) {
  if (!(admissible(P, ul) && admissible(P, ur))) {
    set_err("inadmissible state passed to numerical flux");
    return -1;
  }
  const int V = P->V;
  double fl[MAXV], fr[MAXV];
  switch (tag) {
    case ORC_CENTRAL:
      flux(P, ul, dir, fl);
      flux(P, ur, dir, fr);
      for (int v = 0; v < V; ++v) f[v] = 0.5 * (fl[v] + fr[v]);
      return 0;
    case ORC_RUSANOV: {
      flux(P, ul, dir, fl);
      flux(P, ur, dir, fr);
      const double a = max_wave_speed(P, ul, dir), b = max_wave_speed(P, ur, dir);
      const double lam = (a < b) ? b : a; /* std::max */
      for (int v = 0; v < V; ++v) f[v] = 0.5 * (fl[v] + fr[v]) - 0.5 * lam * (ur[v] - ul[v]);
      return 0;
    }
    case ORC_EC: ec_flux(P, ul, ur, dir, f); return 0;
    case ORC_HLLE: hlle_flux(P, ul, ur, dir, f); return 0;
    case ORC_HLLC: hllc_flux(P, ul, ur, dir, f); return 0;
  }
  set_err("flux not available for Euler physics");
  return -1;
}

/* 2D Navier-Stokes-Fourier viscous flux — oracle extension.  2D analogue of
 * NSFPhysics::viscous_flux (physics.cpp:260-273): Stokes stress with
 * lambda = -2/3 mu, Fourier heat flux q = -kappa grad T, T = p/rho,
 * kappa = gamma/(gamma-1) mu/Pr (physics.hpp:140).  grad is direction-major
 * (physics.hpp:17-18): grad[0..V) = d/dx, grad[V..2V) = d/dy. */
static void viscous_flux_2d(const phys_t* P, const double* u, const double* grad, int dir,
                            double* f) {
  const int V = P->V;
  const double g = P->gamma, mu = P->mu;
  const double kappa = g / (g - 1.0) * mu / P->prandtl;
  const double rho = u[0];
  const double vx = u[1] / rho, vy = u[2] / rho;
  const double* gx = grad;
  const double* gy = grad + V;
  const double vx_x = (gx[1] - vx * gx[0]) / rho, vy_x = (gx[2] - vy * gx[0]) / rho;
  const double vx_y = (gy[1] - vx * gy[0]) / rho, vy_y = (gy[2] - vy * gy[0]) / rho;
  const double t_x = (g - 1.0) * (gx[3] / rho - u[3] * gx[0] / (rho * rho) - (vx * vx_x + vy * vy_x));
  const double t_y = (g - 1.0) * (gy[3] / rho - u[3] * gy[0] / (rho * rho) - (vx * vx_y + vy * vy_y));
  const double tau_xx = mu * (4.0 / 3.0 * vx_x - 2.0 / 3.0 * vy_y);
  const double tau_yy = mu * (4.0 / 3.0 * vy_y - 2.0 / 3.0 * vx_x);
  const double tau_xy = mu * (vx_y + vy_x);
  f[0] = 0.0;
  if (dir == 0) {
    const double q = -kappa * t_x;
    f[1] = tau_xx;
    f[2] = tau_xy;
    f[3] = vx * tau_xx + vy * tau_xy - q;
  } else {
    const double q = -kappa * t_y;
    f[1] = tau_xy;
    f[2] = tau_yy;
    f[3] = vx * tau_xy + vy * tau_yy - q;
  }
}

int orc_numerical_flux(int dim, double gamma, int tag, const double* ul, const double* ur, int dir,
                       double* f) {
  phys_t P = {dim, dim + 2, gamma, 0.0, 1.0};
  return numerical_flux(&P, tag, ul, ur, dir, f);
}

void orc_physics_eval(int dim, double gamma, const double* u, int dir, double* f, double* w,
                      double* s, double* lam) {
  phys_t P = {dim, dim + 2, gamma, 0.0, 1.0};
  flux(&P, u, dir, f);
  entropy_variables(&P, u, w);
  *s = entropy(&P, u);
  *lam = max_wave_speed(&P, u, dir);
}

/* ------------------------------------------------------------------------ */
/* Compensated arithmetic for the accurate relaxation numerics (H1)          */
/* ------------------------------------------------------------------------ */

typedef struct {
  double s, c;
} ksum_t;

static inline void kadd(ksum_t* a, double x) { /* Neumaier */
  const double t = a->s + x;
  if (fabs(a->s) >= fabs(x))
    a->c += (a->s - t) + x;
  else
    a->c += (x - t) + a->s;
  a->s = t;
}
static inline double kval(ksum_t a) { return a.s + a.c; }
/* a += x*y with the product's rounding error kept */
static inline void kaddprod(ksum_t* a, double x, double y) {
  const double p = x * y;
  const double e = fma(x, y, -p);
  kadd(a, p);
  kadd(a, e);
}

/* s(U + delta) - s(U) without forming U + delta:
 *   dkin = (rho (2 m.dm + |dm|^2) - drho |m|^2) / (2 rho (rho + drho))
 *   dp   = (gamma-1)(dE - dkin)
 *   ds   = -drho ln(p_T / rho_T^gamma) - rho [log1p(dp/p) - gamma log1p(drho/rho)] */
static double entropy_difference(const phys_t* P, const double* u, const double* du) {
  const int dim = P->dim;
  const double g = P->gamma;
  const double rho = u[0], drho = du[0];
  double mdm = 0.0, dm2 = 0.0, m2 = 0.0;
  for (int d = 0; d < dim; ++d) {
    mdm += u[1 + d] * du[1 + d];
    dm2 += du[1 + d] * du[1 + d];
    m2 += u[1 + d] * u[1 + d];
  }
  const double rho_t = rho + drho;
  const double dkin = (rho * (2.0 * mdm + dm2) - drho * m2) / (2.0 * rho * rho_t);
  const double p = pressure(P, u);
  const double dp = (g - 1.0) * (du[dim + 1] - dkin);
  const double p_t = p + dp;
  return -drho * (log(p_t) - g * log(rho_t)) - rho * (log1p(dp / p) - g * log1p(drho / rho));
}

double orc_entropy_difference(int dim, double gamma, const double* u, const double* delta) {
  phys_t P = {dim, dim + 2, gamma, 0.0, 1.0};
  return entropy_difference(&P, u, delta);
}

/* ------------------------------------------------------------------------ */
/* Semidiscretization — semidisc.cpp:15-73 (+ 3D extension)                  */
/* ------------------------------------------------------------------------ */

struct orc_semi {
  phys_t P;
  int dim, k, n1, npc; /* npc = nodes per cell */
  int nc[3];           /* cells per axis (nc[2] = 1 in 2D) */
  int64_t ncells, nnodes;
  double* edges[3];
  double nodes[MAXN1], w[MAXN1], D[MAXN1 * MAXN1];
  double* measure;
  int surface_flux, volume_mode, volume_flux, viscous;
  int threads;
  uint64_t evals;
};

static inline double hsz(const orc_semi* s, int axis, int i) {
  return s->edges[axis][i + 1] - s->edges[axis][i];
}

orc_semi* orc_create(const orc_spec* sp) {
  if (sp->dim != 2 && sp->dim != 3) {
    set_err("oracle supports dim 2 and 3");
    return NULL;
  }
  if (sp->k < 1 || sp->k + 1 > MAXN1) {
    set_err("polydeg out of range");
    return NULL;
  }
  if (sp->viscous && sp->dim != 2) {
    set_err("viscous terms implemented in 2D");
    return NULL;
  }
  if (sp->volume_mode == 1 && sp->volume_flux != ORC_CENTRAL && sp->volume_flux != ORC_EC) {
    set_err("flux differencing needs a symmetric consistent volume flux");
    return NULL;
  }
  orc_semi* s = calloc(1, sizeof *s);
  s->dim = sp->dim;
  s->P.dim = sp->dim;
  s->P.V = sp->dim + 2;
  s->P.gamma = sp->gamma;
  s->P.mu = sp->mu;
  s->P.prandtl = sp->prandtl;
  s->k = sp->k;
  s->n1 = sp->k + 1;
  s->npc = sp->dim == 2 ? s->n1 * s->n1 : s->n1 * s->n1 * s->n1;
  s->nc[0] = sp->nx;
  s->nc[1] = sp->ny;
  s->nc[2] = sp->dim == 3 ? sp->nz : 1;
  const double* e[3] = {sp->xe, sp->ye, sp->ze};
  for (int a = 0; a < sp->dim; ++a) {
    s->edges[a] = malloc(sizeof(double) * (s->nc[a] + 1));
    memcpy(s->edges[a], e[a], sizeof(double) * (s->nc[a] + 1));
    for (int i = 0; i < s->nc[a]; ++i)
      if (!(hsz(s, a, i) > 0.0)) {
        set_err("cell sizes must be positive");
        orc_destroy(s);
        return NULL;
      }
  }
  s->ncells = (int64_t)s->nc[0] * s->nc[1] * s->nc[2];
  s->nnodes = s->ncells * s->npc;
  orc_gll(s->k, s->nodes, s->w, s->D);
  s->surface_flux = sp->surface_flux;
  s->volume_mode = sp->volume_mode;
  s->volume_flux = sp->volume_flux;
  s->viscous = sp->viscous;
  s->threads = sp->threads < 1 ? 1 : sp->threads;
  s->measure = malloc(sizeof(double) * s->nnodes);
  const int n1 = s->n1;
  /* semidisc.cpp:56-69: measure = (hx hy / 4) w_ix w_iy; 3D: (hx hy hz / 8) w w w */
  for (int64_t cell = 0; cell < s->ncells; ++cell) {
    const int ci = (int)(cell % s->nc[0]);
    const int cj = (int)((cell / s->nc[0]) % s->nc[1]);
    const int ck = (int)(cell / ((int64_t)s->nc[0] * s->nc[1]));
    const double hx = hsz(s, 0, ci), hy = hsz(s, 1, cj);
    for (int l = 0; l < s->npc; ++l) {
      const int ix = l % n1, iy = (l / n1) % n1, iz = l / (n1 * n1);
      double m;
      if (s->dim == 2)
        m = 0.25 * hx * hy * s->w[ix] * s->w[iy];
      else
        m = 0.125 * hx * hy * hsz(s, 2, ck) * s->w[ix] * s->w[iy] * s->w[iz];
      s->measure[cell * s->npc + l] = m;
    }
  }
  return s;
}

void orc_destroy(orc_semi* s) {
  if (!s) return;
  for (int a = 0; a < 3; ++a) free(s->edges[a]);
  free(s->measure);
  free(s);
}

int64_t orc_num_dofs(const orc_semi* s) { return s->nnodes * s->P.V; }
int64_t orc_num_cells(const orc_semi* s) { return s->ncells; }
int orc_num_vars(const orc_semi* s) { return s->P.V; }
int orc_nodes_per_cell(const orc_semi* s) { return s->npc; }
void orc_set_threads(orc_semi* s, int threads) { s->threads = threads < 1 ? 1 : threads; }
uint64_t orc_rhs_cell_evaluations(const orc_semi* s) { return s->evals; }
void orc_reset_counter(orc_semi* s) { s->evals = 0; }

void orc_node_coords(const orc_semi* s, double* x, double* y, double* z, double* measure) {
  const int n1 = s->n1;
  for (int64_t cell = 0; cell < s->ncells; ++cell) {
    const int ci = (int)(cell % s->nc[0]);
    const int cj = (int)((cell / s->nc[0]) % s->nc[1]);
    const int ck = (int)(cell / ((int64_t)s->nc[0] * s->nc[1]));
    for (int l = 0; l < s->npc; ++l) {
      const int ix = l % n1, iy = (l / n1) % n1, iz = l / (n1 * n1);
      const int64_t n = cell * s->npc + l;
      if (x) x[n] = s->edges[0][ci] + 0.5 * hsz(s, 0, ci) * (s->nodes[ix] + 1.0);
      if (y) y[n] = s->edges[1][cj] + 0.5 * hsz(s, 1, cj) * (s->nodes[iy] + 1.0);
      if (z && s->dim == 3) z[n] = s->edges[2][ck] + 0.5 * hsz(s, 2, ck) * (s->nodes[iz] + 1.0);
      if (measure) measure[n] = s->measure[n];
    }
  }
}

/* node offset (in doubles) of local node (ix,iy,iz) of a cell */
static inline int64_t nidx(const orc_semi* s, int64_t cell, int ix, int iy, int iz) {
  const int n1 = s->n1;
  return (cell * s->npc + ix + n1 * (iy + n1 * iz)) * s->P.V;
}

static inline int64_t cell_id(const orc_semi* s, int ci, int cj, int ck) {
  return ci + (int64_t)s->nc[0] * (cj + (int64_t)s->nc[1] * ck);
}

/* ---- volume term of one cell: semidisc.cpp:425-485 ---------------------- */
static int volume_cell(const orc_semi* s, const double* U, double* out, int64_t cell) {
  const phys_t* P = &s->P;
  const int V = P->V, n1 = s->n1, dim = s->dim;
  const int ci = (int)(cell % s->nc[0]);
  const int cj = (int)((cell / s->nc[0]) % s->nc[1]);
  const int ck = (int)(cell / ((int64_t)s->nc[0] * s->nc[1]));
  const double jac[3] = {2.0 / hsz(s, 0, ci), 2.0 / hsz(s, 1, cj),
                         dim == 3 ? 2.0 / hsz(s, 2, ck) : 0.0};
  const int nz = dim == 3 ? n1 : 1;
  double fv[MAXV];
  if (s->volume_mode == 0) {
    /* weak form, semidisc.cpp:429-445 */
    double* f = malloc(sizeof(double) * s->npc * V);
    for (int dirn = 0; dirn < dim; ++dirn) {
      const double J = jac[dirn];
      for (int l = 0; l < s->npc; ++l) flux(P, &U[cell * s->npc * V + l * V], dirn, &f[l * V]);
      for (int iz = 0; iz < nz; ++iz)
        for (int iy = 0; iy < n1; ++iy)
          for (int ix = 0; ix < n1; ++ix) {
            double* o = &out[nidx(s, cell, ix, iy, iz)];
            const int l = dirn == 0 ? ix : (dirn == 1 ? iy : iz);
            for (int mm = 0; mm < n1; ++mm) {
              const double coef = J * s->D[mm * n1 + l] * s->w[mm] / s->w[l];
              const int src = dirn == 0 ? (mm + n1 * (iy + n1 * iz))
                                        : (dirn == 1 ? (ix + n1 * (mm + n1 * iz))
                                                     : (ix + n1 * (iy + n1 * mm)));
              for (int v = 0; v < V; ++v) o[v] += coef * f[src * V + v];
            }
          }
    }
    free(f);
    return 0;
  }
  /* flux differencing: one line family per direction, in x, y, z order */
  for (int dirn = 0; dirn < dim; ++dirn) {
    const double J = jac[dirn];
    for (int a = 0; a < nz; ++a)       /* outer transverse index */
      for (int bq = 0; bq < n1; ++bq) { /* inner transverse index */
        for (int l = 0; l < n1; ++l) {
          int il[3];
          if (dirn == 0) { il[0] = l; il[1] = bq; il[2] = a; }
          else if (dirn == 1) { il[0] = bq; il[1] = l; il[2] = a; }
          else { il[0] = bq; il[1] = a; il[2] = l; }
          const int64_t nl = nidx(s, cell, il[0], il[1], dim == 3 ? il[2] : 0);
          const double dll = s->D[l * n1 + l];
          if (dll != 0.0) {
            flux(P, &U[nl], dirn, fv);
            for (int v = 0; v < V; ++v) out[nl + v] -= J * 2.0 * dll * fv[v];
          }
          for (int mm = l + 1; mm < n1; ++mm) {
            int im[3] = {il[0], il[1], il[2]};
            im[dirn] = mm;
            const int64_t nm = nidx(s, cell, im[0], im[1], dim == 3 ? im[2] : 0);
            if (numerical_flux(P, s->volume_flux, &U[nl], &U[nm], dirn, fv)) return -1;
            const double clm = J * 2.0 * s->D[l * n1 + mm];
            const double cml = J * 2.0 * s->D[mm * n1 + l];
            for (int v = 0; v < V; ++v) {
              out[nl + v] -= clm * fv[v];
              out[nm + v] -= cml * fv[v];
            }
          }
        }
      }
  }
  return 0;
}

typedef struct {
  const orc_semi* s;
  const double* U;
  double* out;
  const char* mask;
  int64_t lo, hi;
  int rc;
} vol_job;

static void* vol_worker(void* arg) {
  vol_job* j = arg;
  for (int64_t c = j->lo; c < j->hi; ++c)
    if (j->mask[c] && volume_cell(j->s, j->U, j->out, c)) {
      j->rc = -1;
      return NULL;
    }
  return NULL;
}

/* parallel_cells, semidisc.cpp:75-89 */
static int volume_all(const orc_semi* s, const double* U, double* out, const char* mask) {
  const int T = s->threads;
  if (T <= 1 || s->ncells < 2 * T) {
    vol_job j = {s, U, out, mask, 0, s->ncells, 0};
    vol_worker(&j);
    return j.rc;
  }
  pthread_t th[256];
  vol_job jobs[256];
  const int64_t chunk = (s->ncells + T - 1) / T;
  int nt = 0;
  for (int t = 0; t < T && t < 256; ++t) {
    const int64_t lo = t * chunk;
    const int64_t hi = lo + chunk < s->ncells ? lo + chunk : s->ncells;
    if (lo >= hi) break;
    jobs[nt] = (vol_job){s, U, out, mask, lo, hi, 0};
    pthread_create(&th[nt], NULL, vol_worker, &jobs[nt]);
    ++nt;
  }
  int rc = 0;
  for (int t = 0; t < nt; ++t) {
    pthread_join(th[t], NULL);
    rc |= jobs[t].rc;
  }
  return rc;
}

/* ---- surface pass: semidisc.cpp:489-556, one face family per direction --- */
static int faces_all(const orc_semi* s, const double* U, double* out, const char* mask) {
  const phys_t* P = &s->P;
  const int V = P->V, n1 = s->n1, dim = s->dim;
  const int fluxdiff = s->volume_mode == 1;
  const double w0 = s->w[0];
  double fstar[MAXV], ftrace[MAXV];
  const int nz = dim == 3 ? n1 : 1;
  for (int dirn = 0; dirn < dim; ++dirn) {
    const int nd = s->nc[dirn];
    for (int ck = 0; ck < s->nc[2]; ++ck)
      for (int cj = 0; cj < s->nc[1]; ++cj)
        for (int ci = 0; ci < s->nc[0]; ++ci) {
          int cidx[3] = {ci, cj, ck};
          const int64_t cr = cell_id(s, ci, cj, ck);
          int cl_idx[3] = {ci, cj, ck};
          cl_idx[dirn] = (cidx[dirn] + nd - 1) % nd;
          const int64_t cl = cell_id(s, cl_idx[0], cl_idx[1], cl_idx[2]);
          if (!mask[cl] && !mask[cr]) continue;
          for (int a = 0; a < nz; ++a)
            for (int bq = 0; bq < n1; ++bq) {
              int il[3], ir[3];
              if (dirn == 0) { il[0] = n1 - 1; il[1] = bq; il[2] = a; }
              else if (dirn == 1) { il[0] = bq; il[1] = n1 - 1; il[2] = a; }
              else { il[0] = bq; il[1] = a; il[2] = n1 - 1; }
              memcpy(ir, il, sizeof il);
              ir[dirn] = 0;
              const int64_t nl = nidx(s, cl, il[0], il[1], dim == 3 ? il[2] : 0);
              const int64_t nr = nidx(s, cr, ir[0], ir[1], dim == 3 ? ir[2] : 0);
              const double* ul = &U[nl];
              const double* ur = &U[nr];
              if (numerical_flux(P, s->surface_flux, ul, ur, dirn, fstar)) return -1;
              if (mask[cl]) {
                const double coef = 2.0 / (hsz(s, dirn, cl_idx[dirn]) * w0) * 1.0;
                double* o = &out[nl];
                if (fluxdiff) {
                  flux(P, ul, dirn, ftrace);
                  for (int v = 0; v < V; ++v) o[v] -= coef * (fstar[v] - ftrace[v]);
                } else {
                  for (int v = 0; v < V; ++v) o[v] -= coef * fstar[v];
                }
              }
              if (mask[cr]) {
                const double coef = 2.0 / (hsz(s, dirn, cidx[dirn]) * w0);
                double* o = &out[nr];
                if (fluxdiff) {
                  flux(P, ur, dirn, ftrace);
                  for (int v = 0; v < V; ++v) o[v] += coef * (fstar[v] - ftrace[v]);
                } else {
                  for (int v = 0; v < V; ++v) o[v] += coef * fstar[v];
                }
              }
            }
        }
  }
  return 0;
}

/* ---- 2D BR1 (oracle extension; 2D analogue of semidisc.cpp:245-395) ------ */

/* face neighbours of cell c in 2D periodic (left, right, bottom, top) */
static void neighbours_2d(const orc_semi* s, int64_t c, int64_t nb[4]) {
  const int nx = s->nc[0], ny = s->nc[1];
  const int ci = (int)(c % nx), cj = (int)(c / nx);
  nb[0] = cell_id(s, (ci + nx - 1) % nx, cj, 0);
  nb[1] = cell_id(s, (ci + 1) % nx, cj, 0);
  nb[2] = cell_id(s, ci, (cj + ny - 1) % ny, 0);
  nb[3] = cell_id(s, ci, (cj + 1) % ny, 0);
}

/* gradients_1d (semidisc.cpp:245-319) per direction; grad has dim*nnodes*V
 * entries, direction-major: grad[dir][node][v]. */
static void gradients_2d(const orc_semi* s, const double* U, double* grad, const char* mask) {
  const int V = s->P.V, n1 = s->n1;
  const int64_t N = s->nnodes * V;
  memset(grad, 0, sizeof(double) * 2 * N);
  char* gmask = malloc(s->ncells);
  memcpy(gmask, mask, s->ncells);
  for (int64_t c = 0; c < s->ncells; ++c)
    if (mask[c]) {
      int64_t nb[4];
      neighbours_2d(s, c, nb);
      for (int q = 0; q < 4; ++q) gmask[nb[q]] = 1;
    }
  for (int64_t c = 0; c < s->ncells; ++c) {
    if (!gmask[c]) continue;
    const int ci = (int)(c % s->nc[0]), cj = (int)(c / s->nc[0]);
    for (int dirn = 0; dirn < 2; ++dirn) {
      const double jac = 2.0 / hsz(s, dirn, dirn == 0 ? ci : cj);
      double* G = grad + dirn * N;
      for (int b = 0; b < n1; ++b)
        for (int l = 0; l < n1; ++l) {
          const int64_t nl = dirn == 0 ? nidx(s, c, l, b, 0) : nidx(s, c, b, l, 0);
          double* g = &G[nl];
          for (int m = 0; m < n1; ++m) {
            const int64_t nm = dirn == 0 ? nidx(s, c, m, b, 0) : nidx(s, c, b, m, 0);
            const double coef = jac * s->D[l * n1 + m];
            for (int v = 0; v < V; ++v) g[v] += coef * U[nm + v];
          }
        }
    }
  }
  const double w0 = s->w[0];
  double ustar[MAXV];
  for (int dirn = 0; dirn < 2; ++dirn) {
    double* G = grad + dirn * N;
    const int nd = s->nc[dirn];
    for (int cj = 0; cj < s->nc[1]; ++cj)
      for (int ci = 0; ci < s->nc[0]; ++ci) {
        int idx[2] = {ci, cj}, lidx[2] = {ci, cj};
        lidx[dirn] = (idx[dirn] + nd - 1) % nd;
        const int64_t cr = cell_id(s, ci, cj, 0), cl = cell_id(s, lidx[0], lidx[1], 0);
        for (int b = 0; b < n1; ++b) {
          const int64_t nl = dirn == 0 ? nidx(s, cl, n1 - 1, b, 0) : nidx(s, cl, b, n1 - 1, 0);
          const int64_t nr = dirn == 0 ? nidx(s, cr, 0, b, 0) : nidx(s, cr, b, 0, 0);
          for (int v = 0; v < V; ++v) ustar[v] = 0.5 * (U[nl + v] + U[nr + v]);
          if (gmask[cl]) {
            const double coef = 2.0 / (hsz(s, dirn, lidx[dirn]) * w0);
            for (int v = 0; v < V; ++v) G[nl + v] += coef * (ustar[v] - U[nl + v]);
          }
          if (gmask[cr]) {
            const double coef = 2.0 / (hsz(s, dirn, idx[dirn]) * w0);
            for (int v = 0; v < V; ++v) G[nr + v] -= coef * (ustar[v] - U[nr + v]);
          }
        }
      }
  }
  free(gmask);
}

/* add_viscous_1d (semidisc.cpp:321-395) per direction */
static void add_viscous_2d(const orc_semi* s, const double* U, const double* grad, double* out,
                           const char* mask) {
  const int V = s->P.V, n1 = s->n1;
  const int64_t N = s->nnodes * V;
  double* G = calloc(2 * N, sizeof(double)); /* viscous flux per direction */
  for (int64_t c = 0; c < s->ncells; ++c) {
    int needed = mask[c];
    if (!needed) {
      int64_t nb[4];
      neighbours_2d(s, c, nb);
      for (int q = 0; q < 4; ++q) needed |= mask[nb[q]];
    }
    if (!needed) continue;
    for (int l = 0; l < s->npc; ++l) {
      const int64_t n = (c * s->npc + l) * V;
      double g[2 * MAXV];
      for (int v = 0; v < V; ++v) {
        g[v] = grad[n + v];
        g[V + v] = grad[N + n + v];
      }
      viscous_flux_2d(&s->P, &U[n], g, 0, &G[n]);
      viscous_flux_2d(&s->P, &U[n], g, 1, &G[N + n]);
    }
  }
  for (int64_t c = 0; c < s->ncells; ++c) {
    if (!mask[c]) continue;
    const int ci = (int)(c % s->nc[0]), cj = (int)(c / s->nc[0]);
    for (int dirn = 0; dirn < 2; ++dirn) {
      const double jac = 2.0 / hsz(s, dirn, dirn == 0 ? ci : cj);
      const double* Gd = G + dirn * N;
      for (int b = 0; b < n1; ++b)
        for (int l = 0; l < n1; ++l) {
          const int64_t nl = dirn == 0 ? nidx(s, c, l, b, 0) : nidx(s, c, b, l, 0);
          double* o = &out[nl];
          for (int m = 0; m < n1; ++m) {
            const int64_t nm = dirn == 0 ? nidx(s, c, m, b, 0) : nidx(s, c, b, m, 0);
            const double coef = jac * s->D[m * n1 + l] * s->w[m] / s->w[l];
            for (int v = 0; v < V; ++v) o[v] -= coef * Gd[nm + v];
          }
        }
    }
  }
  const double w0 = s->w[0];
  double gstar[MAXV];
  for (int dirn = 0; dirn < 2; ++dirn) {
    const double* Gd = G + dirn * N;
    const int nd = s->nc[dirn];
    for (int cj = 0; cj < s->nc[1]; ++cj)
      for (int ci = 0; ci < s->nc[0]; ++ci) {
        int idx[2] = {ci, cj}, lidx[2] = {ci, cj};
        lidx[dirn] = (idx[dirn] + nd - 1) % nd;
        const int64_t cr = cell_id(s, ci, cj, 0), cl = cell_id(s, lidx[0], lidx[1], 0);
        if (!mask[cl] && !mask[cr]) continue;
        for (int b = 0; b < n1; ++b) {
          const int64_t nl = dirn == 0 ? nidx(s, cl, n1 - 1, b, 0) : nidx(s, cl, b, n1 - 1, 0);
          const int64_t nr = dirn == 0 ? nidx(s, cr, 0, b, 0) : nidx(s, cr, b, 0, 0);
          for (int v = 0; v < V; ++v) gstar[v] = 0.5 * (Gd[nl + v] + Gd[nr + v]);
          if (mask[cl]) {
            const double coef = 2.0 / (hsz(s, dirn, lidx[dirn]) * w0);
            for (int v = 0; v < V; ++v) out[nl + v] += coef * gstar[v];
          }
          if (mask[cr]) {
            const double coef = 2.0 / (hsz(s, dirn, idx[dirn]) * w0);
            for (int v = 0; v < V; ++v) out[nr + v] -= coef * gstar[v];
          }
        }
      }
  }
  free(G);
}

/* rhs_masked, semidisc.cpp:126-138 -> rhs_2d 409-557 */
int orc_rhs_masked(orc_semi* s, double t, const double* U, double* out, const char* mask) {
  (void)t; /* the 2D/3D periodic RHS is autonomous (semidisc.cpp:411) */
  const int64_t N = orc_num_dofs(s);
  char* full = NULL;
  if (!mask) {
    full = malloc(s->ncells);
    memset(full, 1, s->ncells);
    mask = full;
  }
  memset(out, 0, sizeof(double) * N);
  int64_t n_eval = 0;
  for (int64_t c = 0; c < s->ncells; ++c) n_eval += mask[c] ? 1 : 0;
  s->evals += (uint64_t)n_eval * s->npc * s->P.V;
  int rc = volume_all(s, U, out, mask);
  if (!rc) rc = faces_all(s, U, out, mask);
  if (!rc && s->viscous) {
    double* grad = malloc(sizeof(double) * 2 * N);
    gradients_2d(s, U, grad, mask);
    add_viscous_2d(s, U, grad, out, mask);
    free(grad);
  }
  free(full);
  return rc;
}

int orc_br1_gradients(orc_semi* s, double t, const double* U, double* grads) {
  (void)t;
  if (s->dim != 2) {
    set_err("BR1 gradients implemented in 2D");
    return -1;
  }
  char* mask = malloc(s->ncells);
  memset(mask, 1, s->ncells);
  gradients_2d(s, U, grads, mask);
  free(mask);
  return 0;
}

/* ---- reductions: semidisc.cpp:561-607 ------------------------------------ */
double orc_total_entropy(const orc_semi* s, const double* U) {
  double h = 0.0;
  for (int64_t n = 0; n < s->nnodes; ++n) h += s->measure[n] * entropy(&s->P, &U[n * s->P.V]);
  return h;
}

double orc_entropy_inner_product(const orc_semi* s, const double* U, const double* K) {
  const int V = s->P.V;
  double w[MAXV], acc = 0.0;
  for (int64_t n = 0; n < s->nnodes; ++n) {
    entropy_variables(&s->P, &U[n * V], w);
    double dot = 0.0;
    for (int v = 0; v < V; ++v) dot += w[v] * K[n * V + v];
    acc += s->measure[n] * dot;
  }
  return acc;
}

void orc_integral_per_variable(const orc_semi* s, const double* U, double* out) {
  const int V = s->P.V;
  for (int v = 0; v < V; ++v) out[v] = 0.0;
  for (int64_t n = 0; n < s->nnodes; ++n)
    for (int v = 0; v < V; ++v) out[v] += s->measure[n] * U[n * V + v];
}

int orc_admissible(const orc_semi* s, const double* U, int* first_bad_cell) {
  for (int64_t c = 0; c < s->ncells; ++c)
    for (int l = 0; l < s->npc; ++l)
      if (!admissible(&s->P, &U[(c * s->npc + l) * s->P.V])) {
        if (first_bad_cell) *first_bad_cell = (int)c;
        return 0;
      }
  return 1;
}

/* compensated variants (accurate relaxation numerics) */
static ksum_t inner_acc(const orc_semi* s, const double* U, const double* K) {
  const int V = s->P.V;
  double w[MAXV];
  ksum_t acc = {0, 0};
  for (int64_t n = 0; n < s->nnodes; ++n) {
    entropy_variables(&s->P, &U[n * V], w);
    double dot = 0.0;
    for (int v = 0; v < V; ++v) dot += w[v] * K[n * V + v];
    kaddprod(&acc, s->measure[n], dot);
  }
  return acc;
}

static ksum_t entropy_acc(const orc_semi* s, const double* U) {
  ksum_t acc = {0, 0};
  for (int64_t n = 0; n < s->nnodes; ++n)
    kaddprod(&acc, s->measure[n], entropy(&s->P, &U[n * s->P.V]));
  return acc;
}

double orc_total_entropy_acc(const orc_semi* s, const double* U) {
  return kval(entropy_acc(s, U));
}

/* mesh.cpp:97-129 (3D: third direction) */
void orc_characteristic_speed(const orc_semi* s, const double* U, double* nu) {
  const int V = s->P.V;
  for (int64_t c = 0; c < s->ncells; ++c) {
    const int ci = (int)(c % s->nc[0]);
    const int cj = (int)((c / s->nc[0]) % s->nc[1]);
    const int ck = (int)(c / ((int64_t)s->nc[0] * s->nc[1]));
    double r[3] = {0, 0, 0};
    for (int l = 0; l < s->npc; ++l) {
      const double* u = &U[(c * s->npc + l) * V];
      for (int d = 0; d < s->dim; ++d) {
        const double lam = max_wave_speed(&s->P, u, d);
        r[d] = (r[d] < lam) ? lam : r[d];
      }
    }
    double m = r[0] / hsz(s, 0, ci);
    const double y = r[1] / hsz(s, 1, cj);
    m = (m < y) ? y : m;
    if (s->dim == 3) {
      const double z = r[2] / hsz(s, 2, ck);
      m = (m < z) ? z : m;
    }
    nu[c] = (s->k + 1) * m;
  }
}

/* stepper.cpp:116-127 with CflRamp{cfl, cfl, 1} */
double orc_compute_dt(const orc_semi* s, const double* U, int fixed, double dt_or_cfl, double t,
                      double tf) {
  if (fixed) return dt_or_cfl < tf - t ? dt_or_cfl : tf - t;
  double* nu = malloc(sizeof(double) * s->ncells);
  orc_characteristic_speed(s, U, nu);
  double nu_max = 0.0;
  for (int64_t c = 0; c < s->ncells; ++c) nu_max = (nu_max < nu[c]) ? nu[c] : nu_max;
  free(nu);
  /* CflRamp{cfl, cfl, 1}(t - t0) == cfl (stepper.cpp:13-15) */
  const double cfl = dt_or_cfl;
  return cfl / nu_max;
}

/* ------------------------------------------------------------------------ */
/* Relaxation — relax.cpp:26-151 (numerics 0) and the H1 variant (1)          */
/* ------------------------------------------------------------------------ */

typedef struct {
  const orc_semi* s;
  const double* U;
  const double* d;
  double dt, h_ref;
  ksum_t dh;    /* accumulated entropy change */
  double* buf;  /* TrialState buffer (numerics 0) */
  double offset; /* H(U_n) - h_ref (numerics 1, anchored mode) */
  int numerics;
} relax_ctx;

static const double* trial(relax_ctx* r, double gamma) {
  const int64_t N = orc_num_dofs(r->s);
  const double c = gamma * r->dt;
  for (int64_t i = 0; i < N; ++i) r->buf[i] = r->U[i] + c * r->d[i];
  return r->buf;
}

/* r(gamma), relax.cpp:39-43 / H1.2 */
static double residual(relax_ctx* r, double gamma) {
  if (r->numerics == 0)
    return orc_total_entropy(r->s, trial(r, gamma)) - r->h_ref - gamma * kval(r->dh);
  const orc_semi* s = r->s;
  const int V = s->P.V;
  const double gdt = gamma * r->dt;
  ksum_t acc = {0, 0};
  double du[MAXV];
  for (int64_t n = 0; n < s->nnodes; ++n) {
    for (int v = 0; v < V; ++v) du[v] = gdt * r->d[n * V + v];
    kaddprod(&acc, s->measure[n], entropy_difference(&s->P, &r->U[n * V], du));
  }
  kadd(&acc, r->offset);
  kaddprod(&acc, -gamma, r->dh.s);
  kaddprod(&acc, -gamma, r->dh.c);
  return kval(acc);
}

/* r'(gamma), relax.cpp:45-49 */
static double derivative(relax_ctx* r, double gamma) {
  const double* T = trial(r, gamma);
  if (r->numerics == 0) return r->dt * orc_entropy_inner_product(r->s, T, r->d) - kval(r->dh);
  ksum_t ip = inner_acc(r->s, T, r->d);
  ksum_t acc = {0, 0};
  kaddprod(&acc, r->dt, ip.s);
  kaddprod(&acc, r->dt, ip.c);
  kadd(&acc, -r->dh.s);
  kadd(&acc, -r->dh.c);
  return kval(acc);
}

static orc_step_result fallback(int iters, double res) {
  orc_step_result fb;
  memset(&fb, 0, sizeof fb);
  fb.gamma = 1.0;
  fb.iterations = iters;
  fb.residual = res;
  fb.fell_back = 1;
  return fb;
}

/* solve_relaxation, relax.cpp:51-151; returns -1 on a non-finite direction
 * (the reference throws there). */
static int solve_relaxation(relax_ctx* r, const orc_relax* cfg, double gamma_seed,
                            orc_step_result* out) {
  const int64_t N = orc_num_dofs(r->s);
  double dmax = 0.0;
  for (int64_t i = 0; i < N; ++i) {
    const double a = fabs(r->d[i]);
    dmax = (dmax < a) ? a : dmax;
  }
  if (!isfinite(dmax)) {
    set_err("non-finite update direction");
    return -1;
  }
  out->gamma = 1.0;
  out->iterations = 0;
  out->residual = 0.0;
  out->fell_back = 0;
  if (dmax == 0.0) return 0;

  if (cfg->method == 0 && r->numerics == 1) {
    /* H1.4: always take >= 1 Newton step from the seed; stop on a relative
     * step below 1e-13 (from the second step on, the iterate is then kept:
     * the correction is noise) or on noise-floor stagnation; fall back on
     * non-finite values, gamma <= 0, or a last correction above 1e-10 gamma
     * at max_iter (not converged). */
    double gamma = cfg->seed_from_previous ? gamma_seed : 1.0;
    double prev = 0.0;
    for (int it = 1; it <= cfg->max_iter; ++it) {
      const double res = residual(r, gamma);
      const double dr = derivative(r, gamma);
      out->iterations = it;
      out->residual = res;
      if (dr == 0.0 || !isfinite(dr) || !isfinite(res)) {
        *out = fallback(it, res);
        return 0;
      }
      const double step = res / dr;
      /* after the first step, a correction below 1e-13 gamma is under the
       * residual's noise floor: the current iterate is kept as the root */
      if (it >= 2 && fabs(step) <= 1e-13 * gamma && gamma > 0.0) {
        out->gamma = gamma;
        return 0;
      }
      gamma -= step;
      if (!isfinite(gamma) || !(gamma > 0.0)) {
        *out = fallback(it, res);
        return 0;
      }
      out->gamma = gamma;
      if (fabs(step) <= 1e-13 * gamma) return 0;
      if (it >= 2 && fabs(step) < 1e-10 * gamma && fabs(step) > 0.5 * fabs(prev)) return 0;
      /* out of iterations: converged only if the last correction is inside
       * the noise band, else the reference's fallback (relax.cpp:104) */
      if (it == cfg->max_iter && fabs(step) > 1e-10 * gamma) {
        *out = fallback(it, res);
        return 0;
      }
      prev = step;
    }
    return 0; /* accepted after max_iter */
  }

  switch (cfg->method) {
    case 0: { /* Newton, relax.cpp:79-104 */
      double gamma = cfg->seed_from_previous ? gamma_seed : 1.0;
      double res = residual(r, gamma);
      for (int it = 1; it <= cfg->max_iter; ++it) {
        out->iterations = it;
        if (fabs(res) <= cfg->residual_tol) {
          out->gamma = gamma;
          out->residual = res;
          out->iterations = it - 1;
          if (!(gamma > 0.0)) *out = fallback(it - 1, res);
          return 0;
        }
        const double dr = derivative(r, gamma);
        if (dr == 0.0 || !isfinite(dr)) {
          *out = fallback(it, res);
          return 0;
        }
        const double step = res / dr;
        gamma -= step;
        if (!isfinite(gamma)) {
          *out = fallback(it, res);
          return 0;
        }
        res = residual(r, gamma);
        if (fabs(res) <= cfg->residual_tol || fabs(step) <= cfg->step_tol) {
          out->gamma = gamma;
          out->residual = res;
          if (!(gamma > 0.0)) *out = fallback(it, res);
          return 0;
        }
      }
      *out = fallback(cfg->max_iter, res);
      return 0;
    }
    case 1: { /* bisection, relax.cpp:105-127 */
      double lo = cfg->bracket_min, hi = cfg->bracket_max;
      double rlo = residual(r, lo), rhi = residual(r, hi);
      if (signbit(rlo) == signbit(rhi)) {
        *out = fallback(0, rlo);
        return 0;
      }
      double mid = 0.5 * (lo + hi), rmid = 0.0;
      for (int it = 1; it <= cfg->max_iter; ++it) {
        mid = 0.5 * (lo + hi);
        rmid = residual(r, mid);
        out->iterations = it;
        if (fabs(rmid) <= cfg->residual_tol || (hi - lo) <= cfg->step_tol) break;
        if (signbit(rmid) == signbit(rlo)) {
          lo = mid;
          rlo = rmid;
        } else {
          hi = mid;
        }
      }
      out->gamma = mid;
      out->residual = rmid;
      if (!(fabs(rmid) <= cfg->residual_tol || (hi - lo) <= cfg->step_tol) || mid <= 0.0)
        *out = fallback(out->iterations, rmid);
      return 0;
    }
    case 2: { /* secant, relax.cpp:128-148 */
      double g0 = cfg->seed_from_previous ? gamma_seed : 1.0;
      double g1 = g0 - 1e-6;
      double r0 = residual(r, g0), r1 = residual(r, g1);
      for (int it = 1; it <= cfg->max_iter; ++it) {
        out->iterations = it;
        if (r1 == r0) {
          *out = fallback(it, r1);
          return 0;
        }
        const double g2 = g1 - r1 * (g1 - g0) / (r1 - r0);
        if (!isfinite(g2)) {
          *out = fallback(it, r1);
          return 0;
        }
        g0 = g1;
        r0 = r1;
        g1 = g2;
        r1 = residual(r, g1);
        if (fabs(r1) <= cfg->residual_tol || fabs(g1 - g0) <= cfg->step_tol) {
          out->gamma = g1;
          out->residual = r1;
          if (!(g1 > 0.0)) *out = fallback(it, r1);
          return 0;
        }
      }
      *out = fallback(cfg->max_iter, r1);
      return 0;
    }
  }
  set_err("unknown relaxation method");
  return -1;
}

/* ------------------------------------------------------------------------ */
/* perk_step — stepper.cpp:17-114                                            */
/* ------------------------------------------------------------------------ */

/* active_stage_set, butcher.cpp:319-332 */
static void active_stage_set(const orc_family* f, int r, char* act) {
  const int S = f->S;
  const double* A = f->A + (size_t)r * S * S;
  memset(act, 0, S);
  act[0] = 1;
  for (int i = 0; i < S; ++i)
    if (f->b[i] != 0.0) act[i] = 1;
  int grew = 1;
  while (grew) {
    grew = 0;
    for (int i = S - 1; i >= 0; --i)
      if (act[i])
        for (int j = 0; j < i; ++j)
          if (A[i * S + j] != 0.0 && !act[j]) {
            act[j] = 1;
            grew = 1;
          }
  }
}

int orc_perk_step(orc_semi* s, double* U, double* t, double dt, const orc_family* fam,
                  const int* eff, const orc_relax* relax, double gamma_seed, double h_ref,
                  int idt, double gamma_override, orc_step_result* result) {
  if (!(dt > 0.0)) {
    set_err("dt must be positive");
    return -1;
  }
  const int S = fam->S, R = fam->R;
  const double* b = fam->b;
  const double* c = fam->c;
  const int64_t M = orc_num_dofs(s);
  const int64_t n_cells = s->ncells;
  const int per_cell = s->npc * s->P.V;
  memset(result, 0, sizeof *result);
  result->gamma = 1.0;
  result->bad_cell = -1;
  result->bad_stage = -1;

  /* active[level-1][i], member index = R - level (butcher.hpp:47) */
  char* active = calloc((size_t)R * S, 1);
  for (int lvl = 1; lvl <= R; ++lvl) active_stage_set(fam, R - lvl, active + (size_t)(lvl - 1) * S);

  int bad_cell = -1;
  if (!orc_admissible(s, U, &bad_cell)) {
    result->aborted = 1;
    result->bad_cell = bad_cell;
    result->bad_stage = 0;
    free(active);
    return 0;
  }

  double* K1 = malloc(sizeof(double) * M);
  double* Kprev = calloc(M, sizeof(double));
  double* Ustage = malloc(sizeof(double) * M);
  double* d = calloc(M, sizeof(double));
  char* mask = calloc(n_cells, 1);
  const int accurate = relax && relax->numerics == 1;
  ksum_t delta_h = {0, 0};
  int rc = 0;

  rc = orc_rhs_masked(s, *t, U, K1, NULL);
  if (!rc && b[0] != 0.0) {
    if (accurate) {
      const ksum_t ip = inner_acc(s, U, K1);
      kaddprod(&delta_h, dt * b[0], ip.s);
      kaddprod(&delta_h, dt * b[0], ip.c);
    } else {
      delta_h.s += dt * b[0] * orc_entropy_inner_product(s, U, K1);
    }
    for (int64_t m = 0; m < M; ++m) d[m] += b[0] * K1[m];
  }

  for (int i = 1; i < S && !rc; ++i) {
    for (int64_t cell = 0; cell < n_cells; ++cell) {
      const int lvl = eff[cell];
      const double* A = fam->A + (size_t)(R - lvl) * S * S;
      const double a1 = A[i * S + 0];
      const double ap = i >= 2 ? A[i * S + i - 1] : 0.0;
      const int64_t base = cell * per_cell;
      if (ap != 0.0) {
        for (int m = 0; m < per_cell; ++m)
          Ustage[base + m] = U[base + m] + dt * (a1 * K1[base + m] + ap * Kprev[base + m]);
      } else {
        for (int m = 0; m < per_cell; ++m) Ustage[base + m] = U[base + m] + dt * a1 * K1[base + m];
      }
    }
    if (!orc_admissible(s, Ustage, &bad_cell)) {
      result->aborted = 1;
      result->bad_cell = bad_cell;
      result->bad_stage = i;
      goto done;
    }
    for (int64_t cell = 0; cell < n_cells; ++cell)
      mask[cell] = active[(size_t)(eff[cell] - 1) * S + i];
    rc = orc_rhs_masked(s, *t + c[i] * dt, Ustage, Kprev, mask);
    if (!rc && b[i] != 0.0) {
      if (accurate) {
        const ksum_t ip = inner_acc(s, Ustage, Kprev);
        kaddprod(&delta_h, dt * b[i], ip.s);
        kaddprod(&delta_h, dt * b[i], ip.c);
      } else {
        delta_h.s += dt * b[i] * orc_entropy_inner_product(s, Ustage, Kprev);
      }
      for (int64_t m = 0; m < M; ++m) d[m] += b[i] * Kprev[m];
    }
  }
  if (rc) goto done;

  result->delta_h = kval(delta_h);
  double gamma = gamma_override;
  if (relax) {
    relax_ctx rx = {s, U, d, dt, 0.0, delta_h, Ustage, 0.0, relax->numerics};
    if (accurate) {
      rx.offset = isnan(h_ref) ? 0.0 : kval(entropy_acc(s, U)) - h_ref;
    } else {
      rx.h_ref = isnan(h_ref) ? orc_total_entropy(s, U) : h_ref;
    }
    orc_step_result oc;
    rc = solve_relaxation(&rx, relax, gamma_seed, &oc);
    if (rc) goto done;
    result->gamma = oc.gamma;
    result->iterations = oc.iterations;
    result->residual = oc.residual;
    result->fell_back = oc.fell_back;
    gamma = oc.gamma;
  } else {
    result->gamma = gamma;
  }
  {
    const double scale = gamma * dt;
    for (int64_t m = 0; m < M; ++m) U[m] += scale * d[m];
    if (relax && !idt)
      *t += gamma * dt;
    else
      *t += dt;
  }
done:
  free(K1);
  free(Kprev);
  free(Ustage);
  free(d);
  free(mask);
  free(active);
  return rc;
}

/* run() loop body, stepper.cpp:144-188, for exactly nsteps steps; log rows
 * [t, dt, gamma, iters, H, fell_back, inv_0 .. inv_{V-1}, delta_h, H_acc]:
 * delta_h is PerkStepResult::delta_h (stepper.hpp:62-68), H_acc the total
 * entropy as a compensated sum (H is the reference's naive serial sum,
 * semidisc.cpp:561-566) */
int orc_run_steps(orc_semi* s, double* U, double* t, int nsteps, const orc_family* fam,
                  const int* eff, const orc_relax* relax, int fixed, double dt_or_cfl, int anchor,
                  int records, double* log, double* seconds) {
  const int V = s->P.V;
  const double h0 = orc_total_entropy(s, U);
  double gamma_seed = 1.0;
  int taken = 0;
  struct timespec a, b;
  clock_gettime(CLOCK_MONOTONIC, &a);
  for (int step = 0; step < nsteps; ++step) {
    const double dt = orc_compute_dt(s, U, fixed, dt_or_cfl, *t, 1e300);
    orc_step_result r;
    const double seed = relax && relax->seed_from_previous ? gamma_seed : 1.0;
    if (orc_perk_step(s, U, t, dt, fam, eff, relax, seed, anchor ? h0 : NAN, 0, 1.0, &r))
      return -1;
    if (r.aborted) break;
    gamma_seed = r.fell_back ? 1.0 : r.gamma;
    if (records) {
      double* row = log + (size_t)step * (8 + V);
      row[0] = *t;
      row[1] = dt;
      row[2] = r.gamma;
      row[3] = r.iterations;
      row[4] = orc_total_entropy(s, U);
      row[5] = r.fell_back;
      orc_integral_per_variable(s, U, row + 6);
      row[6 + V] = r.delta_h;
      row[7 + V] = kval(entropy_acc(s, U));
    }
    ++taken;
  }
  clock_gettime(CLOCK_MONOTONIC, &b);
  if (seconds) *seconds = (b.tv_sec - a.tv_sec) + 1e-9 * (b.tv_nsec - a.tv_nsec);
  return taken;
}
