// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// C-ABI shim over the UNMODIFIED reference C++ library (compiled from
// /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/).  Only
// tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline leg
// may load it, and only as the checker / the timed reference arm.
//
// Every entry point forwards to the reference API without changing its
// numerics:
//   Semidiscretization        proj/core/include/perrk/semidisc.hpp:40-113
//   perk_step / compute_dt    proj/core/src/stepper.cpp:17-127
//   solve_relaxation          proj/core/src/relax.cpp:51-151
//   build_* families          proj/core/src/butcher.cpp:51-247
//   make_partition_map etc.   proj/core/src/mesh.cpp:56-129
#include <chrono>
#include <cmath>
#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "perrk/basis.hpp"
#include "perrk/butcher.hpp"
#include "perrk/mesh.hpp"
#include "perrk/physics.hpp"
#include "perrk/relax.hpp"
#include "perrk/semidisc.hpp"
#include "perrk/stepper.hpp"

using namespace perrk;

namespace {
thread_local std::string g_err;

FluxTag tag_of(int id) {
  switch (id) {
    case 0: return FluxTag::central;
    case 1: return FluxTag::upwind;
    case 2: return FluxTag::rusanov;
    case 3: return FluxTag::hlle;
    case 4: return FluxTag::hllc;
    case 5: return FluxTag::ec;
  }
  throw Error("bad flux id");
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
}  // namespace

struct ref_ctx {
  std::unique_ptr<Semidiscretization> semi;
};

struct ref_family {
  int S, R, kind;
  const int* E;
  const double* A;  // R*S*S row-major, member r = index in E (ascending)
  const double* b;
  const double* c;
};

struct ref_relax {
  int method;  // 0 newton, 1 bisection, 2 secant
  int max_iter;
  double residual_tol, step_tol, bracket_min, bracket_max;
  int seed_from_previous;
};

struct ref_step_result {
  double gamma;
  int iterations;
  double residual;
  int fell_back;
  double delta_h;
  int aborted, bad_cell, bad_stage;
};

static PartitionFamily make_family(const ref_family* f) {
  PartitionFamily fam;
  fam.kind = static_cast<FamilyKind>(f->kind);
  fam.order = family_order(fam.kind);
  fam.S = f->S;
  fam.R = f->R;
  for (int r = 0; r < f->R; ++r) {
    fam.E.push_back(f->E[r]);
    ButcherTableau t;
    t.S = f->S;
    t.A.assign(f->A + static_cast<std::size_t>(r) * f->S * f->S,
               f->A + static_cast<std::size_t>(r + 1) * f->S * f->S);
    t.b.assign(f->b, f->b + f->S);
    t.c.assign(f->c, f->c + f->S);
    fam.members.push_back(t);
    fam.active_sets.push_back(active_stage_set(fam.members.back()));
  }
  return fam;
}

static RelaxationConfig make_relax(const ref_relax* r) {
  RelaxationConfig c;
  c.method = static_cast<RelaxMethod>(r->method);
  c.max_iter = r->max_iter;
  c.residual_tol = r->residual_tol;
  c.step_tol = r->step_tol;
  c.bracket_min = r->bracket_min;
  c.bracket_max = r->bracket_max;
  c.seed_from_previous = r->seed_from_previous != 0;
  return c;
}

static PartitionMap make_map(const Semidiscretization& semi, const int* eff, int R) {
  PartitionMap map;
  map.R = R;
  map.effective_level.assign(eff, eff + semi.num_cells());
  map.raw_level = map.effective_level;
  return map;
}

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// physics: 0 euler(dim,gamma), 1 advection(vel[dim])
ref_ctx* ref_create(int dim, const double* xe, int nxe, const double* ye, int nye, int k,
                    int physics, double gamma, const double* adv_vel, int surface_flux,
                    int volume_mode, int volume_flux) {
  ref_ctx* ctx = nullptr;
  int rc = guarded([&] {
    SemidiscretizationSpec spec;
    if (dim == 1) {
      Mesh1D m;
      m.edges.assign(xe, xe + nxe);
      m.periodic = true;
      spec.mesh = m;
    } else {
      Mesh2DRect m;
      m.x_edges.assign(xe, xe + nxe);
      m.y_edges.assign(ye, ye + nye);
      spec.mesh = m;
    }
    spec.polydeg = k;
    if (physics == 0)
      spec.physics = std::make_shared<EulerPhysics>(dim, gamma);
    else
      spec.physics = std::make_shared<AdvectionPhysics>(std::vector<double>(adv_vel, adv_vel + dim));
    spec.surface_flux = tag_of(surface_flux);
    spec.volume_mode = volume_mode ? VolumeMode::flux_differencing : VolumeMode::weak;
    spec.volume_flux = tag_of(volume_flux);
    ctx = new ref_ctx{std::make_unique<Semidiscretization>(std::move(spec))};
  });
  return rc ? nullptr : ctx;
}

// 1D compressible Navier-Stokes-Fourier with BR1 (NSFPhysics, physics.hpp:127-146;
// the reference's only viscous path, semidisc.cpp:245-395), periodic
ref_ctx* ref_create_nsf1d(const double* xe, int nxe, int k, double gamma, double mu,
                          double prandtl, int surface_flux, int volume_mode, int volume_flux) {
  ref_ctx* ctx = nullptr;
  int rc = guarded([&] {
    SemidiscretizationSpec spec;
    Mesh1D m;
    m.edges.assign(xe, xe + nxe);
    m.periodic = true;
    spec.mesh = m;
    spec.polydeg = k;
    spec.physics = std::make_shared<NSFPhysics>(gamma, mu, prandtl);
    spec.viscous = true;
    spec.surface_flux = tag_of(surface_flux);
    spec.volume_mode = volume_mode ? VolumeMode::flux_differencing : VolumeMode::weak;
    spec.volume_flux = tag_of(volume_flux);
    ctx = new ref_ctx{std::make_unique<Semidiscretization>(std::move(spec))};
  });
  return rc ? nullptr : ctx;
}

void ref_destroy(ref_ctx* ctx) { delete ctx; }
int ref_num_dofs(ref_ctx* ctx) { return ctx->semi->num_dofs(); }
int ref_num_cells(ref_ctx* ctx) { return ctx->semi->num_cells(); }
void ref_set_threads(ref_ctx* ctx, int n) { ctx->semi->set_threads(n); }
unsigned long long ref_rhs_cell_evaluations(ref_ctx* ctx) {
  return ctx->semi->rhs_cell_evaluations();
}
void ref_reset_counter(ref_ctx* ctx) { ctx->semi->reset_evaluation_counter(); }

void ref_node_coords(ref_ctx* ctx, double* x, double* y, double* measure) {
  const auto& s = *ctx->semi;
  const std::size_t n = s.node_measure().size();
  std::memcpy(x, s.node_x().data(), n * sizeof(double));
  if (y && s.dim() == 2) std::memcpy(y, s.node_y().data(), n * sizeof(double));
  std::memcpy(measure, s.node_measure().data(), n * sizeof(double));
}

int ref_rhs_masked(ref_ctx* ctx, double t, const double* U, double* out, const char* mask) {
  return guarded([&] {
    const auto& s = *ctx->semi;
    StateVector u(U, U + s.num_dofs()), o;
    if (mask) {
      std::vector<char> m(mask, mask + s.num_cells());
      s.rhs_masked(t, u, o, m);
    } else {
      s.rhs(t, u, o);
    }
    std::memcpy(out, o.data(), o.size() * sizeof(double));
  });
}

double ref_total_entropy(ref_ctx* ctx, const double* U) {
  const auto& s = *ctx->semi;
  return s.total_entropy(StateVector(U, U + s.num_dofs()));
}

double ref_entropy_inner_product(ref_ctx* ctx, const double* U, const double* K) {
  const auto& s = *ctx->semi;
  return s.entropy_inner_product(StateVector(U, U + s.num_dofs()),
                                 StateVector(K, K + s.num_dofs()));
}

void ref_integral_per_variable(ref_ctx* ctx, const double* U, double* out) {
  const auto& s = *ctx->semi;
  const auto v = s.integral_per_variable(StateVector(U, U + s.num_dofs()));
  std::memcpy(out, v.data(), v.size() * sizeof(double));
}

int ref_admissible(ref_ctx* ctx, const double* U, int* first_bad) {
  const auto& s = *ctx->semi;
  int bad = -1;
  const bool ok = s.admissible(StateVector(U, U + s.num_dofs()), &bad);
  if (first_bad) *first_bad = bad;
  return ok ? 1 : 0;
}

int ref_characteristic_speed(ref_ctx* ctx, const double* U, double* nu) {
  return guarded([&] {
    const auto& s = *ctx->semi;
    const auto v = characteristic_speed(s.mesh(), s.physics(), StateVector(U, U + s.num_dofs()),
                                        s.basis().k);
    std::memcpy(nu, v.data(), v.size() * sizeof(double));
  });
}

// params: gamma, mach, radius, intensity, rho_inf, vx_inf, vy_inf, half_width
int ref_project_vortex(ref_ctx* ctx, const double* p, double t, double* U) {
  return guarded([&] {
    VortexParams vp;
    vp.gamma = p[0];
    vp.mach = p[1];
    vp.radius = p[2];
    vp.intensity = p[3];
    vp.rho_inf = p[4];
    vp.v_inf = {p[5], p[6]};
    vp.half_width = p[7];
    const auto u = ctx->semi->project(
        [&](double x, double y, double* out) { isentropic_vortex_state(vp, x, y, t, out); });
    std::memcpy(U, u.data(), u.size() * sizeof(double));
  });
}

// error_norms (stepper.cpp:195-265) against the isentropic vortex
int ref_error_norms_vortex(ref_ctx* ctx, const double* U, const double* p, double t, double* l1,
                           double* linf) {
  return guarded([&] {
    VortexParams vp;
    vp.gamma = p[0];
    vp.mach = p[1];
    vp.radius = p[2];
    vp.intensity = p[3];
    vp.rho_inf = p[4];
    vp.v_inf[0] = p[5];
    vp.v_inf[1] = p[6];
    vp.half_width = p[7];
    const auto& s = *ctx->semi;
    StateVector u(U, U + s.num_dofs());
    const auto e = error_norms(
        u, [&](double x, double y, double tt, double* out) { isentropic_vortex_state(vp, x, y, tt, out); },
        t, s);
    std::memcpy(l1, e.l1.data(), sizeof(double) * e.l1.size());
    std::memcpy(linf, e.linf.data(), sizeof(double) * e.linf.size());
  });
}

// the reference's CSV writers (stepper.cpp:267-301, semidisc.cpp:609-632);
// rows: [step, t, dt, gamma, iters, H, fell_back, invariants...]
int ref_write_step_log(ref_ctx* ctx, int n, const double* rows, const char* path) {
  return guarded([&] {
    const int V = ctx->semi->num_vars();
    std::vector<StepRecord> log(n);
    for (int k = 0; k < n; ++k) {
      const double* r = rows + static_cast<std::size_t>(k) * (7 + V);
      log[k].step = static_cast<int>(r[0]);
      log[k].t = r[1];
      log[k].dt = r[2];
      log[k].gamma = r[3];
      log[k].newton_iters = static_cast<int>(r[4]);
      log[k].entropy = r[5];
      log[k].fell_back = r[6] != 0.0;
      log[k].invariants.assign(r + 7, r + 7 + V);
    }
    write_step_log_csv(log, *ctx->semi, path);
  });
}

int ref_write_snapshot(ref_ctx* ctx, const double* U, const char* path) {
  return guarded([&] {
    StateVector u(U, U + ctx->semi->num_dofs());
    write_snapshot_csv(*ctx->semi, u, path);
  });
}

// ---- basis / physics pins ------------------------------------------------
void ref_gll(int k, double* nodes, double* weights, double* D) {
  const auto b = gll_basis(k);
  std::memcpy(nodes, b.nodes.data(), b.nodes.size() * sizeof(double));
  std::memcpy(weights, b.weights.data(), b.weights.size() * sizeof(double));
  std::memcpy(D, b.D.data(), b.D.size() * sizeof(double));
}

double ref_logmean(double a, double b) { return logmean(a, b); }

int ref_numerical_flux(int dim, double gamma, int tag, const double* ul, const double* ur, int dir,
                       double* f) {
  return guarded([&] {
    EulerPhysics e(dim, gamma);
    e.numerical_flux(tag_of(tag), ul, ur, dir, f);
  });
}

int ref_physics_eval(int dim, double gamma, const double* u, int dir, double* f, double* w,
                     double* s, double* lam) {
  return guarded([&] {
    EulerPhysics e(dim, gamma);
    e.flux(u, dir, f);
    e.entropy_variables(u, w);
    *s = e.entropy(u);
    *lam = e.max_wave_speed(u, dir);
  });
}

// ---- families / partitions -------------------------------------------------
// free_flat holds the members' free subdiagonals back to back (ascending E).
int ref_family_build(int kind, int S, int R, const int* E, const double* free_flat,
                     double c_sm3, double* A, double* b, double* c, int* active) {
  return guarded([&] {
    std::vector<int> El(E, E + R);
    std::vector<std::vector<double>> fr;
    std::size_t off = 0;
    for (int r = 0; r < R; ++r) {
      const int n = free_coefficient_count(static_cast<FamilyKind>(kind), E[r]);
      fr.emplace_back(free_flat + off, free_flat + off + n);
      off += n;
    }
    const auto fam = build_family(static_cast<FamilyKind>(kind), S, El, fr, c_sm3);
    for (int r = 0; r < R; ++r) {
      std::memcpy(A + static_cast<std::size_t>(r) * S * S, fam.members[r].A.data(),
                  sizeof(double) * S * S);
      for (int i = 0; i < S; ++i) active[r * S + i] = fam.active_sets[r].count(i) ? 1 : 0;
    }
    std::memcpy(b, fam.members[0].b.data(), sizeof(double) * S);
    std::memcpy(c, fam.members[0].c.data(), sizeof(double) * S);
  });
}

int ref_family_to_text(const ref_family* f, char* buf, int cap) {
  return guarded([&] {
    const std::string s = family_to_text(make_family(f));
    PERRK_REQUIRE(static_cast<int>(s.size()) < cap, "buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

int ref_assign_levels(const double* nu, int n, int R, int* levels) {
  return guarded([&] {
    const auto l = assign_levels(std::vector<double>(nu, nu + n), R);
    std::memcpy(levels, l.data(), sizeof(int) * n);
  });
}

int ref_make_partition_map(ref_ctx* ctx, const int* levels, int R, int* eff) {
  return guarded([&] {
    const auto& s = *ctx->semi;
    const auto m = make_partition_map(s.mesh(), std::vector<int>(levels, levels + s.num_cells()), R);
    std::memcpy(eff, m.effective_level.data(), sizeof(int) * s.num_cells());
  });
}

// ---- stepping ----------------------------------------------------------------
int ref_perk_step(ref_ctx* ctx, double* U, double* t, double dt, const ref_family* f,
                  const int* eff, const ref_relax* relax, double gamma_seed, double h_ref,
                  int idt, double gamma_override, ref_step_result* out) {
  return guarded([&] {
    const auto& s = *ctx->semi;
    const auto fam = make_family(f);
    const auto map = make_map(s, eff, f->R);
    StateVector u(U, U + s.num_dofs());
    RelaxationConfig rc;
    PerkStepOptions opts;
    if (relax) {
      rc = make_relax(relax);
      opts.relaxation = &rc;
    }
    opts.gamma_seed = gamma_seed;
    opts.h_ref = h_ref;
    opts.idt = idt != 0;
    opts.gamma_override = gamma_override;
    const auto r = perk_step(u, *t, dt, fam, map, s, opts);
    std::memcpy(U, u.data(), u.size() * sizeof(double));
    out->gamma = r.outcome.gamma;
    out->iterations = r.outcome.iterations;
    out->residual = r.outcome.residual;
    out->fell_back = r.outcome.fell_back;
    out->delta_h = r.delta_h;
    out->aborted = r.aborted;
    out->bad_cell = r.bad_cell;
    out->bad_stage = r.bad_stage;
  });
}

// analysis::assemble_update_matrix (analysis.cpp:11-32) without its Eigen
// container: column j = perk_step(e_j) with relaxation off and gamma fixed;
// D column-major (D(i, j) = D[j * M + i]).
int ref_update_matrix(ref_ctx* ctx, const ref_family* f, const int* eff, double dt, double gamma,
                      double* D) {
  return guarded([&] {
    const auto& s = *ctx->semi;
    PERRK_REQUIRE(s.physics().name() == "advection", "update matrix needs linear physics");
    const auto fam = make_family(f);
    const auto map = make_map(s, eff, f->R);
    const int M = s.num_dofs();
    PerkStepOptions opts;
    opts.relaxation = nullptr;
    opts.gamma_override = gamma;
    StateVector unit(static_cast<std::size_t>(M));
    for (int j = 0; j < M; ++j) {
      std::fill(unit.begin(), unit.end(), 0.0);
      unit[j] = 1.0;
      double t = 0.0;
      perk_step(unit, t, dt, fam, map, s, opts);
      std::memcpy(D + static_cast<std::size_t>(j) * M, unit.data(), sizeof(double) * M);
    }
  });
}

double ref_compute_dt(ref_ctx* ctx, const double* U, int fixed, double dt_or_cfl, double t,
                      double tf) {
  const auto& s = *ctx->semi;
  IntegratorConfig cfg;
  cfg.t0 = 0.0;
  cfg.tf = tf;
  cfg.time.fixed = fixed != 0;
  cfg.time.dt = dt_or_cfl;
  cfg.time.ramp = CflRamp{dt_or_cfl, dt_or_cfl, 1.0};
  double dt = NAN;
  guarded([&] { dt = compute_dt(StateVector(U, U + s.num_dofs()), s, cfg, t); });
  return dt;
}

// Mirrors the loop body of run() (stepper.cpp:144-188) for exactly nsteps
// steps: compute_dt, perk_step with gamma-seed carry, StepRecord H and
// invariants.  log rows: [t, dt, gamma, iters, H, fell_back, inv0..inv{V-1}].
// Returns the number of steps taken (< nsteps on a positivity abort).
int ref_run_steps(ref_ctx* ctx, double* U, double* t, int nsteps, const ref_family* f,
                  const int* eff, const ref_relax* relax, int fixed, double dt_or_cfl, int anchor,
                  int records, double* log, double* seconds) {
  int taken = 0;
  const int rc = guarded([&] {
    const auto& s = *ctx->semi;
    const auto fam = make_family(f);
    const auto map = make_map(s, eff, f->R);
    StateVector u(U, U + s.num_dofs());
    IntegratorConfig cfg;
    cfg.tf = 1e300;
    cfg.time.fixed = fixed != 0;
    cfg.time.dt = dt_or_cfl;
    cfg.time.ramp = CflRamp{dt_or_cfl, dt_or_cfl, 1.0};
    RelaxationConfig rcfg;
    const double h0 = s.total_entropy(u);
    double gamma_seed = 1.0;
    const int V = s.num_vars();
    const auto t0 = std::chrono::steady_clock::now();
    for (int step = 0; step < nsteps; ++step) {
      const double dt = compute_dt(u, s, cfg, *t);
      PerkStepOptions opts;
      if (relax) {
        rcfg = make_relax(relax);
        opts.relaxation = &rcfg;
        opts.gamma_seed = rcfg.seed_from_previous ? gamma_seed : 1.0;
        if (anchor) opts.h_ref = h0;
      }
      const auto r = perk_step(u, *t, dt, fam, map, s, opts);
      if (r.aborted) break;
      gamma_seed = r.outcome.fell_back ? 1.0 : r.outcome.gamma;
      if (records) {
        double* row = log + static_cast<std::size_t>(step) * (6 + V);
        row[0] = *t;
        row[1] = dt;
        row[2] = r.outcome.gamma;
        row[3] = r.outcome.iterations;
        row[4] = s.total_entropy(u);
        row[5] = r.outcome.fell_back;
        const auto inv = s.integral_per_variable(u);
        for (int v = 0; v < V; ++v) row[6 + v] = inv[v];
      }
      ++taken;
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::memcpy(U, u.data(), u.size() * sizeof(double));
  });
  return rc ? -1 : taken;
}

}  // extern "C"
