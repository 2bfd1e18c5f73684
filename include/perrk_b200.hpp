// perrk_b200.hpp — header-only C++ adapter: the reference's Semidiscretization /
// perk_step API (arxiv/paper_2507_04991, proj/core/include/perrk/) on top of
// the C-ABI in perrk_b200.h.  This is the binding a maintainer of the
// reference adds to switch its hot path to the B200 library: include the
// reference headers first, then this one, and replace
//
//     perrk::Semidiscretization semi(spec);            // semidisc.hpp:40-113
//     perrk::perk_step(U, t, dt, family, map, semi, opts);  // stepper.hpp:72-74
// by
//     perrk_b200::Semidiscretization semi(spec);
//     perrk_b200::perk_step(U, t, dt, family, map, semi, opts);
//
// Same argument meaning, same in-place update of U and t (untouched on a
// positivity abort, stepper.hpp:70-71), same result type, and the same error
// behaviour: precondition violations throw perrk::Error (common.hpp:15-23).
// Without the reference headers the adapter still compiles against plain
// descriptors (perrk_semi_desc / perrk_family_desc) and throws
// perrk_b200::Error.
#ifndef PERRK_B200_HPP
#define PERRK_B200_HPP

#include <cmath>
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <variant>
#include <vector>

#include "perrk_b200.h"

namespace perrk_b200 {

#ifdef PERRK_COMMON_HPP
using ErrorBase = ::perrk::Error;  // reference error type when visible
#else
using ErrorBase = std::runtime_error;
#endif

struct Error : ErrorBase {
  int code;
  Error(int c, const std::string& m) : ErrorBase(m), code(c) {}
};

inline void check(int rc) {
  if (rc != PERRK_OK) throw Error(rc, perrk_last_error());
}

class Semidiscretization {
 public:
  explicit Semidiscretization(const perrk_semi_desc& d) { init(d); }

#ifdef PERRK_SEMIDISC_HPP
  /// From the reference's SemidiscretizationSpec (semidisc.hpp:24-35): a
  /// periodic Mesh2DRect, EulerPhysics (NSFPhysics when viscous), flux tags.
  explicit Semidiscretization(const ::perrk::SemidiscretizationSpec& spec, int device = 0) {
    const auto* rect = std::get_if<::perrk::Mesh2DRect>(&spec.mesh);
    if (!rect) throw Error(PERRK_EUNSUP, "the device path takes periodic 2D/3D rectilinear meshes");
    const auto* euler = dynamic_cast<const ::perrk::EulerPhysics*>(spec.physics.get());
    if (!euler) throw Error(PERRK_EUNSUP, "the device path takes Euler / NSF physics");
    perrk_semi_desc d{};
    d.dim = 2;
    d.n[0] = rect->nx();
    d.n[1] = rect->ny();
    d.edges[0] = rect->x_edges.data();
    d.edges[1] = rect->y_edges.data();
    d.polydeg = spec.polydeg;
    d.physics = spec.viscous ? 1 : 0;
    d.gamma = euler->gamma();
    if (const auto* nsf = dynamic_cast<const ::perrk::NSFPhysics*>(spec.physics.get())) {
      d.mu = nsf->mu();
      d.prandtl = nsf->prandtl();
    }
    d.surface_flux = static_cast<int>(spec.surface_flux);  // FluxTag order == PERRK_FLUX_*
    d.volume_mode = spec.volume_mode == ::perrk::VolumeMode::flux_differencing ? 1 : 0;
    d.volume_flux = static_cast<int>(spec.volume_flux);
    d.device = device;
    init(d);
  }
#endif

  ~Semidiscretization() {
    if (ctx_) perrk_destroy(ctx_);
  }
  Semidiscretization(const Semidiscretization&) = delete;
  Semidiscretization& operator=(const Semidiscretization&) = delete;

  int num_dofs() const { return static_cast<int>(dofs_); }
  int num_nodes() const { return static_cast<int>(nodes_); }
  int num_cells() const { return static_cast<int>(cells_); }
  int num_vars() const { return vars_; }
  int nodes_per_cell() const { return npc_; }
  perrk_ctx* handle() const { return ctx_; }

  void rhs(double t, const std::vector<double>& U, std::vector<double>& out) const {
    size_check(U);
    out.assign(U.size(), 0.0);
    check(perrk_rhs_masked(ctx_, t, U.data(), out.data(), nullptr));
  }
  void rhs_masked(double t, const std::vector<double>& U, std::vector<double>& out,
                  const std::vector<char>& eval_cell) const {
    size_check(U);
    if (static_cast<int64_t>(eval_cell.size()) != cells_)
      throw Error(PERRK_EINVAL, "mask size mismatch");
    out.assign(U.size(), 0.0);
    check(perrk_rhs_masked(ctx_, t, U.data(), out.data(), eval_cell.data()));
  }
  template <class Map>
  void rhs_partition_restricted(double t, const std::vector<double>& U, std::vector<double>& out,
                                const Map& map, int level) const {
    std::vector<char> mask(map.effective_level.size());
    for (std::size_t i = 0; i < mask.size(); ++i) mask[i] = map.effective_level[i] == level;
    rhs_masked(t, U, out, mask);
  }
  double total_entropy(const std::vector<double>& U) const {
    size_check(U);
    double h = 0.0;
    check(perrk_total_entropy(ctx_, U.data(), &h));
    return h;
  }
  double entropy_inner_product(const std::vector<double>& U, const std::vector<double>& K) const {
    size_check(U);
    size_check(K);
    double h = 0.0;
    check(perrk_entropy_inner_product(ctx_, U.data(), K.data(), &h));
    return h;
  }
  std::vector<double> integral_per_variable(const std::vector<double>& U) const {
    size_check(U);
    double out[5] = {};
    check(perrk_integral_per_variable(ctx_, U.data(), out));
    return std::vector<double>(out, out + vars_);
  }
  bool admissible(const std::vector<double>& U, int* first_bad_cell = nullptr) const {
    size_check(U);
    int ok = 0, bad = -1;
    check(perrk_admissible(ctx_, U.data(), &ok, &bad));
    if (first_bad_cell) *first_bad_cell = bad;
    return ok != 0;
  }
  std::uint64_t rhs_cell_evaluations() const {
    uint64_t n = 0;
    check(perrk_rhs_cell_evaluations(ctx_, &n));
    return n;
  }
  void reset_evaluation_counter() const { check(perrk_reset_counter(ctx_)); }

  /// Upload a family + partition map (cached by address and size).
  void bind(const perrk_family_desc& f, const std::vector<int>& effective_level,
            const void* key) const {
    if (key == bound_ && f.S == bound_S_) return;
    check(perrk_set_family(ctx_, &f, effective_level.data()));
    bound_ = key;
    bound_S_ = f.S;
  }

 private:
  void init(const perrk_semi_desc& d) {
    check(perrk_create(&d, &ctx_));
    check(perrk_sizes(ctx_, &dofs_, &nodes_, &cells_, &vars_, &npc_));
  }
  void size_check(const std::vector<double>& U) const {
    if (static_cast<int64_t>(U.size()) != dofs_) throw Error(PERRK_EINVAL, "state size mismatch");
  }
  perrk_ctx* ctx_ = nullptr;
  int64_t dofs_ = 0, nodes_ = 0, cells_ = 0;
  int vars_ = 0, npc_ = 0;
  mutable const void* bound_ = nullptr;
  mutable int bound_S_ = -1;
};

#ifdef PERRK_STEPPER_HPP
/// perk_step (stepper.hpp:72-74) on the device: the reference's family, map,
/// options and result types.
inline ::perrk::PerkStepResult perk_step(std::vector<double>& U, double& t, double dt,
                                         const ::perrk::PartitionFamily& family,
                                         const ::perrk::PartitionMap& map,
                                         const Semidiscretization& semi,
                                         const ::perrk::PerkStepOptions& opts) {
  const int S = family.S, R = family.R;
  std::vector<double> A(static_cast<std::size_t>(R) * S * S);
  for (int r = 0; r < R; ++r)
    for (int q = 0; q < S * S; ++q) A[static_cast<std::size_t>(r) * S * S + q] = family.members[r].A[q];
  perrk_family_desc fd{static_cast<int>(family.kind), S, R, family.E.data(), A.data(),
                       family.members[0].b.data(), family.members[0].c.data()};
  semi.bind(fd, map.effective_level, &family);
  perrk_step_opts o{};
  o.relax_enabled = opts.relaxation != nullptr;
  if (opts.relaxation) {
    const auto& r = *opts.relaxation;
    o.relax = perrk_relax_cfg{static_cast<int>(r.method), r.max_iter, r.residual_tol, r.step_tol,
                              r.bracket_min, r.bracket_max, r.seed_from_previous ? 1 : 0, 0};
  }
  o.gamma_override = opts.gamma_override;
  o.gamma_seed = opts.gamma_seed;
  o.h_ref = opts.h_ref;
  o.idt = opts.idt ? 1 : 0;
  perrk_step_result res{};
  check(perrk_perk_step(semi.handle(), U.data(), &t, dt, &o, &res));
  ::perrk::PerkStepResult out;
  out.outcome.gamma = res.gamma;
  out.outcome.iterations = res.iterations;
  out.outcome.residual = res.residual;
  out.outcome.fell_back = res.fell_back != 0;
  out.delta_h = res.delta_h;
  out.aborted = res.aborted != 0;
  out.bad_cell = res.bad_cell;
  out.bad_stage = res.bad_stage;
  return out;
}
#endif

}  // namespace perrk_b200

#endif
