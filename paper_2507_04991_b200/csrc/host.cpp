// Host layer of perrk_b200: the reference's Semidiscretization / perk_step /
// run API (proj/core/include/perrk/{semidisc,stepper,relax}.hpp) re-expressed
// over device-resident state, plus the host-side inputs of the hot path
// (GLL basis, P-ERK family builders, level assignment, partition map).  The
// exported entry points are the C-ABI declared in include/perrk_b200.h.
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <set>
#include <stdexcept>
#include <string>
#include <algorithm>
#include <vector>

#include <memory>

#include <cuda_runtime.h>
#include <nccl.h>

#include "../../include/perrk_b200.h"
#include "dg_launch.hpp"

namespace perrk {
namespace {

thread_local std::string g_last_error;

struct Fail : std::runtime_error {
  int code;
  Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define REQUIRE(cond, msg)                       \
  do {                                           \
    if (!(cond)) throw Fail(PERRK_EINVAL, (msg)); \
  } while (0)

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Fail(PERRK_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

template <class F>
int guarded(F&& f) {
  try {
    f();
    return PERRK_OK;
  } catch (const Fail& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return PERRK_EINVAL;
  }
}

// ---------------------------------------------------------------------------
// GLL basis: nodes are the endpoints and the roots of P_k' (found by Newton
// from Chebyshev-Lobatto guesses); w_i = 2 / (k(k+1) P_k(x_i)^2);
// D_ij = P_k(x_i) / (P_k(x_j)(x_i - x_j)), D_00 = -k(k+1)/4, D_kk = k(k+1)/4.
// Same construction as the reference's gll_basis (basis.cpp:35-84).
// ---------------------------------------------------------------------------
struct Basis {
  int k;
  std::vector<double> x, w, D;
};

void legendre_pair(int k, double x, double& p, double& dp) {
  double a = 1.0, b = x;  // P_{n-1}, P_n
  if (k == 0) {
    p = 1.0;
    dp = 0.0;
    return;
  }
  for (int n = 1; n < k; ++n) {
    const double c = ((2.0 * n + 1.0) * x * b - n * a) / (n + 1.0);
    a = b;
    b = c;
  }
  p = b;
  dp = k * (a - x * b) / (1.0 - x * x);
}

Basis make_basis(int k) {
  Basis B;
  B.k = k;
  const int n = k + 1;
  B.x.assign(n, 0.0);
  B.x[0] = -1.0;
  B.x[k] = 1.0;
  for (int i = 1; i < k; ++i) {
    double x = -std::cos(M_PI * i / k);
    for (int it = 0; it < 100; ++it) {
      double p, dp;
      legendre_pair(k, x, p, dp);
      const double step = dp / ((2.0 * x * dp - k * (k + 1.0) * p) / (1.0 - x * x));
      x -= step;
      if (std::fabs(step) < 1e-15) break;
    }
    B.x[i] = x;
  }
  for (int i = 0; i < n / 2; ++i) {  // exact antisymmetry
    const double v = 0.5 * (B.x[n - 1 - i] - B.x[i]);
    B.x[i] = -v;
    B.x[n - 1 - i] = v;
  }
  if (n % 2) B.x[n / 2] = 0.0;
  std::vector<double> pk(n);
  B.w.resize(n);
  for (int i = 0; i < n; ++i) {
    double p, dp;
    if (std::fabs(B.x[i]) == 1.0)
      p = (B.x[i] > 0 || k % 2 == 0) ? 1.0 : -1.0;
    else
      legendre_pair(k, B.x[i], p, dp);
    pk[i] = p;
    B.w[i] = 2.0 / (k * (k + 1.0) * p * p);
  }
  B.D.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      if (i != j) B.D[i * n + j] = pk[i] / (pk[j] * (B.x[i] - B.x[j]));
  B.D[0] = -k * (k + 1.0) / 4.0;
  B.D[n * n - 1] = k * (k + 1.0) / 4.0;
  return B;
}

// ---------------------------------------------------------------------------
// P-ERK family builders (butcher.cpp:24-247): shared b and c, first column
// a_{i,1} = c_i, chain rows S-E+2..S-1 (0-based) carry a_{i,i-1}.
// ---------------------------------------------------------------------------
constexpr double kP4cSm2 = 0.479274057836310;
constexpr double kP4aSm2 = 0.114851811257441;  // divided by c_{S-3}
constexpr double kP4aSm1 = 0.648906880894214;
constexpr double kP4aS = 0.0283121635129678;

int free_count(int kind, int E) {
  switch (kind) {
    case PERRK_FAMILY_P2: return E - 2;
    case PERRK_FAMILY_P3_VARIANT:
    case PERRK_FAMILY_P3_ORIGINAL: return E - 3;
    case PERRK_FAMILY_P4: return E - 5;
  }
  throw Fail(PERRK_EINVAL, "unknown family kind");
}

std::vector<double> weights_b(int kind, int S) {
  std::vector<double> b(S, 0.0);
  if (kind == PERRK_FAMILY_P2) {
    b[S - 1] = 1.0;
  } else if (kind == PERRK_FAMILY_P3_VARIANT) {
    b[0] = 1.0 / 6.0;
    b[S - 2] = 1.0 / 6.0;
    b[S - 1] = 2.0 / 3.0;
  } else if (kind == PERRK_FAMILY_P3_ORIGINAL) {
    b[S - 2] = 3.0 / 4.0;
    b[S - 1] = 1.0 / 4.0;
  } else {
    b[S - 2] = 0.5;
    b[S - 1] = 0.5;
  }
  return b;
}

std::vector<double> abscissae(int kind, int S, double c_sm3) {
  std::vector<double> c(S, 0.0);
  if (kind == PERRK_FAMILY_P2) {
    for (int i = 1; i < S; ++i) c[i] = static_cast<double>(i) / (2.0 * (S - 1));
  } else if (kind == PERRK_FAMILY_P3_VARIANT || kind == PERRK_FAMILY_P3_ORIGINAL) {
    for (int i = 1; i <= S - 3; ++i) c[i] = static_cast<double>(i) / (S - 3);
    c[S - 2] = kind == PERRK_FAMILY_P3_VARIANT ? 1.0 : 1.0 / 3.0;
    c[S - 1] = kind == PERRK_FAMILY_P3_VARIANT ? 0.5 : 1.0;
  } else {
    const double r = std::sqrt(3.0) / 6.0;
    for (int i = 1; i <= S - 5; ++i) c[i] = 1.0;
    if (S >= 5) c[S - 4] = c_sm3;
    c[S - 3] = kP4cSm2;
    c[S - 2] = 0.5 + r;
    c[S - 1] = 0.5 - r;
  }
  return c;
}

std::vector<char> reachable_stages(int S, const double* A, const std::vector<double>& b) {
  std::vector<char> act(S, 0);
  act[0] = 1;
  for (int i = 0; i < S; ++i)
    if (b[i] != 0.0) act[i] = 1;
  // a stage feeds stage i through any nonzero A[i][j]: sweep from the back
  for (bool grew = true; grew;) {
    grew = false;
    for (int i = S - 1; i >= 0; --i)
      if (act[i])
        for (int j = 0; j < i; ++j)
          if (A[i * S + j] != 0.0 && !act[j]) act[j] = 1, grew = true;
  }
  return act;
}

void build_member(int kind, int S, int E, const double* fr, const std::vector<double>& b,
                  const std::vector<double>& c, double* A) {
  const int minE = kind == PERRK_FAMILY_P4 ? 5 : 3;
  REQUIRE(E >= minE && E <= S, "member evaluation count out of range for archetype");
  std::fill(A, A + S * S, 0.0);
  for (int i = 1; i < S; ++i) A[i * S] = c[i];
  auto chain = [&](int i, double a) {
    A[i * S + i - 1] = a;
    A[i * S] = c[i] - a;
  };
  const int derived = kind == PERRK_FAMILY_P4 ? 3 : (kind == PERRK_FAMILY_P2 ? 0 : 1);
  int next = 0;
  for (int i = S - E + 2; i < S - derived; ++i) chain(i, fr[next++]);
  if (kind == PERRK_FAMILY_P3_VARIANT || kind == PERRK_FAMILY_P3_ORIGINAL) {
    double acs = 0.0;  // (A c)_{S-2}: pins a_{S,S-1} through b^T A c = 1/6
    for (int j = 0; j < S - 2; ++j) acs += A[(S - 2) * S + j] * c[j];
    const double a_last = (1.0 / 6.0 - b[S - 2] * acs) / (b[S - 1] * c[S - 2]);
    REQUIRE(std::isfinite(a_last), "no solution for the p3 coupling coefficient");
    chain(S - 1, a_last);
  } else if (kind == PERRK_FAMILY_P4) {
    REQUIRE(c[S - 4] != 0.0, "c_{S-3} = 0: division by zero in the p4 base coefficients");
    chain(S - 3, kP4aSm2 / c[S - 4]);
    chain(S - 2, kP4aSm1);
    chain(S - 1, kP4aS);
  }
  const double tol = -1e-14;
  if (kind == PERRK_FAMILY_P2) {
    for (int i = 1; i < S; ++i)
      REQUIRE(A[i * S] >= tol, "free coefficient produces negative first-column entry");
  } else if (kind != PERRK_FAMILY_P3_ORIGINAL) {
    for (int i = 0; i < S; ++i)
      for (int j = 0; j < i; ++j)
        REQUIRE(A[i * S + j] >= tol, "no nonnegative solution for the coupling coefficients");
  }
}

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------
struct StagePlan {
  int* dlist = nullptr;  // nullptr: all cells
  int n = 0;
  // slab decomposition: the stage's cells off the slab boundary (computed
  // while the halo is in flight) and on it (after the halo arrives)
  int *ilist = nullptr, *blist = nullptr;
  int in = 0, bn = 0;
  int* glist = nullptr;  // BR1: active cells and their face neighbours (nullptr: all)
  int gn = 0;
  double bytes = 0.0;    // compulsory HBM bytes of the launch (roofline)
  StageArgs args{};
};

}  // namespace

}  // namespace perrk

using namespace perrk;
using perrk::dev::StepState;

struct perrk_ctx;
namespace perrk {
// A set of contexts that step together: one rank's context under NCCL (one
// process per GPU), or several contexts on one device and one stream that
// exchange through device copies (loopback; the test harness for the
// multi-rank logic on a single GPU).
struct Exchange {
  virtual ~Exchange() = default;
  // every rank's packed traces (sendbuf, per peer) -> the peers' ghost slots
  virtual void halo(std::vector<perrk_ctx*>& g) = 0;
  // the same, overlapped: started after the packing on the compute stream,
  // waited for before the boundary cells' stage launch
  virtual void halo_begin(std::vector<perrk_ctx*>& g) { halo(g); }
  virtual void halo_end(std::vector<perrk_ctx*>&) {}
  // StepState::red_local of every rank -> red_all[rank][NRED] on every rank
  virtual void gather(std::vector<perrk_ctx*>& g) = 0;
};

struct Group {
  std::vector<perrk_ctx*> members;
  std::unique_ptr<Exchange> ex;  // null: a single context on the whole mesh
  cudaStream_t shared_stream = nullptr;  // loopback: owned by the group, not a member
  ~Group() {
    if (shared_stream) cudaStreamDestroy(shared_stream);
  }
};

}  // namespace perrk

struct perrk_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int dim = 2, V = 4, npc = 16, k = 3;
  int nc[3] = {1, 1, 1};
  long long ncells = 0, nnodes = 0, ndofs = 0;
  std::vector<double> edges[3], h[3];
  Basis basis;
  dev::Phys ph{};
  int physics = 0, surface = 2, volume_mode = 1, volume_flux = 5;
  int vol() const {  // the stage kernel's volume variant (dg_launch.hpp)
    return volume_mode == 0 ? VOL_WEAK : (volume_flux == PERRK_FLUX_EC ? VOL_EC : VOL_CENTRAL);
  }
  double mu = 0.0, prandtl = 1.0;
  // device buffers
  double *U = nullptr, *K1 = nullptr, *d = nullptr;
  // second state buffer of perrk_advance's fused relaxation (relax_spec_kernel):
  // each step reads U and writes the new state to Ualt, then the two swap
  double* Ualt = nullptr;
  double *Ka = nullptr, *Kb = nullptr;  // formed stage states U_i, ping-pong by stage parity
  double *tU = nullptr, *tK = nullptr;  // scratch for host-buffer queries
  // staging vector of upload / download: the canonical (reference) layout of
  // a host buffer, transposed on the device to / from the device layout
  // (dev::sidx, cell-blocked SoA)
  double* lay = nullptr;
  double* G = nullptr;                   // BR1 viscous fluxes [2][ndofs] (NSF only)
  double *dh[3] = {}, *djac[3] = {}, *dlift[3] = {};
  int8_t* dlevel = nullptr;
  StepState* st = nullptr;
  double* partials = nullptr;
  unsigned* counter = nullptr;
  double* dout = nullptr;
  int* dint = nullptr;
  int* dlist_tmp = nullptr;
  double* records = nullptr;
  int records_cap = 0;
  // pinned host rows the step records stream into, one D2H copy per step as
  // the step completes (no host synchronisation inside the run)
  double* rec_host = nullptr;
  int rec_host_cap = 0;
  double* dnu = nullptr;
  int grid_stage = 1184, grid_flat = 1184;
  // family
  bool has_family = false;
  int S = 0, R = 0;
  std::vector<double> A, b, c;
  std::vector<int> E, eff;
  std::vector<StagePlan> plan;
  uint64_t evals = 0;
  // domain decomposition: this context owns the cells g of the
  // global mesh with owner[g] == rank, in increasing global id; face
  // neighbours owned elsewhere are ghost trace slots filled by the halo
  bool slab = false;  // decomposed
  int rank = 0, nranks = 1;
  int ncg[3] = {1, 1, 1};
  long long ncells_global = 0;
  std::vector<int> gid;    // local -> global cell
  std::vector<int> nbr_h;  // [local][2 dim]: local neighbour or -1 - ghost slot
  int *d_gid = nullptr, *d_nbr = nullptr, *d_send = nullptr;
  dev::CellRec* d_rec = nullptr;  // static per-cell descriptors of the stage kernel
  long long* d_ghost_gid = nullptr;
  double *ghost = nullptr, *sendbuf = nullptr;  // [slot][FP][V], [entry][FP][V]
  std::vector<int> peers;                       // ascending
  std::vector<long long> recv_off, send_off;    // per peer, in traces
  long long nghost = 0, nsend = 0;
  double* red_all = nullptr;  // [nranks][NRED]
  std::shared_ptr<perrk::Group> group;
  // CUDA graph of one run() step (perrk_advance): launch latency matters for
  // the small configurations (C1 is 4096 nodes, ~20 kernels per step)
  bool use_graphs = true;
  bool use_fused = true;  // perrk_advance: relax_spec_kernel (PERRK_NO_FUSED_RELAX=1 disables)
  // captured steps by key (plan, records, mode, and the current state buffer:
  // the fused path alternates two, so two graphs stay cached)
  struct StepGraph {
    std::string key;
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;  // kernels per graph launch
  };
  std::vector<StepGraph> graphs;
  uint64_t plan_version = 0;
  // instrumentation: launch counter and per-stage-launch event pairs
  bool own_stream = true;
  int64_t launches = 0;
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<double> ev_bytes;

  dev::MeshDev mesh() const {
    dev::MeshDev m{};
    for (int a = 0; a < 3; ++a) {
      m.nc[a] = nc[a];  // global
      m.h[a] = dh[a];
      m.jac[a] = djac[a];
      m.lift[a] = dlift[a];
    }
    m.dim = dim;
    m.level = dlevel;
    m.rec = d_rec;
    if (slab) {
      m.gid = d_gid;
      m.nbr = d_nbr;
      m.ghost = ghost;
      m.ghost_gid = d_ghost_gid;
    }
    return m;
  }
  size_t ndofs_() const { return static_cast<size_t>(ndofs); }
  size_t trace_doubles() const { return static_cast<size_t>(dim == 3 ? 16 : 4) * V; }  // one face trace
  double* sbuf(int parity) { return parity ? Kb : Ka; }  // formed stage states (ping-pong)
};

namespace perrk {
namespace {

void set_device(perrk_ctx* c) { CK(cudaSetDevice(c->device)); }

StepState fresh_state() {
  StepState s{};
  s.bad_code = std::numeric_limits<long long>::max();
  s.h_ref = std::numeric_limits<double>::quiet_NaN();
  s.gamma = s.gamma_seed = s.gamma_override = 1.0;
  s.relax_done = 1;
  return s;
}

void put_state(perrk_ctx* c, const StepState& s) {
  CK(cudaMemcpyAsync(c->st, &s, sizeof s, cudaMemcpyHostToDevice, c->stream));
}

StepState get_state(perrk_ctx* c) {
  StepState s;
  CK(cudaMemcpyAsync(&s, c->st, sizeof s, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return s;
}

// Host buffers are in the reference's canonical layout (common.hpp:11-13),
// device state-shaped buffers in the device layout (dev::sidx): the copies
// go through c->lay and the layout kernel.
void upload(perrk_ctx* c, double* dst, const double* src) {
  if (!c->lay) CK(cudaMalloc(&c->lay, sizeof(double) * c->ndofs));
  CK(cudaMemcpyAsync(c->lay, src, sizeof(double) * c->ndofs, cudaMemcpyHostToDevice, c->stream));
  CK(launch_layout(dst, c->lay, c->ncells, c->npc, c->V, 1, c->grid_flat, c->stream));
}

void download(perrk_ctx* c, double* dst, const double* src) {
  if (!c->lay) CK(cudaMalloc(&c->lay, sizeof(double) * c->ndofs));
  CK(launch_layout(c->lay, src, c->ncells, c->npc, c->V, 0, c->grid_flat, c->stream));
  CK(cudaMemcpyAsync(dst, c->lay, sizeof(double) * c->ndofs, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
}

// Build per-stage launch plans from the family and the effective levels.
// cells of a mask plus their periodic face neighbours (2D), ascending
std::vector<int> with_neighbours_2d(const perrk_ctx* c, const std::vector<char>& on) {
  const int nx = c->nc[0], ny = c->nc[1];
  std::vector<char> g(on);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i)
      if (on[i + nx * j]) {
        g[(i + 1) % nx + nx * j] = 1;
        g[(i + nx - 1) % nx + nx * j] = 1;
        g[i + nx * ((j + 1) % ny)] = 1;
        g[i + nx * ((j + ny - 1) % ny)] = 1;
      }
  std::vector<int> out;
  for (long long q = 0; q < c->ncells; ++q)
    if (g[q]) out.push_back(static_cast<int>(q));
  return out;
}

// Traversal order of a stage's cell list (3D).  The persistent warps of a
// stage kernel walk the list front to back, so the cells in flight at any
// moment are a window of consecutive entries.  In the natural x-fastest
// order a cell's z-neighbours lie nx ny entries away (40 MB of stage traffic
// on a 64^3 mesh), and their face traces are fetched from HBM a second time.
// Ordering the list by bricks of B^3 cells (x-fastest inside a brick and
// between bricks) brings every neighbour within B^2 entries except across
// brick faces.  Measured on C5 (profiles/r02_ab.txt): no change in stage time,
// DRAM bytes -2% with the round-1 kernel and +2% with the direct streaming
// epilogue (shorter contiguous runs), so the natural order is the default;
// PERRK_BRICK=B orders by bricks of B^3.
int brick_edge() {  // read at every perrk_set_family
  const char* e = std::getenv("PERRK_BRICK");
  const int v = e ? std::atoi(e) : 0;
  return v < 0 ? 0 : v;
}

bool brick_order(const perrk_ctx* c, std::vector<int>& list) {
  const int B = brick_edge();
  if (c->dim != 3 || B <= 1) return false;
  const long long nx = c->ncg[0], ny = c->ncg[1], nz = c->ncg[2];
  if (nx <= B && ny <= B && nz <= B) return false;
  const long long nbx = (nx + B - 1) / B, nby = (ny + B - 1) / B;
  auto key = [&](int cell) {
    const long long g = c->slab ? c->gid[cell] : cell;
    const long long ix = g % nx, iy = (g / nx) % ny, iz = g / (nx * ny);
    return ((iz / B) * nby + iy / B) * nbx + ix / B;
  };
  std::vector<std::pair<long long, int>> k(list.size());
  for (size_t i = 0; i < list.size(); ++i) k[i] = {key(list[i]), list[i]};
  std::sort(k.begin(), k.end());  // ties (one brick) in ascending cell order
  for (size_t i = 0; i < list.size(); ++i) list[i] = k[i].second;
  return true;
}

void build_plan(perrk_ctx* c) {
  for (auto& p : c->plan)
    for (int* q : {p.dlist, p.glist, p.ilist, p.blist})
      if (q) cudaFree(q);
  c->plan.clear();
  const int S = c->S, R = c->R;
  std::vector<std::vector<char>> active(R);  // by level-1
  for (int lvl = 1; lvl <= R; ++lvl)
    active[lvl - 1] = reachable_stages(S, &c->A[static_cast<size_t>(R - lvl) * S * S], c->b);
  int first_b = -1, last_b = -1;
  for (int i = 0; i < S; ++i)
    if (c->b[i] != 0.0) {
      if (first_b < 0) first_b = i;
      last_b = i;
    }
  REQUIRE(first_b >= 0, "family has no nonzero weight");
  for (int i = 0; i < S; ++i) {
    StagePlan p;
    StageArgs& a = p.args;
    std::vector<int> list;
    bool all = true;
    for (long long cell = 0; cell < c->ncells; ++cell) {
      const bool on = i == 0 || active[c->eff[cell] - 1][i];
      if (on)
        list.push_back(static_cast<int>(cell));
      else
        all = false;
    }
    p.n = static_cast<int>(list.size());
    if (brick_order(c, list)) all = false;  // a reordered full list is still a list
    if (!all && p.n > 0) {
      CK(cudaMalloc(&p.dlist, sizeof(int) * list.size()));
      CK(cudaMemcpy(p.dlist, list.data(), sizeof(int) * list.size(), cudaMemcpyHostToDevice));
    }
    if (c->slab) {  // interior / boundary (some neighbour is a ghost) split
      std::vector<int> il, bl;
      for (int q : list) {
        bool boundary = false;
        for (int f = 0; f < 2 * c->dim; ++f) boundary |= c->nbr_h[static_cast<size_t>(q) * 2 * c->dim + f] < 0;
        (boundary ? bl : il).push_back(q);
      }
      p.in = static_cast<int>(il.size());
      p.bn = static_cast<int>(bl.size());
      if (p.in > 0) {
        CK(cudaMalloc(&p.ilist, sizeof(int) * il.size()));
        CK(cudaMemcpy(p.ilist, il.data(), sizeof(int) * il.size(), cudaMemcpyHostToDevice));
      }
      if (p.bn > 0) {
        CK(cudaMalloc(&p.blist, sizeof(int) * bl.size()));
        CK(cudaMemcpy(p.blist, bl.data(), sizeof(int) * bl.size(), cudaMemcpyHostToDevice));
      }
    }
    if (c->physics == 1) {  // BR1: gradients on the active cells and their neighbours
      std::vector<char> on(c->ncells, 0);
      for (int q : list) on[q] = 1;
      const std::vector<int> gl = with_neighbours_2d(c, on);
      p.gn = static_cast<int>(gl.size());
      if (p.gn < c->ncells && p.gn > 0) {
        CK(cudaMalloc(&p.glist, sizeof(int) * gl.size()));
        CK(cudaMemcpy(p.glist, gl.data(), sizeof(int) * gl.size(), cudaMemcpyHostToDevice));
      }
    }
    // stage-state data flow ("K4 folded into the loads"): the
    // epilogue of stage i writes U_{i+1} = U + dt (a_{i+1,1} K1 + a_{i+1,i} K_i)
    // for its cells, so stage i+1 reads one formed array for every cell that
    // was active at i; cells that were not are formed from the first column
    // (their a_{i+1,i} is zero: chain rows follow active stages,
    // butcher.cpp:67-77).  Only K1 is ever stored.
    for (int lvl = 0; lvl <= dev::MAXR; ++lvl) {
      a.a1[lvl] = a.a1n[lvl] = a.apn[lvl] = 0.0;
      a.formed[lvl] = 0;
    }
    for (int lvl = 1; lvl <= R; ++lvl) {
      const double* Am = &c->A[static_cast<size_t>(R - lvl) * S * S];
      a.a1[lvl] = i > 0 ? Am[i * S] : 0.0;
      a.formed[lvl] = i == 0 || active[lvl - 1][i - 1] ? 1 : 0;
      if (i >= 1 && !a.formed[lvl])
        REQUIRE(Am[i * S + i - 1] == 0.0, "chain coefficient on a stage following an inactive one");
      if (i + 1 < S) {
        a.a1n[lvl] = Am[(i + 1) * S];
        a.apn[lvl] = i >= 1 ? Am[(i + 1) * S + i] : 0.0;
      }
    }
    a.form = i > 0 ? 1 : 0;
    a.write_next = i + 1 < S ? 1 : 0;
    a.write_k = i == 0 ? 1 : 0;  // K1
    a.b = c->b[i];
    a.d_mode = c->b[i] != 0.0 ? (i == first_b ? 1 : 2) : 0;
    a.want_dh = c->b[i] != 0.0;
    a.want_dmax = i == last_b;
    a.want_h = 0;
    a.stage = i;
    a.ncells = c->ncells_global;
    a.list = p.dlist;
    a.n = p.n;
    // compulsory traffic per active cell, in node-vectors of 8V bytes: the
    // stage state (U_i, or U and K1 where formed from the first column),
    // K1 written at stage 0, U_{i+1} written (its formation reads U and K1),
    // and d (write at the first b-stage, read-modify-write after)
    double vecs = 0.0;
    for (long long cell = 0; cell < c->ncells; ++cell) {
      const int lv = c->eff[cell];
      if (!(i == 0 || active[lv - 1][i])) continue;
      double v = (a.form && !a.formed[lv]) ? 2.0 : 1.0;
      if (a.write_k) v += 1.0;
      if (a.write_next) v += 1.0 + (a.form && a.formed[lv] ? 2.0 : 0.0);
      v += a.d_mode == 1 ? 1.0 : (a.d_mode == 2 ? 2.0 : 0.0);
      vecs += v;
    }
    p.bytes = vecs * c->npc * c->V * 8.0;
    c->plan.push_back(p);
  }
}

// residual evaluations one step may need (each pass is one fused launch)
int relax_passes(const perrk_relax_cfg& r) {
  if (r.method == 0) return r.numerics == 1 ? r.max_iter : r.max_iter + 1;
  return r.max_iter + 2;  // bisection: r(lo), r(hi) + max_iter; secant: r(g0), r(g1) + ...
}

struct StepMode {
  bool relax = false;
  perrk_relax_cfg cfg{};
  bool want_nu = false;
  bool want_record = false;
  double* records = nullptr;  // non-null: each member writes its own c->records
  double* records_of(perrk_ctx* c) const { return records ? c->records : nullptr; }
  // single context, accurate-numerics Newton: Newton pass 2 fused with a
  // speculative out-of-place update (relax_spec_kernel); the step's new state
  // lands in c->Ualt and enqueue_step swaps c->U / c->Ualt
  bool fused = false;
};

// Enqueue the stage launch of stage i of one context; part 0: all the
// stage's cells, 1: those off the slab boundary, 2: those on it.
void enqueue_stage(perrk_ctx* c, int i, bool want_h, int part = 0) {
  StagePlan& p = c->plan[i];
  StageArgs a = p.args;
  if (part == 1) {
    a.list = p.ilist;
    a.n = p.in;
  } else if (part == 2) {
    a.list = p.blist;
    a.n = p.bn;
  }
  if (a.n == 0) return;
  a.U = c->U;
  a.K1 = c->K1;
  a.Us = i > 0 ? c->sbuf(i & 1) : nullptr;
  a.Usn = c->sbuf((i + 1) & 1);
  a.Kout = c->K1;
  a.d = c->d;
  a.want_h = (i == 0 && want_h) ? 1 : 0;
  a.ndofs = c->ndofs;
  if (c->physics == 1) {  // BR1: viscous fluxes of the stage state first
    StageArgs ga = a;
    ga.list = p.glist;
    ga.n = p.gn;
    CK(launch_grad(ga, c->mesh(), c->ph, c->st, c->G, c->ndofs, 0, c->grid_stage, c->stream));
    c->launches += 1;
    a.G = c->G;
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->profiling) {
    if (c->ev_used + 2 > c->ev_pool.size()) {
      for (int q = 0; q < 64; ++q) {
        cudaEvent_t ev;
        CK(cudaEventCreate(&ev));
        c->ev_pool.push_back(ev);
      }
    }
    e0 = c->ev_pool[c->ev_used++];
    e1 = c->ev_pool[c->ev_used++];
    c->ev_bytes.push_back(p.n > 0 ? p.bytes * a.n / p.n : 0.0);
    CK(cudaEventRecord(e0, c->stream));
  }
  CK(launch_stage(c->dim, c->surface, c->vol(), a, c->mesh(), c->ph, c->st, c->partials, c->counter,
                  c->grid_stage, c->stream));
  if (c->profiling) CK(cudaEventRecord(e1, c->stream));
  c->launches += p.n > 0 ? 1 : 0;
}

void enqueue_pack(perrk_ctx* c, int i) {
  StageArgs a = c->plan[i].args;
  a.U = c->U;
  a.K1 = c->K1;
  a.Us = i > 0 ? c->sbuf(i & 1) : nullptr;
  CK(launch_pack_traces(c->dim, a, c->mesh(), c->st, c->d_send, static_cast<int>(c->nsend),
                        c->sendbuf, c->stream));
  c->launches += 1;
}

// One reduction point of the slab decomposition: local partials -> every
// rank -> combined (sums in rank order, so every rank holds the same bits).
void reduce_point(Group& g, int mode, bool stash, double* records = nullptr) {
  if (stash)
    for (perrk_ctx* c : g.members) CK(launch_stash(c->st, mode, c->stream));
  g.ex->gather(g.members);
  for (perrk_ctx* c : g.members) {
    CK(launch_combine(c->st, c->red_all, c->nranks, mode, c->V,
                      mode == RED_UPDATE ? (records ? c->records : nullptr) : nullptr, c->stream));
    c->launches += (stash ? 1 : 0) + 1 + (records && mode == RED_UPDATE ? 1 : 0);
  }
}

// Enqueue one perk_step (stepper.cpp:17-114) on the resident state of every
// member of the group.  Single context on the whole mesh: each kernel's last
// block finishes its own reduction (no host or collective in the chain).
// Slab decomposition: per stage, the boundary traces are packed and
// exchanged before the stage kernels; after the last stage, after every
// relaxation pass and after the update the partials go through reduce_point.
void enqueue_step(Group& g, const StepMode& mode, bool want_h) {
  const bool slab = g.ex != nullptr;
  for (perrk_ctx* c : g.members) {
    CK(launch_begin_step(c->st, c->stream));
    c->launches += 1;
  }
  const int S = g.members[0]->S;
  for (int i = 0; i < S; ++i) {
    if (slab) {
      // boundary traces out, interior cells while they travel, boundary
      // cells once they are in (north_star item 5: halo overlapped with the
      // interior volume work)
      for (perrk_ctx* c : g.members) enqueue_pack(c, i);
      g.ex->halo_begin(g.members);
      for (perrk_ctx* c : g.members) enqueue_stage(c, i, want_h, 1);
      g.ex->halo_end(g.members);
      for (perrk_ctx* c : g.members) enqueue_stage(c, i, want_h, 2);
    } else {
      for (perrk_ctx* c : g.members) enqueue_stage(c, i, want_h);
    }
  }
  if (slab) reduce_point(g, RED_STAGES, true);
  if (mode.relax) {
    const int passes = relax_passes(mode.cfg);
    for (int p = 0; p < passes; ++p) {
      for (perrk_ctx* c : g.members) {
        if (mode.fused && p == 1)
          CK(launch_relax_spec(c->dim, c->U, c->d, c->Ualt, c->mesh(), c->ph, c->st, c->partials,
                               c->counter, c->nnodes, mode.want_nu ? 1 : 0,
                               mode.want_record ? 1 : 0, mode.records_of(c), c->grid_flat,
                               c->stream));
        else
          CK(launch_relax_pass(c->dim, c->U, c->d, c->mesh(), c->ph, c->st, c->partials,
                               c->counter, c->nnodes, c->grid_flat, c->stream));
        c->launches += 1;
      }
      if (slab) reduce_point(g, RED_RELAX, false);
    }
  }
  for (perrk_ctx* c : g.members) {
    CK(launch_update(c->dim, mode.fused ? c->Ualt : c->U, c->U, c->d, c->mesh(), c->ph, c->st,
                     c->partials, c->counter, c->nnodes, mode.want_nu ? 1 : 0,
                     mode.want_record ? 1 : 0, slab ? nullptr : mode.records_of(c), c->grid_flat,
                     c->stream));
    c->launches += 1;
    if (mode.fused) std::swap(c->U, c->Ualt);
  }
  if (slab) reduce_point(g, RED_UPDATE, true, mode.want_record ? mode.records : nullptr);
}

void check_relax_cfg(const perrk_relax_cfg& r) {
  REQUIRE(r.method >= 0 && r.method <= 2, "relaxation method must be 0 newton, 1 bisection, 2 secant");
  if (r.method == 1) REQUIRE(r.bracket_max > r.bracket_min, "empty bisection bracket");
  REQUIRE(r.max_iter >= 1, "relaxation max_iter must be >= 1");
  REQUIRE(r.numerics == 0 || r.numerics == 1, "relaxation numerics must be 0 or 1");
}

void configure_relax(StepState& s, bool enabled, const perrk_relax_cfg& r) {
  s.relax_enabled = enabled ? 1 : 0;
  if (!enabled) return;
  s.numerics = r.numerics;
  s.max_iter = r.max_iter;
  s.seed_from_previous = r.seed_from_previous;
  s.residual_tol = r.residual_tol;
  s.step_tol = r.step_tol;
  s.method = r.method;
  s.bracket_min = r.bracket_min;
  s.bracket_max = r.bracket_max;
}

// Cell-sized device buffers of a context (its slab when decomposed).
void alloc_cell_buffers(perrk_ctx* c) {
  const size_t bytes = sizeof(double) * c->ndofs_();
  for (double** p : {&c->U, &c->K1, &c->Ka, &c->Kb, &c->d, &c->tU, &c->tK}) {
    CK(cudaMalloc(p, bytes));
    CK(cudaMemsetAsync(*p, 0, bytes, c->stream));
  }
  if (c->physics == 1) CK(cudaMalloc(&c->G, 2 * bytes));
  CK(cudaMalloc(&c->dlevel, c->ncells));
  CK(cudaMemset(c->dlevel, 1, c->ncells));
  CK(cudaMalloc(&c->dlist_tmp, sizeof(int) * c->ncells));
  CK(cudaMalloc(&c->dnu, sizeof(double) * c->ncells));
  if (c->slab) {
    const size_t tb = sizeof(double) * c->trace_doubles();
    CK(cudaMalloc(&c->ghost, tb * std::max<long long>(c->nghost, 1)));
    CK(cudaMalloc(&c->sendbuf, tb * std::max<long long>(c->nsend, 1)));
    CK(cudaMemsetAsync(c->ghost, 0, tb * std::max<long long>(c->nghost, 1), c->stream));
    CK(cudaMalloc(&c->red_all, sizeof(double) * dev::NRED * c->nranks));
  }
}

void free_cell_buffers(perrk_ctx* c) {
  for (double** p : {&c->U, &c->K1, &c->Ka, &c->Kb, &c->d, &c->tU, &c->tK, &c->dnu, &c->G,
                     &c->ghost, &c->sendbuf, &c->red_all, &c->Ualt, &c->lay}) {
    if (*p) cudaFree(*p);
    *p = nullptr;
  }
  if (c->dlevel) cudaFree(c->dlevel);
  if (c->dlist_tmp) cudaFree(c->dlist_tmp);
  c->dlevel = nullptr;
  c->dlist_tmp = nullptr;
}

double* red_local_ptr(perrk_ctx* c) {
  return reinterpret_cast<double*>(reinterpret_cast<char*>(c->st) + offsetof(StepState, red_local));
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Fail(PERRK_ECOMM, std::string(what) + ": " + ncclGetErrorString(r));
}
#define NK(x) nccl_check((x), #x)

// One rank per process (GPU): grouped send/recv of the boundary traces to the
// slab neighbours (periodic ring) and an all-gather of the reduction partials,
// all on the context's stream.
struct NcclExchange : Exchange {
  ncclComm_t comm = nullptr;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t packed = nullptr, arrived = nullptr;
  ~NcclExchange() override {
    if (comm) ncclCommDestroy(comm);
    if (packed) cudaEventDestroy(packed);
    if (arrived) cudaEventDestroy(arrived);
    if (comm_stream) cudaStreamDestroy(comm_stream);
  }
  void setup() {
    CK(cudaStreamCreateWithFlags(&comm_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&packed, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&arrived, cudaEventDisableTiming));
  }
  void sendrecv(perrk_ctx* c, cudaStream_t s) {
    const size_t tu = c->trace_doubles();
    NK(ncclGroupStart());
    for (size_t k = 0; k < c->peers.size(); ++k) {
      const size_t ns = c->send_off[k + 1] - c->send_off[k];
      const size_t nr = c->recv_off[k + 1] - c->recv_off[k];
      if (ns) NK(ncclSend(c->sendbuf + c->send_off[k] * tu, ns * tu, ncclDouble, c->peers[k], comm, s));
      if (nr) NK(ncclRecv(c->ghost + c->recv_off[k] * tu, nr * tu, ncclDouble, c->peers[k], comm, s));
    }
    NK(ncclGroupEnd());
  }
  void halo_begin(std::vector<perrk_ctx*>& g) override {
    perrk_ctx* c = g[0];
    CK(cudaEventRecord(packed, c->stream));
    CK(cudaStreamWaitEvent(comm_stream, packed, 0));
    sendrecv(c, comm_stream);
    CK(cudaEventRecord(arrived, comm_stream));
  }
  void halo_end(std::vector<perrk_ctx*>& g) override {
    CK(cudaStreamWaitEvent(g[0]->stream, arrived, 0));
  }
  // grouped send/recv, matched in order per peer, so nranks == 2 (up == dn)
  // pairs correctly
  void halo(std::vector<perrk_ctx*>& g) override { sendrecv(g[0], g[0]->stream); }
  void gather(std::vector<perrk_ctx*>& g) override {
    perrk_ctx* c = g[0];
    NK(ncclAllGather(red_local_ptr(c), c->red_all, dev::NRED, ncclDouble, comm, c->stream));
  }
};

// Several slabs on one device and one stream: the same data movement as
// device-to-device copies, stream-ordered (no kernel waits on another).
struct LoopbackExchange : Exchange {
  void halo(std::vector<perrk_ctx*>& g) override {
    for (perrk_ctx* c : g) {
      const size_t tb = sizeof(double) * c->trace_doubles();
      for (size_t k = 0; k < c->peers.size(); ++k) {
        perrk_ctx* p = g[c->peers[k]];
        const size_t kk = std::lower_bound(p->peers.begin(), p->peers.end(), c->rank) - p->peers.begin();
        const size_t n = c->send_off[k + 1] - c->send_off[k];
        if (n)
          CK(cudaMemcpyAsync(p->ghost + p->recv_off[kk] * c->trace_doubles(),
                             c->sendbuf + c->send_off[k] * c->trace_doubles(), n * tb,
                             cudaMemcpyDeviceToDevice, c->stream));
      }
    }
  }
  void gather(std::vector<perrk_ctx*>& g) override {
    const int P = static_cast<int>(g.size());
    for (int r = 0; r < P; ++r)
      for (int q = 0; q < P; ++q)
        CK(cudaMemcpyAsync(g[q]->red_all + static_cast<size_t>(r) * dev::NRED, red_local_ptr(g[r]),
                           sizeof(double) * dev::NRED, cudaMemcpyDeviceToDevice, g[r]->stream));
  }
};

// device allocations released on every exit path
struct DeviceBuffers {
  std::vector<void*> p;
  ~DeviceBuffers() {
    for (void* q : p) cudaFree(q);
  }
  template <class T>
  T* get(size_t n) {
    void* q = nullptr;
    CK(cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T)));
    p.push_back(q);
    return static_cast<T*>(q);
  }
};

// Periodic face neighbour of global cell g across face f (2 d + side).
long long face_neighbour(int dim, const int* n, long long g, int f) {
  long long co[3] = {g % n[0], (g / n[0]) % n[1], g / (static_cast<long long>(n[0]) * n[1])};
  const int d = f >> 1, side = f & 1;
  co[d] = side ? (co[d] + 1 == n[d] ? 0 : co[d] + 1) : (co[d] == 0 ? n[d] - 1 : co[d] - 1);
  (void)dim;
  return co[0] + n[0] * (co[1] + static_cast<long long>(n[1]) * co[2]);
}

// Static per-cell descriptors of the stage kernel (dev::CellRec): face
// neighbours (periodic, or the halo plan's local / ghost slots), global id
// and the per-axis geometry factors of semidisc.cpp:50-70, 503, 513.
void build_cell_records(perrk_ctx* c) {
  const long long n = c->ncells;
  const int nf = 2 * c->dim;
  const double w0 = c->basis.w[0];
  std::vector<dev::CellRec> r(static_cast<size_t>(n));
  for (long long i = 0; i < n; ++i) {
    const long long g = c->slab ? c->gid[i] : i;
    const long long co[3] = {g % c->nc[0], (g / c->nc[0]) % c->nc[1],
                             g / (static_cast<long long>(c->nc[0]) * c->nc[1])};
    dev::CellRec& q = r[static_cast<size_t>(i)];
    q = dev::CellRec{};
    for (int f = 0; f < nf; ++f)
      q.nb[f] = c->slab ? c->nbr_h[static_cast<size_t>(i) * nf + f]
                        : static_cast<int>(face_neighbour(c->dim, c->nc, g, f));
    q.gid = static_cast<int>(g);
    // levels (perrk_set_family; 1 before a family is set)
    const bool lv = static_cast<long long>(c->eff.size()) == n;
    q.lev[0] = static_cast<signed char>(lv ? c->eff[i] : 1);
    for (int f = 0; f < nf; ++f)
      q.lev[1 + f] = static_cast<signed char>(lv && q.nb[f] >= 0 ? c->eff[q.nb[f]] : 1);
    double meas = 1.0;
    for (int a = 0; a < c->dim; ++a) {
      const double h = c->h[a][co[a]];
      q.J2[a] = 2.0 * (2.0 / h);
      q.lift[a] = 2.0 / (h * w0);  // semidisc.cpp:503,513
      meas *= 0.5 * h;
    }
    q.meas = meas;
  }
  if (c->d_rec) cudaFree(c->d_rec);
  c->d_rec = nullptr;
  CK(cudaMalloc(&c->d_rec, sizeof(dev::CellRec) * r.size()));
  CK(cudaMemcpy(c->d_rec, r.data(), sizeof(dev::CellRec) * r.size(), cudaMemcpyHostToDevice));
}

// Halo plan of one rank for an ownership map: the local cells (ascending
// global id), per local cell and face the local neighbour or a ghost slot, and
// per peer (ascending) the ghost slots it fills and the (local cell, face)
// traces it receives from us.  Both sides order a peer's entries by the
// sender's (global cell, face), so slot k of the receiver is entry k of the
// sender.
struct HaloPlan {
  std::vector<int> gid, nbr, peers, send;  // send: (local cell, face) pairs
  std::vector<long long> ghost_gid, recv_off, send_off;
};

HaloPlan halo_plan(int dim, const int* n, const int* owner, int rank) {
  HaloPlan h;
  const long long NG = static_cast<long long>(n[0]) * n[1] * (dim == 3 ? n[2] : 1);
  std::vector<int> loc(NG, -1);
  for (long long g = 0; g < NG; ++g)
    if (owner[g] == rank) {
      loc[g] = static_cast<int>(h.gid.size());
      h.gid.push_back(static_cast<int>(g));
    }
  REQUIRE(!h.gid.empty(), "a rank owns no cells");
  const int nf = 2 * dim;
  struct Key {
    int peer;
    long long g;  // sender's cell
    int f;        // sender's face
    int local, lf;  // our (receiver) cell and face, or our (sender) cell and face
  };
  std::vector<Key> recv, send;
  h.nbr.assign(h.gid.size() * nf, 0);
  for (size_t c = 0; c < h.gid.size(); ++c)
    for (int f = 0; f < nf; ++f) {
      const long long ng = face_neighbour(dim, n, h.gid[c], f);
      if (owner[ng] == rank) {
        h.nbr[c * nf + f] = loc[ng];
      } else {
        recv.push_back({owner[ng], ng, f ^ 1, static_cast<int>(c), f});
        send.push_back({owner[ng], h.gid[c], f, static_cast<int>(c), f});
      }
    }
  auto by_key = [](const Key& x, const Key& y) {
    return x.peer != y.peer ? x.peer < y.peer : (x.g != y.g ? x.g < y.g : x.f < y.f);
  };
  std::sort(recv.begin(), recv.end(), by_key);
  std::sort(send.begin(), send.end(), by_key);
  for (size_t k = 0; k < recv.size(); ++k) {
    h.nbr[static_cast<size_t>(recv[k].local) * nf + recv[k].lf] = -1 - static_cast<int>(k);
    h.ghost_gid.push_back(recv[k].g);
    if (h.peers.empty() || h.peers.back() != recv[k].peer) {
      h.peers.push_back(recv[k].peer);
      h.recv_off.push_back(static_cast<long long>(k));
    }
  }
  h.recv_off.push_back(static_cast<long long>(recv.size()));
  size_t k = 0;
  for (int p : h.peers) {
    h.send_off.push_back(static_cast<long long>(k));
    while (k < send.size() && send[k].peer == p) {
      h.send.push_back(send[k].local);
      h.send.push_back(send[k].lf);
      ++k;
    }
  }
  h.send_off.push_back(static_cast<long long>(k));
  REQUIRE(k == send.size(), "asymmetric halo");
  return h;
}

// Restrict a context to the cells it owns (owner: global cell -> rank; NULL:
// uniform slabs of last-axis layers).
void make_partition(perrk_ctx* c, int rank, int nranks, const int* owner) {
  REQUIRE(!c->slab, "context is already decomposed");
  REQUIRE(!c->has_family, "decompose before perrk_set_family");
  if (c->physics == 1)
    throw Fail(PERRK_EUNSUP, "the multi-GPU decomposition runs the Euler configurations");
  REQUIRE(nranks >= 2 && rank >= 0 && rank < nranks, "bad rank / rank count");
  const long long NG = c->ncells_global;
  std::vector<int> own(NG);
  if (owner) {
    for (long long g = 0; g < NG; ++g) {
      REQUIRE(owner[g] >= 0 && owner[g] < nranks, "owner out of range");
      own[g] = owner[g];
    }
  } else {
    const int L = c->dim - 1, nl = c->nc[L];
    const long long lc = NG / nl;
    REQUIRE(nranks <= nl, "more ranks than cell layers along the last axis");
    for (long long g = 0; g < NG; ++g) {
      const int layer = static_cast<int>(g / lc);
      int r = 0;
      while (r + 1 < nranks && layer >= (r + 1) * nl / nranks) ++r;
      own[g] = r;
    }
  }
  HaloPlan h = halo_plan(c->dim, c->nc, own.data(), rank);
  set_device(c);
  CK(cudaStreamSynchronize(c->stream));
  free_cell_buffers(c);
  c->slab = true;
  c->rank = rank;
  c->nranks = nranks;
  c->gid = h.gid;
  c->nbr_h = h.nbr;
  c->peers = h.peers;
  c->recv_off = h.recv_off;
  c->send_off = h.send_off;
  c->nghost = static_cast<long long>(h.ghost_gid.size());
  c->nsend = static_cast<long long>(h.send.size() / 2);
  c->ncells = static_cast<long long>(h.gid.size());
  c->nnodes = c->ncells * c->npc;
  c->ndofs = c->nnodes * c->V;
  alloc_cell_buffers(c);
  for (int** p : {&c->d_gid, &c->d_nbr, &c->d_send})
    if (*p) cudaFree(*p);
  if (c->d_ghost_gid) cudaFree(c->d_ghost_gid);
  CK(cudaMalloc(&c->d_gid, sizeof(int) * h.gid.size()));
  CK(cudaMalloc(&c->d_nbr, sizeof(int) * h.nbr.size()));
  CK(cudaMalloc(&c->d_send, sizeof(int) * std::max<size_t>(h.send.size(), 1)));
  CK(cudaMalloc(&c->d_ghost_gid, sizeof(long long) * std::max<size_t>(h.ghost_gid.size(), 1)));
  CK(cudaMemcpy(c->d_gid, h.gid.data(), sizeof(int) * h.gid.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_nbr, h.nbr.data(), sizeof(int) * h.nbr.size(), cudaMemcpyHostToDevice));
  if (!h.send.empty())
    CK(cudaMemcpy(c->d_send, h.send.data(), sizeof(int) * h.send.size(), cudaMemcpyHostToDevice));
  if (!h.ghost_gid.empty())
    CK(cudaMemcpy(c->d_ghost_gid, h.ghost_gid.data(), sizeof(long long) * h.ghost_gid.size(),
                  cudaMemcpyHostToDevice));
  build_cell_records(c);
  CK(cudaStreamSynchronize(c->stream));
}

void no_slab(const perrk_ctx* c, const char* what) {
  if (c->slab)
    throw Fail(PERRK_EUNSUP, std::string(what) + " is not available on a slab-decomposed context");
}

// per-member copy of the step state: the slab flag and rank count
StepState slab_state(const perrk_ctx* c, StepState s) {
  s.slab = c->slab ? 1 : 0;
  s.nranks = c->nranks;
  return s;
}

bool needs_h(bool relax, const perrk_relax_cfg& r, double h_ref) {
  if (!relax) return false;
  return r.numerics == 0 ? std::isnan(h_ref) : !std::isnan(h_ref);
}

uint64_t evals_per_step(const perrk_ctx* c) {
  uint64_t n = 0;
  for (const auto& p : c->plan) n += static_cast<uint64_t>(p.n) * c->npc * c->V;
  return n;
}

void fill_result(const perrk_ctx* c, const StepState& s, bool relax, double gamma_override,
                 perrk_step_result* r) {
  r->gamma = relax ? s.gamma : gamma_override;
  r->iterations = relax ? s.iters : 0;
  r->residual = relax ? s.residual : 0.0;
  r->fell_back = relax ? s.fell_back : 0;
  r->delta_h = s.dh_hi + s.dh_lo;
  r->aborted = s.aborted;
  if (s.aborted && s.bad_code != std::numeric_limits<long long>::max()) {
    r->bad_stage = static_cast<int>(s.bad_code / c->ncells_global);
    r->bad_cell = static_cast<int>(s.bad_code % c->ncells_global);  // global cell id
  } else {
    r->bad_stage = r->bad_cell = -1;
  }
}

const double* stage_input(perrk_ctx* c, const double* U) {
  if (!U) return c->U;
  upload(c, c->tU, U);
  return c->tU;
}

double quad(perrk_ctx* c, const double* dU, const double* dK, int mode, double* outv) {
  CK(launch_quad(c->dim, dU, dK, c->mesh(), c->ph, mode, c->partials, c->counter, c->dout,
                 c->nnodes, c->grid_flat, c->stream));
  double host[5];
  CK(cudaMemcpyAsync(host, c->dout, sizeof host, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (outv) std::memcpy(outv, host, sizeof(double) * c->V);
  return host[0];
}

}  // namespace
}  // namespace perrk

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

const char* perrk_last_error(void) { return g_last_error.c_str(); }
int perrk_abi_version(void) { return PERRK_B200_ABI_VERSION; }

int perrk_create(const perrk_semi_desc* dsc, perrk_ctx** out) {
  perrk_ctx* c = nullptr;
  const int rc = guarded([&] {
    REQUIRE(dsc && out, "null argument");
    REQUIRE(dsc->dim == 2 || dsc->dim == 3, "dim must be 2 or 3");
    if (dsc->polydeg != 3) throw Fail(PERRK_EUNSUP, "the device path is built for polydeg 3");
    REQUIRE(dsc->physics == 0 || dsc->physics == 1, "physics must be 0 (Euler) or 1 (NSF)");
    if (dsc->physics == 1 && dsc->dim != 2)
      throw Fail(PERRK_EUNSUP, "Navier-Stokes/BR1 runs in 2D on the device");
    if (dsc->physics == 1) REQUIRE(dsc->mu >= 0.0 && dsc->prandtl > 0.0, "need mu >= 0 and Pr > 0");
    REQUIRE(dsc->volume_mode == 0 || dsc->volume_mode == 1, "volume_mode must be 0 (weak) or 1");
    // semidisc.cpp:25-28: flux differencing takes the central or the EC two-point flux
    if (dsc->volume_mode == 1 && dsc->volume_flux != PERRK_FLUX_EC &&
        dsc->volume_flux != PERRK_FLUX_CENTRAL)
      throw Fail(PERRK_EINVAL, "flux differencing needs a symmetric consistent volume flux");
    if (dsc->physics == 1 && !(dsc->volume_mode == 1 && dsc->volume_flux == PERRK_FLUX_EC))
      throw Fail(PERRK_EUNSUP, "the 2D Navier-Stokes path runs EC flux differencing");
    const int sf = dsc->surface_flux;
    if (sf == PERRK_FLUX_UPWIND) throw Fail(PERRK_EINVAL, "upwind flux only available for advection");
    REQUIRE(sf >= 0 && sf <= 5, "unknown surface flux");
    REQUIRE(dsc->gamma > 1.0, "gamma must exceed 1");
    c = new perrk_ctx;
    if (const char* e = std::getenv("PERRK_NO_FUSED_RELAX")) c->use_fused = e[0] != '1';
    c->device = dsc->device;
    c->dim = dsc->dim;
    c->V = dsc->dim + 2;
    c->npc = dsc->dim == 2 ? 16 : 64;
    c->physics = dsc->physics;
    c->surface = sf;
    c->volume_mode = dsc->volume_mode;
    c->volume_flux = dsc->volume_flux;
    c->mu = dsc->mu;
    c->prandtl = dsc->prandtl;
    c->ph.gamma = dsc->gamma;
    c->ph.gm1 = dsc->gamma - 1.0;
    c->ph.inv_gm1 = 1.0 / (dsc->gamma - 1.0);
    c->ph.mu = dsc->physics == 1 ? dsc->mu : 0.0;
    c->ph.kappa = dsc->physics == 1 ? dsc->gamma / (dsc->gamma - 1.0) * dsc->mu / dsc->prandtl : 0.0;
    c->basis = make_basis(3);
    for (int a = 0; a < 3; ++a) {
      c->nc[a] = a < dsc->dim ? dsc->n[a] : 1;
      REQUIRE(c->nc[a] >= 1, "need at least one cell per axis");
      if (a < dsc->dim) {
        REQUIRE(dsc->edges[a] != nullptr, "missing edges");
        c->edges[a].assign(dsc->edges[a], dsc->edges[a] + c->nc[a] + 1);
      } else {
        c->edges[a] = {0.0, 1.0};
      }
      c->h[a].resize(c->nc[a]);
      for (int i = 0; i < c->nc[a]; ++i) {
        c->h[a][i] = c->edges[a][i + 1] - c->edges[a][i];
        REQUIRE(c->h[a][i] > 0.0, "cell sizes must be positive");
      }
    }
    c->ncells = static_cast<long long>(c->nc[0]) * c->nc[1] * c->nc[2];
    REQUIRE(c->ncells < (1ll << 31) / 64, "mesh too large for 32-bit cell ids");
    c->nnodes = c->ncells * c->npc;
    c->ndofs = c->nnodes * c->V;
    for (int a = 0; a < 3; ++a) c->ncg[a] = c->nc[a];
    c->ncells_global = c->ncells;
    set_device(c);
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    int sms = 148;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    // persistent stage grid: exactly the resident capacity, so the active
    // cells are swept in order and neighbour traces are L2 hits; a function
    // of the device only, so block partials (and the sums) are reproducible
    const int occ = stage_blocks_per_sm(c->dim, sf, c->vol());
    c->grid_stage = sms * (occ > 0 ? occ : 1);
    c->grid_flat = 8 * sms;
    alloc_cell_buffers(c);
    const double w0 = c->basis.w[0];
    for (int a = 0; a < 3; ++a) {
      std::vector<double> jac(c->nc[a]), lift(c->nc[a]);
      for (int i = 0; i < c->nc[a]; ++i) {
        jac[i] = 2.0 / c->h[a][i];
        lift[i] = 2.0 / (c->h[a][i] * w0);  // semidisc.cpp:503,513
      }
      CK(cudaMalloc(&c->dh[a], sizeof(double) * c->nc[a]));
      CK(cudaMalloc(&c->djac[a], sizeof(double) * c->nc[a]));
      CK(cudaMalloc(&c->dlift[a], sizeof(double) * c->nc[a]));
      CK(cudaMemcpy(c->dh[a], c->h[a].data(), sizeof(double) * c->nc[a], cudaMemcpyHostToDevice));
      CK(cudaMemcpy(c->djac[a], jac.data(), sizeof(double) * c->nc[a], cudaMemcpyHostToDevice));
      CK(cudaMemcpy(c->dlift[a], lift.data(), sizeof(double) * c->nc[a], cudaMemcpyHostToDevice));
    }
    CK(cudaMalloc(&c->st, sizeof(StepState)));
    CK(cudaMalloc(&c->partials, sizeof(double) * 2 * 8 * 4096));
    CK(cudaMalloc(&c->counter, sizeof(unsigned)));
    CK(cudaMemset(c->counter, 0, sizeof(unsigned)));
    CK(cudaMalloc(&c->dout, sizeof(double) * 8));
    CK(cudaMalloc(&c->dint, sizeof(int) * 4));
    c->group = std::make_shared<Group>();
    c->group->members = {c};
    CK(upload_basis(c->basis.D.data(), c->basis.w.data()));
    build_cell_records(c);
    CK(cudaStreamSynchronize(c->stream));
    *out = c;
  });
  if (rc != PERRK_OK && c) perrk_destroy(c);
  return rc;
}

int perrk_destroy(perrk_ctx* c) {
  if (!c) return PERRK_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  free_cell_buffers(c);
  for (double* p : {c->partials, c->dout, c->records})
    if (p) cudaFree(p);
  if (c->rec_host) cudaFreeHost(c->rec_host);
  for (int a = 0; a < 3; ++a)
    for (double* p : {c->dh[a], c->djac[a], c->dlift[a]})
      if (p) cudaFree(p);
  for (auto& p : c->plan)
    for (int* q : {p.dlist, p.glist, p.ilist, p.blist})
      if (q) cudaFree(q);
  if (c->st) cudaFree(c->st);
  for (int* p : {c->d_gid, c->d_nbr, c->d_send})
    if (p) cudaFree(p);
  if (c->d_ghost_gid) cudaFree(c->d_ghost_gid);
  if (c->d_rec) cudaFree(c->d_rec);
  if (c->counter) cudaFree(c->counter);
  if (c->dint) cudaFree(c->dint);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  for (auto& gr : c->graphs) cudaGraphExecDestroy(gr.exec);
  if (c->group) {  // leave the group (the exchange dies with its last member)
    auto& mem = c->group->members;
    for (size_t i = 0; i < mem.size(); ++i)
      if (mem[i] == c) {
        mem.erase(mem.begin() + static_cast<long>(i));
        break;
      }
    c->group.reset();
  }
  if (c->stream && c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
  return PERRK_OK;
}

int perrk_sizes(const perrk_ctx* c, int64_t* dofs, int64_t* nodes, int64_t* cells, int* vars,
                int* npc) {
  return guarded([&] {
    REQUIRE(c, "null context");
    if (dofs) *dofs = c->ndofs;
    if (nodes) *nodes = c->nnodes;
    if (cells) *cells = c->ncells;
    if (vars) *vars = c->V;
    if (npc) *npc = c->npc;
  });
}

int perrk_node_geometry(const perrk_ctx* c, double* x, double* y, double* z, double* measure) {
  return guarded([&] {
    REQUIRE(c, "null context");
    const auto& B = c->basis;
    for (long long cell = 0; cell < c->ncells; ++cell) {
      const long long g = c->slab ? c->gid[cell] : cell;
      const int ci = static_cast<int>(g % c->nc[0]);
      const int cj = static_cast<int>((g / c->nc[0]) % c->nc[1]);
      const int ck = static_cast<int>(g / (static_cast<long long>(c->nc[0]) * c->nc[1]));
      const int cj2 = cj;
      for (int l = 0; l < c->npc; ++l) {
        const int ix = l % 4, iy = (l / 4) % 4, iz = l / 16;
        const long long n = cell * c->npc + l;
        if (x) x[n] = c->edges[0][ci] + 0.5 * c->h[0][ci] * (B.x[ix] + 1.0);
        if (y) y[n] = c->edges[1][cj2] + 0.5 * c->h[1][cj2] * (B.x[iy] + 1.0);
        if (z && c->dim == 3) z[n] = c->edges[2][ck] + 0.5 * c->h[2][ck] * (B.x[iz] + 1.0);
        if (measure)
          measure[n] = c->dim == 2 ? 0.25 * c->h[0][ci] * c->h[1][cj2] * B.w[ix] * B.w[iy]
                                   : 0.125 * c->h[0][ci] * c->h[1][cj] * c->h[2][ck] * B.w[ix] *
                                         B.w[iy] * B.w[iz];
      }
    }
  });
}

int perrk_set_family(perrk_ctx* c, const perrk_family_desc* f, const int* eff) {
  return guarded([&] {
    REQUIRE(c && f && eff, "null argument");
    REQUIRE(f->S >= 1 && f->R >= 1 && f->R <= dev::MAXR, "family size out of range");
    set_device(c);
    c->S = f->S;
    c->R = f->R;
    c->E.assign(f->E, f->E + f->R);
    c->A.assign(f->A, f->A + static_cast<size_t>(f->R) * f->S * f->S);
    c->b.assign(f->b, f->b + f->S);
    c->c.assign(f->c, f->c + f->S);
    // the level map is global; the context keeps its own cells' part
    for (long long i = 0; i < c->ncells_global; ++i)
      REQUIRE(eff[i] >= 1 && eff[i] <= f->R, "level out of range");
    c->eff.resize(c->ncells);
    for (long long i = 0; i < c->ncells; ++i) c->eff[i] = eff[c->slab ? c->gid[i] : i];
    std::vector<int8_t> lv(c->ncells);
    for (long long i = 0; i < c->ncells; ++i) lv[i] = static_cast<int8_t>(c->eff[i]);
    CK(cudaMemcpy(c->dlevel, lv.data(), c->ncells, cudaMemcpyHostToDevice));
    build_cell_records(c);
    build_plan(c);
    c->has_family = true;
    c->plan_version += 1;
  });
}

int perrk_upload_state(perrk_ctx* c, const double* U, size_t n) {
  return guarded([&] {
    REQUIRE(c && U, "null argument");
    REQUIRE(static_cast<long long>(n) == c->ndofs, "state size mismatch");
    set_device(c);
    upload(c, c->U, U);
    CK(cudaStreamSynchronize(c->stream));
  });
}

int perrk_download_state(perrk_ctx* c, double* U, size_t n) {
  return guarded([&] {
    REQUIRE(c && U, "null argument");
    REQUIRE(static_cast<long long>(n) == c->ndofs, "state size mismatch");
    set_device(c);
    download(c, U, c->U);
  });
}

int perrk_state_device_ptr(perrk_ctx* c, double** p) {
  return guarded([&] {
    REQUIRE(c && p, "null argument");
    *p = c->U;
  });
}

int perrk_sync(perrk_ctx* c) {
  return guarded([&] {
    REQUIRE(c, "null context");
    set_device(c);
    CK(cudaStreamSynchronize(c->stream));
  });
}

int perrk_rhs_masked(perrk_ctx* c, double t, const double* U, double* out, const char* mask) {
  (void)t;  // the periodic 2D/3D RHS is autonomous (semidisc.cpp:411)
  return guarded([&] {
    REQUIRE(c && U && out, "null argument");
    no_slab(c, "rhs_masked");
    set_device(c);
    std::vector<int> list;
    for (long long i = 0; i < c->ncells; ++i)
      if (!mask || mask[i]) list.push_back(static_cast<int>(i));
    upload(c, c->tU, U);
    CK(cudaMemsetAsync(c->tK, 0, sizeof(double) * c->ndofs, c->stream));
    c->evals += static_cast<uint64_t>(list.size()) * c->npc * c->V;
    if (!list.empty()) {
      CK(cudaMemcpyAsync(c->dlist_tmp, list.data(), sizeof(int) * list.size(),
                         cudaMemcpyHostToDevice, c->stream));
      StepState s = fresh_state();
      put_state(c, s);
      StageArgs a{};
      a.U = c->tU;
      a.K1 = c->tU;
      a.Kout = c->tK;
      a.list = mask ? c->dlist_tmp : nullptr;
      a.n = static_cast<int>(list.size());
      a.write_k = 1;
      a.ncells = c->ncells_global;
      a.ndofs = c->ndofs;
      int* gl_dev = nullptr;
      if (c->physics == 1) {  // BR1 viscous fluxes on the cells and their neighbours
        std::vector<char> on(c->ncells, 0);
        for (int q : list) on[q] = 1;
        const std::vector<int> gl = with_neighbours_2d(c, on);
        CK(cudaMalloc(&gl_dev, sizeof(int) * gl.size()));
        CK(cudaMemcpyAsync(gl_dev, gl.data(), sizeof(int) * gl.size(), cudaMemcpyHostToDevice,
                           c->stream));
        StageArgs ga = a;
        ga.list = gl_dev;
        ga.n = static_cast<int>(gl.size());
        CK(launch_grad(ga, c->mesh(), c->ph, c->st, c->G, c->ndofs, 0, c->grid_stage, c->stream));
        a.G = c->G;
      }
      CK(launch_stage(c->dim, c->surface, c->vol(), a, c->mesh(), c->ph, c->st, c->partials, c->counter,
                      c->grid_stage, c->stream));
      if (gl_dev) {
        CK(cudaStreamSynchronize(c->stream));
        cudaFree(gl_dev);
      }
      const StepState r = get_state(c);
      if (r.bad_code != std::numeric_limits<long long>::max())
        throw Fail(PERRK_ENUMERIC, "inadmissible state passed to numerical flux");
    }
    download(c, out, c->tK);
  });
}

namespace {
// Full (unmasked) RHS of device state dU into dK, as perrk_rhs_masked(mask = NULL).
static void rhs_full_device(perrk_ctx* c, const double* dU, double* dK, int* gl_all) {
  CK(cudaMemsetAsync(dK, 0, sizeof(double) * c->ndofs, c->stream));
  c->evals += static_cast<uint64_t>(c->ncells) * c->npc * c->V;
  StepState s = fresh_state();
  put_state(c, s);
  StageArgs a{};
  a.U = dU;
  a.K1 = dU;
  a.Kout = dK;
  a.list = nullptr;
  a.n = static_cast<int>(c->ncells);
  a.write_k = 1;
  a.ncells = c->ncells_global;
  a.ndofs = c->ndofs;
  if (c->physics == 1) {
    StageArgs ga = a;
    ga.list = gl_all;
    CK(launch_grad(ga, c->mesh(), c->ph, c->st, c->G, c->ndofs, 0, c->grid_stage, c->stream));
    a.G = c->G;
  }
  CK(launch_stage(c->dim, c->surface, c->vol(), a, c->mesh(), c->ph, c->st, c->partials, c->counter,
                  c->grid_stage, c->stream));
  const StepState r = get_state(c);
  if (r.bad_code != std::numeric_limits<long long>::max())
    throw Fail(PERRK_ENUMERIC, "inadmissible state passed to numerical flux");
}

// Cells whose RHS rows read cell p: its face neighbours out to `rad` steps.
static std::vector<int> probe_stencil(const perrk_ctx* c, int p, int rad) {
  std::vector<int> out{p};
  size_t lo = 0;
  for (int r = 0; r < rad; ++r) {
    const size_t hi = out.size();
    for (size_t q = lo; q < hi; ++q)
      for (int f = 0; f < 2 * c->dim; ++f) {
        const int g = static_cast<int>(face_neighbour(c->dim, c->nc, out[q], f));
        if (std::find(out.begin(), out.end(), g) == out.end()) out.push_back(g);
      }
    lo = hi;
  }
  return out;
}
}  // namespace

int perrk_krylov_hessenberg(perrk_ctx* c, const double* base, double t, double epsilon, int m,
                            const char* cell_mask, double* H, int* m_done) {
  (void)t;  // autonomous RHS (semidisc.cpp:411)
  return guarded([&] {
    REQUIRE(c && H && m_done, "null argument");
    no_slab(c, "krylov_hessenberg");
    REQUIRE(m >= 1, "m must be at least 1");
    REQUIRE(std::isfinite(epsilon) && epsilon > 0.0, "epsilon must be positive");
    const long long M = c->ndofs;
    REQUIRE(m <= M, "m exceeds the number of DOFs");
    set_device(c);
    const int nc = static_cast<int>(c->ncells);
    const long long stride = static_cast<long long>(c->npc) * c->V;
    const int grid = c->grid_flat;
    std::vector<void*> bufs;
    auto dalloc = [&](size_t n) {
      void* q = nullptr;
      CK(cudaMalloc(&q, n));
      bufs.push_back(q);
      return q;
    };
    *m_done = 0;
    try {
      const size_t vb = sizeof(double) * M;
      double* Vb = static_cast<double*>(dalloc(vb * (m + 1)));  // Krylov basis
      double* dbase = static_cast<double*>(dalloc(vb));
      double* up = static_cast<double*>(dalloc(vb));
      double* um = static_cast<double*>(dalloc(vb));
      double* fp = static_cast<double*>(dalloc(vb));
      double* fm = static_cast<double*>(dalloc(vb));
      double* w = static_cast<double*>(dalloc(vb));
      const int nblk = c->grid_flat / 4;  // two blocks per SM
      double* partials = static_cast<double*>(dalloc(sizeof(double) * 2 * nblk * (m + 1)));
      double* coef = static_cast<double*>(dalloc(sizeof(double) * 2 * (m + 1)));
      unsigned char* dmask = nullptr;
      int* dall = static_cast<int*>(dalloc(sizeof(int) * nc));
      std::vector<int> all(nc);
      for (int p = 0; p < nc; ++p) all[p] = p;
      CK(cudaMemcpyAsync(dall, all.data(), sizeof(int) * nc, cudaMemcpyHostToDevice, c->stream));
      if (cell_mask) {
        dmask = static_cast<unsigned char*>(dalloc(nc));
        CK(cudaMemcpyAsync(dmask, cell_mask, nc, cudaMemcpyHostToDevice, c->stream));
      }
      // the base state and its max norm (the step scale of specopt.cpp:25-26)
      std::vector<double> hb;
      const double* bsrc = base;
      if (!base) {
        hb.resize(M);
        download(c, hb.data(), c->U);
        bsrc = hb.data();
      }
      double umax = 0.0;
      for (long long i = 0; i < M; ++i) umax = std::max(umax, std::fabs(bsrc[i]));
      upload(c, dbase, bsrc);
      const double h = epsilon * (1.0 + umax);
      std::vector<double> Hh(static_cast<size_t>(m + 1) * m, 0.0), c1(m + 1), c2(m + 1);
      auto norm2 = [&](const double* x) {
        CK(launch_krylov_dots(x, 0, 1, x, partials, nblk, coef, M, c->stream));
        double r = 0.0;
        CK(cudaMemcpyAsync(&r, coef, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return std::sqrt(r);
      };
      CK(launch_krylov_seed(Vb, dmask, stride, M, 0x5eedULL, grid, c->stream));
      const double n0 = norm2(Vb);
      REQUIRE(n0 > 0.0, "empty cell mask");
      CK(launch_krylov_scale(Vb, Vb, 1.0 / n0, M, grid, c->stream));
      int done = 0;
      for (int k = 0; k < m; ++k) {
        double* vk = Vb + static_cast<long long>(k) * M;
        CK(launch_krylov_perturb(up, um, dbase, vk, h, M, grid, c->stream));
        rhs_full_device(c, up, fp, dall);
        rhs_full_device(c, um, fm, dall);
        CK(launch_krylov_fd(w, fp, fm, 0.5 / h, dmask, stride, M, grid, c->stream));
        // classical Gram-Schmidt, applied twice (CGS2): orthogonal to working precision
        for (int pass = 0; pass < 2; ++pass) {
          CK(launch_krylov_dots(Vb, M, k + 1, w, partials, nblk, coef, M, c->stream));
          CK(launch_krylov_project(w, Vb, M, coef, k + 1, M, grid, c->stream));
          CK(cudaMemcpyAsync((pass ? c2 : c1).data(), coef, sizeof(double) * (k + 1),
                             cudaMemcpyDeviceToHost, c->stream));
        }
        const double beta = norm2(w);  // synchronizes: c1, c2 are on the host
        for (int j = 0; j <= k; ++j) Hh[j + static_cast<size_t>(m + 1) * k] = c1[j] + c2[j];
        Hh[k + 1 + static_cast<size_t>(m + 1) * k] = beta;
        done = k + 1;
        double col = 0.0;
        for (int j = 0; j <= k; ++j) col = std::max(col, std::fabs(c1[j] + c2[j]));
        if (!(beta > 1e-13 * col)) break;  // invariant subspace: the Ritz values are exact
        CK(launch_krylov_scale(Vb + static_cast<long long>(k + 1) * M, w, 1.0 / beta, M, grid,
                               c->stream));
      }
      CK(cudaStreamSynchronize(c->stream));
      std::copy(Hh.begin(), Hh.end(), H);
      *m_done = done;
    } catch (...) {
      cudaStreamSynchronize(c->stream);
      for (void* q : bufs) cudaFree(q);
      throw;
    }
    for (void* q : bufs) cudaFree(q);
  });
}

int perrk_probe_jacobian(perrk_ctx* c, const double* base, double t, double epsilon, double* J,
                         int* n_colours) {
  (void)t;  // autonomous RHS (semidisc.cpp:411)
  return guarded([&] {
    REQUIRE(c && base && J, "null argument");
    no_slab(c, "probe_jacobian");
    const long long M = c->ndofs;
    REQUIRE(M <= 5000, "dense Jacobian probing guarded to M <= 5000");
    REQUIRE(std::isfinite(epsilon) && epsilon > 0.0, "epsilon must be positive");
    set_device(c);
    const int nc = static_cast<int>(c->ncells);
    const long long stride = static_cast<long long>(c->npc) * c->V;
    // Distance-2 greedy colouring of the cells over the RHS dependency graph
    // (BR1 widens each stencil to two face steps, semidisc.cpp:254-263).
    const int rad = c->physics == 1 ? 2 : 1;
    std::vector<std::vector<int>> sten(nc);
    for (int p = 0; p < nc; ++p) sten[p] = probe_stencil(c, p, rad);
    std::vector<std::vector<int>> readers(nc);  // cells whose stencil holds q
    for (int p = 0; p < nc; ++p)
      for (int q : sten[p]) readers[q].push_back(p);
    std::vector<int> colour(nc, -1);
    int ncol = 0;
    for (int p = 0; p < nc; ++p) {
      std::vector<char> used(ncol + 1, 0);
      for (int q : sten[p])
        for (int o : readers[q])
          if (colour[o] >= 0) used[colour[o]] = 1;
      int k = 0;
      while (used[k]) ++k;
      colour[p] = k;
      ncol = std::max(ncol, k + 1);
    }
    std::vector<double> h(M);
    for (long long j = 0; j < M; ++j) h[j] = epsilon * (1.0 + std::fabs(base[j]));
    const size_t vb = sizeof(double) * M;
    std::vector<void*> bufs;
    auto dalloc = [&](size_t n) {
      void* q = nullptr;
      CK(cudaMalloc(&q, n));
      bufs.push_back(q);
      return q;
    };
    try {
      double* dJ = static_cast<double*>(dalloc(vb * M));
      double* dbase = static_cast<double*>(dalloc(vb));
      double* dh = static_cast<double*>(dalloc(vb));
      double* up = static_cast<double*>(dalloc(vb));
      double* um = static_cast<double*>(dalloc(vb));
      double* fp = static_cast<double*>(dalloc(vb));
      double* fm = static_cast<double*>(dalloc(vb));
      int* dcells = static_cast<int*>(dalloc(sizeof(int) * nc));
      int* downer = static_cast<int*>(dalloc(sizeof(int) * nc));
      int* dall = static_cast<int*>(dalloc(sizeof(int) * nc));
      std::vector<int> all(nc);
      for (int p = 0; p < nc; ++p) all[p] = p;
      CK(cudaMemcpyAsync(dall, all.data(), sizeof(int) * nc, cudaMemcpyHostToDevice, c->stream));
      upload(c, dbase, base);  // both to the device layout; the scatter writes J canonically
      upload(c, dh, h.data());
      CK(cudaMemcpyAsync(up, dbase, vb, cudaMemcpyDeviceToDevice, c->stream));
      CK(cudaMemcpyAsync(um, dbase, vb, cudaMemcpyDeviceToDevice, c->stream));
      CK(cudaMemsetAsync(dJ, 0, vb * M, c->stream));
      const int sgrid = static_cast<int>(std::min<long long>((M + 255) / 256, c->grid_flat));
      for (int k = 0; k < ncol; ++k) {
        std::vector<int> cells, owner(nc, -1);
        for (int p = 0; p < nc; ++p)
          if (colour[p] == k) {
            cells.push_back(p);
            for (int q : sten[p]) owner[q] = p;
          }
        CK(cudaMemcpyAsync(dcells, cells.data(), sizeof(int) * cells.size(),
                           cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(downer, owner.data(), sizeof(int) * nc, cudaMemcpyHostToDevice,
                           c->stream));
        const int n = static_cast<int>(cells.size());
        for (int l = 0; l < stride; ++l) {
          CK(launch_probe_set(up, um, dbase, dh, dcells, n, stride, l, 1, c->stream));
          rhs_full_device(c, up, fp, dall);
          rhs_full_device(c, um, fm, dall);
          CK(launch_probe_set(up, um, dbase, dh, dcells, n, stride, l, 0, c->stream));
          CK(launch_probe_scatter(dJ, fp, fm, dh, downer, M, stride, l, c->npc, sgrid,
                                  c->stream));
        }
        CK(cudaStreamSynchronize(c->stream));  // owner / cells host vectors die here
      }
      CK(cudaMemcpyAsync(J, dJ, vb * M, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
    } catch (...) {
      cudaStreamSynchronize(c->stream);
      for (void* q : bufs) cudaFree(q);
      throw;
    }
    for (void* q : bufs) cudaFree(q);
    if (n_colours) *n_colours = ncol;
  });
}

int perrk_br1_gradients(perrk_ctx* c, double t, const double* U, double* grads) {
  (void)t;
  return guarded([&] {
    REQUIRE(c && U && grads, "null argument");
    no_slab(c, "br1_gradients");
    if (c->physics != 1) throw Fail(PERRK_EUNSUP, "BR1 gradients need NSF physics");
    set_device(c);
    upload(c, c->tU, U);
    StepState s = fresh_state();
    put_state(c, s);
    StageArgs a{};
    a.U = a.K1 = c->tU;
    a.n = static_cast<int>(c->ncells);
    CK(launch_grad(a, c->mesh(), c->ph, c->st, c->G, c->ndofs, 1, c->grid_stage, c->stream));
    download(c, grads, c->G);                 // [0][dofs]: d/dx
    download(c, grads + c->ndofs, c->G + c->ndofs);  // [1][dofs]: d/dy
  });
}

int perrk_total_entropy(perrk_ctx* c, const double* U, double* out) {
  return guarded([&] {
    REQUIRE(c && out, "null argument");
    no_slab(c, "total_entropy");
    set_device(c);
    *out = quad(c, stage_input(c, U), nullptr, 0, nullptr);
  });
}

int perrk_entropy_inner_product(perrk_ctx* c, const double* U, const double* K, double* out) {
  return guarded([&] {
    REQUIRE(c && K && out, "null argument");
    no_slab(c, "entropy_inner_product");
    set_device(c);
    const double* dU = stage_input(c, U);
    upload(c, c->tK, K);
    *out = quad(c, dU, c->tK, 1, nullptr);
  });
}

int perrk_integral_per_variable(perrk_ctx* c, const double* U, double* out) {
  return guarded([&] {
    REQUIRE(c && out, "null argument");
    no_slab(c, "integral_per_variable");
    set_device(c);
    quad(c, stage_input(c, U), nullptr, 2, out);
  });
}

int perrk_admissible(perrk_ctx* c, const double* U, int* ok, int* first_bad) {
  return guarded([&] {
    REQUIRE(c && ok, "null argument");
    no_slab(c, "admissible");
    set_device(c);
    const double* dU = stage_input(c, U);
    const int init = std::numeric_limits<int>::max();
    CK(cudaMemcpyAsync(c->dint, &init, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    CK(launch_admissible(c->dim, dU, c->ph, c->dint, c->nnodes, c->grid_flat, c->stream));
    int bad;
    CK(cudaMemcpyAsync(&bad, c->dint, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    *ok = bad == init ? 1 : 0;
    if (first_bad) *first_bad = bad == init ? -1 : bad;
  });
}

int perrk_characteristic_speed(perrk_ctx* c, const double* U, double* nu) {
  return guarded([&] {
    REQUIRE(c && nu, "null argument");
    set_device(c);
    CK(launch_nu_cell(c->dim, stage_input(c, U), c->mesh(), c->ph, c->dnu, c->ncells, c->stream));
    CK(cudaMemcpyAsync(nu, c->dnu, sizeof(double) * c->ncells, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int perrk_compute_dt(perrk_ctx* c, const double* U, int fixed, double dt_or_cfl, double t,
                     double tf, double* dt) {
  return guarded([&] {
    REQUIRE(c && dt, "null argument");
    if (fixed) {
      REQUIRE(dt_or_cfl > 0.0, "fixed dt must be positive");
      *dt = std::fmin(dt_or_cfl, tf - t);
      return;
    }
    set_device(c);
    Group& g = *c->group;
    REQUIRE(g.members.size() == 1 || !U, "a loopback group takes the resident state (U = NULL)");
    StepState s = fresh_state();
    s.numax_bits = 0;
    for (perrk_ctx* m : g.members) {
      put_state(m, slab_state(m, s));
      CK(launch_numax(m->dim, m == c ? stage_input(c, U) : m->U, m->mesh(), m->ph, m->st,
                      m->nnodes, m->grid_flat, m->stream));
    }
    if (g.ex) reduce_point(g, RED_NUMAX, true);  // global max over the slabs
    const StepState r = get_state(c);
    double best;
    std::memcpy(&best, &r.numax_bits, sizeof best);
    const double nu_max = 4.0 * best;
    REQUIRE(nu_max > 0.0, "vanishing characteristic speed");
    *dt = dt_or_cfl / nu_max;
  });
}

static int step_common(perrk_ctx* c, double* t, double dt, const perrk_step_opts* o,
                       perrk_step_result* res) {
  return guarded([&] {
    REQUIRE(c && t && o && res, "null argument");
    REQUIRE(c->has_family, "no family set (perrk_set_family)");
    REQUIRE(dt > 0.0, "dt must be positive");
    if (o->relax_enabled) check_relax_cfg(o->relax);
    Group& g = *c->group;
    for (perrk_ctx* m : g.members) REQUIRE(m->has_family, "no family set on a group member");
    set_device(c);
    StepState s = fresh_state();
    s.t = *t;
    s.dt_mode = 0;
    s.dt_given = dt;
    s.gamma_override = o->gamma_override;
    s.gamma_seed = o->gamma_seed;
    s.h_ref = o->h_ref;
    s.idt = o->idt;
    configure_relax(s, o->relax_enabled != 0, o->relax);
    for (perrk_ctx* m : g.members) put_state(m, slab_state(m, s));
    StepMode mode;
    mode.relax = o->relax_enabled != 0;
    mode.cfg = o->relax;
    enqueue_step(g, mode, needs_h(mode.relax, o->relax, o->h_ref));
    const StepState r = get_state(c);
    if (r.error == 1) throw Fail(PERRK_ENUMERIC, "non-finite update direction");
    for (perrk_ctx* m : g.members) m->evals += evals_per_step(m);
    fill_result(c, r, mode.relax, o->gamma_override, res);
    if (!r.aborted) *t = r.t;
  });
}

int perrk_perk_step_resident(perrk_ctx* c, double* t, double dt, const perrk_step_opts* o,
                             perrk_step_result* res) {
  return step_common(c, t, dt, o, res);
}

int perrk_perk_step(perrk_ctx* c, double* U, double* t, double dt, const perrk_step_opts* o,
                    perrk_step_result* res) {
  int rc = guarded([&] {
    REQUIRE(c && U, "null argument");
    set_device(c);
    upload(c, c->U, U);
  });
  if (rc) return rc;
  rc = step_common(c, t, dt, o, res);
  if (rc) return rc;
  if (res->aborted) return PERRK_OK;  // U untouched on abort (stepper.hpp:70-71)
  return guarded([&] { download(c, U, c->U); });
}

int perrk_advance(perrk_ctx* c, const perrk_run_cfg* cfg, double* t, int nsteps,
                  perrk_step_record* log, int* steps_taken, int* aborted) {
  return guarded([&] {
    REQUIRE(c && cfg && t, "null argument");
    REQUIRE(c->has_family, "no family set (perrk_set_family)");
    REQUIRE(nsteps >= 0, "nsteps must be >= 0");
    if (cfg->relax_enabled) check_relax_cfg(cfg->relax);
    if (cfg->fixed_dt) REQUIRE(cfg->dt_or_cfl > 0.0, "fixed dt must be positive");
    set_device(c);
    StepState s = fresh_state();
    s.t = *t;
    s.run_mode = 1;
    s.tf = cfg->tf;
    s.t_eps = 1e-12 * std::fmax(1.0, std::fabs(cfg->tf));
    s.dt_mode = cfg->fixed_dt ? 1 : 2;
    s.dt_or_cfl = cfg->dt_or_cfl;
    s.cfl0 = cfg->cfl0;
    s.t_ramp = cfg->cfl0 == cfg->dt_or_cfl ? 0.0 : cfg->t_ramp;
    s.t0 = cfg->t0;
    s.idt = cfg->idt;
    // run() keeps the gamma seed and the anchor across its whole loop
    // (stepper.cpp:151,153,170): a continued run carries them in
    s.gamma_seed = cfg->carry ? cfg->gamma_seed : 1.0;
    if (cfg->carry) REQUIRE(cfg->gamma_seed > 0.0, "carried gamma seed must be positive");
    configure_relax(s, cfg->relax_enabled != 0, cfg->relax);
    if (cfg->relax_enabled && cfg->anchor_initial)
      s.h_ref = cfg->carry ? cfg->h_anchor : quad(c, c->U, nullptr, 0, nullptr);  // H(U_0)
    Group& g = *c->group;
    REQUIRE(!(g.ex && cfg->relax_enabled && cfg->anchor_initial),
            "anchored relaxation is not supported with the slab decomposition");
    for (perrk_ctx* m : g.members) {
      REQUIRE(m->has_family, "no family set on a group member");
      put_state(m, slab_state(m, s));
    }
    const bool rec = cfg->records && log;
    // record rows: at least 256, doubling, so that calls of growing length
    // keep the buffer (its address is part of the step-graph key below)
    auto rows_for = [](int have, int need) {
      int n = have > 256 ? have : 256;
      while (n < need) n *= 2;
      return n;
    };
    for (perrk_ctx* m : g.members)
      if (rec && m->records_cap < nsteps) {
        const int rows = rows_for(m->records_cap, nsteps);
        if (m->records) cudaFree(m->records);
        m->records = nullptr;
        m->records_cap = 0;
        CK(cudaMalloc(&m->records, sizeof(double) * dev::REC_COLS * rows));
        m->records_cap = rows;
      }
    if (rec && c->rec_host_cap < nsteps) {
      const int rows = rows_for(c->rec_host_cap, nsteps);
      if (c->rec_host) cudaFreeHost(c->rec_host);
      c->rec_host = nullptr;
      c->rec_host_cap = 0;
      CK(cudaMallocHost(&c->rec_host, sizeof(double) * dev::REC_COLS * rows));
      c->rec_host_cap = rows;
    }
    // each step's StepRecord row leaves for the host right after the step
    auto stream_rows = [&](int k0, int n) {
      if (!rec || n <= 0) return;
      const size_t off = static_cast<size_t>(k0) * dev::REC_COLS;
      CK(cudaMemcpyAsync(c->rec_host + off, c->records + off, sizeof(double) * dev::REC_COLS * n,
                         cudaMemcpyDeviceToHost, c->stream));
    };
    StepMode mode;
    mode.relax = cfg->relax_enabled != 0;
    mode.cfg = cfg->relax;
    mode.want_nu = !cfg->fixed_dt;
    mode.want_record = rec;
    mode.records = rec ? c->records : nullptr;
    if (!cfg->fixed_dt) {
      for (perrk_ctx* m : g.members) {
        CK(launch_numax(m->dim, m->U, m->mesh(), m->ph, m->st, m->nnodes, m->grid_flat,
                        m->stream));
        m->launches += 1;
      }
      if (g.ex) reduce_point(g, RED_NUMAX, true);
    }
    const bool want_h = needs_h(mode.relax, cfg->relax, s.h_ref);
    mode.fused = mode.relax && cfg->relax.numerics == 1 && cfg->relax.method == 0 &&
                 cfg->relax.max_iter >= 2 && !g.ex && g.members.size() == 1 && c->use_fused;
    if (mode.fused && !c->Ualt) CK(cudaMalloc(&c->Ualt, sizeof(double) * c->ndofs_()));
    double* const U_first = c->U;  // the state buffer of step 0; steps alternate with Ualt
    double* const U_second = c->Ualt;
    bool graphs = c->use_graphs && nsteps > 1;
    for (perrk_ctx* m : g.members) graphs = graphs && !m->profiling;
    if (graphs) {
      // every step enqueues the same launches with the same arguments (the
      // step-to-step state lives in the device StepState), so one captured
      // step is replayed nsteps times
      std::string key;
      for (perrk_ctx* m : g.members) key += std::to_string(m->plan_version) + ":" +
                                           std::to_string(reinterpret_cast<uintptr_t>(m->records)) + ";";
      key += std::to_string(reinterpret_cast<uintptr_t>(c->U)) + (mode.fused ? "F" : "-");
      // everything enqueue_step branches on: the relaxation method decides the
      // number of captured passes (relax_passes), so it is part of the key
      key += std::to_string(mode.relax) + std::to_string(mode.cfg.numerics) + ":" +
             std::to_string(mode.cfg.method) + ":" + std::to_string(relax_passes(mode.cfg)) +
             ":" + std::to_string(mode.cfg.max_iter) + std::to_string(mode.want_nu) +
             std::to_string(mode.want_record) + std::to_string(want_h);
      perrk_ctx::StepGraph* gr = nullptr;
      for (auto& x : c->graphs)
        if (x.key == key) gr = &x;
      if (!gr) {
        if (c->graphs.size() >= 4) {  // drop the oldest
          cudaGraphExecDestroy(c->graphs.front().exec);
          c->graphs.erase(c->graphs.begin());
        }
        const int64_t l0 = c->launches;
        cudaGraph_t graph;
        perrk_ctx::StepGraph ng;
        ng.key = key;
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed));
        enqueue_step(g, mode, want_h);
        if (mode.fused) enqueue_step(g, mode, want_h);  // two steps: the buffers are back in place
        CK(cudaStreamEndCapture(c->stream, &graph));
        CK(cudaGraphInstantiate(&ng.exec, graph, 0));
        cudaGraphDestroy(graph);
        ng.launches = c->launches - l0;
        c->launches = l0;
        c->graphs.push_back(ng);
        gr = &c->graphs.back();
      }
      const int per = mode.fused ? 2 : 1;
      int k = 0;
      for (; k + per <= nsteps; k += per) {
        CK(cudaGraphLaunch(gr->exec, c->stream));
        c->launches += gr->launches;
        stream_rows(k, per);
      }
      if (nsteps % per) {
        enqueue_step(g, mode, want_h);
        stream_rows(k, 1);
      }
    } else {
      for (int k = 0; k < nsteps; ++k) {
        enqueue_step(g, mode, want_h);
        stream_rows(k, 1);
      }
    }
    const StepState r = get_state(c);  // synchronizes: the streamed rows are on the host
    if (mode.fused) {  // the state of the last step taken (a stopped step writes nothing)
      const bool odd = (r.steps_taken & 1) != 0;
      c->U = odd ? U_second : U_first;
      c->Ualt = odd ? U_first : U_second;
    }
    if (r.error == 1) throw Fail(PERRK_ENUMERIC, "non-finite update direction");
    if (r.error == 2) throw Fail(PERRK_EINVAL, "vanishing characteristic speed");
    *t = r.t;
    if (steps_taken) *steps_taken = r.steps_taken;
    if (aborted) *aborted = r.aborted;
    for (perrk_ctx* m : g.members)
      m->evals += evals_per_step(m) * static_cast<uint64_t>(r.steps_taken + (r.aborted ? 1 : 0));
    if (rec && r.steps_taken > 0) {
      for (int k = 0; k < r.steps_taken; ++k) {
        const double* row = c->rec_host + static_cast<size_t>(k) * dev::REC_COLS;
        perrk_step_record& o = log[k];
        o.t = row[0];
        o.dt = row[1];
        o.gamma = row[2];
        o.newton_iters = static_cast<int>(row[3]);
        o.fell_back = static_cast<int>(row[4]);
        o.entropy = row[5];
        for (int v = 0; v < 5; ++v) o.invariants[v] = v < c->V ? row[6 + v] : 0.0;
        o.delta_h = row[11];
      }
    }
  });
}

int perrk_error_norms(perrk_ctx* c, const double* U, int exact, const double* params, double t,
                      double* l1, double* linf) {
  return guarded([&] {
    REQUIRE(c && params && l1 && linf, "null argument");
    no_slab(c, "error_norms");
    if (c->dim != 2 || exact != 0)
      throw Fail(PERRK_EUNSUP, "device error norms: 2D isentropic vortex (exact = 0)");
    set_device(c);
    // degree-2k GLL points and the interpolation matrix (basis.cpp:35-110)
    const Basis fine = make_basis(2 * c->basis.k);
    const int nf = static_cast<int>(fine.x.size()), n1 = c->basis.k + 1;
    std::vector<double> buf(2 * nf + nf * n1 + 8 + c->nc[0] + c->nc[1] + 4);
    std::copy(fine.x.begin(), fine.x.end(), buf.begin());
    std::copy(fine.w.begin(), fine.w.end(), buf.begin() + nf);
    std::vector<double> bw(n1, 1.0);
    for (int j = 0; j < n1; ++j)
      for (int q = 0; q < n1; ++q)
        if (q != j) bw[j] /= (c->basis.x[j] - c->basis.x[q]);
    for (int i = 0; i < nf; ++i) {
      double* row = &buf[2 * nf + i * n1];
      int hit = -1;
      for (int j = 0; j < n1; ++j)
        if (fine.x[i] == c->basis.x[j]) hit = j;
      if (hit >= 0) {
        for (int j = 0; j < n1; ++j) row[j] = j == hit ? 1.0 : 0.0;
        continue;
      }
      double den = 0.0;
      for (int j = 0; j < n1; ++j) den += bw[j] / (fine.x[i] - c->basis.x[j]);
      for (int j = 0; j < n1; ++j) row[j] = (bw[j] / (fine.x[i] - c->basis.x[j])) / den;
    }
    const size_t off_vp = 2 * nf + nf * n1, off_x = off_vp + 8, off_y = off_x + c->nc[0];
    std::copy(params, params + 8, buf.begin() + off_vp);
    for (int i = 0; i < c->nc[0]; ++i) buf[off_x + i] = c->edges[0][i];
    for (int j = 0; j < c->nc[1]; ++j) buf[off_y + j] = c->edges[1][j];
    double* dbuf = nullptr;
    unsigned long long* dmax = nullptr;
    CK(cudaMalloc(&dbuf, sizeof(double) * buf.size()));
    CK(cudaMalloc(&dmax, sizeof(unsigned long long) * 4));
    CK(cudaMemcpyAsync(dbuf, buf.data(), sizeof(double) * buf.size(), cudaMemcpyHostToDevice,
                       c->stream));
    CK(cudaMemsetAsync(dmax, 0, sizeof(unsigned long long) * 4, c->stream));
    CK(launch_error_norms(stage_input(c, U), c->mesh(), dbuf + off_x, dbuf + off_y, dbuf, nf,
                          dbuf + off_vp, t, c->partials, c->counter, c->dout, dmax, c->ncells,
                          c->grid_flat, c->stream));
    unsigned long long mx[4];
    CK(cudaMemcpyAsync(l1, c->dout, sizeof(double) * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(mx, dmax, sizeof mx, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(dbuf);
    cudaFree(dmax);
    double dom = 1.0;
    for (int a = 0; a < 2; ++a) dom *= c->edges[a].back() - c->edges[a].front();
    for (int v = 0; v < 4; ++v) {
      l1[v] /= dom;  // domain_measure (semidisc.cpp:71-72)
      std::memcpy(&linf[v], &mx[v], sizeof(double));
    }
  });
}

int perrk_rhs_cell_evaluations(const perrk_ctx* c, uint64_t* out) {
  return guarded([&] {
    REQUIRE(c && out, "null argument");
    *out = c->evals;
  });
}

int perrk_reset_counter(perrk_ctx* c) {
  return guarded([&] {
    REQUIRE(c, "null context");
    c->evals = 0;
  });
}

int perrk_family_build(int kind, int S, int R, const int* E, const double* free_flat,
                       double c_sm3, double* A, double* b, double* cc, int* active) {
  return guarded([&] {
    REQUIRE(E && A && b && cc, "null argument");
    REQUIRE(kind >= 0 && kind <= 3, "unknown family kind");
    REQUIRE(S >= (kind == PERRK_FAMILY_P4 ? 5 : 3), "too few stages for archetype");
    REQUIRE(R >= 1, "empty member list");
    for (int r = 1; r < R; ++r) REQUIRE(E[r] > E[r - 1], "E must be strictly increasing");
    REQUIRE(E[R - 1] == S, "largest member must have E = S");
    const auto bw = weights_b(kind, S);
    const auto cw = abscissae(kind, S, c_sm3);
    size_t off = 0;
    for (int r = 0; r < R; ++r) {
      double* Am = A + static_cast<size_t>(r) * S * S;
      build_member(kind, S, E[r], free_flat ? free_flat + off : nullptr, bw, cw, Am);
      off += free_count(kind, E[r]);
      const auto act = reachable_stages(S, Am, bw);
      int n = 0;
      for (int i = 0; i < S; ++i) {
        n += act[i];
        if (active) active[r * S + i] = act[i];
      }
      REQUIRE(n == E[r], "active stage set does not match E");
    }
    std::copy(bw.begin(), bw.end(), b);
    std::copy(cw.begin(), cw.end(), cc);
  });
}

int perrk_assign_levels(const double* nu, int64_t n, int R, int* levels) {
  return guarded([&] {
    REQUIRE(R >= 1, "R must be at least 1");
    REQUIRE(n > 0 && nu && levels, "empty speed list");
    double nu_max = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      REQUIRE(nu[i] > 0.0, "characteristic speeds must be positive");
      nu_max = std::fmax(nu_max, nu[i]);
    }
    int max_assigned = 1;
    for (int64_t i = 0; i < n; ++i) {
      // cells within a factor 2^(r-1) of the fastest get level r
      int r = 1 + static_cast<int>(std::ceil(std::log2(nu_max / nu[i]) - 1e-12));
      r = r < 1 ? 1 : (r > R ? R : r);
      levels[i] = r;
      max_assigned = r > max_assigned ? r : max_assigned;
    }
    const int shift = R - max_assigned;  // slowest cells on the cheapest member
    if (shift > 0)
      for (int64_t i = 0; i < n; ++i) levels[i] += shift;
  });
}

int perrk_make_partition_map(int dim, const int* n, const int* levels, int R, int* eff) {
  return guarded([&] {
    REQUIRE(R >= 1, "R must be at least 1");
    REQUIRE(dim >= 1 && dim <= 3 && n && levels && eff, "bad arguments");
    const int nx = n[0], ny = dim >= 2 ? n[1] : 1, nz = dim == 3 ? n[2] : 1;
    const long long N = static_cast<long long>(nx) * ny * nz;
    for (long long i = 0; i < N; ++i)
      REQUIRE(levels[i] >= 1 && levels[i] <= R, "level out of range");
    for (int k = 0; k < nz; ++k)
      for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
          const long long cell = i + static_cast<long long>(nx) * (j + static_cast<long long>(ny) * k);
          int lv = levels[cell];
          auto nb = [&](int ii, int jj, int kk) {
            ii = (ii + nx) % nx;
            jj = (jj + ny) % ny;
            kk = (kk + nz) % nz;
            const int o = levels[ii + static_cast<long long>(nx) * (jj + static_cast<long long>(ny) * kk)];
            lv = o < lv ? o : lv;
          };
          nb(i - 1, j, k);
          nb(i + 1, j, k);
          nb(i, j - 1, k);
          nb(i, j + 1, k);
          if (dim == 3) {
            nb(i, j, k - 1);
            nb(i, j, k + 1);
          }
          eff[cell] = lv;
        }
  });
}

int perrk_set_stream(perrk_ctx* c, void* stream) {
  return guarded([&] {
    REQUIRE(c, "null context");
    set_device(c);
    CK(cudaStreamSynchronize(c->stream));
    if (c->own_stream) CK(cudaStreamDestroy(c->stream));
    if (stream) {
      c->stream = static_cast<cudaStream_t>(stream);
      c->own_stream = false;
    } else {
      CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
  });
}

int perrk_profile(perrk_ctx* c, int enable) {
  return guarded([&] {
    REQUIRE(c, "null context");
    c->profiling = enable != 0;
    c->ev_used = 0;
    c->ev_bytes.clear();
  });
}

int perrk_profile_read(perrk_ctx* c, double* stage_ms, int64_t* stage_launches,
                       double* stage_bytes) {
  return guarded([&] {
    REQUIRE(c, "null context");
    set_device(c);
    CK(cudaStreamSynchronize(c->stream));
    double ms = 0.0, bytes = 0.0;
    int64_t n = 0;
    for (size_t q = 0; q + 1 < c->ev_used; q += 2) {
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, c->ev_pool[q], c->ev_pool[q + 1]));
      ms += t;
      bytes += c->ev_bytes[q / 2];
      ++n;
    }
    if (stage_ms) *stage_ms = ms;
    if (stage_launches) *stage_launches = n;
    if (stage_bytes) *stage_bytes = bytes;
  });
}

int perrk_launch_count(const perrk_ctx* c, int64_t* out) {
  return guarded([&] {
    REQUIRE(c && out, "null argument");
    *out = c->launches;
  });
}

int perrk_step_traffic(const perrk_ctx* c, double* stage_bytes, double* pass_bytes,
                       double* update_bytes) {
  return guarded([&] {
    REQUIRE(c, "null context");
    double s = 0.0;
    for (const auto& p : c->plan) s += p.bytes;
    if (stage_bytes) *stage_bytes = s;
    if (pass_bytes) *pass_bytes = 16.0 * c->V * c->nnodes;    // read U, d
    if (update_bytes) *update_bytes = 24.0 * c->V * c->nnodes;  // read U, d; write U
  });
}

int perrk_update_matrix(const perrk_advection_desc* ad, const perrk_family_desc* f,
                        const int* eff, double dt, double gamma, double* D, int64_t* Mout) {
  return guarded([&] {
    REQUIRE(ad && Mout, "null argument");
    REQUIRE(ad->dim == 1 || ad->dim == 2, "advection runs on 1D or 2D meshes");
    const int sf = ad->surface_flux;
    if (sf == PERRK_FLUX_HLLE) throw Fail(PERRK_EINVAL, "HLLE flux not available for this physics");
    if (sf == PERRK_FLUX_HLLC) throw Fail(PERRK_EINVAL, "HLLC flux not available for this physics");
    REQUIRE(sf == PERRK_FLUX_CENTRAL || sf == PERRK_FLUX_UPWIND || sf == PERRK_FLUX_RUSANOV ||
                sf == PERRK_FLUX_EC,
            "unknown surface flux");
    REQUIRE(ad->volume_mode == 0 || ad->volume_mode == 1, "volume_mode must be 0 (weak) or 1");
    if (ad->volume_mode == 1 && ad->volume_flux != PERRK_FLUX_EC &&
        ad->volume_flux != PERRK_FLUX_CENTRAL)
      throw Fail(PERRK_EINVAL, "flux differencing needs a symmetric consistent volume flux");
    const int npc = ad->dim == 1 ? 4 : 16;
    long long ncells = 1;
    std::vector<double> hs[2];
    for (int a = 0; a < ad->dim; ++a) {
      REQUIRE(ad->n[a] >= 1 && ad->edges[a], "bad mesh");
      ncells *= ad->n[a];
      for (int i = 0; i < ad->n[a]; ++i) {
        const double h = ad->edges[a][i + 1] - ad->edges[a][i];
        REQUIRE(h > 0.0, "edges must be strictly increasing");
        hs[a].push_back(h);
      }
    }
    const long long M = ncells * npc;
    *Mout = M;
    if (!D) return;
    REQUIRE(f && eff, "null argument");
    REQUIRE(dt > 0.0, "dt must be positive");
    REQUIRE(f->S >= 1 && f->R >= 1 && f->R <= dev::MAXR, "family size out of range");
    const int S = f->S, R = f->R;
    std::vector<double> A(f->A, f->A + static_cast<size_t>(R) * S * S), b(f->b, f->b + S);
    for (long long i = 0; i < ncells; ++i) REQUIRE(eff[i] >= 1 && eff[i] <= R, "level out of range");
    CK(cudaSetDevice(ad->device));
    const Basis B = make_basis(3);
    CK(upload_basis(B.D.data(), B.w.data()));
    // per-level rows and activity (member R - level, butcher.hpp:47)
    std::vector<std::vector<char>> active(R);
    for (int lvl = 1; lvl <= R; ++lvl)
      active[lvl - 1] = reachable_stages(S, &A[static_cast<size_t>(R - lvl) * S * S], b);
    DeviceBuffers buf;
    AdvArgs base{};
    base.dim = ad->dim;
    for (int a = 0; a < 2; ++a) {
      base.nc[a] = a < ad->dim ? ad->n[a] : 1;
      base.a[a] = a < ad->dim ? ad->velocity[a] : 0.0;
      if (a < ad->dim) {
        double* h = buf.get<double>(hs[a].size());
        CK(cudaMemcpy(h, hs[a].data(), sizeof(double) * hs[a].size(), cudaMemcpyHostToDevice));
        base.h[a] = h;
      }
    }
    std::vector<int8_t> lv(eff, eff + ncells);
    int8_t* dl = buf.get<int8_t>(ncells);
    CK(cudaMemcpy(dl, lv.data(), ncells, cudaMemcpyHostToDevice));
    base.level = dl;
    base.surface = sf;
    base.volume_flux = ad->volume_flux;
    base.weak = ad->volume_mode == 0;
    base.M = M;
    base.dt = dt;
    std::vector<int*> lists(S, nullptr);
    std::vector<int> nlist(S, 0);
    for (int i = 0; i < S; ++i) {
      std::vector<int> l;
      for (long long cell = 0; cell < ncells; ++cell)
        if (i == 0 || active[eff[cell] - 1][i]) l.push_back(static_cast<int>(cell));
      nlist[i] = static_cast<int>(l.size());
      if (nlist[i] > 0 && nlist[i] < ncells) {
        lists[i] = buf.get<int>(l.size());
        CK(cudaMemcpy(lists[i], l.data(), sizeof(int) * l.size(), cudaMemcpyHostToDevice));
      }
    }
    // column chunk: K1, two K buffers, d and the output chunk (5 x B x M doubles)
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    const double budget = std::min(0.5 * static_cast<double>(free_b), 16.0e9);
    long long Bc = static_cast<long long>(budget / (5.0 * 8.0 * static_cast<double>(M)));
    Bc = std::max(1LL, std::min(Bc, M));
    double* K1 = buf.get<double>(static_cast<size_t>(Bc) * M);
    double* Kb[2] = {buf.get<double>(static_cast<size_t>(Bc) * M),
                     buf.get<double>(static_cast<size_t>(Bc) * M)};
    double* d = buf.get<double>(static_cast<size_t>(Bc) * M);
    double* Dd = buf.get<double>(static_cast<size_t>(Bc) * M);
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ad->device));
    for (long long col0 = 0; col0 < M; col0 += Bc) {
      const int nc = static_cast<int>(std::min(Bc, M - col0));
      CK(cudaMemset(d, 0, sizeof(double) * static_cast<size_t>(nc) * M));
      for (int i = 0; i < S; ++i) {
        AdvArgs a = base;
        a.col0 = col0;
        a.ncols = nc;
        a.stage = i;
        a.K1 = K1;
        a.Kp = i >= 2 ? Kb[(i - 1) & 1] : K1;
        a.Kout = i == 0 ? K1 : Kb[i & 1];
        a.d = d;
        a.b = b[i];
        a.list = lists[i];
        a.nlist = nlist[i];
        for (int lvl = 1; lvl <= R; ++lvl) {
          const double* Am = &A[static_cast<size_t>(R - lvl) * S * S];
          a.a1[lvl] = i >= 1 ? Am[static_cast<size_t>(i) * S] : 0.0;
          a.ap[lvl] = i >= 2 ? Am[static_cast<size_t>(i) * S + i - 1] : 0.0;
        }
        const long long work = static_cast<long long>(nlist[i]) * npc * nc;
        if (work == 0) continue;
        const int grid = static_cast<int>(std::min<long long>((work + 255) / 256, 16LL * sms));
        CK(launch_adv_stage(a, grid, nullptr));
      }
      const long long n = static_cast<long long>(nc) * M;
      CK(launch_adv_final(d, M, col0, nc, gamma * dt, Dd,
                          static_cast<int>(std::min<long long>((n + 255) / 256, 16LL * sms)),
                          nullptr));
      CK(cudaMemcpy(D + static_cast<size_t>(col0) * M, Dd, sizeof(double) * n,
                    cudaMemcpyDeviceToHost));
    }
  });
}

int perrk_fp64_peak(int device, double* gflops) {
  return guarded([&] {
    REQUIRE(gflops, "null argument");
    CK(cudaSetDevice(device));
    *gflops = measure_fp64_peak();
  });
}

int perrk_nccl_id(void* out) {
  return guarded([&] {
    REQUIRE(out, "null argument");
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof id);
  });
}

int perrk_comm_init(perrk_ctx* c, const void* nccl_id, int rank, int nranks, const int* owner) {
  return guarded([&] {
    REQUIRE(c && nccl_id, "null argument");
    if (nranks == 1) return;  // the whole periodic mesh: nothing to exchange
    make_partition(c, rank, nranks, owner);
    auto ex = std::make_unique<NcclExchange>();
    ex->setup();
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof id);
    set_device(c);
    NK(ncclCommInitRank(&ex->comm, nranks, id, rank));
    c->group->ex = std::move(ex);
  });
}

int perrk_loopback_group(perrk_ctx** ctxs, int n, const int* owner) {
  return guarded([&] {
    REQUIRE(ctxs && n >= 2, "need at least two contexts");
    for (int r = 0; r < n; ++r) {
      REQUIRE(ctxs[r], "null context");
      REQUIRE(ctxs[r]->device == ctxs[0]->device, "loopback contexts share one device");
      REQUIRE(ctxs[r]->ncells_global == ctxs[0]->ncells_global, "contexts of different meshes");
    }
    auto g = std::make_shared<Group>();
    g->ex = std::make_unique<LoopbackExchange>();
    set_device(ctxs[0]);
    CK(cudaStreamCreateWithFlags(&g->shared_stream, cudaStreamNonBlocking));
    for (int r = 0; r < n; ++r) {
      perrk_ctx* c = ctxs[r];
      make_partition(c, r, n, owner);
      // one stream, owned by the group (it outlives every member), orders
      // every member's work
      CK(cudaStreamSynchronize(c->stream));
      if (c->own_stream) CK(cudaStreamDestroy(c->stream));
      c->stream = g->shared_stream;
      c->own_stream = false;
      g->members.push_back(c);
      c->group = g;
    }
  });
}

int perrk_local_cells(const perrk_ctx* c, int* gids, int64_t* n) {
  return guarded([&] {
    REQUIRE(c && n, "null argument");
    *n = c->ncells;
    if (gids)
      for (long long i = 0; i < c->ncells; ++i) gids[i] = c->slab ? c->gid[i] : static_cast<int>(i);
  });
}

namespace {
long long global_cells(int dim, const int* n) {
  REQUIRE((dim == 2 || dim == 3) && n && n[0] >= 1 && n[1] >= 1 && (dim == 2 || n[2] >= 1),
          "bad mesh shape");
  return static_cast<long long>(n[0]) * n[1] * (dim == 3 ? n[2] : 1);
}
}  // namespace

int perrk_partition_slabs(int dim, const int* n, const double* cell_work, int nranks, int* owner) {
  return guarded([&] {
    const long long NG = global_cells(dim, n);
    const int nl = n[dim - 1];
    const long long lc = NG / nl;
    REQUIRE(owner && nranks >= 1 && nranks <= nl, "bad arguments");
    // contiguous last-axis layers, cut where the running work crosses
    // r / nranks of the total, every rank >= 1 layer
    std::vector<double> pre(nl + 1, 0.0);
    for (int l = 0; l < nl; ++l) {
      double w = 0.0;
      for (long long i = 0; i < lc; ++i) w += cell_work ? cell_work[l * lc + i] : 1.0;
      pre[l + 1] = pre[l] + w;
    }
    std::vector<int> cuts(nranks + 1, 0);
    for (int r = 1; r < nranks; ++r) {
      const double target = pre[nl] * r / nranks;
      int l = cuts[r - 1] + 1;
      while (l < nl - (nranks - r) && pre[l] + 0.5 * (pre[l + 1] - pre[l]) < target) ++l;
      cuts[r] = l;
    }
    cuts[nranks] = nl;
    for (int r = 0; r < nranks; ++r)
      for (long long g = cuts[r] * lc; g < cuts[r + 1] * lc; ++g) owner[g] = r;
  });
}

int perrk_partition_levels(int dim, const int* n, const int* level, int nlevels, int nranks,
                           int* owner) {
  return guarded([&] {
    const long long NG = global_cells(dim, n);
    REQUIRE(level && owner && nlevels >= 1 && nranks >= 1, "bad arguments");
    // every level's cells, in global (last-axis-major) order, cut into nranks
    // contiguous runs of equal size: each rank holds 1/nranks of every level,
    // so every stage's active set is balanced, and a run is a band of layers
    std::vector<long long> cnt(nlevels + 1, 0), seen(nlevels + 1, 0);
    for (long long g = 0; g < NG; ++g) {
      REQUIRE(level[g] >= 1 && level[g] <= nlevels, "level out of range");
      ++cnt[level[g]];
    }
    for (long long g = 0; g < NG; ++g) {
      const int l = level[g];
      owner[g] = static_cast<int>(seen[l]++ * nranks / cnt[l]);
    }
    std::vector<char> has(nranks, 0);
    for (long long g = 0; g < NG; ++g) has[owner[g]] = 1;
    for (int r = 0; r < nranks; ++r) REQUIRE(has[r], "more ranks than cells");
  });
}

int perrk_halo_plan(int dim, const int* n, const int* owner, int rank, int64_t* counts, int* gid,
                    int* nbr, int64_t* ghost_gid, int* peers, int64_t* recv_off,
                    int64_t* send_off, int* send) {
  return guarded([&] {
    const long long NG = global_cells(dim, n);
    REQUIRE(owner && counts, "null argument");
    for (long long g = 0; g < NG; ++g) REQUIRE(owner[g] >= 0, "negative owner");
    HaloPlan h = halo_plan(dim, n, owner, rank);
    counts[0] = static_cast<int64_t>(h.gid.size());
    counts[1] = static_cast<int64_t>(h.ghost_gid.size());
    counts[2] = static_cast<int64_t>(h.send.size() / 2);
    counts[3] = static_cast<int64_t>(h.peers.size());
    auto put = [](auto* dst, const auto& src) {
      if (dst) std::copy(src.begin(), src.end(), dst);
    };
    put(gid, h.gid);
    put(nbr, h.nbr);
    put(ghost_gid, h.ghost_gid);
    put(peers, h.peers);
    put(recv_off, h.recv_off);
    put(send_off, h.send_off);
    put(send, h.send);
  });
}

int perrk_face_nodes(int dim, int face, int* nodes) {
  return guarded([&] {
    REQUIRE((dim == 2 || dim == 3) && face >= 0 && face < 2 * dim && nodes, "bad arguments");
    // trace point pt of face f (pack_traces_kernel / the stage kernel's ghost read)
    const int d = face >> 1, side = face & 1, fp = dim == 3 ? 16 : 4;
    const int stride = d == 0 ? 1 : (d == 1 ? 4 : 16);
    for (int pt = 0; pt < fp; ++pt) {
      const int t1 = pt % 4, t2 = pt / 4;
      const int base = dim == 2 ? (d == 0 ? 4 * t1 : t1)
                                : (d == 0 ? 4 * t1 + 16 * t2 : (d == 1 ? t1 + 16 * t2 : t1 + 4 * t2));
      nodes[pt] = base + (side ? 3 : 0) * stride;
    }
  });
}

}  // extern "C"
