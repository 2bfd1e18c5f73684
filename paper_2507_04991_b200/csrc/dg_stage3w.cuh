// Stage kernel, 3D Euler with the EC volume flux and the Rusanov / central
// surface flux: one warp per cell, two LGL nodes per lane, no block barriers.
//
// Same work per active cell as stage_kernel (dg_stage.cuh; reference
// semidisc.cpp:409-557 via rhs_masked :126-138, stepper.cpp:52-92 around it):
// stage-state formation, flux-differencing volume term with the Ranocha EC
// flux, surface flux + strong-form lift + endpoint diagonal term, b-stage
// epilogue and the next stage's formed state.
//
// Mapping.  A 4x4x4 cell (node n = ix + 4 iy + 16 iz) is one warp: lane l
// owns nodes A = l (iz = l >> 4 in {0, 1}) and B = l + 32 (iz + 2).  Then
//   * x- and y-lines lie in groups of four lanes, once for the A layer and
//     once for the B layer: each node evaluates its pair (j, j+1 mod 4) and
//     receives (j-1, j) by shuffle; the distance-2 pairs of the two layers
//     are split between the lanes (j < 2: the A pair, j >= 2: the B pair) and
//     exchanged with a lane^2 (x) / lane^8 (y) shuffle;
//   * z-lines pair lane l with lane l^16: the distance-2 pair (A, B) is inside
//     the lane, and each node's (j, j+1 mod 4) pair goes to the partner lane
//     by a lane^16 shuffle.
// So every lane evaluates exactly 9 EC fluxes (4.5 per node, each pair once)
// and 3 face points (96 per cell, one direction per round, compile time).
// Warps never wait for one another: the cell's primitives and surface terms
// live in the warp's own shared-memory slice, ordered by __syncwarp.  The
// neighbours' face traces are staged into that slice with cp.async while the
// volume terms are computed.
//
// What binds it (profiles/r02_stage_kernel_ncu.txt): the L1 data pipe (shared
// loads / stores, shuffles, global accesses: 70% of its peak), the FP64 pipe
// (50%) and the issue slots (55%) together, at 3 warps per scheduler.  The
// defaults below are the winners of the same-box A/B runs in
// profiles/r02_ab.txt: fewer wavefronts (own primitives, descriptor and
// z-face terms through registers), straight-line phases (hoisted descriptor
// reads, branch-free staging / surface / gather), and no cache pollution
// (direct streaming epilogue, no bulk L2 prefetch).  The switches keep the
// rejected forms buildable (profiles/tools/mk_variant.sh).
#pragma once

namespace perrk {
namespace dev {

#ifndef PERRK_W3_DESC_CA
#define PERRK_W3_DESC_CA 0  // 1: descriptor prefetch through L1 (cp.async.ca)
#endif

#ifndef PERRK_W3_NOSEL
#define PERRK_W3_NOSEL 0  // 1: distance-2 exchange without selects
#endif

#ifndef PERRK_W3_COAL
// 1: epilogue U / K1 / U_{i+1} blocks through the slice (the round-1 form, for
// the canonical AoS layout); 0: direct loads and stores, which the device
// layout makes coalesced 256-byte warp accesses (A/B: -4% stage time)
#define PERRK_W3_COAL 0
#endif

#ifndef PERRK_W3_WPB
// warps (cells in flight) per block; the default is one 12-warp block per SM
// at 168 registers (two 8-warp blocks at 128 registers: PERRK_W3_WPB=8)
#define PERRK_W3_WPB 12
#endif

#ifndef PERRK_W3_HALFP
#define PERRK_W3_HALFP 1  // 1: the slice holds p / 2 (the EC flux's pressure terms take it as is)
#endif

#ifndef PERRK_W3_OWNPF
#define PERRK_W3_OWNPF 0  // 1: the next cell's own stage-state block arrives by cp.async a cell ahead
#endif

#ifndef PERRK_W3_REGPF
// the next cell's own stage state is loaded into registers a cell ahead
// (coalesced loads of the device layout; its L2 latency hides behind the
// current cell's 1: surface phase and epilogue, 2: epilogue; 3: issued after
// the epilogue, ahead of the next cell's descriptor round trip); 0: loaded at
// the top of its own cell
#define PERRK_W3_REGPF 0
#endif

#ifndef PERRK_W3_L2PF
#define PERRK_W3_L2PF 0  // 1: the next cell's state blocks are bulk-prefetched to L2 a cell ahead; 2: see below
#endif

#ifndef PERRK_W3_CS
// 1: the direct epilogue's read-once / write-once streams (U, K1, d, U_{i+1},
// K_0) use the streaming cache operator (evict first), so that L2 keeps the
// stage-state blocks the neighbours' traces come from
#define PERRK_W3_CS 1
#endif

#ifndef PERRK_W3_EPIREG
// 1 (direct epilogue only): the epilogue's U and K1 values are loaded into
// registers right after the volume phase, so their latency hides behind the
// surface phase
#define PERRK_W3_EPIREG 1
#endif

#ifndef PERRK_W3_EPIPF
// 1: the lines of the epilogue's U / K1 blocks are prefetched (prefetch.global.L1,
// one or two lines per lane) right after the volume phase: the register-free
// form of PERRK_W3_EPIREG for the 128-register configuration
#define PERRK_W3_EPIPF 0
#endif

#ifndef PERRK_W3_DESCREG
// 1: the next cell's descriptor travels through a register of lanes 0-5
// (one 16-byte load a cell ahead, one 16-byte shared store at the top of its
// cell) instead of cp.async (13 L1 wavefronts per cell for its 96 bytes)
#define PERRK_W3_DESCREG 1
#endif

#ifndef PERRK_W3_ZREG
// 1 (with PERRK_W3_ZOWN and PERRK_W3_OWNREG): the z-face round runs first and
// takes its own-side primitives, E and c from the lane's registers
#define PERRK_W3_ZREG 0
#endif

#ifndef PERRK_W3_HOIST
// 1: the descriptor's neighbour ids and the neighbours' formed flags are read
// once at the top of the cell (their shared / constant load latencies
// overlap), the surface phase loads its slot unconditionally, and the
// gather is branch free (0/1 weights instead of divergent blocks)
#define PERRK_W3_HOIST 1
#endif

#ifndef PERRK_W3_FLAT
// 1 (with PERRK_W3_HOIST): the three surface rounds form one straight-line
// block.  Neighbours formed from U and K1 (first active stage of a level) are
// written into their slots by a warp-uniform pre-pass, the admissibility
// report is made once after the rounds, and the z-face terms are added with
// 0/1 weights, so the scheduler can overlap the rounds' dependent chains.
#define PERRK_W3_FLAT 1
#endif

#ifndef PERRK_W3_OWNL1PF
// 1: the 20 lines of the next cell's own stage-state block are prefetched to
// L1 (prefetch.global.L1, lanes 0-19) after the volume phase; 2: after the gather
#define PERRK_W3_OWNL1PF 0
#endif

#ifndef PERRK_W3_UNFPF
#define PERRK_W3_UNFPF 0  // 1: K1 traces of neighbours formed in the surface pre-pass are prefetched to L2 at staging
#endif

#ifndef PERRK_W3_RSQ
#define PERRK_W3_RSQ 1  // 1: beta and the sound speed of the own nodes from one reciprocal square root (A/B -0.8%)
#endif

#ifndef PERRK_W3_OWNCG
#define PERRK_W3_OWNCG 0  // 1: the own formed stage state is loaded past L1 (ld.global.cg); 2: with L1::evict_last
#endif

#ifndef PERRK_W3_ZOWN
#define PERRK_W3_ZOWN 1  // 1: z-face terms are added by the lane that computes them (it owns the node)
#endif

#ifndef PERRK_W3_EPI
#define PERRK_W3_EPI 0  // 1: the epilogue's U / K1 blocks arrive by bulk copies issued at cell start
#endif

struct W3 {
  static constexpr int V = 5, NPC = 64, FP = 16, WPB = PERRK_W3_WPB, T = 32 * WPB;
  // Shared-memory layouts chosen so that every warp access of the kernel is
  // free of bank conflicts (profiles/r01_x1_*: the L1/shared data pipe, not
  // the FP64 pipe, binds this kernel).
  //  * primitives: four arrays of 16-byte pairs, (rho, beta), (vx, vy),
  //    (vz, p), (E, c), 64 nodes each, node n at entry w3_sw(n): the low three
  //    bits of n XORed with h((n >> 3) & 3), h = {0, 1, 6, 7}.  Each of the
  //    kernel's access patterns (own node, x/y/z partners and distance-2
  //    pairs, the face nodes of the three surface rounds) then puts the eight
  //    lanes of every quarter-warp on eight distinct 16-byte bank groups.
  //  * face slots: 5 doubles (40 bytes) per slot, slot s at w3_fs(s) =
  //    s + 4 (s >> 4), read and written with 8-byte accesses: lane-indexed
  //    staging / surface and the node-indexed gather are all conflict free.
  static constexpr int NPR = 8;
  static constexpr int SM_PR = NPR * NPC;
  static constexpr int FS = 5;
  static constexpr int SM_FS = (96 + 4 * 5) * FS;
  // PERRK_W3_EPI: a dedicated [U | K1] epilogue block pair after the slice,
  // filled by two bulk copies at the start of the cell (their latency hides
  // behind the cell's whole volume and surface phases); d (b-stages only)
  // still comes through the dead slice
  static constexpr int SM_EP = PERRK_W3_EPI ? 2 * NPC * V : 0;
  // PERRK_W3_OWNPF: the next cell's own stage-state block ([v][64], read by
  // lane with conflict-free 8-byte loads)
  static constexpr int SM_OB = PERRK_W3_OWNPF ? NPC * V : 0;
  static constexpr int SM_WARP = SM_PR + SM_FS + SM_EP + SM_OB;
  static_assert(SM_PR + SM_FS >= (PERRK_W3_EPI ? 1 : 3) * NPC * V,
                "the epilogue stages its blocks in the slice");
  static_assert(SM_WARP % 2 == 0, "16-byte aligned slices");
  static constexpr int SM_TOTAL = WPB * SM_WARP;  // doubles per block
};

// swizzled entry of node n in the primitive arrays
__device__ __forceinline__ int w3_sw(int n) {
  const int k = (n >> 3) & 3;
  return n ^ ((k & 1) | ((k >> 1) * 6));
}

// first double of face slot s
__device__ __forceinline__ int w3_fs(int s) { return (s + 4 * (s >> 4)) * W3::FS; }

// a face slot (5 doubles) with 8-byte shared loads / stores
__device__ __forceinline__ void w3_slot_load(const double* p, double (&u)[5]) {
#pragma unroll
  for (int v = 0; v < 5; ++v) u[v] = p[v];
}

__device__ __forceinline__ void w3_slot_store(double* p, const double (&u)[5]) {
#pragma unroll
  for (int v = 0; v < 5; ++v) p[v] = u[v];
}

// the flux inputs of one node from the warp slice (three 16-byte loads)
struct W3Prim {
  double rho, beta, v[3], p;
};

__device__ __forceinline__ W3Prim w3_load(const double* pr, int n) {
  const double2* q = reinterpret_cast<const double2*>(pr) + w3_sw(n);
  const double2 a = q[0], b = q[W3::NPC], c = q[2 * W3::NPC];
  W3Prim r;
  r.rho = a.x;
  r.beta = a.y;
  r.v[0] = b.x;
  r.v[1] = b.y;
  r.v[2] = c.x;
  r.p = c.y;
  return r;
}

#ifndef PERRK_W3_MINB
#define PERRK_W3_MINB (16 / PERRK_W3_WPB)
#endif

// node on face (d, side) at face point pt (t1 + 4 t2, the line_base order)
__device__ __forceinline__ int w3_face_node(int d, int side, int pt) {
  const int t1 = pt & 3, t2 = pt >> 2;
  return d == 0 ? 3 * side + 4 * t1 + 16 * t2
                : (d == 1 ? t1 + 12 * side + 16 * t2 : t1 + 4 * t2 + 48 * side);
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async16_ca(void* dst, const void* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int NPENDING>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(NPENDING) : "memory");
}

// bulk (TMA-path) store of a shared-memory block to global memory: the
// writing lanes fence their generic-proxy stores first; one lane issues
__device__ __forceinline__ void bulk_store_fence() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void bulk_store(double* gdst, const double* ssrc, unsigned bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(ssrc));
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// the source of every committed bulk store has been read (smem reusable)
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// per-warp mbarrier of the epilogue blocks (PERRK_W3_EPI): lane 0 arms it
// with the byte count and issues the bulk loads, which complete the
// transaction; the lanes wait on the phase parity before reading
__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_load(double* sdst, const double* gsrc, unsigned bytes,
                                          unsigned long long* bar) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(d), "l"(gsrc), "r"(bytes), "r"(b)
      : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "W3_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W3_WAIT;\n"
      "}\n" ::"r"(b),
      "r"(parity)
      : "memory");
}

// a load that asks L1 to keep its line (PERRK_W3_OWNCG == 2)
__device__ __forceinline__ double w3_ld_l1last(const double* p) {
  double x;
  asm volatile("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(x) : "l"(p));
  return x;
}

// one cell's contiguous block of a state array (64 V doubles) into the warp's slice
__device__ __forceinline__ void w3_stage_cell(double* dst, const double* src, int lane) {
#pragma unroll
  for (int k = 0; k < W3::NPC * W3::V / 2 / 32; ++k)
    cp_async16(dst + 2 * (lane + 32 * k), src + 2 * (lane + 32 * k));
}

#ifndef PERRK_W3_SWZ
#define PERRK_W3_SWZ 1  // 1: partner entries by XOR masks of the own entry (no per-load swizzle arithmetic)
#endif

// the same from a swizzled entry e = w3_sw(n)
__device__ __forceinline__ W3Prim w3_load_e(const double* pr, int e) {
  const double2* q = reinterpret_cast<const double2*>(pr) + e;
  const double2 a = q[0], b = q[W3::NPC], c = q[2 * W3::NPC];
  W3Prim r;
  r.rho = a.x;
  r.beta = a.y;
  r.v[0] = b.x;
  r.v[1] = b.y;
  r.v[2] = c.x;
  r.p = c.y;
  return r;
}

// EC flux between smem nodes p and q in direction D (compile time).  With
// PERRK_W3_SWZ p and q are swizzled entries: w3_sw(n) = n ^ (iy >> 1) ^ 6 (iz & 1),
// so the entry of a node that differs from n in given coordinate bits is the
// entry of n XOR a mask, and the entry of n + 32 is the entry of n plus 32.
template <int D, bool SM>
__device__ __forceinline__ void w3_ec(const Phys& ph, const double* pr, int p, int q, double* f) {
#if PERRK_W3_SWZ
  const W3Prim L = w3_load_e(pr, p), R = w3_load_e(pr, q);
#else
  const W3Prim L = w3_load(pr, p), R = w3_load(pr, q);
#endif
  ec2<3, SM, PERRK_W3_HALFP != 0>(ph, D, L.rho, L.v, L.p, L.beta, R.rho, R.v, R.p, R.beta, f);
}

#ifndef PERRK_W3_OWNREG
// 1: the lane's own primitives stay in registers from the primitive pass
// (the slice is read for partners only): 12 fewer 16-byte shared loads per
// lane and cell; the L1 data pipe, at 70-80% of its peak, binds this kernel
#define PERRK_W3_OWNREG 1
#endif

// EC flux between the register-held node L and the smem entry q (needs PERRK_W3_SWZ)
template <int D, bool SM>
__device__ __forceinline__ void w3_ec_r(const Phys& ph, const double* pr, const W3Prim& L, int q,
                                        double* f) {
  const W3Prim R = w3_load_e(pr, q);
  ec2<3, SM, PERRK_W3_HALFP != 0>(ph, D, L.rho, L.v, L.p, L.beta, R.rho, R.v, R.p, R.beta, f);
}

__device__ __forceinline__ W3Prim w3_select(bool first, const W3Prim& a, const W3Prim& b) {
  W3Prim r;
  r.rho = first ? a.rho : b.rho;
  r.beta = first ? a.beta : b.beta;
#pragma unroll
  for (int i = 0; i < 3; ++i) r.v[i] = first ? a.v[i] : b.v[i];
  r.p = first ? a.p : b.p;
  return r;
}

// x / y lines (D = 0, 1): the lane's two layers.  Each node evaluates
// f(j, j+1 mod 4) and receives f(j-1, j); the distance-2 pairs: lanes with
// j < 2 evaluate the A layer's (j, j+2), lanes with j >= 2 the B layer's
// (j-2, j), exchanged with the lane 2 stride(D) positions away.
template <int D, bool SM>
__device__ __forceinline__ void w3_inplane(const Phys& ph, const double* pr, int lane, int j,
                                           double J2, double* KA, double* KB, const W3Prim& oA,
                                           const W3Prim& oB) {
  constexpr int V = W3::V;
  constexpr int st = D == 0 ? 1 : 4;  // lane / node stride along the line
  const int kn = (j + 1) & 3, kp = (j + 3) & 3;
  const double cn = J2 * c_D[j * N1 + kn], cp = J2 * c_D[j * N1 + kp], c2 = J2 * c_D[j * N1 + (j ^ 2)];
  const int pn = lane + (kn - j) * st;  // partner lane for (j, j+1)
  const int src = lane + (kp - j) * st;
  double f[V];
#if PERRK_W3_SWZ
  // entries: own A (eA), its line partner (j, j+1 mod 4), and the distance-2 partner
  const int eA = w3_sw(lane);
  const int mnext = D == 0 ? (1 | ((j & 1) << 1)) : (4 | ((j & 1) * 9));
  const int ePn = eA ^ mnext;
  constexpr int m2 = D == 0 ? 2 : 9;
#define W3_NODE_A eA
#define W3_NODE_PA ePn
#define W3_NODE_B (eA + 32)
#define W3_NODE_PB (ePn + 32)
#else
#define W3_NODE_A lane
#define W3_NODE_PA pn
#define W3_NODE_B (lane + 32)
#define W3_NODE_PB (pn + 32)
#endif
  // A layer
#if PERRK_W3_OWNREG
  w3_ec_r<D, SM>(ph, pr, oA, W3_NODE_PA, f);
#else
  w3_ec<D, SM>(ph, pr, W3_NODE_A, W3_NODE_PA, f);
#endif
#pragma unroll
  for (int v = 0; v < V; ++v) {
    KA[v] = fma(-cn, f[v], KA[v]);
    KA[v] = fma(-cp, __shfl_sync(0xffffffffu, f[v], src), KA[v]);
  }
  // B layer
#if PERRK_W3_OWNREG
  w3_ec_r<D, SM>(ph, pr, oB, W3_NODE_PB, f);
#else
  w3_ec<D, SM>(ph, pr, W3_NODE_B, W3_NODE_PB, f);
#endif
#undef W3_NODE_A
#undef W3_NODE_PA
#undef W3_NODE_B
#undef W3_NODE_PB
#pragma unroll
  for (int v = 0; v < V; ++v) {
    KB[v] = fma(-cn, f[v], KB[v]);
    KB[v] = fma(-cp, __shfl_sync(0xffffffffu, f[v], src), KB[v]);
  }
  // distance 2: j < 2 -> (A_j, A_j+2); j >= 2 -> (B_j, B_j-2)
  const bool lo = j < 2;
#if PERRK_W3_SWZ
  const int own = lo ? eA : eA + 32;
#if PERRK_W3_OWNREG
  w3_ec_r<D, SM>(ph, pr, w3_select(lo, oA, oB), own ^ m2, f);
#else
  w3_ec<D, SM>(ph, pr, own, own ^ m2, f);
#endif
#else
  const int own = lo ? lane : lane + 32;
  w3_ec<D, SM>(ph, pr, own, own ^ (2 * st), f);
#endif
#if PERRK_W3_NOSEL
  // no selects: the pair's two terms weighted by c2 or 0 (DFMA instead of FSEL pairs)
  const double cA = lo ? c2 : 0.0, cB = lo ? 0.0 : c2;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double r = __shfl_xor_sync(0xffffffffu, f[v], 2 * st);
    KA[v] = fma(-cA, f[v], fma(-cB, r, KA[v]));
    KB[v] = fma(-cB, f[v], fma(-cA, r, KB[v]));
  }
#else
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double r = __shfl_xor_sync(0xffffffffu, f[v], 2 * st);
    KA[v] = fma(-c2, lo ? f[v] : r, KA[v]);
    KB[v] = fma(-c2, lo ? r : f[v], KB[v]);
  }
#endif
}

// z lines: lane l holds z = zA and zA + 2, lane l^16 the other two.
template <bool SM>
__device__ __forceinline__ void w3_z(const Phys& ph, const double* pr, int lane, int zA,
                                     double J2, double* KA, double* KB, const W3Prim& oA,
                                     const W3Prim& oB) {
  constexpr int V = W3::V;
  const int zB = zA + 2;
  double f[V];
#if PERRK_W3_SWZ
  const int nA = w3_sw(lane), nB = nA + 32;  // own entries
#else
  const int nA = lane, nB = lane + 32;
#endif
  // distance 2 inside the lane: (A, B)
#if PERRK_W3_OWNREG
  ec2<3, SM, PERRK_W3_HALFP != 0>(ph, 2, oA.rho, oA.v, oA.p, oA.beta, oB.rho, oB.v, oB.p, oB.beta, f);
#else
  w3_ec<2, SM>(ph, pr, nA, nB, f);
#endif
  const double cab = J2 * c_D[zA * N1 + zB], cba = J2 * c_D[zB * N1 + zA];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    KA[v] = fma(-cab, f[v], KA[v]);
    KB[v] = fma(-cba, f[v], KB[v]);
  }
  // (j, j+1 mod 4) of both nodes; partner lane l^16 holds the j+1 nodes:
  // zA = 0: A(0)-A'(1), B(2)-B'(3);  zA = 1: A(1)-B'(2), B(3)-A'(0)
#if PERRK_W3_SWZ
  const int pl = nA ^ 22;  // lane ^ 16 flips iz & 1: node bit 4 and the swizzle's 6
#else
  const int pl = lane ^ 16;
#endif
  const int pA = zA ? pl + 32 : pl, pB = zA ? pl : pl + 32;
  const double cnA = J2 * c_D[zA * N1 + ((zA + 1) & 3)], cnB = J2 * c_D[zB * N1 + ((zB + 1) & 3)];
  const double cpA = J2 * c_D[zA * N1 + ((zA + 3) & 3)], cpB = J2 * c_D[zB * N1 + ((zB + 3) & 3)];
  double g[V];
#if PERRK_W3_OWNREG
  w3_ec_r<2, SM>(ph, pr, oA, pA, f);  // A's (j, j+1): to the partner's node pA
  w3_ec_r<2, SM>(ph, pr, oB, pB, g);  // B's (j, j+1): to the partner's node pB
#else
  w3_ec<2, SM>(ph, pr, nA, pA, f);  // A's (j, j+1): to the partner's node pA
  w3_ec<2, SM>(ph, pr, nB, pB, g);  // B's (j, j+1): to the partner's node pB
#endif
  // received: the partner's pair ending at my node.  Partner zA' = 1 - zA:
  // zA = 0 -> its A pair (1,2) ends at my B, its B pair (3,0) at my A;
  // zA = 1 -> its A pair (0,1) ends at my A, its B pair (2,3) at my B.
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double rA = __shfl_xor_sync(0xffffffffu, f[v], 16);
    const double rB = __shfl_xor_sync(0xffffffffu, g[v], 16);
    KA[v] = fma(-cnA, f[v], KA[v]);
    KB[v] = fma(-cnB, g[v], KB[v]);
    KA[v] = fma(-cpA, zA ? rA : rB, KA[v]);
    KB[v] = fma(-cpB, zA ? rB : rA, KB[v]);
  }
}

// FORM / NEXT / DM >= 0 fix a.form, a.write_next and a.d_mode at compile time
// (the stage kinds every P-ERK step launches: stage 0, interior stages, the
// b-stages); -1 reads them from the arguments
template <int SURF, int FORM = -1, int NEXT = -1, int DM = -1>
__global__ void __launch_bounds__(W3::T, PERRK_W3_MINB)
    stage3w_kernel(StageArgs a, MeshDev m, Phys ph, StepState* st, double* partials,
                   unsigned* counter) {
  using S = W3;
  constexpr int V = S::V, N = S::NPC, FP = S::FP;
  const bool form_ = FORM >= 0 ? (FORM != 0) : (a.form != 0);
  const bool next_ = NEXT >= 0 ? (NEXT != 0) : (a.write_next != 0);
  const int dm_ = DM >= 0 ? DM : a.d_mode;
  extern __shared__ double smem[];
  __shared__ double s_red[2 * 2 * S::WPB];
  __shared__ CellRec s_rec[S::WPB][2];  // descriptors, prefetched one cell ahead
#if PERRK_W3_EPI
  __shared__ unsigned long long s_mbar[S::WPB];
#endif
  if (st->aborted || st->finished) return;  // uniform across the grid
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* pr = smem + wib * S::SM_WARP;  // [4][64] double2, swizzled (w3_sw)
  double* fs = pr + S::SM_PR;            // face slots (w3_fs): staged traces, then surface terms
#if PERRK_W3_OWNPF
  double* ob = fs + S::SM_FS + S::SM_EP;  // the next cell's own block
  // the block a cell's own state comes from: Us (formed) or U (stage 0);
  // a cell formed from the first column (rare) reads U and K1 directly
  const double* own_src = form_ ? a.Us : a.U;
#endif
#if PERRK_W3_EPI
  double* ep = fs + S::SM_FS;            // epilogue blocks [U | K1] (device layout)
  unsigned ep_phase = 0;
  if (lane == 0) mbar_init(&s_mbar[wib]);
  __syncwarp();
#endif
  // descriptor of one cell into the warp's buffer b (lanes 0-5, 16 B each)
#if PERRK_W3_DESCREG
  static_assert(!PERRK_W3_OWNPF, "PERRK_W3_DESCREG assumes the trace group is the only cp.async group");
  int4 recq = make_int4(0, 0, 0, 0);
  auto fetch_rec = [&](int, int c) {
    if (c >= 0 && lane < static_cast<int>(sizeof(CellRec) / 16))
      recq = __ldg(reinterpret_cast<const int4*>(m.rec + c) + lane);
  };
#else
  auto fetch_rec = [&](int b, int c) {
    if (c >= 0 && lane < static_cast<int>(sizeof(CellRec) / 16))
#if PERRK_W3_DESC_CA
      cp_async16_ca(reinterpret_cast<char*>(&s_rec[wib][b]) + 16 * lane,
                    reinterpret_cast<const char*>(m.rec + c) + 16 * lane);
#else
      cp_async16(reinterpret_cast<char*>(&s_rec[wib][b]) + 16 * lane,
                 reinterpret_cast<const char*>(m.rec + c) + 16 * lane);
#endif
    cp_async_commit();
  };
#endif
  const double dt = st->dt;
#if PERRK_W3_RSQ
  const double sqrt_gamma = sqrt(ph.gamma);
#endif
  const int ix = lane & 3, iy = (lane >> 2) & 3, zA = lane >> 4, zB = zA + 2;
  const int side = zA, pt = lane & 15;
  dd acc_dh = dd_zero(), acc_h = dd_zero();
  unsigned long long dmax_bits = 0;
  const int nw = gridDim.x * S::WPB;
  int slot = blockIdx.x * S::WPB + wib;
  auto cell_at = [&](int sl) { return sl < a.n ? (a.list ? a.list[sl] : sl) : -1; };
  int cell = cell_at(slot);
  int ncell = cell_at(slot + nw);  // list entries are read one cell ahead of their use
  int rb = 0;
  fetch_rec(0, cell);
#if PERRK_W3_OWNPF
  if (cell >= 0) {
    w3_stage_cell(ob, own_src + static_cast<size_t>(cell) * N * V, lane);
    cp_async_commit();
  }
#endif

#if PERRK_W3_REGPF
  // own stage state of a cell into registers (coalesced: variable v of node
  // n at block + v N + n); a cell formed from the first column reads stale
  // Us here and is redone at its top
  double uA[V], uB[V];
  const double* own_reg = form_ ? a.Us : a.U;
  auto load_own = [&](int c) {
    const double* g = own_reg + static_cast<size_t>(c) * N * V + lane;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      uA[v] = __ldg(g + v * N);
      uB[v] = __ldg(g + v * N + 32);
    }
  };
  if (cell >= 0) load_own(cell);
#endif

  while (cell >= 0) {
    // next cell: its state arrays to L2 (bulk prefetch); the one after: list entry
    const int nslot = slot + nw;
    const int nncell = cell_at(nslot + nw);
    if (PERRK_W3_L2PF == 1 && lane == 0 && ncell >= 0) {
      constexpr unsigned kBytes = N * V * sizeof(double);
      const size_t off = static_cast<size_t>(ncell) * N * V;
      if (form_) l2_prefetch(a.Us + off, kBytes);
      if (!form_ || next_) l2_prefetch(a.U + off, kBytes);  // stage 0 state / epilogue
      if (next_ && form_) l2_prefetch(a.K1 + off, kBytes);
      if (dm_ == 2) l2_prefetch(a.d + off, kBytes);
    }
    // ---- descriptor (host.cpp build_cell_records), fetched a cell ago -------
#if PERRK_W3_DESCREG
    if (lane < static_cast<int>(sizeof(CellRec) / 16))
      reinterpret_cast<int4*>(&s_rec[wib][0])[lane] = recq;
#else
    cp_async_wait<0>();
#endif
    if (PERRK_W3_COAL && lane == 0) bulk_wait_read();  // the previous U_{i+1} left the slice
    __syncwarp();
    const CellRec* rp = &s_rec[wib][PERRK_W3_DESCREG ? 0 : rb];
    const unsigned long long lv =
        static_cast<unsigned long long>(*reinterpret_cast<const long long*>(rp->lev));
    const int lev = static_cast<int>(lv & 0xff);
    const double J2x = rp->J2[0], J2y = rp->J2[1], J2z = rp->J2[2];
    // ---- own nodes A, B: formed stage state (stepper.cpp:60-72) -------------
    // device layout (sidx): variable v of node n at cbase + v N + n, so each
    // load below is one coalesced 256-byte warp access
    const size_t cbase = static_cast<size_t>(cell) * N * V;
#if PERRK_W3_EPI
    // the epilogue's U (and K1) blocks, in flight for the whole cell
    if (next_ && lane == 0) {
      constexpr unsigned kBytes = N * V * sizeof(double);
      mbar_expect_tx(&s_mbar[wib], form_ ? 2 * kBytes : kBytes);
      bulk_load(ep, a.U + cbase, kBytes, &s_mbar[wib]);
      if (form_) bulk_load(ep + N * V, a.K1 + cbase, kBytes, &s_mbar[wib]);
    }
#endif
    const size_t gA = cbase + lane, gB = gA + 32;
#if PERRK_W3_REGPF
    // uA / uB arrived a cell ago from Us (U at stage 0); a cell formed from
    // the first column (first active stage of its level) is redone here
    if (form_ && !a.formed[lev]) {
      const double a1 = dt * a.a1[lev];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        uA[v] = fma(a1, __ldg(a.K1 + gA + v * N), __ldg(a.U + gA + v * N));
        uB[v] = fma(a1, __ldg(a.K1 + gB + v * N), __ldg(a.U + gB + v * N));
      }
    }
#else
    double uA[V], uB[V];
#endif
#if PERRK_W3_REGPF
#elif PERRK_W3_OWNPF
    if (!form_ || a.formed[lev]) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        uA[v] = ob[v * N + lane];
        uB[v] = ob[v * N + lane + 32];
      }
    } else
#endif
#if !PERRK_W3_REGPF
    if (!form_) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        uA[v] = __ldg(a.U + gA + v * N);
        uB[v] = __ldg(a.U + gB + v * N);
      }
    } else if (a.formed[lev]) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        uA[v] = PERRK_W3_OWNCG == 2 ? w3_ld_l1last(a.Us + gA + v * N)
                : PERRK_W3_OWNCG  ? __ldcg(a.Us + gA + v * N) : __ldg(a.Us + gA + v * N);
        uB[v] = PERRK_W3_OWNCG == 2 ? w3_ld_l1last(a.Us + gB + v * N)
                : PERRK_W3_OWNCG  ? __ldcg(a.Us + gB + v * N) : __ldg(a.Us + gB + v * N);
      }
    } else {
      const double a1 = dt * a.a1[lev];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        uA[v] = fma(a1, __ldg(a.K1 + gA + v * N), __ldg(a.U + gA + v * N));
        uB[v] = fma(a1, __ldg(a.K1 + gB + v * N), __ldg(a.U + gB + v * N));
      }
    }
#endif
    // ---- neighbour face traces -> the warp's face slots (cp.async), one
    // direction per round: round d, face 2 d + side, point pt -------------------
#if PERRK_W3_HOIST
    int nb3[3];
    unsigned unf = 0;  // bit d: the neighbour on (d, side) is formed from U and K1 in the surface phase
#pragma unroll
    for (int d = 0; d < 3; ++d) nb3[d] = rp->nb[2 * d + side];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int l2 = static_cast<int>((lv >> (8 * (1 + 2 * d + side))) & 0xff);
      if (form_ && nb3[d] >= 0 && !a.formed[l2]) unf |= 1u << d;
    }
#endif
#pragma unroll
    for (int d = 0; d < 3; ++d) {
#if PERRK_W3_HOIST
      const int nbc = nb3[d];
#else
      const int nbc = rp->nb[2 * d + side];
#endif
      double* dst = fs + w3_fs(d * 32 + lane);
#if PERRK_W3_FLAT && PERRK_W3_HOIST
      {
        // branch free: a ghost trace is point-major [pt][V], a cell block
        // variable-major; of a neighbour that is formed in the surface
        // pre-pass the U trace is copied (K1 is added there)
        const bool gh = nbc < 0;
        const double* src =
            gh ? m.ghost + (static_cast<size_t>(-1 - nbc) * FP + pt) * V
               : ((form_ && !((unf >> d) & 1u)) ? a.Us : a.U) + static_cast<size_t>(nbc) * N * V +
                     w3_face_node(d, 1 - side, pt);
        const int vs = gh ? 1 : N;
#pragma unroll
        for (int v = 0; v < V; ++v) cp_async8(dst + v, src + v * vs);
#if PERRK_W3_UNFPF
        // the K1 trace the pre-pass will read: towards L2 now
        if ((unf >> d) & 1u) {
          const double* k1 = a.K1 + static_cast<size_t>(nbc) * N * V + w3_face_node(d, 1 - side, pt);
#pragma unroll
          for (int v = 0; v < V; ++v) asm volatile("prefetch.global.L2 [%0];" ::"l"(k1 + v * N));
        }
#endif
        continue;
      }
#endif
      if (nbc < 0) {
        const double* g = m.ghost + (static_cast<size_t>(-1 - nbc) * FP + pt) * V;
#pragma unroll
        for (int v = 0; v < V; ++v) cp_async8(dst + v, g + v);
      } else {
        const size_t gi = static_cast<size_t>(nbc) * N * V + w3_face_node(d, 1 - side, pt);
#if PERRK_W3_HOIST
        if (!((unf >> d) & 1u)) {
          const double* src = (form_ ? a.Us : a.U) + gi;
#pragma unroll
          for (int v = 0; v < V; ++v) cp_async8(dst + v, src + v * N);
        }  // else: formed from U and K1 in the surface phase (first active stage only)
#else
        const int l2 = static_cast<int>((lv >> (8 * (1 + 2 * d + side))) & 0xff);
        if (!form_) {
#pragma unroll
          for (int v = 0; v < V; ++v) cp_async8(dst + v, a.U + gi + v * N);
        } else if (a.formed[l2]) {
#pragma unroll
          for (int v = 0; v < V; ++v) cp_async8(dst + v, a.Us + gi + v * N);
        }  // else: formed from U and K1 in the surface phase (first active stage only)
#endif
      }
    }
    cp_async_commit();
    fetch_rec(rb ^ 1, ncell);  // the next cell's descriptor
#if PERRK_W3_OWNPF
    __syncwarp();  // every lane has its own state out of the buffer
    if (ncell >= 0) w3_stage_cell(ob, own_src + static_cast<size_t>(ncell) * N * V, lane);
    cp_async_commit();  // (empty past the end) waited at the top of the next cell
#endif
    // ---- primitives of A and B -> the warp's slice -------------------------
    bool okAB = true;
    W3Prim own[2];  // the lane's nodes A and B (PERRK_W3_OWNREG: used by the volume phase)
    double2 ownEc[2];  // (E, c) of A and B (PERRK_W3_ZREG: the z-face round)
    // range of rho and beta over the cell from the high words of the doubles
    // (monotone for positive values; a negative or NaN value lands at the top)
    unsigned hr_lo = 0xffffffffu, hr_hi = 0u, hb_lo = 0xffffffffu, hb_hi = 0u;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int n = lane + 32 * h;
      double ir;
      const Prim<3> q = prim_of<3>(ph, h ? uB : uA, ir);
      okAB = okAB & prim_ok<3>(q);
#if PERRK_W3_RSQ
      // beta = rho / p and c = sqrt(gamma p / rho) from one reciprocal square
      // root of x = p / rho: beta = y^2, c = sqrt(gamma) x y (Rusanov only)
      double be, cs_;
      if (SURF == 2) {
        const double x = q.p * ir;
        const double y = frsqrt(x);
        be = y * y;
        cs_ = sqrt_gamma * (x * y);
      } else {
        be = q.rho * frcp(q.p);
        cs_ = 0.0;
      }
#else
      const double be = q.rho * frcp(q.p);
      const double cs_ = SURF == 2 ? fsqrt(ph.gamma * q.p * ir) : 0.0;
#endif
      double2* dst = reinterpret_cast<double2*>(pr) + w3_sw(n);
      own[h].rho = q.rho;
      own[h].beta = be;
      own[h].v[0] = q.v[0];
      own[h].v[1] = q.v[1];
      own[h].v[2] = q.v[2];
      own[h].p = PERRK_W3_HALFP ? 0.5 * q.p : q.p;
      dst[0] = make_double2(q.rho, be);
      dst[N] = make_double2(q.v[0], q.v[1]);
      dst[2 * N] = make_double2(q.v[2], PERRK_W3_HALFP ? 0.5 * q.p : q.p);
      ownEc[h] = make_double2(q.E, cs_);
      dst[3 * N] = ownEc[h];
      const unsigned hr = static_cast<unsigned>(__double2hiint(q.rho));
      const unsigned hb = static_cast<unsigned>(__double2hiint(be));
      hr_lo = min(hr_lo, hr);
      hr_hi = max(hr_hi, hr);
      hb_lo = min(hb_lo, hb);
      hb_hi = max(hb_hi, hb);
    }
    if (!okAB) report_bad(st, a.stage, a.ncells, m.gid ? m.gid[cell] : cell);
    // smooth cell: max / min < 1.0198 for both, so every pair of the cell has
    // ((a - b) / (a + b))^2 < 9.6e-5, below logmean's series threshold 1e-4
    // (physics.cpp:32) with margin; true values lie below hi + 1
    bool smooth;
    {
      hr_lo = __reduce_min_sync(0xffffffffu, hr_lo);
      hr_hi = __reduce_max_sync(0xffffffffu, hr_hi);
      hb_lo = __reduce_min_sync(0xffffffffu, hb_lo);
      hb_hi = __reduce_max_sync(0xffffffffu, hb_hi);
      auto ratio_ok = [](unsigned lo, unsigned hi) {
        if (hi >= 0x7ff00000u || lo < 0x00100000u) return false;  // inf / NaN / negative, tiny
        return __hiloint2double(static_cast<int>(hi + 1), 0) <
               1.0198 * __hiloint2double(static_cast<int>(lo), 0);
      };
      smooth = ratio_ok(hr_lo, hr_hi) && ratio_ok(hb_lo, hb_hi);
    }
    __syncwarp();

    // ---- flux-differencing volume terms (semidisc.cpp:455-464) --------------
    double KA[V], KB[V];
#pragma unroll
    for (int v = 0; v < V; ++v) KA[v] = KB[v] = 0.0;
    if (smooth) {
      w3_inplane<0, true>(ph, pr, lane, ix, J2x, KA, KB, own[0], own[1]);
      w3_inplane<1, true>(ph, pr, lane, iy, J2y, KA, KB, own[0], own[1]);
      w3_z<true>(ph, pr, lane, zA, J2z, KA, KB, own[0], own[1]);
    } else {
      w3_inplane<0, false>(ph, pr, lane, ix, J2x, KA, KB, own[0], own[1]);
      w3_inplane<1, false>(ph, pr, lane, iy, J2y, KA, KB, own[0], own[1]);
      w3_z<false>(ph, pr, lane, zA, J2z, KA, KB, own[0], own[1]);
    }

    // ---- surface flux + lift + endpoint diagonal at the lane's three face
    // points (semidisc.cpp:489-556, :450-454) ---------------------------------
#if PERRK_W3_REGPF == 1
    if (ncell >= 0) load_own(ncell);
#endif
    if (PERRK_W3_OWNL1PF == 1 && ncell >= 0 && lane < 20)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(
          reinterpret_cast<const char*>((form_ ? a.Us : a.U) + static_cast<size_t>(ncell) * N * V) +
          128 * lane));
    // PERRK_W3_L2PF == 2: only the next cell's own stage-state block, and only
    // now (a surface phase and an epilogue ahead of its use)
    if (PERRK_W3_L2PF == 2 && lane == 0 && ncell >= 0)
      l2_prefetch((form_ ? a.Us : a.U) + static_cast<size_t>(ncell) * N * V,
                  N * V * sizeof(double));
#if PERRK_W3_EPIPF
    if (next_) {
      // 2560-byte blocks: 20 lines of 128 bytes each; lanes 0-19 take U, and
      // (formed stages) lanes 12-31 take K1
      const char* pu = reinterpret_cast<const char*>(a.U + cbase);
      const char* pk = reinterpret_cast<const char*>(a.K1 + cbase);
      if (lane < 20) asm volatile("prefetch.global.L1 [%0];" ::"l"(pu + 128 * lane));
      if (form_ && lane >= 12) asm volatile("prefetch.global.L1 [%0];" ::"l"(pk + 128 * (lane - 12)));
    }
#endif
#if PERRK_W3_EPIREG
    static_assert(!PERRK_W3_COAL, "PERRK_W3_EPIREG needs the direct epilogue");
    double eU[2][V], eK[2][V];
    if (!next_ && dm_ == 2) {  // last b-stage: no U / K1, the d block takes their place
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const size_t g = h ? gB : gA;
#pragma unroll
        for (int v = 0; v < V; ++v)
          eU[h][v] = PERRK_W3_CS ? __ldcs(a.d + g + v * N) : __ldg(a.d + g + v * N);
      }
    }
    if (next_) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const size_t g = h ? gB : gA;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          eU[h][v] = PERRK_W3_CS ? __ldcs(a.U + g + v * N) : __ldg(a.U + g + v * N);
          if (form_) eK[h][v] = PERRK_W3_CS ? __ldcs(a.K1 + g + v * N) : __ldg(a.K1 + g + v * N);
        }
      }
    }
#endif
    // the traces (the next descriptor, and with PERRK_W3_OWNPF the next own block, fly on)
    cp_async_wait<PERRK_W3_DESCREG ? 0 : (PERRK_W3_OWNPF ? 2 : 1)>();
    __syncwarp();
#if PERRK_W3_FLAT && PERRK_W3_HOIST
    if (__any_sync(0xffffffffu, unf != 0u)) {  // rare: a level's first active stage
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        if ((unf >> d) & 1u) {
          const int l2 = static_cast<int>((lv >> (8 * (1 + 2 * d + side))) & 0xff);
          const size_t gi = static_cast<size_t>(nb3[d]) * N * V + w3_face_node(d, 1 - side, pt);
          const double b1 = dt * a.a1[l2];
          double* sl = fs + w3_fs(d * 32 + lane);  // the lane's own slot: the U trace
          double un[V];
#pragma unroll
          for (int v = 0; v < V; ++v) un[v] = fma(b1, __ldg(a.K1 + gi + v * N), sl[v]);
          w3_slot_store(sl, un);
        }
      }
    }
    unsigned badf = 0;  // bit d: the neighbour's trace on (d, side) is inadmissible
#endif
#pragma unroll
    for (int kd = 0; kd < 3; ++kd) {
      // z faces first with PERRK_W3_ZREG (the own registers die early)
      const int d = PERRK_W3_ZREG ? (kd == 0 ? 2 : kd - 1) : kd;
      double* slotp = fs + w3_fs(d * 32 + lane);
#if PERRK_W3_FLAT && PERRK_W3_HOIST
      double un[V];
      w3_slot_load(slotp, un);
#elif PERRK_W3_HOIST
      const int nbc = nb3[d];
      double un[V];
      w3_slot_load(slotp, un);  // (stale where the neighbour is formed below)
      if ((unf >> d) & 1u) {
        const int l2 = static_cast<int>((lv >> (8 * (1 + 2 * d + side))) & 0xff);
        const size_t gi = static_cast<size_t>(nbc) * N * V + w3_face_node(d, 1 - side, pt);
        const double b1 = dt * a.a1[l2];
#pragma unroll
        for (int v = 0; v < V; ++v)
          un[v] = fma(b1, __ldg(a.K1 + gi + v * N), __ldg(a.U + gi + v * N));
      }
#else
      const int nbc = rp->nb[2 * d + side];
      double un[V];
      if (nbc >= 0 && form_) {
        const int l2 = static_cast<int>((lv >> (8 * (1 + 2 * d + side))) & 0xff);
        if (a.formed[l2]) {
          w3_slot_load(slotp, un);
        } else {
          const size_t gi = static_cast<size_t>(nbc) * N * V + w3_face_node(d, 1 - side, pt);
          const double b1 = dt * a.a1[l2];
#pragma unroll
          for (int v = 0; v < V; ++v)
            un[v] = fma(b1, __ldg(a.K1 + gi + v * N), __ldg(a.U + gi + v * N));
        }
      } else {
        w3_slot_load(slotp, un);
      }
#endif
      const double J2 = d == 0 ? J2x : (d == 1 ? J2y : J2z);
      const double lift = rp->lift[d];
      const int j = side ? N1 - 1 : 0;
      double o5[V];
      double2 o0, o1, o2, o3;
      if (PERRK_W3_ZREG && PERRK_W3_ZOWN && PERRK_W3_OWNREG && d == 2) {
        const W3Prim w = w3_select(side == 0, own[0], own[1]);
        o0 = make_double2(w.rho, w.beta);
        o1 = make_double2(w.v[0], w.v[1]);
        o2 = make_double2(w.v[2], w.p);
        o3 = side ? ownEc[1] : ownEc[0];
      } else {
        const double2* on =
            reinterpret_cast<const double2*>(pr) + w3_sw(w3_face_node(d, side, pt));
        o0 = on[0];
        o1 = on[N];
        o2 = on[2 * N];
        o3 = on[3 * N];
      }
      const double vo[3] = {o1.x, o1.y, o2.x};
      const bool ok = rus_lift_v<3, SURF>(ph, o0.x, vo, PERRK_W3_HALFP ? o2.y + o2.y : o2.y,
                                          o3.x, o3.y, un, d, side,
                                          J2 * c_D[j * N1 + j], side ? -lift : lift, false, o5);
#if PERRK_W3_FLAT && PERRK_W3_HOIST
      if (!ok) badf |= 1u << d;
      if (PERRK_W3_ZOWN && d == 2) {
        const double mA = side ? 0.0 : 1.0, mB = side ? 1.0 : 0.0;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          KA[v] = fma(mA, o5[v], KA[v]);
          KB[v] = fma(mB, o5[v], KB[v]);
        }
      } else {
        w3_slot_store(slotp, o5);
      }
      continue;
#else
      if (!ok)
        report_bad(st, a.stage, a.ncells,
                   nbc < 0 ? m.ghost_gid[-1 - nbc] : (m.gid ? m.gid[nbc] : nbc));
#endif
      if (PERRK_W3_ZOWN && d == 2) {
        // z faces: face point (2, side, pt) of lane 16 side + pt belongs to the
        // lane's own node (A on side 0, B on side 1): no trip through the slots
        if (side) {
#pragma unroll
          for (int v = 0; v < V; ++v) KB[v] += o5[v];
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v) KA[v] += o5[v];
        }
      } else {
        w3_slot_store(slotp, o5);
      }
    }
#if PERRK_W3_FLAT && PERRK_W3_HOIST
    if (badf) {
      const int nbc = (badf & 1u) ? nb3[0] : ((badf & 2u) ? nb3[1] : nb3[2]);
      report_bad(st, a.stage, a.ncells,
                 nbc < 0 ? m.ghost_gid[-1 - nbc] : (m.gid ? m.gid[nbc] : nbc));
    }
#endif
    __syncwarp();
    // gather: node A / B on face (d, side) takes the term of face point
    // (d, side, pt(node, d)) = slot d * 32 + 16 side + pt
    {
      const int jA[3] = {ix, iy, zA}, jB[3] = {ix, iy, zB};
#pragma unroll
      for (int d = 0; d < (PERRK_W3_ZOWN ? 2 : 3); ++d) {
        const int ptA = d == 0 ? iy + 4 * zA : (d == 1 ? ix + 4 * zA : ix + 4 * iy);
        const int ptB = d == 0 ? iy + 4 * zB : (d == 1 ? ix + 4 * zB : ix + 4 * iy);
#if PERRK_W3_HOIST
        // every lane reads a written slot (finite values); nodes off the face weigh it with 0
        const double mA = (jA[d] == 0 || jA[d] == N1 - 1) ? 1.0 : 0.0;
        const double mB = (jB[d] == 0 || jB[d] == N1 - 1) ? 1.0 : 0.0;
        double cA[V], cB[V];
        w3_slot_load(fs + w3_fs(d * 32 + 16 * (jA[d] ? 1 : 0) + ptA), cA);
        w3_slot_load(fs + w3_fs(d * 32 + 16 * (jB[d] ? 1 : 0) + ptB), cB);
#pragma unroll
        for (int v = 0; v < V; ++v) {
          KA[v] = fma(mA, cA[v], KA[v]);
          KB[v] = fma(mB, cB[v], KB[v]);
        }
        continue;
#endif
        if (jA[d] == 0 || jA[d] == N1 - 1) {
          double c[V];
          w3_slot_load(fs + w3_fs(d * 32 + 16 * (jA[d] ? 1 : 0) + ptA), c);
#pragma unroll
          for (int v = 0; v < V; ++v) KA[v] += c[v];
        }
        if (jB[d] == 0 || jB[d] == N1 - 1) {
          double c[V];
          w3_slot_load(fs + w3_fs(d * 32 + 16 * (jB[d] ? 1 : 0) + ptB), c);
#pragma unroll
          for (int v = 0; v < V; ++v) KB[v] += c[v];
        }
      }
    }

#if PERRK_W3_REGPF == 2
    if (ncell >= 0) load_own(ncell);
#endif
    if (PERRK_W3_OWNL1PF == 2 && ncell >= 0 && lane < 20)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(
          reinterpret_cast<const char*>((form_ ? a.Us : a.U) + static_cast<size_t>(ncell) * N * V) +
          128 * lane));
    // ---- epilogue (stepper.cpp:52-55, 60-72, 89-92) ---------------------------
    if (a.want_dh || a.want_h) {
      const double meas = rp->meas;
      const double wxy = c_w[ix] * c_w[iy];
      // own primitives from the slice (not kept in registers across the volume phase)
      auto node = [&](int n, const double* K, int iz) {
        const W3Prim q = w3_load(pr, n);
        const double be = q.beta;
        // (admissible here: an inadmissible cell was reported above and the step is
        // discarded, so the unguarded logarithm body is enough)
        const double s_therm = -(flog_core(be) + ph.gm1 * flog_core(q.rho));
        const double om = meas * wxy * c_w[iz];
        if (a.want_dh) {
          double v2 = 0.0, dot = 0.0;
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            v2 = fma(q.v[i], q.v[i], v2);
            dot = fma(ph.gm1 * be * q.v[i], K[1 + i], dot);
          }
          dot = fma(ph.gamma - s_therm - 0.5 * ph.gm1 * be * v2, K[0], dot);
          dot = fma(-ph.gm1 * be, K[V - 1], dot);
          acc_dh = dd_add_prod(acc_dh, om, dot);
        }
        if (a.want_h) acc_h = dd_add_prod(acc_h, om, -q.rho * s_therm);
      };
      node(lane, KA, zA);
      node(lane + 32, KB, zB);
    }
    const double an = dt * a.a1n[lev], pn = dt * a.apn[lev];
#if PERRK_W3_COAL
    // Epilogue through the slice (dead after the gather and the dH terms):
    // the cell's blocks of U, K1 and d (2560 contiguous bytes each) come in by
    // coalesced 16-byte cp.async, are read node-wise with conflict-free 8-byte
    // loads, and the results, U_{i+1} = U + dt (a_{i+1,1} K1 + a_{i+1,i} K_i)
    // in place of U, K1 = K_0 (stage 0) and d in place, leave as bulk copies
    // (cp.async.bulk, the TMA path: no per-lane store wavefronts).  This was
    // the round-1 form, for the canonical layout (a direct 40-byte-stride
    // LDG.64 / STG.64 touched 10 lines per instruction); with the device
    // layout the direct form below is coalesced and costs fewer L1 wavefronts.
    //   slice: U [0, 64V) | K1 or K_0 [64V, 128V) | d [128V, 192V)
    {
#if PERRK_W3_EPI
      double* eu = ep;
      double* ek = ep + N * V;
      double* ed = pr;
      __syncwarp();  // every lane is done with the primitives and face slots
      if (dm_ == 2) {
        w3_stage_cell(ed, a.d + cbase, lane);
        cp_async_commit();
        cp_async_wait<0>();
      }
      if (next_) {
        mbar_wait(&s_mbar[wib], ep_phase);
        ep_phase ^= 1u;
      }
      __syncwarp();
#else
      double* eu = pr;
      double* ek = pr + N * V;
      double* ed = pr + 2 * N * V;
      __syncwarp();  // every lane is done with the primitives and face slots
      if (next_) w3_stage_cell(eu, a.U + cbase, lane);
      if (next_ && form_) w3_stage_cell(ek, a.K1 + cbase, lane);
      if (dm_ == 2) w3_stage_cell(ed, a.d + cbase, lane);
      cp_async_commit();
      cp_async_wait<0>();
      __syncwarp();
#endif
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double* K = h ? KB : KA;
        const int o = lane + 32 * h;  // variable v of this node at o + v N (device layout)
        if (a.write_k) {
#pragma unroll
          for (int v = 0; v < V; ++v) ek[o + v * N] = K[v];
        }
        if (next_) {
          double x[V];
          if (form_) {
#pragma unroll
            for (int v = 0; v < V; ++v) x[v] = eu[o + v * N] + fma(an, ek[o + v * N], pn * K[v]);
          } else {
#pragma unroll
            for (int v = 0; v < V; ++v) x[v] = fma(an, K[v], eu[o + v * N]);
          }
#pragma unroll
          for (int v = 0; v < V; ++v) eu[o + v * N] = x[v];
        }
        if (dm_) {
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const double x = dm_ == 2 ? fma(a.b, K[v], ed[o + v * N]) : a.b * K[v];
            ed[o + v * N] = x;
            const unsigned long long bits =
                static_cast<unsigned long long>(__double_as_longlong(x)) & 0x7fffffffffffffffULL;
            if (a.want_dmax) dmax_bits = bits > dmax_bits ? bits : dmax_bits;
          }
        }
      }
      bulk_store_fence();
      __syncwarp();
      if (lane == 0) {
        constexpr unsigned kBytes = N * V * sizeof(double);
        if (next_) bulk_store(a.Usn + cbase, eu, kBytes);
        if (a.write_k) bulk_store(a.Kout + cbase, ek, kBytes);
        if (dm_) bulk_store(a.d + cbase, ed, kBytes);
      }
    }
#else
#if PERRK_W3_EPIREG
#define W3_EU(h, v) eU[h][v]
#define W3_EK(h, v) eK[h][v]
#else
#define W3_EU(h, v) 0.0
#define W3_EK(h, v) 0.0
#endif
#if PERRK_W3_CS
#define W3_LD(p) __ldcs(p)
#define W3_ST(p, x) __stcs(p, x)
#else
#define W3_LD(p) (*(p))
#define W3_ST(p, x) (*(p) = (x))
#endif
    if (a.write_k) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        W3_ST(a.Kout + gA + v * N, KA[v]);
        W3_ST(a.Kout + gB + v * N, KB[v]);
      }
    }
    // U_{i+1} and d node by node, each batch with all its loads issued before
    // its first store (the compiler cannot tell that Usn / d do not alias
    // U / K1, and would otherwise serialise load -> store pairs)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const double* K = h ? KB : KA;
      const size_t g = h ? gB : gA;  // variable v at g + v N (coalesced)
      double x[V], y[V];
      if (next_) {
#pragma unroll
        for (int v = 0; v < V; ++v) x[v] = PERRK_W3_EPIREG ? W3_EU(h, v) : W3_LD(a.U + g + v * N);
        if (form_) {
#pragma unroll
          for (int v = 0; v < V; ++v) y[v] = PERRK_W3_EPIREG ? W3_EK(h, v) : W3_LD(a.K1 + g + v * N);
#pragma unroll
          for (int v = 0; v < V; ++v) W3_ST(a.Usn + g + v * N, x[v] + fma(an, y[v], pn * K[v]));
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v) W3_ST(a.Usn + g + v * N, fma(an, K[v], x[v]));
        }
      }
      if (dm_) {
        if (dm_ == 2) {
#pragma unroll
          for (int v = 0; v < V; ++v)
            x[v] = fma(a.b, K[v], (PERRK_W3_EPIREG && !next_) ? W3_EU(h, v) : W3_LD(a.d + g + v * N));
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v) x[v] = a.b * K[v];
        }
#pragma unroll
        for (int v = 0; v < V; ++v) {
          W3_ST(a.d + g + v * N, x[v]);
          const unsigned long long bits =
              static_cast<unsigned long long>(__double_as_longlong(x[v])) & 0x7fffffffffffffffULL;
          if (a.want_dmax) dmax_bits = bits > dmax_bits ? bits : dmax_bits;
        }
      }
    }
#undef W3_LD
#undef W3_ST
#undef W3_EU
#undef W3_EK
#endif
#if PERRK_W3_REGPF == 3
    if (ncell >= 0) load_own(ncell);  // the last thing of the cell: ahead of the next cell's descriptor round trip
#endif
    __syncwarp();  // the slice is rewritten by the next cell
    slot = nslot;
    cell = ncell;
    ncell = nncell;
    rb ^= 1;
  }

  if (PERRK_W3_COAL && lane == 0) bulk_wait_all();
  // ---- grid epilogue (as stage_kernel) --------------------------------------
  if (a.want_dmax) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o = __shfl_down_sync(0xffffffffu, dmax_bits, off);
      dmax_bits = o > dmax_bits ? o : dmax_bits;
    }
    if (lane == 0) {
      if (dmax_bits >= 0x7ff0000000000000ULL) st->d_nonfinite = 1;
      else atomicMax(&st->dmax_bits, dmax_bits);
    }
  }
  dd v[2] = {acc_dh, acc_h}, tot[2];
  if (a.want_dh || a.want_h) block_reduce_dd<2>(v, s_red);
  if (grid_reduce_dd<2>(v, partials, counter, s_red, tot) && threadIdx.x == 0) {
    if (a.want_dh) {
      const dd inc = dd_mul_d(tot[0], dt * a.b);
      const dd cur = {st->dh_hi, st->dh_lo};
      const dd nw2 = dd_add(cur, inc);
      st->dh_hi = nw2.hi;
      st->dh_lo = nw2.lo;
    }
    if (a.want_h) {
      st->h_hi = tot[1].hi;
      st->h_lo = tot[1].lo;
    }
    if (st->bad_code != kNoBad) st->aborted = 1;
  }
}

}  // namespace dev
}  // namespace perrk
