// ef_kernels.cu — the sm_100a kernels of one forward-Euler stage.
//
// Per-slot data is SELL-32 (slot-major inside 32-row slices) and per-node data
// structure-of-arrays, so slot loads of consecutive rows coalesce and
// neighbour gathers hit L1/L2 thanks to the Cuthill-McKee numbering.
// Phase map (reference stepper.py):
//   k_edge_visc    = step1 d_ij_low on the upper triangle, one thread per edge (:407-416)
//   k_row_visc     = step1 IndicatorAccumulator (:417-425) + step2 _k_mirror and
//                    _tau_local (:427-434, :66-70)
//   k_low_order    = step3 _k_low_order (+ tau = min(c_cfl tau_min, tau_max), :548)
//   k_edge_lim(q)  = step4 (q = 0: P_ij, P_ji built from R, U, d, alpha, m) and the
//                    limiter of pass q for both rows of an edge + min(l_ij, l_ji)
//                    (:456-474, :478-479, :485-491), one thread per edge
//   k_edge_lim_last = the last pass over the worklist the pass before it built
//   k_row_upd      = step5 non-final limited update (:480-481), one thread per row
//   k_final        = step6 final pass + _k_boundary + _finish_step check
//                    + SSP-RK3 combination + next stage's step0 (:493-504, :612-636, :399-405)
// The edge kernels run one thread per upper edge, the row kernels one thread
// per owned row.  k_edge_visc writes d_ij also into the lower slot of row j
// (d is symmetric) and k_edge_lim writes P and min(l_ij, l_ji) to both rows of
// an edge, so the row kernels stream their own slots instead of gathering
// transposes.  The gather loops of k_row_visc / k_low_order prefetch the next
// slot's neighbour fields with cp.async (row_pipe); step0 (fused into k_final
// and k_nodal) caches v = m / rho and p for the neighbour fluxes.  Variants
// measured slower (row groups, slot-parallel and row-owned limiters, half-edge
// limiter, PDL, ...) are listed in DESIGN.md §6.
// Exact fast paths (every one returns the bits of the full computation; DESIGN
// §6): min(l) == 1 makes the next P zero (later passes tag such slots kZeroP
// instead of limiting them, the last pass only visits a worklist of min(l) < 1
// edges, k_final only rows that have one); identical states (U_i == U_j bit for
// bit) give a closed-form lambda, uniform stencils skip the indicator and
// low-order loops and zero the first pass's P, unchanged rows keep their d_ij
// (the *<..., UNI> variants, chosen per step from a sampled count); in 3D the
// limiter accepts t_R from an fp32 bound of the pow when the margin is clear.
#include <atomic>
#include <cstdio>

#include "ef_kernels.cuh"

namespace ef {

// Bounds checks of every computed index (-DEF_CHECKS debug build, used in place
// of compute-sanitizer, which the GPU pool does not allow): a violated check
// prints its location and traps.
#ifdef EF_CHECKS
#define EF_ASSERT(c)                                                               \
  do {                                                                             \
    if (!(c)) {                                                                    \
      printf("EF_ASSERT failed %s:%d: %s\n", __FILE__, __LINE__, #c);              \
      __trap();                                                                    \
    }                                                                              \
  } while (0)
#else
#define EF_ASSERT(c) \
  do {               \
  } while (0)
#endif
#define EF_IN(x, n) EF_ASSERT((int64_t)(x) >= 0 && (int64_t)(x) < (int64_t)(n))


#ifndef EF_TPB
#define EF_TPB 128
#endif
constexpr int TPB = EF_TPB;  // state I/O, halo and pow kernels
// Stage kernels: 64-thread blocks in 2D (a shorter last wave: +1%), 128 in 3D
// (64 measured -1%).  The register caps below count resident 128-thread
// blocks per SM; EF_LB rescales them to the kernel's block size.
#ifndef EF_TPB2
#define EF_TPB2 64
#endif
#ifndef EF_TPB3
#define EF_TPB3 128
#endif
#define EF_TPB_D(D) ((D) == 3 ? EF_TPB3 : EF_TPB2)
#define EF_LB(n, D) ((n) * 128 / EF_TPB_D(D))
// Resident blocks per SM requested from ptxas (i.e. the register cap) per
// kernel and dimension, measured on B200 (C2 2D, 160^3 periodic 3D): these
// kernels are latency-bound, so occupancy usually beats spill-free code.
#ifndef EF_MINB
#define EF_MINB 8
#endif
#ifndef EF_MINB_EDGE2
#define EF_MINB_EDGE2 9
#endif
#ifndef EF_MINB_ROW2
#define EF_MINB_ROW2 EF_MINB
#endif
#ifndef EF_MINB_LOW2
#define EF_MINB_LOW2 5
#endif
#ifndef EF_MINB_EDGE3
#define EF_MINB_EDGE3 6  // 80 registers, 20 bytes of spills (7: 72 registers, 80 bytes: +0.7% at base clocks, +1.4% on C5 320^3; before the
                         // trimmed pows and lambda 7 was the best: 5: 3.00, 6: 2.90, 7: 2.63, 8: 2.69, 10: 2.97 ms on the 160^3 box)
#endif
#define EF_MINB_EDGE(D) ((D) == 3 ? EF_MINB_EDGE3 : EF_MINB_EDGE2)
#ifndef EF_MINB_ROW3
#define EF_MINB_ROW3 5
#endif
#ifndef EF_MINB_LOW3
#define EF_MINB_LOW3 4
#endif
#define EF_MINB_ROW(D) ((D) == 3 ? EF_MINB_ROW3 : EF_MINB_ROW2)
#define EF_MINB_LOW(D) ((D) == 3 ? EF_MINB_LOW3 : EF_MINB_LOW2)
#ifndef EF_MINB_ELIM2
#define EF_MINB_ELIM2 EF_MINB
#endif
#ifndef EF_MINB_ELIM3
#define EF_MINB_ELIM3 6
#endif
// the first pass (forms P) wants more registers than the rescaling passes
#ifndef EF_MINB_ELIM2_FIRST
#define EF_MINB_ELIM2_FIRST 7
#endif
#ifndef EF_MINB_ELIM3_FIRST
#define EF_MINB_ELIM3_FIRST EF_MINB_ELIM3
#endif
#define EF_MINB_ELIM(D, FIRST) \
  ((D) == 3 ? ((FIRST) ? EF_MINB_ELIM3_FIRST : EF_MINB_ELIM3) : ((FIRST) ? EF_MINB_ELIM2_FIRST : EF_MINB_ELIM2))
#ifndef EF_MINB_UPD
#define EF_MINB_UPD 10
#endif
// 3D k_row_upd at 8 resident blocks: -15% (from 10; 160^3 box)
#ifndef EF_MINB_UPD3
#define EF_MINB_UPD3 8
#endif
#define EF_MINB_PASS(D) ((D) == 3 ? EF_MINB_UPD3 : EF_MINB_UPD)
#ifndef EF_MINB_FINAL3
#define EF_MINB_FINAL3 12  // 3D k_final: -11% from 6 to 8, -4% from 8 to 10, -3% from 10 to 12 resident blocks
#endif
#define EF_MINB_FINAL(D) ((D) == 3 ? EF_MINB_FINAL3 : EF_MINB)

static inline unsigned grid_for(int64_t n) { return (unsigned)((n + TPB - 1) / TPB); }

__device__ __forceinline__ int sidx32(int i, int s, int L) { return (i >> 5) * (32 * L) + s * 32 + (i & 31); }

template <int NV>
__device__ __forceinline__ void load_node(const double* __restrict__ U, int NP, int i, double* out) {
#pragma unroll
  for (int k = 0; k < NV; ++k) out[k] = U[k * NP + i];
}

template <int NV>
__device__ __forceinline__ void load_node(const double* __restrict__ U, int64_t NP, int64_t i,
                                          double* out) {
#pragma unroll
  for (int k = 0; k < NV; ++k) out[k] = U[k * NP + i];
}

// L2 prefetch of the streamed per-edge index arrays about one wave of resident
// threads ahead (k_edge_lim: EF_PF_LIM edges):
// those loads miss L2 (read once per launch), and their DRAM latency otherwise
// heads every edge's dependent load chain.  Measured: limiter passes -2% (2D)
// / -3% (3D); k_edge_visc +3% in 3D (issue-bound), so off there.
// Rows whose whole stencil holds the row's own state (bitwise; w.nonuni == 0)
// take exact closed forms in k_row_visc (alpha = 0), k_low_order (no neighbour
// loads) and k_edge_lim's first pass (P = 0) -- EF_UNIFORM_ROWS, default on.
#ifndef EF_UNIFORM_ROWS
#define EF_UNIFORM_ROWS 1
#endif
// warp-aggregated append of e to a worklist (order is irrelevant: each listed
// edge's work is independent)
__device__ __forceinline__ void wl_append(bool need, int e, int* __restrict__ wl, int* n) {
  const unsigned act = __activemask(), bal = __ballot_sync(act, need);
  if (!bal) return;
  const int lane = threadIdx.x & 31, leader = __ffs(bal) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(n, __popc(bal));
  base = __shfl_sync(act, base, leader);
  EF_ASSERT(base >= 0);
  if (need) wl[base + __popc(bal & ((1u << lane) - 1u))] = e;
}
// warp-aggregated count into one of kSameSlots counters (spread: no hot address)
__device__ __forceinline__ void count_hits(bool hit, unsigned long long* slots) {
  const unsigned act = __activemask(), hits = __ballot_sync(act, hit);
  if ((threadIdx.x & 31) == (unsigned)(__ffs(act) - 1) && hits)
    atomicAdd(slots + ((blockIdx.x * 7 + (threadIdx.x >> 5)) & (kSameSlots - 1)), (unsigned long long)__popc(hits));
}
template <int N>
__device__ __forceinline__ bool all_finite(const double* x) {
  bool ok = true;
#pragma unroll
  for (int k = 0; k < N; ++k) ok = ok && finite(x[k]);
  return ok;
}
// d_ij memo across identical-state stages (EF_MEMO_D, default on)
#ifndef EF_MEMO_D
#define EF_MEMO_D 1
#endif
#ifndef EF_WL
#define EF_WL 1
#endif
#ifndef EF_WL_GRID
#define EF_WL_GRID 1184  // 8 resident-size waves of 148 SMs
#endif
#ifndef EF_PF_VISC_UNI
#define EF_PF_VISC_UNI 131072  // (the memo check makes the identical-state variant latency-bound: -6%)
#endif
// min(l) slot tag: this slot's P is zero for the current and all later passes
// (set instead of storing zero P; a genuine min(l) is in [0, 1])
constexpr double kZeroP = -1.0;
// frozen rows (uniform and unchanged since the previous identical-state stage)
// skip k_row_visc / k_low_order (EF_FROZEN, default on)
#ifndef EF_FROZEN
#define EF_FROZEN 1
#endif
// P = 0 shortcut of the limiter passes after the first (EF_ZSKIP, default on)
#ifndef EF_ZSKIP
#define EF_ZSKIP 1
#endif
#ifndef EF_PF_LIM
#define EF_PF_LIM 131072
#endif
// latch an error: its bit, and its position in the reference's order of checks
__device__ __forceinline__ void raise_err(const Work& w, int bit, int stage, int phase) {
  atomicOr(w.err, bit);
  atomicMin(w.err_first, stage * 8 + phase);
}
__device__ __forceinline__ void pf_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// ---------------------------------------------------------------- state I/O
template <int D>
__global__ void k_gather_state(Layout m, int64_t count, const double* __restrict__ Uaos,
                               const int64_t* __restrict__ orig, double* __restrict__ U, int* err) {
  constexpr int NV = D + 2;
  const int64_t i = blockIdx.x * (int64_t)TPB + threadIdx.x;
  if (i >= count) return;
  const int64_t o = orig[i];
  double x[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    x[k] = Uaos[o * NV + k];
    U[k * m.NP + i] = x[k];
  }
  if (!((x[0] > 0.0) && (internal_energy<D>(x) > 0.0))) atomicOr(err, 1);
}

template <int D>
__global__ void k_scatter_state(Layout m, const double* __restrict__ U,
                                const int64_t* __restrict__ orig, double* __restrict__ Uaos) {
  constexpr int NV = D + 2;
  const int64_t i = blockIdx.x * (int64_t)TPB + threadIdx.x;
  if (i >= m.n_owned) return;
  const int64_t o = orig[i];
#pragma unroll
  for (int k = 0; k < NV; ++k) Uaos[o * NV + k] = U[k * m.NP + i];
}

// ---------------------------------------------------------------- step0
// step0 (stepper.py:399-405) of node i: eta/rho, phi, and the flux inputs
// v = m / rho, p = gm1 * eps that the row kernels reuse for every stencil slot
template <int D>
__device__ __forceinline__ void nodal_one(const double* Ui, const Gas& g, Work& w, int NP, int i) {
  const double rho = Ui[0];
  const Recip rr = recip(rho);  // shared by the divisions by rho
  const double eps = internal_energy<D>(Ui, rr);
  w.eor[i] = qdiv(dpow(rho * eps, g.gp1_inv), rr);  // stepper.py:403
  w.phi[i] = eps * dpow(rho, g.neg_gamma);          // stepper.py:404
#pragma unroll
  for (int a = 0; a < D; ++a) w.vp[a * NP + i] = qdiv(Ui[1 + a], rr);  // physics.py:157
  w.vp[D * NP + i] = g.gm1 * eps;                                        // physics.py:94
}

template <int D>
__global__ void k_nodal(Layout m, Gas g, const double* __restrict__ U, Work w, int64_t lo, int64_t hi) {
  const int64_t i = lo + blockIdx.x * (int64_t)TPB + threadIdx.x;
  if (i >= hi) return;
  double Ui[D + 2];
  load_node<D + 2>(U, m.NP, i, Ui);
  nodal_one<D>(Ui, g, w, (int)m.NP, (int)i);
  w.nonuni[i] = 0;  // a new state (set_state, ghost rows): nothing of it is known
  w.chg[i] = 1;
}

// ---------------------------------------------------------------- step1a
// One thread per upper edge (global id of the column above the row's, i.e. a
// slot after the diagonal; stepper.py:211, 415).  The edge list holds SELL
// positions in ascending order, so a warp reads 32 consecutive positions of
// one slot row (coalesced) and the row / slot are recovered from the position.
// the two states and the geometry record (n_ij, |c_ij|, n_ji, |c_ji|) of an edge
template <int D>
__device__ __forceinline__ void load_edge(const Layout& m, const double* __restrict__ U, int NP, int e, int i, int j,
                                          double* Ui, double* Uj, double* nij, double& norm_ij, double* nji,
                                          double& norm_ji) {
  load_node<D + 2>(U, NP, i, Ui);
  load_node<D + 2>(U, NP, j, Uj);
  double g[2 * (D + 1)];
  const double2* __restrict__ rec = reinterpret_cast<const double2*>(m.egeo) + (size_t)e * (D + 1);
#pragma unroll
  for (int k = 0; k < D + 1; ++k) {
    const double2 v = rec[k];
    g[2 * k] = v.x;
    g[2 * k + 1] = v.y;
  }
#pragma unroll
  for (int a = 0; a < D; ++a) {
    nij[a] = g[a];
    nji[a] = g[D + 1 + a];
  }
  norm_ij = g[D];
  norm_ji = g[2 * D + 1];
}
template <int D, bool UNI>
__global__ void __launch_bounds__(EF_TPB_D(D), EF_LB(EF_MINB_EDGE(D), D)) k_edge_visc(Layout m, Gas g, const double* __restrict__ U,
                                                   Work w, int flags) {  // 1: reset the CFL bound, 2: count,
                                                                         // bits 4-5: stage
  constexpr int NV = D + 2;
  const int e = blockIdx.x * EF_TPB_D(D) + threadIdx.x;
  if ((flags & 1) && e == 0) *w.tau_min_bits = 0x7ff0000000000000ULL;
  if (e >= m.n_edges) return;
  const int NP = (int)m.NP, NE = (int)m.n_edges;
  if (UNI && EF_PF_VISC_UNI > 0 && e + EF_PF_VISC_UNI < NE) {
    pf_l2(m.edges + e + EF_PF_VISC_UNI);
    pf_l2(m.edge_j + e + EF_PF_VISC_UNI);
  }
  if (UNI && EF_MEMO_D) {
    // both rows unchanged since the previous identical-state stage: d_ij (a pure
    // function of U_i, U_j and the static geometry) and the rows' uniformity
    // marks are still those of the previous stage
    const int p0 = m.edges[e];
    const int i0 = (int)fdiv((uint32_t)p0, m.slab) * 32 + (p0 & 31);
    if (!w.chg[i0] && !w.chg[m.edge_j[e]]) return;
  }
  const int p = m.edges[e];
  const int i = (int)fdiv((uint32_t)p, m.slab) * 32 + (p & 31);
  const int j = m.edge_j[e];
  const int pt = m.edge_pt[e];
  EF_IN(p, m.NP * m.L);
  EF_IN(pt, m.NP * m.L);
  EF_IN(i, m.n_local);
  EF_IN(j, m.n_local);
  bool bad = false, same = false, done = false;
  double dv;
  {
    double Ui[NV], Uj[NV], nij[D], nji[D], norm_ij, norm_ji;
    load_edge<D>(m, U, NP, e, i, j, Ui, Uj, nij, norm_ij, nji, norm_ji);
    if (UNI || ((flags & 2) && (blockIdx.x & 7) == 0)) same = same_state<NV>(Ui, Uj);
    if (UNI && !same) {
      w.nonuni[i] = 1;
      w.nonuni[j] = 1;
    }
    // the straight-line evaluation (ef_math.cuh); identical states by their closed form
    done = d_ij_sl<D>(Ui, Uj, nij, norm_ij, nji, norm_ji, g, dv, UNI && same);
  }
  if (!done) {
    // zero or extreme operands, an inadmissible state, vacuum, identical states: the
    // general code on operands loaded again (nothing of the rare path stays live above)
    asm volatile("" ::: "memory");
    double Ui[NV], Uj[NV], nij[D], nji[D], norm_ij, norm_ji;
    load_edge<D>(m, U, NP, e, i, j, Ui, Uj, nij, norm_ij, nji, norm_ji);
    dv = d_ij_geo<D>(Ui, Uj, nij, norm_ij, nji, norm_ji, g, bad, UNI && same);
  }
  // d is symmetric by construction (riemann.py:139-142): the value is also
  // the lower-triangle entry of row j, written straight to its slot (the
  // reference's mirror, stepper.py:427-434, without a gather)
  w.d[p] = dv;
  w.d[pt] = dv;
  if (bad) raise_err(w, ERR_PROJECT, flags >> 4, PH_VISC);
  // with the shortcuts off: sample (1 block in 8, first stage) how many would apply
  if (!UNI && (flags & 2) && (blockIdx.x & 7) == 0) count_hits(same, w.n_same);
}

// ---------------------------------------------------------------- step1b + step2
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Per owned row, in slot order: the entropy-viscosity indicator
// (IndicatorAccumulator.reset/accumulate/result, indicator.py:35-73), the
// mirror of the lower triangle with d_ii = -(numpy pairwise row sum)
// (_k_mirror, stepper.py:427-434) and the CFL bound (_tau_local, :66-70).
// Register-free gather prefetch: cp.async copies a neighbour's fields into this
// thread's own shared-memory column one slot ahead (per-thread completion, no
// block barrier), so a row loop overlaps slot s+1's loads with slot s's math.
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// Row loop over the real slots s != diag in ascending order with a two-stage
// prefetch: slot s+1's fields are issued (issue(s, j, stage)) before slot s is
// consumed (body(s, stage)); the column of slot s+2 is loaded one iteration
// ahead so the issue never waits on it.
template <class Issue, class Body>
__device__ __forceinline__ void row_pipe(const int* __restrict__ col, int base, int card, int dg, Issue issue,
                                         Body body) {
  int sA = (dg == 0) ? 1 : 0;
  int sB = sA + 1 + (sA + 1 == dg ? 1 : 0);
  if (sA < card) issue(sA, col[base + sA * 32], 0);
  cp_commit();
  int jB = (sB < card) ? col[base + sB * 32] : 0;
  for (int it = 0; sA < card; ++it) {
    const int st = it & 1;
    if (sB < card) issue(sB, jB, st ^ 1);
    cp_commit();
    const int sC = sB + 1 + (sB + 1 == dg ? 1 : 0);
    const int jC = (sC < card) ? col[base + sC * 32] : 0;
    cp_wait1();
    body(sA, st);
    sA = sB;
    sB = sC;
    jB = jC;
  }
}
// k_low_order: the prefetch pays once the kernel may keep more registers
// (2D 5 blocks/SM: -21%; 3D 4 blocks/SM: -23%); k_row_visc: -3% in 2D.
// the row kernels form neighbour fluxes from v, p cached by step0 (measured:
// 2D k_row_visc -5%, k_low_order -10%, 3D k_low_order -19%; 3D k_row_visc
// neutral on the 160^3 box, -18% on the Sod box)
#define EF_VP_ROW(D) true
#define EF_VP_LOW(D) true
template <int D, bool USE>
__device__ __forceinline__ void node_flux(const double* Ui, const Work& w, int NP, int i, const Gas& g,
                                          double (*f)[D]) {
  if (USE) {
    double vp[D + 1];
    load_node<D + 1>(w.vp, NP, i, vp);
    flux_vp<D>(Ui, vp, vp[D], f);
  } else {
    flux<D>(Ui, g, f);
  }
}

template <int D>
__global__ void __launch_bounds__(EF_TPB_D(D), EF_LB(EF_MINB_ROW(D), D)) k_row_visc(Layout m, Gas g, const double* __restrict__ U,
                                                  Work w, int want_tau, int uni_on, RowSet rs, int stage) {
  constexpr int NV = D + 2;
  const int t0 = blockIdx.x * EF_TPB_D(D) + threadIdx.x;
  const bool act = t0 < rs.n;
  const int i = act ? rs.row(t0) : 0;
  double cand = __longlong_as_double(0x7ff0000000000000LL);
  bool bad = false;
  // frozen row: uniform stencil and state unchanged since the previous
  // (identical-state) stage -- then so are all its neighbours, all its d_ij
  // (memo), its alpha (0) and d_ii: only the CFL candidate is formed again
  // (and no P of the row's edges was formed in the previous stage: a limited pass
  // then added to U^L in place, so the stored U^L is not this stage's)
  const bool frozen = act && EF_FROZEN && uni_on && !w.nonuni[i] && !w.chg[i] && !w.pnz[i];
  if (frozen && want_tau) {
    const double dii = w.d[sidx32(i, m.diag[i], m.L)];
    if (dii < 0.0) cand = m.m_i[i] / (-2.0 * dii);
  }
  if (act && !frozen) {
    const int NP = (int)m.NP;
    const int L = m.L;
    const int NPL = NP * L;
    const int card = m.card[i], dg = m.diag[i];
    const int base = sidx32(i, 0, L);
    double Ui[NV];
    load_node<NV>(U, NP, i, Ui);
    double fi[NV][D];
    node_flux<D, EF_VP_ROW(D)>(Ui, w, NP, i, g, fi);
    const double eor_i = w.eor[i];
    double A = 0.0, B[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) B[k] = 0.0;
    // Uniform stencil (every neighbour's state is U_i bit for bit, hence the
    // same eor and flux): each slot adds (+0) * x = +-0 to sums that start at
    // +0, which leaves them +0 -- the loop is skipped (finite values assumed,
    // checked), and alpha_i = 0 follows from the unchanged tail.
    const bool uni = EF_UNIFORM_ROWS && uni_on && !w.nonuni[i] && all_finite<NV>(Ui) &&
                     all_finite<NV * D>(&fi[0][0]) && finite(eor_i);
    // one slot j != i (j == i contributes exact zeros), in slot order
    auto slot = [&](const double* Uj, const double* cc, double eor_j, const double* vpj) {
      double mc = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) mc = mc + Uj[1 + a] * cc[a];
      A = A + (eor_j - eor_i) * mc;
      double fj[NV][D];
      if (EF_VP_ROW(D)) flux_vp<D>(Uj, vpj, vpj[D], fj);
      else flux<D>(Uj, g, fj);
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        double t = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) t = t + (fj[k][a] - fi[k][a]) * cc[a];
        B[k] = B[k] + t;
      }
    };
    {
      constexpr int NQ = EF_VP_ROW(D) ? D + 1 : 0;  // v_j, p_j
      constexpr int K0 = EF_VP_ROW(D) ? 1 : 0;      // rho_j is not used once v_j, p_j are cached
      constexpr int F = (NV - K0) + 1 + D + NQ;     // U_j (from K0), eor_j, c, (v_j, p_j)
      __shared__ double buf[2][F][EF_TPB_D(D)];
      const int t = threadIdx.x;
      auto issue = [&](int s, int j, int st) {
        const int p = base + s * 32;
        EF_IN(j, m.n_local);
        EF_IN(p, NPL);
#pragma unroll
        for (int k = K0; k < NV; ++k) cp_async8(&buf[st][k - K0][t], U + k * NP + j);
        cp_async8(&buf[st][NV - K0][t], w.eor + j);
#pragma unroll
        for (int a = 0; a < D; ++a) cp_async8(&buf[st][NV - K0 + 1 + a][t], m.c + (size_t)a * NPL + p);
#pragma unroll
        for (int a = 0; a < NQ; ++a) cp_async8(&buf[st][NV - K0 + 1 + D + a][t], w.vp + a * NP + j);
      };
      auto body = [&](int, int st) {
        double Uj[NV], cc[D], vpj[D + 1];
        Uj[0] = 0.0;  // (unused with the v, p cache)
#pragma unroll
        for (int k = K0; k < NV; ++k) Uj[k] = buf[st][k - K0][t];
#pragma unroll
        for (int a = 0; a < D; ++a) cc[a] = buf[st][NV - K0 + 1 + a][t];
#pragma unroll
        for (int a = 0; a < NQ; ++a) vpj[a] = buf[st][NV - K0 + 1 + D + a][t];
        slot(Uj, cc, buf[st][NV - K0][t], vpj);
      };
      if (!uni) row_pipe(m.col, base, card, dg, issue, body);
    }
    // d row sum over the L padded slots (lower slots were filled by k_edge_visc)
    double* __restrict__ d = w.d;
    auto v = [&](int s) -> double {
      if (s == dg || s >= card) return 0.0;
      return d[base + s * 32];
    };
    double res;
    if (L < 8) {  // numpy pairwise_sum, n < 8: sequential from +0
      res = 0.0;
      for (int s = 0; s < L; ++s) res = res + v(s);
    } else {      // n >= 8: 8 accumulators, fixed tree, sequential tail
      double r[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) r[q] = v(q);
      const int Lm = L - (L % 8);
      for (int b = 8; b < Lm; b += 8) {
#pragma unroll
        for (int q = 0; q < 8; ++q) r[q] = r[q] + v(b + q);
      }
      res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
      for (int s = Lm; s < L; ++s) res = res + v(s);
    }
    const double dii = -res;
    d[base + dg * 32] = dii;
    if (want_tau && dii < 0.0) cand = m.m_i[i] / (-2.0 * dii);
    // IndicatorAccumulator.reset (harten_entropy_derivative, physics.py:133-148)
    double ep[NV];
    const double re = Ui[0] * internal_energy<D>(Ui);
    if (re <= 0.0) bad = true;
    if (uni) {  // A = B = +0: numer = denom = +0, so alpha = 0 whatever eta' is
      w.alpha[i] = 0.0;
    } else {
    {
      const double scale = dpow(re, g.neg_g_gp1_inv) * g.gp1_inv;  // physics.py:143
      ep[0] = scale * Ui[D + 1];
#pragma unroll
      for (int a = 0; a < D; ++a) ep[1 + a] = (-scale) * Ui[1 + a];
      ep[D + 1] = scale * Ui[0];
    }
    // IndicatorAccumulator.result, indicator.py:63-73
    double eb = 0.0;
#pragma unroll
    for (int k = 0; k < NV; ++k) eb = eb + ep[k] * B[k];
    const double numer = fabs((A - eb) + (eor_i * B[0]));
    double wb = 0.0;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const double wk = (k == 0) ? fabs(ep[0] - eor_i) : fabs(ep[k]);
      wb = wb + wk * fabs(B[k]);
    }
    const double denom = fabs(A) + wb;
    const double safe = denom > kDenomFloor ? denom : 1.0;
    const double al = npclip(div0(numer, safe), 0.0, 1.0);
    w.alpha[i] = denom > kDenomFloor ? al : 0.0;
    }
  }
  if (bad) raise_err(w, ERR_PROJECT, stage, PH_INDICATOR);
  if (!want_tau) return;
  __shared__ double red[EF_TPB_D(D) / 32];
  cand = warp_min(cand);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cand;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = red[0];
#pragma unroll
    for (int q = 1; q < EF_TPB_D(D) / 32; ++q) b = fmin(b, red[q]);
    // tau > 0: the IEEE bit pattern orders like the value
    atomicMin(w.tau_min_bits, (unsigned long long)__double_as_longlong(b));
  }
}

// ---------------------------------------------------------------- step3
__device__ __forceinline__ double stage_tau(const Work& w, const StageParams& sp) {
  double tau;
  if (sp.tau_mode == TAU_GIVEN) {
    tau = w.tau_arg[0];
  } else if (sp.tau_mode == TAU_DEVICE) {
    tau = *w.tau;
  } else {  // stepper.py:538-548
    const double tmin = __longlong_as_double((long long)*w.tau_min_bits);
    const double a = sp.c_cfl * tmin;
    const double tau_max = w.tau_arg[1];
    tau = (tau_max < a) ? tau_max : a;
  }
  return tau;
}


template <int D>
__global__ void __launch_bounds__(EF_TPB_D(D), EF_LB(EF_MINB_LOW(D), D)) k_low_order(Layout m, Gas g, const double* __restrict__ U,
                                                   Work w, StageParams sp, RowSet rs) {
  constexpr int NV = D + 2;
  const double tau = stage_tau(w, sp);
  const int t0 = blockIdx.x * EF_TPB_D(D) + threadIdx.x;
  if (t0 == 0 && rs.lead && sp.tau_mode != TAU_DEVICE) {
    *w.tau = tau;
    if (sp.tau_mode == TAU_CFL &&
        !(__longlong_as_double((long long)*w.tau_min_bits) < __longlong_as_double(0x7ff0000000000000LL)))
      raise_err(w, ERR_TAU_UNBOUNDED, sp.stage, PH_TAU);
  }
  if (t0 >= rs.n) return;
  const int i = rs.row(t0);
  if (EF_FROZEN && sp.uni && !w.nonuni[i] && !w.chg[i] && !w.pnz[i]) {  // as k_row_visc decides
    // frozen row (see k_row_visc): U^L, R, bounds and the zero-P mark from the
    // previous stage are this stage's values (U^L = U + (+0) does not depend on
    // tau); only the shortcut count and the row status are kept up
    if (sp.tau_mode != TAU_DEVICE && (blockIdx.x & 7) == 0) count_hits(true, w.n_same);
    w.ust[i] = 2;
    return;
  }
  const int NP = (int)m.NP;
  const int L = m.L;
  const int NPL = NP * L;
  double Ui[NV];
  load_node<NV>(U, NP, i, Ui);
  double fi[NV][D];
  node_flux<D, EF_VP_LOW(D)>(Ui, w, NP, i, g, fi);
  const double ai = w.alpha[i];
  double sumL[NV], sumR[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) sumL[k] = sumR[k] = 0.0;
  // the diagonal (and every pad) yields the bar state U_i and phi_i exactly
  double rmin = Ui[0], rmax = Ui[0], pmin = w.phi[i];
  const int card = m.card[i], dg = m.diag[i];
  const int base = sidx32(i, 0, L);
  // Uniform stencil: dU = +0 and f_j - f_i = +0 in every slot, so each slot adds
  // +0 to sumL / sumR and leaves the bounds at (rho_i, rho_i, phi_i) (the bar
  // state is 0.5 (rho_i + rho_i) - (+0) = rho_i): the loop is skipped.
  const bool uni = EF_UNIFORM_ROWS && sp.uni && !w.nonuni[i] && all_finite<NV>(Ui) &&
                   all_finite<NV * D>(&fi[0][0]) && finite(pmin) && fabs(Ui[0]) < 1e300;
  // one slot j != i of the row, in slot order (stepper.py:441-454)
  auto slot = [&](const double* Uj, const double* cc, double dv, double alj, double phij, const double* vpj) {
    double fj[NV][D];
    if (EF_VP_LOW(D)) flux_vp<D>(Uj, vpj, vpj[D], fj);
    else flux<D>(Uj, g, fj);
    const double dH = dv * (0.5 * (ai + alj));
    double ubar = 0.0;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const double dU = Uj[k] - Ui[k];
      double fdc = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) fdc = fdc + (fj[k][a] - fi[k][a]) * cc[a];
      sumL[k] = sumL[k] + ((dv * dU) - fdc);
      sumR[k] = sumR[k] + ((dH * dU) - fdc);
      if (k == 0) {
        const double corr = dv != 0.0 ? div0(fdc, 2.0 * dv) : 0.0;
        ubar = (0.5 * (Ui[0] + Uj[0])) - corr;
      }
    }
    rmin = npmin(rmin, ubar);
    rmax = npmax(rmax, ubar);
    pmin = npmin(pmin, phij);
  };
  {
    // fields per slot: U_j (NV), alpha_j, phi_j, c (D), d
    constexpr int NQ = EF_VP_LOW(D) ? D + 1 : 0;  // v_j, p_j
    constexpr int F = NV + 2 + D + 1 + NQ;
    __shared__ double buf[2][F][EF_TPB_D(D)];
    const int t = threadIdx.x;
    auto issue = [&](int s, int j, int st) {
      const int p = base + s * 32;
      EF_IN(j, m.n_local);
      EF_IN(p, NPL);
#pragma unroll
      for (int k = 0; k < NV; ++k) cp_async8(&buf[st][k][t], U + k * NP + j);
      cp_async8(&buf[st][NV][t], w.alpha + j);
      cp_async8(&buf[st][NV + 1][t], w.phi + j);
#pragma unroll
      for (int a = 0; a < D; ++a) cp_async8(&buf[st][NV + 2 + a][t], m.c + (size_t)a * NPL + p);
      cp_async8(&buf[st][NV + 2 + D][t], w.d + p);
#pragma unroll
      for (int a = 0; a < NQ; ++a) cp_async8(&buf[st][NV + 3 + D + a][t], w.vp + a * NP + j);
    };
    auto body = [&](int, int st) {
      double Uj[NV], cc[D];
#pragma unroll
      for (int k = 0; k < NV; ++k) Uj[k] = buf[st][k][t];
#pragma unroll
      for (int a = 0; a < D; ++a) cc[a] = buf[st][NV + 2 + a][t];
      double vpj[D + 1];
#pragma unroll
      for (int a = 0; a < NQ; ++a) vpj[a] = buf[st][NV + 3 + D + a][t];
      slot(Uj, cc, buf[st][NV + 2 + D][t], buf[st][NV][t], buf[st][NV + 1][t], vpj);
    };
    if (!uni) row_pipe(m.col, base, card, dg, issue, body);
  }
  const double fac = tau * m.inv_m[i];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    w.Unext[k * NP + i] = Ui[k] + (fac * sumL[k]);
    w.R[k * NP + i] = sumR[k];
  }
  w.bounds[i] = rmin;
  w.bounds[NP + i] = rmax;
  w.bounds[2 * NP + i] = pmin;
  if (EF_UNIFORM_ROWS && sp.uni && sp.passes > 0) {
    // first-pass factor of the edges between two uniform rows (their P is +-0,
    // R_i = R_j = +0 and U_j = U_i): limiter(U^L_i, 0, bounds_i); NaN = no shortcut
    w.ust[i] = uni ? 1 : 0;
    w.pnz[i] = 0;  // the first limiter pass marks the rows of every edge it computes
  }
  // uniform rows (keep the shortcuts on): sampled like k_edge_visc's count
  if (EF_UNIFORM_ROWS && sp.uni && sp.tau_mode != TAU_DEVICE && (blockIdx.x & 7) == 0) count_hits(uni, w.n_same);
}

// ---------------------------------------------------------------- steps 4-6
// Edge-parallel limiter.  For an edge (i, j) the correction fluxes of both
// rows, P_ij (row i, stepper.py:460-468) and P_ji (row j), their limiter
// factors l_ij = limiter(U^L_i, P_ij, bounds_i) and l_ji (limiter.py:149-193)
// and the symmetric factor min(l_ij, l_ji) (stepper.py:478-479) are formed by
// ONE thread, which writes P and min(l) to both rows' slots.  Later passes
// rescale P <- (1 - min l) P per side (stepper.py:485) and re-limit.  The row
// kernels then only stream their own slots.  Every operation is the
// reference's, in its order; each side uses its own m_ij / m_ji, alpha sum and
// factor, so nothing assumes symmetry that the inputs might not have.
template <int D>
__device__ __forceinline__ void edge_lim_store(const Layout& m, const Work& w, const StageParams& sp, int q, int p,
                                               int j, int pt, int e, int i, double li, double lj);

template <int D, bool FIRST, bool UNI>
__device__ __forceinline__ void edge_lim_one(const Layout& m, const Gas& g, const double* __restrict__ U,
                                             const Work& w, const StageParams& sp, int q, int p, int j,
                                             int pt, int e) {
  constexpr int NV = D + 2;
  const int i = (int)fdiv((uint32_t)p, m.slab) * 32 + (p & 31);
  const int NP = (int)m.NP;
  const size_t NPL = (size_t)NP * m.L;
  EF_IN(p, NPL);
  EF_IN(pt, NPL);
  EF_IN(i, m.n_local);
  EF_IN(j, m.n_local);
  double Pi[NV], Pj[NV];
  if (FIRST && UNI && EF_UNIFORM_ROWS) {
    // both rows took k_low_order's uniform shortcut (ust >= 1; owned rows):
    // R_i = R_j = +0 and U_j = U_i, so P_ij and P_ji are +-0 and stay zero in
    // every pass; each later use of the slots' factors multiplies a zero P
    const int no = (int)m.n_owned;
    if (i < no && j < no) {
      const int si = w.ust[i], sj = w.ust[j];
      if (si && sj) {
        // two frozen rows: the previous stage already tagged the slots
        if (si == 2 && sj == 2) return;
        // no P store and no limiter: the slots are tagged kZeroP instead of min(l)
        double* __restrict__ mo = sp.passes == 1 ? w.ml2 : w.ml;
        mo[p] = kZeroP;
        mo[pt] = kZeroP;
        return;
      }
    }
  }
  if (FIRST && UNI) {  // this edge's P is computed: both rows may carry a nonzero P
    w.pnz[i] = 1;
    w.pnz[j] = 1;
  }
  if (FIRST) {  // q == 0
    const double tau = *w.tau;
    const double imi = m.inv_m[i], imj = m.inv_m[j];
    const double fi = (tau * imi) * (double)(m.cardf[i] - 1);  // stepper.py:467 (full card)
    const double fj = (tau * imj) * (double)(m.cardf[j] - 1);
    const double ai = w.alpha[i], aj = w.alpha[j];
    const double dv = w.d[p];  // == d at pt (d is symmetric by construction)
    const double dHi = dv * (0.5 * (ai + aj));
    const double dHj = dv * (0.5 * (aj + ai));
    const double mij = m.mij[p], mji = m.mij[pt];
    const double bi = 0.0 - mij * imj, bTi = 0.0 - mij * imi;  // b_slot / bT_slot, stepper.py:234-236
    const double bj = 0.0 - mji * imi, bTj = 0.0 - mji * imj;
    const double ddi = dHi - dv, ddj = dHj - dv;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const double Uik = U[k * NP + i], Ujk = U[k * NP + j];
      const double Rik = w.R[k * NP + i], Rjk = w.R[k * NP + j];
      Pi[k] = fi * (((bi * Rjk) - (bTi * Rik)) + (ddi * (Ujk - Uik)));
      Pj[k] = fj * (((bj * Rik) - (bTj * Rjk)) + (ddj * (Uik - Ujk)));
    }
  } else {
    // (kZeroP slots and, in the last pass, min(l) == 1 slots never get here: the
    // kernel returns for them before loading anything else, see k_edge_lim)
    const double mli = w.ml[p], mlj = w.ml[pt];
    const double gi = 1.0 - mli, gj = 1.0 - mlj;
    if (EF_ZSKIP && gi == 0.0 && gj == 0.0) {
      // non-last pass, min(l) of the previous pass was 1: P rescales to +-0 on
      // both sides (P is finite, k_edge_lim<FIRST> checks) and stays zero, so
      // every later use of this slot's factor multiplies a zero P (the row
      // update adds +-0, the next P is +-0 again, k_final skips the slot): the
      // slots are tagged kZeroP and the P loads, both limiter evaluations and
      // the P store are skipped
      w.ml[p] = kZeroP;
      w.ml[pt] = kZeroP;
      return;
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      Pi[k] = w.P[(size_t)k * NPL + p] * gi;
      Pj[k] = w.P[(size_t)k * NPL + pt] * gj;
    }
  }
  if (FIRST && sp.passes >= 2) {  // the later passes' P = 0 shortcut assumes finite P
    bool fin = true;
#pragma unroll
    for (int k = 0; k < NV; ++k) fin = fin && finite(Pi[k]) && finite(Pj[k]);
    if (!fin) raise_err(w, ERR_NONFINITE_P, sp.stage, PH_P);
  }
  // The last pass q >= 1 leaves P_(q-1) and min(l) of pass q-1 in place: k_final
  // forms the same product P_(q-1) (1 - min l) itself, which saves the largest
  // write of the stage.  Every other pass stores its P_q.
  const bool last = q == sp.passes - 1;
  if (FIRST || !last) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      w.P[(size_t)k * NPL + p] = Pi[k];
      w.P[(size_t)k * NPL + pt] = Pj[k];
    }
  }
  double Un[NV];
  load_node<NV>(w.Unext, NP, i, Un);
  const double li = limiter<D>(Un, Pi, w.bounds[i], w.bounds[NP + i], w.bounds[2 * NP + i], sp.newton, g);
  load_node<NV>(w.Unext, NP, j, Un);
  const double lj = limiter<D>(Un, Pj, w.bounds[j], w.bounds[NP + j], w.bounds[2 * NP + j], sp.newton, g);
  edge_lim_store<D>(m, w, sp, q, p, j, pt, e, i, li, lj);
}

// min(l) of an edge to both rows' slots, and (pass before the last) the last
// pass's worklist entry and slot-mask bits
template <int D>
__device__ __forceinline__ void edge_lim_store(const Layout& m, const Work& w, const StageParams& sp, int q, int p,
                                               int j, int pt, int e, int i, double li, double lj) {
  const bool last = q == sp.passes - 1;
  double* __restrict__ ml = last ? w.ml2 : w.ml;
  const double mlv = npmin(li, lj);
  ml[p] = mlv;             // row i: np.minimum(l_ij, l_ji)
  ml[pt] = npmin(lj, li);  // row j: np.minimum(l_ji, l_ij)
  // the pass before the last lists the edges the last pass has work for
  if (EF_WL && q == sp.passes - 2) {
    wl_append(mlv != 1.0, e, w.wl, w.wl_n);
    if (mlv != 1.0 && m.L <= 64) {  // the slots of this edge in rows i and j
      const int sL = 32 * m.L;
      EF_IN((p - (i >> 5) * sL) >> 5, m.L);
      EF_IN((pt - (j >> 5) * sL) >> 5, m.L);
      atomicOr(w.lmask + i, 1ull << ((p - (i >> 5) * sL) >> 5));
      atomicOr(w.lmask + j, 1ull << ((pt - (j >> 5) * sL) >> 5));
    }
  }
}

template <int D, bool FIRST, bool UNI>
__global__ void __launch_bounds__(EF_TPB_D(D), EF_LB(EF_MINB_ELIM(D, FIRST), D)) k_edge_lim(Layout m, Gas g,
                                                                        const double* __restrict__ U,
                                                                        Work w, StageParams sp, int q) {
  const int e = blockIdx.x * EF_TPB_D(D) + threadIdx.x;
  const int NE = (int)m.n_edges;
  if (e >= NE) return;
  if (EF_PF_LIM > 0 && e + EF_PF_LIM < NE) {
    const int f = e + EF_PF_LIM;
    pf_l2(m.edges + f);
    pf_l2(m.edge_j + f);
    pf_l2(m.edge_pt + f);
  }
  const int p = m.edges[e];
  if (!FIRST) {
    // kZeroP slot: P stays zero and nothing reads its factor again.  Last pass
    // with min(l) == 1: P rescales to +-0 and k_final skips the slot (its term
    // is ml2 * (+-0)), so neither the factor nor anything else is needed.
    const double mli = w.ml[p];
    if (mli < 0.0 || (EF_ZSKIP && mli == 1.0 && q == sp.passes - 1)) return;
  }
  edge_lim_one<D, FIRST, UNI>(m, g, U, w, sp, q, p, m.edge_j[e], m.edge_pt[e], e);
}

// The last limiter pass over the worklist (grid-stride over its device-side
// count): every other edge has min(l) == 1 or a kZeroP tag from the pass before,
// i.e. nothing to do in the last pass (see k_edge_lim).
template <int D>
__global__ void __launch_bounds__(EF_TPB_D(D), EF_LB(EF_MINB_ELIM(D, false), D))
    k_edge_lim_last(Layout m, Gas g, const double* __restrict__ U, Work w, StageParams sp, int q) {
  const int n = *w.wl_n;
  EF_ASSERT(n <= m.n_edges);
  for (int t = blockIdx.x * EF_TPB_D(D) + threadIdx.x; t < n; t += gridDim.x * EF_TPB_D(D)) {
    const int e = w.wl[t];
    EF_IN(e, m.n_edges);
    edge_lim_one<D, false, false>(m, g, U, w, sp, q, m.edges[e], m.edge_j[e], m.edge_pt[e], e);
  }
}

// step5 (non-final pass): U_next_i += lam_i * sum_s min(l) P in slot order
// (stepper.py:478-481); the rescale of P belongs to the next k_edge_lim.
template <int D>
__global__ void __launch_bounds__(EF_TPB_D(D), EF_LB(EF_MINB_PASS(D), D)) k_row_upd(Layout m, Gas g, const double* __restrict__ U,
                                                                Work w, StageParams sp, RowSet rs, int use_mask) {
  constexpr int NV = D + 2;
  const int t0 = blockIdx.x * EF_TPB_D(D) + threadIdx.x;
  if (t0 >= rs.n) return;
  const int i = rs.row(t0);
  const int NP = (int)m.NP;
  const int L = m.L;
  const size_t NPL = (size_t)NP * L;
  const int card = m.card[i], dg = m.diag[i];
  const int base = sidx32(i, 0, L);
  double upd[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) upd[k] = 0.0;
  // every P of the row is the first pass's stored +0 (kept zero by later
  // passes): each term is +-0 and the sums stay +0, so the loop is skipped
  const int nslots = (EF_UNIFORM_ROWS && sp.uni && !w.pnz[i]) ? 0 : card;
  // use_mask: the pass just done built the slot masks (k_final's) and left no
  // kZeroP tags (first of two passes, no identical-state shortcuts): a slot
  // outside the mask has min(l) == 1 exactly, and 1.0 * P == P, so its factor
  // is not loaded
  const unsigned long long mk = use_mask ? w.lmask[i] : 0ull;
#pragma unroll 1
  for (int s = 0; s < nslots; ++s) {
    if (s == dg) continue;
    const int p = base + s * 32;
    EF_IN(p, NPL);
    const double ml = (use_mask && !((mk >> s) & 1ull)) ? 1.0 : w.ml[p];
    if (ml < 0.0) continue;  // kZeroP: the term is ml * (+-0)
#pragma unroll
    for (int k = 0; k < NV; ++k) upd[k] = upd[k] + ml * w.P[(size_t)k * NPL + p];
  }
  const double lam = m.lam[i];
  double Un[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    Un[k] = w.Unext[k * NP + i] + lam * upd[k];
    w.Unext[k * NP + i] = Un[k];
  }
}

template <int D>
__global__ void __launch_bounds__(EF_TPB_D(D), EF_LB(EF_MINB_FINAL(D), D)) k_final(Layout m, Gas g, const double* __restrict__ U,
                                               const double* __restrict__ U0, double* __restrict__ Uout,
                                               Work w, StageParams sp, RowSet rs) {
  constexpr int NV = D + 2;
  const int t0 = blockIdx.x * EF_TPB_D(D) + threadIdx.x;
  if (t0 >= rs.n) return;
  const int i = rs.row(t0);
  const int NP = (int)m.NP;
  const int L = m.L;
  const size_t NPL = (size_t)NP * L;
  double Un[NV];
  load_node<NV>(w.Unext, NP, i, Un);
  if (sp.passes > 0) {
    const int card = m.card[i], dg = m.diag[i];
    const int base = sidx32(i, 0, L);
    double upd[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) upd[k] = 0.0;
    const bool rescale = sp.passes >= 2;  // P of the last pass = P_(q-1) (1 - min l_(q-1))
    // all P zero (k_row_upd), or (worklist) only the slots of the row's
    // worklist edges -- min(l) < 1 in the pass before the last -- can carry a
    // nonzero rescaled term; the others add +-0 or are tagged zeros.  Their
    // bits are visited in increasing slot order, the order of the full loop.
    // (a zero-P row never gets a mask bit: all its edges are tagged)
    const bool zrow = EF_UNIFORM_ROWS && sp.uni && !w.pnz[i];
    const bool lr = EF_WL && rescale && !zrow && L <= 64;
    unsigned long long mk = 0;
    if (lr) {
      mk = w.lmask[i];
      if (mk) w.lmask[i] = 0;  // cleared for the next stage
    }
    const int nslots = (zrow || lr) ? 0 : card;
    auto term = [&](int s) {
      const int p = base + s * 32;
      EF_IN(p, NPL);
      EF_ASSERT(s < card);
      const double mlp = rescale ? w.ml[p] : 0.0;
      const double gp = rescale ? 1.0 - mlp : 1.0;
      // gp == 0: the term is ml2 * (P * 0) = +-0 (P finite), and adding +-0 to a
      // sum that starts at +0 never changes it (it cannot become -0); kZeroP
      // slots (negative tag) carry a zero P
      if ((EF_ZSKIP && gp == 0.0) || mlp < 0.0) return;
      const double ml = w.ml2[p];
      if (ml < 0.0) return;  // kZeroP from a single-pass first limiter
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const double Pk = rescale ? w.P[(size_t)k * NPL + p] * gp : w.P[(size_t)k * NPL + p];
        upd[k] = upd[k] + ml * Pk;
      }
    };
#pragma unroll 1
    for (int s = 0; s < nslots; ++s)
      if (s != dg) term(s);
    while (mk) {
      term(__ffsll((long long)mk) - 1);
      mk &= mk - 1;
    }
    const double lam = m.lam[i];
#pragma unroll
    for (int k = 0; k < NV; ++k) Un[k] = Un[k] + lam * upd[k];
  }
  // _k_boundary, stepper.py:493-504: slip projection, then inflow reset
  const int kind = m.bc_kind[i];
  if (kind & 1) {
    double nr[D], mn = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      nr[a] = m.bc_n[a * NP + i];
      mn = mn + Un[1 + a] * nr[a];
    }
#pragma unroll
    for (int a = 0; a < D; ++a) Un[1 + a] = Un[1 + a] - mn * nr[a];
  }
  if (kind & 2) {
#pragma unroll
    for (int k = 0; k < NV; ++k) Un[k] = m.farfield[k];
  }
  // _finish_step admissibility, stepper.py:612-621
  if (!((Un[0] > 0.0) && (internal_energy<D>(Un) > 0.0))) {
    raise_err(w, ERR_BAD_STATE, sp.stage, PH_STATE);
    // the earliest failing stage first (the reference stops there), then the
    // smallest CM id of that stage
    atomicMin(w.bad_gid, ((unsigned long long)sp.stage << 56) | (unsigned long long)m.gid[i]);
  }
  double Uo[NV];
  if (sp.rk_a >= 0.0) {  // ssp_rk3_step incremental combination, stepper.py:632,635
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const double u0 = U0[k * NP + i];
      Uo[k] = u0 + sp.rk_a * (Un[k] - u0);
    }
  } else {
#pragma unroll
    for (int k = 0; k < NV; ++k) Uo[k] = Un[k];
  }
#pragma unroll
  for (int k = 0; k < NV; ++k) Uout[k * NP + i] = Uo[k];
  // flags for the next stage: after an identical-state stage, an unchanged row
  // keeps its d_ij memo and its uniformity mark (k_edge_visc recomputes every
  // edge with a changed end); otherwise everything is recomputed
  bool changed = true;
  if (EF_UNIFORM_ROWS && sp.uni) {
    double Ui[NV];
    load_node<NV>(U, NP, i, Ui);
    changed = !same_state<NV>(Uo, Ui);
  }
  w.chg[i] = changed ? 1 : 0;
  if (changed) w.nonuni[i] = 0;
  // next stage's step0; an unchanged row's eor, phi, v, p (pure functions of
  // its state) are already in place
  if (changed) nodal_one<D>(Uo, g, w, NP, i);
}

// ---------------------------------------------------------------- halo packing
// rows: buf[r * ncomp + k] <-> field[k * NP + idx[r]]; slots: buf[q] <-> arr[pos[q]]
__global__ void k_pack_rows(const double* __restrict__ field, int ncomp, int64_t NP,
                            const int32_t* __restrict__ idx, int64_t count, double* __restrict__ buf,
                            int stride, int coff) {
  const int64_t q = blockIdx.x * (int64_t)TPB + threadIdx.x;
  if (q >= count * ncomp) return;
  const int64_t r = q / ncomp;
  const int k = (int)(q - r * ncomp);
  EF_IN(idx[r], NP);
  buf[r * stride + coff + k] = field[k * NP + idx[r]];
}
__global__ void k_unpack_rows(double* __restrict__ field, int ncomp, int64_t NP,
                              const int32_t* __restrict__ idx, int64_t count, const double* __restrict__ buf,
                              int stride, int coff) {
  const int64_t q = blockIdx.x * (int64_t)TPB + threadIdx.x;
  if (q >= count * ncomp) return;
  const int64_t r = q / ncomp;
  const int k = (int)(q - r * ncomp);
  EF_IN(idx[r], NP);
  field[k * NP + idx[r]] = buf[r * stride + coff + k];
}
// min of the CFL bounds of every rank of a same-device group, written back to all
__global__ void k_group_min(unsigned long long* const* bits, int n) {
  unsigned long long v = ~0ull;
  for (int r = 0; r < n; ++r) v = min(v, *bits[r]);
  for (int r = 0; r < n; ++r) *bits[r] = v;
}

__global__ void k_pow(const double* __restrict__ x, double y, double* __restrict__ out, int64_t n) {
  const int64_t q = blockIdx.x * (int64_t)TPB + threadIdx.x;
  if (q < n) out[q] = ef_pow(x[q], y);
}

// ---------------------------------------------------------------- launchers
// process-wide count of kernel launches issued through the launchers below
// (a CUDA-graph replay adds the count its capture recorded; ef_capi.cu)
static std::atomic<long long> g_launches{0};
long long kernel_launches() { return g_launches.load(std::memory_order_relaxed); }
void add_kernel_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
#define EF_COUNT() g_launches.fetch_add(1, std::memory_order_relaxed)
#define EF_DISPATCH(dim, KERNEL, GRID, ...)                                   \
  do {                                                                        \
    EF_COUNT();                                                               \
    if ((dim) == 2) KERNEL<2><<<(GRID), TPB, 0, st>>>(__VA_ARGS__);          \
    else KERNEL<3><<<(GRID), TPB, 0, st>>>(__VA_ARGS__);                     \
  } while (0)
// stage kernels: grid for n items with the dimension's block size
static inline unsigned grid_d(int dim, int64_t n) {
  const int b = dim == 3 ? EF_TPB3 : EF_TPB2;
  return (unsigned)((n + b - 1) / b);
}
#define EF_DISPATCH_STAGE(dim, KERNEL, N, ...)                                                      \
  do {                                                                                              \
    EF_COUNT();                                                                                     \
    if ((dim) == 2) KERNEL<2><<<grid_d(2, (N)), EF_TPB2, 0, st>>>(__VA_ARGS__);                     \
    else KERNEL<3><<<grid_d(3, (N)), EF_TPB3, 0, st>>>(__VA_ARGS__);                                \
  } while (0)

void launch_gather_state(int dim, const Layout& m, int64_t count, const double* U_aos, const int64_t* orig,
                         double* U, int* err, cudaStream_t st) {
  if (count == 0) return;
  EF_DISPATCH(dim, k_gather_state, grid_for(count), m, count, U_aos, orig, U, err);
}
void launch_scatter_state(int dim, const Layout& m, const double* U, const int64_t* orig,
                          double* U_aos, cudaStream_t st) {
  if (m.n_owned == 0) return;
  EF_DISPATCH(dim, k_scatter_state, grid_for(m.n_owned), m, U, orig, U_aos);
}
void launch_nodal(int dim, const Layout& m, const Gas& g, const double* U, Work w, int64_t lo,
                  int64_t hi, cudaStream_t st) {
  if (hi <= lo) return;
  EF_DISPATCH(dim, k_nodal, grid_for(hi - lo), m, g, U, w, lo, hi);
}
void launch_edge_visc(int dim, const Layout& m, const Gas& g, const double* U, Work w, int stage,
                      bool reset_tau, bool uni, bool count, cudaStream_t st) {
  const int64_t n = m.n_edges > 0 ? m.n_edges : 1;
  const int r = (reset_tau ? 1 : 0) | (count ? 2 : 0) | (stage << 4);
  EF_COUNT();
  if (dim == 2) {
    if (uni) k_edge_visc<2, true><<<grid_d(2, n), EF_TPB2, 0, st>>>(m, g, U, w, r);
    else k_edge_visc<2, false><<<grid_d(2, n), EF_TPB2, 0, st>>>(m, g, U, w, r);
  } else {
    if (uni) k_edge_visc<3, true><<<grid_d(3, n), EF_TPB3, 0, st>>>(m, g, U, w, r);
    else k_edge_visc<3, false><<<grid_d(3, n), EF_TPB3, 0, st>>>(m, g, U, w, r);
  }
}
void launch_row_visc(int dim, const Layout& m, const Gas& g, const double* U, Work w, int stage,
                     bool want_tau, bool uni, RowSet rs, cudaStream_t st) {
  EF_DISPATCH_STAGE(dim, k_row_visc, rs.n > 0 ? rs.n : 1, m, g, U, w, want_tau ? 1 : 0, uni ? 1 : 0, rs, stage);
}
void launch_low_order(int dim, const Layout& m, const Gas& g, const double* U, Work w,
                      StageParams sp, RowSet rs, cudaStream_t st) {
  EF_DISPATCH_STAGE(dim, k_low_order, rs.n > 0 ? rs.n : 1, m, g, U, w, sp, rs);
}
bool edge_lim_worklist() { return EF_WL != 0; }

template <int D>
static void edge_lim_launch(const Layout& m, const Gas& g, const double* U, Work w, StageParams sp, int q,
                            cudaStream_t st) {
  constexpr int tb = D == 3 ? EF_TPB3 : EF_TPB2;
  const unsigned grid = grid_d(D, m.n_edges);
  EF_COUNT();
  if (EF_WL && q > 0 && q == sp.passes - 1)
    k_edge_lim_last<D><<<grid < EF_WL_GRID ? grid : EF_WL_GRID, tb, 0, st>>>(m, g, U, w, sp, q);
  else if (q > 0) k_edge_lim<D, false, false><<<grid, tb, 0, st>>>(m, g, U, w, sp, q);
  else if (sp.uni) k_edge_lim<D, true, true><<<grid, tb, 0, st>>>(m, g, U, w, sp, q);
  else k_edge_lim<D, true, false><<<grid, tb, 0, st>>>(m, g, U, w, sp, q);
}

void launch_edge_lim(int dim, const Layout& m, const Gas& g, const double* U, Work w,
                     StageParams sp, int q, cudaStream_t st) {
  if (m.n_edges == 0) return;
  if (dim == 2) edge_lim_launch<2>(m, g, U, w, sp, q, st);
  else edge_lim_launch<3>(m, g, U, w, sp, q, st);
}
void launch_row_upd(int dim, const Layout& m, const Gas& g, const double* U, Work w,
                    StageParams sp, RowSet rs, int q, cudaStream_t st) {
  if (rs.n == 0) return;
  // (two passes: the mask-building pass is the first, which tags only in the
  // identical-state mode; a middle pass of three or more tags its P = 0 slots)
  const int use_mask = (EF_WL && !sp.uni && sp.passes == 2 && q == 0 && m.L <= 64) ? 1 : 0;
  EF_DISPATCH_STAGE(dim, k_row_upd, rs.n, m, g, U, w, sp, rs, use_mask);
}
void launch_final(int dim, const Layout& m, const Gas& g, const double* U, const double* U0,
                  double* Uout, Work w, StageParams sp, RowSet rs, cudaStream_t st) {
  if (rs.n == 0) return;
  EF_DISPATCH_STAGE(dim, k_final, rs.n, m, g, U, U0, Uout, w, sp, rs);
}
void launch_pack_rows(const double* field, int ncomp, int64_t NP, const int32_t* idx, int64_t count,
                      double* buf, int stride, int coff, cudaStream_t st) {
  if (count > 0 && EF_COUNT() >= 0)
    k_pack_rows<<<grid_for(count * ncomp), TPB, 0, st>>>(field, ncomp, NP, idx, count, buf, stride, coff);
}
void launch_unpack_rows(double* field, int ncomp, int64_t NP, const int32_t* idx, int64_t count,
                        const double* buf, int stride, int coff, cudaStream_t st) {
  if (count > 0 && EF_COUNT() >= 0)
    k_unpack_rows<<<grid_for(count * ncomp), TPB, 0, st>>>(field, ncomp, NP, idx, count, buf, stride, coff);
}
void launch_group_min(unsigned long long* const* bits_dev, int n, cudaStream_t st) {
  EF_COUNT();
  k_group_min<<<1, 1, 0, st>>>(bits_dev, n);
}
__global__ void k_pow_ub(const double* __restrict__ x, double y, double* __restrict__ out, int64_t n) {
  const int64_t q = blockIdx.x * (int64_t)TPB + threadIdx.x;
  if (q < n) out[q] = pow_ub(x[q], y);
}
void launch_pow_ub(const double* x, double y, double* out, int64_t n, cudaStream_t st) {
  if (n > 0) k_pow_ub<<<grid_for(n), TPB, 0, st>>>(x, y, out, n);
}
void launch_pow(const double* x, double y, double* out, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  k_pow<<<grid_for(n), TPB, 0, st>>>(x, y, out, n);
}

// ---------------------------------------------------------------- function checks
// d_ij and the limiter on batches of independent inputs (AoS), through exactly
// the device code the stage kernels run (the edge geometry formed as the
// setup forms it: |c| = sqrt(R1(c*c)), n = c / |c|, e_1 for c = 0).
template <int D>
__global__ void k_eval_dij(Gas g, int64_t n, const double* __restrict__ Ui, const double* __restrict__ Uj,
                           const double* __restrict__ cij, const double* __restrict__ cji,
                           double* __restrict__ out, int* __restrict__ bad) {
  constexpr int NV = D + 2;
  const int64_t q = blockIdx.x * (int64_t)TPB + threadIdx.x;
  if (q >= n) return;
  double a[NV], b[NV], nij[D], nji[D];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    a[k] = Ui[q * NV + k];
    b[k] = Uj[q * NV + k];
  }
  double sij = 0.0, sji = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    sij = sij + cij[q * D + k] * cij[q * D + k];
    sji = sji + cji[q * D + k] * cji[q * D + k];
  }
  const double norm_ij = sqrt(sij), norm_ji = sqrt(sji);
#pragma unroll
  for (int k = 0; k < D; ++k) {
    nij[k] = norm_ij > 0.0 ? cij[q * D + k] / norm_ij : (k == 0 ? 1.0 : 0.0);
    nji[k] = norm_ji > 0.0 ? cji[q * D + k] / norm_ji : (k == 0 ? 1.0 : 0.0);
  }
  bool bd = false;
  double dv;
  // as k_edge_visc<D, true>: identical states by their closed form, then the straight-line path, else the general code
  const bool same = same_state<NV>(a, b);
  if (!d_ij_sl<D>(a, b, nij, norm_ij, nji, norm_ji, g, dv, same)) dv = d_ij_geo<D>(a, b, nij, norm_ij, nji, norm_ji, g, bd, same);
  out[q] = dv;
  bad[q] = bd ? 1 : 0;
}

template <int D>
__global__ void k_eval_limiter(Gas g, int64_t n, const double* __restrict__ U, const double* __restrict__ P,
                               const double* __restrict__ bounds, int newton, double* __restrict__ out) {
  constexpr int NV = D + 2;
  const int64_t q = blockIdx.x * (int64_t)TPB + threadIdx.x;
  if (q >= n) return;
  double u[NV], pp[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    u[k] = U[q * NV + k];
    pp[k] = P[q * NV + k];
  }
  out[q] = limiter<D>(u, pp, bounds[3 * q], bounds[3 * q + 1], bounds[3 * q + 2], newton, g);
}

// the straight-line primitives against the compiler's own 1/b, a/b, sqrt (test hook):
// mism[0..2] count operands in the safe range whose results differ
__global__ void k_eval_arith(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                             unsigned long long* __restrict__ mism) {
  const int64_t q = blockIdx.x * (int64_t)TPB + threadIdx.x;
  if (q >= n) return;
  const double x = a[q], y = b[q];
  if (!(exp_within<450>(x) && exp_within<450>(y))) return;
  if (__double_as_longlong(rcp_sl(y)) != __double_as_longlong(1.0 / y)) atomicAdd(mism + 0, 1ULL);
  if (__double_as_longlong(div_sl(x, y)) != __double_as_longlong(x / y)) atomicAdd(mism + 1, 1ULL);
  const double ax = fabs(x);
  if (__double_as_longlong(sqrt_sl(ax)) != __double_as_longlong(sqrt(ax))) atomicAdd(mism + 2, 1ULL);
  const double yr = 1.0 / y;
  if (__double_as_longlong(qdiv_sl(x, y, yr)) != __double_as_longlong(x / y)) atomicAdd(mism + 3, 1ULL);
}
void launch_eval_arith(int64_t n, const double* a, const double* b, unsigned long long* mism, cudaStream_t st) {
  if (n > 0) k_eval_arith<<<grid_for(n), TPB, 0, st>>>(n, a, b, mism);
}

void launch_eval_dij(int dim, const Gas& g, int64_t n, const double* Ui, const double* Uj, const double* cij,
                     const double* cji, double* out, int* bad, cudaStream_t st) {
  if (n <= 0) return;
  EF_DISPATCH(dim, k_eval_dij, grid_for(n), g, n, Ui, Uj, cij, cji, out, bad);
}
void launch_eval_limiter(int dim, const Gas& g, int64_t n, const double* U, const double* P,
                         const double* bounds, int newton, double* out, cudaStream_t st) {
  if (n <= 0) return;
  EF_DISPATCH(dim, k_eval_limiter, grid_for(n), g, n, U, P, bounds, newton, out);
}

}  // namespace ef
