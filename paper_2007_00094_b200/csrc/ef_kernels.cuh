// ef_kernels.cuh — device data layout and kernel launch interface.
//
// Layout in HBM (one rank = owned rows followed by ghost rows, padded to a
// multiple of 32 rows, NP):
//   * per-node fields are structure-of-arrays: field[k * NP + i];
//   * per-slot fields are SELL-32 with the global pad width L, slot-major
//     inside a 32-row slice: sidx(i, s) = (i / 32) * 32 * L + s * 32 + i % 32.
//     A warp owns one slice, so slot s of 32 consecutive rows is one 256-byte
//     coalesced transaction per fp64 field.
//   * slots of a row are sorted by global Cuthill-McKee id (stepper.py:195),
//     so "upper" (global id above the row's) == slot index above the diagonal
//     slot; pads (s >= card) are never touched after setup.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "ef_math.cuh"

namespace ef {

__host__ __device__ __forceinline__ int64_t sidx(int64_t i, int s, int L) {
  return (i >> 5) * (int64_t)(32 * L) + (int64_t)s * 32 + (i & 31);
}

// Division by a runtime constant d < 2^31 for unsigned n < 2^32 (round-up
// multiply-high method): q = (umulhi(n, mul) + n) >> shift.
struct FastDiv {
  uint32_t d, mul, shift;
};

inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  f.shift = l;
  f.mul = (uint32_t)((((1ull << 32) * ((1ull << l) - d)) / d) + 1);
  return f;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return (uint32_t)((((unsigned long long)__umulhi(n, f.mul)) + n) >> f.shift);
}

struct Layout {
  int L;            // global pad width
  int64_t NP;       // padded local rows (multiple of 32)
  int64_t n_local;  // owned + ghost rows
  int64_t n_owned;
  const int32_t* col;    // [NP*L] local column id (pads: the row itself)
  const uint8_t* tslot;  // [NP*L] slot of (col, row) in row col
  const uint8_t* card;   // [NP] valid slots in the (possibly truncated) stencil
  const uint8_t* cardf;  // [NP] full stencil cardinality (ghost rows: the owner's)
  const uint8_t* diag;   // [NP] slot of the diagonal
  const double* c;       // [D][NP*L]  c_ij
  const double* egeo;    // [n_edges][2(D+1)]  n_ij, |c_ij|, n_ji, |c_ji| per upper edge (16-byte aligned records)
  const double* mij;     // [NP*L]     consistent mass m_ij
  const double* m_i;     // [NP] lumped mass
  const double* inv_m;   // [NP]
  const double* lam;     // [NP] 1 / max(card - 1, 1)   (stepper.py:214-215)
  const int64_t* gid;    // [NP] global CM id of each local row
  const int8_t* bc_kind; // [NP] bit0 slip, bit1 inflow
  const double* bc_n;    // [D][NP] slip normal
  const int32_t* edges;  // [n_edges] SELL positions of the upper slots of all local rows, ascending
  const int32_t* edge_j;   // [n_edges] column j of the edge (= col at edges[e])
  const int32_t* edge_pt;  // [n_edges] SELL position of the transposed slot (j, i)
  int64_t n_edges;
  FastDiv slab;          // division by 32 * L (SELL slice size)
  double farfield[5];
};

struct Work {
  double* eor;       // [NP]
  double* phi;       // [NP]
  double* vp;        // [(D+1)*NP] v = m / rho (D comps), p = gm1 * eps: the flux inputs
  double* alpha;     // [NP]
  double* R;         // [NV][NP]
  double* Unext;     // [NV][NP]
  double* bounds;    // [3][NP] rho_min, rho_max, phi_min
  double* d;         // [NP*L]
  double* ml;        // [NP*L] min(l_ij, l_ji) of the current non-final limiter pass
  double* ml2;       // [NP*L] min(l_ij, l_ji) of the last limiter pass
  double* P;         // [NV][NP*L] correction fluxes P_ij, rescaled in place per pass
  uint8_t* nonuni;   // [NP] 1 if some stencil neighbour's state differs from the row's
                     // (bitwise); set by k_edge_visc, cleared by step0 (k_final / k_nodal)
  uint8_t* chg;      // [NP] 1 unless the row's state is bitwise the one of the previous
                     // (identical-state) stage: d_ij of two unchanged rows is kept
  uint8_t* pnz;      // [NP] (identical-state stages) 1 if some P_ij of the row may be nonzero;
                     // 0: every edge of the row took the first pass's P = 0 shortcut
  int* wl;           // [n_edges] worklist of the last limiter pass: the edges whose min(l)
  int* wl_n;         // came out below 1 in the pass before it (count in wl_n)
  unsigned long long* lmask;  // [NP] bit s: slot s of the row belongs to a worklist edge (its
                              // k_final rescaled term can be nonzero); cleared by k_final
  uint8_t* ust;      // [NP] k_low_order's row status for the first limiter pass: 0 general,
                     // 1 uniform-stencil shortcut (R = 0), 2 frozen (also unchanged)
  unsigned long long* tau_min_bits;  // CFL min over owned rows
  double* tau;       // tau of the current RK step / Euler step
  double* tau_arg;   // [2] the step's tau (TAU_GIVEN) and tau_max, written before every step
                     // (kept out of the kernel arguments so one CUDA graph serves every tau)
  int* err;          // ErrBits of every error since the flags were last read (ef_sync /
                     // a synchronous step / set_state): errors latch across async steps
  int* err_first;    // min over the errors of (stage * 8 + phase): the one the reference
                     // would have raised first (stepper.py:508-622 order of the checks)
  unsigned long long* bad_gid;       // min of (stage << 56 | global CM id) of an inadmissible row
  unsigned long long* n_same;        // [kSameSlots] spread counters since the last reset:
                                     // identical-state edges (shortcuts off) or uniform rows (on)
};

constexpr int kSameSlots = 128;
enum TauMode { TAU_CFL = 0, TAU_GIVEN = 1, TAU_DEVICE = 2 };
enum ErrBits { ERR_PROJECT = 1, ERR_BAD_STATE = 2, ERR_TAU_UNBOUNDED = 4, ERR_NONFINITE_P = 8 };
// phase of a check inside a stage, in the reference's order: d_ij projections
// (step1), the indicator's entropy derivative (step1), tau (step2/3), P (step4),
// the admissibility of the result (_finish_step)
enum ErrPhase { PH_VISC = 0, PH_INDICATOR = 1, PH_TAU = 2, PH_P = 3, PH_STATE = 4 };
constexpr int kErrNone = 0x7fffffff;

struct StageParams {
  int tau_mode;
  int stage;  // 0..2: stage of the RK step (error ordering)
  double c_cfl;
  int newton;
  int passes;
  double rk_a;  // < 0: Uout = Unew; else Uout = U0 + rk_a * (Unew - U0)   (stepper.py:632,635)
  int uni;      // identical-state shortcuts on (k_edge_visc marks rows; the row kernels and
                // the first limiter pass use the marks); chosen per step by the host
};

// Owned rows a row kernel covers: [r0, r0 + n0) then [r2, r2 + n - n0).  The
// whole range, or (with communication overlap, stepper.py Alg. 4) the rows
// other ranks import -- a prefix and a suffix of the CM range -- and then the
// interior.  `lead` marks the launch that also writes the stage's scalars.
struct RowSet {
  int r0 = 0, n0 = 0, r2 = 0, n = 0, lead = 1;
  __host__ __device__ int row(int t) const { return t < n0 ? r0 + t : r2 + (t - n0); }
};
inline RowSet all_rows(int64_t n_owned) {
  RowSet r;
  r.n0 = r.n = (int)n_owned;
  r.r2 = (int)n_owned;
  return r;
}

// launch wrappers (ef_kernels.cu); all asynchronous on `st`
void launch_gather_state(int dim, const Layout& m, int64_t count, const double* U_aos, const int64_t* orig_of_local,
                         double* U, int* err, cudaStream_t st);
void launch_scatter_state(int dim, const Layout& m, const double* U, const int64_t* orig_of_local,
                          double* U_aos, cudaStream_t st);
void launch_nodal(int dim, const Layout& m, const Gas& g, const double* U, Work w, int64_t lo,
                  int64_t hi, cudaStream_t st);
// step1a: d_ij on every upper edge (one thread per edge)
void launch_edge_visc(int dim, const Layout& m, const Gas& g, const double* U, Work w, int stage,
                      bool reset_tau, bool uni, bool count, cudaStream_t st);
// step1b+2: per owned row, indicator alpha, mirror of d, d_ii, CFL bound
void launch_row_visc(int dim, const Layout& m, const Gas& g, const double* U, Work w, int stage,
                     bool want_tau, bool uni, RowSet rs, cudaStream_t st);
void launch_low_order(int dim, const Layout& m, const Gas& g, const double* U, Work w,
                      StageParams sp, RowSet rs, cudaStream_t st);
// steps 4-5: P (q = 0) and min(l_ij, l_ji) of limiter pass q, one thread per edge
void launch_edge_lim(int dim, const Layout& m, const Gas& g, const double* U, Work w,
                     StageParams sp, int q, cudaStream_t st);
// true if the last limiter pass runs over the worklist (EF_WL); the pass before it
// then needs *wl_n cleared first
bool edge_lim_worklist();
long long kernel_launches();
void add_kernel_launches(long long n);
// step5: non-final pass row update U_next += lam * sum min(l) P
void launch_row_upd(int dim, const Layout& m, const Gas& g, const double* U, Work w,
                    StageParams sp, RowSet rs, int q, cudaStream_t st);
void launch_final(int dim, const Layout& m, const Gas& g, const double* U, const double* U0,
                  double* Uout, Work w, StageParams sp, RowSet rs, cudaStream_t st);
void launch_pow(const double* x, double y, double* out, int64_t n, cudaStream_t st);
// the limiter's fast-accept upper bound of pow (ef_math.cuh: pow_ub), for tests
void launch_pow_ub(const double* x, double y, double* out, int64_t n, cudaStream_t st);
// halo exchange helpers: buf[r * stride + coff + k] <-> field[k * NP + idx[r]]
void launch_pack_rows(const double* field, int ncomp, int64_t NP, const int32_t* idx, int64_t count,
                      double* buf, int stride, int coff, cudaStream_t st);
void launch_unpack_rows(double* field, int ncomp, int64_t NP, const int32_t* idx, int64_t count,
                        const double* buf, int stride, int coff, cudaStream_t st);
void launch_group_min(unsigned long long* const* bits_dev, int n, cudaStream_t st);
// function-level checks: d_ij and the limiter on independent AoS batches
void launch_eval_arith(int64_t n, const double* a, const double* b, unsigned long long* mism, cudaStream_t st);
void launch_eval_dij(int dim, const Gas& g, int64_t n, const double* Ui, const double* Uj, const double* cij,
                     const double* cji, double* out, int* bad, cudaStream_t st);
void launch_eval_limiter(int dim, const Gas& g, int64_t n, const double* U, const double* P,
                         const double* bounds, int newton, double* out, cudaStream_t st);

}  // namespace ef
