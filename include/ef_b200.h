/*
 * ef_b200.h — C-ABI of the B200 per-stage IDP Euler update (drop-in boundary).
 *
 * The reference has no FFI: its boundary is the Python class
 *   eulerflow.stepper.Solver   /root/reference/pkg/src/eulerflow/stepper.py:87-649
 * plus the pow plug-in point  physics.set_power_function  (physics.py:59-75).
 * Each entry point below replaces one member of that surface; the ctypes
 * binding that a maintainer of the reference would add is shown in
 * INTEGRATION.md and implemented in paper_2007_00094_b200/stepper.py.
 *
 * Conventions: plain pointers and sizes, host memory only in the signatures,
 * no torch types.  Every call returns an EF_* status; on failure
 * ef_last_error() describes it (thread-local).  One handle = one GPU = one
 * rank; a handle is driven by one host thread.  Inputs are copied at create;
 * the library never retains host pointers.
 */
#ifndef EF_B200_H
#define EF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (the Python layer maps them to the reference's exceptions) */
#define EF_OK 0
#define EF_ERR_ARG 1            /* ValueError (stepper.py:104-107, :322-323)           */
#define EF_ERR_INADMISSIBLE 2   /* AdmissibilityError (stepper.py:324-325, :612-621;   */
                                /*   riemann.py:66-67; physics.py:128-130, :141-142)  */
#define EF_ERR_TAU_UNBOUNDED 3  /* ValueError("constant field ...") stepper.py:546-547 */
#define EF_ERR_CUDA 4           /* RuntimeError                                        */
#define EF_ERR_NCCL 5           /* RuntimeError                                        */

typedef struct ef_solver ef_solver;

/* PrecomputedMatrices, assembly.py:22-50 (beta is not read by the time step,
 * indicator.py:49-51, so it is not part of the ABI). CSR in original node ids,
 * columns sorted ascending per row. */
typedef struct {
  int64_t n;
  int32_t dim;               /* 2 or 3 */
  const int64_t* indptr;     /* (n + 1) */
  const int64_t* indices;    /* (nnz)   */
  const double* m;           /* (nnz)      consistent mass m_ij  */
  const double* c;           /* (nnz, dim) c_ij                 */
  const double* m_lumped;    /* (n)  */
  const double* inv_m;       /* (n)  */
} ef_matrices;

/* Solver(...) keyword arguments (stepper.py:90-103) + GasConstants (physics.py:33-52) */
typedef struct {
  double gamma, gm1, gp1_inv, gm1_over_2g, two_g_over_gm1; /* as computed by GasConstants */
  double c_cfl;              /* (0, 1]                       */
  int32_t limiter_passes;    /* >= 0                         */
  int32_t newton_steps;      /* >= 0                         */
  int32_t overlap;           /* Solver(overlap=...), stepper.py:97: with several
                                ranks, compute the exported rows first and move
                                their halo while the interior rows are computed
                                (exchange.py:168-222); results are identical   */
} ef_params;

/* BoundaryConditions, stepper.py:40-52 (original node ids) */
typedef struct {
  int64_t n_inflow;
  const int64_t* inflow;     /* (n_inflow) */
  const double* farfield;    /* (dim + 2)  */
  int64_t n_slip;
  const int64_t* slip;       /* (n_slip)   */
  const double* slip_normals;/* (n_slip, dim) unit outward normals */
} ef_boundary;

/* Partition (exchange.partition, exchange.py:52-104) and device binding. */
typedef struct {
  int32_t rank, nranks;      /* contiguous ranges of the global CM order      */
  int32_t device;            /* CUDA device ordinal                           */
  const int64_t* cm_perm;    /* (n) original id -> global Cuthill-McKee id    */
  const int64_t* ranges;     /* (nranks + 1) CM-id range bounds, or NULL (even split as exchange.py:64-70) */
  const void* nccl_id;       /* 128-byte ncclUniqueId shared by all ranks (nranks > 1), else NULL */
  void* stream;              /* cudaStream_t to launch on, or NULL for a library-owned stream */
} ef_dist;

/* Solver.__init__ (stepper.py:90-139) */
int ef_create(const ef_matrices* mat, const ef_params* prm, const ef_boundary* bc,
              const ef_dist* dist, ef_solver** out);
int ef_destroy(ef_solver* h);

/* Solver.set_state / get_state (stepper.py:319-336): U is (n, dim+2) float64,
 * original node order.  set_state rejects inadmissible input (state unchanged);
 * get_state fills the rows this rank owns. */
int ef_set_state(ef_solver* h, const double* U);
int ef_get_state(ef_solver* h, double* U);

/* Solver.euler_step / ssp_rk3_step (stepper.py:508-610, :624-636).  has_tau=0:
 * CFL step capped by tau_max; has_tau=1: the given tau.  *tau_used = step used
 * (Solver.tau_last).  On error the state is left at its value before the call. */
int ef_euler_step(ef_solver* h, int32_t has_tau, double tau, double tau_max, double* tau_used);
int ef_ssp_rk3_step(ef_solver* h, int32_t has_tau, double tau, double tau_max, double* tau_used);

/* Same steps, asynchronous: no host synchronisation, tau stays on the device,
 * errors are latched and reported by the next ef_sync().  For benchmarks and
 * CUDA-graph capture. */
int ef_ssp_rk3_step_async(ef_solver* h, int32_t has_tau, double tau, double tau_max);
int ef_sync(ef_solver* h, double* tau_used);

/* original id of the inadmissible node behind the last EF_ERR_INADMISSIBLE */
int64_t ef_bad_node(const ef_solver* h);
const char* ef_last_error(void);
/* Number of kernels this process has launched through the library (all handles;
 * a CUDA-graph replay counts the kernels it contains).  bench.py's gpu_launches. */
int64_t ef_kernel_launches(void);

/* Solver.timers (stepper.py:37, 515-607): seconds per phase step0..step6,
 * accumulated while timing is enabled (adds a sync per phase). */
int ef_enable_timers(ef_solver* h, int32_t on);
/* CUDA-graph replay of whole steps (single rank; on by default unless the
 * environment sets EF_GRAPHS=0).  Results are identical either way. */
int ef_enable_graphs(ef_solver* h, int32_t on);
/* Identical-state shortcuts (exact closed forms where U_i == U_j, uniform
 * stencils, P = 0): -1 = automatic (default; on while the last synchronised step
 * saw >= 20% of them, environment EF_UNIFORM=0/1 overrides), 0 = off, 1 = on.
 * Results are identical in every mode. */
int ef_set_uniform(ef_solver* h, int32_t mode);
int ef_phase_times(ef_solver* h, double* seconds7);
/* Solver.n_euler_steps, comm.sync_count, comm.sync_volume (doubles) */
int ef_counters(ef_solver* h, int64_t* out3);

/* Layout facts: out[0]=n_owned, [1]=n_local, [2]=pad width L, [3]=nnz owned,
 * [4]=standard card (most frequent), [5]=dim */
int ef_info(ef_solver* h, int64_t* out6);

/* Per-phase parity hook (the reference exposes these as solver.ranks[r].*,
 * stepper.py:73-84), the last stage's arrays: which = 0 d (n_local*L),
 * 1 alpha (n_local), 2 R (n_local*nvar), 3 bounds (n_local*3), 4 min(l_ij,
 * l_ji) of the last limiter pass (n_local*L; written on the edges that pass
 * limits: those whose previous factor was below 1), 5 eor, 6 phi,
 * 7 U (n_local*nvar), 8 U_next, 9 min(l) of the pass before the last (-1 tags
 * a slot whose P is zero from then on), 10 P as stored by the first limiter
 * pass (n_local*L*nvar; the reference's rk.P is P_0 (1 - min l_0) ... for
 * two or more passes: Solver.fetch("P") forms it).  which_pass is reserved.
 * Rows in local order (owned rows = global CM ids rank_start.., then ghosts
 * ascending), slots in stencil order. */
int ef_debug_fetch(ef_solver* h, int32_t which, int32_t which_pass, double* out);
/* local row -> global CM id, (n_local) */
int ef_local_gids(ef_solver* h, int64_t* out);

/* The shared deterministic pow (csrc/ef_pow.h): host build, to be installed
 * into the reference through physics.set_power_function, and the same code
 * evaluated on the device (test hook). */
/* Function-level checks through the device code of the stage (diagnostics,
 * like ef_debug_fetch): riemann.d_ij_low (riemann.py:119-142) for n pairs
 * (Ui, Uj: (n, dim+2) AoS; cij, cji: (n, dim); out: d_ij; bad: projection
 * error flags) and limiter.limiter_compute (limiter.py:149-193) for n lanes
 * (U, P: (n, dim+2); bounds: (n, 3) rho_min, rho_max, phi_min; newton_steps
 * from prm).  Gas constants from prm; run on the current device. */
int ef_eval_dij(const ef_params* prm, int32_t dim, int64_t n, const double* Ui, const double* Uj,
                const double* cij, const double* cji, double* out, int32_t* bad);
int ef_eval_limiter(const ef_params* prm, int32_t dim, int64_t n, const double* U, const double* P,
                    const double* bounds, double* out);
/* The straight-line division / reciprocal / square root of the d_ij kernel
 * (csrc/ef_math.cuh: rcp_sl, div_sl, sqrt_sl, qdiv_sl) against the IEEE
 * operations they restate (the reference's numpy /, sqrt: riemann.py:56-109):
 * mismatches[0..3] = operands (a[q], b[q]) inside the safe exponent range with
 * 1/b, a/b, sqrt|a| or the shared-reciprocal a/b differing in any bit. */
int ef_eval_arith(int64_t n, const double* a, const double* b, uint64_t* mismatches);

void ef_pow_host(const double* x, double y, double* out, int64_t n);
int ef_pow_device(const double* x, double y, double* out, int64_t n);
/* The limiter's fast-accept upper bound of pow(x, y) (+inf outside its range),
 * evaluated on the device: for tests of the bound. */
int ef_pow_bound_device(const double* x, double y, double* out, int64_t n);

/* Device pointer of the current state, (nvar, stride) structure-of-arrays in
 * local row order (benchmarks / zero-copy consumers). */
int ef_state_device_ptr(ef_solver* h, void** dev_ptr, int64_t* stride);

/* ---- multi-rank (exchange.partition / Communicator, exchange.py:52-222) ----
 * One process per GPU: rank 0 calls ef_nccl_unique_id, broadcasts the 128
 * bytes, every rank passes them in ef_dist.nccl_id to ef_create; halo syncs are
 * NCCL send/recv, the CFL bound an NCCL allreduce(min).  Ranks created with
 * nranks > 1 and nccl_id == NULL instead form a same-device group stepped in
 * lockstep (exchanges by device copies) — the reference's simulated ranks. */
int ef_nccl_unique_id(void* out128);
typedef struct ef_group ef_group;
int ef_group_create(ef_solver** ranks, int32_t nranks, ef_group** out);
int ef_group_destroy(ef_group* g);
int ef_group_set_state(ef_group* g, const double* U);
int ef_group_get_state(ef_group* g, double* U);
int ef_group_euler_step(ef_group* g, int32_t has_tau, double tau, double tau_max, double* tau_used);
int ef_group_ssp_rk3_step(ef_group* g, int32_t has_tau, double tau, double tau_max, double* tau_used);

/* ---- per-rank setup: no rank holds the global matrix ----
 * A rank passes only its rows, in a GLOBAL node order chosen by the caller
 * (its "CM order": the Cuthill-McKee order of exchange.partition,
 * exchange.py:58-62, or any bandwidth-limited order such as the lexicographic
 * order of a structured box).  Rank r owns the contiguous global ids
 * [ranges[r], ranges[r+1]) (exchange.py:64-70) with their full stencils, then
 * its ghost layer = the off-range columns of its owned rows (exchange.py:78-81),
 * each ghost row carrying its stencil truncated to local columns
 * (stepper.py:175-181).  Columns are global ids, ascending per row; values are
 * those of PrecomputedMatrices (assembly.py:22-50) for the same entries. */
typedef struct {
  int64_t n_global;          /* nodes of the whole mesh                        */
  int32_t dim;               /* 2 or 3                                         */
  int32_t pad_width;         /* global max stencil cardinality (stepper.py:128-131) */
  int32_t standard_card;     /* global most frequent cardinality               */
  int64_t n_owned;           /* = ranges[rank + 1] - ranges[rank]              */
  int64_t n_ghost;
  const int64_t* ghost_gid;  /* (n_ghost) ascending global ids                 */
  const int64_t* rowptr;     /* (n_owned + n_ghost + 1): owned rows, then ghosts */
  const int64_t* col_gid;    /* (nnz_local) global column ids                  */
  const double* m;           /* (nnz_local) m_ij  (NULL: plan only)            */
  const double* c;           /* (nnz_local, dim) c_ij                          */
  const double* m_lumped;    /* (n_owned + n_ghost)                            */
  const double* inv_m;       /* (n_owned + n_ghost)                            */
  const int32_t* full_card;  /* (n_owned + n_ghost) row cardinality in the global matrix */
} ef_local_matrices;

/* Solver.__init__ for one rank from its own rows.  bc: global ids (rows this
 * rank does not own are ignored); dist: rank, nranks, device, ranges
 * (required), nccl_id (one process per GPU) or NULL (same-device group),
 * stream; dist.cm_perm is not read. */
int ef_create_local(const ef_local_matrices* lm, const ef_params* prm, const ef_boundary* bc,
                    const ef_dist* dist, ef_solver** out);
/* set_state / get_state of a per-rank handle: U is (n_owned, dim+2), the owned
 * rows in global-id order.  set_state is collective over the ranks (ghost rows
 * come from their owners; every rank accepts or every rank rejects). */
int ef_set_state_owned(ef_solver* h, const double* U);
int ef_get_state_owned(ef_solver* h, double* U);
int ef_group_set_state_owned(ef_group* g, const double* const* U);  /* U[r]: rank r's rows */
int ef_group_get_state_owned(ef_group* g, double* const* U);

/* Host-only partition plan of one rank (no CUDA): sizes = {n_owned, n_local,
 * L, nranks}; rows: global CM ids of the rows sent to / received from a peer
 * (recv = 0 / 1) in message order.  Every exchanged quantity is per row (the
 * edge kernel recomputes ghost-side limiter factors), so there are no slot
 * messages.  Return the count (-1 on a bad peer).  ef_plan_build_local builds
 * the same plan from the rank's own rows (lm->m / lm->c may be NULL). */
typedef struct ef_plan ef_plan;
int ef_plan_build(const ef_matrices* mat, const ef_dist* dist, ef_plan** out);
int ef_plan_build_local(const ef_local_matrices* lm, const ef_dist* dist, ef_plan** out);
int ef_plan_destroy(ef_plan* p);
int ef_plan_sizes(const ef_plan* p, int64_t* out4);
int64_t ef_plan_rows(const ef_plan* p, int32_t peer, int32_t recv, int64_t* out_gids, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* EF_B200_H */
