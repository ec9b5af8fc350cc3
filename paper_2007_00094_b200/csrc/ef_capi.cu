// ef_capi.cu — host side of the C-ABI (include/ef_b200.h): SELL-32 setup from
// the partition plan (ef_plan.h), device memory, the phase-stepped stage
// driver with halo exchanges, transports (NCCL; same-device group), and error
// mapping.
//
// One stage (stepper.py:508-610) = six kernels; on more than one rank the
// reference's five ghost syncs and one tau reduction sit between them:
//   edge_visc, row_visc | alpha (+ tau min) | low_order | R | correction | l_0 |
//   limit_pass(p) | l_{p+1} ... | final | U  (+ step0 of the ghost rows)
// (stepper.py:532, 545, 561, 585, 605).
#include <dlfcn.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include <nccl.h>

#include "../../include/ef_b200.h"
#include "ef_kernels.cuh"
#include "ef_plan.h"

using ef::Gas;
using ef::Layout;
using ef::StageParams;
using ef::Work;

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define EF_CUDA(x)                                                                    \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess)                                                            \
      return fail(EF_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));      \
  } while (0)

#define EF_TRY(x)                 \
  do {                            \
    int rc_ = (x);                \
    if (rc_ != EF_OK) return rc_; \
  } while (0)

// ---------------------------------------------------------------- NCCL (dlopen)
// Bound at run time so the library also loads where NCCL is absent (CPU tests);
// an already loaded libnccl (torch's) is preferred.
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
#define EF_SYM(name) api.name = reinterpret_cast<decltype(api.name)>(dlsym(h, "nccl" #name))
  EF_SYM(GetUniqueId);
  EF_SYM(CommInitRank);
  EF_SYM(CommDestroy);
  EF_SYM(Send);
  EF_SYM(Recv);
  EF_SYM(GroupStart);
  EF_SYM(GroupEnd);
  EF_SYM(AllReduce);
  EF_SYM(GetErrorString);
#undef EF_SYM
  api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv && api.GroupStart &&
           api.GroupEnd && api.AllReduce && api.GetErrorString;
  return api;
}

#define EF_NCCL(x)                                                                             \
  do {                                                                                         \
    ncclResult_t r_ = (x);                                                                     \
    if (r_ != ncclSuccess) return fail(EF_ERR_NCCL, std::string(#x) + ": " + nccl().GetErrorString(r_)); \
  } while (0)

// ---------------------------------------------------------------- handle
struct ef_solver {
  int dim = 0, nvar = 0, L = 0, passes = 0, newton = 0, standard_card = 0;
  double c_cfl = 0.9;
  Gas gas{};
  int64_t n_global = 0, n_owned = 0, n_local = 0, NP = 0, NPL = 0, nnz_owned = 0;
  int rank = 0, nranks = 1, device = 0;
  bool use_nccl = false;   // nranks > 1: NCCL, or a same-device group (ef_group_*)
  ncclComm_t comm = nullptr;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  Layout lay{};
  Work w{};
  std::vector<void*> allocs;
  double* Ubuf[3] = {nullptr, nullptr, nullptr};
  int cur = 0;
  int pending_out = -1;  // buffer holding the result of an async step
  double* aos_dev = nullptr;
  int64_t* orig_dev = nullptr;
  std::vector<int64_t> orig_host, gid_host;
  // halo plans (per peer rank): counts and offsets in rows / slots, device index lists
  std::vector<int64_t> xs_rows, xr_rows;   // counts
  std::vector<int64_t> os_rows, or_rows;   // offsets
  int32_t *send_rows = nullptr, *recv_rows = nullptr;
  int64_t n_send_rows = 0, n_recv_rows = 0;
  bool local_io = false;  // per-rank setup: state I/O over the owned rows (ef_*_state_owned)
  double *sendbuf = nullptr, *recvbuf = nullptr;
  int64_t sync_count = 0, sync_volume = 0;  // Solver.comm counters (exchange.py:131-157)
  // communication overlap (stepper.py Alg. 4, exchange.py:168-222): rows other
  // ranks import (a prefix and a suffix of the CM range) are computed first,
  // their halo travels on `cst` while the interior rows are computed on `st`
  bool overlap = true;
  ef::RowSet rs_all, rs_B, rs_I;
  cudaStream_t cst = nullptr;
  cudaEvent_t evB = nullptr, evX = nullptr;
  // pinned readback block
  struct Readback {
    double tau;
    int err;
    int err_first;
    unsigned long long bad;
    unsigned long long n_same[ef::kSameSlots];
  }* rb = nullptr;
  // identical-state shortcuts: on while the last synchronised step saw at least
  // 20% identical-state edges (EF_UNIFORM=0/1 forces them off/on)
  bool uni_on = true;
  int uni_force = -1;
  double tau_last = 0.0;
  int64_t bad_node = -1;
  bool timing = false;
  double phase_s[7] = {0, 0, 0, 0, 0, 0, 0};
  int64_t n_euler = 0;
  // timing ring: 8 events per stage, recorded without host syncs and folded
  // into phase_s when the ring fills or the timers are read
  std::vector<std::array<cudaEvent_t, 8>> ring;
  int ring_used = 0;
  // CUDA graphs of whole steps (timers off; a group's graph lives on rank 0's
  // handle): one launch replays the ~25 kernels and memsets of an RK step.  Keyed by everything the captured
  // launches depend on; a few entries cover the rotating U buffers.
  // (tau and tau_max are read by the kernels from Work::tau_arg, written before
  // every launch, so they are not part of the key)
  struct GraphKey {
    int rk3, cur, has_tau, uni;
    bool operator==(const GraphKey& o) const {
      return rk3 == o.rk3 && cur == o.cur && has_tau == o.has_tau && uni == o.uni;
    }
  };
  struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec;
    uint64_t used;
    long long launches;  // kernels captured (added to the launch count per replay)
    std::vector<std::pair<int64_t, int64_t>> syncs;  // per rank: halo syncs, volume per replay
  };
  std::vector<GraphEntry> graphs;
  uint64_t graph_clock = 0;
  bool use_graphs = true;

  template <class T>
  int alloc(T** p, size_t count) {
    void* q = nullptr;
    size_t bytes = sizeof(T) * (count > 0 ? count : 1);
    cudaError_t e = cudaMalloc(&q, bytes);
    if (e != cudaSuccess)
      return fail(EF_ERR_CUDA, std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    allocs.push_back(q);
    *p = (T*)q;
    return EF_OK;
  }
  ~ef_solver() {
    for (void* p : allocs) cudaFree(p);
    if (rb) cudaFreeHost(rb);
    for (auto& set : ring)
      for (auto& e : set) cudaEventDestroy(e);
    for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
    if (comm && nccl().ok) nccl().CommDestroy(comm);
    if (evB) cudaEventDestroy(evB);
    if (evX) cudaEventDestroy(evX);
    if (cst) cudaStreamDestroy(cst);
    if (own_stream && st) cudaStreamDestroy(st);
  }
};

struct ef_group {
  std::vector<ef_solver*> hs;
  unsigned long long** bits_dev = nullptr;  // device array of the ranks' tau_min_bits
};

template <class T, class A>
static int upload(ef_solver* h, T** dst, const std::vector<T, A>& src) {
  EF_TRY(h->alloc(dst, src.size()));
  EF_CUDA(cudaMemcpy(*dst, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice));
  return EF_OK;
}

static Gas make_gas(const ef_params* p) {
  Gas g;
  g.gamma = p->gamma;
  g.gm1 = p->gm1;
  g.gp1_inv = p->gp1_inv;
  g.gm1_over_2g = p->gm1_over_2g;
  g.two_g_over_gm1 = p->two_g_over_gm1;
  volatile double gamma = p->gamma;  // evaluate exactly as the reference writes it
  g.gp1 = gamma + 1.0;
  g.gp1_over_2g = (gamma + 1.0) / (2.0 * gamma);
  g.half_gm1 = 0.5 * p->gm1;
  g.neg_gm1_over_2g = -p->gm1_over_2g;
  g.neg_gamma = -gamma;
  g.neg_g_gp1_inv = (-gamma) * p->gp1_inv;
  g.sqrt2 = std::sqrt(2.0);
  const char* fa = std::getenv("EF_FAST_ACCEPT");  // results are identical either way
  g.fast_accept = (fa && fa[0] == '0') ? 0 : 1;
  const char* sl = std::getenv("EF_SL");  // straight-line d_ij path (ef_math.cuh); results are identical either way
  g.sl = (sl && sl[0] == '0') ? 0 : 1;
  g.kind_a = ef_pow_kind(g.neg_gm1_over_2g);
  g.kind_b = ef_pow_kind(g.two_g_over_gm1);
  g.kind_gp1 = ef_pow_kind(g.gp1);
  g.kind_gamma = ef_pow_kind(g.gamma);
  return g;
}

// ---------------------------------------------------------------- setup
// Values behind a plan's local rows: entry values indexed by Plan::src(k), and
// per local row the lumped mass, the full-stencil cardinality and the caller's
// node id (state I/O and boundary lists).
struct Src {
  const double* m = nullptr;
  const double* c = nullptr;
  std::vector<double> m_lumped, inv_m;
  std::vector<uint8_t> cardf;
  std::vector<int64_t> orig;
  const int64_t* cm_perm = nullptr;  // caller id -> global id (boundary lists); null: identity
  bool local_io = false;             // state I/O over the owned rows (per-rank setup)
};

static int build_from_plan(ef_solver* h, ef::Plan& P, Src& S, const ef_boundary* bc);

static int build(ef_solver* h, const ef_matrices* mat, const ef_boundary* bc, const ef_dist* dist) {
  const int64_t n = mat->n;
  if (!dist || !dist->cm_perm) return fail(EF_ERR_ARG, "ef_dist.cm_perm is required");
  ef::Plan P;
  if (!ef::build_plan(n, mat->indptr, mat->indices, dist->cm_perm, h->rank, h->nranks, dist->ranges, P))
    return fail(EF_ERR_ARG, P.error);
  Src S;
  S.m = mat->m;
  S.c = mat->c;
  S.cm_perm = dist->cm_perm;
  const int64_t n_local = P.n_local;
  S.orig.resize(n_local);
  S.m_lumped.resize(n_local);
  S.inv_m.resize(n_local);
  S.cardf.resize(n_local);
  ef::parallel_for(n_local, [&](int64_t a, int64_t b, int) {
    for (int64_t i = a; i < b; ++i) {
      const int64_t o = P.cm_inv[P.gid[i]];
      S.orig[i] = o;
      S.m_lumped[i] = mat->m_lumped[o];
      S.inv_m[i] = mat->inv_m[o];
      S.cardf[i] = (uint8_t)(mat->indptr[o + 1] - mat->indptr[o]);
    }
  });
  return build_from_plan(h, P, S, bc);
}

// per-rank setup: the rank's rows only (ef_create_local)
static int build_local(ef_solver* h, const ef_local_matrices* lm, const ef_boundary* bc, const ef_dist* dist) {
  ef::Plan P;
  if (!ef::build_plan_local(lm->n_global, lm->n_owned, lm->n_ghost, lm->ghost_gid, lm->rowptr, lm->col_gid,
                            lm->pad_width, lm->standard_card, h->rank, h->nranks, dist ? dist->ranges : nullptr, P))
    return fail(EF_ERR_ARG, P.error);
  if (!lm->m || !lm->c || !lm->m_lumped || !lm->inv_m || !lm->full_card)
    return fail(EF_ERR_ARG, "ef_local_matrices values are required");
  Src S;
  S.m = lm->m;
  S.c = lm->c;
  S.local_io = true;
  const int64_t n_local = P.n_local;
  S.orig.assign(P.gid.begin(), P.gid.end());
  S.m_lumped.assign(lm->m_lumped, lm->m_lumped + n_local);
  S.inv_m.assign(lm->inv_m, lm->inv_m + n_local);
  S.cardf.resize(n_local);
  for (int64_t i = 0; i < n_local; ++i) {
    if (lm->full_card[i] < 1 || lm->full_card[i] > P.L) return fail(EF_ERR_ARG, "full_card out of range");
    S.cardf[i] = (uint8_t)lm->full_card[i];
  }
  return build_from_plan(h, P, S, bc);
}

static int build_from_plan(ef_solver* h, ef::Plan& P, Src& S, const ef_boundary* bc) {
  const int D = h->dim, NV = h->nvar;
  const int64_t n = P.n;
  const int L = P.L;
  const int64_t n_owned = P.n_owned, n_local = P.n_local;
  h->L = L;
  h->standard_card = P.standard_card;
  h->n_global = n;
  h->n_owned = n_owned;
  h->n_local = n_local;
  h->NP = std::max<int64_t>((n_local + 31) / 32 * 32, 32);
  h->NPL = h->NP * L;
  const int64_t NP = h->NP, NPL = h->NPL;
  if (NPL >= (int64_t)1 << 31 || (int64_t)NV * NP >= (int64_t)1 << 31)
    return fail(EF_ERR_ARG, "local rows/slots exceed 32-bit indexing (use more ranks)");
  h->gid_host = P.gid;
  h->orig_host = std::move(S.orig);
  h->local_io = S.local_io;
  auto local_of = [&](int64_t g) -> int64_t {
    if (g >= P.s_lo && g < P.s_hi) return g - P.s_lo;
    auto it = std::lower_bound(P.gid.begin() + n_owned, P.gid.end(), g);
    if (it != P.gid.end() && *it == g) return it - P.gid.begin();
    return -1;
  };

  // SELL-32 host images, filled row by row on all host threads (every slot of
  // every row, pads included, is written exactly once)
  ef::hvec<int32_t> col(NPL);
  ef::hvec<uint8_t> tslot(NPL);
  ef::hvec<double> c((size_t)D * NPL), mij(NPL);
  std::vector<uint8_t> card(NP, 1), cardf(NP, 1), diag(NP, 0);
  std::vector<double> m_i(NP, 1.0), inv_m(NP, 1.0), lam(NP, 1.0);
  std::vector<int64_t> gid(NP, 0);
  std::atomic<int64_t> nnz_acc{0};
  std::atomic<int> bad{0};  // 1: not structurally symmetric, 2: missing diagonal
  ef::parallel_for(NP, [&](int64_t a, int64_t b, int) {
    int64_t nnz_part = 0;
    for (int64_t i = a; i < b; ++i) {
      const int64_t cnt = i < n_local ? P.rptr[i + 1] - P.rptr[i] : 0;
      for (int64_t s = cnt; s < L; ++s) {  // pads (and padding rows): self column, zero values
        const int64_t p = ef::sidx(i, (int)s, L);
        col[p] = (int32_t)std::min<int64_t>(i, n_local - 1);
        tslot[p] = 0;
        mij[p] = 0.0;
        for (int d = 0; d < D; ++d) c[(size_t)d * NPL + p] = 0.0;
      }
      if (i >= n_local) continue;
      card[i] = (uint8_t)cnt;
      if (i < n_owned) nnz_part += cnt;
      int dg = -1;
      for (int64_t s = 0; s < cnt; ++s) {
        const int64_t cg = P.cols[P.rptr[i] + s];
        const int64_t j = local_of(cg);
        const int64_t q = P.src(P.rptr[i] + s);
        const int64_t p = ef::sidx(i, (int)s, L);
        col[p] = (int32_t)j;
        if (j == i) dg = (int)s;
        mij[p] = S.m[q];
        for (int d = 0; d < D; ++d) c[(size_t)d * NPL + p] = S.c[q * D + d];
        // transpose slot: position of this row's CM id in row j (both rows local)
        if (j < 0) {
          bad.store(1);
          continue;
        }
        const int64_t* rb = P.cols + P.rptr[j];
        const int64_t* re = P.cols + P.rptr[j + 1];
        const int64_t* it = std::lower_bound(rb, re, P.gid[i]);
        if (it == re || *it != P.gid[i]) {
          bad.store(1);
          tslot[p] = 0;
        } else {
          tslot[p] = (uint8_t)(it - rb);
        }
      }
      if (dg < 0) {
        bad.store(2);
        dg = 0;
      }
      diag[i] = (uint8_t)dg;
      cardf[i] = S.cardf[i];
      m_i[i] = S.m_lumped[i];
      inv_m[i] = S.inv_m[i];
      const int64_t den = std::max<int64_t>(cnt - 1, 1);
      lam[i] = 1.0 / (double)den;  // stepper.py:214-215
      gid[i] = P.gid[i];
    }
    nnz_acc += nnz_part;
  }, 1024);
  if (bad.load() == 1) return fail(EF_ERR_ARG, "stencil pattern is not structurally symmetric");
  if (bad.load() == 2) return fail(EF_ERR_ARG, "every stencil must contain its own row");
  h->nnz_owned = nnz_acc.load();
  // upper-triangle edges with at least one owned endpoint (a ghost row's upper
  // edge to an owned row is that row's lower entry), in ascending SELL position
  std::vector<std::vector<int32_t>> epart(ef::par_threads());
  const int nch = ef::parallel_for(NP / 32, [&](int64_t a, int64_t b, int t) {
    auto& out = epart[t];
    for (int64_t sl = a; sl < b; ++sl)
      for (int s = 0; s < L; ++s)
        for (int ln = 0; ln < 32; ++ln) {
          const int64_t i = sl * 32 + ln;
          if (i >= n_local || !(s > diag[i] && s < card[i])) continue;
          if (i < n_owned || col[ef::sidx(i, s, L)] < n_owned) out.push_back((int32_t)ef::sidx(i, s, L));
        }
  }, 256);
  std::vector<int32_t> edges;
  for (int t = 0; t < nch; ++t) edges.insert(edges.end(), epart[t].begin(), epart[t].end());
  epart.clear();
  const int64_t NE = (int64_t)edges.size();
  // endpoint tables: the edge kernels read j and the transposed position with
  // the edge position (one coalesced load each) instead of through col/tslot
  std::vector<int32_t> edge_j(std::max<int64_t>(NE, 1), 0), edge_pt(std::max<int64_t>(NE, 1), 0);
  // static edge geometry (riemann.py:131-136): n = c / |c|, |c| = sqrt(R1(c*c)),
  // for c_ij and c_ji, evaluated with the reference's operation order; one record of
  // 2 (D + 1) doubles per edge (the edge kernel reads it as 16-byte pairs)
  ef::hvec<double> egeo((size_t)2 * (D + 1) * std::max<int64_t>(NE, 1));
  if (NE == 0)
    for (auto& v : egeo) v = 0.0;
  ef::parallel_for(NE, [&](int64_t a, int64_t b, int) {
    for (int64_t e = a; e < b; ++e) {
      const int64_t p = edges[e];
      const int64_t pt = ef::sidx(col[p], tslot[p], L);
      edge_j[e] = col[p];
      edge_pt[e] = (int32_t)pt;
      for (int dir = 0; dir < 2; ++dir) {
        const int64_t q = dir ? pt : p;
        volatile double ss = 0.0;  // ((0 + c0^2) + c1^2) + c2^2, no contraction
        for (int d = 0; d < D; ++d) {
          volatile double sq = c[(size_t)d * NPL + q] * c[(size_t)d * NPL + q];
          ss = ss + sq;
        }
        const double nrm = std::sqrt((double)ss);
        const int base = dir * (D + 1);
        for (int d = 0; d < D; ++d)
          egeo[(size_t)e * (2 * (D + 1)) + base + d] = nrm > 0.0 ? c[(size_t)d * NPL + q] / nrm : (d == 0 ? 1.0 : 0.0);
        egeo[(size_t)e * (2 * (D + 1)) + base + D] = nrm;
      }
    }
  });
  // EF_CHECKS=1: every real slot (row < n_local, s != diag, s < card) is written
  // by exactly one edge thread -- at p (upper) or pt (lower) -- so the edge
  // kernels' plain stores of d, P and min(l) never collide
  if (const char* ck = std::getenv("EF_CHECKS"); ck && ck[0] == '1') {
    std::vector<uint8_t> hits(NPL, 0);
    for (int64_t e = 0; e < NE; ++e) {
      hits[edges[e]]++;
      hits[edge_pt[e]]++;
    }
    for (int64_t i = 0; i < n_local; ++i)
      for (int s = 0; s < card[i]; ++s) {
        const int64_t p = ef::sidx(i, s, L);
        const bool owned_edge = i < n_owned || col[p] < n_owned;  // edges with an owned end
        const int want = (s == diag[i] || !owned_edge) ? 0 : 1;
        if (hits[p] != want)
          return fail(EF_ERR_ARG, "EF_CHECKS: slot (" + std::to_string(i) + ", " + std::to_string(s) +
                                      ") is written by " + std::to_string(hits[p]) + " edges");
      }
  }
  // boundary data (stepper.py:258-267): owned rows only
  std::vector<int8_t> bc_kind(NP, 0);
  std::vector<double> bc_n((size_t)D * NP, 0.0);
  double farfield[5] = {0, 0, 0, 0, 0};
  if (bc) {
    for (int64_t q = 0; q < bc->n_slip; ++q) {
      const int64_t o = bc->slip[q];
      if (o < 0 || o >= n) return fail(EF_ERR_ARG, "slip node id out of range");
      const int64_t g = S.cm_perm ? S.cm_perm[o] : o;
      if (g < P.s_lo || g >= P.s_hi) continue;
      const int64_t i = g - P.s_lo;
      bc_kind[i] |= 1;
      for (int a = 0; a < D; ++a) bc_n[(size_t)a * NP + i] = bc->slip_normals[q * D + a];
    }
    for (int64_t q = 0; q < bc->n_inflow; ++q) {
      const int64_t o = bc->inflow[q];
      if (o < 0 || o >= n) return fail(EF_ERR_ARG, "inflow node id out of range");
      const int64_t g = S.cm_perm ? S.cm_perm[o] : o;
      if (g < P.s_lo || g >= P.s_hi) continue;
      bc_kind[g - P.s_lo] |= 2;
    }
    if (bc->n_inflow > 0) {
      if (!bc->farfield) return fail(EF_ERR_ARG, "inflow nodes need a farfield state");
      for (int k = 0; k < NV; ++k) farfield[k] = bc->farfield[k];
    }
  }
  // halo plans -> flat device index lists (peer-major)
  const int R = h->nranks;
  h->xs_rows.assign(R, 0);
  h->xr_rows.assign(R, 0);
  h->os_rows.assign(R + 1, 0);
  h->or_rows.assign(R + 1, 0);
  std::vector<int32_t> srows, rrows;
  for (int q = 0; q < R; ++q) {
    for (int64_t i : P.send_rows[q]) srows.push_back((int32_t)i);
    for (int64_t i : P.recv_rows[q]) rrows.push_back((int32_t)i);
    h->xs_rows[q] = (int64_t)P.send_rows[q].size();
    h->xr_rows[q] = (int64_t)P.recv_rows[q].size();
    h->os_rows[q + 1] = h->os_rows[q] + h->xs_rows[q];
    h->or_rows[q + 1] = h->or_rows[q] + h->xr_rows[q];
  }
  h->n_send_rows = (int64_t)srows.size();
  h->n_recv_rows = (int64_t)rrows.size();
  // exported rows B = [0, a) u [b, n_owned) with the fewest rows covering every
  // send row (RCM keeps them near both ends of the range); interior = [a, b)
  h->rs_all = ef::all_rows(n_owned);
  h->rs_B = ef::all_rows(n_owned);
  h->rs_I = ef::all_rows(0);
  if (R > 1) {
    std::vector<int64_t> sr(srows.begin(), srows.end());
    std::sort(sr.begin(), sr.end());
    sr.erase(std::unique(sr.begin(), sr.end()), sr.end());
    int64_t best_a = 0, best_b = n_owned, best = -1;
    for (size_t k = 0; k <= sr.size(); ++k) {  // rows sr[0..k) low, sr[k..) high
      const int64_t a = k > 0 ? sr[k - 1] + 1 : 0;
      const int64_t b = k < sr.size() ? sr[k] : n_owned;
      if (a > b) continue;
      const int64_t cost = a + (n_owned - b);
      if (best < 0 || cost < best) {
        best = cost;
        best_a = a;
        best_b = b;
      }
    }
    if (best < 0) {  // cannot happen (k = 0 covers everything); keep all rows exported
      best_a = n_owned;
      best_b = n_owned;
    }
    ef::RowSet B;
    B.r0 = 0;
    B.n0 = (int)best_a;
    B.r2 = (int)best_b;
    B.n = (int)(best_a + (n_owned - best_b));
    B.lead = 1;
    ef::RowSet I;
    I.r0 = (int)best_a;
    I.n0 = I.n = (int)(best_b - best_a);
    I.r2 = (int)best_b;
    I.lead = 0;
    h->rs_B = B;
    h->rs_I = I;
  }

  // ---- device images
  Layout& m = h->lay;
  m.L = L;
  m.NP = NP;
  m.n_local = n_local;
  m.n_owned = n_owned;
  int32_t* d_col;
  uint8_t *d_tslot, *d_card, *d_cardf, *d_diag;
  double *d_c, *d_egeo, *d_mij, *d_mi, *d_invm, *d_lam, *d_bcn;
  int64_t* d_gid;
  int8_t* d_bck;
  int32_t *d_edges, *d_edge_j, *d_edge_pt;
  EF_TRY(upload(h, &d_col, col));
  EF_TRY(upload(h, &d_tslot, tslot));
  EF_TRY(upload(h, &d_card, card));
  EF_TRY(upload(h, &d_cardf, cardf));
  EF_TRY(upload(h, &d_diag, diag));
  EF_TRY(upload(h, &d_c, c));
  EF_TRY(upload(h, &d_egeo, egeo));
  EF_TRY(upload(h, &d_mij, mij));
  EF_TRY(upload(h, &d_mi, m_i));
  EF_TRY(upload(h, &d_invm, inv_m));
  EF_TRY(upload(h, &d_lam, lam));
  EF_TRY(upload(h, &d_gid, gid));
  EF_TRY(upload(h, &d_bck, bc_kind));
  EF_TRY(upload(h, &d_bcn, bc_n));
  EF_TRY(upload(h, &d_edges, edges));
  EF_TRY(upload(h, &d_edge_j, edge_j));
  EF_TRY(upload(h, &d_edge_pt, edge_pt));
  m.col = d_col;
  m.tslot = d_tslot;
  m.card = d_card;
  m.cardf = d_cardf;
  m.diag = d_diag;
  m.c = d_c;
  m.egeo = d_egeo;
  m.mij = d_mij;
  m.m_i = d_mi;
  m.inv_m = d_invm;
  m.lam = d_lam;
  m.gid = d_gid;
  m.bc_kind = d_bck;
  m.bc_n = d_bcn;
  m.edges = d_edges;
  m.edge_j = d_edge_j;
  m.edge_pt = d_edge_pt;
  m.n_edges = (int64_t)edges.size();
  m.slab = ef::make_fastdiv((uint32_t)(32 * L));
  for (int k = 0; k < 5; ++k) m.farfield[k] = farfield[k];
  if (R > 1) {
    EF_TRY(upload(h, &h->send_rows, srows));
    EF_TRY(upload(h, &h->recv_rows, rrows));
    // the widest message row: R, U^L and bounds after the low-order update
    const int64_t sb = h->n_send_rows * (2 * NV + 3);
    const int64_t rbn = h->n_recv_rows * (2 * NV + 3);
    EF_TRY(h->alloc(&h->sendbuf, sb));
    EF_TRY(h->alloc(&h->recvbuf, rbn));
  }

  Work& w = h->w;
  EF_TRY(h->alloc(&w.eor, NP));
  EF_TRY(h->alloc(&w.phi, NP));
  EF_TRY(h->alloc(&w.vp, (size_t)(D + 1) * NP));
  EF_CUDA(cudaMemset(w.vp, 0, sizeof(double) * (D + 1) * NP));
  EF_TRY(h->alloc(&w.alpha, NP));
  EF_TRY(h->alloc(&w.R, (size_t)NV * NP));
  EF_TRY(h->alloc(&w.Unext, (size_t)NV * NP));
  EF_TRY(h->alloc(&w.bounds, (size_t)3 * NP));
  EF_TRY(h->alloc(&w.d, NPL));
  EF_TRY(h->alloc(&w.ml, NPL));
  EF_TRY(h->alloc(&w.ml2, NPL));
  EF_TRY(h->alloc(&w.P, (size_t)NV * NPL));
  EF_TRY(h->alloc(&w.nonuni, NP));
  EF_CUDA(cudaMemset(w.nonuni, 1, NP));
  EF_TRY(h->alloc(&w.chg, NP));
  EF_CUDA(cudaMemset(w.chg, 1, NP));
  EF_TRY(h->alloc(&w.pnz, NP));
  EF_CUDA(cudaMemset(w.pnz, 1, NP));
  EF_TRY(h->alloc(&w.wl, std::max<int64_t>(h->lay.n_edges, 1)));
  EF_TRY(h->alloc(&w.wl_n, 1));
  EF_TRY(h->alloc(&w.lmask, NP));
  EF_CUDA(cudaMemset(w.lmask, 0, sizeof(unsigned long long) * NP));
  EF_CUDA(cudaMemset(w.wl_n, 0, sizeof(int)));
  EF_TRY(h->alloc(&w.ust, NP));
  EF_CUDA(cudaMemset(w.ust, 0, NP));
  EF_TRY(h->alloc(&w.tau_min_bits, 1));
  EF_TRY(h->alloc(&w.tau, 1));
  EF_TRY(h->alloc(&w.err, 1));
  EF_TRY(h->alloc(&w.err_first, 1));
  EF_TRY(h->alloc(&w.bad_gid, 1));
  EF_TRY(h->alloc(&w.tau_arg, 2));
  EF_CUDA(cudaMemset(w.tau_arg, 0, 2 * sizeof(double)));
  EF_CUDA(cudaMemset(w.err, 0, sizeof(int)));
  EF_CUDA(cudaMemset(w.err_first, 0x7f, sizeof(int)));
  EF_CUDA(cudaMemset(w.bad_gid, 0xff, sizeof(unsigned long long)));
  EF_TRY(h->alloc(&w.n_same, ef::kSameSlots));
  EF_CUDA(cudaMemset(w.n_same, 0, sizeof(unsigned long long) * ef::kSameSlots));
  EF_CUDA(cudaMemset(w.d, 0, sizeof(double) * NPL));
  EF_CUDA(cudaMemset(w.ml, 0, sizeof(double) * NPL));
  EF_CUDA(cudaMemset(w.ml2, 0, sizeof(double) * NPL));
  EF_CUDA(cudaMemset(w.P, 0, sizeof(double) * NV * NPL));
  EF_CUDA(cudaMemset(w.alpha, 0, sizeof(double) * NP));
  EF_CUDA(cudaMemset(w.R, 0, sizeof(double) * NV * NP));
  EF_CUDA(cudaMemset(w.eor, 0, sizeof(double) * NP));
  EF_CUDA(cudaMemset(w.phi, 0, sizeof(double) * NP));
  for (int k = 0; k < 3; ++k) {
    EF_TRY(h->alloc(&h->Ubuf[k], (size_t)NV * NP));
    EF_CUDA(cudaMemset(h->Ubuf[k], 0, sizeof(double) * NV * NP));
  }
  if (h->local_io) {  // owned rows only: no rank holds an n_global-sized array
    EF_TRY(h->alloc(&h->aos_dev, (size_t)n_owned * NV));
    std::vector<int64_t> iota(n_owned);
    for (int64_t i = 0; i < n_owned; ++i) iota[i] = i;
    EF_TRY(upload(h, &h->orig_dev, iota));
  } else {
    EF_TRY(h->alloc(&h->aos_dev, (size_t)n * NV));
    EF_TRY(upload(h, &h->orig_dev, h->orig_host));
  }
  EF_CUDA(cudaMallocHost((void**)&h->rb, sizeof(ef_solver::Readback)));
  return EF_OK;
}

// ---------------------------------------------------------------- driver
// A Driver steps one NCCL rank (hs.size() == 1) or every rank of a same-device
// group in lockstep (all handles on one stream, exchanges by device copies).
struct Driver {
  std::vector<ef_solver*> hs;
  bool group = false;
  unsigned long long** bits_dev = nullptr;
  ef_solver* h0() const { return hs[0]; }
  bool multi() const { return hs[0]->nranks > 1; }
};

static int flush_timers(ef_solver* h) {
  for (int q = 0; q < h->ring_used; ++q) {
    EF_CUDA(cudaEventSynchronize(h->ring[q][7]));
    for (int k = 0; k < 7; ++k) {
      float ms = 0.f;
      EF_CUDA(cudaEventElapsedTime(&ms, h->ring[q][k], h->ring[q][k + 1]));
      h->phase_s[k] += ms * 1e-3;
    }
  }
  h->ring_used = 0;
  return EF_OK;
}

static int mark(ef_solver* h, int k) {
  if (!h->timing) return EF_OK;
  if (k == 0 && h->ring_used == (int)h->ring.size()) {
    if (h->ring.size() < 256) {
      std::array<cudaEvent_t, 8> set;
      for (auto& e : set) EF_CUDA(cudaEventCreate(&e));
      h->ring.push_back(set);
    } else {
      EF_TRY(flush_timers(h));
    }
  }
  EF_CUDA(cudaEventRecord(h->ring[h->ring_used][k], h->st));
  if (k == 7) h->ring_used++;
  return EF_OK;
}

// Halo exchange of several row fields in one message per peer
// (exchange.py:145-157 semantics: owners' values overwrite the ghost copies).
// A message row holds the fields' components back to back; `fld.of(r)` is rank
// r's device array (index into Driver::hs).  Everything runs on stream `s`.
struct Fld {
  std::function<double*(size_t)> of;
  int ncomp;
};
static int exchange(Driver& d, const std::vector<Fld>& flds, cudaStream_t s) {
  if (!d.multi()) return EF_OK;
  int C = 0;
  for (const Fld& f : flds) C += f.ncomp;
  for (size_t r = 0; r < d.hs.size(); ++r) {
    ef_solver* h = d.hs[r];
    int off = 0;
    for (const Fld& f : flds) {
      ef::launch_pack_rows(f.of(r), f.ncomp, h->NP, h->send_rows, h->n_send_rows, h->sendbuf, C, off, s);
      off += f.ncomp;
    }
  }
  if (d.group) {
    for (ef_solver* h : d.hs)
      for (int q = 0; q < h->nranks; ++q) {
        const int64_t cnt = h->xr_rows[q] * C;
        if (cnt == 0) continue;
        ef_solver* src = d.hs[q];
        EF_CUDA(cudaMemcpyAsync(h->recvbuf + h->or_rows[q] * C, src->sendbuf + src->os_rows[h->rank] * C,
                                sizeof(double) * cnt, cudaMemcpyDeviceToDevice, s));
      }
  } else {
    ef_solver* h = d.h0();
    EF_NCCL(nccl().GroupStart());
    for (int q = 0; q < h->nranks; ++q) {
      const int64_t sc = h->xs_rows[q] * C, rc = h->xr_rows[q] * C;
      if (sc) EF_NCCL(nccl().Send(h->sendbuf + h->os_rows[q] * C, (size_t)sc, ncclFloat64, q, h->comm, s));
      if (rc) EF_NCCL(nccl().Recv(h->recvbuf + h->or_rows[q] * C, (size_t)rc, ncclFloat64, q, h->comm, s));
    }
    EF_NCCL(nccl().GroupEnd());
  }
  for (size_t r = 0; r < d.hs.size(); ++r) {
    ef_solver* h = d.hs[r];
    int off = 0;
    for (const Fld& f : flds) {
      ef::launch_unpack_rows(f.of(r), f.ncomp, h->NP, h->recv_rows, h->n_recv_rows, h->recvbuf, C, off, s);
      off += f.ncomp;
    }
    h->sync_count++;
    h->sync_volume += h->n_recv_rows * C;
  }
  return EF_OK;
}

// allreduce_min of the CFL bound (exchange.py:160-165): bit patterns of
// positive doubles order like their values, so a uint64 min is exact.
static int allreduce_tau(Driver& d, cudaStream_t s) {
  if (!d.multi()) return EF_OK;
  if (d.group) {
    ef::launch_group_min(d.bits_dev, (int)d.hs.size(), s);
    EF_CUDA(cudaGetLastError());
    return EF_OK;
  }
  ef_solver* h = d.h0();
  EF_NCCL(nccl().AllReduce(h->w.tau_min_bits, h->w.tau_min_bits, 1, ncclUint64, ncclMin, h->comm, s));
  return EF_OK;
}

struct StageIO {
  const double* U;
  const double* U0;
  double* Uout;
};

static int run_stage(Driver& d, const std::vector<StageIO>& io, StageParams sp) {
  const bool want_tau = sp.tau_mode == ef::TAU_CFL;
  auto each = [&](auto fn) {
    for (size_t r = 0; r < d.hs.size(); ++r) fn(d.hs[r], io[r]);
  };
  ef_solver* t = d.h0();  // timers, comm stream and events are kept on the first handle
  const bool multi = d.multi();
  const bool ov = multi && t->overlap;
  cudaStream_t st = t->st;  // the ranks of a same-device group share it
  const int NV = t->nvar;
  // Run a row kernel launch(h, x, rows) over the owned rows, then the halo
  // exchange of `flds`.  With overlap: exported rows first, their halo on the
  // comm stream while the interior rows run, joined before the next phase.
  auto produce = [&](auto launch, const std::vector<Fld>& flds) -> int {
    if (!multi || flds.empty()) {
      each([&](ef_solver* h, const StageIO& x) { launch(h, x, h->rs_all); });
      return EF_OK;
    }
    if (!ov) {
      each([&](ef_solver* h, const StageIO& x) { launch(h, x, h->rs_all); });
      return exchange(d, flds, st);
    }
    each([&](ef_solver* h, const StageIO& x) { launch(h, x, h->rs_B); });
    EF_CUDA(cudaEventRecord(t->evB, st));
    EF_CUDA(cudaStreamWaitEvent(t->cst, t->evB, 0));
    EF_TRY(exchange(d, flds, t->cst));
    EF_CUDA(cudaEventRecord(t->evX, t->cst));
    each([&](ef_solver* h, const StageIO& x) { launch(h, x, h->rs_I); });
    EF_CUDA(cudaStreamWaitEvent(st, t->evX, 0));
    return EF_OK;
  };
  auto fld = [&](double* Work::*member, int ncomp) {
    return Fld{[&d, member](size_t r) { return d.hs[r]->w.*member; }, ncomp};
  };
  EF_TRY(mark(t, 0));
  EF_TRY(mark(t, 1));  // step0 is fused into the previous stage's final kernel
  each([&](ef_solver* h, const StageIO& x) { ef::launch_edge_visc(h->dim, h->lay, h->gas, x.U, h->w, sp.stage, want_tau, sp.uni != 0,
                                                                   sp.tau_mode != ef::TAU_DEVICE, st); });
  EF_TRY(mark(t, 2));
  EF_TRY(produce([&](ef_solver* h, const StageIO& x, ef::RowSet rs) {
    ef::launch_row_visc(h->dim, h->lay, h->gas, x.U, h->w, sp.stage, want_tau, sp.uni != 0, rs, st);
  }, {fld(&Work::alpha, 1)}));
  if (want_tau) EF_TRY(allreduce_tau(d, st));
  EF_TRY(mark(t, 3));
  // ghost rows need R for P, U^L and bounds for their own limiter side
  std::vector<Fld> lo_flds;
  if (t->passes > 0) lo_flds = {fld(&Work::R, NV), fld(&Work::Unext, NV), fld(&Work::bounds, 3)};
  EF_TRY(produce([&](ef_solver* h, const StageIO& x, ef::RowSet rs) {
    ef::launch_low_order(h->dim, h->lay, h->gas, x.U, h->w, sp, rs, st);
  }, lo_flds));
  EF_TRY(mark(t, 4));
  // the pass before the last fills the last pass's worklist
  auto clear_wl = [&](int q) -> int {
    if (ef::edge_lim_worklist() && q == t->passes - 2)
      for (ef_solver* h : d.hs) EF_CUDA(cudaMemsetAsync(h->w.wl_n, 0, sizeof(int), st));
    return EF_OK;
  };
  if (t->passes > 0) {
    EF_TRY(clear_wl(0));
    each([&](ef_solver* h, const StageIO& x) { ef::launch_edge_lim(h->dim, h->lay, h->gas, x.U, h->w, sp, 0, st); });
    EF_TRY(mark(t, 5));
    for (int p = 0; p + 1 < t->passes; ++p) {
      EF_TRY(produce([&](ef_solver* h, const StageIO& x, ef::RowSet rs) {
        ef::launch_row_upd(h->dim, h->lay, h->gas, x.U, h->w, sp, rs, p, st);
      }, {fld(&Work::Unext, NV)}));
      EF_TRY(clear_wl(p + 1));
      each([&](ef_solver* h, const StageIO& x) { ef::launch_edge_lim(h->dim, h->lay, h->gas, x.U, h->w, sp, p + 1, st); });
    }
    EF_TRY(mark(t, 6));
  } else {
    EF_TRY(mark(t, 5));
    EF_TRY(mark(t, 6));
  }
  EF_TRY(produce([&](ef_solver* h, const StageIO& x, ef::RowSet rs) {
    ef::launch_final(h->dim, h->lay, h->gas, x.U, x.U0, x.Uout, h->w, sp, rs, st);
  }, {Fld{[&io](size_t r) { return io[r].Uout; }, NV}}));
  if (multi) {
    each([&](ef_solver* h, const StageIO& x) {  // step0 of the ghost rows
      ef::launch_nodal(h->dim, h->lay, h->gas, x.Uout, h->w, h->n_owned, h->n_local, st);
    });
  }
  EF_TRY(mark(t, 7));
  for (ef_solver* h : d.hs) {
    EF_CUDA(cudaGetLastError());
    h->n_euler++;
  }
  return EF_OK;
}

static StageParams stage_params(ef_solver* h, int mode, int stage, double rk_a) {
  StageParams sp;
  sp.tau_mode = mode;
  sp.stage = stage;
  sp.c_cfl = h->c_cfl;
  sp.newton = h->newton;
  sp.passes = h->passes;
  sp.rk_a = rk_a;
  sp.uni = h->uni_on ? 1 : 0;
  return sp;
}

// Per step: the identical-state sample counters.  The error flags are NOT reset
// here: they latch across a chain of async steps and are cleared only after
// they have been read (finish) or by set_state (clear_err).
static int reset_counters(Driver& d) {
  for (ef_solver* h : d.hs)
    EF_CUDA(cudaMemsetAsync(h->w.n_same, 0, sizeof(unsigned long long) * ef::kSameSlots, h->st));
  return EF_OK;
}

static int clear_err(ef_solver* h) {
  EF_CUDA(cudaMemsetAsync(h->w.err, 0, sizeof(int), h->st));
  EF_CUDA(cudaMemsetAsync(h->w.err_first, 0x7f, sizeof(int), h->st));  // 0x7f7f7f7f > every code
  EF_CUDA(cudaMemsetAsync(h->w.bad_gid, 0xff, sizeof(unsigned long long), h->st));
  return EF_OK;
}

static int euler_async(Driver& d, int32_t has_tau, int* out_buf) {
  const int in = d.h0()->cur, out = (in + 1) % 3;
  EF_TRY(reset_counters(d));
  std::vector<StageIO> io;
  for (ef_solver* h : d.hs) io.push_back({h->Ubuf[in], h->Ubuf[in], h->Ubuf[out]});
  StageParams sp = stage_params(d.h0(), has_tau ? ef::TAU_GIVEN : ef::TAU_CFL, 0, -1.0);
  EF_TRY(run_stage(d, io, sp));
  *out_buf = out;
  return EF_OK;
}

static int rk3_async(Driver& d, int32_t has_tau, int* out_buf) {
  const int u0 = d.h0()->cur, a = (u0 + 1) % 3, b = (u0 + 2) % 3;
  EF_TRY(reset_counters(d));
  auto io_of = [&](int in, int out) {
    std::vector<StageIO> io;
    for (ef_solver* h : d.hs) io.push_back({h->Ubuf[in], h->Ubuf[u0], h->Ubuf[out]});
    return io;
  };
  EF_TRY(run_stage(d, io_of(u0, a), stage_params(d.h0(), has_tau ? ef::TAU_GIVEN : ef::TAU_CFL, 0, -1.0)));
  EF_TRY(run_stage(d, io_of(a, b), stage_params(d.h0(), ef::TAU_DEVICE, 1, 0.25)));        // stepper.py:632
  EF_TRY(run_stage(d, io_of(b, a), stage_params(d.h0(), ef::TAU_DEVICE, 2, 2.0 / 3.0)));   // stepper.py:635
  *out_buf = a;
  return EF_OK;
}

// One step (forward Euler or SSP-RK3) queued on the stream.  A single rank with
// the timers off replays a CUDA graph of the step's launches, captured on first
// use per (kind, U buffer, tau arguments); anything else launches directly.  A
// capture that fails turns graphs off for the handle and runs the step directly.
// One step (forward Euler or SSP-RK3) queued on the stream.  With the timers
// off, the step's launches (all ranks of a same-device group, or one NCCL rank
// with its send/recv and allreduce calls and the comm-stream halo overlap) are
// captured once per key into a CUDA graph and replayed with one
// cudaGraphLaunch; the step counters and halo statistics the capture recorded
// are re-added per replay.  A capture that fails turns graphs off for the
// handle and runs the step directly.  EF_GRAPHS_NCCL=0 keeps NCCL ranks on
// direct launches.
static bool graphs_nccl() {
  const char* e = std::getenv("EF_GRAPHS_NCCL");
  return !(e && e[0] == '0');
}

static int step_async(Driver& d, bool rk3, int32_t has_tau, double tau, double tau_max, int* out_buf) {
  ef_solver* h = d.h0();
  // the step's tau arguments: a pageable-source copy is staged at the call, so the
  // host values may change before the copy executes (async chains)
  const double targ[2] = {has_tau ? tau : 0.0, tau_max};
  for (ef_solver* r : d.hs)
    EF_CUDA(cudaMemcpyAsync(r->w.tau_arg, targ, sizeof targ, cudaMemcpyHostToDevice, r->st));
  auto body = [&]() {
    return rk3 ? rk3_async(d, has_tau, out_buf) : euler_async(d, has_tau, out_buf);
  };
  if (!h->use_graphs || h->timing || (h->use_nccl && !graphs_nccl())) return body();
  int uni_mask = 0;  // every rank picks its identical-state mode on its own
  for (size_t r = 0; r < d.hs.size(); ++r) uni_mask |= (d.hs[r]->uni_on ? 1 : 0) << (r & 31);
  const ef_solver::GraphKey key{rk3 ? 1 : 0, h->cur, has_tau ? 1 : 0, uni_mask};
  for (auto& g : h->graphs)
    if (g.key == key) {
      g.used = ++h->graph_clock;
      EF_CUDA(cudaGraphLaunch(g.exec, h->st));
      ef::add_kernel_launches(g.launches);
      *out_buf = (h->cur + 1) % 3;  // euler: in + 1; rk3: u0 + 1
      for (size_t r = 0; r < d.hs.size(); ++r) {
        d.hs[r]->n_euler += rk3 ? 3 : 1;
        d.hs[r]->sync_count += g.syncs[r].first;
        d.hs[r]->sync_volume += g.syncs[r].second;
      }
      return EF_OK;
    }
  std::vector<std::array<int64_t, 3>> before;
  for (ef_solver* r : d.hs) before.push_back({r->n_euler, r->sync_count, r->sync_volume});
  const long long l0 = ef::kernel_launches();
  cudaError_t e = cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal);
  int rc = e == cudaSuccess ? body() : EF_ERR_CUDA;
  cudaGraph_t graph = nullptr;
  if (e == cudaSuccess) e = cudaStreamEndCapture(h->st, &graph);
  cudaGraphExec_t exec = nullptr;
  if (rc == EF_OK && e == cudaSuccess && graph) e = cudaGraphInstantiate(&exec, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  if (rc != EF_OK || e != cudaSuccess || !exec) {
    if (exec) cudaGraphExecDestroy(exec);
    cudaGetLastError();
    h->use_graphs = false;
    for (size_t r = 0; r < d.hs.size(); ++r) {
      d.hs[r]->n_euler = before[r][0];
      d.hs[r]->sync_count = before[r][1];
      d.hs[r]->sync_volume = before[r][2];
    }
    return body();
  }
  if (h->graphs.size() >= 8) {
    auto old = std::min_element(h->graphs.begin(), h->graphs.end(),
                                [](const auto& a, const auto& b) { return a.used < b.used; });
    cudaGraphExecDestroy(old->exec);
    h->graphs.erase(old);
  }
  std::vector<std::pair<int64_t, int64_t>> syncs;
  for (size_t r = 0; r < d.hs.size(); ++r)
    syncs.push_back({d.hs[r]->sync_count - before[r][1], d.hs[r]->sync_volume - before[r][2]});
  h->graphs.push_back({key, exec, ++h->graph_clock, ef::kernel_launches() - l0, syncs});
  EF_CUDA(cudaGraphLaunch(exec, h->st));  // the counters were advanced by the captured body
  return EF_OK;
}

static int readback(ef_solver* h) {
  EF_CUDA(cudaMemcpyAsync(&h->rb->tau, h->w.tau, sizeof(double), cudaMemcpyDeviceToHost, h->st));
  EF_CUDA(cudaMemcpyAsync(&h->rb->err, h->w.err, sizeof(int), cudaMemcpyDeviceToHost, h->st));
  EF_CUDA(cudaMemcpyAsync(&h->rb->err_first, h->w.err_first, sizeof(int), cudaMemcpyDeviceToHost, h->st));
  EF_CUDA(cudaMemcpyAsync(&h->rb->bad, h->w.bad_gid, sizeof(unsigned long long), cudaMemcpyDeviceToHost, h->st));
  EF_CUDA(cudaMemcpyAsync(h->rb->n_same, h->w.n_same, sizeof(unsigned long long) * ef::kSameSlots,
                          cudaMemcpyDeviceToHost, h->st));
  EF_CUDA(cudaStreamSynchronize(h->st));
  EF_CUDA(cudaGetLastError());
  return EF_OK;
}

// Reads the step's flags (made identical on every rank: NCCL max / min, or a
// host reduction over the group) and commits the output buffer on success.
static int finish(Driver& d, int out_buf, double* tau_used) {
  ef_solver* h0 = d.h0();
  if (d.multi() && !d.group) {
    EF_NCCL(nccl().AllReduce(h0->w.err, h0->w.err, 1, ncclInt32, ncclMax, h0->comm, h0->st));
    EF_NCCL(nccl().AllReduce(h0->w.err_first, h0->w.err_first, 1, ncclInt32, ncclMin, h0->comm, h0->st));
    EF_NCCL(nccl().AllReduce(h0->w.bad_gid, h0->w.bad_gid, 1, ncclUint64, ncclMin, h0->comm, h0->st));
  }
  int err = 0, first = ef::kErrNone;
  unsigned long long bad = ~0ull;
  for (ef_solver* h : d.hs) {
    EF_TRY(readback(h));
    err |= h->rb->err;
    first = std::min(first, h->rb->err_first);
    bad = std::min(bad, h->rb->bad);
  }
  bad &= (1ull << 56) - 1;  // drop the stage tag
  if (err) {  // the state rolls back: nothing computed for the failed stages may be reused --
              // step0 of the current state again (it also clears the memo marks)
    for (ef_solver* h : d.hs) {
      EF_TRY(clear_err(h));
      ef::launch_nodal(h->dim, h->lay, h->gas, h->Ubuf[h->cur], h->w, 0, h->lay.n_local, h->st);
      EF_CUDA(cudaGetLastError());
    }
  }
  // report the error the reference would have raised first: the earliest stage,
  // and inside it the earliest check (kernels latch min(stage * 8 + phase))
  int which = 0;
  if (err) {
    switch (first == ef::kErrNone ? -1 : first % 8) {
      case ef::PH_VISC:
      case ef::PH_INDICATOR: which = ef::ERR_PROJECT; break;
      case ef::PH_TAU: which = ef::ERR_TAU_UNBOUNDED; break;
      case ef::PH_P: which = ef::ERR_NONFINITE_P; break;
      case ef::PH_STATE: which = ef::ERR_BAD_STATE; break;
      default:
        which = (err & ef::ERR_TAU_UNBOUNDED) ? ef::ERR_TAU_UNBOUNDED
              : (err & ef::ERR_PROJECT)       ? ef::ERR_PROJECT
              : (err & ef::ERR_NONFINITE_P)   ? ef::ERR_NONFINITE_P
                                              : ef::ERR_BAD_STATE;
    }
  }
  if (which == ef::ERR_TAU_UNBOUNDED) return fail(EF_ERR_TAU_UNBOUNDED, "constant field, the time step bound is unbounded");
  if (which == ef::ERR_PROJECT) return fail(EF_ERR_INADMISSIBLE, "projected state requires rho > 0 and p > 0");
  if (which == ef::ERR_NONFINITE_P) return fail(EF_ERR_INADMISSIBLE, "non-finite correction flux P_ij (overflow)");
  if (which == ef::ERR_BAD_STATE) {
    int64_t orig = -1;  // original id of the smallest inadmissible CM id (any local copy)
    for (ef_solver* h : d.hs)
      for (int64_t i = 0; i < h->n_local && orig < 0; ++i)
        if (h->gid_host[i] == (int64_t)bad) orig = h->orig_host[i];
    for (ef_solver* h : d.hs) h->bad_node = orig;
    return fail(EF_ERR_INADMISSIBLE, "inadmissible state at node " + std::to_string(orig));
  }
  for (ef_solver* h : d.hs) {
    h->cur = out_buf;
    h->tau_last = h0->rb->tau;
    if (h->uni_force >= 0) {
      h->uni_on = h->uni_force != 0;
    } else {  // counted over the step's stages: uniform rows (on) or identical-state edges (off)
      unsigned long long c = 0;
      for (int k = 0; k < ef::kSameSlots; ++k) c += h->rb->n_same[k];
      const double base = h->uni_on ? (double)h->n_owned : (double)h->lay.n_edges;
      // 1-in-8 block sample of the first stage; the shortcut variants' checks cost
      // ~10-18% in k_edge_visc / the first limiter pass where nothing is uniform
      // (160^3 box), so they run while >= 20% of the edges / rows qualify
      h->uni_on = 8.0 * (double)c >= 0.20 * base;
    }
  }
  if (tau_used) *tau_used = h0->rb->tau;
  return EF_OK;
}

// Us[r]: rank r's input -- the whole state in original node order (global
// setup), or the rank's owned rows (per-rank setup; ghost rows then come from
// their owners through one halo exchange).  Every rank reaches the same verdict
// (NCCL max of the flags), so a rejected state leaves every rank unchanged.
static int set_state_all(Driver& d, const double* const* Us) {
  int bad = 0;
  for (size_t r = 0; r < d.hs.size(); ++r) {
    ef_solver* h = d.hs[r];
    if (h->pending_out >= 0) {  // a new state replaces an unchecked async result
      EF_CUDA(cudaStreamSynchronize(h->st));
      h->pending_out = -1;
    }
    const int spare = (h->cur + 1) % 3;
    EF_TRY(clear_err(h));
    const int64_t rows = h->local_io ? h->n_owned : h->n_global;
    EF_CUDA(cudaMemcpyAsync(h->aos_dev, Us[r], sizeof(double) * h->nvar * rows, cudaMemcpyHostToDevice, h->st));
    ef::launch_gather_state(h->dim, h->lay, h->local_io ? h->n_owned : h->n_local, h->aos_dev, h->orig_dev,
                            h->Ubuf[spare], h->w.err, h->st);
  }
  if (d.multi() && d.hs[0]->local_io) {
    const int NV = d.hs[0]->nvar;
    EF_TRY(exchange(d, {Fld{[&d](size_t r) { return d.hs[r]->Ubuf[(d.hs[r]->cur + 1) % 3]; }, NV}}, d.hs[0]->st));
  }
  if (d.multi() && !d.group) {
    ef_solver* h0 = d.h0();
    EF_NCCL(nccl().AllReduce(h0->w.err, h0->w.err, 1, ncclInt32, ncclMax, h0->comm, h0->st));
  }
  for (ef_solver* h : d.hs) {
    EF_TRY(readback(h));
    bad |= h->rb->err;
  }
  for (ef_solver* h : d.hs) EF_TRY(clear_err(h));  // (the gather used w.err for its check)
  if (bad) return fail(EF_ERR_INADMISSIBLE, "initial state is not admissible");
  for (ef_solver* h : d.hs) {
    h->cur = (h->cur + 1) % 3;
    h->pending_out = -1;
    ef::launch_nodal(h->dim, h->lay, h->gas, h->Ubuf[h->cur], h->w, 0, h->lay.n_local, h->st);
    EF_CUDA(cudaGetLastError());
  }
  return EF_OK;
}

static int get_state_one(ef_solver* h, double* U) {
  const int NV = h->nvar;
  if (h->local_io) {  // the owned rows, in order
    ef::launch_scatter_state(h->dim, h->lay, h->Ubuf[h->cur], h->orig_dev, h->aos_dev, h->st);
    EF_CUDA(cudaMemcpyAsync(U, h->aos_dev, sizeof(double) * NV * h->n_owned, cudaMemcpyDeviceToHost, h->st));
    EF_CUDA(cudaStreamSynchronize(h->st));
    return EF_OK;
  }
  if (h->nranks == 1) {
    ef::launch_scatter_state(h->dim, h->lay, h->Ubuf[h->cur], h->orig_dev, h->aos_dev, h->st);
    EF_CUDA(cudaMemcpyAsync(U, h->aos_dev, sizeof(double) * NV * h->n_global, cudaMemcpyDeviceToHost, h->st));
    EF_CUDA(cudaStreamSynchronize(h->st));
    return EF_OK;
  }
  std::vector<double> soa((size_t)NV * h->NP);
  EF_CUDA(cudaMemcpyAsync(soa.data(), h->Ubuf[h->cur], sizeof(double) * NV * h->NP, cudaMemcpyDeviceToHost, h->st));
  EF_CUDA(cudaStreamSynchronize(h->st));
  for (int64_t i = 0; i < h->n_owned; ++i)
    for (int k = 0; k < NV; ++k) U[h->orig_host[i] * NV + k] = soa[(size_t)k * h->NP + i];
  return EF_OK;
}

// ---------------------------------------------------------------- C-ABI
struct ef_plan {
  ef::Plan p;
};

// scratch device buffers of the function-check entry points, freed on every path
struct DevBufs {
  std::vector<void*> p;
  ~DevBufs() {
    for (void* q : p) cudaFree(q);
  }
  template <class T>
  int get(T** out, size_t count, const T* host = nullptr) {
    void* q = nullptr;
    EF_CUDA(cudaMalloc(&q, sizeof(T) * (count > 0 ? count : 1)));
    p.push_back(q);
    if (host) EF_CUDA(cudaMemcpy(q, host, sizeof(T) * count, cudaMemcpyHostToDevice));
    *out = (T*)q;
    return EF_OK;
  }
};

// common part of ef_create / ef_create_local: `build` fills the layout
template <class Build>
static int create_handle(int dim, const ef_params* prm, const ef_dist* dist, ef_solver** out, Build build) {
  *out = nullptr;
  if (!(prm->c_cfl > 0.0 && prm->c_cfl <= 1.0)) return fail(EF_ERR_ARG, "c_cfl must lie in (0, 1]");
  if (prm->limiter_passes < 0) return fail(EF_ERR_ARG, "limiter_passes must be >= 0");
  if (prm->newton_steps < 0) return fail(EF_ERR_ARG, "newton_steps must be >= 0");
  if (dim != 2 && dim != 3) return fail(EF_ERR_ARG, "dim must be 2 or 3");
  if (dist && (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks))
    return fail(EF_ERR_ARG, "bad rank/nranks");
  ef_solver* h = new ef_solver();
  h->dim = dim;
  h->nvar = dim + 2;
  h->passes = prm->limiter_passes;
  h->newton = prm->newton_steps;
  h->c_cfl = prm->c_cfl;
  h->gas = make_gas(prm);
  h->rank = dist ? dist->rank : 0;
  h->nranks = dist ? dist->nranks : 1;
  h->device = dist ? dist->device : 0;
  auto bail = [&](int rc) {
    std::string msg = g_err;
    delete h;
    g_err = msg;
    return rc;
  };
  cudaError_t e = cudaSetDevice(h->device);
  if (e != cudaSuccess) return bail(fail(EF_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e)));
  if (dist && dist->stream) {
    h->st = (cudaStream_t)dist->stream;
  } else {
    e = cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking);
    if (e != cudaSuccess) return bail(fail(EF_ERR_CUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e)));
    h->own_stream = true;
  }
  h->overlap = prm->overlap != 0;
  {
    const char* ge = std::getenv("EF_GRAPHS");
    h->use_graphs = !(ge && ge[0] == '0');
    const char* ue = std::getenv("EF_UNIFORM");
    if (ue && (ue[0] == '0' || ue[0] == '1')) h->uni_force = ue[0] - '0';
    h->uni_on = h->uni_force != 0;
  }
  int rc = build(h);
  if (rc != EF_OK) return bail(rc);
  if (h->nranks > 1) {
    e = cudaStreamCreateWithFlags(&h->cst, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->evB, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->evX, cudaEventDisableTiming);
    if (e != cudaSuccess) return bail(fail(EF_ERR_CUDA, std::string("comm stream: ") + cudaGetErrorString(e)));
  }
  if (h->nranks > 1 && dist->nccl_id) {
    if (!nccl().ok) return bail(fail(EF_ERR_NCCL, "libnccl.so.2 could not be loaded"));
    ncclUniqueId id;
    std::memcpy(&id, dist->nccl_id, sizeof id);
    ncclResult_t r = nccl().CommInitRank(&h->comm, h->nranks, id, h->rank);
    if (r != ncclSuccess) return bail(fail(EF_ERR_NCCL, std::string("ncclCommInitRank: ") + nccl().GetErrorString(r)));
    h->use_nccl = true;
  }
  *out = h;
  return EF_OK;
}

extern "C" {
int ef_sync(ef_solver* h, double* tau_used);

// A synchronous call after ef_ssp_rk3_step_async first settles the pending
// chain (ef_sync: its latched errors are reported by this call).
static int settle(ef_solver* h) {
  if (h->pending_out < 0) return EF_OK;
  return ef_sync(h, nullptr);
}


const char* ef_last_error(void) { return g_err.c_str(); }

int64_t ef_kernel_launches(void) { return (int64_t)ef::kernel_launches(); }

int ef_nccl_unique_id(void* out128) {
  if (!out128) return fail(EF_ERR_ARG, "null argument");
  if (!nccl().ok) return fail(EF_ERR_NCCL, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  EF_NCCL(nccl().GetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, sizeof id);
  return EF_OK;
}

int ef_create(const ef_matrices* mat, const ef_params* prm, const ef_boundary* bc, const ef_dist* dist,
              ef_solver** out) {
  if (!mat || !prm || !out) return fail(EF_ERR_ARG, "null argument");
  *out = nullptr;
  if (mat->n <= 0) return fail(EF_ERR_ARG, "empty mesh");
  return create_handle(mat->dim, prm, dist, out, [&](ef_solver* h) { return build(h, mat, bc, dist); });
}

int ef_create_local(const ef_local_matrices* lm, const ef_params* prm, const ef_boundary* bc, const ef_dist* dist,
                    ef_solver** out) {
  if (!lm || !prm || !out) return fail(EF_ERR_ARG, "null argument");
  *out = nullptr;
  if (lm->n_global <= 0 || lm->n_owned < 0 || lm->n_ghost < 0 || !lm->rowptr || !lm->col_gid ||
      (lm->n_ghost > 0 && !lm->ghost_gid))
    return fail(EF_ERR_ARG, "bad ef_local_matrices");
  return create_handle(lm->dim, prm, dist, out, [&](ef_solver* h) { return build_local(h, lm, bc, dist); });
}

int ef_destroy(ef_solver* h) {
  if (h) {
    cudaSetDevice(h->device);
    if (h->own_stream) cudaStreamSynchronize(h->st);  // a group rank borrows rank 0's stream
    delete h;
    cudaGetLastError();  // teardown errors must not surface in a later call
  }
  return EF_OK;
}

static int single_driver(ef_solver* h, Driver& d) {
  if (!h) return fail(EF_ERR_ARG, "null handle");
  if (h->nranks > 1 && !h->use_nccl)
    return fail(EF_ERR_ARG, "a rank created without nccl_id must be stepped through an ef_group");
  cudaSetDevice(h->device);
  d.hs = {h};
  d.group = false;
  return EF_OK;
}

int ef_set_state(ef_solver* h, const double* U) {
  if (!h || !U) return fail(EF_ERR_ARG, "null argument");
  if (h->local_io) return fail(EF_ERR_ARG, "a per-rank handle takes its owned rows: ef_set_state_owned");
  cudaSetDevice(h->device);
  Driver d;
  d.hs = {h};
  d.group = h->nranks > 1 && !h->use_nccl;
  const double* Us[1] = {U};
  return set_state_all(d, Us);
}

int ef_get_state(ef_solver* h, double* U) {
  if (!h || !U) return fail(EF_ERR_ARG, "null argument");
  cudaSetDevice(h->device);
  EF_TRY(settle(h));
  return get_state_one(h, U);
}

int ef_euler_step(ef_solver* h, int32_t has_tau, double tau, double tau_max, double* tau_used) {
  Driver d;
  EF_TRY(single_driver(h, d));
  EF_TRY(settle(h));
  int out;
  EF_TRY(step_async(d, false, has_tau, tau, tau_max, &out));
  return finish(d, out, tau_used);
}

int ef_ssp_rk3_step(ef_solver* h, int32_t has_tau, double tau, double tau_max, double* tau_used) {
  Driver d;
  EF_TRY(single_driver(h, d));
  EF_TRY(settle(h));
  int out;
  EF_TRY(step_async(d, true, has_tau, tau, tau_max, &out));
  return finish(d, out, tau_used);
}

int ef_set_state_owned(ef_solver* h, const double* U) {
  if (!h || !U) return fail(EF_ERR_ARG, "null argument");
  if (!h->local_io) return fail(EF_ERR_ARG, "ef_set_state_owned needs a handle from ef_create_local");
  Driver d;
  EF_TRY(single_driver(h, d));
  const double* Us[1] = {U};
  return set_state_all(d, Us);
}

int ef_get_state_owned(ef_solver* h, double* U) {
  if (!h || !U) return fail(EF_ERR_ARG, "null argument");
  if (!h->local_io) return fail(EF_ERR_ARG, "ef_get_state_owned needs a handle from ef_create_local");
  cudaSetDevice(h->device);
  EF_TRY(settle(h));
  return get_state_one(h, U);
}

int ef_ssp_rk3_step_async(ef_solver* h, int32_t has_tau, double tau, double tau_max) {
  Driver d;
  EF_TRY(single_driver(h, d));
  if (h->pending_out >= 0) h->cur = h->pending_out;  // chain on the unchecked result
  int out;
  EF_TRY(step_async(d, true, has_tau, tau, tau_max, &out));
  h->pending_out = out;
  return EF_OK;
}

int ef_sync(ef_solver* h, double* tau_used) {
  Driver d;
  EF_TRY(single_driver(h, d));
  if (h->pending_out < 0) {
    EF_CUDA(cudaStreamSynchronize(h->st));
    if (tau_used) *tau_used = h->tau_last;
    return EF_OK;
  }
  const int out = h->pending_out;
  h->pending_out = -1;
  return finish(d, out, tau_used);
}

int64_t ef_bad_node(const ef_solver* h) { return h ? h->bad_node : -1; }

int ef_enable_timers(ef_solver* h, int32_t on) {
  if (!h) return fail(EF_ERR_ARG, "null handle");
  h->timing = on != 0;
  return EF_OK;
}

int ef_set_uniform(ef_solver* h, int32_t mode) {
  if (!h) return fail(EF_ERR_ARG, "null handle");
  if (mode < -1 || mode > 1) return fail(EF_ERR_ARG, "mode must be -1 (auto), 0 (off) or 1 (on)");
  h->uni_force = mode;
  if (mode >= 0) h->uni_on = mode != 0;  // automatic: keep the current choice until the next sync
  return EF_OK;
}

int ef_enable_graphs(ef_solver* h, int32_t on) {
  if (!h) return fail(EF_ERR_ARG, "null handle");
  h->use_graphs = on != 0;
  return EF_OK;
}

int ef_phase_times(ef_solver* h, double* s7) {
  if (!h || !s7) return fail(EF_ERR_ARG, "null argument");
  EF_TRY(flush_timers(h));
  for (int k = 0; k < 7; ++k) s7[k] = h->phase_s[k];
  return EF_OK;
}

int ef_counters(ef_solver* h, int64_t* out3) {
  if (!h || !out3) return fail(EF_ERR_ARG, "null argument");
  out3[0] = h->n_euler;
  out3[1] = h->sync_count;
  out3[2] = h->sync_volume;
  return EF_OK;
}

int ef_info(ef_solver* h, int64_t* out6) {
  if (!h || !out6) return fail(EF_ERR_ARG, "null argument");
  out6[0] = h->n_owned;
  out6[1] = h->n_local;
  out6[2] = h->L;
  out6[3] = h->nnz_owned;
  out6[4] = h->standard_card;
  out6[5] = h->dim;
  return EF_OK;
}

int ef_local_gids(ef_solver* h, int64_t* out) {
  if (!h || !out) return fail(EF_ERR_ARG, "null argument");
  std::copy(h->gid_host.begin(), h->gid_host.end(), out);
  return EF_OK;
}

int ef_debug_fetch(ef_solver* h, int32_t which, int32_t which_pass, double* out) {
  if (!h || !out) return fail(EF_ERR_ARG, "null argument");
  cudaSetDevice(h->device);
  EF_CUDA(cudaStreamSynchronize(h->st));
  const int64_t n = h->n_local, NP = h->NP, L = h->L, NPL = h->NPL;
  const int NV = h->nvar;
  auto node_field = [&](const double* dev, int ncomp) -> int {
    std::vector<double> tmp((size_t)ncomp * NP);
    EF_CUDA(cudaMemcpy(tmp.data(), dev, sizeof(double) * ncomp * NP, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n; ++i)
      for (int k = 0; k < ncomp; ++k) out[i * ncomp + k] = tmp[(size_t)k * NP + i];
    return EF_OK;
  };
  auto slot_field = [&](const double* dev) -> int {
    std::vector<double> tmp(NPL);
    EF_CUDA(cudaMemcpy(tmp.data(), dev, sizeof(double) * NPL, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n; ++i)
      for (int s = 0; s < L; ++s) out[i * L + s] = tmp[ef::sidx(i, s, (int)L)];
    return EF_OK;
  };
  switch (which) {
    case 0: return slot_field(h->w.d);
    case 1: return node_field(h->w.alpha, 1);
    case 2: return node_field(h->w.R, NV);
    case 3: return node_field(h->w.bounds, 3);
    case 4:  // min(l_ij, l_ji) of the last limiter pass
      (void)which_pass;
      return slot_field(h->w.ml2);
    case 5: return node_field(h->w.eor, 1);
    case 6: return node_field(h->w.phi, 1);
    case 7: return node_field(h->Ubuf[h->cur], NV);
    case 8: return node_field(h->w.Unext, NV);
    case 9: return slot_field(h->w.ml);  // min(l_ij, l_ji) of the last non-final pass
    case 10: {  // P_0 as stored: (n_local, L, nvar); the pass structure is applied by the caller
      std::vector<double> tmp((size_t)NV * NPL);
      EF_CUDA(cudaMemcpy(tmp.data(), h->w.P, sizeof(double) * NV * NPL, cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < n; ++i)
        for (int s = 0; s < L; ++s)
          for (int k = 0; k < NV; ++k) out[(i * L + s) * NV + k] = tmp[(size_t)k * NPL + ef::sidx(i, s, (int)L)];
      return EF_OK;
    }
  }
  return fail(EF_ERR_ARG, "unknown field");
}

void ef_pow_host(const double* x, double y, double* out, int64_t n) {
  for (int64_t q = 0; q < n; ++q) out[q] = ef_pow(x[q], y);
}

int ef_pow_device(const double* x, double y, double* out, int64_t n) {
  if (n <= 0) return EF_OK;
  double *dx = nullptr, *dy = nullptr;
  EF_CUDA(cudaMalloc(&dx, sizeof(double) * n));
  EF_CUDA(cudaMalloc(&dy, sizeof(double) * n));
  EF_CUDA(cudaMemcpy(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice));
  ef::launch_pow(dx, y, dy, n, 0);
  EF_CUDA(cudaGetLastError());
  EF_CUDA(cudaMemcpy(out, dy, sizeof(double) * n, cudaMemcpyDeviceToHost));
  cudaFree(dx);
  cudaFree(dy);
  return EF_OK;
}

int ef_pow_bound_device(const double* x, double y, double* out, int64_t n) {
  if (n <= 0) return EF_OK;
  if (!x || !out) return fail(EF_ERR_ARG, "null argument");
  DevBufs b;
  double *dx, *dy;
  EF_TRY(b.get(&dx, (size_t)n, x));
  EF_TRY(b.get(&dy, (size_t)n));
  ef::launch_pow_ub(dx, y, dy, n, 0);
  EF_CUDA(cudaGetLastError());
  EF_CUDA(cudaMemcpy(out, dy, sizeof(double) * n, cudaMemcpyDeviceToHost));
  return EF_OK;
}

int ef_eval_arith(int64_t n, const double* a, const double* b, uint64_t* mismatches) {
  if (n < 0 || !mismatches) return fail(EF_ERR_ARG, "bad arguments");
  for (int k = 0; k < 4; ++k) mismatches[k] = 0;
  if (n == 0) return EF_OK;
  if (!a || !b) return fail(EF_ERR_ARG, "null argument");
  DevBufs bufs;
  double *da, *db;
  unsigned long long* dm;
  EF_TRY(bufs.get(&da, (size_t)n, a));
  EF_TRY(bufs.get(&db, (size_t)n, b));
  EF_TRY(bufs.get(&dm, (size_t)4));
  EF_CUDA(cudaMemset(dm, 0, 4 * sizeof(unsigned long long)));
  ef::launch_eval_arith(n, da, db, dm, 0);
  EF_CUDA(cudaGetLastError());
  EF_CUDA(cudaMemcpy(mismatches, dm, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  return EF_OK;
}

int ef_eval_dij(const ef_params* prm, int32_t dim, int64_t n, const double* Ui, const double* Uj,
                const double* cij, const double* cji, double* out, int32_t* bad) {
  if (!prm || (dim != 2 && dim != 3) || n < 0) return fail(EF_ERR_ARG, "bad arguments");
  if (n == 0) return EF_OK;
  if (!Ui || !Uj || !cij || !cji || !out || !bad) return fail(EF_ERR_ARG, "null argument");
  const Gas g = make_gas(prm);
  const size_t nv = (size_t)dim + 2;
  DevBufs b;
  double *dUi, *dUj, *dci, *dcj, *dout;
  int* dbad;
  EF_TRY(b.get(&dUi, n * nv, Ui));
  EF_TRY(b.get(&dUj, n * nv, Uj));
  EF_TRY(b.get(&dci, n * (size_t)dim, cij));
  EF_TRY(b.get(&dcj, n * (size_t)dim, cji));
  EF_TRY(b.get(&dout, (size_t)n));
  EF_TRY(b.get(&dbad, (size_t)n));
  ef::launch_eval_dij(dim, g, n, dUi, dUj, dci, dcj, dout, dbad, 0);
  EF_CUDA(cudaGetLastError());
  EF_CUDA(cudaMemcpy(out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost));
  EF_CUDA(cudaMemcpy(bad, dbad, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  return EF_OK;
}

int ef_eval_limiter(const ef_params* prm, int32_t dim, int64_t n, const double* U, const double* P,
                    const double* bounds, double* out) {
  if (!prm || (dim != 2 && dim != 3) || n < 0) return fail(EF_ERR_ARG, "bad arguments");
  if (n == 0) return EF_OK;
  if (!U || !P || !bounds || !out) return fail(EF_ERR_ARG, "null argument");
  const Gas g = make_gas(prm);
  const size_t nv = (size_t)dim + 2;
  DevBufs b;
  double *dU, *dP, *dB, *dout;
  EF_TRY(b.get(&dU, n * nv, U));
  EF_TRY(b.get(&dP, n * nv, P));
  EF_TRY(b.get(&dB, n * (size_t)3, bounds));
  EF_TRY(b.get(&dout, (size_t)n));
  ef::launch_eval_limiter(dim, g, n, dU, dP, dB, prm->newton_steps, dout, 0);
  EF_CUDA(cudaGetLastError());
  EF_CUDA(cudaMemcpy(out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost));
  return EF_OK;
}

int ef_state_device_ptr(ef_solver* h, void** dev_ptr, int64_t* stride) {
  if (!h || !dev_ptr || !stride) return fail(EF_ERR_ARG, "null argument");
  *dev_ptr = h->Ubuf[h->cur];
  *stride = h->NP;
  return EF_OK;
}

// ---- same-device group: all ranks of a partition in one process/GPU
int ef_group_create(ef_solver** hs, int32_t n, ef_group** out) {
  if (!hs || !out || n < 1) return fail(EF_ERR_ARG, "null argument");
  for (int r = 0; r < n; ++r) {
    if (!hs[r] || hs[r]->rank != r || hs[r]->nranks != n) return fail(EF_ERR_ARG, "group needs ranks 0..n-1 of one partition");
    if (hs[r]->device != hs[0]->device) return fail(EF_ERR_ARG, "group ranks must share one device");
    if (hs[r]->use_nccl) return fail(EF_ERR_ARG, "group ranks must be created without nccl_id");
  }
  ef_group* g = new ef_group();
  g->hs.assign(hs, hs + n);
  cudaSetDevice(hs[0]->device);
  for (int r = 1; r < n; ++r) {  // one stream for the whole group: ordered phases, no waiting kernels
    cudaStreamSynchronize(hs[r]->st);
    if (hs[r]->own_stream && hs[r]->st && hs[r]->st != hs[0]->st) cudaStreamDestroy(hs[r]->st);
    hs[r]->own_stream = false;
    hs[r]->st = hs[0]->st;
  }
  std::vector<unsigned long long*> bits;
  for (auto* h : g->hs) bits.push_back(h->w.tau_min_bits);
  cudaError_t e = cudaMalloc(&g->bits_dev, sizeof(unsigned long long*) * n);
  if (e == cudaSuccess) e = cudaMemcpy(g->bits_dev, bits.data(), sizeof(unsigned long long*) * n, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    delete g;
    return fail(EF_ERR_CUDA, std::string("group setup: ") + cudaGetErrorString(e));
  }
  *out = g;
  return EF_OK;
}

int ef_group_destroy(ef_group* g) {
  if (g) {
    cudaSetDevice(g->hs[0]->device);
    cudaStreamSynchronize(g->hs[0]->st);
    if (g->bits_dev) cudaFree(g->bits_dev);
    delete g;
    cudaGetLastError();
  }
  return EF_OK;
}

static Driver group_driver(ef_group* g) {
  Driver d;
  d.hs = g->hs;
  d.group = true;
  d.bits_dev = g->bits_dev;
  cudaSetDevice(g->hs[0]->device);
  return d;
}

int ef_group_set_state(ef_group* g, const double* U) {
  if (!g || !U) return fail(EF_ERR_ARG, "null argument");
  if (g->hs[0]->local_io) return fail(EF_ERR_ARG, "per-rank handles take their owned rows: ef_group_set_state_owned");
  Driver d = group_driver(g);
  std::vector<const double*> Us(d.hs.size(), U);
  return set_state_all(d, Us.data());
}

int ef_group_set_state_owned(ef_group* g, const double* const* U) {
  if (!g || !U) return fail(EF_ERR_ARG, "null argument");
  if (!g->hs[0]->local_io) return fail(EF_ERR_ARG, "ef_group_set_state_owned needs handles from ef_create_local");
  for (size_t r = 0; r < g->hs.size(); ++r)
    if (!U[r]) return fail(EF_ERR_ARG, "null argument");
  Driver d = group_driver(g);
  return set_state_all(d, U);
}

int ef_group_get_state_owned(ef_group* g, double* const* U) {
  if (!g || !U) return fail(EF_ERR_ARG, "null argument");
  if (!g->hs[0]->local_io) return fail(EF_ERR_ARG, "ef_group_get_state_owned needs handles from ef_create_local");
  for (size_t r = 0; r < g->hs.size(); ++r) {
    if (!U[r]) return fail(EF_ERR_ARG, "null argument");
    EF_TRY(get_state_one(g->hs[r], U[r]));
  }
  return EF_OK;
}

int ef_group_get_state(ef_group* g, double* U) {
  if (!g || !U) return fail(EF_ERR_ARG, "null argument");
  for (ef_solver* h : g->hs) EF_TRY(get_state_one(h, U));
  return EF_OK;
}

int ef_group_euler_step(ef_group* g, int32_t has_tau, double tau, double tau_max, double* tau_used) {
  if (!g) return fail(EF_ERR_ARG, "null handle");
  Driver d = group_driver(g);
  int out;
  EF_TRY(step_async(d, false, has_tau, tau, tau_max, &out));
  return finish(d, out, tau_used);
}

int ef_group_ssp_rk3_step(ef_group* g, int32_t has_tau, double tau, double tau_max, double* tau_used) {
  if (!g) return fail(EF_ERR_ARG, "null handle");
  Driver d = group_driver(g);
  int out;
  EF_TRY(step_async(d, true, has_tau, tau, tau_max, &out));
  return finish(d, out, tau_used);
}

// ---- host-only partition plans (no CUDA; CPU tests)
int ef_plan_build(const ef_matrices* mat, const ef_dist* dist, ef_plan** out) {
  if (!mat || !dist || !out || !dist->cm_perm) return fail(EF_ERR_ARG, "null argument");
  if (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks) return fail(EF_ERR_ARG, "bad rank/nranks");
  ef_plan* p = new ef_plan();
  if (!ef::build_plan(mat->n, mat->indptr, mat->indices, dist->cm_perm, dist->rank, dist->nranks, dist->ranges, p->p)) {
    std::string msg = p->p.error;
    delete p;
    return fail(EF_ERR_ARG, msg);
  }
  *out = p;
  return EF_OK;
}

int ef_plan_build_local(const ef_local_matrices* lm, const ef_dist* dist, ef_plan** out) {
  if (!lm || !dist || !out || !lm->rowptr || !lm->col_gid) return fail(EF_ERR_ARG, "null argument");
  if (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks) return fail(EF_ERR_ARG, "bad rank/nranks");
  ef_plan* p = new ef_plan();
  if (!ef::build_plan_local(lm->n_global, lm->n_owned, lm->n_ghost, lm->ghost_gid, lm->rowptr, lm->col_gid,
                            lm->pad_width, lm->standard_card, dist->rank, dist->nranks, dist->ranges, p->p)) {
    std::string msg = p->p.error;
    delete p;
    return fail(EF_ERR_ARG, msg);
  }
  *out = p;
  return EF_OK;
}

int ef_plan_destroy(ef_plan* p) {
  delete p;
  return EF_OK;
}

int ef_plan_sizes(const ef_plan* p, int64_t* out4) {
  if (!p || !out4) return fail(EF_ERR_ARG, "null argument");
  out4[0] = p->p.n_owned;
  out4[1] = p->p.n_local;
  out4[2] = p->p.L;
  out4[3] = p->p.nranks;
  return EF_OK;
}

int64_t ef_plan_rows(const ef_plan* p, int32_t peer, int32_t recv, int64_t* out_gids, int64_t cap) {
  if (!p || peer < 0 || peer >= p->p.nranks) return -1;
  const auto& v = recv ? p->p.recv_rows[peer] : p->p.send_rows[peer];
  if (out_gids)
    for (int64_t k = 0; k < (int64_t)v.size() && k < cap; ++k) out_gids[k] = p->p.gid[v[k]];
  return (int64_t)v.size();
}

}  // extern "C"
