// ef_capi.cu — host side of the C-ABI (include/ef_b200.h): setup of the
// SELL-32 layout, device memory, stage orchestration and error mapping.
//
// Setup restates the reference's ordering contract natively (the reference
// does it with per-row Python loops, stepper.py:163-268, sparsity.py:168-309):
//   * rows live in global Cuthill-McKee order (cm_perm from exchange.partition);
//   * a row's slots are its stencil columns sorted by CM id (stepper.py:195);
//   * the pad width L is the global maximum cardinality (stepper.py:128-129);
//   * ghost rows (nranks > 1) carry the stencil truncated to local rows
//     (stepper.py:175-181).
#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ef_b200.h"
#include "ef_kernels.cuh"

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

struct ef_solver {
  int dim = 0, nvar = 0, L = 0, passes = 0, newton = 0, standard_card = 0;
  double c_cfl = 0.9;
  Gas gas{};
  int64_t n_global = 0, n_owned = 0, n_local = 0, NP = 0, NPL = 0, nnz_owned = 0;
  int rank = 0, nranks = 1, device = 0;
  int64_t range_lo = 0;
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
  // pinned readback block: [0] tau (double), [1] err (int), [2] bad gid
  struct Readback {
    double tau;
    int err;
    int pad;
    unsigned long long bad;
  }* rb = nullptr;
  double tau_last = 0.0;
  int64_t bad_node = -1;
  bool timing = false;
  double phase_s[7] = {0, 0, 0, 0, 0, 0, 0};
  int64_t n_euler = 0;
  // timing ring: 8 events per stage, recorded without host syncs and folded
  // into phase_s when the ring fills or the timers are read
  std::vector<std::array<cudaEvent_t, 8>> ring;
  int ring_used = 0;

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
    if (own_stream && st) cudaStreamDestroy(st);
  }
};

#define EF_TRY(x)                 \
  do {                            \
    int rc_ = (x);                \
    if (rc_ != EF_OK) return rc_; \
  } while (0)

template <class T>
static int upload(ef_solver* h, T** dst, const std::vector<T>& src) {
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
  return g;
}

static int build(ef_solver* h, const ef_matrices* mat, const ef_params* prm, const ef_boundary* bc,
                 const ef_dist* dist) {
  const int D = h->dim, NV = h->nvar;
  const int64_t n = mat->n;
  const int R = dist ? dist->nranks : 1;
  const int r = dist ? dist->rank : 0;
  if (!dist || !dist->cm_perm) return fail(EF_ERR_ARG, "ef_dist.cm_perm is required");
  const int64_t* cm_perm = dist->cm_perm;
  std::vector<int64_t> cm_inv(n, -1);
  for (int64_t o = 0; o < n; ++o) {
    const int64_t g = cm_perm[o];
    if (g < 0 || g >= n || cm_inv[g] >= 0) return fail(EF_ERR_ARG, "cm_perm is not a permutation");
    cm_inv[g] = o;
  }
  // owned range (exchange.py:405-411 when ranges == NULL)
  int64_t s_lo, s_hi;
  if (dist->ranges) {
    s_lo = dist->ranges[r];
    s_hi = dist->ranges[r + 1];
  } else {
    const int64_t base = n / R, extra = n % R;
    s_lo = r * base + std::min<int64_t>(r, extra);
    s_hi = s_lo + base + (r < extra ? 1 : 0);
  }
  h->range_lo = s_lo;
  // global pad width and the most frequent cardinality
  int64_t L = 0;
  std::vector<int64_t> card_hist(1, 0);
  for (int64_t o = 0; o < n; ++o) {
    const int64_t c = mat->indptr[o + 1] - mat->indptr[o];
    L = std::max(L, c);
    if ((int64_t)card_hist.size() <= c) card_hist.resize(c + 1, 0);
    card_hist[c]++;
  }
  if (L > 255) return fail(EF_ERR_ARG, "stencil cardinality above 255 is not supported");
  h->L = (int)L;
  h->standard_card = (int)(std::max_element(card_hist.begin(), card_hist.end()) - card_hist.begin());
  // local rows: owned CM ids, then ghosts (ascending CM id)
  const int64_t n_owned = s_hi - s_lo;
  h->n_global = n;
  std::vector<int64_t> ghosts;
  for (int64_t g = s_lo; g < s_hi; ++g) {
    const int64_t o = cm_inv[g];
    for (int64_t q = mat->indptr[o]; q < mat->indptr[o + 1]; ++q) {
      const int64_t cg = cm_perm[mat->indices[q]];
      if (cg < s_lo || cg >= s_hi) ghosts.push_back(cg);
    }
  }
  std::sort(ghosts.begin(), ghosts.end());
  ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
  const int64_t n_local = n_owned + (int64_t)ghosts.size();
  auto local_of = [&](int64_t g) -> int64_t {
    if (g >= s_lo && g < s_hi) return g - s_lo;
    auto it = std::lower_bound(ghosts.begin(), ghosts.end(), g);
    if (it != ghosts.end() && *it == g) return n_owned + (it - ghosts.begin());
    return -1;
  };
  h->n_owned = n_owned;
  h->n_local = n_local;
  h->NP = (n_local + 31) / 32 * 32;
  if (h->NP == 0) h->NP = 32;
  h->NPL = h->NP * L;
  const int64_t NP = h->NP, NPL = h->NPL;
  h->gid_host.resize(n_local);
  h->orig_host.resize(n_local);
  for (int64_t i = 0; i < n_owned; ++i) h->gid_host[i] = s_lo + i;
  for (size_t k = 0; k < ghosts.size(); ++k) h->gid_host[n_owned + k] = ghosts[k];
  for (int64_t i = 0; i < n_local; ++i) h->orig_host[i] = cm_inv[h->gid_host[i]];

  // per local row: slots sorted by CM id, truncated to local columns
  std::vector<int64_t> rptr(n_local + 1, 0);
  std::vector<int64_t> rcm;   // CM id per slot
  std::vector<int64_t> rsrc;  // source nnz index per slot
  rcm.reserve((size_t)n_local * L);
  rsrc.reserve((size_t)n_local * L);
  std::vector<std::pair<int64_t, int64_t>> tmp;
  for (int64_t i = 0; i < n_local; ++i) {
    const int64_t o = h->orig_host[i];
    tmp.clear();
    for (int64_t q = mat->indptr[o]; q < mat->indptr[o + 1]; ++q) {
      const int64_t cg = cm_perm[mat->indices[q]];
      if (i >= n_owned && local_of(cg) < 0) continue;
      tmp.emplace_back(cg, q);
    }
    std::sort(tmp.begin(), tmp.end());
    for (auto& t : tmp) {
      rcm.push_back(t.first);
      rsrc.push_back(t.second);
    }
    rptr[i + 1] = (int64_t)rcm.size();
  }
  // SELL-32 host images
  std::vector<int32_t> col(NPL);
  std::vector<uint8_t> tslot(NPL, 0), card(NP, 1), diag(NP, 0);
  std::vector<double> c((size_t)D * NPL, 0.0), cT((size_t)D * NPL, 0.0), mij(NPL, 0.0);
  std::vector<double> m_i(NP, 1.0), inv_m(NP, 1.0), lam(NP, 1.0);
  std::vector<int64_t> gid(NP, 0);
  for (int64_t i = 0; i < NP; ++i)
    for (int s = 0; s < L; ++s) col[ef::sidx(i, s, (int)L)] = (int32_t)std::min<int64_t>(i, n_local > 0 ? n_local - 1 : 0);
  int64_t nnz_owned = 0;
  for (int64_t i = 0; i < n_local; ++i) {
    const int64_t o = h->orig_host[i];
    const int64_t cnt = rptr[i + 1] - rptr[i];
    card[i] = (uint8_t)cnt;
    if (i < n_owned) nnz_owned += cnt;
    int dg = -1;
    for (int64_t s = 0; s < cnt; ++s) {
      const int64_t cg = rcm[rptr[i] + s];
      const int64_t j = local_of(cg);
      const int64_t q = rsrc[rptr[i] + s];
      const int64_t p = ef::sidx(i, (int)s, (int)L);
      col[p] = (int32_t)j;
      if (j == i) dg = (int)s;
      mij[p] = mat->m[q];
      for (int a = 0; a < D; ++a) c[(size_t)a * NPL + p] = mat->c[q * D + a];
      // transpose slot: position of this row's CM id in row j
      const int64_t* b = rcm.data() + rptr[j];
      const int64_t* e = rcm.data() + rptr[j + 1];
      const int64_t* it = std::lower_bound(b, e, h->gid_host[i]);
      if (it == e || *it != h->gid_host[i]) {
        if (i < n_owned || j < n_owned)
          return fail(EF_ERR_ARG, "stencil pattern is not structurally symmetric");
        tslot[p] = 0;
      } else {
        tslot[p] = (uint8_t)(it - b);
      }
    }
    if (dg < 0) return fail(EF_ERR_ARG, "every stencil must contain its own row");
    diag[i] = (uint8_t)dg;
    m_i[i] = mat->m_lumped[o];
    inv_m[i] = mat->inv_m[o];
    const int64_t den = std::max<int64_t>(cnt - 1, 1);
    lam[i] = 1.0 / (double)den;
    gid[i] = h->gid_host[i];
  }
  for (int64_t i = 0; i < n_local; ++i) {
    const int64_t cnt = rptr[i + 1] - rptr[i];
    for (int64_t s = 0; s < cnt; ++s) {
      const int64_t p = ef::sidx(i, (int)s, (int)L);
      const int64_t j = col[p];
      const int64_t pt = ef::sidx(j, tslot[p], (int)L);
      for (int a = 0; a < D; ++a) cT[(size_t)a * NPL + p] = c[(size_t)a * NPL + pt];
    }
  }
  h->nnz_owned = nnz_owned;
  // upper-triangle edge list (all local rows: ghost rows need d for the mirror)
  if (NPL >= (int64_t)1 << 31) return fail(EF_ERR_ARG, "local slot count exceeds int32 positions");
  std::vector<int32_t> edges;
  for (int64_t sl = 0; sl < NP / 32; ++sl)
    for (int s = 0; s < L; ++s)
      for (int ln = 0; ln < 32; ++ln) {
        const int64_t i = sl * 32 + ln;
        if (i >= n_local) continue;
        if (s > diag[i] && s < card[i]) edges.push_back((int32_t)ef::sidx(i, s, (int)L));
      }
  // boundary data (stepper.py:258-267): owned rows only
  std::vector<int8_t> bc_kind(NP, 0);
  std::vector<double> bc_n((size_t)D * NP, 0.0);
  double farfield[5] = {0, 0, 0, 0, 0};
  if (bc) {
    for (int64_t q = 0; q < bc->n_slip; ++q) {
      const int64_t o = bc->slip[q];
      if (o < 0 || o >= n) return fail(EF_ERR_ARG, "slip node id out of range");
      const int64_t g = cm_perm[o];
      if (g < s_lo || g >= s_hi) continue;
      const int64_t i = g - s_lo;
      bc_kind[i] |= 1;
      for (int a = 0; a < D; ++a) bc_n[(size_t)a * NP + i] = bc->slip_normals[q * D + a];
    }
    for (int64_t q = 0; q < bc->n_inflow; ++q) {
      const int64_t o = bc->inflow[q];
      if (o < 0 || o >= n) return fail(EF_ERR_ARG, "inflow node id out of range");
      const int64_t g = cm_perm[o];
      if (g < s_lo || g >= s_hi) continue;
      bc_kind[g - s_lo] |= 2;
    }
    if (bc->n_inflow > 0) {
      if (!bc->farfield) return fail(EF_ERR_ARG, "inflow nodes need a farfield state");
      for (int k = 0; k < NV; ++k) farfield[k] = bc->farfield[k];
    }
  }

  // ---- device images
  Layout& m = h->lay;
  m.L = (int)L;
  m.NP = NP;
  m.n_local = n_local;
  m.n_owned = n_owned;
  int32_t* d_col;
  uint8_t *d_tslot, *d_card, *d_diag;
  double *d_c, *d_cT, *d_mij, *d_mi, *d_invm, *d_lam, *d_bcn;
  int64_t* d_gid;
  int8_t* d_bck;
  EF_TRY(upload(h, &d_col, col));
  EF_TRY(upload(h, &d_tslot, tslot));
  EF_TRY(upload(h, &d_card, card));
  EF_TRY(upload(h, &d_diag, diag));
  EF_TRY(upload(h, &d_c, c));
  EF_TRY(upload(h, &d_cT, cT));
  EF_TRY(upload(h, &d_mij, mij));
  EF_TRY(upload(h, &d_mi, m_i));
  EF_TRY(upload(h, &d_invm, inv_m));
  EF_TRY(upload(h, &d_lam, lam));
  EF_TRY(upload(h, &d_gid, gid));
  EF_TRY(upload(h, &d_bck, bc_kind));
  EF_TRY(upload(h, &d_bcn, bc_n));
  int32_t* d_edges;
  EF_TRY(upload(h, &d_edges, edges));
  m.edges = d_edges;
  m.n_edges = (int64_t)edges.size();
  m.slab = ef::make_fastdiv((uint32_t)(32 * L));
  m.col = d_col;
  m.tslot = d_tslot;
  m.card = d_card;
  m.diag = d_diag;
  m.c = d_c;
  m.cT = d_cT;
  m.mij = d_mij;
  m.m_i = d_mi;
  m.inv_m = d_invm;
  m.lam = d_lam;
  m.gid = d_gid;
  m.bc_kind = d_bck;
  m.bc_n = d_bcn;
  for (int k = 0; k < 5; ++k) m.farfield[k] = farfield[k];

  Work& w = h->w;
  EF_TRY(h->alloc(&w.eor, NP));
  EF_TRY(h->alloc(&w.phi, NP));
  EF_TRY(h->alloc(&w.alpha, NP));
  EF_TRY(h->alloc(&w.R, (size_t)NV * NP));
  EF_TRY(h->alloc(&w.Unext, (size_t)NV * NP));
  EF_TRY(h->alloc(&w.bounds, (size_t)3 * NP));
  EF_TRY(h->alloc(&w.d, NPL));
  EF_TRY(h->alloc(&w.l, (size_t)std::max(1, h->passes) * NPL));
  EF_TRY(h->alloc(&w.P, (size_t)NV * NPL));
  EF_CUDA(cudaMemset(w.P, 0, sizeof(double) * NV * NPL));

  EF_TRY(h->alloc(&w.tau_min_bits, 1));
  EF_TRY(h->alloc(&w.tau, 1));
  EF_TRY(h->alloc(&w.err, 1));
  EF_TRY(h->alloc(&w.bad_gid, 1));
  EF_CUDA(cudaMemset(w.d, 0, sizeof(double) * NPL));
  EF_CUDA(cudaMemset(w.l, 0, sizeof(double) * std::max(1, h->passes) * NPL));
  EF_CUDA(cudaMemset(w.alpha, 0, sizeof(double) * NP));
  EF_CUDA(cudaMemset(w.R, 0, sizeof(double) * NV * NP));
  EF_CUDA(cudaMemset(w.eor, 0, sizeof(double) * NP));
  EF_CUDA(cudaMemset(w.phi, 0, sizeof(double) * NP));
  for (int k = 0; k < 3; ++k) {
    EF_TRY(h->alloc(&h->Ubuf[k], (size_t)NV * NP));
    EF_CUDA(cudaMemset(h->Ubuf[k], 0, sizeof(double) * NV * NP));
  }
  EF_TRY(h->alloc(&h->aos_dev, (size_t)n * NV));
  EF_TRY(upload(h, &h->orig_dev, h->orig_host));
  EF_CUDA(cudaMallocHost((void**)&h->rb, sizeof(ef_solver::Readback)));
  (void)prm;
  return EF_OK;
}

extern "C" {

const char* ef_last_error(void) { return g_err.c_str(); }

int ef_create(const ef_matrices* mat, const ef_params* prm, const ef_boundary* bc,
              const ef_dist* dist, ef_solver** out) {
  if (!mat || !prm || !out) return fail(EF_ERR_ARG, "null argument");
  *out = nullptr;
  if (!(prm->c_cfl > 0.0 && prm->c_cfl <= 1.0)) return fail(EF_ERR_ARG, "c_cfl must lie in (0, 1]");
  if (prm->limiter_passes < 0) return fail(EF_ERR_ARG, "limiter_passes must be >= 0");
  if (prm->newton_steps < 0) return fail(EF_ERR_ARG, "newton_steps must be >= 0");
  if (mat->dim != 2 && mat->dim != 3) return fail(EF_ERR_ARG, "dim must be 2 or 3");
  if (mat->n <= 0) return fail(EF_ERR_ARG, "empty mesh");
  if (dist && (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks))
    return fail(EF_ERR_ARG, "bad rank/nranks");
  if (dist && dist->nranks > 1)
    return fail(EF_ERR_ARG, "multi-rank halo exchange is not built into this library version");
  ef_solver* h = new ef_solver();
  h->dim = mat->dim;
  h->nvar = mat->dim + 2;
  h->passes = prm->limiter_passes;
  h->newton = prm->newton_steps;
  h->c_cfl = prm->c_cfl;
  h->gas = make_gas(prm);
  h->rank = dist ? dist->rank : 0;
  h->nranks = dist ? dist->nranks : 1;
  h->device = dist ? dist->device : 0;
  cudaError_t e = cudaSetDevice(h->device);
  if (e != cudaSuccess) {
    delete h;
    return fail(EF_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  }
  if (dist && dist->stream) {
    h->st = (cudaStream_t)dist->stream;
  } else {
    e = cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete h;
      return fail(EF_ERR_CUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
    }
    h->own_stream = true;
  }
  int rc = build(h, mat, prm, bc, dist);
  if (rc != EF_OK) {
    std::string msg = g_err;
    delete h;
    g_err = msg;
    return rc;
  }
  *out = h;
  return EF_OK;
}

int ef_destroy(ef_solver* h) {
  if (h) {
    cudaSetDevice(h->device);
    cudaStreamSynchronize(h->st);
    delete h;
  }
  return EF_OK;
}

static int readback(ef_solver* h) {
  EF_CUDA(cudaMemcpyAsync(&h->rb->tau, h->w.tau, sizeof(double), cudaMemcpyDeviceToHost, h->st));
  EF_CUDA(cudaMemcpyAsync(&h->rb->err, h->w.err, sizeof(int), cudaMemcpyDeviceToHost, h->st));
  EF_CUDA(cudaMemcpyAsync(&h->rb->bad, h->w.bad_gid, sizeof(unsigned long long), cudaMemcpyDeviceToHost, h->st));
  EF_CUDA(cudaStreamSynchronize(h->st));
  EF_CUDA(cudaGetLastError());
  return EF_OK;
}

int ef_set_state(ef_solver* h, const double* U) {
  if (!h || !U) return fail(EF_ERR_ARG, "null argument");
  cudaSetDevice(h->device);
  const int NV = h->nvar;
  // upload the full array, permute it into local SoA order on the device
  // (into a spare buffer, so a rejected state leaves the current one intact)
  const int spare = (h->cur + 1) % 3;
  EF_CUDA(cudaMemsetAsync(h->w.err, 0, sizeof(int), h->st));
  EF_CUDA(cudaMemcpyAsync(h->aos_dev, U, sizeof(double) * NV * h->n_global, cudaMemcpyHostToDevice, h->st));
  ef::launch_gather_state(h->dim, h->lay, h->aos_dev, h->orig_dev, h->Ubuf[spare], h->w.err, h->st);
  EF_TRY(readback(h));
  if (h->rb->err) return fail(EF_ERR_INADMISSIBLE, "initial state is not admissible");
  h->cur = spare;
  h->pending_out = -1;
  ef::launch_nodal(h->dim, h->lay, h->gas, h->Ubuf[h->cur], h->w, 0, h->lay.n_local, h->st);
  EF_CUDA(cudaGetLastError());
  return EF_OK;
}

int ef_get_state(ef_solver* h, double* U) {
  if (!h || !U) return fail(EF_ERR_ARG, "null argument");
  cudaSetDevice(h->device);
  const int NV = h->nvar;
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

// ---- one forward-Euler stage (stepper.py:508-610) --------------------------------
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

static int run_stage(ef_solver* h, const double* U, const double* U0, double* Uout, StageParams sp) {
  const int D = h->dim;
  const bool want_tau = sp.tau_mode == ef::TAU_CFL;
  EF_TRY(mark(h, 0));
  EF_TRY(mark(h, 1));  // step0 is fused into the previous stage's final kernel
  ef::launch_edge_visc(D, h->lay, h->gas, U, h->w, want_tau, h->st);
  EF_TRY(mark(h, 2));
  ef::launch_row_visc(D, h->lay, h->gas, U, h->w, want_tau, h->st);
  EF_TRY(mark(h, 3));
  ef::launch_low_order(D, h->lay, h->gas, U, h->w, sp, h->st);
  EF_TRY(mark(h, 4));
  if (h->passes > 0) {
    ef::launch_limiter0(D, h->lay, h->gas, U, h->w, sp, h->st);
    EF_TRY(mark(h, 5));
    for (int p = 0; p + 1 < h->passes; ++p) ef::launch_pass(D, h->lay, h->gas, U, h->w, sp, p, h->st);
    EF_TRY(mark(h, 6));
  } else {
    EF_TRY(mark(h, 5));
    EF_TRY(mark(h, 6));
  }
  ef::launch_final(D, h->lay, h->gas, U, U0, Uout, h->w, sp, h->st);
  EF_TRY(mark(h, 7));
  EF_CUDA(cudaGetLastError());
  h->n_euler++;
  return EF_OK;
}

static StageParams stage_params(ef_solver* h, int mode, double tau, double tau_max, double rk_a) {
  StageParams sp;
  sp.tau_mode = mode;
  sp.tau_given = tau;
  sp.tau_max = tau_max;
  sp.c_cfl = h->c_cfl;
  sp.newton = h->newton;
  sp.passes = h->passes;
  sp.rk_a = rk_a;
  return sp;
}

static int reset_flags(ef_solver* h) {
  EF_CUDA(cudaMemsetAsync(h->w.err, 0, sizeof(int), h->st));
  EF_CUDA(cudaMemsetAsync(h->w.bad_gid, 0xff, sizeof(unsigned long long), h->st));
  return EF_OK;
}

static int finish(ef_solver* h, int out_buf, double* tau_used) {
  EF_TRY(readback(h));
  const int err = h->rb->err;
  if (err & ef::ERR_TAU_UNBOUNDED) return fail(EF_ERR_TAU_UNBOUNDED, "constant field, the time step bound is unbounded");
  if (err & ef::ERR_PROJECT) return fail(EF_ERR_INADMISSIBLE, "projected state requires rho > 0 and p > 0");
  if (err & ef::ERR_BAD_STATE) {
    const int64_t g = (int64_t)h->rb->bad;
    int64_t orig = -1;
    for (int64_t i = 0; i < h->n_local; ++i)
      if (h->gid_host[i] == g) orig = h->orig_host[i];
    h->bad_node = orig;
    return fail(EF_ERR_INADMISSIBLE, "inadmissible state at node " + std::to_string(orig));
  }
  h->cur = out_buf;
  h->tau_last = h->rb->tau;
  if (tau_used) *tau_used = h->rb->tau;
  return EF_OK;
}

static int euler_async(ef_solver* h, int32_t has_tau, double tau, double tau_max, int* out_buf) {
  const int in = h->cur, out = (h->cur + 1) % 3;
  EF_TRY(reset_flags(h));
  StageParams sp = stage_params(h, has_tau ? ef::TAU_GIVEN : ef::TAU_CFL, tau, tau_max, -1.0);
  EF_TRY(run_stage(h, h->Ubuf[in], h->Ubuf[in], h->Ubuf[out], sp));
  *out_buf = out;
  return EF_OK;
}

static int rk3_async(ef_solver* h, int32_t has_tau, double tau, double tau_max, int* out_buf) {
  const int u0 = h->cur, a = (h->cur + 1) % 3, b = (h->cur + 2) % 3;
  EF_TRY(reset_flags(h));
  StageParams s1 = stage_params(h, has_tau ? ef::TAU_GIVEN : ef::TAU_CFL, tau, tau_max, -1.0);
  EF_TRY(run_stage(h, h->Ubuf[u0], h->Ubuf[u0], h->Ubuf[a], s1));
  StageParams s2 = stage_params(h, ef::TAU_DEVICE, 0.0, 0.0, 0.25);
  EF_TRY(run_stage(h, h->Ubuf[a], h->Ubuf[u0], h->Ubuf[b], s2));
  StageParams s3 = stage_params(h, ef::TAU_DEVICE, 0.0, 0.0, 2.0 / 3.0);
  EF_TRY(run_stage(h, h->Ubuf[b], h->Ubuf[u0], h->Ubuf[a], s3));
  *out_buf = a;
  return EF_OK;
}

int ef_euler_step(ef_solver* h, int32_t has_tau, double tau, double tau_max, double* tau_used) {
  if (!h) return fail(EF_ERR_ARG, "null handle");
  cudaSetDevice(h->device);
  int out;
  EF_TRY(euler_async(h, has_tau, tau, tau_max, &out));
  return finish(h, out, tau_used);
}

int ef_ssp_rk3_step(ef_solver* h, int32_t has_tau, double tau, double tau_max, double* tau_used) {
  if (!h) return fail(EF_ERR_ARG, "null handle");
  cudaSetDevice(h->device);
  int out;
  EF_TRY(rk3_async(h, has_tau, tau, tau_max, &out));
  return finish(h, out, tau_used);
}

int ef_ssp_rk3_step_async(ef_solver* h, int32_t has_tau, double tau, double tau_max) {
  if (!h) return fail(EF_ERR_ARG, "null handle");
  cudaSetDevice(h->device);
  if (h->pending_out >= 0) h->cur = h->pending_out;  // chain on the unchecked result
  int out;
  EF_TRY(rk3_async(h, has_tau, tau, tau_max, &out));
  h->pending_out = out;
  return EF_OK;
}

int ef_sync(ef_solver* h, double* tau_used) {
  if (!h) return fail(EF_ERR_ARG, "null handle");
  cudaSetDevice(h->device);
  if (h->pending_out < 0) {
    EF_CUDA(cudaStreamSynchronize(h->st));
    if (tau_used) *tau_used = h->tau_last;
    return EF_OK;
  }
  const int out = h->pending_out;
  h->pending_out = -1;
  return finish(h, out, tau_used);
}

int64_t ef_bad_node(const ef_solver* h) { return h ? h->bad_node : -1; }

int ef_enable_timers(ef_solver* h, int32_t on) {
  if (!h) return fail(EF_ERR_ARG, "null handle");
  h->timing = on != 0;
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
  out3[1] = 0;
  out3[2] = 0;
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
    case 4:
      if (which_pass < 0 || which_pass >= std::max(1, h->passes)) return fail(EF_ERR_ARG, "bad pass");
      return slot_field(h->w.l + (size_t)which_pass * NPL);
    case 5: return node_field(h->w.eor, 1);
    case 6: return node_field(h->w.phi, 1);
    case 7: return node_field(h->Ubuf[h->cur], NV);
    case 8: return node_field(h->w.Unext, NV);
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

int ef_state_device_ptr(ef_solver* h, void** dev_ptr, int64_t* stride) {
  if (!h || !dev_ptr || !stride) return fail(EF_ERR_ARG, "null argument");
  *dev_ptr = h->Ubuf[h->cur];
  *stride = h->NP;
  return EF_OK;
}

}  // extern "C"
