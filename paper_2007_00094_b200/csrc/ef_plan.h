// ef_plan.h — host-side partition, local numbering and halo-exchange plans.
//
// Restates the reference's distribution scheme natively
// (/root/reference/pkg/src/eulerflow/exchange.py:52-104, stepper.py:163-315):
//   * rank r owns a contiguous range of the global Cuthill-McKee order
//     (even split as exchange.py:64-70 unless explicit ranges are given);
//   * its ghost layer = off-range columns of its owned rows (exchange.py:78-81);
//   * local rows = owned rows (CM order) then ghosts (ascending CM id); a
//     ghost row carries its stencil truncated to local columns
//     (stepper.py:175-181); slots of every row are sorted by CM id;
//   * row messages (alpha, R, U) go owner -> ghost copies
//     (_build_row_sends, stepper.py:270-285).  The reference's limiter-factor
//     messages (_build_l_sends, stepper.py:287-315) have no counterpart: the
//     edge kernel recomputes a ghost row's factors from halo'd rows (U^L, R,
//     bounds), so every message is per row.
// build_plan derives every rank's plan from the same global CSR + permutation;
// build_plan_local (per-rank setup) from the rank's own rows only: with a
// structurally symmetric pattern, owned row g is a ghost on rank q exactly when
// one of g's columns is owned by q, so send and receive sides agree without any
// negotiation either way.  No CUDA here: the CPU tests exercise these plans
// across gloo ranks.
#pragma once
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

#include "ef_par.h"

namespace ef {

struct Plan {
  int rank = 0, nranks = 1;
  int64_t n = 0, s_lo = 0, s_hi = 0, n_owned = 0, n_local = 0;
  int L = 0, standard_card = 0;
  std::vector<int64_t> ranges;        // nranks + 1
  std::vector<int64_t> cm_inv;        // CM id -> original id
  std::vector<int64_t> gid;           // local row -> CM id
  std::vector<int64_t> rptr;          // local stencils: row pointers,
  hvec<int64_t> rcm, rsrc;            // CM column ids, source nnz index (empty: identity)
  const int64_t* cols = nullptr;      // = rcm.data(), or the caller's local columns
  // halo plans, one entry per peer rank (index = peer rank, empty when none)
  std::vector<std::vector<int64_t>> send_rows, recv_rows;  // local row ids
  std::string error;
  int64_t src(int64_t k) const { return rsrc.empty() ? k : rsrc[k]; }
};

// ranges given, or the even split of exchange.py:64-70
inline bool plan_ranges(int64_t n, int nranks, const int64_t* ranges_in, Plan& P) {
  P.ranges.resize(nranks + 1);
  if (ranges_in) {
    for (int q = 0; q <= nranks; ++q) P.ranges[q] = ranges_in[q];
    if (P.ranges[0] != 0 || P.ranges[nranks] != n) {
      P.error = "ranges must start at 0 and end at n";
      return false;
    }
    for (int q = 0; q < nranks; ++q)
      if (P.ranges[q + 1] < P.ranges[q]) {
        P.error = "ranges must be non-decreasing";
        return false;
      }
  } else {
    const int64_t base = n / nranks, extra = n % nranks;
    int64_t start = 0;
    for (int q = 0; q < nranks; ++q) {
      P.ranges[q] = start;
      start += base + (q < extra ? 1 : 0);
    }
    P.ranges[nranks] = n;
  }
  return true;
}

inline int plan_owner(const Plan& P, int64_t g) {
  return (int)(std::upper_bound(P.ranges.begin(), P.ranges.end(), g) - P.ranges.begin()) - 1;
}

// Per-rank plan from the rank's own rows: owned rows
// [ranges[rank], ranges[rank+1]) with full stencils, then the ghost rows
// (ascending global id) with stencils truncated to local columns; columns are
// global ids, ascending per row.  Nothing global is read or allocated.
inline bool build_plan_local(int64_t n, int64_t n_owned, int64_t n_ghost, const int64_t* ghost_gid,
                             const int64_t* rowptr, const int64_t* col_gid, int L, int standard_card, int rank,
                             int nranks, const int64_t* ranges_in, Plan& P) {
  P.rank = rank;
  P.nranks = nranks;
  P.n = n;
  if (!ranges_in && nranks > 1) {
    P.error = "per-rank setup needs the ranges of every rank";
    return false;
  }
  if (!plan_ranges(n, nranks, ranges_in, P)) return false;
  P.s_lo = P.ranges[rank];
  P.s_hi = P.ranges[rank + 1];
  P.n_owned = P.s_hi - P.s_lo;
  if (P.n_owned != n_owned) {
    P.error = "n_owned does not match ranges[rank + 1] - ranges[rank]";
    return false;
  }
  if (L < 1 || L > 255) {
    P.error = "pad width must lie in [1, 255]";
    return false;
  }
  P.L = L;
  P.standard_card = standard_card;
  P.n_local = n_owned + n_ghost;
  P.gid.resize(P.n_local);
  for (int64_t i = 0; i < n_owned; ++i) P.gid[i] = P.s_lo + i;
  for (int64_t k = 0; k < n_ghost; ++k) {
    const int64_t g = ghost_gid[k];
    if (g < 0 || g >= n || (g >= P.s_lo && g < P.s_hi) || (k > 0 && g <= ghost_gid[k - 1])) {
      P.error = "ghost ids must be ascending, in range and not owned";
      return false;
    }
    P.gid[n_owned + k] = g;
  }
  P.rptr.assign(rowptr, rowptr + P.n_local + 1);
  P.cols = col_gid;
  // validation (parallel): row sizes, ascending local columns, owned rows reach
  // only local rows (their stencils are complete)
  std::atomic<int> bad{0};
  auto is_local = [&](int64_t c) -> bool {
    if (c >= P.s_lo && c < P.s_hi) return true;
    return std::binary_search(ghost_gid, ghost_gid + n_ghost, c);
  };
  parallel_for(P.n_local, [&](int64_t a, int64_t b, int) {
    for (int64_t i = a; i < b; ++i) {
      const int64_t lo = rowptr[i], hi = rowptr[i + 1];
      if (hi < lo || hi - lo > L) {
        bad.store(1);
        return;
      }
      for (int64_t k = lo; k < hi; ++k)
        if ((k > lo && col_gid[k] <= col_gid[k - 1]) || !is_local(col_gid[k])) {
          bad.store(2);
          return;
        }
    }
  });
  if (bad.load() == 1) {
    P.error = "row longer than the pad width (or rowptr not ascending)";
    return false;
  }
  if (bad.load() == 2) {
    P.error = "columns must be ascending local ids (owned rows need every column in the ghost layer)";
    return false;
  }
  // halo plans: receive my ghosts from their owners; send an owned row to every
  // rank owning one of its columns (pattern symmetry: then it is a ghost there)
  P.send_rows.assign(nranks, {});
  P.recv_rows.assign(nranks, {});
  for (int64_t k = 0; k < n_ghost; ++k) P.recv_rows[plan_owner(P, ghost_gid[k])].push_back(n_owned + k);
  if (nranks > 1) {
    std::vector<std::vector<std::vector<int64_t>>> part(par_threads(), std::vector<std::vector<int64_t>>(nranks));
    const int nch = parallel_for(n_owned, [&](int64_t a, int64_t b, int t) {
      auto& out = part[t];
      std::vector<int> seen;
      for (int64_t i = a; i < b; ++i) {
        seen.clear();
        for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
          const int64_t c = col_gid[k];
          if (c >= P.s_lo && c < P.s_hi) continue;
          const int q = plan_owner(P, c);
          if (std::find(seen.begin(), seen.end(), q) == seen.end()) seen.push_back(q);
        }
        for (int q : seen) out[q].push_back(i);
      }
    });
    for (int t = 0; t < nch; ++t)  // chunks are ascending row ranges in thread order
      for (int q = 0; q < nranks; ++q) P.send_rows[q].insert(P.send_rows[q].end(), part[t][q].begin(), part[t][q].end());
  }
  return true;
}

inline bool build_plan(int64_t n, const int64_t* indptr, const int64_t* indices, const int64_t* cm_perm,
                       int rank, int nranks, const int64_t* ranges_in, Plan& P) {
  P.rank = rank;
  P.nranks = nranks;
  P.n = n;
  P.cm_inv.assign(n, -1);
  for (int64_t o = 0; o < n; ++o) {
    const int64_t g = cm_perm[o];
    if (g < 0 || g >= n || P.cm_inv[g] >= 0) {
      P.error = "cm_perm is not a permutation";
      return false;
    }
    P.cm_inv[g] = o;
  }
  if (!plan_ranges(n, nranks, ranges_in, P)) return false;  // exchange.py:64-70
  auto owner = [&](int64_t g) -> int { return plan_owner(P, g); };
  // global pad width and most frequent cardinality (stepper.py:128-131)
  int64_t L = 0;
  std::vector<int64_t> hist(1, 0);
  for (int64_t o = 0; o < n; ++o) {
    const int64_t c = indptr[o + 1] - indptr[o];
    L = std::max(L, c);
    if ((int64_t)hist.size() <= c) hist.resize(c + 1, 0);
    hist[c]++;
  }
  if (L > 255) {
    P.error = "stencil cardinality above 255 is not supported";
    return false;
  }
  P.L = (int)L;
  P.standard_card = (int)(std::max_element(hist.begin(), hist.end()) - hist.begin());
  // ghost layer of every rank (exchange.py:78-81); none with one rank
  std::vector<std::vector<int64_t>> ghosts(nranks);
  for (int q = 0; q < nranks && nranks > 1; ++q) {
    const int64_t lo = P.ranges[q], hi = P.ranges[q + 1];
    std::vector<std::vector<int64_t>> part(par_threads());
    const int nch = parallel_for(hi - lo, [&](int64_t a, int64_t b, int t) {
      auto& out = part[t];
      for (int64_t g = lo + a; g < lo + b; ++g) {
        const int64_t o = P.cm_inv[g];
        for (int64_t k = indptr[o]; k < indptr[o + 1]; ++k) {
          const int64_t c = cm_perm[indices[k]];
          if (c < lo || c >= hi) out.push_back(c);
        }
      }
      std::sort(out.begin(), out.end());
      out.erase(std::unique(out.begin(), out.end()), out.end());
    });
    auto& gq = ghosts[q];
    for (int t = 0; t < nch; ++t) gq.insert(gq.end(), part[t].begin(), part[t].end());
    std::sort(gq.begin(), gq.end());
    gq.erase(std::unique(gq.begin(), gq.end()), gq.end());
  }
  auto is_local = [&](int q, int64_t c) -> bool {
    if (c >= P.ranges[q] && c < P.ranges[q + 1]) return true;
    return std::binary_search(ghosts[q].begin(), ghosts[q].end(), c);
  };
  P.s_lo = P.ranges[rank];
  P.s_hi = P.ranges[rank + 1];
  P.n_owned = P.s_hi - P.s_lo;
  const auto& mine = ghosts[rank];
  P.n_local = P.n_owned + (int64_t)mine.size();
  P.gid.resize(P.n_local);
  for (int64_t i = 0; i < P.n_owned; ++i) P.gid[i] = P.s_lo + i;
  for (size_t k = 0; k < mine.size(); ++k) P.gid[P.n_owned + k] = mine[k];
  // local stencils sorted by CM id; ghost rows truncated to local columns
  P.rptr.assign(P.n_local + 1, 0);
  parallel_for(P.n_local, [&](int64_t a, int64_t b, int) {
    for (int64_t i = a; i < b; ++i) {
      const int64_t o = P.cm_inv[P.gid[i]];
      int64_t cnt = indptr[o + 1] - indptr[o];
      if (i >= P.n_owned) {
        cnt = 0;
        for (int64_t k = indptr[o]; k < indptr[o + 1]; ++k) cnt += is_local(rank, cm_perm[indices[k]]) ? 1 : 0;
      }
      P.rptr[i + 1] = cnt;
    }
  });
  for (int64_t i = 0; i < P.n_local; ++i) P.rptr[i + 1] += P.rptr[i];
  P.rcm.resize(P.rptr[P.n_local]);
  P.rsrc.resize(P.rptr[P.n_local]);
  parallel_for(P.n_local, [&](int64_t a, int64_t b, int) {
    std::vector<std::pair<int64_t, int64_t>> tmp;
    for (int64_t i = a; i < b; ++i) {
      const int64_t o = P.cm_inv[P.gid[i]];
      tmp.clear();
      for (int64_t k = indptr[o]; k < indptr[o + 1]; ++k) {
        const int64_t c = cm_perm[indices[k]];
        if (i >= P.n_owned && !is_local(rank, c)) continue;
        tmp.emplace_back(c, k);
      }
      std::sort(tmp.begin(), tmp.end());
      int64_t q = P.rptr[i];
      for (auto& t : tmp) {
        P.rcm[q] = t.first;
        P.rsrc[q] = t.second;
        ++q;
      }
    }
  });
  P.cols = P.rcm.data();
  // halo plans (row messages only: every exchanged quantity is per row)
  P.send_rows.assign(nranks, {});
  P.recv_rows.assign(nranks, {});
  for (size_t k = 0; k < mine.size(); ++k)  // receives: my ghosts by owner, ascending CM id
    P.recv_rows[owner(mine[k])].push_back(P.n_owned + (int64_t)k);
  for (int q = 0; q < nranks; ++q) {  // sends: my owned rows that are ghosts on q
    if (q == rank) continue;
    const auto& gq = ghosts[q];
    auto lo = std::lower_bound(gq.begin(), gq.end(), P.s_lo);
    auto hi = std::lower_bound(gq.begin(), gq.end(), P.s_hi);
    for (auto it = lo; it != hi; ++it) P.send_rows[q].push_back(*it - P.s_lo);
  }
  return true;
}

}  // namespace ef
