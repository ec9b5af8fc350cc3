// ef_plan.h — host-side partition, local numbering and halo-exchange plans.
//
// Restates the reference's distribution scheme natively
// (/root/reference/pkg/src/eulerflow/exchange.py:393-445, stepper.py:163-315):
//   * rank r owns a contiguous range of the global Cuthill-McKee order
//     (even split as exchange.py:405-411 unless explicit ranges are given);
//   * its ghost layer = off-range columns of its owned rows (exchange.py:419-422);
//   * local rows = owned rows (CM order) then ghosts (ascending CM id); a
//     ghost row carries its stencil truncated to local columns
//     (stepper.py:175-181); slots of every row are sorted by CM id;
//   * row messages (alpha, R, U) go owner -> ghost copies
//     (_build_row_sends, stepper.py:270-285), limiter-factor messages send the
//     owner's l restricted to the ghost row's truncated stencil
//     (_build_l_sends, stepper.py:287-315).
// Every rank derives every plan from the same global CSR + permutation, so
// send and receive sides agree without any negotiation.  No CUDA here: the
// CPU tests exercise these plans across gloo ranks.
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
  hvec<int64_t> rcm, rsrc;            // CM column ids, source nnz index
  // halo plans, one entry per peer rank (index = peer rank, empty when none)
  std::vector<std::vector<int64_t>> send_rows, recv_rows;  // local row ids
  std::vector<std::vector<int64_t>> send_slots, recv_slots;  // local row * 256 + slot
  std::string error;
};

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
  P.ranges.resize(nranks + 1);
  if (ranges_in) {
    for (int q = 0; q <= nranks; ++q) P.ranges[q] = ranges_in[q];
    if (P.ranges[0] != 0 || P.ranges[nranks] != n) {
      P.error = "ranges must start at 0 and end at n";
      return false;
    }
  } else {  // exchange.py:405-411
    const int64_t base = n / nranks, extra = n % nranks;
    int64_t start = 0;
    for (int q = 0; q < nranks; ++q) {
      P.ranges[q] = start;
      start += base + (q < extra ? 1 : 0);
    }
    P.ranges[nranks] = n;
  }
  auto owner = [&](int64_t g) -> int {
    return (int)(std::upper_bound(P.ranges.begin(), P.ranges.end(), g) - P.ranges.begin()) - 1;
  };
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
  // ghost layer of every rank (exchange.py:419-422); none with one rank
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
  // halo plans
  P.send_rows.assign(nranks, {});
  P.recv_rows.assign(nranks, {});
  P.send_slots.assign(nranks, {});
  P.recv_slots.assign(nranks, {});
  for (size_t k = 0; k < mine.size(); ++k) {  // receives: my ghosts by owner, ascending CM id
    const int64_t g = mine[k];
    const int q = owner(g);
    const int64_t j = P.n_owned + (int64_t)k;
    P.recv_rows[q].push_back(j);
    for (int64_t t = 0; t < P.rptr[j + 1] - P.rptr[j]; ++t) P.recv_slots[q].push_back(j * 256 + t);
  }
  for (int q = 0; q < nranks; ++q) {  // sends: my owned rows that are ghosts on q
    if (q == rank) continue;
    const auto& gq = ghosts[q];
    auto lo = std::lower_bound(gq.begin(), gq.end(), P.s_lo);
    auto hi = std::lower_bound(gq.begin(), gq.end(), P.s_hi);
    for (auto it = lo; it != hi; ++it) {
      const int64_t i = *it - P.s_lo;
      P.send_rows[q].push_back(i);
      for (int64_t t = 0; t < P.rptr[i + 1] - P.rptr[i]; ++t)
        if (is_local(q, P.rcm[P.rptr[i] + t])) P.send_slots[q].push_back(i * 256 + t);
    }
  }
  return true;
}

}  // namespace ef
