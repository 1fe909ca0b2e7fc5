// brute.cpp — exhaustive minimum-footprint search for small conflict graphs
// (host code; smartpool.py:167-221).  The reference's test oracle A2 runs it
// on 200 random graphs per test; in Python the DFS dominates the test.
//
// Same search, same order: variables in placement order, offsets drawn from
// the sorted subset sums of the sizes, candidate loop cut at
// off + size >= best, first complete layout at or below `lower` ends it.
#include <stdint.h>

#include <vector>

#include "../../include/memplan_b200.h"

namespace {

struct Search {
  int n;
  const int64_t *size;
  const int64_t *nb_off;
  const int32_t *nb;
  const int64_t *cand;
  int64_t ncand, lower, best;
  std::vector<int64_t> off;

  bool dfs(int k, int64_t cur) {
    if (k == n) {
      best = cur;
      return best <= lower;
    }
    const int64_t sk = size[k];
    for (int64_t c = 0; c < ncand; c++) {
      const int64_t o = cand[c];
      if (o + sk >= best) break;
      bool ok = true;
      for (int64_t e = nb_off[k]; e < nb_off[k + 1]; e++) {
        const int j = nb[e];
        if (o < off[j] + size[j] && off[j] < o + sk) { ok = false; break; }
      }
      if (!ok) continue;
      off[k] = o;
      if (dfs(k + 1, cur > o + sk ? cur : o + sk)) return true;
    }
    return false;
  }
};

}  // namespace

extern "C" int mp_brute_force_footprint(int32_t n, const int64_t *size, const int64_t *nb_off, const int32_t *nb,
                                        const int64_t *cand, int64_t ncand, int64_t lower, int64_t *best) {
  Search s{n, size, nb_off, nb, cand, ncand, lower, *best, std::vector<int64_t>(n > 0 ? n : 1, 0)};
  s.dfs(0, 0);
  *best = s.best;
  return MP_OK;
}
