// Global minimum 2-cut (Stoer-Wagner maximum-adjacency phases) on the host: the
// native twin of the reference's only compiled component, hetplan's
// ``min_cut_kernel`` (_mincut_c.pyx:16-82; Python twin _mincut_py.py:19-73).
// Same arithmetic in the same order and the same tie rules (smallest lexicographic
// rank wins, merged supervertices keep the smallest rank of their members), so cut
// weights and sides are bit-identical to the reference's backends.
#include "zb_internal.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

using namespace zb;

extern "C" int zb_min_cut(const double* weights, int64_t n, const int64_t* lexrank, double* cut_out,
                          int64_t* side_out, int64_t* side_len) {
  if (n < 2) return set_error(ZB_ERR_INVALID, "min cut needs >= 2 vertices");
  if (!weights || !lexrank || !cut_out || !side_out || !side_len)
    return set_error(ZB_ERR_INVALID, "min_cut: NULL argument");
  std::vector<double> w(weights, weights + n * n);
  std::vector<int64_t> minid(lexrank, lexrank + n);
  std::vector<uint8_t> active(n, 1), in_a(n, 0);
  std::vector<double> conn(n, 0.0);
  std::vector<std::vector<int64_t>> members(n);
  for (int64_t i = 0; i < n; ++i) members[i].push_back(i);
  double best_w = INFINITY;
  std::vector<int64_t> best_side;
  int64_t n_active = n;
  while (n_active > 1) {
    // phase start: active slot with the smallest lexicographic rank
    int64_t start = -1;
    for (int64_t i = 0; i < n; ++i)
      if (active[i] && (start < 0 || minid[i] < minid[start])) start = i;
    for (int64_t i = 0; i < n; ++i) {
      in_a[i] = 0;
      conn[i] = w[start * n + i];
    }
    in_a[start] = 1;
    int64_t prev = start, last = start;
    double cut_val = 0.0;
    for (int64_t step = 0; step < n_active - 1; ++step) {
      int64_t sel = -1;
      double top = 0.0;
      for (int64_t j = 0; j < n; ++j)
        if (active[j] && !in_a[j])
          if (sel < 0 || conn[j] > top || (conn[j] == top && minid[j] < minid[sel])) {
            sel = j;
            top = conn[j];
          }
      cut_val = conn[sel];
      prev = last;
      last = sel;
      in_a[sel] = 1;
      for (int64_t j = 0; j < n; ++j)
        if (active[j] && !in_a[j]) conn[j] += w[sel * n + j];
    }
    if (cut_val < best_w) {
      best_w = cut_val;
      best_side = members[last];
    }
    // merge `last` into `prev` (the second-to-last vertex of the phase)
    for (int64_t j = 0; j < n; ++j) w[prev * n + j] += w[last * n + j];
    w[prev * n + prev] = 0.0;
    w[prev * n + last] = 0.0;
    for (int64_t j = 0; j < n; ++j) w[j * n + prev] = w[prev * n + j];
    active[last] = 0;
    members[prev].insert(members[prev].end(), members[last].begin(), members[last].end());
    if (minid[last] < minid[prev]) minid[prev] = minid[last];
    --n_active;
  }
  std::sort(best_side.begin(), best_side.end());
  *cut_out = best_w;
  *side_len = (int64_t)best_side.size();
  std::copy(best_side.begin(), best_side.end(), side_out);
  return 0;
}
