// packing.cpp -- layer-pack decomposition (paper Algorithm 2), native.
//
// The search (paper Algorithm 1) packs the chain once per backward
// microbatch size and once per (forward, backward) pair, so packing sits in
// the planner's inner loop; here it is O(R) per trial pack count on prefix
// sums of the per-layer time and memory tables instead of re-summing ranges.
//
// Semantics are the reference's (`pkg/src/wrapsched/packing.py:67-186`):
//   * trial pack counts S = max(1, ceil(sum(mem) / alpha)) .. R, fewest first;
//   * for S packs, the S-1 cut points are the first layer whose accumulated
//     time exceeds k * (total / S) (k = 1..S-1) -- a layer whose running sum
//     equals a target stays in the earlier pack; when S == R the packs are
//     singletons, and all-zero times split by count (k * R / S);
//   * cuts at 0, at R or not after the previous cut are dropped (the
//     degenerate pack merges into its left neighbour);
//   * the first S whose every pack fits alpha wins.  A forward pack's memory
//     includes the checkpointed input activation x(first layer, u);
//   * greedy baseline: grow each pack while the next layer still fits.
// Errors: a single layer above alpha (LayerTooLarge, reporting the layer),
// no feasible S (Unpackable).
#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/harmony_b200.h"

namespace hm {
namespace {

struct Tables {
  int n;
  std::vector<int64_t> t, m;  // prefix sums, size n + 1
  const int64_t *ckpt;        // per-layer checkpoint bytes (forward packs) or null
  int64_t mem(int lo, int hi) const { return m[hi + 1] - m[lo] + (ckpt ? ckpt[lo] : 0); }
};

Tables make_tables(int n, const int64_t *time, const int64_t *mem, const int64_t *ckpt) {
  Tables T{n, std::vector<int64_t>(n + 1, 0), std::vector<int64_t>(n + 1, 0), ckpt};
  for (int i = 0; i < n; ++i) {
    T.t[i + 1] = T.t[i] + time[i];
    T.m[i + 1] = T.m[i] + mem[i];
  }
  return T;
}

// index of the first prefix entry (over layers 0..n-1, i.e. T.t[1..n]) whose
// value exceeds x: Python's bisect_right over the running sums
int first_above(const Tables &T, double x) {
  int lo = 0, hi = T.n;
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    if ((double)T.t[mid + 1] <= x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

}  // namespace
}  // namespace hm

extern "C" int hm_pack_layers(int32_t mode, int32_t count, const int64_t *time, const int64_t *mem,
                              const int64_t *ckpt, int64_t alpha, int32_t *first_layer, int32_t *n_packs,
                              int32_t *bad_layer) {
  if (count < 1 || !time || !mem || !first_layer || !n_packs || alpha <= 0) return HM_ERR_VALIDATION;
  const hm::Tables T = hm::make_tables(count, time, mem, ckpt);
  for (int L = 0; L < count; ++L)
    if (T.mem(L, L) > alpha) {
      if (bad_layer) *bad_layer = L;
      return HM_ERR_LAYER_TOO_LARGE;
    }
  std::vector<int> starts;
  if (mode == 1) {  // greedy: grow while the next layer fits
    for (int lo = 0; lo < count;) {
      int hi = lo;
      while (hi + 1 < count && T.mem(lo, hi + 1) <= alpha) ++hi;
      starts.push_back(lo);
      lo = hi + 1;
    }
  } else {
    const int64_t total_t = T.t[count], total_m = T.m[count];
    const int64_t s_min = std::max<int64_t>(1, (total_m + alpha - 1) / alpha);
    bool found = false;
    for (int64_t s = s_min; s <= count && !found; ++s) {
      const double target = (double)total_t / (double)s;
      starts.assign(1, 0);
      for (int64_t k = 1; k < s; ++k) {
        int64_t cut;
        if (s == count) cut = k;
        else if (total_t == 0) cut = k * count / s;
        else cut = hm::first_above(T, (double)k * target);
        if (cut > 0 && cut < count && cut > starts.back()) starts.push_back((int)cut);
      }
      found = true;
      for (size_t i = 0; i < starts.size() && found; ++i) {
        const int hi = (i + 1 < starts.size() ? starts[i + 1] : count) - 1;
        found = T.mem(starts[i], hi) <= alpha;
      }
    }
    if (!found) return HM_ERR_UNPACKABLE;
  }
  if ((int)starts.size() > *n_packs) return HM_ERR_VALIDATION;
  for (size_t i = 0; i < starts.size(); ++i) first_layer[i] = starts[i];
  *n_packs = (int32_t)starts.size();
  return HM_OK;
}
