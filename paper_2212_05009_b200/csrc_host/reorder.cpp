// Host-side locality ordering for the device layout.
//
// Deterministic asynchronous label propagation over a symmetric pattern:
// every vertex (in id order) adopts the label held by most of its neighbours
// (ties: the smallest label; its own label counts once), for a fixed number
// of sweeps.  Rows are then laid out community by community, so a tile of
// consecutive rows gathers mostly rows of its own community and those rows sit
// next to each other in the feature block — the gathers hit L2 instead of HBM.
// This is a layout choice only: global vertex ids, plans and results are
// unchanged.
#include <algorithm>
#include <cstdint>
#include <vector>

extern "C" int gcnb_label_propagation(int64_t n, const int64_t* rp, const int64_t* ci, int32_t sweeps,
                                      int64_t* labels) {
  if (n < 0 || !rp || !ci || !labels || sweeps < 0) return 1;
  for (int64_t v = 0; v < n; ++v) labels[v] = v;
  std::vector<int64_t> nb;
  for (int s = 0; s < sweeps; ++s) {
    int64_t changed = 0;
    for (int64_t v = 0; v < n; ++v) {
      nb.clear();
      nb.push_back(labels[v]);
      for (int64_t e = rp[v]; e < rp[v + 1]; ++e)
        if (ci[e] != v) nb.push_back(labels[ci[e]]);
      std::sort(nb.begin(), nb.end());
      int64_t best = labels[v], best_cnt = 0;
      for (size_t i = 0; i < nb.size();) {
        size_t j = i;
        while (j < nb.size() && nb[j] == nb[i]) ++j;
        const int64_t cnt = (int64_t)(j - i);
        if (cnt > best_cnt) {  // ascending scan: ties keep the smaller label
          best_cnt = cnt;
          best = nb[i];
        }
        i = j;
      }
      if (best != labels[v]) {
        labels[v] = best;
        ++changed;
      }
    }
    if (changed == 0) break;
  }
  return 0;
}
