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
  // O(deg) label histogram per vertex: counts in a dense array, reset through
  // the list of labels touched (the winner is the most frequent label, ties
  // to the smallest — the same choice as an ascending scan of the sorted list)
  std::vector<int32_t> cnt(n, 0);
  std::vector<int64_t> touched;
  for (int s = 0; s < sweeps; ++s) {
    int64_t changed = 0;
    for (int64_t v = 0; v < n; ++v) {
      touched.clear();
      touched.push_back(labels[v]);
      cnt[labels[v]] = 1;
      for (int64_t e = rp[v]; e < rp[v + 1]; ++e) {
        const int64_t u = ci[e];
        if (u == v) continue;
        const int64_t l = labels[u];
        if (cnt[l]++ == 0) touched.push_back(l);
      }
      int64_t best = labels[v];
      int32_t best_cnt = 0;
      for (const int64_t l : touched) {
        if (cnt[l] > best_cnt || (cnt[l] == best_cnt && l < best)) {
          best_cnt = cnt[l];
          best = l;
        }
        cnt[l] = 0;
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

// Chain order of the communities: a maximum-adjacency (Prim-like) ordering of
// the contracted community graph.  Starting from `start`, repeatedly place the
// unplaced community with the largest total edge weight to the already-placed
// set (ties: lowest id; disconnected remainder: lowest unplaced id).  Laying
// communities out in this order puts the communities a row's off-community
// neighbours live in next to it, so those gathers also stay in L2's reuse
// window.  rank_out[c] = position of community c in the chain.
#include <queue>
#include <utility>

extern "C" int gcnb_chain_order(int64_t C, const int64_t* ptr, const int64_t* adj, const double* w, int64_t start,
                                int64_t* rank_out) {
  if (C < 0 || !ptr || !rank_out || (C > 0 && (start < 0 || start >= C))) return 1;
  std::vector<double> conn(C, 0.0);
  std::vector<char> placed(C, 0);
  using Item = std::pair<double, int64_t>;  // (weight, -id): max weight, then lowest id
  std::priority_queue<Item> heap;
  int64_t next = 0, scan = 0;
  if (C > 0) heap.push({0.0, -start});
  while (next < C) {
    if (heap.empty()) {
      while (placed[scan]) ++scan;
      heap.push({0.0, -scan});
    }
    const Item it = heap.top();
    heap.pop();
    const int64_t v = -it.second;
    if (placed[v] || it.first != conn[v]) continue;  // stale entry
    placed[v] = 1;
    rank_out[v] = next++;
    for (int64_t e = ptr[v]; e < ptr[v + 1]; ++e) {
      const int64_t u = adj[e];
      if (u < 0 || u >= C) return 1;
      if (!placed[u]) {
        conn[u] += w[e];
        heap.push({conn[u], -u});
      }
    }
  }
  return 0;
}
