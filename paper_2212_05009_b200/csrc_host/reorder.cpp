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
#include <omp.h>

#include <algorithm>
#include <cstdint>
#include <utility>
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

// The contracted community graph chain_keys orders (locality.py): for labels
// lab[0..n) in 0..C-1 and the pattern (rp, ci), the edge weight between
// communities a != b is the number of nonzeros (u, v) with {lab[u], lab[v]} =
// {a, b} counted in both directions (a nonzero u->v adds 1 to (a, b) and 1 to
// (b, a)); edges sorted by (src, dst).  O(nnz + C + E log E) instead of numpy's
// unique over 2·nnz keys.  Call with ptr/adj/w == nullptr for the edge count
// (*m_out), then with arrays of C+1 / m / m entries.
extern "C" int gcnb_community_graph(int64_t n, const int64_t* rp, const int64_t* ci, const int64_t* lab, int64_t C,
                                    int64_t* m_out, int64_t* ptr, int64_t* adj, double* w) {
  if (n < 0 || C < 0 || !rp || !ci || !lab || !m_out) return 1;
  // members of each community (counting sort by label)
  std::vector<int64_t> mptr(C + 1, 0), members(n);
  for (int64_t v = 0; v < n; ++v) {
    if (lab[v] < 0 || lab[v] >= C) return 1;
    ++mptr[lab[v] + 1];
  }
  for (int64_t c = 0; c < C; ++c) mptr[c + 1] += mptr[c];
  {
    std::vector<int64_t> next(mptr.begin(), mptr.end() - 1);
    for (int64_t v = 0; v < n; ++v) members[next[lab[v]]++] = v;
  }
  // out(a -> b): nonzeros from a's rows to b's columns, per a (dense counter +
  // touched list per thread; communities in parallel, every host core)
  std::vector<std::vector<std::pair<int64_t, int64_t>>> outs(C);
  int bad = 0;
  const int nt = std::max(1, std::min(omp_get_num_procs(), 32));
#pragma omp parallel num_threads(nt)
  {
    std::vector<int64_t> cnt(C, 0), touched;
#pragma omp for schedule(dynamic, 64)
    for (int64_t a = 0; a < C; ++a) {
      touched.clear();
      for (int64_t i = mptr[a]; i < mptr[a + 1]; ++i) {
        const int64_t u = members[i];
        for (int64_t e = rp[u]; e < rp[u + 1]; ++e) {
          const int64_t v = ci[e];
          if (v < 0 || v >= n) {
            bad = 1;
            continue;
          }
          const int64_t b = lab[v];
          if (b == a) continue;
          if (cnt[b]++ == 0) touched.push_back(b);
        }
      }
      std::sort(touched.begin(), touched.end());
      auto& o = outs[a];
      o.reserve(touched.size());
      for (int64_t b : touched) {
        o.emplace_back(b, cnt[b]);
        cnt[b] = 0;
      }
    }
  }
  if (bad) return 1;
  std::vector<int64_t> optr(C + 1, 0);
  for (int64_t a = 0; a < C; ++a) optr[a + 1] = optr[a] + (int64_t)outs[a].size();
  std::vector<int64_t> odst(optr[C]), ocnt(optr[C]);
  for (int64_t a = 0; a < C; ++a) {
    int64_t k = optr[a];
    for (const auto& pr : outs[a]) {
      odst[k] = pr.first;
      ocnt[k++] = pr.second;
    }
    std::vector<std::pair<int64_t, int64_t>>().swap(outs[a]);
  }
  // symmetric weights: w(a, b) = out(a -> b) + out(b -> a); the reverse lists by a counting sort
  const int64_t E = (int64_t)odst.size();
  std::vector<int64_t> rptr(C + 1, 0), rsrc(E), rcnt(E);
  for (int64_t e = 0; e < E; ++e) ++rptr[odst[e] + 1];
  for (int64_t c = 0; c < C; ++c) rptr[c + 1] += rptr[c];
  {
    std::vector<int64_t> next(rptr.begin(), rptr.end() - 1);
    for (int64_t a = 0; a < C; ++a)  // a ascending: each reverse list comes out sorted by source
      for (int64_t e = optr[a]; e < optr[a + 1]; ++e) {
        const int64_t k = next[odst[e]]++;
        rsrc[k] = a;
        rcnt[k] = ocnt[e];
      }
  }
  // merge the two sorted lists of every community
  int64_t m = 0;
  const bool fill = ptr && adj && w;
  if (fill) ptr[0] = 0;
  for (int64_t a = 0; a < C; ++a) {
    int64_t i = optr[a], j = rptr[a];
    while (i < optr[a + 1] || j < rptr[a + 1]) {
      int64_t b;
      double x = 0.0;
      if (j >= rptr[a + 1] || (i < optr[a + 1] && odst[i] < rsrc[j])) {
        b = odst[i];
        x = (double)ocnt[i++];
      } else if (i >= optr[a + 1] || rsrc[j] < odst[i]) {
        b = rsrc[j];
        x = (double)rcnt[j++];
      } else {
        b = odst[i];
        x = (double)(ocnt[i++] + rcnt[j++]);
      }
      if (fill) {
        adj[m] = b;
        w[m] = x;
      }
      ++m;
    }
    if (fill) ptr[a + 1] = m;
  }
  *m_out = m;
  return 0;
}
