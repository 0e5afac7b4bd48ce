// Host (C++) bisection engine of the hypergraph partitioner (HP) — the
// reference's connectivity-1 recursive-bisection FM (gcnpart partition.py:
// HypergraphBisection 117-199, _grow_bfs 206-240, _repair_sides 243-265,
// _fm_passes 268-323, restart selection 344-360), restated with bucketed
// gains so a pass costs O(pins·log n) instead of O(n) per move.
//
// Semantics are kept move-for-move: the FM pick is the legal unlocked vertex
// of maximal gain with the LOWEST id on ties (numpy argmax), legality is the
// reference's (other side's weight + w(v) <= cap_move, source side keeps one
// vertex), rollback to the best balanced prefix, pass stops without strict
// improvement; BFS growth visits neighbours in ascending id and jumps to the
// lowest unvisited vertex when a component is exhausted.  Random draws stay in
// Python (numpy Generator): the caller passes the BFS seed of every restart,
// so small instances reproduce the reference's assignment bit-exactly.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <set>
#include <vector>

namespace {

// vertex → nets incidence, built once per bisection node and shared
// read-only by the restarts (which run concurrently)
struct Incidence {
  std::vector<int64_t> vptr;
  std::vector<int32_t> vnets;
};

struct Engine {
  int n = 0, m = 0;
  const int64_t* nptr = nullptr;   // net → pins (local vertex ids, ascending)
  const int32_t* pins = nullptr;
  const int32_t* cost = nullptr;
  const int64_t* vptr = nullptr;   // vertex → nets (Incidence)
  const int32_t* vnets = nullptr;
  std::vector<int8_t> side;
  std::vector<int32_t> c0, c1;
  std::vector<int64_t> s0, s1;     // sum of the ids of a net's pins on side 0 / 1
  std::vector<int64_t> gain;
  int64_t cut = 0;

  static void build_incidence(int n, int m, const int64_t* nptr, const int32_t* pins, Incidence& inc) {
    inc.vptr.assign(n + 1, 0);
    for (int j = 0; j < m; ++j)
      for (int64_t e = nptr[j]; e < nptr[j + 1]; ++e) ++inc.vptr[pins[e] + 1];
    for (int v = 0; v < n; ++v) inc.vptr[v + 1] += inc.vptr[v];
    inc.vnets.assign(inc.vptr[n], 0);
    std::vector<int64_t> fill(inc.vptr.begin(), inc.vptr.end() - 1);
    for (int j = 0; j < m; ++j)
      for (int64_t e = nptr[j]; e < nptr[j + 1]; ++e) inc.vnets[fill[pins[e]]++] = j;
  }

  void init_structure(int n_, int m_, const int64_t* nptr_, const int32_t* pins_, const int32_t* cost_,
                      const Incidence& inc) {
    n = n_; m = m_; nptr = nptr_; pins = pins_; cost = cost_;
    vptr = inc.vptr.data();
    vnets = inc.vnets.data();
    c0.assign(m, 0);
    c1.assign(m, 0);
    s0.assign(m, 0);
    s1.assign(m, 0);
    gain.assign(n, 0);
  }

  int count(int j, int s) const { return s ? c1[j] : c0[j]; }
  int& countr(int j, int s) { return s ? c1[j] : c0[j]; }

  int64_t gain_of(int v) const {
    const int sv = side[v];
    int64_t g = 0;
    for (int64_t e = vptr[v]; e < vptr[v + 1]; ++e) {
      const int j = vnets[e];
      if (count(j, 1 - sv) > 0) g += cost[j];
      if (count(j, sv) > 1) g -= cost[j];
    }
    return g;
  }

  void rebuild() {
    std::fill(c0.begin(), c0.end(), 0);
    std::fill(c1.begin(), c1.end(), 0);
    std::fill(s0.begin(), s0.end(), 0);
    std::fill(s1.begin(), s1.end(), 0);
    cut = 0;
    for (int j = 0; j < m; ++j) {
      for (int64_t e = nptr[j]; e < nptr[j + 1]; ++e) {
        const int u = pins[e];
        ++countr(j, side[u]);
        (side[u] ? s1 : s0)[j] += u;
      }
      if (c0[j] > 0 && c1[j] > 0) cut += cost[j];
    }
    for (int v = 0; v < n; ++v) gain[v] = gain_of(v);
  }

  // the one pin of net j on side s (count(j, s) == 1): the side's id sum, O(1)
  int single_pin(int j, int s) const { return (int)(s ? s1[j] : s0[j]); }

  // move v to the other side, maintaining counts, cut and every pin's gain;
  // on_gain(u, old, new) is called for each changed gain of u != v, after
  // gain[u] holds the new value.
  template <class F>
  void move(int v, F&& on_gain) {
    const int sv = side[v], ov = 1 - sv;
    for (int64_t e = vptr[v]; e < vptr[v + 1]; ++e) {
      const int j = vnets[e];
      const int64_t c = cost[j];
      const int f = count(j, sv), t = count(j, ov);
      const bool was_cut = t > 0;
      if (t == 0) {
        for (int64_t q = nptr[j]; q < nptr[j + 1]; ++q) {
          const int u = pins[q];
          if (u != v) { gain[u] += c; on_gain(u, gain[u] - c, gain[u]); }
        }
      } else if (t == 1) {
        const int u = single_pin(j, ov);
        gain[u] -= c;
        on_gain(u, gain[u] + c, gain[u]);
      }
      countr(j, sv) = f - 1;
      countr(j, ov) = t + 1;
      (sv ? s1 : s0)[j] -= v;
      (sv ? s0 : s1)[j] += v;
      if (f - 1 == 0) {
        for (int64_t q = nptr[j]; q < nptr[j + 1]; ++q) {
          const int u = pins[q];
          if (u != v) { gain[u] -= c; on_gain(u, gain[u] + c, gain[u]); }
        }
      } else if (f - 1 == 1) {
        const int u = single_pin(j, sv);
        gain[u] += c;
        on_gain(u, gain[u] - c, gain[u]);
      }
      const bool is_cut = (f - 1) > 0;
      cut += c * ((int)is_cut - (int)was_cut);
    }
    side[v] = (int8_t)ov;
    gain[v] = gain_of(v);
  }
};

void grow_bfs(const Engine& eng, const double* w, int seed, int64_t min_count, double target,
              std::vector<int8_t>& side) {
  const int n = eng.n;
  std::vector<char> visited(n, 0);
  std::vector<char> expanded(eng.m, 0);  // a net's pins are all visited once one of its pins was expanded
  std::deque<int> queue;
  queue.push_back(seed);
  visited[seed] = 1;
  double acc = 0.0;
  int64_t taken = 0;
  int next_unvisited = 0;
  std::vector<int> nb;
  while (true) {
    if (queue.empty()) {
      while (next_unvisited < n && visited[next_unvisited]) ++next_unvisited;
      if (next_unvisited >= n) break;
      queue.push_back(next_unvisited);
      visited[next_unvisited] = 1;
    }
    const int v = queue.front();
    queue.pop_front();
    const double wv = w[v];
    const bool closer = std::fabs(acc + wv - target) < std::fabs(acc - target);
    if (!closer && taken >= min_count) break;
    side[v] = 0;
    acc += wv;
    ++taken;
    // unvisited neighbours in ascending id; a net already expanded adds none
    nb.clear();
    for (int64_t e = eng.vptr[v]; e < eng.vptr[v + 1]; ++e) {
      const int j = eng.vnets[e];
      if (expanded[j]) continue;
      expanded[j] = 1;
      for (int64_t q = eng.nptr[j]; q < eng.nptr[j + 1]; ++q)
        if (!visited[eng.pins[q]]) nb.push_back(eng.pins[q]);
    }
    std::sort(nb.begin(), nb.end());
    nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
    for (int u : nb) { visited[u] = 1; queue.push_back(u); }
    if (taken >= n - min_count) break;
  }
}

void repair_sides(std::vector<int8_t>& side, const double* w, int n, double cap, int64_t min_count) {
  double sw[2] = {0.0, 0.0};
  for (int v = 0; v < n; ++v) sw[side[v]] += w[v];
  while (std::max(sw[0], sw[1]) > cap) {
    const int heavy = sw[0] >= sw[1] ? 0 : 1;
    int64_t members = 0;
    for (int v = 0; v < n; ++v) members += side[v] == heavy;
    if (members <= min_count) return;
    const double diff = sw[heavy] - sw[1 - heavy];
    int best = -1;
    double best_score = 0.0;
    for (int v = 0; v < n; ++v) {
      if (side[v] != heavy) continue;
      const double score = std::fabs(w[v] - diff / 2.0);
      if (best < 0 || score < best_score) { best = v; best_score = score; }
    }
    if (!(0 < w[best] && w[best] < diff)) return;
    side[best] = (int8_t)(1 - heavy);
    sw[heavy] -= w[best];
    sw[1 - heavy] += w[best];
  }
}

// Candidate moves of one side: the side's vertices sorted by weight at the
// start of a pass, under a segment tree whose node holds the best unlocked
// vertex of its range — highest gain, then LOWER id (numpy argmax's
// tie-break).  A move of v is legal iff other + w(v) <= cap_move, i.e. iff v
// lies in the prefix of weights <= cap_move - other, so the reference's pick
// (the highest gain holding a legal vertex, its lowest legal id) is one prefix
// query; a gain change or a lock re-evaluates one leaf-to-root path.
struct MoveTree {
  const int64_t* gain = nullptr;
  int size = 1;
  std::vector<int> t;         // best vertex of the node's range, -1 if none
  std::vector<int> leaf;      // vertex -> leaf position, -1 if not on this side
  std::vector<double> wsort;  // weights in leaf order

  int pick(int a, int b) const {
    if (a < 0) return b;
    if (b < 0) return a;
    return (gain[a] > gain[b] || (gain[a] == gain[b] && a < b)) ? a : b;
  }
  void build(const std::vector<int>& verts, const double* w, int n, const int64_t* g) {
    gain = g;
    const int k = (int)verts.size();
    size = 1;
    while (size < std::max(k, 1)) size <<= 1;
    t.assign(2 * size, -1);
    leaf.assign(n, -1);
    wsort.resize(k);
    for (int i = 0; i < k; ++i) {
      t[size + i] = verts[i];
      leaf[verts[i]] = i;
      wsort[i] = w[verts[i]];
    }
    for (int x = size - 1; x >= 1; --x) t[x] = pick(t[2 * x], t[2 * x + 1]);
  }
  void refresh(int v) {
    int x = leaf[v];
    if (x < 0) return;
    x = (x + size) >> 1;
    for (; x >= 1; x >>= 1) t[x] = pick(t[2 * x], t[2 * x + 1]);
  }
  void lock(int v) {
    const int x = leaf[v];
    if (x < 0) return;
    t[size + x] = -1;
    refresh(v);
  }
  // best vertex among the leaves [0, k)
  int best_prefix(int k) const {
    int res = -1;
    int lo = size, hi = size + k;  // [lo, hi)
    while (lo < hi) {
      if (lo & 1) res = pick(res, t[lo++]);
      if (hi & 1) res = pick(res, t[--hi]);
      lo >>= 1;
      hi >>= 1;
    }
    return res;
  }
  int best_legal(double limit) const {
    const int k = (int)(std::upper_bound(wsort.begin(), wsort.end(), limit) - wsort.begin());
    return k > 0 ? best_prefix(k) : -1;
  }
};

void fm_passes(Engine& eng, const double* w, double cap, int64_t min_count, int max_passes) {
  const int n = eng.n;
  double side_w[2] = {0.0, 0.0};
  int64_t side_n[2] = {0, 0};
  double wmax = 0.0, total = 0.0;
  for (int v = 0; v < n; ++v) {
    side_w[eng.side[v]] += w[v];
    ++side_n[eng.side[v]];
    wmax = std::max(wmax, w[v]);
    total += w[v];
  }
  const double cap_move = std::max(cap, total / 2.0 + wmax);
  MoveTree mt[2];
  std::vector<char> locked(n);
  std::vector<int> moves, verts[2];
  moves.reserve(n);
  for (int pass = 0; pass < max_passes; ++pass) {
    const int64_t start_cut = eng.cut;
    int64_t best_cut = start_cut;
    size_t best_len = 0;
    moves.clear();
    std::fill(locked.begin(), locked.end(), 0);
    for (int s = 0; s < 2; ++s) verts[s].clear();
    for (int v = 0; v < n; ++v) verts[eng.side[v]].push_back(v);
    for (int s = 0; s < 2; ++s) {
      std::stable_sort(verts[s].begin(), verts[s].end(), [&](int a, int b) { return w[a] < w[b]; });
      mt[s].build(verts[s], w, n, eng.gain.data());
    }
    auto on_gain = [&](int u, int64_t, int64_t) {
      if (!locked[u]) mt[eng.side[u]].refresh(u);
    };
    while (true) {
      int pick = -1;
      int64_t pick_gain = 0;
      for (int s = 0; s < 2; ++s) {
        if (side_n[s] - 1 < 1) continue;
        const int found = mt[s].best_legal(cap_move - side_w[1 - s]);
        if (found < 0) continue;
        const int64_t g = eng.gain[found];
        if (pick < 0 || g > pick_gain || (g == pick_gain && found < pick)) {
          pick = found;
          pick_gain = g;
        }
      }
      if (pick < 0) break;
      const int v = pick;
      const int s = eng.side[v];
      locked[v] = 1;
      mt[s].lock(v);
      eng.move(v, on_gain);
      side_w[s] -= w[v];
      side_w[1 - s] += w[v];
      --side_n[s];
      ++side_n[1 - s];
      moves.push_back(v);
      const bool balanced = std::max(side_w[0], side_w[1]) <= cap && std::min(side_n[0], side_n[1]) >= min_count;
      if (balanced && eng.cut < best_cut) {
        best_cut = eng.cut;
        best_len = moves.size();
      }
    }
    auto noop = [](int, int64_t, int64_t) {};
    for (size_t i = moves.size(); i > best_len; --i) {
      const int v = moves[i - 1];
      const int s = eng.side[v];
      eng.move(v, noop);
      side_w[s] -= w[v];
      side_w[1 - s] += w[v];
      --side_n[s];
      ++side_n[1 - s];
    }
    if (std::getenv("GCNB_HP_TRACE"))
      std::fprintf(stderr, "  fm pass %d: %zu moves, best prefix %zu, cut %lld -> %lld\n", pass, moves.size(), best_len,
                   (long long)start_cut, (long long)best_cut);
    if (!(best_cut < start_cut)) break;
  }
}

}  // namespace

extern "C" {

// One bisection node of the recursive-bisection HP (partition.py:326-370).
// Hypergraph on n local vertices: net j pins pins[net_ptr[j] .. net_ptr[j+1])
// (ascending local ids, >= 2 pins), cost[j].  For each restart r a BFS grows
// side 0 from seeds[r]; sides are repaired to `cap`, FM-refined (fm_passes),
// and the best restart (balanced first, then lowest cut) is returned in
// side_out.  Returns 0, or 1 on invalid input.
int gcnb_hp_bisect(int32_t n, int32_t m, const int64_t* net_ptr, const int32_t* pins, const int32_t* cost,
                   const double* w, double cap, int64_t min_count, const int32_t* seeds, int32_t restarts,
                   int32_t fm_passes_n, int32_t refinement, int8_t* side_out, int64_t* cut_out) {
  if (n <= 0 || m < 0 || restarts < 1 || !w || !seeds || !side_out) return 1;
  for (int r = 0; r < restarts; ++r)
    if (seeds[r] < 0 || seeds[r] >= n) return 1;
  Incidence inc;
  Engine::build_incidence(n, m, net_ptr, pins, inc);
  double total = 0.0;
  for (int v = 0; v < n; ++v) total += w[v];
  // the restarts are independent (own sides, counts and gains over the shared
  // incidence): run them concurrently, then select in restart order exactly
  // as the sequential loop does (balanced first, then the strictly lower cut)
  std::vector<std::vector<int8_t>> sides(restarts);
  std::vector<int64_t> cuts(restarts, 0);
  std::vector<char> unbals(restarts, 1);
#pragma omp parallel for schedule(dynamic, 1) num_threads(restarts) if (restarts > 1)
  for (int r = 0; r < restarts; ++r) {
    Engine eng;
    eng.init_structure(n, m, net_ptr, pins, cost, inc);
    std::vector<int8_t> side(n, 1);
    auto t0 = std::chrono::steady_clock::now();
    grow_bfs(eng, w, seeds[r], min_count, total / 2.0, side);
    auto t1 = std::chrono::steady_clock::now();
    repair_sides(side, w, n, cap, min_count);
    auto t2 = std::chrono::steady_clock::now();
    eng.side = side;
    eng.rebuild();
    auto t3 = std::chrono::steady_clock::now();
    if (refinement && fm_passes_n > 0) fm_passes(eng, w, cap, min_count, fm_passes_n);
    auto t4 = std::chrono::steady_clock::now();
    if (std::getenv("GCNB_HP_TRACE")) {
      auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
      std::fprintf(stderr, "hp bisect n=%d r=%d bfs %.0f repair %.0f rebuild %.0f fm %.0f ms\n", n, r, ms(t0, t1),
                   ms(t1, t2), ms(t2, t3), ms(t3, t4));
    }
    double w0 = 0.0;
    for (int v = 0; v < n; ++v)
      if (eng.side[v] == 0) w0 += w[v];
    unbals[r] = std::max(w0, total - w0) > cap;
    cuts[r] = eng.cut;
    sides[r] = std::move(eng.side);
  }
  int best = 0;
  for (int r = 1; r < restarts; ++r)
    if (unbals[r] < unbals[best] || (unbals[r] == unbals[best] && cuts[r] < cuts[best])) best = r;
  const int64_t best_cut = cuts[best];
  std::memcpy(side_out, sides[best].data(), n);
  if (cut_out) *cut_out = best_cut;
  return 0;
}

}  // extern "C"

// k-way boundary refinement of a p-way partition under the connectivity-1 cost
// of the column-net model of a SYMMETRIC pattern (net j pins the rows of
// column j, i.e. of row j): the uncoarsening step of the multilevel
// partitioners (hp.py), after a projected coarse partition.  Vertices are
// visited in id order; each moves to the part with the largest positive gain
//   gain(v, a -> b) = #{nets j of v : cnt[j][a] == 1} - #{nets j of v : cnt[j][b] == 0}
// (lowest part id on ties) if that part stays within `cap` and `a` keeps a
// vertex.  Only strictly improving moves: the cost never increases, and the
// result is deterministic.  owner (int64) is updated in place; *moved_out /
// *gain_out report the moves and the total cost reduction.
extern "C" int gcnb_kway_refine(int64_t n, const int64_t* rp, const int64_t* ci, int64_t* owner, int32_t p,
                                const int64_t* weight, double cap, int32_t passes, int64_t* moved_out,
                                int64_t* gain_out) {
  if (n < 0 || p < 2 || p > 1024 || !rp || !ci || !owner || !weight) return 1;
  std::vector<int32_t> cnt((size_t)n * p, 0);
  std::vector<double> load(p, 0.0);
  std::vector<int64_t> members(p, 0);
  for (int64_t v = 0; v < n; ++v) {
    const int64_t a = owner[v];
    if (a < 0 || a >= p) return 1;
    load[a] += (double)weight[v];
    ++members[a];
  }
  for (int64_t j = 0; j < n; ++j)  // net j's pins: row j of the symmetric pattern
    for (int64_t e = rp[j]; e < rp[j + 1]; ++e) {
      const int64_t u = ci[e];
      if (u < 0 || u >= n) return 1;
      ++cnt[(size_t)j * p + owner[u]];
    }
  std::vector<int64_t> gain(p);
  std::vector<char> seen(p);
  int64_t moved = 0, total = 0;
  for (int pass = 0; pass < passes; ++pass) {
    int64_t moved_pass = 0;
    for (int64_t v = 0; v < n; ++v) {
      const int64_t a = owner[v];
      if (members[a] <= 1) continue;
      // candidate parts: those some net of v already touches
      std::fill(gain.begin(), gain.end(), 0);
      std::fill(seen.begin(), seen.end(), 0);
      int64_t leave = 0;  // nets where v is the only pin in a
      for (int64_t e = rp[v]; e < rp[v + 1]; ++e) {
        const int32_t* c = &cnt[(size_t)ci[e] * p];
        if (c[a] == 1) ++leave;
        for (int q = 0; q < p; ++q)
          if (c[q] > 0) seen[q] = 1;
      }
      if (!leave) continue;  // no net would lose part a: no move can gain
      int best = -1;
      int64_t best_gain = 0;
      for (int q = 0; q < p; ++q) {
        if (q == a || !seen[q] || load[q] + (double)weight[v] > cap) continue;
        int64_t join = 0;  // nets of v with no pin in q yet
        for (int64_t e = rp[v]; e < rp[v + 1]; ++e)
          if (cnt[(size_t)ci[e] * p + q] == 0) ++join;
        const int64_t g = leave - join;
        if (g > best_gain) {
          best_gain = g;
          best = q;
        }
      }
      if (best < 0) continue;
      for (int64_t e = rp[v]; e < rp[v + 1]; ++e) {
        int32_t* c = &cnt[(size_t)ci[e] * p];
        --c[a];
        ++c[best];
      }
      load[a] -= (double)weight[v];
      load[best] += (double)weight[v];
      --members[a];
      ++members[best];
      owner[v] = best;
      total += best_gain;
      ++moved_pass;
    }
    moved += moved_pass;
    if (!moved_pass) break;
  }
  if (moved_out) *moved_out = moved;
  if (gain_out) *gain_out = total;
  return 0;
}
