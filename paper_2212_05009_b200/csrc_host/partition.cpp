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
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <set>
#include <vector>

namespace {

struct Engine {
  int n = 0, m = 0;
  const int64_t* nptr = nullptr;   // net → pins (local vertex ids, ascending)
  const int32_t* pins = nullptr;
  const int32_t* cost = nullptr;
  std::vector<int64_t> vptr;       // vertex → nets
  std::vector<int32_t> vnets;
  std::vector<int8_t> side;
  std::vector<int32_t> c0, c1;
  std::vector<int64_t> gain;
  int64_t cut = 0;

  void init_structure(int n_, int m_, const int64_t* nptr_, const int32_t* pins_, const int32_t* cost_) {
    n = n_; m = m_; nptr = nptr_; pins = pins_; cost = cost_;
    vptr.assign(n + 1, 0);
    for (int j = 0; j < m; ++j)
      for (int64_t e = nptr[j]; e < nptr[j + 1]; ++e) ++vptr[pins[e] + 1];
    for (int v = 0; v < n; ++v) vptr[v + 1] += vptr[v];
    vnets.assign(vptr[n], 0);
    std::vector<int64_t> fill(vptr.begin(), vptr.end() - 1);
    for (int j = 0; j < m; ++j)
      for (int64_t e = nptr[j]; e < nptr[j + 1]; ++e) vnets[fill[pins[e]]++] = j;
    c0.assign(m, 0);
    c1.assign(m, 0);
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
    cut = 0;
    for (int j = 0; j < m; ++j) {
      for (int64_t e = nptr[j]; e < nptr[j + 1]; ++e) ++countr(j, side[pins[e]]);
      if (c0[j] > 0 && c1[j] > 0) cut += cost[j];
    }
    for (int v = 0; v < n; ++v) gain[v] = gain_of(v);
  }

  int single_pin_on(int j, int s, int exclude) const {
    for (int64_t e = nptr[j]; e < nptr[j + 1]; ++e)
      if (pins[e] != exclude && side[pins[e]] == s) return pins[e];
    return -1;
  }

  // move v to the other side, maintaining counts, cut and every pin's gain;
  // on_gain(u, old, new) is called for each changed gain of u != v.
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
          if (u != v) { on_gain(u, gain[u], gain[u] + c); gain[u] += c; }
        }
      } else if (t == 1) {
        const int u = single_pin_on(j, ov, v);
        on_gain(u, gain[u], gain[u] - c);
        gain[u] -= c;
      }
      countr(j, sv) = f - 1;
      countr(j, ov) = t + 1;
      if (f - 1 == 0) {
        for (int64_t q = nptr[j]; q < nptr[j + 1]; ++q) {
          const int u = pins[q];
          if (u != v) { on_gain(u, gain[u], gain[u] - c); gain[u] -= c; }
        }
      } else if (f - 1 == 1) {
        const int u = single_pin_on(j, sv, v);
        on_gain(u, gain[u], gain[u] + c);
        gain[u] += c;
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
    nb.clear();
    for (int64_t e = eng.vptr[v]; e < eng.vptr[v + 1]; ++e) {
      const int j = eng.vnets[e];
      for (int64_t q = eng.nptr[j]; q < eng.nptr[j + 1]; ++q)
        if (eng.pins[q] != v) nb.push_back(eng.pins[q]);
    }
    std::sort(nb.begin(), nb.end());
    nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
    for (int u : nb)
      if (!visited[u]) { visited[u] = 1; queue.push_back(u); }
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

// Gain buckets per side with ids ordered ascending (lowest-id tie-break).
struct Buckets {
  int64_t off = 0;
  std::vector<std::set<int>> b[2];
  int64_t top[2] = {-1, -1};

  void reset(int64_t max_abs) {
    off = max_abs;
    for (int s = 0; s < 2; ++s) {
      b[s].assign(2 * max_abs + 1, std::set<int>());
      top[s] = -1;
    }
  }
  void insert(int s, int64_t g, int v) {
    const int64_t i = g + off;
    b[s][i].insert(v);
    if (i > top[s]) top[s] = i;
  }
  void erase(int s, int64_t g, int v) { b[s][g + off].erase(v); }
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
  int64_t max_abs = 1;
  for (int v = 0; v < n; ++v) {
    int64_t s = 0;
    for (int64_t e = eng.vptr[v]; e < eng.vptr[v + 1]; ++e) s += eng.cost[eng.vnets[e]];
    max_abs = std::max(max_abs, s);
  }
  Buckets bk;
  std::vector<char> locked(n);
  std::vector<int> moves;
  moves.reserve(n);
  for (int pass = 0; pass < max_passes; ++pass) {
    const int64_t start_cut = eng.cut;
    int64_t best_cut = start_cut;
    size_t best_len = 0;
    moves.clear();
    std::fill(locked.begin(), locked.end(), 0);
    bk.reset(max_abs);
    // unlocked weights per side: a side whose lightest unlocked vertex cannot
    // move under cap_move is skipped in O(1) instead of scanning its buckets
    std::multiset<double> wset[2];
    for (int v = 0; v < n; ++v) {
      bk.insert(eng.side[v], eng.gain[v], v);
      wset[eng.side[v]].insert(w[v]);
    }
    auto on_gain = [&](int u, int64_t g_old, int64_t g_new) {
      if (locked[u]) return;
      bk.erase(eng.side[u], g_old, u);
      bk.insert(eng.side[u], g_new, u);
    };
    while (true) {
      int pick = -1;
      int64_t pick_gain = 0;
      for (int s = 0; s < 2; ++s) {
        if (side_n[s] - 1 < 1) continue;
        const double other = side_w[1 - s];
        if (wset[s].empty() || other + *wset[s].begin() > cap_move) continue;
        for (int64_t i = bk.top[s]; i >= 0; --i) {
          auto& set = bk.b[s][i];
          if (set.empty()) {
            if (i == bk.top[s]) bk.top[s] = i - 1;
            continue;
          }
          int found = -1;
          for (int v : set)
            if (other + w[v] <= cap_move) { found = v; break; }
          if (found >= 0) {
            const int64_t g = i - bk.off;
            if (pick < 0 || g > pick_gain || (g == pick_gain && found < pick)) {
              pick = found;
              pick_gain = g;
            }
            break;
          }
        }
      }
      if (pick < 0) break;
      const int v = pick;
      const int s = eng.side[v];
      bk.erase(s, eng.gain[v], v);
      wset[s].erase(wset[s].find(w[v]));
      locked[v] = 1;
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
  Engine eng;
  eng.init_structure(n, m, net_ptr, pins, cost);
  double total = 0.0;
  for (int v = 0; v < n; ++v) total += w[v];
  bool have = false;
  bool best_unbal = true;
  int64_t best_cut = 0;
  std::vector<int8_t> best_side;
  for (int r = 0; r < restarts; ++r) {
    std::vector<int8_t> side(n, 1);
    if (seeds[r] < 0 || seeds[r] >= n) return 1;
    grow_bfs(eng, w, seeds[r], min_count, total / 2.0, side);
    repair_sides(side, w, n, cap, min_count);
    eng.side = side;
    eng.rebuild();
    if (refinement && fm_passes_n > 0) fm_passes(eng, w, cap, min_count, fm_passes_n);
    double w0 = 0.0;
    for (int v = 0; v < n; ++v)
      if (eng.side[v] == 0) w0 += w[v];
    const bool unbal = std::max(w0, total - w0) > cap;
    if (!have || (unbal < best_unbal) || (unbal == best_unbal && eng.cut < best_cut)) {
      have = true;
      best_unbal = unbal;
      best_cut = eng.cut;
      best_side = eng.side;
    }
  }
  std::memcpy(side_out, best_side.data(), n);
  if (cut_out) *cut_out = best_cut;
  return 0;
}

}  // extern "C"
