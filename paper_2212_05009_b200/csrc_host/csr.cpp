// Host-side CSR helpers for setup (not the device path).
//
// gcnb_csr_transpose: Aᵀ by a stable counting sort — entries are placed into
// their column's bucket in row order, which is exactly the order a stable
// argsort of the column indices gives (sparse.py:226-234), in O(nnz).
#include <cstdint>
#include <vector>

extern "C" int gcnb_csr_transpose(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int64_t* ci,
                                  const double* val, int64_t* rp_t, int64_t* ci_t, double* val_t) {
  if (n_rows < 0 || n_cols < 0 || !rp || !rp_t) return 1;
  const int64_t nnz = rp[n_rows];
  for (int64_t c = 0; c <= n_cols; ++c) rp_t[c] = 0;
  for (int64_t e = 0; e < nnz; ++e) {
    if (ci[e] < 0 || ci[e] >= n_cols) return 1;
    ++rp_t[ci[e] + 1];
  }
  for (int64_t c = 0; c < n_cols; ++c) rp_t[c + 1] += rp_t[c];
  std::vector<int64_t> next(rp_t, rp_t + n_cols);
  for (int64_t r = 0; r < n_rows; ++r)
    for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
      const int64_t pos = next[ci[e]]++;
      ci_t[pos] = r;
      if (val && val_t) val_t[pos] = val[e];
    }
  return 0;
}

// out[i] = number of cum entries < x[i] (numpy searchsorted side='left'),
// parallel over queries; used by the synthetic generators' inverse-CDF draws.
#include <algorithm>

extern "C" int gcnb_searchsorted_f64(const double* cum, int64_t n, const double* x, int64_t k, int64_t* out) {
  if (n < 0 || k < 0 || (k > 0 && (!cum || !x || !out))) return 1;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < k; ++i) out[i] = std::lower_bound(cum, cum + n, x[i]) - cum;
  return 0;
}

// The column-net model of a square CSR pattern (net j pins the rows with a
// nonzero in column j, models.py:175-186) contracted onto vertex clusters
// labels[0..n) (0..C-1): net j's pins become the distinct clusters of its
// rows, ascending; nets inside one cluster are dropped.  Nets come out in
// ascending j.  O(nnz) with a per-thread cluster stamp, parallel over columns.
// Call with ptr_out == pins_out == nullptr to get the sizes (*m_out nets,
// *p_out pins), then again with arrays of those sizes.  Returns 2 when a row
// has no diagonal entry (the column-net model needs self loops).
#include <omp.h>

extern "C" int gcnb_coarse_column_nets(int64_t n, const int64_t* rp, const int64_t* ci, const int64_t* labels,
                                       int64_t C, int64_t* m_out, int64_t* p_out, int64_t* ptr_out,
                                       int64_t* pins_out) {
  if (n < 0 || C < 1 || !rp || !ci || !labels || !m_out || !p_out) return 1;
  const int64_t nnz = rp[n];
  std::vector<int64_t> cp(n + 1, 0), rows(nnz);
  for (int64_t e = 0; e < nnz; ++e) {
    if (ci[e] < 0 || ci[e] >= n) return 1;
    ++cp[ci[e] + 1];
  }
  for (int64_t c = 0; c < n; ++c) cp[c + 1] += cp[c];
  {
    std::vector<int64_t> next(cp.begin(), cp.end() - 1);
    for (int64_t r = 0; r < n; ++r) {
      bool diag = false;
      for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
        rows[next[ci[e]]++] = r;
        diag |= ci[e] == r;
      }
      if (!diag) return 2;
    }
  }
  // all host cores (torchrun sets OMP_NUM_THREADS=1 for the bench processes)
  const int nt = std::max(1, std::min(omp_get_num_procs(), 32));
  const int64_t chunk = (n + nt - 1) / std::max(nt, 1);
  std::vector<int64_t> nets_t(nt, 0), pins_t(nt, 0);
  const bool fill = ptr_out && pins_out;
  std::vector<int64_t> net_base(nt + 1, 0), pin_base(nt + 1, 0);
  for (int pass = 0; pass < (fill ? 2 : 1); ++pass) {
#pragma omp parallel num_threads(nt)
    {
      const int t = omp_get_thread_num();
      const int64_t c0 = std::min(n, t * chunk), c1 = std::min(n, c0 + chunk);
      std::vector<int64_t> stamp(C, -1), cl;
      int64_t nets = 0, pins = 0;
      int64_t nb = pass ? net_base[t] : 0, pb = pass ? pin_base[t] : 0;
      for (int64_t c = c0; c < c1; ++c) {
        cl.clear();
        for (int64_t e = cp[c]; e < cp[c + 1]; ++e) {
          const int64_t k = labels[rows[e]];
          if (stamp[k] != c) {
            stamp[k] = c;
            cl.push_back(k);
          }
        }
        if (cl.size() < 2) continue;
        if (pass) {
          std::sort(cl.begin(), cl.end());
          for (int64_t k : cl) pins_out[pb++] = k;
          ptr_out[++nb] = pb;
        }
        ++nets;
        pins += (int64_t)cl.size();
      }
      nets_t[t] = nets;
      pins_t[t] = pins;
    }
    if (!pass) {
      for (int t = 0; t < nt; ++t) {
        net_base[t + 1] = net_base[t] + nets_t[t];
        pin_base[t + 1] = pin_base[t] + pins_t[t];
      }
      *m_out = net_base[nt];
      *p_out = pin_base[nt];
      if (fill) ptr_out[0] = 0;
    }
  }
  return 0;
}
