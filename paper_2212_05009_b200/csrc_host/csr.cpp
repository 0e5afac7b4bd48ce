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
