/*
 * oracle.c — TEST INFRASTRUCTURE ONLY (CPU checker and CPU baseline).
 *
 * fp64 restatement of the reference's dense/sparse arithmetic for the GCN
 * training path, used by tests/ (as the parity checker), by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
 * leg.  The product path never links or calls this file.
 *
 *   oracle_spmm_f64     gcnpart sparse.spmm (sparse.py:196-207): row i is
 *                       accumulated over its nonzeros in ascending column
 *                       (CSR) order; empty rows stay 0.  Rows are independent,
 *                       so rows are split over OpenMP threads (the per-row
 *                       accumulation order is unchanged).
 *   oracle_gemm_f64     the `@` of gcn.py:125/178 and runtime.py:299/353
 *                       (C = A·B, k-ascending accumulation per element)
 *   oracle_gemm_tn_f64  `h.T @ aggregated` of runtime.py:356 / gcn.py:176
 *                       (C = Aᵀ·B, row-ascending accumulation per element)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

void oracle_spmm_f64(int64_t n_rows, const int64_t* rp, const int64_t* ci, const double* v, const double* x,
                     int64_t d, double* y, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 256)
#endif
  for (int64_t i = 0; i < n_rows; ++i) {
    double* yi = y + i * d;
    for (int64_t j = 0; j < d; ++j) yi[j] = 0.0;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
      const double a = v[e];
      const double* xr = x + ci[e] * d;
      for (int64_t j = 0; j < d; ++j) yi[j] += a * xr[j];
    }
  }
}

void oracle_gemm_f64(int64_t n, int64_t k, int64_t m, const double* a, const double* b, double* c, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
  for (int64_t i = 0; i < n; ++i) {
    double* ci = c + i * m;
    for (int64_t j = 0; j < m; ++j) ci[j] = 0.0;
    for (int64_t t = 0; t < k; ++t) {
      const double av = a[i * k + t];
      const double* br = b + t * m;
      for (int64_t j = 0; j < m; ++j) ci[j] += av * br[j];
    }
  }
}

/* C (k×m) = Aᵀ·B with A n×k, B n×m.  Each thread owns a contiguous row range
 * and a private partial; partials are added in thread order (deterministic for
 * a fixed thread count). */
void oracle_gemm_tn_f64(int64_t n, int64_t k, int64_t m, const double* a, const double* b, double* c,
                        int nthreads) {
  int nt = 1;
#ifdef _OPENMP
  nt = nthreads > 0 ? nthreads : omp_get_max_threads();
#endif
  double* part = (double*)calloc((size_t)nt * k * m, sizeof(double));
#ifdef _OPENMP
#pragma omp parallel num_threads(nt)
#endif
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    const int64_t lo = n * tid / nt, hi = n * (tid + 1) / nt;
    double* p = part + (size_t)tid * k * m;
    for (int64_t i = lo; i < hi; ++i)
      for (int64_t t = 0; t < k; ++t) {
        const double av = a[i * k + t];
        if (av == 0.0) continue;
        const double* br = b + i * m;
        double* pr = p + t * m;
        for (int64_t j = 0; j < m; ++j) pr[j] += av * br[j];
      }
  }
  memset(c, 0, sizeof(double) * k * m);
  for (int t = 0; t < nt; ++t)
    for (int64_t j = 0; j < k * m; ++j) c[j] += part[(size_t)t * k * m + j];
  free(part);
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
