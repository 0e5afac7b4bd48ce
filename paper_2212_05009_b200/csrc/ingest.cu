// Graph ingest on the device (reference sparse.py:167-193,
// 226-234 and models.py:254-276), bit-exact with the reference's numpy:
//
//   gcnb_normalize_f64   Â = D^-1/2 (A+I) D^-1/2 (sparse.py:167-193): the A+I
//                        merge per row (a present diagonal gets +1, an absent one
//                        is inserted in column order, as from_coo's duplicate sum
//                        does), row degrees summed entry by entry in column order
//                        (np.add.at's sequential order), s = 1/sqrt(deg) with
//                        IEEE-rounded fp64 sqrt and division, v·s_i·s_j in that order;
//   gcnb_transpose_f64   Aᵀ by a stable radix sort of the column ids
//                        (sparse.py:226-234's stable argsort);
//   gcnb_induced_pattern the vertex-induced sub-pattern of a sorted batch with
//                        unit values, indexed by batch position (models.py:254-276,
//                        add_diagonal = False: the mini-batch training path).
//
// All three are setup-time code: they synchronise the stream to size outputs.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>

#include "common.cuh"

namespace gcnb {
namespace {

constexpr int IG_T = 256;

int ig_grid(long long work) {
  return (int)std::max<long long>(1, std::min<long long>((work + IG_T - 1) / IG_T, 148LL * 32));
}

struct IgTemp {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t st;
  explicit IgTemp(cudaStream_t s) : st(s) {}
  int ensure(size_t b) {
    if (b <= bytes) return 0;
    if (p) cudaFreeAsync(p, st);
    bytes = b;
    return cudaMallocAsync(&p, b, st) == cudaSuccess ? 0 : 1;
  }
  ~IgTemp() {
    if (p) cudaFreeAsync(p, st);
  }
};

// rows of A+I: length = len + (no diagonal present)
__global__ void k_tilde_len(const int64_t* __restrict__ rp, const int64_t* __restrict__ ci, long long n,
                            long long* __restrict__ len) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    bool diag = false;
    for (long long e = rp[r]; e < rp[r + 1]; ++e) diag |= ci[e] == r;
    len[r] = rp[r + 1] - rp[r] + (diag ? 0 : 1);
  }
}

// A+I row r in column order (duplicate (r, r) summed: v + 1), and the row's
// degree summed sequentially in that order
__global__ void k_tilde_fill(const int64_t* __restrict__ rp, const int64_t* __restrict__ ci,
                             const double* __restrict__ val, long long n, const long long* __restrict__ orp,
                             int64_t* __restrict__ oci, double* __restrict__ oval, double* __restrict__ deg) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    long long o = orp[r];
    bool placed = false;
    double d = 0.0;
    for (long long e = rp[r]; e < rp[r + 1]; ++e) {
      const long long c = ci[e];
      if (!placed && c > r) {
        oci[o] = r;
        oval[o] = 1.0;
        d += 1.0;
        ++o;
        placed = true;
      }
      double v = val[e];
      if (c == r) {
        v = v + 1.0;  // from_coo sums the duplicate (r, r): A's entry first, then I's
        placed = true;
      }
      oci[o] = c;
      oval[o] = v;
      d += v;
      ++o;
    }
    if (!placed) {
      oci[o] = r;
      oval[o] = 1.0;
      d += 1.0;
    }
    deg[r] = d;
  }
}

__global__ void k_inv_sqrt(const double* __restrict__ deg, long long n, double* __restrict__ s, int* __restrict__ bad) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const double d = deg[r];
    if (!(d > 0.0)) atomicMin(bad, (int)r);
    s[r] = 1.0 / sqrt(d);
  }
}

__global__ void k_scale(const long long* __restrict__ orp, const int64_t* __restrict__ oci, const double* __restrict__ s,
                        long long n, double* __restrict__ oval) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const double si = s[r];
    for (long long e = orp[r]; e < orp[r + 1]; ++e) oval[e] = oval[e] * si * s[oci[e]];
  }
}

// row id of every entry
__global__ void k_row_of(const int64_t* __restrict__ rp, long long n, int64_t* __restrict__ row_of) {
  const int lane = threadIdx.x & 31;
  for (long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; r < n;
       r += ((long long)gridDim.x * blockDim.x) >> 5)
    for (long long e = rp[r] + lane; e < rp[r + 1]; e += 32) row_of[e] = r;
}

__global__ void k_iota64(int64_t* __restrict__ x, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    x[i] = i;
}

__global__ void k_count_cols(const int64_t* __restrict__ ci, long long nnz, long long* __restrict__ cnt) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz; e += (long long)gridDim.x * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(cnt + ci[e]), 1ull);
}

__global__ void k_transpose_gather(const int64_t* __restrict__ perm, const int64_t* __restrict__ row_of,
                                   const double* __restrict__ val, long long nnz, int64_t* __restrict__ oci,
                                   double* __restrict__ oval) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nnz; i += (long long)gridDim.x * blockDim.x) {
    const long long e = perm[i];
    oci[i] = row_of[e];
    oval[i] = val[e];
  }
}

__global__ void k_batch_pos(const int64_t* __restrict__ batch, long long B, int64_t* __restrict__ pos) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < B; i += (long long)gridDim.x * blockDim.x)
    pos[batch[i]] = i;
}

__global__ void k_induced_len(const int64_t* __restrict__ rp, const int64_t* __restrict__ ci,
                              const int64_t* __restrict__ batch, long long B, const int64_t* __restrict__ pos,
                              long long* __restrict__ len) {
  const int lane = threadIdx.x & 31;
  for (long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; i < B;
       i += ((long long)gridDim.x * blockDim.x) >> 5) {
    const long long g = batch[i];
    int c = 0;
    for (long long e = rp[g] + lane; e < rp[g + 1]; e += 32) c += pos[ci[e]] >= 0;
    for (int s = 16; s > 0; s >>= 1) c += __shfl_xor_sync(0xffffffffu, c, s);
    if (lane == 0) len[i] = c;
  }
}

__global__ void k_induced_fill(const int64_t* __restrict__ rp, const int64_t* __restrict__ ci,
                               const int64_t* __restrict__ batch, long long B, const int64_t* __restrict__ pos,
                               const long long* __restrict__ orp, int64_t* __restrict__ oci, double* __restrict__ oval) {
  const int lane = threadIdx.x & 31;
  for (long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; i < B;
       i += ((long long)gridDim.x * blockDim.x) >> 5) {
    const long long g = batch[i];
    long long o = orp[i];
    for (long long e0 = rp[g]; e0 < rp[g + 1]; e0 += 32) {
      const long long e = e0 + lane;
      const long long p = e < rp[g + 1] ? pos[ci[e]] : -1;
      const unsigned b = __ballot_sync(0xffffffffu, p >= 0);
      if (p >= 0) {
        const long long at = o + __popc(b & ((1u << lane) - 1u));
        oci[at] = p;  // columns ascend with the batch ids (batch sorted, row sorted)
        oval[at] = 1.0;
      }
      o += __popc(b);
    }
  }
}

int scan_rows(const long long* len, long long n, int64_t* out_rp, cudaStream_t st, IgTemp& tmp) {
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, len, reinterpret_cast<long long*>(out_rp), n + 1, st);
  if (tmp.ensure(tb)) return set_error(GCNB_ECUDA, "ingest: out of memory");
  cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp.p, tb, len, reinterpret_cast<long long*>(out_rp), n + 1, st);
  if (e != cudaSuccess) return cuda_fail(e, "ingest: scan");
  return GCNB_OK;
}

}  // namespace
}  // namespace gcnb

using namespace gcnb;

#define IG_CUDA(x)                                                          \
  do {                                                                      \
    cudaError_t _e = (x);                                                   \
    if (_e != cudaSuccess) return cuda_fail(_e, "ingest: " #x);             \
  } while (0)

/* Pass 1 (out_ci == NULL): out_rp (n+1) and *nnz_out.  Pass 2: fill out_ci /
 * out_val (size *nnz_out) and scale.  Returns GCNB_EINVAL if a degree is <= 0. */
extern "C" int gcnb_normalize_f64(const int64_t* rp, const int64_t* ci, const double* val, int64_t n,
                                  int64_t* out_rp, int64_t* out_ci, double* out_val, int64_t* nnz_out,
                                  void* stream) {
  GCNB_REQUIRE(n >= 0 && rp && ci && val && out_rp && nnz_out, "normalize: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  IgTemp tmp(st);
  if (!out_ci) {
    long long* len = nullptr;
    IG_CUDA(cudaMallocAsync(&len, sizeof(long long) * (n + 1), st));
    IG_CUDA(cudaMemsetAsync(len + n, 0, sizeof(long long), st));
    if (n > 0) k_tilde_len<<<ig_grid(n), IG_T, 0, st>>>(rp, ci, n, len);
    if (int rc = scan_rows(len, n, out_rp, st, tmp)) return rc;
    cudaFreeAsync(len, st);
    IG_CUDA(cudaMemcpyAsync(nnz_out, out_rp + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    IG_CUDA(cudaStreamSynchronize(st));
    GCNB_AFTER_LAUNCH("normalize (sizes)");
    return GCNB_OK;
  }
  GCNB_REQUIRE(out_val, "normalize: null out_val");
  double *deg = nullptr, *s = nullptr;
  int* bad = nullptr;
  IG_CUDA(cudaMallocAsync(&deg, sizeof(double) * std::max<int64_t>(n, 1), st));
  IG_CUDA(cudaMallocAsync(&s, sizeof(double) * std::max<int64_t>(n, 1), st));
  IG_CUDA(cudaMallocAsync(&bad, sizeof(int), st));
  const int big = 0x7fffffff;
  IG_CUDA(cudaMemcpyAsync(bad, &big, sizeof(int), cudaMemcpyHostToDevice, st));
  if (n > 0) {
    k_tilde_fill<<<ig_grid(n), IG_T, 0, st>>>(rp, ci, val, n, reinterpret_cast<const long long*>(out_rp), out_ci,
                                              out_val, deg);
    k_inv_sqrt<<<ig_grid(n), IG_T, 0, st>>>(deg, n, s, bad);
    k_scale<<<ig_grid(n), IG_T, 0, st>>>(reinterpret_cast<const long long*>(out_rp), out_ci, s, n, out_val);
  }
  int bad_h = big;
  IG_CUDA(cudaMemcpyAsync(&bad_h, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  cudaFreeAsync(deg, st);
  cudaFreeAsync(s, st);
  cudaFreeAsync(bad, st);
  GCNB_AFTER_LAUNCH("normalize");
  IG_CUDA(cudaStreamSynchronize(st));
  if (bad_h != big) return set_error(GCNB_EINVAL, "row %d has non-positive degree; cannot normalize", bad_h);
  return GCNB_OK;
}

/* Aᵀ of an n_rows × n_cols CSR (nnz entries): out_rp (n_cols+1), out_ci / out_val (nnz). */
extern "C" int gcnb_transpose_f64(const int64_t* rp, const int64_t* ci, const double* val, int64_t n_rows,
                                  int64_t n_cols, int64_t* out_rp, int64_t* out_ci, double* out_val, void* stream) {
  GCNB_REQUIRE(n_rows >= 0 && n_cols >= 0 && rp && ci && val && out_rp && out_ci && out_val,
               "transpose: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  IgTemp tmp(st);
  long long nnz = 0;
  IG_CUDA(cudaMemcpyAsync(&nnz, rp + n_rows, sizeof(long long), cudaMemcpyDeviceToHost, st));
  IG_CUDA(cudaStreamSynchronize(st));
  long long* cnt = nullptr;
  IG_CUDA(cudaMallocAsync(&cnt, sizeof(long long) * (n_cols + 1), st));
  IG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(long long) * (n_cols + 1), st));
  if (nnz > 0) k_count_cols<<<ig_grid(nnz), IG_T, 0, st>>>(ci, nnz, cnt);
  if (int rc = scan_rows(cnt, n_cols, out_rp, st, tmp)) return rc;
  if (nnz > 0) {
    int64_t *row_of = nullptr, *iota = nullptr, *perm = nullptr, *keys_out = nullptr;
    IG_CUDA(cudaMallocAsync(&row_of, sizeof(int64_t) * nnz, st));
    IG_CUDA(cudaMallocAsync(&iota, sizeof(int64_t) * nnz, st));
    IG_CUDA(cudaMallocAsync(&perm, sizeof(int64_t) * nnz, st));
    IG_CUDA(cudaMallocAsync(&keys_out, sizeof(int64_t) * nnz, st));
    k_row_of<<<ig_grid((long long)n_rows * 32), IG_T, 0, st>>>(rp, n_rows, row_of);
    k_iota64<<<ig_grid(nnz), IG_T, 0, st>>>(iota, nnz);
    int bits = 1;
    while (bits < 63 && (1ll << bits) <= n_cols) ++bits;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, ci, keys_out, iota, perm, nnz, 0, bits, st);
    if (tmp.ensure(tb)) return set_error(GCNB_ECUDA, "transpose: out of memory");
    IG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, ci, keys_out, iota, perm, nnz, 0, bits, st));
    k_transpose_gather<<<ig_grid(nnz), IG_T, 0, st>>>(perm, row_of, val, nnz, out_ci, out_val);
    cudaFreeAsync(row_of, st);
    cudaFreeAsync(iota, st);
    cudaFreeAsync(perm, st);
    cudaFreeAsync(keys_out, st);
  }
  cudaFreeAsync(cnt, st);
  GCNB_AFTER_LAUNCH("transpose");
  IG_CUDA(cudaStreamSynchronize(st));
  return GCNB_OK;
}

/* Induced sub-pattern of the sorted batch (B ids): pass 1 (out_ci == NULL)
 * fills out_rp (B+1) and *nnz_out, pass 2 the columns (batch positions) and
 * unit values.  pos_scratch: n int64 entries set to -1 by the caller. */
extern "C" int gcnb_induced_pattern(const int64_t* rp, const int64_t* ci, int64_t n, const int64_t* batch,
                                    int64_t B, int64_t* pos_scratch, int64_t* out_rp, int64_t* out_ci,
                                    double* out_val, int64_t* nnz_out, void* stream) {
  GCNB_REQUIRE(n >= 0 && B >= 0 && rp && ci && batch && pos_scratch && out_rp && nnz_out,
               "induced pattern: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  IgTemp tmp(st);
  if (B > 0) k_batch_pos<<<ig_grid(B), IG_T, 0, st>>>(batch, B, pos_scratch);
  if (!out_ci) {
    long long* len = nullptr;
    IG_CUDA(cudaMallocAsync(&len, sizeof(long long) * (B + 1), st));
    IG_CUDA(cudaMemsetAsync(len + B, 0, sizeof(long long), st));
    if (B > 0) k_induced_len<<<ig_grid(B * 32), IG_T, 0, st>>>(rp, ci, batch, B, pos_scratch, len);
    if (int rc = scan_rows(len, B, out_rp, st, tmp)) return rc;
    cudaFreeAsync(len, st);
    IG_CUDA(cudaMemcpyAsync(nnz_out, out_rp + B, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    IG_CUDA(cudaStreamSynchronize(st));
    GCNB_AFTER_LAUNCH("induced pattern (sizes)");
    return GCNB_OK;
  }
  GCNB_REQUIRE(out_val, "induced pattern: null out_val");
  if (B > 0)
    k_induced_fill<<<ig_grid(B * 32), IG_T, 0, st>>>(rp, ci, batch, B, pos_scratch,
                                                    reinterpret_cast<const long long*>(out_rp), out_ci, out_val);
  GCNB_AFTER_LAUNCH("induced pattern");
  IG_CUDA(cudaStreamSynchronize(st));
  return GCNB_OK;
}
