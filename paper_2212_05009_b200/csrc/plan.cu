// Device communication plan and rank layout builder: the
// reference's build_comm_plan (comm.py:59-93) and the per-rank split of
// scatter (runtime.py:203-275), bit-exact with both, as sorts and scans over
// the nonzeros instead of per-row Python loops.
//
//   gcnb_plan_build   all ranks' plan at once: every cut nonzero (r, c) with
//                     owner[r] != owner[c] becomes the key
//                     (consumer = owner[r], sender = owner[c], c); one radix
//                     sort + unique gives, per (consumer, sender) block, the
//                     sorted distinct columns = send[sender][consumer]
//                     (comm.py:79-92) — and, per consumer, its halo in the
//                     reference's positional order (sender asc, then id asc);
//                     also every rank's own rows (ascending id) and their
//                     positions;
//   gcnb_layout_fill  one rank's extended CSR over [own rows | halo] in a
//                     given row order (values kept fp64 for the host views),
//                     each row's entries sorted by extended column when the
//                     rank has a halo (layout.py:build_op_layout), plus the
//                     interior / boundary row lists.
//
// Sizes that the caller must know before allocating (unique key count, the
// rank's nonzero count) come back through small host-visible outputs; the
// builder is setup-time code (never inside a captured epoch).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>

#include "common.cuh"

namespace gcnb {
namespace {

constexpr int PL_T = 256;

// Scratch for CUB: stream-ordered allocation, freed on the same stream.
struct Temp {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t st;
  explicit Temp(cudaStream_t s) : st(s) {}
  int ensure(size_t b) {
    if (b <= bytes) return 0;
    if (p) cudaFreeAsync(p, st);
    bytes = b;
    return cudaMallocAsync(&p, b, st) == cudaSuccess ? 0 : 1;
  }
  ~Temp() {
    if (p) cudaFreeAsync(p, st);
  }
};

template <typename T>
int dmalloc(T** p, size_t n, cudaStream_t st) {
  return cudaMallocAsync(reinterpret_cast<void**>(p), std::max<size_t>(n, 1) * sizeof(T), st) == cudaSuccess ? 0 : 1;
}

constexpr int KEY_RANK_BITS = 7;                       // p <= 64 (GCNB_MAX_PEERS) fits 7 bits with room
constexpr int KEY_COL_BITS = 64 - 2 * KEY_RANK_BITS - 1;  // 49 bits of column id

__device__ __forceinline__ unsigned long long cut_key(int consumer, int sender, long long c) {
  return ((unsigned long long)consumer << (KEY_COL_BITS + KEY_RANK_BITS)) |
         ((unsigned long long)sender << KEY_COL_BITS) | (unsigned long long)c;
}

// cut nonzeros per row (warp per row)
__global__ void k_cut_count(const int64_t* __restrict__ rp, const int64_t* __restrict__ ci,
                            const int* __restrict__ owner, long long n_rows, long long* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  for (long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; r < n_rows;
       r += ((long long)gridDim.x * blockDim.x) >> 5) {
    const int o = owner[r];
    int c = 0;
    for (long long e = rp[r] + lane; e < rp[r + 1]; e += 32) c += owner[ci[e]] != o;
    for (int s = 16; s > 0; s >>= 1) c += __shfl_xor_sync(0xffffffffu, c, s);
    if (lane == 0) cnt[r] = c;
  }
}

__global__ void k_cut_emit(const int64_t* __restrict__ rp, const int64_t* __restrict__ ci,
                           const int* __restrict__ owner, long long n_rows, const long long* __restrict__ off,
                           unsigned long long* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  for (long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; r < n_rows;
       r += ((long long)gridDim.x * blockDim.x) >> 5) {
    const int o = owner[r];
    long long base = off[r];
    for (long long e0 = rp[r]; e0 < rp[r + 1]; e0 += 32) {
      const long long e = e0 + lane;
      const bool ok = e < rp[r + 1];
      const long long c = ok ? ci[e] : 0;
      const bool cut = ok && owner[c] != o;
      const unsigned b = __ballot_sync(0xffffffffu, cut);
      if (cut) keys[base + __popc(b & ((1u << lane) - 1u))] = cut_key(o, owner[c], c);
      base += __popc(b);
    }
  }
}

// block [start, end) of every (consumer, sender) pair in the sorted unique keys
__global__ void k_pair_bounds(const unsigned long long* __restrict__ keys, long long n_keys, int p,
                              long long* __restrict__ bounds) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > p * p) return;
  // first key >= pair i's smallest key (i == p*p: the end)
  const unsigned long long lo = i == p * p ? ~0ull : cut_key(i / p, i % p, 0);
  long long a = 0, b = n_keys;
  while (a < b) {
    const long long mid = (a + b) >> 1;
    if (keys[mid] < lo) a = mid + 1;
    else b = mid;
  }
  bounds[i] = i == p * p ? n_keys : a;
}

// (row << 32 | extended column) keys of a layout's entries, warp per row, and
// their positions: one radix sort of them orders every row by column.
__global__ void k_row_col_keys(const long long* __restrict__ row_ptr, int n_rows, const int* __restrict__ col,
                               unsigned long long* __restrict__ key, int* __restrict__ pos) {
  const int lane = threadIdx.x & 31;
  for (long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; r < n_rows;
       r += ((long long)gridDim.x * blockDim.x) >> 5) {
    const long long e0 = row_ptr[r], e1 = row_ptr[r + 1];
    for (long long e = e0 + lane; e < e1; e += 32) {
      key[e] = ((unsigned long long)r << 32) | (unsigned int)col[e];
      pos[e] = (int)e;
    }
  }
}

__global__ void k_key_col(const unsigned long long* __restrict__ key, long long n, int* __restrict__ col) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    col[i] = (int)(unsigned int)(key[i] & 0xffffffffull);
}

__global__ void k_iota(int* __restrict__ x, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    x[i] = (int)i;
}

// rank_ptr from the sorted owners (every rank q's first index, empty ranks included)
__global__ void k_rank_rows(const int* __restrict__ owner_sorted, long long n, int p, int* __restrict__ rank_ptr) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int o = owner_sorted[i];
    if (i == 0 || owner_sorted[i - 1] != o)
      for (int q = i == 0 ? 0 : owner_sorted[i - 1] + 1; q <= o; ++q) rank_ptr[q] = (int)i;
    if (i == n - 1)
      for (int q = o + 1; q <= p; ++q) rank_ptr[q] = (int)n;
  }
}

__global__ void k_localpos(const int* __restrict__ owner_sorted, const int* __restrict__ rows_sorted, long long n,
                           const int* __restrict__ rank_ptr, int* __restrict__ localpos) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    localpos[rows_sorted[i]] = (int)(i - rank_ptr[owner_sorted[i]]);
}

int grid_for(long long work, int per_block) {
  return (int)std::max<long long>(1, std::min<long long>((work + per_block - 1) / per_block, 148LL * 32));
}

// extended column of every column id for rank m: own rows -> layout position,
// halo columns -> n_own + position in the consumer block, others untouched
__global__ void k_colmap_own(const int* __restrict__ layout_rows, int n_own, int* __restrict__ colmap) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_own; i += gridDim.x * blockDim.x)
    colmap[layout_rows[i]] = i;
}

__global__ void k_colmap_halo(const unsigned long long* __restrict__ keys, long long k0, long long n_halo, int n_own,
                              int* __restrict__ colmap) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_halo;
       i += (long long)gridDim.x * blockDim.x)
    colmap[keys[k0 + i] & ((1ull << KEY_COL_BITS) - 1ull)] = n_own + (int)i;
}

__global__ void k_row_len(const int64_t* __restrict__ rp, const int* __restrict__ layout_rows, int n_own,
                          long long* __restrict__ len) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_own; i += gridDim.x * blockDim.x) {
    const int r = layout_rows[i];
    len[i] = rp[r + 1] - rp[r];
  }
}

// warp per layout row: entries with extended columns (CSR order), halo flag
__global__ void k_fill(const int64_t* __restrict__ rp, const int64_t* __restrict__ ci, const double* __restrict__ val,
                       const int* __restrict__ layout_rows, int n_own, const long long* __restrict__ out_ptr,
                       const int* __restrict__ colmap, int* __restrict__ ext_col, double* __restrict__ out_val,
                       int* __restrict__ has_halo) {
  const int lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_own; i += (gridDim.x * blockDim.x) >> 5) {
    const int r = layout_rows[i];
    const long long s = rp[r], e = rp[r + 1], o = out_ptr[i];
    int halo = 0;
    for (long long k = s + lane; k < e; k += 32) {
      const int x = colmap[ci[k]];
      ext_col[o + (k - s)] = x;
      out_val[o + (k - s)] = val[k];
      halo |= x >= n_own;
    }
    halo = __any_sync(0xffffffffu, halo);
    if (lane == 0) has_halo[i] = halo;
  }
}

__global__ void k_to_i32(const long long* __restrict__ x, long long n, int* __restrict__ y) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = (int)x[i];
}

__global__ void k_gather_val(const int* __restrict__ perm, const double* __restrict__ v, long long n,
                             double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = v[perm[i]];
}

}  // namespace
}  // namespace gcnb

using namespace gcnb;

#define PL_CUDA(x)                                                         \
  do {                                                                     \
    cudaError_t _e = (x);                                                  \
    if (_e != cudaSuccess) return cuda_fail(_e, "plan build: " #x);        \
  } while (0)

/* See include/gcnb.h. */
extern "C" int gcnb_plan_build(const int64_t* rp, const int64_t* ci, int64_t n, const int32_t* owner, int32_t p,
                               uint64_t** keys_out, int64_t* n_keys_out, int64_t* pair_bounds, int32_t* rows_sorted,
                               int32_t* rank_ptr, int32_t* localpos, void* stream) {
  GCNB_REQUIRE(n >= 0 && n < (1ll << 31) && p >= 1 && p <= GCNB_MAX_PEERS, "plan build: bad sizes (n %lld, p %d)",
               (long long)n, p);
  GCNB_REQUIRE(rp && ci && owner && keys_out && n_keys_out && pair_bounds && rows_sorted && rank_ptr && localpos,
               "plan build: null argument");
  cudaStream_t st = (cudaStream_t)stream;
  Temp tmp(st);
  // 1. every rank's own rows, ascending (stable radix sort of (owner, v))
  int *own_sorted = nullptr, *iota = nullptr;
  if (dmalloc(&own_sorted, n, st) || dmalloc(&iota, n, st)) return set_error(GCNB_ECUDA, "plan build: out of memory");
  if (n > 0) {
    k_iota<<<grid_for(n, PL_T), PL_T, 0, st>>>(iota, n);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, owner, own_sorted, iota, rows_sorted, (int)n, 0, KEY_RANK_BITS, st);
    if (tmp.ensure(tb)) return set_error(GCNB_ECUDA, "plan build: out of memory");
    PL_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, owner, own_sorted, iota, rows_sorted, (int)n, 0,
                                            KEY_RANK_BITS, st));
    k_rank_rows<<<grid_for(n, PL_T), PL_T, 0, st>>>(own_sorted, n, p, rank_ptr);
    k_localpos<<<grid_for(n, PL_T), PL_T, 0, st>>>(own_sorted, rows_sorted, n, rank_ptr, localpos);
  } else {
    PL_CUDA(cudaMemsetAsync(rank_ptr, 0, sizeof(int32_t) * (p + 1), st));
  }
  // 2. cut keys (consumer, sender, column): count, scan, emit, sort, unique
  long long *cnt = nullptr, *off = nullptr;
  if (dmalloc(&cnt, n + 1, st) || dmalloc(&off, n + 1, st)) return set_error(GCNB_ECUDA, "plan build: out of memory");
  PL_CUDA(cudaMemsetAsync(cnt + n, 0, sizeof(long long), st));
  if (n > 0) k_cut_count<<<grid_for(n * 32, PL_T), PL_T, 0, st>>>(rp, ci, owner, n, cnt);
  {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, (int)(n + 1), st);
    if (tmp.ensure(tb)) return set_error(GCNB_ECUDA, "plan build: out of memory");
    PL_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt, off, (int)(n + 1), st));
  }
  long long n_cut = 0;
  PL_CUDA(cudaMemcpyAsync(&n_cut, off + n, sizeof(long long), cudaMemcpyDeviceToHost, st));
  PL_CUDA(cudaStreamSynchronize(st));
  unsigned long long *keys = nullptr, *sorted = nullptr, *uniq = nullptr;
  long long* n_uniq_d = nullptr;
  if (dmalloc(&keys, n_cut, st) || dmalloc(&sorted, n_cut, st) || dmalloc(&n_uniq_d, 1, st))
    return set_error(GCNB_ECUDA, "plan build: out of memory");
  if (n > 0) k_cut_emit<<<grid_for(n * 32, PL_T), PL_T, 0, st>>>(rp, ci, owner, n, off, keys);
  long long n_uniq = 0;
  if (n_cut > 0) {
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, sorted, n_cut, 0, 64, st);
    if (tmp.ensure(tb)) return set_error(GCNB_ECUDA, "plan build: out of memory");
    PL_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, keys, sorted, n_cut, 0, 64, st));
    cub::DeviceSelect::Unique(nullptr, tb, sorted, keys, n_uniq_d, n_cut, st);
    if (tmp.ensure(tb)) return set_error(GCNB_ECUDA, "plan build: out of memory");
    PL_CUDA(cub::DeviceSelect::Unique(tmp.p, tb, sorted, keys, n_uniq_d, n_cut, st));
    PL_CUDA(cudaMemcpyAsync(&n_uniq, n_uniq_d, sizeof(long long), cudaMemcpyDeviceToHost, st));
    PL_CUDA(cudaStreamSynchronize(st));
  }
  if (dmalloc(&uniq, n_uniq, st)) return set_error(GCNB_ECUDA, "plan build: out of memory");
  if (n_uniq > 0)
    PL_CUDA(cudaMemcpyAsync(uniq, keys, sizeof(unsigned long long) * n_uniq, cudaMemcpyDeviceToDevice, st));
  k_pair_bounds<<<(p * p + 1 + 127) / 128, 128, 0, st>>>(uniq, n_uniq, p, reinterpret_cast<long long*>(pair_bounds));
  cudaFreeAsync(own_sorted, st);
  cudaFreeAsync(iota, st);
  cudaFreeAsync(cnt, st);
  cudaFreeAsync(off, st);
  cudaFreeAsync(keys, st);
  cudaFreeAsync(sorted, st);
  cudaFreeAsync(n_uniq_d, st);
  GCNB_AFTER_LAUNCH("plan build");
  PL_CUDA(cudaStreamSynchronize(st));
  *keys_out = reinterpret_cast<uint64_t*>(uniq);
  *n_keys_out = n_uniq;
  return GCNB_OK;
}

extern "C" int gcnb_plan_free(void* p) {
  if (p) {
    cudaError_t e = cudaFree(p);
    if (e != cudaSuccess) return cuda_fail(e, "plan free");
  }
  return GCNB_OK;
}

/* See include/gcnb.h. */
extern "C" int gcnb_layout_fill(const int64_t* rp, const int64_t* ci, const double* val, int64_t n,
                                const int32_t* layout_rows, int32_t n_own, const uint64_t* keys, int64_t halo_k0,
                                int64_t n_halo, int32_t sort_rows, int64_t* row_ptr_out, int32_t* ext_col_out,
                                double* val_out, int32_t* has_halo_out, int32_t* colmap_scratch, void* stream) {
  GCNB_REQUIRE(n >= 0 && n_own >= 0 && n_halo >= 0, "layout fill: bad sizes");
  GCNB_REQUIRE(rp && ci && val && row_ptr_out && colmap_scratch && (n_own == 0 || (layout_rows && has_halo_out)),
               "layout fill: null argument");
  cudaStream_t st = (cudaStream_t)stream;
  Temp tmp(st);
  if (n_own > 0) k_colmap_own<<<grid_for(n_own, PL_T), PL_T, 0, st>>>(layout_rows, n_own, colmap_scratch);
  if (n_halo > 0)
    k_colmap_halo<<<grid_for(n_halo, PL_T), PL_T, 0, st>>>(reinterpret_cast<const unsigned long long*>(keys), halo_k0,
                                                           n_halo, n_own, colmap_scratch);
  long long* len = nullptr;
  if (dmalloc(&len, (size_t)n_own + 1, st)) return set_error(GCNB_ECUDA, "layout fill: out of memory");
  PL_CUDA(cudaMemsetAsync(len + n_own, 0, sizeof(long long), st));
  if (n_own > 0) k_row_len<<<grid_for(n_own, PL_T), PL_T, 0, st>>>(rp, layout_rows, n_own, len);
  {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, len, reinterpret_cast<long long*>(row_ptr_out), n_own + 1, st);
    if (tmp.ensure(tb)) return set_error(GCNB_ECUDA, "layout fill: out of memory");
    PL_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, len, reinterpret_cast<long long*>(row_ptr_out), n_own + 1, st));
  }
  long long nnz = 0;
  PL_CUDA(cudaMemcpyAsync(&nnz, row_ptr_out + n_own, sizeof(long long), cudaMemcpyDeviceToHost, st));
  PL_CUDA(cudaStreamSynchronize(st));
  GCNB_REQUIRE(nnz < (1ll << 31), "layout fill: rank block has %lld nonzeros (int32 limit)", nnz);
  if (n_own > 0)
    k_fill<<<grid_for((long long)n_own * 32, PL_T), PL_T, 0, st>>>(rp, ci, val, layout_rows, n_own,
                                                                  reinterpret_cast<const long long*>(row_ptr_out),
                                                                  colmap_scratch, ext_col_out, val_out, has_halo_out);
  if (sort_rows && n_halo > 0 && nnz > 0) {
    // each row by extended column (column ids are distinct within a row, so
    // any sort reproduces the host layout's stable sort): one radix sort of
    // (row, column) keys over all entries — a segmented sort over ~10^5 short
    // rows cost ~45 ms per layout on a 2^20-vertex mini-batch
    unsigned long long *kin = nullptr, *kout = nullptr;
    int *perm_in = nullptr, *perm = nullptr;
    double* vtmp = nullptr;
    if (dmalloc(&kin, nnz, st) || dmalloc(&kout, nnz, st) || dmalloc(&perm_in, nnz, st) || dmalloc(&perm, nnz, st) ||
        dmalloc(&vtmp, nnz, st))
      return set_error(GCNB_ECUDA, "layout fill: out of memory");
    k_row_col_keys<<<grid_for((long long)n_own * 32, PL_T), PL_T, 0, st>>>(
        reinterpret_cast<const long long*>(row_ptr_out), n_own, ext_col_out, kin, perm_in);
    int row_bits = 1;
    while ((1ll << row_bits) < (long long)n_own) ++row_bits;
    {
      size_t tb = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, perm_in, perm, nnz, 0, 32 + row_bits, st);
      if (tmp.ensure(tb)) return set_error(GCNB_ECUDA, "layout fill: out of memory");
      PL_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, kin, kout, perm_in, perm, nnz, 0, 32 + row_bits, st));
    }
    k_key_col<<<grid_for(nnz, PL_T), PL_T, 0, st>>>(kout, nnz, ext_col_out);
    PL_CUDA(cudaMemcpyAsync(vtmp, val_out, sizeof(double) * nnz, cudaMemcpyDeviceToDevice, st));
    k_gather_val<<<grid_for(nnz, PL_T), PL_T, 0, st>>>(perm, vtmp, nnz, val_out);
    cudaFreeAsync(kin, st);
    cudaFreeAsync(kout, st);
    cudaFreeAsync(perm_in, st);
    cudaFreeAsync(perm, st);
    cudaFreeAsync(vtmp, st);
  }
  cudaFreeAsync(len, st);
  GCNB_AFTER_LAUNCH("layout fill");
  PL_CUDA(cudaStreamSynchronize(st));
  return GCNB_OK;
}
