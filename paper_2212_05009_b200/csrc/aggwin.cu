// Windowed aggregation: Y = act(A·X) over all own rows with the feature rows
// of a sliding row window staged in shared memory (the SpMM of sparse.py:196-207
// for the whole row block, i.e. runtime.py:299/346 with rows = all).
//
// Why: the gather of neighbour rows is bound by L2→SM bandwidth, not by HBM
// (every nonzero pulls a d-wide fp32 row through L2; products fwd1 moves
// ~50 GB through L2 for ~3 GB of compulsory HBM bytes).  With the locality
// layout (locality.py) most neighbours of a row sit within a couple of
// thousand rows of it, so a CTA that walks a contiguous row range can keep
// those rows on chip and read them from shared memory (3x the L2 bandwidth
// per SM) — each staged once per CTA instead of once per nonzero.
//
// Layout (built once per operator by k_wincsr):
//   * rows are split in tiles of AW_T = 128; the window of tile t is the data
//     tiles [t - bt, t + bt] (W = (2bt+1)·128 rows), the shared-memory ring
//     holds RT = 2bt + 3 data tiles (two tiles of lookahead);
//   * every row's nonzeros are re-ordered near-first: a nonzero is *near* when
//     its column is an own row inside the row's window; near entries store the
//     ring slot ((col/128) mod RT)·128 + col mod 128, far entries the column;
//     entries are int2 {slot|col, val bits}, nnear[r] counts the near ones.
//   Accumulation order per row: near entries then far entries, each in CSR
//   order — fixed, so reruns are bit-identical (the reference sums in CSR
//   order; the reassociation is within fp32 rounding, far below 1e-4).
//
// Kernel: grid = n_ranges × n_slices.  A CTA owns a contiguous, tile-aligned,
// nnz-balanced row range and one feature slice of CS float4 chunks (CS·16 bytes
// per row), so a ring data tile is 128 × CS·16 bytes (CS = 5: 10 KB; 21 tiles =
// 210 KB).  Warp 15 is the producer: one TMA (cp.async.bulk.tensor.2d) per data
// tile, completion on that ring slot's mbarrier; it refills the slot of data
// tile c - bt with tile c + bt + 3 once every row of tile c has been released
// (per-tile "empty" mbarriers, 128 arrivals).  Warps 0-14 grab GPW rows at a
// time from a shared counter (rows stay in order: a warp can lag the producer
// by at most two tiles), check the ring slots their rows need, and aggregate a
// row per group of CS lanes: near entries from shared memory (LDS.128), far
// entries from global (batched 16-byte loads).
#include <cuda.h>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "common.cuh"
#include "sync.cuh"

namespace gcnb {

namespace {

constexpr int AW_T = 128;           // rows per tile
constexpr int AW_WARPS = 16;        // 15 consumer warps + 1 producer warp
constexpr int AW_THREADS = AW_WARPS * 32;
constexpr int AW_EMPTY = 4;         // per-tile release barriers (tiles in flight <= 3)

__device__ __forceinline__ int2 ldg_int2(const int2* p) {
  int2 v;
  asm volatile("ld.global.nc.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ float4 ldg4_pred(const float4* p, bool pred) {
  float4 v;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "mov.b32 %0, 0;\n\tmov.b32 %1, 0;\n\tmov.b32 %2, 0;\n\tmov.b32 %3, 0;\n\t"
      "@q ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];\n\t}"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p), "r"((int)pred));
  return v;
}

__device__ __forceinline__ float4 lds4_pred(uint32_t addr, bool pred) {
  float4 v;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "mov.b32 %0, 0;\n\tmov.b32 %1, 0;\n\tmov.b32 %2, 0;\n\tmov.b32 %3, 0;\n\t"
      "@q ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n\t}"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "r"(addr), "r"((int)pred));
  return v;
}

__host__ __device__ constexpr int aw_ring_tiles(int bt) { return 2 * bt + 3; }

constexpr int SE = 16;  // near entries staged per row group and pass

// per-warp entry staging: 2 passes × GPW groups × (SE + 1) int2 (the +1 pad
// spreads the groups' broadcast reads over different banks)
__host__ __device__ constexpr int aw_stage_int2(int cs) { return (AW_WARPS - 1) * 2 * (32 / cs) * (SE + 1); }

__host__ __device__ inline size_t aw_smem_bytes(int cs, int bt) {
  return (size_t)aw_ring_tiles(bt) * AW_T * cs * 16 + (size_t)aw_stage_int2(cs) * 8 +
         (size_t)(aw_ring_tiles(bt) + AW_EMPTY) * 8 + 16;
}

// First tile of range j: smallest tile whose first row starts at or after
// nonzero j·nnz/n_ranges (ranges are contiguous, tile-aligned, nnz-balanced).
__device__ __forceinline__ int range_bound(const int* __restrict__ rp, int n_rows, int n_tiles, int j,
                                           int n_ranges) {
  if (j <= 0) return 0;
  if (j >= n_ranges) return n_tiles;
  const long long target = (long long)__ldg(rp + n_rows) * j / n_ranges;
  int lo = 0, hi = n_tiles;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(rp + min(mid * AW_T, n_rows)) >= target) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

template <int CS>
__global__ void __launch_bounds__(AW_THREADS, 1)
    k_aggwin(const __grid_constant__ CUtensorMap xmap, int c4, const int* __restrict__ rp,
             const int* __restrict__ nnear, const int2* __restrict__ ent, int n_rows, int n_ranges, int n_slices,
             int bt, float4* __restrict__ Y4, int ldy4) {
  constexpr int G = CS;          // lanes per row group (one float4 chunk each)
  constexpr int GPW = 32 / G;    // row groups per warp
  const int RT = aw_ring_tiles(bt);
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t ring = smem_u32(smem);
  int2* stage = reinterpret_cast<int2*>(smem + (size_t)RT * AW_T * CS * 16);
  uint64_t* bars = reinterpret_cast<uint64_t*>(stage + aw_stage_int2(CS));
  const uint32_t full0 = smem_u32(bars);               // RT ring-slot barriers
  const uint32_t empty0 = smem_u32(bars + RT);          // AW_EMPTY tile-release barriers
  int* next = reinterpret_cast<int*>(bars + RT + AW_EMPTY);

  const int range = blockIdx.x / n_slices, slice = blockIdx.x - range * n_slices;
  const int n_tiles = (n_rows + AW_T - 1) / AW_T;
  const int ta = range_bound(rp, n_rows, n_tiles, range, n_ranges);
  const int tb = range_bound(rp, n_rows, n_tiles, range + 1, n_ranges);
  if (ta >= tb) return;  // uniform over the CTA
  const int c0 = slice * CS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < RT; ++i) mbar_init(full0 + 8 * i, 1);
    for (int i = 0; i < AW_EMPTY; ++i) mbar_init(empty0 + 8 * i, AW_T);
    *next = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  constexpr uint32_t TILE_BYTES = AW_T * CS * 16;
  const int d_first = ta - bt;          // first data tile of the range (phase 0 of every slot)

  if (warp == AW_WARPS - 1) {
    // producer: data tiles d_first .. tb-1+bt in order; tile d lands in slot d mod RT
    if (lane == 0) {
      auto issue = [&](int d) {
        const int slot = ((d % RT) + RT) % RT;
        const uint32_t fb = full0 + 8 * slot;
        if (d >= 0 && d < n_tiles) {
          mbar_expect_tx(fb, TILE_BYTES);
          tma_load_2d(ring + (uint32_t)slot * TILE_BYTES, &xmap, c0 * 4, d * AW_T, fb);
        } else {
          mbar_arrive(fb);  // outside the matrix: complete the phase, no data (never read)
        }
      };
      const int d_last = tb - 1 + bt;
      int d = d_first;
      for (; d < d_first + RT && d <= d_last; ++d) issue(d);
      for (int c = ta; d <= d_last; ++c, ++d) {
        // slot of data tile d = c + bt + 3 held data tile c - bt, which only
        // windows of tiles <= c read: wait until tile c has been released
        mbar_wait(empty0 + 8 * ((c - ta) % AW_EMPTY), (uint32_t)((c - ta) / AW_EMPTY) & 1u);
        issue(d);
      }
    }
    return;
  }

  // consumers (near pass): a group of G = CS lanes per row, GPW rows per
  // warp.  A row's near entries are staged SE at a time in the warp's slice of
  // shared memory (loaded one pass ahead into registers, then stored), and read
  // back as broadcast LDS.64 — no shuffles, so no warp-convergence
  // requirement inside the loops — then each lane reads its 16-byte chunk of
  // the neighbour row from the ring (LDS.128).  No global data loads here:
  // the far entries are the second pass (launch_agg_far).
  const int g = lane / G, gl = lane - g * G;
  const bool lane_on = g < GPW;
  const int q = c0 + gl;
  const bool q_on = lane_on && q < c4;
  const int row0 = ta * AW_T, row_end = tb * AW_T;
  const uint32_t ring_q = ring + (uint32_t)gl * 16;
  int2* wst = stage + (size_t)warp * 2 * GPW * (SE + 1);
  int vhi = d_first - 1;  // highest data tile this warp has seen complete
  auto grab = [&]() {
    int b = 0;
    if (lane == 0) b = atomicAdd(next, GPW);
    return __shfl_sync(0xffffffffu, b, 0) + row0;
  };
  auto extent = [&](int b, int& s, int& nn) {
    const int r = b + g;
    s = nn = 0;
    if (lane_on && b < row_end && r < min(row_end, n_rows)) {
      s = __ldg(rp + r);
      nn = __ldg(nnear + r);
    }
  };
  constexpr int JE = (SE + G - 1) / G;
  int b = grab();
  int s, nn;
  extent(b, s, nn);
  while (b < row_end) {
    const int b_n = grab();  // the near pass is short: the next batch's extent is fetched now
    int s_n, nn_n;
    extent(b_n, s_n, nn_n);
    const int r = b + g;
    const bool r_in = lane_on && r < row_end;   // counts toward its tile's release
    {
      const int t_lo = b / AW_T;
      const int t_hi = (min(b + GPW, row_end) - 1) / AW_T;
      const int dneed = min(t_hi + bt, n_tiles - 1);
      for (int d = max(vhi + 1, max(t_lo - bt, 0)); d <= dneed; ++d)
        mbar_wait(full0 + 8 * (d % RT), (uint32_t)((d - d_first) / RT) & 1u);
      vhi = max(vhi, dneed);
    }
    const int2* er = ent + s;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const int maxnn = __reduce_max_sync(0xffffffffu, nn);
    int2 e[JE];
#pragma unroll
    for (int j = 0; j < JE; ++j) {
      const int k = j * G + gl;
      e[j] = (k < SE && k < nn) ? ldg_int2(er + k) : make_int2(0, 0);
    }
    for (int base = 0; base < maxnn; base += SE) {
      // idle lanes (g == GPW when 32 % G != 0) address group GPW - 1's slots (never stored)
      int2* buf = wst + ((base / SE) & 1) * GPW * (SE + 1) + min(g, GPW - 1) * (SE + 1);
#pragma unroll
      for (int j = 0; j < JE; ++j) {
        const int k = j * G + gl;
        if (lane_on && k < SE) buf[k] = e[j];
      }
      if (base + SE < maxnn) {
#pragma unroll
        for (int j = 0; j < JE; ++j) {
          const int k = base + SE + j * G + gl;
          e[j] = (j * G + gl < SE && k < nn) ? ldg_int2(er + k) : make_int2(0, 0);
        }
      }
      __syncwarp();
      const int cnt = min(SE, maxnn - base);
      for (int kk = 0; kk < cnt; kk += 4) {
        int2 t[4];
        float4 x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) t[u] = (kk + u < SE) ? buf[kk + u] : make_int2(0, 0);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          x[u] = lds4_pred(ring_q + (uint32_t)t[u].x * (CS * 16), q_on && base + kk + u < nn);
#pragma unroll
        for (int u = 0; u < 4; ++u) acc = fma4(__int_as_float(t[u].y), x[u], acc);
      }
      __syncwarp();
    }
    // release the row's ring data, store the near partial sum (the far pass adds the rest)
    if (r_in && gl == 0) mbar_arrive(empty0 + 8 * (((r / AW_T) - ta) % AW_EMPTY));
    if (r_in && r < n_rows && q_on) Y4[(size_t)r * ldy4 + q] = acc;
    b = b_n;
    s = s_n;
    nn = nn_n;
  }
}

// One warp per row: stable near-first partition of the row's nonzeros into
// int2 entries {slot | col, val bits} (see the file comment).
__global__ void k_wincsr(const int* __restrict__ rp, const int* __restrict__ col, const float* __restrict__ val,
                         int n_rows, int n_own, int bt, int* __restrict__ nnear, int2* __restrict__ ent) {
  const int lane = threadIdx.x & 31;
  const int RT = aw_ring_tiles(bt);
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_rows; r += (gridDim.x * blockDim.x) >> 5) {
    const int s = rp[r], e = rp[r + 1];
    const int rt = r / AW_T;
    auto is_near = [&](int c) { return c < n_own && abs(c / AW_T - rt) <= bt; };
    int cnt = 0;
    for (int k0 = s; k0 < e; k0 += 32) {
      const int k = k0 + lane;
      cnt += __popc(__ballot_sync(0xffffffffu, k < e && is_near(col[k])));
    }
    int nb = 0, fb = 0;
    for (int k0 = s; k0 < e; k0 += 32) {
      const int k = k0 + lane;
      const bool ok = k < e;
      const int c = ok ? col[k] : 0;
      const bool nr = ok && is_near(c);
      const unsigned bn = __ballot_sync(0xffffffffu, nr);
      const unsigned bf = __ballot_sync(0xffffffffu, ok && !nr);
      const unsigned lt = (1u << lane) - 1u;
      if (ok) {
        const int2 v = nr ? make_int2((c / AW_T % RT) * AW_T + c % AW_T, __float_as_int(val[k]))
                          : make_int2(c, __float_as_int(val[k]));
        const int pos = nr ? s + nb + __popc(bn & lt) : s + cnt + fb + __popc(bf & lt);
        ent[pos] = v;
      }
      nb += __popc(bn);
      fb += __popc(bf);
    }
    if (lane == 0) nnear[r] = cnt;
  }
}

}  // namespace

// Passes gcnb_aggwin_f32 runs (bit 0 near, bit 1 far): a measurement knob
// (gcnb_set_aggwin_passes), 3 = both = the aggregation.
int g_aggwin_passes = 3;

// Chunk count per slice for a row of c4 float4 chunks.
static int aggwin_cs(int c4) { return (c4 % 5 == 0 && c4 % 4 != 0) ? 5 : 4; }

}  // namespace gcnb

using namespace gcnb;

extern "C" int gcnb_window_csr(const int32_t* row_ptr, const int32_t* col, const float* val, int32_t n_rows,
                               int32_t n_own, int32_t bt, int32_t* nnear, void* entries, void* stream) {
  GCNB_REQUIRE(n_rows >= 0 && n_own >= 0 && bt >= 0, "window csr: bad sizes");
  if (n_rows == 0) return GCNB_OK;
  GCNB_REQUIRE(row_ptr && col && val && nnear && entries, "window csr: null pointer");
  const int threads = 256;
  const int blocks = std::min((n_rows + 7) / 8, 148 * 16);
  k_wincsr<<<blocks, threads, 0, (cudaStream_t)stream>>>(row_ptr, col, val, n_rows, n_own, bt, nnear,
                                                         static_cast<int2*>(entries));
  GCNB_AFTER_LAUNCH("window csr");
  return GCNB_OK;
}

extern "C" int gcnb_aggwin_applies(int32_t d, int32_t bt, int32_t* out) {
  GCNB_REQUIRE(out, "aggwin_applies: null out");
  const int c4 = (d + 3) / 4;
  *out = d >= 16 && bt >= 0 && aw_smem_bytes(aggwin_cs(c4), bt) <= 227 * 1024 ? 1 : 0;
  return GCNB_OK;
}

extern "C" int gcnb_aggwin_f32(const int32_t* row_ptr, const int32_t* nnear, const void* entries, int32_t n_rows,
                               int32_t bt, const float* x, int32_t ldx, int32_t d, float* y, int32_t ldy,
                               int32_t act, void* stream) {
  GCNB_REQUIRE(n_rows >= 0 && d > 0 && bt >= 0, "aggwin: bad sizes");
  if (n_rows == 0) return GCNB_OK;
  GCNB_REQUIRE(row_ptr && nnear && entries && x && y, "aggwin: null pointer");
  GCNB_REQUIRE(ldx % 4 == 0 && ldy % 4 == 0 && ldx >= d && ldy >= d && aligned16(x) && aligned16(y),
               "aggwin: rows must be 16-byte aligned with ld >= d (ld %% 4 == 0)");
  const int c4 = (d + 3) / 4;
  const int cs = aggwin_cs(c4);
  const size_t smem = aw_smem_bytes(cs, bt);
  GCNB_REQUIRE(smem <= 227 * 1024, "aggwin: window of %d tiles does not fit shared memory", 2 * bt + 1);
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  // the map covers the n_rows own rows only: halo rows are never near
  GCNB_REQUIRE(tmap_2d(&map, x, ldx, n_rows, ldx, cs * 4, AW_T, CU_TENSOR_MAP_SWIZZLE_NONE),
               "aggwin: tensor map encode failed");
  const int n_slices = (c4 + cs - 1) / cs;
  const int n_tiles = (n_rows + AW_T - 1) / AW_T;
  const int n_ranges = std::max(1, std::min(n_tiles, num_sms() / n_slices));
  cudaStream_t st = (cudaStream_t)stream;
  auto fn = cs == 5 ? k_aggwin<5> : k_aggwin<4>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (!(g_aggwin_passes & 1)) return (g_aggwin_passes & 2) ? launch_agg_far(row_ptr, nnear, entries, n_rows, x, ldx, d, y, ldy, act, st) : GCNB_OK;
  fn<<<n_ranges * n_slices, AW_THREADS, smem, st>>>(map, c4, row_ptr, nnear, static_cast<const int2*>(entries),
                                                    n_rows, n_ranges, n_slices, bt, reinterpret_cast<float4*>(y),
                                                    ldy / 4);
  GCNB_AFTER_LAUNCH("aggregation (windowed, near pass)");
  if (!(g_aggwin_passes & 2)) return GCNB_OK;
  return launch_agg_far(row_ptr, nnear, entries, n_rows, x, ldx, d, y, ldy, act, st);
}

extern "C" int gcnb_set_aggwin_passes(int32_t mask) {
  GCNB_REQUIRE(mask >= 0 && mask <= 3, "aggwin passes: mask in [0, 3]");
  gcnb::g_aggwin_passes = mask;
  return GCNB_OK;
}
