// Halo pack fused into a producing kernel's epilogue (north_star subsystem 2;
// the reference's send side, runtime.py:289-294 / 336-341 + SimNetwork.send):
// row r of the output, as it is stored, is also stored into every receiver's
// halo slot the plan assigns to it (map[map_ptr[r] .. map_ptr[r+1]) =
// {segment, position}; segment s is receiver s's halo block for this rank, a
// peer-mapped NVLink address), and once every block's stores are visible the
// last block rings the receivers' doorbells — the k_pack protocol without the
// separate launch and without re-reading the rows.  An EpiPack with
// map_ptr == nullptr disables both (the plain kernels).
#pragma once

#include <cstdint>

#include "common.cuh"

namespace gcnb {

struct EpiPack {
  float4* dst[GCNB_MAX_PEERS];
  unsigned long long* flag[GCNB_MAX_PEERS];
  const int* map_ptr;
  const int2* map;
  int* counter;
  int n_seg;
  int ldd4;
};

__device__ __forceinline__ void red_release_sys_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void epi_store(const EpiPack& pk, int row, int ch, float4 v) {
  if (!pk.map_ptr) return;
  const int e1 = __ldg(pk.map_ptr + row + 1);
  for (int e = __ldg(pk.map_ptr + row); e < e1; ++e) {
    const int2 m = __ldg(pk.map + e);
    pk.dst[m.x][(size_t)m.y * pk.ldd4 + ch] = v;
  }
}

// The rows this block produced — tiles blockIdx.x, blockIdx.x + gridDim.x, ...
// of T row positions; position i is own row rows[i] (rows == nullptr: i) —
// stored into their receiver slots after the fact, which keeps the pack out of
// the producer's register-tight main loop.  A warp tests 32 rows per step (one
// coalesced map_ptr load per lane, a ballot), then spreads the (boundary row,
// float4 chunk) pairs of those rows over its lanes, 32 independent copies per
// round (plain loads: the rows were written by this block, visible after its
// barrier).  All
// threads call it after the block's last store of Y and a __syncthreads.
__device__ __forceinline__ void epi_forward(const EpiPack& pk, const float* Y, int ldy, const int* rows, int n_rows,
                                            int T, int c4) {
  if (!pk.map_ptr) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int n_tiles = (n_rows + T - 1) / T;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int t1 = min(n_rows, (tile + 1) * T);
    for (int i0 = tile * T + warp * 32; i0 < t1; i0 += nw * 32) {
      const int i = i0 + lane;
      int row = 0, e0 = 0, e1 = 0;
      if (i < t1) {
        row = rows ? __ldg(rows + i) : i;
        e0 = __ldg(pk.map_ptr + row);
        e1 = __ldg(pk.map_ptr + row + 1);
      }
      const unsigned todo = __ballot_sync(0xffffffffu, e1 > e0);
      const int items = __popc(todo) * c4;  // (boundary row, chunk) pairs, spread over the lanes
      for (int base = 0; base < items; base += 32) {
        const int idx = base + lane;
        const int k = idx / c4, ch = idx - k * c4;
        const int src = idx < items ? (int)__fns(todo, 0, k + 1) : 0;
        const int r = __shfl_sync(0xffffffffu, row, src);
        const int a = __shfl_sync(0xffffffffu, e0, src);
        const int b = __shfl_sync(0xffffffffu, e1, src);
        if (idx < items) {
          const float4 v = reinterpret_cast<const float4*>(Y + (size_t)r * ldy)[ch];
          for (int e = a; e < b; ++e) {
            const int2 m = __ldg(pk.map + e);
            pk.dst[m.x][(size_t)m.y * pk.ldd4 + ch] = v;
          }
        }
      }
    }
  }
}

// All threads of the block call this once, after their last epi_store.
__device__ __forceinline__ void epi_signal(const EpiPack& pk) {
  if (!pk.map_ptr) return;
  __syncthreads();
  __shared__ int last;
  if (threadIdx.x == 0) {
    __threadfence_system();
    last = (atomicAdd(pk.counter, 1) == (int)gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence_system();
    *pk.counter = 0;
    for (int s = 0; s < pk.n_seg; ++s)
      if (pk.flag[s]) red_release_sys_add(pk.flag[s], 1ull);
  }
}

// Host: fill an EpiPack from the ABI's arrays (n_seg == 0: disabled).
int make_epipack(EpiPack* pk, const int32_t* map_ptr, const int32_t* map, float* const* dst, uint64_t* const* flags,
                 int32_t n_seg, int32_t ldd, int32_t* counter);

}  // namespace gcnb
