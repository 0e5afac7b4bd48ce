// Tensor-core (tcgen05) fp32-class dense transform Y[r] = act(X[r]·W) for the
// wide layers (the `@ w` of runtime.py:299/304), 3xTF32:
//
//   x·w ≈ hi(x)·hi(w) + hi(x)·lo(w) + lo(x)·hi(w),  hi = tf32 truncation, lo = x − hi
//
// (relative error ~2^-21 per product, fp32 accumulation in TMEM; a single
// TF32 product misses the 1e-4 bar, SURVEY key facts).  The tensor core reads
// tf32 operands as fp32 bit patterns and ignores the low 13 mantissa bits, so
// the raw fp32 tile *is* hi(x); lo(x) is written over the tile in place once
// the hi MMAs have drained.
//
// One persistent CTA per SM (256 threads): W (K×N, fp32) is staged once as the
// K-major B operand in both hi and lo form; 128-row X tiles are double
// buffered with cp.async (tile i+1 streams in while tile i is multiplied), in
// the canonical no-swizzle K-major layout (8-row × 16-byte core matrices).
// Thread 0 issues the MMAs (M=128, N=round16(d_out), K=8 per instruction)
// into a TMEM accumulator; completion is tracked with tcgen05.commit → an
// mbarrier; all 8 warps drain the accumulator with tcgen05.ld (warp w reads
// TMEM lanes 32·(w%4).., half the columns each), apply the activation and store.
#include <algorithm>
#include <cstdint>

#include "common.cuh"

namespace gcnb {

namespace {

constexpr int TC_M = 128;        // rows per tile = MMA M = TMEM lanes
constexpr int TC_THREADS = 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Canonical K-major, no-swizzle shared-memory matrix descriptor (sm_100):
// start>>4 [0,14), LBO>>4 [16,30) (next 16-byte K chunk), SBO>>4 [32,46)
// (next 8-row group), version 1 at [46,48), layout type 0 (SWIZZLE_NONE).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

// Instruction descriptor, kind::tf32: D f32 [4,6)=1, A tf32 [7,10)=2, B tf32
// [10,13)=2, both K-major, N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}" ::"r"(mbar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
      "@q cp.async.ca.shared.global [%0], [%1], 16;\n\t}" ::"r"(dst),
      "l"(src), "r"((int)pred)
      : "memory");
}

__device__ __forceinline__ float tf32_lo(float x) {
  return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// Byte offset of 16-byte chunk c of row r in a K-major canonical tile with
// `nch` chunks per row: core matrix (r/8, c) is 128 contiguous bytes.
__device__ __forceinline__ uint32_t kmaj_off(int r, int c, int nch) {
  return (uint32_t)(((r >> 3) * nch + c) * 128 + (r & 7) * 16);
}

// Stream one 128-row X tile into a stage: lanes map (row-in-group, chunk) so
// a quarter-warp fills one 128-byte core matrix (bank-conflict free) and four
// lanes of a row read 64 contiguous bytes.
__device__ __forceinline__ void load_tile(uint32_t stage, const float* __restrict__ X, int ldx,
                                          const int* __restrict__ rows, int n_rows, int m0, int kc, int nch) {
  const int quads = (kc + 3) >> 2;
  const int total = (TC_M / 8) * quads * 32;
  for (int idx = threadIdx.x; idx < total; idx += TC_THREADS) {
    const int rr = idx & 7, cc = (idx >> 3) & 3, gq = idx >> 5;
    const int g = gq % (TC_M / 8), q = gq / (TC_M / 8);
    const int r = g * 8 + rr, c = q * 4 + cc;
    const int i = m0 + r;
    const bool ok = c < kc && i < n_rows;
    const int xr = ok ? (rows ? __ldg(rows + i) : i) : 0;
    cp16(stage + kmaj_off(r, c, nch), X + (size_t)xr * ldx + 4 * c, ok);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

}  // namespace

namespace {
int g_dense_mode = 0;  // 0 auto, 1 force SIMT, 2 force tensor core (where it applies)
}

__global__ void __launch_bounds__(TC_THREADS, 1)
    k_dense_tc(const float* __restrict__ X, int ldx, const int* __restrict__ rows, int n_rows, int K,
               const float* __restrict__ W, int ldw, int w_nk, int N, float* __restrict__ Y, int ldy, int act,
               const float* __restrict__ Hm, int ldhm) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base_slot;
  const int Kp = (K + 7) & ~7, nch = Kp / 4, kc = (K + 3) / 4;  // chunks per row (padded / valid)
  const int Np = (N + 15) & ~15;
  const uint32_t tile_bytes = TC_M * Kp * 4, b_bytes = Np * Kp * 4;
  uint8_t* a_stage[2] = {smem, smem + tile_bytes};
  uint8_t* b_hi = smem + 2 * tile_bytes;
  uint8_t* b_lo = b_hi + b_bytes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles = (n_rows + TC_M - 1) / TC_M;
  const uint32_t tmem_cols = Np <= 32 ? 32 : Np <= 64 ? 64 : Np <= 128 ? 128 : 256;

  // first tile in flight before the one-time setup
  if ((int)blockIdx.x < n_tiles) load_tile(smem_u32(a_stage[0]), X, ldx, rows, n_rows, blockIdx.x * TC_M, kc, nch);

  // zero the K pad chunks of both stages (never written by the loads)
  for (int idx = threadIdx.x; idx < 2 * TC_M * (nch - kc); idx += TC_THREADS) {
    const int s = idx / (TC_M * (nch - kc)), rem = idx % (TC_M * (nch - kc));
    const int r = rem % TC_M, c = kc + rem / TC_M;
    *reinterpret_cast<float4*>(a_stage[s] + kmaj_off(r, c, nch)) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // B operand = Wᵀ (N rows × Kp, K-major): element (n, k) = W[k][n]; pad rows/cols zero
  for (int idx = threadIdx.x; idx < Np * nch; idx += TC_THREADS) {
    const int n = idx % Np, c = idx / Np;
    float v[4], l[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int k = 4 * c + e;
      v[e] = (n < N && k < K) ? __ldg(W + (w_nk ? (size_t)n * ldw + k : (size_t)k * ldw + n)) : 0.0f;
      l[e] = tf32_lo(v[e]);
    }
    *reinterpret_cast<float4*>(b_hi + kmaj_off(n, c, nch)) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(b_lo + kmaj_off(n, c, nch)) = make_float4(l[0], l[1], l[2], l[3]);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_slot)),
                 "r"(tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_async_smem();
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = tmem_base_slot;
  const uint32_t mb = smem_u32(&mbar);
  const uint32_t idesc = idesc_tf32(TC_M, Np);
  const uint32_t sbo_a = nch * 128, sbo_b = nch * 128;
  uint32_t phase = 0;

  int it = 0;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
    const int next = tile + gridDim.x;
    if (next < n_tiles) {
      load_tile(smem_u32(a_stage[(it + 1) & 1]), X, ldx, rows, n_rows, next * TC_M, kc, nch);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    fence_async_smem();
    __syncthreads();
    uint8_t* a = a_stage[it & 1];
    const uint32_t a_addr = smem_u32(a), bh = smem_u32(b_hi), bl = smem_u32(b_lo);
    // hi(x)·hi(w) + hi(x)·lo(w)
    if (threadIdx.x == 0) {
      tc_after_sync();
      for (int s = 0; s < Kp / 8; ++s) {
        const uint64_t da = smem_desc(a_addr + s * 256, 128, sbo_a);
        mma_tf32(tmem, da, smem_desc(bh + s * 256, 128, sbo_b), idesc, s > 0);
        mma_tf32(tmem, da, smem_desc(bl + s * 256, 128, sbo_b), idesc, 1);
      }
      mma_commit(mb);
    }
    mbar_wait(mb, phase);
    phase ^= 1;
    // lo(x) in place, then + lo(x)·hi(w)
    for (int idx = threadIdx.x; idx < TC_M * kc; idx += TC_THREADS) {
      const int r = idx % TC_M, c = idx / TC_M;
      float4* p = reinterpret_cast<float4*>(a + kmaj_off(r, c, nch));
      const float4 v = *p;
      *p = make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w));
    }
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_after_sync();
      for (int s = 0; s < Kp / 8; ++s)
        mma_tf32(tmem, smem_desc(a_addr + s * 256, 128, sbo_a), smem_desc(bh + s * 256, 128, sbo_b), idesc, 1);
      mma_commit(mb);
    }
    mbar_wait(mb, phase);
    phase ^= 1;
    tc_after_sync();
    // epilogue: warp w drains TMEM lanes 32(w%4).. (rows), columns [half·Np/2, (half+1)·Np/2)
    {
      const int quarter = warp & 3, half = warp >> 2;
      const int r = quarter * 32 + lane;
      const int i = tile * TC_M + r;
      const bool ok = i < n_rows;
      const int yr = ok ? (rows ? __ldg(rows + i) : i) : 0;
      const int c_lo = half * (Np / 2), c_hi = c_lo + Np / 2;
      for (int c0 = c_lo; c0 < c_hi; c0 += 8) {
        uint32_t v[8];
        const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (ok) {
          float* y = Y + (size_t)yr * ldy + c0;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (c0 + 4 * h < ldy) {
              float4 o = make_float4(__uint_as_float(v[4 * h]), __uint_as_float(v[4 * h + 1]),
                                     __uint_as_float(v[4 * h + 2]), __uint_as_float(v[4 * h + 3]));
              if (Hm) {  // backward: (agg·Wᵀ) ⊙ σ'(H_prev), σ' from h (gcn.py:101-104)
                const float4 hv = __ldg(reinterpret_cast<const float4*>(Hm + (size_t)yr * ldhm + c0) + h);
                o.x *= act_grad_from_h(hv.x, act);
                o.y *= act_grad_from_h(hv.y, act);
                o.z *= act_grad_from_h(hv.z, act);
                o.w *= act_grad_from_h(hv.w, act);
              } else {
                o = act_fwd4(o, act);
              }
              reinterpret_cast<float4*>(y)[h] = o;
            }
          }
        }
      }
    }
    tc_before_sync();
    __syncthreads();  // TMEM drained and stage (it & 1) free before they are reused
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols) : "memory");
}

bool dense_tc_applies(int d_in, int d_out) {
  if (g_dense_mode == 1) return false;
  const int Kp = (d_in + 7) & ~7, Np = (d_out + 15) & ~15;
  const size_t smem = (size_t)2 * TC_M * Kp * 4 + (size_t)2 * Np * Kp * 4;
  const bool fits = d_in <= 256 && d_out <= 256 && smem <= 220 * 1024;
  if (g_dense_mode == 2) return fits;
  return fits && d_in >= 32 && d_out >= 32;
}

int launch_dense_tc(const float* x, int ldx, const int* rows, int n_rows, int d_in, const float* w, int d_out,
                    float* y, int ldy, int act, cudaStream_t st, const float* w_nk, int ld_wnk, const float* hmask,
                    int ldhm) {
  const int Kp = (d_in + 7) & ~7, Np = (d_out + 15) & ~15;
  const size_t smem = (size_t)2 * TC_M * Kp * 4 + (size_t)2 * Np * Kp * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_dense_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int tiles = (n_rows + TC_M - 1) / TC_M;
  const int grid = std::max(1, std::min(tiles, num_sms()));
  k_dense_tc<<<grid, TC_THREADS, smem, st>>>(x, ldx, rows, n_rows, d_in, w_nk ? w_nk : w, w_nk ? ld_wnk : round4(d_out),
                                             w_nk ? 1 : 0, d_out, y, ldy, act, hmask, ldhm);
  GCNB_AFTER_LAUNCH("dense (tcgen05 3xTF32)");
  return GCNB_OK;
}

// ---------------------------------------------------------------------------
// ΔW partial per CTA: P[cta] = Σ_{rows of the CTA's tiles} H[r]ᵀ·A[r]  (the
// `h_prev.T @ agg` of runtime.py:355), 3xTF32 on tcgen05 with K = graph rows:
// A-operand = Hᵀ and B-operand = A, both MN-major straight from the row-major
// rows, M = 128 (d_prev padded), N = round16(d_k).  MN-major tf32 operands
// must use the 128B-swizzle-with-32B-atoms layout (SWIZZLE_128B_BASE32B): an
// atom is 4 K-rows × 128 bytes (32 features), its 32-byte granules XOR-permuted
// by the row index (bits [5,7) ^= bits [7,9) of the address); atoms repeat
// along the features at LBO = 512 B and along K at SBO = atoms·512 B.  A
// 16-byte chunk of 4 features never straddles a granule, so rows stream in
// with plain 16-byte cp.async.  The accumulator lives in TMEM for the CTA's
// whole tile range and is written once; partials fold in fixed order
// (k_reduce*), so results are deterministic.
//   ΔW += H·A + lo(H)·A  [lo(H) in its own buffer],  then A → lo(A) in place,  ΔW += H·lo(A)
constexpr int DW_T = 64;  // rows per tile (8 MMA K-steps of 8 rows)

namespace {

// Byte offset of feature m of tile row k in an MN-major SW128_32B tile with `na` atoms per 4-row group.
__device__ __forceinline__ uint32_t mn_off(int k, int m, int na) {
  return (uint32_t)((k >> 2) * (na * 512) + (m >> 5) * 512 + (k & 3) * 128 + ((((m & 31) >> 3) ^ (k & 3)) << 5) +
                    ((m & 7) << 2));
}

__device__ __forceinline__ void load_rows_mn(uint32_t stage, const float* __restrict__ X, int ldx,
                                             const int* __restrict__ rows, int n_rows, int m0, int kc, int na) {
  for (int idx = threadIdx.x; idx < DW_T * kc; idx += TC_THREADS) {
    const int k = idx / kc, c = idx - k * kc;
    const int i = m0 + k;
    const bool ok = i < n_rows;  // rows past the end must be zero: they are summed over
    const int xr = ok ? (rows ? __ldg(rows + i) : i) : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(stage + mn_off(k, 4 * c, na)),
                 "l"(X + (size_t)xr * ldx + 4 * c), "r"(ok ? 16 : 0)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__device__ __forceinline__ uint64_t desc_mn_sw32(uint32_t addr, int na) {
  // LBO = next 32-feature atom (512 B), SBO = next 4-row group, layout type 1
  return smem_desc(addr, 512, (uint32_t)na * 512) | (1ull << 61);
}

__device__ __forceinline__ void lo_inplace(uint8_t* dst, const uint8_t* src, int bytes) {
  for (int i = threadIdx.x; i < bytes / 16; i += TC_THREADS) {
    const float4 v = reinterpret_cast<const float4*>(src)[i];
    reinterpret_cast<float4*>(dst)[i] = make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w));
  }
}

}  // namespace

__global__ void __launch_bounds__(TC_THREADS, 1)
    k_dw_tc(const float* __restrict__ H, int ldh, int d_prev, const float* __restrict__ A, int lda, int d_k,
            const int* __restrict__ rows, int n_rows, float* __restrict__ partials, int n_slots) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base_slot;
  constexpr int NA_H = 4;                                // M = 128 features = 4 atoms
  const int Np = (d_k + 15) & ~15, na_a = (Np + 31) / 32;
  const int kc_h = (d_prev + 3) / 4, kc_a = (d_k + 3) / 4;
  const int h_bytes = (DW_T / 4) * NA_H * 512, a_bytes = (DW_T / 4) * na_a * 512;
  uint8_t* st_h[2] = {smem, smem + h_bytes + a_bytes};
  uint8_t* st_a[2] = {smem + h_bytes, smem + 2 * h_bytes + a_bytes};
  uint8_t* h_lo = smem + 2 * (h_bytes + a_bytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles = (n_rows + DW_T - 1) / DW_T;
  const uint32_t tmem_cols = Np <= 32 ? 32 : Np <= 64 ? 64 : Np <= 128 ? 128 : 256;

  // pad features (never loaded) must read as zero: clear everything once
  for (int i = threadIdx.x; i < (3 * h_bytes + 2 * a_bytes) / 16; i += TC_THREADS)
    reinterpret_cast<float4*>(smem)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  if ((int)blockIdx.x < n_tiles) {
    load_rows_mn(smem_u32(st_h[0]), H, ldh, rows, n_rows, blockIdx.x * DW_T, kc_h, NA_H);
    load_rows_mn(smem_u32(st_a[0]), A, lda, rows, n_rows, blockIdx.x * DW_T, kc_a, na_a);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_slot)),
                 "r"(tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = tmem_base_slot;
  const uint32_t mb = smem_u32(&mbar);
  const uint32_t idesc = idesc_tf32(128, Np) | (1u << 15) | (1u << 16);  // A and B MN-major
  const uint32_t kstep_h = 2 * NA_H * 512, kstep_a = 2 * na_a * 512;   // 8 rows = two 4-row groups
  uint32_t phase = 0;
  bool first = true;

  int it = 0;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
    const int next = tile + gridDim.x;
    if (next < n_tiles) {
      load_rows_mn(smem_u32(st_h[(it + 1) & 1]), H, ldh, rows, n_rows, next * DW_T, kc_h, NA_H);
      load_rows_mn(smem_u32(st_a[(it + 1) & 1]), A, lda, rows, n_rows, next * DW_T, kc_a, na_a);
      asm volatile("cp.async.wait_group 2;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    uint8_t* hs = st_h[it & 1];
    uint8_t* as = st_a[it & 1];
    lo_inplace(h_lo, hs, h_bytes);
    fence_async_smem();
    __syncthreads();
    const uint32_t ha = smem_u32(hs), hl = smem_u32(h_lo), aa = smem_u32(as);
    if (threadIdx.x == 0) {
      tc_after_sync();
      for (int s = 0; s < DW_T / 8; ++s) {
        const uint64_t db = desc_mn_sw32(aa + s * kstep_a, na_a);
        mma_tf32(tmem, desc_mn_sw32(ha + s * kstep_h, NA_H), db, idesc, first ? 0u : 1u);
        first = false;
        mma_tf32(tmem, desc_mn_sw32(hl + s * kstep_h, NA_H), db, idesc, 1u);
      }
      mma_commit(mb);
    }
    mbar_wait(mb, phase);
    phase ^= 1;
    lo_inplace(as, as, a_bytes);
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_after_sync();
      for (int s = 0; s < DW_T / 8; ++s)
        mma_tf32(tmem, desc_mn_sw32(ha + s * kstep_h, NA_H), desc_mn_sw32(aa + s * kstep_a, na_a), idesc, 1u);
      mma_commit(mb);
    }
    mbar_wait(mb, phase);
    phase ^= 1;
    __syncthreads();  // stage (it & 1) and lo(H) free for reuse
  }
  tc_after_sync();
  // partial[m][n] for m < d_prev, n < round4(d_k): TMEM lane m, column n
  const int ld_k = (d_k + 3) & ~3;
  {
    const int quarter = warp & 3, half = warp >> 2;
    const int m = quarter * 32 + lane;
    float* out = partials + (size_t)blockIdx.x * d_prev * ld_k + (size_t)m * ld_k;
    const int c_lo = half * (Np / 2), c_hi = c_lo + Np / 2;
    for (int c0 = c_lo; c0 < c_hi; c0 += 8) {
      uint32_t v[8];
      const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (m < d_prev) {
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (c0 + e < ld_k) out[c0 + e] = n_tiles > (int)blockIdx.x ? __uint_as_float(v[e]) : 0.0f;
      }
    }
  }
  // slots beyond the grid (the caller sized the partials for another engine) are zero
  {
    const size_t slot = (size_t)d_prev * ld_k;
    for (int sl = blockIdx.x + gridDim.x; sl < n_slots; sl += gridDim.x)
      for (size_t e = threadIdx.x; e < slot; e += TC_THREADS) partials[sl * slot + e] = 0.0f;
  }
  tc_before_sync();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols) : "memory");
}

bool dw_tc_applies(int d_prev, int d_k) {
  if (g_dense_mode == 1) return false;
  const int Np = (d_k + 15) & ~15, na = (Np + 31) / 32;
  const size_t smem = (size_t)3 * (DW_T / 4) * 4 * 512 + (size_t)2 * (DW_T / 4) * na * 512;
  return d_prev <= 128 && d_k <= 256 && smem <= 220 * 1024;
}

int dw_tc_grid(int n_rows) { return std::max(1, std::min((n_rows + DW_T - 1) / DW_T, num_sms())); }

int launch_dw_tc(const float* h, int ldh, int d_prev, const float* a, int lda, int d_k, const int* rows, int n_rows,
                 float* partials, int n_slots, cudaStream_t st) {
  const int grid = std::min(dw_tc_grid(n_rows), n_slots);
  const int Np = (d_k + 15) & ~15, na = (Np + 31) / 32;
  const size_t smem = (size_t)3 * (DW_T / 4) * 4 * 512 + (size_t)2 * (DW_T / 4) * na * 512;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_dw_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_dw_tc<<<grid, TC_THREADS, smem, st>>>(h, ldh, d_prev, a, lda, d_k, rows, n_rows, partials, n_slots);
  GCNB_AFTER_LAUNCH("bwd ΔW (tcgen05 3xTF32)");
  return GCNB_OK;
}

}  // namespace gcnb

extern "C" int gcnb_set_dense_mode(int32_t mode) {
  GCNB_REQUIRE(mode >= 0 && mode <= 2, "dense mode must be 0 (auto), 1 (SIMT) or 2 (tensor core)");
  gcnb::g_dense_mode = mode;
  return GCNB_OK;
}
