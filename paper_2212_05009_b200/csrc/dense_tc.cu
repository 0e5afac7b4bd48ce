// Tensor-core (tcgen05) fp32-class dense transforms for the wide layers (the
// `@ w` of runtime.py:299/304, `agg @ weights.T` and `h.T @ aggregated` of
// runtime.py:353-356), 3xTF32:
//
//   x·w ≈ hi(x)·hi(w) + hi(x)·lo(w) + lo(x)·hi(w),  hi = tf32 truncation, lo = x − hi
//
// (relative error ~2^-21 per product, fp32 accumulation in TMEM; a single
// TF32 product misses the 1e-4 bar, SURVEY key facts).  The tensor core reads
// tf32 operands as fp32 bit patterns and ignores the low 13 mantissa bits, so
// a raw fp32 tile *is* hi(x); lo(x) is written over the tile in place once
// the hi MMAs have drained.
//
// k_dense_tc: Y[r] = act(X[r]·W) or (X[r]·Wᵀ) ⊙ σ'(H[r]) — warp-specialised,
// persistent, MMA M = output features (see the kernel comment).
// k_dw_tc:    per-CTA ΔW partials Σ_r H[r]ᵀ·A[r] with K = graph rows.
#include <cuda.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <cstdio>

#include "common.cuh"
#include "epipack.cuh"
#include "sync.cuh"

namespace gcnb {

// Extra dynamic shared memory each tcgen05 kernel asks for so that it can align
// its stage ring to 1024 bytes itself (swizzle atoms).
constexpr size_t SMEM_ALIGN_PAD = 1024;

namespace {



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

// Byte offset of 16-byte chunk c (4 floats of K) of row r in a K-major
// SWIZZLE_128B tile of `rows` rows: K runs in blocks of 32 floats (one 128-byte
// line per row); a block is `rows` lines, 8-row atoms of 1024 bytes, and the
// chunk's position inside its line is XOR-permuted by the row (r & 7).  The
// tile base must be 1024-byte aligned.
__device__ __forceinline__ uint32_t sw128_off(int r, int c, int rows) {
  return (uint32_t)((c >> 3) * rows * 128 + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

// Descriptor of MMA K-step s (8 tf32 = 32 bytes) of a SWIZZLE_128B K-major
// tile: the start advances 32 bytes inside the 128-byte line and a whole
// block of `rows` lines every 4 steps; SBO = 1024 (next 8-row atom), LBO
// unused (1), layout type 2 (SWIZZLE_128B) at bits [61,64).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t base, int s, int rows) {
  const uint32_t addr = base + (uint32_t)((s >> 2) * rows * 128 + (s & 3) * 32);
  return smem_desc(addr, 16, 1024) | (2ull << 61);
}

}  // namespace

namespace {
int g_dense_mode = 0;  // 0 auto, 1 force SIMT, 2 force tensor core (where it applies)
int g_dw_v2 = 1;       // 1: k_dw_tc2 (Hᵀ in TMEM) where it applies, 0: k_dw_tc (gcnb_set_dw_mode)
}

// Warp-specialised, transposed-orientation transform: the MMA computes
// Dᵀ = Wᵀ·Xᵀ, i.e. M = 128 output features (TMEM lanes), N = NT_ rows of X per
// tile (TMEM columns), K = d_in.  A = Wᵀ (hi and lo) lives in TENSOR memory for
// the whole persistent CTA (columns [0, 2·Kp)), so shared memory holds only the
// X stages (SWIZZLE_128B, 2-4 of them) and each MMA reads one operand from
// shared memory.  With the features on TMEM lanes, the epilogue thread for
// feature m holds consecutive rows, so a warp store writes 32 consecutive
// features of one row (128 contiguous bytes).
//   warps 0-7   epilogue: tcgen05.ld → act / ⊙σ'(mask) → coalesced stores
//               (two warps per TMEM lane quarter, each half of the tile's rows);
//               warps 0-3 also write Wᵀ hi/lo into TMEM at start
//   warps 8-11  converter: lo(x) in place once the stage's hi MMAs drained
//   warps 12-14 producer: cp.async X (and mask) tile → stage (TMA: one thread)
//   warp 15     TMEM owner; lane 0 issues the MMAs, software-pipelined as
//               hi(t) · lo(t-1) so the tensor core runs while tile t converts
// Accumulators: two buffers of NT_ columns at TMEM column 256.
constexpr int DT_WARPS = 16;  // 4 per SM sub-partition: up to 128 registers per thread
constexpr int DT_THREADS = DT_WARPS * 32;
constexpr int DT_PROD = 96;   // producer threads (warps 12-14)
constexpr int DT_CONV = 128;  // converter threads (warps 8-11)
constexpr int DT_EPI = 256;   // epilogue threads (warps 0-7)
constexpr int DT_MAX_STAGES = 4;

namespace {



// D (tmem) (+)= A (tmem) · B (smem descriptor), kind::tf32
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}



// X rows [m0, m0+N) (through the row list) into a K-major SWIZZLE_128B tile.
__device__ __forceinline__ void load_x_rows(uint32_t stage, const float* __restrict__ X, int ldx,
                                            const int* __restrict__ rows, int n_rows, int m0, int N, int kc, int tid) {
  for (int idx = tid; idx < N * kc; idx += DT_PROD) {
    const int r = idx / kc, c = idx - r * kc;   // a row's chunks are consecutive lanes (coalesced)
    const int i = m0 + r;
    const bool ok = i < n_rows;
    const int xr = ok ? (rows ? __ldg(rows + i) : i) : 0;
    cp16(stage + sw128_off(r, c, N), X + (size_t)xr * ldx + 4 * c, ok);
  }
}

// Mask rows (H_prev of the backward epilogue) into a row-major [N][mpad] tile.
__device__ __forceinline__ void load_mask_rows(uint32_t stage, const float* __restrict__ Hm, int ldhm,
                                               const int* __restrict__ rows, int n_rows, int m0, int N, int mpad,
                                               int tid) {
  const int c4 = mpad / 4;
  for (int idx = tid; idx < N * c4; idx += DT_PROD) {
    const int r = idx / c4, c = idx - r * c4;
    const int i = m0 + r;
    const bool ok = i < n_rows;
    const int hr = ok ? (rows ? __ldg(rows + i) : i) : 0;
    cp16(stage + (uint32_t)(r * mpad + 4 * c) * 4, Hm + (size_t)hr * ldhm + 4 * c, ok);
  }
}

}  // namespace

// TMA (rows == nullptr): one thread of warp 12 streams each tile with Kb/32
// SWIZZLE_128B boxes of 32 floats × NT_ rows (out-of-range K and rows arrive
// as zeros) plus, masked, one box of the mask rows; completion is counted by
// the stage's mbarrier (expect_tx), so loads run up to S tiles ahead.
// MK (mask kind): 0 act(X·W); 1 ⊙σ'(Hm) with Hm fp32 rows (ldhm floats);
// 2 ⊙σ'(H) from packed sign bits (Hm = uint32 words, ldhm words per row, bit m
// of word m/32 = (H[m] > 0)), which the forward writes through `bits_out`.
template <bool RELU, int MK, bool TMA>
__global__ void __launch_bounds__(DT_THREADS, 1)
    k_dense_tc(const float* __restrict__ X, int ldx, const int* __restrict__ rows, int n_rows, int K,
               const float* __restrict__ W, int ldw, int w_nk, int M, int NT_, int S, float* __restrict__ Y,
               int ldy, const float* __restrict__ Hm, int ldhm, uint32_t* __restrict__ bits_out, int ld_bits,
               const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmm,
               const EpiPack pk) {
  constexpr bool MASKED = MK != 0;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // swizzle atoms need 1024-byte alignment: align by hand (the launch adds
  // SMEM_ALIGN_PAD bytes) rather than trust the placement of the dynamic region
  uint8_t* const smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bars[4 * DT_MAX_STAGES + 4];
  __shared__ uint32_t tmem_base_slot;
  const int Kp = (K + 7) & ~7, kc = (K + 3) / 4;  // MMA K extent, loaded chunks per row
  const int Kb = (K + 31) & ~31;                  // smem K extent (whole 128-byte swizzle lines)
  const int mpad = (M + 3) & ~3;                  // mask tile row stride (floats)
  const uint32_t x_bytes = (uint32_t)NT_ * Kb * 4;
  const int mrow = MK == 2 ? ldhm : mpad;           // mask tile row: floats (MK 1) or words (MK 2)
  const uint32_t m_bytes = MASKED ? (uint32_t)NT_ * mrow * 4 : 0;
  const uint32_t st_bytes = (x_bytes + m_bytes + 1023) & ~1023u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles = (n_rows + NT_ - 1) / NT_;
  // barriers: full[S] hi_done[S] lo_ready[S] empty[S] | acc_full[2] acc_empty[2]
  auto bar = [&](int kind, int i) { return smem_u32(&bars[kind * DT_MAX_STAGES + i]); };
  auto abar = [&](int kind, int i) { return smem_u32(&bars[4 * DT_MAX_STAGES + 2 * kind + i]); };

  // K pad chunks of every X stage are never loaded: zero them once
  const int pad_ch = Kp / 4 - kc;
  for (int idx = threadIdx.x; idx < S * NT_ * pad_ch; idx += DT_THREADS) {
    const int sidx = idx / (NT_ * pad_ch), rem = idx % (NT_ * pad_ch);
    const int r = rem % NT_, c = kc + rem / NT_;
    *reinterpret_cast<float4*>(smem + sidx * st_bytes + sw128_off(r, c, NT_)) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (warp == 15) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&tmem_base_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(bar(0, i), TMA ? 1 : DT_PROD);
      mbar_init(bar(1, i), 1);
      mbar_init(bar(2, i), DT_CONV);
      mbar_init(bar(3, i), MASKED ? 1 + DT_EPI : 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(abar(0, i), 1);
      mbar_init(abar(1, i), DT_EPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_async_smem();
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = tmem_base_slot;
  const uint32_t acc0 = tmem + 256;

  if (warp < 4) {
    // Wᵀ hi → columns [0, Kp), lo → [Kp, 2Kp): lane m = output feature, column k.
    // Element (m, k) = W[k][m] (w_nk: W[m][k]); pad features / K zero.
    const int m = warp * 32 + lane;
    for (int c0 = 0; c0 < Kp; c0 += 8) {
      uint32_t hi[8], lo[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int k = c0 + e;
        const float v = (m < M && k < K) ? __ldg(W + (w_nk ? (size_t)m * ldw + k : (size_t)k * ldw + m)) : 0.0f;
        hi[e] = __float_as_uint(v);
        lo[e] = __float_as_uint(tf32_lo(v));
      }
      const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(hi[0]),
                   "r"(hi[1]), "r"(hi[2]), "r"(hi[3]), "r"(hi[4]), "r"(hi[5]), "r"(hi[6]), "r"(hi[7])
                   : "memory");
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta + Kp),
                   "r"(lo[0]), "r"(lo[1]), "r"(lo[2]), "r"(lo[3]), "r"(lo[4]), "r"(lo[5]), "r"(lo[6]), "r"(lo[7])
                   : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();

  if (TMA && warp >= 12 && warp < 15) {
    // ---------------- producer (TMA)
    if (warp == 12 && lane == 0) {
      const uint32_t tx = (uint32_t)(Kb / 32) * NT_ * 128 + m_bytes;
      int t = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++t) {
        const int s = t % S;
        if (t >= S) mbar_wait(bar(3, s), (uint32_t)(t / S - 1) & 1u);
        const uint32_t st = smem_u32(smem + s * st_bytes);
        mbar_expect_tx(bar(0, s), tx);
        for (int j = 0; j < Kb / 32; ++j) tma_load_2d(st + j * NT_ * 128, &tmx, 32 * j, tile * NT_, bar(0, s));
        if (MASKED) tma_load_2d(st + x_bytes, &tmm, 0, tile * NT_, bar(0, s));
      }
    }
    __syncwarp();
  } else if (warp >= 12 && warp < 15) {
    // ---------------- producer (cp.async, row list)
    const int tid = threadIdx.x - 384;
    int t = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++t) {
      const int s = t % S;
      if (t >= S) mbar_wait(bar(3, s), (uint32_t)(t / S - 1) & 1u);
      const uint32_t st = smem_u32(smem + s * st_bytes);
      load_x_rows(st, X, ldx, rows, n_rows, tile * NT_, NT_, kc, tid);
      if (MASKED) load_mask_rows(st + x_bytes, Hm, ldhm, rows, n_rows, tile * NT_, NT_, mrow, tid);
      asm volatile("cp.async.commit_group;" ::: "memory");
      if (t >= 1) {
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        fence_async_smem();
        mbar_arrive(bar(0, (t - 1) % S));
      }
    }
    if (t >= 1) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      fence_async_smem();
      mbar_arrive(bar(0, (t - 1) % S));
    }
  } else if (warp >= 8 && warp < 12) {
    // ---------------- lo(x) converter
    const int tid = threadIdx.x - 256;
    int t = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++t) {
      const int s = t % S;
      const uint32_t par = (uint32_t)(t / S) & 1u;
      mbar_wait(bar(0, s), par);  // every producer's copies visible
      mbar_wait(bar(1, s), par);  // hi MMAs have read the tile
      uint8_t* xs = smem + s * st_bytes;
      for (int idx = tid; idx < NT_ * kc; idx += DT_CONV) {
        const int r = idx % NT_, c = idx / NT_;
        float4* q = reinterpret_cast<float4*>(xs + sw128_off(r, c, NT_));
        const float4 v = *q;
        *q = make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w));
      }
      fence_async_smem();
      mbar_arrive(bar(2, s));
    }
  } else if (warp == 15) {
    // ---------------- MMA issuer: hi(t) then lo(t-1)
    if (lane == 0) {
      const uint32_t idesc = idesc_tf32(128, NT_);
      const int ksteps = Kp / 8;
      int t = 0;
      for (int tile = blockIdx.x;; tile += gridDim.x, ++t) {
        const bool live = tile < n_tiles;
        if (live) {
          const int s = t % S, b = t & 1;
          const uint32_t xs = smem_u32(smem + s * st_bytes);
          mbar_wait(bar(0, s), (uint32_t)(t / S) & 1u);
          if (t >= 2) mbar_wait(abar(1, b), (uint32_t)((t >> 1) - 1) & 1u);
          tc_after_sync();
          const uint32_t d = acc0 + (uint32_t)(b * NT_);
          for (int k = 0; k < ksteps; ++k) {
            const uint64_t db = sw128_desc(xs, k, NT_);
            mma_tf32_ts(d, tmem + 8 * k, db, idesc, k > 0);
            mma_tf32_ts(d, tmem + Kp + 8 * k, db, idesc, 1);
          }
          mma_commit(bar(1, s));
        }
        if (t >= 1) {
          const int tp = t - 1, sp = tp % S, bp = tp & 1;
          const uint32_t xs = smem_u32(smem + sp * st_bytes);
          mbar_wait(bar(2, sp), (uint32_t)(tp / S) & 1u);
          tc_after_sync();
          const uint32_t d = acc0 + (uint32_t)(bp * NT_);
          for (int k = 0; k < ksteps; ++k) mma_tf32_ts(d, tmem + 8 * k, sw128_desc(xs, k, NT_), idesc, 1);
          mma_commit(bar(3, sp));
          mma_commit(abar(0, bp));
        }
        if (!live) break;
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue: warp e drains TMEM lanes 32(e%4).. (features),
    // columns (tile rows) of its half e/4 of the tile
    const int q = warp & 3, hs = warp >> 2;
    const int span = NT_ / 2;
    const int m = q * 32 + lane;
    const bool m_out = m < ldy, m_mask = m < mpad;
    int t = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++t) {
      const int s = t % S, b = t & 1;
      mbar_wait(abar(0, b), (uint32_t)(t >> 1) & 1u);
      if (MASKED) mbar_wait(bar(0, s), (uint32_t)(t / S) & 1u);
      tc_after_sync();
      const float* ms = reinterpret_cast<const float*>(smem + s * st_bytes + x_bytes);
      const uint32_t* mw = reinterpret_cast<const uint32_t*>(ms);
      const int i0 = tile * NT_;
      // drain this warp's half of the accumulator into registers first and
      // release it, so the MMAs of tile t+2 overlap the stores of tile t
      const int ng = span / 16;
      uint32_t v[4][16];
#pragma unroll
      for (int gi = 0; gi < 4; ++gi) {
        if (gi < ng) {
          const uint32_t taddr = acc0 + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * NT_ + hs * span + 16 * gi);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(v[gi][0]), "=r"(v[gi][1]), "=r"(v[gi][2]), "=r"(v[gi][3]), "=r"(v[gi][4]), "=r"(v[gi][5]),
                "=r"(v[gi][6]), "=r"(v[gi][7]), "=r"(v[gi][8]), "=r"(v[gi][9]), "=r"(v[gi][10]), "=r"(v[gi][11]),
                "=r"(v[gi][12]), "=r"(v[gi][13]), "=r"(v[gi][14]), "=r"(v[gi][15])
              : "r"(taddr));
        }
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      tc_before_sync();
      mbar_arrive(abar(1, b));
#pragma unroll
      for (int gi = 0; gi < 4; ++gi) {
        const int n0 = hs * span + 16 * gi;
        if (gi >= ng || i0 + n0 >= n_rows) continue;
        float o[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          o[j] = __uint_as_float(v[gi][j]);
          if (MK == 1) {
            const float hv = m_mask ? ms[(n0 + j) * mpad + m] : 1.0f;
            o[j] = RELU ? (hv > 0.0f ? o[j] : 0.0f) : o[j];
          } else if (MK == 2) {
            const uint32_t w = mw[(n0 + j) * ldhm + q];
            o[j] = RELU ? (((w >> lane) & 1u) ? o[j] : 0.0f) : o[j];
          } else if (RELU) {
            o[j] = fmaxf(o[j], 0.0f);
          }
        }
        if (MK == 0 && RELU && bits_out != nullptr) {
          // σ' of this layer's output for the backward pass: one ballot per row
          uint32_t mine = 0;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const uint32_t bw = __ballot_sync(0xffffffffu, o[j] > 0.0f);
            if (lane == j) mine = bw;
          }
          const int i = i0 + n0 + lane;
          if (lane < 16 && i < n_rows) bits_out[(size_t)(rows ? __ldg(rows + i) : i) * ld_bits + q] = mine;
        }
        if (!m_out) continue;
        if (rows == nullptr && i0 + n0 + 16 <= n_rows) {
          float* p = Y + (size_t)(i0 + n0) * ldy + m;
#pragma unroll
          for (int j = 0; j < 16; ++j) p[(size_t)j * ldy] = o[j];
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int i = i0 + n0 + j;
            if (i < n_rows) Y[(size_t)(rows ? __ldg(rows + i) : i) * ldy + m] = o[j];
          }
        }
      }
      if (MASKED) mbar_arrive(bar(3, s));
    }
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  epi_forward(pk, Y, ldy, rows, n_rows, NT_, mpad / 4);
  epi_signal(pk);
  if (warp == 15) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

namespace {
constexpr size_t DT_SMEM_MAX = 227 * 1024 - 1024;  // leaves room for SMEM_ALIGN_PAD

// Rows per tile (MMA N) and stage count: the largest tile of 128/64/32 rows
// for which enough stages fit (up to DT_MAX_STAGES).  The cp.async producer
// needs three: it signals tile t-1 only after it has waited for the stage of
// tile t to drain (lo MMAs of tile t-S), while the MMA issuer needs tile t-1
// before it issues those lo MMAs of tile t-2 — with S = 2 that is a cycle.
// TMA completion does not wait on later tiles, so two suffice there.
// mask_row: floats (or bit words) of the mask tile per row, 0 when unmasked.
int dense_tc_tile(int d_in, int d_out, int mask_row, bool tma, int* stages, size_t* smem_out) {
  if (d_in > 128 || d_out > 128) return 0;  // Wᵀ hi+lo ≤ 256 TMEM columns; one 128-lane half
  const bool masked = mask_row > 0;
  const int Kb = (d_in + 31) & ~31;
  for (int nt = 128; nt >= 32; nt >>= 1) {
    const size_t st = ((size_t)nt * (Kb + mask_row) * 4 + 1023) & ~(size_t)1023;
    const int s = (int)std::min<size_t>(DT_MAX_STAGES, DT_SMEM_MAX / st);
    // masked: the epilogue releases a stage only after reading its mask rows,
    // so two stages would serialise load, MMA and epilogue — keep three
    if (s >= (tma && !masked ? 2 : 3)) {
      *stages = s;
      *smem_out = s * st;
      return nt;
    }
  }
  return 0;
}
}  // namespace

bool dense_tc_applies(int d_in, int d_out) {
  if (g_dense_mode == 1) return false;
  int stages = 0;
  size_t smem = 0;
  // the backward form carries a mask tile: require that it fits too
  const bool fits = dense_tc_tile(d_in, d_out, (d_out + 3) & ~3, false, &stages, &smem) > 0;
  if (g_dense_mode == 2) return fits;
  return fits && d_in >= 32 && d_out >= 32;
}

namespace {
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      p = nullptr;
    }
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

}  // namespace

// 2-D fp32 tensor map: dim0 = `cols` contiguous floats, dim1 = `n_rows` rows
// `ld` floats apart; box {box0, box1}; out-of-range elements read as zero.
bool tmap_2d(CUtensorMap* m, const float* base, int cols, int n_rows, int ld, int box0, int box1,
             CUtensorMapSwizzle sw) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)n_rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  const cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)box1};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int launch_dense_tc(const float* x, int ldx, const int* rows, int n_rows, int d_in, const float* w, int d_out,
                    float* y, int ldy, int act, cudaStream_t st, const float* w_nk, int ld_wnk, const float* hmask,
                    int ldhm, const uint32_t* hbits, int ld_hbits, uint32_t* bits_out, int ld_bits_out,
                    const EpiPack* pk) {
  GCNB_REQUIRE(!pk || !pk->map_ptr || rows == nullptr, "dense (tcgen05): a fused halo pack needs rows 0..n-1");
  const int mk = hbits ? 2 : hmask ? 1 : 0;
  const int mpad = (d_out + 3) & ~3;
  const int mask_row = mk == 2 ? ld_hbits : mk == 1 ? mpad : 0;
  const float* mptr = mk == 2 ? reinterpret_cast<const float*>(hbits) : hmask;
  const int mld = mk == 2 ? ld_hbits : ldhm;
  GCNB_REQUIRE(mk != 1 || ldhm >= mpad, "dense (tcgen05): mask stride too small");
  GCNB_REQUIRE(mk != 2 || (ld_hbits % 4 == 0 && ld_hbits * 32 >= d_out), "dense (tcgen05): mask-bit stride");
  GCNB_REQUIRE(!bits_out || (act == GCNB_ACT_RELU && mk == 0 && ld_bits_out * 32 >= d_out),
               "dense (tcgen05): sign bits are written for an unmasked ReLU transform only");
  CUtensorMap tmx, tmm;
  std::memset(&tmx, 0, sizeof(tmx));
  std::memset(&tmm, 0, sizeof(tmm));
  int stages = 0;
  size_t smem = 0;
  bool tma = rows == nullptr && n_rows > 0;
  int nt = tma ? dense_tc_tile(d_in, d_out, mask_row, true, &stages, &smem) : 0;
  if (tma) {
    tma = nt > 0 && tmap_2d(&tmx, x, d_in, n_rows, ldx, 32, nt, CU_TENSOR_MAP_SWIZZLE_128B) &&
          (mk == 0 || tmap_2d(&tmm, mptr, mask_row, n_rows, mld, mask_row, nt, CU_TENSOR_MAP_SWIZZLE_NONE));
  }
  if (!tma) nt = dense_tc_tile(d_in, d_out, mask_row, false, &stages, &smem);
  GCNB_REQUIRE(nt > 0, "dense (tcgen05): widths %d -> %d not supported", d_in, d_out);
  const bool relu = act == GCNB_ACT_RELU;
  using Fn = void (*)(const float*, int, const int*, int, int, const float*, int, int, int, int, int, float*, int,
                      const float*, int, uint32_t*, int, const CUtensorMap, const CUtensorMap, const EpiPack);
#define GCNB_DT_PICK(T)                                                                              \
  (mk == 2 ? (relu ? k_dense_tc<true, 2, T> : k_dense_tc<false, 2, T>)                               \
           : mk == 1 ? (relu ? k_dense_tc<true, 1, T> : k_dense_tc<false, 1, T>)                     \
                     : (relu ? k_dense_tc<true, 0, T> : k_dense_tc<false, 0, T>))
  Fn fn = tma ? GCNB_DT_PICK(true) : GCNB_DT_PICK(false);
#undef GCNB_DT_PICK
  smem += SMEM_ALIGN_PAD;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int tiles = (n_rows + nt - 1) / nt;
  const int grid = std::max(1, std::min(tiles, num_sms()));
  fn<<<grid, DT_THREADS, smem, st>>>(x, ldx, rows, n_rows, d_in, w_nk ? w_nk : w, w_nk ? ld_wnk : round4(d_out),
                                     w_nk ? 1 : 0, d_out, nt, stages, y, ldy, mptr, mld, bits_out, ld_bits_out, tmx,
                                     tmm, pk ? *pk : EpiPack{});
  GCNB_AFTER_LAUNCH(tma ? "dense (tcgen05 3xTF32, TMA)" : "dense (tcgen05 3xTF32)");
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
//   ΔW += H·A + lo(H)·A + H·lo(A)
// Warp-specialised pipeline over DW_T-row tiles and S stages (raw H, raw A,
// lo(H), lo(A) per stage):
//   warps 0-3  converter (lo buffers of each landed stage), then the final
//              TMEM → partial epilogue
//   warps 4-7  producer (cp.async rows, zero-filled past the end)
//   warp 8     TMEM owner; lane 0 issues the 3 × DW_T/8 MMAs of a tile
constexpr int DW_T = 32;            // rows per tile (4 MMA K-steps of 8 rows)
constexpr int DW_WARPS = 9;
constexpr int DW_THREADS = DW_WARPS * 32;
constexpr int DW_MAX_STAGES = 4;
constexpr int DW_NA_H = 4;          // M = 128 features = 4 atoms
constexpr int DW_CHUNK = 8;         // tiles (8 × 32 = 256 rows) per TMEM accumulation chunk
constexpr int DW_REG_COLS = 128;    // ΔW columns accumulated in registers (the rest in the partial row)

namespace {

// Byte offset of feature m of tile row k in an MN-major SW128_32B tile: each
// 32-feature atom holds the tile's DW_T rows contiguously (128 bytes per row,
// its 32-byte granules XOR-permuted by k & 3) — the layout a TMA box of
// {32 features, DW_T rows} with SWIZZLE_128B_ATOM_32B writes.
__device__ __forceinline__ uint32_t mn_off(int k, int m) {
  return (uint32_t)((m >> 5) * (DW_T * 128) + k * 128 + ((((m & 31) >> 3) ^ (k & 3)) << 5) + ((m & 7) << 2));
}

__device__ __forceinline__ void load_rows_mn(uint32_t stage, const float* __restrict__ X, int ldx,
                                             const int* __restrict__ rows, int n_rows, int m0, int kc, int tid) {
  for (int idx = tid; idx < DW_T * kc; idx += 128) {
    const int k = idx / kc, c = idx - k * kc;
    const int i = m0 + k;
    const bool ok = i < n_rows;  // rows past the end must be zero: they are summed over
    const int xr = ok ? (rows ? __ldg(rows + i) : i) : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(stage + mn_off(k, 4 * c)),
                 "l"(X + (size_t)xr * ldx + 4 * c), "r"(ok ? 16 : 0)
                 : "memory");
  }
}

__device__ __forceinline__ uint64_t desc_mn_sw32(uint32_t addr) {
  // LBO = next 32-feature atom (DW_T rows × 128 B), SBO = next 4-row group (512 B), layout type 1
  return smem_desc(addr, DW_T * 128, 512) | (1ull << 61);
}

__device__ __forceinline__ void lo_copy(uint8_t* dst, const uint8_t* src, int bytes, int tid) {
  for (int i = tid; i < bytes / 16; i += 128) {
    const float4 v = reinterpret_cast<const float4*>(src)[i];
    reinterpret_cast<float4*>(dst)[i] = make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w));
  }
}

struct DwGeom {
  int na_a, h_bytes, a_bytes, st_bytes, stages;
};

__host__ __device__ inline DwGeom dw_geom(int d_k) {
  DwGeom g;
  const int Np = (d_k + 15) & ~15;
  g.na_a = (Np + 31) / 32;
  g.h_bytes = (DW_T / 4) * DW_NA_H * 512;
  g.a_bytes = (DW_T / 4) * g.na_a * 512;
  g.st_bytes = 2 * (g.h_bytes + g.a_bytes);
  const int fit = (int)((size_t)(220 * 1024) / (size_t)g.st_bytes);
  g.stages = fit < DW_MAX_STAGES ? fit : DW_MAX_STAGES;
  return g;
}

}  // namespace

template <bool TMA>
__global__ void __launch_bounds__(DW_THREADS, 1)
    k_dw_tc(const float* __restrict__ H, int ldh, int d_prev, const float* __restrict__ A, int lda, int d_k,
            const int* __restrict__ rows, int n_rows, float* __restrict__ partials, int n_slots,
            const __grid_constant__ CUtensorMap tmh, const __grid_constant__ CUtensorMap tma_) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // swizzle atoms need 1024-byte alignment: align by hand (the launch adds
  // SMEM_ALIGN_PAD bytes) rather than trust the placement of the dynamic region
  uint8_t* const smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bars[3 * DW_MAX_STAGES + 1];
  __shared__ uint64_t accb[4];  // accumulator full[2] (MMA commit) / empty[2] (128 epilogue arrivals)
  __shared__ uint32_t tmem_base_slot;
  const DwGeom g = dw_geom(d_k);
  const int S = g.stages;
  const int Np = (d_k + 15) & ~15;
  const int kc_h = (d_prev + 3) / 4, kc_a = (d_k + 3) / 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles = (n_rows + DW_T - 1) / DW_T;
  // two accumulators of acc_cols columns: chunk c of DW_CHUNK tiles accumulates in
  // buffer c & 1 while the epilogue drains chunk c - 1 into fp32 registers
  const uint32_t acc_cols = Np <= 32 ? 32 : Np <= 64 ? 64 : Np <= 128 ? 128 : 256;
  const uint32_t tmem_cols = 2 * acc_cols;
  // stage s: [H | A | lo(H) | lo(A)]
  auto st_h = [&](int s) { return smem + s * g.st_bytes; };
  auto st_a = [&](int s) { return smem + s * g.st_bytes + g.h_bytes; };
  auto st_hl = [&](int s) { return smem + s * g.st_bytes + g.h_bytes + g.a_bytes; };
  auto st_al = [&](int s) { return smem + s * g.st_bytes + 2 * g.h_bytes + g.a_bytes; };
  // barriers: full[S] (producers) conv[S] (converters) empty[S] (MMA commit) | done
  auto bar = [&](int kind, int i) { return smem_u32(&bars[kind * DW_MAX_STAGES + i]); };
  const uint32_t b_done = smem_u32(&bars[3 * DW_MAX_STAGES]);

  // pad features (never loaded) must read as zero in every buffer: clear once
  for (int i = threadIdx.x; i < S * g.st_bytes / 16; i += DW_THREADS)
    reinterpret_cast<float4*>(smem)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_slot)),
                 "r"(tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(bar(0, i), TMA ? 1 : 128);
      mbar_init(bar(1, i), 128);
      mbar_init(bar(2, i), 1);
    }
    mbar_init(b_done, 1);
    mbar_init(smem_u32(&accb[0]), 1);
    mbar_init(smem_u32(&accb[1]), 1);
    mbar_init(smem_u32(&accb[2]), 128);
    mbar_init(smem_u32(&accb[3]), 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_async_smem();
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = tmem_base_slot;

  if (TMA && warp >= 4 && warp < 8) {
    // ---------------- producer (TMA: one box per 32-feature atom of H and A)
    if (warp == 4 && lane == 0) {
      const uint32_t tx = (uint32_t)(DW_NA_H + g.na_a) * DW_T * 128;
      int t = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++t) {
        const int s = t % S;
        if (t >= S) mbar_wait(bar(2, s), (uint32_t)(t / S - 1) & 1u);
        mbar_expect_tx(bar(0, s), tx);
        for (int a = 0; a < DW_NA_H; ++a)
          tma_load_2d(smem_u32(st_h(s)) + a * DW_T * 128, &tmh, 32 * a, tile * DW_T, bar(0, s));
        for (int a = 0; a < g.na_a; ++a)
          tma_load_2d(smem_u32(st_a(s)) + a * DW_T * 128, &tma_, 32 * a, tile * DW_T, bar(0, s));
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 8) {
    // ---------------- producer (cp.async, row list)
    const int tid = threadIdx.x - 128;
    int t = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++t) {
      const int s = t % S;
      if (t >= S) mbar_wait(bar(2, s), (uint32_t)(t / S - 1) & 1u);
      load_rows_mn(smem_u32(st_h(s)), H, ldh, rows, n_rows, tile * DW_T, kc_h, tid);
      load_rows_mn(smem_u32(st_a(s)), A, lda, rows, n_rows, tile * DW_T, kc_a, tid);
      asm volatile("cp.async.commit_group;" ::: "memory");
      if (t >= 1) {
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        fence_async_smem();
        mbar_arrive(bar(0, (t - 1) % S));
      }
    }
    if (t >= 1) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      fence_async_smem();
      mbar_arrive(bar(0, (t - 1) % S));
    }
  } else if (warp == 8) {
    // ---------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_tf32(128, Np) | (1u << 15) | (1u << 16);  // A and B MN-major
      const uint32_t kstep = 2 * 512;  // 8 rows = two 4-row groups
      int t = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++t) {
        const int s = t % S;
        const int c = t / DW_CHUNK, buf = c & 1;
        const bool first = t % DW_CHUNK == 0;
        const bool last = t % DW_CHUNK == DW_CHUNK - 1 || tile + (int)gridDim.x >= n_tiles;
        if (first && c >= 2) {  // the epilogue has drained chunk c - 2 out of this buffer
          mbar_wait(smem_u32(&accb[2 + buf]), (uint32_t)(c / 2 - 1) & 1u);
          tc_after_sync();
        }
        mbar_wait(bar(1, s), (uint32_t)(t / S) & 1u);
        tc_after_sync();
        const uint32_t acc = tmem + (uint32_t)buf * acc_cols;
        const uint32_t ha = smem_u32(st_h(s)), hl = smem_u32(st_hl(s));
        const uint32_t aa = smem_u32(st_a(s)), al = smem_u32(st_al(s));
        for (int k = 0; k < DW_T / 8; ++k) {
          const uint64_t dh = desc_mn_sw32(ha + k * kstep);
          const uint64_t da = desc_mn_sw32(aa + k * kstep);
          mma_tf32(acc, dh, da, idesc, (!first || k > 0) ? 1u : 0u);
          mma_tf32(acc, desc_mn_sw32(hl + k * kstep), da, idesc, 1u);
          mma_tf32(acc, dh, desc_mn_sw32(al + k * kstep), idesc, 1u);
        }
        mma_commit(bar(2, s));
        if (last) mma_commit(smem_u32(&accb[buf]));
      }
      mma_commit(b_done);
    }
    __syncwarp();
  } else {
    // ---------------- converter (warps 0-3), and the epilogue: every chunk of
    // DW_CHUNK tiles (K = 256 rows) is drained from TMEM and added into fp32
    // registers (round-to-nearest).  The tensor core's own accumulation does
    // not round to nearest, so its error grows with K: one accumulator over
    // the CTA's ~16 K rows measured 3e-4 relative on products ΔW², chunks of
    // 256 rows keep it at the level of the products themselves (~2^-21).
    const int tid = threadIdx.x;
    const int ld_k = (d_k + 3) & ~3;
    const int m = warp * 32 + lane;
    float* out = partials + (size_t)blockIdx.x * d_prev * ld_k + (size_t)m * ld_k;
    float accr[DW_REG_COLS];
#pragma unroll
    for (int e = 0; e < DW_REG_COLS; ++e) accr[e] = 0.0f;
    // columns >= DW_REG_COLS (d_k > 128) accumulate in this thread's row of the partial slot
    for (int c = DW_REG_COLS; c < ld_k; ++c)
      if (m < d_prev) out[c] = 0.0f;
    auto drain = [&](int c) {
      const int buf = c & 1;
      mbar_wait(smem_u32(&accb[buf]), (uint32_t)(c / 2) & 1u);
      tc_after_sync();
      const uint32_t base = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)buf * acc_cols;
#pragma unroll
      for (int c0 = 0; c0 < 256; c0 += 8) {
        if (c0 < Np) {
          uint32_t v[8];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
              : "r"(base + (uint32_t)c0));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            if (c0 + e < DW_REG_COLS) accr[c0 + e] += __uint_as_float(v[e]);
            else if (m < d_prev && c0 + e < ld_k) out[c0 + e] += __uint_as_float(v[e]);
          }
        }
      }
      tc_before_sync();
      mbar_arrive(smem_u32(&accb[2 + buf]));
    };
    int t = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++t) {
      const int s = t % S;
      mbar_wait(bar(0, s), (uint32_t)(t / S) & 1u);
      lo_copy(st_hl(s), st_h(s), g.h_bytes, tid);
      lo_copy(st_al(s), st_a(s), g.a_bytes, tid);
      fence_async_smem();
      mbar_arrive(bar(1, s));
      // one chunk behind: chunk c is drained once chunk c + 1 is fully converted
      if ((t + 1) % DW_CHUNK == 0 && t + 1 >= 2 * DW_CHUNK) drain((t + 1) / DW_CHUNK - 2);
    }
    const int n_chunks = (t + DW_CHUNK - 1) / DW_CHUNK;
    for (int c = std::max(0, t / DW_CHUNK - 1); c < n_chunks; ++c) drain(c);  // the ones the loop left
    if (n_tiles > (int)blockIdx.x) mbar_wait(b_done, 0);
    tc_after_sync();
    // partial[m][n] for m < d_prev, n < round4(d_k)
    if (m < d_prev) {
#pragma unroll
      for (int e = 0; e < DW_REG_COLS; ++e)
        if (e < ld_k) out[e] = accr[e];
    }
  }
  // slots beyond the grid (the caller sized the partials for another engine) are zero
  {
    const int ld_k = (d_k + 3) & ~3;
    const size_t slot = (size_t)d_prev * ld_k;
    for (int sl = blockIdx.x + gridDim.x; sl < n_slots; sl += gridDim.x)
      for (size_t e = threadIdx.x; e < slot; e += DW_THREADS) partials[sl * slot + e] = 0.0f;
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols) : "memory");
}

// ---------------------------------------------------------------------------
// k_dw_tc2: the same partials with Hᵀ (hi and lo) written to TENSOR memory as
// the MMA A operand (tcgen05.mma with A from TMEM), contiguous row ranges by
// TMA.  k_dw_tc keeps hi/lo of both operands in shared memory, so every tile
// costs TMA writes + the converters' read/write + three MMAs' operand reads:
// ~140 KB of shared-memory traffic per 32-row tile, which bounds it near 40 % of
// HBM (ncu, products).  Here H arrives row-major (one TMA box per tile), the
// converter thread of feature m reads its 32 values (conflict-free: a warp
// reads one 128-byte row segment per step) and stores hi / lo to its own TMEM
// lane; only A and lo(A) stay in shared memory.  Smaller stages (no lo(H), no
// swizzle atoms for H) and no MMA reads of H: deeper pipeline, ~half the traffic.
// TMEM columns: [0, 2·acc_cols) accumulators (double-buffered 256-row chunks,
// drained into fp32 registers as in k_dw_tc), then 64 columns (hi | lo of the
// 32-row K tile) per stage.
//   warps 0-3  converter (Hᵀ → TMEM, lo(A) in place), then the epilogue
//   warp 4     producer (one thread: TMA boxes for H and A)
//   warp 5     TMEM owner; lane 0 issues the 3 × 4 MMAs of a tile
constexpr int DW2_WARPS = 6;
constexpr int DW2_THREADS = DW2_WARPS * 32;
constexpr int DW2_MAX_STAGES = 6;

namespace {
struct Dw2Geom {
  int na_a, hstride, h_bytes, a_bytes, st_bytes, stages, acc_cols;
};

__host__ __device__ inline Dw2Geom dw2_geom(int d_prev, int d_k) {
  Dw2Geom g;
  const int Np = (d_k + 15) & ~15;
  g.na_a = (Np + 31) / 32;
  g.hstride = (d_prev + 3) & ~3;
  g.h_bytes = ((DW_T * g.hstride * 4 + 1023) / 1024) * 1024;  // A atoms stay 1024-byte aligned
  g.a_bytes = g.na_a * DW_T * 128;
  g.st_bytes = g.h_bytes + 2 * g.a_bytes;
  g.acc_cols = Np <= 32 ? 32 : Np <= 64 ? 64 : Np <= 128 ? 128 : 256;
  const int by_smem = (int)((size_t)(220 * 1024) / (size_t)g.st_bytes);
  const int by_tmem = (512 - 2 * g.acc_cols) / 64;
  int st = by_smem < by_tmem ? by_smem : by_tmem;
  g.stages = st < DW2_MAX_STAGES ? st : DW2_MAX_STAGES;
  return g;
}
}  // namespace

__global__ void __launch_bounds__(DW2_THREADS, 1)
    k_dw_tc2(int d_prev, int d_k, int n_rows, float* __restrict__ partials, int n_slots,
             const __grid_constant__ CUtensorMap tmh, const __grid_constant__ CUtensorMap tma_) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // swizzle atoms need 1024-byte alignment: align by hand (the launch adds
  // SMEM_ALIGN_PAD bytes) rather than trust the placement of the dynamic region
  uint8_t* const smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bars[3 * DW2_MAX_STAGES + 1];
  __shared__ uint64_t accb[4];
  __shared__ uint32_t tmem_base_slot;
  const Dw2Geom g = dw2_geom(d_prev, d_k);
  const int S = g.stages;
  const int Np = (d_k + 15) & ~15;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles = (n_rows + DW_T - 1) / DW_T;
  const uint32_t acc_cols = g.acc_cols;
  auto st_h = [&](int s) { return smem + s * g.st_bytes; };
  auto st_a = [&](int s) { return smem + s * g.st_bytes + g.h_bytes; };
  auto st_al = [&](int s) { return smem + s * g.st_bytes + g.h_bytes + g.a_bytes; };
  auto bar = [&](int kind, int i) { return smem_u32(&bars[kind * DW2_MAX_STAGES + i]); };
  const uint32_t b_done = smem_u32(&bars[3 * DW2_MAX_STAGES]);
  // lo(A) pad columns (never loaded) must read as zero: clear once
  for (int i = threadIdx.x; i < S * g.st_bytes / 16; i += DW2_THREADS)
    reinterpret_cast<float4*>(smem)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (warp == 5) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&tmem_base_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(bar(0, i), 1);     // full: TMA
      mbar_init(bar(1, i), 128);   // converted
      mbar_init(bar(2, i), 1);     // empty: MMA commit
    }
    mbar_init(b_done, 1);
    mbar_init(smem_u32(&accb[0]), 1);
    mbar_init(smem_u32(&accb[1]), 1);
    mbar_init(smem_u32(&accb[2]), 128);
    mbar_init(smem_u32(&accb[3]), 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_async_smem();
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = tmem_base_slot;
  auto a_col = [&](int s) { return tmem + 2 * acc_cols + (uint32_t)(64 * s); };

  if (warp == 4) {
    // ---------------- producer
    if (lane == 0) {
      const uint32_t tx = (uint32_t)(DW_T * g.hstride * 4 + g.a_bytes);
      int t = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++t) {
        const int s = t % S;
        if (t >= S) mbar_wait(bar(2, s), (uint32_t)(t / S - 1) & 1u);
        mbar_expect_tx(bar(0, s), tx);
        tma_load_2d(smem_u32(st_h(s)), &tmh, 0, tile * DW_T, bar(0, s));
        for (int a = 0; a < g.na_a; ++a)
          tma_load_2d(smem_u32(st_a(s)) + a * DW_T * 128, &tma_, 32 * a, tile * DW_T, bar(0, s));
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ---------------- MMA issuer: D[m][n] += Σ_k Hᵀ[m][k] · A[k][n]
    if (lane == 0) {
      const uint32_t idesc = idesc_tf32(128, Np) | (1u << 16);  // A from TMEM (K-major), B MN-major
      const uint32_t kstep = 2 * 512;                            // 8 rows = two 4-row groups
      int t = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++t) {
        const int s = t % S;
        const int c = t / DW_CHUNK, buf = c & 1;
        const bool first = t % DW_CHUNK == 0;
        const bool last = t % DW_CHUNK == DW_CHUNK - 1 || tile + (int)gridDim.x >= n_tiles;
        if (first && c >= 2) {
          mbar_wait(smem_u32(&accb[2 + buf]), (uint32_t)(c / 2 - 1) & 1u);
          tc_after_sync();
        }
        mbar_wait(bar(1, s), (uint32_t)(t / S) & 1u);
        tc_after_sync();
        const uint32_t acc = tmem + (uint32_t)buf * acc_cols;
        const uint32_t ah = a_col(s), al = ah + 32;
        const uint32_t ba = smem_u32(st_a(s)), bl = smem_u32(st_al(s));
        for (int k = 0; k < DW_T / 8; ++k) {
          const uint64_t dhi = desc_mn_sw32(ba + k * kstep);
          mma_tf32_ts(acc, ah + 8 * k, dhi, idesc, (!first || k > 0) ? 1u : 0u);
          mma_tf32_ts(acc, al + 8 * k, dhi, idesc, 1u);
          mma_tf32_ts(acc, ah + 8 * k, desc_mn_sw32(bl + k * kstep), idesc, 1u);
        }
        mma_commit(bar(2, s));
        if (last) mma_commit(smem_u32(&accb[buf]));
      }
      mma_commit(b_done);
    }
    __syncwarp();
  } else {
    // ---------------- converter (warps 0-3: TMEM lanes 0-127 = features), then the epilogue
    const int tid = threadIdx.x;
    const int m = warp * 32 + lane;
    const int ld_k = (d_k + 3) & ~3;
    float* out = partials + (size_t)blockIdx.x * d_prev * ld_k + (size_t)m * ld_k;
    float accr[DW_REG_COLS];
#pragma unroll
    for (int e = 0; e < DW_REG_COLS; ++e) accr[e] = 0.0f;
    for (int c = DW_REG_COLS; c < ld_k; ++c)
      if (m < d_prev) out[c] = 0.0f;
    auto drain = [&](int c) {
      const int buf = c & 1;
      mbar_wait(smem_u32(&accb[buf]), (uint32_t)(c / 2) & 1u);
      tc_after_sync();
      const uint32_t base = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)buf * acc_cols;
#pragma unroll
      for (int c0 = 0; c0 < 256; c0 += 8) {
        if (c0 < Np) {
          uint32_t v[8];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
              : "r"(base + (uint32_t)c0));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            if (c0 + e < DW_REG_COLS) accr[c0 + e] += __uint_as_float(v[e]);
            else if (m < d_prev && c0 + e < ld_k) out[c0 + e] += __uint_as_float(v[e]);
          }
        }
      }
      tc_before_sync();
      mbar_arrive(smem_u32(&accb[2 + buf]));
    };
    int t = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++t) {
      const int s = t % S;
      mbar_wait(bar(0, s), (uint32_t)(t / S) & 1u);
      // Hᵀ hi / lo of this K tile → TMEM lane m, columns [a_col(s), +32) / [+32, +64).
      // (The MMAs of tile t - S, which read these columns, completed before the
      // producer refilled stage s: its TMA waited on their commit.)
      const float* hs = reinterpret_cast<const float*>(st_h(s));
      const uint32_t ta = a_col(s) + ((uint32_t)(warp * 32) << 16);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const float v = m < d_prev ? hs[(half * 16 + r) * g.hstride + m] : 0.0f;
          hi[r] = __float_as_uint(v);
          lo[r] = __float_as_uint(tf32_lo(v));
        }
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
            ::"r"(ta + 16 * half), "r"(hi[0]), "r"(hi[1]), "r"(hi[2]), "r"(hi[3]), "r"(hi[4]), "r"(hi[5]),
            "r"(hi[6]), "r"(hi[7]), "r"(hi[8]), "r"(hi[9]), "r"(hi[10]), "r"(hi[11]), "r"(hi[12]), "r"(hi[13]),
            "r"(hi[14]), "r"(hi[15])
            : "memory");
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
            ::"r"(ta + 32 + 16 * half), "r"(lo[0]), "r"(lo[1]), "r"(lo[2]), "r"(lo[3]), "r"(lo[4]), "r"(lo[5]),
            "r"(lo[6]), "r"(lo[7]), "r"(lo[8]), "r"(lo[9]), "r"(lo[10]), "r"(lo[11]), "r"(lo[12]), "r"(lo[13]),
            "r"(lo[14]), "r"(lo[15])
            : "memory");
      }
      lo_copy(st_al(s), st_a(s), g.a_bytes, tid);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      fence_async_smem();
      tc_before_sync();
      mbar_arrive(bar(1, s));
      if ((t + 1) % DW_CHUNK == 0 && t + 1 >= 2 * DW_CHUNK) drain((t + 1) / DW_CHUNK - 2);
    }
    const int n_chunks = (t + DW_CHUNK - 1) / DW_CHUNK;
    for (int c = std::max(0, t / DW_CHUNK - 1); c < n_chunks; ++c) drain(c);
    if (n_tiles > (int)blockIdx.x) mbar_wait(b_done, 0);
    tc_after_sync();
    if (m < d_prev) {
#pragma unroll
      for (int e = 0; e < DW_REG_COLS; ++e)
        if (e < ld_k) out[e] = accr[e];
    }
  }
  {
    const int ld_k = (d_k + 3) & ~3;
    const size_t slot = (size_t)d_prev * ld_k;
    for (int sl = blockIdx.x + gridDim.x; sl < n_slots; sl += gridDim.x)
      for (size_t e = threadIdx.x; e < slot; e += DW2_THREADS) partials[sl * slot + e] = 0.0f;
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  if (warp == 5) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

bool dw_tc_applies(int d_prev, int d_k) {
  if (g_dense_mode == 1) return false;
  return d_prev <= 128 && d_k <= 256 && dw_geom(d_k).stages >= 2;
}

int dw_tc_grid(int n_rows) { return std::max(1, std::min((n_rows + DW_T - 1) / DW_T, num_sms())); }

int launch_dw_tc(const float* h, int ldh, int d_prev, const float* a, int lda, int d_k, const int* rows, int n_rows,
                 float* partials, int n_slots, cudaStream_t st) {
  const int grid = std::min(dw_tc_grid(n_rows), n_slots);
  const DwGeom g = dw_geom(d_k);
  const size_t smem = (size_t)g.stages * g.st_bytes;
  CUtensorMap tmh, tma_;
  std::memset(&tmh, 0, sizeof(tmh));
  std::memset(&tma_, 0, sizeof(tma_));
  const bool tma = rows == nullptr && n_rows > 0 &&
                   tmap_2d(&tmh, h, d_prev, n_rows, ldh, 32, DW_T, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) &&
                   tmap_2d(&tma_, a, d_k, n_rows, lda, 32, DW_T, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  const Dw2Geom g2 = dw2_geom(d_prev, d_k);
  if (tma && g_dw_v2 && g2.stages >= 2) {
    // Hᵀ in TMEM (k_dw_tc2): H as plain row-major boxes of the whole (padded) row
    CUtensorMap tmh2;
    std::memset(&tmh2, 0, sizeof(tmh2));
    if (tmap_2d(&tmh2, h, d_prev, n_rows, ldh, g2.hstride, DW_T, CU_TENSOR_MAP_SWIZZLE_NONE)) {
      const size_t smem2 = (size_t)g2.stages * g2.st_bytes + SMEM_ALIGN_PAD;
      cudaFuncSetAttribute(k_dw_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
      k_dw_tc2<<<grid, DW2_THREADS, smem2, st>>>(d_prev, d_k, n_rows, partials, n_slots, tmh2, tma_);
      GCNB_AFTER_LAUNCH("bwd ΔW (tcgen05 3xTF32, Hᵀ in TMEM, TMA)");
      return GCNB_OK;
    }
  }
  auto fn = tma ? k_dw_tc<true> : k_dw_tc<false>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem + SMEM_ALIGN_PAD));
  fn<<<grid, DW_THREADS, smem + SMEM_ALIGN_PAD, st>>>(h, ldh, d_prev, a, lda, d_k, rows, n_rows, partials, n_slots,
                                                      tmh, tma_);
  GCNB_AFTER_LAUNCH(tma ? "bwd ΔW (tcgen05 3xTF32, TMA)" : "bwd ΔW (tcgen05 3xTF32)");
  return GCNB_OK;
}

}  // namespace gcnb

extern "C" int gcnb_set_dense_mode(int32_t mode) {
  GCNB_REQUIRE(mode >= 0 && mode <= 2, "dense mode must be 0 (auto), 1 (SIMT) or 2 (tensor core)");
  gcnb::g_dense_mode = mode;
  return GCNB_OK;
}

extern "C" int gcnb_set_dw_mode(int32_t v2) {
  gcnb::g_dw_v2 = v2 ? 1 : 0;
  return GCNB_OK;
}
