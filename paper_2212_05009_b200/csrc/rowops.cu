// Row-partitioned GCN layer kernels for sm_100a.
//
//   gcnb_spmm_f32       sparse.spmm                (sparse.py:196-207)
//   gcnb_fwd_layer_f32  runtime._fwd_compute       (runtime.py:297-306)
//   gcnb_dense_f32      the `@ w` of runtime.py:299 hoisted before aggregation
//   gcnb_bwd_layer_f32  runtime._bwd_compute       (runtime.py:344-356)
//   gcnb_reduce_*       allreduce-side ΔW reduction (+ fused SGD, runtime.py:359-360)
//
// Design: the aggregation Σ_j A[r,j]·X[j] is HBM/L2-gather
// bound.  A group of LPR lanes owns one CSR row; each lane owns a 16-byte
// float4 chunk of the feature row, so one gather of a neighbour row is a
// single coalesced LPR×16-byte access.  Column indices and values are loaded
// cooperatively (one per lane, coalesced) and broadcast with shuffles.  The
// dense epilogue (·W, ReLU, ·Wᵀ ⊙ σ', Hᵀ·agg) runs on a T-row tile staged in
// shared memory with W resident in shared memory for the whole persistent
// block, so the aggregated rows never round-trip through HBM.  All
// accumulation orders are fixed (CSR order per row, fixed tile→block map,
// fixed partial-reduction order): reruns are bit-identical.
#include <algorithm>

#include "common.cuh"
#include "epipack.cuh"

namespace gcnb {

// 16-byte read-only gather as a volatile asm: volatile loads keep their program
// order, so a batch of them is issued back to back (all in flight) before the
// dependent FMAs — the compiler otherwise interleaves load→fma pairs to save
// registers and keeps one gather in flight per lane.
__device__ __forceinline__ float4 ldg_batch(const float4* p, bool pred) {
  float4 v;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "mov.b32 %0, 0;\n\tmov.b32 %1, 0;\n\tmov.b32 %2, 0;\n\tmov.b32 %3, 0;\n\t"
      "@q ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];\n\t}"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p), "r"((int)pred));
  return v;
}

// Row extent [s, s+len) of CSR row `row` (row < 0: empty).
__device__ __forceinline__ void row_extent(const int* __restrict__ rp, int row, int& s, int& len) {
  s = 0;
  len = 0;
  if (row >= 0) {
    s = __ldg(rp + row);
    len = __ldg(rp + row + 1) - s;
  }
}

// Cooperative aggregation of one CSR row (extent s, len) by a group of LPR
// lanes.  Must be called by all 32 lanes of the warp (warp-uniform trip
// count).  The (col, val) chunk for the next LPR nonzeros is loaded before
// the current chunk's gathers are issued, so the index stream and the
// feature-row gathers overlap instead of forming two dependent round trips
// per chunk.
template <bool ENT>
__device__ __forceinline__ void load_nz(const int* __restrict__ col, const float* __restrict__ val, int e, int& c,
                                        float& v);

template <int LPR, int VPL, bool ENT = false>
__device__ __forceinline__ void aggregate_span(const int* __restrict__ col, const float* __restrict__ val, int s,
                                               int len, const float4* __restrict__ X4, int ldx4, int c4, int gl,
                                               float4 (&acc)[VPL]) {
  const int maxlen = __reduce_max_sync(0xffffffffu, len);
  int cj = 0;
  float vj = 0.0f;
  if (gl < len) load_nz<ENT>(col, val, s + gl, cj, vj);
  for (int base = 0; base < maxlen; base += LPR) {
    int cn = 0;
    float vn = 0.0f;
    if (base + LPR + gl < len) load_nz<ENT>(col, val, s + base + LPR + gl, cn, vn);
    const int cnt = min(LPR, maxlen - base);
    // Issue U independent row gathers into distinct registers before any is
    // consumed: a load→fma→load chain would keep only one gather in flight
    // per lane (the compiler reuses the destination registers otherwise).
    constexpr int U = LPR < 8 ? LPR : 8;
    for (int t0 = 0; t0 < cnt; t0 += U) {
      float4 xv[U][VPL];
      float vv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int t = t0 + u;
        const int c = __shfl_sync(0xffffffffu, cj, t & (LPR - 1), LPR);
        const float v = __shfl_sync(0xffffffffu, vj, t & (LPR - 1), LPR);
        const bool ok = t < cnt && base + t < len;
        vv[u] = ok ? v : 0.0f;
        const float4* xr = X4 + (size_t)c * ldx4;
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
          const int ch = gl + q * LPR;
          xv[u][q] = ldg_batch(xr + ch, ok && ch < c4);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int q = 0; q < VPL; ++q) acc[q] = fma4(vv[u], xv[u][q], acc[q]);
      }
    }
    cj = cn;
    vj = vn;
  }
}

// The same aggregation with the U gathers of a batch issued as cp.async into a
// per-warp shared-memory staging slot (stage: [U][VPL][32 lanes] float4): the
// copies are memory operations the scheduler cannot sink next to their uses,
// so U gathers per lane are genuinely in flight, at no register cost.  Each
// lane reads back only the slot it filled itself (no warp barrier needed).
// Predicated off (not zero-filled) when !pred: a src-size-0 copy still sends
// its sector request through L1/L2 (ncu measured 1.5x the algorithmic gather
// bytes on products from the idle chunk lanes), a predicated one does not.
// The slot then holds stale data, so callers must not consume it.
// CA: allocate the gathered sectors in L1 as well (cp.async.ca) so warps of one
// SM that share neighbours (locality layout) hit L1 instead of the L2 fabric.
template <bool CA = false>
__device__ __forceinline__ void cp_async_16(void* smem_dst, const void* gmem_src, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  if constexpr (CA)
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
        "@q cp.async.ca.shared.global [%0], [%1], 16;\n\t}" ::"r"(s), "l"(gmem_src), "r"((int)pred)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
        "@q cp.async.cg.shared.global [%0], [%1], 16;\n\t}" ::"r"(s), "l"(gmem_src), "r"((int)pred)
        : "memory");
}

// (column, value) of nonzero e: separate CSR arrays, or (ENT) the int2
// {column, value bits} entries of the windowed layout (aggwin.cu).
template <bool ENT>
__device__ __forceinline__ void load_nz(const int* __restrict__ col, const float* __restrict__ val, int e, int& c,
                                        float& v) {
  if constexpr (ENT) {
    const int2 t = __ldg(reinterpret_cast<const int2*>(col) + e);
    c = t.x;
    v = __int_as_float(t.y);
  } else {
    c = __ldg(col + e);
    v = __ldg(val + e);
  }
}

template <int LPR, int VPL, int U, bool CA = false, bool ENT = false>
__device__ __forceinline__ void aggregate_span_cp(const int* __restrict__ col, const float* __restrict__ val, int s,
                                                  int len, const float4* __restrict__ X4, int ldx4, int c4, int gl,
                                                  float4 (&acc)[VPL], float4* __restrict__ stage) {
  const int lane = threadIdx.x & 31;
  const int maxlen = __reduce_max_sync(0xffffffffu, len);
  int cj = 0;
  float vj = 0.0f;
  if (gl < len) load_nz<ENT>(col, val, s + gl, cj, vj);
  for (int base = 0; base < maxlen; base += LPR) {
    int cn = 0;
    float vn = 0.0f;
    if (base + LPR + gl < len) load_nz<ENT>(col, val, s + base + LPR + gl, cn, vn);
    const int cnt = min(LPR, maxlen - base);
    for (int t0 = 0; t0 < cnt; t0 += U) {
      float vv[U];
      bool okv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int t = t0 + u;
        const int c = __shfl_sync(0xffffffffu, cj, t & (LPR - 1), LPR);
        const float v = __shfl_sync(0xffffffffu, vj, t & (LPR - 1), LPR);
        okv[u] = t < cnt && base + t < len;
        vv[u] = v;
        const float4* xr = X4 + (size_t)c * ldx4;
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
          const int ch = gl + q * LPR;
          cp_async_16<CA>(stage + (u * VPL + q) * 32 + lane, xr + ch, okv[u] && ch < c4);
        }
      }
      asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
      // chunks past c4 are never stored by the caller, so only okv gates
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int q = 0; q < VPL; ++q)
          if (okv[u]) acc[q] = fma4(vv[u], stage[(u * VPL + q) * 32 + lane], acc[q]);
      }
    }
    cj = cn;
    vj = vn;
  }
}

template <int LPR, int VPL>
__device__ __forceinline__ void aggregate_row(const int* __restrict__ rp, const int* __restrict__ col,
                                              const float* __restrict__ val, int row,
                                              const float4* __restrict__ X4, int ldx4, int c4, int gl,
                                              float4 (&acc)[VPL]) {
  int s, len;
  row_extent(rp, row, s, len);
  aggregate_span<LPR, VPL>(col, val, s, len, X4, ldx4, c4, gl, acc);
}

// ---------------------------------------------------------------------------
// Gathers batched per lane before one cp.async wait: ~8 float4 chunks in flight.
__host__ __device__ constexpr int agg_batch(int lpr, int vpl) {
  return lpr < 8 / vpl ? lpr : (8 / vpl > 0 ? 8 / vpl : 1);
}

// Aggregate-only: Y[r] = act(A[r,:]·X)  (act < 0: plain store)
//
// Rows are handed out dynamically: a warp grabs the next AGG_ROWS_PER_GRAB
// rows from a per-stream work counter (sched[0], one atomic per grab), so all
// warps sweep the (locality-ordered) rows together in a window of about
// warps × AGG_ROWS_PER_GRAB rows.  A static row-strided assignment lets warps
// drift apart by tens of thousands of rows over a launch (per-row work is
// skewed), which spreads the gathered neighbourhoods over more than the L2 can
// hold: on the products shape an LRU model of the two schedules gives 26 GB vs
// 4 GB of DRAM gathers for the first layer, and ncu measured 23 GB for the
// static one.  Each row is still reduced by one warp in CSR order, so results
// do not depend on the schedule.  The last warp to finish resets the counter
// (sched[1] counts finished warps), so the slot is ready for the next launch
// on the stream.
constexpr int AGG_ROWS_PER_GRAB = 4;
constexpr int AGG_NNZ_PER_GRAB = 1024;

// FAR: the second pass of the windowed aggregation (aggwin.cu): only the far
// entries [rp[r] + nnear[r], rp[r+1]) of the int2 entry array (`col`), added to
// the near partial sum already in Y (order: near entries, then far entries).
//
// VPO > 0: the narrow dense transform is fused into the epilogue (the
// aggregate-first layer with a small W, runtime.py:297-306): Y[r] =
// act((A[r,:]·X)·W) with W (d_in × 4·c4o, zero pad columns) staged in shared
// memory; lane gl of a row group produces output chunks gl + v·LPR (v < VPO)
// from the group's aggregated row, broadcast chunk by chunk with shuffles.
// The products are summed over k ascending from zero, as tile_gemm does.
template <int LPR, int VPL, bool FAR = false, int VPO = 0>
__global__ void __launch_bounds__(NT) k_agg(const int* __restrict__ rp, const int* __restrict__ col,
                                            const float* __restrict__ val, const int* __restrict__ rows,
                                            int n_rows, const float4* __restrict__ X4, int ldx4, int c4,
                                            float4* __restrict__ Y4, int ldy4, int act, int* __restrict__ sched,
                                            int regs, const int* __restrict__ nnear, const float4* __restrict__ W4,
                                            int d_in, int c4o) {
  constexpr int GPW = 32 / LPR;
  // Rows per ticket.  Wide rows keep AGG_ROWS_PER_GRAB (the L2 sweep window
  // above).  Narrow rows (LPR <= 8) size the ticket to ~AGG_NNZ_PER_GRAB
  // nonzeros from the operator's mean row length (contiguous rows: two loads
  // of rp), up to 64 rows: with a few nonzeros per row one atomic per row
  // group makes the shared counter the limit (roadNet fwd2, d = 8: 0.121 ->
  // 0.068 ms; products' labelled-column bwd2: 0.56 -> 0.32 ms).
  constexpr int CH_WIDE = AGG_ROWS_PER_GRAB > GPW ? AGG_ROWS_PER_GRAB / GPW : 1;
  int CH = CH_WIDE;  // row groups per grab
  if constexpr (LPR <= 8) {
    int rows_per_grab = 16;
    if (!rows && n_rows > 0) {
      const int mean = max(1, (__ldg(rp + n_rows) - __ldg(rp)) / n_rows);
      rows_per_grab = min(64, AGG_NNZ_PER_GRAB / mean);
    }
    // ... but not so many that half the grid's warps would get no ticket
    // (config 1, 10 K rows: 64-row tickets left 3/4 of the warps idle)
    rows_per_grab = min(rows_per_grab, 2 * n_rows / (int)(gridDim.x * WARPS));
    CH = max(1, rows_per_grab / GPW);
  }
  const int RPG = GPW * CH;  // rows per grab
  const int lane = threadIdx.x & 31;
  const int gl = lane & (LPR - 1);
  const int gw = lane / LPR;
  constexpr int U = agg_batch(LPR, VPL);
  extern __shared__ __align__(16) float4 stage_all[];
  float4* stage = stage_all + (threadIdx.x >> 5) * (U * VPL * 32);
  float4* Ws4 = stage_all + WARPS * (U * VPL * 32);  // VPO > 0: W, d_in rows of c4o chunks
  if constexpr (VPO > 0) {
    for (int i = threadIdx.x; i < d_in * c4o; i += NT) Ws4[i] = __ldg(W4 + i);
    __syncthreads();
  }
  auto grab = [&]() {
    int b = 0;
    if (lane == 0) b = atomicAdd(sched, 1);
    b = __shfl_sync(0xffffffffu, b, 0);
    return b < (n_rows + RPG - 1) / RPG ? b * RPG : n_rows;
  };
  auto row_of = [&](int b, int c) {
    const int i = b + c * GPW + gw;
    return (b < n_rows && i < n_rows) ? (rows ? __ldg(rows + i) : i) : -1;
  };
  auto extent = [&](int row, int& s, int& len) {
    row_extent(rp, row, s, len);
    if (FAR && row >= 0) {
      const int nn = __ldg(nnear + row);
      s += nn;
      len -= nn;
    }
  };
  int base = grab(), c = 0;
  int row = row_of(base, 0);
  int s, len;
  extent(row, s, len);
  while (base < n_rows) {
    // next row group (grabbing the next chunk one row early), its extent
    // prefetched while this row is aggregated
    int base_n = base, c_n = c + 1;
    if (c_n == CH) {
      base_n = grab();
      c_n = 0;
    }
    const int row_n = row_of(base_n, c_n);
    int s_n, len_n;
    extent(row_n, s_n, len_n);
    float4 acc[VPL];
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
      acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (FAR && row >= 0 && gl + q * LPR < c4) acc[q] = Y4[(size_t)row * ldy4 + gl + q * LPR];
    }
    if (regs == 1) aggregate_span<LPR, VPL, FAR>(col, val, s, len, X4, ldx4, c4, gl, acc);
    else if (regs == 2) aggregate_span_cp<LPR, VPL, U, true, FAR>(col, val, s, len, X4, ldx4, c4, gl, acc, stage);
    else aggregate_span_cp<LPR, VPL, U, false, FAR>(col, val, s, len, X4, ldx4, c4, gl, acc, stage);
    if constexpr (VPO > 0) {
      float4 o[VPO];
#pragma unroll
      for (int v = 0; v < VPO; ++v) o[v] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int ic = 0; ic < c4; ++ic) {  // warp-uniform
        const int q = ic / LPR;
        float4 mine = acc[0];
#pragma unroll
        for (int qq = 1; qq < VPL; ++qq)
          if (qq == q) mine = acc[qq];
        const int src = ic & (LPR - 1);
        float a[4];
        a[0] = __shfl_sync(0xffffffffu, mine.x, src, LPR);
        a[1] = __shfl_sync(0xffffffffu, mine.y, src, LPR);
        a[2] = __shfl_sync(0xffffffffu, mine.z, src, LPR);
        a[3] = __shfl_sync(0xffffffffu, mine.w, src, LPR);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int k = 4 * ic + e;
          if (k < d_in) {
#pragma unroll
            for (int v = 0; v < VPO; ++v) {
              const int oc = gl + v * LPR;
              if (oc < c4o) o[v] = fma4(a[e], Ws4[k * c4o + oc], o[v]);
            }
          }
        }
      }
      if (row >= 0) {
#pragma unroll
        for (int v = 0; v < VPO; ++v) {
          const int oc = gl + v * LPR;
          if (oc < c4o) Y4[(size_t)row * ldy4 + oc] = act_fwd4(o[v], act);
        }
      }
    } else if (row >= 0) {
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const int ch = gl + q * LPR;
        if (ch < c4) Y4[(size_t)row * ldy4 + ch] = act >= 0 ? act_fwd4(acc[q], act) : acc[q];
      }
    }
    base = base_n;
    c = c_n;
    row = row_n;
    s = s_n;
    len = len_n;
  }
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(sched + 1, 1) == (int)(gridDim.x * WARPS) - 1) {
      atomicExch(sched, 0);
      atomicExch(sched + 1, 0);
    }
  }
}

// ---------------------------------------------------------------------------
// Tile GEMM: acc[u] (tile rows trg + u*RG, cols 4tc..4tc+3) = Σ_k Ys[r][k]·Ws[k][4tc..]
template <int RPT>
// (Reading Y four k at a time measured no faster on products and raised
// register counts of the RPT = 8 variants; kept as one k per step.)
__device__ __forceinline__ void tile_gemm(const float* __restrict__ Ys, int ys_ld, const float* __restrict__ Ws,
                                          int ws_ld, int K, int trg, int RG, int tc, int rpt, float4 (&acc)[RPT]) {
#pragma unroll
  for (int u = 0; u < RPT; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4* W4 = reinterpret_cast<const float4*>(Ws);
  const int ws_ld4 = ws_ld / 4;
#pragma unroll 4
  for (int k = 0; k < K; ++k) {
    const float4 w = W4[k * ws_ld4 + tc];
#pragma unroll
    for (int u = 0; u < RPT; ++u)
      if (u < rpt) acc[u] = fma4(Ys[(trg + u * RG) * ys_ld + k], w, acc[u]);
  }
}

// Stage T rows of the tile into Ys (row stride ys_ld): aggregated (AGG; a
// group of LPR lanes per row, next-row extent prefetched) or loaded directly
// from X.
template <int LPR, int VPL, bool AGG>
__device__ __forceinline__ void stage_tile(const int* __restrict__ rp, const int* __restrict__ col,
                                           const float* __restrict__ val, const int* __restrict__ rows,
                                           int n_rows, int t0, int T, const float4* __restrict__ X4, int ldx4,
                                           int c4, float* __restrict__ Ys, int ys_ld) {
  if (AGG) {
    constexpr int NG = NT / LPR;
    const int lane = threadIdx.x & 31;
    const int gl = lane & (LPR - 1);
    const int grp = threadIdx.x / LPR;
    auto row_of = [&](int r) {
      const int i = t0 + r;
      return (r < T && i < n_rows) ? (rows ? __ldg(rows + i) : i) : -1;
    };
    int s, len;
    row_extent(rp, row_of(grp), s, len);
    for (int r0 = 0; r0 < T; r0 += NG) {
      const int r = r0 + grp;
      int s_n, len_n;
      row_extent(rp, row_of(r + NG), s_n, len_n);
      float4 acc[VPL];
#pragma unroll
      for (int q = 0; q < VPL; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      aggregate_span<LPR, VPL>(col, val, s, len, X4, ldx4, c4, gl, acc);
      s = s_n;
      len = len_n;
      if (r < T) {
        float4* dst = reinterpret_cast<float4*>(Ys + r * ys_ld);
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
          const int ch = gl + q * LPR;
          if (ch < c4) dst[ch] = acc[q];
        }
      }
    }
  } else {
    for (int idx = threadIdx.x; idx < T * c4; idx += NT) {
      const int r = idx / c4, ch = idx - r * c4;
      const int i = t0 + r;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i < n_rows) {
        const int row = rows ? __ldg(rows + i) : i;
        v = __ldg(X4 + (size_t)row * ldx4 + ch);
      }
      reinterpret_cast<float4*>(Ys + r * ys_ld)[ch] = v;
    }
  }
}

// Forward layer with the dense transform fused: H[r] = act((A[r,:]·X)·W)
// (AGG) or H[r] = act(X[r]·W) (!AGG, the hoisted dense transform); with
// W == nullptr (AGG only) H[r] = act(A[r,:]·X).
template <int LPR, int VPL, bool AGG, int RPT>
__global__ void __launch_bounds__(NT) k_fwd_gemm(const int* __restrict__ rp, const int* __restrict__ col,
                                                 const float* __restrict__ val, const int* __restrict__ rows,
                                                 int n_rows, const float* __restrict__ X, int ldx, int d_in,
                                                 const float* __restrict__ W, int d_out, float* __restrict__ H,
                                                 int ldh, int act, int T, const EpiPack pk) {
  extern __shared__ __align__(16) float smem[];
  const int ld_in = (d_in + 3) & ~3;
  const int ld_out = (d_out + 3) & ~3;
  const int ys_ld = ld_in + 4;
  const int w_floats = W ? ld_in * ld_out : 0;
  float* Ws = smem;                     // ld_in × ld_out (rows >= d_in zero)
  float* Ys = smem + w_floats;          // T × ys_ld
  if (W) {
    const float4* W4 = reinterpret_cast<const float4*>(W);
    float4* Ws4 = reinterpret_cast<float4*>(Ws);
    for (int idx = threadIdx.x; idx < ld_in * ld_out / 4; idx += NT)
      Ws4[idx] = idx < d_in * ld_out / 4 ? __ldg(W4 + idx) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const int c4o = ld_out / 4;
  const int RG = NT / c4o;
  const int tc = threadIdx.x % c4o, trg = threadIdx.x / c4o;
  const int c4i = ld_in / 4;
  const int n_tiles = (n_rows + T - 1) / T;
  const int rpt = trg < RG ? (T - trg + RG - 1) / RG : 0;
  __syncthreads();
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int t0 = tile * T;
    stage_tile<LPR, VPL, AGG>(rp, col, val, rows, n_rows, t0, T, reinterpret_cast<const float4*>(X), ldx / 4,
                              c4i, Ys, ys_ld);
    __syncthreads();
    if (!W) {
      for (int idx = threadIdx.x; idx < T * c4i; idx += NT) {
        const int r = idx / c4i, ch = idx - r * c4i;
        const int i = t0 + r;
        if (i < n_rows) {
          const int row = rows ? __ldg(rows + i) : i;
          reinterpret_cast<float4*>(H + (size_t)row * ldh)[ch] =
              act_fwd4(reinterpret_cast<const float4*>(Ys + r * ys_ld)[ch], act);
        }
      }
    } else if (rpt > 0) {
      float4 acc[RPT];
      tile_gemm<RPT>(Ys, ys_ld, Ws, ld_out, d_in, trg, RG, tc, rpt, acc);
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        if (u < rpt) {
          const int i = t0 + trg + u * RG;
          if (i < n_rows) {
            const int row = rows ? __ldg(rows + i) : i;
            reinterpret_cast<float4*>(H + (size_t)row * ldh)[tc] = act_fwd4(acc[u], act);
          }
        }
      }
    }
    __syncthreads();
  }
  epi_forward(pk, H, ldh, rows, n_rows, T, (W ? ld_out : ld_in) / 4);
  epi_signal(pk);
}

// ---------------------------------------------------------------------------
// Backward layer: agg = A_back[r,:]·G;  G_prev[r] = (agg·Wᵀ) ⊙ σ'(H_prev[r])  (GP);
// per-block ΔW partial = Σ_r H_prev[r]ᵀ·agg[r]  (fixed tile order).
template <int LPR, int VPL, int IPT, bool GP, int RPT>
__global__ void __launch_bounds__(NT) k_bwd(const int* __restrict__ rp, const int* __restrict__ col,
                                            const float* __restrict__ val, const int* __restrict__ rows,
                                            int n_rows, const float* __restrict__ G, int ldg, int d_k,
                                            const float* __restrict__ Hp, int ldhp, int d_prev,
                                            const float* __restrict__ W, float* __restrict__ Gp, int ldgp,
                                            int act, float* __restrict__ partials, int T, const EpiPack pk) {
  extern __shared__ __align__(16) float smem[];
  const int ld_k = (d_k + 3) & ~3;
  const int ld_p = (d_prev + 3) & ~3;
  const int as_ld = ld_k + 4;
  const int hs_ld = ld_p + 4;
  float* Wts = smem;                              // ld_k × ld_p  (Wᵀ, pad rows/cols zero), GP only
  float* As = smem + (GP ? ld_k * ld_p : 0);      // T × as_ld
  float* Hs = As + T * as_ld;                     // T × hs_ld
  if (GP) {
    for (int idx = threadIdx.x; idx < ld_k * ld_p; idx += NT) {
      const int c = idx / ld_p, i = idx - c * ld_p;
      Wts[idx] = (i < d_prev && c < d_k) ? __ldg(W + (size_t)i * ld_k + c) : 0.0f;
    }
  }
  const int c4k = ld_k / 4, c4p = ld_p / 4;
  // S = agg·Wᵀ mapping (output d_prev wide)
  const int RG = NT / c4p;
  const int tc = threadIdx.x % c4p, trg = threadIdx.x / c4p;
  const int rpt = trg < RG ? (T - trg + RG - 1) / RG : 0;
  // ΔW mapping over the float4 chunks of the d_prev × ld_k partial (C chunks):
  //  C >= NT: thread owns rows i = ig + ii*RGi, cols 4kc.., accumulating every tile row;
  //  C <  NT: RS = NT / C row groups; thread owns one chunk for tile rows r ≡ rs (mod RS),
  //           and the RS group partials are combined in a fixed order at the end.
  const int C = d_prev * c4k;
  const int RS = C >= NT ? 1 : NT / C;
  const int CG = RS > 1 ? C : NT;
  const int q = threadIdx.x % CG, rs = threadIdx.x / CG;
  const int RGi = NT / c4k;
  const int kc = q % c4k, ig = q / c4k;
  int ipt;
  if (RS > 1) ipt = rs < RS ? 1 : 0;
  else ipt = ig < RGi && ig < d_prev ? (d_prev - ig + RGi - 1) / RGi : 0;
  float4 dw[IPT];
#pragma unroll
  for (int ii = 0; ii < IPT; ++ii) dw[ii] = make_float4(0.f, 0.f, 0.f, 0.f);

  const int n_tiles = (n_rows + T - 1) / T;
  __syncthreads();
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int t0 = tile * T;
    const int tv = min(T, n_rows - t0);
    if (rp)
      stage_tile<LPR, VPL, true>(rp, col, val, rows, n_rows, t0, T, reinterpret_cast<const float4*>(G), ldg / 4,
                                 c4k, As, as_ld);
    else  // split mode: G already holds agg = A_back·G (own-row positions)
      stage_tile<LPR, VPL, false>(nullptr, nullptr, nullptr, rows, n_rows, t0, T,
                                  reinterpret_cast<const float4*>(G), ldg / 4, c4k, As, as_ld);
    stage_tile<LPR, VPL, false>(nullptr, nullptr, nullptr, rows, n_rows, t0, T,
                                reinterpret_cast<const float4*>(Hp), ldhp / 4, c4p, Hs, hs_ld);
    __syncthreads();
    if (GP && rpt > 0) {
      float4 acc[RPT];
      tile_gemm<RPT>(As, as_ld, Wts, ld_p, d_k, trg, RG, tc, rpt, acc);
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        if (u < rpt) {
          const int r = trg + u * RG;
          const int i = t0 + r;
          if (i < n_rows) {
            const int row = rows ? __ldg(rows + i) : i;
            const float4 h = reinterpret_cast<const float4*>(Hs + r * hs_ld)[tc];
            float4 o = acc[u];
            o.x *= act_grad_from_h(h.x, act);
            o.y *= act_grad_from_h(h.y, act);
            o.z *= act_grad_from_h(h.z, act);
            o.w *= act_grad_from_h(h.w, act);
            reinterpret_cast<float4*>(Gp + (size_t)row * ldgp)[tc] = o;
          }
        }
      }
    }
    if (ipt > 0) {
      for (int r = rs; r < tv; r += RS) {
        const float4 a = reinterpret_cast<const float4*>(As + r * as_ld)[kc];
        const float* hr = Hs + r * hs_ld + ig;
#pragma unroll
        for (int ii = 0; ii < IPT; ++ii)
          if (ii < ipt) dw[ii] = fma4(hr[ii * RGi], a, dw[ii]);
      }
    }
    __syncthreads();
  }
  if (GP) {
    epi_forward(pk, Gp, ldgp, rows, n_rows, T, c4p);
    epi_signal(pk);
  }
  float* part = partials + (size_t)blockIdx.x * d_prev * ld_k;
  if (RS > 1) {
    float4* red = reinterpret_cast<float4*>(Hs + T * hs_ld);  // NT float4 of dedicated scratch
    if (ipt) red[rs * C + q] = dw[0];
    __syncthreads();
    if (threadIdx.x < C) {
      float4 t = red[threadIdx.x];
      for (int g = 1; g < RS; ++g) {
        const float4 u = red[g * C + threadIdx.x];
        t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
      }
      reinterpret_cast<float4*>(part)[threadIdx.x] = t;  // chunk q == threadIdx.x
    }
    return;
  }
#pragma unroll
  for (int ii = 0; ii < IPT; ++ii)
    if (ii < ipt) reinterpret_cast<float4*>(part + (size_t)(ig + ii * RGi) * ld_k)[kc] = dw[ii];
}

// out = Σ_s partials[s] in a fixed order (float4 chunks).  A 1024-thread block
// owns 64 chunks; its 16 slot groups stride the slots with two independent
// accumulators each and are combined in a fixed order.  With w != null the
// SGD update w -= lr·out is fused (runtime.py:359-360).
constexpr int RED_T = 1024;
constexpr int RED_SPB = 64;  // slots folded per level-1 block

// Level 1 (many SMs): block (bx, by) folds slots [by*SPB, by*SPB+SPB) of its 64
// chunks and writes the fixed-order sum back IN PLACE into slot by*SPB.
__global__ void __launch_bounds__(RED_T) k_reduce_l1(float4* __restrict__ partials, int n_slots, long long size4) {
  __shared__ float4 red[16][64];
  const int lane = threadIdx.x & 63, grp = threadIdx.x >> 6;
  const long long chunk = blockIdx.x * 64LL + lane;
  const int s0 = blockIdx.y * RED_SPB;
  const int s1 = min(n_slots, s0 + RED_SPB);
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a, c = a, d = a;
  if (chunk < size4) {
    // 4 slots per group: s0 + grp + 16*j, j < 4 (independent loads)
    const int b0 = s0 + grp;
    if (b0 < s1) a = partials[(size_t)b0 * size4 + chunk];
    if (b0 + 16 < s1) b = partials[(size_t)(b0 + 16) * size4 + chunk];
    if (b0 + 32 < s1) c = partials[(size_t)(b0 + 32) * size4 + chunk];
    if (b0 + 48 < s1) d = partials[(size_t)(b0 + 48) * size4 + chunk];
  }
  red[grp][lane] = make_float4(a.x + b.x + c.x + d.x, a.y + b.y + c.y + d.y, a.z + b.z + c.z + d.z,
                               a.w + b.w + c.w + d.w);
  __syncthreads();  // every read of this block's slot range is done before the in-place write
  if (grp == 0 && chunk < size4) {
    float4 t = red[0][lane];
#pragma unroll
    for (int g = 1; g < 16; ++g) {
      t.x += red[g][lane].x; t.y += red[g][lane].y; t.z += red[g][lane].z; t.w += red[g][lane].w;
    }
    partials[(size_t)s0 * size4 + chunk] = t;
  }
}

// Level 2 (or the only level): fold slots 0, stride, 2*stride, ... (< n_slots).
__global__ void __launch_bounds__(RED_T) k_reduce4(const float4* __restrict__ partials, int n_slots, int stride,
                                                  long long size4, float4* __restrict__ out, int accumulate,
                                                  float4* __restrict__ w, float lr) {
  __shared__ float4 red[16][64];
  const int lane = threadIdx.x & 63, grp = threadIdx.x >> 6;
  const long long chunk = blockIdx.x * 64LL + lane;
  const int n_fold = (n_slots + stride - 1) / stride;  // slots 0, stride, 2*stride, ...
  // 8 independent accumulation chains per thread (folded slots grp + 16*(8*j + c)),
  // combined in a fixed order: few dependent L2 round trips, deterministic.
  constexpr int CH = 8;
  float4 s[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) s[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (chunk < size4) {
    for (int b0 = grp; b0 < n_fold; b0 += 16 * CH) {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const int b = b0 + 16 * c;
        if (b < n_fold) {
          const float4 u = __ldg(partials + (size_t)b * stride * size4 + chunk);
          s[c].x += u.x; s[c].y += u.y; s[c].z += u.z; s[c].w += u.w;
        }
      }
    }
  }
#pragma unroll
  for (int c = 1; c < CH; ++c) {
    s[0].x += s[c].x; s[0].y += s[c].y; s[0].z += s[c].z; s[0].w += s[c].w;
  }
  red[grp][lane] = s[0];
  __syncthreads();
  if (grp == 0 && chunk < size4) {
    float4 t = accumulate ? out[chunk] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int g = 0; g < 16; ++g) {
      t.x += red[g][lane].x; t.y += red[g][lane].y; t.z += red[g][lane].z; t.w += red[g][lane].w;
    }
    out[chunk] = t;
    if (w) {
      float4 x = w[chunk];
      x.x -= lr * t.x; x.y -= lr * t.y; x.z -= lr * t.z; x.w -= lr * t.w;
      w[chunk] = x;
    }
  }
}

// ---------------------------------------------------------------------------
// host side

namespace {

struct AggShape {
  int lpr;
  int vpl;
};

// Forced (lpr, vpl) for the aggregation-only kernel (gcnb_set_agg_shape; 0 = auto).
int g_agg_lpr = 0, g_agg_vpl = 0;
int g_agg_regs = 0;  // 1: register-batched gathers, 2: L1-allocating cp.async.ca staging (gcnb_set_agg_gather)

AggShape agg_shape(int d) {
  const int c4 = round4(d) / 4;
  if (c4 > 32) return {32, (c4 + 31) / 32};
  int lpr = 1;
  while (lpr < c4) lpr <<= 1;
  return {std::max(lpr, 2), 1};
}

int occupancy_grid(const void* fn, size_t smem, int n_tiles) {
  if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, smem) != cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    per_sm = 1;
  }
  return std::max(1, std::min(n_tiles, per_sm * num_sms()));
}

// Tile height for an output width d_out (<= RPT_MAX rows per thread) that is
// also a multiple of the aggregation group count NG; *rpt_out = rows per thread.
int tile_rows(int d_out, int lpr, int* rpt_out) {
  const int c4o = round4(d_out) / 4;
  const int rg = NT / c4o;
  const int ng = NT / lpr;
  int t = 4 * rg;
  t = ((t + ng - 1) / ng) * ng;
  while (t > RPT_MAX * rg && t > ng) t -= ng;
  t = std::max(t, ng);
  *rpt_out = (t + rg - 1) / rg;
  return t;
}

#define GCNB_LPR_CASES(M) M(2, 1) M(4, 1) M(8, 1) M(16, 1) M(32, 1) M(32, 2)

using AggFn = void (*)(const int*, const int*, const float*, const int*, int, const float4*, int, int, float4*, int,
                       int, int*, int, const int*, const float4*, int, int);
// Shape of the aggregation-only kernel over all own rows: two float4 chunks per
// lane from 9 chunks up, so 2-4 rows share a warp (rows of similar length side by
// side after the degree-sorted layout windows): measured on the products shape,
// d=104 took 3.43 ms as (16,2) vs 3.59 ms as (32,1), d=48 1.82 ms as (8,2) vs
// 1.86 ms as (16,1) (profiles/r01_spmm_shapes_products.txt).  On the interior /
// boundary row lists of 2-4 GPU runs the same shapes were 10-25 % slower.
AggShape agg_shape_spmm(int d) {
  const int c4 = round4(d) / 4;
  if (c4 > 8 && c4 <= 16) return {8, 2};
  if (c4 > 16 && c4 <= 32) return {16, 2};
  return agg_shape(d);
}

#define GCNB_AGG_EXTRA_CASES(M) M(4, 3) M(8, 2) M(8, 4) M(16, 2)
AggFn pick_agg(AggShape s, bool far = false) {
#define M(L, V) if (s.lpr == L && s.vpl == V) return far ? k_agg<L, V, true> : k_agg<L, V, false>;
  GCNB_LPR_CASES(M)
  GCNB_AGG_EXTRA_CASES(M)
#undef M
  return nullptr;
}

using FwdFn = void (*)(const int*, const int*, const float*, const int*, int, const float*, int, int, const float*,
                       int, float*, int, int, int, const EpiPack);
template <bool AGG, int RPT>
FwdFn pick_fwd_rpt(AggShape s) {
#define M(L, V) if (s.lpr == L && s.vpl == V) return k_fwd_gemm<L, V, AGG, RPT>;
  GCNB_LPR_CASES(M)
#undef M
  return nullptr;
}
template <bool AGG>
FwdFn pick_fwd(AggShape s, int rpt) {
  return rpt <= 4 ? pick_fwd_rpt<AGG, 4>(s) : pick_fwd_rpt<AGG, RPT_MAX>(s);
}

using BwdFn = void (*)(const int*, const int*, const float*, const int*, int, const float*, int, int, const float*,
                       int, int, const float*, float*, int, int, float*, int, const EpiPack);
template <int IPT, bool GP, int RPT>
BwdFn pick_bwd_t(AggShape s) {
#define M(L, V) if (s.lpr == L && s.vpl == V) return k_bwd<L, V, IPT, GP, RPT>;
  GCNB_LPR_CASES(M)
#undef M
  return nullptr;
}
template <int IPT>
BwdFn pick_bwd_ipt(AggShape s, bool gp, int rpt) {
  if (gp) return rpt <= 4 ? pick_bwd_t<IPT, true, 4>(s) : pick_bwd_t<IPT, true, RPT_MAX>(s);
  return pick_bwd_t<IPT, false, 4>(s);  // no S-GEMM without G_prev: RPT is unused
}

// Large ΔW tiles make the fused backward kernel register-bound (2 blocks/SM):
// then the aggregation and the dense epilogue run as two kernels.
int g_split_all = 0;  // measurement knob (gcnb_set_split_all): split every layer
int g_fwd_tf = 1;     // gcnb_set_fwd_tf: 1 = k_agg with the fused transform, 0 = tile kernel k_fwd_gemm
bool bwd_split(int d_prev, int d_k) { return g_split_all || (long)d_prev * round4(d_k) > 2048; }

struct BwdPlan {
  BwdFn fn;
  int T;
  size_t smem;
  int grid;
};

int bwd_plan(int n_rows, int d_prev, int d_k, bool with_gp, BwdPlan* out) {
  const AggShape s = agg_shape(d_k);
  const int ld_k = round4(d_k), ld_p = round4(d_prev);
  const int c4k = ld_k / 4;
  const int rgi = NT / c4k;
  const int ipt = d_prev * c4k < NT ? 1 : (d_prev + rgi - 1) / rgi;
  int rpt = 0;
  const int T = tile_rows(d_prev, s.lpr, &rpt);
  BwdFn fn = nullptr;
  if (ipt <= 1) fn = pick_bwd_ipt<1>(s, with_gp, rpt);
  else if (ipt <= 4) fn = pick_bwd_ipt<4>(s, with_gp, rpt);
  else if (ipt <= 8) fn = pick_bwd_ipt<8>(s, with_gp, rpt);
  else if (ipt <= 16) fn = pick_bwd_ipt<16>(s, with_gp, rpt);
  else if (ipt <= 32) fn = pick_bwd_ipt<32>(s, with_gp, rpt);
  GCNB_REQUIRE(fn != nullptr, "bwd layer: unsupported widths d_prev=%d d_k=%d", d_prev, d_k);
  const size_t smem = sizeof(float) * ((with_gp ? (size_t)ld_k * ld_p : 0) + (size_t)T * (ld_k + 4) +
                                       (size_t)T * (ld_p + 4) + 4 * NT);
  GCNB_REQUIRE(smem <= 227 * 1024, "bwd layer: tile does not fit shared memory (d_prev=%d d_k=%d)", d_prev, d_k);
  const int n_tiles = std::max(1, (n_rows + T - 1) / T);
  out->fn = fn;
  out->T = T;
  out->smem = smem;
  out->grid = occupancy_grid(reinterpret_cast<const void*>(fn), smem, n_tiles);
  return GCNB_OK;
}

// Dense part of the backward layer from a resident aggregate: G_prev =
// (agg·Wᵀ) ⊙ σ'(H_prev) (when g_prev) and the ΔW partials H_prevᵀ·agg, on the
// tcgen05 engines where they apply, else the SIMT backward kernel without CSR.
int launch_bwd_epilogue(const float* agg, int ldagg, int d_k, const float* h_prev, int ldhp, int d_prev,
                        const float* w, float* g_prev, int ldgp, int act, const int32_t* rows, int n_rows,
                        float* dw_partials, const BwdPlan& plan, cudaStream_t st, const uint32_t* hbits = nullptr,
                        int ld_hbits = 0, const EpiPack& pk = EpiPack{}) {
  if (dw_tc_applies(d_prev, d_k) && (!g_prev || dense_tc_applies(d_k, d_prev))) {
    if (g_prev) {
      if (int rc = launch_dense_tc(agg, ldagg, rows, n_rows, d_k, nullptr, d_prev, g_prev, ldgp, act, st, w,
                                   round4(d_k), h_prev, ldhp, hbits, ld_hbits, nullptr, 0, &pk))
        return rc;
    }
    return launch_dw_tc(h_prev, ldhp, d_prev, agg, ldagg, d_k, rows, n_rows, dw_partials, plan.grid, st);
  }
  plan.fn<<<plan.grid, NT, plan.smem, st>>>(nullptr, nullptr, nullptr, rows, n_rows, agg, ldagg, d_k, h_prev, ldhp,
                                            d_prev, w, g_prev, ldgp, act, dw_partials, plan.T, pk);
  GCNB_AFTER_LAUNCH("bwd layer (dense epilogue)");
  return GCNB_OK;
}

int check_csr_args(const int32_t* row_ptr, const int32_t* col, const float* val, int32_t n_rows) {
  GCNB_REQUIRE(n_rows >= 0, "n_rows must be >= 0");
  GCNB_REQUIRE(n_rows == 0 || (row_ptr && col && val), "CSR arrays must be non-null");
  return GCNB_OK;
}

int launch_agg(const int32_t* row_ptr, const int32_t* col, const float* val, const int32_t* rows, int32_t n_rows,
               const float* x, int32_t ldx, int32_t d, float* y, int32_t ldy, int32_t act, cudaStream_t st,
               const char* what, const int32_t* nnear = nullptr) {
  // row lists (interior / boundary rows of an overlapped exchange) keep one row
  // group per 16-32 lanes: pairing rows of a list measured slower at 2-4 GPUs
  AggShape s = rows ? agg_shape(d) : agg_shape_spmm(d);
  if (g_agg_lpr > 0 && g_agg_lpr * g_agg_vpl * 4 >= round4(d)) s = {g_agg_lpr, g_agg_vpl};
  AggFn fn = pick_agg(s, nnear != nullptr);
  GCNB_REQUIRE(fn != nullptr, "%s: no aggregation kernel for lpr=%d vpl=%d", what, s.lpr, s.vpl);
  const size_t smem = (size_t)WARPS * agg_batch(s.lpr, s.vpl) * s.vpl * 32 * sizeof(float4);
  const int rows_per_block = NT / s.lpr;
  int per_sm = 0;
  if (smem > 48 * 1024) cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(fn), NT, smem) !=
          cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    per_sm = 1;
  }
  const int grid = std::max(1, std::min((n_rows + rows_per_block - 1) / rows_per_block, num_sms() * per_sm));
  int* sched = sched_counter(st);
  GCNB_REQUIRE(sched != nullptr, "%s: no work-counter slot for this stream", what);
  fn<<<grid, NT, smem, st>>>(row_ptr, col, val, rows, n_rows, reinterpret_cast<const float4*>(x), ldx / 4,
                             round4(d) / 4, reinterpret_cast<float4*>(y), ldy / 4, act, sched, g_agg_regs, nnear,
                             nullptr, 0, 0);
  GCNB_AFTER_LAUNCH(what);
  return GCNB_OK;
}

// Aggregate-first layer with the narrow transform fused into k_agg's epilogue
// (VPO output chunks per lane): rows handed out dynamically like the plain
// aggregation, W in shared memory.  agg_tf_shape says whether the widths have
// such a kernel (otherwise the tile kernel k_fwd_gemm runs the layer).
AggFn pick_agg_tf(int lpr, int vpo) {
#define M(L)                                                    \
  if (lpr == L) {                                               \
    if (vpo == 1) return k_agg<L, 1, false, 1>;                 \
    if (vpo == 2) return k_agg<L, 1, false, 2>;                 \
    if (vpo == 4) return k_agg<L, 1, false, 4>;                 \
  }
  M(2) M(4) M(8) M(16)
#undef M
  return nullptr;
}

bool agg_tf_shape(int d_in, int d_out, int* lpr, int* vpo) {
  const AggShape s = agg_shape(d_in);
  if (s.vpl != 1 || s.lpr > 16) return false;
  const int c4o = round4(d_out) / 4;
  const int v = (c4o + s.lpr - 1) / s.lpr;
  const int vp = v <= 1 ? 1 : v <= 2 ? 2 : v <= 4 ? 4 : 0;
  if (!vp) return false;
  *lpr = s.lpr;
  *vpo = vp;
  return true;
}

int launch_agg_tf(const int32_t* row_ptr, const int32_t* col, const float* val, const int32_t* rows, int32_t n_rows,
                  const float* x, int32_t ldx, int32_t d_in, const float* w, int32_t d_out, float* y, int32_t ldy,
                  int32_t act, cudaStream_t st, const char* what) {
  int lpr = 0, vpo = 0;
  GCNB_REQUIRE(agg_tf_shape(d_in, d_out, &lpr, &vpo), "%s: no fused narrow transform for %d -> %d", what, d_in,
               d_out);
  AggFn fn = pick_agg_tf(lpr, vpo);
  GCNB_REQUIRE(fn != nullptr, "%s: no kernel for lpr=%d vpo=%d", what, lpr, vpo);
  const int c4o = round4(d_out) / 4;
  const size_t smem = (size_t)WARPS * agg_batch(lpr, 1) * 32 * sizeof(float4) + (size_t)d_in * c4o * sizeof(float4);
  GCNB_REQUIRE(smem <= 200 * 1024, "%s: W tile too large for the fused transform", what);
  if (smem > 48 * 1024) cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(fn), NT, smem) !=
          cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    per_sm = 1;
  }
  const int rows_per_block = NT / lpr;
  const int grid = std::max(1, std::min((n_rows + rows_per_block - 1) / rows_per_block, num_sms() * per_sm));
  int* sched = sched_counter(st);
  GCNB_REQUIRE(sched != nullptr, "%s: no work-counter slot for this stream", what);
  fn<<<grid, NT, smem, st>>>(row_ptr, col, val, rows, n_rows, reinterpret_cast<const float4*>(x), ldx / 4,
                             round4(d_in) / 4, reinterpret_cast<float4*>(y), ldy / 4, act, sched, g_agg_regs,
                             nullptr, reinterpret_cast<const float4*>(w), d_in, c4o);
  GCNB_AFTER_LAUNCH(what);
  return GCNB_OK;
}

int launch_fwd_gemm(bool agg, const int32_t* row_ptr, const int32_t* col, const float* val, const int32_t* rows,
                    int32_t n_rows, const float* x, int32_t ldx, int32_t d_in, const float* w, int32_t d_out,
                    float* h, int32_t ldh, int32_t act, cudaStream_t st, const char* what,
                    const EpiPack& pk = EpiPack{}) {
  const AggShape s = agg_shape(d_in);
  int rpt = 0;
  const int T = tile_rows(d_out, s.lpr, &rpt);
  FwdFn fn = agg ? pick_fwd<true>(s, rpt) : pick_fwd<false>(s, rpt);
  GCNB_REQUIRE(fn != nullptr, "%s: unsupported width %d", what, d_in);
  const size_t smem =
      sizeof(float) * ((w ? (size_t)round4(d_in) * round4(d_out) : 0) + (size_t)T * (round4(d_in) + 4));
  GCNB_REQUIRE(smem <= 227 * 1024, "%s: tile does not fit shared memory", what);
  const int grid = occupancy_grid(reinterpret_cast<const void*>(fn), smem, (n_rows + T - 1) / T);
  fn<<<grid, NT, smem, st>>>(row_ptr, col, val, rows, n_rows, x, ldx, d_in, w, d_out, h, ldh, act, T, pk);
  GCNB_AFTER_LAUNCH(what);
  return GCNB_OK;
}

}  // namespace

int launch_agg_far(const int32_t* row_ptr, const int32_t* nnear, const void* entries, int32_t n_rows, const float* x,
                   int32_t ldx, int32_t d, float* y, int32_t ldy, int32_t act, cudaStream_t st) {
  return launch_agg(row_ptr, static_cast<const int32_t*>(entries), nullptr, nullptr, n_rows, x, ldx, d, y, ldy, act,
                    st, "aggregation (windowed, far pass)", nnear);
}

}  // namespace gcnb

using namespace gcnb;

extern "C" int gcnb_set_agg_shape(int32_t lpr, int32_t vpl) {
  GCNB_REQUIRE((lpr == 0 && vpl == 0) || (lpr >= 2 && lpr <= 32 && vpl >= 1 && vpl <= 4),
               "agg shape: lpr in [2, 32], vpl in [1, 4] (or 0, 0 = auto)");
  if (lpr && !pick_agg({lpr, vpl})) return set_error(GCNB_EINVAL, "agg shape (%d, %d) not instantiated", lpr, vpl);
  g_agg_lpr = lpr;
  g_agg_vpl = vpl;
  return GCNB_OK;
}

extern "C" int gcnb_set_agg_gather(int32_t mode) {
  GCNB_REQUIRE(mode >= 0 && mode <= 2,
               "agg gather mode: 0 (cp.async.cg staging), 1 (register batches), 2 (cp.async.ca staging)");
  g_agg_regs = mode;
  return GCNB_OK;
}

extern "C" int gcnb_spmm_f32(const int32_t* row_ptr, const int32_t* col, const float* val, const int32_t* rows,
                             int32_t n_rows, const float* x, int32_t ldx, int32_t d, float* y, int32_t ldy,
                             void* stream) {
  if (int rc = check_csr_args(row_ptr, col, val, n_rows)) return rc;
  GCNB_REQUIRE(d >= 1 && d <= 256, "spmm: width d=%d out of range [1, 256]", d);
  GCNB_REQUIRE(ldx % 4 == 0 && ldy % 4 == 0 && ldx >= round4(d) && ldy >= round4(d),
               "spmm: row strides must be multiples of 4 and >= round4(d)");
  GCNB_REQUIRE(aligned16(x) && aligned16(y), "spmm: X and Y must be 16-byte aligned");
  if (n_rows == 0) return GCNB_OK;
  return launch_agg(row_ptr, col, val, rows, n_rows, x, ldx, d, y, ldy, -1, (cudaStream_t)stream, "spmm");
}

extern "C" int gcnb_fwd_layer_f32(const int32_t* row_ptr, const int32_t* col, const float* val,
                                  const int32_t* rows, int32_t n_rows, const float* x, int32_t ldx, int32_t d_in,
                                  const float* w, int32_t d_out, float* h, int32_t ldh, int32_t act,
                                  void* stream) {
  if (int rc = check_csr_args(row_ptr, col, val, n_rows)) return rc;
  GCNB_REQUIRE(act == GCNB_ACT_RELU || act == GCNB_ACT_IDENTITY, "fwd layer: unknown activation %d", act);
  GCNB_REQUIRE(d_in >= 1 && d_in <= 256 && d_out >= 1 && d_out <= 256, "fwd layer: widths out of range");
  GCNB_REQUIRE(w != nullptr || d_out == d_in, "fwd layer: without W, d_out must equal d_in");
  GCNB_REQUIRE(ldx % 4 == 0 && ldh % 4 == 0 && ldx >= round4(d_in) && ldh >= round4(d_out),
               "fwd layer: row strides must be multiples of 4 and cover the widths");
  GCNB_REQUIRE(aligned16(x) && aligned16(h) && (!w || aligned16(w)), "fwd layer: operands must be 16-byte aligned");
  if (n_rows == 0) return GCNB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (!w)  // aggregate-only: no tile (no barrier, full occupancy)
    return launch_agg(row_ptr, col, val, rows, n_rows, x, ldx, d_in, h, ldh, act, st, "fwd layer (aggregate)");
  int lpr = 0, vpo = 0;
  if (g_fwd_tf && agg_tf_shape(d_in, d_out, &lpr, &vpo))
    return launch_agg_tf(row_ptr, col, val, rows, n_rows, x, ldx, d_in, w, d_out, h, ldh, act, st,
                         "fwd layer (aggregate+transform, fused epilogue)");
  return launch_fwd_gemm(true, row_ptr, col, val, rows, n_rows, x, ldx, d_in, w, d_out, h, ldh, act, st,
                         "fwd layer (aggregate+transform)");
}

extern "C" int gcnb_dense_f32(const float* x, int32_t ldx, const int32_t* rows, int32_t n_rows, int32_t d_in,
                              const float* w, int32_t d_out, float* y, int32_t ldy, int32_t act, void* stream) {
  GCNB_REQUIRE(n_rows >= 0, "dense: n_rows must be >= 0");
  GCNB_REQUIRE(act == GCNB_ACT_RELU || act == GCNB_ACT_IDENTITY, "dense: unknown activation %d", act);
  GCNB_REQUIRE(d_in >= 1 && d_in <= 256 && d_out >= 1 && d_out <= 256, "dense: widths out of range");
  GCNB_REQUIRE(ldx % 4 == 0 && ldy % 4 == 0 && ldx >= round4(d_in) && ldy >= round4(d_out),
               "dense: row strides must be multiples of 4 and cover the widths");
  GCNB_REQUIRE(x && w && y && aligned16(x) && aligned16(w) && aligned16(y), "dense: operands must be 16-byte aligned");
  if (n_rows == 0) return GCNB_OK;
  if (dense_tc_applies(d_in, d_out))
    return launch_dense_tc(x, ldx, rows, n_rows, d_in, w, d_out, y, ldy, act, (cudaStream_t)stream);
  if (dense_blocked_applies(d_in, d_out))
    return launch_dense_blocked(x, ldx, rows, n_rows, d_in, w, d_out, y, ldy, act, (cudaStream_t)stream);
  return launch_fwd_gemm(false, nullptr, nullptr, nullptr, rows, n_rows, x, ldx, d_in, w, d_out, y, ldy, act,
                         (cudaStream_t)stream, "dense");
}

extern "C" int gcnb_dense_tc_applies(int32_t d_in, int32_t d_out, int32_t* out) {
  GCNB_REQUIRE(out != nullptr, "dense tc applies: null output");
  *out = dense_tc_applies(d_in, d_out) ? 1 : 0;
  return GCNB_OK;
}

extern "C" int gcnb_dense_bits_f32(const float* x, int32_t ldx, int32_t n_rows, int32_t d_in, const float* w,
                                   int32_t d_out, float* y, int32_t ldy, uint32_t* bits, int32_t ld_bits,
                                   void* stream) {
  GCNB_REQUIRE(n_rows >= 0, "dense bits: n_rows must be >= 0");
  GCNB_REQUIRE(d_in >= 1 && d_in <= 256 && d_out >= 1 && d_out <= 256, "dense bits: widths out of range");
  GCNB_REQUIRE(ldx % 4 == 0 && ldy % 4 == 0 && ldx >= round4(d_in) && ldy >= round4(d_out),
               "dense bits: row strides must be multiples of 4 and cover the widths");
  GCNB_REQUIRE(x && w && y && bits && aligned16(x) && aligned16(w) && aligned16(y) && aligned16(bits),
               "dense bits: operands must be non-null and 16-byte aligned");
  GCNB_REQUIRE(ld_bits % 4 == 0 && ld_bits * 32 >= d_out, "dense bits: bit-row stride must be a multiple of 4 "
               "words covering d_out");
  GCNB_REQUIRE(dense_tc_applies(d_in, d_out), "dense bits: widths %d -> %d have no tcgen05 engine", d_in, d_out);
  if (n_rows == 0) return GCNB_OK;
  return launch_dense_tc(x, ldx, nullptr, n_rows, d_in, w, d_out, y, ldy, GCNB_ACT_RELU, (cudaStream_t)stream,
                         nullptr, 0, nullptr, 0, nullptr, 0, bits, ld_bits);
}

extern "C" int gcnb_bwd_grid(int32_t n_rows, int32_t d_prev, int32_t d_k, int32_t with_gprev, int32_t* grid_out) {
  GCNB_REQUIRE(grid_out != nullptr, "bwd grid: null output");
  GCNB_REQUIRE(d_prev >= 1 && d_prev <= 256 && d_k >= 1 && d_k <= 256, "bwd grid: widths out of range");
  BwdPlan plan;
  if (int rc = bwd_plan(n_rows, d_prev, d_k, with_gprev != 0, &plan)) return rc;
  *grid_out = plan.grid;
  return GCNB_OK;
}

extern "C" int gcnb_bwd_layer_f32(const int32_t* row_ptr, const int32_t* col, const float* val,
                                  const int32_t* rows, int32_t n_rows, const float* g, int32_t ldg, int32_t d_k,
                                  const float* h_prev, int32_t ldhp, int32_t d_prev, const float* w,
                                  float* g_prev, int32_t ldgp, int32_t act, float* dw_partials, float* workspace,
                                  void* stream) {
  if (int rc = check_csr_args(row_ptr, col, val, n_rows)) return rc;
  GCNB_REQUIRE(act == GCNB_ACT_RELU || act == GCNB_ACT_IDENTITY, "bwd layer: unknown activation %d", act);
  GCNB_REQUIRE(d_prev >= 1 && d_prev <= 256 && d_k >= 1 && d_k <= 256, "bwd layer: widths out of range");
  GCNB_REQUIRE(ldg % 4 == 0 && ldhp % 4 == 0 && ldg >= round4(d_k) && ldhp >= round4(d_prev),
               "bwd layer: row strides must be multiples of 4 and cover the widths");
  GCNB_REQUIRE(!g_prev || (ldgp % 4 == 0 && ldgp >= round4(d_prev) && aligned16(g_prev) && w && aligned16(w)),
               "bwd layer: G_prev needs W and an aligned stride >= round4(d_prev)");
  GCNB_REQUIRE(g && h_prev && dw_partials && aligned16(g) && aligned16(h_prev) && aligned16(dw_partials),
               "bwd layer: operands must be non-null and 16-byte aligned");
  GCNB_REQUIRE(!workspace || aligned16(workspace), "bwd layer: workspace must be 16-byte aligned");
  BwdPlan plan;
  if (int rc = bwd_plan(n_rows, d_prev, d_k, g_prev != nullptr, &plan)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (workspace && bwd_split(d_prev, d_k) && n_rows > 0) {
    // split mode: the gather-bound aggregation runs at full occupancy (k_agg,
    // cp.async staging), the register-heavy dense epilogue streams agg back
    if (int rc = launch_agg(row_ptr, col, val, rows, n_rows, g, ldg, d_k, workspace, round4(d_k), -1, st,
                            "bwd layer (aggregate)"))
      return rc;
    return launch_bwd_epilogue(workspace, round4(d_k), d_k, h_prev, ldhp, d_prev, w, g_prev, ldgp, act, rows, n_rows,
                               dw_partials, plan, st);
  }
  plan.fn<<<plan.grid, NT, plan.smem, st>>>(row_ptr, col, val, rows, n_rows, g, ldg, d_k, h_prev, ldhp, d_prev, w,
                                            g_prev, ldgp, act, dw_partials, plan.T, EpiPack{});
  GCNB_AFTER_LAUNCH("bwd layer");
  return GCNB_OK;
}

extern "C" int gcnb_dw_f32(const float* x, int32_t ldx, int32_t d_prev, const float* a, int32_t lda, int32_t d_k,
                           const int32_t* rows, int32_t n_rows, float* dw_partials, void* stream) {
  GCNB_REQUIRE(n_rows >= 0, "dw: n_rows must be >= 0");
  GCNB_REQUIRE(d_prev >= 1 && d_prev <= 256 && d_k >= 1 && d_k <= 256, "dw: widths out of range");
  GCNB_REQUIRE(ldx % 4 == 0 && lda % 4 == 0 && ldx >= round4(d_prev) && lda >= round4(d_k),
               "dw: row strides must be multiples of 4 and cover the widths");
  GCNB_REQUIRE(x && a && dw_partials && aligned16(x) && aligned16(a) && aligned16(dw_partials),
               "dw: operands must be non-null and 16-byte aligned");
  BwdPlan plan;
  if (int rc = bwd_plan(n_rows, d_prev, d_k, false, &plan)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (dw_tc_applies(d_prev, d_k))
    return launch_dw_tc(x, ldx, d_prev, a, lda, d_k, rows, n_rows, dw_partials, plan.grid, st);
  // SIMT: the backward kernel without CSR reads A's rows directly as its aggregated tile
  plan.fn<<<plan.grid, NT, plan.smem, st>>>(nullptr, nullptr, nullptr, rows, n_rows, a, lda, d_k, x, ldx, d_prev,
                                            nullptr, nullptr, 0, GCNB_ACT_IDENTITY, dw_partials, plan.T, EpiPack{});
  GCNB_AFTER_LAUNCH("dw");
  return GCNB_OK;
}

extern "C" int gcnb_bwd_epilogue_f32(const float* agg, int32_t ldagg, int32_t d_k, const float* h_prev,
                                     int32_t ldhp, int32_t d_prev, const float* w, float* g_prev, int32_t ldgp,
                                     int32_t act, const uint32_t* hbits, int32_t ld_hbits, const int32_t* rows,
                                     int32_t n_rows, float* dw_partials, void* stream) {
  GCNB_REQUIRE(!hbits || (ld_hbits % 4 == 0 && ld_hbits * 32 >= d_prev && aligned16(hbits)),
               "bwd epilogue: sign-bit rows need a stride of >= d_prev/32 words, a multiple of 4");
  GCNB_REQUIRE(n_rows >= 0, "bwd epilogue: n_rows must be >= 0");
  GCNB_REQUIRE(act == GCNB_ACT_RELU || act == GCNB_ACT_IDENTITY, "bwd epilogue: unknown activation %d", act);
  GCNB_REQUIRE(d_prev >= 1 && d_prev <= 256 && d_k >= 1 && d_k <= 256, "bwd epilogue: widths out of range");
  GCNB_REQUIRE(ldagg % 4 == 0 && ldhp % 4 == 0 && ldagg >= round4(d_k) && ldhp >= round4(d_prev),
               "bwd epilogue: row strides must be multiples of 4 and cover the widths");
  GCNB_REQUIRE(!g_prev || (ldgp % 4 == 0 && ldgp >= round4(d_prev) && aligned16(g_prev) && w && aligned16(w)),
               "bwd epilogue: G_prev needs W and an aligned stride >= round4(d_prev)");
  GCNB_REQUIRE(agg && h_prev && dw_partials && aligned16(agg) && aligned16(h_prev) && aligned16(dw_partials),
               "bwd epilogue: operands must be non-null and 16-byte aligned");
  BwdPlan plan;
  if (int rc = bwd_plan(n_rows, d_prev, d_k, g_prev != nullptr, &plan)) return rc;
  if (n_rows == 0) return GCNB_OK;
  return launch_bwd_epilogue(agg, ldagg, d_k, h_prev, ldhp, d_prev, w, g_prev, ldgp, act, rows, n_rows, dw_partials,
                             plan, (cudaStream_t)stream, hbits, ld_hbits);
}

extern "C" int gcnb_bwd_workspace_ld(int32_t d_prev, int32_t d_k, int32_t* ld_out) {
  GCNB_REQUIRE(ld_out != nullptr, "bwd workspace: null output");
  GCNB_REQUIRE(d_prev >= 1 && d_prev <= 256 && d_k >= 1 && d_k <= 256, "bwd workspace: widths out of range");
  *ld_out = bwd_split(d_prev, d_k) ? round4(d_k) : 0;
  return GCNB_OK;
}

extern "C" int gcnb_reduce_sgd_f32(const float* partials, int32_t n_slots, int64_t size, float* out,
                                   int32_t accumulate, float* w, float lr, void* stream) {
  GCNB_REQUIRE(n_slots >= 0 && size >= 0 && size % 4 == 0, "reduce partials: size must be a multiple of 4");
  GCNB_REQUIRE(out && (n_slots == 0 || partials), "reduce partials: null operands");
  GCNB_REQUIRE(aligned16(out) && (!partials || aligned16(partials)) && (!w || aligned16(w)),
               "reduce partials: operands must be 16-byte aligned");
  GCNB_REQUIRE(!w || (lr > 0.0f && lr < 1e30f), "reduce+sgd: learning rate must be positive and finite");
  if (size == 0) return GCNB_OK;
  const long long size4 = size / 4;
  const int grid = (int)((size4 + 63) / 64);
  cudaStream_t st = (cudaStream_t)stream;
  int stride = 1;
  if (n_slots > RED_SPB) {
    // spread the slot fold over many SMs first (one SM's L2 bandwidth would
    // otherwise bound a ~1 MB partial read), folding in place
    const dim3 g1(grid, (n_slots + RED_SPB - 1) / RED_SPB);
    k_reduce_l1<<<g1, RED_T, 0, st>>>(const_cast<float4*>(reinterpret_cast<const float4*>(partials)), n_slots,
                                       size4);
    GCNB_AFTER_LAUNCH("reduce partials (level 1)");
    stride = RED_SPB;
  }
  k_reduce4<<<grid, RED_T, 0, st>>>(reinterpret_cast<const float4*>(partials), n_slots, stride, size4,
                                    reinterpret_cast<float4*>(out), accumulate, reinterpret_cast<float4*>(w), lr);
  GCNB_AFTER_LAUNCH(w ? "reduce partials + sgd" : "reduce partials");
  return GCNB_OK;
}

extern "C" int gcnb_reduce_partials_f32(const float* partials, int32_t n_slots, int64_t size, float* out,
                                        int32_t accumulate, void* stream) {
  return gcnb_reduce_sgd_f32(partials, n_slots, size, out, accumulate, nullptr, 0.0f, stream);
}

// ---------------------------------------------------------------------------
// Producers with the halo pack fused into their epilogue (epipack.cuh).

namespace {
int pack_of(const gcnb_halo_pack* hp, int ld_out, EpiPack* pk, const char* what) {
  if (!hp || hp->n_seg == 0) {
    *pk = EpiPack{};
    return GCNB_OK;
  }
  GCNB_REQUIRE(hp->ldd >= ld_out, "%s: halo stride %d below the row stride %d", what, hp->ldd, ld_out);
  return make_epipack(pk, hp->map_ptr, hp->map, hp->dst, hp->flags, hp->n_seg, hp->ldd, hp->counter);
}
}  // namespace

extern "C" int gcnb_dense_pack_f32(const float* x, int32_t ldx, int32_t n_rows, int32_t d_in, const float* w,
                                   int32_t d_out, float* y, int32_t ldy, int32_t act, uint32_t* bits,
                                   int32_t ld_bits, const gcnb_halo_pack* pack, void* stream) {
  GCNB_REQUIRE(n_rows >= 0, "dense pack: n_rows must be >= 0");
  GCNB_REQUIRE(act == GCNB_ACT_RELU || act == GCNB_ACT_IDENTITY, "dense pack: unknown activation %d", act);
  GCNB_REQUIRE(d_in >= 1 && d_in <= 256 && d_out >= 1 && d_out <= 256, "dense pack: widths out of range");
  GCNB_REQUIRE(ldx % 4 == 0 && ldy % 4 == 0 && ldx >= round4(d_in) && ldy >= round4(d_out),
               "dense pack: row strides must be multiples of 4 and cover the widths");
  GCNB_REQUIRE(x && w && y && aligned16(x) && aligned16(w) && aligned16(y),
               "dense pack: operands must be 16-byte aligned");
  GCNB_REQUIRE(!bits || (act == GCNB_ACT_RELU && ld_bits % 4 == 0 && ld_bits * 32 >= d_out && aligned16(bits) &&
                         dense_tc_applies(d_in, d_out)),
               "dense pack: sign bits need a ReLU tcgen05 transform and a stride of >= d_out/32 words");
  EpiPack pk;
  if (int rc = pack_of(pack, ldy, &pk, "dense pack")) return rc;
  if (n_rows == 0) return GCNB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dense_tc_applies(d_in, d_out))
    return launch_dense_tc(x, ldx, nullptr, n_rows, d_in, w, d_out, y, ldy, act, st, nullptr, 0, nullptr, 0, nullptr,
                           0, bits, ld_bits, &pk);
  if (dense_blocked_applies(d_in, d_out))
    return launch_dense_blocked(x, ldx, nullptr, n_rows, d_in, w, d_out, y, ldy, act, st, &pk);
  return launch_fwd_gemm(false, nullptr, nullptr, nullptr, nullptr, n_rows, x, ldx, d_in, w, d_out, y, ldy, act, st,
                         "dense pack", pk);
}

extern "C" int gcnb_fwd_layer_pack_f32(const int32_t* row_ptr, const int32_t* col, const float* val, int32_t n_rows,
                                       const float* x, int32_t ldx, int32_t d_in, const float* w, int32_t d_out,
                                       float* h, int32_t ldh, int32_t act, const gcnb_halo_pack* pack,
                                       void* stream) {
  if (int rc = check_csr_args(row_ptr, col, val, n_rows)) return rc;
  GCNB_REQUIRE(act == GCNB_ACT_RELU || act == GCNB_ACT_IDENTITY, "fwd layer pack: unknown activation %d", act);
  GCNB_REQUIRE(d_in >= 1 && d_in <= 256 && d_out >= 1 && d_out <= 256, "fwd layer pack: widths out of range");
  GCNB_REQUIRE(w != nullptr, "fwd layer pack: the fused form needs W (aggregate-only layers pack separately)");
  GCNB_REQUIRE(ldx % 4 == 0 && ldh % 4 == 0 && ldx >= round4(d_in) && ldh >= round4(d_out),
               "fwd layer pack: row strides must be multiples of 4 and cover the widths");
  GCNB_REQUIRE(aligned16(x) && aligned16(h) && aligned16(w), "fwd layer pack: operands must be 16-byte aligned");
  EpiPack pk;
  if (int rc = pack_of(pack, ldh, &pk, "fwd layer pack")) return rc;
  if (n_rows == 0) return GCNB_OK;
  return launch_fwd_gemm(true, row_ptr, col, val, nullptr, n_rows, x, ldx, d_in, w, d_out, h, ldh, act,
                         (cudaStream_t)stream, "fwd layer pack (aggregate+transform)", pk);
}

extern "C" int gcnb_bwd_layer_pack_f32(const int32_t* row_ptr, const int32_t* col, const float* val, int32_t n_rows,
                                       const float* g, int32_t ldg, int32_t d_k, const float* h_prev, int32_t ldhp,
                                       int32_t d_prev, const float* w, float* g_prev, int32_t ldgp, int32_t act,
                                       float* dw_partials, float* workspace, const gcnb_halo_pack* pack,
                                       void* stream) {
  if (int rc = check_csr_args(row_ptr, col, val, n_rows)) return rc;
  GCNB_REQUIRE(act == GCNB_ACT_RELU || act == GCNB_ACT_IDENTITY, "bwd layer pack: unknown activation %d", act);
  GCNB_REQUIRE(d_prev >= 1 && d_prev <= 256 && d_k >= 1 && d_k <= 256, "bwd layer pack: widths out of range");
  GCNB_REQUIRE(ldg % 4 == 0 && ldhp % 4 == 0 && ldg >= round4(d_k) && ldhp >= round4(d_prev),
               "bwd layer pack: row strides must be multiples of 4 and cover the widths");
  GCNB_REQUIRE(g_prev && w && ldgp % 4 == 0 && ldgp >= round4(d_prev) && aligned16(g_prev) && aligned16(w),
               "bwd layer pack: the packed G_prev needs W and an aligned stride >= round4(d_prev)");
  GCNB_REQUIRE(g && h_prev && dw_partials && aligned16(g) && aligned16(h_prev) && aligned16(dw_partials),
               "bwd layer pack: operands must be non-null and 16-byte aligned");
  GCNB_REQUIRE(!workspace || aligned16(workspace), "bwd layer pack: workspace must be 16-byte aligned");
  EpiPack pk;
  if (int rc = pack_of(pack, ldgp, &pk, "bwd layer pack")) return rc;
  BwdPlan plan;
  if (int rc = bwd_plan(n_rows, d_prev, d_k, true, &plan)) return rc;
  if (n_rows == 0) return GCNB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (workspace && bwd_split(d_prev, d_k)) {
    if (int rc = launch_agg(row_ptr, col, val, nullptr, n_rows, g, ldg, d_k, workspace, round4(d_k), -1, st,
                            "bwd layer pack (aggregate)"))
      return rc;
    return launch_bwd_epilogue(workspace, round4(d_k), d_k, h_prev, ldhp, d_prev, w, g_prev, ldgp, act, nullptr,
                               n_rows, dw_partials, plan, st, nullptr, 0, pk);
  }
  plan.fn<<<plan.grid, NT, plan.smem, st>>>(row_ptr, col, val, nullptr, n_rows, g, ldg, d_k, h_prev, ldhp, d_prev, w,
                                            g_prev, ldgp, act, dw_partials, plan.T, pk);
  GCNB_AFTER_LAUNCH("bwd layer pack");
  return GCNB_OK;
}

extern "C" int gcnb_bwd_epilogue_pack_f32(const float* agg, int32_t ldagg, int32_t d_k, const float* h_prev,
                                          int32_t ldhp, int32_t d_prev, const float* w, float* g_prev, int32_t ldgp,
                                          int32_t act, const uint32_t* hbits, int32_t ld_hbits, int32_t n_rows,
                                          float* dw_partials, const gcnb_halo_pack* pack, void* stream) {
  GCNB_REQUIRE(!hbits || (ld_hbits % 4 == 0 && ld_hbits * 32 >= d_prev && aligned16(hbits)),
               "bwd epilogue pack: sign-bit rows need a stride of >= d_prev/32 words, a multiple of 4");
  GCNB_REQUIRE(n_rows >= 0, "bwd epilogue pack: n_rows must be >= 0");
  GCNB_REQUIRE(act == GCNB_ACT_RELU || act == GCNB_ACT_IDENTITY, "bwd epilogue pack: unknown activation %d", act);
  GCNB_REQUIRE(d_prev >= 1 && d_prev <= 256 && d_k >= 1 && d_k <= 256, "bwd epilogue pack: widths out of range");
  GCNB_REQUIRE(ldagg % 4 == 0 && ldhp % 4 == 0 && ldagg >= round4(d_k) && ldhp >= round4(d_prev),
               "bwd epilogue pack: row strides must be multiples of 4 and cover the widths");
  GCNB_REQUIRE(g_prev && w && ldgp % 4 == 0 && ldgp >= round4(d_prev) && aligned16(g_prev) && aligned16(w),
               "bwd epilogue pack: the packed G_prev needs W and an aligned stride >= round4(d_prev)");
  GCNB_REQUIRE(agg && h_prev && dw_partials && aligned16(agg) && aligned16(h_prev) && aligned16(dw_partials),
               "bwd epilogue pack: operands must be non-null and 16-byte aligned");
  EpiPack pk;
  if (int rc = pack_of(pack, ldgp, &pk, "bwd epilogue pack")) return rc;
  BwdPlan plan;
  if (int rc = bwd_plan(n_rows, d_prev, d_k, true, &plan)) return rc;
  if (n_rows == 0) return GCNB_OK;
  return launch_bwd_epilogue(agg, ldagg, d_k, h_prev, ldhp, d_prev, w, g_prev, ldgp, act, nullptr, n_rows,
                             dw_partials, plan, (cudaStream_t)stream, hbits, ld_hbits, pk);
}

extern "C" int gcnb_set_split_all(int32_t on) {
  GCNB_REQUIRE(on == 0 || on == 1, "split all: 0 or 1");
  g_split_all = on;
  return GCNB_OK;
}

extern "C" int gcnb_set_fwd_tf(int32_t on) {
  GCNB_REQUIRE(on == 0 || on == 1, "fwd tf: 0 or 1");
  g_fwd_tf = on;
  return GCNB_OK;
}
