// Register-blocked SIMT fp32 transform Y[r] = act(X[r]·W) for the dense half of
// a layer (the `@ w` of runtime.py:299/304): tall-skinny X (n × K) times a
// small resident W (K × N, K·N ≤ 24 Ki floats).
//
// Exact fp32 is required (TF32 misses the 1e-4 bar, SURVEY key facts), so this
// runs on the FMA pipes: each thread owns an 8 × 8 output block; per k it reads
// 8 X values and 8 W values with four 16-byte shared loads and issues 64 FMAs
// (the generic tile epilogue does 5 loads per 16 FMAs).  X is staged in
// transposed 16-wide k chunks; W stays in shared memory for the persistent
// block.  Per-output accumulation is k-ascending: identical to every other
// transform path in the library (bit-identical results).
#include <algorithm>

#include "common.cuh"
#include "epipack.cuh"

namespace gcnb {

constexpr int DT_M = 8, DT_N = 8, DT_BK = 16;

__global__ void __launch_bounds__(NT) k_dense(const float4* __restrict__ X4, int ldx4, const int* __restrict__ rows,
                                              int n_rows, int K, const float4* __restrict__ W4, int ldN, int N,
                                              float* __restrict__ Y, int ldy, int act, const EpiPack pk) {
  extern __shared__ __align__(16) float sm[];
  const int K4 = (K + 3) & ~3;
  float* Ws = sm;                                  // K4 × ldN (rows >= K zero)
  const int CG = (ldN + DT_N - 1) / DT_N;          // column groups of 8
  const int RG = NT / CG;                          // row groups
  const int BM = RG * DT_M;
  const int xs_ld = BM + 4;
  float* Xs = Ws + K4 * ldN;                       // DT_BK × xs_ld (transposed X chunk)
  for (int idx = threadIdx.x; idx < K4 * ldN / 4; idx += NT)
    reinterpret_cast<float4*>(Ws)[idx] = idx < K * ldN / 4 ? __ldg(W4 + idx) : make_float4(0.f, 0.f, 0.f, 0.f);
  const int cg = threadIdx.x % CG, rg = threadIdx.x / CG;
  const bool active = rg < RG;
  const int n_tiles = (n_rows + BM - 1) / BM;
  __syncthreads();
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int m0 = tile * BM;
    float acc[DT_M][DT_N];
#pragma unroll
    for (int i = 0; i < DT_M; ++i)
#pragma unroll
      for (int j = 0; j < DT_N; ++j) acc[i][j] = 0.0f;
    for (int k0 = 0; k0 < K4; k0 += DT_BK) {
      const int kq_n = min(DT_BK, K4 - k0) / 4;
      for (int idx = threadIdx.x; idx < BM * kq_n; idx += NT) {
        const int m = idx / kq_n, kq = idx - m * kq_n;
        const int i = m0 + m;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < n_rows) {
          const int r = rows ? __ldg(rows + i) : i;
          v = __ldg(X4 + (size_t)r * ldx4 + k0 / 4 + kq);
        }
        float* col = Xs + (4 * kq) * xs_ld + m;
        col[0] = v.x;
        col[xs_ld] = v.y;
        col[2 * xs_ld] = v.z;
        col[3 * xs_ld] = v.w;
      }
      __syncthreads();
      if (active) {
        const int kn = min(DT_BK, K4 - k0);
#pragma unroll 4
        for (int kk = 0; kk < kn; ++kk) {
          const float4 a0 = *reinterpret_cast<const float4*>(Xs + kk * xs_ld + rg * DT_M);
          const float4 a1 = *reinterpret_cast<const float4*>(Xs + kk * xs_ld + rg * DT_M + 4);
          const float4 b0 = *reinterpret_cast<const float4*>(Ws + (k0 + kk) * ldN + cg * DT_N);
          const float4 b1 = *reinterpret_cast<const float4*>(Ws + (k0 + kk) * ldN + cg * DT_N + 4);
          const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
          const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
          for (int i = 0; i < DT_M; ++i)
#pragma unroll
            for (int j = 0; j < DT_N; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
      }
      __syncthreads();
    }
    if (active) {
#pragma unroll
      for (int i = 0; i < DT_M; ++i) {
        const int gi = m0 + rg * DT_M + i;
        if (gi >= n_rows) continue;
        const int r = rows ? __ldg(rows + gi) : gi;
        float* y = Y + (size_t)r * ldy + cg * DT_N;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (cg * DT_N + 4 * h < ldN)
            reinterpret_cast<float4*>(y)[h] =
                act_fwd4(make_float4(acc[i][4 * h], acc[i][4 * h + 1], acc[i][4 * h + 2], acc[i][4 * h + 3]), act);
        }
      }
    }
  }
  if (pk.map_ptr) {
    __syncthreads();
    epi_forward(pk, Y, ldy, rows, n_rows, BM, ldN / 4);
    epi_signal(pk);
  }
}

// Used by gcnb_dense_f32 when the blocked kernel applies (returns false otherwise).
bool dense_blocked_applies(int d_in, int d_out) {
  const int ldN = round4(d_out);
  return ldN >= 32 && round4(d_in) * ldN <= 24 * 1024;
}

int launch_dense_blocked(const float* x, int ldx, const int* rows, int n_rows, int d_in, const float* w, int d_out,
                         float* y, int ldy, int act, cudaStream_t st, const EpiPack* pk) {
  const int ldN = round4(d_out), K4 = round4(d_in);
  const int CG = (ldN + DT_N - 1) / DT_N;
  const int RG = NT / CG;
  const int BM = RG * DT_M;
  const size_t smem = sizeof(float) * ((size_t)K4 * ldN + (size_t)DT_BK * (BM + 4));
  GCNB_REQUIRE(smem <= 227 * 1024, "dense: blocked tile does not fit shared memory");
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dense, NT, smem) != cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    per_sm = 1;
  }
  const int tiles = (n_rows + BM - 1) / BM;
  const int grid = std::max(1, std::min(tiles, per_sm * num_sms()));
  k_dense<<<grid, NT, smem, st>>>(reinterpret_cast<const float4*>(x), ldx / 4, rows, n_rows, d_in,
                                  reinterpret_cast<const float4*>(w), ldN, d_out, y, ldy, act,
                                  pk ? *pk : EpiPack{});
  GCNB_AFTER_LAUNCH("dense (blocked)");
  return GCNB_OK;
}

}  // namespace gcnb
