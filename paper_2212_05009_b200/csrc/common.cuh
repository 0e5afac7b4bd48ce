// Shared helpers for the gcnb sm_100a kernels (error plumbing, launch
// accounting, small vector math).  See include/gcnb.h for the ABI contract.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>

#include "../../include/gcnb.h"

namespace gcnb {

struct EpiPack;  // epipack.cuh

constexpr int NT = 256;          // threads per block for the row kernels
constexpr int WARPS = NT / 32;
constexpr int RPT_MAX = 8;       // output rows per thread in the tile GEMMs
constexpr int MAX_DEVICES = 64;

extern std::atomic<uint64_t> g_launches;

int set_error(int code, const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);
int num_sms();
// Work counter (2 ints, zero between launches) for dynamically scheduled
// kernels launched on `st`: one slot per (device, stream), so kernels running
// concurrently on different streams never share a counter.
int* sched_counter(cudaStream_t st);

// rowops.cu: far pass of the windowed aggregation (aggwin.cu) — k_agg over the
// far int2 entries of each row, added to the near partial sums in y, then act.
int launch_agg_far(const int32_t* row_ptr, const int32_t* nnear, const void* entries, int32_t n_rows, const float* x,
                   int32_t ldx, int32_t d, float* y, int32_t ldy, int32_t act, cudaStream_t st);
// dense.cu: register-blocked SIMT transform for the wide dense layers
bool dense_blocked_applies(int d_in, int d_out);
int launch_dense_blocked(const float* x, int ldx, const int* rows, int n_rows, int d_in, const float* w, int d_out,
                         float* y, int ldy, int act, cudaStream_t st, const EpiPack* pk = nullptr);
// dense_tc.cu: tcgen05 3xTF32 transform for the wide dense layers
bool dense_tc_applies(int d_in, int d_out);
// w_nk != nullptr: B = w_nk stored N×K (row stride ld_wnk) instead of w (K×N);
// hmask != nullptr: epilogue y = acc ⊙ σ'(hmask) (backward) instead of act(acc)
// hbits != nullptr: the mask comes from packed sign bits (ld_hbits words per
// row) instead of hmask; bits_out != nullptr (unmasked ReLU): also write the
// sign bits of the output (ld_bits_out words per row) for the backward pass.
int launch_dense_tc(const float* x, int ldx, const int* rows, int n_rows, int d_in, const float* w, int d_out,
                    float* y, int ldy, int act, cudaStream_t st, const float* w_nk = nullptr, int ld_wnk = 0,
                    const float* hmask = nullptr, int ldhm = 0, const uint32_t* hbits = nullptr, int ld_hbits = 0,
                    uint32_t* bits_out = nullptr, int ld_bits_out = 0, const EpiPack* pk = nullptr);
bool dw_tc_applies(int d_prev, int d_k);
int dw_tc_grid(int n_rows);
int launch_dw_tc(const float* h, int ldh, int d_prev, const float* a, int lda, int d_k, const int* rows, int n_rows,
                 float* partials, int n_slots, cudaStream_t st);

// After every <<<>>> launch: surface launch errors, count the launch.
#define GCNB_AFTER_LAUNCH(what)                                         \
  do {                                                                  \
    cudaError_t _e = cudaGetLastError();                                \
    if (_e != cudaSuccess) return ::gcnb::cuda_fail(_e, what);          \
    ::gcnb::g_launches.fetch_add(1, std::memory_order_relaxed);         \
  } while (0)

#define GCNB_REQUIRE(cond, ...)                                         \
  do {                                                                  \
    if (!(cond)) return ::gcnb::set_error(GCNB_EINVAL, __VA_ARGS__);    \
  } while (0)

inline int round4(int d) { return (d + 3) & ~3; }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

__device__ __forceinline__ float4 fma4(float s, const float4& x, float4 a) {
  a.x = fmaf(s, x.x, a.x);
  a.y = fmaf(s, x.y, a.y);
  a.z = fmaf(s, x.z, a.z);
  a.w = fmaf(s, x.w, a.w);
  return a;
}

__device__ __forceinline__ float act_fwd(float z, int act) {
  return act == GCNB_ACT_RELU ? fmaxf(z, 0.0f) : z;
}

__device__ __forceinline__ float4 act_fwd4(float4 z, int act) {
  return make_float4(act_fwd(z.x, act), act_fwd(z.y, act), act_fwd(z.z, act), act_fwd(z.w, act));
}

// σ'(z) expressed through h = σ(z): relu'(z) = (z > 0) = (h > 0) (gcn.py:101-104).
__device__ __forceinline__ float act_grad_from_h(float h, int act) {
  return act == GCNB_ACT_RELU ? (h > 0.0f ? 1.0f : 0.0f) : 1.0f;
}

}  // namespace gcnb
