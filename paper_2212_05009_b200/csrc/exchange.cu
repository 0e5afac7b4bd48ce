// Halo exchange, loss, reductions and the update step for sm_100a.
//
//   gcnb_pack_rows_f32     sparse.gather_rows + SimNetwork.send (sparse.py:237-261, runtime.py:85-91)
//   gcnb_wait_flags        SimNetwork.recv                      (runtime.py:93-108)
//   gcnb_loss_grad_f32     runtime._local_loss_grad             (runtime.py:309-333)
//   gcnb_sum_buffers_*     allreduce_sum                        (runtime.py:147-157)
//   gcnb_sgd_f32           runtime._apply_update                (runtime.py:359-360)
//
// The send side writes each boundary row once, straight into the receiver's
// halo slot (a peer-mapped NVLink address when ranks live in different
// processes), then rings a per-(src,dst) doorbell with a system-scope release
// increment once every block's stores are globally visible.  The receiver's
// wait kernel acquires the doorbell; no unpack is needed because the halo is
// laid out exactly as the receiver's CSR column space expects.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "epipack.cuh"

namespace gcnb {

struct PackArgs {
  float* dst[GCNB_MAX_PEERS];
  unsigned long long* flag[GCNB_MAX_PEERS];
  int seg_ptr[GCNB_MAX_PEERS + 1];
  int n_seg;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(NT) k_pack(const float4* __restrict__ X4, int ldx4, int c4,
                                             const int* __restrict__ idx, PackArgs a, int ldd4, int* counter,
                                             int signal) {
  const int total = a.seg_ptr[a.n_seg];
  const long long work = (long long)total * c4;
  for (long long t = blockIdx.x * (long long)NT + threadIdx.x; t < work; t += (long long)gridDim.x * NT) {
    const int e = (int)(t / c4);
    const int ch = (int)(t - (long long)e * c4);
    int s = 0;
    while (e >= a.seg_ptr[s + 1]) ++s;
    const float4 v = __ldg(X4 + (size_t)__ldg(idx + e) * ldx4 + ch);
    reinterpret_cast<float4*>(a.dst[s])[(size_t)(e - a.seg_ptr[s]) * ldd4 + ch] = v;
  }
  if (!signal) return;
  // The block's (possibly remote) stores happen-before thread 0's system-scope
  // fence through the barrier (fences are cumulative), so one fence per block
  // suffices; the last block to arrive rings the doorbells.
  __syncthreads();
  if (gridDim.x == 1) {  // small halo: one block, one fence, no election
    if (threadIdx.x == 0) {
      __threadfence_system();
      for (int s = 0; s < a.n_seg; ++s)
        if (a.seg_ptr[s + 1] > a.seg_ptr[s] && a.flag[s]) red_release_sys_add(a.flag[s], 1ull);
    }
    return;
  }
  __shared__ int last;
  if (threadIdx.x == 0) {
    __threadfence_system();
    last = (atomicAdd(counter, 1) == (int)gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence_system();
    *counter = 0;  // every block has arrived: safe to re-arm for the next launch
    for (int s = 0; s < a.n_seg; ++s)
      if (a.seg_ptr[s + 1] > a.seg_ptr[s] && a.flag[s]) red_release_sys_add(a.flag[s], 1ull);
  }
}

struct WaitArgs {
  int src[GCNB_MAX_PEERS];
  int n;
};

__global__ void k_wait(const unsigned long long* flags, WaitArgs a, unsigned long long* expected, int* err,
                       long long timeout_ns) {
  const int i = threadIdx.x;
  if (i >= a.n) return;
  const int s = a.src[i];
  const unsigned long long target = expected[s] + 1ull;
  expected[s] = target;
  if (*(volatile int*)err) return;  // an earlier exchange already failed: do not stack timeouts
  const unsigned long long t0 = globaltimer_ns();
  while (ld_acquire_sys(flags + s) < target) {
    if ((long long)(globaltimer_ns() - t0) > timeout_ns) {
      atomicExch(err, 1);
      return;
    }
    __nanosleep(64);
  }
}

// label[r] >= 0 marks a labelled own row.
constexpr int LOSS_BLOCKS_MAX = 148 * 8;

// A group of LPR lanes owns a row; each lane owns VPL float4 column chunks
// (one 16-byte load/store each).  Unlabelled rows write zeros without reading
// H.  All lanes of a warp run the group shuffles (warp-uniform loop).
__device__ __forceinline__ float f4get(const float4& v, int e) {
  return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
}

template <int LPR, int VPL>
__global__ void __launch_bounds__(NT) k_loss(const float4* __restrict__ H4, int ldh4, int n_rows, int d,
                                             const int* __restrict__ label, double inv_n, float4* __restrict__ G4,
                                             int ldg4, int act, double* __restrict__ partials, const EpiPack pk) {
  constexpr int GPW = 32 / LPR;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int gl = lane & (LPR - 1), gw = lane / LPR;
  const int c4 = (d + 3) / 4;
  const float inv = (float)inv_n;
  double local = 0.0;
  const int warp_global = blockIdx.x * WARPS + warp;
  const int stride = gridDim.x * WARPS * GPW;
  // the next row's label is fetched one iteration ahead (hides its latency)
  int y_next = warp_global * GPW + gw < n_rows ? __ldg(label + warp_global * GPW + gw) : -1;
  for (int row0 = warp_global * GPW; row0 < n_rows; row0 += stride) {
    const int row = row0 + gw;
    const int y = y_next;
    y_next = row + stride < n_rows ? __ldg(label + row + stride) : -1;
    if (!__any_sync(0xffffffffu, y >= 0)) {  // no labelled row in this warp (warp-uniform): zeros only
      if (row < n_rows)
        for (int ch = gl; ch < ldg4; ch += LPR) {
          G4[(size_t)row * ldg4 + ch] = make_float4(0.f, 0.f, 0.f, 0.f);
          epi_store(pk, row, ch, make_float4(0.f, 0.f, 0.f, 0.f));
        }
      continue;
    }
    float4 hv[VPL];
    float m = -INFINITY;
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
      const int ch = gl + q * LPR;
      hv[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (y >= 0 && ch < c4) {
        hv[q] = __ldg(H4 + (size_t)row * ldh4 + ch);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (4 * ch + e < d) m = fmaxf(m, f4get(hv[q], e));
      }
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o, LPR));
    float s = 0.0f;
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
      const int ch = gl + q * LPR;
      if (y >= 0 && ch < c4) {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (4 * ch + e < d) s += expf(f4get(hv[q], e) - m);
      }
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, LPR);
    if (row >= n_rows) continue;
    float4* g = G4 + (size_t)row * ldg4;
    if (y < 0) {
      for (int ch = gl; ch < ldg4; ch += LPR) {
        g[ch] = make_float4(0.f, 0.f, 0.f, 0.f);
        epi_store(pk, row, ch, make_float4(0.f, 0.f, 0.f, 0.f));
      }
      continue;
    }
    const float lse = logf(s);
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
      const int ch = gl + q * LPR;
      if (ch >= ldg4) continue;
      float o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = 4 * ch + e;
        o[e] = 0.0f;
        if (j < d) {
          const float hj = f4get(hv[q], e);
          const float logp = (hj - m) - lse;
          if (j == y) local -= (double)logp;
          o[e] = (expf(logp) - (j == y ? 1.0f : 0.0f)) * inv * act_grad_from_h(hj, act);
        }
      }
      g[ch] = make_float4(o[0], o[1], o[2], o[3]);
      epi_store(pk, row, ch, make_float4(o[0], o[1], o[2], o[3]));
    }
    for (int ch = gl + VPL * LPR; ch < ldg4; ch += LPR) {
      g[ch] = make_float4(0.f, 0.f, 0.f, 0.f);
      epi_store(pk, row, ch, make_float4(0.f, 0.f, 0.f, 0.f));
    }
  }
  // fixed-order block reduction of the per-lane NLL sums
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  __shared__ double wsum[WARPS];
  if (lane == 0) wsum[warp] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < WARPS; ++w) t += wsum[w];
    partials[blockIdx.x] = t;
  }
  epi_signal(pk);
}

// One warp: lane-strided partial sums, then a fixed xor tree (deterministic).
__global__ void k_sum_partials_f64(const double* __restrict__ partials, int n, double* out) {
  double t = 0.0;
  for (int i = threadIdx.x; i < n; i += 32) t += partials[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (threadIdx.x == 0) *out = t;
}

// One vector pushed to several (peer) destinations, then one doorbell per
// destination once every block's stores are visible (the allreduce_sum
// contribution exchange of runtime.py:147-157 over NVLink).
struct PushArgs {
  float4* dst[GCNB_MAX_PEERS];
  unsigned long long* flag[GCNB_MAX_PEERS];
  int n_dst;
};

__global__ void __launch_bounds__(NT) k_push(const float4* __restrict__ src, long long n4, PushArgs a, int* counter) {
  const long long work = n4 * a.n_dst;
  for (long long t = blockIdx.x * (long long)NT + threadIdx.x; t < work; t += (long long)gridDim.x * NT) {
    const int d = (int)(t / n4);
    const long long j = t - (long long)d * n4;
    a.dst[d][j] = __ldg(src + j);
  }
  __syncthreads();  // see k_pack: one cumulative system fence per block
  __shared__ int last;
  if (threadIdx.x == 0) {
    __threadfence_system();
    last = (atomicAdd(counter, 1) == (int)gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence_system();
    *counter = 0;
    for (int d = 0; d < a.n_dst; ++d) red_release_sys_add(a.flag[d], 1ull);
  }
}

// out[j] = Σ_r slots[r*stride + j] in ascending rank order; the f64 in the two
// words after n_f32 of every slot is summed the same way into *loss.
__global__ void k_sum_slots(const float* __restrict__ slots, int p, long long stride, long long n_f32,
                            float* __restrict__ out, double* loss) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n_f32; j += (long long)gridDim.x * blockDim.x) {
    float s = slots[j];
    for (int r = 1; r < p; ++r) s += slots[(size_t)r * stride + j];
    out[j] = s;
  }
  if (loss && blockIdx.x == 0 && threadIdx.x == 0) {
    double t = 0.0;
    for (int r = 0; r < p; ++r) t += *reinterpret_cast<const double*>(slots + (size_t)r * stride + n_f32);
    *loss = t;
  }
}

struct PtrArgsF {
  const float* p[GCNB_MAX_PEERS];
};
struct PtrArgsD {
  const double* p[GCNB_MAX_PEERS];
};

__global__ void k_sum_f32(PtrArgsF a, int p, long long n, float* __restrict__ out) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    float s = a.p[0][j];
    for (int r = 1; r < p; ++r) s += a.p[r][j];
    out[j] = s;
  }
}

__global__ void k_sum_f64(PtrArgsD a, int p, long long n, double* __restrict__ out) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    double s = a.p[0][j];
    for (int r = 1; r < p; ++r) s += a.p[r][j];
    out[j] = s;
  }
}

__global__ void k_sgd(float* __restrict__ w, const float* __restrict__ dw, long long n, float lr) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x)
    w[j] = w[j] - lr * dw[j];
}

__global__ void k_cast_pad(const double* __restrict__ src, int ld_src, long long n_rows, int d,
                           float* __restrict__ dst, int ld_dst) {
  const long long total = n_rows * ld_dst;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long r = t / ld_dst;
    const int j = (int)(t - r * ld_dst);
    dst[t] = j < d ? (float)src[r * ld_src + j] : 0.0f;
  }
}

}  // namespace gcnb

using namespace gcnb;

extern "C" int gcnb_pack_rows_f32(const float* x, int32_t ldx, int32_t d, const int32_t* idx,
                                  const int32_t* seg_ptr, int32_t n_seg, float* const* dst, int32_t ld_dst,
                                  uint64_t* const* flags, int32_t* counter, void* stream) {
  GCNB_REQUIRE(n_seg >= 0 && n_seg <= GCNB_MAX_PEERS, "pack: n_seg=%d out of range", n_seg);
  GCNB_REQUIRE(d >= 1 && d <= 256, "pack: width %d out of range", d);
  GCNB_REQUIRE(ldx % 4 == 0 && ld_dst % 4 == 0 && ldx >= round4(d) && ld_dst >= round4(d),
               "pack: row strides must be multiples of 4 and cover the width");
  if (n_seg == 0) return GCNB_OK;
  GCNB_REQUIRE(seg_ptr && dst && x, "pack: null arguments");
  PackArgs a{};
  a.n_seg = n_seg;
  a.seg_ptr[0] = seg_ptr[0];
  GCNB_REQUIRE(seg_ptr[0] == 0, "pack: seg_ptr[0] must be 0");
  for (int s = 0; s < n_seg; ++s) {
    GCNB_REQUIRE(seg_ptr[s + 1] >= seg_ptr[s], "pack: seg_ptr must be non-decreasing");
    a.seg_ptr[s + 1] = seg_ptr[s + 1];
    a.dst[s] = dst[s];
    a.flag[s] = flags ? reinterpret_cast<unsigned long long*>(flags[s]) : nullptr;
    GCNB_REQUIRE(seg_ptr[s + 1] == seg_ptr[s] || (dst[s] && aligned16(dst[s])),
                 "pack: destination %d must be non-null and 16-byte aligned", s);
  }
  const int total = a.seg_ptr[n_seg];
  const int signal = flags != nullptr;
  GCNB_REQUIRE(!signal || counter, "pack: signalling needs a device counter");
  if (total == 0 && !signal) return GCNB_OK;
  GCNB_REQUIRE(total == 0 || (idx && aligned16(x)), "pack: index list and 16-byte aligned source required");
  const int c4 = round4(d) / 4;
  const long long work = (long long)total * c4;
  // a few rows per thread: fewer blocks → fewer fences and counter arrivals
  // (up to 4·NT chunks a single block: one fence, no last-block election)
  const int grid = (int)std::max<long long>(1, std::min<long long>((work + 4 * NT - 1) / (4 * NT), num_sms() * 2));
  k_pack<<<grid, NT, 0, (cudaStream_t)stream>>>(reinterpret_cast<const float4*>(x), ldx / 4, c4, idx, a, ld_dst / 4,
                                                counter, signal);
  GCNB_AFTER_LAUNCH("pack rows");
  return GCNB_OK;
}

extern "C" int gcnb_wait_flags(const uint64_t* flags, const int32_t* srcs_host, int32_t n, uint64_t* expected,
                               int32_t* err, int32_t timeout_ms, void* stream) {
  GCNB_REQUIRE(n >= 0 && n <= GCNB_MAX_PEERS, "wait: n=%d out of range", n);
  if (n == 0) return GCNB_OK;
  GCNB_REQUIRE(flags && srcs_host && expected && err, "wait: null arguments");
  GCNB_REQUIRE(timeout_ms > 0, "wait: timeout must be positive");
  WaitArgs a{};
  a.n = n;
  for (int i = 0; i < n; ++i) {
    GCNB_REQUIRE(srcs_host[i] >= 0 && srcs_host[i] < GCNB_MAX_PEERS, "wait: source rank out of range");
    a.src[i] = srcs_host[i];
  }
  k_wait<<<1, 64, 0, (cudaStream_t)stream>>>(reinterpret_cast<const unsigned long long*>(flags), a,
                                             reinterpret_cast<unsigned long long*>(expected), err,
                                             (long long)timeout_ms * 1000000LL);
  GCNB_AFTER_LAUNCH("wait flags");
  return GCNB_OK;
}

extern "C" int gcnb_loss_scratch_doubles(void) { return LOSS_BLOCKS_MAX; }

namespace {
int loss_grad(const float* h, int32_t ldh, int32_t n_rows, int32_t d, const int32_t* label, double inv_n_labeled,
              float* g, int32_t ldg, int32_t act, double* scratch, double* loss_sum, cudaStream_t st,
              const EpiPack& pk);
}  // namespace

extern "C" int gcnb_loss_grad_f32(const float* h, int32_t ldh, int32_t n_rows, int32_t d, const int32_t* label,
                                  double inv_n_labeled, float* g, int32_t ldg, int32_t act, double* scratch,
                                  double* loss_sum, void* stream) {
  EpiPack pk{};
  return loss_grad(h, ldh, n_rows, d, label, inv_n_labeled, g, ldg, act, scratch, loss_sum, (cudaStream_t)stream,
                   pk);
}

namespace gcnb {
int make_epipack(EpiPack* pk, const int32_t* map_ptr, const int32_t* map, float* const* dst, uint64_t* const* flags,
                 int32_t n_seg, int32_t ldd, int32_t* counter) {
  *pk = EpiPack{};
  GCNB_REQUIRE(n_seg >= 0 && n_seg <= GCNB_MAX_PEERS, "pack: n_seg=%d out of range", n_seg);
  if (n_seg == 0) return GCNB_OK;
  GCNB_REQUIRE(map_ptr && map && dst && counter && ldd % 4 == 0, "pack: null or inconsistent pack arguments");
  pk->map_ptr = map_ptr;
  pk->map = reinterpret_cast<const int2*>(map);
  pk->counter = counter;
  pk->n_seg = n_seg;
  pk->ldd4 = ldd / 4;
  for (int s = 0; s < n_seg; ++s) {
    GCNB_REQUIRE(dst[s] && aligned16(dst[s]), "pack: destination %d invalid", s);
    pk->dst[s] = reinterpret_cast<float4*>(dst[s]);
    pk->flag[s] = reinterpret_cast<unsigned long long*>(flags ? flags[s] : nullptr);
  }
  return GCNB_OK;
}
}  // namespace gcnb

extern "C" int gcnb_loss_grad_pack_f32(const float* h, int32_t ldh, int32_t n_rows, int32_t d, const int32_t* label,
                                       double inv_n_labeled, float* g, int32_t ldg, int32_t act, double* scratch,
                                       double* loss_sum, const int32_t* map_ptr, const int32_t* map,
                                       float* const* dst, uint64_t* const* flags, int32_t n_seg, int32_t ldd,
                                       int32_t* counter, void* stream) {
  GCNB_REQUIRE(n_seg == 0 || ldd >= ldg, "loss pack: destination stride below the row stride");
  EpiPack pk;
  if (int rc = make_epipack(&pk, map_ptr, map, dst, flags, n_seg, ldd, counter)) return rc;
  return loss_grad(h, ldh, n_rows, d, label, inv_n_labeled, g, ldg, act, scratch, loss_sum, (cudaStream_t)stream,
                   pk);
}

namespace {
int loss_grad(const float* h, int32_t ldh, int32_t n_rows, int32_t d, const int32_t* label, double inv_n_labeled,
              float* g, int32_t ldg, int32_t act, double* scratch, double* loss_sum, cudaStream_t st,
              const EpiPack& pk) {
  GCNB_REQUIRE(n_rows >= 0 && d >= 1 && ldh >= d && ldg >= d, "loss: bad shapes");
  GCNB_REQUIRE(act == GCNB_ACT_RELU || act == GCNB_ACT_IDENTITY, "loss: unknown activation %d", act);
  GCNB_REQUIRE(scratch && loss_sum, "loss: scratch and loss_sum required");
  GCNB_REQUIRE(n_rows == 0 || (h && g && label), "loss: null operands");
  GCNB_REQUIRE(d <= 256, "loss: class count %d above 256", d);
  GCNB_REQUIRE(ldh % 4 == 0 && ldg % 4 == 0 && (n_rows == 0 || (aligned16(h) && aligned16(g))),
               "loss: row strides must be multiples of 4 floats and operands 16-byte aligned");
  const int c4 = (d + 3) / 4;
  int lpr = 1;
  while (lpr < 32 && lpr < c4) lpr <<= 1;
  const int vpl = (c4 + lpr - 1) / lpr;  // 1 or 2
  const int rows_per_block = NT / lpr;
  const int grid = std::max(1, std::min((n_rows + rows_per_block - 1) / rows_per_block, LOSS_BLOCKS_MAX));
  if (n_rows > 0) {
    using LossFn = void (*)(const float4*, int, int, int, const int*, double, float4*, int, int, double*,
                            const EpiPack);
    LossFn fn = vpl == 2 ? k_loss<32, 2>
              : lpr == 1 ? k_loss<1, 1> : lpr == 2 ? k_loss<2, 1> : lpr == 4 ? k_loss<4, 1>
              : lpr == 8 ? k_loss<8, 1> : lpr == 16 ? k_loss<16, 1> : k_loss<32, 1>;
    fn<<<grid, NT, 0, st>>>(reinterpret_cast<const float4*>(h), ldh / 4, n_rows, d, label, inv_n_labeled,
                            reinterpret_cast<float4*>(g), ldg / 4, act, scratch, pk);
    GCNB_AFTER_LAUNCH(pk.map_ptr ? "loss grad (+ fused halo pack)" : "loss grad");
  }
  k_sum_partials_f64<<<1, 32, 0, st>>>(scratch, n_rows > 0 ? grid : 0, loss_sum);
  GCNB_AFTER_LAUNCH("loss sum");
  return GCNB_OK;
}
}  // namespace

extern "C" int gcnb_push_f32(const float* src, int64_t n, float* const* dst, uint64_t* const* flags, int32_t n_dst,
                             int32_t* counter, void* stream) {
  GCNB_REQUIRE(n_dst >= 1 && n_dst <= GCNB_MAX_PEERS, "push: n_dst=%d out of range", n_dst);
  GCNB_REQUIRE(n > 0 && n % 4 == 0, "push: length must be a positive multiple of 4");
  GCNB_REQUIRE(src && dst && flags && counter && aligned16(src), "push: null or misaligned arguments");
  PushArgs a{};
  a.n_dst = n_dst;
  for (int d = 0; d < n_dst; ++d) {
    GCNB_REQUIRE(dst[d] && aligned16(dst[d]) && flags[d], "push: destination %d invalid", d);
    a.dst[d] = reinterpret_cast<float4*>(dst[d]);
    a.flag[d] = reinterpret_cast<unsigned long long*>(flags[d]);
  }
  const long long work = (n / 4) * n_dst;
  const int grid = (int)std::max<long long>(1, std::min<long long>((work + NT - 1) / NT, num_sms() * 2));
  k_push<<<grid, NT, 0, (cudaStream_t)stream>>>(reinterpret_cast<const float4*>(src), n / 4, a, counter);
  GCNB_AFTER_LAUNCH("push");
  return GCNB_OK;
}

__global__ void k_signal(PushArgs a) {
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int d = 0; d < a.n_dst; ++d) red_release_sys_add(a.flag[d], 1ull);
  }
}

extern "C" int gcnb_signal_peers(uint64_t* const* flags, int32_t n, void* stream) {
  GCNB_REQUIRE(n >= 0 && n <= GCNB_MAX_PEERS && (n == 0 || flags), "signal: bad arguments");
  if (n == 0) return GCNB_OK;
  PushArgs a{};
  a.n_dst = n;
  for (int d = 0; d < n; ++d) {
    GCNB_REQUIRE(flags[d] != nullptr, "signal: null flag %d", d);
    a.flag[d] = reinterpret_cast<unsigned long long*>(flags[d]);
  }
  k_signal<<<1, 32, 0, (cudaStream_t)stream>>>(a);
  GCNB_AFTER_LAUNCH("signal peers");
  return GCNB_OK;
}

extern "C" int gcnb_sum_slots_f32(const float* slots, int32_t p, int64_t stride, int64_t n_f32, float* out,
                                  double* loss_out, void* stream) {
  GCNB_REQUIRE(p >= 1 && n_f32 >= 0 && stride >= n_f32 + (loss_out ? 2 : 0), "sum slots: bad shapes");
  GCNB_REQUIRE(slots && out, "sum slots: null operands");
  GCNB_REQUIRE(!loss_out || ((n_f32 % 2) == 0 && (stride % 2) == 0), "sum slots: loss words must be 8-byte aligned");
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n_f32 + NT - 1) / NT, num_sms() * 4));
  k_sum_slots<<<grid, NT, 0, (cudaStream_t)stream>>>(slots, p, stride, n_f32, out, loss_out);
  GCNB_AFTER_LAUNCH("sum slots");
  return GCNB_OK;
}

extern "C" int gcnb_sum_buffers_f32(const float* const* bufs, int32_t p, int64_t n, float* out, void* stream) {
  GCNB_REQUIRE(p >= 1 && p <= GCNB_MAX_PEERS && n >= 0 && bufs && out, "sum buffers: bad arguments");
  if (n == 0) return GCNB_OK;
  PtrArgsF a{};
  for (int r = 0; r < p; ++r) {
    GCNB_REQUIRE(bufs[r] != nullptr, "sum buffers: null buffer %d", r);
    a.p[r] = bufs[r];
  }
  const int grid = (int)std::min<int64_t>((n + NT - 1) / NT, num_sms() * 4);
  k_sum_f32<<<grid, NT, 0, (cudaStream_t)stream>>>(a, p, n, out);
  GCNB_AFTER_LAUNCH("sum buffers f32");
  return GCNB_OK;
}

extern "C" int gcnb_sum_buffers_f64(const double* const* bufs, int32_t p, int64_t n, double* out, void* stream) {
  GCNB_REQUIRE(p >= 1 && p <= GCNB_MAX_PEERS && n >= 0 && bufs && out, "sum buffers: bad arguments");
  if (n == 0) return GCNB_OK;
  PtrArgsD a{};
  for (int r = 0; r < p; ++r) {
    GCNB_REQUIRE(bufs[r] != nullptr, "sum buffers: null buffer %d", r);
    a.p[r] = bufs[r];
  }
  const int grid = (int)std::min<int64_t>((n + NT - 1) / NT, num_sms() * 4);
  k_sum_f64<<<grid, NT, 0, (cudaStream_t)stream>>>(a, p, n, out);
  GCNB_AFTER_LAUNCH("sum buffers f64");
  return GCNB_OK;
}

extern "C" int gcnb_sgd_f32(float* w, const float* dw, int64_t n, float lr, void* stream) {
  GCNB_REQUIRE(n >= 0 && (n == 0 || (w && dw)), "sgd: bad arguments");
  GCNB_REQUIRE(std::isfinite(lr) && lr > 0.0f, "sgd: learning rate must be positive and finite");
  if (n == 0) return GCNB_OK;
  const int grid = (int)std::min<int64_t>((n + NT - 1) / NT, num_sms() * 4);
  k_sgd<<<grid, NT, 0, (cudaStream_t)stream>>>(w, dw, n, lr);
  GCNB_AFTER_LAUNCH("sgd");
  return GCNB_OK;
}

extern "C" int gcnb_cast_pad_f64_f32(const double* src, int32_t ld_src, int64_t n_rows, int32_t d, float* dst,
                                     int32_t ld_dst, void* stream) {
  GCNB_REQUIRE(n_rows >= 0 && d >= 0 && ld_src >= d && ld_dst >= d, "cast: bad shapes");
  if (n_rows == 0 || ld_dst == 0) return GCNB_OK;
  GCNB_REQUIRE(src && dst, "cast: null operands");
  const long long total = n_rows * (long long)ld_dst;
  const int grid = (int)std::min<long long>((total + NT - 1) / NT, num_sms() * 8);
  k_cast_pad<<<grid, NT, 0, (cudaStream_t)stream>>>(src, ld_src, n_rows, d, dst, ld_dst);
  GCNB_AFTER_LAUNCH("cast pad");
  return GCNB_OK;
}
