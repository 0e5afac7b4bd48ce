// Shared-memory mbarrier and TMA helpers (sm_100a) used by the pipelined
// kernels (dense_tc.cu, aggwin.cu).
//
// Watchdog: a parity wait that never completes (a pipeline bug) would hang
// the device.  The wait checks %globaltimer and traps after g_watchdog_ns
// (default 60 s; gcnb_set_watchdog_ms / GCNB_WATCHDOG_MS, 0 = never).  The
// limit is four orders of magnitude above any healthy wait (these kernels run
// for milliseconds), so preemption, time slicing or MPS do not trip it.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

namespace gcnb {

// One copy per translation unit (no relocatable device code); every copy
// registers a host setter with abi.cu at load time.
void register_watchdog_setter(int (*fn)(unsigned long long));
static __device__ unsigned long long g_watchdog_ns = 60000000000ull;
static int watchdog_setter(unsigned long long ns) {
  return cudaMemcpyToSymbol(g_watchdog_ns, &ns, sizeof(ns)) == cudaSuccess ? 0 : 1;
}
static const int g_watchdog_registered = (register_watchdog_setter(&watchdog_setter), 0);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t mbar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(mbar) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}

__device__ __forceinline__ bool mbar_try(uint32_t mbar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(done)
      : "r"(mbar), "r"(parity)
      : "memory");
  return done != 0;
}

// Wait until the phase with `parity` has completed (acquire).
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  if (mbar_try(mbar, parity)) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  const unsigned long long limit = g_watchdog_ns;
  for (;;) {
    if (mbar_try(mbar, parity)) return;
    if (limit) {
      uint64_t now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > limit) {
        printf("gcnb: mbarrier wait timed out (block %d thread %d bar 0x%x parity %u)\n", blockIdx.x, threadIdx.x,
               mbar, parity);
        __trap();
      }
    }
  }
}

// TMA: box at (x, y) of a 2-D tensor map into shared memory, completion counted on mbar
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(mbar)
      : "memory");
}

// 2-D fp32 tensor map: dim0 = `cols` contiguous floats, dim1 = `n_rows` rows
// `ld` floats apart; box {box0, box1}; out-of-range elements read as zero.
// (dense_tc.cu; cuTensorMapEncodeTiled through the runtime's driver entry point.)
bool tmap_2d(CUtensorMap* m, const float* base, int cols, int n_rows, int ld, int box0, int box1,
             CUtensorMapSwizzle sw);

}  // namespace gcnb
