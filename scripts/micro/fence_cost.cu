// Micro-benchmark: what a doorbell-signalled NVLink halo store costs on B200.
// GPU0 kernels store into GPU1 memory (peer access) and signal a flag there;
// each variant is timed with CUDA events over many back-to-back launches.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fence_cost fence_cost.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void red_rel_sys(unsigned long long* p) {
  asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void red_rel_gpu_ctr(int* p, int* old) {
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(*old) : "l"(p) : "memory");
}

// mode bits: 1 store rows, 2 per-block fence.sys, 4 election + last-block signal, 8 per-block gpu atomic
// election (acq_rel.gpu, no sys fence) + last block red.release.sys, 16 per-block red.release.sys
__global__ void k(float4* dst, int rows_per_block, int c4, unsigned long long* flag, int* counter, int mode) {
  if (mode & 1) {
    for (int i = threadIdx.x; i < rows_per_block * c4; i += blockDim.x)
      dst[(size_t)blockIdx.x * rows_per_block * c4 + i] = make_float4(1.f, 2.f, 3.f, 4.f);
  }
  __syncthreads();
  __shared__ int last;
  if (mode & 2) {
    if (threadIdx.x == 0) __threadfence_system();
  }
  if (mode & 4) {
    if (threadIdx.x == 0) {
      __threadfence_system();
      last = atomicAdd(counter, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
      __threadfence_system();
      *counter = 0;
      red_rel_sys(flag);
    }
  }
  if (mode & 8) {
    if (threadIdx.x == 0) {
      int old;
      red_rel_gpu_ctr(counter, &old);
      last = old == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
      *counter = 0;
      red_rel_sys(flag);
    }
  }
  if (mode & 16) {
    if (threadIdx.x == 0) red_rel_sys(flag);
  }
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  const bool peer = n >= 2;
  float4* dst = nullptr;
  unsigned long long* flag = nullptr;
  if (peer) {
    CK(cudaSetDevice(1));
    CK(cudaMalloc(&dst, 256 << 20));
    CK(cudaMalloc(&flag, 64));
    CK(cudaMemset(flag, 0, 64));
    CK(cudaSetDevice(0));
    CK(cudaDeviceEnablePeerAccess(1, 0));
  } else {
    CK(cudaMalloc(&dst, 256 << 20));
    CK(cudaMalloc(&flag, 64));
  }
  float4* ldst = nullptr;
  CK(cudaMalloc(&ldst, 256 << 20));
  int* counter = nullptr;
  CK(cudaMalloc(&counter, 64));
  CK(cudaMemset(counter, 0, 64));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grids[] = {1, 148, 296, 592};
  const int modes[] = {0, 1, 2, 3, 4, 5, 8, 9, 16, 17};
  const char* names[] = {"empty", "store", "fence.sys", "store+fence.sys", "elect(fence.sys)+signal",
                         "store+elect(fence.sys)+signal", "elect(acq_rel.gpu)+signal",
                         "store+elect(acq_rel.gpu)+signal", "per-block red.release.sys",
                         "store+per-block red.release.sys"};
  for (int where = 0; where < (peer ? 2 : 1); ++where) {
    float4* d = where ? dst : ldst;
    for (int g : grids) {
      for (int mi = 0; mi < 10; ++mi) {
        const int mode = modes[mi];
        const int rows = 8, c4 = 4;  // 8 rows x 64 B per block
        for (int w = 0; w < 20; ++w) k<<<g, 256>>>(d, rows, c4, flag, counter, mode);
        CK(cudaDeviceSynchronize());
        const int it = 200;
        cudaEventRecord(a);
        for (int i = 0; i < it; ++i) k<<<g, 256>>>(d, rows, c4, flag, counter, mode);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("%s grid=%4d %-36s %7.2f us/launch\n", where ? "peer " : "local", g, names[mi], 1000.f * ms / it);
      }
    }
  }
  // one launch between events (launch + single kernel latency, not pipelined)
  for (int mi = 0; mi < 10; ++mi) {
    float tot = 0;
    for (int i = 0; i < 50; ++i) {
      cudaEventRecord(a);
      k<<<296, 256>>>(peer ? dst : ldst, 8, 4, flag, counter, modes[mi]);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      tot += ms;
    }
    printf("single grid=296 %-36s %7.2f us\n", names[mi], 1000.f * tot / 50);
  }
  return 0;
}
