// Library plumbing for the gcnb C ABI: error reporting, launch accounting,
// device memory that can be mapped into peer processes (CUDA IPC), peer access.
#include <cstdarg>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"

namespace gcnb {

std::atomic<uint64_t> g_launches{0};

namespace {
thread_local char t_err[512] = "";
int g_sms[MAX_DEVICES] = {0};
std::mutex g_sms_mu;
}  // namespace

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(t_err, sizeof(t_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return set_error(GCNB_ECUDA, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

int num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= MAX_DEVICES) return 148;
  if (g_sms[dev] == 0) {
    std::lock_guard<std::mutex> lk(g_sms_mu);
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 148;
    }
    g_sms[dev] = n;
  }
  return g_sms[dev];
}

// Zero-initialised at module load on every device; a kernel that takes a
// slot leaves it zero when it finishes (see k_agg).
constexpr int SCHED_SLOTS = 4096;
__device__ int g_sched[2 * SCHED_SLOTS];

int* sched_counter(cudaStream_t st) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, int> slot_of;
  static int next_slot[MAX_DEVICES] = {0};
  static int* base[MAX_DEVICES] = {nullptr};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= MAX_DEVICES) {
    cudaGetLastError();
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(mu);
  if (!base[dev]) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_sched) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    base[dev] = static_cast<int*>(p);
  }
  // A launch captured into a CUDA graph gets a slot of its own (baked into that
  // graph node, never shared): graphs captured on one stream and replayed
  // concurrently on different streams then never race on a counter.  Eager
  // launches share one slot per (device, stream): stream order serialises them.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) != cudaSuccess) cudaGetLastError();
  auto key = std::make_pair(dev, st);
  auto it = slot_of.find(key);
  int slot;
  if (cap == cudaStreamCaptureStatusActive) {
    if (next_slot[dev] >= SCHED_SLOTS) {
      set_error(GCNB_EINVAL, "more than %d captured or per-stream dynamically scheduled launches", SCHED_SLOTS);
      return nullptr;
    }
    slot = next_slot[dev]++;
  } else if (it != slot_of.end()) {
    slot = it->second;
  } else {
    if (next_slot[dev] >= SCHED_SLOTS) {
      set_error(GCNB_EINVAL, "more than %d streams used with dynamically scheduled kernels", SCHED_SLOTS);
      return nullptr;
    }
    slot = next_slot[dev]++;
    slot_of.emplace(key, slot);
  }
  return base[dev] + 2 * slot;
}

}  // namespace gcnb

using namespace gcnb;

extern "C" const char* gcnb_last_error(void) { return t_err; }

namespace gcnb {
// Host setters of every translation unit's watchdog limit (sync.cuh).
static std::vector<int (*)(unsigned long long)>& watchdog_setters() {
  static std::vector<int (*)(unsigned long long)> v;
  return v;
}
void register_watchdog_setter(int (*fn)(unsigned long long)) { watchdog_setters().push_back(fn); }
}  // namespace gcnb

extern "C" int gcnb_set_watchdog_ms(int64_t ms) {
  GCNB_REQUIRE(ms >= 0, "watchdog: negative limit");
  for (auto fn : gcnb::watchdog_setters())
    if (fn((unsigned long long)ms * 1000000ull) != 0) return gcnb::set_error(GCNB_ECUDA, "watchdog: symbol copy failed");
  return GCNB_OK;
}

extern "C" int gcnb_version(void) { return 200; }  // 0.2.0

extern "C" uint64_t gcnb_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

extern "C" int gcnb_device_count(int* out) {
  GCNB_REQUIRE(out != nullptr, "device count: null output");
  cudaError_t e = cudaGetDeviceCount(out);
  if (e != cudaSuccess) {
    *out = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  return GCNB_OK;
}

extern "C" int gcnb_copy_d2h(void* dst_host, const void* src_dev, size_t bytes) {
  GCNB_REQUIRE(dst_host && src_dev, "copy d2h: null pointer");
  cudaError_t e = cudaMemcpy(dst_host, src_dev, bytes, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "copy d2h");
  return GCNB_OK;
}

extern "C" int gcnb_malloc(void** dptr, size_t bytes) {
  GCNB_REQUIRE(dptr != nullptr, "malloc: null output");
  cudaError_t e = cudaMalloc(dptr, bytes ? bytes : 16);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  return GCNB_OK;
}

extern "C" int gcnb_free(void* dptr) {
  if (!dptr) return GCNB_OK;
  cudaError_t e = cudaFree(dptr);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFree");
  return GCNB_OK;
}

extern "C" int gcnb_memset_async(void* dptr, int value, size_t bytes, void* stream) {
  if (bytes == 0) return GCNB_OK;
  GCNB_REQUIRE(dptr != nullptr, "memset: null pointer");
  cudaError_t e = cudaMemsetAsync(dptr, value, bytes, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  return GCNB_OK;
}

extern "C" int gcnb_ipc_get_handle(const void* dptr, uint8_t handle_out[64]) {
  GCNB_REQUIRE(dptr && handle_out, "ipc get handle: null arguments");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dptr));
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  std::memcpy(handle_out, &h, 64);
  return GCNB_OK;
}

extern "C" int gcnb_ipc_open_handle(const uint8_t handle[64], void** dptr_out) {
  GCNB_REQUIRE(handle && dptr_out, "ipc open handle: null arguments");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  cudaError_t e = cudaIpcOpenMemHandle(dptr_out, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
  return GCNB_OK;
}

extern "C" int gcnb_ipc_close_handle(void* dptr) {
  if (!dptr) return GCNB_OK;
  cudaError_t e = cudaIpcCloseMemHandle(dptr);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcCloseMemHandle");
  return GCNB_OK;
}

extern "C" int gcnb_enable_peer_access(int peer_device) {
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return GCNB_OK;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
  return GCNB_OK;
}

extern "C" int gcnb_event_create(void** ev) {
  GCNB_REQUIRE(ev != nullptr, "event create: null output");
  cudaError_t e = cudaEventCreate(reinterpret_cast<cudaEvent_t*>(ev));
  if (e != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
  return GCNB_OK;
}

extern "C" int gcnb_event_destroy(void* ev) {
  if (!ev) return GCNB_OK;
  cudaError_t e = cudaEventDestroy(reinterpret_cast<cudaEvent_t>(ev));
  if (e != cudaSuccess) return cuda_fail(e, "cudaEventDestroy");
  return GCNB_OK;
}

extern "C" int gcnb_event_record(void* ev, void* stream, int32_t external) {
  GCNB_REQUIRE(ev != nullptr, "event record: null event");
  cudaError_t e = cudaEventRecordWithFlags(reinterpret_cast<cudaEvent_t>(ev), (cudaStream_t)stream,
                                           external ? cudaEventRecordExternal : cudaEventRecordDefault);
  if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecordWithFlags");
  return GCNB_OK;
}

extern "C" int gcnb_event_elapsed_ms(void* ev0, void* ev1, float* ms_out) {
  GCNB_REQUIRE(ev0 && ev1 && ms_out, "event elapsed: null arguments");
  cudaError_t e = cudaEventElapsedTime(ms_out, reinterpret_cast<cudaEvent_t>(ev0), reinterpret_cast<cudaEvent_t>(ev1));
  if (e != cudaSuccess) return cuda_fail(e, "cudaEventElapsedTime");
  return GCNB_OK;
}

extern "C" int gcnb_stream_is_capturing(void* stream, int32_t* out) {
  GCNB_REQUIRE(out != nullptr, "stream capture status: null output");
  cudaStreamCaptureStatus st;
  cudaError_t e = cudaStreamIsCapturing((cudaStream_t)stream, &st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamIsCapturing");
  *out = st == cudaStreamCaptureStatusActive ? 1 : 0;
  return GCNB_OK;
}
