// C-ABI runtime utilities: errors, host memory, copies, events.
//
// These are the primitives of the copy-engine weight streamer (SURVEY.md
// §8a row a17): pinned host memory (cudaHostAlloc, exact size, mapped so
// CPU-placed shards can be read zero-copy), cudaMemcpyAsync on a dedicated
// stream, and events that order ring-slot reuse against compute.
#include <stdarg.h>
#include <string.h>

#include <mutex>
#include <vector>

#include "common.cuh"
#include "../../include/pshard.h"

static thread_local char g_err[1024] = "";

void ps_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// Host ranges visible to kernels (mapped cudaHostAlloc / cudaHostRegister). The
// GEMV dispatcher reads weights that live here with the register-burst kernel
// (zero-copy over PCIe) instead of the bulk-copy kernel.
namespace {
std::mutex g_host_mu;
std::vector<std::pair<uintptr_t, size_t>> g_host_ranges;

void host_range_add(const void* p, size_t n) {
  std::lock_guard<std::mutex> g(g_host_mu);
  g_host_ranges.emplace_back(reinterpret_cast<uintptr_t>(p), n);
}

void host_range_remove(const void* p) {
  std::lock_guard<std::mutex> g(g_host_mu);
  for (size_t i = 0; i < g_host_ranges.size(); ++i)
    if (g_host_ranges[i].first == reinterpret_cast<uintptr_t>(p)) {
      g_host_ranges.erase(g_host_ranges.begin() + i);
      return;
    }
}
}  // namespace

namespace ps {
bool is_host_ptr(const void* p) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  std::lock_guard<std::mutex> g(g_host_mu);
  for (const auto& r : g_host_ranges)
    if (a >= r.first && a < r.first + r.second) return true;
  return false;
}
}  // namespace ps

int ps_preload_gemv();
int ps_preload_gemv_tma();
int ps_preload_gemv_tc();
int ps_preload_gemm();
int ps_preload_attention();
int ps_preload_elementwise();
int ps_preload_moe();
int ps_preload_moe_decode();
extern "C" int ps_preload_fetcher();
int ps_preload_striper();
int ps_preload_attention_tc();
int ps_preload_hx();

namespace ps {
int g_pdl = 0;

namespace {
std::once_flag g_fault_once;
unsigned* g_fault_h = nullptr;
unsigned* g_fault_d = nullptr;
void fault_init() {
  if (cudaHostAlloc(reinterpret_cast<void**>(&g_fault_h), 64, cudaHostAllocMapped | cudaHostAllocPortable) !=
      cudaSuccess) {
    cudaGetLastError();
    g_fault_h = nullptr;
    return;
  }
  memset(g_fault_h, 0, 64);
  if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&g_fault_d), g_fault_h, 0) != cudaSuccess) {
    cudaGetLastError();
    g_fault_d = nullptr;
  }
}
}  // namespace

unsigned* fault_host() {
  std::call_once(g_fault_once, fault_init);
  return g_fault_h;
}
unsigned* fault_dev() {
  std::call_once(g_fault_once, fault_init);
  return g_fault_d;
}
}  // namespace ps

extern "C" {

int ps_fault_status(unsigned* words, int reset) {
  volatile unsigned* h = ps::fault_host();
  PS_REQUIRE(h != nullptr && ps::fault_dev() != nullptr, "ps_fault_status: no mapped fault words");
  PS_REQUIRE(words != nullptr, "ps_fault_status: null argument");
  for (int i = 0; i < ps::FAULT_WORDS; ++i) {
    words[i] = h[i];
    if (reset) h[i] = 0;
  }
  return PS_OK;
}

int ps_preload_kernels(int* n_loaded) {
  static int loaded = -1;
  if (loaded < 0)
    loaded = ps_preload_gemv() + ps_preload_gemv_tma() + ps_preload_gemv_tc() + ps_preload_gemm() + ps_preload_attention() +
             ps_preload_elementwise() + ps_preload_moe() + ps_preload_moe_decode() + ps_preload_fetcher() + ps_preload_striper() +
             ps_preload_attention_tc() + ps_preload_hx();
  if (n_loaded) *n_loaded = loaded;
  return PS_OK;
}

const char* ps_last_error(void) { return g_err; }

int ps_abi_version(void) { return PS_ABI_VERSION; }

int ps_device_info(int device, int* sm_count, int* cc_major, int* cc_minor,
                   size_t* total_mem) {
  cudaDeviceProp prop;
  PS_CHECK_CUDA(cudaGetDeviceProperties(&prop, device));
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  if (total_mem) *total_mem = prop.totalGlobalMem;
  return PS_OK;
}

int ps_set_device(int device) {
  PS_CHECK_CUDA(cudaSetDevice(device));
  return PS_OK;
}

int ps_host_alloc(size_t bytes, int mapped, void** out) {
  PS_REQUIRE(out != nullptr, "ps_host_alloc: out is null");
  unsigned flags = cudaHostAllocPortable | (mapped ? cudaHostAllocMapped : 0);
  PS_CHECK_CUDA(cudaHostAlloc(out, bytes, flags));
  if (mapped) host_range_add(*out, bytes);
  return PS_OK;
}

int ps_host_free(void* ptr) {
  if (ptr) {
    host_range_remove(ptr);
    PS_CHECK_CUDA(cudaFreeHost(ptr));
  }
  return PS_OK;
}

int ps_host_register(void* ptr, size_t bytes, int portable) {
  unsigned flags = cudaHostRegisterMapped | (portable ? cudaHostRegisterPortable : 0);
  PS_CHECK_CUDA(cudaHostRegister(ptr, bytes, flags));
  host_range_add(ptr, bytes);
  return PS_OK;
}

int ps_host_unregister(void* ptr) {
  host_range_remove(ptr);
  PS_CHECK_CUDA(cudaHostUnregister(ptr));
  return PS_OK;
}

int ps_host_device_pointer(void* host_ptr, void** dev_ptr) {
  PS_CHECK_CUDA(cudaHostGetDevicePointer(dev_ptr, host_ptr, 0));
  return PS_OK;
}

int ps_device_alloc(size_t bytes, void** out) {
  PS_CHECK_CUDA(cudaMalloc(out, bytes));
  return PS_OK;
}

int ps_device_free(void* ptr) {
  if (ptr) PS_CHECK_CUDA(cudaFree(ptr));
  return PS_OK;
}

int ps_memcpy_async(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes == 0) return PS_OK;
  PS_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream));
  return PS_OK;
}

int ps_memset_async(void* dst, int value, size_t bytes, void* stream) {
  if (bytes == 0) return PS_OK;
  PS_CHECK_CUDA(cudaMemsetAsync(dst, value, bytes, (cudaStream_t)stream));
  return PS_OK;
}

int ps_stream_create(int high_priority, void** out) {
  int lo = 0, hi = 0;
  PS_CHECK_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  cudaStream_t s;
  PS_CHECK_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, high_priority ? hi : lo));
  *out = (void*)s;
  return PS_OK;
}

int ps_stream_destroy(void* stream) {
  if (stream) PS_CHECK_CUDA(cudaStreamDestroy((cudaStream_t)stream));
  return PS_OK;
}

int ps_set_pdl(int on) {
  ps::g_pdl = on ? 1 : 0;
  return PS_OK;
}

int ps_stream_synchronize(void* stream) {
  PS_CHECK_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return PS_OK;
}

int ps_device_synchronize(void) {
  PS_CHECK_CUDA(cudaDeviceSynchronize());
  return PS_OK;
}

int ps_event_create(int timing, void** out) {
  cudaEvent_t e;
  PS_CHECK_CUDA(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
  *out = (void*)e;
  return PS_OK;
}

int ps_event_destroy(void* ev) {
  if (ev) PS_CHECK_CUDA(cudaEventDestroy((cudaEvent_t)ev));
  return PS_OK;
}

int ps_event_record(void* ev, void* stream) {
  PS_CHECK_CUDA(cudaEventRecord((cudaEvent_t)ev, (cudaStream_t)stream));
  return PS_OK;
}

int ps_stream_wait_event(void* stream, void* ev) {
  PS_CHECK_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)ev, 0));
  return PS_OK;
}

int ps_event_synchronize(void* ev) {
  PS_CHECK_CUDA(cudaEventSynchronize((cudaEvent_t)ev));
  return PS_OK;
}

int ps_event_query(void* ev) {
  cudaError_t e = cudaEventQuery((cudaEvent_t)ev);
  if (e == cudaSuccess) return 1;
  if (e == cudaErrorNotReady) { cudaGetLastError(); return 0; }
  ps_set_error("cudaEventQuery -> %s", cudaGetErrorString(e));
  return -PS_ERR_CUDA;
}

int ps_event_elapsed_ms(void* start, void* stop, float* ms) {
  PS_CHECK_CUDA(cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)stop));
  return PS_OK;
}

}  // extern "C"
