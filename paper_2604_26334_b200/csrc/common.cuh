// Shared helpers for the pshard sm_100a kernels and the C-ABI layer.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>

#define PS_OK 0
#define PS_ERR_CUDA 1
#define PS_ERR_ARG 2
#define PS_ERR_UNSUPPORTED 3

// Thread-local last error text, read through ps_last_error().
void ps_set_error(const char* fmt, ...);

#define PS_CHECK_CUDA(expr)                                                        \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess) {                                                       \
      ps_set_error("%s:%d %s -> %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return PS_ERR_CUDA;                                                          \
    }                                                                              \
  } while (0)

#define PS_CHECK_LAUNCH() PS_CHECK_CUDA(cudaGetLastError())

#define PS_REQUIRE(cond, ...)                                                      \
  do {                                                                             \
    if (!(cond)) {                                                                 \
      ps_set_error(__VA_ARGS__);                                                   \
      return PS_ERR_ARG;                                                           \
    }                                                                              \
  } while (0)

namespace ps {

__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// 128-bit streaming load that does not allocate in L1 (weights are read once).
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ float silu(float g) { return g / (1.0f + __expf(-g)); }

__device__ __forceinline__ float block_sum(float v, float* red) {
  // red: >= 32 floats of shared memory
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  int nw = (blockDim.x + 31) >> 5;
  v = (threadIdx.x < nw) ? red[threadIdx.x] : 0.f;
  if (warp == 0) v = warp_sum(v);
  if (threadIdx.x == 0) red[0] = v;
  __syncthreads();
  return red[0];
}

// ---- paged KV cache ----------------------------------------
// A layer's cache is a pool of pages; a page holds 2^page_shift consecutive positions of
// ONE request, each a row of row_elems bf16 ([K heads | V heads]). table[slot *
// bt_stride + p >> page_shift] is the physical page holding request slot's position p
// (the same block table serves every layer). Pages are allocated on demand by the
// executor, in any order; kernels only ever touch pages the table names.
struct KvPages {
  __nv_bfloat16* pool;
  const int* table;
  int bt_stride;
  int page_shift;
  int row_elems;
  __device__ __forceinline__ long long row(int slot, int p) const {
    const int pg = __ldg(table + (long long)slot * bt_stride + (p >> page_shift));
    return ((((long long)pg) << page_shift) + (p & ((1 << page_shift) - 1))) * row_elems;
  }
};

// Host side: validate the C-ABI arguments of a paged cache and build the descriptor.
// page_rows must be a power of two >= 64 (a 64-position TMA box never crosses a page).
inline bool kv_pages(KvPages& kv, const void* pool, int row_elems, const int* table, int bt_stride,
                     int page_rows) {
  if (!pool || !table || bt_stride < 1 || row_elems < 1 || page_rows < 64 || (page_rows & (page_rows - 1)))
    return false;
  kv.pool = static_cast<__nv_bfloat16*>(const_cast<void*>(pool));
  kv.table = table;
  kv.bt_stride = bt_stride;
  kv.page_shift = __builtin_ctz((unsigned)page_rows);
  kv.row_elems = row_elems;
  return true;
}

}  // namespace ps

// Module preloading: touch a kernel so CUDA's lazy loader loads it now. Every TU
// lists the kernels it launches in ps_preload_<tu>(); ps_preload_kernels() calls
// them all. A kernel loaded for the first time while another kernel spins on the
// device (ps_wait_flag) would stall the load until the spin ends — so the executor
// preloads everything before its first pass.
namespace ps {
// ---- programmatic dependent launch (PDL) ---------------------------------------
// Passes whose weights are all VRAM-resident (no ring copies, no fetcher) are
// chains of small dependent kernels; with PDL the next kernel is launched while
// the previous one runs and blocks in griddepcontrol.wait until it completed, so
// the ~2 us launch gap between them disappears (the bulk-copy GEMV additionally
// starts streaming its weights before the wait). Kernels launched through
// launch_k() call pdl_trigger() first and pdl_wait() before touching any buffer
// an earlier kernel writes or reads; both are no-ops for a normal launch.
extern int g_pdl;   // ps_set_pdl(): launch_k() adds the PDL attribute while set

// ---- device-side faults ----------------------------------------------------------
// Spin-waits that give up (fetcher flag, stripe flags, tcgen05 attention barriers)
// record a code in ONE host-mapped word array instead of hanging the GPU; the host
// reads it with a plain load after every pass (ps_fault_status) and raises, so a
// timed-out wait can never return wrong tokens silently. Slots: FAULT_FETCH (the
// sequence number the expert wait gave up on), FAULT_STRIPE (stripe seq),
// FAULT_ATTN (role/barrier code of tcgen05 attention), FAULT_HOST (host-side code),
// FAULT_HEAD (pass sequence the early-head GEMV gave up waiting for).
enum { FAULT_FETCH = 0, FAULT_STRIPE = 1, FAULT_ATTN = 2, FAULT_HOST = 3, FAULT_HEAD = 4, FAULT_WORDS = 5 };
unsigned* fault_host();     // host address of the words (mapped, zero-initialised)
unsigned* fault_dev();      // device alias of the same words
__device__ __forceinline__ void raise_fault(unsigned* words, int slot, unsigned code) {
  atomicCAS_system(words + slot, 0u, code ? code : 1u);
  __threadfence_system();
}

__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

template <typename F>
inline void touch_kernel(F* f, int& n) {
  cudaFuncAttributes a;
  if (cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(f)) == cudaSuccess) ++n;
  else cudaGetLastError();
}
}  // namespace ps
