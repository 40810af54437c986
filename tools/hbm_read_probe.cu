// HBM read ceiling probe (tooling, not product): how fast can one B200 stream
// a 1 GiB buffer it only reads? Three readers, CUDA-event timed, best of 10:
//   ldg    : grid-stride 128-bit ld.global.nc.L1::no_allocate, xor-accumulated
//   bulk   : one CTA per SM, one producer lane keeping S stages of 16 KB
//            cp.async.bulk copies in flight, consumers only release the stages
//            (the GEMV's memory pipeline with the arithmetic removed)
//   bulk2  : the same with 2 CTAs per SM
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_read_probe hbm_read_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void ldg_kernel(const uint4* __restrict__ p, size_t n, unsigned* out) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678) out[0] = acc;
}

constexpr int STAGE = 16384;

__global__ void bulk_kernel(const char* __restrict__ p, size_t bytes, int stages, unsigned* out) {
  extern __shared__ __align__(128) char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * STAGE);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int consumers = blockDim.x / 32 - 1;
  const size_t per = (bytes / gridDim.x) / STAGE * STAGE;
  const char* base = p + blockIdx.x * per;
  const int n = (int)(per / STAGE);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(consumers));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < n; ++i) {
        int s = i % stages;
        uint32_t ph = ((i / stages) & 1) ^ 1;
        asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}"
                     ::"r"(su32(&empty[s])), "r"(ph));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(STAGE));
        for (int c = 0; c < 4; ++c)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(su32(smem + s * STAGE + c * 4096)), "l"(base + (size_t)i * STAGE + c * 4096),
                       "r"(4096), "r"(su32(&full[s])));
      }
    }
    return;
  }
  unsigned acc = 0;
  for (int i = 0; i < n; ++i) {
    int s = i % stages;
    uint32_t ph = (i / stages) & 1;
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}"
                 ::"r"(su32(&full[s])), "r"(ph));
    acc ^= reinterpret_cast<const unsigned*>(smem + s * STAGE)[threadIdx.x];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])));
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  const size_t bytes = 1ull << 30;
  char* buf;
  unsigned* out;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&out, 4);
  cudaMemset(buf, 1, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto best_of = [&](auto launch) {
    float best = 1e9;
    for (int r = 0; r < 12; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r >= 2 && ms < best) best = ms;
    }
    return bytes / (best / 1e3) / 1e9;
  };
  for (int per_sm : {4, 8, 16})
    printf("{\"reader\": \"ldg\", \"ctas_per_sm\": %d, \"GBps\": %.1f}\n", per_sm,
           best_of([&] { ldg_kernel<<<sms * per_sm, 256>>>((const uint4*)buf, bytes / 16, out); }));
  for (int ctas : {1, 2})
    for (int stages : {4, 6, 8, 12}) {
      if (ctas == 2 && stages > 6) continue;
      size_t smem = stages * (STAGE + 16);
      cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      printf("{\"reader\": \"bulk\", \"ctas_per_sm\": %d, \"stages\": %d, \"GBps\": %.1f}\n", ctas, stages,
             best_of([&] { bulk_kernel<<<sms * ctas, 288, smem>>>(buf, bytes, stages, out); }));
    }
  cudaError_t e = cudaGetLastError();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
