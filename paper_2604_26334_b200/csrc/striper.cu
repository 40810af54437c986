// NVLink-striped streaming: the executing GPU's ring pieces
// are split into stripes and every GPU of the node pulls one stripe over ITS OWN
// PCIe link, writing it straight into the executing GPU's ring through a CUDA-IPC
// mapping (the helper's copy engine reads host memory and writes peer memory over
// NVLink / NVSwitch). Batch-1 decode is host-link bound on one GPU; with N GPUs
// of a node pulling stripes, the link roofline scales with N.
//
// Control path (no NCCL, no host round trip on the executing GPU's critical path):
//   leader host   posts piece commands (seq, source offset in the node-shared
//                 weight blob, destination offset in its ring, stripe size) into a
//                 shared control block (/dev/shm) as it enqueues the pass;
//   leader GPU    on its copy stream, after the ring region's release events:
//                 ps_stripe_signal writes go_seq = seq into the control block
//                 (host-mapped), then copies its own stripe 0;
//   helper j      (one host thread per helper process) waits for go_seq >= seq,
//                 cudaMemcpyAsync(leader ring + stripe j <- shared blob) on its own
//                 stream, then writes seq into done[j] in the leader's device memory;
//   leader GPU    before a piece's first consumer: ps_stripe_wait spins (1 thread,
//                 2 s timeout -> error flag, never a hang) until done[j] >= seq for
//                 every helper.
// The same code runs N processes on one GPU (functional test; no bandwidth gain,
// the stripes share one link) and one process per GPU on a multi-GPU node.
#include <stdint.h>
#include <string.h>

#include <atomic>
#include <chrono>
#include <thread>

#include <cuda.h>

#include "common.cuh"
#include "../../include/pshard.h"

namespace ps {

constexpr int STRIPE_MAX_HELPERS = 15;
constexpr int STRIPE_CMDS = 4096;   // command ring (power of two)

struct StripeCmd {
  uint32_t seq;
  uint32_t pad;
  uint64_t src_off;      // bytes into the shared weight blob
  uint64_t dst_off;      // bytes into the leader's ring base
  uint64_t bytes;        // whole piece
  uint64_t stripe;       // stripe size (last stripe may be shorter)
};

// Lives in a /dev/shm segment mapped by every process of the group.
struct StripeCtl {
  uint32_t magic;
  uint32_t n_helpers;
  volatile uint32_t go_seq;             // written by the leader's GPU
  volatile uint32_t posted;             // commands posted by the leader host
  volatile uint32_t stop;
  volatile uint32_t helper_ready[STRIPE_MAX_HELPERS];
  volatile uint32_t helper_error[STRIPE_MAX_HELPERS];
  cudaIpcMemHandle_t ring_handle;       // leader's ring allocation
  uint64_t ring_offset;                 // ring base - allocation base
  cudaIpcMemHandle_t done_handle;       // leader's done[] flags (device)
  StripeCmd cmds[STRIPE_CMDS];
};

constexpr uint32_t STRIPE_MAGIC = 0x53545250;  // "STRP"

__global__ void stripe_signal_kernel(volatile uint32_t* go, uint32_t seq) {
  __threadfence_system();
  *go = seq;
  __threadfence_system();
}

__global__ void stripe_wait_kernel(const volatile uint32_t* done, int n, uint32_t seq, uint32_t* err,
                                   unsigned* fault, unsigned long long timeout_ns) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int j = 0; j < n; ++j) {
    while ((int)(done[j] - seq) < 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        atomicExch(err, seq);
        if (fault) raise_fault(fault, FAULT_STRIPE, seq);
        return;
      }
      __nanosleep(200);
    }
  }
  __threadfence();
}

}  // namespace ps

using namespace ps;

int ps_preload_striper() {
  int n = 0;
  touch_kernel(stripe_signal_kernel, n);
  touch_kernel(stripe_wait_kernel, n);
  return n;
}

extern "C" {

int ps_stripe_ctl_bytes(long long* n) {
  *n = (long long)sizeof(StripeCtl);
  return PS_OK;
}

// Leader: initialise the control block `ctl_host` (already mapped and registered with
// ps_host_register), export the ring allocation and a fresh done[] array.
typedef CUresult (*GetAddressRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);

int ps_stripe_leader_init(void* ctl_host, int n_helpers, void* ring, void** done_dev) {
  PS_REQUIRE(ctl_host && n_helpers >= 1 && n_helpers <= STRIPE_MAX_HELPERS,
             "ps_stripe_leader_init: n_helpers=%d", n_helpers);
  auto* c = static_cast<StripeCtl*>(ctl_host);
  memset((void*)c, 0, sizeof(StripeCtl));
  c->n_helpers = (uint32_t)n_helpers;
  // an IPC handle names a whole allocation: find the one holding the ring
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  PS_CHECK_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
  PS_REQUIRE(fn && q == cudaDriverEntryPointSuccess, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  PS_REQUIRE(reinterpret_cast<GetAddressRangeFn>(fn)(&base, &size, (CUdeviceptr)ring) == CUDA_SUCCESS,
             "cuMemGetAddressRange failed");
  PS_CHECK_CUDA(cudaIpcGetMemHandle(&c->ring_handle, (void*)base));
  c->ring_offset = (uint64_t)((CUdeviceptr)ring - base);
  void* done = nullptr;
  PS_CHECK_CUDA(cudaMalloc(&done, 512));   // [0, 16) helper flags, [64] wait-timeout flag
  PS_CHECK_CUDA(cudaMemset(done, 0, 512));
  PS_CHECK_CUDA(cudaDeviceSynchronize());
  PS_CHECK_CUDA(cudaIpcGetMemHandle(&c->done_handle, done));
  *done_dev = done;
  std::atomic_thread_fence(std::memory_order_release);
  c->magic = STRIPE_MAGIC;
  return PS_OK;
}

int ps_stripe_leader_free(void* done_dev) {
  if (done_dev) PS_CHECK_CUDA(cudaFree(done_dev));
  return PS_OK;
}

// Leader host: post the command of piece `seq` (before enqueueing its signal).
int ps_stripe_post(void* ctl_host, unsigned seq, long long src_off, long long dst_off, long long bytes,
                   long long stripe) {
  auto* c = static_cast<StripeCtl*>(ctl_host);
  PS_REQUIRE(c && c->magic == STRIPE_MAGIC, "ps_stripe_post: control block not initialised");
  const uint32_t i = c->posted;
  StripeCmd& m = c->cmds[i % STRIPE_CMDS];
  m.seq = seq;
  m.src_off = (uint64_t)src_off;
  m.dst_off = (uint64_t)dst_off;
  m.bytes = (uint64_t)bytes;
  m.stripe = (uint64_t)stripe;
  std::atomic_thread_fence(std::memory_order_release);
  c->posted = i + 1;
  return PS_OK;
}

// Leader GPU, on its copy stream after the region's release waits.
int ps_stripe_signal(void* ctl_dev, unsigned seq, void* stream) {
  auto* go = reinterpret_cast<volatile uint32_t*>(static_cast<char*>(ctl_dev) + offsetof(StripeCtl, go_seq));
  stripe_signal_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(go, seq);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

// Leader GPU, on its compute stream before a striped piece's first consumer.
int ps_stripe_wait(void* done_dev, int n_helpers, unsigned seq, void* stream) {
  auto* done = static_cast<uint32_t*>(done_dev);
  stripe_wait_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(done, n_helpers, seq, done + 64, fault_dev(),
                                                        2000000000ull);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

int ps_stripe_error(void* done_dev, unsigned* seq_out) {
  PS_CHECK_CUDA(cudaMemcpy(seq_out, static_cast<uint32_t*>(done_dev) + 64, 4, cudaMemcpyDeviceToHost));
  return PS_OK;
}

// Helper j (1-based): serve commands until ctl->stop. `blob_host` is this process's
// mapping of the node-shared weight blob (registered pinned). Blocks the calling
// thread; returns the number of bytes this helper copied through *bytes_out.
int ps_stripe_helper_run(void* ctl_host, int j, void* blob_host, long long* bytes_out) {
  auto* c = static_cast<StripeCtl*>(ctl_host);
  PS_REQUIRE(c && j >= 1, "ps_stripe_helper_run: bad arguments");
  auto t_start = std::chrono::steady_clock::now();
  while (c->magic != STRIPE_MAGIC) {
    if (std::chrono::steady_clock::now() - t_start > std::chrono::seconds(120)) {
      ps_set_error("ps_stripe_helper_run: leader never initialised the control block");
      return PS_ERR_ARG;
    }
    std::this_thread::sleep_for(std::chrono::milliseconds(1));
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  PS_REQUIRE(j <= (int)c->n_helpers, "ps_stripe_helper_run: helper %d of %u", j, c->n_helpers);
  const int n_ranks = (int)c->n_helpers + 1;
  void* ring_alloc = nullptr;
  void* done = nullptr;
  PS_CHECK_CUDA(cudaIpcOpenMemHandle(&ring_alloc, c->ring_handle, cudaIpcMemLazyEnablePeerAccess));
  PS_CHECK_CUDA(cudaIpcOpenMemHandle(&done, c->done_handle, cudaIpcMemLazyEnablePeerAccess));
  char* ring = static_cast<char*>(ring_alloc) + c->ring_offset;
  cudaStream_t s;
  PS_CHECK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  uint32_t* seq_src = nullptr;
  PS_CHECK_CUDA(cudaHostAlloc(&seq_src, 1024 * sizeof(uint32_t), cudaHostAllocDefault));
  c->helper_ready[j - 1] = 1;
  long long copied = 0;
  uint32_t next = 0, ring_i = 0;
  int rc = PS_OK;
  while (!c->stop) {
    if (next == c->posted) {   // nothing posted yet
      std::this_thread::yield();
      continue;
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    const StripeCmd m = c->cmds[next % STRIPE_CMDS];
    // wait for the leader's GPU to release the ring region of this piece
    while ((int)(c->go_seq - m.seq) < 0 && !c->stop) std::this_thread::yield();
    if (c->stop) break;
    const uint64_t off = (uint64_t)j * m.stripe;
    if (off < m.bytes) {
      const uint64_t n = m.bytes - off < m.stripe ? m.bytes - off : m.stripe;
      if (cudaMemcpyAsync(ring + m.dst_off + off, static_cast<char*>(blob_host) + m.src_off + off, n,
                          cudaMemcpyHostToDevice, s) != cudaSuccess) {
        c->helper_error[j - 1] = 1;
        rc = PS_ERR_CUDA;
      }
      copied += (long long)n;
    }
    uint32_t* src = seq_src + (ring_i++ % 1024);
    *src = m.seq;
    if (cudaMemcpyAsync(static_cast<uint32_t*>(done) + (j - 1), src, 4, cudaMemcpyHostToDevice, s) != cudaSuccess) {
      c->helper_error[j - 1] = 2;
      rc = PS_ERR_CUDA;
    }
    ++next;
  }
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  cudaFreeHost(seq_src);
  cudaIpcCloseMemHandle(ring_alloc);
  cudaIpcCloseMemHandle(done);
  (void)n_ranks;
  if (bytes_out) *bytes_out = copied;
  if (rc) ps_set_error("ps_stripe_helper_run: a copy failed");
  return rc;
}

int ps_stripe_ready(void* ctl_host, int* n_ready) {
  auto* c = static_cast<StripeCtl*>(ctl_host);
  int n = 0;
  for (uint32_t j = 0; j < c->n_helpers && j < (uint32_t)STRIPE_MAX_HELPERS; ++j) n += c->helper_ready[j] ? 1 : 0;
  *n_ready = n;
  return PS_OK;
}

int ps_stripe_stop(void* ctl_host) {
  auto* c = static_cast<StripeCtl*>(ctl_host);
  c->stop = 1;
  return PS_OK;
}

}  // extern "C"
