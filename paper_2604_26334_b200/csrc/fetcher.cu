// Routed-expert fetcher: copy-engine uploads of the experts a router picked.
//
// A MoE layer's experts are known only after its router runs on the GPU
// (SURVEY.md §7 hard part 6), so a copy-engine upload cannot be enqueued
// ahead of time the way the streamer enqueues dense pieces. Reading the
// routed experts zero-copy works but costs ~8 % of the host link (SM reads
// travel as 128-byte PCIe requests; the copy engine moves larger ones:
// 51 vs 55.6 GB/s measured). The fetcher closes that gap with one host
// thread per executor:
//
//   compute stream:  ... router -> top-k -> ps_moe_publish -> ps_wait_flag -> experts ...
//   host thread:     sees the published expert list (host-mapped, seq-tagged),
//                    enqueues one cudaMemcpyAsync per routed expert into fixed
//                    VRAM slots on its own copy stream, then a 4-byte copy of
//                    the sequence number into a device flag
//   ps_wait_flag:    one thread spins (nanosleep) until the flag reaches seq
//
// ps_moe_publish also writes slot_of_expert[E] (rank among the routed experts,
// -1 otherwise), which the mapped expert kernels use to find each expert's
// slot. The wait kernel gives up after a timeout and raises a device-side
// error flag instead of hanging the GPU if the host thread ever stalls.
#include <stdint.h>
#include <string.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>

#include "common.cuh"
#include "../../include/pshard.h"

namespace ps {

// publish block (host-mapped, 64-bit words tagged with the sequence number in the high
// half): [0] = seq:count, [1 + r] = seq:expert id of rank r (ascending ids). Every word
// carries its own tag, so the host can accept the block word by word and the GPU
// needs no system-scope fence (which would queue behind the copy engines' PCIe reads).
constexpr int PUB_HEADER = 1;

__global__ void __launch_bounds__(1024)
moe_publish_kernel(const int* __restrict__ ids, int P, int E, int* __restrict__ slot_of_expert,
                   volatile unsigned long long* __restrict__ pub, unsigned seq) {
  extern __shared__ int mark[];            // E flags, then 32 warp totals
  int* warp_tot = mark + E;
  __shared__ int base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int e = threadIdx.x; e < E; e += blockDim.x) mark[e] = 0;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int p = threadIdx.x; p < P; p += blockDim.x) mark[ids[p]] = 1;
  __syncthreads();
  // ranks in ascending expert id: ballot prefix within a warp, scan of warp totals
  for (int e0 = 0; e0 < E; e0 += blockDim.x) {
    const int e = e0 + threadIdx.x;
    const bool hit = e < E && mark[e];
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) warp_tot[warp] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = base;
      for (int w = 0; w < nwarps; ++w) { const int t = warp_tot[w]; warp_tot[w] = acc; acc += t; }
      base = acc;
    }
    __syncthreads();
    if (e < E) {
      const int rank = warp_tot[warp] + __popc(m & ((1u << lane) - 1));
      slot_of_expert[e] = hit ? rank : -1;
      if (hit) pub[PUB_HEADER + rank] = ((unsigned long long)seq << 32) | (unsigned)e;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) pub[0] = ((unsigned long long)seq << 32) | (unsigned)base;
}

__global__ void wait_flag_kernel(const volatile unsigned* __restrict__ flag, unsigned seq,
                                 unsigned* __restrict__ error_flag, unsigned* fault,
                                 unsigned long long timeout_ns) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (true) {
    unsigned v = *flag;
    if ((int)(v - seq) >= 0) break;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      atomicExch(error_flag, seq);
      if (fault) raise_fault(fault, FAULT_FETCH, seq);
      break;
    }
    __nanosleep(200);
  }
  __threadfence();
}

struct FetchJob {
  unsigned seq;
  const char* host_base;
  long long expert_stride, expert_bytes;
  char* slot_base;
  long long slot_stride;
  int split;   // > 0: after the first `split` ranks are issued, raise the flag to seq - 1
};

class ExpertFetcher {
 public:
  ExpertFetcher(int max_experts) : max_experts_(max_experts) {}

  int init() {
    PS_CHECK_CUDA(cudaHostAlloc(&pub_host_, (PUB_HEADER + max_experts_) * sizeof(unsigned long long),
                                cudaHostAllocMapped));
    memset((void*)pub_host_, 0, (PUB_HEADER + max_experts_) * sizeof(unsigned long long));
    PS_CHECK_CUDA(cudaHostGetDevicePointer((void**)&pub_dev_, (void*)pub_host_, 0));
    PS_CHECK_CUDA(cudaHostAlloc(&seq_src_, kSeqRing * sizeof(unsigned), cudaHostAllocDefault));
    PS_CHECK_CUDA(cudaMalloc(&flag_dev_, 2 * sizeof(unsigned)));   // [flag, error]
    PS_CHECK_CUDA(cudaMemset(flag_dev_, 0, 2 * sizeof(unsigned)));
    PS_CHECK_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    PS_CHECK_CUDA(cudaGetDevice(&device_));
    thread_ = std::thread([this] { run(); });
    return PS_OK;
  }

  ~ExpertFetcher() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    if (thread_.joinable()) thread_.join();
    if (stream_) {
      cudaStreamSynchronize(stream_);
      cudaStreamDestroy(stream_);
    }
    if (flag_dev_) cudaFree(flag_dev_);
    if (seq_src_) cudaFreeHost(seq_src_);
    if (pub_host_) cudaFreeHost((void*)pub_host_);
  }

  void submit(const FetchJob& j) {
    {
      std::lock_guard<std::mutex> g(mu_);
      q_.push_back(j);
    }
    cv_.notify_one();
  }

  unsigned long long* pub_dev() const { return pub_dev_; }
  unsigned* flag_dev() const { return flag_dev_; }
  cudaStream_t stream() const { return stream_; }
  long long experts_copied() const { return copied_.load(); }
  long long bytes_copied() const { return bytes_.load(); }
  int error() const { return error_.load(); }

 private:
  static constexpr int kSeqRing = 1024;

  void run() {
    cudaSetDevice(device_);
    while (true) {
      FetchJob j;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [this] { return stop_ || !q_.empty(); });
        if (stop_ && q_.empty()) return;
        j = q_.front();
        q_.pop_front();
      }
      // wait for the GPU to publish this layer's routed experts
      auto t0 = std::chrono::steady_clock::now();
      unsigned spins = 0;
      bool seen = true;
      while ((unsigned)(pub_host_[0] >> 32) != j.seq) {
        if (++spins > 4096) {
          std::this_thread::yield();
          if (stopping() || std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30)) {
            error_.store(1);
            seen = false;
            break;
          }
        }
      }
      std::atomic_thread_fence(std::memory_order_acquire);
      if (!seen) {
        // the GPU never published this layer: copy nothing and do NOT raise the
        // sequence flag, so the wait kernel times out and faults instead of letting
        // the expert kernels read whatever the slots hold
        volatile unsigned* fw = fault_host();
        if (fw && fw[FAULT_HOST] == 0) fw[FAULT_HOST] = j.seq ? j.seq : 1;
        continue;
      }
      unsigned n = (unsigned)(pub_host_[0] & 0xffffffffu);
      if (n > (unsigned)max_experts_) n = 0, error_.store(2);
      // one copy per run of consecutive expert ids when host and slot strides agree
      // (slots are in ascending-id order, so the run is contiguous on both sides)
      const bool coalesce = j.expert_stride == j.slot_stride;
      unsigned ids[4096];
      for (unsigned r = 0; r < n; ++r) {      // each word carries the tag: wait for this seq's
        unsigned long long w;
        while ((unsigned)((w = pub_host_[PUB_HEADER + r]) >> 32) != j.seq) {
          if (stopping()) break;
        }
        ids[r] = (unsigned)(w & 0xffffffffu);
        if (ids[r] >= (unsigned)max_experts_) {   // never copy outside the group
          error_.store(2);
          n = r;
          break;
        }
      }
      bool half_sent = j.split <= 0;
      for (unsigned r = 0; r < n;) {
        if (!half_sent && r >= (unsigned)j.split) {   // the first ranks have landed: seq - 1
          unsigned* hs = seq_src_ + (ring_i_++ % kSeqRing);
          *hs = j.seq - 1;
          if (cudaMemcpyAsync(flag_dev_, hs, sizeof(unsigned), cudaMemcpyHostToDevice, stream_) != cudaSuccess)
            error_.store(3);
          half_sent = true;
        }
        const unsigned e = ids[r];
        unsigned run = 1;
        const unsigned lim = half_sent ? n : (unsigned)j.split;   // runs never cross the split
        while (coalesce && r + run < lim && ids[r + run] == e + run) ++run;
        const long long bytes = (long long)(run - 1) * j.expert_stride + j.expert_bytes;
        if (cudaMemcpyAsync(j.slot_base + r * j.slot_stride, j.host_base + (long long)e * j.expert_stride, bytes,
                            cudaMemcpyHostToDevice, stream_) != cudaSuccess)
          error_.store(3);
        r += run;
      }
      copied_ += n;
      bytes_ += (long long)n * j.expert_bytes;
      unsigned* src = seq_src_ + (ring_i_++ % kSeqRing);
      *src = j.seq;
      if (cudaMemcpyAsync(flag_dev_, src, sizeof(unsigned), cudaMemcpyHostToDevice, stream_) != cudaSuccess)
        error_.store(3);
    }
  }

  bool stopping() {
    std::lock_guard<std::mutex> g(mu_);
    return stop_;
  }

  int max_experts_;
  int device_ = 0;
  volatile unsigned long long* pub_host_ = nullptr;
  unsigned long long* pub_dev_ = nullptr;
  unsigned* seq_src_ = nullptr;
  unsigned* flag_dev_ = nullptr;
  unsigned ring_i_ = 0;
  cudaStream_t stream_ = nullptr;
  std::thread thread_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<FetchJob> q_;
  bool stop_ = false;
  std::atomic<long long> copied_{0}, bytes_{0};
  std::atomic<int> error_{0};
};

}  // namespace ps

using namespace ps;

extern "C" {

int ps_preload_fetcher() {
  int n = 0;
  touch_kernel(moe_publish_kernel, n);
  touch_kernel(wait_flag_kernel, n);
  return n;
}

int ps_preload_kernels(int* n_loaded);

int ps_fetcher_create(int max_experts, void** out) {
  PS_REQUIRE(out && max_experts >= 1 && max_experts <= 4096, "ps_fetcher_create: max_experts=%d", max_experts);
  int loaded = 0;
  ps_preload_kernels(&loaded);   // no lazy module load may happen while ps_wait_flag spins
  auto* f = new ExpertFetcher(max_experts);
  int rc = f->init();
  if (rc) {
    delete f;
    return rc;
  }
  *out = f;
  return PS_OK;
}

int ps_fetcher_destroy(void* f) {
  delete static_cast<ExpertFetcher*>(f);
  return PS_OK;
}

int ps_fetcher_info(void* f, void** copy_stream, void** flag_dev, long long* experts_copied, long long* bytes_copied,
                    int* error) {
  auto* x = static_cast<ExpertFetcher*>(f);
  PS_REQUIRE(x != nullptr, "ps_fetcher_info: null fetcher");
  if (copy_stream) *copy_stream = x->stream();
  if (flag_dev) *flag_dev = x->flag_dev();
  if (experts_copied) *experts_copied = x->experts_copied();
  if (bytes_copied) *bytes_copied = x->bytes_copied();
  if (error) *error = x->error();
  return PS_OK;
}

int ps_fetcher_submit(void* f, unsigned seq, const void* host_base, long long expert_stride, long long expert_bytes,
                      void* slot_base, long long slot_stride) {
  auto* x = static_cast<ExpertFetcher*>(f);
  PS_REQUIRE(x != nullptr, "ps_fetcher_submit: null fetcher");
  PS_REQUIRE(expert_bytes > 0 && slot_stride >= expert_bytes, "ps_fetcher_submit: bad sizes");
  x->submit(FetchJob{seq, static_cast<const char*>(host_base), expert_stride, expert_bytes,
                     static_cast<char*>(slot_base), slot_stride, 0});
  return PS_OK;
}

int ps_fetcher_submit_split(void* f, unsigned seq, const void* host_base, long long expert_stride,
                            long long expert_bytes, void* slot_base, long long slot_stride, int split) {
  auto* x = static_cast<ExpertFetcher*>(f);
  PS_REQUIRE(x != nullptr, "ps_fetcher_submit_split: null fetcher");
  PS_REQUIRE(expert_bytes > 0 && slot_stride >= expert_bytes && split >= 1 && seq >= 2,
             "ps_fetcher_submit_split: bad sizes / split %d / seq %u", split, seq);
  x->submit(FetchJob{seq, static_cast<const char*>(host_base), expert_stride, expert_bytes,
                     static_cast<char*>(slot_base), slot_stride, split});
  return PS_OK;
}

int ps_moe_publish(void* f, const int* ids, int P, int E, int* slot_of_expert, unsigned seq, void* stream) {
  auto* x = static_cast<ExpertFetcher*>(f);
  PS_REQUIRE(x != nullptr && P >= 1 && E >= 1, "ps_moe_publish: P=%d E=%d", P, E);
  const int threads = E >= 1024 ? 1024 : (E + 31) / 32 * 32;
  moe_publish_kernel<<<1, threads, (E + 32) * sizeof(int), (cudaStream_t)stream>>>(ids, P, E, slot_of_expert,
                                                                                   x->pub_dev(), seq);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

int ps_wait_flag(void* f, unsigned seq, void* stream) {
  auto* x = static_cast<ExpertFetcher*>(f);
  PS_REQUIRE(x != nullptr, "ps_wait_flag: null fetcher");
  wait_flag_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(x->flag_dev(), seq, x->flag_dev() + 1, fault_dev(),
                                                      2000000000ull /* 2 s */);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

int ps_fetcher_device_error(void* f, unsigned* seq_out) {
  auto* x = static_cast<ExpertFetcher*>(f);
  PS_REQUIRE(x != nullptr && seq_out, "ps_fetcher_device_error: null argument");
  PS_CHECK_CUDA(cudaMemcpy(seq_out, x->flag_dev() + 1, sizeof(unsigned), cudaMemcpyDeviceToHost));
  return PS_OK;
}

}  // extern "C"
