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
//
// Speculative (pre-gated) prefetch, ps_moe_publish_spec: the publish of layer i also
// carries S experts PREDICTED for layer i+1 (the next router applied to layer i's
// state). The host thread copies layer i's experts, raises the flag, then copies the
// predictions into one of two spare slot sets, so they cross the link while layer i
// computes and layer i+1 routes — time the link would otherwise idle. Layer i+1's
// publish skips every routed expert already in its prediction set (a hit) and lists
// only the misses; slot_of_rank[r] tells the expansion where rank r's bytes are.
// Predictions that miss are wasted link bytes, never wrong results: every expert is
// read from the slot its bytes were copied into.
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
// half): [0] = seq:(count | nspec << 16), [1 + r] = seq:(expert id | slot << 16) for the
// `count` copies of this layer (ascending ids), then the `nspec` speculative copies.
// Every word carries its own tag, so the host can accept the block word by word and the
// GPU needs no system-scope fence (which would queue behind the copy engines' PCIe reads).
constexpr int PUB_HEADER = 1;
constexpr int PUB_SPEC_MAX = 64;

__device__ __forceinline__ unsigned long long pub_word(unsigned seq, int e, int slot) {
  return ((unsigned long long)seq << 32) | (unsigned)e | ((unsigned)slot << 16);
}

// spec == false: every routed expert is copied into slot = its rank. spec == true (one
// CTA, P <= blockDim): rank r's expert is looked up in this layer's prediction set
// (spec_state[set_cur][0..S), set_cur < 0: none) — a hit is already in slot
// k_base + set_cur * S + q and is not copied; a miss goes to slot r. Then the S
// predictions for the next layer (pred[0..S), set_next >= 0) are recorded in
// spec_state[set_next] and published for slots k_base + set_next * S + q.
__global__ void __launch_bounds__(1024)
moe_publish_kernel(const int* __restrict__ ids, int P, int E, int* __restrict__ slot_of_expert,
                   volatile unsigned long long* __restrict__ pub, unsigned seq, bool spec,
                   const int* __restrict__ pred, int S, int* __restrict__ spec_state, int set_cur, int set_next,
                   int k_base, int* __restrict__ slot_of_rank) {
  extern __shared__ int mark[];            // E flags, then 32 warp totals, then E rank -> id
  int* warp_tot = mark + E;
  int* rid = warp_tot + 32;
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
      if (hit) {
        if (spec) rid[rank] = e;
        else pub[PUB_HEADER + rank] = pub_word(seq, e, rank);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  if (!spec) {
    pub[0] = ((unsigned long long)seq << 32) | (unsigned)base;
    return;
  }
  int cnt = 0;
  for (int r = 0; r < base; ++r) {   // <= P entries, serial: a handful in a one-token pass
    const int e = rid[r];
    int slot = r;
    if (set_cur >= 0)
      for (int q = 0; q < S; ++q)
        if (spec_state[set_cur * S + q] == e) slot = k_base + set_cur * S + q;
    slot_of_rank[r] = slot;
    if (slot == r) pub[PUB_HEADER + cnt++] = pub_word(seq, e, slot);
  }
  int ns = 0;
  if (set_next >= 0)
    for (int q = 0; q < S; ++q) {
      const int e = pred[q];
      spec_state[set_next * S + q] = e;
      if (e >= 0 && e < E) pub[PUB_HEADER + cnt + ns++] = pub_word(seq, e, k_base + set_next * S + q);
    }
  pub[0] = ((unsigned long long)seq << 32) | (unsigned)(cnt | ns << 16);
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
  int n_slots; // slots the published slot numbers may name
  // predictions are experts of the NEXT layer: its group's host base, stride, bytes
  const char* spec_base;
  long long spec_stride, spec_bytes;
};

class ExpertFetcher {
 public:
  ExpertFetcher(int max_experts) : max_experts_(max_experts) {}

  int init() {
    PS_CHECK_CUDA(cudaHostAlloc(&pub_host_, pub_words() * sizeof(unsigned long long), cudaHostAllocMapped));
    memset((void*)pub_host_, 0, pub_words() * sizeof(unsigned long long));
    for (auto& b : seq_bytes_) b.store(-1);
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
  int max_experts() const { return max_experts_; }
  long long experts_copied() const { return copied_.load(); }
  // bytes the job of `seq` copies (-1: not processed yet; the slot is reused every kSeqRing seqs)
  long long seq_bytes(unsigned seq) const {
    return seq_tag_[seq % kSeqRing].load(std::memory_order_acquire) == seq ? seq_bytes_[seq % kSeqRing].load() : -1;
  }
  long long bytes_copied() const { return bytes_.load(); }
  int error() const { return error_.load(); }

 private:
  static constexpr int kSeqRing = 1 << 16;

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
      const unsigned hdr = (unsigned)(pub_host_[0] & 0xffffffffu);
      unsigned n = hdr & 0xffffu, ns = hdr >> 16;
      if (n > (unsigned)max_experts_ || ns > (unsigned)PUB_SPEC_MAX) n = ns = 0, error_.store(2);
      // one copy per run of consecutive expert ids into consecutive slots when host and
      // slot strides agree (the run is contiguous on both sides)
      unsigned ids[4096 + PUB_SPEC_MAX], slot[4096 + PUB_SPEC_MAX];
      unsigned total = n + ns;
      for (unsigned r = 0; r < total; ++r) {      // each word carries the tag: wait for this seq's
        unsigned long long w;
        while ((unsigned)((w = pub_host_[PUB_HEADER + r]) >> 32) != j.seq) {
          if (stopping()) break;
        }
        ids[r] = (unsigned)(w & 0xffffu);
        slot[r] = (unsigned)((w >> 16) & 0xffffu);
        if (ids[r] >= (unsigned)max_experts_ || slot[r] >= (unsigned)j.n_slots) {   // never copy outside
          error_.store(2);
          if (r < n) n = r, ns = 0; else ns = r - n;
          total = n + ns;
          break;
        }
      }
      const long long moved = (long long)n * j.expert_bytes + (long long)ns * j.spec_bytes;
      copied_ += total;
      bytes_ += moved;
      seq_bytes_[j.seq % kSeqRing].store(moved);
      seq_tag_[j.seq % kSeqRing].store(j.seq, std::memory_order_release);
      bool half_sent = j.split <= 0;
      auto copy_runs = [&](unsigned r, unsigned end, const char* hbase, long long hstride, long long hbytes) {
        const bool coalesce = hstride == j.slot_stride;
        while (r < end) {
          if (!half_sent && r >= (unsigned)j.split) {   // the first ranks have landed: seq - 1
            flag(j.seq - 1);
            half_sent = true;
          }
          const unsigned e = ids[r];
          unsigned run = 1;
          const unsigned lim = half_sent ? end : (unsigned)j.split;   // runs never cross the split
          while (coalesce && r + run < lim && ids[r + run] == e + run && slot[r + run] == slot[r] + run) ++run;
          const long long bytes = (long long)(run - 1) * hstride + hbytes;
          if (cudaMemcpyAsync(j.slot_base + (long long)slot[r] * j.slot_stride, hbase + (long long)e * hstride,
                              bytes, cudaMemcpyHostToDevice, stream_) != cudaSuccess)
            error_.store(3);
          r += run;
        }
      };
      if (ns && !j.spec_base) error_.store(2);   // predictions published for a job that cannot copy them
      copy_runs(0, n, j.host_base, j.expert_stride, j.expert_bytes);
      flag(j.seq);
      if (ns && j.spec_base)   // predictions for the next layer: behind the flag, link otherwise idle
        copy_runs(n, total, j.spec_base, j.spec_stride, j.spec_bytes);
    }
  }

  void flag(unsigned v) {
    unsigned* src = seq_src_ + (ring_i_++ % kSeqRing);
    *src = v;
    if (cudaMemcpyAsync(flag_dev_, src, sizeof(unsigned), cudaMemcpyHostToDevice, stream_) != cudaSuccess)
      error_.store(3);
  }

  bool stopping() {
    std::lock_guard<std::mutex> g(mu_);
    return stop_;
  }

  int pub_words() const { return PUB_HEADER + max_experts_ + PUB_SPEC_MAX; }

  int max_experts_;
  int device_ = 0;
  std::atomic<long long> seq_bytes_[kSeqRing];
  std::atomic<unsigned> seq_tag_[kSeqRing] = {};
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
                     static_cast<char*>(slot_base), slot_stride, 0, x->max_experts(), nullptr, 0, 0});
  return PS_OK;
}

int ps_fetcher_submit_spec(void* f, unsigned seq, const void* host_base, long long expert_stride,
                           long long expert_bytes, void* slot_base, long long slot_stride, int n_slots,
                           const void* next_base, long long next_stride, long long next_bytes) {
  auto* x = static_cast<ExpertFetcher*>(f);
  PS_REQUIRE(x != nullptr, "ps_fetcher_submit_spec: null fetcher");
  PS_REQUIRE(expert_bytes > 0 && slot_stride >= expert_bytes && n_slots >= 1 && n_slots <= 65535 &&
                 (!next_base || (next_bytes > 0 && slot_stride >= next_bytes)),
             "ps_fetcher_submit_spec: bad sizes / n_slots %d", n_slots);
  x->submit(FetchJob{seq, static_cast<const char*>(host_base), expert_stride, expert_bytes,
                     static_cast<char*>(slot_base), slot_stride, 0, n_slots, static_cast<const char*>(next_base),
                     next_stride, next_bytes});
  return PS_OK;
}

int ps_fetcher_seq_bytes(void* f, unsigned seq, long long* bytes) {
  auto* x = static_cast<ExpertFetcher*>(f);
  PS_REQUIRE(x != nullptr && bytes, "ps_fetcher_seq_bytes: null argument");
  *bytes = x->seq_bytes(seq);
  return PS_OK;
}

int ps_fetcher_submit_split(void* f, unsigned seq, const void* host_base, long long expert_stride,
                            long long expert_bytes, void* slot_base, long long slot_stride, int split) {
  auto* x = static_cast<ExpertFetcher*>(f);
  PS_REQUIRE(x != nullptr, "ps_fetcher_submit_split: null fetcher");
  PS_REQUIRE(expert_bytes > 0 && slot_stride >= expert_bytes && split >= 1 && seq >= 2,
             "ps_fetcher_submit_split: bad sizes / split %d / seq %u", split, seq);
  x->submit(FetchJob{seq, static_cast<const char*>(host_base), expert_stride, expert_bytes,
                     static_cast<char*>(slot_base), slot_stride, split, x->max_experts(), nullptr, 0, 0});
  return PS_OK;
}

int ps_moe_publish(void* f, const int* ids, int P, int E, int* slot_of_expert, unsigned seq, void* stream) {
  auto* x = static_cast<ExpertFetcher*>(f);
  PS_REQUIRE(x != nullptr && P >= 1 && E >= 1, "ps_moe_publish: P=%d E=%d", P, E);
  const int threads = E >= 1024 ? 1024 : (E + 31) / 32 * 32;
  moe_publish_kernel<<<1, threads, (2 * E + 32) * sizeof(int), (cudaStream_t)stream>>>(
      ids, P, E, slot_of_expert, x->pub_dev(), seq, false, nullptr, 0, nullptr, -1, -1, 0, nullptr);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

int ps_moe_publish_spec(void* f, const int* ids, int P, int E, int* slot_of_expert, unsigned seq, const int* pred,
                        int S, int* spec_state, int set_cur, int set_next, int k_base, int* slot_of_rank,
                        void* stream) {
  auto* x = static_cast<ExpertFetcher*>(f);
  PS_REQUIRE(x != nullptr && P >= 1 && E >= 1 && E <= x->max_experts() && P <= 1024 && S >= 0 &&
                 S <= PUB_SPEC_MAX && set_cur >= -1 && set_cur <= 1 && set_next >= -1 && set_next <= 1 &&
                 (S == 0 || spec_state) && slot_of_rank && (set_next < 0 || pred) && k_base >= P,
             "ps_moe_publish_spec: P=%d E=%d S=%d sets %d/%d k_base %d", P, E, S, set_cur, set_next, k_base);
  const int threads = E >= 1024 ? 1024 : (E + 31) / 32 * 32;
  moe_publish_kernel<<<1, threads, (2 * E + 32) * sizeof(int), (cudaStream_t)stream>>>(
      ids, P, E, slot_of_expert, x->pub_dev(), seq, true, pred, S, spec_state, set_cur, set_next, k_base,
      slot_of_rank);
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
