/*
 * pshard.h — C-ABI of the B200-native pipelined-sharding inference path.
 *
 * The reference (`shardplan`, pure Python) has no native interface: its
 * hot path prices these operations analytically and simulates the
 * pipeline. Each entry point below REPLACES the priced/simulated operation
 * cited beside it with real sm_100a work; the Python host
 * (`paper_2604_26334_b200/runtime/`) binds it through ctypes
 * (INTEGRATION.md shows the binding).
 *
 * Conventions: plain pointers and sizes, no framework types. Device
 * pointers unless stated; "host-mapped" pointers come from ps_host_alloc
 * (mapped=1) and are valid in kernels (zero-copy). `stream` is a
 * cudaStream_t. Every function returns 0 on success, non-zero on error;
 * ps_last_error() returns the thread-local message. No function allocates
 * device memory behind the caller's back (the VRAM budget is enforced by
 * the caller's capped arena).
 */
#ifndef PSHARD_H
#define PSHARD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PS_ABI_VERSION 1

/* GEMV / GEMM epilogues */
#define PS_EPI_STORE 0      /* y = acc (fp32) */
#define PS_EPI_ACCUM 1      /* y += acc (fp32; fused residual add) */
#define PS_EPI_SWIGLU 2     /* rows/cols interleaved gate,up: y[j] = silu(acc[2j]) * acc[2j+1] */
#define PS_EPI_STORE_BF16 3 /* y = bf16(acc) (GEMM only) */

/* ---- errors / device ------------------------------------------------------ */
const char* ps_last_error(void);
int ps_abi_version(void);
int ps_device_info(int device, int* sm_count, int* cc_major, int* cc_minor, size_t* total_mem);
int ps_set_device(int device);
/* Load every kernel of the library now (CUDA lazy module loading would otherwise load
 * a kernel at its first launch — stalling behind any spinning kernel, e.g. ps_wait_flag).
 * The executor calls it once before its first pass; n_loaded may be NULL. */
int ps_preload_kernels(int* n_loaded);

/* ---- host memory and the copy engine --------------------------------------
 * Replace the simulated PCIe channels of `pkg/src/shardplan/simulator.py:156-207`
 * (in-order H2D / D2H uploads, slot release by compute) and the link rate of
 * `pkg/src/shardplan/machine.py:99-101`. */
int ps_host_alloc(size_t bytes, int mapped, void** out);         /* cudaHostAlloc, exact size */
int ps_host_free(void* ptr);
int ps_host_register(void* ptr, size_t bytes, int portable);     /* pin existing memory (/dev/shm) */
int ps_host_unregister(void* ptr);
int ps_host_device_pointer(void* host_ptr, void** dev_ptr);
int ps_device_alloc(size_t bytes, void** out);
int ps_device_free(void* ptr);
int ps_memcpy_async(void* dst, const void* src, size_t bytes, void* stream);
int ps_memset_async(void* dst, int value, size_t bytes, void* stream);
int ps_stream_create(int high_priority, void** out);
int ps_stream_destroy(void* stream);
int ps_stream_synchronize(void* stream);
int ps_device_synchronize(void);
int ps_event_create(int timing, void** out);
int ps_event_destroy(void* ev);
int ps_event_record(void* ev, void* stream);
int ps_stream_wait_event(void* stream, void* ev);
int ps_event_synchronize(void* ev);
int ps_event_query(void* ev);                                    /* 1 done, 0 pending, <0 error */
int ps_event_elapsed_ms(void* start, void* stop, float* ms);

/* ---- K1 / K8: GEMV / skinny GEMM, t <= 32 rows ------------------------------
 * Replaces MATMUL (t, d, n) requests of `pkg/src/shardplan/model_graph.py:147-153`
 * (attention projection), `:173-179` (FFN) and `:202-209` (output head).
 * y[t, n] (epi)= sum_k x[t, k] * W[n, k]; x fp32 [t x ldx], W bf16 [N x ldw]
 * (device, ring slot, or host-mapped for CPU-placed shards), y fp32 [t x ldy].
 * SWIGLU writes N/2 columns. */
int ps_gemv_bf16(const float* x, int ldx, int t, const void* W, int N, int K, long long ldw,
                 float* y, int ldy, int epilogue, void* stream);
/* Device-resident W runs the bulk-copy kernel (8-stage cp.async.bulk ring per SM,
 * gemv_tma.cu); host-mapped W (zero-copy) runs the register-burst kernel (gemv.cu).
 * _cfg forces the kernel (tuning / tests): rows = 0 -> bulk-copy kernel with
 * grid_cap CTAs (0 = one per SM); rows = 2|4 -> register-burst kernel with rows per
 * warp, ksplit warps per row group (1|2|4|8, 0 = auto), grid cap (0 = resident CTAs). */
int ps_gemv_bf16_cfg(const float* x, int ldx, int t, const void* W, int N, int K, long long ldw,
                     float* y, int ldy, int epilogue, void* stream, int rows, int ksplit, int grid_cap);

/* ---- K3: tcgen05/TMEM/TMA GEMM (prefill, batched projections) ---------------
 * Same MATMUL requests at t >= 64. C[M x N] (epi)= A[M x K] * B[N x K]^T,
 * A, B bf16 K-major (row-major), K % 64 == 0. C fp32 (STORE/ACCUM) or bf16
 * (STORE_BF16, SWIGLU: N/2 columns). */
int ps_gemm_bf16(const void* A, int M, int K, long long lda, const void* B, int N, long long ldb,
                 void* C, int ldc, int epilogue, void* stream);
/* Same, kernel forced (tuning / tests): 0 = auto (M > 128 -> 2), 1 = one 128 x 256 tile
 * per CTA, 2 = persistent CTA-pair kernel (tcgen05.mma.cta_group::2, 256 x 256 tiles,
 * double-buffered TMEM accumulator). */
int ps_gemm_bf16_cfg(const void* A, int M, int K, long long lda, const void* B, int N, long long ldb,
                     void* C, int ldc, int epilogue, void* stream, int variant);

/* ---- K2: normalisation, RoPE, KV append ------------------------------------
 * Folded into elementwise_epsilon by the reference
 * (`pkg/src/shardplan/model_graph.py:35,142`); KV append is the KV shard's
 * ELEMENT_WISE request (`:164-171`, kv_append_bytes `:241-246`). */
int ps_rmsnorm(const float* x, int ldx, const int* rows, int n_rows, const void* w, int d,
               float eps, void* out, int ldo, int out_bf16, void* stream);
int ps_qkv_rope_append(float* qkv, int ldq, int t, int n_heads, int n_kv, int head_dim,
                       const int* pos, const int* req, void* kv_pool, int row_elems,
                       const int* block_table, int bt_stride, int page_rows, const void* rope_cs,
                       const void* q_norm, const void* k_norm, float eps, void* stream);

/* ---- K4: attention (GQA / MHA) ----------------------------------------------
 * Replaces GQA/MHA requests (`pkg/src/shardplan/model_graph.py:154-161`) over a PAGED
 * KV cache (KV shard sizing `:299-304,331`): a layer's cache is a pool of pages of
 * page_rows positions (a power of two >= 64) of ONE request each, a row being bf16
 * [K heads | V heads] (row_elems = 2 * n_kv * head_dim). Request slot s's position p is
 * row p % page_rows of physical page block_table[s * bt_stride + p / page_rows]; one
 * block table serves every layer. slot(b) = req_slot[b], or b when req_slot is NULL.
 * kv_pool may be a VRAM-pinned pool, a ring-staged window of a host pool (pages at the
 * same page offsets), or host-mapped memory. */
int ps_attn_decode(const float* q, int ldq, int batch, int n_heads, int n_kv, int head_dim,
                   const int* req_slot, const void* kv_pool, int row_elems, const int* block_table,
                   int bt_stride, int page_rows, const int* lens, int max_len, float scale, float* out,
                   int ldo, float* workspace, long long workspace_floats, void* stream);
/* Workspace floats ps_attn_decode needs for this shape (0 when one split covers max_len). */
int ps_attn_decode_workspace(int batch, int n_heads, int head_dim, int max_len, long long* floats);
int ps_attn_prefill(const float* q, int ldq, int batch, const int* q_start, const int* p0,
                    const int* req_slot, int max_new, int n_heads, int n_kv, int head_dim,
                    const void* kv_pool, int row_elems, const int* block_table, int bt_stride,
                    int page_rows, float scale, void* out, int ldo, int out_bf16, void* stream);

/* Same attention on the tcgen05 tensor cores (attention_tc.cu): S and O accumulate in
 * TMEM, K/V tiles arrive by TMA from the page pool viewed as a 3-D tensor
 * [pool_pages * page_rows][2 * n_kv heads][head_dim], one 64-row box per page half-tile
 * at the block-table row. head_dim 64 or 128. */
int ps_attn_prefill_tc(const float* q, int ldq, int batch, const int* q_start, const int* p0,
                       const int* req_slot, int max_new, int n_heads, int n_kv, int head_dim,
                       const void* kv_pool, int row_elems, const int* block_table, int bt_stride,
                       int page_rows, int pool_pages, float scale, void* out, int ldo, int out_bf16,
                       void* stream);
/* Pipeline watchdog of ps_attn_prefill_tc: non-zero = a barrier wait gave up after 1 s
 * ((role << 24) | (barrier << 16) | key block); reset clears it. */
int ps_attn_tc_watchdog(unsigned* code, int reset);

/* Device-side faults of every spin-wait with a timeout, in host-mapped memory (a plain
 * host load, no CUDA call, no synchronisation): words[0] = expert-fetch sequence the
 * wait gave up on, [1] = stripe sequence, [2] = tcgen05 attention barrier code,
 * [3] = host-side fetcher timeout (sequence never published), [4] = pass sequence the
 * early-head GEMV gave up waiting for. All zero = healthy;
 * reset clears them. The executor raises on any non-zero word after every pass. */
int ps_fault_status(unsigned* words /* [5] */, int reset);

/* "Early head" for one-token passes whose output head is CPU-placed (zero-copy): y[N] =
 * x . W rows, launched on a side stream at the start of the pass with at most grid_cap
 * CTAs; its producers stream W (bf16, or 12-bit coded rows with coded = 1 and ldw bytes)
 * from host memory while the layers compute, its consumers wait for *xflag >= xseq.
 * ps_set_flag writes the flag on the compute stream once x is final. */
int ps_gemv_head_early(const float* x, int K, const void* W, int N, long long ldw, int coded, float* y, int grid_cap,
                       const unsigned* xflag, unsigned xseq, void* stream);
int ps_set_flag(unsigned* flag, unsigned value, void* stream);

/* Coded rows (format of ps_gemv_bf16c, ld_in bytes each) -> bf16 rows (ld_out elements):
 * a GEMM pass that streams coded pieces expands each piece in VRAM for the tcgen05 GEMM. */
int ps_expand_coded(const void* coded, long long ld_in, int rows, int K, void* out, long long ld_out,
                    void* stream);

/* GPU encoder of the exponent-coded rows (csrc/wencode.cu), byte-identical to
 * runtime/wcomp.py encode: per row of a bf16 [N x K] matrix (row stride ld elements,
 * K % 256 == 0) the window base and escape count, then the coded rows (ld_out bytes each,
 * trailer_bytes >= 16 * ceil((1 + max count) / 4)). Replaces the numpy encoder at model
 * load (no reference counterpart: the link format is this build's). */
int ps_wencode_stats(const void* bits, int N, int K, long long ld, int* base_out, int* count_out, void* stream);
int ps_wencode_rows(const void* bits, int N, int K, long long ld, const int* base, int trailer_bytes, void* out,
                    long long ld_out, void* stream);

/* Huffman-coded exponents ("hx", csrc/hx.cu, format in runtime/hxcodec.py): ~10.1 bits
 * per bf16 weight, lossless. ps_hx_expand decodes `rows` rows (whole 64-row blocks;
 * block_off[b] = byte offset of block b from `piece`, device memory) to bf16 rows of
 * ld_out elements, with the matrix's 4096-entry lookup table (runtime/hxcodec.pair_table: uint32
 * s1 | s2 << 8 | bits << 16 | n << 24).
 * Encoder passes: ps_hx_stats (row max exponent + histogram of rowmax - exponent),
 * ps_hx_sizes (bits per 256-weight sub-block, bytes per row, given the code table
 * uint32 length << 16 | bit-reversed code), ps_hx_write (the coded rows at row_off into a
 * zeroed buffer). No reference counterpart: the link format is this build's. */
int ps_hx_expand(const void* piece, const unsigned* block_off, int rows, int K, const void* lut, void* out,
                 long long ld_out, void* stream);
/* The k routed experts of a MoE layer fetched hx-coded into slots (rank j in slot j, or in
 * slot slot_of_rank[j] when non-null — ps_moe_publish_spec's placement; slot stride
 * slot_stride): each slot's span carries the uint32 block offsets of matrix A at
 * word hdr_a and of B at hdr_b, the matrices at mat_a / mat_b; both are expanded in one
 * launch (latency-bound: one launch's latency on the routing chain, not two) into scratch
 * expert j at out_a / out_b (bf16 rows of K_a / K_b) for the bf16 one-token kernels. */
int ps_hx_expand_experts2(const void* slots, long long slot_stride, const int* slot_of_rank, int k, int hdr_a,
                          long long mat_a, int rows_a,
                          int K_a, const void* lut_a, long long out_a, int hdr_b, long long mat_b, int rows_b, int K_b,
                          const void* lut_b, long long out_b, void* scratch, long long scratch_stride, void* stream);
int ps_hx_stats(const void* bits, int N, int K, long long ld, int* rowmax, unsigned long long* hist, void* stream);
int ps_hx_sizes(const void* bits, int N, int K, long long ld, const int* rowmax, const unsigned* table,
                unsigned short* sublen, unsigned* rowbytes, void* stream);
int ps_hx_write(const void* bits, int N, int K, long long ld, const int* rowmax, const unsigned* table,
                const unsigned short* sublen, const unsigned* rowbytes, const unsigned long long* row_off, void* out,
                void* stream);

/* Decode GEMV for 9..32 tokens on the tcgen05 tensor cores (gemv_tc.cu): y[t, n] (epi)=
 * x[t, :] . W[n, :] reading W ONCE (the CUDA-core GEMV takes 8 tokens per launch). W is
 * bf16 [N x K] (row stride ldw elements) or, with coded = 1, exponent-coded rows of ldw
 * bytes (the format of ps_gemv_bf16c). x is split into three bf16 planes (x1 + x2 + x3 =
 * x to fp32 precision) and the three products accumulate in fp32 TMEM: fp32-faithful.
 * Split-K partials are summed in a fixed order (deterministic). workspace: device bytes,
 * 256-byte aligned, at least the x planes (3 * 32 * K * 2 bytes); ps_gemv_tc_workspace(N, K)
 * is the size at which the split-K choice is unconstrained (smaller: fewer splits, the
 * same results up to summation order). t <= 32, K % 64 == 0. */
int ps_gemv_tc(const float* x, int ldx, int t, const void* W, int N, int K, long long ldw, int coded,
               float* y, int ldy, int epilogue, void* workspace, long long workspace_bytes, void* stream);
int ps_gemv_tc_workspace(int N, int K, long long* bytes);

/* Exponent-coded GEMV: y[t, n] (epi)= x[t, :] . W[n, :] with W in the 12-bit format of
 * runtime/wcomp.py: row n (stride ldw bytes) = K sign|mantissa bytes, K/2 bytes of 4-bit
 * exponent codes relative to the row's base (15 = escape), then a trailer of ldw - 1.5 K
 * bytes (16..256): uint32 [base | n_esc << 8, (col << 8 | exp) x n_esc, 0xFFFFFFFF ...].
 * Every row carries its own base and escapes, so one bulk copy per row segment brings
 * everything the decoder needs into shared memory. Same decomposition and accumulation
 * order as ps_gemv_bf16's bulk-copy kernel: bit-identical to ps_gemv_bf16 on the decoded
 * weights, with 25 % fewer weight bytes. t <= 8, K % 256 == 0, Wc 16-byte aligned. */
int ps_gemv_bf16c(const float* x, int ldx, int t, const void* Wc, int N, int K, long long ldw,
                  float* y, int ldy, int epilogue, void* stream);

/* Programmatic dependent launch for the decode-pass kernels (rmsnorm, qkv/RoPE,
 * decode attention + merge, GEMVs, embed, argmax, add, small uploads): while on,
 * each is launched with cudaLaunchAttributeProgrammaticStreamSerialization and
 * waits (griddepcontrol.wait) for the previous kernel inside, so launch gaps
 * overlap. Only valid while no copy or other stream produces a kernel's inputs
 * (the executor enables it for passes over fully resident weights). Default off. */
int ps_set_pdl(int on);

/* ---- K5: MoE router + routed experts ------------------------------------------
 * Replace MOE_ROUTE (t, d, E) and the expert MATMUL (t*k, d, mats*eff) of
 * `pkg/src/shardplan/model_graph.py:181-200`. Everything stays on the device:
 * route_topk (softmax, top-k with ties to the lower id, optional renormalisation)
 * -> plan (pairs grouped by expert, int buffer of ps_moe_plan_ints() ints)
 * -> expert_gu (h = silu(x Wg^T) * (x Wu^T)) -> expert_down -> combine (y += sum_j w_j out_j).
 * Expert e's gate/up rows live at expert_base + e * expert_stride + gu_off
 * ([2*eff x d], gate/up interleaved) and its down matrix at ... + down_off ([d x eff]);
 * expert_base may be host-mapped (zero-copy: only routed experts cross the link).
 * [e_lo, e_hi) restricts the experts processed (a ring piece holding those experts). */
int ps_moe_route_topk(const float* logits, int ldl, int T, int E, int k, int renorm, int* ids,
                      float* w, void* stream);
int ps_moe_plan_ints(int P, int E, long long* n_ints);
int ps_moe_plan(const int* ids, int P, int E, int* plan, void* stream);
int ps_moe_expert_gu(const void* x, int ldx, int x_bf16, const int* plan, int E, int P, int k,
                     const void* expert_base, long long expert_stride, long long gu_off, int eff,
                     int d, float* h, int e_lo, int e_hi, void* stream);
int ps_moe_expert_down(const float* h, const int* plan, int E, int P, const void* expert_base,
                       long long expert_stride, long long down_off, int eff, int d, float* out,
                       int e_lo, int e_hi, void* stream);
/* Same expert kernels with an expert -> slot map: expert e is read from
 * expert_base + slot_of_expert[e] * expert_stride (the routed-expert fetcher's VRAM slots). */
int ps_moe_expert_gu_mapped(const void* x, int ldx, int x_bf16, const int* plan, int E, int P, int k,
                            const void* expert_base, long long expert_stride, long long gu_off, int eff,
                            int d, float* h, int e_lo, int e_hi, const int* slot_of_expert, void* stream);
int ps_moe_expert_down_mapped(const float* h, const int* plan, int E, int P, const void* expert_base,
                              long long expert_stride, long long down_off, int eff, int d, float* out,
                              int e_lo, int e_hi, const int* slot_of_expert, void* stream);
int ps_moe_combine(const float* out, const int* plan, int E, int P, const float* w, int T, int k,
                   int d, float* y, int ldy, void* stream);
/* One-token decode (t = 1) in two launches, no plan: CTA group j streams routed expert
 * ids[j] (slot_of_expert[ids[j]] when not NULL) through a bulk-copy ring,
 * h[j] = silu(x Wg^T) * (x Wu^T) ([k x eff] fp32 scratch); then each CTA streams one
 * row block of all k down matrices and adds sum_j w[j] (h[j] Wd_j^T), j ascending (the
 * order of ps_moe_combine), into y. x, y fp32 [d]; d, eff multiples of 8, <= 2048. */
int ps_moe_decode_experts(const float* x, const int* ids, int k, const int* slot_of_expert,
                          const void* expert_base, long long expert_stride, long long gu_off,
                          long long down_off, int eff, int d, float* h, const float* w, float* y,
                          void* stream);
/* The same on exponent-coded experts (runtime/wcomp.py rows; gu_row_bytes = 1.5 d +
 * trailer, down_row_bytes = 1.5 eff + trailer, every expert of the group the same size):
 * decoded in the consumer loops, bit-identical to ps_moe_decode_experts on the decoded
 * weights. d and eff multiples of 256. */
int ps_moe_decode_experts_c(const float* x, const int* ids, int k, const int* slot_of_expert,
                            const void* expert_base, long long expert_stride, long long gu_off,
                            long long down_off, int eff, int d, int gu_row_bytes, int down_row_bytes,
                            float* h, const float* w, float* y, void* stream);
/* ps_moe_decode_experts (bf16 rows) in phases: phase 1 = gate/up + SwiGLU into h for the
 * routed experts whose slot (rank, slot_of_expert) lies in [rank_lo, rank_hi); phase 2 =
 * down + combine over all k (the same order as the one-call form: bit-identical); 3 =
 * both. Lets the first experts of a layer compute while the rest are still arriving. */
int ps_moe_decode_experts_phase(const float* x, const int* ids, int k, const int* slot_of_expert,
                                const void* expert_base, long long expert_stride, long long gu_off,
                                long long down_off, int eff, int d, float* h, const float* w, float* y, int phase,
                                int rank_lo, int rank_hi, void* stream);

/* ---- routed-expert fetcher (copy-engine uploads of router-selected experts) --
 * Replaces the zero-copy read of a streamed expert group in decode passes: the GPU
 * publishes the routed expert ids (ps_moe_publish, host-mapped, seq-tagged), a host
 * thread enqueues one cudaMemcpyAsync per routed expert into VRAM slots on its own
 * copy stream and then copies `seq` into a device flag; ps_wait_flag holds the
 * compute stream until the flag reaches seq (2 s timeout -> device error flag, no hang).
 * ps_fetcher_submit must be called once per published seq, in seq order. */
int ps_fetcher_create(int max_experts, void** out);
int ps_fetcher_destroy(void* fetcher);
int ps_fetcher_info(void* fetcher, void** copy_stream, void** flag_dev, long long* experts_copied,
                    long long* bytes_copied, int* error);
int ps_fetcher_submit(void* fetcher, unsigned seq, const void* host_base, long long expert_stride,
                      long long expert_bytes, void* slot_base, long long slot_stride);
/* The same, raising the flag to seq - 1 once the first `split` ranks' copies are issued
 * (then to seq after the rest): ps_wait_flag(seq - 1) releases the first experts early.
 * seq >= 2; the caller advances its sequence by 2 per layer. */
int ps_fetcher_submit_split(void* fetcher, unsigned seq, const void* host_base, long long expert_stride,
                            long long expert_bytes, void* slot_base, long long slot_stride, int split);
int ps_moe_publish(void* fetcher, const int* ids, int P, int E, int* slot_of_expert, unsigned seq,
                   void* stream);
/* Speculative (pre-gated) prefetch. ps_moe_publish_spec publishes, for the job submitted
 * with ps_fetcher_submit_spec (slots numbered 0 .. n_slots-1):
 *  - this layer's routed experts NOT already in its prediction set spec_state[set_cur]
 *    (set_cur = -1: no prediction), each into slot = its rank; a predicted expert stays
 *    in slot k_base + set_cur * S + q. slot_of_rank[r] receives rank r's slot (for
 *    ps_hx_expand_experts2);
 *  - then, when set_next >= 0, the S experts pred[0..S) predicted for the next layer,
 *    recorded in spec_state[set_next] and copied AFTER the flag is raised into slots
 *    k_base + set_next * S + q (k_base >= P; the two sets alternate by layer).
 * Predictions only move bytes earlier or waste them; every expert is read from the slot
 * its bytes were copied into. Predictions are copied from the next layer's group
 * (next_base / next_stride / next_bytes; null next_base: none are copied).
 * ps_fetcher_seq_bytes: bytes the job of `seq` copied (-1: not processed yet), for the
 * pass's link-byte count. */
int ps_fetcher_submit_spec(void* fetcher, unsigned seq, const void* host_base, long long expert_stride,
                           long long expert_bytes, void* slot_base, long long slot_stride, int n_slots,
                           const void* next_base, long long next_stride, long long next_bytes);
int ps_moe_publish_spec(void* fetcher, const int* ids, int P, int E, int* slot_of_expert, unsigned seq,
                        const int* pred, int S, int* spec_state, int set_cur, int set_next, int k_base,
                        int* slot_of_rank, void* stream);
int ps_fetcher_seq_bytes(void* fetcher, unsigned seq, long long* bytes);
int ps_wait_flag(void* fetcher, unsigned seq, void* stream);
int ps_fetcher_device_error(void* fetcher, unsigned* seq_out);

/* ---- NVLink-striped streaming (runtime/striping.py) ----------------------------
 * Every GPU of a node pulls one stripe of each leader ring piece over its own PCIe
 * link into the leader's ring (CUDA IPC, peer writes over NVLink). The control block
 * (ps_stripe_ctl_bytes bytes) lives in shared host memory mapped by every process and
 * registered (ps_host_register). Leader: ps_stripe_leader_init exports the VRAM
 * allocation holding `ring` and creates the helpers' done[] flags; per piece,
 * ps_stripe_post (host, before) + ps_stripe_signal (its copy stream, after the
 * region's release waits) + its own stripe; consumers wait with ps_stripe_wait
 * (2 s timeout -> ps_stripe_error). Helper j >= 1: ps_stripe_helper_run serves
 * until ps_stripe_stop. Replaces the single-link channel priced at
 * `pkg/src/shardplan/machine.py:99-101` by N links. */
int ps_stripe_ctl_bytes(long long* n);
int ps_stripe_leader_init(void* ctl_host, int n_helpers, void* ring, void** done_dev);
int ps_stripe_leader_free(void* done_dev);
int ps_stripe_post(void* ctl_host, unsigned seq, long long src_off, long long dst_off, long long bytes,
                   long long stripe);
int ps_stripe_signal(void* ctl_dev, unsigned seq, void* stream);
int ps_stripe_wait(void* done_dev, int n_helpers, unsigned seq, void* stream);
int ps_stripe_error(void* done_dev, unsigned* seq_out);
int ps_stripe_helper_run(void* ctl_host, int j, void* blob_host, long long* bytes_out);
int ps_stripe_ready(void* ctl_host, int* n_ready);   /* helpers attached so far */
int ps_stripe_stop(void* ctl_host);

/* ---- K6: embedding gather (zero-copy from host-mapped table), greedy -------
 * Not priced by the reference (embeddings are outside the plan,
 * `pkg/src/shardplan/model_graph.py:279-297`); the head's MATMUL is
 * `:202-209`. */
int ps_embed_gather(const void* table, const int* ids, int n, int d, float* out, int ldo,
                    void* stream);
int ps_argmax(const float* logits, int rows, int V, int ldl, int* out, void* stream);
int ps_cast_f32_bf16(const float* src, int lds, void* dst, int ldd, int rows, int cols, void* stream);
int ps_add_f32(float* dst, const float* src, long long n, void* stream);
/* <= 4000 bytes host -> device through a kernel's parameter block (no copy engine). */
int ps_upload_small(void* dst, const void* src, int nbytes, void* stream);

/* ---- model load: deterministic random init ----------------------------------
 * dst[i] = bf16_rne(fmaf(2u - 1, scale, bias)), u = splitmix64(seed ^ ((offset + i) * golden)) >> 40
 * scaled to [0, 1). Restated on the CPU by oracle/c/weights.c. */
int ps_init_uniform_bf16(void* dst, size_t n, unsigned long long seed, unsigned long long offset,
                         float scale, float bias, void* stream);
/* Gate/up rows interleaved for the fused SwiGLU epilogue: rows [row_begin, row_begin + n_rows)
 * of the [2 * rows_each x cols] interleaved matrix; row 2j is tensor a's row j (seed_a),
 * row 2j+1 tensor b's row j (seed_b); element (j, c) uses counter j * cols + c. */
/* Output-head init: element i of a [rows x cols] tensor (from `offset`) is the uniform
 * value of ps_init_uniform_bf16 (bias 0) with scale * s_row, s_row = min(u^-1/2, 64) from
 * the row's own hash (heavy-tailed row norms: a clear top-1 logit). */
int ps_init_rowscaled_bf16(void* dst, size_t n, unsigned long long seed, unsigned long long offset,
                           long long cols, float scale, void* stream);
int ps_init_interleaved_bf16(void* dst, long long rows_each, long long row_begin, long long n_rows,
                             int cols, unsigned long long seed_a, unsigned long long seed_b,
                             float scale, float bias, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PSHARD_H */
