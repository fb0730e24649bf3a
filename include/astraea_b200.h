/*
 * astraea_b200.h -- C ABI of the B200 (sm_100a) data path driven by
 * Astraea's state-aware scheduler (arXiv 2512.14142).
 *
 * The reference (pkg/src/agentsched, pure Python) has no FFI: every GPU
 * action is a cost-model delay. Each entry point below names the reference
 * symbol whose *delay* it replaces with real device work; the host plugin
 * (paper_2512_14142_b200.gpu, and the ctypes stub in INTEGRATION.md) calls
 * them at exactly those seams.
 *
 * Conventions
 *   - Every function returns int: 0 on success, a positive cudaError_t, or
 *     a negative ASTRAEA_E* code. Nothing throws across the ABI.
 *   - Pointers named *_dev are device (HBM) pointers; *_host are host
 *     pointers (pinned where a copy engine or SM reads them directly).
 *   - All device work is stream-ordered on the caller's stream (a
 *     cudaStream_t passed as void*); no call synchronises the device except
 *     where stated.
 *   - bf16 tensors are row-major and contiguous unless a stride is given.
 *
 * KV pool layout (HBM), block-major so a swap moves whole blocks:
 *   pool[num_blocks][num_layers][2 (K,V)][num_kv_heads][block_tokens][head_dim]  bf16
 * One (block, layer, K|V, head) page is block_tokens*head_dim*2 bytes and
 * contiguous (4 KiB for head_dim 128): the unit the decode kernel stages
 * into shared memory with one cp.async.bulk.
 *
 * Host swap slot layout (pinned), token-compact, exactly
 * n_tokens * kv_bytes_per_token bytes:
 *   slot[num_layers][2][num_kv_heads][n_tokens][head_dim]  bf16
 */
#ifndef ASTRAEA_B200_H
#define ASTRAEA_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define ASTRAEA_API __attribute__((visibility("default")))
#else
#define ASTRAEA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ASTRAEA_OK = 0,
  ASTRAEA_EINVAL = -1,      /* bad argument / shape */
  ASTRAEA_ENOBLOCKS = -2,   /* allocator cannot satisfy the request (nothing taken) */
  ASTRAEA_EDOUBLEFREE = -3, /* block returned twice or out of range */
  ASTRAEA_EUNSUPPORTED = -4 /* shape/dtype combination not compiled in */
};

ASTRAEA_API const char* astraea_status_string(int status);
ASTRAEA_API int astraea_abi_version(void);

typedef struct {
  int32_t num_layers;
  int32_t num_kv_heads;
  int32_t head_dim;      /* 64 or 128 */
  int32_t block_tokens;  /* 16 */
  int32_t num_blocks;
} astraea_kv_geometry;

/* Bytes of one pool block (all layers, K and V). */
ASTRAEA_API size_t astraea_kv_block_bytes(const astraea_kv_geometry* g);
/* Bytes per token of KV: the reference's MemoryModel.bytes_per_token
 * (kvcache.py:87-99) made concrete. */
ASTRAEA_API size_t astraea_kv_bytes_per_token(const astraea_kv_geometry* g);

/* ---- block allocator (host free list over [0, num_blocks)) --------------
 * Mirrors MemoryModel.allocate / release (kvcache.py:118-134) at block
 * granularity. LIFO reuse keeps recently freed (L2-warm) blocks hot. */
typedef struct astraea_block_allocator astraea_block_allocator;
ASTRAEA_API int astraea_alloc_create(int32_t num_blocks, astraea_block_allocator** out);
ASTRAEA_API int astraea_alloc_destroy(astraea_block_allocator* a);
/* Take n blocks into out_ids_host; ASTRAEA_ENOBLOCKS (and nothing taken) if short. */
ASTRAEA_API int astraea_alloc_take(astraea_block_allocator* a, int32_t n, int32_t* out_ids_host);
/* Return blocks; ASTRAEA_EDOUBLEFREE if any id is free already or out of range
 * (in which case nothing is returned). */
ASTRAEA_API int astraea_alloc_give(astraea_block_allocator* a, const int32_t* ids_host, int32_t n);
ASTRAEA_API int32_t astraea_alloc_free_count(const astraea_block_allocator* a);

/* ---- K1 / K2: KV swap ----------------------------------------------------------
 * Replace the swap delay kv_tokens / swap_bandwidth (kvcache.py:136-137)
 * scheduled at simulator.py:239-245 (out) and simulator.py:299-325 (in),
 * completed by KvCacheManager.complete_swap_out / complete_swap_in
 * (kvcache.py:230-258).
 * block_ids_host lists the request's blocks in context order; only the first
 * n_tokens tokens are moved (the last block's padding is not).
 * mode 0: SM gather/scatter kernel writing/reading the pinned slot through
 *         its mapped device address (zero-copy over the host link);
 * mode 1: copy engines, one strided 2-D DMA per block;
 * mode 2: staged -- the SM kernel gathers (scatters) the token-compact slot
 *         image in a stream-ordered device buffer (HBM to HBM, tens of us)
 *         and ONE contiguous copy-engine transfer crosses the host link, so
 *         the SMs are busy only briefly beside a running decode.
 * host slot must be pinned (cudaHostAlloc / cudaHostRegister). */
enum { ASTRAEA_SWAP_KERNEL = 0, ASTRAEA_SWAP_DMA = 1, ASTRAEA_SWAP_STAGED = 2 };
ASTRAEA_API int astraea_kv_swap_out(const astraea_kv_geometry* g, const void* pool_dev,
                        const int32_t* block_ids_host, int32_t n_blocks, int32_t n_tokens,
                        void* slot_host, int mode, void* stream);
ASTRAEA_API int astraea_kv_swap_in(const astraea_kv_geometry* g, void* pool_dev,
                       const int32_t* block_ids_host, int32_t n_blocks, int32_t n_tokens,
                       const void* slot_host, int mode, void* stream);
/* Device-to-device block copy (pool compaction / defragmentation). */
ASTRAEA_API int astraea_kv_copy_blocks(const astraea_kv_geometry* g, void* pool_dev,
                           const int32_t* src_ids_host, const int32_t* dst_ids_host,
                           int32_t n, void* stream);

/* ---- K3: block table build / compaction ------------------------------------------
 * Replaces the implicit per-request residency of kvcache.py:219-222,
 * 260-292 with the dense table the attention kernels read.
 * csr_ptr_dev[R+1], csr_ids_dev[...]: every request's block list.
 * rows_dev[B]: which CSR rows form the batch (retired members are simply
 * left out -> compaction). Writes table_dev[B][max_blocks] (pad -1) and
 * ctx_dev[B] = ctx_src_dev[rows[b]]. */
ASTRAEA_API int astraea_block_table_build(const int32_t* csr_ptr_dev, const int32_t* csr_ids_dev,
                              const int32_t* rows_dev, const int32_t* ctx_src_dev, int32_t B,
                              int32_t max_blocks, int32_t* table_dev, int32_t* ctx_dev,
                              void* stream);

/* ---- decode-loop driver (device side, CUDA-graph capturable) ----------------------------
 * Advances the batch by one decode step without host involvement, so the
 * whole step (advance + layers + sampling) is one replayable graph.
 * step = *step_dev (then *step_dev += 1). For row b with step < n_gen[b]:
 *   fed token  = step == 0 ? first_tok[b] : token of sampled_keys[b]
 *                (an ARGMAX-epilogue key; the kernel re-zeroes it for the next step)
 *   position   = base_pos[b] + step;  ctx[b] = position + 1
 *   slot       = table[b][position / block_tokens] * block_tokens + position % block_tokens
 *   hist[b * hist_stride + step] = fed token
 * and at step == n_gen[b]: hist[b * hist_stride + n_gen[b]] = that token (the
 * row's pending next token), so hist rows need n_gen[b] + 1 entries.
 * Rows with step >= n_gen[b] are retired: slot -1, ctx 0 (attention and
 * append skip them) -- the compaction the reference's parallel-max batch
 * implies when members finish at their own n_gen (simulator.py:96-98). */
ASTRAEA_API int astraea_decode_advance(int32_t* step_dev, int32_t B, const int32_t* n_gen_dev,
                           const int32_t* base_pos_dev, const int32_t* first_tok_dev,
                           unsigned long long* sampled_keys_dev, const int32_t* table_dev,
                           int32_t max_blocks, int32_t block_tokens, int32_t* tokens_dev,
                           int32_t* positions_dev, int32_t* slots_dev, int32_t* ctx_dev,
                           int32_t* hist_dev, int32_t hist_stride, void* stream);

/* ---- K5: RoPE + KV append ------------------------------------------------------------
 * Materialises state.kv_tokens = context_after(...) (simulator.py:367-369)
 * as real K/V rows. qkv_dev[T][(Hq + 2*Hkv) * D] is the fused projection
 * output; RoPE (theta, NeoX half-split) is applied to q (in place) and k;
 * k and v are written to pool slot slots_dev[t] = block * block_tokens + offset
 * (slot < 0: row skipped). positions_dev[T] are absolute token positions. */
ASTRAEA_API int astraea_rope_kv_append(const astraea_kv_geometry* g, void* pool_dev, int32_t layer,
                           void* qkv_dev, int32_t T, int32_t num_q_heads,
                           const int32_t* positions_dev, const int32_t* slots_dev,
                           float rope_theta, void* stream);

/* ---- K4: paged decode attention ------------------------------------------------------------
 * Replaces n_gen * seconds_per_token (simulator.py:337) -- one decode step
 * of the scheduler's mixed batch. q_dev: row b at q_dev + b*q_row_stride elements
 * holds [Hq][D] (so q can be read in place from the fused QKV rows);
 * table_dev[B][max_blocks];
 * ctx_dev[B] = tokens visible to the row (0 -> output zeros). out_dev[B][Hq][D].
 * workspace: astraea_decode_workspace_bytes(...) bytes, zero-filled once
 * before first use (it holds split arrival counters the kernel resets);
 * splits of long contexts are merged inside the same launch. */
ASTRAEA_API size_t astraea_decode_workspace_bytes(int32_t B, int32_t num_q_heads, int32_t head_dim,
                                      int32_t max_blocks);
ASTRAEA_API int astraea_paged_decode_attention(const astraea_kv_geometry* g, const void* pool_dev,
                                   int32_t layer, const void* q_dev, int32_t q_row_stride,
                                   int32_t B, int32_t num_q_heads, const int32_t* table_dev,
                                   int32_t max_blocks, const int32_t* ctx_dev, float scale,
                                   void* out_dev, void* workspace_dev, size_t workspace_bytes,
                                   void* stream);

/* ---- K7: paged prefill attention (causal, varlen) ---------------------------------------------
 * Replaces prefill_seconds(n_in + extra) (simulator.py:335-336): the
 * appended API result, or the whole context after a discard.
 * q_dev rows of [Hq][D] at stride q_row_stride (T = cu_q[S] rows); out_dev is
 * dense [T][Hq][D]; sequence s owns q rows [cu_q[s], cu_q[s+1])
 * whose absolute positions are ctx[s]-len_s .. ctx[s]-1 and attends causally
 * to its paged context table[s][*] of ctx[s] tokens. */
ASTRAEA_API int astraea_paged_prefill_attention(const astraea_kv_geometry* g, const void* pool_dev,
                                    int32_t layer, const void* q_dev, int32_t q_row_stride,
                                    const int32_t* cu_q_dev,
                                    int32_t S, int32_t max_q_len, int32_t num_q_heads,
                                    const int32_t* table_dev, int32_t max_blocks,
                                    const int32_t* ctx_dev, float scale, void* out_dev,
                                    void* stream);

/* ---- K6 / K9: dense projections on tcgen05 ------------------------------------------------------
 * C[M][N] = A[M][K] . W[N][K]^T (+ residual[M][N]), bf16 in, fp32 TMEM
 * accumulate, bf16 out. lda/ldw/ldc in elements. Prefill (M large) and decode
 * (M = batch) both run on tcgen05.mma; decode uses the swapped-operand form
 * (W rows on the MMA M axis) with deterministic split-K. workspace may be
 * NULL when astraea_gemm_workspace_bytes() returns 0; otherwise it must be
 * zero-filled once before first use (its arrival counters are reset by the
 * kernel itself) and not shared by concurrently running GEMMs. */
enum { ASTRAEA_EPI_NONE = 0, ASTRAEA_EPI_RESIDUAL = 1, ASTRAEA_EPI_SILU = 2, ASTRAEA_EPI_QKV_ROPE = 3,
       ASTRAEA_EPI_ARGMAX = 4 };
ASTRAEA_API size_t astraea_gemm_workspace_bytes(int32_t M, int32_t N, int32_t K);
ASTRAEA_API int astraea_gemm_bf16(const void* A_dev, int32_t lda, const void* W_dev, int32_t ldw,
                      void* C_dev, int32_t ldc, int32_t M, int32_t N, int32_t K,
                      const void* residual_dev, int32_t epilogue, void* workspace_dev,
                      size_t workspace_bytes, void* stream);

/* Fused epilogue programs of the Llama block (the small per-layer kernels
 * never run as separate launches on the decode path):
 *   NONE       C = acc
 *   RESIDUAL   C = acc + residual (may alias C); if ssq_out_dev != NULL also
 *              writes ssq_out[ceil(N/128)][M]: per-128-column sums of squares
 *              of the bf16 output -- the statistics of the next RMSNorm
 *   SILU       W rows interleaved [64 gate | 64 up] per 128 rows (N = 2F):
 *              C[M][F] = silu(gate) * up
 *   QKV_ROPE   N = (Hq + 2 Hkv) * head_dim: RoPE (theta, NeoX half split) on
 *              q and k at positions[t]; C[M][Hq*D] receives q; k and v rows
 *              are written to the pool at slots[t] (slot < 0: skipped)
 *   ARGMAX     greedy sampling fused into the lm_head: atomicMax of a packed
 *              (order-preserving value, ~column) key into argmax_keys[t]
 *              (zero before the launch; lowest index wins ties); C may be
 *              NULL, otherwise it also receives the bf16 logits
 * and for any program, input RMS scaling when ssq_in_dev != NULL:
 *   acc[t][:] *= rsqrt(sum_p ssq_in[p][t] / rms_dim + rms_eps)
 * (the norm weight is folded into W by the caller). */
typedef struct {
  int32_t kind;
  const void* residual_dev;
  float* ssq_out_dev;
  const float* ssq_in_dev;
  int32_t ssq_in_parts;
  int32_t rms_dim;
  float rms_eps;
  void* pool_dev;
  astraea_kv_geometry geo;
  int32_t layer;
  int32_t num_q_heads;
  const int32_t* positions_dev;
  const int32_t* slots_dev;
  float rope_theta;
  const float* rope_table_dev; /* optional [M][head_dim/2] (cos, sin) pairs from astraea_rope_table */
  unsigned long long* argmax_keys_dev; /* ARGMAX: [M] */
  int32_t argmax_col_offset;           /* ARGMAX: added to the column index in the key (vocab-sharded lm_head) */
} astraea_epilogue;
/* A chain of dependent decode GEMMs (M <= 64 tokens) in ONE persistent launch
 * (e.g. O-proj -> gate/up -> down -> next layer's QKV, or ... -> lm_head +
 * argmax). Phase p+1 may read phase p's output: its activation tiles wait on
 * a device-side phase barrier while its weight tiles already stream. At most
 * 4 phases. workspace: astraea_gemm_chain_workspace_bytes(), zero-filled
 * once before first use, not shared by concurrently running launches. */
typedef struct {
  const void* A;
  int32_t lda;
  const void* W;
  int32_t ldw;
  void* C;
  int32_t ldc;
  int32_t N;
  int32_t K;
  astraea_epilogue epi;
} astraea_gemm_phase;
ASTRAEA_API size_t astraea_gemm_chain_workspace_bytes(int32_t M, int32_t nphases,
                                          const astraea_gemm_phase* phases);
ASTRAEA_API int astraea_gemm_chain(int32_t M, int32_t nphases, const astraea_gemm_phase* phases,
                       void* workspace_dev, size_t workspace_bytes, void* stream);
/* A layer's decode attention followed by its chained GEMMs, in ONE launch:
 * the epilogue warps of every CTA run the paged decode attention of `attn`
 * (tensor cores, splits merged in CTA order) while the weight producer
 * already streams phase 0's weights; phase 0's A must be attn->out_dev
 * ([M][num_q_heads * head_dim]). Replaces the separate decode-attention
 * launch of K4 (simulator.py:337); same workspace as astraea_gemm_chain.
 * Supported: head_dim 128 with 4 q heads per kv head, head_dim 64 with 2 or 4. */
typedef struct {
  const void* pool_dev;
  astraea_kv_geometry geo;
  int32_t layer;
  int32_t num_q_heads;
  const void* q_dev;
  int32_t q_row_stride;
  const int32_t* table_dev;
  int32_t max_blocks;
  const int32_t* ctx_dev;
  float scale;
  void* out_dev;
} astraea_attn_phase;
/* attn[k] runs right before GEMM phase attn_before[k] (strictly increasing;
 * attn[k].out_dev must be that phase's A): nattn <= 2, nphases <= 8, so one
 * launch can carry two whole decoder layers. */
ASTRAEA_API int astraea_gemm_chain_attn(int32_t M, int32_t nattn, const astraea_attn_phase* attn,
                           const int32_t* attn_before, int32_t nphases, const astraea_gemm_phase* phases,
                           void* workspace_dev, size_t workspace_bytes, void* stream);
ASTRAEA_API int astraea_gemm_bf16_ex(const void* A_dev, int32_t lda, const void* W_dev, int32_t ldw,
                         void* C_dev, int32_t ldc, int32_t M, int32_t N, int32_t K,
                         const astraea_epilogue* epilogue, void* workspace_dev,
                         size_t workspace_bytes, void* stream);

/* ---- one decode step as one persistent kernel ------------------------------------------------
 * The whole decode step (every layer's QKV+RoPE+append, paged attention, O,
 * gate/up+SiLU, down, then lm_head+argmax) as ONE launch over a *program* of
 * phases, for M <= 64 rows. Phases are ordered; dependencies point backwards
 * and are tracked per chunk (128-feature GEMM tile, kv head) with epoch flags,
 * so phases overlap across SMs with no grid-wide barrier while the weight
 * stream never waits. Replaces the n_gen * seconds_per_token term of
 * Engine._actual_seconds (simulator.py:329-337) for the decode loop.
 *   GEMM phase: `gemm` as in astraea_gemm_chain (A rows = M);
 *     a_from   = phase producing A (-1: A is ready at launch)
 *     epi_from = phase whose output the epilogue reads (RMS statistics or the
 *                residual), -1: none / ready at launch
 *   ATTN phase: paged decode attention of `layer`; q rows at q_dev (row
 *     stride q_row_stride elements, [Hq][D]); out_dev dense [M][Hq*D];
 *     qkv_from = the QKV_ROPE GEMM phase that produced q and this step's K/V.
 * Program: astraea_step_program_bytes(n) bytes; build writes the phase
 * descriptors into program_host (any host memory, 128-byte aligned), the
 * caller copies them to a device buffer of the same size (stream-ordered,
 * e.g. from pinned memory) that astraea_step_launch reads. Workspace:
 * astraea_step_workspace_bytes(...) bytes of device memory, zero-filled once
 * before first use; programs built on one workspace may be launched one
 * after another on one stream, never concurrently. */
enum { ASTRAEA_PHASE_GEMM = 0, ASTRAEA_PHASE_ATTN = 1 };
typedef struct {
  int32_t kind;
  astraea_gemm_phase gemm;
  int32_t a_from;
  int32_t epi_from;
  const void* pool_dev;
  astraea_kv_geometry geo;
  int32_t layer;
  int32_t num_q_heads;
  const void* q_dev;
  int32_t q_row_stride;
  const int32_t* table_dev;
  int32_t max_blocks;
  const int32_t* ctx_dev;
  float scale;
  void* out_dev;
  int32_t qkv_from;
} astraea_step_phase;
ASTRAEA_API size_t astraea_step_program_bytes(int32_t nphases);
ASTRAEA_API size_t astraea_step_workspace_bytes(int32_t M, int32_t nphases, const astraea_step_phase* phases);
ASTRAEA_API int astraea_step_program_build(int32_t M, int32_t nphases, const astraea_step_phase* phases,
                               void* program_host, size_t program_bytes, void* workspace_dev,
                               size_t workspace_bytes);
/* l2_lookahead: weight tiles per CTA prefetched into L2 ahead of the smem ring (0: off). */
/* Diagnostics: when buf != NULL, following step launches write %globaltimer
 * stamps [grid][nphases][4] (+[grid] entry stamps) into buf; NULL disables. */
ASTRAEA_API int astraea_debug_step_trace(void* buf);
ASTRAEA_API int astraea_step_launch(int32_t M, int32_t nphases, const void* program_dev, void* workspace_dev,
                        int32_t l2_lookahead, void* stream);

/* Diagnostics: when buf != NULL, each following decode (stream-K / chain)
 * GEMM launch writes per-CTA %globaltimer stamps [grid][32] into the next of
 * `slots` slots of `slot_stride` u64 each: [0] entry, [1+p] activations of
 * phase p released, [5+p] epilogue of phase p done, [9] MMAs done, [10] exit.
 * Pass NULL to disable. */
ASTRAEA_API int astraea_debug_gemm_trace(void* buf, int32_t slots, int32_t slot_stride);

/* Diagnostics: when buf != NULL, each following tcgen05 prefill-attention
 * launch writes per-CTA %globaltimer stamps [grid][16] into buf (see
 * prefill_tc.cu); NULL disables. */
ASTRAEA_API int astraea_debug_prefill_trace(void* buf);

/* RoPE angle table for a batch: table[t][i] = (cos, sin)(positions[t] * theta^(-2i/D)),
 * i < D/2 -- computed once per forward and shared by every layer's QKV epilogue. */
ASTRAEA_API int astraea_rope_table(const int32_t* positions_dev, int32_t T, int32_t head_dim, float rope_theta,
                       float* table_dev, void* stream);

/* Per-row sums of squares in 128-column groups: ssq_out[ceil(dim/128)][rows]
 * (the layout the GEMM epilogues' ssq_in reads) -- the RMSNorm statistics of
 * a hidden state produced outside a fused epilogue (e.g. after a
 * tensor-parallel all-reduce). */
ASTRAEA_API int astraea_row_ssq(const void* x_dev, int32_t rows, int32_t dim, float* ssq_out_dev, void* stream);

/* ---- K8: small fused ops --------------------------------------------------------------------------- */
/* y = rmsnorm(x + r) * w ; if resid_out_dev != NULL it receives x + r. r may be NULL. */
ASTRAEA_API int astraea_rmsnorm(const void* x_dev, const void* r_dev, const void* w_dev, void* y_dev,
                    void* resid_out_dev, int32_t rows, int32_t dim, float eps, void* stream);
/* out[T][F] = silu(gu[T][0:F]) * gu[T][F:2F] */
ASTRAEA_API int astraea_silu_mul(const void* gu_dev, void* out_dev, int32_t T, int32_t F, void* stream);
/* out[T][dim] = table[ids[T]][dim]; if ssq_out_dev != NULL, ssq_out[t] = sum of
 * squares of the row (one-part RMS statistics for the first layer's norm). */
ASTRAEA_API int astraea_embedding(const int32_t* ids_dev, const void* table_dev, void* out_dev, int32_t T,
                      int32_t dim, float* ssq_out_dev, void* stream);
/* ids_out[r] = argmax_j logits[r][j] (lowest index on ties); logits bf16 [rows][vocab]. */
ASTRAEA_API int astraea_argmax(const void* logits_dev, int32_t rows, int32_t vocab, int32_t* ids_out_dev,
                   void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ASTRAEA_B200_H */
