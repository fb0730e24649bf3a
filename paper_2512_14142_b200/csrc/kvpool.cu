// Paged KV pool: block allocator, swap gather/scatter (K1/K2), block table
// build (K3), RoPE + KV append (K5), device block copy.
//
// Reference seams (pkg/src/agentsched): the swap delay kv_tokens/bandwidth
// (kvcache.py:136-137; simulator.py:239-245, 299-325), complete_swap_out /
// try_begin_swap_in / complete_swap_in (kvcache.py:230-258), release and
// discard (kvcache.py:219-222, 260-292) and admission's
// kv_tokens = context_after(...) (simulator.py:365-369).
#include <algorithm>
#include <new>
#include <vector>

#include "common.cuh"

using namespace astraea;

extern "C" const char* astraea_status_string(int status) {
  switch (status) {
    case ASTRAEA_OK: return "ok";
    case ASTRAEA_EINVAL: return "invalid argument";
    case ASTRAEA_ENOBLOCKS: return "not enough free KV blocks";
    case ASTRAEA_EDOUBLEFREE: return "block freed twice or out of range";
    case ASTRAEA_EUNSUPPORTED: return "unsupported shape";
    default: return status > 0 ? cudaGetErrorString((cudaError_t)status) : "unknown error";
  }
}

extern "C" int astraea_abi_version(void) { return 1; }

static bool geometry_ok(const astraea_kv_geometry* g) {
  return g && g->num_layers > 0 && g->num_kv_heads > 0 &&
         (g->head_dim == 64 || g->head_dim == 128) && g->block_tokens == 16 &&
         g->num_blocks > 0;
}

extern "C" size_t astraea_kv_block_bytes(const astraea_kv_geometry* g) {
  return (size_t)g->num_layers * 2 * g->num_kv_heads * g->block_tokens * g->head_dim * 2;
}

extern "C" size_t astraea_kv_bytes_per_token(const astraea_kv_geometry* g) {
  return (size_t)g->num_layers * 2 * g->num_kv_heads * g->head_dim * 2;
}

// ---------------------------------------------------------------------------
// Block allocator: LIFO free stack + an in-use bitmap for double-free checks.
// ---------------------------------------------------------------------------
struct astraea_block_allocator {
  std::vector<int32_t> stack;
  std::vector<uint8_t> used;
};

extern "C" int astraea_alloc_create(int32_t num_blocks, astraea_block_allocator** out) {
  if (num_blocks <= 0 || !out) return ASTRAEA_EINVAL;
  auto* a = new (std::nothrow) astraea_block_allocator();
  if (!a) return ASTRAEA_EINVAL;
  a->stack.resize(num_blocks);
  a->used.assign(num_blocks, 0);
  // Pop order 0,1,2,...: push in reverse.
  for (int32_t i = 0; i < num_blocks; ++i) a->stack[i] = num_blocks - 1 - i;
  *out = a;
  return ASTRAEA_OK;
}

extern "C" int astraea_alloc_destroy(astraea_block_allocator* a) {
  delete a;
  return ASTRAEA_OK;
}

extern "C" int astraea_alloc_take(astraea_block_allocator* a, int32_t n, int32_t* out) {
  if (!a || n < 0 || (n > 0 && !out)) return ASTRAEA_EINVAL;
  if ((size_t)n > a->stack.size()) return ASTRAEA_ENOBLOCKS;
  for (int32_t i = 0; i < n; ++i) {
    int32_t id = a->stack.back();
    a->stack.pop_back();
    a->used[id] = 1;
    out[i] = id;
  }
  return ASTRAEA_OK;
}

extern "C" int astraea_alloc_give(astraea_block_allocator* a, const int32_t* ids, int32_t n) {
  if (!a || n < 0 || (n > 0 && !ids)) return ASTRAEA_EINVAL;
  const int32_t nb = (int32_t)a->used.size();
  for (int32_t i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= nb || !a->used[ids[i]]) return ASTRAEA_EDOUBLEFREE;
    for (int32_t j = 0; j < i; ++j)
      if (ids[j] == ids[i]) return ASTRAEA_EDOUBLEFREE;
  }
  // Push in reverse so that the first id of the list is reused first.
  for (int32_t i = n - 1; i >= 0; --i) {
    a->used[ids[i]] = 0;
    a->stack.push_back(ids[i]);
  }
  return ASTRAEA_OK;
}

extern "C" int32_t astraea_alloc_free_count(const astraea_block_allocator* a) {
  return a ? (int32_t)a->stack.size() : 0;
}

// ---------------------------------------------------------------------------
// K1/K2 swap. A "chunk" is one (block, layer, K|V, head) page: up to
// block_tokens * head_dim bf16, contiguous on both sides. One warp moves one
// chunk per iteration with 16-byte vectors; all loads of a chunk are issued
// before its stores so each warp keeps a whole page in flight over the link.
// Block ids travel in the kernel parameter block (no H2D copy per swap).
// ---------------------------------------------------------------------------
constexpr int kSwapMaxIds = 900;

struct SwapArgs {
  const char* src;
  char* dst;
  long long block_bytes;   // pool block stride
  int lanes;               // num_layers * 2 * num_kv_heads
  int page_bytes;          // block_tokens * head_dim * 2
  int row_bytes;           // head_dim * 2
  int n_tokens;            // tokens of the whole slot (lane stride in the slot)
  int token_base;          // first token covered by this launch
  int n_blocks;            // blocks in this launch
  int last_tokens;         // valid tokens in the final block of this launch
  int ids[kSwapMaxIds];
};

constexpr int kSwapCtas = 32;   // default grid of the SM swap path (tools/swap_load.py sweep)

constexpr int kSwapThreads = 128;

template <bool kOut>
__global__ void __launch_bounds__(kSwapThreads) swap_kernel(const __grid_constant__ SwapArgs a) {
  const int lane_id = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const long long total = (long long)a.lanes * a.n_blocks;
  const long long slot_lane_bytes = (long long)a.n_tokens * a.row_bytes;
  for (long long c = warp; c < total; c += nwarps) {
    const int blk = (int)(c % a.n_blocks);  // block fastest: consecutive warps, consecutive slot bytes
    const int lane = (int)(c / a.n_blocks);
    const int tokens = (blk == a.n_blocks - 1) ? a.last_tokens : (a.page_bytes / a.row_bytes);
    const int bytes = tokens * a.row_bytes;
    const long long pool_off = (long long)a.ids[blk] * a.block_bytes + (long long)lane * a.page_bytes;
    const long long slot_off = (long long)lane * slot_lane_bytes +
                               ((long long)a.token_base + (long long)blk * (a.page_bytes / a.row_bytes)) * a.row_bytes;
    const char* s = a.src + (kOut ? pool_off : slot_off);
    char* d = a.dst + (kOut ? slot_off : pool_off);
    const int nvec = bytes >> 4;
    // page_bytes <= 4096 -> at most 8 vectors per lane.
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      int idx = lane_id + 32 * k;
      if (idx < nvec) v[k] = ld_stream(s + 16 * idx);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      int idx = lane_id + 32 * k;
      if (idx < nvec) st_stream(d + 16 * idx, v[k]);
    }
  }
}

static void* mapped(const void* host) {
  void* dev = nullptr;
  if (cudaHostGetDevicePointer(&dev, const_cast<void*>(host), 0) != cudaSuccess) {
    cudaGetLastError();
    return const_cast<void*>(host);  // UVA: pinned host pointers are device-addressable
  }
  return dev;
}

static int swap_impl(bool out, const astraea_kv_geometry* g, const void* pool, void* pool_mut,
                     const int32_t* ids, int32_t n_blocks, int32_t n_tokens, const void* slot,
                     void* slot_mut, int mode, void* stream) {
  if (!geometry_ok(g) || !ids || n_blocks <= 0 || n_tokens <= 0) return ASTRAEA_EINVAL;
  const int bt = g->block_tokens;
  if ((n_tokens + bt - 1) / bt != n_blocks) return ASTRAEA_EINVAL;
  for (int32_t i = 0; i < n_blocks; ++i)
    if (ids[i] < 0 || ids[i] >= g->num_blocks) return ASTRAEA_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const long long block_bytes = (long long)astraea_kv_block_bytes(g);
  const int row_bytes = g->head_dim * 2;
  const int page_bytes = bt * row_bytes;
  const int lanes = g->num_layers * 2 * g->num_kv_heads;
  if (mode == ASTRAEA_SWAP_DMA) {
    const size_t slot_pitch = (size_t)n_tokens * row_bytes;
    for (int32_t i = 0; i < n_blocks; ++i) {
      const int tokens = std::min(bt, n_tokens - i * bt);
      char* pool_page = (char*)(out ? pool : pool_mut) + (long long)ids[i] * block_bytes;
      char* slot_col = (char*)(out ? slot_mut : slot) + (size_t)i * page_bytes;
      cudaError_t e;
      if (out)
        e = cudaMemcpy2DAsync(slot_col, slot_pitch, pool_page, page_bytes, (size_t)tokens * row_bytes,
                              lanes, cudaMemcpyDeviceToHost, st);
      else
        e = cudaMemcpy2DAsync(pool_page, page_bytes, slot_col, slot_pitch, (size_t)tokens * row_bytes,
                              lanes, cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) return (int)e;
    }
    return ASTRAEA_OK;
  }
  if (mode != ASTRAEA_SWAP_KERNEL && mode != ASTRAEA_SWAP_STAGED) return ASTRAEA_EINVAL;
  {
    // The SM path dereferences the slot over the host link: it must be pinned.
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, out ? slot_mut : slot) != cudaSuccess ||
        (attr.type != cudaMemoryTypeHost && attr.type != cudaMemoryTypeManaged)) {
      cudaGetLastError();
      return ASTRAEA_EINVAL;
    }
  }
  // Co-residence with the persistent decode kernel (1 CTA/SM, ~200 KB of
  // shared memory): a swap CTA must not pin its SM to a small-shared-memory
  // carveout (the decode CTA could then not start there until the swap CTA
  // exits), and its registers must fit beside the decode CTA's.
  static const bool carveout = [] {
    cudaFuncSetAttribute(swap_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(swap_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    cudaGetLastError();
    return true;
  }();
  (void)carveout;
  const size_t slot_bytes = (size_t)n_tokens * row_bytes * lanes;
  char* slot_dev = nullptr;
  if (mode == ASTRAEA_SWAP_STAGED) {
    // stream-ordered staging image of the slot; the device pool keeps freed
    // memory cached (no release threshold), so steady-state swaps allocate nothing
    static const bool pool_cfg = [] {
      int dev = 0;
      cudaMemPool_t mp;
      if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&mp, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      cudaGetLastError();
      return true;
    }();
    (void)pool_cfg;
    ASTRAEA_TRY(cudaMallocAsync((void**)&slot_dev, slot_bytes, st));
    if (!out) ASTRAEA_TRY(cudaMemcpyAsync(slot_dev, slot, slot_bytes, cudaMemcpyHostToDevice, st));
  } else {
    slot_dev = (char*)mapped(out ? slot_mut : slot);
  }
  // A few CTAs keep the host link full (a warp moves up to 4 KiB per
  // round trip); more only steal issue slots and memory-pipe share from the
  // persistent decode kernel running beside the swap. ASTRAEA_SWAP_CTAS
  // overrides (read per call, for the load sweeps).
  const char* env = getenv("ASTRAEA_SWAP_CTAS");
  const int grid = mode == ASTRAEA_SWAP_STAGED ? 2 * num_sms()   // HBM to HBM: a short full-width burst
                                               : std::max(1, std::min(env ? atoi(env) : kSwapCtas, 4 * num_sms()));
  for (int32_t first = 0; first < n_blocks; first += kSwapMaxIds) {
    SwapArgs a;
    const int nb = std::min<int32_t>(kSwapMaxIds, n_blocks - first);
    a.block_bytes = block_bytes;
    a.lanes = lanes;
    a.page_bytes = page_bytes;
    a.row_bytes = row_bytes;
    a.n_tokens = n_tokens;
    a.token_base = first * bt;
    a.n_blocks = nb;
    a.last_tokens = std::min(bt, n_tokens - (first + nb - 1) * bt);
    for (int i = 0; i < nb; ++i) a.ids[i] = ids[first + i];
    if (out) {
      a.src = (const char*)pool;
      a.dst = slot_dev;
      swap_kernel<true><<<grid, kSwapThreads, 0, st>>>(a);
    } else {
      a.src = slot_dev;
      a.dst = (char*)pool_mut;
      swap_kernel<false><<<grid, kSwapThreads, 0, st>>>(a);
    }
    ASTRAEA_CHECK_LAUNCH();
  }
  if (mode == ASTRAEA_SWAP_STAGED) {
    if (out) ASTRAEA_TRY(cudaMemcpyAsync(slot_mut, slot_dev, slot_bytes, cudaMemcpyDeviceToHost, st));
    ASTRAEA_TRY(cudaFreeAsync(slot_dev, st));
  }
  return ASTRAEA_OK;
}

extern "C" int astraea_kv_swap_out(const astraea_kv_geometry* g, const void* pool,
                                   const int32_t* ids, int32_t n_blocks, int32_t n_tokens,
                                   void* slot, int mode, void* stream) {
  return swap_impl(true, g, pool, nullptr, ids, n_blocks, n_tokens, nullptr, slot, mode, stream);
}

extern "C" int astraea_kv_swap_in(const astraea_kv_geometry* g, void* pool, const int32_t* ids,
                                  int32_t n_blocks, int32_t n_tokens, const void* slot, int mode,
                                  void* stream) {
  return swap_impl(false, g, nullptr, pool, ids, n_blocks, n_tokens, slot, nullptr, mode, stream);
}

extern "C" int astraea_kv_copy_blocks(const astraea_kv_geometry* g, void* pool,
                                      const int32_t* src_ids, const int32_t* dst_ids, int32_t n,
                                      void* stream) {
  if (!geometry_ok(g) || n < 0 || (n > 0 && (!src_ids || !dst_ids))) return ASTRAEA_EINVAL;
  const size_t bb = astraea_kv_block_bytes(g);
  for (int32_t i = 0; i < n; ++i) {
    if (src_ids[i] < 0 || src_ids[i] >= g->num_blocks || dst_ids[i] < 0 ||
        dst_ids[i] >= g->num_blocks)
      return ASTRAEA_EINVAL;
    ASTRAEA_TRY(cudaMemcpyAsync((char*)pool + dst_ids[i] * bb, (char*)pool + src_ids[i] * bb, bb,
                                cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  }
  return ASTRAEA_OK;
}

// ---------------------------------------------------------------------------
// K3: dense block table for the active rows of a batch.
// ---------------------------------------------------------------------------
__global__ void table_build_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ ids,
                                   const int32_t* __restrict__ rows, const int32_t* __restrict__ ctx_src,
                                   int32_t max_blocks, int32_t* __restrict__ table,
                                   int32_t* __restrict__ ctx) {
  const int b = blockIdx.x;
  pdl_wait();
  pdl_launch();
  const int r = rows[b];
  const int begin = ptr[r];
  const int n = ptr[r + 1] - begin;
  for (int j = threadIdx.x; j < max_blocks; j += blockDim.x)
    table[(long long)b * max_blocks + j] = j < n ? ids[begin + j] : -1;
  if (threadIdx.x == 0) ctx[b] = ctx_src[r];
}

extern "C" int astraea_block_table_build(const int32_t* ptr, const int32_t* ids, const int32_t* rows,
                                         const int32_t* ctx_src, int32_t B, int32_t max_blocks,
                                         int32_t* table, int32_t* ctx, void* stream) {
  if (B < 0 || max_blocks <= 0) return ASTRAEA_EINVAL;
  if (B == 0) return ASTRAEA_OK;
  ASTRAEA_TRY(launch_k(table_build_kernel, dim3(B), dim3(128), 0, (cudaStream_t)stream, ptr, ids, rows, ctx_src, max_blocks, table, ctx));
  ASTRAEA_CHECK_LAUNCH();
  return ASTRAEA_OK;
}

// ---------------------------------------------------------------------------
// K5: RoPE (NeoX half split, as in Llama) on q and k, then write k, v rows
// into their pool slots. One CTA per token.
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256) rope_append_kernel(
    bf16* __restrict__ qkv, int Hq, int Hkv, const int32_t* __restrict__ positions,
    const int32_t* __restrict__ slots, bf16* __restrict__ pool, long long block_bytes_el,
    int layer, int bt, float theta) {
  const int t = blockIdx.x;
  pdl_wait();
  pdl_launch();
  const int H = Hq + 2 * Hkv;
  bf16* row = qkv + (long long)t * H * D;
  const float pos = (float)positions[t];
  const int slot = slots[t];
  constexpr int half = D / 2;
  bf16* kdst = nullptr;
  bf16* vdst = nullptr;
  if (slot >= 0) {
    const int blk = slot / bt, off = slot % bt;
    bf16* base = pool + (long long)blk * block_bytes_el + (long long)layer * 2 * Hkv * bt * D;
    kdst = base + (long long)off * D;                 // + head * bt * D
    vdst = base + (long long)Hkv * bt * D + (long long)off * D;
  }
  // Rotations: (Hq + Hkv) heads x half pairs.
  for (int w = threadIdx.x; w < (Hq + Hkv) * half; w += blockDim.x) {
    const int h = w / half, i = w % half;
    const float inv_freq = 1.0f / powf(theta, (float)(2 * i) / (float)D);  // as torch's fp32 RoPE
    float sn, cs;
    sincosf(pos * inv_freq, &sn, &cs);
    bf16* hp = row + h * D;
    const float x0 = bf2f(hp[i]), x1 = bf2f(hp[i + half]);
    const bf16 y0 = f2bf(x0 * cs - x1 * sn);
    const bf16 y1 = f2bf(x1 * cs + x0 * sn);
    if (h < Hq) {
      hp[i] = y0;
      hp[i + half] = y1;
    } else if (kdst) {
      bf16* kd = kdst + (long long)(h - Hq) * bt * D;
      kd[i] = y0;
      kd[i + half] = y1;
    }
  }
  if (vdst) {
    const bf16* vsrc = row + (Hq + Hkv) * D;
    for (int w = threadIdx.x; w < Hkv * D / 8; w += blockDim.x) {
      const int h = w / (D / 8), c = w % (D / 8);
      *reinterpret_cast<uint4*>(vdst + (long long)h * bt * D + c * 8) =
          *reinterpret_cast<const uint4*>(vsrc + h * D + c * 8);
    }
  }
}

extern "C" int astraea_rope_kv_append(const astraea_kv_geometry* g, void* pool, int32_t layer,
                                      void* qkv, int32_t T, int32_t Hq, const int32_t* positions,
                                      const int32_t* slots, float theta, void* stream) {
  if (!geometry_ok(g) || layer < 0 || layer >= g->num_layers || T < 0 || Hq <= 0 ||
      Hq % g->num_kv_heads)
    return ASTRAEA_EINVAL;
  if (T == 0) return ASTRAEA_OK;
  const long long bbe = (long long)astraea_kv_block_bytes(g) / 2;
  cudaStream_t st = (cudaStream_t)stream;
  if (g->head_dim == 128)
    ASTRAEA_TRY(launch_k(rope_append_kernel<128>, dim3(T), dim3(256), 0, st, (bf16*)qkv, (int)Hq, (int)g->num_kv_heads,
                         positions, slots, (bf16*)pool, bbe, (int)layer, (int)g->block_tokens, theta));
  else
    ASTRAEA_TRY(launch_k(rope_append_kernel<64>, dim3(T), dim3(256), 0, st, (bf16*)qkv, (int)Hq, (int)g->num_kv_heads,
                         positions, slots, (bf16*)pool, bbe, (int)layer, (int)g->block_tokens, theta));
  ASTRAEA_CHECK_LAUNCH();
  return ASTRAEA_OK;
}

// ---------------------------------------------------------------------------
// Decode-loop driver: one CTA advances every row of the batch by one step.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int key_token(unsigned long long k) {
  return (int)(0xFFFFFFFFu - (uint32_t)(k & 0xFFFFFFFFull));
}

__global__ void decode_advance_kernel(int32_t* __restrict__ step_ctr, int B, const int32_t* __restrict__ n_gen,
                                      const int32_t* __restrict__ base_pos, const int32_t* __restrict__ first_tok,
                                      unsigned long long* __restrict__ keys, const int32_t* __restrict__ table,
                                      int max_blocks, int bt, int32_t* __restrict__ tokens,
                                      int32_t* __restrict__ positions, int32_t* __restrict__ slots,
                                      int32_t* __restrict__ ctx, int32_t* __restrict__ hist, int hist_stride) {
  pdl_wait();
  pdl_launch();
  const int step = *step_ctr;
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const int sampled = step == 0 ? 0 : key_token(keys[b]);
    keys[b] = 0ull;  // ready for this step's lm_head argmax
    if (step < n_gen[b]) {
      const int tok = step == 0 ? first_tok[b] : sampled;
      const int pos = base_pos[b] + step;
      tokens[b] = tok;
      positions[b] = pos;
      ctx[b] = pos + 1;
      slots[b] = table[(long long)b * max_blocks + pos / bt] * bt + pos % bt;
      if (hist) hist[(long long)b * hist_stride + step] = tok;
    } else {
      // first step after retirement: record the token sampled by the row's
      // last step (the request's pending next token)
      if (hist && step == n_gen[b]) hist[(long long)b * hist_stride + step] = sampled;
      tokens[b] = 0;
      positions[b] = 0;
      ctx[b] = 0;
      slots[b] = -1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *step_ctr = step + 1;
}

extern "C" int astraea_decode_advance(int32_t* step, int32_t B, const int32_t* n_gen, const int32_t* base_pos,
                                      const int32_t* first_tok, unsigned long long* sampled, const int32_t* table,
                                      int32_t max_blocks, int32_t bt, int32_t* tokens, int32_t* positions,
                                      int32_t* slots, int32_t* ctx, int32_t* hist, int32_t hist_stride,
                                      void* stream) {
  if (!step || B <= 0 || B > 1024 || max_blocks <= 0 || bt <= 0) return ASTRAEA_EINVAL;
  ASTRAEA_TRY(launch_k(decode_advance_kernel, dim3(1), dim3(256), 0, (cudaStream_t)stream, step, (int)B, n_gen,
                       base_pos, first_tok, sampled, table, (int)max_blocks, (int)bt, tokens, positions, slots, ctx,
                       hist, (int)hist_stride));
  ASTRAEA_CHECK_LAUNCH();
  return ASTRAEA_OK;
}
