// Paged attention over the block pool.
//
// K4 decode: the step the reference models as n_gen * seconds_per_token
//   (pkg/src/agentsched/simulator.py:329-337) over the scheduler's mixed
//   batch (execute_batch parallel-max, simulator.py:96-98).
//   One CTA per (row, kv head, context split). K/V pages of the kv head
//   (block_tokens x head_dim bf16, contiguous in the pool) are staged into a
//   shared-memory ring with cp.async.bulk + mbarrier (TMA bulk engine); the
//   GQA group's q heads share every staged page. Scores are reduced with
//   warp shuffles, softmax is online in the exp2 domain, and context splits
//   are merged (log-sum-exp, split order) by the last split CTA to finish.
//
// K7 prefill: the recompute-on-resume prefill (simulator.py:335-336),
//   flash-attention style on mma.sync m16n8k16 tensor-core tiles: one CTA
//   per (64 query rows, q head, sequence), K/V tiles gathered from pool
//   pages with cp.async into XOR-swizzled shared memory, causal mask on
//   absolute positions.
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "attn_mma.cuh"

using namespace astraea;

namespace astraea {
// K7 on tcgen05 (prefill_tc.cu)
int prefill_tc_launch(const astraea_kv_geometry* g, const void* pool, int32_t layer, const void* q, int32_t q_stride,
                      const int32_t* cu_q, int32_t S, int32_t max_q_len, int32_t Hq, const int32_t* table,
                      int32_t max_blocks, const int32_t* ctx, float scale, void* out, cudaStream_t st);
}

namespace {

constexpr int kBT = 16;         // tokens per block
constexpr int kMaxSplits = 64;  // context splits per (row, kv head)
constexpr int kMaxBlocksPerSplit = 512;
constexpr float kLog2e = 1.4426950408889634f;

struct DecodeParams {
  const bf16* pool;
  const bf16* q;
  const int32_t* table;
  const int32_t* ctx;
  bf16* out;
  long long q_stride;
  float* ws_o;     // [B][Hq][splits][D]
  float* ws_lse;   // [B][Hq][splits]
  int* counters;   // [B][Hkv] split arrival counters (zero between launches)
  long long block_el;  // elements per pool block
  int layer, Hkv, Hq, max_blocks, blocks_per_split, splits;
  float scale_log2;
  int block_rows;  // TMA path: rows of one pool block in the [blocks x L x 2 x Hkv x 16][D] view
};

// Warp-per-tile decode attention. Each of the 4 warps owns a private 2-deep
// ring of (K, V) page stages and processes tiles j = warp, warp + 4, ... of
// the CTA's block range independently: scores with lanes split over
// (token, head group), softmax with 16-lane shuffles, PV with lanes split
// over head_dim. No block-wide barrier inside the tile loop; the 4 warp
// states are merged once at the end.
template <int D, int G>
__global__ void __launch_bounds__(128) decode_kernel(const __grid_constant__ DecodeParams p) {
  constexpr int PAGE = kBT * D;             // elements per page
  constexpr int CPR = D / 8;                // 16-byte chunks per row
  constexpr int WST = 2;                    // stages per warp
  constexpr int HPL = G >= 2 ? G / 2 : 1;   // heads per lane in the score phase
  constexpr int DPL = D / 32;               // dims per lane in the PV phase

  extern __shared__ __align__(128) uint8_t dsm[];
  bf16 (*ks)[PAGE] = reinterpret_cast<bf16 (*)[PAGE]>(dsm);                       // [4*WST][PAGE]
  bf16 (*vs)[PAGE] = reinterpret_cast<bf16 (*)[PAGE]>(dsm + 4 * WST * PAGE * 2);  // [4*WST][PAGE]
  float (*acc_w)[G][D] = reinterpret_cast<float (*)[G][D]>(dsm);                  // aliases ks after the loop
  __shared__ __align__(16) float qs[G][D];
  __shared__ __align__(8) uint64_t bar[4 * WST];
  __shared__ float m_w[4][G], l_w[4][G];

  const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  pdl_wait();
  pdl_launch();
  const int ctx = p.ctx[b];
  const int nblk = (ctx + kBT - 1) / kBT;
  const int b0 = split * p.blocks_per_split;
  const int b1 = min(nblk, b0 + p.blocks_per_split);
  const int ntile = max(0, b1 - b0);

  // Block ids of this split (one per lane, loaded in parallel with q), so the
  // first TMA issue does not wait on a dependent table load.
  __shared__ int blk_ids[kMaxBlocksPerSplit];
  const int32_t* trow = p.table + (long long)b * p.max_blocks;
  for (int i = tid; i < ntile; i += 128) blk_ids[i] = trow[b0 + i];
  for (int i = tid; i < G * D / 8; i += 128) {
    const int g = i / (D / 8), c = i % (D / 8);
    float f[8];
    unpack8(*reinterpret_cast<const uint4*>(p.q + (long long)b * p.q_stride + (h * G + g) * D + c * 8), f);
#pragma unroll
    for (int k = 0; k < 8; ++k) qs[g][c * 8 + k] = f[k] * p.scale_log2;
  }
  if (tid < 4 * WST) mbar_init(&bar[tid], 1);
  fence_barrier_init();
  __syncthreads();

  const long long head_off = ((long long)p.layer * 2 * p.Hkv + h) * PAGE;
  const long long v_off = (long long)p.Hkv * PAGE;
  // tiles of this warp: j = warp + 4 k, k = 0, 1, ...
  const int my_tiles = ntile > warp ? (ntile - warp + 3) / 4 : 0;
  auto issue = [&](int k) {
    const int st = warp * WST + (k % WST);
    const long long base = (long long)blk_ids[warp + 4 * k] * p.block_el + head_off;
    mbar_arrive_expect_tx(&bar[st], 2 * PAGE * 2);
    bulk_g2s(ks[st], p.pool + base, PAGE * 2, &bar[st]);
    bulk_g2s(vs[st], p.pool + base + v_off, PAGE * 2, &bar[st]);
  };
  if (lane == 0)
    for (int k = 0; k < min(my_tiles, WST); ++k) issue(k);

  const int t = lane & 15;          // score phase: token of this lane
  const int hg = lane >> 4;         // head group (HPL heads)
  float m[G], l[G], acc[G][DPL];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int i = 0; i < DPL; ++i) acc[g][i] = 0.f;
  }

  for (int k = 0; k < my_tiles; ++k) {
    const int j = warp + 4 * k;
    const int st = warp * WST + (k % WST);
    const int valid = min(kBT, ctx - (b0 + j) * kBT);
    mbar_wait(&bar[st], (k / WST) & 1);
    // ---- scores (log2 domain, q pre-scaled): lane -> token t, heads hg*HPL ..
    float s[HPL];
#pragma unroll
    for (int e = 0; e < HPL; ++e) s[e] = 0.f;
    const bf16* krow = &ks[st][t * D];
#pragma unroll 4
    for (int c = 0; c < CPR; ++c) {
      const int cc = (c + t) & (CPR - 1);   // rotate to spread smem banks across tokens
      float kf[8];
      unpack8(*reinterpret_cast<const uint4*>(krow + cc * 8), kf);
#pragma unroll
      for (int e = 0; e < HPL; ++e) {
        const int g = hg * HPL + e;
        if (g < G) {
          const float4 q0 = *reinterpret_cast<const float4*>(&qs[g][cc * 8]);
          const float4 q1 = *reinterpret_cast<const float4*>(&qs[g][cc * 8 + 4]);
          s[e] += q0.x * kf[0] + q0.y * kf[1] + q0.z * kf[2] + q0.w * kf[3] + q1.x * kf[4] + q1.y * kf[5] +
                  q1.z * kf[6] + q1.w * kf[7];
        }
      }
    }
    // ---- online softmax per head over the 16 tokens of this tile. Lane
    // half hg owns heads hg*HPL + e; m/l of all heads are replicated in
    // every lane (register arrays, compile-time indexed only).
    float pr[HPL], mnew[HPL], lnew[HPL], alpha[HPL];
#pragma unroll
    for (int e = 0; e < HPL; ++e) {
      const int g = hg * HPL + e;
      float mold = -INFINITY, lold = 0.f;
#pragma unroll
      for (int gg = 0; gg < G; ++gg)
        if (gg == g) {
          mold = m[gg];
          lold = l[gg];
        }
      const float sv = (t < valid && g < G) ? s[e] : -INFINITY;
      float mx = sv;
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mnew[e] = fmaxf(mold, mx);
      alpha[e] = mnew[e] == -INFINITY ? 1.f : exp2f(mold - mnew[e]);
      pr[e] = sv == -INFINITY ? 0.f : exp2f(sv - mnew[e]);
      float sum = pr[e];
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      lnew[e] = lold * alpha[e] + sum;
    }
    // broadcast per-head (m, alpha, l) to all lanes: head g lives in half g / HPL
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int src = (g / HPL) * 16;
      const int e = g % HPL;
      m[g] = __shfl_sync(0xffffffffu, mnew[e], src);
      l[g] = __shfl_sync(0xffffffffu, lnew[e], src);
      const float al = __shfl_sync(0xffffffffu, alpha[e], src);
#pragma unroll
      for (int i = 0; i < DPL; ++i) acc[g][i] *= al;
    }
    // ---- PV: lane -> dims lane*DPL .. ; p[g][tok] from the score lanes
    const bf16* vbase = &vs[st][lane * DPL];
#pragma unroll 4
    for (int tok = 0; tok < kBT; ++tok) {
      if (tok >= valid) break;
      float vf[DPL];
      if constexpr (DPL == 4) {
        const uint2 u = *reinterpret_cast<const uint2*>(vbase + tok * D);
        const float2 a0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
        const float2 a1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
        vf[0] = a0.x; vf[1] = a0.y; vf[2] = a1.x; vf[3] = a1.y;
      } else {
        const float2 a0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vbase + tok * D));
        vf[0] = a0.x; vf[1] = a0.y;
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float pg = __shfl_sync(0xffffffffu, pr[g % HPL], (g / HPL) * 16 + tok);
#pragma unroll
        for (int i = 0; i < DPL; ++i) acc[g][i] += pg * vf[i];
      }
    }
    __syncwarp();
    if (lane == 0 && k + WST < my_tiles) issue(k + WST);
  }
  // ---- merge the 4 warps (acc_w aliases the stage ring: wait for every warp)
  __syncthreads();
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if (lane == 0) {
      m_w[warp][g] = m[g];
      l_w[warp][g] = l[g];
    }
#pragma unroll
    for (int i = 0; i < DPL; ++i) acc_w[warp][g][lane * DPL + i] = acc[g][i];
  }
  __syncthreads();
  constexpr int TPH = 128 / G;              // threads per head in the output phase
  constexpr int DPT = D / TPH;
  const int pg = tid / TPH, pd = (tid % TPH) * DPT;
  float mt = -INFINITY;
#pragma unroll
  for (int w = 0; w < 4; ++w) mt = fmaxf(mt, m_w[w][pg]);
  float lsum = 0.f, o[DPT];
#pragma unroll
  for (int i = 0; i < DPT; ++i) o[i] = 0.f;
  if (mt != -INFINITY) {
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float sc = m_w[w][pg] == -INFINITY ? 0.f : exp2f(m_w[w][pg] - mt);
      lsum += l_w[w][pg] * sc;
#pragma unroll
      for (int i = 0; i < DPT; ++i) o[i] += acc_w[w][pg][pd + i] * sc;
    }
  }
  const int hq = h * G + pg;
  const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
  if (p.splits == 1) {
    bf16* dst = p.out + ((long long)b * p.Hq + hq) * D + pd;
#pragma unroll
    for (int i = 0; i < DPT; ++i) dst[i] = f2bf(o[i] * inv);
  } else {
    // Split-K over the context: store this split's normalised partial and
    // log-sum-exp; the last split CTA of (row, kv head) to arrive merges all
    // splits in split order (deterministic) and writes the G output heads.
    __shared__ int s_last;
    const long long row = ((long long)b * p.Hq + hq) * p.splits + split;
    float* dst = p.ws_o + row * D + pd;
#pragma unroll
    for (int i = 0; i < DPT; ++i) __stcg(dst + i, o[i] * inv);
    if ((tid % TPH) == 0) __stcg(p.ws_lse + row, lsum > 0.f ? mt + log2f(lsum) : -INFINITY);
    __threadfence();
    __syncthreads();
    int* ctr = p.counters + (long long)b * p.Hkv + h;
    if (tid == 0) s_last = atomicAdd(ctr, 1) == p.splits - 1;
    __syncthreads();
    if (s_last) {
      __threadfence();
      // merge: per q head, log-sum-exp weights of all splits (split order)
      __shared__ float wsh[G][kMaxSplits];
      __shared__ float den_sh[G];
      const long long bh0 = (long long)b * p.Hq + h * G;
      for (int i = tid; i < G * p.splits; i += 128) {
        const int g = i / p.splits, sp = i % p.splits;
        wsh[g][sp] = __ldcg(p.ws_lse + (bh0 + g) * p.splits + sp);
      }
      __syncthreads();
      if (tid < G) {
        float mx = -INFINITY;
        for (int sp = 0; sp < p.splits; ++sp) mx = fmaxf(mx, wsh[tid][sp]);
        float den = 0.f;
        for (int sp = 0; sp < p.splits; ++sp) {
          const float w = (mx == -INFINITY || wsh[tid][sp] == -INFINITY) ? 0.f : exp2f(wsh[tid][sp] - mx);
          wsh[tid][sp] = w;
          den += w;
        }
        den_sh[tid] = den;
      }
      __syncthreads();
      const long long row0 = ((long long)b * p.Hq + hq) * p.splits;
      float num[DPT];
#pragma unroll
      for (int i = 0; i < DPT; ++i) num[i] = 0.f;
      int sp = 0;
      for (; sp + 4 <= p.splits; sp += 4) {
        float o[4][DPT];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int i = 0; i < DPT; ++i) o[k][i] = __ldcg(p.ws_o + (row0 + sp + k) * D + pd + i);
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int i = 0; i < DPT; ++i) num[i] += wsh[pg][sp + k] * o[k][i];
      }
      for (; sp < p.splits; ++sp)
#pragma unroll
        for (int i = 0; i < DPT; ++i) num[i] += wsh[pg][sp] * __ldcg(p.ws_o + (row0 + sp) * D + pd + i);
      const float den = den_sh[pg];
      bf16* out = p.out + ((long long)b * p.Hq + hq) * D + pd;
#pragma unroll
      for (int i = 0; i < DPT; ++i) out[i] = f2bf(den > 0.f ? num[i] / den : 0.f);
      if (tid == 0) *ctr = 0;
    }
  }
}

// Tensor-core decode attention: one CTA per (context split, kv head, row),
// four warps taking every fourth page of the split (attn_mma.cuh: mma.sync
// scores and PV with the G q heads as the M rows), merged in shared memory;
// splits are merged (log-sum-exp, split order) by the last split CTA. Only
// ~17 KB of shared memory, so the next layer's GEMM CTAs (PDL) are resident
// beside it and stream their first weight tiles during the attention.
template <int D, int G>
constexpr int decode_mma_warp_bytes() {   // a V page, or the warp's merged state ([G] m, [G] l, [G][D] o)
  return kBT * D * 2 > (2 * G + G * D) * 4 ? kBT * D * 2 : (2 * G + G * D) * 4;
}

// Shared tail of the tensor-core decode kernels: merge the 4 warps' states
// (warp order) through shared memory (each warp's region of wreg bf16
// elements is free once its page loop is done), then either write the
// output (one split) or the split partial, the last split CTA merging all
// splits in split order.
template <int D, int G>
__device__ __forceinline__ void decode_merge_tail(const DecodeParams& p, bf16* vs_all, int wreg,
                                                  const astraea::attn::AttnAcc<D>& st, int b, int h,
                                                  int split, int tid, int warp, int lane) {
  constexpr int EPT = (G * D + 127) / 128;
  const int r8 = lane >> 2, quad = lane & 3;
  bf16* vs = vs_all + warp * wreg;
  float* wst = reinterpret_cast<float*>(vs);   // [G] m, [G] l, [G][D] o (the warp's V page is free now)
  __syncwarp();
  if (r8 < G) {
#pragma unroll
    for (int n = 0; n < D / 8; ++n)
      *reinterpret_cast<float2*>(wst + 2 * G + r8 * D + 8 * n + 2 * quad) = make_float2(st.o[n][0], st.o[n][1]);
    if (quad == 0) {
      wst[r8] = st.m;
      wst[G + r8] = st.l;
    }
  }
  __syncthreads();
  float Mv[EPT], Lv[EPT], Ov[EPT];
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    const int idx = tid * EPT + e, g = idx / D, dd = idx % D;
    Mv[e] = -INFINITY;
    Lv[e] = 0.f;
    Ov[e] = 0.f;
    if (idx < G * D) {
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const float* ws = reinterpret_cast<const float*>(vs_all + w * wreg);
        const float mk = ws[g], mn = fmaxf(Mv[e], mk);
        const float a0 = mn == -INFINITY ? 0.f : exp2f(Mv[e] - mn), a1 = mn == -INFINITY ? 0.f : exp2f(mk - mn);
        Lv[e] = Lv[e] * a0 + ws[G + g] * a1;
        Ov[e] = Ov[e] * a0 + ws[2 * G + g * D + dd] * a1;
        Mv[e] = mn;
      }
    }
  }
  if (p.splits == 1) {
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const int idx = tid * EPT + e, g = idx / D, dd = idx % D;
      if (idx < G * D) p.out[((long long)b * p.Hq + h * G + g) * D + dd] = f2bf(Lv[e] > 0.f ? Ov[e] / Lv[e] : 0.f);
    }
    return;
  }
  // split partial: normalised o and log-sum-exp per q head
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    const int idx = tid * EPT + e, g = idx / D, dd = idx % D;
    if (idx < G * D) {
      const long long row = ((long long)b * p.Hq + h * G + g) * p.splits + split;
      __stcg(p.ws_o + row * D + dd, Lv[e] > 0.f ? Ov[e] / Lv[e] : 0.f);
      if (dd == 0) __stcg(p.ws_lse + row, Lv[e] > 0.f ? Mv[e] + log2f(Lv[e]) : -INFINITY);
    }
  }
  __threadfence();
  __syncthreads();
  __shared__ int s_last;
  int* ctr = p.counters + (long long)b * p.Hkv + h;
  if (tid == 0) s_last = atomicAdd(ctr, 1) == p.splits - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  __shared__ float wsh[G][kMaxSplits];
  __shared__ float den_sh[G];
  const long long bh0 = (long long)b * p.Hq + h * G;
  for (int i = tid; i < G * p.splits; i += 128) {
    const int g = i / p.splits, sp = i % p.splits;
    wsh[g][sp] = __ldcg(p.ws_lse + (bh0 + g) * p.splits + sp);
  }
  __syncthreads();
  if (tid < G) {
    float mx = -INFINITY;
    for (int sp = 0; sp < p.splits; ++sp) mx = fmaxf(mx, wsh[tid][sp]);
    float den = 0.f;
    for (int sp = 0; sp < p.splits; ++sp) {
      const float w = (mx == -INFINITY || wsh[tid][sp] == -INFINITY) ? 0.f : exp2f(wsh[tid][sp] - mx);
      wsh[tid][sp] = w;
      den += w;
    }
    den_sh[tid] = den;
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    const int idx = tid * EPT + e, g = idx / D, dd = idx % D;
    if (idx >= G * D) continue;
    const long long row0 = (bh0 + g) * p.splits;
    float num = 0.f;
    int sp = 0;
    for (; sp + 4 <= p.splits; sp += 4) {
      float o4[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) o4[k] = __ldcg(p.ws_o + (row0 + sp + k) * D + dd);
#pragma unroll
      for (int k = 0; k < 4; ++k) num += wsh[g][sp + k] * o4[k];
    }
    for (; sp < p.splits; ++sp) num += wsh[g][sp] * __ldcg(p.ws_o + (row0 + sp) * D + dd);
    const float den = den_sh[g];
    p.out[(bh0 + g) * D + dd] = f2bf(den > 0.f ? num / den : 0.f);
  }
  if (tid == 0) *ctr = 0;
}

template <int D, int G>
__global__ void __launch_bounds__(128) decode_mma_kernel(const __grid_constant__ DecodeParams p) {
  using namespace astraea::attn;
  constexpr int WREG = decode_mma_warp_bytes<D, G>() / 2;   // per-warp region (bf16 elements)
  extern __shared__ __align__(128) uint8_t dsm[];
  bf16* vs_all = reinterpret_cast<bf16*>(dsm);   // [4][WREG]: V page, then the warp's state
  const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  pdl_wait();
  pdl_launch();
  const int ctx = p.ctx[b];
  const int nblk = (ctx + kBT - 1) / kBT;
  const int b0 = split * p.blocks_per_split;
  const int b1 = min(nblk, b0 + p.blocks_per_split);
  const int r8 = lane >> 2, quad = lane & 3;
  uint32_t qa[D / 8];
  attn_load_q<D>(p.q + (long long)b * p.q_stride + (long long)(h * G + r8) * D, r8 < G, quad, qa);
  const PageSrc src = page_src<D>(p.pool, p.block_el, p.layer, p.Hkv, h, p.table + (long long)b * p.max_blocks,
                                  p.scale_log2);
  bf16* vs = vs_all + warp * WREG;
  AttnAcc<D> st;
  attn_pages<D>(src, b0 + warp, b1, 4, ctx, qa, vs, st, lane);
  decode_merge_tail<D, G>(p, vs_all, WREG, st, b, h, split, tid, warp, lane);
}

// ---------------------------------------------------------------------------
// K4 for the larger batches: the same tensor-core page math, but every warp
// keeps S pages in flight. K and V pages arrive by TMA (a 2-D tensor map over
// the pool viewed as [pages x 16 rows][D], 128-byte swizzle, one box of 16
// rows x 64 columns per half page) into a per-warp ring of S stages with one
// mbarrier each; the warp computes page k while pages k+1..k+S-1 are in
// flight, and lane 0 refills the stage as soon as the warp has read it. The
// swizzle keeps the ldmatrix reads of K (scores) and V (transposed, PV)
// conflict-free. With S = 3 and 96 KB per CTA, two CTAs per SM keep up to
// 24 pages (192 KB) per SM in flight -- what HBM latency x per-SM bandwidth
// asks for -- where the one-page-per-warp walk keeps ~32 KB.
// ---------------------------------------------------------------------------
template <int D, int G, int S>
__global__ void __launch_bounds__(128) decode_tma_kernel(const __grid_constant__ CUtensorMap pool_map,
                                                         const __grid_constant__ DecodeParams p) {
  using namespace astraea::attn;
  constexpr int PB = tma_page_bytes<D>();
  extern __shared__ __align__(1024) uint8_t dsm_raw[];
  uint8_t* dsm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar[4 * S];
  const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (lane < S) mbar_init(&bar[warp * S + lane], 1);
  fence_barrier_init();
  __syncwarp();
  if (tid == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&pool_map) : "memory");
  pdl_wait();
  pdl_launch();
  const int ctx = p.ctx[b];
  const int nblk = (ctx + kBT - 1) / kBT;
  const int b0 = split * p.blocks_per_split;
  const int b1 = min(nblk, b0 + p.blocks_per_split);
  const int r8 = lane >> 2, quad = lane & 3;
  uint32_t qs[D / 16][2];
  attn_load_q_std<D>(p.q + (long long)b * p.q_stride + (long long)(h * G + r8) * D, r8 < G, quad, qs);
  TmaPages T;
  T.map = &pool_map;
  T.block_rows = p.block_rows;
  T.k_row0 = (p.layer * 2 * p.Hkv + h) * kBT;
  T.v_row0 = T.k_row0 + p.Hkv * kBT;
  AttnAcc<D> st;
  uint32_t cnt = 0;
  attn_pages_tma<D, S>(T, p.table + (long long)b * p.max_blocks, b0 + warp, b1, 4, ctx, p.scale_log2, qs,
                       dsm + (size_t)warp * S * PB, &bar[warp * S], cnt, st, lane);
  // the merge reuses each warp's ring (all of its pages have landed and been read)
  decode_merge_tail<D, G>(p, reinterpret_cast<bf16*>(dsm), S * PB / 2, st, b, h, split, tid, warp, lane);
}

// ---------------------------------------------------------------------------
// K7 prefill (mma.sync m16n8k16, bf16 in, fp32 accumulate)
// ---------------------------------------------------------------------------
constexpr int kQT = 64;  // q rows per CTA (4 warps x 16)
constexpr int kKT = 64;  // kv tokens per tile (4 blocks)

struct PrefillParams {
  const bf16* pool;
  const bf16* q;
  const int32_t* cu_q;
  const int32_t* table;
  const int32_t* ctx;
  bf16* out;
  long long q_stride;
  long long block_el;
  int layer, Hkv, Hq, max_blocks;
  float scale_log2;
};

// Swizzled offset (elements) of 16-byte chunk c in row r of a [rows][D] tile.
template <int D>
__device__ __forceinline__ int swz(int r, int c) {
  return r * D + ((c ^ (r & 7)) << 3);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

__device__ __forceinline__ void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(smem_u32(p)));
}
__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int D>
__global__ void __launch_bounds__(128) prefill_kernel(const __grid_constant__ PrefillParams p) {
  constexpr int CPR = D / 8;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  bf16* qs = reinterpret_cast<bf16*>(smem_raw);          // [64][D]
  bf16* ks = qs + kQT * D;                                // [2][64][D]
  bf16* vs = ks + 2 * kKT * D;                            // [2][64][D]

  const int s = blockIdx.z, hq = blockIdx.y, qt = blockIdx.x;
  pdl_wait();
  pdl_launch();
  const int q_begin = p.cu_q[s], len = p.cu_q[s + 1] - q_begin;
  if (qt * kQT >= len) return;
  const int ctx = p.ctx[s];
  const int pos0 = ctx - len;  // absolute position of q row 0
  const int G = p.Hq / p.Hkv;
  const int h = hq / G;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int row0 = qt * kQT;
  const int rows = min(kQT, len - row0);

  // Q tile -> smem (swizzled)
  for (int i = tid; i < kQT * CPR; i += 128) {
    const int r = i / CPR, c = i % CPR;
    const bool ok = r < rows;
    const bf16* src = p.q + (long long)(q_begin + row0 + (ok ? r : 0)) * p.q_stride + hq * D + c * 8;
    cp_async16(qs + swz<D>(r, c), src, ok);
  }
  const int32_t* trow = p.table + (long long)s * p.max_blocks;
  const long long head_off = ((long long)p.layer * 2 * p.Hkv + h) * kBT * D;
  const long long v_off = (long long)p.Hkv * kBT * D;
  const int last_pos = pos0 + row0 + rows - 1;
  const int ntiles = last_pos / kKT + 1;
  auto load_kv = [&](int t, int buf) {
    for (int i = tid; i < kKT * CPR; i += 128) {
      const int r = i / CPR, c = i % CPR;
      const int tok = t * kKT + r;
      const bool ok = tok < ctx;
      const long long base =
          (long long)trow[ok ? tok / kBT : 0] * p.block_el + head_off + (tok % kBT) * D + c * 8;
      cp_async16(ks + buf * kKT * D + swz<D>(r, c), p.pool + (ok ? base : 0), ok);
      cp_async16(vs + buf * kKT * D + swz<D>(r, c), p.pool + (ok ? base + v_off : 0), ok);
    }
  };
  load_kv(0, 0);
  cp_async_commit();

  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  uint32_t qf[D / 16][4];
  const int g = lane >> 2, t4 = lane & 3;
  const int my_pos[2] = {pos0 + row0 + warp * 16 + g, pos0 + row0 + warp * 16 + g + 8};

  for (int t = 0; t < ntiles; ++t) {
    if (t + 1 < ntiles) load_kv(t + 1, (t + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (t == 0) {
      // Q fragments (A operand): rows warp*16 + (lane%16), chunk kk*2 + lane/16
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const int r = warp * 16 + (lane & 15);
        const int c = kk * 2 + (lane >> 4);
        ldsm_x4(qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], qs + swz<D>(r, c));
      }
    }
    const bf16* kb = ks + (t & 1) * kKT * D;
    const bf16* vb = vs + (t & 1) * kKT * D;
    // S = Q K^T : 16 x 64 per warp -> 8 n-tiles of 8 tokens
    float sfr[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) sfr[n][0] = sfr[n][1] = sfr[n][2] = sfr[n][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
      for (int n2 = 0; n2 < 4; ++n2) {
        // two n-tiles (16 tokens) x k16: matrices (tok 0-7,k0-7)(tok 0-7,k8-15)(tok 8-15,k0-7)(tok 8-15,k8-15)
        const int r = n2 * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int c = kk * 2 + ((lane >> 3) & 1);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(b0, b1, b2, b3, kb + swz<D>(r, c));
        mma16816(sfr[2 * n2], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b0, b1);
        mma16816(sfr[2 * n2 + 1], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b2, b3);
      }
    }
    // mask + online softmax (rows g and g+8 of this warp's 16)
    float mt[2] = {mrow[0], mrow[1]};
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int tok = t * kKT + n * 8 + t4 * 2 + (e & 1);
        const int ri = e >> 1;
        float v = sfr[n][e] * p.scale_log2;
        if (tok > my_pos[ri] || tok >= ctx) v = -INFINITY;
        sfr[n][e] = v;
        mt[ri] = fmaxf(mt[ri], v);
      }
    }
#pragma unroll
    for (int ri = 0; ri < 2; ++ri) {
      mt[ri] = fmaxf(mt[ri], __shfl_xor_sync(0xffffffffu, mt[ri], 1));
      mt[ri] = fmaxf(mt[ri], __shfl_xor_sync(0xffffffffu, mt[ri], 2));
    }
    float alpha[2], rs[2] = {0.f, 0.f};
#pragma unroll
    for (int ri = 0; ri < 2; ++ri) alpha[ri] = mt[ri] == -INFINITY ? 1.f : exp2f(mrow[ri] - mt[ri]);
    uint32_t pf[4][4];  // P as A fragments: 4 k16 steps over 64 tokens
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      float pv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int ri = e >> 1;
        pv[e] = mt[ri] == -INFINITY ? 0.f : exp2f(sfr[n][e] - mt[ri]);
        rs[ri] += pv[e];
      }
      // n-tile n covers tokens n*8..n*8+7 = k-step n/2, half n&1
      pf[n >> 1][(n & 1) * 2 + 0] = pack_bf16(pv[0], pv[1]);
      pf[n >> 1][(n & 1) * 2 + 1] = pack_bf16(pv[2], pv[3]);
    }
#pragma unroll
    for (int ri = 0; ri < 2; ++ri) {
      rs[ri] += __shfl_xor_sync(0xffffffffu, rs[ri], 1);
      rs[ri] += __shfl_xor_sync(0xffffffffu, rs[ri], 2);
      lrow[ri] = lrow[ri] * alpha[ri] + rs[ri];
      mrow[ri] = mt[ri];
    }
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      o[i][0] *= alpha[0]; o[i][1] *= alpha[0];
      o[i][2] *= alpha[1]; o[i][3] *= alpha[1];
    }
    // O += P V : A = P (16 x 64 tokens), B = V (64 tokens x D) via ldmatrix.trans
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      // A fragment order: a0 (rows g, k 0-7) a1 (rows g+8, k 0-7) a2 (rows g, k 8-15) a3 (rows g+8, k 8-15)
      const uint32_t a0 = pf[kk][0], a1 = pf[kk][1], a2 = pf[kk][2], a3 = pf[kk][3];
#pragma unroll
      for (int dn = 0; dn < D / 16; ++dn) {
        // matrices: (tok 0-7, d 0-7)(tok 8-15, d 0-7)(tok 0-7, d 8-15)(tok 8-15, d 8-15)
        const int r = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
        const int c = dn * 2 + (lane >> 4);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(b0, b1, b2, b3, vb + swz<D>(r, c));
        mma16816(o[2 * dn], a0, a1, a2, a3, b0, b1);
        mma16816(o[2 * dn + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    __syncthreads();
  }
  // write O / l
#pragma unroll
  for (int ri = 0; ri < 2; ++ri) {
    const int r = warp * 16 + g + ri * 8;
    if (r >= rows) continue;
    const float inv = lrow[ri] > 0.f ? 1.f / lrow[ri] : 0.f;
    bf16* dst = p.out + ((long long)(q_begin + row0 + r) * p.Hq + hq) * D;
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      *reinterpret_cast<__nv_bfloat162*>(dst + n * 8 + t4 * 2) =
          __floats2bfloat162_rn(o[n][ri * 2] * inv, o[n][ri * 2 + 1] * inv);
    }
  }
}

int decode_splits(int B, int Hkv, int max_blocks, int* bps, int min_blocks = 0) {
  // Enough CTAs to cover the SMs, but at least kMinBlocks blocks (8 KiB of
  // K+V per head per block) per CTA so per-CTA fixed costs stay small.
  static const int kEnvMin = [] {
    const char* e = getenv("ASTRAEA_DECODE_MIN_BLOCKS");
    return e ? std::max(1, atoi(e)) : 8;
  }();
  const int kMinBlocks = min_blocks > 0 ? min_blocks : kEnvMin;
  const int target = 2 * num_sms();
  const int base = B * Hkv;
  int want = (target + base - 1) / base;
  want = max(1, min(want, (max_blocks + kMinBlocks - 1) / kMinBlocks));
  int per = (max_blocks + want - 1) / want;
  int splits = (max_blocks + per - 1) / per;
  if (splits > kMaxSplits) {
    per = (max_blocks + kMaxSplits - 1) / kMaxSplits;
    splits = (max_blocks + per - 1) / per;
  }
  if (per > kMaxBlocksPerSplit) return -1;   // > 64 x 512 x 16 tokens: not supported
  *bps = per;
  return splits;
}

}  // namespace

// Decode workspace: [counters: 4096 ints][partials o: B*Hq*splits*D][lse: B*Hq*splits].
constexpr size_t kDecCounterBytes = 4096 * sizeof(int);

extern "C" size_t astraea_decode_workspace_bytes(int32_t B, int32_t Hq, int32_t D, int32_t max_blocks) {
  // Upper bound over any B / Hkv (see decode_splits).
  const size_t splits = (size_t)std::min(max_blocks, kMaxSplits);
  return kDecCounterBytes + (size_t)B * Hq * splits * (D + 1) * sizeof(float);
}

extern "C" int astraea_paged_decode_attention(const astraea_kv_geometry* g, const void* pool,
                                              int32_t layer, const void* q, int32_t q_stride,
                                              int32_t B, int32_t Hq,
                                              const int32_t* table, int32_t max_blocks,
                                              const int32_t* ctx, float scale, void* out, void* ws,
                                              size_t ws_bytes, void* stream) {
  if (!g || B < 0 || max_blocks <= 0 || layer < 0 || layer >= g->num_layers || g->block_tokens != kBT)
    return ASTRAEA_EINVAL;
  if (B == 0) return ASTRAEA_OK;
  const int Hkv = g->num_kv_heads, D = g->head_dim;
  if (Hq % Hkv || q_stride < Hq * D) return ASTRAEA_EINVAL;
  const int G = Hq / Hkv;
  DecodeParams p;
  p.pool = (const bf16*)pool;
  p.q = (const bf16*)q;
  p.q_stride = q_stride;
  p.table = table;
  p.ctx = ctx;
  p.out = (bf16*)out;
  p.block_el = (long long)astraea_kv_block_bytes(g) / 2;
  p.layer = layer;
  p.Hkv = Hkv;
  p.Hq = Hq;
  p.max_blocks = max_blocks;
  p.scale_log2 = scale * kLog2e;
  int bps = 0;
  p.splits = decode_splits(B, Hkv, max_blocks, &bps);
  if (p.splits < 0) return ASTRAEA_EUNSUPPORTED;
  p.blocks_per_split = bps;
  const size_t need = kDecCounterBytes + (size_t)B * Hq * p.splits * (D + 1) * sizeof(float);
  if (p.splits > 1 && (!ws || ws_bytes < need || (size_t)B * Hkv * sizeof(int) > kDecCounterBytes))
    return ASTRAEA_EINVAL;
  p.counters = (int*)ws;
  p.ws_o = (float*)((char*)ws + kDecCounterBytes);
  p.ws_lse = p.ws_o + (size_t)B * Hq * p.splits * D;
  dim3 grid(p.splits, Hkv, B);
  cudaStream_t st = (cudaStream_t)stream;
#define LAUNCH_DEC(DD, GG)                                                                         \
  do {                                                                                               \
    constexpr size_t smem = std::max<size_t>(2 * 8 * kBT * DD * 2, 4 * GG * DD * 4);                \
    static bool attr = false;                                                                        \
    if (!attr) {                                                                                     \
      ASTRAEA_TRY(cudaFuncSetAttribute(decode_kernel<DD, GG>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                       (int)smem));                                                  \
      attr = true;                                                                                   \
    }                                                                                                \
    ASTRAEA_TRY(launch_k(decode_kernel<DD, GG>, grid, dim3(128), smem, st, p));                     \
  } while (0)
#define LAUNCH_MMA(DD, GG)                                                                         \
  do {                                                                                               \
    constexpr size_t smem = 4 * decode_mma_warp_bytes<DD, GG>();                                   \
    ASTRAEA_TRY(launch_k(decode_mma_kernel<DD, GG>, grid, dim3(128), smem, st, p));                 \
  } while (0)
#define LAUNCH_TMA(DD, GG)                                                                         \
  do {                                                                                               \
    constexpr int S = 3;                                                                             \
    constexpr size_t smem = 1024 + (size_t)4 * S * astraea::attn::tma_page_bytes<DD>();             \
    static bool attr = false;                                                                        \
    if (!attr) {                                                                                     \
      ASTRAEA_TRY(cudaFuncSetAttribute(decode_tma_kernel<DD, GG, S>,                                 \
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));     \
      attr = true;                                                                                   \
    }                                                                                                \
    ASTRAEA_TRY(launch_k(decode_tma_kernel<DD, GG, S>, grid, dim3(128), smem, st, map, p));         \
  } while (0)
  static const char mode = [] {
    const char* e = getenv("ASTRAEA_DECODE_ATTN");
    return e ? e[0] : 't';   // 't' TMA-staged (default), 'm' one page per warp, 's' CUDA cores
  }();
  const bool use_mma = mode != 's';
  if (mode == 't' && D * 2 <= 256 && (D == 128 || D == 64)) {
    // TMA-staged kernel: its own split (each warp >= S pages: 12 blocks per split)
    int bps2 = 0;
    const int sp2 = decode_splits(B, Hkv, max_blocks, &bps2, 12);
    const bool ok_g = (D == 128 && (G == 4 || G == 8)) || (D == 64 && (G == 2 || G == 4));
    if (sp2 > 0 && ok_g) {
      const size_t need2 = kDecCounterBytes + (size_t)B * Hq * sp2 * (D + 1) * sizeof(float);
      if (sp2 > 1 && (!ws || ws_bytes < need2)) return ASTRAEA_EINVAL;
      p.splits = sp2;
      p.blocks_per_split = bps2;
      p.ws_lse = p.ws_o + (size_t)B * Hq * p.splits * D;
      p.block_rows = g->num_layers * 2 * Hkv * kBT;
      CUtensorMap map;
      int rc = astraea::tc::make_map(&map, pool, (long long)g->num_blocks * p.block_rows, D, D, kBT);
      if (rc) return rc;
      dim3 grid2(p.splits, Hkv, B);
      grid = grid2;
      if (D == 128 && G == 4) LAUNCH_TMA(128, 4);
      else if (D == 128 && G == 8) LAUNCH_TMA(128, 8);
      else if (D == 64 && G == 4) LAUNCH_TMA(64, 4);
      else LAUNCH_TMA(64, 2);
      ASTRAEA_CHECK_LAUNCH();
      return ASTRAEA_OK;
    }
  }
  if (use_mma && D == 128 && G == 4) LAUNCH_MMA(128, 4);
  else if (use_mma && D == 128 && G == 8) LAUNCH_MMA(128, 8);
  else if (use_mma && D == 64 && G == 4) LAUNCH_MMA(64, 4);
  else if (use_mma && D == 64 && G == 2) LAUNCH_MMA(64, 2);
  else if (D == 128 && G == 4) LAUNCH_DEC(128, 4);
  else if (D == 128 && G == 8) LAUNCH_DEC(128, 8);
  else if (D == 64 && G == 4) LAUNCH_DEC(64, 4);
  else if (D == 64 && G == 8) LAUNCH_DEC(64, 8);
  else if (D == 128 && G == 2) LAUNCH_DEC(128, 2);
  else if (D == 64 && G == 2) LAUNCH_DEC(64, 2);
  else if (D == 128 && G == 1) LAUNCH_DEC(128, 1);
  else return ASTRAEA_EUNSUPPORTED;
#undef LAUNCH_DEC
#undef LAUNCH_MMA
#undef LAUNCH_TMA
  ASTRAEA_CHECK_LAUNCH();
  return ASTRAEA_OK;
}

extern "C" int astraea_paged_prefill_attention(const astraea_kv_geometry* g, const void* pool,
                                               int32_t layer, const void* q, int32_t q_stride,
                                               const int32_t* cu_q,
                                               int32_t S, int32_t max_q_len, int32_t Hq,
                                               const int32_t* table, int32_t max_blocks,
                                               const int32_t* ctx, float scale, void* out,
                                               void* stream) {
  if (!g || S < 0 || max_q_len < 0 || layer < 0 || layer >= g->num_layers || g->block_tokens != kBT)
    return ASTRAEA_EINVAL;
  if (S == 0 || max_q_len == 0) return ASTRAEA_OK;
  if (Hq % g->num_kv_heads || q_stride < Hq * g->head_dim) return ASTRAEA_EINVAL;
  static const bool use_tc = [] {
    const char* e = getenv("ASTRAEA_PREFILL_ATTN");
    return !(e && e[0] == 'm');   // "m": the mma.sync kernel below
  }();
  if (use_tc) {
    const int rc = astraea::prefill_tc_launch(g, pool, layer, q, q_stride, cu_q, S, max_q_len, Hq, table, max_blocks,
                                              ctx, scale, out, (cudaStream_t)stream);
    if (rc != ASTRAEA_EUNSUPPORTED) return rc;
  }
  PrefillParams p;
  p.pool = (const bf16*)pool;
  p.q = (const bf16*)q;
  p.q_stride = q_stride;
  p.cu_q = cu_q;
  p.table = table;
  p.ctx = ctx;
  p.out = (bf16*)out;
  p.block_el = (long long)astraea_kv_block_bytes(g) / 2;
  p.layer = layer;
  p.Hkv = g->num_kv_heads;
  p.Hq = Hq;
  p.max_blocks = max_blocks;
  p.scale_log2 = scale * kLog2e;
  dim3 grid((max_q_len + kQT - 1) / kQT, Hq, S);
  cudaStream_t st = (cudaStream_t)stream;
  const int D = g->head_dim;
  const size_t smem = (size_t)(kQT + 4 * kKT) * D * 2;
  if (D == 128) {
    static bool attr = false;
    if (!attr) {
      ASTRAEA_TRY(cudaFuncSetAttribute(prefill_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr = true;
    }
    ASTRAEA_TRY(launch_k(prefill_kernel<128>, grid, dim3(128), smem, st, p));
  } else if (D == 64) {
    ASTRAEA_TRY(launch_k(prefill_kernel<64>, grid, dim3(128), smem, st, p));
  } else {
    return ASTRAEA_EUNSUPPORTED;
  }
  ASTRAEA_CHECK_LAUNCH();
  return ASTRAEA_OK;
}
