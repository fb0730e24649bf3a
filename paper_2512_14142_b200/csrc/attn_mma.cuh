// Tensor-core paged decode attention of one warp over a (row, kv head)'s
// pages: shared by the per-layer decode kernel (attention.cu) and the
// decode-step kernel's attention phase (decode_step.cu).
#pragma once

#include "common.cuh"
#include "tc.cuh"

namespace astraea {
namespace attn {

using tc::atom_add_acq_rel;
using tc::epi_bar;

constexpr int kAttnBT = 16;   // tokens per block (page)

__device__ __forceinline__ uint4 ldcg16(const void* p) { return __ldcg(reinterpret_cast<const uint4*>(p)); }
__device__ __forceinline__ unsigned long long gtimer_() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------------------
// Paged decode attention of one (row, kv head) page range, by one warp, one
// page (16 tokens) per iteration, on tensor cores (mma.sync m16n8k16, bf16 in,
// fp32 accumulate), the GQA group's G <= 8 q heads as the M rows:
//   S[g][tok] = Q[g] . K[tok]     two n8 tiles x D/16 k-steps. The head dims
//              are contracted in a permuted order (thread q of a quad owns the
//              contiguous dims [q*D/4, (q+1)*D/4)), applied to Q and K alike,
//              so a thread's K fragment is four 16-byte loads of one K row;
//   softmax    online, exp2 domain, row reductions inside the quad;
//   O[g][d]  += P[g][tok] . V[tok][d]  the S accumulator layout is reused as
//              the A operand (FA2 register reuse); V goes through a swizzled
//              shared-memory page (cp.async, zero-filled past the context)
//              and ldmatrix.trans.
// Thread t holds head row g = t/4 and output dims {8n + 2(t%4), +1}.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mma_16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                          uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4_trans(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int D>
struct AttnAcc {
  float m, l;            // running max (log2 domain) and sum of row g = lane / 4
  float o[D / 8][4];     // O fragments (c2, c3: padding rows, stay 0)
};

// Q fragments of row g (zeros for g >= G): the thread's D/4 dims as bf16 pairs.
template <int D>
__device__ __forceinline__ void attn_load_q(const bf16* q_row, bool ok, int quad, uint32_t* qa) {
  const uint4* src = reinterpret_cast<const uint4*>(q_row + quad * (D / 4));
#pragma unroll
  for (int i = 0; i < D / 32; ++i) {
    const uint4 v = ok ? __ldcg(src + i) : make_uint4(0u, 0u, 0u, 0u);
    qa[4 * i] = v.x;
    qa[4 * i + 1] = v.y;
    qa[4 * i + 2] = v.z;
    qa[4 * i + 3] = v.w;
  }
}

// Where one (row, kv head)'s pages live: page p of the row is block trow[p];
// its K page is at pool + block * block_el + k_off, V at + v_off.
struct PageSrc {
  const bf16* pool;
  long long block_el, k_off, v_off;
  const int32_t* trow;
  float scale_log2;
};

template <int D>
__device__ __forceinline__ PageSrc page_src(const bf16* pool, long long block_el, int layer, int Hkv, int h,
                                            const int32_t* trow, float scale_log2) {
  PageSrc s;
  s.pool = pool;
  s.block_el = block_el;
  s.k_off = ((long long)(layer * 2) * Hkv + h) * kAttnBT * D;
  s.v_off = ((long long)(layer * 2 + 1) * Hkv + h) * kAttnBT * D;
  s.trow = trow;
  s.scale_log2 = scale_log2;
  return s;
}

template <int D>
__device__ __forceinline__ void attn_pages(const PageSrc& A, int pa, int pb, int pstep, int ctx_b,
                                           const uint32_t* qa, bf16* vs, AttnAcc<D>& st, int lane,
                                           unsigned long long* itr = nullptr) {
  // itr (diagnostics): first iteration: [0] start, [1] K arrived, [2] scores, [3] softmax, [4] PV done
  constexpr int NT = D / 8;     // output n8 tiles
  constexpr int KS = D / 16;    // k-steps of the score MMA
  constexpr int CPR = D / 8;    // 16-byte chunks per V row
  const int quad = lane & 3, r8 = lane >> 2;
  st.m = -INFINITY;
  st.l = 0.f;
#pragma unroll
  for (int n = 0; n < NT; ++n)
#pragma unroll
    for (int i = 0; i < 4; ++i) st.o[n][i] = 0.f;
  const long long k_off = A.k_off, v_off = A.v_off;
  const int32_t* trow = A.trow;
  int blk_l = -1;
  for (int p = pa, it = 0; p < pb; p += pstep, ++it) {
    if ((it & 31) == 0) blk_l = (p + lane * pstep < pb) ? __ldg(trow + p + lane * pstep) : -1;   // 32 block ids at once
    const int blk = __shfl_sync(0xffffffffu, blk_l, it & 31);
    const int n_valid = min(kAttnBT, ctx_b - p * kAttnBT);
    if (n_valid <= 0 || blk < 0) continue;
    const bool trace_it = itr && p == pa && lane == 0;
    if (trace_it) itr[0] = gtimer_();
    const bf16* page = A.pool + (long long)blk * A.block_el;
    // V page -> shared memory (XOR-swizzled 16-byte chunks), rows past the context zero
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 2 * D / 32; ++i) {
      const int j = lane + 32 * i, row = j / CPR, c = j % CPR;
      cp_async16_zfill(vs + row * D + ((c ^ (row & 7)) * 8), page + v_off + row * D + c * 8, row < n_valid);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    // K fragments of tokens r8 (n-tile 0) and 8 + r8 (n-tile 1)
    uint4 k0[D / 32], k1[D / 32];
    {
      const bf16* s0 = page + k_off + r8 * D + quad * (D / 4);
      const bf16* s1 = s0 + 8 * D;
#pragma unroll
      for (int i = 0; i < D / 32; ++i) {
        k0[i] = r8 < n_valid ? ldcg16(s0 + i * 8) : make_uint4(0u, 0u, 0u, 0u);
        k1[i] = 8 + r8 < n_valid ? ldcg16(s1 + i * 8) : make_uint4(0u, 0u, 0u, 0u);
      }
    }
    if (trace_it) itr[1] = gtimer_() + (k0[0].x == 0x12345678u);
    float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const uint32_t* w0 = reinterpret_cast<const uint32_t*>(&k0[ks / 2]) + 2 * (ks & 1);
      const uint32_t* w1 = reinterpret_cast<const uint32_t*>(&k1[ks / 2]) + 2 * (ks & 1);
      mma_16816(s0, qa[2 * ks], 0u, qa[2 * ks + 1], 0u, w0[0], w0[1]);
      mma_16816(s1, qa[2 * ks], 0u, qa[2 * ks + 1], 0u, w1[0], w1[1]);
    }
    if (trace_it) itr[2] = gtimer_() + (s0[0] == 1234.5f);
    // online softmax of row r8 over the page's 16 tokens (2q, 2q+1, 8+2q, 9+2q in this thread)
    const int t0 = 2 * quad;
    const float v00 = t0 < n_valid ? s0[0] * A.scale_log2 : -INFINITY;
    const float v01 = t0 + 1 < n_valid ? s0[1] * A.scale_log2 : -INFINITY;
    const float v10 = t0 + 8 < n_valid ? s1[0] * A.scale_log2 : -INFINITY;
    const float v11 = t0 + 9 < n_valid ? s1[1] * A.scale_log2 : -INFINITY;
    float mx = fmaxf(fmaxf(v00, v01), fmaxf(v10, v11));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float mnew = fmaxf(st.m, mx);
    const float alpha = mnew == -INFINITY ? 1.f : exp2f(st.m - mnew);
    const float p00 = v00 == -INFINITY ? 0.f : exp2f(v00 - mnew), p01 = v01 == -INFINITY ? 0.f : exp2f(v01 - mnew);
    const float p10 = v10 == -INFINITY ? 0.f : exp2f(v10 - mnew), p11 = v11 == -INFINITY ? 0.f : exp2f(v11 - mnew);
    float sum = (p00 + p01) + (p10 + p11);
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    st.l = st.l * alpha + sum;
    st.m = mnew;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      st.o[n][0] *= alpha;
      st.o[n][1] *= alpha;
    }
    const uint32_t pa0 = pack_bf2(p00, p01), pa2 = pack_bf2(p10, p11);
    if (trace_it) itr[3] = gtimer_() + (p00 == 1234.5f);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    // PV: ldmatrix.trans gives the B fragments of n-tiles 2m, 2m+1
    const int lt = lane & 7, mi = lane >> 3;          // row within matrix, matrix index
    const int vrow = (mi & 1) * 8 + lt;
#pragma unroll
    for (int m2 = 0; m2 < NT / 2; ++m2) {
      const int chunk = 2 * m2 + (mi >> 1);
      uint32_t b0, b1, b2, b3;
      ldsm_x4_trans(b0, b1, b2, b3, vs + vrow * D + ((chunk ^ (vrow & 7)) * 8));
      mma_16816(st.o[2 * m2], pa0, 0u, pa2, 0u, b0, b1);
      mma_16816(st.o[2 * m2 + 1], pa0, 0u, pa2, 0u, b2, b3);
    }
    if (trace_it) itr[4] = gtimer_() + (st.o[0][0] == 1234.5f);
  }
}

constexpr int kAttnWarpBytes = kAttnBT * 128 * 2;   // per attention warp: one V page (D <= 128)

__device__ __forceinline__ unsigned long long tagged(float v, unsigned tag) {
  return (unsigned long long)__float_as_uint(v) | ((unsigned long long)tag << 32);
}

__device__ __forceinline__ int warp_max_int(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ void l2_prefetch_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// One layer's paged decode attention for the scheduler's mixed batch.
struct AttnWork {
  const bf16* pool;
  long long block_el;
  int layer, Hq, Hkv;
  const bf16* q;
  int q_stride;
  const int32_t* table;
  int max_blocks;
  const int32_t* ctx;
  bf16* out;             // [M][Hq*D]
  float scale_log2;
  unsigned long long* ws;  // [grid][G][D+2] tagged split partials (fp32 bits | tag << 32)
  unsigned tag;          // unique per launch and phase
  int prefetch;          // L2-prefetch the pages before the (q/k/v) wait: worth it only when there is a wait
  int min_pages;
  int M;
};

// One layer's attention by the 4 epilogue warps of every CTA. The (row, kv
// head) sequences' pages are split evenly over the CTAs; inside a CTA the
// four warps take every fourth page of the CTA's piece and merge in shared
// memory, so each sequence has at most one partial per CTA. The last CTA to
// finish a split sequence merges the partials (CTA order: deterministic); the
// kv head's flag is raised when all M rows of that head are written.
// L2 prefetch of the K/V pages this warp will read in attn_cta_phase (same
// work distribution): issued ahead -- e.g. by the previous layer's launch --
// so the attention's page loads hit L2.
template <int D>
__device__ __forceinline__ void attn_cta_prefetch(const AttnWork& A, int cta, int grid, int warp, int lane) {
  const int M = A.M, Hkv = A.Hkv;
  // pages per row (retired rows count one empty page so that every (row, head) is written)
  int pg0 = 0, pg1 = 0;
  if (lane < M) pg0 = max(1, (__ldg(A.ctx + lane) + kAttnBT - 1) / kAttnBT);
  if (lane + 32 < M) pg1 = max(1, (__ldg(A.ctx + lane + 32) + kAttnBT - 1) / kAttnBT);
  int s0 = pg0, s1 = pg1;   // inclusive scan over rows 0..63 (lane holds rows lane and lane+32)
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, s0, o), c = __shfl_up_sync(0xffffffffu, s1, o);
    if (lane >= o) {
      s0 += a;
      s1 += c;
    }
  }
  s1 += __shfl_sync(0xffffffffu, s0, 31);
  const int total_pages = __shfl_sync(0xffffffffu, s1, 31);
  const int U = Hkv * total_pages;
  // pages per CTA: cover the SMs, >= 4 * min_pages, <= 32 parts per sequence
  const int maxpg = warp_max_int(max(pg0, pg1));
  const int qc = max(max(4 * A.min_pages, (U + grid - 1) / grid), (maxpg + 30) / 31);
  const int my0 = cta * qc, my1 = min(U, my0 + qc);
  const int ex0 = s0 - pg0, ex1 = s1 - pg1;   // exclusive prefixes of rows lane, lane+32
  auto resolve = [&](int cur, int& b, int& h, int& seq0, int& seq1, int& pe) {
    const unsigned b0 = __ballot_sync(0xffffffffu, lane < M && Hkv * ex0 <= cur);
    const unsigned b1 = __ballot_sync(0xffffffffu, lane + 32 < M && Hkv * ex1 <= cur);
    b = __popc(b0) + __popc(b1) - 1;
    const int exb = __shfl_sync(0xffffffffu, b < 32 ? ex0 : ex1, b & 31);
    const int pgb = __shfl_sync(0xffffffffu, b < 32 ? pg0 : pg1, b & 31);
    const int row_start = Hkv * exb;
    h = (cur - row_start) / pgb;
    seq0 = row_start + h * pgb;
    seq1 = seq0 + pgb;
    pe = min(my1, seq1);
  };
  // L2 prefetch of this warp's K/V pages before waiting for the QKV flags
  for (int cur = my0; cur < my1;) {
    int b, h, seq0, seq1, pe;
    resolve(cur, b, h, seq0, seq1, pe);
    const int ctx_b = __ldg(A.ctx + b);
    const int32_t* trow = A.table + (long long)b * A.max_blocks;
    const long long k_off = ((long long)(A.layer * 2) * A.Hkv + h) * kAttnBT * D;
    const long long v_off = ((long long)(A.layer * 2 + 1) * A.Hkv + h) * kAttnBT * D;
    for (int p = cur - seq0 + warp + 4 * lane; p < pe - seq0; p += 128) {
      const int blk = p * kAttnBT < ctx_b ? __ldg(trow + p) : -1;
      if (blk >= 0) {
        const bf16* page = A.pool + (long long)blk * A.block_el;
        l2_prefetch_bulk(page + k_off, kAttnBT * D * 2);
        l2_prefetch_bulk(page + v_off, kAttnBT * D * 2);
      }
    }
    cur = pe;
  }
}

template <int D, int G, class WaitHead, class DoneHead>
__device__ __forceinline__ void attn_cta_phase(const AttnWork& A, int cta, int grid, int warp, int lane,
                                               bf16* vs_all, const WaitHead& wait_head, const DoneHead& done_head,
                                               unsigned long long* atr = nullptr) {
  // atr (diagnostics, may be null): this warp's first piece: [0] entry,
  // [1] q/k/v flags seen, [2] q loaded, [3] pages done, [4] CTA merge +
  // partial published, [5] split merge done, [6] output published, [7] exit
  auto mark = [&](int k, bool first) {
    if (atr && first && lane == 0) atr[k] = gtimer_();
  };
  mark(0, true);
  const int M = A.M, Hkv = A.Hkv;
  const int et = warp * 32 + lane;
  bf16* vs = vs_all + warp * (kAttnWarpBytes / 2);
  // pages per row (retired rows count one empty page so that every (row, head) is written)
  int pg0 = 0, pg1 = 0;
  if (lane < M) pg0 = max(1, (__ldg(A.ctx + lane) + kAttnBT - 1) / kAttnBT);
  if (lane + 32 < M) pg1 = max(1, (__ldg(A.ctx + lane + 32) + kAttnBT - 1) / kAttnBT);
  int s0 = pg0, s1 = pg1;   // inclusive scan over rows 0..63 (lane holds rows lane and lane+32)
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, s0, o), c = __shfl_up_sync(0xffffffffu, s1, o);
    if (lane >= o) {
      s0 += a;
      s1 += c;
    }
  }
  s1 += __shfl_sync(0xffffffffu, s0, 31);
  const int total_pages = __shfl_sync(0xffffffffu, s1, 31);
  const int U = Hkv * total_pages;
  // pages per CTA: cover the SMs, >= 4 * min_pages, <= 32 parts per sequence
  const int maxpg = warp_max_int(max(pg0, pg1));
  const int qc = max(max(4 * A.min_pages, (U + grid - 1) / grid), (maxpg + 30) / 31);
  const int my0 = cta * qc, my1 = min(U, my0 + qc);
  const int ex0 = s0 - pg0, ex1 = s1 - pg1;   // exclusive prefixes of rows lane, lane+32
  auto resolve = [&](int cur, int& b, int& h, int& seq0, int& seq1, int& pe) {
    const unsigned b0 = __ballot_sync(0xffffffffu, lane < M && Hkv * ex0 <= cur);
    const unsigned b1 = __ballot_sync(0xffffffffu, lane + 32 < M && Hkv * ex1 <= cur);
    b = __popc(b0) + __popc(b1) - 1;
    const int exb = __shfl_sync(0xffffffffu, b < 32 ? ex0 : ex1, b & 31);
    const int pgb = __shfl_sync(0xffffffffu, b < 32 ? pg0 : pg1, b & 31);
    const int row_start = Hkv * exb;
    h = (cur - row_start) / pgb;
    seq0 = row_start + h * pgb;
    seq1 = seq0 + pgb;
    pe = min(my1, seq1);
  };
  // L2 prefetch of this warp's K/V pages before waiting for the QKV flags
  if (A.prefetch) {
  for (int cur = my0; cur < my1;) {
    int b, h, seq0, seq1, pe;
    resolve(cur, b, h, seq0, seq1, pe);
    const int ctx_b = __ldg(A.ctx + b);
    const int32_t* trow = A.table + (long long)b * A.max_blocks;
    const long long k_off = ((long long)(A.layer * 2) * A.Hkv + h) * kAttnBT * D;
    const long long v_off = ((long long)(A.layer * 2 + 1) * A.Hkv + h) * kAttnBT * D;
    for (int p = cur - seq0 + warp + 4 * lane; p < pe - seq0; p += 128) {
      const int blk = p * kAttnBT < ctx_b ? __ldg(trow + p) : -1;
      if (blk >= 0) {
        const bf16* page = A.pool + (long long)blk * A.block_el;
        l2_prefetch_bulk(page + k_off, kAttnBT * D * 2);
        l2_prefetch_bulk(page + v_off, kAttnBT * D * 2);
      }
    }
    cur = pe;
  }
  }
  constexpr int EPT = (G * D + 128 - 1) / 128;   // merged elements per thread
  unsigned heads_ready = 0;
  for (int cur = my0; cur < my1;) {
    int b, h, seq0, seq1, pe;
    resolve(cur, b, h, seq0, seq1, pe);
    const int pa = cur - seq0, pb = pe - seq0;
    const bool first_piece = cur == my0;
    if (!(heads_ready >> h & 1)) {
      wait_head(h, lane);
      heads_ready |= 1u << h;
    }
    mark(1, first_piece);
    const int ctx_b = __ldg(A.ctx + b);
    const int r8 = lane >> 2, quad = lane & 3;
    uint32_t qa[D / 8];
    attn_load_q<D>(A.q + (long long)b * A.q_stride + (long long)(h * G + r8) * D, r8 < G, quad, qa);
    mark(2, first_piece);
    AttnAcc<D> st;
    const PageSrc src = page_src<D>(A.pool, A.block_el, A.layer, A.Hkv, h, A.table + (long long)b * A.max_blocks,
                                    A.scale_log2);
    attn_pages<D>(src, pa + warp, pb, 4, ctx_b, qa, vs, st, lane, (atr && first_piece) ? atr + 8 : nullptr);
    mark(3, first_piece);
    // ---- CTA merge of the 4 warps' states (warp order) through shared memory
    float* wst = reinterpret_cast<float*>(vs);   // this warp's V page is free now: [G] m, [G] l, [G][D] o
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
    epi_bar();
    float Mv[EPT], Lv[EPT], Ov[EPT];
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const int idx = et * EPT + e, g = idx / D, dd = idx % D;
      Mv[e] = -INFINITY;
      Lv[e] = 0.f;
      Ov[e] = 0.f;
      if (idx < G * D) {
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const float* ws = reinterpret_cast<const float*>(vs_all + w * (kAttnWarpBytes / 2));
          const float mk = ws[g], mn = fmaxf(Mv[e], mk);
          const float a0 = mn == -INFINITY ? 0.f : exp2f(Mv[e] - mn), a1 = mn == -INFINITY ? 0.f : exp2f(mk - mn);
          Lv[e] = Lv[e] * a0 + ws[G + g] * a1;
          Ov[e] = Ov[e] * a0 + ws[2 * G + g * D + dd] * a1;
          Mv[e] = mn;
        }
      }
    }
    // Split sequences: the CTA owning the sequence's first pages merges. Its
    // piece closes its range, while the other parts open the ranges of the
    // following CTAs, so they are normally published first; parts are
    // self-validating 64-bit words (fp32 bits | tag << 32) -- one round trip,
    // no arrival counter. Merge order: own part, then the CTAs in order.
    const int first_c = seq0 / qc, last_c = (seq1 - 1) / qc;
    const bool merger = cta == first_c;
    bool done = first_c == last_c;
    if (!done && !merger) {
      // contributor: this piece opens this CTA's range (slot 0)
      unsigned long long* part = A.ws + (long long)cta * G * (D + 2);
#pragma unroll
      for (int e = 0; e < EPT; ++e) {
        const int idx = et * EPT + e, g = idx / D, dd = idx % D;
        if (idx < G * D) {
          tc::st_relaxed_u64(part + 2 * G + idx, tagged(Ov[e], A.tag));
          if (dd == 0) {
            tc::st_relaxed_u64(part + g, tagged(Mv[e], A.tag));
            tc::st_relaxed_u64(part + G + g, tagged(Lv[e], A.tag));
          }
        }
      }
      mark(4, first_piece);
    } else if (!done) {
      // a thread's EPT elements lie in one head row g: per part, m and l are
      // two words and o is EPT words; eight parts are polled together
      const int g_me = min(et * EPT, G * D - 1) / D;
      for (int c0 = first_c + 1; c0 <= last_c; c0 += 8) {
        unsigned long long pm[8], pl[8], po[8][EPT];
        for (int spin = 0;; ++spin) {
          bool ready = true;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const unsigned long long* pp = A.ws + (long long)(c0 + k) * G * (D + 2);
            const bool ok = c0 + k <= last_c;
            pm[k] = ok ? tc::ld_relaxed_u64(pp + g_me) : tagged(-INFINITY, A.tag);
            pl[k] = ok ? tc::ld_relaxed_u64(pp + G + g_me) : tagged(0.f, A.tag);
#pragma unroll
            for (int e = 0; e < EPT; ++e) {
              const int idx = et * EPT + e;
              po[k][e] = (ok && idx < G * D) ? tc::ld_relaxed_u64(pp + 2 * G + idx) : tagged(0.f, A.tag);
            }
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            ready &= (unsigned)(pm[k] >> 32) == A.tag && (unsigned)(pl[k] >> 32) == A.tag;
#pragma unroll
            for (int e = 0; e < EPT; ++e) ready &= (unsigned)(po[k][e] >> 32) == A.tag;
          }
          if (ready) {
            if (atr && lane == 0 && first_piece && c0 == first_c + 1) atr[14] = (unsigned long long)spin;
            break;
          }
          __nanosleep(64);
        }
        if (atr && first_piece && c0 == first_c + 1) {
          __syncwarp();
          if (lane == 0) atr[13] = gtimer_();   // every lane of the warp has its words
        }
        // a thread's EPT elements share one head row: one (m, l) rescale per part
        float mc = Mv[0], lc = Lv[0];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (c0 + k > last_c) continue;   // warp-uniform
          const float mk = __uint_as_float((unsigned)pm[k]), lk = __uint_as_float((unsigned)pl[k]);
          const float mn = fmaxf(mc, mk);
          const float mr = mn == -INFINITY ? 0.f : mn;   // all -inf: both scales 0
          const float a0 = exp2f(mc - mr), a1 = exp2f(mk - mr);
          lc = lc * a0 + lk * a1;
#pragma unroll
          for (int e = 0; e < EPT; ++e) Ov[e] = Ov[e] * a0 + __uint_as_float((unsigned)po[k][e]) * a1;
          mc = mn;
        }
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
          Mv[e] = mc;
          Lv[e] = lc;
        }
      }
      done = true;
      mark(5, first_piece);
    }
    if (done) {
      bf16* out = A.out + (long long)b * (A.Hq * D) + (long long)h * G * D;
#pragma unroll
      for (int e = 0; e < EPT; ++e) {
        const int idx = et * EPT + e;
        if (idx < G * D) out[idx] = f2bf(Lv[e] > 0.f ? Ov[e] / Lv[e] : 0.f);
      }
      done_head(h, warp * 32 + lane);   // all 128 threads
    }
    mark(6, first_piece);
    epi_bar();   // the warps' shared-memory states are rewritten by the next piece
    cur = pe;
  }
  mark(7, true);
}

}  // namespace attn
}  // namespace astraea
