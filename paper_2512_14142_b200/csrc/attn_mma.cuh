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

// ---------------------------------------------------------------------------
// The same page math with S pages in flight per warp (S >= 2): K and V pages
// arrive by TMA -- a 2-D tensor map over the pool viewed as
// [blocks x L x 2 x Hkv x 16 rows][D], 128-byte swizzle, one 16-row x
// 64-column box per half page -- into the warp's ring of S stages (one
// mbarrier each). The warp computes page k while pages k+1..k+S-1 land; lane
// 0 refills a stage as soon as the warp has read it. The swizzle keeps the
// ldmatrix reads of K (scores) and V (transposed, PV) conflict-free. Q is in
// the standard A-fragment layout (attn_load_q_std). ``cnt``: the warp's
// running page count (ring position and barrier phase), carried across
// pieces and launches' phases.
// ---------------------------------------------------------------------------
template <int D>
constexpr int tma_page_bytes() { return 2 * kAttnBT * D * 2; }   // K + V page

__device__ __forceinline__ uint32_t sw128_off(int row, int chunk) {   // in [16 rows][64 cols] half pages
  return (uint32_t)((chunk >> 3) * (kAttnBT * 128) + row * 128 + (((chunk & 7) ^ (row & 7)) << 4));
}

template <int D>
__device__ __forceinline__ void attn_load_q_std(const bf16* q_row, bool ok, int quad, uint32_t (*qa)[2]) {
#pragma unroll
  for (int ks = 0; ks < D / 16; ++ks) {
    qa[ks][0] = ok ? __ldcg(reinterpret_cast<const unsigned int*>(q_row + 16 * ks + 2 * quad)) : 0u;
    qa[ks][1] = ok ? __ldcg(reinterpret_cast<const unsigned int*>(q_row + 16 * ks + 8 + 2 * quad)) : 0u;
  }
}

struct TmaPages {
  const CUtensorMap* map;
  int block_rows;          // rows of one pool block in the 2-D view (L * 2 * Hkv * 16)
  int k_row0, v_row0;      // (layer, head) row offsets of the K and V pages within a block
};

// Issue the TMA of page k (of pages pa, pa + pstep, ...) into stage (cnt + k) % S.
template <int D, int S>
__device__ __forceinline__ void attn_tma_issue(const TmaPages& T, int k, int blk, uint8_t* ring, uint64_t* bars,
                                               uint32_t cnt) {
  constexpr int PB = tma_page_bytes<D>();
  constexpr int HALF = kAttnBT * 128;
  const uint32_t slot = (cnt + k) % S;
  uint64_t* bb = bars + slot;
  uint8_t* stw = ring + slot * PB;
  const int kr = blk * T.block_rows + T.k_row0, vr = blk * T.block_rows + T.v_row0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // the warp's reads of the stage come first
  mbar_arrive_expect_tx(bb, PB);
#pragma unroll
  for (int hf = 0; hf < D / 64; ++hf) {
    tc::tma_load_2d(stw + hf * HALF, T.map, bb, hf * 64, kr);
    tc::tma_load_2d(stw + (D / 64) * HALF + hf * HALF, T.map, bb, hf * 64, vr);
  }
}

// Before the wait for the previous kernel: issue the first stages' pages
// that hold only older tokens. In a decode step the previous kernel appends
// just the newest token (position ctx - 1) of this layer; every kernel that
// wrote older pages completed before the step began. Returns how many of the
// first S pages were issued (a prefix); attn_pages_tma(pre = that) issues the rest.
template <int D, int S>
__device__ __forceinline__ int attn_pages_tma_preissue(const TmaPages& T, const int32_t* trow, int pa, int pb,
                                                       int pstep, int ctx_b, uint8_t* ring, uint64_t* bars,
                                                       uint32_t cnt, int lane) {
  const int my = pb > pa ? (pb - pa + pstep - 1) / pstep : 0;
  const int new_page = (ctx_b - 1) / kAttnBT;
  int n = 0;
  while (n < S && n < my && pa + pstep * n < new_page) ++n;
  const int blk = lane < n ? __ldg(trow + pa + pstep * lane) : 0;
#pragma unroll
  for (int k = 0; k < S; ++k) {
    const int b = __shfl_sync(0xffffffffu, blk, k);
    if (lane == 0 && k < n) attn_tma_issue<D, S>(T, k, b, ring, bars, cnt);
  }
  return n;
}

template <int D, int S>
__device__ __forceinline__ void attn_pages_tma(const TmaPages& T, const int32_t* trow, int pa, int pb, int pstep,
                                               int ctx_b, float scale_log2, const uint32_t (*qa)[2],
                                               uint8_t* ring, uint64_t* bars, uint32_t& cnt, AttnAcc<D>& st,
                                               int lane, int pre = 0) {
  // pre: the first `pre` pages were issued already (attn_pages_tma_preissue)
  constexpr int PB = tma_page_bytes<D>();
  constexpr int HALF = kAttnBT * 128;
  constexpr int KS = D / 16, NT = D / 8;
  st.m = -INFINITY;
  st.l = 0.f;
#pragma unroll
  for (int n = 0; n < NT; ++n)
#pragma unroll
    for (int i = 0; i < 4; ++i) st.o[n][i] = 0.f;
  const int my = pb > pa ? (pb - pa + pstep - 1) / pstep : 0;
  if (my == 0) return;
  auto ids_of = [&](int w0) { return w0 + lane < my ? __ldg(trow + pa + pstep * (w0 + lane)) : 0; };
  int blk_c = ids_of(0), blk_n = ids_of(32);
  auto issue = [&](int k, int blk) { attn_tma_issue<D, S>(T, k, blk, ring, bars, cnt); };   // lane 0
#pragma unroll
  for (int k = 0; k < S; ++k) {
    const int blk = __shfl_sync(0xffffffffu, blk_c, k);
    if (lane == 0 && k < my && k >= pre) issue(k, blk);
  }
  const int quad = lane & 3;
  for (int k = 0; k < my; ++k) {
    const int pg = pa + pstep * k;
    const int n_valid = min(kAttnBT, ctx_b - pg * kAttnBT);
    const int nxt = k + S;
    if ((nxt & 31) == 1) blk_n = ids_of(nxt + 31);   // the next 32-page window, early
    if ((nxt & 31) == 0) blk_c = blk_n;
    const int nxt_blk = __shfl_sync(0xffffffffu, blk_c, nxt & 31);
    const uint32_t slot = (cnt + k) % S;
    mbar_wait(bars + slot, ((cnt + k) / S) & 1);
    const uint32_t kb = smem_u32(ring + slot * PB), vb = kb + (D / 64) * HALF;
    // S = Q K^T: ldmatrix.x4 gives (tok 0-7, k lo)(tok 0-7, k hi)(tok 8-15, k lo)(tok 8-15, k hi)
    float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int r = (lane & 7) + ((lane >> 4) << 3);
      const int c = 2 * ks + ((lane >> 3) & 1);
      uint32_t b0, b1, b2, b3;
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                   : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3) : "r"(kb + sw128_off(r, c)));
      mma_16816(s0, qa[ks][0], 0u, qa[ks][1], 0u, b0, b1);
      mma_16816(s1, qa[ks][0], 0u, qa[ks][1], 0u, b2, b3);
    }
    // online softmax of row lane/4 over the page (tokens 2q, 2q+1, 8+2q, 9+2q)
    const int t0 = 2 * quad;
    const float v00 = t0 < n_valid ? s0[0] * scale_log2 : -INFINITY;
    const float v01 = t0 + 1 < n_valid ? s0[1] * scale_log2 : -INFINITY;
    const float v10 = t0 + 8 < n_valid ? s1[0] * scale_log2 : -INFINITY;
    const float v11 = t0 + 9 < n_valid ? s1[1] * scale_log2 : -INFINITY;
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
    // O += P V: ldmatrix.trans of (tok 0-7, d)(tok 8-15, d)(tok 0-7, d+8)(tok 8-15, d+8)
#pragma unroll
    for (int m2 = 0; m2 < NT / 2; ++m2) {
      const int r = (lane & 7) + (((lane >> 3) & 1) << 3);
      const int c = 2 * m2 + (lane >> 4);
      uint32_t b0, b1, b2, b3;
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                   : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3) : "r"(vb + sw128_off(r, c)));
      mma_16816(st.o[2 * m2], pa0, 0u, pa2, 0u, b0, b1);
      mma_16816(st.o[2 * m2 + 1], pa0, 0u, pa2, 0u, b2, b3);
    }
    __syncwarp();
    if (lane == 0 && nxt < my) issue(nxt, nxt_blk);   // refill this stage with page k + S
  }
  cnt += (uint32_t)my;
}

// per attention warp: one V page (D <= 128), reused after the page loop for
// the warp's merge state ([G] m, [G] l, [G][D] o fp32: 4,160 B at G = 8, D = 128)
constexpr int kAttnWarpBytes = kAttnBT * 128 * 2 + 128;

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

// Work split of one layer's attention over the CTAs (every lane of a warp
// computes the same result). A (row, kv head) sequence has pg pages (retired
// rows count one empty page, so every output row is written).
//  * aligned (sequences <= CTAs): each sequence is cut into ceil(pg / qc)
//    parts of qc consecutive pages on consecutive CTAs, one part per CTA;
//    qc >= 4 * min_pages, <= 32 parts per sequence, the smallest qc (from the
//    even share up) whose parts fit the grid. No CTA works on two sequences,
//    so no piece waits behind another.
//  * contiguous (more sequences than CTAs): the concatenated pages are cut
//    into equal ranges of qc pages; a CTA walks the pieces of its range.
// A piece = (row b, head h, pages [pa, pb)); its sequence's parts live on
// CTAs first_c..last_c, first_c merges.
struct AttnPiece {
  int b, h, pa, pb, first_c, last_c;
};

__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct AttnSplit {
  const AttnWork* A;
  int lane, cta;
  bool aligned;
  int qc, my0, my1;       // contiguous: this CTA's page range
  int pg0, pg1;           // pages of rows lane, lane + 32
  int ex0, ex1;           // exclusive prefixes: pages (contiguous) or parts (aligned) of rows lane, lane + 32
  int np0, np1;           // aligned: parts of rows lane, lane + 32
  int n_pieces;           // this CTA's pieces (aligned: 0 or 1)
  int cur;                // contiguous: next page of the range

  __device__ __forceinline__ void init(const AttnWork& W, int cta_, int grid, int lane_) {
    A = &W;
    lane = lane_;
    cta = cta_;
    const int M = W.M, Hkv = W.Hkv;
    pg0 = pg1 = 0;
    if (lane < M) pg0 = max(1, (__ldg(W.ctx + lane) + kAttnBT - 1) / kAttnBT);
    if (lane + 32 < M) pg1 = max(1, (__ldg(W.ctx + lane + 32) + kAttnBT - 1) / kAttnBT);
    const int total = warp_sum_int(pg0 + pg1);
    const int maxpg = warp_max_int(max(pg0, pg1));
    qc = max(max(4 * W.min_pages, (Hkv * total + grid - 1) / grid), (maxpg + 31) / 32);
    aligned = Hkv * M <= grid;
    int v0 = pg0, v1 = pg1;
    if (aligned) {
      for (int it = 0; it < 64; ++it) {
        np0 = (pg0 + qc - 1) / qc;
        np1 = (pg1 + qc - 1) / qc;
        if (Hkv * warp_sum_int(np0 + np1) <= grid) break;
        qc += max(1, qc / 8);
      }
      v0 = np0;
      v1 = np1;
    }
    int s0 = v0, s1 = v1;   // inclusive scan over rows 0..63
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int x = __shfl_up_sync(0xffffffffu, s0, o), y = __shfl_up_sync(0xffffffffu, s1, o);
      if (lane >= o) {
        s0 += x;
        s1 += y;
      }
    }
    s1 += __shfl_sync(0xffffffffu, s0, 31);
    ex0 = s0 - v0;
    ex1 = s1 - v1;
    const int all = Hkv * __shfl_sync(0xffffffffu, s1, 31);
    if (aligned) {
      n_pieces = cta < all ? 1 : 0;
    } else {
      my0 = cta * qc;
      my1 = min(all, my0 + qc);
      cur = my0;
      n_pieces = my0 < my1 ? 1 : 0;   // at least one; next() tells when the range ends
    }
  }
  // the row whose prefix (in units of one head) covers position x
  __device__ __forceinline__ int row_of(int x, int& ex, int& pg, int& np) const {
    const int Hkv = A->Hkv, M = A->M;
    const unsigned b0 = __ballot_sync(0xffffffffu, lane < M && Hkv * ex0 <= x);
    const unsigned b1 = __ballot_sync(0xffffffffu, lane + 32 < M && Hkv * ex1 <= x);
    const int b = max(0, __popc(b0) + __popc(b1) - 1);
    ex = __shfl_sync(0xffffffffu, b < 32 ? ex0 : ex1, b & 31);
    pg = __shfl_sync(0xffffffffu, b < 32 ? pg0 : pg1, b & 31);
    np = aligned ? __shfl_sync(0xffffffffu, b < 32 ? np0 : np1, b & 31) : 0;
    return b;
  }
  // the piece starting at the current position; false when the CTA is done
  __device__ __forceinline__ bool next(AttnPiece& pc) {
    const int Hkv = A->Hkv;
    int ex, pg, np;
    if (aligned) {
      if (n_pieces == 0) return false;
      n_pieces = 0;
      pc.b = row_of(cta, ex, pg, np);
      np = max(1, np);
      const int r0 = cta - Hkv * ex, part = r0 % np;
      pc.h = r0 / np;
      pc.pa = part * qc;
      pc.pb = min(pg, pc.pa + qc);
      pc.first_c = cta - part;
      pc.last_c = pc.first_c + np - 1;
      return true;
    }
    if (cur >= my1) return false;
    pc.b = row_of(cur, ex, pg, np);
    const int row_start = Hkv * ex;
    pc.h = (cur - row_start) / pg;
    const int seq0 = row_start + pc.h * pg, seq1 = seq0 + pg, pe = min(my1, seq1);
    pc.pa = cur - seq0;
    pc.pb = pe - seq0;
    pc.first_c = seq0 / qc;
    pc.last_c = (seq1 - 1) / qc;
    cur = pe;
    return true;
  }
};

// L2 prefetch of the K/V pages this CTA's warps read in attn_cta_phase (same
// work split), e.g. issued by the previous layer's launch.
template <int D>
__device__ __forceinline__ void attn_cta_prefetch(const AttnWork& A, int cta, int grid, int warp, int lane) {
  AttnSplit sp;
  sp.init(A, cta, grid, lane);
  AttnPiece pc;
  while (sp.next(pc)) {
    const int ctx_b = __ldg(A.ctx + pc.b);
    const int32_t* trow = A.table + (long long)pc.b * A.max_blocks;
    const long long k_off = ((long long)(A.layer * 2) * A.Hkv + pc.h) * kAttnBT * D;
    const long long v_off = ((long long)(A.layer * 2 + 1) * A.Hkv + pc.h) * kAttnBT * D;
    for (int p = pc.pa + warp + 4 * lane; p < pc.pb; p += 128) {
      const int blk = p * kAttnBT < ctx_b ? __ldg(trow + p) : -1;
      if (blk >= 0) {
        const bf16* page = A.pool + (long long)blk * A.block_el;
        l2_prefetch_bulk(page + k_off, kAttnBT * D * 2);
        l2_prefetch_bulk(page + v_off, kAttnBT * D * 2);
      }
    }
  }
}

// One layer's attention by the 4 epilogue warps of every CTA: this CTA's
// piece (attn_split) -- the four warps take every fourth page and merge in
// shared memory; a split sequence's part-0 CTA merges the other parts'
// self-validating partials (CTA order: deterministic) and writes the output.
// wait_head(h, lane) runs before the first q / page load (e.g. waits for the
// kernel that produced q and the new K/V); done_head(h, thread) after the
// merged output is written.
// AS > 1: the TMA-staged page loop (attn_pages_tma) with AS stages per warp
// in vs_all ([4][AS][K + V page], 1024-byte aligned), barriers abar[4][AS] and
// the warps' running page counts acnt (caller-initialised, carried over).
template <int D, int G, int AS = 1, class WaitHead, class DoneHead>
__device__ __forceinline__ void attn_cta_phase(const AttnWork& A, int cta, int grid, int warp, int lane,
                                               bf16* vs_all, const WaitHead& wait_head, const DoneHead& done_head,
                                               unsigned long long* atr = nullptr, const TmaPages* tp = nullptr,
                                               uint64_t* abar = nullptr, uint32_t* acnt = nullptr) {
  // acnt: this warp's running page count (AS > 1), one word per calling thread
  // atr (diagnostics, may be null): [0] entry, [1] wait_head passed, [2] q
  // loaded, [3] pages done, [4] CTA merge + partial published, [5] split
  // merge done, [6] output published, [7] exit, [8..12] first page, [13]
  // merger: all parts seen, [14] merger: spins
  auto mark = [&](int k) {
    if (atr && lane == 0) atr[k] = gtimer_();
  };
  mark(0);
  const int et = warp * 32 + lane;
  constexpr int WREG = (AS > 1 ? AS * tma_page_bytes<D>() : kAttnWarpBytes) / 2;   // per-warp region (bf16)
  bf16* vs = vs_all + warp * WREG;
  AttnSplit sp;
  sp.init(A, cta, grid, lane);
  constexpr int EPT = (G * D + 128 - 1) / 128;   // merged elements per thread
  unsigned heads_ready = 0;
  AttnPiece pc;
  while (sp.next(pc)) {
    const int b = pc.b, h = pc.h;
    const int ctx_b = __ldg(A.ctx + b);   // the step's contexts and tables: ready before any wait
    int pre = 0;
    TmaPages T;
    if constexpr (AS > 1) {
      T = *tp;
      T.k_row0 = (A.layer * 2 * A.Hkv + h) * kAttnBT;
      T.v_row0 = T.k_row0 + A.Hkv * kAttnBT;
      // pages of older tokens stream while the previous kernel finishes
      pre = attn_pages_tma_preissue<D, AS>(T, A.table + (long long)b * A.max_blocks, pc.pa + warp, pc.pb, 4,
                                           ctx_b, reinterpret_cast<uint8_t*>(vs), abar + warp * AS, *acnt, lane);
    }
    if (!(heads_ready >> h & 1)) {
      wait_head(h, lane);
      heads_ready |= 1u << h;
    }
    mark(1);
    const int r8 = lane >> 2, quad = lane & 3;
    AttnAcc<D> st;
    if constexpr (AS > 1) {
      uint32_t qs[D / 16][2];
      attn_load_q_std<D>(A.q + (long long)b * A.q_stride + (long long)(h * G + r8) * D, r8 < G, quad, qs);
      mark(2);
      attn_pages_tma<D, AS>(T, A.table + (long long)b * A.max_blocks, pc.pa + warp, pc.pb, 4, ctx_b, A.scale_log2,
                            qs, reinterpret_cast<uint8_t*>(vs), abar + warp * AS, *acnt, st, lane, pre);
    } else {
      uint32_t qa[D / 8];
      attn_load_q<D>(A.q + (long long)b * A.q_stride + (long long)(h * G + r8) * D, r8 < G, quad, qa);
      mark(2);
      const PageSrc src = page_src<D>(A.pool, A.block_el, A.layer, A.Hkv, h,
                                      A.table + (long long)b * A.max_blocks, A.scale_log2);
      attn_pages<D>(src, pc.pa + warp, pc.pb, 4, ctx_b, qa, vs, st, lane, atr ? atr + 8 : nullptr);
    }
    mark(3);
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
          const float* ws = reinterpret_cast<const float*>(vs_all + w * WREG);
          const float mk = ws[g], mn = fmaxf(Mv[e], mk);
          const float a0 = mn == -INFINITY ? 0.f : exp2f(Mv[e] - mn), a1 = mn == -INFINITY ? 0.f : exp2f(mk - mn);
          Lv[e] = Lv[e] * a0 + ws[G + g] * a1;
          Ov[e] = Ov[e] * a0 + ws[2 * G + g * D + dd] * a1;
          Mv[e] = mn;
        }
      }
    }
    // Split sequences: part 0's CTA merges. Parts are self-validating 64-bit
    // words (fp32 bits | tag << 32) -- one round trip, no arrival counter.
    // Merge order: own part, then the CTAs in order.
    const int first_c = pc.first_c, last_c = pc.last_c;
    const bool merger = cta == first_c;
    bool done = first_c == last_c;
    if (!done && !merger) {
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
      mark(4);
    } else if (!done) {
      // a thread's EPT elements lie in one head row g: per part, m and l are
      // two words and o is EPT words; eight parts are polled together
      const int g_me = min(et * EPT, G * D - 1) / D;
      constexpr int KP = EPT <= 4 ? 8 : 4;   // parts polled per round (32 words of o per thread)
      for (int c0 = first_c + 1; c0 <= last_c; c0 += KP) {
        unsigned long long pm[KP], pl[KP], po[KP][EPT];
        for (int spin = 0;; ++spin) {
          bool ready = true;
#pragma unroll
          for (int k = 0; k < KP; ++k) {
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
          for (int k = 0; k < KP; ++k) {
            ready &= (unsigned)(pm[k] >> 32) == A.tag && (unsigned)(pl[k] >> 32) == A.tag;
#pragma unroll
            for (int e = 0; e < EPT; ++e) ready &= (unsigned)(po[k][e] >> 32) == A.tag;
          }
          if (ready) {
            if (atr && lane == 0 && c0 == first_c + 1) atr[14] = (unsigned long long)spin;
            break;
          }
          __nanosleep(64);
        }
        if (atr && c0 == first_c + 1) {
          __syncwarp();
          if (lane == 0) atr[13] = gtimer_();   // every lane of the warp has its words
        }
        // a thread's EPT elements share one head row: one (m, l) rescale per part
        float mc = Mv[0], lc = Lv[0];
#pragma unroll
        for (int k = 0; k < KP; ++k) {
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
      mark(5);
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
    mark(6);
    epi_bar();   // the warps' shared-memory states are rewritten by the next piece
  }
  mark(7);
}

}  // namespace attn
}  // namespace astraea
