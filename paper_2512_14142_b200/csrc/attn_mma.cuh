// Tensor-core paged decode attention of one warp over a (row, kv head)'s
// pages: shared by the per-layer decode kernel (attention.cu) and the
// decode-step kernel's attention phase (decode_step.cu).
#pragma once

#include "common.cuh"
#include "tc.cuh"

namespace astraea {
namespace attn {

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

}  // namespace attn
}  // namespace astraea
