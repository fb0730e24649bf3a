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

using namespace astraea;

namespace {

constexpr int kBT = 16;         // tokens per block
constexpr int kStages = 4;      // decode smem ring depth
constexpr int kMaxSplits = 64;  // context splits per (row, kv head)
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
};

template <int D, int G>
__global__ void __launch_bounds__(128) decode_kernel(const __grid_constant__ DecodeParams p) {
  constexpr int PAGE = kBT * D;             // elements per page
  constexpr int CPR = D / 8;                // 16-byte chunks per row
  constexpr int CPT = CPR / 8;              // chunks per score thread (8 threads per token)
  constexpr int TPH = 128 / G;              // PV threads per q head
  constexpr int DPT = D / TPH;              // dims per PV thread
  static_assert(DPT >= 1 && DPT <= 8, "PV mapping");

  __shared__ __align__(128) bf16 ks[kStages][PAGE];
  __shared__ __align__(128) bf16 vs[kStages][PAGE];
  __shared__ float qs[G][D];
  __shared__ float sc[G][kBT];
  __shared__ __align__(8) uint64_t bar[kStages];

  const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x;
  pdl_wait();
  pdl_launch();
  const int ctx = p.ctx[b];
  const int nblk = (ctx + kBT - 1) / kBT;
  const int b0 = split * p.blocks_per_split;
  const int b1 = min(nblk, b0 + p.blocks_per_split);
  const int ntile = b1 - b0;

  for (int i = tid; i < G * D; i += 128) {
    const int g = i / D, d = i % D;
    qs[g][d] = bf2f(p.q[(long long)b * p.q_stride + (h * G + g) * D + d]);
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();

  const int32_t* trow = p.table + (long long)b * p.max_blocks;
  const long long head_off = ((long long)p.layer * 2 * p.Hkv + h) * PAGE;
  const long long v_off = (long long)p.Hkv * PAGE;
  auto issue = [&](int j) {
    const int slot = j % kStages;
    const long long base = (long long)trow[b0 + j] * p.block_el + head_off;
    mbar_arrive_expect_tx(&bar[slot], 2 * PAGE * 2);
    bulk_g2s(ks[slot], p.pool + base, PAGE * 2, &bar[slot]);
    bulk_g2s(vs[slot], p.pool + base + v_off, PAGE * 2, &bar[slot]);
  };
  if (tid == 0)
    for (int j = 0; j < min(ntile, kStages); ++j) issue(j);

  // score mapping
  const int st = tid >> 3, part = tid & 7;
  // PV mapping
  const int pg = tid / TPH, pd = (tid % TPH) * DPT;
  float m = -INFINITY, l = 0.f;
  float acc[DPT];
#pragma unroll
  for (int i = 0; i < DPT; ++i) acc[i] = 0.f;

  for (int j = 0; j < ntile; ++j) {
    const int slot = j % kStages;
    const int valid = min(kBT, ctx - (b0 + j) * kBT);
    mbar_wait(&bar[slot], (j / kStages) & 1);
    // ---- scores: thread (token st, part) covers chunks part, part+8, ...
    float dot[G];
#pragma unroll
    for (int g = 0; g < G; ++g) dot[g] = 0.f;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int chunk = part + 8 * c;
      float kf[8];
      unpack8(*reinterpret_cast<const uint4*>(&ks[slot][st * D + chunk * 8]), kf);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float4 q0 = *reinterpret_cast<const float4*>(&qs[g][chunk * 8]);
        const float4 q1 = *reinterpret_cast<const float4*>(&qs[g][chunk * 8 + 4]);
        dot[g] += q0.x * kf[0] + q0.y * kf[1] + q0.z * kf[2] + q0.w * kf[3] + q1.x * kf[4] +
                  q1.y * kf[5] + q1.z * kf[6] + q1.w * kf[7];
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      dot[g] += __shfl_xor_sync(0xffffffffu, dot[g], 4);
      dot[g] += __shfl_xor_sync(0xffffffffu, dot[g], 2);
      dot[g] += __shfl_xor_sync(0xffffffffu, dot[g], 1);
    }
    if (part == 0) {
#pragma unroll
      for (int g = 0; g < G; ++g) sc[g][st] = st < valid ? dot[g] * p.scale_log2 : -INFINITY;
    }
    __syncthreads();
    // ---- online softmax + PV for (head pg, dims pd..pd+DPT)
    float mt = m;
    for (int t = 0; t < valid; ++t) mt = fmaxf(mt, sc[pg][t]);
    const float alpha = exp2f(m - mt);
    l *= alpha;
#pragma unroll
    for (int i = 0; i < DPT; ++i) acc[i] *= alpha;
    for (int t = 0; t < valid; ++t) {
      const float pr = exp2f(sc[pg][t] - mt);
      l += pr;
      const bf16* vr = &vs[slot][t * D + pd];
      if constexpr (DPT == 8) {
        float vf[8];
        unpack8(*reinterpret_cast<const uint4*>(vr), vf);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += pr * vf[i];
      } else if constexpr (DPT == 4) {
        const uint2 u = *reinterpret_cast<const uint2*>(vr);
        const float2 a0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
        const float2 a1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
        acc[0] += pr * a0.x; acc[1] += pr * a0.y; acc[2] += pr * a1.x; acc[3] += pr * a1.y;
      } else if constexpr (DPT == 2) {
        const float2 a0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vr));
        acc[0] += pr * a0.x; acc[1] += pr * a0.y;
      } else {
        acc[0] += pr * bf2f(*vr);
      }
    }
    m = mt;
    __syncthreads();  // slot and sc free
    if (tid == 0 && j + kStages < ntile) issue(j + kStages);
  }

  const int hq = h * G + pg;
  if (p.splits == 1) {
    const float inv = l > 0.f ? 1.f / l : 0.f;
    float o[DPT];
#pragma unroll
    for (int i = 0; i < DPT; ++i) o[i] = acc[i] * inv;
    bf16* dst = p.out + ((long long)b * p.Hq + hq) * D + pd;
    if constexpr (DPT == 1) {
      dst[0] = f2bf(o[0]);
    } else {
#pragma unroll
      for (int i = 0; i < DPT; i += 2)
        *reinterpret_cast<__nv_bfloat162*>(dst + i) = __floats2bfloat162_rn(o[i], o[i + 1]);
    }
  } else {
    // Split-K over the context: store this split's normalised partial and
    // log-sum-exp; the last split CTA of (row, kv head) to arrive merges all
    // splits in split order (deterministic) and writes the G output heads.
    __shared__ int s_last;
    const long long row = ((long long)b * p.Hq + hq) * p.splits + split;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    float* dst = p.ws_o + row * D + pd;
#pragma unroll
    for (int i = 0; i < DPT; ++i) __stcg(dst + i, acc[i] * inv);
    if ((tid % TPH) == 0) __stcg(p.ws_lse + row, l > 0.f ? m + log2f(l) : -INFINITY);
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

int decode_splits(int B, int Hkv, int max_blocks, int* bps) {
  // Enough CTAs to cover the SMs, but at least kMinBlocks blocks (8 KiB of
  // K+V per head per block) per CTA so per-CTA fixed costs stay small.
  constexpr int kMinBlocks = 8;
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
  p.blocks_per_split = bps;
  const size_t need = kDecCounterBytes + (size_t)B * Hq * p.splits * (D + 1) * sizeof(float);
  if (p.splits > 1 && (!ws || ws_bytes < need || (size_t)B * Hkv * sizeof(int) > kDecCounterBytes))
    return ASTRAEA_EINVAL;
  p.counters = (int*)ws;
  p.ws_o = (float*)((char*)ws + kDecCounterBytes);
  p.ws_lse = p.ws_o + (size_t)B * Hq * p.splits * D;
  dim3 grid(p.splits, Hkv, B);
  cudaStream_t st = (cudaStream_t)stream;
#define LAUNCH_DEC(DD, GG) ASTRAEA_TRY(launch_k(decode_kernel<DD, GG>, grid, dim3(128), 0, st, p))
  if (D == 128 && G == 4) LAUNCH_DEC(128, 4);
  else if (D == 128 && G == 8) LAUNCH_DEC(128, 8);
  else if (D == 64 && G == 4) LAUNCH_DEC(64, 4);
  else if (D == 64 && G == 8) LAUNCH_DEC(64, 8);
  else if (D == 128 && G == 2) LAUNCH_DEC(128, 2);
  else if (D == 64 && G == 2) LAUNCH_DEC(64, 2);
  else if (D == 128 && G == 1) LAUNCH_DEC(128, 1);
  else return ASTRAEA_EUNSUPPORTED;
#undef LAUNCH_DEC
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
