// tcgen05 / TMEM / TMA building blocks and the fused epilogue program shared
// by the GEMM kernels (gemm.cu) and the decode-step kernel (decode_step.cu).
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace astraea {
namespace tc {

constexpr int kBM = 128;   // MMA M
constexpr int kBK = 64;    // K per stage = one 128-byte swizzle atom of bf16

// ---- PTX wrappers -------------------------------------------------------------------

__device__ __forceinline__ void tma_load_2d(void* smem, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(smem_u32(smem)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 consecutive fp32 columns: thread i of the warp gets row (quarter*32 + i).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x 32 consecutive fp32 columns back into TMEM (the inverse of tmem_ld32).
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  uint32_t r[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(v[i]);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
      "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
      "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row groups of
// 1024 bytes (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc_sw128(const void* p) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;            // start address
  d |= (uint64_t)1 << 16;                  // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;        // SBO
  d |= (uint64_t)1 << 46;                  // version
  d |= (uint64_t)2 << 61;                  // SWIZZLE_128B
  return d;
}

// Instruction descriptor: D=f32, A=B=bf16, both K-major, M=128, N=n.
__host__ __device__ constexpr uint32_t instr_desc(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
}

__device__ __forceinline__ float round_bf(float x) { return bf2f(f2bf(x)); }

__device__ __forceinline__ float silu_rounded(float g) {
  // silu(g) is materialised in bf16 by the reference formulation. Fast
  // division: an IEEE divide takes its slow path whenever exp(-g)
  // overflows (g < -88), ~100 instructions per element.
  return round_bf(__fdividef(g, 1.f + __expf(-g)));
}

// ---- epilogue program --------------------------------------------------------------

struct Epi {
  int kind;
  const bf16* residual;
  float* ssq_out;          // [ceil(N/128)][M]
  const float* ssq_in;     // [parts][M]
  int ssq_parts;
  int rms_dim;
  float eps;
  bf16* pool;
  long long block_el;
  int layer, Hq, Hkv, D, bt;
  const int32_t* pos;
  const int32_t* slots;
  float theta;
  const float2* cs;        // optional [M][D/2] (cos, sin) table
  unsigned long long* amax;  // ARGMAX: [M] packed (value, index) keys
  int amax_off;              // ARGMAX: column offset of this shard
};

// Greedy-sampling key: order-preserving float bits in the high word, the
// complemented column in the low word, so atomicMax picks the largest value
// and, among equal values, the lowest index (torch.argmax's tie rule).
__device__ __forceinline__ unsigned long long argmax_key(float x, int col) {
  const uint32_t b = __float_as_uint(x);
  const uint32_t u = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return ((unsigned long long)u << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)col);
}

__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) {
  return a > b ? a : b;
}

__device__ __forceinline__ unsigned long long warp_max64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = umax64(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// (cos, sin) of token t's rotation for frequency index i (< D/2).
__device__ __forceinline__ float2 rope_cs(const Epi& e, int t, int i) {
  if (e.cs) return e.cs[(long long)t * (e.D / 2) + i];
  float sn, cs;
  sincosf((float)e.pos[t] * (1.0f / powf(e.theta, (float)(2 * i) / (float)e.D)), &sn, &cs);
  return make_float2(cs, sn);
}

__device__ __forceinline__ float rms_scale(const Epi& e, int M, int t) {
  // independent loads in groups of 8 (the sum order stays p = 0, 1, 2, ...)
  float s = 0.f;
  int p = 0;
  for (; p + 8 <= e.ssq_parts; p += 8) {
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldcg(e.ssq_in + (long long)(p + k) * M + t);
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
  }
  for (; p < e.ssq_parts; ++p) s += __ldcg(e.ssq_in + (long long)p * M + t);
  return rsqrtf(s / (float)e.rms_dim + e.eps);
}

// Destination of a rotated/plain head element in QKV_ROPE: q -> C, k/v -> pool.
// slot_pre: token t's pool slot when the caller staged it (>= -1), else -2
__device__ __forceinline__ void qkv_store(const Epi& e, bf16* C, int ldc, int t, int head, int hrow, float y,
                                          int slot_pre = -2) {
  if (head < e.Hq) {
    C[(long long)t * ldc + head * e.D + hrow] = f2bf(y);
    return;
  }
  const int slot = slot_pre >= -1 ? slot_pre : e.slots[t];
  if (slot < 0) return;
  const int kv = head < e.Hq + e.Hkv ? 0 : 1;
  const int h = head - e.Hq - kv * e.Hkv;
  const int blk = e.bt == 16 ? slot >> 4 : slot / e.bt;   // 16-token pages: no integer division
  const int off = e.bt == 16 ? slot & 15 : slot % e.bt;
  bf16* base = e.pool + (long long)blk * e.block_el + ((long long)(e.layer * 2 + kv) * e.Hkv + h) * e.bt * e.D;
  base[(long long)off * e.D + hrow] = f2bf(y);
}

enum { EPI_NONE = 0, EPI_RESIDUAL = 1, EPI_SILU = 2, EPI_QKV_ROPE = 3, EPI_ARGMAX = 4 };

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
  int prev;
  asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], %2;" : "=r"(prev) : "l"(p), "r"(v) : "memory");
  return prev;
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Sums of MT per-lane values over a warp, written to out[0..MT): recursive
// halving -- at each step a lane keeps half of its values and adds its
// partner's copy of them (MT/2 + MT/4 + ... shuffles, then a butterfly over
// the remaining lane bits), 2*MT - 1 + log2(32 / MT) shuffles in all instead
// of 5 * MT. MT: power of two <= 32. v is clobbered.
template <int MT>
__device__ __forceinline__ void warp_multi_sum(float* v, int lane, float* out) {
  int base = 0;
#pragma unroll
  for (int w = MT, o = 16; w > 1; w >>= 1, o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < w / 2; ++i) {
      const float send = up ? v[i] : v[i + w / 2];
      const float keep = up ? v[i + w / 2] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
    if (up) base += w / 2;
  }
#pragma unroll
  for (int o = 16 / MT; o > 0; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
  if ((lane & (32 / MT - 1)) == 0) out[base] = v[0];
}

// Finish one 128-feature tile: thread `row` holds v[t] (t < M) of feature
// tile*128 + row. All 128 epilogue threads call this together. MT (<= BN):
// compile-time bound of the token loops (MT = 1 for a batch of one keeps the
// code executed per tile small -- it runs once per phase, from a cold cache).
template <int BN, typename A, int MT = BN>
__device__ __forceinline__ void sk_finish(const A& a, int tile, int row, float* v, const float* rs,
                                          bf16* xch, float* red, const float* res_pre = nullptr,
                                          const int* slot_s = nullptr, const float2* cs_s = nullptr,
                                          unsigned long long* ftr = nullptr) {
  // ftr (diagnostics, thread row 0 only): [0] exchange written, [1] stores issued
  // slot_s / cs_s (optional): the tokens' pool slots and the [M][D/2] RoPE
  // table staged in shared memory by the caller (QKV_ROPE)
  const Epi& e = a.epi;
  const int M = a.M;
  const int f = tile * kBM + row;
  const bool fok = f < a.N;
  if (e.ssq_in) {
#pragma unroll
    for (int t = 0; t < MT; ++t) v[t] *= rs[t];
  }
  // (as in the QKV path below: pointers and strides into registers before the
  // token loops, so the parameter-space program is not re-read behind the stores)
  bf16* __restrict__ cbase = a.C;
  const long long ldc = a.ldc;
  if (e.kind == EPI_ARGMAX) {
    unsigned long long* __restrict__ amax = e.amax;
    const int col = f + e.amax_off;
#pragma unroll
    for (int t = 0; t < MT; ++t) {
      if (t >= M) break;
      if (cbase && fok) cbase[t * ldc + f] = f2bf(v[t]);
      const unsigned long long k = warp_max64(fok ? argmax_key(v[t], col) : 0ull);
      if ((row & 31) == 0) atomicMax(amax + t, k);
    }
    return;
  }
  if (e.kind == EPI_NONE || e.kind == EPI_RESIDUAL) {
    float sq[BN];
    const bool resid = e.kind == EPI_RESIDUAL;
    const bf16* __restrict__ rbase = e.residual;
#pragma unroll
    for (int t = 0; t < MT; ++t) {
      sq[t] = 0.f;
      if (t < M && fok) {
        float o = v[t];
        if (resid)   // preloaded by the caller, or from L2 (produced by other CTAs)
          o += res_pre ? res_pre[t] : bf2f(__ldcg(rbase + t * ldc + f));
        const bf16 ob = f2bf(o);
        cbase[t * ldc + f] = ob;
        sq[t] = bf2f(ob) * bf2f(ob);
      }
    }
    if (ftr) ftr[0] = gtimer();
    if (e.ssq_out) {
      const int q = row >> 5, lane = row & 31;
      if constexpr (MT <= 32) {
        warp_multi_sum<MT>(sq, lane, red + q * BN);
      } else {
        warp_multi_sum<32>(sq, lane, red + q * BN);
        warp_multi_sum<32>(sq + 32, lane, red + q * BN + 32);
      }
      epi_bar();
      if (row < M) e.ssq_out[(long long)tile * M + row] = red[row] + red[BN + row] + red[2 * BN + row] + red[3 * BN + row];
      epi_bar();
    }
    if (ftr) ftr[1] = gtimer();
    return;
  }
  // pair exchange through shared memory (values rounded to bf16, as the
  // unfused formulation materialises them)
#pragma unroll
  for (int t = 0; t < MT; ++t) xch[t * kBM + row] = f2bf(v[t]);
  epi_bar();
  if (ftr) ftr[0] = gtimer();
  if (e.kind == EPI_SILU) {
    if (row >= 64) {
      const int out_f = tile * 64 + (row - 64);
      if (fok) {
        bf16* __restrict__ cs = cbase + out_f;
#pragma unroll
        for (int t = 0; t < MT; ++t)
          if (t < M)
            cs[t * ldc] = f2bf(silu_rounded(bf2f(xch[t * kBM + row - 64])) * bf2f(xch[t * kBM + row]));
      }
    }
  } else {  // QKV_ROPE
    // Everything the token loop needs is read into registers first: the
    // epilogue program lives in kernel-parameter space and, behind the
    // loop's global stores, the compiler would re-read it every token
    // (0.4 us per token at batch 16 before this).
    const int D = e.D, half = D / 2, Hq = e.Hq, Hkv = e.Hkv;
    const int head = f / D, hrow = f % D;
    const int partner = row ^ half;
    const bool rot = head < Hq + Hkv;
    const int fr = hrow % half;
    // The (cos, sin) source is chosen once, outside the token loops: with a
    // per-token `cs_s ? table : rope_cs()` the compiler may evaluate the
    // sincos/pow fallback speculatively for every token.
    const float2* __restrict__ cst = cs_s ? cs_s : e.cs;
    if (fok && !cst) {
#pragma unroll 1
      for (int t = 0; t < M; ++t) {   // no table at all (not used by the runners): compute in place
        const float x = bf2f(xch[t * kBM + row]);
        float y = x;
        if (rot) {
          const float xp = bf2f(xch[t * kBM + partner]);
          const float2 r = rope_cs(e, t, fr);
          y = hrow < half ? x * r.x - xp * r.y : x * r.x + xp * r.y;
        }
        qkv_store(e, cbase, ldc, t, head, hrow, y, slot_s ? slot_s[t] : -2);
      }
    } else if (fok) {
      if (head < Hq) {
        bf16* __restrict__ cq = cbase + (long long)head * D + hrow;
#pragma unroll 4
        for (int t = 0; t < MT; ++t) {
          if (t >= M) break;
          const float x = bf2f(xch[t * kBM + row]);
          const float xp = bf2f(xch[t * kBM + partner]);
          const float2 r = cst[t * half + fr];
          cq[t * ldc] = f2bf(hrow < half ? x * r.x - xp * r.y : x * r.x + xp * r.y);
        }
      } else {
        const int kv = head < Hq + Hkv ? 0 : 1;
        const int h = head - Hq - kv * Hkv;
        bf16* __restrict__ pool = e.pool;
        const long long bel = e.block_el;
        const int bt = e.bt;
        const long long hoff = ((long long)(e.layer * 2 + kv) * Hkv + h) * bt * D + hrow;
        const int32_t* __restrict__ sl = slot_s ? slot_s : e.slots;   // chosen once (no speculative global load)
#pragma unroll 4
        for (int t = 0; t < MT; ++t) {
          if (t >= M) break;
          const float x = bf2f(xch[t * kBM + row]);
          float y = x;
          if (rot) {
            const float xp = bf2f(xch[t * kBM + partner]);
            const float2 r = cst[t * half + fr];
            y = hrow < half ? x * r.x - xp * r.y : x * r.x + xp * r.y;
          }
          const int slot = sl[t];
          if (slot >= 0) {
            if (bt == 16)   // 16-token pages: no integer division
              pool[(long long)(slot >> 4) * bel + hoff + (long long)(slot & 15) * D] = f2bf(y);
            else
              pool[(long long)(slot / bt) * bel + hoff + (long long)(slot % bt) * D] = f2bf(y);
          }
        }
      }
    }
  }
  if (ftr) ftr[1] = gtimer();
  epi_bar();
}

// 2-D bf16 tensor [rows][cols] (row stride ld elements) -> TMA descriptor with a
// box of kBK cols x box_rows rows, 128B swizzle (cached by (ptr, shape, box)).
int make_map(CUtensorMap* out, const void* ptr, long long rows, long long cols, long long ld, int box_rows);

}  // namespace tc
}  // namespace astraea
