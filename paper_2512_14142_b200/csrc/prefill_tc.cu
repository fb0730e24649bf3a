// K7 on the 5th-generation tensor cores: paged flash-attention prefill of
// the recompute-on-resume segment (the reference's prefill_seconds(n_in +
// extra), simulator.py:329-337; PrefillProfile, predictor.py:47-57).
//
// One CTA per (tile of 128 / G query tokens, kv head, sequence); the G q
// heads of the kv head are the 128 MMA rows (row = g * QT + t), so every
// staged K/V page serves the whole GQA group and short appends (n_in 32..512
// onto a resident context) still fill the M = 128 rows. Per KV tile of 128
// tokens (8 pages):
//   warp 0   TMA producer: the pages' K and V boxes (16 rows x 64 cols, 128B
//            swizzle) from the pool viewed as [blocks x L x 2 x Hkv x 16][D]
//            into a 2-stage ring (block ids from the table; pages past the
//            context re-load the last page -- finite data, masked);
//   warp 1   MMA issuer (one thread): S_j = Q K_j^T into one of two TMEM
//            score buffers (tcgen05.mma kind::f16, both operands K-major in
//            shared memory), then O += P_j V_j into the TMEM accumulator (P
//            K-major in shared memory, V MN-major: the page rows are tokens);
//            S_{j+1} is issued before P_j is ready, so the tensor pipe runs
//            the next scores while the softmax warps work;
//   warps 2-5  softmax, one thread per row: tcgen05.ld of the row's 128
//            scores, causal mask on absolute positions, online softmax in the
//            exp2 domain with a lazy reference max (O and l are rescaled only
//            when the row max grows by more than 2^8 -- exact, the final
//            normalisation uses the same reference), P as bf16 into shared
//            memory; at the end O / l from TMEM to global.
// Accumulation is fp32 (TMEM); P is rounded to bf16 for the PV MMA as in the
// mma.sync kernel it replaces.
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "tc.cuh"

using namespace astraea;
using namespace astraea::tc;

namespace {

constexpr int kPT = 16;         // tokens per page (block)
constexpr int kKT = 128;        // KV tokens per tile
constexpr int kThreads = 192;

struct TcPrefillParams {
  const bf16* q;
  const int32_t* cu_q;
  const int32_t* table;
  const int32_t* ctx;
  bf16* out;
  long long q_stride;
  int layer, Hkv, Hq, G, QT, max_blocks, block_rows;
  float scale_log2;
  unsigned long long* trace;   // diagnostics: [grid][16] %globaltimer stamps, or NULL
};

unsigned long long* g_ptrace = nullptr;

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// MN-major operand, 128-byte swizzle: LBO = stride between 64-element atoms
// along MN, SBO = stride between 8-row groups along K.
__device__ __forceinline__ uint64_t smem_desc_mn_sw128(const void* p, uint32_t lbo, uint32_t sbo) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// 32 lanes x 32 columns without waiting (tcgen05.ld is asynchronous until
// tcgen05.wait::ld); tmem_wait32 waits and ties the registers to the wait so
// no use is scheduled before it.
__device__ __forceinline__ void tmem_ld32_async(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait32(uint32_t* r) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}

// One non-blocking probe of an mbarrier phase (true: the phase completed).
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 16-byte chunk c of row r in a [128 rows][64 cols] K-major 128B-swizzled region
__device__ __forceinline__ uint32_t swz_off(int r, int c) { return (uint32_t)(r * 128 + (((c & 7) ^ (r & 7)) << 4)); }

template <int D>
struct TcLayout {
  static constexpr int REG = 128 * 128;                 // one [128 rows][64 cols] bf16 region (16 KB)
  static constexpr int NH = D / 64;                     // 64-column halves of the head dim
  static constexpr int Q = 0;                           // [NH] regions
  static constexpr int KV = NH * REG;                   // 2 stages x (K [NH] + V [NH]) regions
  static constexpr int STAGE = 2 * NH * REG;
  static constexpr int P = KV + 2 * STAGE;              // 2 buffers x 2 regions (tokens 0-63, 64-127)
  static constexpr int PBUF = 2 * REG;
  static constexpr int BAR = P + 2 * PBUF;
  static constexpr int SMEM = BAR + 256 + 1024;         // + barriers, TMEM slot, alignment
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1) prefill_tc_kernel(const __grid_constant__ CUtensorMap pool_map,
                                                                 const __grid_constant__ TcPrefillParams p) {
  using Lay = TcLayout<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Lay::BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;    // [2]
  uint64_t* kv_empty = bars + 3;   // [2]
  uint64_t* s_full = bars + 5;     // [2] per score buffer
  uint64_t* p_full = bars + 7;     // [2] per P buffer
  uint64_t* pv_done = bars + 9;    // [2] per P buffer
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 11);

  const int s = blockIdx.z, h = blockIdx.y;
  const int qt = gridDim.x - 1 - blockIdx.x;   // heaviest (latest) query tiles first
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* tr =
      p.trace ? p.trace + ((long long)(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 16 : nullptr;
  // tr: [0] entry [1] MMA warp saw Q [2] first scores seen [3] tiles [4] last P published [5] last PV seen
  //     [6] output written [7] exit [8] first KV tile issued [9] last KV tile issued
  if (tr && threadIdx.x == 0) tr[0] = gtime();
  pdl_wait();
  const int q_begin = p.cu_q[s], len = p.cu_q[s + 1] - q_begin;
  const int QT = p.QT;
  const int row0 = qt * QT;
  if (row0 >= len) {
    pdl_launch();
    return;
  }
  const int rows = min(QT, len - row0);
  const int ctx = p.ctx[s];
  const int pos0 = ctx - len;                  // absolute position of the sequence's first query
  const int kv_end = pos0 + row0 + rows;       // keys this tile needs: [0, kv_end)
  const int ntiles = (kv_end + kKT - 1) / kKT;

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&pool_map) : "memory");
    mbar_init(q_full, 128);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&pv_done[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_launch();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t kSCol = 0, kOCol = 256;   // S buffers at columns 0 / 128, O at 256

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer: KV tile j = pages 8j .. 8j+7 into stage j % 2
      const int32_t* trow = p.table + (long long)s * p.max_blocks;
      const int last_page = (kv_end - 1) / kPT;
      const int k_row0 = (p.layer * 2 * p.Hkv + h) * kPT, v_row0 = k_row0 + p.Hkv * kPT;
      if (tr) tr[3] = (unsigned long long)ntiles;
      for (int j = 0; j < ntiles; ++j) {
        const int st = j & 1;
        if (j >= 2) mbar_wait(&kv_empty[st], ((j >> 1) - 1) & 1);
        if (tr && (j == 0 || j == ntiles - 1)) tr[j == 0 ? 8 : 9] = gtime();
        if (tr && j == 4) tr[10] = gtime();   // tile 4 issued (stage free)
        uint8_t* kb = sm + Lay::KV + st * Lay::STAGE;
        uint8_t* vb = kb + Lay::NH * Lay::REG;
        mbar_arrive_expect_tx(&kv_full[st], (uint32_t)(2 * kKT * D * 2));
#pragma unroll 1
        for (int pg = 0; pg < kKT / kPT; ++pg) {
          const int page = min(j * (kKT / kPT) + pg, last_page);
          const int blk = __ldg(trow + page);
          const int kr = blk * p.block_rows + k_row0, vr = blk * p.block_rows + v_row0;
#pragma unroll
          for (int hf = 0; hf < Lay::NH; ++hf) {
            tma_load_2d(kb + hf * Lay::REG + pg * kPT * 128, &pool_map, &kv_full[st], hf * 64, kr);
            tma_load_2d(vb + hf * Lay::REG + pg * kPT * 128, &pool_map, &kv_full[st], hf * 64, vr);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer
    constexpr uint32_t idesc_s = instr_desc(kKT);                 // M 128, N 128, both K-major
    constexpr uint32_t idesc_pv = instr_desc(D) | (1u << 16);     // B (V) MN-major
    mbar_wait(q_full, 0);
    tc_fence_after();
    if (tr && lane == 0) tr[1] = gtime();
    auto issue_s = [&](int j) {
      const int st = j & 1;
      mbar_wait(&kv_full[st], (j >> 1) & 1);   // returns at once when the caller saw it land
      tc_fence_after();
      if (tr && j == 4 && lane == 0) tr[11] = gtime();   // tile 4 landed
      if (lane == 0) {
        const uint8_t* kb = sm + Lay::KV + st * Lay::STAGE;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t da = smem_desc_sw128(sm + Lay::Q + (kk / 4) * Lay::REG) + 2 * (kk % 4);
          const uint64_t db = smem_desc_sw128(kb + (kk / 4) * Lay::REG) + 2 * (kk % 4);
          mma_bf16(tmem + kSCol + st * kKT, da, db, idesc_s, kk > 0 ? 1u : 0u);
        }
        mma_commit(&s_full[st]);
      }
      __syncwarp();
    };
    issue_s(0);
    for (int j = 0; j < ntiles; ++j) {
      // S(j+1) and PV(j) in whichever order their inputs arrive (the next
      // KV tile or the softmax's P), so a late tile never holds up PV(j)
      const int pb = j & 1;
      bool s_next = j + 1 >= ntiles;
      for (;;) {
        if (!s_next && mbar_test(&kv_full[(j + 1) & 1], ((j + 1) >> 1) & 1)) {
          issue_s(j + 1);
          s_next = true;
        }
        if (mbar_test(&p_full[pb], (j >> 1) & 1)) break;
      }
      tc_fence_after();
      if (tr && j == 4 && lane == 0) tr[14] = gtime();   // P(4) seen by the MMA warp
      if (lane == 0) {
        const uint8_t* vb = sm + Lay::KV + (j & 1) * Lay::STAGE + Lay::NH * Lay::REG;
        const uint8_t* pbuf = sm + Lay::P + pb * Lay::PBUF;
#pragma unroll
        for (int kk = 0; kk < kKT / 16; ++kk) {
          const uint64_t da = smem_desc_sw128(pbuf + (kk / 4) * Lay::REG) + 2 * (kk % 4);
          const uint64_t db = smem_desc_mn_sw128(vb + kk * 16 * 128, Lay::REG, 1024);
          mma_bf16(tmem + kOCol, da, db, idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&pv_done[pb]);
        mma_commit(&kv_empty[j & 1]);
      }
      __syncwarp();
      if (!s_next) issue_s(j + 1);
    }
  } else {
    // ---- softmax warps: thread = row r (TMEM lane r)
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
    const int g = r / QT, t = r % QT;
    const bool valid = t < rows && g < p.G;
    // Q row -> shared memory (K-major, 128B swizzle; zero rows past the tile)
    {
      const bf16* src = p.q + (long long)(q_begin + row0 + t) * p.q_stride + (long long)(h * p.G + g) * D;
#pragma unroll
      for (int c = 0; c < D / 8; ++c) {
        const uint4 v = valid ? __ldg(reinterpret_cast<const uint4*>(src) + c) : make_uint4(0u, 0u, 0u, 0u);
        *reinterpret_cast<uint4*>(sm + Lay::Q + (c / 8) * Lay::REG + swz_off(r, c)) = v;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(q_full);
    }
    const int qp = pos0 + row0 + t;                        // this row's absolute position
    const int lim = valid ? qp : kv_end - 1;               // keys kt <= lim are visible
    const float c2 = p.scale_log2;
    float m_ref = -INFINITY, l = 0.f;
    for (int j = 0; j < ntiles; ++j) {
      const int st = j & 1;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      if (tr && j == 0 && threadIdx.x == 64) tr[2] = gtime();
      if (tr && j == 4 && threadIdx.x == 64) tr[12] = gtime();   // S(4) seen by softmax
      const uint32_t scol = lane_addr + kSCol + st * kKT;
      const int kt0 = j * kKT;
      // the row's 128 scores: four loads in flight, one wait
      uint32_t sv[kKT];
#pragma unroll
      for (int c = 0; c < kKT / 32; ++c) tmem_ld32_async(scol + c * 32, sv + c * 32);
#pragma unroll
      for (int c = 0; c < kKT / 32; ++c) tmem_wait32(sv + c * 32);
      const int nvis = min(kKT, lim - kt0 + 1);          // keys kt0 .. kt0 + nvis - 1 are visible
      float mt = -INFINITY;
#pragma unroll
      for (int i = 0; i < kKT; ++i)
        if (i < nvis) mt = fmaxf(mt, __uint_as_float(sv[i]));
      // lazy reference max: move it (and rescale O, l) only for growth > 2^8
      float alpha = 1.f;
      bool resc = false;
      if (mt > m_ref && (m_ref == -INFINITY || (mt - m_ref) * c2 > 8.f)) {
        alpha = m_ref == -INFINITY ? 0.f : ex2((m_ref - mt) * c2);
        m_ref = mt;
        resc = j > 0;
      }
      const float mo = m_ref * c2;
      // P buffer j & 1 is free once PV(j-2) is done; a rescale of O needs
      // every earlier PV done (PV(j-1) completes after PV(j-2): in order)
      const int pb = j & 1;
      const bool any_resc = __any_sync(0xffffffffu, resc);
      if (any_resc) {
        mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
        tc_fence_after();
      } else if (j >= 2) {
        mbar_wait(&pv_done[pb], ((j >> 1) - 1) & 1);
      }
      if (j > 0) {
        if (any_resc) {
          const float a = resc ? alpha : 1.f;
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            float v[32];
            tmem_ld32(lane_addr + kOCol + c * 32, v);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] *= a;
            tmem_st32(lane_addr + kOCol + c * 32, v);
          }
        }
      }
      // P = exp2(s * c - m_ref * c) as bf16 -> shared memory (K-major: tokens
      // 0-63 | 64-127, 128B swizzle); the row sum of the rounded values
      float sum0 = 0.f, sum1 = 0.f;
      uint8_t* prow = sm + Lay::P + pb * Lay::PBUF;
      if (nvis >= kKT) {   // every key of the tile visible (all but the diagonal tiles)
#pragma unroll
        for (int c = 0; c < kKT / 8; ++c) {
          uint32_t w[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int i = 8 * c + 2 * k;
            const float p0 = ex2(fmaf(__uint_as_float(sv[i]), c2, -mo));
            const float p1 = ex2(fmaf(__uint_as_float(sv[i + 1]), c2, -mo));
            sum0 += p0;
            sum1 += p1;
            const __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
            w[k] = *reinterpret_cast<const uint32_t*>(&b2);
          }
          *reinterpret_cast<uint4*>(prow + (c / 8) * Lay::REG + swz_off(r, c)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < kKT / 8; ++c) {
          uint32_t w[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int i = 8 * c + 2 * k;
            const float p0 = i < nvis ? ex2(fmaf(__uint_as_float(sv[i]), c2, -mo)) : 0.f;
            const float p1 = i + 1 < nvis ? ex2(fmaf(__uint_as_float(sv[i + 1]), c2, -mo)) : 0.f;
            sum0 += p0;
            sum1 += p1;
            const __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
            w[k] = *reinterpret_cast<const uint32_t*>(&b2);
          }
          *reinterpret_cast<uint4*>(prow + (c / 8) * Lay::REG + swz_off(r, c)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
      const float sum = sum0 + sum1;
      l = l * alpha + sum;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      mbar_arrive(&p_full[pb]);
      if (tr && j == ntiles - 1 && threadIdx.x == 64) tr[4] = gtime();
      if (tr && j == 4 && threadIdx.x == 64) tr[13] = gtime();   // P(4) published
    }
    // O / l -> global
    mbar_wait(&pv_done[(ntiles - 1) & 1], ((ntiles - 1) >> 1) & 1);
    tc_fence_after();
    if (tr && threadIdx.x == 64) tr[5] = gtime();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    bf16* dst = p.out + (long long)(q_begin + row0 + t) * p.Hq * D + (long long)(h * p.G + g) * D;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      float v[32];
      tmem_ld32(lane_addr + kOCol + c * 32, v);
      if (valid) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          float f[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) f[k] = v[i + k] * inv;
          *reinterpret_cast<uint4*>(dst + c * 32 + i) = pack8(f);
        }
      }
    }
  }
  if (tr && threadIdx.x == 64) tr[6] = gtime();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
  if (tr && threadIdx.x == 0) tr[7] = gtime();
}

}  // namespace

namespace astraea {

// Launch the tcgen05 prefill for a kv geometry; ASTRAEA_EUNSUPPORTED when
// the shape is not covered (head_dim 64 / 128, G | 128, G <= 8).
int prefill_tc_launch(const astraea_kv_geometry* g, const void* pool, int32_t layer, const void* q, int32_t q_stride,
                      const int32_t* cu_q, int32_t S, int32_t max_q_len, int32_t Hq, const int32_t* table,
                      int32_t max_blocks, const int32_t* ctx, float scale, void* out, cudaStream_t st) {
  const int D = g->head_dim, Hkv = g->num_kv_heads, G = Hq / Hkv;
  if ((D != 64 && D != 128) || G < 1 || G > 8 || (128 % G) || g->block_tokens != kPT) return ASTRAEA_EUNSUPPORTED;
  TcPrefillParams p;
  p.q = (const bf16*)q;
  p.cu_q = cu_q;
  p.table = table;
  p.ctx = ctx;
  p.out = (bf16*)out;
  p.q_stride = q_stride;
  p.layer = layer;
  p.Hkv = Hkv;
  p.Hq = Hq;
  p.G = G;
  p.QT = 128 / G;
  p.max_blocks = max_blocks;
  p.block_rows = g->num_layers * 2 * Hkv * kPT;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.trace = g_ptrace;
  CUtensorMap map;
  int rc = tc::make_map(&map, pool, (long long)g->num_blocks * p.block_rows, D, D, kPT);
  if (rc) return rc;
  dim3 grid((max_q_len + p.QT - 1) / p.QT, Hkv, S);
  if (D == 128) {
    constexpr size_t smem = TcLayout<128>::SMEM;
    static bool attr = false;
    if (!attr) {
      ASTRAEA_TRY(cudaFuncSetAttribute(prefill_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr = true;
    }
    ASTRAEA_TRY(launch_k(prefill_tc_kernel<128>, grid, dim3(kThreads), smem, st, map, p));
  } else {
    constexpr size_t smem = TcLayout<64>::SMEM;
    static bool attr = false;
    if (!attr) {
      ASTRAEA_TRY(cudaFuncSetAttribute(prefill_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr = true;
    }
    ASTRAEA_TRY(launch_k(prefill_tc_kernel<64>, grid, dim3(kThreads), smem, st, map, p));
  }
  ASTRAEA_CHECK_LAUNCH();
  return ASTRAEA_OK;
}

}  // namespace astraea

extern "C" int astraea_debug_prefill_trace(void* buf) {
  g_ptrace = (unsigned long long*)buf;
  return ASTRAEA_OK;
}
