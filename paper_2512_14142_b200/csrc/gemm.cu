// K6 / K9: bf16 GEMM on 5th-generation tensor cores (tcgen05 + TMEM + TMA),
// with the Llama block's elementwise work fused into the epilogue.
//
//   C[M][N] = epilogue( A[M][K] . W[N][K]^T )
//
// These are the dense projections of the recompute-on-resume prefill and of
// every decode step -- the work the reference reduces to the profile lookup
// prefill_seconds(n_in + extra) and n_gen * seconds_per_token
// (pkg/src/agentsched/predictor.py:47-66, simulator.py:329-337).
//
// Kernel anatomy (192 threads):
//   warp 0      TMA producer: 128B-swizzled A/B tiles into a smem ring
//               (cp.async.bulk.tensor.2d, mbarrier complete_tx); weight tiles
//               of the first stages are fetched before griddepcontrol.wait,
//               i.e. while the previous kernel drains (PDL);
//   warp 1      allocates TMEM; one elected lane issues tcgen05.mma
//               (kind::f16, M=128, fp32 accumulators in TMEM) and commits
//               each stage back to the producer with tcgen05.commit;
//   warps 2..5  epilogue: tcgen05.ld 32x32b -> registers -> fused epilogue.
//
// Orientations:
//   kRows  (prefill, M > 64): MMA M axis = 128 rows of A (tokens), N axis =
//          128/256 rows of W, one output tile per CTA.
//   stream-K (decode, M <= 64): MMA M axis = 128 rows of W (output features),
//          N axis = the M tokens padded to 16/32/64 ("swap AB"); persistent,
//          one CTA per SM, deterministic split-tile fix-up.
//
// Epilogue programs (astraea_epilogue.kind):
//   NONE       C = acc
//   RESIDUAL   C = acc + residual (may alias C); optionally emits per-128-
//              column sums of squares of the bf16 output (the next RMSNorm's
//              statistics, so the norm itself never runs as a kernel)
//   SILU       W rows interleaved as [64 gate | 64 up] per 128: C = silu(g)*u
//   QKV_ROPE   N = (Hq + 2 Hkv) D: RoPE on q and k, q -> C, k/v -> KV pool slots
// plus, for any program, input RMS scaling: acc[t][:] *= rsqrt(ssq_t/d + eps)
// with the norm weight folded into W offline (x*w @ W^T == x @ (W diag w)^T).
#include <cuda.h>

#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "tc.cuh"
#include "attn_mma.cuh"


using namespace astraea;
using namespace astraea::tc;

namespace {

constexpr int kThreads = 192;
constexpr int kMaxPhases = 8;   // GEMMs per chain launch (two layers)
constexpr int kMaxAttn = 2;     // attention phases per chain launch

struct GemmArgs {
  bf16* C;
  int M, N, K, ldc;
  Epi epi;
  // CTA-pair kernel split-K (splits > 1 only when tiles * splits <= pairs):
  int splits;
  unsigned long long* part;    // [tiles][splits - 1][2 CTAs][128][256] tagged fp32 partials
  int* ctr;                    // workspace counters: [kMaxPhases] exit, [kMaxPhases + 1] launch epoch
  // one-CTA kernel split-K (short prefills): K cut into gridDim.z ranges
  float* rpart;                // [tiles][splits][128][BN] fp32 partials
  int* rctr;                   // [tiles] arrival counters (zero between uses)
  unsigned long long* trace;   // diagnostics (astraea_debug_gemm_trace): 16 words per CTA, or null
  int trace_ctas;
};

// Epilogue of one 128-row x BN-column accumulator tile: thread = token row m
// (mok: m < M), TMEM columns at lane_addr (this warp's 32 lanes), output
// columns n_tile * BN ... (+BN). Shared by the one-CTA and the CTA-pair kernel.
struct NoFix {
  __device__ __forceinline__ void operator()(float*, int) const {}
};

template <int BN, class Fix = NoFix>
__device__ __forceinline__ void rows_epilogue(const GemmArgs& args, int m, bool mok, float rs, uint32_t lane_addr,
                                              int tile_b, const Fix& fix = Fix()) {
  const Epi& e = args.epi;
    bf16* crow = args.C + (long long)m * args.ldc;
#pragma unroll 1
  for (int g = 0; g < BN / 128; ++g) {
    const int n_group = tile_b * BN + g * 128;    // first output column of the 128-group
    if (e.kind == EPI_SILU || e.kind == EPI_QKV_ROPE) {
      const int pair = (e.kind == EPI_SILU || e.D == 128) ? 2 : 1;   // chunk distance of a pair
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        if ((c / pair) % 2) continue;                 // c is the low half of its pair
        float lo[32], hi[32];
        tmem_ld32(lane_addr + g * 128 + c * 32, lo);
        tmem_ld32(lane_addr + g * 128 + (c + pair) * 32, hi);
        fix(lo, g * 128 + c * 32);
        fix(hi, g * 128 + (c + pair) * 32);
        if (!mok || n_group >= args.N) continue;
        if (e.kind == EPI_SILU) {
          const int f0 = (n_group / 128) * 64 + c * 32;   // output feature of lo[0]
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            float o[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
              o[q] = silu_rounded(round_bf(lo[j + q] * rs)) * round_bf(hi[j + q] * rs);
            *reinterpret_cast<uint4*>(crow + f0 + j) = pack8(o);
          }
        } else {
          // 32 consecutive columns of one head: low half hrow0.., high half +D/2
          const int col0 = n_group + c * 32;
          const int head = col0 / e.D, hrow0 = col0 % e.D;
          const bool rot = head < e.Hq + e.Hkv;
          float ylo[32], yhi[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float x0 = round_bf(lo[j] * rs), x1 = round_bf(hi[j] * rs);
            if (rot) {
              const float2 r = rope_cs(e, m, hrow0 + j);
              ylo[j] = x0 * r.x - x1 * r.y;
              yhi[j] = x1 * r.x + x0 * r.y;
            } else {
              ylo[j] = x0;
              yhi[j] = x1;
            }
          }
          bf16* dst = nullptr;
          long long half_stride = e.D / 2;
          if (head < e.Hq) {
            dst = args.C + (long long)m * args.ldc + head * e.D + hrow0;
          } else if (e.slots[m] >= 0) {
            const int slot = e.slots[m];
            const int kv = head < e.Hq + e.Hkv ? 0 : 1;
            const int hk = head - e.Hq - kv * e.Hkv;
            dst = e.pool + (long long)(slot / e.bt) * e.block_el +
                  ((long long)(e.layer * 2 + kv) * e.Hkv + hk) * e.bt * e.D + (long long)(slot % e.bt) * e.D + hrow0;
          }
          if (dst) {
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
              *reinterpret_cast<uint4*>(dst + j) = pack8(ylo + j);
              *reinterpret_cast<uint4*>(dst + half_stride + j) = pack8(yhi + j);
            }
          }
        }
      }
      continue;
    }
    if (e.kind == EPI_ARGMAX) {
      unsigned long long best = 0ull;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float v[32];
        tmem_ld32(lane_addr + g * 128 + c * 32, v);
        fix(v, g * 128 + c * 32);
        const int n0 = n_group + c * 32;
        if (!mok) continue;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          if (n0 + k < args.N) {
            const float o = v[k] * rs;
            if (args.C) crow[n0 + k] = f2bf(o);
            best = umax64(best, argmax_key(o, n0 + k + e.amax_off));
          }
        }
      }
      if (mok) atomicMax(e.amax + m, best);
      continue;
    }
    float ssq = 0.f;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      float v[32];
      tmem_ld32(lane_addr + g * 128 + c * 32, v);
      fix(v, g * 128 + c * 32);
      const int n0 = n_group + c * 32;
      if (!mok || n0 >= args.N) continue;
      bf16* dst = crow + n0;
      const bf16* res = e.kind == EPI_RESIDUAL ? e.residual + (long long)m * args.ldc + n0 : nullptr;
      if (n0 + 32 <= args.N) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float o[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) o[k] = v[q * 8 + k] * rs;
          if (res) {
            float r[8];
            unpack8(*reinterpret_cast<const uint4*>(res + q * 8), r);
#pragma unroll
            for (int k = 0; k < 8; ++k) o[k] += r[k];
          }
          const uint4 packed = pack8(o);
          *reinterpret_cast<uint4*>(dst + q * 8) = packed;
          float ob[8];
          unpack8(packed, ob);
#pragma unroll
          for (int k = 0; k < 8; ++k) ssq += ob[k] * ob[k];
        }
      } else {
        for (int k = 0; k < 32 && n0 + k < args.N; ++k) {
          float o = v[k] * rs;
          if (res) o += bf2f(res[k]);
          const bf16 ob = f2bf(o);
          dst[k] = ob;
          ssq += bf2f(ob) * bf2f(ob);
        }
      }
    }
    if (e.ssq_out && mok && n_group < args.N) e.ssq_out[(long long)(n_group / 128) * args.M + m] = ssq;
  }
}

// The one-CTA kernel's epilogue staged through shared memory (the drained
// stage ring): each thread still owns one token row of the accumulator, but
// every global access is made by the 128 epilogue threads together, a row of
// 16-byte chunks per 16 (or 8) consecutive lanes -- a thread-per-row global
// access touches 32 rows (32 L2 transactions) per instruction, which made
// the epilogue of a 128 x 128 tile cost more than its main loop
// (tools/rows_trace.py). Chunk j of row r lives at r * CH + (j ^ (r & 7)):
// conflict-free for both the per-row and the per-chunk walks.
// Same arithmetic, same order as rows_epilogue (bit-identical results).
template <int CH>
__device__ __forceinline__ int swz(int r, int j) {
  return r * CH + (j ^ (r & 7));
}

template <int BN>
__device__ __forceinline__ void rows_epilogue_staged(const GemmArgs& args, int tile_a, int tile_b, int row, float rs,
                                                     uint32_t lane_addr, uint8_t* stage,
                                                     unsigned long long* tr = nullptr) {
  const Epi& e = args.epi;
  const int et = threadIdx.x - 64;   // 0..127: cooperative index
  const int m = tile_a * kBM + row;
  const bool mok = m < args.M;
  uint4* ob = reinterpret_cast<uint4*>(stage);               // [128][16] chunks: one 128-column group
  uint4* cs4 = reinterpret_cast<uint4*>(stage + 32768);      // QKV: [128][D/4] chunks of (cos, sin) pairs
  int* sl = reinterpret_cast<int*>(stage + 32768 + 65536);   // QKV: [128] pool slots
  const bool qkv = e.kind == EPI_QKV_ROPE;
  if (qkv) {
    const int chq = e.D / 4;   // 16-byte chunks per row of the table: D/2 float2
    if (et < kBM) sl[et] = (tile_a * kBM + et < args.M) ? e.slots[tile_a * kBM + et] : -1;
    // the (cos, sin) pairs of the tile's 128 tokens, staged with batches of
    // 16 independent loads per thread (a dependent load per iteration would
    // serialise 32 L2 round trips). Recomputing them per element instead
    // (IEEE sincosf) measured slower: QKV 34.6 -> 36.1 us at 128 tokens.
#pragma unroll 1
    for (int i0 = 0; i0 < kBM * chq; i0 += 16 * kBM) {
      uint4 v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int i = i0 + k * kBM + et, r = i / chq, j = i % chq, mm = tile_a * kBM + r;
        v[k] = make_uint4(0, 0, 0, 0);
        if (i < kBM * chq && mm < args.M) {
          if (e.cs) {
            v[k] = __ldg(reinterpret_cast<const uint4*>(e.cs + (long long)mm * (e.D / 2)) + j);
          } else {
            const float2 a = rope_cs(e, mm, 2 * j), b = rope_cs(e, mm, 2 * j + 1);
            v[k] = make_uint4(__float_as_uint(a.x), __float_as_uint(a.y), __float_as_uint(b.x), __float_as_uint(b.y));
          }
        }
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int i = i0 + k * kBM + et, r = i / chq, j = i % chq;
        if (i < kBM * chq) cs4[r * chq + (j ^ (r & 7))] = v[k];
      }
    }
  }
#pragma unroll 1
  for (int g = 0; g < BN / 128; ++g) {
    const int n_group = tile_b * BN + g * 128;
    if (n_group >= args.N) break;
    if (g) epi_bar();   // the previous group's stores have left the buffer
    if (tr && g == 0 && et == 0) tr[12] = gtimer();
    if (e.kind == EPI_SILU) {
      // gate chunk c pairs with up chunk c + 2: 64 output columns, 8 chunks
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        float lo[32], hi[32];
        tmem_ld32(lane_addr + g * 128 + c * 32, lo);
        tmem_ld32(lane_addr + g * 128 + (c + 2) * 32, hi);
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          float o[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) o[q] = silu_rounded(round_bf(lo[j + q] * rs)) * round_bf(hi[j + q] * rs);
          ob[swz<8>(row, c * 4 + j / 8)] = pack8(o);
        }
      }
      if (tr && g == 0 && et == 0) tr[13] = gtimer();
      epi_bar();
      if (tr && g == 0 && et == 0) tr[14] = gtimer();
      const int f0 = (n_group / 128) * 64;
      for (int i = et; i < kBM * 8; i += kBM) {
        const int r = i >> 3, j = i & 7, mm = tile_a * kBM + r;
        if (mm < args.M) *reinterpret_cast<uint4*>(args.C + (long long)mm * args.ldc + f0 + j * 8) = ob[swz<8>(r, j)];
      }
      continue;
    }
    if (qkv) {
      const int pair = e.D == 128 ? 2 : 1;
      const int chq = e.D / 4;
      if (g == 0) epi_bar();   // table and slots staged
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        if ((c / pair) % 2) continue;
        float lo[32], hi[32];
        tmem_ld32(lane_addr + g * 128 + c * 32, lo);
        tmem_ld32(lane_addr + g * 128 + (c + pair) * 32, hi);
        const int col0 = n_group + c * 32;
        const int head = col0 / e.D, hrow0 = col0 % e.D;
        const bool rot = head < e.Hq + e.Hkv;
        float ylo[32], yhi[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float x0 = round_bf(lo[j] * rs), x1 = round_bf(hi[j] * rs);
          if (rot) {
            const int fi = hrow0 + j;
            const float* cj = reinterpret_cast<const float*>(cs4 + row * chq + ((fi >> 1) ^ (row & 7)));
            const float2 r = make_float2(cj[(fi & 1) * 2], cj[(fi & 1) * 2 + 1]);
            ylo[j] = x0 * r.x - x1 * r.y;
            yhi[j] = x1 * r.x + x0 * r.y;
          } else {
            ylo[j] = x0;
            yhi[j] = x1;
          }
        }
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          ob[swz<16>(row, c * 4 + j / 8)] = pack8(ylo + j);
          ob[swz<16>(row, (c + pair) * 4 + j / 8)] = pack8(yhi + j);
        }
      }
      if (tr && g == 0 && et == 0) tr[13] = gtimer();
      epi_bar();
      if (tr && g == 0 && et == 0) tr[14] = gtimer();
      for (int i = et; i < kBM * 16; i += kBM) {
        const int r = i >> 4, j = i & 15, mm = tile_a * kBM + r;
        const int col = n_group + j * 8;
        if (mm >= args.M || col >= args.N) continue;
        const int head = col / e.D, hrow = col % e.D;
        bf16* dst;
        if (head < e.Hq) {
          dst = args.C + (long long)mm * args.ldc + col;
        } else {
          const int slot = sl[r];
          if (slot < 0) continue;
          const int kv = head < e.Hq + e.Hkv ? 0 : 1;
          const int hk = head - e.Hq - kv * e.Hkv;
          dst = e.pool + (long long)(slot / e.bt) * e.block_el +
                ((long long)(e.layer * 2 + kv) * e.Hkv + hk) * e.bt * e.D + (long long)(slot % e.bt) * e.D + hrow;
        }
        *reinterpret_cast<uint4*>(dst) = ob[swz<16>(r, j)];
      }
      continue;
    }
    // NONE / RESIDUAL (+ sums of squares of the bf16 output)
    const bool resid = e.kind == EPI_RESIDUAL;
    if (resid) {
      uint4 v[16];   // all 16 loads in flight before the first use
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int i = k * kBM + et, r = i >> 4, j = i & 15, mm = tile_a * kBM + r;
        const int col = n_group + j * 8;
        v[k] = (mm < args.M && col < args.N)
                   ? __ldcg(reinterpret_cast<const uint4*>(e.residual + (long long)mm * args.ldc + col))
                   : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int i = k * kBM + et;
        ob[swz<16>(i >> 4, i & 15)] = v[k];
      }
      epi_bar();
    }
    float ssq = 0.f;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      float v[32];
      tmem_ld32(lane_addr + g * 128 + c * 32, v);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = c * 4 + q;
        if (n_group + j * 8 >= args.N) continue;
        float o[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] = v[q * 8 + k] * rs;
        if (resid) {
          float r[8];
          unpack8(ob[swz<16>(row, j)], r);
#pragma unroll
          for (int k = 0; k < 8; ++k) o[k] += r[k];
        }
        const uint4 packed = pack8(o);
        ob[swz<16>(row, j)] = packed;
        float obf[8];
        unpack8(packed, obf);
#pragma unroll
        for (int k = 0; k < 8; ++k) ssq += obf[k] * obf[k];
      }
    }
    if (e.ssq_out && mok) e.ssq_out[(long long)(n_group / 128) * args.M + m] = ssq;
    if (tr && g == 0 && et == 0) tr[13] = gtimer();
    epi_bar();
    if (tr && g == 0 && et == 0) tr[14] = gtimer();
    for (int i = et; i < kBM * 16; i += kBM) {
      const int r = i >> 4, j = i & 15, mm = tile_a * kBM + r;
      const int col = n_group + j * 8;
      if (mm < args.M && col < args.N)
        *reinterpret_cast<uint4*>(args.C + (long long)mm * args.ldc + col) = ob[swz<16>(r, j)];
    }
  }
}

// ---------------------------------------------------------------------------
// kRows (prefill): one 128 x BN output tile per CTA. Epilogue thread = one
// token row; columns are processed in 128-column groups (4 TMEM chunks of
// 32), pairing chunk c with chunk c + 2 (SILU, RoPE at D=128) or c + 1 (RoPE
// at D=64) so every rotation / gate-up pair is register local.
// ---------------------------------------------------------------------------
template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_rows_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                     const __grid_constant__ GemmArgs args) {
  constexpr int A_BYTES = kBM * kBK * 2;
  constexpr int B_BYTES = BN * kBK * 2;
  constexpr uint32_t TMEM_COLS = BN;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile_a = blockIdx.x;   // tokens (128)
  const int tile_b = blockIdx.y;   // output columns (BN)
  // split-K: this CTA's k-block range (gridDim.z splits of the K dimension)
  const int nkb_all = (args.K + kBK - 1) / kBK;
  const int S = gridDim.z, z = blockIdx.z;
  const int kb0 = (int)((long long)z * nkb_all / S), kb1 = (int)((long long)(z + 1) * nkb_all / S);
  const int nkb = kb1 - kb0;
  const int lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  unsigned long long* tr = (args.trace && lin < args.trace_ctas) ? args.trace + lin * 16 : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = gtimer();

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tr && threadIdx.x == 0) tr[1] = gtimer();

  pdl_launch();
  if (warp == 0) {
    if (lane == 0) {
      const int pre = min(nkb, STAGES);
      for (int i = 0; i < pre; ++i) {  // weights first, before the dependency wait
        mbar_arrive_expect_tx(&full[i], A_BYTES + B_BYTES);
        tma_load_2d(sb + i * B_BYTES, &map_b, &full[i], (kb0 + i) * kBK, tile_b * BN);
      }
      pdl_wait();
      for (int i = 0; i < pre; ++i) tma_load_2d(sa + i * A_BYTES, &map_a, &full[i], (kb0 + i) * kBK, tile_a * kBM);
      for (int i = pre; i < nkb; ++i) {
        const int s = i % STAGES;
        mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], A_BYTES + B_BYTES);
        tma_load_2d(sa + s * A_BYTES, &map_a, &full[s], (kb0 + i) * kBK, tile_a * kBM);
        tma_load_2d(sb + s * B_BYTES, &map_b, &full[s], (kb0 + i) * kBK, tile_b * BN);
      }
    }
  } else if (warp == 1) {
    pdl_wait();
    constexpr uint32_t idesc = instr_desc(BN);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % STAGES;
      mbar_wait(&full[s], (i / STAGES) & 1);
      tc_fence_after();
      if (tr && i == 0 && lane == 0) tr[2] = gtimer();
      if (lane == 0) {
        const uint64_t da = smem_desc_sw128(sa + s * A_BYTES);
        const uint64_t db = smem_desc_sw128(sb + s * B_BYTES);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) mma_bf16(tmem, da + 2 * k, db + 2 * k, idesc, (i | k) != 0);
        mma_commit(&empty[s]);
        if (i == nkb - 1) mma_commit(done);
      }
      __syncwarp();
    }
  } else {
    pdl_wait();
    const Epi& e = args.epi;
    const int quarter = warp & 3;
    const int m = tile_a * kBM + quarter * 32 + lane;
    const bool mok = m < args.M;
    const float rs = (e.ssq_in && mok) ? rms_scale(e, args.M, m) : 1.f;
    mbar_wait(done, 0);
    tc_fence_after();
    if (tr && threadIdx.x == 64) tr[3] = gtimer();
    if (tr && lane == 0) tr[8 + warp - 2] = gtimer();
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
    bool finish = true;
    if (S > 1) {
      // every split publishes its fp32 partial; the last to arrive sums all
      // of them in split order (deterministic) back into its TMEM tile and
      // runs the epilogue
      const int row = quarter * 32 + lane;
      const long long tile = (long long)tile_a * gridDim.y + tile_b;
      // partial layout per (tile, split): [BN / 4][128 rows][4] -- a warp's
      // float4 for one column quad covers 32 consecutive rows (512 B)
      float* mine = args.rpart + (tile * S + z) * kBM * BN + row * 4;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        float v[32];
        tmem_ld32(lane_addr + c, v);
#pragma unroll
        for (int k = 0; k < 32; k += 4)
          __stcg(reinterpret_cast<float4*>(mine + (c + k) * kBM), make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]));
      }
      __threadfence();
      epi_bar();
      __shared__ int s_last;
      if (threadIdx.x == 64) s_last = atom_add_acq_rel(args.rctr + tile, 1) == S - 1;
      epi_bar();
      finish = s_last;
      if (tr && threadIdx.x == 64) tr[4] = gtimer();
      if (finish) {
        __threadfence();
        const float* base = args.rpart + tile * S * kBM * BN + row * 4;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          float sum[32], own[32];
          tmem_ld32(lane_addr + c, own);
#pragma unroll
          for (int k = 0; k < 32; ++k) sum[k] = 0.f;
          for (int zz = 0; zz < S; ++zz) {
            if (zz == z) {
#pragma unroll
              for (int k = 0; k < 32; ++k) sum[k] += own[k];
            } else {
              const float* src = base + (long long)zz * kBM * BN + c * kBM;
#pragma unroll
              for (int k = 0; k < 32; k += 4) {
                const float4 w = __ldcg(reinterpret_cast<const float4*>(src + k * kBM));
                sum[k] += w.x;
                sum[k + 1] += w.y;
                sum[k + 2] += w.z;
                sum[k + 3] += w.w;
              }
            }
          }
          tmem_st32(lane_addr + c, sum);
        }
        tc_fence_before();
        epi_bar();
        tc_fence_after();
        if (threadIdx.x == 64) args.rctr[tile] = 0;
        if (tr && threadIdx.x == 64) tr[5] = gtimer();
      }
    }
    if (finish) {
      static_assert(STAGES * (A_BYTES + B_BYTES) >= 32768 + 65536 + 512, "epilogue staging area");
      if (e.kind != EPI_ARGMAX && (args.N % 8) == 0)
        rows_epilogue_staged<BN>(args, tile_a, tile_b, quarter * 32 + lane, rs, lane_addr, smem, tr);
      else
        rows_epilogue<BN>(args, m, mok, rs, lane_addr, tile_b);
    }
    if (tr && threadIdx.x == 64) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      tr[6] = gtimer();
      tr[7] = (unsigned long long)smid | ((unsigned long long)z << 16) | ((unsigned long long)finish << 31);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, TMEM_COLS);
}

// ---------------------------------------------------------------------------
// Prefill GEMM on a CTA pair (tcgen05 cta_group::2), persistent.
//
// A cluster of two CTAs on one TPC computes 256 x 256 output tiles: CTA r
// stages rows [128 r, 128 r + 128) of the A tile and of the W tile, the
// leader issues tcgen05.mma.cta_group::2 (M = 256, N = 256) reading both
// CTAs' shared memory, and each CTA's TMEM receives its 128 rows. Per CTA a
// stage is 32 KB (instead of 48 KB for a one-CTA 128 x 256 tile), so six
// stages fit and cover the TMA latency at tensor-core rate; the two 256-column
// accumulators (all 512 TMEM columns) let the epilogue of one tile overlap
// the main loop of the next. Tiles are walked M-fastest so consecutive tiles
// of a pair reuse the same weight columns from L2.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* smem, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                 int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(smem)),
      "l"(map), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {   // to the same barrier in both CTAs
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

// Partial sums of the other K-splits of a tile, added to each 32-column chunk
// the finisher (split 0) loads from TMEM: self-validating 64-bit words
// (fp32 bits | tag << 32), stale words re-polled together. Partials are column-major
// ([256 cols][128 rows] per CTA and split): a warp's lanes are consecutive
// rows, so every load and store is coalesced.
struct PairSplitFix {
  const unsigned long long* base;   // (tile, split 1, this CTA) row `row`
  long long stride;                 // between splits
  int extra;                        // splits - 1
  unsigned tag;
  __device__ __forceinline__ void operator()(float* v, int col) const {
    for (int s = 0; s < extra; ++s) {
      const unsigned long long* p = base + s * stride + (long long)col * 128;
      unsigned long long w[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) w[j] = ld_relaxed_u64(p + j * 128);
      for (;;) {   // stale words re-polled together
        bool ready = true;
#pragma unroll
        for (int j = 0; j < 32; ++j) ready &= (unsigned)(w[j] >> 32) == tag;
        if (ready) break;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if ((unsigned)(w[j] >> 32) != tag) w[j] = ld_relaxed_u64(p + j * 128);
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] += __uint_as_float((unsigned)w[j]);
    }
  }
};

template <int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                     const __grid_constant__ GemmArgs args) {
  constexpr int HALF = 128;                    // rows of A and of W staged per CTA
  constexpr int A_BYTES = HALF * kBK * 2;
  constexpr int B_BYTES = HALF * kBK * 2;
  constexpr uint32_t TMEM_COLS = 512;          // two 256-column accumulators
  constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) |
                             ((uint32_t)(256 >> 4) << 24);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int TM = (args.M + 255) / 256, TN = (args.N + 255) / 256, tiles = TM * TN;
  const int KB = (args.K + kBK - 1) / kBK;
  const int S = args.splits, units = tiles * S;   // unit = (tile, K-split)

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);   // 4 epilogue warps x 2 CTAs
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_launch();

  if (warp == 0) {
    if (lane == 0) {
      pdl_wait();
      int idx = 0;
      for (int u = pair; u < units; u += npairs) {
        const int t = u / S, sp = u % S;
        const int tm = t % TM, tn = t / TM;
        const int k0 = sp * KB / S, k1 = (sp + 1) * KB / S;
        for (int kb = k0; kb < k1; ++kb, ++idx) {
          const int s = idx % STAGES;
          if (idx >= STAGES) mbar_wait(&empty[s], ((idx / STAGES) - 1) & 1);
          if (leader) mbar_arrive_expect_tx(&full[s], 2 * (A_BYTES + B_BYTES));
          const uint32_t bar = mapa_shared(smem_u32(&full[s]), 0);   // the leader's barrier counts both CTAs
          tma_load_2d_pair(sa + s * A_BYTES, &map_a, bar, kb * kBK, tm * 256 + (int)rank * HALF);
          tma_load_2d_pair(sb + s * B_BYTES, &map_b, bar, kb * kBK, tn * 256 + (int)rank * HALF);
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      int i = 0, lt = 0;
      for (int u = pair; u < units; u += npairs, ++lt) {
        const int sp = u % S;
        const int k0 = sp * KB / S, k1 = (sp + 1) * KB / S;
        const int buf = lt & 1;
        if (lt >= 2) mbar_wait(&tempty[buf], ((lt >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + buf * 256;
        for (int kb = k0; kb < k1; ++kb, ++i) {
          const int s = i % STAGES;
          mbar_wait(&full[s], (i / STAGES) & 1);
          tc_fence_after();
          if (lane == 0) {
            const uint64_t da = smem_desc_sw128(sa + s * A_BYTES);
            const uint64_t db = smem_desc_sw128(sb + s * B_BYTES);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              mma_bf16_pair(acc, da + 2 * k, db + 2 * k, idesc, (kb != k0 || k != 0) ? 1u : 0u);
            mma_commit_pair(&empty[s]);
          }
          __syncwarp();
        }
        if (lane == 0) mma_commit_pair(&tfull[buf]);
        __syncwarp();
      }
    }
  } else {
    pdl_wait();
    const Epi& e = args.epi;
    const int quarter = warp & 3;
    const uint32_t tempty_leader[2] = {mapa_shared(smem_u32(&tempty[0]), 0), mapa_shared(smem_u32(&tempty[1]), 0)};
    const unsigned tag = S > 1 ? (((unsigned)__ldcg(args.ctr + kMaxPhases + 1) + 1u) << 4) | 15u : 0u;
    const int row_local = quarter * 32 + lane;
    constexpr long long kPartCta = (long long)HALF * 256;   // words per CTA partial
    int lt = 0;
    for (int u = pair; u < units; u += npairs, ++lt) {
      const int t = u / S, sp = u % S;
      const int tm = t % TM, tn = t / TM;
      const int buf = lt & 1;
      const int m = tm * 256 + (int)rank * HALF + row_local;
      const bool mok = m < args.M;
      const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + buf * 256;
      mbar_wait(&tfull[buf], (lt >> 1) & 1);
      tc_fence_after();
      if (sp < S - 1) {
        // contributor: publish this split's accumulator rows as tagged partials
        unsigned long long* p =
            args.part + (((long long)t * (S - 1) + sp) * 2 + rank) * kPartCta + row_local;
        for (int c = 0; c < 8; ++c) {
          float v[32];
          tmem_ld32(taddr + c * 32, v);
#pragma unroll
          for (int j = 0; j < 32; ++j)
            st_relaxed_u64(p + (c * 32 + j) * 128,
                           (unsigned long long)__float_as_uint(v[j]) | ((unsigned long long)tag << 32));
        }
      } else {
        const float rs = (e.ssq_in && mok) ? rms_scale(e, args.M, m) : 1.f;
        if (S > 1) {
          PairSplitFix fix{args.part + ((long long)t * (S - 1) * 2 + rank) * kPartCta + row_local,
                           2 * kPartCta, S - 1, tag};
          rows_epilogue<256>(args, m, mok, rs, taddr, tn, fix);
        } else {
          rows_epilogue<256>(args, m, mok, rs, taddr, tn);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(tempty_leader[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  if (threadIdx.x == 0 && args.ctr) {
    // the last CTA to leave advances the workspace's launch epoch (partial tags)
    if (atom_add_acq_rel(args.ctr + kMaxPhases, 1) == (int)gridDim.x - 1) {
      args.ctr[kMaxPhases] = 0;
      args.ctr[kMaxPhases + 1] += 1;
    }
  }
}

// ---------------------------------------------------------------------------
// Decode GEMM: persistent stream-K on tcgen05 (swap-AB orientation).
//
// MMA A = W rows (128 output features per tile), MMA B = the M <= 64 tokens
// (BN = 16/32/64). The tiles x k-blocks work units are split evenly over one
// CTA per SM, so every SM streams the same number of weight bytes (the
// roofline of a decode step is the weight stream). A CTA walks its units in
// order: the TMA ring runs continuously across tile boundaries, the MMA warp
// accumulates each tile *segment* into one of two TMEM accumulators, and the
// epilogue drains the other. Segments covering a whole tile finish directly;
// split tiles are fixed up deterministically -- each segment stores an fp32
// partial, the last to arrive sums them in segment order and finishes.
// Epilogue thread = one output feature of the tile, all M tokens; pairs that
// straddle warps (RoPE, gate/up) are exchanged through shared memory.
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Decode GEMM chain: persistent stream-K on tcgen05 (swap-AB orientation),
// running up to kMaxPhases dependent GEMMs in one launch.
//
// Per phase, MMA A = W rows (128 output features per tile), MMA B = the M <= 64
// tokens (BN = 16/32/64); the tiles x k-blocks units are split evenly over
// one CTA per SM so every SM streams the same number of weight bytes (the
// roofline of a decode step is the weight stream). A CTA walks its units in
// order; the TMA ring runs continuously across tile *and phase* boundaries,
// the MMA warp accumulates each tile segment into one of two TMEM
// accumulators and the epilogue drains the other. Segments covering a whole
// tile finish directly; split tiles are fixed up deterministically (each
// segment stores an fp32 partial, the last to arrive sums them in segment
// order and finishes).
//
// Phase p+1 reads phase p's output, so its activation tiles wait on a
// device-side phase barrier (every CTA's epilogue arrives after finishing
// phase p); its *weight* tiles do not, and stream into the ring while phase p
// drains -- the same trick PDL plays at kernel boundaries (phase 0 waits on
// griddepcontrol.wait instead).
// ---------------------------------------------------------------------------

struct SkPhase {
  bf16* C;
  int M, N, K, ldc;
  int tiles, kbs, maxseg;
  int geff;          // CTAs sharing this phase's units: min(grid, units); the rest idle in it
  long long units;
  Epi epi;
};

// Stream-K range of CTA `cta` in a phase: [u0, u1) (empty for cta >= geff).
__device__ __forceinline__ void sk_range(const SkPhase& P, int cta, long long& u0, long long& u1) {
  if (cta < P.geff) {
    u0 = (long long)cta * P.units / P.geff;
    u1 = (long long)(cta + 1) * P.units / P.geff;
  } else {
    u0 = u1 = P.units;
  }
}

struct ChainMaps {
  CUtensorMap w[kMaxPhases];
  CUtensorMap x[kMaxPhases];
  CUtensorMap pool;            // attention (AS > 1): the KV pool as [blocks x L x 2 x Hkv x 16][D]
};

struct ChainArgs {
  unsigned long long* trace;   // diagnostics: [grid][8] globaltimer stamps, or NULL
  float* ws;                   // split-tile partials [tiles][maxseg][M][128] (reused by every phase)
  int* counters;               // [tiles] arrival counters, zero between uses
  int* phase_ctr;              // [kMaxPhases + 1] phase / kernel arrival counters, zero between launches
  int M, grid, nph;
  int l2_pre;                  // weight tiles per CTA prefetched into L2 before griddepcontrol.wait
  int nattn;                   // attention phases (layers) in this launch
  int attn_kind[kMaxAttn];     // 1: D128 G4; 2: D64 G2; 3: D64 G4
  int attn_before[kMaxAttn];   // the GEMM phase that attention k precedes (its output is that phase's A)
  attn::AttnWork at[kMaxAttn];
  int pf_layer;                // >= 0: prefetch that layer's K/V pages into L2 during the last phase
  int attn_early;              // the first attention's work split runs before griddepcontrol.wait
  int block_rows;              // attention (AS > 1): rows of one pool block in ChainMaps::pool
  int trace_phase;             // diagnostics: the phase whose split-tile finishers are traced
  SkPhase ph[kMaxPhases];
};
constexpr int kAttnCtr = kMaxPhases + 2;   // phase_ctr slots kAttnCtr + k: CTAs done with attention k


// Stream-K fix-up loads of a split tile's finisher: the words of segments
// c_first+1..c_last for tokens T0 <= t < min(M, T0 + MT) (compile-time
// range), 32/MT segments per round. All words of a round are loaded together and the stale
// ones (tag not yet this launch's) re-polled together: a late segment costs
// one round trip after it lands, not one per word. Summed in CTA order.
template <int MT, int T0, int BN>
__device__ __forceinline__ void sk_collect(const unsigned long long* tpart, int c_first, int c_last,
                                           long long cstride, int M, unsigned tag, float (&acc)[BN]) {
  static_assert(MT <= 32 && T0 + MT <= BN, "token range");
  constexpr int KG = 32 / MT;
  const unsigned long long ready_word = (unsigned long long)tag << 32;
  for (int c0 = c_first + 1; c0 <= c_last; c0 += KG) {
    unsigned long long pv[KG][MT];
    const unsigned long long* base = tpart + (long long)(c0 - c_first) * cstride;
#pragma unroll
    for (int k = 0; k < KG; ++k)
#pragma unroll
      for (int t = 0; t < MT; ++t)
        pv[k][t] = (c0 + k <= c_last && T0 + t < M) ? ld_relaxed_u64(base + k * cstride + (long long)(T0 + t) * kBM)
                                                    : ready_word;
    for (;;) {
      bool ready = true;
#pragma unroll
      for (int k = 0; k < KG; ++k)
#pragma unroll
        for (int t = 0; t < MT; ++t) ready &= (unsigned)(pv[k][t] >> 32) == tag;
      if (ready) break;
#pragma unroll
      for (int k = 0; k < KG; ++k)
#pragma unroll
        for (int t = 0; t < MT; ++t)
          if ((unsigned)(pv[k][t] >> 32) != tag) pv[k][t] = ld_relaxed_u64(base + k * cstride + (long long)(T0 + t) * kBM);
    }
#pragma unroll
    for (int k = 0; k < KG; ++k) {
      if (c0 + k > c_last) break;
#pragma unroll
      for (int t = 0; t < MT; ++t)
        if (T0 + t < M) acc[T0 + t] += __uint_as_float((unsigned)pv[k][t]);
    }
  }
}

__device__ __forceinline__ int sk_owner(long long u, long long units, int grid) {
  return (int)(((u + 1) * grid - 1) / units);
}

__device__ __forceinline__ void wait_phase(const int* ctr, int target) {
  while (ld_acquire(ctr) < target) __nanosleep(32);
}


// MT: token loops' bound (1: batch of one). AS: pages in flight per attention
// warp (1: one page, cp.async; > 1: the TMA-staged ring, for larger batches).
template <int BN, int STAGES, int MINB, int MT = BN, int AS = 1>
__global__ void __launch_bounds__(kThreads, MINB)
    gemm_chain_kernel(const __grid_constant__ ChainMaps maps, const __grid_constant__ ChainArgs args) {
  constexpr int A_BYTES = kBM * kBK * 2;
  constexpr int B_BYTES = BN * kBK * 2;
  constexpr uint32_t TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  bf16* xch = reinterpret_cast<bf16*>(tmem_slot + 4);        // [BN][128]
  float* red = reinterpret_cast<float*>(xch + BN * kBM);     // [4][BN]
  float* rs = red + 4 * BN;                                  // [BN]
  int* slot_s = reinterpret_cast<int*>(rs + BN);             // [64] QKV phases: the tokens' pool slots
  constexpr bool kAttn = MINB == 1;                          // deep (layer) chains carry the attention phase
  uint64_t* abar = reinterpret_cast<uint64_t*>(slot_s + 64);  // [4][AS] attention page barriers (AS > 1)
  constexpr uintptr_t kVsAlign = AS > 1 ? 1024 : 128;         // TMA 128-byte-swizzle destinations
  bf16* vs_all = reinterpret_cast<bf16*>((reinterpret_cast<uintptr_t>(abar + 4 * AS) + kVsAlign - 1) &
                                         ~(kVsAlign - 1));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const int G = args.grid;
  unsigned long long* tr = args.trace ? args.trace + (long long)cta * 32 : nullptr;   // [0..15] phases, [16..31] attention
  if (tr && threadIdx.x == 0) tr[0] = gtimer();

  if (warp == 0 && lane == 0) {
    for (int p = 0; p < args.nph; ++p) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.w[p]) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.x[p]) : "memory");
    }
    if constexpr (AS > 1)
      if (args.nattn) asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.pool) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    if constexpr (AS > 1)
      for (int i = 0; i < 4 * AS; ++i) mbar_init(&abar[i], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  pdl_launch();
  if (warp == 0) {
    if (lane == 0) {
      int i = 0;   // ring position, continuous across phases
      for (int p = 0; p < args.nph; ++p) {
        const SkPhase& P = args.ph[p];
        const int KB = P.kbs;
        long long u0, u1;
        sk_range(P, cta, u0, u1);
        // nothing to load: no counter wait either (the last phase's counter
        // may be reset for the next launch as soon as every epilogue has
        // arrived) -- but griddepcontrol.wait still comes first, before this
        // thread reads any counter of a later phase
        if (u0 == u1) {
          if (p == 0) pdl_wait();
          continue;
        }
        const int pre = (int)(u1 - u0 < STAGES ? u1 - u0 : STAGES);
        // weights first: independent of the previous phase / kernel
        for (int k = 0; k < pre; ++k) {
          const int idx = i + k, s = idx % STAGES;
          if (idx >= STAGES) mbar_wait(&empty[s], ((idx / STAGES) - 1) & 1);
          const long long u = u0 + k;
          mbar_arrive_expect_tx(&full[s], A_BYTES + B_BYTES);
          tma_load_2d(sa + s * A_BYTES, &maps.w[p], &full[s], (int)(u % KB) * kBK, (int)(u / KB) * kBM);
        }
        int ak = -1;
        if (kAttn)
          for (int k = 0; k < args.nattn; ++k)
            if (args.attn_before[k] == p) ak = k;
        if (p == 0) {
          // While the previous kernel finishes and the layer's attention runs,
          // prefetch the next l2_pre weight tiles of this CTA's stream (beyond
          // the smem ring) into L2 (default 0: measured slower at every depth,
          // profiles/r2_chain_l2pre_rejected.txt).
          if (args.l2_pre > 0) {
            int q = p;
            long long uu = u0 + pre, qu1 = u1;
            for (int k = 0; k < args.l2_pre; ++k, ++uu) {
              while (uu >= qu1 && ++q < args.nph) {
                long long a0, a1;
                sk_range(args.ph[q], cta, a0, a1);
                uu = a0;
                qu1 = a1;
              }
              if (q >= args.nph) break;
              const int qkb = args.ph[q].kbs;
              asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(&maps.w[q]),
                           "r"((int)(uu % qkb) * kBK), "r"((int)(uu / qkb) * kBM)
                           : "memory");
            }
          }
          pdl_wait();
          if (ak >= 0) {
            wait_phase(args.phase_ctr + kAttnCtr + ak, G);   // every CTA's share of the attention is written
            asm volatile("fence.proxy.async;" ::: "memory");
          }
        } else if (ak >= 0) {
          wait_phase(args.phase_ctr + kAttnCtr + ak, G);
          asm volatile("fence.proxy.async;" ::: "memory");
        } else {
          wait_phase(args.phase_ctr + p - 1, G);
          asm volatile("fence.proxy.async;" ::: "memory");   // generic-proxy writes -> TMA reads
        }
        if (tr && p < 4) tr[1 + p] = gtimer();   // activations of phase p released (first layer only)
        for (int k = 0; k < pre; ++k) {
          const int s = (i + k) % STAGES;
          tma_load_2d(sb + s * B_BYTES, &maps.x[p], &full[s], (int)((u0 + k) % KB) * kBK, 0);
        }
        int idx = i + pre;
        for (long long u = u0 + pre; u < u1; ++u, ++idx) {
          const int s = idx % STAGES;
          if (idx >= STAGES) mbar_wait(&empty[s], ((idx / STAGES) - 1) & 1);
          mbar_arrive_expect_tx(&full[s], A_BYTES + B_BYTES);
          const int kc = (int)(u % KB) * kBK;
          tma_load_2d(sa + s * A_BYTES, &maps.w[p], &full[s], kc, (int)(u / KB) * kBM);
          tma_load_2d(sb + s * B_BYTES, &maps.x[p], &full[s], kc, 0);
        }
        i += (int)(u1 - u0);
      }
    }
  } else if (warp == 1) {
    pdl_wait();
    constexpr uint32_t idesc = instr_desc(BN);
    int i = 0, seg = 0;
    for (int p = 0; p < args.nph; ++p) {
      const SkPhase& P = args.ph[p];
      const int KB = P.kbs;
      long long u0, u1;
      sk_range(P, cta, u0, u1);
      for (long long u = u0; u < u1; ++seg) {
        const long long tile = u / KB;
        const long long seg_end = min(u1, (tile + 1) * KB);
        const int buf = seg & 1;
        if (seg >= 2) mbar_wait(&tempty[buf], ((seg >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + buf * BN;
        const long long seg_begin = u;
        for (; u < seg_end; ++u, ++i) {
          const int s = i % STAGES;
          mbar_wait(&full[s], (i / STAGES) & 1);
          tc_fence_after();
          if (lane == 0) {

            const uint64_t da = smem_desc_sw128(sa + s * A_BYTES);
            const uint64_t db = smem_desc_sw128(sb + s * B_BYTES);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              mma_bf16(acc, da + 2 * k, db + 2 * k, idesc, (u != seg_begin || k != 0) ? 1u : 0u);
            mma_commit(&empty[s]);
          }
          __syncwarp();
        }
        if (lane == 0) mma_commit(&tfull[buf]);
        __syncwarp();
      }
    }
    if (tr && lane == 0) tr[9] = gtimer();
  } else {
    bool attn0_done = false;
    uint32_t acnt = 0;   // this attention warp's running page count (AS > 1)
    attn::TmaPages tpg;
    tpg.map = &maps.pool;
    tpg.block_rows = args.block_rows;
    if constexpr (kAttn) {
      if (args.attn_early && args.nattn && args.attn_before[0] == 0) {
        // The first attention starts before griddepcontrol.wait: its work
        // split needs only the step's inputs (contexts, block tables); each
        // warp waits for the previous kernel (q, the new token's K/V, the
        // workspace epoch) right before its first q / page loads.
        const int ew = warp - 2;
        attn::AttnWork aw = args.at[0];
        auto wait_prev = [&aw, &args](int, int) {
          pdl_wait();
          aw.tag = (((unsigned)__ldcg(args.phase_ctr + kMaxPhases + 1) + 1u) << 4) | 8u;
        };
        auto done = [](int, int) { asm volatile("fence.proxy.async;" ::: "memory"); };
        unsigned long long* atr = (tr && ew == 0) ? tr + 16 : nullptr;
        if (args.attn_kind[0] == 1)
          attn::attn_cta_phase<128, 4, AS>(aw, cta, G, ew, lane, vs_all, wait_prev, done, atr, &tpg, abar, &acnt);
        else if (args.attn_kind[0] == 2)
          attn::attn_cta_phase<64, 2, AS>(aw, cta, G, ew, lane, vs_all, wait_prev, done, nullptr, &tpg, abar, &acnt);
        else if (args.attn_kind[0] == 4)
          attn::attn_cta_phase<128, 8, AS>(aw, cta, G, ew, lane, vs_all, wait_prev, done, nullptr, &tpg, abar, &acnt);
        else
          attn::attn_cta_phase<64, 4, AS>(aw, cta, G, ew, lane, vs_all, wait_prev, done, nullptr, &tpg, abar, &acnt);
        pdl_wait();
        asm volatile("fence.proxy.async;" ::: "memory");
        epi_bar();
        if (threadIdx.x == 64) {
          atom_add_acq_rel(args.phase_ctr + kAttnCtr, 1);
          if (tr) tr[15] = gtimer();   // this CTA's share of attention 0 written
        }
        attn0_done = true;
      }
    }
    pdl_wait();
    const int epoch = __ldcg(args.phase_ctr + kMaxPhases + 1) + 1;   // launches completed on this workspace + 1
    const int quarter = warp & 3;
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
    const int row = quarter * 32 + lane;  // feature within the tile
    int seg = 0;
    for (int p = 0; p < args.nph; ++p) {
      const SkPhase& P = args.ph[p];
      const int KB = P.kbs;
      const long long U = P.units;
      long long u0, u1;
      sk_range(P, cta, u0, u1);
      // Everything this phase's epilogue reads from earlier phases (residual,
      // norm statistics) was published by those phases' barrier: acquire it
      // once, then order the other epilogue threads behind it.
      if (p > 0) {
        if (threadIdx.x == 64) wait_phase(args.phase_ctr + p - 1, G);
        epi_bar();
      }
      if constexpr (kAttn) {
        for (int k = attn0_done ? 1 : 0; k < args.nattn; ++k) {
          if (args.attn_before[k] != p) continue;
          // A layer's paged decode attention (attn_mma.cuh), by this CTA's
          // epilogue warps, while warp 0 already streams phase p's weight
          // tiles into the ring; its output is phase p's A.
          const int ew = warp - 2;
          auto no_wait = [](int, int) {};
          auto done = [](int, int) { asm volatile("fence.proxy.async;" ::: "memory"); };
          attn::AttnWork aw = args.at[k];
          aw.tag = ((unsigned)epoch << 4) | (unsigned)(8 + k);
          unsigned long long* atr = (tr && ew == 0 && k == 0) ? tr + 16 : nullptr;
          if (args.attn_kind[k] == 1)
            attn::attn_cta_phase<128, 4, AS>(aw, cta, G, ew, lane, vs_all, no_wait, done, atr, &tpg, abar, &acnt);
          else if (args.attn_kind[k] == 2)
            attn::attn_cta_phase<64, 2, AS>(aw, cta, G, ew, lane, vs_all, no_wait, done, nullptr, &tpg, abar, &acnt);
          else if (args.attn_kind[k] == 4)
            attn::attn_cta_phase<128, 8, AS>(aw, cta, G, ew, lane, vs_all, no_wait, done, nullptr, &tpg, abar, &acnt);
          else
            attn::attn_cta_phase<64, 4, AS>(aw, cta, G, ew, lane, vs_all, no_wait, done, nullptr, &tpg, abar, &acnt);
          asm volatile("fence.proxy.async;" ::: "memory");
          epi_bar();
          if (threadIdx.x == 64) {
            atom_add_acq_rel(args.phase_ctr + kAttnCtr + k, 1);
            if (tr && k == 0) tr[15] = gtimer();   // this CTA's share of attention 0 written
          }
        }
      }
      // per-phase token data staged in shared memory: RMS scales, and for a
      // QKV phase the pool slots and (deep chains: in the attention's V-page
      // space, free during the GEMM phases) the RoPE table -- the finisher's
      // epilogue then reads no global memory but its outputs' inputs
      const bool qkv = P.epi.kind == EPI_QKV_ROPE;
      const float2* cs_s = nullptr;
      bool stage = false;
      if constexpr (kAttn) {
        const int n = args.M * (P.epi.D / 2);
        stage = qkv && P.epi.cs && n * (int)sizeof(float2) <= 4 * attn::kAttnWarpBytes;
        if (stage) {
          if (row < args.M) slot_s[row] = P.epi.slots[row];
          float2* cs = reinterpret_cast<float2*>(vs_all);
          for (int i = row; i < n; i += kBM) cs[i] = P.epi.cs[i];
          cs_s = cs;
        }
      }
      if (P.epi.ssq_in && row < args.M) rs[row] = rms_scale(P.epi, args.M, row);
      if (P.epi.ssq_in || stage) epi_bar();
      if constexpr (kAttn) {
        if (args.nattn && args.pf_layer >= 0 && p == args.nph - 1) {
          // the next layer's attention (next launch) reads these pages: warm L2 now
          attn::AttnWork nx = args.at[args.nattn - 1];
          nx.layer = args.pf_layer;
          if (args.attn_kind[0] == 1 || args.attn_kind[0] == 4) attn::attn_cta_prefetch<128>(nx, cta, G, warp - 2, lane);
          else attn::attn_cta_prefetch<64>(nx, cta, G, warp - 2, lane);
        }
      }
      // Split tiles are finished by c_first, the CTA owning the tile's first
      // k-blocks: its segment closes its range while the others open theirs,
      // so their partials are normally in L2 long before. Partials are
      // self-validating 64-bit words (fp32 bits | tag << 32, single-copy
      // atomic): the finisher loads them while its own last MMAs run and
      // spins only on words not yet written -- no arrival counter and no
      // round trip after the last MMA. Sum order: the other segments in CTA
      // order, then the finisher's own (deterministic).
      const unsigned tag = ((unsigned)epoch << 4) | (unsigned)p;
      const bool resid = P.epi.kind == EPI_RESIDUAL;
      unsigned long long* wsq = reinterpret_cast<unsigned long long*>(args.ws);
      for (long long u = u0; u < u1; ++seg) {
        const long long tile = u / KB;
        const long long seg_end = min(u1, (tile + 1) * KB);
        const bool whole = (u == tile * KB) && (seg_end == (tile + 1) * KB);
        u = seg_end;
        const int buf = seg & 1;
        const long long first_u = tile * KB;
        const int c_first = whole ? cta : sk_owner(first_u, U, P.geff);
        const int c_last = whole ? cta : sk_owner(first_u + KB - 1, U, P.geff);
        const bool finisher = cta == c_first;
        unsigned long long* tpart = wsq + ((tile * P.maxseg) * (long long)args.M) * kBM + row;
        constexpr bool kPreRes = BN <= 32;   // register budget: BN = 64 reads the residual in the epilogue
        float res[BN], acc[BN];
        // diagnostics (phase trace_phase, the last finished tile): [11] collect start, [12] collect done,
        // [13] own MMAs done, [14] epilogue done
        const bool ftr = tr && finisher && !whole && p == args.trace_phase && threadIdx.x == 64;
        if (ftr) tr[11] = gtimer();
        if (finisher) {
          if (kPreRes && resid) {
            const int f = (int)tile * kBM + row;
#pragma unroll
            for (int t = 0; t < MT; ++t)
              res[t] = (t < args.M && f < P.N) ? bf2f(__ldcg(P.epi.residual + (long long)t * P.ldc + f)) : 0.f;
            // pin the loads here (issued before the collect, consumed after it):
            // the compiler would otherwise sink them into the epilogue loop and
            // pay an L2 round trip there
#pragma unroll
            for (int t = 0; t < MT; ++t) asm volatile("" : "+f"(res[t]));
          }
#pragma unroll
          for (int t = 0; t < MT; ++t) acc[t] = 0.f;
          // the other segments' words: up to 32 per thread in flight (several
          // segments at once when M is small), stale words re-polled together
          const long long cstride = (long long)args.M * kBM;
          const int M = args.M;
          if (MT == 1 || M <= 1) sk_collect<1, 0>(tpart, c_first, c_last, cstride, M, tag, acc);
          else if (MT == 2) sk_collect<2, 0>(tpart, c_first, c_last, cstride, M, tag, acc);
          else if (MT == 4) sk_collect<4, 0>(tpart, c_first, c_last, cstride, M, tag, acc);
          else if (MT == 8) sk_collect<8, 0>(tpart, c_first, c_last, cstride, M, tag, acc);
          else if (M <= 2) sk_collect<2, 0>(tpart, c_first, c_last, cstride, M, tag, acc);
          else if (M <= 4) sk_collect<4, 0>(tpart, c_first, c_last, cstride, M, tag, acc);
          else if (M <= 8) sk_collect<8, 0>(tpart, c_first, c_last, cstride, M, tag, acc);
          else if (M <= 16) sk_collect<16, 0>(tpart, c_first, c_last, cstride, M, tag, acc);
          else if constexpr (BN >= 32) {
            sk_collect<16, 0>(tpart, c_first, c_last, cstride, M, tag, acc);
            sk_collect<16, 16>(tpart, c_first, c_last, cstride, M, tag, acc);
            if constexpr (BN == 64) {
              if (M > 32) {
                sk_collect<16, 32>(tpart, c_first, c_last, cstride, M, tag, acc);
                sk_collect<16, 48>(tpart, c_first, c_last, cstride, M, tag, acc);
              }
            }
          }
        }
        if (ftr) tr[12] = gtimer();
        mbar_wait(&tfull[buf], (seg >> 1) & 1);
        tc_fence_after();
        if (ftr) tr[13] = gtimer();
        float v[BN < 32 ? 32 : BN];
#pragma unroll
        for (int c0 = 0; c0 < BN; c0 += 32) tmem_ld32(lane_addr + buf * BN + c0, v + c0);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        if (ftr) tr[30] = gtimer();   // accumulator read back from TMEM
        if (!finisher) {
          unsigned long long* pp = tpart + (long long)(cta - c_first) * args.M * kBM;
#pragma unroll
          for (int t = 0; t < MT; ++t)
            if (t < args.M)
              st_relaxed_u64(pp + (long long)t * kBM,
                             (unsigned long long)__float_as_uint(v[t]) | ((unsigned long long)tag << 32));
          continue;
        }
        if (!whole) {
#pragma unroll
          for (int t = 0; t < MT; ++t) v[t] = acc[t] + v[t];
        }
        if (ftr) tr[31] = gtimer() + (v[0] == 1234.5f);   // partials added
        sk_finish<BN, SkPhase, MT>(P, (int)tile, row, v, rs, xch, red, (kPreRes && resid) ? res : nullptr, stage ? slot_s : nullptr,
                      cs_s, ftr ? tr + 28 : nullptr);
        if (ftr) tr[14] = gtimer();
      }
      // phase p done in this CTA: publish (release) for the other CTAs. The
      // last CTA to finish the last phase resets the counters for the next
      // launch: every CTA has passed all of its counter waits by then (its
      // producer waited before loading this phase's activations), and the
      // next launch touches them only after griddepcontrol.wait.
      epi_bar();
      if (threadIdx.x == 64) {
        const int before = atom_add_acq_rel(args.phase_ctr + p, 1);
        if (tr && p < 4) tr[5 + p] = gtimer();
        if (p == args.nph - 1 && before == G - 1) {
          for (int q = 0; q <= kMaxPhases; ++q) args.phase_ctr[q] = 0;
          for (int k = 0; k < kMaxAttn; ++k) args.phase_ctr[kAttnCtr + k] = 0;
          args.phase_ctr[kMaxPhases + 1] += 1;   // launch epoch (tags of the stream-K partials)
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, TMEM_COLS);
  if (tr && threadIdx.x == 0) tr[10] = gtimer();
}

__global__ void rope_table_kernel(const int32_t* __restrict__ pos, int T, int half, float theta,
                                  float2* __restrict__ out) {
  pdl_wait();
  pdl_launch();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < T * half; i += gridDim.x * blockDim.x) {
    const int t = i / half, k = i % half;
    float sn, cs;
    sincosf((float)pos[t] * (1.0f / powf(theta, (float)(2 * k) / (float)(2 * half))), &sn, &cs);
    out[i] = make_float2(cs, sn);
  }
}

// ---- host side ----------------------------------------------------------------------------

template <int BN, int STAGES>
int launch_rows(const CUtensorMap& ma, const CUtensorMap& mb, const GemmArgs& a, dim3 grid, cudaStream_t st) {
  auto kern = gemm_rows_kernel<BN, STAGES>;
  constexpr size_t smem = 1024 + (size_t)STAGES * (kBM * kBK * 2 + BN * kBK * 2) + (2 * STAGES + 1) * 8 + 16;
  static bool attr = false;
  if (!attr) {
    ASTRAEA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  ASTRAEA_TRY(launch_k(kern, grid, dim3(kThreads), smem, st, ma, mb, a));
  return 0;
}

template <int STAGES>
int launch_pair(const CUtensorMap& ma, const CUtensorMap& mb, const GemmArgs& a, cudaStream_t st) {
  auto kern = gemm_pair_kernel<STAGES>;
  constexpr size_t smem = 1024 + (size_t)STAGES * (2 * 128 * kBK * 2) + (2 * STAGES + 4) * 8 + 16;
  static bool attr = false;
  if (!attr) {
    ASTRAEA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  const int tiles = ((a.M + 255) / 256) * ((a.N + 255) / 256);
  const int pairs = std::max(1, std::min(tiles * a.splits, num_sms() / 2));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  ASTRAEA_TRY(cudaLaunchKernelEx(&cfg, kern, ma, mb, a));
  return 0;
}

bool pair_gemm_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ASTRAEA_GEMM_PAIR");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

constexpr int kColsMaxM = 64;

struct SkPlan {
  int bn, tiles, kbs, grid, maxseg;
  long long units;
};

SkPlan sk_plan(int M, int N, int K) {
  SkPlan p;
  p.bn = M <= 16 ? 16 : (M <= 32 ? 32 : 64);
  p.tiles = (N + kBM - 1) / kBM;
  p.kbs = (K + kBK - 1) / kBK;
  p.units = (long long)p.tiles * p.kbs;
  p.grid = num_sms();
  p.maxseg = (p.grid + p.tiles - 1) / p.tiles + 1;
  return p;
}

// Workspace layout: a fixed tile-counter region shared by every GEMM shape
// (so GEMMs of different tile counts reuse one workspace in stream order
// without clobbering each other's counters), the phase counters, then the
// fp32 partials of split tiles.
constexpr size_t kCounterBytes = 16384 * sizeof(int);
constexpr size_t kPhaseBytes = 256;
// attention phase of a layer chain: [grid <= 192][G <= 4][D + 2 <= 130] tagged split partials
constexpr size_t kAttnWsBytes = (size_t)192 * 8 * 130 * sizeof(unsigned long long);   // grid x G x (D + 2), G*D <= 1024
constexpr size_t kHeadBytes = kCounterBytes + kPhaseBytes + kAttnWsBytes;   // before the GEMM partials

size_t partial_bytes(int M, const SkPlan& p) { return (size_t)p.tiles * p.maxseg * M * kBM * sizeof(unsigned long long); }

template <int BN, bool DEEP = false, int AS = 1>
constexpr size_t sk_extra_bytes() {
  // DEEP (layer) chains also hold the attention phase's four V pages, or
  // with AS > 1 four rings of AS (K + V) pages (D = 128 sized, 1 KB aligned)
  return (size_t)BN * kBM * 2 + 5 * BN * sizeof(float) + 64 * sizeof(int) + 64 +
         (DEEP ? (AS > 1 ? 1024 + 4 * AS * 8 + 4 * (size_t)AS * attn::tma_page_bytes<128>()
                         : 128 + 4 * (size_t)attn::kAttnWarpBytes)
               : 0);
}
// Single GEMMs: ~104 KB so two CTAs fit per SM and the next kernel's CTA can
// become resident and prefetch its weights (PDL) while this one drains.
// Chains: one deep ring per SM (~200 KB), the phases hide each other's tails.
#ifndef ASTRAEA_DEEP_RING_KB
#define ASTRAEA_DEEP_RING_KB 200   // smem budget of a deep chain's ring + extras (KB)
#endif
template <int BN, bool DEEP, int AS = 1>
constexpr int sk_stages() {
  return (int)(((DEEP ? ASTRAEA_DEEP_RING_KB : 104) * 1024 - sk_extra_bytes<BN, DEEP, AS>()) /
               (kBM * kBK * 2 + BN * kBK * 2));
}

// Attention pages in flight per warp for the batches a BN / MT instantiation
// serves: batches <= 4 keep the one-page walk and the deepest weight ring,
// 5-8 two TMA page stages, above 8 three (weight-ring stages traded for
// pages in flight; ASTRAEA_CHAIN_ATTN_STAGES* at build time; same-box A/B in
// profiles/r2_attn_stages_small_ab.txt: batch 8 3.646 -> 3.560 ms with two
// stages, batches 1-4 within +-0.7%).
#ifndef ASTRAEA_CHAIN_ATTN_STAGES
#define ASTRAEA_CHAIN_ATTN_STAGES 3
#endif
#ifndef ASTRAEA_CHAIN_ATTN_STAGES_SMALL
#define ASTRAEA_CHAIN_ATTN_STAGES_SMALL 1
#endif
template <int BN, int MT>
constexpr int chain_attn_stages() {
  return (BN == 16 && MT <= 4) ? ASTRAEA_CHAIN_ATTN_STAGES_SMALL
         : (BN == 16 && MT == 8) ? 2 : ASTRAEA_CHAIN_ATTN_STAGES;
}

template <int BN, bool DEEP, int MT>
int launch_chain_mt(const ChainMaps& maps, const ChainArgs& a, cudaStream_t st, int which) {
  constexpr int AS = DEEP ? chain_attn_stages<BN, MT>() : 1;
  constexpr int S = sk_stages<BN, DEEP, AS>();
  constexpr int MB = DEEP ? 1 : 2;
  auto kern = gemm_chain_kernel<BN, S, MB, MT, AS>;
  constexpr size_t smem = 1024 + (size_t)S * (kBM * kBK * 2 + BN * kBK * 2) + (2 * S + 4) * 8 + 16 +
                          sk_extra_bytes<BN, DEEP, AS>();
  static bool attr = false;
  if (!attr) {
    ASTRAEA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  (void)which;
  ASTRAEA_TRY(launch_k(kern, dim3(a.grid), dim3(kThreads), smem, st, maps, a));
  return 0;
}

template <int BN, bool DEEP>
int launch_chain(const ChainMaps& maps, const ChainArgs& a, cudaStream_t st) {
  // token-loop bound: the next power of two >= M (its own instantiation, so
  // the per-phase epilogue code a small batch executes stays small)
  if constexpr (BN == 16) {
    if (a.M <= 1) return launch_chain_mt<BN, DEEP, 1>(maps, a, st, 1);
    if (a.M <= 2) return launch_chain_mt<BN, DEEP, 2>(maps, a, st, 2);
    if (a.M <= 4) return launch_chain_mt<BN, DEEP, 4>(maps, a, st, 3);
    if (a.M <= 8) return launch_chain_mt<BN, DEEP, 8>(maps, a, st, 4);
  }
  return launch_chain_mt<BN, DEEP, BN>(maps, a, st, 0);
}

int to_epi(const astraea_epilogue* in, int N, Epi* e) {
  *e = Epi{};
  if (!in) return 0;
  e->kind = in->kind;
  if (in->kind < EPI_NONE || in->kind > EPI_ARGMAX) return ASTRAEA_EINVAL;
  e->amax = in->argmax_keys_dev;
  e->amax_off = in->argmax_col_offset;
  if (e->kind == EPI_ARGMAX && !e->amax) return ASTRAEA_EINVAL;
  e->residual = (const bf16*)in->residual_dev;
  e->ssq_out = in->ssq_out_dev;
  e->ssq_in = in->ssq_in_dev;
  e->ssq_parts = in->ssq_in_parts;
  e->rms_dim = in->rms_dim;
  e->eps = in->rms_eps;
  if (e->kind == EPI_RESIDUAL && !e->residual) return ASTRAEA_EINVAL;
  if (e->ssq_in && (e->ssq_parts <= 0 || e->rms_dim <= 0)) return ASTRAEA_EINVAL;
  if (e->kind != EPI_RESIDUAL && e->kind != EPI_NONE && e->ssq_out) return ASTRAEA_EINVAL;
  if (e->kind == EPI_SILU && (N % 128)) return ASTRAEA_EINVAL;
  if (e->kind == EPI_QKV_ROPE) {
    const astraea_kv_geometry& g = in->geo;
    if (!in->pool_dev || !in->positions_dev || !in->slots_dev || (g.head_dim != 64 && g.head_dim != 128) ||
        in->num_q_heads <= 0 || N != (in->num_q_heads + 2 * g.num_kv_heads) * g.head_dim || in->layer < 0 ||
        in->layer >= g.num_layers)
      return ASTRAEA_EINVAL;
    e->pool = (bf16*)in->pool_dev;
    e->block_el = (long long)g.num_layers * 2 * g.num_kv_heads * g.block_tokens * g.head_dim;
    e->layer = in->layer;
    e->Hq = in->num_q_heads;
    e->Hkv = g.num_kv_heads;
    e->D = g.head_dim;
    e->bt = g.block_tokens;
    e->pos = in->positions_dev;
    e->slots = in->slots_dev;
    e->theta = in->rope_theta;
    e->cs = reinterpret_cast<const float2*>(in->rope_table_dev);
  }
  return 0;
}

}  // namespace

namespace astraea {
namespace tc {
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

struct MapKey {
  const void* ptr;
  long long rows, cols, ld;
  int box_rows;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && rows == o.rows && cols == o.cols && ld == o.ld && box_rows == o.box_rows;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = std::hash<const void*>()(k.ptr);
    h ^= std::hash<long long>()(k.rows * 1315423911ll + k.cols * 2654435761ll + k.ld) + 0x9e3779b9 + (h << 6);
    return h ^ (size_t)k.box_rows;
  }
};

// 2-D bf16 tensor [rows][cols] (row stride ld elements), box = kBK cols x box_rows rows, 128B swizzle.
int make_map(CUtensorMap* out, const void* ptr, long long rows, long long cols, long long ld, int box_rows) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  MapKey key{ptr, rows, cols, ld, box_rows};
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *out = it->second;
      return 0;
    }
  }
  EncodeTiledFn fn = encode_fn();
  if (!fn) return ASTRAEA_EUNSUPPORTED;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return ASTRAEA_EINVAL;
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, *out);
  return 0;
}

}  // namespace tc
}  // namespace astraea

static unsigned long long* g_trace = nullptr;
static int g_trace_slots = 0, g_trace_next = 0, g_trace_stride = 0;

extern "C" int astraea_debug_gemm_trace(void* buf, int32_t slots, int32_t slot_stride) {
  g_trace = (unsigned long long*)buf;
  g_trace_slots = slots;
  g_trace_stride = slot_stride;
  g_trace_next = 0;
  return ASTRAEA_OK;
}

extern "C" int astraea_rope_table(const int32_t* positions, int32_t T, int32_t head_dim, float theta,
                                  float* table, void* stream) {
  if (T < 0 || (head_dim != 64 && head_dim != 128) || !table) return ASTRAEA_EINVAL;
  if (T == 0) return ASTRAEA_OK;
  const int n = T * head_dim / 2;
  ASTRAEA_TRY(launch_k(rope_table_kernel, dim3((n + 255) / 256), dim3(256), 0, (cudaStream_t)stream, positions,
                       (int)T, (int)(head_dim / 2), theta, reinterpret_cast<float2*>(table)));
  return ASTRAEA_OK;
}

static size_t chain_ws_bytes(int M, int nph, const astraea_gemm_phase* ph) {
  size_t part = 0;
  for (int p = 0; p < nph; ++p) part = std::max(part, partial_bytes(M, sk_plan(M, ph[p].N, ph[p].K)));
  return kHeadBytes + part;
}

// K-splits of the CTA-pair GEMM (units = tiles x splits, dealt round-robin
// to the pairs; the last split of a tile finishes it, so its contributors
// come earlier on every pair). Only when the tiles leave pairs idle (small
// M, e.g. a short recompute prefill): at most pairs / tiles splits, >= 32
// k-blocks each. Measured on B200 (tools/gemm_bench.py, CUDA graph,
// profiles/r1_prefill_splitk.txt): the down projection at M <= 512 drops
// from 71-72 us to 47-54 us, the K = 4096 shapes at M <= 256 from 24.5-26
// to 22.7-24.7 us; splitting when tiles >= pairs is 1.2-4x slower (the fp32
// partial exchange through L2 outweighs the balance). ASTRAEA_PAIR_SPLITK=0
// disables, ASTRAEA_PAIR_SPLITS forces S (experiments).
static int pair_splits(int M, int N, int K) {
  static const bool on = [] {
    const char* e = getenv("ASTRAEA_PAIR_SPLITK");
    return !(e && e[0] == '0');
  }();
  static const int min_kbs = [] {
    const char* e = getenv("ASTRAEA_PAIR_SPLIT_MIN_KB");
    return e ? std::max(1, atoi(e)) : 32;
  }();
  static const int forced = [] {
    const char* e = getenv("ASTRAEA_PAIR_SPLITS");
    return e ? std::max(1, std::min(8, atoi(e))) : 0;
  }();
  if (!on) return 1;
  const int tiles = ((M + 255) / 256) * ((N + 255) / 256);
  const int pairs = num_sms() / 2;
  const int kb = (K + kBK - 1) / kBK;
  if (forced) return std::min(forced, std::max(1, kb / 4));
  if (tiles >= pairs) return 1;
  return std::max(1, std::min(std::min(pairs / tiles, kb / min_kbs), 8));
}
// One-CTA kernel plan for short prefills: BN and the split-K count that fill
// the SMs (>= 8 k-blocks per split, <= 4 splits).
struct RowsPlan {
  int bn, splits;
};
static RowsPlan rows_plan(int M, int N, int K) {
  RowsPlan p;
  static const int force_bn = [] {
    const char* e = getenv("ASTRAEA_ROWS_BN");
    return e ? atoi(e) : 0;
  }();
  // 256-column tiles once 128-column ones would need more than one wave
  // (gate/up at 128 tokens: 224 -> 112 CTAs, the activation tile read once
  // per 256 weight rows; 76 -> 67 us)
  p.bn = (N % 256 == 0 && (long long)((M + kBM - 1) / kBM) * ((N + 127) / 128) > num_sms()) ? 256 : 128;
  if (force_bn == 256 && N % 256 == 0) p.bn = 256;
  if (force_bn == 128) p.bn = 128;
  const long long tiles = (long long)((M + kBM - 1) / kBM) * ((N + p.bn - 1) / p.bn);
  const int nkb = (K + kBK - 1) / kBK;
  static const int max_splits = [] {
    const char* e = getenv("ASTRAEA_ROWS_SPLITS");
    return e ? std::max(1, std::min(8, atoi(e))) : 2;   // 128-token prefill 6.78 -> 6.68 ms; 4: no better
  }();
  static const int max_splits_long = [] {
    const char* e = getenv("ASTRAEA_ROWS_SPLITS_LONG");
    return e ? std::max(1, std::min(8, atoi(e))) : 3;   // down at 128 tokens: 63.7 (CTA pairs) -> 47.5 us
  }();
  int s = 1;
  const int cap = nkb > 64 ? max_splits_long : max_splits;
  if (tiles < num_sms()) s = (int)std::min<long long>(num_sms() / tiles, cap);   // one wave
  s = std::max(1, std::min(s, nkb / 8));
  p.splits = s;
  return p;
}
static bool short_rows(int M, int N, int K) {
  static const int long_k = [] {
    const char* e = getenv("ASTRAEA_ROWS_LONGK");
    return e ? atoi(e) : 1;
  }();
  static const int long_k_m = [] {
    const char* e = getenv("ASTRAEA_ROWS_LONGK_M");
    return e ? atoi(e) : 256;   // down projection at 129-256 tokens: 63 -> 48 us (CTA pairs -> split-K rows)
  }();
  static const int rows_m = [] {
    const char* e = getenv("ASTRAEA_ROWS_M");
    return e ? atoi(e) : 512;   // QKV / O at 257-512 tokens: 54 / 38 -> 40-51 / 28 us (one wave of 128-row tiles)
  }();
  if (long_k && (M <= 128 || (M <= long_k_m && N <= 8192))) return true;
  return K <= 4096 && (M <= 128 || (M <= rows_m && N <= 6144));
}
static size_t rows_partial_bytes(int M, int N, int K) {
  const RowsPlan p = rows_plan(M, N, K);
  if (p.splits <= 1) return 0;
  const long long tiles = (long long)((M + kBM - 1) / kBM) * ((N + p.bn - 1) / p.bn);
  return (size_t)tiles * p.splits * kBM * p.bn * sizeof(float);
}

static size_t pair_partial_bytes(int M, int N, int K) {
  const int S = pair_splits(M, N, K);
  const long long tiles = (long long)((M + 255) / 256) * ((N + 255) / 256);
  return (size_t)tiles * (S - 1) * 2 * 128 * 256 * sizeof(unsigned long long);
}

extern "C" size_t astraea_gemm_workspace_bytes(int32_t M, int32_t N, int32_t K) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  if (M > kColsMaxM) {
    const size_t p = short_rows(M, N, K) ? rows_partial_bytes(M, N, K) : pair_partial_bytes(M, N, K);
    return p ? kHeadBytes + p : 0;
  }
  return kHeadBytes + partial_bytes(M, sk_plan(M, N, K));
}

extern "C" size_t astraea_gemm_chain_workspace_bytes(int32_t M, int32_t nphases, const astraea_gemm_phase* phases) {
  if (M <= 0 || M > kColsMaxM || nphases <= 0 || nphases > kMaxPhases || !phases) return 0;
  return chain_ws_bytes(M, nphases, phases);
}

// Build and launch a chain of 1..kMaxPhases decode GEMMs (M <= 64 tokens).
static int run_chain(int M, int nph, const astraea_gemm_phase* ph, void* ws, size_t ws_bytes, bool deep,
                     cudaStream_t st, int nattn = 0, const astraea_attn_phase* ats = nullptr,
                     const int32_t* attn_before = nullptr) {
  if (M <= 0 || M > kColsMaxM || nph <= 0 || nph > kMaxPhases) return ASTRAEA_EINVAL;
  if (!ws || ws_bytes < chain_ws_bytes(M, nph, ph)) return ASTRAEA_EINVAL;
  ChainMaps maps;
  ChainArgs a;
  a.trace = nullptr;
  if (g_trace && g_trace_slots > 0) {
    a.trace = g_trace + (size_t)(g_trace_next % g_trace_slots) * g_trace_stride;
    ++g_trace_next;
  }
  a.counters = (int*)ws;
  a.phase_ctr = (int*)((char*)ws + kCounterBytes);
  a.ws = (float*)((char*)ws + kHeadBytes);
  a.nattn = 0;
  a.pf_layer = -1;
  if (nattn < 0 || nattn > kMaxAttn || (nattn && (!ats || !attn_before || !deep))) return ASTRAEA_EINVAL;
  for (int k = 0; k < nattn; ++k) {
    const astraea_attn_phase* at = ats + k;
    const astraea_kv_geometry& g = at->geo;
    if (!at->pool_dev || !at->q_dev || !at->table_dev || !at->ctx_dev || !at->out_dev || g.block_tokens != 16 ||
        g.num_kv_heads <= 0 || g.num_kv_heads > 32 || at->num_q_heads % g.num_kv_heads || at->layer < 0 ||
        at->layer >= g.num_layers || at->max_blocks <= 0 || attn_before[k] < 0 || attn_before[k] >= nph ||
        (k && attn_before[k] <= attn_before[k - 1]))
      return ASTRAEA_EINVAL;
    const int G = at->num_q_heads / g.num_kv_heads, D = g.head_dim;
    a.attn_kind[k] = (D == 128 && G == 4) ? 1 : (D == 64 && G == 2) ? 2 : (D == 64 && G == 4) ? 3
                   : (D == 128 && G == 8) ? 4 : 0;   // 4: a Llama-3-70B TP=8 rank (8 q heads on 1 kv head)
    if (!a.attn_kind[k] || num_sms() > 192) return ASTRAEA_EUNSUPPORTED;
    a.attn_before[k] = attn_before[k];
    attn::AttnWork& w = a.at[k];
    w.pool = (const bf16*)at->pool_dev;
    w.block_el = (long long)astraea_kv_block_bytes(&g) / 2;
    w.layer = at->layer;
    w.Hq = at->num_q_heads;
    w.Hkv = g.num_kv_heads;
    w.q = (const bf16*)at->q_dev;
    w.q_stride = at->q_row_stride;
    w.table = at->table_dev;
    w.max_blocks = at->max_blocks;
    w.ctx = at->ctx_dev;
    w.out = (bf16*)at->out_dev;
    w.scale_log2 = at->scale * 1.4426950408889634f;
    w.ws = (unsigned long long*)((char*)ws + kCounterBytes + kPhaseBytes);
    w.tag = 0;        // set on the device from the launch epoch
    w.prefetch = 0;   // no wait before the page loads: nothing to overlap
    static const int min_pages = [] {
      const char* e = getenv("ASTRAEA_CHAIN_ATTN_MIN_PAGES");
      return e ? std::max(1, atoi(e)) : 2;   // pages per warp: measured best at batch 1-16
    }();
    w.min_pages = min_pages;
    w.M = M;
    if (ph[attn_before[k]].A != at->out_dev) return ASTRAEA_EINVAL;   // the attention output is that phase's A
    static const bool pf = [] {
      const char* e = getenv("ASTRAEA_CHAIN_KV_PREFETCH");
      return e && e[0] == '1';   // measured neutral at batch 1, -3% at batch 16: off
    }();
    a.pf_layer = (pf && at->layer + 1 < g.num_layers) ? at->layer + 1 : -1;
  }
  a.nattn = nattn;
  a.block_rows = 0;
  static const int trace_phase = [] {
    const char* e = getenv("ASTRAEA_TRACE_PHASE");
    return e ? atoi(e) : 2;
  }();
  a.trace_phase = trace_phase;
  if (nattn > 0) {
    // the TMA-staged attention instantiations (AS > 1) read pages through
    // this map; every attention of a launch uses the same pool
    const astraea_kv_geometry& g = ats[0].geo;
    for (int k = 1; k < nattn; ++k)
      if (ats[k].pool_dev != ats[0].pool_dev || ats[k].geo.num_blocks != g.num_blocks ||
          ats[k].geo.head_dim != g.head_dim || ats[k].geo.num_kv_heads != g.num_kv_heads ||
          ats[k].geo.num_layers != g.num_layers)
        return ASTRAEA_EINVAL;
    a.block_rows = g.num_layers * 2 * g.num_kv_heads * g.block_tokens;
    const int rc = make_map(&maps.pool, ats[0].pool_dev, (long long)g.num_blocks * a.block_rows, g.head_dim,
                            g.head_dim, g.block_tokens);
    if (rc) return rc;
  }
  static const int attn_early = [] {
    const char* e = getenv("ASTRAEA_CHAIN_ATTN_EARLY");
    return e ? atoi(e) : 1;
  }();
  a.attn_early = attn_early;
  a.M = M;
  a.grid = num_sms();
  a.nph = nph;
  static const int l2_pre = [] {
    const char* e = getenv("ASTRAEA_CHAIN_L2PRE");
    return e ? atoi(e) : 0;
  }();
  a.l2_pre = deep ? l2_pre : 0;
  const int bn = M <= 16 ? 16 : (M <= 32 ? 32 : 64);
  for (int p = 0; p < nph; ++p) {
    const astraea_gemm_phase& q = ph[p];
    if (q.N <= 0 || q.K <= 0 || q.lda < q.K || q.ldw < q.K || (q.lda % 8) || (q.ldw % 8) || (q.N % 8))
      return ASTRAEA_EINVAL;
    Epi e;
    int rc = to_epi(&q.epi, q.N, &e);
    if (rc) return rc;
    const int out_cols = e.kind == EPI_SILU ? q.N / 2 : (e.kind == EPI_QKV_ROPE ? e.Hq * e.D : q.N);
    if ((q.C && (q.ldc < out_cols || (q.ldc % 8))) || (!q.C && e.kind != EPI_ARGMAX)) return ASTRAEA_EINVAL;
    const SkPlan pl = sk_plan(M, q.N, q.K);
    if ((size_t)pl.tiles * sizeof(int) > kCounterBytes) return ASTRAEA_EUNSUPPORTED;
    SkPhase& P = a.ph[p];
    P.C = (bf16*)q.C;
    P.M = M;
    P.N = q.N;
    P.K = q.K;
    P.ldc = q.ldc;
    P.tiles = pl.tiles;
    P.kbs = pl.kbs;
    P.maxseg = pl.maxseg;
    P.units = pl.units;
    P.geff = (int)std::min<long long>(a.grid, pl.units);
    P.epi = e;
    if ((rc = make_map(&maps.w[p], q.W, q.N, q.K, q.ldw, kBM))) return rc;
    if ((rc = make_map(&maps.x[p], q.A, M, q.K, q.lda, bn))) return rc;
  }
  if (deep) {
    if (bn == 16) return launch_chain<16, true>(maps, a, st);
    if (bn == 32) return launch_chain<32, true>(maps, a, st);
    return launch_chain<64, true>(maps, a, st);
  }
  if (bn == 16) return launch_chain<16, false>(maps, a, st);
  if (bn == 32) return launch_chain<32, false>(maps, a, st);
  return launch_chain<64, false>(maps, a, st);
}

extern "C" int astraea_gemm_chain(int32_t M, int32_t nphases, const astraea_gemm_phase* phases, void* ws,
                                  size_t ws_bytes, void* stream) {
  if (!phases) return ASTRAEA_EINVAL;
  return run_chain(M, nphases, phases, ws, ws_bytes, true, (cudaStream_t)stream);
}

extern "C" int astraea_gemm_chain_attn(int32_t M, int32_t nattn, const astraea_attn_phase* attn,
                                       const int32_t* attn_before, int32_t nphases, const astraea_gemm_phase* phases,
                                       void* ws, size_t ws_bytes, void* stream) {
  if (!phases || !attn || nattn <= 0) return ASTRAEA_EINVAL;
  return run_chain(M, nphases, phases, ws, ws_bytes, true, (cudaStream_t)stream, nattn, attn, attn_before);
}

extern "C" int astraea_gemm_bf16_ex(const void* A, int32_t lda, const void* W, int32_t ldw, void* C, int32_t ldc,
                                    int32_t M, int32_t N, int32_t K, const astraea_epilogue* epi, void* ws,
                                    size_t ws_bytes, void* stream) {
  if (M < 0 || N <= 0 || K <= 0 || lda < K || ldw < K) return ASTRAEA_EINVAL;
  if ((lda % 8) || (ldw % 8) || (ldc % 8) || (N % 8)) return ASTRAEA_EINVAL;
  Epi e;
  int rc = to_epi(epi, N, &e);
  if (rc) return rc;
  const int out_cols = e.kind == EPI_SILU ? N / 2 : (e.kind == EPI_QKV_ROPE ? e.Hq * e.D : N);
  if (C && ldc < out_cols) return ASTRAEA_EINVAL;
  if (!C && e.kind != EPI_ARGMAX) return ASTRAEA_EINVAL;
  if (M == 0) return ASTRAEA_OK;
  cudaStream_t st = (cudaStream_t)stream;
  static const int chain_max_m = [] {
    const char* e = getenv("ASTRAEA_GEMM_CHAIN_MAX_M");
    // a single GEMM of 33-64 rows (a short prefill) runs faster on the
    // one-CTA kernel than on the BN = 64 stream-K kernel, whose epilogue
    // loops over 64 tokens: 64-token prefill 8.33 -> 5.52 ms
    return e ? std::min(kColsMaxM, std::max(1, atoi(e))) : 32;
  }();
  if (M <= chain_max_m) {
    astraea_gemm_phase ph;
    ph.A = A;
    ph.lda = lda;
    ph.W = W;
    ph.ldw = ldw;
    ph.C = C;
    ph.ldc = ldc;
    ph.N = N;
    ph.K = K;
    ph.epi = epi ? *epi : astraea_epilogue{};
    return run_chain(M, 1, &ph, ws, ws_bytes, false, st);
  }
  CUtensorMap ma, mb;
  GemmArgs a{};
  a.C = (bf16*)C;
  a.M = M;
  a.N = N;
  a.K = K;
  a.ldc = ldc;
  a.epi = e;
  // Short prefills (recompute-on-resume appends) are weight-streaming bound:
  // there the one-CTA 128-row tiles keep more SMs streaming than 256x256
  // CTA-pair tiles -- every projection at M <= 128 (down included, split-K
  // over up to 3 CTAs: 63.7 -> 47.5 us), N <= 8192 ones at M <= 256 (down:
  // 63 -> 48 us) and N <= 6144 ones (QKV, O) at M <= 512 (tools/gpu_r2t.sh sweep: 128 tokens 50 -> 37 us QKV, 37.5 ->
  // 31.8 O, 90.5 -> 76 gate/up per layer; profiles/r2_prefill_rows_v2.txt).
  const bool rows_short = short_rows(M, N, K);
  a.trace = nullptr;
  a.trace_ctas = 0;
  if (g_trace && g_trace_slots > 0) {
    a.trace = g_trace + (size_t)(g_trace_next % g_trace_slots) * g_trace_stride;
    a.trace_ctas = g_trace_stride / 16;
    ++g_trace_next;
  }
  a.splits = 1;
  a.rpart = nullptr;
  a.rctr = nullptr;
  if (pair_gemm_enabled() && !rows_short) {
    if ((rc = make_map(&ma, A, M, K, lda, 128))) return rc;
    if ((rc = make_map(&mb, W, N, K, ldw, 128))) return rc;
    a.splits = pair_splits(M, N, K);
    a.part = nullptr;
    a.ctr = nullptr;
    if (a.splits > 1) {
      if (ws && ws_bytes >= kHeadBytes + pair_partial_bytes(M, N, K)) {
        a.ctr = (int*)((char*)ws + kCounterBytes);
        a.part = (unsigned long long*)((char*)ws + kHeadBytes);
      } else {
        a.splits = 1;   // no workspace: unsplit (fewer pairs busy, same result)
      }
    }
    return launch_pair<6>(ma, mb, a, st);
  }
  const RowsPlan rp = rows_plan(M, N, K);
  const int bn = rp.bn;
  int splits = rows_short ? rp.splits : 1;
  const long long rtiles = (long long)((M + kBM - 1) / kBM) * ((N + bn - 1) / bn);
  if (splits > 1) {
    if (ws && ws_bytes >= kHeadBytes + rows_partial_bytes(M, N, K) && rtiles * sizeof(int) <= kCounterBytes) {
      a.rpart = (float*)((char*)ws + kHeadBytes);
      a.rctr = (int*)ws;   // the tile counters (zero between uses, as for the chain)
    } else {
      splits = 1;          // no workspace: unsplit (fewer SMs busy, same result)
    }
  }
  if ((rc = make_map(&ma, A, M, K, lda, kBM))) return rc;
  if ((rc = make_map(&mb, W, N, K, ldw, bn))) return rc;
  dim3 grid((M + kBM - 1) / kBM, (N + bn - 1) / bn, splits);
  if (bn == 256) return launch_rows<256, 4>(ma, mb, a, grid, st);
  return launch_rows<128, 6>(ma, mb, a, grid, st);
}

extern "C" int astraea_gemm_bf16(const void* A, int32_t lda, const void* W, int32_t ldw, void* C, int32_t ldc,
                                 int32_t M, int32_t N, int32_t K, const void* residual, int32_t epilogue,
                                 void* ws, size_t ws_bytes, void* stream) {
  if (epilogue != ASTRAEA_EPI_NONE && epilogue != ASTRAEA_EPI_RESIDUAL) return ASTRAEA_EINVAL;
  astraea_epilogue e = {};
  e.kind = epilogue;
  e.residual_dev = residual;
  return astraea_gemm_bf16_ex(A, lda, W, ldw, C, ldc, M, N, K, &e, ws, ws_bytes, stream);
}
