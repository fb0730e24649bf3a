// One decode step of the scheduler's mixed batch as ONE persistent kernel.
//
// The reference models a decode step as n_gen * seconds_per_token
// (pkg/src/agentsched/simulator.py:329-337, predictor.py:60-66). On B200 the
// step is bound by streaming every weight byte from HBM once (15 GB for
// Llama-3-8B), so the kernel is organised around an uninterrupted weight
// stream and everything else hides under it:
//
//   program   a list of phases in global memory (astraea_step_phase):
//             GEMM phases (QKV+RoPE+KV-append, O+residual, gate/up+SiLU,
//             down+residual, lm_head+argmax -- the fused epilogues of
//             tc.cuh) and ATTN phases (paged decode attention of one layer);
//   dataflow  no grid-wide barriers. Every phase publishes per-chunk ready
//             flags (one per 128-feature GEMM tile, one per kv head for
//             attention) holding the launch epoch; a consumer waits only for
//             the chunks it reads, so phases overlap across CTAs and a
//             straggler delays only its own dependants;
//   roles     (224 threads, one CTA per SM, all CTAs co-resident)
//             warp 0  weight producer: TMA weight tiles of every GEMM phase
//                     into the smem ring in stream-K order, never waiting on
//                     data dependencies (and optionally L2 prefetches further
//                     ahead); it starts before griddepcontrol.wait;
//             warp 6  activation producer: for each ring slot, waits for the
//                     producing chunk's flag (acquire), fences the async
//                     proxy and TMA-loads the activation k-block;
//             warp 1  tcgen05.mma issuer (M=128 weight rows x N=BN tokens,
//                     fp32 accumulators double-buffered in TMEM);
//             warps 2-5  epilogue: drain TMEM, deterministic stream-K fix-up,
//                     fused epilogue, publish tile flags; in ATTN phases they
//                     run the paged attention (K/V pages read straight from
//                     the pool into registers, warp-shuffle online softmax,
//                     deterministic split merge) while warp 0 keeps
//                     streaming the next projection's weights.
//
// Safety of the overlap (why no barrier is needed): a GEMM tile is finished
// only after all k-blocks of its input, and every projection's input spans
// all of the previous phase's output; attention of head h needs q/k/v of
// head h, and the O projection needs every head. Hence every read of a
// buffer by phase p completes before phase p+2 can finish anything, which
// makes all write-after-read reuse of x/q/att/h/statistics safe, and lets
// stream-K partials and counters alternate between two regions.
#include <cuda.h>

#include <algorithm>
#include <cstring>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "tc.cuh"
#include "attn_mma.cuh"

using namespace astraea;
using namespace astraea::tc;
using namespace astraea::attn;

namespace {

constexpr int kMkThreads = 224;
constexpr int kEpiThreads = 128;
#ifndef MK_RING_KB
#define MK_RING_KB 220
#endif
constexpr int kRingBytes = MK_RING_KB * 1024;
constexpr int kBT = 16;
constexpr int kAttnSmem = kBT * 128 * 2;   // per attention warp: one V page (D <= 128), bf16

enum { PK_GEMM = 0, PK_ATTN = 1 };

struct AttnDesc {
  const bf16* pool;
  long long block_el;
  int layer, Hq, Hkv, D, G;
  const bf16* q;
  int q_stride;
  const int32_t* table;
  int max_blocks;
  const int32_t* ctx;
  bf16* out;            // [M][Hq*D]
  float scale_log2;
  const int* qkv_flags; // tile flags of the QKV phase (128 features per tile)
  int* seq_ctr;         // [M][Hkv] split arrival counters
  int* head_ctr;        // [Hkv] finished rows per head
  float* ws;            // [4*grid][2][G][D+2] split partials
  int min_pages;
};

struct alignas(128) MkPhase {
  CUtensorMap wmap;     // GEMM: W [N][K]
  CUtensorMap xmap;     // GEMM: A [M][K]
  int kind;
  int M;
  // dependencies (flags hold the launch epoch when ready)
  const int* x_flags;   // chunks of A (nullptr: ready at launch)
  int x_chunk_cols;
  const int* dep_flags; // what the epilogue reads from an earlier phase (RMS stats / residual)
  int n_dep;
  int* out_flags;       // this phase's chunk flags
  // GEMM
  bf16* C;
  int N, K, ldc, tiles, kbs, geff;
  int units;            // tiles * kbs (< 2^31 / grid)
  unsigned long long* partials;   // [grid][2][M][128] tagged fp32 (bits | tag << 32)
  Epi epi;
  AttnDesc attn;
};

struct MkState {
  int epoch;            // completed launches
  int exit_ctr;
};

__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_all() { asm volatile("fence.proxy.async;" ::: "memory"); }
__device__ __forceinline__ void l2_prefetch_tile(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map), "r"(c0), "r"(c1)
               : "memory");
}
// Ready flags: one per 128-byte line (no false sharing between the writer
// and the pollers of neighbouring chunks). Polls are relaxed loads; the
// acquire is a fence after the flag was seen.
constexpr int kFlagStride = 32;
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ bool flag_set(const int* flags, int i, int epoch) {
  return ld_relaxed(flags + i * kFlagStride) == epoch;
}
__device__ __forceinline__ void l2_prefetch_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void spin_flag(const int* flags, int i, int epoch) {
  int ns = 64;
  while (!flag_set(flags, i, epoch)) {
    __nanosleep(ns);
    ns = ns < 512 ? 2 * ns : 512;
  }
  fence_acquire();
}
__device__ __forceinline__ void set_flag(int* flags, int i, int epoch) {
#if defined(MK_UNSAFE_NOFENCE)   // perf experiment only: no release ordering
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(flags + i * kFlagStride), "r"(epoch) : "memory");
#elif defined(MK_FLAG_FENCE_RELAXED)
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(flags + i * kFlagStride), "r"(epoch) : "memory");
#else
  st_release(flags + i * kFlagStride, epoch);
#endif
}
__device__ __forceinline__ int warp_max_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}


__device__ __forceinline__ void mk_range(const MkPhase& P, int cta, int& u0, int& u1) {
  const int g = P.geff;
  if (cta < g) {
    u0 = cta * P.units / g;
    u1 = (cta + 1) * P.units / g;
  } else {
    u0 = u1 = P.units;
  }
}
__device__ __forceinline__ int mk_owner(int u, int units, int g) {
  return ((u + 1) * g - 1) / units;
}

// Walks the (GEMM phase, unit) sequence of one CTA; used for L2 prefetch.
struct UnitCursor {
  int p;
  int u, u1;
  __device__ void seek(const MkPhase* prog, int nph, int cta, int from) {
    for (p = from; p < nph; ++p) {
      if (prog[p].kind != PK_GEMM) continue;
      int a, b;
      mk_range(prog[p], cta, a, b);
      if (a < b) {
        u = a;
        u1 = b;
        return;
      }
    }
  }
  __device__ bool valid(int nph) const { return p < nph; }
  __device__ void next(const MkPhase* prog, int nph, int cta) {
    if (++u >= u1) seek(prog, nph, cta, p + 1);
  }
};

// Acquire the QKV tiles head h reads (q heads hG.., k head h, v head h).
__device__ __forceinline__ void attn_wait_qkv(const AttnDesc& A, int h, int epoch, int lane) {
  const int D = A.D;
  const int q0 = (h * A.G * D) / 128, q1 = ((h + 1) * A.G * D - 1) / 128;
  const int k0 = (A.Hq * D + h * D) / 128, k1 = (A.Hq * D + (h + 1) * D - 1) / 128;
  const int v0 = ((A.Hq + A.Hkv) * D + h * D) / 128, v1 = ((A.Hq + A.Hkv) * D + (h + 1) * D - 1) / 128;
  const int nq = q1 - q0 + 1, nk = k1 - k0 + 1, nv = v1 - v0 + 1;
  if (lane < nq + nk + nv) {
    const int t = lane < nq ? q0 + lane : (lane < nq + nk ? k0 + lane - nq : v0 + lane - nq - nk);
    spin_flag(A.qkv_flags, t, epoch);
  }
  __syncwarp();
}

// One layer's attention by the 4 epilogue warps of every CTA. The (row, kv
// head) sequences' pages are split evenly over the CTAs; inside a CTA the
// four warps take every fourth page of the CTA's piece and merge in shared
// memory, so each sequence has at most one partial per CTA. The last CTA to
// finish a split sequence merges the partials (CTA order: deterministic); the
// kv head's flag is raised when all M rows of that head are written.
template <int D, int G>
__device__ __noinline__ void attn_phase(const MkPhase& P, int epoch, int cta, int grid, int warp, int lane, bf16* vs_all,
                                        int* out_flags, unsigned long long* atr) {
  // atr (diagnostics, may be null): this warp's first piece: [0] entry,
  // [1] q/k/v flags seen, [2] q loaded, [3] pages done, [4] CTA merge +
  // partial published, [5] split merge done, [6] output published, [7] exit
  auto mark = [&](int k, bool first) {
    if (atr && first && lane == 0) atr[k] = gtimer();
  };
  mark(0, true);
  const AttnDesc& A = P.attn;
  const int M = P.M, Hkv = A.Hkv;
  const int et = warp * 32 + lane;
  bf16* vs = vs_all + warp * (kAttnSmem / 2);
  // pages per row (retired rows count one empty page so that every (row, head) is written)
  int pg0 = 0, pg1 = 0;
  if (lane < M) pg0 = max(1, (__ldg(A.ctx + lane) + kBT - 1) / kBT);
  if (lane + 32 < M) pg1 = max(1, (__ldg(A.ctx + lane + 32) + kBT - 1) / kBT);
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
  const int maxpg = warp_max_i(max(pg0, pg1));
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
    const long long k_off = ((long long)(A.layer * 2) * A.Hkv + h) * kBT * D;
    const long long v_off = ((long long)(A.layer * 2 + 1) * A.Hkv + h) * kBT * D;
    for (int p = cur - seq0 + warp + 4 * lane; p < pe - seq0; p += 128) {
      const int blk = p * kBT < ctx_b ? __ldg(trow + p) : -1;
      if (blk >= 0) {
        const bf16* page = A.pool + (long long)blk * A.block_el;
        l2_prefetch_bulk(page + k_off, kBT * D * 2);
        l2_prefetch_bulk(page + v_off, kBT * D * 2);
      }
    }
    cur = pe;
  }
  __shared__ int s_attn_last;
  constexpr int EPT = (G * D + kEpiThreads - 1) / kEpiThreads;   // merged elements per thread
  unsigned heads_ready = 0;
  for (int cur = my0; cur < my1;) {
    int b, h, seq0, seq1, pe;
    resolve(cur, b, h, seq0, seq1, pe);
    const int pa = cur - seq0, pb = pe - seq0;
    const bool first_piece = cur == my0;
    if (!(heads_ready >> h & 1)) {
      attn_wait_qkv(A, h, epoch, lane);
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
          const float* ws = reinterpret_cast<const float*>(vs_all + w * (kAttnSmem / 2));
          const float mk = ws[g], mn = fmaxf(Mv[e], mk);
          const float a0 = mn == -INFINITY ? 0.f : exp2f(Mv[e] - mn), a1 = mn == -INFINITY ? 0.f : exp2f(mk - mn);
          Lv[e] = Lv[e] * a0 + ws[G + g] * a1;
          Ov[e] = Ov[e] * a0 + ws[2 * G + g * D + dd] * a1;
          Mv[e] = mn;
        }
      }
    }
    const int first_c = seq0 / qc, last_c = (seq1 - 1) / qc;
    const int nparts = last_c - first_c + 1;
    bool done = nparts == 1;
    if (!done) {
      // CTA partial (layout m[G], l[G], o[G][D]); slot 0: the CTA's first piece
      float* part = A.ws + ((long long)cta * 2 + (first_piece ? 0 : 1)) * G * (D + 2);
#pragma unroll
      for (int e = 0; e < EPT; ++e) {
        const int idx = et * EPT + e, g = idx / D, dd = idx % D;
        if (idx < G * D) {
          __stcg(part + 2 * G + idx, Ov[e]);
          if (dd == 0) {
            __stcg(part + g, Mv[e]);
            __stcg(part + G + g, Lv[e]);
          }
        }
      }
      // publish the partial: one release/acquire RMW for the CTA after the
      // barrier (cumulativity), as in the GEMM fix-up
      epi_bar();
      int* ctr = A.seq_ctr + b * Hkv + h;
      if (et == 0) s_attn_last = atom_add_acq_rel(ctr, 1) == nparts - 1;
      epi_bar();
      mark(4, first_piece);
      if (s_attn_last) {
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
          Mv[e] = -INFINITY;
          Lv[e] = 0.f;
          Ov[e] = 0.f;
        }
        for (int c0 = first_c; c0 <= last_c; c0 += 8) {
          float pm[8][EPT], pl[8][EPT], po[8][EPT];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int c = c0 + k;
            const float* pp = A.ws + ((long long)c * 2 + ((c == first_c && c * qc < seq0) ? 1 : 0)) * G * (D + 2);
#pragma unroll
            for (int e = 0; e < EPT; ++e) {
              const int idx = et * EPT + e, g = idx / D;
              const bool ok = c <= last_c && idx < G * D;
              pm[k][e] = ok ? __ldcg(pp + g) : -INFINITY;
              pl[k][e] = ok ? __ldcg(pp + G + g) : 0.f;
              po[k][e] = ok ? __ldcg(pp + 2 * G + idx) : 0.f;
            }
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
#pragma unroll
            for (int e = 0; e < EPT; ++e) {
              const float mn = fmaxf(Mv[e], pm[k][e]);
              const float a0 = mn == -INFINITY ? 0.f : exp2f(Mv[e] - mn);
              const float a1 = mn == -INFINITY ? 0.f : exp2f(pm[k][e] - mn);
              Lv[e] = Lv[e] * a0 + pl[k][e] * a1;
              Ov[e] = Ov[e] * a0 + po[k][e] * a1;
              Mv[e] = mn;
            }
          }
        }
        if (et == 0) *ctr = 0;
        done = true;
        mark(5, first_piece);
      }
    }
    if (done) {
      bf16* out = A.out + (long long)b * (A.Hq * D) + (long long)h * G * D;
#pragma unroll
      for (int e = 0; e < EPT; ++e) {
        const int idx = et * EPT + e;
        if (idx < G * D) out[idx] = f2bf(Lv[e] > 0.f ? Ov[e] / Lv[e] : 0.f);
      }
      // publish: the O projection reads att through TMA (async proxy)
      fence_proxy_async_all();
      epi_bar();
      if (et == 0) {
        if (atom_add_acq_rel(A.head_ctr + h, 1) == M - 1) {
          A.head_ctr[h] = 0;
          set_flag(out_flags, h, epoch);
        }
      }
    }
    mark(6, first_piece);
    epi_bar();   // the warps' shared-memory states are rewritten by the next piece
    cur = pe;
  }
  mark(7, true);
}

__device__ void attn_dispatch(const MkPhase& P, int epoch, int cta, int grid, int warp, int lane, bf16* vs,
                              unsigned long long* atr) {
  const int D = P.attn.D, G = P.attn.G;
  if (D == 128 && G == 4) attn_phase<128, 4>(P, epoch, cta, grid, warp, lane, vs, P.out_flags, atr);
#ifndef MK_ONLY_8B
  else if (D == 64 && G == 2) attn_phase<64, 2>(P, epoch, cta, grid, warp, lane, vs, P.out_flags, atr);
  else if (D == 64 && G == 4) attn_phase<64, 4>(P, epoch, cta, grid, warp, lane, vs, P.out_flags, atr);
#endif
}

constexpr size_t kSmemMax = 232448 - 4096;   // 227 KB per CTA, less static shared memory and slack
template <int BN>
constexpr size_t mk_fixed() {   // everything but the ring
  return 1024 + 4 * 8 + 64 + (size_t)BN * kBM * 2 + 5 * BN * sizeof(float) + 128 + 4 * (size_t)kAttnSmem + 64;
}
template <int BN>
constexpr int mk_stages() {
  constexpr size_t stage = kBM * kBK * 2 + BN * kBK * 2 + 16;   // tiles + two mbarriers
  constexpr size_t room = kSmemMax - mk_fixed<BN>();
  return (int)((kRingBytes < room ? (size_t)kRingBytes : room) / stage);
}
template <int BN>
constexpr size_t mk_smem() {
  return mk_fixed<BN>() + (size_t)mk_stages<BN>() * (kBM * kBK * 2 + BN * kBK * 2 + 16);
}

template <int BN>
__global__ void __launch_bounds__(kMkThreads, 1)
    decode_step_kernel(const MkPhase* __restrict__ prog, int nph, MkState* state, int l2_ahead,
                       unsigned long long* trace) {
  constexpr int S = mk_stages<BN>();
  constexpr int A_BYTES = kBM * kBK * 2;
  constexpr int B_BYTES = BN * kBK * 2;
  constexpr uint32_t TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + S * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + S * B_BYTES);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  bf16* xch = reinterpret_cast<bf16*>(tmem_slot + 16);            // [BN][128]
  float* red = reinterpret_cast<float*>(xch + BN * kBM);      // [4][BN]
  float* rs = red + 4 * BN;                                   // [BN]
  bf16* vs_all = reinterpret_cast<bf16*>(
      (reinterpret_cast<uintptr_t>(rs + BN) + 127) & ~uintptr_t(127));   // [4][16][D] V pages (attention)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x, grid = gridDim.x;
  // diagnostics: trace[(cta * nph + p) * 8 + k] = %globaltimer when
  //   k=0 the weight producer issued phase p's first tile, k=1 the activation
  //   producer issued its first k-block, k=2 the epilogue finished phase p,
  //   k=3 the MMA warp finished phase p, k=4 the epilogue began its segments,
  //   k=5 the last split's partials were seen, k=6 the last accumulator
  //   arrived, k=7 the last tile was finished; trace[grid*nph*8 + cta] = entry.
  auto stamp = [&](int p, int k) {
    if (trace) trace[((long long)cta * nph + p) * 8 + k] = gtimer();
  };
  if (trace && threadIdx.x == 0) trace[(long long)grid * nph * 8 + cta] = gtimer();

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 2);   // weight + activation producers each arrive (with their tx bytes)
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_launch();

  if (warp == 0) {
    // ---- weight producer: independent of every data dependency
    if (lane == 0) {
      UnitCursor pf;
      pf.seek(prog, nph, cta, 0);
      for (int k = 0; k < l2_ahead && pf.valid(nph); ++k) {
        const MkPhase& Q = prog[pf.p];
        l2_prefetch_tile(&Q.wmap, (int)(pf.u % Q.kbs) * kBK, (int)(pf.u / Q.kbs) * kBM);
        pf.next(prog, nph, cta);
      }
      int idx = 0;
      for (int p = 0; p < nph; ++p) {
        const MkPhase& P = prog[p];
        if (P.kind != PK_GEMM) continue;
        asm volatile("prefetch.tensormap [%0];" ::"l"(&P.wmap) : "memory");
        int u0, u1;
        mk_range(P, cta, u0, u1);
        const int KB = P.kbs;
        for (int u = u0; u < u1; ++u, ++idx) {
          const int s = idx % S;
          if (idx >= S) mbar_wait(&empty[s], ((idx / S) - 1) & 1);
          if (u == u0) stamp(p, 0);
          mbar_arrive_expect_tx(&full[s], A_BYTES);
          tma_load_2d(sa + s * A_BYTES, &P.wmap, &full[s], (int)(u % KB) * kBK, (int)(u / KB) * kBM);
          if (l2_ahead > 0 && pf.valid(nph)) {
            const MkPhase& Q = prog[pf.p];
            l2_prefetch_tile(&Q.wmap, (int)(pf.u % Q.kbs) * kBK, (int)(pf.u / Q.kbs) * kBM);
            pf.next(prog, nph, cta);
          }
        }
      }
    }
  } else if (warp == 6) {
    // ---- activation producer (whole warp polls flags, lane 0 issues the TMA):
    // a k-block is loaded once the chunk producing it is flagged; missing
    // chunks are re-polled all at once (one memory round trip per poll).
    pdl_wait();
    const int epoch = __ldcg(&state->epoch) + 1;
    int idx = 0;
    for (int p = 0; p < nph; ++p) {
      const MkPhase& P = prog[p];
      if (P.kind != PK_GEMM) continue;
      if (lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&P.xmap) : "memory");
      int u0, u1;
      mk_range(P, cta, u0, u1);
      const int KB = P.kbs;
      const int* xf = P.x_flags;
      const int ccols = P.x_chunk_cols;
      const int nchunks = xf ? (P.K + ccols - 1) / ccols : 0;
      for (int u = u0; u < u1; ++u, ++idx) {
        const int s = idx % S;
        const int kb = u % KB;
        if (xf && u == u0) {
          // every k-block of this phase's activations is read by this CTA's
          // range (a full tile spans all of K): wait for all producer chunks
          for (;;) {
            bool all = true;
            for (int ch = lane; ch < nchunks; ch += 32) all &= flag_set(xf, ch, epoch);
            if (__all_sync(0xffffffffu, all)) break;
            __nanosleep(128);
          }
          fence_acquire();
          if (lane == 0) fence_proxy_async_all();
        }
        if (lane == 0) {
          if (idx >= S) mbar_wait(&empty[s], ((idx / S) - 1) & 1);
          if (u == u0) stamp(p, 1);
          mbar_arrive_expect_tx(&full[s], B_BYTES);
          tma_load_2d(sb + s * B_BYTES, &P.xmap, &full[s], kb * kBK, 0);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer
    constexpr uint32_t idesc = instr_desc(BN);
    int i = 0, seg = 0;
    for (int p = 0; p < nph; ++p) {
      const MkPhase& P = prog[p];
      if (P.kind != PK_GEMM) continue;
      int u0, u1;
      mk_range(P, cta, u0, u1);
      const int KB = P.kbs;
      for (int u = u0; u < u1; ++seg) {
        const int seg_end = min(u1, (u / KB + 1) * KB);
        const int buf = seg & 1;
        if (seg >= 2) mbar_wait(&tempty[buf], ((seg >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + buf * BN;
        const int seg_begin = u;
        for (; u < seg_end; ++u, ++i) {
          const int s = i % S;
          mbar_wait(&full[s], (i / S) & 1);
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
      if (lane == 0) stamp(p, 3);
    }
  } else {
    // ---- epilogue / attention warps (2..5)
    pdl_wait();
    const int epoch = __ldcg(&state->epoch) + 1;
    const int ew = warp - 2;                 // 0..3
    const int quarter = warp & 3;            // TMEM lane quarter of this warp
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
    const int row = quarter * 32 + lane;     // feature within the tile
    const int et = threadIdx.x - 64;         // 0..127
    int seg = 0;
    for (int p = 0; p < nph; ++p) {
      const MkPhase& P = prog[p];
      if (P.kind == PK_ATTN) {
        attn_dispatch(P, epoch, cta, grid, ew, lane, vs_all,
                      (trace && p == 1) ? trace + (long long)grid * nph * 8 + grid + (cta * 4 + ew) * 16 : nullptr);
        epi_bar();
        if (et == 0) stamp(p, 2);
        continue;
      }
      const int M = P.M;
      const int KB = P.kbs;
      const int U = P.units;
      int u0, u1;
      mk_range(P, cta, u0, u1);
      // What the epilogue reads from earlier phases (RMS statistics, the
      // residual) is acquired up front, while the MMA warp fills the first
      // accumulator, so it is off the phase's critical tail.
      if (u0 < u1) {
        for (int i = et; i < P.n_dep; i += kEpiThreads) spin_flag(P.dep_flags, i, epoch);
        epi_bar();
        if (P.epi.ssq_in) {
          if (row < M) rs[row] = rms_scale(P.epi, M, row);
          epi_bar();
        }
      }
      const bool resid = P.epi.kind == EPI_RESIDUAL;
      auto publish = [&](int tile) {
#ifndef MK_NO_PUBLISH_FENCE
        fence_proxy_async_all();   // consumers read C with TMA
#endif
        epi_bar();
        if (et == 0) set_flag(P.out_flags, tile, epoch);
      };
      // Split tiles: the CTA that owns the tile's first k-blocks (c_first)
      // finishes it. Its segment is the end of its range, while the other
      // segments open the ranges of c_first+1.. -- so their partials are
      // normally published long before, and c_first sums them (CTA order,
      // deterministic) while its own last MMAs still run: the fix-up is off
      // the phase's critical tail (no arrival counter, no round trip after
      // the last MMA).
      const int tag = (epoch << 8) | (p & 255);
      if (et == 0) stamp(p, 4);
      for (int u = u0; u < u1; ++seg) {
        const int tile = u / KB;
        const int seg_end = min(u1, (tile + 1) * KB);
        const bool whole = (u == tile * KB) && (seg_end == (tile + 1) * KB);
        const bool first_seg = u == u0;
        u = seg_end;
        const int buf = seg & 1;
        const int first_u = tile * KB;
        const int c_first = whole ? cta : mk_owner(first_u, U, P.geff);
        const int c_last = whole ? cta : mk_owner(first_u + KB - 1, U, P.geff);
        const bool finisher = cta == c_first;
        const int f = tile * kBM + row;
        float res[BN], acc[BN];
        if (finisher) {
          // the residual of this tile's features, loaded before the accumulator wait
          if (resid) {
#pragma unroll
            for (int t = 0; t < BN; ++t)
              res[t] = (t < M && f < P.N) ? bf2f(__ldcg(P.epi.residual + (long long)t * P.ldc + f)) : 0.f;
          }
#pragma unroll
          for (int t = 0; t < BN; ++t) acc[t] = 0.f;
          if (!whole) {
            // Partials are self-validating 64-bit words (fp32 bits | tag << 32,
            // single-copy atomic): each thread spins on its own values, so
            // waiting and loading are one round trip and need no flag.
            constexpr int GRP = 1;
            for (int c0 = c_first + 1; c0 <= c_last; c0 += GRP) {
              unsigned long long pv[GRP][BN];
#pragma unroll
              for (int k = 0; k < GRP; ++k) {
                const int c = c0 + k;
                const unsigned long long* pp = P.partials + ((long long)(c * 2) * M) * kBM + row;   // slot 0
#pragma unroll
                for (int t = 0; t < BN; ++t) pv[k][t] = (c <= c_last && t < M) ? ld_relaxed_u64(pp + (long long)t * kBM) : 0ull;
              }
#pragma unroll
              for (int k = 0; k < GRP; ++k) {
                const int c = c0 + k;
                if (c <= c_last) {
                  const unsigned long long* pp = P.partials + ((long long)(c * 2) * M) * kBM + row;
#pragma unroll
                  for (int t = 0; t < BN; ++t) {
                    if (t < M) {
                      while ((unsigned)(pv[k][t] >> 32) != (unsigned)tag) pv[k][t] = ld_relaxed_u64(pp + (long long)t * kBM);
                      acc[t] += __uint_as_float((unsigned)pv[k][t]);
                    }
                  }
                }
              }
            }
            if (et == 0) stamp(p, 5);
          }
        }
        mbar_wait(&tfull[buf], (seg >> 1) & 1);
        if (et == 0) stamp(p, 6);
        tc_fence_after();
        float v[BN < 32 ? 32 : BN];
#pragma unroll
        for (int c0 = 0; c0 < BN; c0 += 32) tmem_ld32(lane_addr + buf * BN + c0, v + c0);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        if (!finisher) {
          // contributor: publish this segment's tagged fp32 partial (slot 0 = first segment of the range)
          const int slot = first_seg ? 0 : 1;
          unsigned long long* part = P.partials + ((long long)(cta * 2 + slot) * M) * kBM + row;
#pragma unroll
          for (int t = 0; t < BN; ++t)
            if (t < M) st_relaxed_u64(part + (long long)t * kBM, (unsigned long long)__float_as_uint(v[t]) |
                                                                  ((unsigned long long)(unsigned)tag << 32));
          continue;
        }
        if (!whole) {
#pragma unroll
          for (int t = 0; t < BN; ++t) v[t] = acc[t] + v[t];
        }
        sk_finish<BN>(P, tile, row, v, rs, xch, red, resid ? res : nullptr);
        publish(tile);
        if (et == 0) stamp(p, 7);
      }
      if (et == 0) stamp(p, 2);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, TMEM_COLS);
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&state->exit_ctr, 1) == grid - 1) {
      state->exit_ctr = 0;
      state->epoch = state->epoch + 1;
      __threadfence();
    }
  }
}

unsigned long long* g_step_trace = nullptr;

template <int BN>
int launch_step(const MkPhase* prog, int nph, MkState* state, int l2_ahead, cudaStream_t st) {
  auto kern = decode_step_kernel<BN>;
  constexpr size_t smem = mk_smem<BN>();
  static bool attr = false;
  if (!attr) {
    ASTRAEA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  ASTRAEA_TRY(launch_k(kern, dim3(num_sms()), dim3(kMkThreads), smem, st, prog, nph, state, l2_ahead, g_step_trace));
  return 0;
}

int gemm_out_chunk_cols(const astraea_step_phase& p) {
  return p.gemm.epi.kind == ASTRAEA_EPI_SILU ? 64 : 128;
}

struct Layout {
  size_t state = 0, flags = 0, regions = 0, region_bytes = 0, attn = 0, total = 0;
  std::vector<size_t> flag_off;
  int max_tiles = 0;
  size_t attn_seq = 0, attn_head = 0, attn_ws = 0;
};

int plan_layout(int M, int nph, const astraea_step_phase* ph, Layout& L) {
  const int grid = num_sms();
  size_t off = 256;   // MkState
  L.flag_off.resize(nph);
  int maxHkv = 0, maxG = 0, maxD = 0;
  for (int p = 0; p < nph; ++p) {
    int n = 0;
    if (ph[p].kind == ASTRAEA_PHASE_GEMM) {
      n = (ph[p].gemm.N + kBM - 1) / kBM;
      L.max_tiles = std::max(L.max_tiles, n);
    } else if (ph[p].kind == ASTRAEA_PHASE_ATTN) {
      n = ph[p].geo.num_kv_heads;
      maxHkv = std::max(maxHkv, n);
      maxG = std::max(maxG, ph[p].num_q_heads / std::max(1, n));
      maxD = std::max(maxD, ph[p].geo.head_dim);
    } else {
      return ASTRAEA_EINVAL;
    }
    L.flag_off[p] = off;
    off += (size_t)n * kFlagStride * sizeof(int);
  }
  off = (off + 255) & ~size_t(255);
  L.regions = off;
  L.region_bytes = (size_t)grid * 2 * M * kBM * sizeof(unsigned long long);
  off += 2 * L.region_bytes;
  L.attn = off;
  L.attn_seq = off;
  off += (((size_t)M * std::max(1, maxHkv) * sizeof(int)) + 255) & ~size_t(255);
  L.attn_head = off;
  off += 256;
  L.attn_ws = off;
  off += (size_t)4 * grid * 2 * std::max(1, maxG) * (std::max(1, maxD) + 2) * sizeof(float);
  L.total = off;
  return 0;
}

}  // namespace

extern "C" size_t astraea_step_program_bytes(int32_t nphases) {
  return nphases > 0 ? (size_t)nphases * sizeof(MkPhase) : 0;
}

extern "C" size_t astraea_step_workspace_bytes(int32_t M, int32_t nphases, const astraea_step_phase* phases) {
  if (M <= 0 || M > 64 || nphases <= 0 || !phases) return 0;
  Layout L;
  if (plan_layout(M, nphases, phases, L)) return 0;
  return L.total;
}

extern "C" int astraea_step_program_build(int32_t M, int32_t nph, const astraea_step_phase* ph, void* prog_host,
                                          size_t prog_bytes, void* ws_dev, size_t ws_bytes) {
  if (M <= 0 || M > 64 || nph <= 0 || nph > 255 || !ph || !prog_host || !ws_dev) return ASTRAEA_EINVAL;
  if (prog_bytes < (size_t)nph * sizeof(MkPhase)) return ASTRAEA_EINVAL;
  Layout L;
  int rc = plan_layout(M, nph, ph, L);
  if (rc) return rc;
  if (ws_bytes < L.total) return ASTRAEA_EINVAL;
  char* ws = (char*)ws_dev;
  const int bn = M <= 16 ? 16 : (M <= 32 ? 32 : 64);
  const int grid = num_sms();
  MkPhase* host = (MkPhase*)prog_host;
  int gemm_idx = 0;
  for (int p = 0; p < nph; ++p) {
    MkPhase& P = host[p];
    memset(&P, 0, sizeof(P));
    const astraea_step_phase& q = ph[p];
    P.kind = q.kind == ASTRAEA_PHASE_GEMM ? PK_GEMM : PK_ATTN;
    P.M = M;
    P.out_flags = (int*)(ws + L.flag_off[p]);
    auto flags_of = [&](int from) -> const int* { return from >= 0 ? (const int*)(ws + L.flag_off[from]) : nullptr; };
    auto nflags_of = [&](int from) -> int {
      if (from < 0) return 0;
      return ph[from].kind == ASTRAEA_PHASE_GEMM ? (ph[from].gemm.N + kBM - 1) / kBM : ph[from].geo.num_kv_heads;
    };
    if (q.epi_from >= p || q.a_from >= p || (q.kind == ASTRAEA_PHASE_ATTN && (q.qkv_from < 0 || q.qkv_from >= p)))
      return ASTRAEA_EINVAL;   // dependencies must point backwards
    P.dep_flags = flags_of(q.epi_from);
    P.n_dep = nflags_of(q.epi_from);
    if (q.kind == ASTRAEA_PHASE_GEMM) {
      const astraea_gemm_phase& g = q.gemm;
      if (g.N <= 0 || g.K <= 0 || g.lda < g.K || g.ldw < g.K || (g.lda % 8) || (g.ldw % 8) || (g.N % 8))
        return ASTRAEA_EINVAL;
      Epi e = {};
      // reuse the GEMM library's epilogue validation
      e.kind = g.epi.kind;
      if (e.kind < EPI_NONE || e.kind > EPI_ARGMAX) return ASTRAEA_EINVAL;
      e.amax = g.epi.argmax_keys_dev;
      e.amax_off = g.epi.argmax_col_offset;
      e.residual = (const bf16*)g.epi.residual_dev;
      e.ssq_out = g.epi.ssq_out_dev;
      e.ssq_in = g.epi.ssq_in_dev;
      e.ssq_parts = g.epi.ssq_in_parts;
      e.rms_dim = g.epi.rms_dim;
      e.eps = g.epi.rms_eps;
      if ((e.kind == EPI_ARGMAX && !e.amax) || (e.kind == EPI_RESIDUAL && !e.residual) ||
          (e.ssq_in && (e.ssq_parts <= 0 || e.rms_dim <= 0)) || (e.kind == EPI_SILU && (g.N % 128)))
        return ASTRAEA_EINVAL;
      if (e.kind == EPI_QKV_ROPE) {
        const astraea_kv_geometry& gg = g.epi.geo;
        if (!g.epi.pool_dev || !g.epi.positions_dev || !g.epi.slots_dev || (gg.head_dim != 64 && gg.head_dim != 128) ||
            g.epi.num_q_heads <= 0 || g.N != (g.epi.num_q_heads + 2 * gg.num_kv_heads) * gg.head_dim)
          return ASTRAEA_EINVAL;
        e.pool = (bf16*)g.epi.pool_dev;
        e.block_el = (long long)gg.num_layers * 2 * gg.num_kv_heads * gg.block_tokens * gg.head_dim;
        e.layer = g.epi.layer;
        e.Hq = g.epi.num_q_heads;
        e.Hkv = gg.num_kv_heads;
        e.D = gg.head_dim;
        e.bt = gg.block_tokens;
        e.pos = g.epi.positions_dev;
        e.slots = g.epi.slots_dev;
        e.theta = g.epi.rope_theta;
        e.cs = reinterpret_cast<const float2*>(g.epi.rope_table_dev);
      }
      if (!g.C && e.kind != EPI_ARGMAX) return ASTRAEA_EINVAL;
      P.epi = e;
      P.C = (bf16*)g.C;
      P.N = g.N;
      P.K = g.K;
      P.ldc = g.ldc;
      P.tiles = (g.N + kBM - 1) / kBM;
      P.kbs = (g.K + kBK - 1) / kBK;
      if ((long long)P.tiles * P.kbs * grid >= (1ll << 31)) return ASTRAEA_EUNSUPPORTED;
      P.units = P.tiles * P.kbs;
      P.geff = std::min(grid, P.units);
      char* region = ws + L.regions + (size_t)(gemm_idx & 1) * L.region_bytes;
      P.partials = (unsigned long long*)region;
      ++gemm_idx;
      if (q.a_from >= 0) {
        const astraea_step_phase& src = ph[q.a_from];
        P.x_flags = flags_of(q.a_from);
        P.x_chunk_cols = src.kind == ASTRAEA_PHASE_GEMM ? gemm_out_chunk_cols(src)
                                                        : (src.num_q_heads / src.geo.num_kv_heads) * src.geo.head_dim;
        if (P.x_chunk_cols % kBK) return ASTRAEA_EINVAL;
        if (g.K / P.x_chunk_cols > 256) return ASTRAEA_EUNSUPPORTED;
      }
      if ((rc = make_map(&P.wmap, g.W, g.N, g.K, g.ldw, kBM))) return rc;
      if ((rc = make_map(&P.xmap, g.A, M, g.K, g.lda, bn))) return rc;
    } else {
      const astraea_kv_geometry& gg = q.geo;
      if (!q.pool_dev || !q.q_dev || !q.table_dev || !q.ctx_dev || !q.out_dev || gg.block_tokens != kBT ||
          gg.num_kv_heads <= 0 || q.num_q_heads % gg.num_kv_heads || q.layer < 0 || q.layer >= gg.num_layers)
        return ASTRAEA_EINVAL;
      const int G = q.num_q_heads / gg.num_kv_heads, D = gg.head_dim;
      if (!((D == 128 && G == 4) || (D == 64 && (G == 2 || G == 4)))) return ASTRAEA_EUNSUPPORTED;
      if (gg.num_kv_heads > 32 || G > 8 || D * kBT * 2 > kAttnSmem) return ASTRAEA_EUNSUPPORTED;
      const astraea_step_phase& src = ph[q.qkv_from];
      if (src.kind != ASTRAEA_PHASE_GEMM || src.gemm.epi.kind != ASTRAEA_EPI_QKV_ROPE) return ASTRAEA_EINVAL;
      AttnDesc& A = P.attn;
      A.pool = (const bf16*)q.pool_dev;
      A.block_el = (long long)astraea_kv_block_bytes(&gg) / 2;
      A.layer = q.layer;
      A.Hq = q.num_q_heads;
      A.Hkv = gg.num_kv_heads;
      A.D = D;
      A.G = G;
      A.q = (const bf16*)q.q_dev;
      A.q_stride = q.q_row_stride;
      A.table = q.table_dev;
      A.max_blocks = q.max_blocks;
      A.ctx = q.ctx_dev;
      A.out = (bf16*)q.out_dev;
      A.scale_log2 = q.scale * 1.4426950408889634f;
      A.qkv_flags = flags_of(q.qkv_from);
      A.seq_ctr = (int*)(ws + L.attn_seq);
      A.head_ctr = (int*)(ws + L.attn_head);
      A.ws = (float*)(ws + L.attn_ws);
      static int min_pages = [] {
        const char* e = getenv("ASTRAEA_ATTN_MIN_PAGES");
        return e ? std::max(1, atoi(e)) : 1;
      }();
      A.min_pages = min_pages;
    }
  }
  return ASTRAEA_OK;
}

extern "C" int astraea_debug_step_trace(void* buf) {
  g_step_trace = (unsigned long long*)buf;
  return ASTRAEA_OK;
}

extern "C" int astraea_step_launch(int32_t M, int32_t nph, const void* prog_dev, void* ws_dev, int32_t l2_ahead,
                                   void* stream) {
  if (M <= 0 || M > 64 || nph <= 0 || !prog_dev || !ws_dev) return ASTRAEA_EINVAL;
  const MkPhase* prog = (const MkPhase*)prog_dev;
  MkState* state = (MkState*)ws_dev;
  cudaStream_t st = (cudaStream_t)stream;
  if (M <= 16) return launch_step<16>(prog, nph, state, l2_ahead, st);
  if (M <= 32) return launch_step<32>(prog, nph, state, l2_ahead, st);
  return launch_step<64>(prog, nph, state, l2_ahead, st);
}
