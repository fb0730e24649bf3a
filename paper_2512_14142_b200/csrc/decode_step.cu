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
constexpr int kAttnSmem = attn::kAttnWarpBytes;   // per attention warp: one V page (D <= 128) + merge room

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
  int* head_ctr;        // [Hkv] finished rows per head
  unsigned long long* ws;   // [grid][G][D+2] tagged split partials
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

// The step kernel's attention phase: attn_cta_phase (attn_mma.cuh) with the
// QKV tile flags as the per-head dependency and the kv-head flag as output.
template <int D, int G>
__device__ __noinline__ void attn_phase(const MkPhase& P, int pidx, int epoch, int cta, int grid, int warp, int lane,
                                        bf16* vs_all, int* out_flags, unsigned long long* atr) {
  const AttnDesc& D_ = P.attn;
  AttnWork A;
  A.pool = D_.pool;
  A.block_el = D_.block_el;
  A.layer = D_.layer;
  A.Hq = D_.Hq;
  A.Hkv = D_.Hkv;
  A.q = D_.q;
  A.q_stride = D_.q_stride;
  A.table = D_.table;
  A.max_blocks = D_.max_blocks;
  A.ctx = D_.ctx;
  A.out = D_.out;
  A.scale_log2 = D_.scale_log2;
  A.ws = D_.ws;
  A.tag = ((unsigned)epoch << 8) | (unsigned)(pidx & 255);
  A.prefetch = 1;
  A.min_pages = D_.min_pages;
  A.M = P.M;
  auto wait_head = [&](int h, int ln) { attn_wait_qkv(D_, h, epoch, ln); };
  auto done_head = [&](int h, int et) {
    // publish: the O projection reads att through TMA (async proxy)
    fence_proxy_async_all();
    epi_bar();
    if (et == 0) {
      if (atom_add_acq_rel(D_.head_ctr + h, 1) == P.M - 1) {
        D_.head_ctr[h] = 0;
        set_flag(out_flags, h, epoch);
      }
    }
  };
  attn_cta_phase<D, G>(A, cta, grid, warp, lane, vs_all, wait_head, done_head, atr);
}

__device__ void attn_dispatch(const MkPhase& P, int pidx, int epoch, int cta, int grid, int warp, int lane, bf16* vs,
                              unsigned long long* atr) {
  const int D = P.attn.D, G = P.attn.G;
  if (D == 128 && G == 4) attn_phase<128, 4>(P, pidx, epoch, cta, grid, warp, lane, vs, P.out_flags, atr);
#ifndef MK_ONLY_8B
  else if (D == 64 && G == 2) attn_phase<64, 2>(P, pidx, epoch, cta, grid, warp, lane, vs, P.out_flags, atr);
  else if (D == 64 && G == 4) attn_phase<64, 4>(P, pidx, epoch, cta, grid, warp, lane, vs, P.out_flags, atr);
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
      (reinterpret_cast<uintptr_t>(rs + BN) + 127) & ~uintptr_t(127));   // [4][kAttnWarpBytes] (attention)

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
        attn_dispatch(P, p, epoch, cta, grid, ew, lane, vs_all,
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
      A.head_ctr = (int*)(ws + L.attn_head);
      A.ws = (unsigned long long*)(ws + L.attn_ws);
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
