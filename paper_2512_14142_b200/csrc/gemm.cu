// K6 / K9: bf16 GEMM on 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
//   C[M][N] = A[M][K] . W[N][K]^T  (+ residual)
//
// These are the dense projections of the recompute-on-resume prefill and of
// every decode step -- the work the reference reduces to the profile lookup
// prefill_seconds(n_in + extra) and n_gen * seconds_per_token
// (pkg/src/agentsched/predictor.py:47-66, simulator.py:329-337).
//
// Kernel anatomy (one output tile per CTA, 192 threads):
//   warp 0      TMA producer: 128B-swizzled A/B tiles into a smem ring
//               (cp.async.bulk.tensor.2d, mbarrier complete_tx);
//   warp 1      allocates TMEM; one elected lane issues tcgen05.mma
//               (kind::f16, M=128, fp32 accumulators in TMEM) and commits
//               each stage back to the producer with tcgen05.commit;
//   warps 2..5  epilogue: tcgen05.ld 32x32b -> registers -> global.
//
// Two operand orientations:
//   kRows  (prefill, M large): MMA M axis = rows of A (tokens), N axis =
//          rows of W; bf16 output (+ residual) stored directly.
//   kCols  (decode, M <= 64): MMA M axis = rows of W (128 output features),
//          N axis = the M tokens padded to 16/32/64 ("swap AB"), with
//          split-K across CTAs so the weight stream covers all SMs; the
//          last CTA of each tile reduces the fp32 partials in split order
//          (deterministic) and applies the bf16 (+ residual) epilogue.
#include <cuda.h>

#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "common.cuh"

using namespace astraea;

namespace {

constexpr int kBM = 128;   // MMA M
constexpr int kBK = 64;    // K per stage = one 128-byte swizzle atom of bf16
constexpr int kThreads = 192;

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

enum Orient { kRows = 0, kCols = 1 };

struct GemmArgs {
  bf16* C;
  const bf16* residual;
  float* ws;          // kCols split-K: fp32 [splits][M][N] partials
  int* counters;      // kCols split-K: per-tile arrival counters (zero between launches)
  int M, N, K, ldc;
  int kb_per_split;   // K blocks per CTA (split-K)
};

// BN: MMA N (tile width along the N axis of the MMA).
template <int BN, int STAGES, int ORIENT>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                const __grid_constant__ GemmArgs args) {
  // map_a feeds the MMA "A" (M axis, 128 rows), map_b the MMA "B" (BN rows).
  constexpr int A_BYTES = kBM * kBK * 2;
  constexpr int B_BYTES = BN * kBK * 2;
  constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile_a = blockIdx.x;   // along the MMA M axis (128)
  const int tile_b = blockIdx.y;   // along the MMA N axis (BN)
  const int split = blockIdx.z;
  const int total_kb = (args.K + kBK - 1) / kBK;
  const int kb0 = split * args.kb_per_split;
  const int kb1 = min(total_kb, kb0 + args.kb_per_split);
  const int nkb = kb1 - kb0;

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

  pdl_launch();
  if (warp == 0) {
    if (lane == 0) {
      // Weights (map_b) do not depend on the previous kernel: prefetch the
      // first stages before the grid-dependency wait.
      const int pre = min(nkb, STAGES);
      for (int i = 0; i < pre; ++i) {
        mbar_arrive_expect_tx(&full[i], A_BYTES + B_BYTES);
        tma_load_2d(sb + i * B_BYTES, &map_b, &full[i], (kb0 + i) * kBK, tile_b * BN);
      }
      pdl_wait();
      for (int i = 0; i < pre; ++i) tma_load_2d(sa + i * A_BYTES, &map_a, &full[i], (kb0 + i) * kBK, tile_a * kBM);
      for (int i = pre; i < nkb; ++i) {
        const int s = i % STAGES;
        mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], A_BYTES + B_BYTES);
        const int kc = (kb0 + i) * kBK;
        tma_load_2d(sa + s * A_BYTES, &map_a, &full[s], kc, tile_a * kBM);
        tma_load_2d(sb + s * B_BYTES, &map_b, &full[s], kc, tile_b * BN);
      }
    }
  } else if (warp == 1) {
    pdl_wait();
    constexpr uint32_t idesc = instr_desc(BN);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % STAGES;
      mbar_wait(&full[s], (i / STAGES) & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint64_t da = smem_desc_sw128(sa + s * A_BYTES);
        const uint64_t db = smem_desc_sw128(sb + s * B_BYTES);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {
          // advance 16 bf16 = 32 bytes along K inside the swizzle atom (>>4 -> +2)
          mma_bf16(tmem, da + 2 * k, db + 2 * k, idesc, (i | k) != 0);
        }
        mma_commit(&empty[s]);
        if (i == nkb - 1) mma_commit(done);
      }
      __syncwarp();
    }
    if (nkb == 0 && lane == 0) mbar_arrive(done);
  } else {
    // epilogue: warps 2..5 -> TMEM lane quarter (warp % 4)
    pdl_wait();
    const int quarter = warp & 3;
    mbar_wait(done, 0);
    tc_fence_after();
    const int row_in_tile = quarter * 32 + lane;
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
    if constexpr (ORIENT == kRows) {
      const int m = tile_a * kBM + row_in_tile;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        tmem_ld32(lane_addr + c0, v);
        const int n0 = tile_b * BN + c0;
        if (m < args.M && nkb > 0) {
          bf16* dst = args.C + (long long)m * args.ldc + n0;
          if (n0 + 32 <= args.N) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float o[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) o[e] = v[q * 8 + e];
              if (args.residual) {
                float r[8];
                unpack8(*reinterpret_cast<const uint4*>(args.residual + (long long)m * args.ldc + n0 + q * 8), r);
#pragma unroll
                for (int e = 0; e < 8; ++e) o[e] += r[e];
              }
              *reinterpret_cast<uint4*>(dst + q * 8) = pack8(o);
            }
          } else {
            for (int e = 0; e < 32 && n0 + e < args.N; ++e) {
              float o = v[e];
              if (args.residual) o += bf2f(args.residual[(long long)m * args.ldc + n0 + e]);
              dst[e] = f2bf(o);
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, TMEM_COLS);
}

// ---------------------------------------------------------------------------
// Decode GEMM: persistent stream-K on tcgen05 (swap-AB orientation).
//
// MMA A = W rows (128 output features per tile), MMA B = the M <= 64 tokens
// (BN = 16/32/64). The tiles x k-blocks work units are split evenly over one
// CTA per SM, so every SM streams the same number of weight bytes (the
// roofline of a decode step is the weight stream). A CTA walks its units
// in order: the TMA ring runs continuously across tile boundaries, the MMA
// warp accumulates each tile *segment* into one of two TMEM accumulators,
// and the epilogue drains the other. Segments that cover a whole tile are
// written directly; split tiles are fixed up deterministically -- each
// segment stores an fp32 partial, the last to arrive sums them in segment
// order and applies the bf16 (+ residual) epilogue.
// ---------------------------------------------------------------------------
struct SkArgs {
  bf16* C;
  const bf16* residual;
  float* ws;        // [tiles][maxseg][M][128] partials
  int* counters;    // [tiles] arrival counters, zero between launches
  int M, N, K, ldc;
  int tiles, kbs, grid, maxseg;
  long long units;
};

__device__ __forceinline__ int sk_owner(long long u, long long units, int grid) {
  return (int)(((u + 1) * grid - 1) / units);
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 2)
    gemm_streamk_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x,
                        const __grid_constant__ SkArgs args) {
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
  __shared__ int s_last;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const long long U = args.units;
  const long long u0 = (long long)cta * U / args.grid;
  const long long u1 = (long long)(cta + 1) * U / args.grid;
  const int KB = args.kbs;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_w) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
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
    if (lane == 0) {
      // Weight tiles are independent of the previous kernel: stream the first
      // STAGES of them while the predecessor drains, then wait for it and
      // fetch the matching activation tiles.
      const int pre = (int)(u1 - u0 < STAGES ? u1 - u0 : STAGES);
      for (int i = 0; i < pre; ++i) {
        const long long u = u0 + i;
        mbar_arrive_expect_tx(&full[i], A_BYTES + B_BYTES);
        tma_load_2d(sa + i * A_BYTES, &map_w, &full[i], (int)(u % KB) * kBK, (int)(u / KB) * kBM);
      }
      pdl_wait();
      for (int i = 0; i < pre; ++i) tma_load_2d(sb + i * B_BYTES, &map_x, &full[i], (int)((u0 + i) % KB) * kBK, 0);
      int i = pre;
      for (long long u = u0 + pre; u < u1; ++u, ++i) {
        const int s = i % STAGES;
        mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], A_BYTES + B_BYTES);
        const int tile = (int)(u / KB), kc = (int)(u % KB) * kBK;
        tma_load_2d(sa + s * A_BYTES, &map_w, &full[s], kc, tile * kBM);
        tma_load_2d(sb + s * B_BYTES, &map_x, &full[s], kc, 0);
      }
    }
  } else if (warp == 1) {
    pdl_wait();
    constexpr uint32_t idesc = instr_desc(BN);
    int i = 0, seg = 0;
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
  } else {
    pdl_wait();
    const int quarter = warp & 3;
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
    const int row = quarter * 32 + lane;  // feature within the tile
    int seg = 0;
    for (long long u = u0; u < u1; ++seg) {
      const long long tile = u / KB;
      const long long seg_end = min(u1, (tile + 1) * KB);
      const bool whole = (u == tile * KB) && (seg_end == (tile + 1) * KB);
      u = seg_end;
      const int buf = seg & 1;
      mbar_wait(&tfull[buf], (seg >> 1) & 1);
      tc_fence_after();
      float v[BN < 32 ? 32 : BN];
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 32) tmem_ld32(lane_addr + buf * BN + c0, v + c0);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      const int f = (int)tile * kBM + row;
      const bool fok = f < args.N;
      if (whole) {
#pragma unroll
        for (int t = 0; t < BN; ++t) {
          if (t < args.M && fok) {
            float o = v[t];
            if (args.residual) o += bf2f(args.residual[(long long)t * args.ldc + f]);
            args.C[(long long)t * args.ldc + f] = f2bf(o);
          }
        }
        continue;
      }
      const long long first_u = tile * KB;
      const int c_first = sk_owner(first_u, U, args.grid);
      const int nseg = sk_owner(first_u + KB - 1, U, args.grid) - c_first + 1;
      const int sidx = cta - c_first;
      float* part = args.ws + ((tile * args.maxseg + sidx) * (long long)args.M) * kBM;
#pragma unroll
      for (int t = 0; t < BN; ++t)
        if (t < args.M) __stcg(part + (long long)t * kBM + row, v[t]);
      __threadfence();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 64) s_last = atomicAdd(args.counters + tile, 1) == nseg - 1;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (s_last) {
        __threadfence();
        const float* base = args.ws + (tile * args.maxseg * (long long)args.M) * kBM + row;
        for (int t = 0; t < args.M; ++t) {
          float o = 0.f;
          for (int sg = 0; sg < nseg; ++sg) o += __ldcg(base + ((long long)sg * args.M + t) * kBM);
          if (fok) {
            if (args.residual) o += bf2f(args.residual[(long long)t * args.ldc + f]);
            args.C[(long long)t * args.ldc + f] = f2bf(o);
          }
        }
        if (threadIdx.x == 64) args.counters[tile] = 0;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, TMEM_COLS);
}

// ---- host side ----------------------------------------------------------------------------

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

template <int BN, int STAGES>
constexpr size_t smem_bytes() {
  return 1024 + (size_t)STAGES * (kBM * kBK * 2 + BN * kBK * 2) + (2 * STAGES + 1) * 8 + 16;
}

template <int BN, int STAGES, int ORIENT>
int launch(const CUtensorMap& ma, const CUtensorMap& mb, const GemmArgs& a, dim3 grid, cudaStream_t st) {
  auto kern = gemm_kernel<BN, STAGES, ORIENT>;
  constexpr size_t smem = smem_bytes<BN, STAGES>();
  static bool attr = false;
  if (!attr) {
    ASTRAEA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  ASTRAEA_TRY(launch_k(kern, grid, dim3(kThreads), smem, st, ma, mb, a));
  return 0;
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
  p.grid = (int)std::min<long long>(num_sms(), p.units);
  p.maxseg = (p.grid + p.tiles - 1) / p.tiles + 1;
  return p;
}

// Workspace layout: a fixed counter region shared by every GEMM shape (so
// GEMMs of different tile counts reuse one workspace in stream order without
// clobbering each other's counters), then the fp32 partials.
constexpr size_t kCounterBytes = 16384 * sizeof(int);

size_t sk_ws_bytes(int M, const SkPlan& p) {
  return kCounterBytes + (size_t)p.tiles * p.maxseg * M * kBM * sizeof(float);
}

template <int BN>
constexpr int sk_stages() {
  // ~100 KB: two CTAs fit per SM, so the next GEMM's CTA can become resident
  // and prefetch its weights (PDL) while this one drains.
  return (100 * 1024) / (kBM * kBK * 2 + BN * kBK * 2);
}

template <int BN>
int launch_sk(const CUtensorMap& mw, const CUtensorMap& mx, const SkArgs& a, cudaStream_t st) {
  constexpr int S = sk_stages<BN>();
  auto kern = gemm_streamk_kernel<BN, S>;
  constexpr size_t smem = 1024 + (size_t)S * (kBM * kBK * 2 + BN * kBK * 2) + (2 * S + 4) * 8 + 16;
  static bool attr = false;
  if (!attr) {
    ASTRAEA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  ASTRAEA_TRY(launch_k(kern, dim3(a.grid), dim3(kThreads), smem, st, mw, mx, a));
  return 0;
}

}  // namespace

extern "C" size_t astraea_gemm_workspace_bytes(int32_t M, int32_t N, int32_t K) {
  if (M <= 0 || M > kColsMaxM || N <= 0 || K <= 0) return 0;
  return sk_ws_bytes(M, sk_plan(M, N, K));
}

extern "C" int astraea_gemm_bf16(const void* A, int32_t lda, const void* W, int32_t ldw, void* C, int32_t ldc,
                                 int32_t M, int32_t N, int32_t K, const void* residual, int32_t epilogue,
                                 void* ws, size_t ws_bytes, void* stream) {
  if (M < 0 || N <= 0 || K <= 0 || lda < K || ldw < K || ldc < N) return ASTRAEA_EINVAL;
  if ((lda % 8) || (ldw % 8) || (ldc % 8) || (N % 8)) return ASTRAEA_EINVAL;
  if (epilogue == ASTRAEA_EPI_RESIDUAL && !residual) return ASTRAEA_EINVAL;
  if (epilogue == ASTRAEA_EPI_NONE) residual = nullptr;
  if (M == 0) return ASTRAEA_OK;
  cudaStream_t st = (cudaStream_t)stream;
  CUtensorMap ma, mb;
  int rc;
  if (M <= kColsMaxM) {
    const SkPlan p = sk_plan(M, N, K);
    if (!ws || ws_bytes < sk_ws_bytes(M, p)) return ASTRAEA_EINVAL;
    if ((size_t)p.tiles * sizeof(int) > kCounterBytes) return ASTRAEA_EUNSUPPORTED;
    SkArgs a;
    a.C = (bf16*)C;
    a.residual = (const bf16*)residual;
    a.counters = (int*)ws;
    a.ws = (float*)((char*)ws + kCounterBytes);
    a.M = M;
    a.N = N;
    a.K = K;
    a.ldc = ldc;
    a.tiles = p.tiles;
    a.kbs = p.kbs;
    a.grid = p.grid;
    a.maxseg = p.maxseg;
    a.units = p.units;
    if ((rc = make_map(&ma, W, N, K, ldw, kBM))) return rc;
    if ((rc = make_map(&mb, A, M, K, lda, p.bn))) return rc;
    if (p.bn == 16) return launch_sk<16>(ma, mb, a, st);
    if (p.bn == 32) return launch_sk<32>(ma, mb, a, st);
    return launch_sk<64>(ma, mb, a, st);
  }
  GemmArgs a;
  a.C = (bf16*)C;
  a.residual = (const bf16*)residual;
  a.ws = nullptr;
  a.counters = nullptr;
  a.M = M;
  a.N = N;
  a.K = K;
  a.ldc = ldc;
  a.kb_per_split = (K + kBK - 1) / kBK;
  const int bn = (N % 256 == 0 && (long long)((M + kBM - 1) / kBM) * (N / 256) >= num_sms()) ? 256 : 128;
  if ((rc = make_map(&ma, A, M, K, lda, kBM))) return rc;
  if ((rc = make_map(&mb, W, N, K, ldw, bn))) return rc;
  dim3 grid((M + kBM - 1) / kBM, (N + bn - 1) / bn, 1);
  if (bn == 256) return launch<256, 4, kRows>(ma, mb, a, grid, st);
  return launch<128, 6, kRows>(ma, mb, a, grid, st);
}
