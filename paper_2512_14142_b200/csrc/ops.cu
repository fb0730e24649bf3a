// K8 small fused ops of the Llama block: RMSNorm (+ residual add),
// SiLU(gate) * up, embedding gather, greedy argmax sampling.
// None of these exist in the reference (it has no model);
// they complete the recompute-prefill and decode steps whose durations the
// reference only predicts (predictor.py:47-66).
#include <float.h>

#include "common.cuh"

using namespace astraea;

namespace {

// One CTA per row; the row is held in registers as 8-element vectors.
template <int VPT>
__global__ void __launch_bounds__(256) rmsnorm_kernel(const bf16* __restrict__ x, const bf16* __restrict__ r,
                                                      const bf16* __restrict__ w, bf16* __restrict__ y,
                                                      bf16* __restrict__ resid_out, int dim, float eps) {
  const long long row = blockIdx.x;
  pdl_wait();
  pdl_launch();
  const int nvec = dim / 8;
  float v[VPT][8];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    if (i < nvec) {
      unpack8(*reinterpret_cast<const uint4*>(x + row * dim + i * 8), v[k]);
      if (r) {
        float rv[8];
        unpack8(*reinterpret_cast<const uint4*>(r + row * dim + i * 8), rv);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[k][e] += rv[e];
      }
      if (resid_out) {
        // the residual stream is kept in bf16, as the model's hidden state
        *reinterpret_cast<uint4*>(resid_out + row * dim + i * 8) = pack8(v[k]);
        float rt[8];
        unpack8(pack8(v[k]), rt);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[k][e] = rt[e];
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) ss += v[k][e] * v[k][e];
    }
  }
  __shared__ float red[32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / dim + eps);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    if (i < nvec) {
      float wv[8], o[8];
      unpack8(*reinterpret_cast<const uint4*>(w + i * 8), wv);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = v[k][e] * inv * wv[e];
      *reinterpret_cast<uint4*>(y + row * dim + i * 8) = pack8(o);
    }
  }
}

__global__ void silu_mul_kernel(const bf16* __restrict__ gu, bf16* __restrict__ out, int F, long long total_vec) {
  pdl_wait();
  pdl_launch();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total_vec;
       i += (long long)gridDim.x * blockDim.x) {
    const long long t = i / (F / 8);
    const int c = (int)(i % (F / 8));
    float g[8], u[8], o[8];
    unpack8(*reinterpret_cast<const uint4*>(gu + t * 2 * F + c * 8), g);
    unpack8(*reinterpret_cast<const uint4*>(gu + t * 2 * F + F + c * 8), u);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      // round silu(g) to bf16 first, as the reference bf16 model does
      const float s = bf2f(f2bf(g[e] / (1.f + __expf(-g[e]))));
      o[e] = s * u[e];
    }
    *reinterpret_cast<uint4*>(out + t * F + c * 8) = pack8(o);
  }
}

__global__ void embedding_kernel(const int32_t* __restrict__ ids, const bf16* __restrict__ table,
                                 bf16* __restrict__ out, int dim, float* __restrict__ ssq_out) {
  const long long t = blockIdx.x;
  pdl_wait();
  pdl_launch();
  const long long id = ids[t];
  float ss = 0.f;
  for (int i = threadIdx.x; i < dim / 8; i += blockDim.x) {
    const uint4 u = *reinterpret_cast<const uint4*>(table + id * dim + i * 8);
    *reinterpret_cast<uint4*>(out + t * dim + i * 8) = u;
    float f[8];
    unpack8(u, f);
#pragma unroll
    for (int k = 0; k < 8; ++k) ss += f[k] * f[k];
  }
  if (ssq_out) {
    __shared__ float red[32];
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
      float s = 0.f;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
      ssq_out[t] = s;
    }
  }
}

__global__ void __launch_bounds__(1024) argmax_kernel(const bf16* __restrict__ logits, int vocab,
                                                      int32_t* __restrict__ out) {
  const long long row = blockIdx.x;
  pdl_wait();
  pdl_launch();
  const bf16* lr = logits + row * vocab;
  float best = -FLT_MAX;
  int bidx = 0x7fffffff;
  for (int i = threadIdx.x; i < vocab; i += blockDim.x) {
    const float v = bf2f(lr[i]);
    if (v > best || (v == best && i < bidx)) {
      best = v;
      bidx = i;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (ov > best || (ov == best && oi < bidx)) {
      best = ov;
      bidx = oi;
    }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = best;
    si[threadIdx.x >> 5] = bidx;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x >> 5;
    best = threadIdx.x < nw ? sv[threadIdx.x] : -FLT_MAX;
    bidx = threadIdx.x < nw ? si[threadIdx.x] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (ov > best || (ov == best && oi < bidx)) {
        best = ov;
        bidx = oi;
      }
    }
    if (threadIdx.x == 0) out[row] = bidx < vocab ? bidx : 0;  // all-NaN row: never emit an invalid id
  }
}

// One warp per (row, 128-column group): lane holds 4 columns.
__global__ void row_ssq_kernel(const bf16* __restrict__ x, int rows, int dim, float* __restrict__ out) {
  pdl_wait();
  pdl_launch();
  const int groups = (dim + 127) / 128;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (gw >= rows * groups) return;
  const int row = gw / groups, g = gw % groups;
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int c = g * 128 + lane * 4 + k;
    if (c < dim) {
      const float v = bf2f(x[(long long)row * dim + c]);
      s += v * v;
    }
  }
  s = warp_sum(s);
  if (lane == 0) out[(long long)g * rows + row] = s;
}

}  // namespace

extern "C" int astraea_rmsnorm(const void* x, const void* r, const void* w, void* y, void* resid_out,
                               int32_t rows, int32_t dim, float eps, void* stream) {
  if (rows < 0 || dim <= 0 || dim % 8 || dim > 256 * 8 * 8) return ASTRAEA_EINVAL;
  if (rows == 0) return ASTRAEA_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int nvec = dim / 8;
  const int threads = nvec >= 256 ? 256 : ((nvec + 31) / 32) * 32;
  const int vpt = (nvec + threads - 1) / threads;
  cudaError_t err = cudaSuccess;
  auto args = [&](auto kern) {
    err = launch_k(kern, dim3(rows), dim3(threads), 0, st, (const bf16*)x, (const bf16*)r, (const bf16*)w, (bf16*)y,
                   (bf16*)resid_out, (int)dim, eps);
  };
  if (vpt <= 1) args(rmsnorm_kernel<1>);
  else if (vpt <= 2) args(rmsnorm_kernel<2>);
  else if (vpt <= 4) args(rmsnorm_kernel<4>);
  else args(rmsnorm_kernel<8>);
  ASTRAEA_TRY(err);
  return ASTRAEA_OK;
}

extern "C" int astraea_silu_mul(const void* gu, void* out, int32_t T, int32_t F, void* stream) {
  if (T < 0 || F <= 0 || F % 8) return ASTRAEA_EINVAL;
  if (T == 0) return ASTRAEA_OK;
  const long long total = (long long)T * F / 8;
  long long want = (total + 255) / 256, cap = 8LL * num_sms();
  const int grid = (int)(want < cap ? want : cap);
  ASTRAEA_TRY(launch_k(silu_mul_kernel, dim3(grid), dim3(256), 0, (cudaStream_t)stream, (const bf16*)gu, (bf16*)out,
                       (int)F, total));
  ASTRAEA_CHECK_LAUNCH();
  return ASTRAEA_OK;
}

extern "C" int astraea_embedding(const int32_t* ids, const void* table, void* out, int32_t T, int32_t dim,
                                 float* ssq_out, void* stream) {
  if (T < 0 || dim <= 0 || dim % 8) return ASTRAEA_EINVAL;
  if (T == 0) return ASTRAEA_OK;
  ASTRAEA_TRY(launch_k(embedding_kernel, dim3(T), dim3(128), 0, (cudaStream_t)stream, ids, (const bf16*)table,
                       (bf16*)out, (int)dim, ssq_out));
  ASTRAEA_CHECK_LAUNCH();
  return ASTRAEA_OK;
}

extern "C" int astraea_argmax(const void* logits, int32_t rows, int32_t vocab, int32_t* ids_out, void* stream) {
  if (rows < 0 || vocab <= 0) return ASTRAEA_EINVAL;
  if (rows == 0) return ASTRAEA_OK;
  ASTRAEA_TRY(launch_k(argmax_kernel, dim3(rows), dim3(1024), 0, (cudaStream_t)stream, (const bf16*)logits,
                       (int)vocab, ids_out));
  ASTRAEA_CHECK_LAUNCH();
  return ASTRAEA_OK;
}

extern "C" int astraea_row_ssq(const void* x, int32_t rows, int32_t dim, float* out, void* stream) {
  if (!x || !out || rows < 0 || dim <= 0) return ASTRAEA_EINVAL;
  if (rows == 0) return ASTRAEA_OK;
  const long long warps = (long long)rows * ((dim + 127) / 128);
  ASTRAEA_TRY(launch_k(row_ssq_kernel, dim3((unsigned)((warps * 32 + 255) / 256)), dim3(256), 0, (cudaStream_t)stream,
                       (const bf16*)x, (int)rows, (int)dim, out));
  return ASTRAEA_OK;
}
