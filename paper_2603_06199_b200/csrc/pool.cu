// pool.cu — K1: block-mean key pooling (discovery.hpp:39-70) and operand conversions.
//
// HBM-bound.  One 64-thread CTA owns one (kv head, key block); each thread owns 2 channels and
// sums the block's rows sequentially in fp32 — the reference's order (discovery.hpp:51-53) — then
// multiplies by the fp32 reciprocal 1/len (discovery.hpp:55-56), so `pooled` is bit-identical to
// the reference for identical inputs.  The same pass writes the bf16 hi/lo split of k̄ that the
// tensor-core discovery kernel consumes (k̄ = hi + lo to 16 significant bits).
#include <cuda_bf16.h>

#include "fp_kernels.h"

namespace fpb {

template <bool kBf16>
__global__ void __launch_bounds__(64) pool_keys_kernel(const void* __restrict__ K,
                                                       float* __restrict__ pooled,
                                                       __nv_bfloat16* __restrict__ split, int ZH,
                                                       int L, int M, int last_len, int j0, int nj) {
  // one CTA of 64 threads per (zh, key block j in [j0, j0 + nj)); thread t owns channels 2t, 2t+1
  const int zh = blockIdx.x / nj, j = j0 + blockIdx.x % nj;
  const int c0 = threadIdx.x * 2;
  const int len = (j + 1 == M) ? last_len : kBlock;
  const size_t row0 = (size_t)zh * L + (size_t)j * kBlock;
  float s0 = 0.f, s1 = 0.f;
  constexpr int U = 16;  // independent row loads in flight; the add chain stays sequential in r
  int r = 0;
  for (; r + U <= len; r += U) {
    float v[U][2];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t off = (row0 + r + u) * kHeadDim + c0;
      if constexpr (kBf16) {
        const uint32_t raw = __ldg(reinterpret_cast<const unsigned int*>(
            reinterpret_cast<const __nv_bfloat16*>(K) + off));
        const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&raw);
        v[u][0] = __low2float(a);
        v[u][1] = __high2float(a);
      } else {
        const float2 f = __ldg(reinterpret_cast<const float2*>(reinterpret_cast<const float*>(K) + off));
        v[u][0] = f.x;
        v[u][1] = f.y;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {  // discovery.hpp:51-53: out[c] += row[c], r ascending
      s0 = __fadd_rn(s0, v[u][0]);
      s1 = __fadd_rn(s1, v[u][1]);
    }
  }
  for (; r < len; ++r) {
    const size_t off = (row0 + r) * kHeadDim + c0;
    float v0, v1;
    if constexpr (kBf16) {
      const __nv_bfloat16* p = reinterpret_cast<const __nv_bfloat16*>(K) + off;
      v0 = __bfloat162float(p[0]);
      v1 = __bfloat162float(p[1]);
    } else {
      const float* p = reinterpret_cast<const float*>(K) + off;
      v0 = p[0];
      v1 = p[1];
    }
    s0 = __fadd_rn(s0, v0);
    s1 = __fadd_rn(s1, v1);
  }
  const float inv = __fdiv_rn(1.0f, (float)len);  // discovery.hpp:55-56
  const float o0 = __fmul_rn(s0, inv), o1 = __fmul_rn(s1, inv);
  const size_t dst = ((size_t)zh * M + j) * kHeadDim + c0;
  if (pooled) *reinterpret_cast<float2*>(pooled + dst) = make_float2(o0, o1);
  if (split) {
    const __nv_bfloat16 h0 = __float2bfloat16_rn(o0), h1 = __float2bfloat16_rn(o1);
    const __nv_bfloat162 hi = __halves2bfloat162(h0, h1);
    const __nv_bfloat162 lo = __halves2bfloat162(
        __float2bfloat16_rn(__fsub_rn(o0, __bfloat162float(h0))),
        __float2bfloat16_rn(__fsub_rn(o1, __bfloat162float(h1))));
    const size_t plane = (size_t)ZH * M * kHeadDim;
    *reinterpret_cast<__nv_bfloat162*>(split + dst) = hi;
    *reinterpret_cast<__nv_bfloat162*>(split + plane + dst) = lo;
  }
}

cudaError_t launch_pool_keys(const Dims& D, bool bf16_in, const void* K, float* pooled,
                             __nv_bfloat16* kbar_split, cudaStream_t s, int j0, int nj) {
  const int ZH = D.Z * D.Hkv;
  if (nj < 0) nj = D.M - j0;
  if (nj <= 0) return cudaSuccess;
  const dim3 grid(ZH * nj);
  if (bf16_in)
    pool_keys_kernel<true><<<grid, 64, 0, s>>>(K, pooled, kbar_split, ZH, D.L, D.M, D.last_len,
                                               j0, nj);
  else
    pool_keys_kernel<false><<<grid, 64, 0, s>>>(K, pooled, kbar_split, ZH, D.L, D.M, D.last_len,
                                                j0, nj);
  return cudaGetLastError();
}

// pooled fp32 (caller-provided, approx_block_scores API) -> bf16 hi/lo planes.
__global__ void split_pooled_kernel(const float* __restrict__ pooled,
                                    __nv_bfloat16* __restrict__ split, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const float x = pooled[i];
    const __nv_bfloat16 hi = __float2bfloat16_rn(x);
    split[i] = hi;
    split[n + i] = __float2bfloat16_rn(__fsub_rn(x, __bfloat162float(hi)));
  }
}

cudaError_t launch_split_pooled(const Dims& D, const float* pooled, __nv_bfloat16* kbar_split,
                                cudaStream_t s) {
  const size_t n = (size_t)D.Z * D.Hkv * D.M * kHeadDim;
  split_pooled_kernel<<<1184, 256, 0, s>>>(pooled, kbar_split, n);
  return cudaGetLastError();
}

// fp32 -> bf16 (hi) and optionally the residual plane (lo), 4 elements per thread.
__global__ void f32_to_bf16_kernel(const float4* __restrict__ src, uint2* __restrict__ hi,
                                   uint2* __restrict__ lo, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
       i += (size_t)gridDim.x * blockDim.x) {
    const float4 f = src[i];
    const float v[4] = {f.x, f.y, f.z, f.w};
    __nv_bfloat16 h[4], l[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      h[c] = __float2bfloat16_rn(v[c]);
      l[c] = __float2bfloat16_rn(__fsub_rn(v[c], __bfloat162float(h[c])));
    }
    hi[i] = *reinterpret_cast<const uint2*>(h);
    if (lo) lo[i] = *reinterpret_cast<const uint2*>(l);
  }
}

cudaError_t launch_f32_to_bf16(const float* src, __nv_bfloat16* hi, __nv_bfloat16* lo, size_t n,
                               cudaStream_t s) {
  const size_t n4 = n / 4;  // n is a multiple of d = 128
  f32_to_bf16_kernel<<<148 * 8, 256, 0, s>>>(reinterpret_cast<const float4*>(src),
                                             reinterpret_cast<uint2*>(hi),
                                             reinterpret_cast<uint2*>(lo), n4);
  return cudaGetLastError();
}

}  // namespace fpb
