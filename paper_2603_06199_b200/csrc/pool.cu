// pool.cu — K1: block-mean key pooling (discovery.hpp:39-70) and operand conversions.
//
// HBM-bound.  One CTA per (kv head, key block): a single bulk copy (cp.async.bulk, TMA engine)
// stages the block's rows — contiguous in K (Z x Hkv x L x d) — in shared memory, 32 KiB for
// bf16; one thread per channel then sums the rows sequentially in fp32, the reference's order
// (discovery.hpp:51-53), and multiplies by the fp32 reciprocal 1/len (discovery.hpp:55-56), so
// `pooled` is bit-identical to the reference for identical inputs.  With every block's copy in
// flight at once (one wave: 7 CTAs of 32 KiB per SM) the kernel streams K at HBM rate.  The same
// pass writes the bf16 hi/lo split of k̄ that the tensor-core discovery kernel consumes
// (k̄ = hi + lo to 16 significant bits).
#include <cuda_bf16.h>

#include <type_traits>

#include "fp_kernels.h"

namespace fpb {

using namespace ptx;

template <bool kBf16>
__global__ void __launch_bounds__(kHeadDim) pool_keys_kernel(const void* __restrict__ K,
                                                             float* __restrict__ pooled,
                                                             __nv_bfloat16* __restrict__ split,
                                                             int ZH, int L, int M, int last_len,
                                                             int j0, int nj) {
  using T = typename std::conditional<kBf16, __nv_bfloat16, float>::type;
  extern __shared__ __align__(128) uint8_t tile_raw[];
  const T* tile = reinterpret_cast<const T*>(tile_raw);
  __shared__ uint64_t bar;
  const int zh = blockIdx.x / nj, j = j0 + blockIdx.x % nj;
  const int len = (j + 1 == M) ? last_len : kBlock;
  const size_t row0 = (size_t)zh * L + (size_t)j * kBlock;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t bytes = (uint32_t)(len * kHeadDim * sizeof(T));
    mbar_arrive_expect_tx(smem_u32(&bar), bytes);
    bulk_load_1d(smem_u32(tile_raw), reinterpret_cast<const T*>(K) + row0 * kHeadDim, bytes,
                 smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  const int c = threadIdx.x;  // one channel per thread
  float sum = 0.f;
  for (int r = 0; r < len; ++r)  // discovery.hpp:51-53: out[c] += row[c], r ascending
    sum = __fadd_rn(sum, static_cast<float>(tile[r * kHeadDim + c]));
  const float o = __fmul_rn(sum, __fdiv_rn(1.0f, (float)len));  // discovery.hpp:55-56
  const size_t dst = ((size_t)zh * M + j) * kHeadDim + c;
  if (pooled) pooled[dst] = o;
  if (split) {
    const __nv_bfloat16 hi = __float2bfloat16_rn(o);
    split[dst] = hi;
    split[(size_t)ZH * M * kHeadDim + dst] = __float2bfloat16_rn(__fsub_rn(o, __bfloat162float(hi)));
  }
}

cudaError_t launch_pool_keys(const Dims& D, bool bf16_in, const void* K, float* pooled,
                             __nv_bfloat16* kbar_split, cudaStream_t s, int j0, int nj) {
  const int ZH = D.Z * D.Hkv;
  if (nj < 0) nj = D.M - j0;
  if (nj <= 0) return cudaSuccess;
  const dim3 grid(ZH * nj);
  if (bf16_in) {
    pool_keys_kernel<true><<<grid, kHeadDim, kBlock * kHeadDim * 2, s>>>(
        K, pooled, kbar_split, ZH, D.L, D.M, D.last_len, j0, nj);
  } else {
    constexpr int smem = kBlock * kHeadDim * 4;  // 64 KiB of fp32 rows
    cudaError_t e = cudaFuncSetAttribute(pool_keys_kernel<false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    pool_keys_kernel<false><<<grid, kHeadDim, smem, s>>>(K, pooled, kbar_split, ZH, D.L, D.M,
                                                         D.last_len, j0, nj);
  }
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
