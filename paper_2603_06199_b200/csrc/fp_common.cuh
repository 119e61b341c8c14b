// fp_common.cuh — shared definitions for the FlashPrefill sm_100a kernels.
#pragma once

#include <cfloat>
#include <cstdint>

#include "fp_ptx.cuh"

namespace fpb {

constexpr int kBlock = 128;      // B: token block == MMA tile edge (core.hpp:88)
constexpr int kHeadDim = 128;    // d
constexpr float kLog2e = 1.4426950408889634f;  // core.hpp:13
constexpr float kNegSentinel = -FLT_MAX;       // discovery.hpp:12

// Shapes + PipelineConfig resolved on the host (core.hpp:96-111).
struct Dims {
  int Z, Hq, Hkv, L, M;     // M == N == ceil(L / B)
  int group;                // Hq / Hkv
  int last_len;             // length of block M-1
  float to_bits;            // tau * log2(e)
  float eps, alpha;
  int sink_blocks, window_blocks;
  int B, d;                 // block size and head dim (128 / 128 on the tensor-core path)
  // Row shard: only query blocks I = rb + rs * k (k < Mr) are processed (rb = 0, rs = 1,
  // Mr = M for the whole problem).  Every (z, h, I) is independent (discovery.hpp:87-88,
  // selection.hpp:71-72, attention.hpp:59-60), so rs ranks with rb = rank split any density
  // profile evenly.
  int rb, rs, Mr;
  // Zigzag shard (zz = 1): 2G contiguous chunks of ceil(M / 2G) query blocks; rank r owns chunk r
  // and chunk 2G-1-r (equal causal work, contiguous rows for K/V locality in L2).  zh_end / zh_n:
  // end and size of the high chunk, zl_end: end of the low chunk; Mr = both sizes.
  int zz, zh_end, zh_n, zl_end;
};
using GenDims = Dims;

// t-th owned query block, heaviest (longest causal row) first.
__host__ __device__ __forceinline__ int owned_row(const Dims& D, int t) {
  if (D.zz) return t < D.zh_n ? D.zh_end - 1 - t : D.zl_end - 1 - (t - D.zh_n);
  return D.rb + D.rs * (D.Mr - 1 - t);
}

__host__ __device__ __forceinline__ int block_len(const Dims& D, int blk) {
  return blk + 1 == D.M ? D.last_len : D.B;
}

// Block-wide reductions over `nthreads` (multiple of 32) threads using `scratch` (>= 32 floats).
template <int kThreads>
__device__ __forceinline__ float block_max(float v, float* scratch) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) scratch[w] = v;
  __syncthreads();
  v = (l < kThreads / 32) ? scratch[l] : -INFINITY;
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <int kThreads>
__device__ __forceinline__ float block_sum(float v, float* scratch) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) scratch[w] = v;
  __syncthreads();
  v = (l < kThreads / 32) ? scratch[l] : 0.0f;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// Exclusive prefix count of `pred` across the block (ascending thread order); returns the slot and
// writes the block total to *total.
template <int kThreads>
__device__ __forceinline__ int block_prefix_count(bool pred, int* scratch, int* total) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const unsigned bal = __ballot_sync(0xffffffffu, pred);
  const int in_warp = __popc(bal & ((1u << l) - 1u));
  __syncthreads();
  if (l == 0) scratch[w] = __popc(bal);
  __syncthreads();
  int before = 0, all = 0;
#pragma unroll
  for (int i = 0; i < kThreads / 32; ++i) {
    const int c = scratch[i];
    before += (i < w) ? c : 0;
    all += c;
  }
  *total = all;
  return before + in_warp;
}

}  // namespace fpb
