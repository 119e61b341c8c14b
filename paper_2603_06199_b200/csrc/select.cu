// select.cu — standalone kernels for the unfused API entry points:
//   normalize_block_scores (discovery.hpp:119-148), max_threshold_mask (selection.hpp:63-92),
//   compress_indices (selection.hpp:176-192), visit_count (selection.hpp:195-200),
//   full_causal_plan (attention.hpp:178-192).
// All are HBM-bound integer/compare work: one warp per score row, warp-level reductions, ballot
// compaction.  max/compare/compaction are exact, so given the same score map the mask, idx and
// counts are bit-identical to the reference.  The fused hot path (discover.cu) does the same work
// in the epilogue of the discovery kernel instead.
#include "fp_kernels.h"

namespace fpb {

__device__ __forceinline__ float warp_max(float v) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One warp per (z, h, i) row.
__global__ void normalize_kernel(Dims D, const float* __restrict__ energy,
                                 const float* __restrict__ local_max, float* __restrict__ score) {
  const long row = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long rows = (long)D.Z * D.Hq * D.M;
  if (row >= rows) return;
  const int lane = threadIdx.x & 31;
  const int i = (int)(row % D.M), N = D.M;
  const float* en = energy + row * N;
  const float* lm = local_max + row * N;
  float* dst = score + row * N;
  float rmax = kNegSentinel;
  for (int j = lane; j <= i; j += 32) rmax = fmaxf(rmax, lm[j]);
  rmax = warp_max(rmax);
  float total = 0.f;
  for (int j = lane; j <= i; j += 32) total += en[j] * exp2f(lm[j] - rmax);
  total = warp_sum(total);
  const float inv = 1.0f / (total + D.eps);
  for (int j = lane; j < N; j += 32) dst[j] = (j <= i) ? (en[j] * exp2f(lm[j] - rmax)) * inv : 0.f;
}

cudaError_t launch_normalize(const Dims& D, const float* energy, const float* local_max,
                             float* score, cudaStream_t s) {
  const long rows = (long)D.Z * D.Hq * D.M;
  normalize_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(D, energy, local_max, score);
  return cudaGetLastError();
}

// One warp per (z, h, i) score row; writes the head-last mask row mask[z, i, :, h].
__global__ void threshold_kernel(Dims D, const float* __restrict__ score, uint8_t* __restrict__ mask,
                                 unsigned long long* __restrict__ comparisons) {
  const long row = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long rows = (long)D.Z * D.Hq * D.M;
  if (row >= rows) return;
  const int lane = threadIdx.x & 31;
  const int i = (int)(row % D.M), N = D.M;
  const int h = (int)((row / D.M) % D.Hq), z = (int)(row / ((long)D.M * D.Hq));
  const float* srow = score + row * N;
  float max_val = 0.0f;  // selection.hpp:75 — initialised to 0, not -inf
  for (int j = lane; j <= i; j += 32) max_val = fmaxf(max_val, srow[j]);
  max_val = warp_max(max_val);
  const float thresh = D.alpha * max_val;  // selection.hpp:80
  uint8_t* mrow = mask + ((size_t)z * D.M + i) * (size_t)N * D.Hq + h;
  for (int j = lane; j < N; j += 32) {
    uint8_t a = 0;
    if (j <= i)
      a = (srow[j] >= thresh) || j < D.sink_blocks || (i - j) < D.window_blocks;  // :82-84
    mrow[(size_t)j * D.Hq] = a;
  }
  if (comparisons && lane == 0) atomicAdd(comparisons, 2ull * (unsigned long long)(i + 1));
}

cudaError_t launch_threshold(const Dims& D, const float* score, uint8_t* mask,
                             unsigned long long* comparisons, cudaStream_t s) {
  const long rows = (long)D.Z * D.Hq * D.M;
  threshold_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(D, score, mask, comparisons);
  return cudaGetLastError();
}

// One warp per (z, i, h): ballot-compaction of active j in ascending order, then the fill value N.
__global__ void compress_kernel(Dims D, const uint8_t* __restrict__ mask, int32_t* __restrict__ idx,
                                int32_t* __restrict__ counts) {
  const long row = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long rows = (long)D.Z * D.M * D.Hq;
  if (row >= rows) return;
  const int lane = threadIdx.x & 31;
  const int h = (int)(row % D.Hq);
  const long zi = row / D.Hq;
  const int N = D.M, H = D.Hq;
  const uint8_t* mrow = mask + (size_t)zi * N * H + h;
  int32_t* irow = idx + (size_t)zi * N * H + h;
  int base = 0;
  for (int j0 = 0; j0 < N; j0 += 32) {
    const int j = j0 + lane;
    const bool a = j < N && mrow[(size_t)j * H] != 0;
    const unsigned bal = __ballot_sync(0xffffffffu, a);
    if (a) irow[(size_t)(base + __popc(bal & ((1u << lane) - 1u))) * H] = j;
    base += __popc(bal);
  }
  for (int slot = base + lane; slot < N; slot += 32) irow[(size_t)slot * H] = N;
  if (lane == 0) counts[row] = base;
}

cudaError_t launch_compress(const Dims& D, const uint8_t* mask, int32_t* idx, int32_t* counts,
                            cudaStream_t s) {
  const long rows = (long)D.Z * D.M * D.Hq;
  compress_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(D, mask, idx, counts);
  return cudaGetLastError();
}

// Plan rows of the owned query blocks set to the fill value N (selection.hpp:176-192), with
// coalesced 16-byte stores: the fused discovery epilogue then writes only the active slots.
// Row (z, I) is N * Hq contiguous int32.
__global__ void fill_plan_kernel(Dims D, int32_t* __restrict__ idx) {
  const size_t row_ints = (size_t)D.M * D.Hq, row_vec = row_ints / 4;
  const int rows = D.Z * D.Mr;
  const int4 f = make_int4(D.M, D.M, D.M, D.M);
  for (int r = blockIdx.y; r < rows; r += gridDim.y) {
    const int z = r / D.Mr, I = owned_row(D, r % D.Mr);  // interleaved, zigzag or all rows
    int32_t* row = idx + ((size_t)z * D.M + I) * row_ints;
    int4* row4 = reinterpret_cast<int4*>(row);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < row_vec;
         i += (size_t)gridDim.x * blockDim.x)
      row4[i] = f;
    for (size_t i = row_vec * 4 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < row_ints;
         i += (size_t)gridDim.x * blockDim.x)
      row[i] = D.M;
  }
}

// Two-pass plan-only discovery, second pass.  One CTA per owned (z, I) plan row and one warp per
// head: normalize_block_scores (discovery.hpp:131-143), the max-based threshold with sink /
// window retention (selection.hpp:63-92) and compress_indices (selection.hpp:176-192) in three
// sweeps over the head's row of the packed (local max, energy) triangle.  The plan is head-last
// (Z x M x N x H, selection.hpp:14-21), so the CTA assembles the N x Hc slab of a chunk of Hc
// heads in shared memory (fill value N included) and writes it with coalesced stores; Hc is a
// power of two and the slab is XOR-swizzled so both the per-head compaction writes (consecutive
// slots) and the row-major copy-out are bank-conflict free.
__global__ void __launch_bounds__(1024, 2) select_rows_kernel(Dims D, const float2* __restrict__ rows,
                                                           int32_t* __restrict__ idx,
                                                           int32_t* __restrict__ counts, int hc_log2) {
  extern __shared__ int32_t slab[];
  const int Hc = 1 << hc_log2;
  const int N = D.M, H = D.Hq;
  const int z = blockIdx.x / D.Mr;
  const int I = owned_row(D, blockIdx.x % D.Mr);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t plan_row = ((size_t)z * D.M + I) * (size_t)N;
  auto at = [&](int slot, int hc) { return slot * Hc + (hc ^ (slot & (Hc - 1))); };
  for (int h0 = 0; h0 < H; h0 += Hc) {
    const int Hv = min(Hc, H - h0);
    for (int e = threadIdx.x; e < N * Hc; e += blockDim.x) slab[e] = N;
    __syncthreads();
    if (w < Hv) {
      const int h = h0 + w;
      const float2* r = rows + ((size_t)z * H + h) * ((size_t)D.M * (D.M + 1) / 2) +
                        (size_t)I * (I + 1) / 2;
      float rmax = kNegSentinel;
      for (int J = lane; J <= I; J += 32) rmax = fmaxf(rmax, r[J].x);
      rmax = warp_max(rmax);
      float total = 0.f, pmax = 0.f;
      for (int J = lane; J <= I; J += 32) {
        const float2 ms = r[J];
        const float sp = __fmul_rn(ms.y, exp2f(__fsub_rn(ms.x, rmax)));
        total += sp;
        pmax = fmaxf(pmax, sp);
      }
      total = warp_sum(total);
      pmax = warp_max(pmax);
      const float inv = __fdiv_rn(1.0f, __fadd_rn(total, D.eps));
      // max_J fl(S'_J inv) == fl(max_J S'_J * inv) (monotone rounding, inv > 0); max_val >= 0
      const float thresh = __fmul_rn(D.alpha, __fmul_rn(pmax, inv));
      int base = 0;
      for (int J0 = 0; J0 <= I; J0 += 32) {
        const int J = J0 + lane;
        bool act = false;
        if (J <= I) {
          const float2 ms = r[J];
          const float sc = __fmul_rn(__fmul_rn(ms.y, exp2f(__fsub_rn(ms.x, rmax))), inv);
          act = sc >= thresh || J < D.sink_blocks || (I - J) < D.window_blocks;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, act);
        if (act) slab[at(base + __popc(bal & ((1u << lane) - 1u)), w)] = J;
        base += __popc(bal);
      }
      if (lane == 0) counts[((size_t)z * D.M + I) * H + h] = base;
    }
    __syncthreads();
    int32_t* dst = idx + plan_row * H + h0;
    if (Hv == H && (H & 3) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
      // the whole (z, I) row is one contiguous N x H run
      int4* d4 = reinterpret_cast<int4*>(dst);
      for (int e = threadIdx.x; e < N * H / 4; e += blockDim.x) {
        const int k = e * 4, slot = k / Hc, hc = k % Hc;
        d4[e] = make_int4(slab[at(slot, hc)], slab[at(slot, hc + 1)], slab[at(slot, hc + 2)],
                          slab[at(slot, hc + 3)]);
      }
    } else {
      for (int e = threadIdx.x; e < N * Hv; e += blockDim.x) {
        const int slot = e / Hv, hc = e % Hv;
        dst[(size_t)slot * H + hc] = slab[at(slot, hc)];
      }
    }
    __syncthreads();
  }
}

cudaError_t launch_select_rows(const Dims& D, const float2* rows, int32_t* idx, int32_t* counts,
                               bool prefilled, cudaStream_t s) {
  (void)prefilled;  // the slab carries the fill value; every slot of an owned row is written
  const long nrows = (long)D.Z * D.Mr;
  if (nrows == 0 || D.Hq == 0) return cudaSuccess;
  int hc_log2 = 0;
  while (hc_log2 < 5 && (2 << hc_log2) <= D.Hq) ++hc_log2;  // largest power of two <= min(H, 32)
  while (hc_log2 > 0 && (size_t)D.M * (1u << hc_log2) * 4 > 96 * 1024) --hc_log2;
  const size_t smem = (size_t)D.M * (1u << hc_log2) * 4;
  if (smem > 96 * 1024) return cudaErrorInvalidValue;  // M > 24K blocks: not a two-pass size
  cudaError_t e = cudaFuncSetAttribute(select_rows_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  if (e != cudaSuccess) return e;
  select_rows_kernel<<<(unsigned)nrows, 32 << hc_log2, smem, s>>>(D, rows, idx, counts, hc_log2);
  return cudaGetLastError();
}

cudaError_t launch_fill_plan(const Dims& D, int32_t* idx, cudaStream_t s) {
  if (D.Mr == 0) return cudaSuccess;
  const size_t row_vec = (size_t)D.M * D.Hq / 4;
  const int bx = (int)((row_vec + 255) / 256 < 8 ? (row_vec + 255) / 256 : 8);
  const int rows = D.Z * D.Mr;
  const dim3 grid(bx < 1 ? 1 : bx, rows < 4096 ? rows : 4096);
  fill_plan_kernel<<<grid, 256, 0, s>>>(D, idx);
  return cudaGetLastError();
}

__global__ void visit_count_kernel(const int32_t* __restrict__ counts, size_t n,
                                   unsigned long long* __restrict__ total) {
  unsigned long long acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    acc += (unsigned long long)(long long)counts[i];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(total, acc);
}

cudaError_t launch_visit_count(const Dims& D, const int32_t* counts, unsigned long long* total,
                               cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(total, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  const size_t n = (size_t)D.Z * D.M * D.Hq;
  visit_count_kernel<<<148, 256, 0, s>>>(counts, n, total);
  return cudaGetLastError();
}

__global__ void full_plan_kernel(Dims D, int32_t* __restrict__ idx, int32_t* __restrict__ counts) {
  const int N = D.M, H = D.Hq;
  const size_t n = (size_t)D.Z * D.M * N * H;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n;
       e += (size_t)gridDim.x * blockDim.x) {
    const int h = (int)(e % H);
    const int slot = (int)((e / H) % N);
    const int i = (int)((e / ((size_t)H * N)) % D.M);
    idx[e] = slot <= i ? slot : N;
    if (slot == 0) counts[(e / ((size_t)H * N)) * H + h] = i + 1;
  }
}

cudaError_t launch_full_causal_plan(const Dims& D, int32_t* idx, int32_t* counts, cudaStream_t s) {
  full_plan_kernel<<<148 * 8, 256, 0, s>>>(D, idx, counts);
  return cudaGetLastError();
}

}  // namespace fpb
