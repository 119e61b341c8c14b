// baselines.cu — the reference's comparison methods, on the GPU so the drop-in
// covers the whole bsattn API, not only the FlashPrefill path:
//   topk_select / topp_select        selection.hpp:94-159 (sort-based baselines the paper argues
//                                    against)
//   discover_pool_both               discovery.hpp:164-195 (mean-pool Q as well)
//   discover_exact                   discovery.hpp:201-279 (per-query softmax over pooled keys)
// Arithmetic follows the reference order (4-lane dot, sequential sums, double accumulation for
// top-p) with FMA contraction disabled; only exp2f may differ by a few ulp from glibc.
#include "fp_kernels.h"

namespace fpb {

namespace {

__device__ __forceinline__ float dot4f(const float* a, const float* b, int n) {
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  int i = 0;
  for (; i + 4 <= n; i += 4) {
    s0 = __fadd_rn(s0, __fmul_rn(a[i], b[i]));
    s1 = __fadd_rn(s1, __fmul_rn(a[i + 1], b[i + 1]));
    s2 = __fadd_rn(s2, __fmul_rn(a[i + 2], b[i + 2]));
    s3 = __fadd_rn(s3, __fmul_rn(a[i + 3], b[i + 3]));
  }
  for (; i < n; ++i) s0 = __fadd_rn(s0, __fmul_rn(a[i], b[i]));
  return __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3));
}
template <typename T>
__device__ __forceinline__ float ldv(const T* p, size_t i) {
  if constexpr (sizeof(T) == 2) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
  else return reinterpret_cast<const float*>(p)[i];
}
template <typename T>
__device__ float dot4q(const T* q, size_t qo, const float* k, int n) {
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  int i = 0;
  for (; i + 4 <= n; i += 4) {
    s0 = __fadd_rn(s0, __fmul_rn(ldv(q, qo + i), k[i]));
    s1 = __fadd_rn(s1, __fmul_rn(ldv(q, qo + i + 1), k[i + 1]));
    s2 = __fadd_rn(s2, __fmul_rn(ldv(q, qo + i + 2), k[i + 2]));
    s3 = __fadd_rn(s3, __fmul_rn(ldv(q, qo + i + 3), k[i + 3]));
  }
  for (; i < n; ++i) s0 = __fadd_rn(s0, __fmul_rn(ldv(q, qo + i), k[i]));
  return __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3));
}
__device__ __forceinline__ float rmax(float a, float b) { return (a < b) ? b : a; }

constexpr int kSortMax = 4096;  // row length supported by the in-SMEM bitonic sort

// ---------------------------------------------------------------- top-k / top-p
// One CTA per (z, h, i) score row: bitonic sort of (score desc, index asc) == std::stable_sort
// with `row[a] > row[b]` (selection.hpp:112, 142), then the selection rule, then the structural
// retention (selection.hpp:116-117, 153-154).
__global__ void __launch_bounds__(256) sort_select_kernel(Dims D, const float* __restrict__ score,
                                                          uint8_t* __restrict__ mask, int mode,
                                                          int k, float p) {
  __shared__ float key[kSortMax];
  __shared__ int ord[kSortMax];
  const long row = blockIdx.x;
  const int i = (int)(row % D.M), N = D.M;
  const int h = (int)((row / D.M) % D.Hq), z = (int)(row / ((long)D.M * D.Hq));
  const float* srow = score + row * N;
  const int n = i + 1;
  int P = 1;
  while (P < n) P <<= 1;
  for (int t = threadIdx.x; t < P; t += blockDim.x) {
    key[t] = t < n ? srow[t] : -INFINITY;
    ord[t] = t < n ? t : 0x7fffffff;
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < P; t += blockDim.x) {
        const int u = t ^ stride;
        if (u > t) {
          // "before" = larger score first; equal scores keep the lower index first
          const bool t_first = key[t] > key[u] || (key[t] == key[u] && ord[t] < ord[u]);
          const bool up = (t & size) == 0;
          if (up ? !t_first : t_first) {
            const float kk = key[t];
            key[t] = key[u];
            key[u] = kk;
            const int oo = ord[t];
            ord[t] = ord[u];
            ord[u] = oo;
          }
        }
      }
      __syncthreads();
    }
  }
  // key[] now holds the scores in selection order; ord[] their indices
  __shared__ int take;
  if (threadIdx.x == 0) {
    if (mode == 0) {
      take = min(k, n);
    } else {  // top-p (selection.hpp:144-152): double accumulation in the reference order
      double total = 0.0;
      for (int j = 0; j < n; ++j) total += (double)srow[j];
      double cum = 0.0;
      int r = 0;
      for (; r < n; ++r) {
        if (total <= 0.0 || key[r] <= 0.0f) break;
        cum += (double)key[r] / total;
        if (cum >= (double)p - 1e-9) {
          ++r;
          break;
        }
      }
      take = r;
    }
  }
  __syncthreads();
  uint8_t* mrow = mask + ((size_t)z * D.M + i) * (size_t)N * D.Hq + h;
  for (int j = threadIdx.x; j < N; j += blockDim.x) mrow[(size_t)j * D.Hq] = 0;
  __syncthreads();
  for (int r = threadIdx.x; r < take; r += blockDim.x) mrow[(size_t)ord[r] * D.Hq] = 1;
  __syncthreads();
  for (int j = threadIdx.x; j <= i; j += blockDim.x)
    if (j < D.sink_blocks || (i - j) < D.window_blocks) mrow[(size_t)j * D.Hq] = 1;
}

// ---------------------------------------------------------------- pool-both
// discovery.hpp:177-192: one logit per block pair, energy 1, sentinel above the diagonal.
__global__ void pool_both_kernel(Dims D, const float* __restrict__ pq, const float* __restrict__ pk,
                                 float* __restrict__ energy, float* __restrict__ local_max) {
  const size_t n = (size_t)D.Z * D.Hq * D.M * D.M;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n;
       e += (size_t)gridDim.x * blockDim.x) {
    const int J = (int)(e % D.M);
    const int I = (int)((e / D.M) % D.M);
    const size_t zh = e / ((size_t)D.M * D.M);
    const int z = (int)(zh / D.Hq), h = (int)(zh % D.Hq);
    if (J > I) {
      energy[e] = 0.f;
      local_max[e] = -FLT_MAX;
    } else {
      const float* qb = pq + (zh * D.M + I) * D.d;
      const float* kb = pk + (((size_t)z * D.Hkv + h / D.group) * D.M + J) * D.d;
      local_max[e] = __fmul_rn(dot4f(qb, kb, D.d), D.to_bits);
      energy[e] = 1.0f;
    }
  }
}

// ---------------------------------------------------------------- exact
// discovery.hpp:222-229: table[t][kj] = kj <= block(t) ? dot(q_t, kbar_kj) * to_bits : sentinel
template <typename T>
__global__ void exact_logits_kernel(Dims D, const T* __restrict__ Q, const float* __restrict__ pk,
                                    float* __restrict__ table) {
  const size_t n = (size_t)D.Z * D.Hq * D.L * D.M;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n;
       e += (size_t)gridDim.x * blockDim.x) {
    const int kj = (int)(e % D.M);
    const size_t tr = e / D.M;  // (zh, t)
    const int t = (int)(tr % D.L);
    const size_t zh = tr / D.L;
    const int z = (int)(zh / D.Hq), h = (int)(zh % D.Hq);
    const int visible = t / D.B;
    table[e] = kj <= visible
                   ? __fmul_rn(dot4q(Q, tr * D.d, pk + (((size_t)z * D.Hkv + h / D.group) * D.M + kj) * D.d, D.d),
                               D.to_bits)
                   : -FLT_MAX;
  }
}
// discovery.hpp:235-248: block-pair max and sum of exp2 over the tile's rows (sequential r)
__global__ void exact_energy_kernel(Dims D, const float* __restrict__ table,
                                    float* __restrict__ energy, float* __restrict__ local_max) {
  const size_t n = (size_t)D.Z * D.Hq * D.M * D.M;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n;
       e += (size_t)gridDim.x * blockDim.x) {
    const int kj = (int)(e % D.M);
    const int qi = (int)((e / D.M) % D.M);
    const size_t zh = e / ((size_t)D.M * D.M);
    if (kj > qi) {
      energy[e] = 0.f;
      local_max[e] = -FLT_MAX;
      continue;
    }
    const int rows = block_len(D, qi);
    const float* col = table + (zh * D.L + (size_t)qi * D.B) * D.M + kj;
    float m = -FLT_MAX;
    for (int r = 0; r < rows; ++r) m = rmax(m, col[(size_t)r * D.M]);
    float s = 0.f;
    for (int r = 0; r < rows; ++r) s = __fadd_rn(s, exp2f(__fsub_rn(col[(size_t)r * D.M], m)));
    local_max[e] = m;
    energy[e] = s;
  }
}
// discovery.hpp:251-263: per-query softmax over the visible pooled keys, in place
__global__ void exact_softmax_kernel(Dims D, float* __restrict__ table) {
  const size_t n = (size_t)D.Z * D.Hq * D.L;
  for (size_t tr = blockIdx.x * (size_t)blockDim.x + threadIdx.x; tr < n;
       tr += (size_t)gridDim.x * blockDim.x) {
    const int visible = (int)(tr % D.L) / D.B;
    float* row = table + tr * D.M;
    float m = -FLT_MAX;
    for (int kj = 0; kj <= visible; ++kj) m = rmax(m, row[kj]);
    float total = 0.f;
    for (int kj = 0; kj <= visible; ++kj) {
      row[kj] = exp2f(__fsub_rn(row[kj], m));
      total = __fadd_rn(total, row[kj]);
    }
    const float inv = __fdiv_rn(1.0f, __fadd_rn(total, D.eps));
    for (int kj = 0; kj <= visible; ++kj) row[kj] = __fmul_rn(row[kj], inv);
  }
}
// discovery.hpp:265-274: score = average over the block's rows
__global__ void exact_score_kernel(Dims D, const float* __restrict__ table, float* __restrict__ score) {
  const size_t n = (size_t)D.Z * D.Hq * D.M * D.M;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n;
       e += (size_t)gridDim.x * blockDim.x) {
    const int kj = (int)(e % D.M);
    const int qi = (int)((e / D.M) % D.M);
    const size_t zh = e / ((size_t)D.M * D.M);
    if (kj > qi) {
      score[e] = 0.f;
      continue;
    }
    const int rows = block_len(D, qi);
    const float* col = table + (zh * D.L + (size_t)qi * D.B) * D.M + kj;
    float acc = 0.f;
    for (int r = 0; r < rows; ++r) acc = __fadd_rn(acc, col[(size_t)r * D.M]);
    score[e] = __fmul_rn(acc, __fdiv_rn(1.0f, (float)rows));
  }
}

}  // namespace

cudaError_t launch_sort_select(const Dims& D, const float* score, uint8_t* mask, int mode, int k,
                               float p, cudaStream_t s) {
  if (D.M > kSortMax) return cudaErrorInvalidValue;
  sort_select_kernel<<<(unsigned)((size_t)D.Z * D.Hq * D.M), 256, 0, s>>>(D, score, mask, mode, k, p);
  return cudaGetLastError();
}

cudaError_t launch_pool_both(const Dims& D, bool bf16_in, const void* Q, const void* K,
                             float* pooled_q, float* pooled_k, float* energy, float* local_max,
                             cudaStream_t s) {
  Dims Dq = D;
  Dq.Hkv = D.Hq;  // pool all Q heads with the same kernel
  cudaError_t e = g_launch_pool(Dq, bf16_in, Q, pooled_q, s);
  if (e == cudaSuccess) e = g_launch_pool(D, bf16_in, K, pooled_k, s);
  if (e != cudaSuccess) return e;
  pool_both_kernel<<<592, 256, 0, s>>>(D, pooled_q, pooled_k, energy, local_max);
  return cudaGetLastError();
}

size_t exact_table_bytes(const Dims& D) { return sizeof(float) * (size_t)D.Z * D.Hq * D.L * D.M; }

cudaError_t launch_exact(const Dims& D, bool bf16_in, const void* Q, const void* K, float* pooled,
                         float* table, float* energy, float* local_max, float* score,
                         cudaStream_t s) {
  cudaError_t e = g_launch_pool(D, bf16_in, K, pooled, s);
  if (e != cudaSuccess) return e;
  if (bf16_in)
    exact_logits_kernel<__nv_bfloat16><<<1184, 256, 0, s>>>(D, static_cast<const __nv_bfloat16*>(Q),
                                                           pooled, table);
  else
    exact_logits_kernel<float><<<1184, 256, 0, s>>>(D, static_cast<const float*>(Q), pooled, table);
  exact_energy_kernel<<<592, 256, 0, s>>>(D, table, energy, local_max);
  exact_softmax_kernel<<<592, 256, 0, s>>>(D, table);
  exact_score_kernel<<<592, 256, 0, s>>>(D, table, score);
  return cudaGetLastError();
}

}  // namespace fpb
