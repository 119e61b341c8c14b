// generic.cu — SIMT CUDA kernels for shapes outside the tensor-core tile (d != 128 or B != 128).
//
// The tcgen05 kernels cover the production shape (d = 128, B = 128).  The reference
// API accepts any d >= 1 and B >= 1 (core.hpp:31-41, 96-101), and its own tests use d = 4..64 and
// B = 4..128; these kernels keep the drop-in complete for those shapes.  They follow the reference
// arithmetic literally — the 4-lane dot_f32 order (core.hpp:116-127), sequential row sums, max
// initialised to the sentinel, multiply-by-reciprocal — with FMA contraction disabled
// (__fmul_rn/__fadd_rn), so logits, maxima and pooled keys are bit-identical to the reference and
// only exp2f/log2f can differ (CUDA <= 2 ulp vs glibc).  Performance is not a goal here.
#include "fp_kernels.h"

namespace fpb {

namespace {

template <typename T>
__device__ __forceinline__ float ld(const T* p, size_t i) {
  if constexpr (sizeof(T) == 2) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
  else return reinterpret_cast<const float*>(p)[i];
}

// core.hpp:116-127 — four stride-4 partial sums combined as (s0+s1)+(s2+s3).
template <typename TA, typename TB>
__device__ float dot4(const TA* a, size_t ao, const TB* b, size_t bo, int n) {
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  int i = 0;
  for (; i + 4 <= n; i += 4) {
    s0 = __fadd_rn(s0, __fmul_rn(ld(a, ao + i), ld(b, bo + i)));
    s1 = __fadd_rn(s1, __fmul_rn(ld(a, ao + i + 1), ld(b, bo + i + 1)));
    s2 = __fadd_rn(s2, __fmul_rn(ld(a, ao + i + 2), ld(b, bo + i + 2)));
    s3 = __fadd_rn(s3, __fmul_rn(ld(a, ao + i + 3), ld(b, bo + i + 3)));
  }
  for (; i < n; ++i) s0 = __fadd_rn(s0, __fmul_rn(ld(a, ao + i), ld(b, bo + i)));
  return __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3));
}

__device__ __forceinline__ float ref_max(float a, float b) { return (a < b) ? b : a; }  // std::max

// discovery.hpp:39-59: one thread per (zh, j, c), sequential sum over the block's rows.
template <typename T>
__global__ void g_pool_kernel(const T* __restrict__ K, float* __restrict__ pooled,
                              __nv_bfloat16* __restrict__ split, int ZH, int L, int d, int B,
                              int M, int last_len) {
  const size_t n = (size_t)ZH * M * d;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n;
       e += (size_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % d);
    const int j = (int)((e / d) % M);
    const size_t zh = e / ((size_t)d * M);
    const int len = (j + 1 == M) ? last_len : B;
    float s = 0.f;
    const size_t base = (zh * L + (size_t)j * B) * d + c;
    for (int r = 0; r < len; ++r) s = __fadd_rn(s, ld(K, base + (size_t)r * d));
    const float out = __fmul_rn(s, __fdiv_rn(1.0f, (float)len));
    if (pooled) pooled[e] = out;
    if (split) {  // unused by the generic path, kept for symmetry with pool.cu
      const __nv_bfloat16 hi = __float2bfloat16_rn(out);
      split[e] = hi;
      split[n + e] = __float2bfloat16_rn(__fsub_rn(out, __bfloat162float(hi)));
    }
  }
}

// discovery.hpp:75-115: one CTA per (z, h, I); logits of the tile into shared memory, max,
// then the sequential sum of exp2f(x - m) in row order by one thread.
template <typename T>
__global__ void g_approx_kernel(GenDims G, const T* __restrict__ Q, const float* __restrict__ pooled,
                                float* __restrict__ energy, float* __restrict__ local_max) {
  extern __shared__ float logits[];
  const int I = blockIdx.x % G.M;
  const int zh = blockIdx.x / G.M;
  const int z = zh / G.Hq, h = zh % G.Hq;
  const int rows = (I + 1 == G.M) ? G.last_len : G.B;
  const size_t qoff = ((size_t)zh * G.L + (size_t)I * G.B) * G.d;
  const size_t koff0 = ((size_t)(z * G.Hkv + h / G.group) * G.M) * G.d;
  const size_t row = ((size_t)zh * G.M + I) * G.M;
  for (int J = 0; J < G.M; ++J) {
    if (J > I) {  // discovery.hpp:84
      if (threadIdx.x == 0) {
        energy[row + J] = 0.f;
        local_max[row + J] = -FLT_MAX;
      }
      continue;
    }
    for (int r = threadIdx.x; r < rows; r += blockDim.x)
      logits[r] = __fmul_rn(dot4(Q, qoff + (size_t)r * G.d, pooled, koff0 + (size_t)J * G.d, G.d),
                            G.to_bits);
    __syncthreads();
    if (threadIdx.x == 0) {
      float m = -FLT_MAX;
      for (int r = 0; r < rows; ++r) m = ref_max(m, logits[r]);
      float s = 0.f;
      for (int r = 0; r < rows; ++r) s = __fadd_rn(s, exp2f(__fsub_rn(logits[r], m)));
      energy[row + J] = s;
      local_max[row + J] = m;
    }
    __syncthreads();
  }
}

// attention.hpp:38-174 per query row: one thread per row of a (z, h, qi) tile, the reference's
// two-pass online softmax over the listed blocks (dense: the implicit list 0..qi).
template <typename T, bool kOutBf16>
__global__ void g_attention_kernel(GenDims G, const T* __restrict__ Q, const T* __restrict__ K,
                                   const T* __restrict__ V, const int32_t* __restrict__ idx,
                                   const int32_t* __restrict__ counts, void* __restrict__ out,
                                   float* __restrict__ lse, unsigned long long* visits,
                                   int32_t* plan_error, float* __restrict__ scratch) {
  const int qi = blockIdx.x % G.M;
  const int zh = blockIdx.x / G.M;
  const int z = zh / G.Hq, h = zh % G.Hq;
  const int rows = (qi + 1 == G.M) ? G.last_len : G.B;
  const int N = G.M;
  const bool dense = idx == nullptr;
  int C = dense ? qi + 1 : counts[((size_t)z * G.M + qi) * G.Hq + h];
  if (C > N) {  // malformed plan: a row has N slots, never read past it
    if (threadIdx.x == 0 && plan_error) atomicExch(plan_error, 1);
    C = N;
  }
  const size_t kvh = (size_t)z * G.Hkv + h / G.group;
  // per-thread scratch: acc[d] + logits[B]
  for (int r = threadIdx.x; r < rows; r += blockDim.x) {
    float* acc = scratch + ((size_t)blockIdx.x * G.B + r) * (G.d + G.B);
    float* lg = acc + G.d;
    for (int c = 0; c < G.d; ++c) acc[c] = 0.f;
    float run_max = -INFINITY, run_sum = 0.f;
    const size_t qoff = ((size_t)zh * G.L + (size_t)qi * G.B + r) * G.d;
    unsigned long long vis = 0;
    for (int slot = 0; slot < C; ++slot) {
      const int bid = dense ? slot : idx[(((size_t)z * G.M + qi) * N + slot) * G.Hq + h];
      if (bid < 0 || bid >= N) {  // attention.hpp:78-81
        if (plan_error) atomicExch(plan_error, 1);
        continue;
      }
      ++vis;
      const int cols = (bid + 1 == G.M) ? G.last_len : G.B;
      const int cols_r = (bid == qi) ? min(cols, r + 1) : cols;
      const size_t kbase = (kvh * G.L + (size_t)bid * G.B) * G.d;
      float lmax = -INFINITY;
      for (int c = 0; c < cols_r; ++c) {
        lg[c] = __fmul_rn(dot4(Q, qoff, K, kbase + (size_t)c * G.d, G.d), G.to_bits);
        lmax = ref_max(lmax, lg[c]);
      }
      const float m_new = ref_max(run_max, lmax);
      const float rescale = run_max == -INFINITY ? 0.f : exp2f(__fsub_rn(run_max, m_new));
      for (int c = 0; c < G.d; ++c) acc[c] = __fmul_rn(acc[c], rescale);
      float bsum = 0.f;
      for (int c = 0; c < cols_r; ++c) {
        const float w = exp2f(__fsub_rn(lg[c], m_new));
        bsum = __fadd_rn(bsum, w);
        const size_t vrow = kbase + (size_t)c * G.d;
        for (int cc = 0; cc < G.d; ++cc) acc[cc] = __fadd_rn(acc[cc], __fmul_rn(w, ld(V, vrow + cc)));
      }
      run_sum = __fadd_rn(__fmul_rn(run_sum, rescale), bsum);
      run_max = m_new;
    }
    if (r == 0 && visits && vis) atomicAdd(visits, vis);
    const float inv = __fdiv_rn(1.0f, run_sum);
    const size_t t = (size_t)zh * G.L + (size_t)qi * G.B + r;
    for (int c = 0; c < G.d; ++c) {
      const float o = __fmul_rn(acc[c], inv);
      if constexpr (kOutBf16) reinterpret_cast<__nv_bfloat16*>(out)[t * G.d + c] = __float2bfloat16_rn(o);
      else reinterpret_cast<float*>(out)[t * G.d + c] = o;
    }
    lse[t] = __fadd_rn(run_max, log2f(run_sum));
  }
}

int gen_threads(int B) { return B >= 128 ? 128 : ((B + 31) / 32) * 32; }

}  // namespace

cudaError_t g_launch_pool(const GenDims& G, bool bf16_in, const void* K, float* pooled,
                          cudaStream_t s) {
  const int ZH = G.Z * G.Hkv;
  if (bf16_in)
    g_pool_kernel<__nv_bfloat16><<<592, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(K), pooled,
                                                     nullptr, ZH, G.L, G.d, G.B, G.M, G.last_len);
  else
    g_pool_kernel<float><<<592, 256, 0, s>>>(static_cast<const float*>(K), pooled, nullptr, ZH,
                                             G.L, G.d, G.B, G.M, G.last_len);
  return cudaGetLastError();
}

cudaError_t g_launch_approx(const GenDims& G, bool bf16_in, const void* Q, const float* pooled,
                            float* energy, float* local_max, cudaStream_t s) {
  const dim3 grid((unsigned)((size_t)G.Z * G.Hq * G.M));
  const size_t smem = sizeof(float) * (size_t)G.B;
  if (bf16_in)
    g_approx_kernel<__nv_bfloat16><<<grid, gen_threads(G.B), smem, s>>>(
        G, static_cast<const __nv_bfloat16*>(Q), pooled, energy, local_max);
  else
    g_approx_kernel<float><<<grid, gen_threads(G.B), smem, s>>>(G, static_cast<const float*>(Q),
                                                               pooled, energy, local_max);
  return cudaGetLastError();
}

size_t g_attention_scratch_bytes(const GenDims& G) {
  return sizeof(float) * (size_t)G.Z * G.Hq * G.M * G.B * (G.d + G.B);
}

cudaError_t g_launch_attention(const GenDims& G, bool bf16_in, const void* Q, const void* K,
                               const void* V, const int32_t* idx, const int32_t* counts,
                               bool out_bf16, void* out, float* lse, unsigned long long* visits,
                               int32_t* plan_error, float* scratch, cudaStream_t s) {
  const dim3 grid((unsigned)((size_t)G.Z * G.Hq * G.M));
  const int th = gen_threads(G.B);
#define FPB_GEN_ATTN(T, OB)                                                                       \
  g_attention_kernel<T, OB><<<grid, th, 0, s>>>(G, static_cast<const T*>(Q), static_cast<const T*>(K), \
                                                static_cast<const T*>(V), idx, counts, out, lse,  \
                                                visits, plan_error, scratch)
  if (bf16_in) {
    if (out_bf16) FPB_GEN_ATTN(__nv_bfloat16, true);
    else FPB_GEN_ATTN(__nv_bfloat16, false);
  } else {
    if (out_bf16) FPB_GEN_ATTN(float, true);
    else FPB_GEN_ATTN(float, false);
  }
#undef FPB_GEN_ATTN
  return cudaGetLastError();
}

}  // namespace fpb
