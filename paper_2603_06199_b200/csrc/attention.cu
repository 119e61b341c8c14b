// attention.cu — K4 block-sparse / K5 dense-causal FlashAttention prefill on tcgen05 + TMEM + TMA.
//
// Restates block_sparse_attention (attention.hpp:38-132) and dense_attention (:135-174):
//   * index-driven iteration over the compacted plan row idx[z, i, 0..C), never a scan over N
//     (the reference's "physical jumping", attention.hpp:76-81); dense = the implicit list 0..i;
//   * causal mask only inside the diagonal block (attention.hpp:85-91); listed blocks j > i are
//     attended in full; ragged last key block masked to its real length;
//   * base-2 online softmax; lse = m + log2(l) (attention.hpp:119-126); C = 0 gives NaN / -inf;
//   * GQA: Q head h reads KV head h / (Hq / Hkv).
//
// One CTA per (z, h, query block i); 256 threads:
//   w0  TMA producer  (Q once; then K_n / V_n into 3- and 2-stage rings, in MMA consumption order)
//   w1  MMA issuer    S_b = Q K_n^T (SS, K-major)  then  O += P_{n-1} V_{n-1} (TS: P from TMEM)
//   w2  TMEM allocator (512 cols: S0 | S1 | O)
//   w4..w7 softmax    thread = query row = TMEM lane: rowmax, lazy rescale (FA4-style, only when
//                     the max grows by > 2^8), exp2, P (bf16) written back over S_b in TMEM.
#include <cstdlib>

#include "fp_kernels.h"

namespace fpb {

using namespace ptx;

namespace {

constexpr int kThreads = 256;
constexpr int kTile = kBlock * kHeadDim * 2;  // 32 KiB bf16 tile
constexpr int kVStages = 2;
// bf16 inputs: one K tile per block, 3-slot ring.  fp32 inputs (NS = 2): Q and K are fed as bf16
// hi + lo splits (S = Qh Kh + Ql Kh + Qh Kl, ~fp32 logits); two K tiles per block, 2-slot ring.
template <int NS>
constexpr int k_slots() { return NS == 1 ? 3 : 2; }
constexpr float kRescaleThreshold = 8.0f;     // log2 units

struct AttnParams {
  Dims D;
  const int32_t* idx;     // nullptr -> dense causal
  const int32_t* counts;
  void* out;
  float* lse;
  unsigned long long* visits;
  int32_t* plan_error;
  int out_bf16;
};

template <int NS>
struct AttnSmem {
  static constexpr int kKStages = k_slots<NS>();
  uint8_t q[NS][kTile];
  uint8_t k[kKStages][kTile];
  uint8_t v[kVStages][kTile];
  uint64_t q_full;
  uint64_t k_full[kKStages], k_empty[kKStages];
  uint64_t v_full[kVStages], v_empty[kVStages];
  uint64_t s_full[2], s_free[2], p_full[2];
  uint64_t o_ready;
  uint32_t tmem_base;
  int nblk;
  int ired[32];
  // followed by int list[M] (dynamic)
};

template <int NS>
__global__ void __launch_bounds__(kThreads, 1)
    attention_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const AttnParams prm) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  using Smem = AttnSmem<NS>;
  constexpr int kKStages = Smem::kKStages;
  auto& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                     ~uintptr_t(1023));
  int* list = reinterpret_cast<int*>(&s + 1);
  const Dims& D = prm.D;
  const int N = D.M;

  const int h = blockIdx.x % D.Hq;
  const int t = blockIdx.x / D.Hq;
  const int qi = owned_row(D, t % D.Mr);
  const int z = t / D.Mr;
  const int zkv = z * D.Hkv + h / D.group;
  const int rows = block_len(D, qi);
  const bool dense = prm.idx == nullptr;
  const uint32_t warp = warp_id(), lane = lane_id();

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    mbar_init(smem_u32(&s.q_full), 1);
    for (int i = 0; i < kKStages; ++i) {
      mbar_init(smem_u32(&s.k_full[i]), 1);
      mbar_init(smem_u32(&s.k_empty[i]), 1);
    }
    for (int i = 0; i < kVStages; ++i) {
      mbar_init(smem_u32(&s.v_full[i]), 1);
      mbar_init(smem_u32(&s.v_empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&s.s_full[i]), 1);
      mbar_init(smem_u32(&s.s_free[i]), 1);
      mbar_init(smem_u32(&s.p_full[i]), 4);
    }
    mbar_init(smem_u32(&s.o_ready), 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(smem_u32(&s.tmem_base));

  // ---- plan row -> validated block list (attention.hpp:76-81)
  if (dense) {
    if (threadIdx.x == 0) s.nblk = qi + 1;
  } else {
    int C = prm.counts[((size_t)z * D.M + qi) * D.Hq + h];
    if (C > N) {  // malformed plan: a row has N slots, never read past it
      if (threadIdx.x == 0 && prm.plan_error) atomicExch(prm.plan_error, 1);
      C = N;
    }
    const size_t prow = ((size_t)z * D.M + qi) * (size_t)N;
    int base = 0;
    for (int s0 = 0; s0 < C; s0 += kThreads) {
      const int slot = s0 + threadIdx.x;
      int bid = 0;
      bool ok = false;
      if (slot < C) {
        bid = prm.idx[(prow + slot) * D.Hq + h];
        ok = bid >= 0 && bid < N;
        if (!ok && prm.plan_error) atomicExch(prm.plan_error, 1);
      }
      int tot;
      const int pos = base + block_prefix_count<kThreads>(ok, s.ired, &tot);
      if (ok) list[pos] = bid;
      base += tot;
    }
    if (threadIdx.x == 0) {
      s.nblk = base;
      if (prm.visits && base) atomicAdd(prm.visits, (unsigned long long)base);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;
  const int nblk = s.nblk;
  auto kv_of = [&](int n) { return dense ? n : list[n]; };

  if (warp == 0) {
    // ===================== TMA producer: K_0, K_1, V_0, K_2, V_1, ... (MMA consumption order)
    if (elect_one() && nblk > 0) {
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      const uint32_t qb = smem_u32(&s.q_full);
      mbar_arrive_expect_tx(qb, NS * kTile);
      for (int sp = 0; sp < NS; ++sp)
        for (int a = 0; a < 2; ++a)
          tma_load_3d_hint(smem_u32(s.q[sp]) + a * (kTile / 2), &tm_q, qb, a * 64, qi * kBlock,
                           sp * D.Z * D.Hq + z * D.Hq + h, pol_q);
      for (int n = 0; n <= nblk; ++n) {
        for (int sp = 0; n < nblk && sp < NS; ++sp) {
          const int item = n * NS + sp;
          const int st = item % kKStages;
          if (item >= kKStages) mbar_wait(smem_u32(&s.k_empty[st]), ((item / kKStages) - 1) & 1);
          const uint32_t fb = smem_u32(&s.k_full[st]);
          mbar_arrive_expect_tx(fb, kTile);
          const int row = kv_of(n) * kBlock;
          for (int a = 0; a < 2; ++a)
            tma_load_3d_hint(smem_u32(s.k[st]) + a * (kTile / 2), &tm_k, fb, a * 64, row,
                             sp * D.Z * D.Hkv + zkv, pol_kv);
        }
        if (n >= 1) {
          const int m = n - 1;
          const int st = m % kVStages;
          if (m >= kVStages) mbar_wait(smem_u32(&s.v_empty[st]), ((m / kVStages) - 1) & 1);
          const uint32_t fb = smem_u32(&s.v_full[st]);
          mbar_arrive_expect_tx(fb, kTile);
          const int row = kv_of(m) * kBlock;
          for (int a = 0; a < 2; ++a)
            tma_load_3d_hint(smem_u32(s.v[st]) + a * (kTile / 2), &tm_v, fb, a * 64, row, zkv,
                             pol_kv);
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer
    if (elect_one() && nblk > 0) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(128, 128, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(128, 128, false, true);
      const uint32_t o_tmem = tmem + 256;
      mbar_wait(smem_u32(&s.q_full), 0);
      auto issue_pv = [&](int m) {
        const int b = m & 1, st = m % kVStages;
        mbar_wait(smem_u32(&s.p_full[b]), (m >> 1) & 1);
        mbar_wait(smem_u32(&s.v_full[st]), (m / kVStages) & 1);
        tc_fence_after();
        const uint32_t p_tmem = tmem + b * 128;
        const uint32_t vbase = smem_u32(s.v[st]);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          mma_bf16_ts(o_tmem, p_tmem + ks * 8, sdesc_sw128(vbase + ks * 2048, kTile / 2, 1024),
                      idesc_pv, (m > 0 || ks > 0) ? 1u : 0u);
        mma_commit(smem_u32(&s.v_empty[st]));
        mma_commit(smem_u32(&s.s_free[b]));
        mma_commit(smem_u32(&s.o_ready));
      };
      for (int n = 0; n < nblk; ++n) {
        const int b = n & 1;
        if (n >= 2) mbar_wait(smem_u32(&s.s_free[b]), ((n >> 1) - 1) & 1);
        const uint32_t s_tmem = tmem + b * 128;
        for (int sp = 0; sp < NS; ++sp) {  // sp 0: K hi (x Q hi [+ Q lo]); sp 1: K lo (x Q hi)
          const int item = n * NS + sp;
          const int st = item % kKStages;
          mbar_wait(smem_u32(&s.k_full[st]), (item / kKStages) & 1);
          tc_fence_after();
          const uint32_t kbase = smem_u32(s.k[st]);
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const uint32_t off = (ks >> 2) * (kTile / 2) + (ks & 3) * 32;
            const uint64_t kd = sdesc_sw128(kbase + off, 16, 1024);
            mma_bf16_ss(s_tmem, sdesc_sw128(smem_u32(s.q[0]) + off, 16, 1024), kd, idesc_qk,
                        (sp > 0 || ks > 0) ? 1u : 0u);
            if (NS == 2 && sp == 0)
              mma_bf16_ss(s_tmem, sdesc_sw128(smem_u32(s.q[1]) + off, 16, 1024), kd, idesc_qk, 1u);
          }
          mma_commit(smem_u32(&s.k_empty[st]));
        }
        mma_commit(smem_u32(&s.s_full[b]));
        if (n >= 1) issue_pv(n - 1);
      }
      issue_pv(nblk - 1);
    }
  } else if (warp >= 4) {
    // ===================== softmax + epilogue: thread == query row == TMEM lane
    const int r = (warp - 4) * 32 + lane;
    const uint32_t lane_addr = static_cast<uint32_t>((warp - 4) * 32) << 16;
    const uint32_t o_addr = tmem + lane_addr + 256;
    float m_used = -INFINITY, l = 0.f;
    for (int n = 0; n < nblk; ++n) {
      const int b = n & 1;
      const int kv = kv_of(n);
      const int cols = block_len(D, kv);
      const int lim = (kv == qi) ? min(cols, r + 1) : cols;  // attention.hpp:88
      mbar_wait(smem_u32(&s.s_full[b]), (n >> 1) & 1);
      tc_fence_after();
      const uint32_t s_addr = tmem + lane_addr + b * 128;
      float mx = -INFINITY;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t v[32];
        tmem_ld32(s_addr + cc * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < 32; ++k)
          if (cc * 32 + k < lim) mx = fmaxf(mx, __uint_as_float(v[k]));
      }
      const float m_blk = mx * D.to_bits;
      const float m_new = fmaxf(m_used, m_blk);
      if (n == 0) {
        m_used = m_new;
      } else if (__any_sync(0xffffffffu, m_new > m_used + kRescaleThreshold)) {
        // O must contain PV_{n-1} before it is rescaled.
        mbar_wait(smem_u32(&s.o_ready), (n - 1) & 1);
        tc_fence_after();
        const float f = ex2_approx(m_used - m_new);
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t v[32];
          tmem_ld32(o_addr + cc * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 32; ++k) v[k] = __float_as_uint(__uint_as_float(v[k]) * f);
          tmem_st32(o_addr + cc * 32, v);
        }
        tmem_st_wait();
        l *= f;
        m_used = m_new;
      }
      const float neg_m = -m_used;
      float bsum = 0.f;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t v[32];
        tmem_ld32(s_addr + cc * 32, v);
        tmem_ld_wait();
        uint32_t pk[16];
#pragma unroll
        for (int k = 0; k < 32; k += 2) {
          const float p0 = (cc * 32 + k < lim)
                               ? ex2_approx(fmaf(__uint_as_float(v[k]), D.to_bits, neg_m)) : 0.f;
          const float p1 = (cc * 32 + k + 1 < lim)
                               ? ex2_approx(fmaf(__uint_as_float(v[k + 1]), D.to_bits, neg_m)) : 0.f;
          bsum += p0 + p1;
          pk[k >> 1] = pack_bf16x2(p0, p1);
        }
        tmem_st16(s_addr + cc * 16, pk);  // P_b occupies columns [0, 64) of S_b
      }
      l += bsum;
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&s.p_full[b]));
    }
    // ---- epilogue (attention.hpp:119-126)
    const size_t orow = ((size_t)z * D.Hq + h) * (size_t)D.L + (size_t)qi * kBlock + r;
    if (nblk > 0) {
      mbar_wait(smem_u32(&s.o_ready), (nblk - 1) & 1);
      tc_fence_after();
    }
    const float inv = (nblk > 0) ? 1.0f / l : __int_as_float(0x7fc00000);
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      uint32_t v[32];
      if (nblk > 0) {
        tmem_ld32(o_addr + cc * 32, v);
        tmem_ld_wait();
      }
      if (r < rows) {
        if (prm.out_bf16) {
          uint32_t pk[16];
#pragma unroll
          for (int k = 0; k < 32; k += 2)
            pk[k >> 1] = pack_bf16x2(nblk > 0 ? __uint_as_float(v[k]) * inv : inv,
                                     nblk > 0 ? __uint_as_float(v[k + 1]) * inv : inv);
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(prm.out) +
                                                orow * kHeadDim + cc * 32);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4)
            dst[q4] = make_uint4(pk[4 * q4], pk[4 * q4 + 1], pk[4 * q4 + 2], pk[4 * q4 + 3]);
        } else {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(prm.out) +
                                                  orow * kHeadDim + cc * 32);
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4) {
            float o[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              o[u] = nblk > 0 ? __uint_as_float(v[4 * q4 + u]) * inv : inv;
            dst[q4] = make_float4(o[0], o[1], o[2], o[3]);
          }
        }
      }
    }
    if (r < rows) prm.lse[orow] = (nblk > 0) ? m_used + log2f(l) : -INFINITY;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

template <int NS>
cudaError_t launch_ns(const Dims& D, const CUtensorMap& tm_q, const CUtensorMap& tm_k,
                      const CUtensorMap& tm_v, const AttnParams& prm, cudaStream_t s) {
  const size_t smem = sizeof(AttnSmem<NS>) + 1024 + sizeof(int) * (size_t)D.M;
  cudaError_t e = cudaFuncSetAttribute(attention_kernel<NS>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const dim3 grid((unsigned)((size_t)D.Z * D.Hq * D.Mr));
  attention_kernel<NS><<<grid, kThreads, smem, s>>>(tm_q, tm_k, tm_v, prm);
  return cudaGetLastError();
}

}  // namespace

// Q / K: `splits` bf16 planes each ([hi][lo] for fp32 inputs); V: one bf16 plane.
// bf16 (splits == 1) runs the persistent two-slot kernel (attention_fa.cu); the split-precision
// fp32 path runs the one-tile kernel above.
cudaError_t launch_attention(const Dims& D, int splits, const __nv_bfloat16* Q,
                             const __nv_bfloat16* K, const __nv_bfloat16* V, const int32_t* idx,
                             const int32_t* counts, bool out_bf16, void* out, float* lse,
                             unsigned long long* visits, int32_t* plan_error, int* sched,
                             uint16_t* lists, uint8_t* phase_ws, cudaStream_t s) {
  if (splits == 1)
    return launch_attention_fa(D, Q, K, V, idx, counts, out_bf16, out, lse, visits, plan_error,
                               sched, lists, phase_ws, s);
  CUtensorMap tm_q, tm_k, tm_v;
  if (!make_tmap_rows128(&tm_q, Q, D.L, (uint64_t)splits * D.Z * D.Hq) ||
      !make_tmap_rows128(&tm_k, K, D.L, (uint64_t)splits * D.Z * D.Hkv) ||
      !make_tmap_rows128(&tm_v, V, D.L, (uint64_t)D.Z * D.Hkv))
    return cudaErrorInvalidValue;
  AttnParams prm{D, idx, counts, out, lse, visits, plan_error, out_bf16 ? 1 : 0};
  return launch_ns<2>(D, tm_q, tm_k, tm_v, prm, s);
}

size_t attention_f32_smem_bytes(const Dims& D) {
  return sizeof(AttnSmem<2>) + 1024 + sizeof(int) * (size_t)D.M;
}

size_t attention_list_bytes(const Dims& D) { return (size_t)256 * 4 * D.M * sizeof(uint16_t); }

}  // namespace fpb
