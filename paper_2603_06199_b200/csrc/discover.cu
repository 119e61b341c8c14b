// discover.cu — K2 (+K3): fused block-approximate pattern discovery on tcgen05 tensor cores.
//
// Restates approx_block_scores (discovery.hpp:75-115), normalize_block_scores (:119-148) and —
// when idx/counts are requested — max_threshold_mask (selection.hpp:63-92) + compress_indices
// (selection.hpp:176-192) in ONE pass over Q, without materialising the M x N maps unless asked.
//
// One CTA per (z, h, query block I), heavy rows first, h fastest (so the head-last mask/idx rows
// of one (z, I) are written by co-resident CTAs and merge in L2).
//
//   logits^T[J, r] = k̄_J . q_r   is one UMMA per 128-block chunk of J:
//     A = k̄ chunk (M = 128 key blocks J on TMEM lanes, K = d), B = Q tile (N = 128 query rows).
//   With J on the lane axis, thread J owns the 128 logits of pair (I, J) and reduces them
//   serially in the reference's order r = 0..rows-1 (discovery.hpp:101-107) — no shuffles.
//
// Precision: k̄ is fp32 (a mean) and is fed as a bf16 hi + lo split (16 significant bits, two
// accumulating MMAs); bf16 Q is exact.  fp32 Q (the C1 config) is split too (3 MMAs: hh, hl, lh).
// Naively rounding k̄ to bf16 flips mask bits (SURVEY §7 hard part 1).
//
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM allocator,
// w4..w7 epilogue (TMEM -> (m, S) per pair), then all 8 warps normalise / threshold / compact.
#include "fp_kernels.h"

namespace fpb {

using namespace ptx;

namespace {

constexpr int kThreads = 256;
constexpr int kTile = kBlock * kHeadDim * 2;  // one bf16 128x128 operand tile: 32 KiB
constexpr int kStages = 2;                    // k̄ chunk ring

struct DiscParams {
  Dims D;
  DiscoverOut out;
};

template <int NQ>
struct DiscSmem {
  uint8_t q[NQ][kTile];               // Q tile(s): hi (and lo for fp32 inputs)
  uint8_t kb[kStages][2][kTile];      // k̄ chunk: hi, lo
  uint64_t q_full;
  uint64_t kb_full[kStages], kb_empty[kStages];
  uint64_t d_full[2], d_empty[2];
  uint32_t tmem_base;
  float red[32];
  int ired[32];
  // followed by float m_s[M], S_s[M] (dynamic)
};

template <int NQ>
__global__ void __launch_bounds__(kThreads, 1)
    discover_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kb,
                    const DiscParams prm) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  auto& s = *reinterpret_cast<DiscSmem<NQ>*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  float* m_s = reinterpret_cast<float*>(&s + 1);
  const Dims& D = prm.D;
  float* S_s = m_s + D.M;

  // ---- work item: h fastest, heavy (large I) first
  const int h = blockIdx.x % D.Hq;
  const int t = blockIdx.x / D.Hq;
  const int I = D.M - 1 - (t % D.M);
  const int z = t / D.M;
  const int zkv = z * D.Hkv + h / D.group;
  const int rows = block_len(D, I);
  const int nchunks = I / kBlock + 1;  // J-chunks of 128 covering 0..I

  const uint32_t warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_kb);
    mbar_init(smem_u32(&s.q_full), 1);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(smem_u32(&s.kb_full[i]), 1);
      mbar_init(smem_u32(&s.kb_empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&s.d_full[i]), 1);
      mbar_init(smem_u32(&s.d_empty[i]), 4);  // one arrive per epilogue warp
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<256>(smem_u32(&s.tmem_base));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;

  if (warp == 0) {
    // ===================== TMA producer
    if (elect_one()) {
      const uint32_t qb = smem_u32(&s.q_full);
      mbar_arrive_expect_tx(qb, NQ * kTile);
      for (int p = 0; p < NQ; ++p)
        for (int a = 0; a < 2; ++a)
          tma_load_3d(smem_u32(s.q[p]) + a * (kTile / 2), &tm_q, qb, a * 64, I * kBlock,
                      p * D.Z * D.Hq + z * D.Hq + h);
      for (int c = 0; c < nchunks; ++c) {
        const int st = c % kStages;
        if (c >= kStages) mbar_wait(smem_u32(&s.kb_empty[st]), ((c / kStages) - 1) & 1);
        const uint32_t fb = smem_u32(&s.kb_full[st]);
        mbar_arrive_expect_tx(fb, 2 * kTile);
        for (int sp = 0; sp < 2; ++sp)
          for (int a = 0; a < 2; ++a)
            tma_load_3d(smem_u32(s.kb[st][sp]) + a * (kTile / 2), &tm_kb, fb, a * 64, c * kBlock,
                        sp * D.Z * D.Hkv + zkv);
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (one thread)
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, 128, false, false);
      mbar_wait(smem_u32(&s.q_full), 0);
      tc_fence_after();
      for (int c = 0; c < nchunks; ++c) {
        const int st = c % kStages, buf = c & 1;
        if (c >= 2) mbar_wait(smem_u32(&s.d_empty[buf]), ((c >> 1) - 1) & 1);
        mbar_wait(smem_u32(&s.kb_full[st]), (c / kStages) & 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem + buf * 128;
        for (int ks = 0; ks < 8; ++ks) {
          const uint32_t off = (ks >> 2) * (kTile / 2) + (ks & 3) * 32;
          const uint64_t a_hi = sdesc_sw128(smem_u32(s.kb[st][0]) + off, 16, 1024);
          const uint64_t a_lo = sdesc_sw128(smem_u32(s.kb[st][1]) + off, 16, 1024);
          const uint64_t b_q0 = sdesc_sw128(smem_u32(s.q[0]) + off, 16, 1024);
          mma_bf16_ss(d_tmem, a_hi, b_q0, idesc, ks > 0);
          mma_bf16_ss(d_tmem, a_lo, b_q0, idesc, 1);
          if constexpr (NQ == 2) {
            const uint64_t b_q1 = sdesc_sw128(smem_u32(s.q[1]) + off, 16, 1024);
            mma_bf16_ss(d_tmem, a_hi, b_q1, idesc, 1);
          }
        }
        mma_commit(smem_u32(&s.kb_empty[st]));
        mma_commit(smem_u32(&s.d_full[buf]));
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue: TMEM row J -> (local max m, energy S)
    const int jl = (warp - 4) * 32 + lane;  // TMEM lane == key block within the chunk
    const uint32_t lane_addr = static_cast<uint32_t>((warp - 4) * 32) << 16;
    for (int c = 0; c < nchunks; ++c) {
      const int buf = c & 1;
      mbar_wait(smem_u32(&s.d_full[buf]), (c >> 1) & 1);
      tc_fence_after();
      const uint32_t base = tmem + lane_addr + buf * 128;
      float m = kNegSentinel;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t v[32];
        tmem_ld32(base + cc * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float x = __fmul_rn(__uint_as_float(v[k]), D.to_bits);
          if (cc * 32 + k < rows) m = fmaxf(m, x);
        }
      }
      float S = 0.f;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t v[32];
        tmem_ld32(base + cc * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float x = __fmul_rn(__uint_as_float(v[k]), D.to_bits);
          if (cc * 32 + k < rows) S = __fadd_rn(S, exp2f(__fsub_rn(x, m)));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&s.d_empty[buf]));
      const int J = c * kBlock + jl;
      if (J <= I) {
        m_s[J] = m;
        S_s[J] = S;
      }
    }
  }
  __syncthreads();

  // ===================== row normalisation (discovery.hpp:131-143), all 256 threads
  const int N = D.M;
  const size_t map_row = (((size_t)z * D.Hq + h) * D.M + I) * (size_t)N;
  if (prm.out.energy || prm.out.local_max) {
    for (int J = threadIdx.x; J < N; J += kThreads) {
      if (prm.out.energy) prm.out.energy[map_row + J] = (J <= I) ? S_s[J] : 0.f;
      if (prm.out.local_max) prm.out.local_max[map_row + J] = (J <= I) ? m_s[J] : kNegSentinel;
    }
  }
  if (prm.out.normalize) {
    float rmax = kNegSentinel;
    for (int J = threadIdx.x; J <= I; J += kThreads) rmax = fmaxf(rmax, m_s[J]);
    rmax = block_max<kThreads>(rmax, s.red);
    float total = 0.f;
    for (int J = threadIdx.x; J <= I; J += kThreads) {
      const float r = __fmul_rn(S_s[J], exp2f(__fsub_rn(m_s[J], rmax)));
      S_s[J] = r;
      total += r;
    }
    total = block_sum<kThreads>(total, s.red);
    const float inv = __fdiv_rn(1.0f, __fadd_rn(total, D.eps));
    float smax = 0.0f;  // selection.hpp:75
    for (int J = threadIdx.x; J <= I; J += kThreads) {
      const float sc = __fmul_rn(S_s[J], inv);
      S_s[J] = sc;
      smax = fmaxf(smax, sc);
    }
    if (prm.out.score)
      for (int J = threadIdx.x; J < N; J += kThreads)
        prm.out.score[map_row + J] = (J <= I) ? S_s[J] : 0.f;

    // ===================== fused max-threshold + compaction (selection.hpp:63-92, 176-192)
    if (prm.out.idx || prm.out.mask) {
      smax = block_max<kThreads>(smax, s.red);
      const float thresh = __fmul_rn(D.alpha, smax);
      const size_t plan_row = ((size_t)z * D.M + I) * (size_t)N;  // [z, I, :, :]
      int base = 0;
      for (int J0 = 0; J0 < N; J0 += kThreads) {
        const int J = J0 + threadIdx.x;
        bool act = false;
        if (J <= I)
          act = (S_s[J] >= thresh) || J < D.sink_blocks || (I - J) < D.window_blocks;
        int total_act;
        const int slot = base + block_prefix_count<kThreads>(act, s.ired, &total_act);
        if (prm.out.mask && J < N) prm.out.mask[(plan_row + J) * D.Hq + h] = act ? 1 : 0;
        if (prm.out.idx && act) prm.out.idx[(plan_row + slot) * D.Hq + h] = J;
        base += total_act;
        if (J0 + kThreads > I) {  // nothing active beyond I: finish mask row only
          for (int J2 = J0 + kThreads + threadIdx.x; prm.out.mask && J2 < N; J2 += kThreads)
            prm.out.mask[(plan_row + J2) * D.Hq + h] = 0;
          break;
        }
      }
      if (prm.out.idx)
        for (int slot = base + threadIdx.x; slot < N; slot += kThreads)
          prm.out.idx[(plan_row + slot) * D.Hq + h] = N;
      if (prm.out.counts && threadIdx.x == 0) prm.out.counts[((size_t)z * D.M + I) * D.Hq + h] = base;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<256>(tmem);
}

template <int NQ>
size_t disc_smem_bytes(int M) {
  return sizeof(DiscSmem<NQ>) + 1024 + 2 * sizeof(float) * (size_t)M;
}

}  // namespace

cudaError_t launch_discover(const Dims& D, int q_splits, const __nv_bfloat16* q_planes,
                            const __nv_bfloat16* kbar_split, const DiscoverOut& out,
                            cudaStream_t s) {
  CUtensorMap tm_q, tm_kb;
  if (!make_tmap_rows128(&tm_q, q_planes, D.L, (uint64_t)q_splits * D.Z * D.Hq) ||
      !make_tmap_rows128(&tm_kb, kbar_split, D.M, 2ull * D.Z * D.Hkv))
    return cudaErrorInvalidValue;
  DiscParams prm{D, out};
  const dim3 grid((unsigned)((size_t)D.Z * D.Hq * D.M));
  if (q_splits == 1) {
    const size_t smem = disc_smem_bytes<1>(D.M);
    cudaError_t e = cudaFuncSetAttribute(discover_kernel<1>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    discover_kernel<1><<<grid, kThreads, smem, s>>>(tm_q, tm_kb, prm);
  } else {
    const size_t smem = disc_smem_bytes<2>(D.M);
    cudaError_t e = cudaFuncSetAttribute(discover_kernel<2>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    discover_kernel<2><<<grid, kThreads, smem, s>>>(tm_q, tm_kb, prm);
  }
  return cudaGetLastError();
}

}  // namespace fpb
