// discover.cu — K2 (+K3): fused block-approximate pattern discovery on tcgen05 tensor cores.
//
// Restates approx_block_scores (discovery.hpp:75-115), normalize_block_scores (:119-148) and —
// when idx/counts are requested — max_threshold_mask (selection.hpp:63-92) + compress_indices
// (selection.hpp:176-192) in ONE pass over Q, without materialising the M x N maps unless asked.
//
// Work item = (z, h, query block I), dealt heavy-first (large I) by a dynamic scheduler to a
// persistent grid of one CTA per SM.  For every item:
//   logits^T[J, r] = k̄_J . q_r   is one UMMA per 128-block chunk of J:
//     A = k̄ chunk (M = 128 key blocks J on TMEM lanes, K = d), B = Q tile (N = 128 query rows).
//   With J on the lane axis, thread J owns the 128 logits of pair (I, J) and reduces them
//   serially in the reference's order r = 0..rows-1 (discovery.hpp:101-107) — no shuffles.
//
// Precision: k̄ is fp32 (a mean) and is fed as a bf16 hi + lo split (16 significant bits, two
// accumulating MMAs); bf16 Q is exact.  fp32 Q (the C1 config) is split too (3 MMAs: hh, hl, lh).
// Naively rounding k̄ to bf16 flips mask bits (SURVEY §7 hard part 1).
//
// Pooling (discovery.hpp:39-70) runs in the same launch for bf16 keys: every CTA first claims
// (z, kv head, key block) units from a global counter, stages each block's 128 contiguous K rows
// in shared memory with one bulk copy (TMA engine; two in flight per warpgroup), sums one channel
// per thread in the reference's order and writes the k̄ hi/lo planes, then publishes the block
// on a per-(kv head, 128-block chunk) counter (release).  The TMA producer acquires a chunk's
// counter before its first k̄ load of that chunk.  Units are claimed dynamically and a CTA waits
// only after the claims ran out, so every claimed unit belongs to a running CTA: no co-residency
// assumption, no deadlock with concurrent kernels.
//
// Warp roles (384 threads, persistent):
//   w2  TMEM allocator (512 cols), then scheduler + TMA producer: item ring (with each item's
//       chunk count), Q tiles (double-buffered), k̄ chunk ring
//   w3  MMA issuer (single thread); TMEM accumulators double-buffered per epilogue warpgroup
//   w0, w1 idle (the control roles sit on the sub-partitions with the lightest epilogue load)
//   w4..w7, w8..w11  two epilogue warpgroups, items alternating: TMEM -> (m, S) per pair, then
//          row normalisation, threshold and compaction for the item while the MMA warp and the
//          other warpgroup already work on the next ones.
#include <cstddef>
#include <cstdlib>

#include "fp_kernels.h"

namespace fpb {

using namespace ptx;

namespace {

constexpr int kThreads = 384;
constexpr int kEpiThreads = 128;               // per epilogue warpgroup (two of them)
constexpr int kTile = kBlock * kHeadDim * 2;  // one bf16 128x128 operand tile: 32 KiB
constexpr int kStages = 2;                    // k̄ chunk ring (hi + lo per stage)
constexpr int kItemRing = 4;
constexpr int kPoolTiles = 6;  // in-kernel pooling staging ring (the q and kb tiles of NQ = 1)
constexpr uint32_t kEpiBar = 1;               // named barriers 1, 2: the two epilogue warpgroups
// Control roles sit on the SM sub-partitions whose epilogue warps are least loaded: epilogue warp
// w4 + i serves key blocks J = 32i..32i+31 of a chunk, and short causal chunks leave the high
// quarters idle, so the single MMA-issuing thread (whose serial bookkeeping competes for issue
// slots with the epilogue warps of its sub-partition) runs on warp 3.
#ifndef FPB_DISC_MMA_WARP
#define FPB_DISC_MMA_WARP 3
#endif
#ifndef FPB_DISC_PRODUCER_WARP
#define FPB_DISC_PRODUCER_WARP 2
#endif
constexpr uint32_t kMmaWarp = FPB_DISC_MMA_WARP;
#ifndef FPB_DISC_TMEM0
#define FPB_DISC_TMEM0 0
#endif
#ifndef FPB_DISC_M64
#define FPB_DISC_M64 1
#endif
constexpr uint32_t kProducerWarp = FPB_DISC_PRODUCER_WARP;

struct DiscParams {
  Dims D;
  DiscoverOut out;
  int* sched;      // zeroed work counter
  int num_items;
  int prefilled;   // idx rows already hold the fill value N (launch_fill_plan)
  float* mscratch;  // per-CTA m/S rows in global memory when they do not fit in shared memory
  // in-kernel pooling (bf16 keys): K, the k̄ hi/lo destination, optional fp32 k̄, and the zeroed
  // counters [claim, pooled blocks per (z * Hkv + kv, chunk)]; kpool == nullptr: k̄ is given
  const __nv_bfloat16* kpool;
  __nv_bfloat16* kbar;
  float* pooled;
  int* pool_ctr;
};

template <int NQ>
struct DiscSmem {
  static constexpr int kQBuf = NQ == 1 ? 2 : 1;  // Q double-buffered across items (bf16 input)
  uint8_t q[kQBuf][NQ][kTile];
  uint8_t kb[kStages][2][kTile];
  uint64_t q_full[kQBuf], q_empty[kQBuf];
  uint64_t kb_full[kStages], kb_empty[kStages];
  uint64_t d_full[4], d_empty[4];  // TMEM accumulators: 2 per epilogue warpgroup
  uint64_t it_full[kItemRing], it_empty[kItemRing];
  int items[kItemRing];
  int nch[kItemRing];  // k̄ chunks of the item (I / 128 + 1), decoded once by the producer
  int lastlive[kItemRing];  // causal key blocks of its last chunk (I % 128 + 1)
  uint32_t tmem_base;
  float red[2][3][4];
  uint64_t pool_full[6], pool_empty[6];  // in-kernel pooling: 6 staging tiles over q and kb
  int pool_unit[6];
  // followed by float m_s[M], S_s[M] per epilogue warpgroup, then int counts[ceil(M/128)][4]
  // per epilogue warpgroup (dynamic)
};

// the in-kernel pooling ring spans the q and kb tiles of the bf16 (NQ = 1) layout
static_assert(offsetof(DiscSmem<1>, kb) == offsetof(DiscSmem<1>, q) + 2 * kTile &&
                  sizeof(DiscSmem<1>::q) + sizeof(DiscSmem<1>::kb) == kPoolTiles * kTile,
              "pooling tiles");

__device__ __forceinline__ void decode_item(const Dims& D, int item, int& z, int& h, int& I) {
  h = item % D.Hq;  // h fastest: co-running CTAs fill the head-last plan rows of one (z, I)
  const int t = item / D.Hq;
  I = owned_row(D, t % D.Mr);  // heavy rows first
  z = t / D.Mr;
}

#ifdef FPB_TRACE
// cycle accounting (tools/trace_discover.py): per-thread accumulators, lane 0 of each warp flushes
__device__ unsigned long long g_dtrace[32];
#define DT_DECL unsigned long long dt_acc[32] = {}; long long _dt = 0
#define DT_T0() _dt = clock64()
#define DT_ADD(i)                                \
  do {                                           \
    const long long _n = clock64();              \
    dt_acc[i] += (unsigned long long)(_n - _dt); \
    _dt = _n;                                    \
  } while (0)
#define DT_FLUSH()                                                         \
  do {                                                                     \
    if (lane_id() == 0)                                                    \
      for (int _i = 0; _i < 32; ++_i)                                      \
        if (dt_acc[_i]) atomicAdd(&g_dtrace[_i], dt_acc[_i]);              \
  } while (0)
#else
#define DT_DECL
#define DT_T0()
#define DT_ADD(i)
#define DT_FLUSH()
#endif

template <int NQ>
__global__ void __launch_bounds__(kThreads, 1)
    discover_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kb,
                    const DiscParams prm) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  using Smem = DiscSmem<NQ>;
  constexpr int kQBuf = Smem::kQBuf;
  auto& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                     ~uintptr_t(1023));
  const Dims& D = prm.D;

  const uint32_t warp = warp_id(), lane = lane_id();
  DT_DECL;
#ifdef FPB_TRACE
  const long long t_begin = clock64();
  auto gtimer = [] {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
  };
  if (threadIdx.x == 0) {  // CTA start spread (globaltimer ns): [28] = ~min, [29] = max
    const unsigned long long t0 = gtimer();
    atomicMax(&g_dtrace[28], ~t0);
    atomicMax(&g_dtrace[29], t0);
  }
#endif

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_kb);
    for (int i = 0; i < kQBuf; ++i) {
      mbar_init(smem_u32(&s.q_full[i]), 1);
      mbar_init(smem_u32(&s.q_empty[i]), 1);
    }
    for (int i = 0; i < kStages; ++i) {
      mbar_init(smem_u32(&s.kb_full[i]), 1);
      mbar_init(smem_u32(&s.kb_empty[i]), 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(smem_u32(&s.d_full[i]), 1);
      mbar_init(smem_u32(&s.d_empty[i]), 4);  // one arrive per epilogue warp
    }
    for (int i = 0; i < kItemRing; ++i) {
      mbar_init(smem_u32(&s.it_full[i]), 1);
      mbar_init(smem_u32(&s.it_empty[i]), 1 + 4);  // MMA thread + the owning epilogue warpgroup
    }
    for (int t = 0; t < kPoolTiles; ++t) {
      mbar_init(smem_u32(&s.pool_full[t]), 1);
      mbar_init(smem_u32(&s.pool_empty[t]), 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(smem_u32(&s.tmem_base));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
#if FPB_DISC_TMEM0
  // the whole TMEM (512 columns) is allocated, so the allocation starts at lane 0, column 0
  constexpr uint32_t tmem = 0;
  if (threadIdx.x == 0 && s.tmem_base != 0u) __trap();
#else
  const uint32_t tmem = s.tmem_base;
#endif
  const int nck = (D.M + kBlock - 1) / kBlock;

  if constexpr (NQ == 1) {
    if (prm.kpool) {
      // ===================== pooling (discovery.hpp:39-70).  Warp 0 lane 0 claims units (one
      // k̄ block each) in batches from the global counter and streams them with bulk copies into
      // a 6-tile ring over the (still unused) q and kb tiles; the two epilogue warpgroups take
      // alternate tiles, one channel per thread, and publish each block on its chunk counter.
      const int units = D.Z * D.Hkv * D.M;
      const uint32_t stage0 = smem_u32(s.q);
      if (warp == 0) {
        if (lane == 0) {
          // guided self-scheduling: each claim takes half the fair share of what is left, so the
          // CTAs that start first cannot take whole shares that later CTAs then wait for
          int next_u = 0, have = 0, ends = 0;
          for (int k = 0; ends < 2; ++k) {
            const int t = k % kPoolTiles;
            DT_T0();
            if (k >= kPoolTiles) mbar_wait(smem_u32(&s.pool_empty[t]), ((k / kPoolTiles) - 1) & 1);
            DT_ADD(25);  // pooling loader: waiting for a free tile
            int u = units;
            if (!ends) {
              if (have == 0) {
                const int batch = min(16, max(1, (units - next_u) / (2 * (int)gridDim.x)));
                next_u = atomicAdd(prm.pool_ctr, batch);
                have = batch;
              }
              u = next_u++;
              --have;
            }
            DT_ADD(24);  // pooling loader: claims
            const uint32_t fb = smem_u32(&s.pool_full[t]);
            if (u >= units) {  // one end marker per consumer warpgroup (k, k + 1)
              s.pool_unit[t] = -1;
              mbar_arrive(fb);
              ++ends;
              continue;
            }
            s.pool_unit[t] = u;
            const int zkv = u / D.M, j = u % D.M;
            const uint32_t bytes = (uint32_t)(block_len(D, j) * kHeadDim * 2);
            mbar_arrive_expect_tx(fb, bytes);
            bulk_load_1d(stage0 + t * kTile,
                         prm.kpool + ((size_t)zkv * D.L + (size_t)j * kBlock) * kHeadDim, bytes, fb);
          }
        }
      } else if (warp >= 4) {
        const int g = (warp - 4) >> 2, c = threadIdx.x & 127;
        const size_t plane = (size_t)D.Z * D.Hkv * D.M * kHeadDim;
        // blocks are published per chunk run: one proxy fence + release per run of consecutive
        // units of the same (kv head, chunk), not per block
        int run_key = -1, run_len = 0;
        auto publish = [&]() {
          if (run_len == 0) return;
          fence_proxy_async_global();  // k̄ is read by TMA (async proxy), in other CTAs
          named_bar_sync(3 + g, 128);
          if (c == 0) {
            __threadfence();
            red_add_release_gpu(prm.pool_ctr + 1 + run_key, run_len);
          }
          run_len = 0;
        };
        for (int k = g;; k += 2) {
          const int t = k % kPoolTiles;
          DT_T0();
          mbar_wait(smem_u32(&s.pool_full[t]), (k / kPoolTiles) & 1);
          DT_ADD(25);  // pooling: waiting for the block's rows
          const int u = s.pool_unit[t];
          if (u < 0) break;
          const int zkv = u / D.M, j = u % D.M, len = block_len(D, j);
          const int key = zkv * nck + j / kBlock;
          if (key != run_key) {
            publish();
            run_key = key;
          }
          // channel c of row r at stage + 2 (r d + c); explicit ld.shared (the aligned Smem view
          // hides the address space from the compiler)
          const uint32_t col = stage0 + t * kTile + 2 * c;
          auto row = [&](int r) {
            uint16_t x;
            asm volatile("ld.shared.u16 %0, [%1];" : "=h"(x) : "r"(col + r * 2 * kHeadDim));
            return __bfloat162float(__ushort_as_bfloat16(x));
          };
          float sum = 0.f;  // discovery.hpp:51-53: out[c] += row[c], r ascending
          if (len == kBlock) {
#pragma unroll 32
            for (int r = 0; r < kBlock; ++r) sum = __fadd_rn(sum, row(r));
          } else {
            for (int r = 0; r < len; ++r) sum = __fadd_rn(sum, row(r));
          }
          DT_ADD(26);  // pooling: channel sums
          const float o = __fmul_rn(sum, __fdiv_rn(1.0f, (float)len));  // discovery.hpp:55-56
          const size_t dst = ((size_t)zkv * D.M + j) * kHeadDim + c;
          if (prm.pooled) prm.pooled[dst] = o;
          const __nv_bfloat16 hi = __float2bfloat16_rn(o);
          prm.kbar[dst] = hi;
          prm.kbar[plane + dst] = __float2bfloat16_rn(__fsub_rn(o, __bfloat162float(hi)));
          fence_proxy_async_smem();  // the tile is refilled by a bulk copy
          named_bar_sync(3 + g, 128);
          if (c == 0) mbar_arrive(smem_u32(&s.pool_empty[t]));
          ++run_len;
          DT_ADD(27);  // pooling: k̄ stores, tile release
        }
        publish();
      }
      __syncthreads();  // the staging tiles become the Q / k̄ rings
#ifdef FPB_TRACE
      if (threadIdx.x == 0) {
        dt_acc[6] += (unsigned long long)(clock64() - t_begin);
        atomicMax(&g_dtrace[30], gtimer());  // latest prologue end
      }
#endif
    }
  }

  if (warp == kProducerWarp) {
    // ===================== scheduler + TMA producer
    if (elect_one()) {
      int gc = 0;  // global chunk counter (same sequence as the MMA issuer)
      uint64_t ready = 0;  // in-kernel pooling: k̄ chunks already seen complete (first 64 keys)
      auto wait_pooled = [&](int zkv, int c) {
        const int key = zkv * nck + c;
        if (key < 64 && ((ready >> key) & 1)) return;
        const int need = min(kBlock, D.M - c * kBlock);
        while (ld_acquire_gpu(prm.pool_ctr + 1 + key) < need) __nanosleep(64);
        fence_proxy_async_global();  // the acquired k̄ stores before this CTA's TMA reads
        if (key < 64) ready |= 1ull << key;
#ifdef FPB_TRACE
        atomicMax(&g_dtrace[31], gtimer());  // latest first sight of a pooled chunk
#endif
      };
      for (int t = 0;; ++t) {
        const int slot = t % kItemRing;
        DT_T0();
        if (t >= kItemRing) mbar_wait(smem_u32(&s.it_empty[slot]), ((t / kItemRing) - 1) & 1);
        DT_ADD(12);  // producer: item ring full (epilogue behind)
        int item = atomicAdd(prm.sched, 1);
        DT_ADD(15);  // producer: work-counter atomic
        if (item >= prm.num_items) item = -1;
        int z = 0, h = 0, I = 0;
        if (item >= 0) {
          decode_item(D, item, z, h, I);
          s.nch[slot] = I / kBlock + 1;
          s.lastlive[slot] = I % kBlock + 1;
        }
        s.items[slot] = item;
        mbar_arrive(smem_u32(&s.it_full[slot]));
        if (item < 0) {  // the other epilogue warpgroup needs its own end marker
          const int t2 = t + 1, slot2 = t2 % kItemRing;
          if (t2 >= kItemRing) mbar_wait(smem_u32(&s.it_empty[slot2]), ((t2 / kItemRing) - 1) & 1);
          s.items[slot2] = -1;
          mbar_arrive(smem_u32(&s.it_full[slot2]));
          break;
        }
        const int zkv = z * D.Hkv + h / D.group;
        const int qb = t % kQBuf;
        DT_T0();
        if (t >= kQBuf) mbar_wait(smem_u32(&s.q_empty[qb]), ((t / kQBuf) - 1) & 1);
        DT_ADD(13);  // producer: Q buffer busy (MMA behind)
        const uint32_t qf = smem_u32(&s.q_full[qb]);
        mbar_arrive_expect_tx(qf, NQ * kTile);
        for (int p = 0; p < NQ; ++p)
          for (int a = 0; a < 2; ++a)
            tma_load_3d(smem_u32(s.q[qb][p]) + a * (kTile / 2), &tm_q, qf, a * 64, I * kBlock,
                        p * D.Z * D.Hq + z * D.Hq + h);
        const int nchunks = I / kBlock + 1;
        for (int c = 0; c < nchunks; ++c, ++gc) {
          const int st = gc % kStages;
          DT_T0();
          if (gc >= kStages) mbar_wait(smem_u32(&s.kb_empty[st]), ((gc / kStages) - 1) & 1);
          DT_ADD(14);  // producer: k̄ ring full
          if (NQ == 1 && prm.kpool) wait_pooled(zkv, c);
          DT_ADD(23);  // producer: waiting for in-kernel pooling
          const uint32_t fb = smem_u32(&s.kb_full[st]);
          mbar_arrive_expect_tx(fb, 2 * kTile);
          for (int sp = 0; sp < 2; ++sp)
            for (int a = 0; a < 2; ++a)
              tma_load_3d(smem_u32(s.kb[st][sp]) + a * (kTile / 2), &tm_kb, fb, a * 64,
                          c * kBlock, sp * D.Z * D.Hkv + zkv);
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer (one thread)
    if (elect_one()) {
      constexpr uint32_t idesc128 = idesc_bf16_f32(128, 128, false, false);
      // a last chunk with at most 64 causal key blocks: an M = 64 MMA on its first 64 k̄ rows
      // (half the tensor work; the accumulator rows land in lanes 0-15 of each TMEM quarter)
      constexpr uint32_t idesc64 = idesc_bf16_f32(64, 128, false, false);
      int gc = 0, dc0 = 0, dc1 = 0;  // chunks issued in total / per epilogue warpgroup
      for (int t = 0;; ++t) {
        const int slot = t % kItemRing;
        DT_T0();
        mbar_wait(smem_u32(&s.it_full[slot]), (t / kItemRing) & 1);
        DT_ADD(19);  // MMA: waiting for the next item
        const int item = s.items[slot];
        const int nchunks = s.nch[slot];
        const int lastlive = s.lastlive[slot];
        mbar_arrive(smem_u32(&s.it_empty[slot]));
        if (item < 0) break;
        const int qb = t % kQBuf, wg = t & 1;
        DT_ADD(21);  // MMA: item decode
        mbar_wait(smem_u32(&s.q_full[qb]), (t / kQBuf) & 1);
        DT_ADD(8);  // MMA: waiting for Q
        for (int c = 0; c < nchunks; ++c, ++gc) {
          const int dc = wg ? dc1++ : dc0++;
          const int st = gc % kStages, buf = wg * 2 + (dc & 1);
          DT_ADD(22);  // MMA: loop overhead between chunks
          if (dc >= 2) mbar_wait(smem_u32(&s.d_empty[buf]), ((dc >> 1) - 1) & 1);
          DT_ADD(9);  // MMA: waiting for the accumulator (epilogue behind)
          mbar_wait(smem_u32(&s.kb_full[st]), (gc / kStages) & 1);
          DT_ADD(10);  // MMA: waiting for the k̄ chunk
          tc_fence_after();
          const uint32_t d_tmem = tmem + buf * 128;
          // SW128 descriptors are linear in the address field: base + constant per K step
          const uint64_t a_hi = sdesc_sw128(smem_u32(s.kb[st][0]), 16, 1024);
          const uint64_t a_lo = sdesc_sw128(smem_u32(s.kb[st][1]), 16, 1024);
          const uint64_t b_q0 = sdesc_sw128(smem_u32(s.q[qb][0]), 16, 1024);
          const uint64_t b_q1 = sdesc_sw128(smem_u32(s.q[qb][NQ - 1]), 16, 1024);
          const uint32_t idesc =
              (FPB_DISC_M64 && c == nchunks - 1 && lastlive <= 64) ? idesc64 : idesc128;
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const uint64_t off = ((ks >> 2) * (kTile / 2) + (ks & 3) * 32) >> 4;
            mma_bf16_ss(d_tmem, a_hi + off, b_q0 + off, idesc, ks > 0);
            mma_bf16_ss(d_tmem, a_lo + off, b_q0 + off, idesc, 1);
            if constexpr (NQ == 2) mma_bf16_ss(d_tmem, a_hi + off, b_q1 + off, idesc, 1);
          }
          mma_commit(smem_u32(&s.kb_empty[st]));
          mma_commit(smem_u32(&s.d_full[buf]));
          DT_ADD(11);  // MMA: issue
        }
        mma_commit(smem_u32(&s.q_empty[qb]));
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue: two warpgroups, items alternate between them
    // Thread et owns key blocks J = c*128 + et (TMEM lane et of every chunk c) end to end, so the
    // per-J state (m_s, S_s) never crosses threads and an item needs only three barrier rounds:
    // row max of m, (sum, max) of the rescaled energies, and the compaction counts.
    const int wg = (warp - 4) >> 2;
    const uint32_t ebar = kEpiBar + wg;
    const int w4 = warp & 3;
    float(*red)[4] = s.red[wg];       // [0]: row max, [1]/[2]: total / max of S'
    const int nck = (D.M + kBlock - 1) / kBlock;
    float* dyn = reinterpret_cast<float*>(&s + 1);
    // m_s/S_s rows are thread-owned (J = c*128 + et): shared memory, or a per-CTA global
    // scratch (coalesced, L1-resident) for sequences whose rows do not fit next to the rings
    float* m_s = prm.mscratch ? prm.mscratch + ((size_t)blockIdx.x * 2 + wg) * 2 * D.M
                              : dyn + (size_t)wg * 2 * D.M;
    float* S_s = m_s + D.M;
    int* ired = reinterpret_cast<int*>(dyn + (prm.mscratch ? 0 : 4 * (size_t)D.M)) +
                (size_t)wg * 4 * nck;  // [chunk][warp] active counts
    const int et = (threadIdx.x - 128) & 127;  // 0..127 within the warpgroup
    const uint32_t lane_addr = static_cast<uint32_t>(w4 * 32) << 16;
    const int N = D.M;
    int dc = 0;
    for (int t = wg;; t += 2) {
      const int slot = t % kItemRing;
      DT_T0();
      mbar_wait(smem_u32(&s.it_full[slot]), (t / kItemRing) & 1);
      DT_ADD(5);  // epilogue: waiting for an item
      const int item = s.items[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&s.it_empty[slot]));
      if (item < 0) break;
      int z, h, I;
      decode_item(D, item, z, h, I);
      const int rows = block_len(D, I);
      const int nchunks = I / kBlock + 1;
      float tmax = kNegSentinel;  // this thread's max of m over its J <= I

      // ---- per chunk: TMEM row J -> (local max m, energy S)  (discovery.hpp:96-110)
      for (int c = 0; c < nchunks; ++c, ++dc) {
        const int buf = wg * 2 + (dc & 1);
        DT_T0();
        mbar_wait(smem_u32(&s.d_full[buf]), (dc >> 1) & 1);
        DT_ADD(0);  // epilogue: waiting for the accumulator
        tc_fence_after();
        // M = 64 last chunks (see the MMA issuer): key block 16 q + i sits in lane i < 16 of
        // TMEM quarter q; lanes 16-31 hold nothing (J past the row)
        const bool m64 = FPB_DISC_M64 && c == nchunks - 1 && (I % kBlock) < 64;
        const int jl = m64 ? (lane < 16 ? w4 * 16 + (int)lane : kBlock) : et;
        const int J = c * kBlock + jl;
        const bool warp_live = c * kBlock + w4 * (m64 ? 16 : 32) <= I;  // warp-uniform
        float m = kNegSentinel, S = 0.f;
        if (warp_live) {
          uint32_t v[128];
          const uint32_t base = tmem + lane_addr + buf * 128;
          tmem_ld32(base + 0, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
          tmem_ld32(base + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
          tmem_ld32(base + 64, *reinterpret_cast<uint32_t(*)[32]>(&v[64]));
          tmem_ld32(base + 96, *reinterpret_cast<uint32_t(*)[32]>(&v[96]));
          tmem_ld_wait();
          DT_ADD(1);  // epilogue: TMEM load
          // TMEM is in registers: release the accumulator to the MMA warp right away
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&s.d_empty[buf]));
          // max commutes with the positive scale: max_r fl(a_r t) == fl(max_r(a_r) t).
          // Four independent chains (max is exact, so the order is free).
          float a0 = -INFINITY, a1 = -INFINITY, a2 = -INFINITY, a3 = -INFINITY;
          if (rows == kBlock) {
#pragma unroll
            for (int r = 0; r < 128; r += 4) {
              a0 = fmaxf(a0, __uint_as_float(v[r]));
              a1 = fmaxf(a1, __uint_as_float(v[r + 1]));
              a2 = fmaxf(a2, __uint_as_float(v[r + 2]));
              a3 = fmaxf(a3, __uint_as_float(v[r + 3]));
            }
          } else {
#pragma unroll
            for (int r = 0; r < 128; r += 4) {
              a0 = fmaxf(a0, r < rows ? __uint_as_float(v[r]) : -INFINITY);
              a1 = fmaxf(a1, r + 1 < rows ? __uint_as_float(v[r + 1]) : -INFINITY);
              a2 = fmaxf(a2, r + 2 < rows ? __uint_as_float(v[r + 2]) : -INFINITY);
              a3 = fmaxf(a3, r + 3 < rows ? __uint_as_float(v[r + 3]) : -INFINITY);
            }
          }
          m = __fmul_rn(fmaxf(fmaxf(a0, a1), fmaxf(a2, a3)), D.to_bits);
          const float nm = -m;
          // S = sum_r exp2(x_r - m) over the tile's real rows (discovery.hpp:101-107) in four
          // interleaved partial sums (the exp2 is ex2.approx, so the reference's sequential
          // rounding is not reproduced bit-for-bit anyway; scores stay within 1e-6 relative)
          float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
          if (rows == kBlock) {
#pragma unroll
            for (int r = 0; r < 128; r += 4) {
              s0 += ex2_approx(fmaf(__uint_as_float(v[r]), D.to_bits, nm));
              s1 += ex2_approx(fmaf(__uint_as_float(v[r + 1]), D.to_bits, nm));
              s2 += ex2_approx(fmaf(__uint_as_float(v[r + 2]), D.to_bits, nm));
              s3 += ex2_approx(fmaf(__uint_as_float(v[r + 3]), D.to_bits, nm));
            }
          } else {
#pragma unroll
            for (int r = 0; r < 128; r += 4) {
              s0 += r < rows ? ex2_approx(fmaf(__uint_as_float(v[r]), D.to_bits, nm)) : 0.f;
              s1 += r + 1 < rows ? ex2_approx(fmaf(__uint_as_float(v[r + 1]), D.to_bits, nm)) : 0.f;
              s2 += r + 2 < rows ? ex2_approx(fmaf(__uint_as_float(v[r + 2]), D.to_bits, nm)) : 0.f;
              s3 += r + 3 < rows ? ex2_approx(fmaf(__uint_as_float(v[r + 3]), D.to_bits, nm)) : 0.f;
            }
          }
          S = (s0 + s1) + (s2 + s3);
        } else {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&s.d_empty[buf]));
        }
        if (J <= I) {
          if (prm.out.rows) {  // two-pass mode: coalesced (m, S) pairs, the select kernel does the rest
            prm.out.rows[((size_t)z * D.Hq + h) * ((size_t)D.M * (D.M + 1) / 2) +
                         (size_t)I * (I + 1) / 2 + J] = make_float2(m, S);
          } else {
            m_s[J] = m;
            S_s[J] = S;
            tmax = fmaxf(tmax, m);
          }
        }
        DT_ADD(2);  // epilogue: per-chunk max / exp2 / sums
      }
      if (prm.out.rows) continue;  // no per-item tail in two-pass mode
      DT_T0();

      // ---- outputs: energy / local_max rows (thread-owned J), then normalisation
      const size_t map_row = (((size_t)z * D.Hq + h) * D.M + I) * (size_t)N;
      if (prm.out.energy || prm.out.local_max) {
        // an M = 64 last chunk wrote its m / S entries through another thread-to-J mapping
        if (FPB_DISC_M64) named_bar_sync(ebar, kEpiThreads);
        for (int J = et; J < N; J += kEpiThreads) {
          if (prm.out.energy) prm.out.energy[map_row + J] = (J <= I) ? S_s[J] : 0.f;
          if (prm.out.local_max) prm.out.local_max[map_row + J] = (J <= I) ? m_s[J] : kNegSentinel;
        }
      }
      if (prm.out.normalize) {
        // round 1: M_I = max_J m (discovery.hpp:131-134)
        for (int o = 16; o > 0; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
        if (lane == 0) red[0][w4] = tmax;
        named_bar_sync(ebar, kEpiThreads);
        DT_ADD(3);  // epilogue: first barrier (warps of the item wait for its slowest warp)
        const float rmax = fmaxf(fmaxf(red[0][0], red[0][1]), fmaxf(red[0][2], red[0][3]));
        // S'_J = S_J exp2(m_J - M_I); total = sum S'; max S' (for the threshold) in one round
        float total = 0.f, pmax = 0.f;
        for (int J = et; J <= I; J += kEpiThreads) {
          const float r = __fmul_rn(S_s[J], ex2_approx(__fsub_rn(m_s[J], rmax)));
          S_s[J] = r;
          total += r;
          pmax = fmaxf(pmax, r);
        }
        for (int o = 16; o > 0; o >>= 1) {
          total += __shfl_xor_sync(0xffffffffu, total, o);
          pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
        }
        if (lane == 0) {
          red[1][w4] = total;
          red[2][w4] = pmax;
        }
        named_bar_sync(ebar, kEpiThreads);
        total = (red[1][0] + red[1][1]) + (red[1][2] + red[1][3]);
        pmax = fmaxf(fmaxf(red[2][0], red[2][1]), fmaxf(red[2][2], red[2][3]));
        const float inv = __fdiv_rn(1.0f, __fadd_rn(total, D.eps));  // discovery.hpp:141-142
        DT_ADD(16);  // epilogue: rescaled energies, second barrier
        if (prm.out.score)
          for (int J = et; J < N; J += kEpiThreads)
            prm.out.score[map_row + J] = (J <= I) ? __fmul_rn(S_s[J], inv) : 0.f;

        // ---- fused max-threshold + compaction (selection.hpp:63-92, 176-192)
        if (prm.out.idx || prm.out.mask || prm.out.counts) {
          // max_J fl(S'_J inv) == fl(max_J S'_J * inv): rounding is monotone for inv > 0;
          // max_val starts at 0 (selection.hpp:75), scores are >= 0.
          const float smax = __fmul_rn(pmax, inv);
          const float thresh = __fmul_rn(D.alpha, smax);
          const size_t plan_row = ((size_t)z * D.M + I) * (size_t)N;  // [z, I, :, :]
          // round 3: per-(chunk, warp) active counts -> exclusive prefix in (J) order
          auto active = [&](int J) {
            return J <= I && ((__fmul_rn(S_s[J], inv) >= thresh) || J < D.sink_blocks ||
                              (I - J) < D.window_blocks);
          };
          for (int c = 0; c < nchunks; ++c) {
            const int J = c * kBlock + et;
            const bool act = active(J);
            const unsigned bal = __ballot_sync(0xffffffffu, act);
            if (lane == 0) ired[c * 4 + w4] = __popc(bal);
            if (prm.out.mask && J < N) prm.out.mask[(plan_row + J) * D.Hq + h] = act ? 1 : 0;
          }
          named_bar_sync(ebar, kEpiThreads);
          DT_ADD(17);  // epilogue: threshold, ballots, third barrier
          int base = 0;
          for (int c = 0; c < nchunks; ++c) {
            const int J = c * kBlock + et;
            const bool act = active(J);
            const unsigned bal = __ballot_sync(0xffffffffu, act);
            int before = base;
#pragma unroll
            for (int w = 0; w < 4; ++w) before += (w < w4) ? ired[c * 4 + w] : 0;
            if (prm.out.idx && act)
              prm.out.idx[(plan_row + before + __popc(bal & ((1u << lane) - 1u))) * D.Hq + h] = J;
            base += (ired[c * 4 + 0] + ired[c * 4 + 1]) + (ired[c * 4 + 2] + ired[c * 4 + 3]);
          }
          DT_ADD(18);  // epilogue: compaction (active idx stores)
          if (prm.out.mask)
            for (int J = nchunks * kBlock + et; J < N; J += kEpiThreads)
              prm.out.mask[(plan_row + J) * D.Hq + h] = 0;
          if (prm.out.idx && !prm.prefilled)
            for (int slot_j = base + et; slot_j < N; slot_j += kEpiThreads)
              prm.out.idx[(plan_row + slot_j) * D.Hq + h] = N;
          if (prm.out.counts && et == 0)
            prm.out.counts[((size_t)z * D.M + I) * D.Hq + h] = base;
        }
      }
      // the next item's M = 64 last chunk writes m_s / S_s entries that other threads of this
      // warpgroup read in the tail above: nobody starts it before everyone is done (racecheck)
      if (FPB_DISC_M64) named_bar_sync(ebar, kEpiThreads);
      DT_ADD(4);  // epilogue: fill + counts
    }
  }
#ifdef FPB_TRACE
  if (threadIdx.x == kMmaWarp * 32) dt_acc[20] += (unsigned long long)(clock64() - t_begin);
#endif
  DT_FLUSH();
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

constexpr size_t kMaxSmem = 227 * 1024;

template <int NQ>
size_t disc_smem_bytes(int M, bool rows_in_smem) {
  return sizeof(DiscSmem<NQ>) + 1024 + (rows_in_smem ? 4 * sizeof(float) * (size_t)M : 0) +
         2 * 4 * sizeof(int) * (size_t)((M + kBlock - 1) / kBlock);
}

int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

template <int NQ>
cudaError_t launch_nq(const Dims& D, const CUtensorMap& tm_q, const CUtensorMap& tm_kb,
                      const DiscParams& prm, cudaStream_t s) {
  const size_t smem = disc_smem_bytes<NQ>(D.M, prm.mscratch == nullptr);
  cudaError_t e = cudaFuncSetAttribute(discover_kernel<NQ>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int sms = sm_count();
  // in-kernel pooling wants every SM streaming K, whether or not it gets discovery items
  const int grid = (prm.num_items < sms && !prm.kpool) ? prm.num_items : sms;
  discover_kernel<NQ><<<grid, kThreads, smem, s>>>(tm_q, tm_kb, prm);
  return cudaGetLastError();
}

}  // namespace

size_t discover_scratch_bytes(const Dims& D) {
  // FPB_DISC_FORCE_SCRATCH=1 takes the long-sequence path at any length (parity tests)
  const char* force = std::getenv("FPB_DISC_FORCE_SCRATCH");
  if (!(force && force[0] == '1') && disc_smem_bytes<1>(D.M, true) <= kMaxSmem &&
      disc_smem_bytes<2>(D.M, true) <= kMaxSmem)
    return 0;
  return (size_t)sm_count() * 2 * 2 * sizeof(float) * D.M;
}

size_t discover_pool_ctr_bytes(const Dims& D) {
  return sizeof(int) * (1 + (size_t)D.Z * D.Hkv * ((D.M + kBlock - 1) / kBlock));
}

cudaError_t launch_discover(const Dims& D, int q_splits, const __nv_bfloat16* q_planes,
                            __nv_bfloat16* kbar_split, const DiscoverOut& out, int* sched,
                            float* mscratch, cudaStream_t s, const __nv_bfloat16* kpool,
                            float* pooled, int* pool_ctr) {
  if (kpool && (q_splits != 1 || !pool_ctr)) return cudaErrorInvalidValue;
  if (discover_scratch_bytes(D) == 0) mscratch = nullptr;
  else if (!mscratch) return cudaErrorInvalidValue;
  CUtensorMap tm_q, tm_kb;
  if (!make_tmap_rows128(&tm_q, q_planes, D.L, (uint64_t)q_splits * D.Z * D.Hq) ||
      !make_tmap_rows128(&tm_kb, kbar_split, D.M, 2ull * D.Z * D.Hkv))
    return cudaErrorInvalidValue;
  cudaError_t e;
  if (kpool && pool_ctr == sched + 1) {  // counters right behind the work counter: one memset
    e = cudaMemsetAsync(sched, 0, sizeof(int) + discover_pool_ctr_bytes(D), s);
  } else {
    e = cudaMemsetAsync(sched, 0, sizeof(int), s);
    if (e == cudaSuccess && kpool) e = cudaMemsetAsync(pool_ctr, 0, discover_pool_ctr_bytes(D), s);
  }
  if (e != cudaSuccess) return e;
  // Long rows: the fill value N of the unused plan slots goes in first as coalesced 16-byte
  // stores (at 256K, one 4-byte store per slot at stride Hq from the epilogue costs as much as
  // the compaction itself); short rows keep the in-epilogue fill (a second launch costs more).
  const int prefilled = out.idx != nullptr && D.M >= 1024 && (D.M * D.Hq) % 4 == 0 &&
                        reinterpret_cast<uintptr_t>(out.idx) % 16 == 0;
  if (prefilled) {
    cudaError_t e = launch_fill_plan(D, out.idx, s);
    if (e != cudaSuccess) return e;
  }
  DiscParams prm{D,      out,        sched,  D.Z * D.Hq * D.Mr, prefilled, mscratch,
                 kpool,  kbar_split, pooled, pool_ctr};
  e = q_splits == 1 ? launch_nq<1>(D, tm_q, tm_kb, prm, s) : launch_nq<2>(D, tm_q, tm_kb, prm, s);
  if (e != cudaSuccess || !out.rows) return e;
  return launch_select_rows(D, out.rows, out.idx, out.counts, prefilled != 0, s);
}

}  // namespace fpb

#ifdef FPB_TRACE
extern "C" int fpb_dtrace_read(unsigned long long* host24, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(host24, fpb::g_dtrace, sizeof(unsigned long long) * 32);
  if (reset) {
    unsigned long long z[32] = {};
    cudaMemcpyToSymbol(fpb::g_dtrace, z, sizeof(z));
  }
  return (int)e;
}
#endif
