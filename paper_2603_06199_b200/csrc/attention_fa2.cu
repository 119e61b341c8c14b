// attention_fa2.cu — K4 block-sparse / K5 dense-causal FlashAttention prefill, bf16, persistent,
// one work item per CTA at a time, QK^T running two blocks ahead of the softmax.
//
// Same semantics as attention_fa.cu / attention.cu (block_sparse_attention, attention.hpp:38-132;
// dense_attention, :135-174): index-driven jumps over the compacted plan row, causal mask only on
// the diagonal block, listed j > i blocks attended in full, ragged last block, base-2 LSE,
// C = 0 -> NaN / -inf, GQA by h / (Hq / Hkv).
//
// Why this shape (profiles/r2_probe*.jsonl, Qwen3 32K).  In the two-slot kernel each slot's
// QK^T -> softmax -> PV chain is serial, and the hand-offs alone (mbarrier round trips through
// the tensor-core commit path, no math at all) cost ~1000 cycles per visit; two slots do not hide
// that: removing the MMAs makes the kernel 24% faster, removing MUFU 2%, halving the K/V bytes
// 7%.  Here every block has its own S buffer two blocks ahead and its own P buffer, so the
// softmax never waits for the tensor core in steady state and the tensor core never waits for a
// hand-off that is not already late:
//
//   TMEM (512 columns): O | S0 | S1 | P0 | P1.  QK^T(g) -> S[g&1] is issued as soon as the
//   softmax of block g-2 has loaded S[g&1] into registers (s_free); the softmax writes P(g) (bf16)
//   into P[g&1] once PV(g-2) has consumed it (pv_done[g&1]); PV(g) reads P[g&1] from TMEM.
//   SMEM: Q[2] (items alternate; after an item's last QK^T its Q tile is the staging buffer of its
//   bf16 O tile) + a 4-tile K/V ring, filled by TMA in the MMA consumption order, one global
//   stream over all items of the CTA.  The producer and the MMA issuer derive that order with the
//   same rule (`qk_next`): QK^T up to two blocks ahead of PV, except that the first QK^T of item t
//   waits until the last PV of item t-2 has been issued (its epilogue frees Q[t&1]).
//
// Warps (16): w0 K/V producer; w1 MMA issuer; w2 TMEM allocator, then Q producer; w3 scheduler
// (dynamic work counter, plan-row fetch + range check + compaction into a global list, up to
// kMeta items ahead); w4..w11 softmax: warp w serves TMEM lane quarter w % 4 (32 query rows) and
// column half (w - 4) / 4 of every S tile — each SM sub-partition runs two softmax warps on the
// same rows; w12..w15 epilogue: O / l, bf16 pack, TMA store, LSE, overlapping the next item.  The
// two column halves of a row exchange their block maxima through shared memory (one 64-thread
// named barrier per block) and so agree on the running max and on the lazy O rescale.
#include <cstdlib>

#include "fp_kernels.h"

namespace fpb {

using namespace ptx;

namespace {

constexpr int kThreads = 512;
constexpr int kTile = kBlock * kHeadDim * 2;  // 32 KiB bf16 tile
constexpr int kRing = 4;                      // K/V tile ring
constexpr int kMeta = 4;                      // scheduler -> roles item ring
constexpr int kAhead = 2;                     // QK^T runs this many blocks ahead of PV
constexpr float kRescaleThreshold = 8.0f;     // lazy O rescale (log2 units)
constexpr uint32_t kColO = 0, kColS = 128, kColP = 384;  // TMEM column map
#ifndef FPB_SCHED_SLEEP
#define FPB_SCHED_SLEEP 256
#endif
#ifndef FA2_REG_CTRL
#define FA2_REG_CTRL 56
#endif
#ifndef FA2_REG_SOFTMAX
#define FA2_REG_SOFTMAX 160
#endif
#ifndef FA2_REG_EPI
#define FA2_REG_EPI 96
#endif

#ifdef FPB_TRACE
// cycle accounting (tools/trace_fa2.py): per-thread register accumulators, lane 0 flushes
__device__ unsigned long long g_trace2[24];
#define T2_DECL unsigned long long t2_acc[24] = {}; long long _t2 = 0
#define T2_T0() _t2 = clock64()
#define T2_ADD(i)                                \
  do {                                           \
    const long long _n = clock64();              \
    t2_acc[i] += (unsigned long long)(_n - _t2); \
    _t2 = _n;                                    \
  } while (0)
#define T2_FLUSH()                                                        \
  do {                                                                    \
    if (lane_id() == 0)                                                   \
      for (int _i = 0; _i < 24; ++_i)                                     \
        if (t2_acc[_i]) atomicAdd(&g_trace2[_i], t2_acc[_i]);             \
  } while (0)
#else
#define T2_DECL
#define T2_T0()
#define T2_ADD(i)
#define T2_FLUSH()
#endif

struct Fa2Params {
  Dims D;
  const int32_t* idx;  // nullptr -> dense causal
  const int32_t* counts;
  void* out;
  float* lse;
  unsigned long long* visits;
  int32_t* plan_error;
  int* sched;
  uint16_t* lists;  // global scratch: [grid][kMeta][M] compacted plan rows
  int num_items;
  int out_bf16;
  int gs;  // KV groups per super-group of the work order (divides Hkv)
};

struct ItemMeta {
  int item;  // -1: no more work
  int nblk;
};

struct Fa2Smem {
  uint8_t q[2][kTile];
  uint8_t ring[kRing][kTile];
  float xch[2][2][128];   // [block & 1][column half][row] row maxima of the two column halves
  float stat[2][3][128];  // [item & 1][m, l of half 0, l of half 1][row] for the epilogue
  uint64_t q_full[2], q_empty[2];
  uint64_t kv_full[kRing], kv_empty[kRing];
  uint64_t s_full[2], s_free[2], p_half[2][2], pv_done[2], max_ready[4][2];
  uint64_t o_full, o_empty, st_full[2], st_empty[2];
  uint64_t meta_full[kMeta], meta_empty[kMeta];
  ItemMeta meta[kMeta];
  uint32_t tmem_base;
};

// Work-item order: (z, KV super-group, query block heavy-first, head within the super-group),
// as in attention_fa.cu: a KV group's Q heads are adjacent, so their K/V tiles are re-read from L2.
__device__ __forceinline__ void decode(const Dims& D, int gs, int item, int& z, int& h, int& qi) {
  const int hs = gs * D.group;
  const int hh = item % hs;
  int t = item / hs;
  qi = owned_row(D, t % D.Mr);
  t /= D.Mr;
  const int nsg = D.Hkv / gs;
  h = (t % nsg) * hs + hh;
  z = t / nsg;
}

// The block stream as seen by the K/V producer and the MMA issuer: a QK cursor and a PV cursor
// over the same items, with the item boundaries (first block index of every item in flight).
struct Stream {
  int gq = 0, gp = 0;          // global block index of the next QK^T / PV
  int tq = 0, tp = 0;          // item of the next QK^T / PV
  int jq = 0, jp = 0;          // block within that item
  bool q_live = true;          // the QK cursor has not reached the sentinel
  int nblk[kMeta] = {};        // blocks of the items in flight (by meta slot)
  int first[kMeta] = {};       // global index of their first block
  // the next operation is a QK^T: it is at most kAhead blocks ahead of PV, and the first QK^T of
  // item t comes after the last PV of item t-2 (whose epilogue stages O through Q[t & 1])
  __device__ __forceinline__ bool qk_next() const {
    if (!q_live || gq > gp + kAhead) return false;
    if (jq == 0 && tq >= 2) {
      const int last_prev2 = first[(tq - 1) % kMeta] - 1;  // last block of item tq - 2
      if (gp <= last_prev2) return false;
    }
    return true;
  }
};

__global__ void __launch_bounds__(kThreads, 1)
    fa2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
               const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
               const Fa2Params prm) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  auto& s = *reinterpret_cast<Fa2Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                        ~uintptr_t(1023));
  const Dims& D = prm.D;
  const int N = D.M;
  uint16_t* lists = prm.lists + (size_t)blockIdx.x * kMeta * D.M;
  auto list_of = [&](int t) { return lists + (size_t)(t % kMeta) * D.M; };
  const bool dense = prm.idx == nullptr;
  const uint32_t warp = warp_id(), lane = lane_id();
  T2_DECL;
#ifdef FPB_TRACE
  const long long t_begin = clock64();
#endif

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_o);
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&s.q_full[i]), 1);
      mbar_init(smem_u32(&s.q_empty[i]), 1);
      mbar_init(smem_u32(&s.s_full[i]), 1);
      mbar_init(smem_u32(&s.s_free[i]), 8);
      mbar_init(smem_u32(&s.p_half[i][0]), 4);
      mbar_init(smem_u32(&s.p_half[i][1]), 4);
      mbar_init(smem_u32(&s.pv_done[i]), 1);
      mbar_init(smem_u32(&s.st_full[i]), 8);
      mbar_init(smem_u32(&s.st_empty[i]), 4);
      for (int qq = 0; qq < 4; ++qq) mbar_init(smem_u32(&s.max_ready[qq][i]), 2);
    }
    mbar_init(smem_u32(&s.o_full), 1);
    mbar_init(smem_u32(&s.o_empty), 4);
    for (int i = 0; i < kRing; ++i) {
      mbar_init(smem_u32(&s.kv_full[i]), 1);
      mbar_init(smem_u32(&s.kv_empty[i]), 1);
    }
    for (int i = 0; i < kMeta; ++i) {
      mbar_init(smem_u32(&s.meta_full[i]), 1);
      // K/V producer + issuer + Q producer + 8 softmax warps + 4 epilogue warps
      mbar_init(smem_u32(&s.meta_empty[i]), 15);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(smem_u32(&s.tmem_base));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;

  auto meta_wait = [&](int t) {
    mbar_wait(smem_u32(&s.meta_full[t % kMeta]), (t / kMeta) & 1);
    return s.meta[t % kMeta];
  };
  auto meta_release = [&](int t) {  // one arrive per warp (lane 0), after the warp is done with t
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&s.meta_empty[t % kMeta]));
  };
  // Stream bookkeeping shared by the K/V producer and the MMA issuer: entering item t with the QK
  // cursor reads its meta; the PV cursor leaving item t releases it.
  auto q_enter = [&](Stream& st) {
    const ItemMeta m = meta_wait(st.tq);
    st.q_live = m.item >= 0;
    st.jq = 0;
    if (st.q_live) {
      st.nblk[st.tq % kMeta] = m.nblk;
      st.first[st.tq % kMeta] = st.gq;
    }
  };
  auto q_advance = [&](Stream& st) {
    ++st.gq;
    if (++st.jq == st.nblk[st.tq % kMeta]) {
      ++st.tq;
      q_enter(st);
    }
  };
  auto p_advance = [&](Stream& st) {  // returns false once the PV cursor passed the last item
    ++st.gp;
    if (++st.jp == st.nblk[st.tp % kMeta]) {
      meta_release(st.tp);
      ++st.tp;
      st.jp = 0;
      if (st.tp == st.tq && !st.q_live) return false;
    }
    return true;
  };

  // 512 threads x 128 registers at launch: the control and epilogue warpgroups hand registers to
  // the two softmax warpgroups (128 x 56 + 128 x 96 + 256 x 160 = 60416 <= 65536).  setmaxnreg is
  // warpgroup-aligned: one instruction per warpgroup, before its roles branch.
  if (warp < 4) {
    setmaxnreg_dec<FA2_REG_CTRL>();
    if (warp == 3) {
      // ===================== scheduler: fetch items, compact plan rows, publish metas
      for (int t = 0;; ++t) {
        const int slot = t % kMeta;
        if (t >= kMeta) {
          const uint32_t bar = smem_u32(&s.meta_empty[slot]);
          const uint32_t par = ((t / kMeta) - 1) & 1;
          while (!mbar_try_wait(bar, par)) {
#if FPB_SCHED_SLEEP > 0
            __nanosleep(FPB_SCHED_SLEEP);  // running kMeta items ahead: yield the issue slots
#endif
          }
        }
        int item, nblk;
        for (;;) {  // skip (and write) empty plan rows: they never become work items
          item = 0;
          if (lane == 0) item = atomicAdd(prm.sched, 1);
          item = __shfl_sync(0xffffffffu, item, 0);
          if (item >= prm.num_items) item = -1;
          nblk = 0;
          if (item < 0) break;
          int z, h, qi;
          decode(D, prm.gs, item, z, h, qi);
          if (dense) {
            nblk = qi + 1;
            break;
          }
          int C = prm.counts[((size_t)z * D.M + qi) * D.Hq + h];
          if (C > N) {  // a row has N slots: more is a malformed plan, never read past it
            if (lane == 0 && prm.plan_error) atomicExch(prm.plan_error, 1);
            C = N;
          }
          const size_t prow = ((size_t)z * D.M + qi) * (size_t)N;
          uint16_t* lst = list_of(t);
          for (int s0 = 0; s0 < C; s0 += 32) {  // attention.hpp:76-81: range-check each slot
            const int slot_i = s0 + lane;
            int bid = -1;
            if (slot_i < C) bid = prm.idx[(prow + slot_i) * D.Hq + h];
            const bool ok = slot_i < C && bid >= 0 && bid < N;
            if (slot_i < C && !ok && prm.plan_error) atomicExch(prm.plan_error, 1);
            const unsigned bal = __ballot_sync(0xffffffffu, ok);
            if (ok) lst[nblk + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)bid;
            nblk += __popc(bal);
          }
          if (lane == 0 && prm.visits && nblk) atomicAdd(prm.visits, (unsigned long long)nblk);
          if (nblk > 0) break;
          // C = 0 (or only out-of-range slots): out = 0 * (1/0) = NaN, lse = -inf
          // (attention.hpp:121-125), written here
          const int rows = block_len(D, qi);
          const size_t orow0 = ((size_t)z * D.Hq + h) * (size_t)D.L + (size_t)qi * kBlock;
          const float nan = __int_as_float(0x7fc00000);
          const int vec_per_row = prm.out_bf16 ? kHeadDim / 8 : kHeadDim / 4;
          for (int e = lane; e < rows * vec_per_row; e += 32) {
            const size_t row = orow0 + e / vec_per_row;
            const int v4 = e % vec_per_row;
            if (prm.out_bf16) {
              const uint32_t pn = pack_bf16x2(nan, nan);
              reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(prm.out) +
                                       row * kHeadDim)[v4] = make_uint4(pn, pn, pn, pn);
            } else {
              reinterpret_cast<float4*>(reinterpret_cast<float*>(prm.out) + row * kHeadDim)[v4] =
                  make_float4(nan, nan, nan, nan);
            }
          }
          for (int r = lane; r < rows; r += 32) prm.lse[orow0 + r] = -INFINITY;
          __syncwarp();
        }
        __syncwarp();
        if (lane == 0) {
          s.meta[slot].item = item;
          s.meta[slot].nblk = nblk;
          mbar_arrive(smem_u32(&s.meta_full[slot]));
        }
        __syncwarp();
        if (item < 0) break;
      }
    } else if (warp == 2) {
      // ===================== Q producer: one tile per item into Q[t & 1] once its previous
      // occupant's epilogue has TMA-stored the O tile staged there
      const uint64_t pol_q = policy_evict_first();
      for (int t = 0;; ++t) {
        const ItemMeta m = meta_wait(t);
        if (m.item < 0) break;
        int z, h, qi;
        decode(D, prm.gs, m.item, z, h, qi);
        const int qb = t & 1;
        if (t >= 2) mbar_wait(smem_u32(&s.q_empty[qb]), ((t >> 1) - 1) & 1);
        if (lane == 0) {
          const uint32_t bar = smem_u32(&s.q_full[qb]);
          mbar_arrive_expect_tx(bar, kTile);
          tma_load_4d_hint(smem_u32(s.q[qb]), &tm_q, bar, 0, qi * kBlock, 0, z * D.Hq + h, pol_q);
        }
        meta_release(t);
      }
    } else if (warp == 0) {
      // ===================== K/V producer: tiles in the MMA consumption order
      const uint64_t pol_kv = policy_evict_last();
      int kvc = 0;
      int zkv[kMeta];
      auto push = [&](const CUtensorMap* map, int t, int j) {
        const int r = kvc % kRing;
        T2_T0();
        if (kvc >= kRing) mbar_wait(smem_u32(&s.kv_empty[r]), ((kvc / kRing) - 1) & 1);
        T2_ADD(14);  // producer: ring slot busy
        if (lane == 0) {
          const int b = dense ? j : (int)list_of(t)[j];
          const uint32_t fb = smem_u32(&s.kv_full[r]);
          mbar_arrive_expect_tx(fb, kTile);
          tma_load_4d_hint(smem_u32(s.ring[r]), map, fb, 0, b * kBlock, 0, zkv[t % kMeta],
                           pol_kv);
        }
        __syncwarp();
        ++kvc;
      };
      Stream st;
      q_enter(st);
      bool more = st.q_live;
      while (more) {
        if (st.qk_next()) {
          if (st.jq == 0) {  // the QK cursor enters item tq: its K/V plane
            int z, h, qi;
            decode(D, prm.gs, s.meta[st.tq % kMeta].item, z, h, qi);
            zkv[st.tq % kMeta] = z * D.Hkv + h / D.group;
          }
          push(&tm_k, st.tq, st.jq);
          q_advance(st);
        } else {
          push(&tm_v, st.tp, st.jp);
          more = p_advance(st);
        }
      }
    } else {
      // ===================== MMA issuer (warp 1): the same stream, same order
      const bool leader = elect_one();
      constexpr uint32_t idesc_qk = idesc_bf16_f32(128, 128, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(128, 128, false, true);
      int kvc = 0;
      Stream st;
      q_enter(st);
      bool more = st.q_live;
      while (more) {
        const int r = kvc % kRing;
        if (st.qk_next()) {
          // QK(gq): S[gq & 1] = Q[tq & 1] K^T, once softmax(gq - 2) has S[gq & 1] in registers
          const int g = st.gq, qb = st.tq & 1;
          T2_T0();
          if (st.jq == 0) mbar_wait(smem_u32(&s.q_full[qb]), (st.tq >> 1) & 1);
          T2_ADD(7);  // MMA: waiting for Q (per item)
          if (g >= 2) mbar_wait(smem_u32(&s.s_free[g & 1]), ((g >> 1) - 1) & 1);
          T2_ADD(8);  // MMA: waiting for a free S buffer
          mbar_wait(smem_u32(&s.kv_full[r]), (kvc / kRing) & 1);
          T2_ADD(9);  // MMA: waiting for K
          tc_fence_after();
          if (leader) {
            const uint32_t s_tmem = tmem + kColS + (g & 1) * 128;
            const uint64_t qdesc = sdesc_sw128(smem_u32(s.q[qb]), 16, 1024);
            const uint64_t kdesc = sdesc_sw128(smem_u32(s.ring[r]), 16, 1024);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
              const uint64_t off = ((ks >> 2) * (kTile / 2) + (ks & 3) * 32) >> 4;
              mma_bf16_ss(s_tmem, qdesc + off, kdesc + off, idesc_qk, ks > 0 ? 1u : 0u);
            }
            mma_commit(smem_u32(&s.kv_empty[r]));
            mma_commit(smem_u32(&s.s_full[g & 1]));
          }
          __syncwarp();
          q_advance(st);
        } else {
          // PV(gp): O (+)= P[gp & 1] [TMEM] x V [ring, MN-major]
          const int g = st.gp;
          const bool first = st.jp == 0, last = st.jp + 1 == st.nblk[st.tp % kMeta];
          T2_T0();
          if (first && st.tp >= 1) mbar_wait(smem_u32(&s.o_empty), (st.tp - 1) & 1);
          T2_ADD(10);  // MMA: waiting for the O accumulator (per item)
          mbar_wait(smem_u32(&s.kv_full[r]), (kvc / kRing) & 1);
          T2_ADD(11);  // MMA: waiting for V
          const uint64_t vdesc = sdesc_sw128(smem_u32(s.ring[r]), kTile / 2, 1024);
          const uint32_t p_tmem = tmem + kColP + (g & 1) * 64;
          for (int half = 0; half < 2; ++half) {
            mbar_wait(smem_u32(&s.p_half[g & 1][half]), (g >> 1) & 1);
            T2_ADD(12 + half);  // MMA: waiting for P half
            tc_fence_after();
            if (leader) {
#pragma unroll
              for (int k4 = 0; k4 < 4; ++k4) {
                const int ks = half * 4 + k4;
                mma_bf16_ts(tmem + kColO, p_tmem + ks * 8, vdesc + (uint64_t)(ks * 2048 >> 4),
                            idesc_pv, (!first || ks > 0) ? 1u : 0u);
              }
            }
            __syncwarp();
          }
          if (leader) {
            mma_commit(smem_u32(&s.kv_empty[r]));
            mma_commit(smem_u32(&s.pv_done[g & 1]));
            if (last) mma_commit(smem_u32(&s.o_full));
          }
          __syncwarp();
          more = p_advance(st);
        }
        ++kvc;
      }
    }
  } else if (warp < 12) {
    setmaxnreg_inc<FA2_REG_SOFTMAX>();
    // ===================== softmax: lane quarter q (rows 32q..32q+31), column half hf
    const int q = warp & 3, hf = (warp - 4) >> 2;
    const int r = q * 32 + lane;  // query row == TMEM lane
    const uint32_t lane_addr = static_cast<uint32_t>(q * 32) << 16;
    const float sc = D.to_bits;
    int g = 0;
    for (int t = 0;; ++t) {
      const ItemMeta mt = meta_wait(t);
      if (mt.item < 0) break;
      const uint16_t* lst = list_of(t);
      int z, h, qi;
      decode(D, prm.gs, mt.item, z, h, qi);
      float m_used = -INFINITY, l = 0.f;
      for (int n = 0; n < mt.nblk; ++n, ++g) {
        const int kv = dense ? n : (int)lst[n];
        const int cols = block_len(D, kv);
        const int lim = (kv == qi) ? min(cols, r + 1) : cols;  // attention.hpp:85-91
        const bool full = __all_sync(0xffffffffu, lim == kBlock);
        T2_T0();
        mbar_wait(smem_u32(&s.s_full[g & 1]), (g >> 1) & 1);
        T2_ADD(0);  // softmax: waiting for S
        tc_fence_after();
        const uint32_t s_addr = tmem + lane_addr + kColS + (g & 1) * 128 + hf * 64;
        uint32_t v[64];
        auto load_s = [&]() {  // this half's 64 logits; columns >= lim do not exist
          tmem_ld64(s_addr, v);
          tmem_ld_wait();
          if (!full) {  // causal diagonal / ragged tail (attention.hpp:85-91)
#pragma unroll
            for (int c = 0; c < 64; ++c)
              if (hf * 64 + c >= lim) v[c] = __float_as_uint(-INFINITY);
          }
        };
        load_s();
        float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
        for (int c = 0; c < 64; c += 8) {
          mx0 = fmaxf(mx0, fmaxf(__uint_as_float(v[c + 0]), __uint_as_float(v[c + 1])));
          mx1 = fmaxf(mx1, fmaxf(__uint_as_float(v[c + 2]), __uint_as_float(v[c + 3])));
          mx2 = fmaxf(mx2, fmaxf(__uint_as_float(v[c + 4]), __uint_as_float(v[c + 5])));
          mx3 = fmaxf(mx3, fmaxf(__uint_as_float(v[c + 6]), __uint_as_float(v[c + 7])));
        }
        const float mloc = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * sc;
        // publish this half's block maxima to the partner warp (same rows, other columns)
        s.xch[g & 1][hf][r] = mloc;
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&s.max_ready[q][g & 1]));
        T2_ADD(1);  // softmax: S load + mask + max
        auto partner_max = [&]() {
          mbar_wait(smem_u32(&s.max_ready[q][g & 1]), (g >> 1) & 1);
          return s.xch[g & 1][hf ^ 1][r];
        };
        // P = exp2(S * to_bits - m) packed in place: v[c/2] <- bf16x2(p_c, p_c+1)
        float bs[8];
        auto exp_block = [&](float m) {
          const float neg_m = -m;
#pragma unroll
          for (int a = 0; a < 8; ++a) bs[a] = 0.f;
          if (full) {
#pragma unroll
            for (int c = 0; c < 64; c += 2) {
              float x0, x1;
              ffma2(x0, x1, __uint_as_float(v[c]), __uint_as_float(v[c + 1]), sc, sc, neg_m,
                    neg_m);
              const float p0 = ex2_approx(x0), p1 = ex2_approx(x1);
              const int a = ((c >> 1) & 3) * 2;
              fadd2(bs[a], bs[a + 1], bs[a], bs[a + 1], p0, p1);
              v[c >> 1] = pack_bf16x2(p0, p1);
            }
          } else {
#pragma unroll
            for (int c = 0; c < 64; c += 2) {
              const float p0 = ex2_approx(fmaf(__uint_as_float(v[c]), sc, neg_m));
              const float p1 = ex2_approx(fmaf(__uint_as_float(v[c + 1]), sc, neg_m));
              const int a = ((c >> 1) & 3) * 2;
              fadd2(bs[a], bs[a + 1], bs[a], bs[a + 1], p0, p1);
              v[c >> 1] = pack_bf16x2(p0, p1);
            }
          }
        };
        if (n == 0) {  // first block of the item: the row max needs both halves first
          m_used = fmaxf(mloc, partner_max());
          T2_ADD(2);
          exp_block(m_used);
          T2_ADD(3);
        } else {
          // speculate on the agreed running max (lazy rescale: exact while the new block max
          // stays within 2^8 of it), then check the partner's half; the warps of a pair only
          // meet here, so their exp2 phases need not line up on the shared MUFU
          exp_block(m_used);
          T2_ADD(3);  // softmax: exp2 + pack
          const float m_new = fmaxf(m_used, fmaxf(mloc, partner_max()));
          if (__any_sync(0xffffffffu, m_new > m_used + kRescaleThreshold)) {
            // rare: rescale this half's 64 O columns and l to the new max (both halves see the
            // same rows and make the same decision); O must hold PV(g - 1); redo P from S
            mbar_wait(smem_u32(&s.pv_done[(g - 1) & 1]), ((g - 1) >> 1) & 1);
            tc_fence_after();
            const float f = ex2_approx(m_used - m_new);
            const uint32_t o_addr = tmem + lane_addr + kColO + hf * 64;
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
              uint32_t o[32];
              tmem_ld32(o_addr + cc * 32, o);
              tmem_ld_wait();
#pragma unroll
              for (int k = 0; k < 32; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * f);
              tmem_st32(o_addr + cc * 32, o);
            }
            l *= f;
            m_used = m_new;
            load_s();
            exp_block(m_used);
          }
          T2_ADD(2);  // softmax: max agreement (+ rare rescale and redo)
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&s.s_free[g & 1]));  // S[g & 1] may take QK(g + 2)
        // P[g & 1] is free once PV(g - 2) has read it
        if (g >= 2) mbar_wait(smem_u32(&s.pv_done[g & 1]), ((g >> 1) - 1) & 1);
        T2_ADD(4);  // softmax: waiting for the P buffer
        tc_fence_after();
        tmem_st32(tmem + lane_addr + kColP + (g & 1) * 64 + hf * 32,
                  *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&s.p_half[g & 1][hf]));
        T2_ADD(5);  // softmax: P store + arrive
        l += ((bs[0] + bs[1]) + (bs[2] + bs[3])) + ((bs[4] + bs[5]) + (bs[6] + bs[7]));
      }
      // row statistics of this item for the epilogue warps: m (half 0) and l of each half
      if (t >= 2) mbar_wait(smem_u32(&s.st_empty[t & 1]), ((t >> 1) - 1) & 1);  // epilogue t-2
      if (hf == 0) s.stat[t & 1][0][r] = m_used;
      s.stat[t & 1][1 + hf][r] = l;
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&s.st_full[t & 1]));
      meta_release(t);
    }
  } else {
    setmaxnreg_dec<FA2_REG_EPI>();
    // ===================== epilogue (attention.hpp:119-126): O / l, LSE, store
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t lane_addr = static_cast<uint32_t>(q * 32) << 16;
    for (int t = 0;; ++t) {
      const ItemMeta mt = meta_wait(t);
      if (mt.item < 0) break;
      int z, h, qi;
      decode(D, prm.gs, mt.item, z, h, qi);
      const int rows = block_len(D, qi);
      const int qb = t & 1;
      T2_T0();
      mbar_wait(smem_u32(&s.st_full[qb]), (t >> 1) & 1);
      T2_ADD(15);  // epilogue: waiting for the row statistics
      const float m = s.stat[qb][0][r];
      const float l = s.stat[qb][1][r] + s.stat[qb][2][r];
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&s.st_empty[qb]));
      const float inv = 1.0f / l;
      mbar_wait(smem_u32(&s.o_full), t & 1);  // last PV of item t done => its QK^Ts too
      T2_ADD(16);  // epilogue: waiting for O
      tc_fence_after();
      const size_t orow = ((size_t)z * D.Hq + h) * (size_t)D.L + (size_t)qi * kBlock + r;
      const uint32_t stage = smem_u32(s.q[qb]);  // this item's Q tile is free: O staging
      const uint32_t o_addr = tmem + lane_addr + kColO;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t o[32];
        tmem_ld32(o_addr + cc * 32, o);
        tmem_ld_wait();
        if (cc == 3) {  // O fully read: the next item's first PV may overwrite it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&s.o_empty));
        }
        if (prm.out_bf16) {
          // row r, columns 32cc..32cc+31 -> SW128 tile layout of the TMA box (64 cols x 128 rows)
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const int col = cc * 32 + q4 * 8;
            const uint32_t off = (col >> 6) * (kTile / 2) + r * 128 +
                                 ((((col & 63) >> 3) ^ (r & 7)) << 4);
            const uint4 val = make_uint4(
                pack_bf16x2(__uint_as_float(o[8 * q4 + 0]) * inv, __uint_as_float(o[8 * q4 + 1]) * inv),
                pack_bf16x2(__uint_as_float(o[8 * q4 + 2]) * inv, __uint_as_float(o[8 * q4 + 3]) * inv),
                pack_bf16x2(__uint_as_float(o[8 * q4 + 4]) * inv, __uint_as_float(o[8 * q4 + 5]) * inv),
                pack_bf16x2(__uint_as_float(o[8 * q4 + 6]) * inv, __uint_as_float(o[8 * q4 + 7]) * inv));
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(stage + off),
                         "r"(val.x), "r"(val.y), "r"(val.z), "r"(val.w)
                         : "memory");
          }
        } else if (r < rows) {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(prm.out) +
                                                  orow * kHeadDim + cc * 32);
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4)
            dst[q4] = make_float4(__uint_as_float(o[4 * q4]) * inv,
                                  __uint_as_float(o[4 * q4 + 1]) * inv,
                                  __uint_as_float(o[4 * q4 + 2]) * inv,
                                  __uint_as_float(o[4 * q4 + 3]) * inv);
        }
      }
      if (r < rows) prm.lse[orow] = m + log2f(l);
      T2_ADD(17);  // epilogue: O load + normalise + stage
      if (prm.out_bf16) {
        fence_proxy_async_smem();
        named_bar_sync(5, 128);
        if (r == 0) {  // rows beyond L are clipped by the tensor map
          tma_store_3d(&tm_o, stage, 0, qi * kBlock, z * D.Hq + h);
          tma_store_3d(&tm_o, stage + kTile / 2, 64, qi * kBlock, z * D.Hq + h);
          bulk_commit();
          bulk_wait_read0();
          mbar_arrive(smem_u32(&s.q_empty[qb]));
        }
      } else if (r == 0) {
        mbar_arrive(smem_u32(&s.q_empty[qb]));
      }
      T2_ADD(18);  // epilogue: TMA store
      meta_release(t);
    }
    if (prm.out_bf16 && r == 0) bulk_wait0();
  }
#ifdef FPB_TRACE
  if (threadIdx.x == 32) t2_acc[19] += (unsigned long long)(clock64() - t_begin);
#endif
  T2_FLUSH();
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

}  // namespace

cudaError_t launch_attention_fa2(const Dims& D, const __nv_bfloat16* Q, const __nv_bfloat16* K,
                                 const __nv_bfloat16* V, const int32_t* idx, const int32_t* counts,
                                 bool out_bf16, void* out, float* lse, unsigned long long* visits,
                                 int32_t* plan_error, int* sched, uint16_t* lists, cudaStream_t s) {
  CUtensorMap tm_q, tm_k, tm_v, tm_o;
  if (!make_tmap_tiles128(&tm_q, Q, D.L, (uint64_t)D.Z * D.Hq) ||
      !make_tmap_tiles128(&tm_k, K, D.L, (uint64_t)D.Z * D.Hkv) ||
      !make_tmap_tiles128(&tm_v, V, D.L, (uint64_t)D.Z * D.Hkv) ||
      !make_tmap_rows128(&tm_o, out_bf16 ? out : Q, D.L, (uint64_t)D.Z * D.Hq))
    return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(sched, 0, sizeof(int), s);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int num_items = D.Z * D.Hq * D.Mr;
  const int grid = num_items < sms ? num_items : sms;
  // K/V bytes of one KV group = 2 tensors x L x d x 2 B; keep gs groups' worth <= 64 MiB
  static const int gs_env = [] {
    const char* e = std::getenv("FPB_FA_GS");
    return e ? std::atoi(e) : 0;
  }();
  int gs = gs_env;
  if (gs <= 0) {
    const double group_bytes = 2.0 * D.L * D.d * 2.0;
    gs = (int)((64.0 * 1024 * 1024) / group_bytes);
  }
  gs = gs < 1 ? 1 : (gs > D.Hkv ? D.Hkv : gs);
  while (D.Hkv % gs) --gs;
  Fa2Params prm{D, idx, counts, out, lse, visits, plan_error, sched, lists, num_items,
                out_bf16 ? 1 : 0, gs};
  const size_t smem = sizeof(Fa2Smem) + 1024;
  e = cudaFuncSetAttribute(fa2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  fa2_kernel<<<grid, kThreads, smem, s>>>(tm_q, tm_k, tm_v, tm_o, prm);
  return cudaGetLastError();
}

}  // namespace fpb

#ifdef FPB_TRACE
extern "C" int fpb_trace2_read(unsigned long long* host24, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(host24, fpb::g_trace2, sizeof(unsigned long long) * 24);
  if (reset) {
    unsigned long long z[24] = {};
    cudaMemcpyToSymbol(fpb::g_trace2, z, sizeof(z));
  }
  return (int)e;
}
#endif
