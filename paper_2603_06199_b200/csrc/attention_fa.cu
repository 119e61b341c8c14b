// attention_fa.cu — K4 block-sparse / K5 dense-causal FlashAttention prefill, bf16, persistent.
//
// Same semantics as attention.cu (block_sparse_attention, attention.hpp:38-132; dense_attention,
// :135-174): index-driven jumps over the compacted plan row, causal mask only on the diagonal
// block, listed j > i blocks attended in full, ragged last block, base-2 LSE, C = 0 -> NaN/-inf,
// GQA by h / (Hq / Hkv).
//
// Persistent CTA per SM, FA4-style two-slot ping-pong: each CTA runs two independent work items
// (z, h, query block i) at once, one per softmax warpgroup, so one slot's softmax (MUFU-bound)
// overlaps the other slot's tensor-core work.
//   TMEM (512 cols): S0 | S1 | O0 | O1; P (bf16) is written back over S and read by the PV MMA
//   straight from TMEM (ts form).  Issue order per slot unit: PV(j-1) then QK(j) — in-order
//   tcgen05 execution makes the S/P aliasing safe.
//   SMEM: Q0, Q1 (32 KiB each) + a 5-tile K/V ring shared by both slots, filled by TMA (one 4-D
//   box per 128 x 128 tile: both 64-column SW128 halves in one instruction) in exactly
//   the MMA consumption order (both warps run the same deterministic unit schedule).  At the end
//   of an item the slot's Q tile is the staging buffer of the O tile, written by one TMA store.
//   Compacted plan rows live in a global scratch (L2-resident), not in SMEM.
//
// Warps: w0 TMA producer; w1 MMA issuer; w2 TMEM allocator; w3 scheduler (dynamic work counter,
// plan-row fetch + range check + compaction, two items ahead per slot); w4..w7 softmax/epilogue
// slot 0; w8..w11 softmax/epilogue slot 1.  PV(j) is issued in two K-halves, each released as
// soon as that half of P is in TMEM.
#include <cstdlib>

#include "fp_kernels.h"

namespace fpb {

using namespace ptx;

namespace {

constexpr int kThreads = 384;
constexpr int kTile = kBlock * kHeadDim * 2;  // 32 KiB bf16 tile
constexpr int kRing = 5;                      // shared K/V tile ring
#ifndef FPB_SCHED_SLEEP
#define FPB_SCHED_SLEEP 256  // ns; measured: 128K -5.7%, 32K / 256K neutral (r1_ab_fa_sched_sleep)
#endif
constexpr float kRescaleThreshold = 8.0f;     // lazy O rescale (log2 units)
// P is handed to the PV MMA in kPParts column parts (keys 128 / kPParts each), one mbarrier each
#ifndef FPB_FA_TMEM0
#define FPB_FA_TMEM0 1  // measured: 32K -0.6%, 128K -2.5% (profiles/r2_ab_tmem0.jsonl)
#endif
#ifndef FPB_FA_PPARTS
#define FPB_FA_PPARTS 2
#endif
constexpr int kPParts = FPB_FA_PPARTS;
static_assert(kPParts == 1 || kPParts == 2 || kPParts == 4, "P parts");
constexpr int kPartFloats = kBlock * kHeadDim + 2 * kBlock;  // one row's partial: O, m, l
constexpr double kPhaseBytes = 64.0 * 1024 * 1024;  // K/V bytes of one KV-range phase (L2 budget)
// Timing probes (wrong numerics; tools/ab_probe.sh): 1 = softmax without max/exp2 (P = raw S),
// 2 = exp2 replaced by one FMA (no MUFU), 3 = no MMA issued (barriers only), 4 = 1 + 3,
// 5 = K/V tiles loaded as one 64-column half (half the L2 -> SMEM bytes), 6 = 4 without the
// tcgen05.ld of S, 7 = 6 loading a quarter of S.
#ifndef FPB_FA_PROBE
#define FPB_FA_PROBE 0
#endif
#if FPB_FA_PROBE == 2
#define FA_EX2(x) fmaf((x), 0.001f, 1.0f)
#else
#define FA_EX2(x) ex2_approx(x)
#endif

struct FaParams {
  Dims D;
  const int32_t* idx;  // nullptr -> dense causal
  const int32_t* counts;
  void* out;
  float* lse;
  unsigned long long* visits;
  int32_t* plan_error;
  int* sched;
  uint16_t* lists;  // global scratch: [grid][2 slots][2 bufs][M] compacted plan rows
  int num_items;
  int out_bf16;
  int gs;     // KV groups per super-group of the work order (divides Hkv)
  // KV-range phases (fa_phases): one KV group's key blocks in `phases` ranges of `chunk` blocks,
  // one launch per range (`phase`); stream order makes range p-1 complete before range p starts
  int phases, chunk, phase;
  float* part;   // partial (O, m, l) of rows that continue in a later phase
  int* pflag;    // per (z, h, query block): 1 when the row's partial holds visited blocks
};

#ifdef FPB_TRACE
// cycle accounting (tools/trace_attention.py): per-warp register accumulators, flushed once
__device__ unsigned long long g_trace[16];
#define TR_DECL unsigned long long tr_acc[16] = {}
#define TR_T0() long long _tr = clock64()
#define TR_ADD(i)                                  \
  do {                                             \
    const long long _n = clock64();                \
    tr_acc[i] += (unsigned long long)(_n - _tr);   \
    _tr = _n;                                      \
  } while (0)
#define TR_FLUSH()                                                          \
  do {                                                                      \
    if (lane_id() == 0)                                                     \
      for (int _i = 0; _i < 16; ++_i)                                       \
        if (tr_acc[_i]) atomicAdd(&g_trace[_i], tr_acc[_i]);                \
  } while (0)
#else
#define TR_DECL
#define TR_T0()
#define TR_ADD(i)
#define TR_FLUSH()
#endif

struct SlotMeta {
  int item;  // -1: no more work
  int nblk;
  int zh, qi, zkv;  // (z * Hq + h), query block, K/V plane
  int jbase;        // first key block of the item's KV range (dense lists)
  int mode;         // kContinue: O/m/l start from the row's partial; kPartialOut: write one
};
constexpr int kContinue = 1, kPartialOut = 2;

struct FaSmem {
  uint8_t q[2][kTile];
  uint8_t ring[kRing][kTile];
  uint64_t q_full[2], q_empty[2];
  uint64_t kv_full[kRing], kv_empty[kRing];
  uint64_t s_full[2], p_part[2][kPParts], o_done[2], o_free[2];
  uint64_t meta_full[2][2], meta_empty[2][2];
  SlotMeta meta[2][2];
  uint32_t tmem_base;
};

// Work-item order: (z, KV super-group, query block heavy-first, head within the super-group).
// A super-group is `gs` adjacent KV groups.  The Q heads of one KV group are adjacent within a
// query block, so their K/V tiles are fetched once and re-read from L2; `gs` bounds the K/V
// working set of the ~296 concurrent items to gs groups (chosen on the host so that it stays
// well inside the 126 MB L2).  gs == Hkv is "all heads fastest" (best while everything fits).
__device__ __forceinline__ void decode(const Dims& D, int gs, int item, int& z, int& h, int& qi) {
  const int hs = gs * D.group;
  const int hh = item % hs;
  int t = item / hs;
  qi = owned_row(D, t % D.Mr);  // heavy (long rows) first
  t /= D.Mr;
  const int nsg = D.Hkv / gs;
  h = (t % nsg) * hs + hh;
  z = t / nsg;
}

// A KV-range phase launch holds the rows qi >= phase * chunk of every (z, KV group): per (z, KV
// group) heavy (long) rows first, the group's Q heads fastest.
__device__ __forceinline__ void decode_phased(const Dims& D, int phase, int chunk, int item,
                                              int& z, int& h, int& qi) {
  const int per_zg = (D.M - phase * chunk) * D.group;
  const int zg = item / per_zg, u = item % per_zg;
  z = zg / D.Hkv;
  h = (zg % D.Hkv) * D.group + u % D.group;
  qi = D.M - 1 - u / D.group;
}

// Per-slot progress shared by the producer's and the MMA issuer's identical unit schedules.
struct SlotState {
  int t = 0;      // items taken by this slot (incl. empty ones and the final sentinel)
  int j = 0;      // unit within the current item (0..nblk)
  int nblk = 0;
  int item = 0;
  int qc = 0;     // items with nblk > 0 (Q loads / O lifetimes)
  int zkv = 0;    // K/V plane of the current item (producer)
  int jbase = 0;  // first key block of the item's range (dense lists, producer)
  bool cont = false;  // the item's O starts from a partial (issuer: accumulate from PV(0))
  int bc = 0;     // blocks processed (P / S / O barrier phases)
  bool active = true;
};

__global__ void __launch_bounds__(kThreads, 1)
    fa_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
              const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
              const FaParams prm) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  auto& s = *reinterpret_cast<FaSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                       ~uintptr_t(1023));
  const Dims& D = prm.D;
  const int N = D.M;
  uint16_t* lists = prm.lists + (size_t)blockIdx.x * 4 * D.M;
  auto list_of = [&](int slot, int p) { return lists + (size_t)(slot * 2 + p) * D.M; };
  const bool dense = prm.idx == nullptr;
  const uint32_t warp = warp_id(), lane = lane_id();
  TR_DECL;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_o);
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&s.q_full[i]), 1);
      mbar_init(smem_u32(&s.q_empty[i]), 1);
      mbar_init(smem_u32(&s.s_full[i]), 1);
      for (int k = 0; k < kPParts; ++k) mbar_init(smem_u32(&s.p_part[i][k]), 4);
      mbar_init(smem_u32(&s.o_done[i]), 1);
      mbar_init(smem_u32(&s.o_free[i]), 4);
      for (int p = 0; p < 2; ++p) {
        mbar_init(smem_u32(&s.meta_full[i][p]), 1);
        mbar_init(smem_u32(&s.meta_empty[i][p]), 4);
      }
    }
    for (int i = 0; i < kRing; ++i) {
      mbar_init(smem_u32(&s.kv_full[i]), 1);
      mbar_init(smem_u32(&s.kv_empty[i]), 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(smem_u32(&s.tmem_base));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
#if FPB_FA_TMEM0
  // all 512 columns of the SM's TMEM are allocated, so the allocation starts at lane 0, column 0:
  // a compile-time base keeps the TMEM addresses out of the control warps' (spilled) registers
  constexpr uint32_t tmem = 0;
  if (threadIdx.x == 0 && s.tmem_base != 0u) __trap();
#else
  const uint32_t tmem = s.tmem_base;
#endif
  // 384 threads x 168 regs at launch; hand the control warpgroup's share to the softmax WGs
  // (128 x 72 + 256 x 216 = 64512 = the launch allocation: any more and setmaxnreg.inc blocks)
  if (warp < 4) {
  setmaxnreg_dec<72>();
  if (warp == 3) {
    // ===================== scheduler: fetch items, compact plan rows, publish per-slot metas
    // (runs up to two items ahead per slot so plan-row loads never stall the TMA producer)
    int t[2] = {0, 0};
    bool done[2] = {false, false};
    while (!done[0] || !done[1]) {
      for (int sl = 0; sl < 2; ++sl) {
        if (done[sl]) continue;
        const int p = t[sl] & 1;
        if (t[sl] >= 2) {
          const bool ready = mbar_try_wait(smem_u32(&s.meta_empty[sl][p]), ((t[sl] >> 1) - 1) & 1);
          if (!__shfl_sync(0xffffffffu, ready, 0)) {
#if FPB_SCHED_SLEEP > 0
            __nanosleep(FPB_SCHED_SLEEP);  // both slots run ahead: yield the issue slots
#endif
            continue;
          }
        }
        __syncwarp();
        int item = 0;
        if (lane == 0) item = atomicAdd(prm.sched, 1);
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item >= prm.num_items) item = -1;
        int nblk = 0;
        SlotMeta mt{item, 0, 0, 0, 0, 0, 0};
        if (item >= 0) {
          int z, h, qi;
          const int ph = prm.phase;
          if (prm.phases > 1)
            decode_phased(D, ph, prm.chunk, item, z, h, qi);
          else
            decode(D, prm.gs, item, z, h, qi);
          mt.zh = z * D.Hq + h;
          mt.qi = qi;
          mt.zkv = z * D.Hkv + h / D.group;
          // this item's KV range: [lo, hi); a row's last phase also takes every listed block
          // beyond its own range (listed j > i blocks, attended in full)
          const int last_ph = prm.phases > 1 ? min(qi / prm.chunk, prm.phases - 1) : 0;
          const int lo = ph * prm.chunk, hi = ph == last_ph ? N : lo + prm.chunk;
          mt.jbase = lo;
          if (ph < last_ph) mt.mode |= kPartialOut;
          bool valid = false;  // the earlier phases visited blocks: a partial (O, m, l) exists
          if (ph > 0) {
            valid = __ldcg(prm.pflag + (size_t)mt.zh * D.M + qi) != 0;
            if (valid) mt.mode |= kContinue;
          }
          if (dense) {
            nblk = max(0, min(qi + 1, hi) - lo);
          } else {
            int C = prm.counts[((size_t)z * D.M + qi) * D.Hq + h];
            if (C > N) {  // a row has N slots: more is a malformed plan, never read past it
              if (lane == 0 && prm.plan_error) atomicExch(prm.plan_error, 1);
              C = N;
            }
            const size_t prow = ((size_t)z * D.M + qi) * (size_t)N;
            uint16_t* lst = list_of(sl, p);
            for (int s0 = 0; s0 < C; s0 += 32) {  // attention.hpp:76-81: range-check each slot
              const int slot = s0 + lane;
              int bid = -1;
              if (slot < C) bid = prm.idx[(prow + slot) * D.Hq + h];
              const bool ok = slot < C && bid >= 0 && bid < N;
              if (slot < C && !ok && prm.plan_error) atomicExch(prm.plan_error, 1);
              const bool mine = ok && bid >= lo && bid < hi;
              const unsigned bal = __ballot_sync(0xffffffffu, mine);
              if (mine) lst[nblk + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)bid;
              nblk += __popc(bal);
            }
            if (lane == 0 && prm.visits && nblk) atomicAdd(prm.visits, (unsigned long long)nblk);
          }
          if (nblk == 0) {
            // Nothing to attend in this range.  An empty item never reaches the other roles
            // (its softmax warps would release the meta / list buffer before the producer and
            // the MMA issuer had read it): the scheduler settles it here.
            if (mt.mode & kPartialOut) {
              // the row goes on: its partial state (or its absence) passes along unchanged
            } else {
              // final: out = O / l and lse = m + log2 l from the partial, or, with no block
              // visited at all (C = 0), out = 0 * (1/0) = NaN, lse = -inf (attention.hpp:121-125)
              const int rows = block_len(D, qi);
              const size_t orow0 = (size_t)mt.zh * D.L + (size_t)qi * kBlock;
              const size_t ps = valid ? (size_t)mt.zh * (D.M - prm.chunk) + (qi - prm.chunk) : 0;
              const float* po = prm.part + ps * (kBlock * kHeadDim + 2 * kBlock);
              const float* pml = po + kBlock * kHeadDim;
              for (int e = lane; e < rows * kHeadDim; e += 32) {
                const int rr = e / kHeadDim;  // out = O * (1 / l), as in the epilogue
                const float val = valid ? __ldcg(po + e) * (1.0f / __ldcg(pml + kBlock + rr))
                                        : __int_as_float(0x7fc00000);
                if (prm.out_bf16)
                  reinterpret_cast<__nv_bfloat16*>(prm.out)[orow0 * kHeadDim + e] =
                      __float2bfloat16_rn(val);
                else
                  reinterpret_cast<float*>(prm.out)[orow0 * kHeadDim + e] = val;
              }
              for (int rr = lane; rr < rows; rr += 32)
                prm.lse[orow0 + rr] =
                    valid ? __ldcg(pml + rr) + log2f(__ldcg(pml + kBlock + rr)) : -INFINITY;
            }
            __syncwarp();
            continue;  // fetch another item for this slot; nothing is published
          }
        }
        mt.nblk = nblk;
        __syncwarp();
        if (lane == 0) {
          s.meta[sl][p] = mt;
          mbar_arrive(smem_u32(&s.meta_full[sl][p]));
        }
        __syncwarp();
        ++t[sl];
        if (item < 0) done[sl] = true;
      }
    }
  } else if (warp == 0) {
    // ===================== TMA producer (whole warp; lane 0 issues)
    const uint64_t pol_q = policy_evict_first();
    const uint64_t pol_kv = policy_evict_last();
    SlotState st[2];
    int kvc = 0;  // tiles pushed through the ring
    auto push = [&](const CUtensorMap* map, int row, int plane) {
      const int r = kvc % kRing;
      TR_T0();
      if (kvc >= kRing) mbar_wait(smem_u32(&s.kv_empty[r]), ((kvc / kRing) - 1) & 1);
      TR_ADD(12);  // producer: waiting for a free ring slot
      if (lane == 0) {
        const uint32_t fb = smem_u32(&s.kv_full[r]);
        mbar_arrive_expect_tx(fb, (FPB_FA_PROBE == 5 || FPB_FA_PROBE == 8) ? kTile / 2 : kTile);
        tma_load_4d_hint(smem_u32(s.ring[r]), map, fb, 0, row, 0, plane, pol_kv);  // whole tile
      }
      __syncwarp();
      ++kvc;
    };
    while (st[0].active || st[1].active) {
      for (int sl = 0; sl < 2; ++sl) {
        SlotState& S = st[sl];
        if (!S.active) continue;
        const int p = S.t & 1;
        if (S.j == 0) {
          {
            TR_T0();
            mbar_wait(smem_u32(&s.meta_full[sl][p]), (S.t >> 1) & 1);
            TR_ADD(14);  // producer: waiting for the scheduler
          }
          const SlotMeta mt = s.meta[sl][p];
          S.item = mt.item;
          S.nblk = mt.nblk;
          if (S.item < 0) {
            S.active = false;
            continue;
          }
          S.zkv = mt.zkv;
          S.jbase = mt.jbase;
          {
            TR_T0();
            if (S.qc >= 1) mbar_wait(smem_u32(&s.q_empty[sl]), (S.qc - 1) & 1);
            TR_ADD(13);  // producer: waiting for the slot's Q tile (previous epilogue)
          }
          if (lane == 0) {
            const uint32_t qb = smem_u32(&s.q_full[sl]);
            mbar_arrive_expect_tx(qb, kTile);
            tma_load_4d_hint(smem_u32(s.q[sl]), &tm_q, qb, 0, mt.qi * kBlock, 0, mt.zh, pol_q);
          }
          __syncwarp();
          ++S.qc;
        }
        // ---- one unit: V(j-1) then K(j), matching the MMA issue order PV(j-1), QK(j)
        const int zkv = S.zkv;
        const uint16_t* lst = list_of(sl, p);
        if (S.j >= 1) push(&tm_v, (dense ? S.jbase + S.j - 1 : (int)lst[S.j - 1]) * kBlock, zkv);
        if (S.j < S.nblk) push(&tm_k, (dense ? S.jbase + S.j : (int)lst[S.j]) * kBlock, zkv);
        if (++S.j == S.nblk + 1) {
          S.j = 0;
          ++S.t;
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer: mirrors the producer's unit schedule
    const bool leader = elect_one();
    constexpr uint32_t idesc_qk = idesc_bf16_f32(128, 128, false, false);
    constexpr uint32_t idesc_pv = idesc_bf16_f32(128, 128, false, true);
    SlotState st[2];
    int kvc = 0;
    while (st[0].active || st[1].active) {
      for (int sl = 0; sl < 2; ++sl) {
        SlotState& S = st[sl];
        if (!S.active) continue;
        const int p = S.t & 1;
        const uint32_t s_tmem = tmem + sl * 128, o_tmem = tmem + 256 + sl * 128;
        if (S.j == 0) {
          mbar_wait(smem_u32(&s.meta_full[sl][p]), (S.t >> 1) & 1);
          S.item = s.meta[sl][p].item;
          S.nblk = s.meta[sl][p].nblk;
          S.cont = (s.meta[sl][p].mode & kContinue) != 0;
          if (S.item < 0) {
            S.active = false;
            continue;
          }
          {
            TR_T0();
            mbar_wait(smem_u32(&s.q_full[sl]), S.qc & 1);
            TR_ADD(15);  // MMA: waiting for Q
          }
          ++S.qc;
        }
        if (S.j >= 1) {
          // PV(j-1): O_sl (+)= P(j-1) [TMEM, aliasing S_sl] x V(j-1) [ring, MN-major]
          const int m = S.j - 1;
          if (m == 0 && S.qc >= 2) mbar_wait(smem_u32(&s.o_free[sl]), (S.qc - 2) & 1);
          const int r = kvc % kRing;
          TR_T0();
          mbar_wait(smem_u32(&s.kv_full[r]), (kvc / kRing) & 1);
          TR_ADD(8);  // MMA: waiting for V
          // SW128 descriptors are linear in the address field (addr >> 4, 14 bits; SMEM < 256 KiB),
          // so every K step is the tile's base descriptor plus a constant
          const uint64_t vdesc = sdesc_sw128(smem_u32(s.ring[r]), kTile / 2, 1024);
          // each part of the keys as soon as that part of P is in TMEM
          for (int part = 0; part < kPParts; ++part) {
            mbar_wait(smem_u32(&s.p_part[sl][part]), (S.bc - 1) & 1);
            tc_fence_after();
            TR_ADD(part + 1 == kPParts ? 10 : 9);  // MMA: waiting for a P part
            if (leader && FPB_FA_PROBE != 3 && FPB_FA_PROBE != 4 && FPB_FA_PROBE < 6) {
#pragma unroll
              for (int k4 = 0; k4 < 8 / kPParts; ++k4) {
                const int ks = part * (8 / kPParts) + k4;
                mma_bf16_ts(o_tmem, s_tmem + ks * 8, vdesc + (uint64_t)(ks * 2048 >> 4), idesc_pv,
                            (m > 0 || ks > 0 || S.cont) ? 1u : 0u);
              }
            }
            __syncwarp();
          }
          if (leader) {
            mma_commit(smem_u32(&s.kv_empty[r]));
            mma_commit(smem_u32(&s.o_done[sl]));
          }
          __syncwarp();
          ++kvc;
        }
        if (S.j < S.nblk) {
          // QK(j): S_sl = Q_sl K(j)^T
          const int r = kvc % kRing;
          TR_T0();
          mbar_wait(smem_u32(&s.kv_full[r]), (kvc / kRing) & 1);
          tc_fence_after();
          TR_ADD(11);  // MMA: waiting for K
          if (leader) {
            const uint64_t qdesc = sdesc_sw128(smem_u32(s.q[sl]), 16, 1024);
            const uint64_t kdesc = sdesc_sw128(smem_u32(s.ring[r]), 16, 1024);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
              const uint64_t off = ((ks >> 2) * (kTile / 2) + (ks & 3) * 32) >> 4;
              if (FPB_FA_PROBE != 3 && FPB_FA_PROBE != 4 && FPB_FA_PROBE < 6)
                mma_bf16_ss(s_tmem, qdesc + off, kdesc + off, idesc_qk, ks > 0 ? 1u : 0u);
            }
            mma_commit(smem_u32(&s.kv_empty[r]));
            mma_commit(smem_u32(&s.s_full[sl]));

          }
          __syncwarp();
          ++kvc;
          ++S.bc;
        }
        if (++S.j == S.nblk + 1) {
          S.j = 0;
          ++S.t;
        }
      }
    }
  }
  } else {
    setmaxnreg_inc<216>();
    // ===================== softmax + epilogue, one warpgroup per slot
    const int sl = (warp - 4) >> 2;
    const int r = ((warp - 4) & 3) * 32 + lane;  // query row == TMEM lane
    const uint32_t lane_addr = static_cast<uint32_t>(((warp - 4) & 3) * 32) << 16;
    const uint32_t s_addr = tmem + lane_addr + sl * 128;
    const uint32_t o_addr = tmem + lane_addr + 256 + sl * 128;
    int bc = 0, qc = 0;
    for (int t = 0;; ++t) {
      const int p = t & 1;
      mbar_wait(smem_u32(&s.meta_full[sl][p]), (t >> 1) & 1);
      const SlotMeta mt = s.meta[sl][p];
      if (mt.item < 0) break;
      const int nblk = mt.nblk, qi = mt.qi, zh = mt.zh;
      const bool cont = (mt.mode & kContinue) != 0;
      const uint16_t* lst = list_of(sl, p);
      const int rows = block_len(D, qi);
      float m_used = -INFINITY, l = 0.f;
      // rows that span several KV-range phases carry (O, m, l) between them (fa_phases)
      float* po = nullptr;
      if (mt.mode & (kContinue | kPartialOut))
        po = prm.part + ((size_t)zh * (D.M - prm.chunk) + (qi - prm.chunk)) * kPartFloats;
      if (cont) {  // O starts from the partial (the slot's previous O was read out above)
        m_used = __ldcg(po + kBlock * kHeadDim + r);
        l = __ldcg(po + kBlock * kHeadDim + kBlock + r);
        const float4* src = reinterpret_cast<const float4*>(po + (size_t)r * kHeadDim);
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t o[32];
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4) {
            const float4 x = __ldcs(src + cc * 8 + q4);  // read once: evict first
            o[4 * q4] = __float_as_uint(x.x);
            o[4 * q4 + 1] = __float_as_uint(x.y);
            o[4 * q4 + 2] = __float_as_uint(x.z);
            o[4 * q4 + 3] = __float_as_uint(x.w);
          }
          tmem_st32(o_addr + cc * 32, o);
        }
        tmem_st_wait();
      }
      for (int n = 0; n < nblk; ++n, ++bc) {
        const int kv = dense ? mt.jbase + n : (int)lst[n];
        const int cols = block_len(D, kv);
        const int lim = (kv == qi) ? min(cols, r + 1) : cols;  // attention.hpp:85-91
        const bool full = __all_sync(0xffffffffu, lim == kBlock);
        TR_T0();
        mbar_wait(smem_u32(&s.s_full[sl]), bc & 1);
        tc_fence_after();
        TR_ADD(0);  // softmax: waiting for S
        uint32_t v[128];
        const float sc = D.to_bits;
        float bs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        // causal diagonal / ragged tail: columns >= lim do not exist (attention.hpp:85-91)
        auto mask_half = [&](int half) {
          if (!full) {
#pragma unroll
            for (int c = half * 64; c < half * 64 + 64; ++c)
              if (c >= lim) v[c] = __float_as_uint(-INFINITY);
          }
        };
        auto max_half = [&](int half) {  // 4 independent 3-input max chains
          float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
          for (int c = half * 64; c < half * 64 + 64; c += 8) {
            mx0 = fmaxf(mx0, fmaxf(__uint_as_float(v[c + 0]), __uint_as_float(v[c + 1])));
            mx1 = fmaxf(mx1, fmaxf(__uint_as_float(v[c + 2]), __uint_as_float(v[c + 3])));
            mx2 = fmaxf(mx2, fmaxf(__uint_as_float(v[c + 4]), __uint_as_float(v[c + 5])));
            mx3 = fmaxf(mx3, fmaxf(__uint_as_float(v[c + 6]), __uint_as_float(v[c + 7])));
          }
          return fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
        };
        // P = exp2(S * to_bits - m) for the columns of one part, packed in place:
        // v[c/2] <- bf16x2(p_c, p_c+1); row sums in 8 independent accumulators
        constexpr int kPC = kBlock / kPParts;  // columns per part
        auto exp_half = [&](int half, float neg_m) {
          if (full) {
#pragma unroll
            for (int c = half * kPC; c < half * kPC + kPC; c += 2) {
              // MUFU ex2 for every element: FMA-pipe emulation measured slower on B200
              // (profiles/r1_fa_trace.txt)
              float x0, x1;
              ffma2(x0, x1, __uint_as_float(v[c]), __uint_as_float(v[c + 1]), sc, sc, neg_m, neg_m);
              const float p0 = FA_EX2(x0), p1 = FA_EX2(x1);
              const int a = ((c >> 1) & 3) * 2;
              fadd2(bs[a], bs[a + 1], bs[a], bs[a + 1], p0, p1);
              v[c >> 1] = pack_bf16x2(p0, p1);
            }
          } else {
#pragma unroll
            for (int c = half * kPC; c < half * kPC + kPC; c += 2) {
              const float p0 = FA_EX2(fmaf(__uint_as_float(v[c]), sc, neg_m));
              const float p1 = FA_EX2(fmaf(__uint_as_float(v[c + 1]), sc, neg_m));
              const int a = ((c >> 1) & 3) * 2;
              fadd2(bs[a], bs[a + 1], bs[a], bs[a + 1], p0, p1);
              v[c >> 1] = pack_bf16x2(p0, p1);
            }
          }
        };
        // lazy O rescale (exact: numerator and denominator share the stale max)
        auto rescale = [&](float m_new) {
          mbar_wait(smem_u32(&s.o_done[sl]), (bc - 1) & 1);  // O must hold PV(n-1)
          tc_fence_after();
          const float f = ex2_approx(m_used - m_new);
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            uint32_t o[32];
            tmem_ld32(o_addr + cc * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 32; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * f);
            tmem_st32(o_addr + cc * 32, o);
          }
          l *= f;
          m_used = m_new;
        };
        {
#if FPB_FA_PROBE == 6 || FPB_FA_PROBE == 7
#pragma unroll
          for (int c = 0; c < 128; ++c) v[c] = (uint32_t)c;
#if FPB_FA_PROBE == 7
          tmem_ld32(s_addr + 0, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));  // a quarter of S
          tmem_ld_wait();
#endif
#else
          tmem_ld64(s_addr + 0, &v[0]);
          tmem_ld64(s_addr + 64, &v[64]);
          tmem_ld_wait();
#endif
#if FPB_FA_PROBE == 1 || FPB_FA_PROBE == 4 || FPB_FA_PROBE == 6 || FPB_FA_PROBE == 7 || FPB_FA_PROBE == 8
          const float m_new = 0.f;
#else
          mask_half(0);
          mask_half(1);
          const float m_new = fmaxf(m_used, fmaxf(max_half(0), max_half(1)) * sc);
#endif
          TR_ADD(1);  // softmax: TMEM load + mask + row max
          if (n == 0 && !cont)
            m_used = m_new;
          else if (__any_sync(0xffffffffu, m_new > m_used + kRescaleThreshold))
            rescale(m_new);
          TR_ADD(2);  // softmax: lazy O rescale (rare)
#if FPB_FA_PROBE != 1 && FPB_FA_PROBE != 4 && FPB_FA_PROBE < 6
          exp_half(0, -m_used);
#endif
        }
#pragma unroll
        for (int half = 0; half < kPParts; ++half) {
#if FPB_FA_PROBE != 1 && FPB_FA_PROBE != 4 && FPB_FA_PROBE < 6
          if (half > 0) exp_half(half, -m_used);
#endif
          // P of this part's keys -> TMEM columns (kPC / 2) half .. (bf16 pairs over S)
          if constexpr (kPParts == 1) {
            tmem_st32(s_addr, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
            tmem_st32(s_addr + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
          } else if constexpr (kPParts == 2)
            tmem_st32(s_addr + half * 32, *reinterpret_cast<uint32_t(*)[32]>(&v[half * 32]));
          else
            tmem_st16(s_addr + half * 16, *reinterpret_cast<uint32_t(*)[16]>(&v[half * 16]));
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&s.p_part[sl][half]));
          TR_ADD(half + 1 == kPParts ? 4 : 3);  // softmax: exp + pack + TMEM store, per part
        }
        l += ((bs[0] + bs[1]) + (bs[2] + bs[3])) + ((bs[4] + bs[5]) + (bs[6] + bs[7]));
      }
      TR_T0();
      // ---- epilogue (attention.hpp:119-126)
      const size_t orow = (size_t)zh * D.L + (size_t)qi * kBlock + r;
      if (mt.mode & kPartialOut) {
        // the row continues in a later KV-range phase: hand over O (unnormalised), m and l
        mbar_wait(smem_u32(&s.o_done[sl]), (bc - 1) & 1);
        tc_fence_after();
        float4* dst = reinterpret_cast<float4*>(po + (size_t)r * kHeadDim);
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t o[32];
          tmem_ld32(o_addr + cc * 32, o);
          tmem_ld_wait();
          if (cc == 3) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&s.o_free[sl]));
          }
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4)
            __stcs(dst + cc * 8 + q4,  // streamed (re-read only by the next phase's launch)
                   make_float4(__uint_as_float(o[4 * q4]), __uint_as_float(o[4 * q4 + 1]),
                               __uint_as_float(o[4 * q4 + 2]), __uint_as_float(o[4 * q4 + 3])));
        }
        __stcg(po + kBlock * kHeadDim + r, m_used);
        __stcg(po + kBlock * kHeadDim + kBlock + r, l);
        named_bar_sync(1 + sl, 128);
        if (r == 0) {
          prm.pflag[(size_t)zh * D.M + qi] = 1;  // read by the next phase's launch
          mbar_arrive(smem_u32(&s.q_empty[sl]));
        }
        ++qc;
      } else if (nblk > 0) {
        mbar_wait(smem_u32(&s.o_done[sl]), (bc - 1) & 1);  // last PV done => last QK done too
        tc_fence_after();
        const float inv = 1.0f / l;
        const uint32_t stage = smem_u32(s.q[sl]);  // this slot's Q tile is free: O staging
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t o[32];
          tmem_ld32(o_addr + cc * 32, o);
          tmem_ld_wait();
          if (cc == 3) {  // O fully read: release the accumulator for the slot's next item
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&s.o_free[sl]));
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
        if (r < rows) prm.lse[orow] = m_used + log2f(l);
        if (prm.out_bf16) {
          fence_proxy_async_smem();
          named_bar_sync(1 + sl, 128);
          if (r == 0) {  // rows beyond L are clipped by the tensor map
            // O is written once and never re-read here: keep it from evicting K/V lines
            const uint64_t pol_o = policy_evict_first();
            tma_store_3d_hint(&tm_o, stage, 0, qi * kBlock, zh, pol_o);
            tma_store_3d_hint(&tm_o, stage + kTile / 2, 64, qi * kBlock, zh, pol_o);
            bulk_commit();
            bulk_wait_read0();
            mbar_arrive(smem_u32(&s.q_empty[sl]));
          }
        } else {
          named_bar_sync(1 + sl, 128);  // every thread is past its tcgen05.ld of O
          if (r == 0) mbar_arrive(smem_u32(&s.q_empty[sl]));
        }
        ++qc;
      } else if (r < rows) {  // C = 0: out = 0 * (1/0) = NaN, lse = -inf (attention.hpp:121-125)
        const float nan = __int_as_float(0x7fc00000);
        if (prm.out_bf16) {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(prm.out) + orow * kHeadDim);
          const uint32_t pn = pack_bf16x2(nan, nan);
          for (int q4 = 0; q4 < 16; ++q4) dst[q4] = make_uint4(pn, pn, pn, pn);
        } else {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(prm.out) + orow * kHeadDim);
          for (int q4 = 0; q4 < 32; ++q4) dst[q4] = make_float4(nan, nan, nan, nan);
        }
        prm.lse[orow] = -INFINITY;
      }
      TR_ADD(5);  // softmax warps: item epilogue
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&s.meta_empty[sl][p]));
    }
    (void)qc;
  }
  TR_FLUSH();
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

}  // namespace

// KV-range phases: when one KV group's K and V exceed the L2 budget (kPhaseBytes), its key blocks
// are processed in `phases` ranges of `chunk` blocks, one launch per range; within a launch the
// work order is still KV-group-major, so all Q heads of a group stream the same L2-sized slice of
// its K/V (at 256K one Qwen3 group's K/V is 128 MB, above the 126 MB L2).  Rows
// spanning several ranges carry their exact fp32 (O, m, l) through a global partial buffer, so the
// arithmetic, and the result, equal the single-launch kernel's bit for bit.  Whole-row problems
// only (no row shards); FPB_FA_PHASES overrides (measurement switch).
int fa_phases(const Dims& D, int* chunk) {
  static const int env = [] {
    const char* e = std::getenv("FPB_FA_PHASES");
    return e ? std::atoi(e) : 0;
  }();
  int P = 1;
  if (D.rs == 1 && !D.zz && D.Mr == D.M) {
    const double group_bytes = 2.0 * D.L * D.d * 2.0;
    P = env > 0 ? env : (int)((group_bytes + kPhaseBytes - 1) / kPhaseBytes);
    P = P < 1 ? 1 : (P > 8 ? 8 : P);
  }
  int c = (D.M + P - 1) / P;
  if (P > 1 && c < 4) P = 1;  // not worth it for a few key blocks
  if (P == 1) c = D.M;
  P = (D.M + c - 1) / c;
  if (chunk) *chunk = c;
  return P;
}

size_t attention_phase_bytes(const Dims& D) {
  int c;
  if (fa_phases(D, &c) == 1) return 0;
  const size_t flags = ((size_t)D.Z * D.Hq * D.M * sizeof(int) + 1023) / 1024 * 1024;
  return flags + (size_t)D.Z * D.Hq * (D.M - c) * kPartFloats * sizeof(float);
}

cudaError_t launch_attention_fa(const Dims& D, const __nv_bfloat16* Q, const __nv_bfloat16* K,
                                const __nv_bfloat16* V, const int32_t* idx, const int32_t* counts,
                                bool out_bf16, void* out, float* lse, unsigned long long* visits,
                                int32_t* plan_error, int* sched, uint16_t* lists,
                                uint8_t* phase_ws, cudaStream_t s) {
  CUtensorMap tm_q, tm_k, tm_v, tm_o;
  if (!make_tmap_tiles128(&tm_q, Q, D.L, (uint64_t)D.Z * D.Hq) ||
      !make_tmap_tiles128(&tm_k, K, D.L, (uint64_t)D.Z * D.Hkv, (FPB_FA_PROBE == 5 || FPB_FA_PROBE == 8) ? 1 : 2) ||
      !make_tmap_tiles128(&tm_v, V, D.L, (uint64_t)D.Z * D.Hkv, (FPB_FA_PROBE == 5 || FPB_FA_PROBE == 8) ? 1 : 2) ||
      !make_tmap_rows128(&tm_o, out_bf16 ? out : Q, D.L, (uint64_t)D.Z * D.Hq))
    return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(sched, 0, sizeof(int), s);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int chunk = D.M;
  const int phases = fa_phases(D, &chunk);
  int* pflag = nullptr;
  float* part = nullptr;
  if (phases > 1) {
    if (!phase_ws) return cudaErrorInvalidValue;
    pflag = reinterpret_cast<int*>(phase_ws);
    part = reinterpret_cast<float*>(
        phase_ws + ((size_t)D.Z * D.Hq * D.M * sizeof(int) + 1023) / 1024 * 1024);
    e = cudaMemsetAsync(pflag, 0, (size_t)D.Z * D.Hq * D.M * sizeof(int), s);
    if (e != cudaSuccess) return e;
  }
  // K/V bytes of one KV group = 2 tensors x L x d x 2 B; keep gs groups' worth <= 64 MiB
  // (measured: 32K prefers all 4 Qwen3 groups interleaved, 128K/256K one group at a time).
  // FPB_FA_GS overrides (measurement switch).
  static const int gs_env = [] {
    const char* e = std::getenv("FPB_FA_GS");
    return e ? std::atoi(e) : 0;
  }();
  int gs = gs_env;
  if (gs <= 0) {
    const double group_bytes = 2.0 * D.L * D.d * 2.0;
    gs = (int)(kPhaseBytes / group_bytes);
  }
  gs = gs < 1 ? 1 : (gs > D.Hkv ? D.Hkv : gs);
  while (D.Hkv % gs) --gs;
  if (phases > 1) gs = 1;
  const size_t smem = sizeof(FaSmem) + 1024;
  e = cudaFuncSetAttribute(fa_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  for (int ph = 0; ph < phases; ++ph) {
    const int num_items = phases > 1 ? D.Z * D.Hq * (D.M - ph * chunk) : D.Z * D.Hq * D.Mr;
    if (ph > 0) {  // the next launch restarts the work counter
      e = cudaMemsetAsync(sched, 0, sizeof(int), s);
      if (e != cudaSuccess) return e;
    }
    const int grid = num_items < sms ? num_items : sms;
    FaParams prm{D,     idx,   counts, out,   lse,    visits, plan_error, sched,
                 lists, num_items, out_bf16 ? 1 : 0, gs, phases, chunk, ph, part, pflag};
    fa_kernel<<<grid, kThreads, smem, s>>>(tm_q, tm_k, tm_v, tm_o, prm);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace fpb

#ifdef FPB_TRACE
extern "C" int fpb_trace_read(unsigned long long* host16, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(host16, fpb::g_trace, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(fpb::g_trace, z, sizeof(z));
  }
  return (int)e;
}
#endif
