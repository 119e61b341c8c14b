// fp_kernels.h — host-side launchers of the sm_100a kernels (internal to libfpb200.so).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "fp_common.cuh"

namespace fpb {

// pool.cu
// Pools key blocks [j0, j0 + nj) (all blocks by default).
cudaError_t launch_pool_keys(const Dims& D, bool bf16_in, const void* K, float* pooled,
                             __nv_bfloat16* kbar_split, cudaStream_t s, int j0 = 0, int nj = -1);
cudaError_t launch_split_pooled(const Dims& D, const float* pooled, __nv_bfloat16* kbar_split,
                                cudaStream_t s);
cudaError_t launch_f32_to_bf16(const float* src, __nv_bfloat16* hi, __nv_bfloat16* lo, size_t n,
                               cudaStream_t s);

// select.cu
cudaError_t launch_normalize(const Dims& D, const float* energy, const float* local_max,
                             float* score, cudaStream_t s);
cudaError_t launch_threshold(const Dims& D, const float* score, uint8_t* mask,
                             unsigned long long* comparisons, cudaStream_t s);
// Owned plan rows (Z x [rb + rs k] x N x Hq) set to the fill value N.
cudaError_t launch_fill_plan(const Dims& D, int32_t* idx, cudaStream_t s);
cudaError_t launch_compress(const Dims& D, const uint8_t* mask, int32_t* idx, int32_t* counts,
                            cudaStream_t s);
cudaError_t launch_visit_count(const Dims& D, const int32_t* counts, unsigned long long* total,
                               cudaStream_t s);
cudaError_t launch_full_causal_plan(const Dims& D, int32_t* idx, int32_t* counts, cudaStream_t s);

// discover.cu — fused block approximation (+ normalisation, + optional threshold/compaction).
struct DiscoverOut {
  float* energy = nullptr;
  float* local_max = nullptr;
  float* score = nullptr;
  uint8_t* mask = nullptr;
  int32_t* idx = nullptr;
  int32_t* counts = nullptr;
  bool normalize = true;  // false: only energy/local_max (approx_block_scores)
  // Two-pass plan-only mode: the discovery kernel writes the causal (local max, energy) pairs
  // of every row to `rows` (packed triangle per (z, h): row I at I(I+1)/2) and a warp-per-row
  // select kernel normalises, thresholds and compacts them (select.cu).
  float2* rows = nullptr;
};
// Bytes of the packed (m, S) triangle of the two-pass mode.
inline size_t discover_rows_bytes(const Dims& D) {
  return (size_t)D.Z * D.Hq * ((size_t)D.M * (D.M + 1) / 2) * sizeof(float2);
}
cudaError_t launch_select_rows(const Dims& D, const float2* rows, int32_t* idx, int32_t* counts,
                               bool prefilled, cudaStream_t s);
// kpool != nullptr (bf16 keys, q_splits == 1): the kernel pools K itself into kbar_split (and
// `pooled` if given), using the pool_ctr counters (discover_pool_ctr_bytes, zeroed here);
// otherwise kbar_split already holds k̄.
cudaError_t launch_discover(const Dims& D, int q_splits, const __nv_bfloat16* q_planes,
                            __nv_bfloat16* kbar_split, const DiscoverOut& out, int* sched,
                            float* mscratch, cudaStream_t s, const __nv_bfloat16* kpool = nullptr,
                            float* pooled = nullptr, int* pool_ctr = nullptr);
size_t discover_pool_ctr_bytes(const Dims& D);
// Global scratch launch_discover needs (0 while the per-key-block rows fit in shared memory,
// i.e. up to ~270K tokens at B = 128).
size_t discover_scratch_bytes(const Dims& D);

// attention.cu / attention_fa.cu — block-sparse (idx/counts) or dense-causal (idx == nullptr).
cudaError_t launch_attention(const Dims& D, int splits, const __nv_bfloat16* Q,
                             const __nv_bfloat16* K, const __nv_bfloat16* V, const int32_t* idx,
                             const int32_t* counts, bool out_bf16, void* out, float* lse,
                             unsigned long long* visits, int32_t* plan_error, int* sched,
                             uint16_t* lists, uint8_t* phase_ws, cudaStream_t s);
cudaError_t launch_attention_fa(const Dims& D, const __nv_bfloat16* Q, const __nv_bfloat16* K,
                                const __nv_bfloat16* V, const int32_t* idx, const int32_t* counts,
                                bool out_bf16, void* out, float* lse, unsigned long long* visits,
                                int32_t* plan_error, int* sched, uint16_t* lists,
                                uint8_t* phase_ws, cudaStream_t s);
// KV-range phases of the bf16 attention kernel (1 = none) and their workspace (flags + partials)
int fa_phases(const Dims& D, int* chunk);
size_t attention_phase_bytes(const Dims& D);
// bytes of the compacted-plan scratch launch_attention needs (grid x 2 slots x 2 bufs x M x u16)
size_t attention_list_bytes(const Dims& D);
size_t attention_f32_smem_bytes(const Dims& D);  // fp32-input kernel (attention.cu)

// generic.cu — SIMT kernels for shapes outside the tensor-core tile (d != 128 or B != 128)
cudaError_t g_launch_pool(const GenDims& G, bool bf16_in, const void* K, float* pooled,
                          cudaStream_t s);
cudaError_t g_launch_approx(const GenDims& G, bool bf16_in, const void* Q, const float* pooled,
                            float* energy, float* local_max, cudaStream_t s);
size_t g_attention_scratch_bytes(const GenDims& G);
cudaError_t g_launch_attention(const GenDims& G, bool bf16_in, const void* Q, const void* K,
                               const void* V, const int32_t* idx, const int32_t* counts,
                               bool out_bf16, void* out, float* lse, unsigned long long* visits,
                               int32_t* plan_error, float* scratch, cudaStream_t s);

// baselines.cu — comparison methods of the reference (top-k / top-p, pool-both, exact)
cudaError_t launch_sort_select(const Dims& D, const float* score, uint8_t* mask, int mode, int k,
                               float p, cudaStream_t s);  // mode 0: top-k, 1: top-p
cudaError_t launch_pool_both(const Dims& D, bool bf16_in, const void* Q, const void* K,
                             float* pooled_q, float* pooled_k, float* energy, float* local_max,
                             cudaStream_t s);
size_t exact_table_bytes(const Dims& D);
cudaError_t launch_exact(const Dims& D, bool bf16_in, const void* Q, const void* K, float* pooled,
                         float* table, float* energy, float* local_max, float* score,
                         cudaStream_t s);

// tensor maps (abi.cu)
bool make_tmap_rows128(CUtensorMap* map, const void* base, uint64_t rows, uint64_t planes);
bool make_tmap_tiles128(CUtensorMap* map, const void* base, uint64_t rows, uint64_t planes,
                        uint32_t box_halves = 2);

}  // namespace fpb
