/* fpb200.h — C ABI of the B200-native FlashPrefill hot path (sm_100a CUDA kernels).
 *
 * Drop-in boundary for the reference's header-only C++ API (namespace bsattn,
 * /root/reference/proj/include/bsattn/).  Each entry point below names the reference function it
 * replaces (file:line).  Tensor layouts, the block grid, and the alpha / sink / window / scale /
 * epsilon parameters are exactly the reference's:
 *
 *   Q          Z x Hq  x L x d            (bf16 or fp32)
 *   K, V       Z x Hkv x L x d            (Hkv divides Hq; Hkv == Hq is the reference case)
 *   pooled     Z x Hkv x N x d   fp32     (discovery.hpp:19-21)
 *   energy, local_max, score   Z x Hq x M x N   fp32   (discovery.hpp:25-34)
 *   mask       Z x M x N x Hq    u8       (selection.hpp:14-21, head axis last)
 *   idx        Z x M x N x Hq    i32      (selection.hpp:26-34, fill value N)
 *   counts     Z x M x Hq        i32
 *   out        Z x Hq x L x d    (bf16 or fp32)      lse  Z x Hq x L  fp32, base 2
 * with M = N = ceil(L / B) (core.hpp:31-41).  GQA (not in the reference): Q head h reads
 * KV head h / (Hq / Hkv); maps and plans stay per Q head.
 *
 * Conventions
 *   - fpb_* functions take DEVICE pointers and are stream-ordered on `stream` (cudaStream_t passed
 *     as void*; NULL = legacy default stream).  They never allocate on the hot path: scratch comes
 *     from a caller-provided workspace sized by fpb_workspace_bytes().
 *   - With d = B = 128 (the tcgen05 path) Q, K, V and out must be 16-byte aligned (TMA / bulk
 *     copies); a misaligned base address returns 2 (validation) instead of faulting.
 *   - fpb_host_* functions take HOST pointers, copy in, run, copy out and synchronise; they are what
 *     the C++ drop-in layer (include/fpb200/bsattn.hpp) calls.
 *   - Return codes mirror the reference CLI's exit codes (bsattn_main.cpp:671-692):
 *     0 ok, 1 usage, 2 validation / config / plan error, 3 format / io, 4 CUDA runtime error.
 *     fpb_last_error() returns a thread-local message for the last failure on this thread.
 *   - Reentrant across streams; the only global state is the thread-local error string and a
 *     per-device cache of kernel attributes.
 */
#ifndef FPB200_H
#define FPB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FPB_OK 0
#define FPB_EUSAGE 1
#define FPB_EVALIDATION 2
#define FPB_EFORMAT 3
#define FPB_ECUDA 4

typedef enum { FPB_F32 = 0, FPB_BF16 = 1 } fpb_dtype;

/* Problem description: shapes plus PipelineConfig (core.hpp:87-112). */
typedef struct {
  int64_t Z, Hq, Hkv, L, d; /* d must be 128 (the tcgen05 tile width) */
  int32_t block_size;       /* B; must be 128 (core.hpp:88) */
  float alpha;              /* core.hpp:89, >= 0 */
  int32_t sink_tokens;      /* core.hpp:90 */
  int32_t window_tokens;    /* core.hpp:91, >= 1 */
  float scale;              /* core.hpp:92, <= 0 selects d^-1/2 */
  float epsilon;            /* core.hpp:93, > 0 */
} fpb_problem;

/* Fills the reference defaults (core.hpp:87-94) for the given shape. */
void fpb_problem_init(fpb_problem* p, int64_t Z, int64_t Hq, int64_t Hkv, int64_t L, int64_t d);

int fpb_version(void);
const char* fpb_last_error(void);

/* Scratch bytes for every fpb_* call of this problem (max over entry points). */
int fpb_workspace_bytes(const fpb_problem* p, fpb_dtype dtype, size_t* bytes);

/* ---- Instantaneous Pattern Discovery (discovery.hpp) ------------------------------------- */
/* pool_keys (discovery.hpp:65-70): pooled[z,h,j,:] = (sum of the block's key rows) * (1/len). */
int fpb_pool_keys(const fpb_problem* p, fpb_dtype dtype, const void* K, float* pooled,
                  void* stream);
/* approx_block_scores (discovery.hpp:75-115) from caller-provided pooled keys. */
int fpb_approx_block_scores(const fpb_problem* p, fpb_dtype dtype, const void* Q,
                            const float* pooled, float* energy, float* local_max, void* workspace,
                            size_t workspace_bytes, void* stream);
/* normalize_block_scores (discovery.hpp:119-148). */
int fpb_normalize_block_scores(const fpb_problem* p, const float* energy, const float* local_max,
                               float* score, void* stream);
/* discover (discovery.hpp:153-159): pooling + fused block approximation + normalisation.
 * energy / local_max may be NULL (not materialised). */
int fpb_discover(const fpb_problem* p, fpb_dtype dtype, const void* Q, const void* K,
                 float* energy, float* local_max, float* score, void* workspace,
                 size_t workspace_bytes, void* stream);

/* ---- Max-based Dynamic Thresholding (selection.hpp) -------------------------------------- */
/* max_threshold_mask (selection.hpp:63-92, 161-164).  comparisons (nullable, device u64) is
 * incremented by the reference's SelectionStats count (2 per causal cell). */
int fpb_max_threshold_mask(const fpb_problem* p, const float* score, uint8_t* mask,
                           unsigned long long* comparisons, void* stream);
/* compress_indices (selection.hpp:176-192). */
int fpb_compress_indices(const fpb_problem* p, const uint8_t* mask, int32_t* idx, int32_t* counts,
                         void* stream);
/* Fused discover -> max_threshold_mask -> compress_indices in one pass over Q (no M x N maps
 * unless requested).  energy / local_max / score / mask are nullable. */
int fpb_discover_select(const fpb_problem* p, fpb_dtype dtype, const void* Q, const void* K,
                        float* energy, float* local_max, float* score, uint8_t* mask, int32_t* idx,
                        int32_t* counts, void* workspace, size_t workspace_bytes, void* stream);
/* visit_count (selection.hpp:195-200) into a device u64 (overwritten). */
int fpb_visit_count(const fpb_problem* p, const int32_t* counts, unsigned long long* total,
                    void* stream);

/* ---- Block-sparse attention (attention.hpp) ---------------------------------------------- */
/* block_sparse_attention (attention.hpp:38-132).  visits (nullable, device u64) is incremented
 * by AttentionStats.block_visits; plan_error (nullable, device i32) is set to 1 when a plan row
 * lists a block outside [0, N) — the reference's PlanError (attention.hpp:78-81). */
int fpb_block_sparse_attention(const fpb_problem* p, fpb_dtype dtype, const void* Q, const void* K,
                               const void* V, const int32_t* idx, const int32_t* counts,
                               fpb_dtype out_dtype, void* out, float* lse,
                               unsigned long long* visits, int32_t* plan_error, void* workspace,
                               size_t workspace_bytes, void* stream);

/* ---- Row-sharded execution (multi-GPU partition; no reference counterpart) ---------------- */
/* Same as fpb_discover_select / fpb_block_sparse_attention restricted to the query blocks
 * I = row_begin + row_step * k (0 <= row_begin < row_step).  Every (z, h, I) is independent
 * (discovery.hpp:87-88, selection.hpp:71-72, attention.hpp:59-60), so row_step ranks with
 * row_begin = rank split the work evenly whatever the per-head density; plan rows and output rows
 * of blocks the shard does not own are left untouched.  Buffers keep the full-problem layout
 * (every rank holds K/V and the pooled keys of the whole sequence).  d = block_size = 128 only. */
int fpb_discover_select_rows(const fpb_problem* p, int32_t row_begin, int32_t row_step,
                             fpb_dtype dtype, const void* Q, const void* K, float* energy,
                             float* local_max, float* score, uint8_t* mask, int32_t* idx,
                             int32_t* counts, void* workspace, size_t workspace_bytes,
                             void* stream);
int fpb_block_sparse_attention_rows(const fpb_problem* p, int32_t row_begin, int32_t row_step,
                                    fpb_dtype dtype, const void* Q, const void* K, const void* V,
                                    const int32_t* idx, const int32_t* counts,
                                    fpb_dtype out_dtype, void* out, float* lse,
                                    unsigned long long* visits, int32_t* plan_error,
                                    void* workspace, size_t workspace_bytes, void* stream);
/* Zigzag shard: the query blocks are cut into 2 * world contiguous chunks of
 * ceil(M / (2 * world)) blocks and rank owns chunks `rank` and `2 * world - 1 - rank` -- equal
 * causal work per rank like the interleaved shard above, but contiguous rows, so the concurrently
 * processed rows of a rank share their K/V blocks in L2 as in the unsharded call.
 * 0 <= rank < world; otherwise as the _rows entry points. */
int fpb_discover_select_zigzag(const fpb_problem* p, int32_t rank, int32_t world,
                               fpb_dtype dtype, const void* Q, const void* K, float* energy,
                               float* local_max, float* score, uint8_t* mask, int32_t* idx,
                               int32_t* counts, void* workspace, size_t workspace_bytes,
                               void* stream);
int fpb_block_sparse_attention_zigzag(const fpb_problem* p, int32_t rank, int32_t world,
                                      fpb_dtype dtype, const void* Q, const void* K,
                                      const void* V, const int32_t* idx, const int32_t* counts,
                                      fpb_dtype out_dtype, void* out, float* lse,
                                      unsigned long long* visits, int32_t* plan_error,
                                      void* workspace, size_t workspace_bytes, void* stream);

/* dense_attention (attention.hpp:135-174): the dense causal kernel, the speedup denominator. */
int fpb_dense_attention(const fpb_problem* p, fpb_dtype dtype, const void* Q, const void* K,
                        const void* V, fpb_dtype out_dtype, void* out, float* lse, void* workspace,
                        size_t workspace_bytes, void* stream);
/* full_causal_plan (attention.hpp:178-192). */
int fpb_full_causal_plan(const fpb_problem* p, int32_t* idx, int32_t* counts, void* stream);

/* ---- Comparison baselines of the reference (not on the FlashPrefill path) ---------------- */
/* topk_select (selection.hpp:96-123): min(k, i+1) highest scores per causal row, ties toward the
 * lower block index, plus sink/window retention.  Rows up to 4096 blocks. */
int fpb_topk_select(const fpb_problem* p, const float* score, int32_t k, uint8_t* mask,
                    void* stream);
/* topp_select (selection.hpp:127-159): shortest descending prefix reaching mass p (0 < p <= 1). */
int fpb_topp_select(const fpb_problem* p, const float* score, float top_p, uint8_t* mask,
                    void* stream);
/* discover_pool_both (discovery.hpp:164-195) and discover_exact (discovery.hpp:201-279).
 * Scratch: fpb_baseline_workspace_bytes. */
int fpb_baseline_workspace_bytes(const fpb_problem* p, size_t* bytes);
int fpb_discover_pool_both(const fpb_problem* p, fpb_dtype dtype, const void* Q, const void* K,
                           float* energy, float* local_max, float* score, void* workspace,
                           size_t workspace_bytes, void* stream);
int fpb_discover_exact(const fpb_problem* p, fpb_dtype dtype, const void* Q, const void* K,
                       float* energy, float* local_max, float* score, void* workspace,
                       size_t workspace_bytes, void* stream);

/* ---- Host-buffer entry points (copy in, run, copy out, synchronise) ----------------------- */
int fpb_host_pool_keys(const fpb_problem* p, fpb_dtype dtype, const void* K, float* pooled);
int fpb_host_approx_block_scores(const fpb_problem* p, fpb_dtype dtype, const void* Q,
                                 const float* pooled, float* energy, float* local_max);
int fpb_host_normalize_block_scores(const fpb_problem* p, const float* energy,
                                    const float* local_max, float* score);
int fpb_host_discover(const fpb_problem* p, fpb_dtype dtype, const void* Q, const void* K,
                      float* energy, float* local_max, float* score);
int fpb_host_max_threshold_mask(const fpb_problem* p, const float* score, uint8_t* mask,
                                unsigned long long* comparisons);
int fpb_host_topk_select(const fpb_problem* p, const float* score, int32_t k, uint8_t* mask);
int fpb_host_topp_select(const fpb_problem* p, const float* score, float top_p, uint8_t* mask);
/* method: 0 approx (== fpb_host_discover), 1 pool-both, 2 exact */
int fpb_host_discover_method(const fpb_problem* p, fpb_dtype dtype, int method, const void* Q,
                             const void* K, float* energy, float* local_max, float* score);
int fpb_host_compress_indices(const fpb_problem* p, const uint8_t* mask, int32_t* idx,
                              int32_t* counts);
int fpb_host_block_sparse_attention(const fpb_problem* p, fpb_dtype dtype, const void* Q,
                                    const void* K, const void* V, const int32_t* idx,
                                    const int32_t* counts, fpb_dtype out_dtype, void* out,
                                    float* lse, unsigned long long* visits);
int fpb_host_dense_attention(const fpb_problem* p, fpb_dtype dtype, const void* Q, const void* K,
                             const void* V, fpb_dtype out_dtype, void* out, float* lse);
/* The whole prefill (acceptance.cpp:357-360): discover -> mask -> compress -> sparse attention.
 * idx / counts are nullable (returned to the host only when given). */
int fpb_host_prefill(const fpb_problem* p, fpb_dtype dtype, const void* Q, const void* K,
                     const void* V, fpb_dtype out_dtype, void* out, float* lse, int32_t* idx,
                     int32_t* counts, unsigned long long* visits);

#ifdef __cplusplus
}
#endif
#endif /* FPB200_H */
