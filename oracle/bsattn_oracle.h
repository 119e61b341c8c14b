/* bsattn_oracle.h — CPU restatement of the reference FlashPrefill hot path (TEST INFRASTRUCTURE).
 *
 * This is the parity oracle, not product code.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load it.  Every function restates one reference function
 * (file:line under /root/reference/proj/include/bsattn/) with the same arithmetic order, so the
 * oracle is bit-identical to the reference when both are built with the same flags
 * (gcc -O3, no -march, -ffp-contract=off); tests/test_oracle_golden.py pins that against
 * golden vectors produced by the reference itself (oracle/_ref).
 *
 * GQA generalisation (the reference has none): K/V carry Hkv heads and Q head h
 * reads KV head h / (Hq / Hkv).  With Hkv == Hq this is exactly the reference; otherwise it
 * equals calling the reference once per Q head with its KV head's slice.
 *
 * Layouts (row-major, identical to the reference):
 *   Q: Z x Hq x L x d   K, V: Z x Hkv x L x d   pooled: Z x Hkv x N x d
 *   energy / local_max / score: Z x Hq x M x N   mask: Z x M x N x Hq (u8)
 *   idx: Z x M x N x Hq (i32, fill N)   counts: Z x M x Hq (i32)
 *   out: Z x Hq x L x d   lse: Z x Hq x L (base 2)
 */
#ifndef BSATTN_ORACLE_H
#define BSATTN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_OK 0
#define OR_EVALIDATION 2 /* ValidationError / ConfigError / PlanError */

/* core.hpp:13-14 */
#define OR_LOG2E 1.4426950408889634f
#define OR_DEFAULT_EPS 1e-10f

typedef struct {
  uint32_t block_size, num_blocks, last_block_len;
} or_grid;

int or_make_grid(uint64_t L, uint32_t B, or_grid* g);                          /* core.hpp:31-41 */
float or_resolved_scale(float scale, uint64_t d);                              /* core.hpp:109-111 */
float or_dot_f32(const float* a, const float* b, uint64_t n);                  /* core.hpp:116-127 */

int or_pool_keys(const float* k, uint64_t Z, uint64_t Hkv, uint64_t L, uint64_t d, uint32_t B,
                 float* pooled);                                                /* discovery.hpp:39-70 */
int or_approx_block_scores(const float* q, const float* pooled, uint64_t Z, uint64_t Hq,
                           uint64_t Hkv, uint64_t L, uint64_t d, uint32_t B, float tau,
                           float* energy, float* local_max);                    /* discovery.hpp:75-115 */
int or_normalize_block_scores(const float* energy, const float* local_max, uint64_t Z,
                              uint64_t H, uint32_t M, float eps, float* score); /* discovery.hpp:119-148 */
int or_discover(const float* q, const float* k, uint64_t Z, uint64_t Hq, uint64_t Hkv, uint64_t L,
                uint64_t d, uint32_t B, float tau, float eps, float* energy, float* local_max,
                float* score);                                                  /* discovery.hpp:153-159 */

int or_max_threshold_mask(const float* score, uint64_t Z, uint64_t H, uint32_t M, uint32_t N,
                          uint32_t block_size, float alpha, uint32_t sink_tokens,
                          uint32_t window_tokens, float epsilon, uint8_t* mask,
                          uint64_t* comparisons);                               /* selection.hpp:63-92 */
int or_compress_indices(const uint8_t* mask, uint64_t Z, uint32_t M, uint32_t N, uint64_t H,
                        int32_t* idx, int32_t* counts);                         /* selection.hpp:176-192 */
uint64_t or_visit_count(const int32_t* counts, uint64_t n);                     /* selection.hpp:195-200 */
double or_density(const int32_t* counts, uint64_t Z, uint64_t H, uint32_t M);   /* selection.hpp:203-209 */

int or_block_sparse_attention(const float* q, const float* k, const float* v, uint64_t Z,
                              uint64_t Hq, uint64_t Hkv, uint64_t L, uint64_t d, uint32_t B,
                              const int32_t* idx, const int32_t* counts, float tau, float* out,
                              float* lse, uint64_t* visits);                    /* attention.hpp:38-132 */
int or_dense_attention(const float* q, const float* k, const float* v, uint64_t Z, uint64_t Hq,
                       uint64_t Hkv, uint64_t L, uint64_t d, float tau, float* out,
                       float* lse);                                             /* attention.hpp:135-174 */
int or_full_causal_plan(uint64_t Z, uint64_t H, uint32_t M, int32_t* idx,
                        int32_t* counts);                                       /* attention.hpp:178-192 */

/* Comparison baselines (not on the FlashPrefill path): selection.hpp:96-159, discovery.hpp:164-279 */
int or_topk_select(const float* score, uint64_t Z, uint64_t H, uint32_t M, uint32_t k,
                   uint32_t block_size, uint32_t sink_tokens, uint32_t window_tokens,
                   uint8_t* mask);
int or_topp_select(const float* score, uint64_t Z, uint64_t H, uint32_t M, float p,
                   uint32_t block_size, uint32_t sink_tokens, uint32_t window_tokens,
                   uint8_t* mask);
int or_discover_pool_both(const float* q, const float* k, uint64_t Z, uint64_t Hq, uint64_t Hkv,
                          uint64_t L, uint64_t d, uint32_t B, float tau, float eps, float* energy,
                          float* local_max, float* score);
int or_discover_exact(const float* q, const float* k, uint64_t Z, uint64_t Hq, uint64_t Hkv,
                      uint64_t L, uint64_t d, uint32_t B, float tau, float eps, float* energy,
                      float* local_max, float* score);

/* Head-parallel pipeline used as the CPU baseline: discover -> mask -> compress -> sparse attn
 * for the given (z, h) slices on `threads` POSIX threads.  Returns wall seconds. */
double or_pipeline_threads(const float* q, const float* k, const float* v, uint64_t Z, uint64_t Hq,
                           uint64_t Hkv, uint64_t L, uint64_t d, uint32_t B, float alpha,
                           uint32_t sink_tokens, uint32_t window_tokens, float tau, float eps,
                           const int32_t* head_list, int n_heads, int threads, float* out,
                           float* lse, uint64_t* visits);

/* workloads.hpp:16-46 — mt19937_64 + Box-Muller, and the planted generator (workloads.hpp:149-263)
 * used to feed the parity harness the reference's own synthetic inputs. */
int or_generate_planted(int kind, float strength, int64_t target_a, int64_t target_b,
                        float base_noise, uint64_t seed, uint64_t Z, uint64_t H, uint64_t L,
                        uint64_t d, uint32_t B, float tau, float* q, float* k, float* v,
                        uint8_t* ground_truth);
int or_random_batch(uint64_t n, uint64_t seed, float stddev, float* out); /* acceptance.cpp:29-35 */

#ifdef __cplusplus
}
#endif
#endif
