/* bsattn_oracle.c — CPU restatement of the reference FlashPrefill hot path.
 *
 * TEST INFRASTRUCTURE ONLY: this is the checker the CUDA path is compared against, and the
 * "port" CPU baseline.  It is never linked into the product library.
 *
 * Each function cites the reference function it restates (path:line under
 * /root/reference/proj/include/bsattn/).  Arithmetic order is kept exactly: the 4-lane
 * dot_f32, sequential fp32 row sums, exp2f/log2f from libm, multiply-by-reciprocal, and the
 * online-softmax update of attention.hpp.  Build with -O3 -ffp-contract=off and no -march so
 * that no FMA contraction happens (the reference's bits are pinned the same way).
 */
#include "bsattn_oracle.h"

#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define NEG_SENTINEL (-FLT_MAX) /* discovery.hpp:12, numeric_limits<float>::lowest() */

static inline float fmaxf_ref(float a, float b) { return (a < b) ? b : a; } /* std::max(a, b) */

/* core.hpp:31-41 */
int or_make_grid(uint64_t L, uint32_t B, or_grid* g) {
  if (L < 1 || B < 1) return OR_EVALIDATION;
  uint64_t blocks = (L + B - 1) / B;
  g->block_size = B;
  g->num_blocks = (uint32_t)blocks;
  g->last_block_len = (uint32_t)(L - (blocks - 1) * B);
  return OR_OK;
}

static inline uint32_t block_len(const or_grid* g, uint32_t blk) { /* core.hpp:23-25 */
  return blk + 1 == g->num_blocks ? g->last_block_len : g->block_size;
}

/* core.hpp:109-111 */
float or_resolved_scale(float scale, uint64_t d) {
  return scale > 0.0f ? scale : 1.0f / sqrtf((float)d);
}

/* core.hpp:116-127: four stride-4 partial sums, combined as (s0+s1)+(s2+s3). */
float or_dot_f32(const float* a, const float* b, uint64_t n) {
  float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f, s3 = 0.0f;
  uint64_t i = 0;
  for (; i + 4 <= n; i += 4) {
    s0 += a[i] * b[i];
    s1 += a[i + 1] * b[i + 1];
    s2 += a[i + 2] * b[i + 2];
    s3 += a[i + 3] * b[i + 3];
  }
  for (; i < n; ++i) s0 += a[i] * b[i];
  return (s0 + s1) + (s2 + s3);
}

/* discovery.hpp:39-59 (detail::pool_blocks): sequential row sum, then multiply by 1/len. */
int or_pool_keys(const float* k, uint64_t Z, uint64_t H, uint64_t L, uint64_t d, uint32_t B,
                 float* pooled) {
  or_grid g;
  if (or_make_grid(L, B, &g)) return OR_EVALIDATION;
  const uint32_t N = g.num_blocks;
  for (uint64_t zh = 0; zh < Z * H; ++zh) {
    const float* src = k + zh * L * d;
    float* dst = pooled + zh * N * d;
    for (uint32_t j = 0; j < N; ++j) {
      const uint32_t len = block_len(&g, j);
      float* out = dst + (uint64_t)j * d;
      for (uint64_t c = 0; c < d; ++c) out[c] = 0.0f;
      for (uint32_t r = 0; r < len; ++r) {
        const float* row = src + ((uint64_t)j * B + r) * d;
        for (uint64_t c = 0; c < d; ++c) out[c] += row[c];
      }
      const float inv = 1.0f / (float)len;
      for (uint64_t c = 0; c < d; ++c) out[c] *= inv;
    }
  }
  return OR_OK;
}

/* discovery.hpp:75-115: for every causal pair (I, J<=I): x_r = dot_f32(q_r, kbar_J) * to_bits,
 * m = max_r x_r (init kNegSentinel), S = sum_r exp2f(x_r - m) over the tile's real rows.
 * Non-causal entries hold energy 0 and local_max kNegSentinel (discovery.hpp:84). */
int or_approx_block_scores(const float* q, const float* pooled, uint64_t Z, uint64_t Hq,
                           uint64_t Hkv, uint64_t L, uint64_t d, uint32_t B, float tau,
                           float* energy, float* local_max) {
  or_grid g;
  if (or_make_grid(L, B, &g) || Hkv == 0 || Hq % Hkv) return OR_EVALIDATION;
  const uint32_t M = g.num_blocks, N = g.num_blocks;
  const uint64_t group = Hq / Hkv;
  const float to_bits = tau * OR_LOG2E;
  float* logits = (float*)malloc(sizeof(float) * B);
  for (uint64_t i = 0; i < Z * Hq * M * N; ++i) {
    energy[i] = 0.0f;
    local_max[i] = NEG_SENTINEL;
  }
  for (uint64_t z = 0; z < Z; ++z)
    for (uint64_t h = 0; h < Hq; ++h) {
      const float* qbase = q + (z * Hq + h) * L * d;
      const float* kbase = pooled + (z * Hkv + h / group) * N * d;
      float* en = energy + (z * Hq + h) * M * N;
      float* lm = local_max + (z * Hq + h) * M * N;
      for (uint32_t qi = 0; qi < M; ++qi) {
        const uint32_t rows = block_len(&g, qi);
        const float* tile = qbase + (uint64_t)qi * B * d;
        for (uint32_t kj = 0; kj <= qi; ++kj) {
          const float* kbar = kbase + (uint64_t)kj * d;
          float m = NEG_SENTINEL;
          for (uint32_t r = 0; r < rows; ++r) {
            const float x = or_dot_f32(tile + (uint64_t)r * d, kbar, d) * to_bits;
            logits[r] = x;
            m = fmaxf_ref(m, x);
          }
          float s = 0.0f;
          for (uint32_t r = 0; r < rows; ++r) s += exp2f(logits[r] - m);
          en[(uint64_t)qi * N + kj] = s;
          lm[(uint64_t)qi * N + kj] = m;
        }
      }
    }
  free(logits);
  return OR_OK;
}

/* discovery.hpp:119-148: row max of local maxima, S' = S * exp2f(m - M_I), sequential total,
 * score = S' * (1 / (total + eps)); score = 0 for J > I. */
int or_normalize_block_scores(const float* energy, const float* local_max, uint64_t Z,
                              uint64_t H, uint32_t M, float eps, float* score) {
  const uint32_t N = M;
  for (uint64_t i = 0; i < Z * H * M * N; ++i) score[i] = 0.0f;
  for (uint64_t zh = 0; zh < Z * H; ++zh) {
    const float* en = energy + zh * M * N;
    const float* lm = local_max + zh * M * N;
    float* dst = score + zh * M * N;
    for (uint32_t qi = 0; qi < M; ++qi) {
      const uint64_t row = (uint64_t)qi * N;
      float row_max = NEG_SENTINEL;
      for (uint32_t kj = 0; kj <= qi; ++kj) row_max = fmaxf_ref(row_max, lm[row + kj]);
      float total = 0.0f;
      for (uint32_t kj = 0; kj <= qi; ++kj) {
        const float rescaled = en[row + kj] * exp2f(lm[row + kj] - row_max);
        dst[row + kj] = rescaled;
        total += rescaled;
      }
      const float inv = 1.0f / (total + eps);
      for (uint32_t kj = 0; kj <= qi; ++kj) dst[row + kj] *= inv;
    }
  }
  return OR_OK;
}

/* discovery.hpp:153-159 */
int or_discover(const float* q, const float* k, uint64_t Z, uint64_t Hq, uint64_t Hkv, uint64_t L,
                uint64_t d, uint32_t B, float tau, float eps, float* energy, float* local_max,
                float* score) {
  or_grid g;
  if (or_make_grid(L, B, &g) || Hkv == 0 || Hq % Hkv) return OR_EVALIDATION;
  float* pooled = (float*)malloc(sizeof(float) * Z * Hkv * g.num_blocks * d);
  int rc = or_pool_keys(k, Z, Hkv, L, d, B, pooled);
  if (!rc) rc = or_approx_block_scores(q, pooled, Z, Hq, Hkv, L, d, B, tau, energy, local_max);
  if (!rc) rc = or_normalize_block_scores(energy, local_max, Z, Hq, g.num_blocks, eps, score);
  free(pooled);
  return rc;
}

/* selection.hpp:63-92 with PipelineConfig::validate / sink_blocks / window_blocks
 * (core.hpp:96-108) and detail::structural (selection.hpp:53-56). */
int or_max_threshold_mask(const float* score, uint64_t Z, uint64_t H, uint32_t M, uint32_t N,
                          uint32_t block_size, float alpha, uint32_t sink_tokens,
                          uint32_t window_tokens, float epsilon, uint8_t* mask,
                          uint64_t* comparisons) {
  if (block_size < 1 || !(alpha >= 0.0f) || window_tokens < 1 || !(epsilon > 0.0f))
    return OR_EVALIDATION;
  const uint32_t sink = (sink_tokens + block_size - 1) / block_size;
  const uint32_t window = (window_tokens + block_size - 1) / block_size;
  uint64_t cmp = 0;
  memset(mask, 0, Z * M * N * H);
  for (uint64_t z = 0; z < Z; ++z)
    for (uint64_t h = 0; h < H; ++h) {
      const float* srow = score + (z * H + h) * M * N;
      for (uint32_t i = 0; i < M; ++i) {
        float max_val = 0.0f;
        for (uint32_t j = 0; j <= i; ++j) {
          max_val = fmaxf_ref(max_val, srow[(uint64_t)i * N + j]);
          ++cmp;
        }
        const float thresh = alpha * max_val;
        for (uint32_t j = 0; j <= i; ++j) {
          const int by_score = srow[(uint64_t)i * N + j] >= thresh;
          ++cmp;
          if (by_score || j < sink || (i - j) < window)
            mask[((z * M + i) * N + j) * H + h] = 1;
        }
      }
    }
  if (comparisons) *comparisons += cmp;
  return OR_OK;
}

/* selection.hpp:176-192: ascending active j into slots, fill value N, counts. */
int or_compress_indices(const uint8_t* mask, uint64_t Z, uint32_t M, uint32_t N, uint64_t H,
                        int32_t* idx, int32_t* counts) {
  for (uint64_t i = 0; i < Z * M * N * H; ++i) idx[i] = (int32_t)N;
  for (uint64_t z = 0; z < Z; ++z)
    for (uint64_t i = 0; i < M; ++i)
      for (uint64_t h = 0; h < H; ++h) {
        int32_t count = 0;
        for (uint64_t j = 0; j < N; ++j)
          if (mask[((z * M + i) * N + j) * H + h])
            idx[((z * M + i) * N + (uint64_t)(count++)) * H + h] = (int32_t)j;
        counts[(z * M + i) * H + h] = count;
      }
  return OR_OK;
}

/* selection.hpp:195-200 */
uint64_t or_visit_count(const int32_t* counts, uint64_t n) {
  uint64_t total = 0;
  for (uint64_t i = 0; i < n; ++i) total += (uint64_t)counts[i];
  return total;
}

/* selection.hpp:203-209 */
double or_density(const int32_t* counts, uint64_t Z, uint64_t H, uint32_t M) {
  const double pairs = (double)Z * (double)H * ((double)M * (M + 1) / 2.0);
  return (double)or_visit_count(counts, Z * M * H) / pairs;
}

/* attention.hpp:38-132 for one (z, h) slice; returns OR_EVALIDATION on a PlanError. */
static int sparse_slice(const float* qbase, const float* kbase, const float* vbase, uint64_t L,
                        uint64_t d, const or_grid* g, const int32_t* idx, const int32_t* counts,
                        uint64_t z, uint64_t h, uint64_t H, float to_bits, float* obase,
                        float* lbase, float* run_max, float* run_sum, float* acc, float* logits,
                        uint64_t* visits) {
  const uint32_t M = g->num_blocks, N = g->num_blocks, B = g->block_size;
  (void)L;
  for (uint32_t qi = 0; qi < M; ++qi) {
    const uint32_t rows = block_len(g, qi);
    const float* tile = qbase + (uint64_t)qi * B * d;
    for (uint32_t r = 0; r < rows; ++r) {
      run_max[r] = -INFINITY;
      run_sum[r] = 0.0f;
    }
    for (uint64_t c = 0; c < (uint64_t)rows * d; ++c) acc[c] = 0.0f;
    const int32_t active = counts[(z * M + qi) * H + h];
    for (int32_t slot = 0; slot < active; ++slot) {
      const int32_t bid = idx[((z * M + qi) * N + (uint64_t)slot) * H + h];
      if (bid < 0 || bid >= (int32_t)N) return OR_EVALIDATION; /* attention.hpp:78-81 */
      ++*visits;
      const uint32_t kj = (uint32_t)bid;
      const uint32_t cols = block_len(g, kj);
      const int is_diag = kj == qi;
      const float* kblk = kbase + (uint64_t)kj * B * d;
      const float* vblk = vbase + (uint64_t)kj * B * d;
      for (uint32_t r = 0; r < rows; ++r) {
        const uint32_t cols_r = is_diag ? (cols < r + 1 ? cols : r + 1) : cols;
        const float* qrow = tile + (uint64_t)r * d;
        float m_new = run_max[r];
        float logits_max = -INFINITY;
        float block_sum = 0.0f;
        float* acc_row = acc + (uint64_t)r * d;
        for (uint32_t c = 0; c < cols_r; ++c) {
          logits[c] = or_dot_f32(qrow, kblk + (uint64_t)c * d, d) * to_bits;
          logits_max = fmaxf_ref(logits_max, logits[c]);
        }
        m_new = fmaxf_ref(m_new, logits_max);
        const float rescale = run_max[r] == -INFINITY ? 0.0f : exp2f(run_max[r] - m_new);
        for (uint64_t c = 0; c < d; ++c) acc_row[c] *= rescale;
        for (uint32_t c = 0; c < cols_r; ++c) {
          const float w = exp2f(logits[c] - m_new);
          block_sum += w;
          const float* vrow = vblk + (uint64_t)c * d;
          for (uint64_t cc = 0; cc < d; ++cc) acc_row[cc] += w * vrow[cc];
        }
        run_sum[r] = run_sum[r] * rescale + block_sum;
        run_max[r] = m_new;
      }
    }
    for (uint32_t r = 0; r < rows; ++r) {
      const uint64_t t = (uint64_t)qi * B + r;
      const float inv = 1.0f / run_sum[r];
      const float* acc_row = acc + (uint64_t)r * d;
      float* orow = obase + t * d;
      for (uint64_t c = 0; c < d; ++c) orow[c] = acc_row[c] * inv;
      lbase[t] = run_max[r] + log2f(run_sum[r]);
    }
  }
  return OR_OK;
}

int or_block_sparse_attention(const float* q, const float* k, const float* v, uint64_t Z,
                              uint64_t Hq, uint64_t Hkv, uint64_t L, uint64_t d, uint32_t B,
                              const int32_t* idx, const int32_t* counts, float tau, float* out,
                              float* lse, uint64_t* visits) {
  or_grid g;
  if (or_make_grid(L, B, &g) || Hkv == 0 || Hq % Hkv) return OR_EVALIDATION;
  const uint64_t group = Hq / Hkv;
  const float to_bits = tau * OR_LOG2E;
  float* run_max = (float*)malloc(sizeof(float) * B);
  float* run_sum = (float*)malloc(sizeof(float) * B);
  float* acc = (float*)malloc(sizeof(float) * B * d);
  float* logits = (float*)malloc(sizeof(float) * B);
  uint64_t vis = 0;
  int rc = OR_OK;
  for (uint64_t i = 0; i < Z * Hq * L * d; ++i) out[i] = 0.0f;
  for (uint64_t i = 0; i < Z * Hq * L; ++i) lse[i] = 0.0f;
  for (uint64_t z = 0; z < Z && !rc; ++z)
    for (uint64_t h = 0; h < Hq && !rc; ++h) {
      const uint64_t kvh = z * Hkv + h / group;
      rc = sparse_slice(q + (z * Hq + h) * L * d, k + kvh * L * d, v + kvh * L * d, L, d, &g, idx,
                        counts, z, h, Hq, to_bits, out + (z * Hq + h) * L * d,
                        lse + (z * Hq + h) * L, run_max, run_sum, acc, logits, &vis);
    }
  free(run_max);
  free(run_sum);
  free(acc);
  free(logits);
  if (visits) *visits += vis;
  return rc;
}

/* attention.hpp:135-174: exact causal base-2 softmax, one logit row at a time. */
int or_dense_attention(const float* q, const float* k, const float* v, uint64_t Z, uint64_t Hq,
                       uint64_t Hkv, uint64_t L, uint64_t d, float tau, float* out, float* lse) {
  if (Hkv == 0 || Hq % Hkv) return OR_EVALIDATION;
  const uint64_t group = Hq / Hkv;
  const float to_bits = tau * OR_LOG2E;
  float* logits = (float*)malloc(sizeof(float) * L);
  for (uint64_t i = 0; i < Z * Hq * L * d; ++i) out[i] = 0.0f;
  for (uint64_t z = 0; z < Z; ++z)
    for (uint64_t h = 0; h < Hq; ++h) {
      const float* qbase = q + (z * Hq + h) * L * d;
      const float* kbase = k + (z * Hkv + h / group) * L * d;
      const float* vbase = v + (z * Hkv + h / group) * L * d;
      float* obase = out + (z * Hq + h) * L * d;
      float* lbase = lse + (z * Hq + h) * L;
      for (uint64_t t = 0; t < L; ++t) {
        const float* qrow = qbase + t * d;
        float m = -INFINITY;
        for (uint64_t s = 0; s <= t; ++s) {
          logits[s] = or_dot_f32(qrow, kbase + s * d, d) * to_bits;
          m = fmaxf_ref(m, logits[s]);
        }
        float total = 0.0f;
        float* orow = obase + t * d;
        for (uint64_t s = 0; s <= t; ++s) {
          const float w = exp2f(logits[s] - m);
          total += w;
          const float* vrow = vbase + s * d;
          for (uint64_t c = 0; c < d; ++c) orow[c] += w * vrow[c];
        }
        const float inv = 1.0f / total;
        for (uint64_t c = 0; c < d; ++c) orow[c] *= inv;
        lbase[t] = m + log2f(total);
      }
    }
  free(logits);
  return OR_OK;
}

/* attention.hpp:178-192 */
int or_full_causal_plan(uint64_t Z, uint64_t H, uint32_t M, int32_t* idx, int32_t* counts) {
  const uint32_t N = M;
  for (uint64_t i = 0; i < Z * M * N * H; ++i) idx[i] = (int32_t)N;
  for (uint64_t z = 0; z < Z; ++z)
    for (uint64_t i = 0; i < M; ++i)
      for (uint64_t h = 0; h < H; ++h) {
        for (uint64_t j = 0; j <= i; ++j) idx[((z * M + i) * N + j) * H + h] = (int32_t)j;
        counts[(z * M + i) * H + h] = (int32_t)(i + 1);
      }
  return OR_OK;
}

/* ------------------------------------------------------------------------------------------
 * Comparison baselines.  std::stable_sort(order, row[a] > row[b]) == sort by (score desc,
 * index asc); restated with qsort on (score, index) pairs. */
typedef struct {
  float s;
  uint32_t j;
} or_pair;

static int pair_cmp(const void* a, const void* b) {
  const or_pair* x = (const or_pair*)a;
  const or_pair* y = (const or_pair*)b;
  if (x->s > y->s) return -1;
  if (y->s > x->s) return 1;
  return (x->j < y->j) ? -1 : (x->j > y->j);
}

static int sort_select(const float* score, uint64_t Z, uint64_t H, uint32_t M, int mode,
                       uint32_t k, float p, uint32_t B, uint32_t sink_tokens,
                       uint32_t window_tokens, uint8_t* mask) {
  if (B < 1 || window_tokens < 1) return OR_EVALIDATION; /* PipelineConfig::validate */
  if (mode == 0 && k < 1) return OR_EVALIDATION;         /* selection.hpp:98 */
  if (mode == 1 && (!(p > 0.0f) || p > 1.0f)) return OR_EVALIDATION; /* selection.hpp:128 */
  const uint32_t sink = (sink_tokens + B - 1) / B, window = (window_tokens + B - 1) / B;
  const uint32_t N = M;
  or_pair* order = (or_pair*)malloc(sizeof(or_pair) * M);
  memset(mask, 0, Z * M * N * H);
  for (uint64_t z = 0; z < Z; ++z)
    for (uint64_t h = 0; h < H; ++h) {
      const float* srow = score + (z * H + h) * M * N;
      for (uint32_t i = 0; i < M; ++i) {
        const float* row = srow + (uint64_t)i * N;
        for (uint32_t j = 0; j <= i; ++j) {
          order[j].s = row[j];
          order[j].j = j;
        }
        qsort(order, i + 1, sizeof(or_pair), pair_cmp);
        if (mode == 0) { /* selection.hpp:114-115 */
          const uint32_t take = k < i + 1 ? k : i + 1;
          for (uint32_t r = 0; r < take; ++r) mask[((z * M + i) * N + order[r].j) * H + h] = 1;
        } else { /* selection.hpp:144-152 */
          double total = 0.0;
          for (uint32_t j = 0; j <= i; ++j) total += row[j];
          double cumulative = 0.0;
          for (uint32_t r = 0; r <= i; ++r) {
            if (total <= 0.0 || order[r].s <= 0.0f) break;
            mask[((z * M + i) * N + order[r].j) * H + h] = 1;
            cumulative += order[r].s / total;
            if (cumulative >= (double)p - 1e-9) break;
          }
        }
        for (uint32_t j = 0; j <= i; ++j)
          if (j < sink || (i - j) < window) mask[((z * M + i) * N + j) * H + h] = 1;
      }
    }
  free(order);
  return OR_OK;
}

int or_topk_select(const float* score, uint64_t Z, uint64_t H, uint32_t M, uint32_t k,
                   uint32_t block_size, uint32_t sink_tokens, uint32_t window_tokens,
                   uint8_t* mask) {
  return sort_select(score, Z, H, M, 0, k, 0.f, block_size, sink_tokens, window_tokens, mask);
}

int or_topp_select(const float* score, uint64_t Z, uint64_t H, uint32_t M, float p,
                   uint32_t block_size, uint32_t sink_tokens, uint32_t window_tokens,
                   uint8_t* mask) {
  return sort_select(score, Z, H, M, 1, 1, p, block_size, sink_tokens, window_tokens, mask);
}

/* discovery.hpp:164-195 */
int or_discover_pool_both(const float* q, const float* k, uint64_t Z, uint64_t Hq, uint64_t Hkv,
                          uint64_t L, uint64_t d, uint32_t B, float tau, float eps, float* energy,
                          float* local_max, float* score) {
  or_grid g;
  if (or_make_grid(L, B, &g) || Hkv == 0 || Hq % Hkv) return OR_EVALIDATION;
  const uint32_t M = g.num_blocks, N = M;
  const uint64_t group = Hq / Hkv;
  const float to_bits = tau * OR_LOG2E;
  float* pq = (float*)malloc(sizeof(float) * Z * Hq * M * d);
  float* pk = (float*)malloc(sizeof(float) * Z * Hkv * M * d);
  or_pool_keys(q, Z, Hq, L, d, B, pq); /* detail::pool_blocks on the queries */
  or_pool_keys(k, Z, Hkv, L, d, B, pk);
  for (uint64_t i = 0; i < Z * Hq * M * N; ++i) {
    energy[i] = 0.0f;
    local_max[i] = NEG_SENTINEL;
  }
  for (uint64_t z = 0; z < Z; ++z)
    for (uint64_t h = 0; h < Hq; ++h) {
      const float* qb = pq + (z * Hq + h) * M * d;
      const float* kb = pk + (z * Hkv + h / group) * N * d;
      float* en = energy + (z * Hq + h) * M * N;
      float* lm = local_max + (z * Hq + h) * M * N;
      for (uint32_t qi = 0; qi < M; ++qi)
        for (uint32_t kj = 0; kj <= qi; ++kj) {
          lm[(uint64_t)qi * N + kj] =
              or_dot_f32(qb + (uint64_t)qi * d, kb + (uint64_t)kj * d, d) * to_bits;
          en[(uint64_t)qi * N + kj] = 1.0f;
        }
    }
  free(pq);
  free(pk);
  return or_normalize_block_scores(energy, local_max, Z, Hq, M, eps, score);
}

/* discovery.hpp:201-279 */
int or_discover_exact(const float* q, const float* k, uint64_t Z, uint64_t Hq, uint64_t Hkv,
                      uint64_t L, uint64_t d, uint32_t B, float tau, float eps, float* energy,
                      float* local_max, float* score) {
  or_grid g;
  if (or_make_grid(L, B, &g) || Hkv == 0 || Hq % Hkv) return OR_EVALIDATION;
  const uint32_t M = g.num_blocks, N = M;
  const uint64_t group = Hq / Hkv;
  const float to_bits = tau * OR_LOG2E;
  float* pk = (float*)malloc(sizeof(float) * Z * Hkv * N * d);
  or_pool_keys(k, Z, Hkv, L, d, B, pk);
  float* table = (float*)malloc(sizeof(float) * L * N);
  for (uint64_t i = 0; i < Z * Hq * M * N; ++i) {
    energy[i] = 0.0f;
    local_max[i] = NEG_SENTINEL;
    score[i] = 0.0f;
  }
  for (uint64_t z = 0; z < Z; ++z)
    for (uint64_t h = 0; h < Hq; ++h) {
      const float* qbase = q + (z * Hq + h) * L * d;
      const float* kbase = pk + (z * Hkv + h / group) * N * d;
      for (uint64_t t = 0; t < L; ++t) { /* pass 1: discovery.hpp:222-229 */
        const uint32_t visible = (uint32_t)(t / B);
        float* row = table + t * N;
        for (uint32_t kj = 0; kj < N; ++kj)
          row[kj] = kj <= visible ? or_dot_f32(qbase + t * d, kbase + (uint64_t)kj * d, d) * to_bits
                                  : NEG_SENTINEL;
      }
      float* en = energy + (z * Hq + h) * M * N;
      float* lm = local_max + (z * Hq + h) * M * N;
      for (uint32_t qi = 0; qi < M; ++qi) { /* discovery.hpp:235-248 */
        const uint32_t rows = block_len(&g, qi);
        for (uint32_t kj = 0; kj <= qi; ++kj) {
          float m = NEG_SENTINEL;
          for (uint32_t r = 0; r < rows; ++r)
            m = fmaxf_ref(m, table[((uint64_t)qi * B + r) * N + kj]);
          float s = 0.0f;
          for (uint32_t r = 0; r < rows; ++r) s += exp2f(table[((uint64_t)qi * B + r) * N + kj] - m);
          lm[(uint64_t)qi * N + kj] = m;
          en[(uint64_t)qi * N + kj] = s;
        }
      }
      for (uint64_t t = 0; t < L; ++t) { /* pass 2: discovery.hpp:251-263 */
        const uint32_t visible = (uint32_t)(t / B);
        float* row = table + t * N;
        float m = NEG_SENTINEL;
        for (uint32_t kj = 0; kj <= visible; ++kj) m = fmaxf_ref(m, row[kj]);
        float total = 0.0f;
        for (uint32_t kj = 0; kj <= visible; ++kj) {
          row[kj] = exp2f(row[kj] - m);
          total += row[kj];
        }
        const float inv = 1.0f / (total + eps);
        for (uint32_t kj = 0; kj <= visible; ++kj) row[kj] *= inv;
      }
      float* dst = score + (z * Hq + h) * M * N;
      for (uint32_t qi = 0; qi < M; ++qi) { /* discovery.hpp:265-274 */
        const uint32_t rows = block_len(&g, qi);
        const float inv_rows = 1.0f / (float)rows;
        for (uint32_t kj = 0; kj <= qi; ++kj) {
          float acc = 0.0f;
          for (uint32_t r = 0; r < rows; ++r) acc += table[((uint64_t)qi * B + r) * N + kj];
          dst[(uint64_t)qi * N + kj] = acc * inv_rows;
        }
      }
    }
  free(pk);
  free(table);
  return OR_OK;
}

/* ------------------------------------------------------------------------------------------
 * CPU baseline: the whole pipeline per (z, h) slice, slices spread over POSIX threads.
 * Per-slice calls are bit-identical to the batched reference call.           */
typedef struct {
  const float *q, *k, *v;
  uint64_t Z, Hq, Hkv, L, d;
  uint32_t B, sink, window;
  float alpha, tau, eps;
  const int32_t* heads;
  int n_heads;
  int next;
  pthread_mutex_t mu;
  float *out, *lse;
  uint64_t visits;
  int rc;
} pipe_job;

static void* pipe_worker(void* arg) {
  pipe_job* J = (pipe_job*)arg;
  or_grid g;
  or_make_grid(J->L, J->B, &g);
  const uint32_t M = g.num_blocks, N = g.num_blocks;
  const uint64_t MN = (uint64_t)M * N, Ld = J->L * J->d;
  float* en = (float*)malloc(sizeof(float) * MN);
  float* lm = (float*)malloc(sizeof(float) * MN);
  float* sc = (float*)malloc(sizeof(float) * MN);
  uint8_t* mask = (uint8_t*)malloc(MN);
  int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * MN);
  int32_t* counts = (int32_t*)malloc(sizeof(int32_t) * M);
  for (;;) {
    pthread_mutex_lock(&J->mu);
    const int slot = J->next++;
    pthread_mutex_unlock(&J->mu);
    if (slot >= J->n_heads) break;
    const uint64_t zh = (uint64_t)J->heads[slot];
    const uint64_t z = zh / J->Hq, h = zh % J->Hq;
    const uint64_t kvh = z * J->Hkv + h / (J->Hq / J->Hkv);
    const float *q = J->q + zh * Ld, *k = J->k + kvh * Ld, *v = J->v + kvh * Ld;
    uint64_t vis = 0;
    int rc = or_discover(q, k, 1, 1, 1, J->L, J->d, J->B, J->tau, J->eps, en, lm, sc);
    if (!rc)
      rc = or_max_threshold_mask(sc, 1, 1, M, N, J->B, J->alpha, J->sink, J->window, J->eps, mask,
                                 NULL);
    if (!rc) rc = or_compress_indices(mask, 1, M, N, 1, idx, counts);
    if (!rc)
      rc = or_block_sparse_attention(q, k, v, 1, 1, 1, J->L, J->d, J->B, idx, counts, J->tau,
                                     J->out + (uint64_t)slot * Ld, J->lse + (uint64_t)slot * J->L,
                                     &vis);
    pthread_mutex_lock(&J->mu);
    J->visits += vis;
    if (rc) J->rc = rc;
    pthread_mutex_unlock(&J->mu);
  }
  free(en);
  free(lm);
  free(sc);
  free(mask);
  free(idx);
  free(counts);
  return NULL;
}

double or_pipeline_threads(const float* q, const float* k, const float* v, uint64_t Z, uint64_t Hq,
                           uint64_t Hkv, uint64_t L, uint64_t d, uint32_t B, float alpha,
                           uint32_t sink_tokens, uint32_t window_tokens, float tau, float eps,
                           const int32_t* head_list, int n_heads, int threads, float* out,
                           float* lse, uint64_t* visits) {
  pipe_job J;
  J.q = q; J.k = k; J.v = v; J.Z = Z; J.Hq = Hq; J.Hkv = Hkv; J.L = L; J.d = d; J.B = B;
  J.sink = sink_tokens; J.window = window_tokens; J.alpha = alpha; J.tau = tau; J.eps = eps;
  J.heads = head_list; J.n_heads = n_heads; J.next = 0; J.out = out; J.lse = lse;
  J.visits = 0; J.rc = 0;
  pthread_mutex_init(&J.mu, NULL);
  if (threads < 1) threads = 1;
  pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (int i = 0; i < threads; ++i) pthread_create(&tids[i], NULL, pipe_worker, &J);
  for (int i = 0; i < threads; ++i) pthread_join(tids[i], NULL);
  clock_gettime(CLOCK_MONOTONIC, &t1);
  free(tids);
  pthread_mutex_destroy(&J.mu);
  if (visits) *visits = J.visits;
  if (J.rc) return -1.0;
  return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}

/* ------------------------------------------------------------------------------------------
 * workloads.hpp:16-46 — std::mt19937_64 and the hand-rolled Box-Muller Rng. */
typedef struct {
  uint64_t mt[312];
  int idx;
  double spare;
  int have_spare;
} or_rng;

static void rng_seed(or_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
  r->have_spare = 0;
  r->spare = 0.0;
}

static uint64_t rng_next(or_rng* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

static double rng_uniform(or_rng* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }

static double rng_gaussian(or_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = rng_uniform(r);
  if (u1 <= 0.0) u1 = 0x1.0p-53;
  const double u2 = rng_uniform(r);
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = 6.283185307179586 * u2;
  r->spare = radius * sin(angle);
  r->have_spare = 1;
  return radius * cos(angle);
}

static float rng_gaussian_f(or_rng* r, float stddev) { return (float)rng_gaussian(r) * stddev; }

/* acceptance.cpp:29-35 random_batch */
int or_random_batch(uint64_t n, uint64_t seed, float stddev, float* out) {
  or_rng r;
  rng_seed(&r, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = rng_gaussian_f(&r, stddev);
  return OR_OK;
}

/* workloads.hpp:82-101 */
static void unit_direction(or_rng* r, float* dst, uint64_t d) {
  double norm_sq = 0.0;
  for (uint64_t c = 0; c < d; ++c) {
    dst[c] = (float)rng_gaussian(r);
    norm_sq += (double)dst[c] * dst[c];
  }
  const float inv = (float)(1.0 / sqrt(norm_sq > 0.0 ? norm_sq : 1.0));
  for (uint64_t c = 0; c < d; ++c) dst[c] *= inv;
}
static void add_scaled(float* row, const float* dir, uint64_t d, float scale) {
  for (uint64_t c = 0; c < d; ++c) row[c] += scale * dir[c];
}

/* workloads.hpp:149-263 generate_planted; kind 0 vertical, 1 slash, 2 block, 3 needle.
 * ground_truth (nullable) is Z x M x M x H u8 (workloads.hpp:103-140). */
int or_generate_planted(int kind, float strength, int64_t target_a, int64_t target_b,
                        float base_noise, uint64_t seed, uint64_t Z, uint64_t H, uint64_t L,
                        uint64_t d, uint32_t B, float tau, float* q, float* k, float* v,
                        uint8_t* gt) {
  if (strength < 0.0f || base_noise < 0.0f) return OR_EVALIDATION;
  or_grid g;
  if (or_make_grid(L, B, &g)) return OR_EVALIDATION;
  const uint32_t M = g.num_blocks;
  if (tau <= 0.0f) tau = 1.0f / sqrtf((float)d);
  const float boost = strength / tau;
  or_rng r;
  rng_seed(&r, seed);
  const uint64_t n = Z * H * L * d;
  for (uint64_t i = 0; i < n; ++i) q[i] = rng_gaussian_f(&r, base_noise);
  for (uint64_t i = 0; i < n; ++i) k[i] = rng_gaussian_f(&r, base_noise);
  for (uint64_t i = 0; i < n; ++i) v[i] = rng_gaussian_f(&r, base_noise);
  if (gt) {
    memset(gt, 0, Z * M * M * H);
    for (uint64_t z = 0; z < Z; ++z)
      for (uint64_t i = 0; i < M; ++i)
        for (uint64_t h = 0; h < H; ++h) gt[((z * M + i) * M + i) * H + h] = 1;
  }
  float* dir = (float*)malloc(sizeof(float) * d);
  int rc = OR_OK;
  if (strength > 0.0f) {
    if (kind == 0) { /* vertical */
      const int64_t col = target_a;
      if (col < 0 || col >= (int64_t)M) { rc = OR_EVALIDATION; goto done; }
      for (uint64_t zh = 0; zh < Z * H; ++zh) {
        unit_direction(&r, dir, d);
        float* qs = q + zh * L * d;
        float* ks = k + zh * L * d;
        for (uint64_t t = 0; t < L; ++t) add_scaled(qs + t * d, dir, d, boost);
        const uint64_t lo = (uint64_t)col * B, hi = lo + B < L ? lo + B : L;
        for (uint64_t s = lo; s < hi; ++s) add_scaled(ks + s * d, dir, d, 1.0f);
      }
      if (gt)
        for (uint64_t z = 0; z < Z; ++z)
          for (uint64_t i = (uint64_t)col; i < M; ++i)
            for (uint64_t h = 0; h < H; ++h) gt[((z * M + i) * M + (uint64_t)col) * H + h] = 1;
    } else if (kind == 1) { /* slash */
      const int64_t offset = target_a;
      if (offset < 1 || offset >= (int64_t)L) { rc = OR_EVALIDATION; goto done; }
      float* dirs = (float*)malloc(sizeof(float) * M * d);
      for (uint64_t zh = 0; zh < Z * H; ++zh) {
        for (uint32_t i = 0; i < M; ++i) unit_direction(&r, dirs + (uint64_t)i * d, d);
        float* qs = q + zh * L * d;
        float* ks = k + zh * L * d;
        for (uint64_t t = 0; t < L; ++t) add_scaled(qs + t * d, dirs + (t / B) * d, d, boost);
        for (uint64_t t = (uint64_t)offset; t < L; ++t)
          add_scaled(ks + (t - (uint64_t)offset) * d, dirs + (t / B) * d, d, 1.0f);
      }
      free(dirs);
      if (gt) /* workloads.hpp:116-129 mark_slash_rows */
        for (uint32_t i = 0; i < M; ++i) {
          const uint64_t t_lo = (uint64_t)i * B;
          const uint64_t t_hi = (t_lo + B < L ? t_lo + B : L) - 1;
          if (t_hi < (uint64_t)offset) continue;
          const uint32_t j_lo = (uint32_t)((t_lo >= (uint64_t)offset ? t_lo - offset : 0) / B);
          const uint32_t j_hi = (uint32_t)((t_hi - offset) / B);
          for (uint32_t j = j_lo; j <= j_hi && j <= i; ++j)
            for (uint64_t z = 0; z < Z; ++z)
              for (uint64_t h = 0; h < H; ++h) gt[((z * M + i) * M + j) * H + h] = 1;
        }
    } else if (kind == 2) { /* block */
      const int64_t row = target_a, col = target_b;
      if (row < 0 || row >= (int64_t)M || col < 0 || col >= (int64_t)M || col > row) {
        rc = OR_EVALIDATION;
        goto done;
      }
      for (uint64_t zh = 0; zh < Z * H; ++zh) {
        unit_direction(&r, dir, d);
        float* qs = q + zh * L * d;
        float* ks = k + zh * L * d;
        const uint64_t q_lo = (uint64_t)row * B, q_hi = q_lo + B < L ? q_lo + B : L;
        for (uint64_t t = q_lo; t < q_hi; ++t) add_scaled(qs + t * d, dir, d, boost);
        const uint64_t k_lo = (uint64_t)col * B, k_hi = k_lo + B < L ? k_lo + B : L;
        for (uint64_t s = k_lo; s < k_hi; ++s) add_scaled(ks + s * d, dir, d, 1.0f);
      }
      if (gt)
        for (uint64_t z = 0; z < Z; ++z)
          for (uint64_t h = 0; h < H; ++h)
            gt[((z * M + (uint64_t)row) * M + (uint64_t)col) * H + h] = 1;
    } else if (kind == 3) { /* needle */
      const int64_t token = target_a;
      if (token < 0 || token >= (int64_t)L) { rc = OR_EVALIDATION; goto done; }
      const uint32_t col = (uint32_t)((uint64_t)token / B);
      const float row_weight = (float)block_len(&g, col);
      for (uint64_t zh = 0; zh < Z * H; ++zh) {
        unit_direction(&r, dir, d);
        float* qs = q + zh * L * d;
        float* ks = k + zh * L * d;
        for (uint64_t t = 0; t < L; ++t) add_scaled(qs + t * d, dir, d, boost);
        add_scaled(ks + (uint64_t)token * d, dir, d, row_weight);
      }
      if (gt)
        for (uint64_t z = 0; z < Z; ++z)
          for (uint64_t i = col; i < M; ++i)
            for (uint64_t h = 0; h < H; ++h) gt[((z * M + i) * M + col) * H + h] = 1;
    } else {
      rc = OR_EVALIDATION;
    }
  }
done:
  free(dir);
  return rc;
}
