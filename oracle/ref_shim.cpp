// ref_shim.cpp — extern "C" shim over the UNMODIFIED reference headers (TEST INFRASTRUCTURE).
//
// Compiled by oracle/Makefile against /root/reference/proj/include into oracle/_ref/
// (git-ignored, travels to the GPU box as a prebuilt .so).  It lets the Python tests and
// bench.py's reference arm call the reference's own bsattn:: functions with plain pointers:
// inputs are copied into bsattn::Tensor, the reference function runs, outputs are copied out.
// No reference source is copied into this repository.
#include <atomic>
#include <chrono>
#include <cstring>
#include <thread>
#include <vector>

#include "bsattn/attention.hpp"
#include "bsattn/discovery.hpp"
#include "bsattn/selection.hpp"
#include "bsattn/tensor.hpp"
#include "bsattn/workloads.hpp"

using namespace bsattn;

namespace {

Tensor<float> make4(const float* p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  Tensor<float> t({a, b, c, d});
  std::memcpy(t.data(), p, sizeof(float) * t.numel());
  return t;
}

SequenceBatch batch(const float* p, uint64_t Z, uint64_t H, uint64_t L, uint64_t d, Role role) {
  return make_sequence_batch(make4(p, Z, H, L, d), role);
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const PlanError&) {
    return 2;
  } catch (const ValidationError&) {
    return 2;
  } catch (const FormatError&) {
    return 3;
  } catch (const IoError&) {
    return 3;
  } catch (...) {
    return 1;
  }
}

}  // namespace

extern "C" {

int ref_pool_keys(const float* k, uint64_t Z, uint64_t H, uint64_t L, uint64_t d, uint32_t B,
                  float* pooled) {
  return guarded([&] {
    const auto kb = batch(k, Z, H, L, d, Role::kKey);
    const auto p = pool_keys(kb, make_block_grid(L, B));
    std::memcpy(pooled, p.data.data(), sizeof(float) * p.data.numel());
  });
}

int ref_discover(const float* q, const float* k, uint64_t Z, uint64_t H, uint64_t L, uint64_t d,
                 uint32_t B, float tau, float eps, float* energy, float* local_max, float* score) {
  return guarded([&] {
    const auto qb = batch(q, Z, H, L, d, Role::kQuery);
    const auto kb = batch(k, Z, H, L, d, Role::kKey);
    const auto map = discover(qb, kb, make_block_grid(L, B), tau, eps);
    const size_t n = map.score.numel();
    std::memcpy(energy, map.energy.data(), sizeof(float) * n);
    std::memcpy(local_max, map.local_max.data(), sizeof(float) * n);
    std::memcpy(score, map.score.data(), sizeof(float) * n);
  });
}

int ref_max_threshold_mask(const float* score, uint64_t Z, uint64_t H, uint32_t M, uint32_t N,
                           uint32_t block_size, float alpha, uint32_t sink_tokens,
                           uint32_t window_tokens, float epsilon, uint8_t* mask,
                           uint64_t* comparisons) {
  return guarded([&] {
    PipelineConfig cfg;
    cfg.block_size = block_size;
    cfg.alpha = alpha;
    cfg.sink_tokens = sink_tokens;
    cfg.window_tokens = window_tokens;
    cfg.epsilon = epsilon;
    SelectionStats stats;
    const auto m = max_threshold_mask(make4(score, Z, H, M, N), cfg, &stats);
    std::memcpy(mask, m.active.data(), m.active.numel());
    if (comparisons) *comparisons += stats.score_comparisons;
  });
}

int ref_topk_select(const float* score, uint64_t Z, uint64_t H, uint32_t M, uint32_t k,
                    uint32_t block_size, uint32_t sink_tokens, uint32_t window_tokens,
                    uint8_t* mask) {
  return guarded([&] {
    PipelineConfig cfg;
    cfg.block_size = block_size;
    cfg.sink_tokens = sink_tokens;
    cfg.window_tokens = window_tokens;
    const auto m = topk_select(make4(score, Z, H, M, M), k, cfg);
    std::memcpy(mask, m.active.data(), m.active.numel());
  });
}

int ref_topp_select(const float* score, uint64_t Z, uint64_t H, uint32_t M, float p,
                    uint32_t block_size, uint32_t sink_tokens, uint32_t window_tokens,
                    uint8_t* mask) {
  return guarded([&] {
    PipelineConfig cfg;
    cfg.block_size = block_size;
    cfg.sink_tokens = sink_tokens;
    cfg.window_tokens = window_tokens;
    const auto m = topp_select(make4(score, Z, H, M, M), p, cfg);
    std::memcpy(mask, m.active.data(), m.active.numel());
  });
}

static int ref_discover_variant(int which, const float* q, const float* k, uint64_t Z, uint64_t H,
                                uint64_t L, uint64_t d, uint32_t B, float tau, float eps,
                                float* energy, float* local_max, float* score) {
  return guarded([&] {
    const auto qb = batch(q, Z, H, L, d, Role::kQuery);
    const auto kb = batch(k, Z, H, L, d, Role::kKey);
    const auto grid = make_block_grid(L, B);
    const auto map = which == 1 ? discover_pool_both(qb, kb, grid, tau, eps)
                                : discover_exact(qb, kb, grid, tau, eps);
    const size_t n = map.score.numel();
    std::memcpy(energy, map.energy.data(), sizeof(float) * n);
    std::memcpy(local_max, map.local_max.data(), sizeof(float) * n);
    std::memcpy(score, map.score.data(), sizeof(float) * n);
  });
}

int ref_discover_pool_both(const float* q, const float* k, uint64_t Z, uint64_t H, uint64_t L,
                           uint64_t d, uint32_t B, float tau, float eps, float* energy,
                           float* local_max, float* score) {
  return ref_discover_variant(1, q, k, Z, H, L, d, B, tau, eps, energy, local_max, score);
}

int ref_discover_exact(const float* q, const float* k, uint64_t Z, uint64_t H, uint64_t L,
                       uint64_t d, uint32_t B, float tau, float eps, float* energy,
                       float* local_max, float* score) {
  return ref_discover_variant(2, q, k, Z, H, L, d, B, tau, eps, energy, local_max, score);
}

int ref_compress_indices(const uint8_t* mask, uint64_t Z, uint32_t M, uint32_t N, uint64_t H,
                         int32_t* idx, int32_t* counts) {
  return guarded([&] {
    ActiveMask m{Tensor<std::uint8_t>({Z, M, N, H})};
    std::memcpy(m.active.data(), mask, m.active.numel());
    const auto plan = compress_indices(m);
    std::memcpy(idx, plan.indices.data(), sizeof(int32_t) * plan.indices.numel());
    std::memcpy(counts, plan.counts.data(), sizeof(int32_t) * plan.counts.numel());
  });
}

int ref_block_sparse_attention(const float* q, const float* k, const float* v, uint64_t Z,
                               uint64_t H, uint64_t L, uint64_t d, uint32_t B, const int32_t* idx,
                               const int32_t* counts, float tau, float* out, float* lse,
                               uint64_t* visits) {
  return guarded([&] {
    const BlockGrid grid = make_block_grid(L, B);
    const uint64_t M = grid.num_query_blocks, N = grid.num_key_blocks;
    SparseBlockPlan plan{Tensor<std::int32_t>({Z, M, N, H}), Tensor<std::int32_t>({Z, M, H})};
    std::memcpy(plan.indices.data(), idx, sizeof(int32_t) * plan.indices.numel());
    std::memcpy(plan.counts.data(), counts, sizeof(int32_t) * plan.counts.numel());
    AttentionStats stats;
    const auto res = block_sparse_attention(batch(q, Z, H, L, d, Role::kQuery),
                                            batch(k, Z, H, L, d, Role::kKey),
                                            batch(v, Z, H, L, d, Role::kValue), plan, grid, tau,
                                            &stats);
    std::memcpy(out, res.out.data(), sizeof(float) * res.out.numel());
    std::memcpy(lse, res.lse.data(), sizeof(float) * res.lse.numel());
    if (visits) *visits += stats.block_visits;
  });
}

int ref_dense_attention(const float* q, const float* k, const float* v, uint64_t Z, uint64_t H,
                        uint64_t L, uint64_t d, float tau, float* out, float* lse) {
  return guarded([&] {
    const auto res = dense_attention(batch(q, Z, H, L, d, Role::kQuery),
                                     batch(k, Z, H, L, d, Role::kKey),
                                     batch(v, Z, H, L, d, Role::kValue), tau);
    std::memcpy(out, res.out.data(), sizeof(float) * res.out.numel());
    std::memcpy(lse, res.lse.data(), sizeof(float) * res.lse.numel());
  });
}

int ref_generate_planted(int kind, float strength, int64_t target_a, int64_t target_b,
                         float base_noise, uint64_t seed, uint64_t Z, uint64_t H, uint64_t L,
                         uint64_t d, uint32_t B, float tau, float* q, float* k, float* v,
                         uint8_t* gt) {
  return guarded([&] {
    PlantedSpec spec;
    spec.pattern_kind = static_cast<PatternKind>(kind);
    spec.strength = strength;
    spec.target_a = target_a;
    spec.target_b = target_b;
    spec.base_noise = base_noise;
    spec.rng_seed = seed;
    const auto w = generate_planted(spec, Z, H, L, d, B, tau);
    const size_t n = w.q.data.numel();
    std::memcpy(q, w.q.data.data(), sizeof(float) * n);
    std::memcpy(k, w.k.data.data(), sizeof(float) * n);
    std::memcpy(v, w.v.data.data(), sizeof(float) * n);
    if (gt) std::memcpy(gt, w.ground_truth.active.data(), w.ground_truth.active.numel());
  });
}

// workloads.hpp:269-311 (pins the CLI's alt-slash generator, tools/cli/workloads.hpp)
int ref_generate_alternating_slash(float strength, int64_t offset, float base_noise, uint64_t seed,
                                   uint64_t Z, uint64_t H, uint64_t L, uint64_t d, uint32_t B,
                                   float tau, float* q, float* k, float* v, uint8_t* gt) {
  return guarded([&] {
    PlantedSpec spec;
    spec.pattern_kind = PatternKind::kSlash;
    spec.strength = strength;
    spec.target_a = offset;
    spec.base_noise = base_noise;
    spec.rng_seed = seed;
    const auto w = generate_alternating_slash(spec, Z, H, L, d, B, tau);
    const size_t n = w.q.data.numel();
    std::memcpy(q, w.q.data.data(), sizeof(float) * n);
    std::memcpy(k, w.k.data.data(), sizeof(float) * n);
    std::memcpy(v, w.v.data.data(), sizeof(float) * n);
    std::memcpy(gt, w.ground_truth.active.data(), w.ground_truth.active.numel());
  });
}

// workloads.hpp:378-399: score n x n, head_index n
int ref_heavy_tail_sweep_map(uint32_t n, float head_mass, float alpha, uint64_t seed, float* score,
                             int32_t* head_index) {
  return guarded([&] {
    const auto m = heavy_tail_sweep_map(n, head_mass, alpha, seed);
    std::memcpy(score, m.score.data(), sizeof(float) * m.score.numel());
    std::memcpy(head_index, m.head_index.data(), sizeof(int32_t) * n);
  });
}

// tensor.hpp save_tensor: the reference's FPT1 writer (pins the container bytes)
int ref_save_tensor_f32(const float* data, const uint64_t* shape, int ndim, const char* path) {
  return guarded([&] {
    Tensor<float> t(std::vector<std::uint64_t>(shape, shape + ndim));
    std::memcpy(t.data(), data, sizeof(float) * t.numel());
    save_tensor(t, path);
  });
}
int ref_save_tensor_i32(const int32_t* data, const uint64_t* shape, int ndim, const char* path) {
  return guarded([&] {
    Tensor<std::int32_t> t(std::vector<std::uint64_t>(shape, shape + ndim));
    std::memcpy(t.data(), data, sizeof(int32_t) * t.numel());
    save_tensor(t, path);
  });
}

// The reference pipeline (discover -> max_threshold_mask -> compress_indices ->
// block_sparse_attention, acceptance.cpp:357-360) per (z, h_q) slice on `threads` std::threads.
// GQA: each Q head is paired with its KV head's K/V slice.  Returns wall seconds, <0 on error.
double ref_pipeline_threads(const float* q, const float* k, const float* v, uint64_t Z,
                            uint64_t Hq, uint64_t Hkv, uint64_t L, uint64_t d, uint32_t B,
                            float alpha, uint32_t sink_tokens, uint32_t window_tokens, float tau,
                            float eps, const int32_t* head_list, int n_heads, int threads,
                            float* out, float* lse, uint64_t* visits) {
  PipelineConfig cfg;
  cfg.block_size = B;
  cfg.alpha = alpha;
  cfg.sink_tokens = sink_tokens;
  cfg.window_tokens = window_tokens;
  cfg.epsilon = eps;
  const BlockGrid grid = make_block_grid(L, B);
  const uint64_t Ld = L * d;
  // Inputs are wrapped once (outside the timed region) so the timing covers the pipeline only.
  std::vector<SequenceBatch> qs, ks, vs;
  for (int s = 0; s < n_heads; ++s) {
    const uint64_t zh = static_cast<uint64_t>(head_list[s]);
    const uint64_t z = zh / Hq, h = zh % Hq, kvh = z * Hkv + h / (Hq / Hkv);
    qs.push_back(batch(q + zh * Ld, 1, 1, L, d, Role::kQuery));
    ks.push_back(batch(k + kvh * Ld, 1, 1, L, d, Role::kKey));
    vs.push_back(batch(v + kvh * Ld, 1, 1, L, d, Role::kValue));
  }
  std::atomic<int> next{0}, err{0};
  std::atomic<uint64_t> vis_total{0};
  auto worker = [&] {
    for (;;) {
      const int s = next.fetch_add(1);
      if (s >= n_heads) break;
      const int rc = guarded([&] {
        const auto map = discover(qs[s], ks[s], grid, tau, eps);
        const auto mask = max_threshold_mask(map, cfg);
        const auto plan = compress_indices(mask);
        AttentionStats stats;
        const auto res = block_sparse_attention(qs[s], ks[s], vs[s], plan, grid, tau, &stats);
        std::memcpy(out + static_cast<uint64_t>(s) * Ld, res.out.data(), sizeof(float) * Ld);
        std::memcpy(lse + static_cast<uint64_t>(s) * L, res.lse.data(), sizeof(float) * L);
        vis_total += stats.block_visits;
      });
      if (rc) err = rc;
    }
  };
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int i = 0; i < (threads < 1 ? 1 : threads); ++i) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
  const double secs =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (visits) *visits = vis_total.load();
  return err ? -1.0 : secs;
}

// The same reference pipeline, also returning what the full-size parity tests compare: per sampled
// slice s the score map (M x N), the plan (idx M x N, counts M) exactly as compress_indices wrote
// them, and out / lse.  `row_keep` (M bytes, nullable) bounds the CPU cost at long L: before
// block_sparse_attention the counts of rows with row_keep[i] == 0 are set to 0 (the reference
// then writes NaN / -inf there, attention.hpp:119-126); the returned counts are the original ones.
double ref_pipeline_detail(const float* q, const float* k, const float* v, uint64_t Z,
                           uint64_t Hq, uint64_t Hkv, uint64_t L, uint64_t d, uint32_t B,
                           float alpha, uint32_t sink_tokens, uint32_t window_tokens, float tau,
                           float eps, const int32_t* head_list, int n_heads, int threads,
                           const uint8_t* row_keep, float* score, int32_t* idx, int32_t* counts,
                           uint64_t* comparisons, float* out, float* lse, uint64_t* visits) {
  PipelineConfig cfg;
  cfg.block_size = B;
  cfg.alpha = alpha;
  cfg.sink_tokens = sink_tokens;
  cfg.window_tokens = window_tokens;
  cfg.epsilon = eps;
  const BlockGrid grid = make_block_grid(L, B);
  const uint64_t Ld = L * d, MN = (uint64_t)grid.num_query_blocks * grid.num_key_blocks;
  const uint32_t M = grid.num_query_blocks;
  std::atomic<int> next{0}, err{0};
  std::atomic<uint64_t> vis_total{0}, cmp_total{0};
  auto worker = [&] {
    for (;;) {
      const int s = next.fetch_add(1);
      if (s >= n_heads) break;
      const int rc = guarded([&] {
        const uint64_t zh = static_cast<uint64_t>(head_list[s]);
        const uint64_t z = zh / Hq, h = zh % Hq, kvh = z * Hkv + h / (Hq / Hkv);
        const auto qs = batch(q + zh * Ld, 1, 1, L, d, Role::kQuery);
        const auto ks = batch(k + kvh * Ld, 1, 1, L, d, Role::kKey);
        const auto vs = batch(v + kvh * Ld, 1, 1, L, d, Role::kValue);
        const auto map = discover(qs, ks, grid, tau, eps);
        SelectionStats sst;
        const auto mask = max_threshold_mask(map, cfg, &sst);
        auto plan = compress_indices(mask);
        cmp_total += sst.score_comparisons;
        if (score) std::memcpy(score + s * MN, map.score.data(), sizeof(float) * MN);
        if (idx) std::memcpy(idx + s * MN, plan.indices.data(), sizeof(int32_t) * MN);
        if (counts) std::memcpy(counts + s * (uint64_t)M, plan.counts.data(), sizeof(int32_t) * M);
        if (row_keep)
          for (uint32_t i = 0; i < M; ++i)
            if (!row_keep[i]) plan.counts.data()[i] = 0;
        AttentionStats stats;
        const auto res = block_sparse_attention(qs, ks, vs, plan, grid, tau, &stats);
        if (out) std::memcpy(out + static_cast<uint64_t>(s) * Ld, res.out.data(), sizeof(float) * Ld);
        if (lse) std::memcpy(lse + static_cast<uint64_t>(s) * L, res.lse.data(), sizeof(float) * L);
        vis_total += stats.block_visits;
      });
      if (rc) err = rc;
    }
  };
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int i = 0; i < (threads < 1 ? 1 : threads); ++i) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
  const double secs =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (visits) *visits = vis_total.load();
  if (comparisons) *comparisons = cmp_total.load();
  return err ? -1.0 : secs;
}

}  // extern "C"
