// test_dropin.cpp — the reference's own unit-test expectations, restated against the C++ drop-in
// (include/fpb200/bsattn.hpp) so they read like proj/tests/test_*.cpp with `bsattn::` swapped
// for `fpb200::`.  Shapes are widened to the kernels' tile (d = 128, B = 128) by zero-padding
// channels, which leaves every dot product unchanged.  Needs a GPU; run by
// tests/test_gpu_dropin.py.  Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <random>
#include <set>

#include "fpb200/bsattn.hpp"

using namespace fpb200;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                       \
  do {                                                                    \
    ++g_checks;                                                           \
    if (!(cond)) {                                                        \
      ++g_fail;                                                           \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);         \
    }                                                                     \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                          \
  do {                                                                    \
    ++g_checks;                                                           \
    bool ok = false;                                                      \
    try {                                                                 \
      (void)(expr);                                                       \
    } catch (const T&) {                                                  \
      ok = true;                                                          \
    } catch (...) {                                                       \
    }                                                                     \
    if (!ok) {                                                            \
      ++g_fail;                                                           \
      std::printf("FAIL %s:%d: %s does not throw %s\n", __FILE__, __LINE__, #expr, #T); \
    }                                                                     \
  } while (0)

static bool approx(double a, double b, double tol) { return std::fabs(a - b) <= tol; }

static SequenceBatch random_batch(std::uint64_t Z, std::uint64_t H, std::uint64_t L, Role role,
                                  std::uint64_t seed) {
  std::mt19937_64 eng(seed);
  std::normal_distribution<float> n(0.0f, 1.0f);
  Tensor<float> t({Z, H, L, 128});
  for (std::size_t i = 0; i < t.numel(); ++i) t.data()[i] = n(eng);
  return make_sequence_batch(std::move(t), role);
}

int main() {
  // test_discovery.cpp:24-35 — pooling hand arithmetic (partial block of 2 tokens)
  {
    Tensor<float> k({1, 1, 2, 128}, 0.0f);
    k(0, 0, 0, 0) = 1.0f, k(0, 0, 0, 1) = 3.0f, k(0, 0, 1, 0) = 3.0f, k(0, 0, 1, 1) = 1.0f;
    const auto pooled = pool_keys(make_sequence_batch(std::move(k), Role::kKey), make_block_grid(2, 128));
    CHECK(pooled.data(0, 0, 0, 0) == 2.0f && pooled.data(0, 0, 0, 1) == 2.0f);
    CHECK(pooled.data(0, 0, 0, 2) == 0.0f);
    CHECK_THROWS_AS(pool_keys(random_batch(1, 1, 4, Role::kQuery, 1), make_block_grid(4, 128)),
                    ValidationError);
  }
  // test_discovery.cpp:70-89 — identical query rows: m = scaled logit, S = B
  {
    const std::uint32_t B = 128;
    Tensor<float> q({1, 1, B, 128}, 0.0f), k({1, 1, B, 128}, 0.0f);
    for (std::uint32_t r = 0; r < B; ++r) {
      q(0, 0, r, 0) = 1.0f, q(0, 0, r, 1) = -2.0f, q(0, 0, r, 2) = 0.5f;
      k(0, 0, r, 0) = 0.25f, k(0, 0, r, 1) = 1.0f, k(0, 0, r, 2) = -1.0f;
    }
    const float tau = 0.5f;
    const BlockGrid grid = make_block_grid(B, B);
    const auto pooled = pool_keys(make_sequence_batch(std::move(k), Role::kKey), grid);
    const auto e = approx_block_scores(make_sequence_batch(std::move(q), Role::kQuery), pooled, grid, tau);
    const float expected = (1.0f * 0.25f - 2.0f * 1.0f + 0.5f * -1.0f) * tau * kLog2e;
    CHECK(approx(e.local_max(0, 0, 0, 0), expected, 1e-5));
    CHECK(approx(e.energy(0, 0, 0, 0), 128.0, 1e-3));
  }
  // test_discovery.cpp:91-134 — sentinels and the energy bound on a ragged grid
  {
    const auto q = random_batch(1, 2, 300, Role::kQuery, 3);
    const auto k = random_batch(1, 2, 300, Role::kKey, 4);
    const BlockGrid grid = make_block_grid(300, 128);
    const auto m = discover(q, k, grid, 1.0f / std::sqrt(128.0f));
    for (std::uint64_t h = 0; h < 2; ++h)
      for (std::uint32_t i = 0; i < 3; ++i)
        for (std::uint32_t j = 0; j < 3; ++j) {
          if (j > i) {
            CHECK(m.energy(0, h, i, j) == 0.0f && m.local_max(0, h, i, j) == kNegSentinel);
            CHECK(m.score(0, h, i, j) == 0.0f);
          } else {
            const float s = m.energy(0, h, i, j);
            CHECK(s >= 1.0f - 1e-5f && s <= grid.block_len(i) * (1.0f + 1e-5f));
          }
        }
    // rows are normalised: sum = total / (total + eps) < 1
    for (std::uint32_t i = 0; i < 3; ++i) {
      double sum = 0;
      for (std::uint32_t j = 0; j <= i; ++j) sum += m.score(0, 0, i, j);
      CHECK(approx(sum, 1.0, 1e-5));
    }
  }
  // test_selection.cpp:59-75, 111-119 — hand enumeration, alpha limits, 2 comparisons per cell
  {
    Tensor<float> score({1, 1, 4, 4}, 0.0f);
    const float row[4] = {0.50f, 0.30f, 0.05f, 0.15f};
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j <= i; ++j) score(0, 0, i, j) = row[j];
    PipelineConfig cfg;
    cfg.sink_tokens = 0;
    cfg.window_tokens = 1;
    auto active = [&](const ActiveMask& m, int i) {
      std::set<int> s;
      for (int j = 0; j < 4; ++j)
        if (m.active(0, i, j, 0)) s.insert(j);
      return s;
    };
    cfg.alpha = 0.5f;
    SelectionStats st;
    CHECK(active(max_threshold_mask(score, cfg, &st), 3) == (std::set<int>{0, 1, 3}));
    CHECK(st.score_comparisons == 2 * 10);
    cfg.alpha = 0.0f;
    const auto all = max_threshold_mask(score, cfg);
    for (int i = 0; i < 4; ++i) CHECK(active(all, i).size() == static_cast<std::size_t>(i + 1));
    cfg.alpha = 1.0f;
    CHECK(active(max_threshold_mask(score, cfg), 3) == (std::set<int>{0, 3}));
    cfg.alpha = -1.0f;
    CHECK_THROWS_AS(max_threshold_mask(score, cfg), ConfigError);
  }
  // test_selection.cpp:123-139 — fill-and-compact
  {
    ActiveMask mask{Tensor<std::uint8_t>({1, 4, 4, 1}, 0)};
    mask.active(0, 0, 0, 0) = 1;
    mask.active(0, 0, 2, 0) = 1;
    const auto plan = compress_indices(mask);
    CHECK(plan.counts(0, 0, 0) == 2);
    CHECK(plan.indices(0, 0, 0, 0) == 0 && plan.indices(0, 0, 1, 0) == 2);
    CHECK(plan.indices(0, 0, 2, 0) == 4 && plan.indices(0, 0, 3, 0) == 4);
  }
  // test_attention.cpp:26-42 — two keys with equal logits average the values
  {
    Tensor<float> q({1, 1, 2, 128}, 0.0f), k({1, 1, 2, 128}, 0.0f), v({1, 1, 2, 128}, 0.0f);
    q(0, 0, 1, 0) = 1.0f;
    k(0, 0, 0, 1) = 1.0f;
    v(0, 0, 0, 0) = 1.0f;
    v(0, 0, 1, 1) = 1.0f;
    const BlockGrid grid = make_block_grid(2, 128);
    const auto out = block_sparse_attention(
        make_sequence_batch(std::move(q), Role::kQuery), make_sequence_batch(std::move(k), Role::kKey),
        make_sequence_batch(std::move(v), Role::kValue), full_causal_plan(1, 1, grid), grid, 1.0f);
    CHECK(approx(out.out(0, 0, 1, 0), 0.5, 2e-3) && approx(out.out(0, 0, 1, 1), 0.5, 2e-3));
    CHECK(approx(out.lse(0, 0, 1), 1.0, 1e-5));
  }
  // acceptance.cpp:59-109 (criterion 1) — full plan == dense <= 1e-4, ragged shapes, visits exact
  {
    for (std::uint64_t L : {128ull, 300ull, 1000ull}) {
      const auto q = random_batch(1, 2, L, Role::kQuery, 100 + L);
      const auto k = random_batch(1, 2, L, Role::kKey, 200 + L);
      const auto v = random_batch(1, 2, L, Role::kValue, 300 + L);
      const BlockGrid grid = make_block_grid(L, 128);
      const float tau = 1.0f / std::sqrt(128.0f);
      const auto plan = full_causal_plan(1, 2, grid);
      AttentionStats stats;
      const auto sp = block_sparse_attention(q, k, v, plan, grid, tau, &stats);
      const auto de = dense_attention(q, k, v, tau);
      double dmax = 0, lmax = 0;
      for (std::size_t i = 0; i < sp.out.numel(); ++i)
        dmax = std::fmax(dmax, std::fabs(sp.out.data()[i] - de.out.data()[i]));
      for (std::size_t i = 0; i < sp.lse.numel(); ++i)
        lmax = std::fmax(lmax, std::fabs(sp.lse.data()[i] - de.lse.data()[i]));
      CHECK(dmax <= 1e-4 && lmax <= 1e-4);
      CHECK(stats.block_visits == visit_count(plan));
    }
  }
  // test_attention.cpp:238-258 — plan corruption raises PlanError; wrong grid ValidationError
  {
    const auto q = random_batch(1, 1, 256, Role::kQuery, 51);
    const auto k = random_batch(1, 1, 256, Role::kKey, 52);
    const auto v = random_batch(1, 1, 256, Role::kValue, 53);
    const BlockGrid grid = make_block_grid(256, 128);
    auto plan = full_causal_plan(1, 1, grid);
    plan.indices(0, 1, 0, 0) = 2;  // == N, the fill value, inside the counted prefix
    CHECK_THROWS_AS(block_sparse_attention(q, k, v, plan, grid, 0.5f), PlanError);
    plan = full_causal_plan(1, 1, grid);
    plan.indices(0, 1, 0, 0) = -1;
    CHECK_THROWS_AS(block_sparse_attention(q, k, v, plan, grid, 0.5f), PlanError);
    const auto other = full_causal_plan(1, 1, make_block_grid(512, 128));
    CHECK_THROWS_AS(block_sparse_attention(q, k, v, other, grid, 0.5f), ValidationError);
  }
  // the full drop-in pipeline (acceptance.cpp:357-360)
  {
    const auto q = random_batch(1, 2, 1024, Role::kQuery, 7);
    const auto k = random_batch(1, 2, 1024, Role::kKey, 8);
    const auto v = random_batch(1, 2, 1024, Role::kValue, 9);
    const BlockGrid grid = make_block_grid(1024, 128);
    PipelineConfig cfg;
    const auto map = discover(q, k, grid, cfg.resolved_scale(128));
    const auto plan = compress_indices(max_threshold_mask(map, cfg));
    AttentionStats stats;
    const auto res = block_sparse_attention(q, k, v, plan, grid, cfg.resolved_scale(128), &stats);
    CHECK(stats.block_visits == visit_count(plan) && density(plan, grid) <= 1.0);
    bool finite = true;
    for (std::size_t i = 0; i < res.out.numel(); ++i) finite = finite && std::isfinite(res.out.data()[i]);
    CHECK(finite);
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail;
}
