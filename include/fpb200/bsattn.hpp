// fpb200/bsattn.hpp — C++ drop-in for the reference's header-only `bsattn::` API.
//
// Same type names, member names, layouts, function signatures and exception types as
// /root/reference/proj/include/bsattn/{tensor,core,discovery,selection,attention}.hpp, so a
// reference user switches by replacing `#include "bsattn/..."` with `#include "fpb200/bsattn.hpp"`
// and `bsattn::` with `fpb200::` (or `namespace bsattn = fpb200;`).  Every compute call goes to the
// sm_100a kernels through the C ABI (include/fpb200.h, host-buffer entry points): inputs are copied
// to HBM, the kernels run, outputs come back.  Link with -lfpb200 (paper_2603_06199_b200/).
//
// Differences, all supersets: K/V may have fewer heads than Q (GQA; the reference requires equal
// shapes, core.hpp:81-85).  d == 128 with block_size == 128 runs the tcgen05 kernels (fp32 inputs
// through the split-precision path); every other shape runs the SIMT kernels of generic.cu.
// The comparison baselines (topk_select, topp_select, discover_pool_both, discover_exact) are here
// too, so the whole bsattn surface is covered.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../fpb200.h"

namespace fpb200 {

// ----------------------------------------------------------------------------- tensor.hpp:18-38
class IoError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};
class FormatError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};
class ValidationError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};
class ConfigError : public ValidationError {
  using ValidationError::ValidationError;
};
class PlanError : public ValidationError {
  using ValidationError::ValidationError;
};
class CudaError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(int rc, const char* what, bool plan = false) {
  if (rc == FPB_OK) return;
  const std::string msg = std::string(what) + ": " + fpb_last_error();
  if (rc == FPB_EVALIDATION) {
    if (plan) throw PlanError(msg);
    throw ValidationError(msg);
  }
  if (rc == FPB_EFORMAT) throw FormatError(msg);
  if (rc == FPB_ECUDA) throw CudaError(msg);
  throw std::invalid_argument(msg);
}
}  // namespace detail

// ----------------------------------------------------------------------------- tensor.hpp:53-95
template <typename T>
class Tensor {
 public:
  Tensor() = default;
  explicit Tensor(std::vector<std::uint64_t> shape, T fill = T{}) : shape_(std::move(shape)) {
    std::size_t n = 1;
    for (auto d : shape_) n *= static_cast<std::size_t>(d);
    data_.assign(n, fill);
  }
  const std::vector<std::uint64_t>& shape() const noexcept { return shape_; }
  std::size_t ndim() const noexcept { return shape_.size(); }
  std::uint64_t dim(std::size_t axis) const { return shape_.at(axis); }
  std::size_t numel() const noexcept { return data_.size(); }
  bool empty() const noexcept { return data_.empty(); }
  T* data() noexcept { return data_.data(); }
  const T* data() const noexcept { return data_.data(); }
  template <typename... Ix>
  std::size_t offset(Ix... ix) const noexcept {
    const std::size_t idx[] = {static_cast<std::size_t>(ix)...};
    std::size_t off = 0;
    for (std::size_t a = 0; a < sizeof...(Ix); ++a) off = off * shape_[a] + idx[a];
    return off;
  }
  template <typename... Ix>
  T& operator()(Ix... ix) noexcept {
    return data_[offset(ix...)];
  }
  template <typename... Ix>
  const T& operator()(Ix... ix) const noexcept {
    return data_[offset(ix...)];
  }
  bool same_shape(const Tensor& o) const noexcept { return shape_ == o.shape_; }

 private:
  std::vector<std::uint64_t> shape_;
  std::vector<T> data_;
};

// ----------------------------------------------------------------------------- core.hpp
inline constexpr float kLog2e = 1.4426950408889634f;
inline constexpr float kDefaultEpsilon = 1e-10f;
inline constexpr float kNegSentinel = std::numeric_limits<float>::lowest();

struct BlockGrid {
  std::uint32_t block_size = 0;
  std::uint32_t num_query_blocks = 0;
  std::uint32_t num_key_blocks = 0;
  std::uint32_t last_block_len = 0;
  std::uint32_t block_len(std::uint32_t block) const noexcept {
    return block + 1 == num_key_blocks ? last_block_len : block_size;
  }
  std::uint32_t block_of(std::uint64_t token) const noexcept {
    return static_cast<std::uint32_t>(token / block_size);
  }
};

inline BlockGrid make_block_grid(std::uint64_t seq_len, std::uint32_t block_size) {
  if (seq_len < 1) throw ValidationError("sequence length must be >= 1");
  if (block_size < 1) throw ValidationError("block size must be >= 1");
  BlockGrid g;
  g.block_size = block_size;
  const std::uint64_t blocks = (seq_len + block_size - 1) / block_size;
  g.num_query_blocks = g.num_key_blocks = static_cast<std::uint32_t>(blocks);
  g.last_block_len = static_cast<std::uint32_t>(seq_len - (blocks - 1) * block_size);
  return g;
}

enum class Role { kQuery, kKey, kValue };

struct SequenceBatch {
  Tensor<float> data;
  Role role = Role::kQuery;
  std::uint64_t batch() const { return data.dim(0); }
  std::uint64_t heads() const { return data.dim(1); }
  std::uint64_t seq_len() const { return data.dim(2); }
  std::uint64_t head_dim() const { return data.dim(3); }
  const float* slice(std::uint64_t z, std::uint64_t h) const {
    return data.data() + ((z * heads() + h) * seq_len()) * head_dim();
  }
};

inline SequenceBatch make_sequence_batch(Tensor<float> data, Role role) {
  if (data.ndim() != 4) throw ValidationError("sequence batch must be Z x H x L x d");
  for (std::size_t a = 0; a < 4; ++a)
    if (data.dim(a) < 1) throw ValidationError("sequence batch dims must be >= 1");
  for (std::size_t i = 0; i < data.numel(); ++i)
    if (!std::isfinite(data.data()[i])) throw ValidationError("non-finite value in sequence batch");
  return SequenceBatch{std::move(data), role};
}

struct PipelineConfig {
  std::uint32_t block_size = 128;
  float alpha = 0.12f;
  std::uint32_t sink_tokens = 256;
  std::uint32_t window_tokens = 512;
  float scale = 0.0f;
  float epsilon = kDefaultEpsilon;
  std::uint64_t rng_seed = 0;
  void validate() const {
    if (block_size < 1) throw ConfigError("block_size must be >= 1");
    if (!(alpha >= 0.0f)) throw ConfigError("alpha must be >= 0");
    if (window_tokens < 1) throw ConfigError("window_tokens must be >= 1");
    if (!(epsilon > 0.0f)) throw ConfigError("epsilon must be > 0");
  }
  std::uint32_t sink_blocks() const noexcept { return (sink_tokens + block_size - 1) / block_size; }
  std::uint32_t window_blocks() const noexcept {
    return (window_tokens + block_size - 1) / block_size;
  }
  float resolved_scale(std::uint64_t head_dim) const noexcept {
    return scale > 0.0f ? scale : 1.0f / std::sqrt(static_cast<float>(head_dim));
  }
};

// ----------------------------------------------------------------------------- result types
struct PooledKeys {
  Tensor<float> data;
};
struct BlockEnergies {
  Tensor<float> energy, local_max;
};
struct BlockScoreMap {
  Tensor<float> energy, local_max, score;
};
struct ActiveMask {
  Tensor<std::uint8_t> active;
  std::uint64_t batch() const { return active.dim(0); }
  std::uint64_t query_blocks() const { return active.dim(1); }
  std::uint64_t key_blocks() const { return active.dim(2); }
  std::uint64_t heads() const { return active.dim(3); }
};
struct SparseBlockPlan {
  Tensor<std::int32_t> indices;
  Tensor<std::int32_t> counts;
  std::uint64_t batch() const { return indices.dim(0); }
  std::uint64_t query_blocks() const { return indices.dim(1); }
  std::uint64_t key_blocks() const { return indices.dim(2); }
  std::uint64_t heads() const { return indices.dim(3); }
};
struct SelectionStats {
  std::uint64_t score_comparisons = 0;
};
struct AttentionOutput {
  Tensor<float> out, lse;
};
struct AttentionStats {
  std::uint64_t block_visits = 0;
};

namespace detail {
inline fpb_problem problem(std::uint64_t Z, std::uint64_t Hq, std::uint64_t Hkv, std::uint64_t L,
                           std::uint64_t d, std::uint32_t block_size) {
  fpb_problem p;
  fpb_problem_init(&p, static_cast<int64_t>(Z), static_cast<int64_t>(Hq),
                   static_cast<int64_t>(Hkv), static_cast<int64_t>(L), static_cast<int64_t>(d));
  p.block_size = static_cast<int32_t>(block_size);
  return p;
}
inline void require_qk(const SequenceBatch& q, const SequenceBatch& k) {
  if (q.batch() != k.batch() || q.seq_len() != k.seq_len() || q.head_dim() != k.head_dim() ||
      q.heads() % k.heads())
    throw ValidationError("query/key shape mismatch");
}
inline std::uint64_t grid_len(const BlockGrid& g) {
  return static_cast<std::uint64_t>(g.num_query_blocks - 1) * g.block_size + g.last_block_len;
}
}  // namespace detail

// ----------------------------------------------------------------------------- discovery.hpp
inline PooledKeys pool_keys(const SequenceBatch& keys, const BlockGrid& grid) {
  if (keys.role != Role::kKey) throw ValidationError("pool_keys expects a key batch");
  if (grid.num_key_blocks * static_cast<std::uint64_t>(grid.block_size) < keys.seq_len())
    throw ValidationError("grid does not cover the key sequence");
  auto p = detail::problem(keys.batch(), keys.heads(), keys.heads(), keys.seq_len(),
                           keys.head_dim(), grid.block_size);
  PooledKeys out{Tensor<float>({keys.batch(), keys.heads(), grid.num_key_blocks, keys.head_dim()})};
  detail::check(fpb_host_pool_keys(&p, FPB_F32, keys.data.data(), out.data.data()), "pool_keys");
  return out;
}

inline BlockEnergies approx_block_scores(const SequenceBatch& q, const PooledKeys& pooled,
                                         const BlockGrid& grid, float tau) {
  const auto& pk = pooled.data;
  if (pk.ndim() != 4 || pk.dim(0) != q.batch() || pk.dim(2) != grid.num_key_blocks ||
      pk.dim(3) != q.head_dim() || q.heads() % pk.dim(1))
    throw ValidationError("pooled keys shape mismatch");
  auto p = detail::problem(q.batch(), q.heads(), pk.dim(1), q.seq_len(), q.head_dim(),
                           grid.block_size);
  p.scale = tau;
  const std::uint64_t M = grid.num_query_blocks;
  BlockEnergies e{Tensor<float>({q.batch(), q.heads(), M, M}), Tensor<float>({q.batch(), q.heads(), M, M})};
  detail::check(fpb_host_approx_block_scores(&p, FPB_F32, q.data.data(), pk.data(),
                                             e.energy.data(), e.local_max.data()),
                "approx_block_scores");
  return e;
}

inline BlockScoreMap normalize_block_scores(BlockEnergies energies, const BlockGrid& grid,
                                            float epsilon = kDefaultEpsilon) {
  const auto& sh = energies.energy.shape();
  auto p = detail::problem(sh[0], sh[1], sh[1], detail::grid_len(grid), 128, grid.block_size);
  p.epsilon = epsilon;
  Tensor<float> score(sh);
  detail::check(fpb_host_normalize_block_scores(&p, energies.energy.data(),
                                                energies.local_max.data(), score.data()),
                "normalize_block_scores");
  return BlockScoreMap{std::move(energies.energy), std::move(energies.local_max), std::move(score)};
}

inline BlockScoreMap discover(const SequenceBatch& q, const SequenceBatch& k, const BlockGrid& grid,
                              float tau, float epsilon = kDefaultEpsilon) {
  detail::require_qk(q, k);
  auto p = detail::problem(q.batch(), q.heads(), k.heads(), q.seq_len(), q.head_dim(),
                           grid.block_size);
  p.scale = tau;
  p.epsilon = epsilon;
  const std::uint64_t M = grid.num_query_blocks;
  BlockScoreMap m{Tensor<float>({q.batch(), q.heads(), M, M}),
                  Tensor<float>({q.batch(), q.heads(), M, M}),
                  Tensor<float>({q.batch(), q.heads(), M, M})};
  detail::check(fpb_host_discover(&p, FPB_F32, q.data.data(), k.data.data(), m.energy.data(),
                                  m.local_max.data(), m.score.data()),
                "discover");
  return m;
}

// comparison methods (discovery.hpp:164-279), method 1 = pool-both, 2 = exact
namespace detail {
inline BlockScoreMap discover_method(int method, const SequenceBatch& q, const SequenceBatch& k,
                                     const BlockGrid& grid, float tau, float epsilon) {
  require_qk(q, k);
  auto p = problem(q.batch(), q.heads(), k.heads(), q.seq_len(), q.head_dim(), grid.block_size);
  p.scale = tau;
  p.epsilon = epsilon;
  const std::uint64_t M = grid.num_query_blocks;
  BlockScoreMap m{Tensor<float>({q.batch(), q.heads(), M, M}),
                  Tensor<float>({q.batch(), q.heads(), M, M}),
                  Tensor<float>({q.batch(), q.heads(), M, M})};
  check(fpb_host_discover_method(&p, FPB_F32, method, q.data.data(), k.data.data(),
                                 m.energy.data(), m.local_max.data(), m.score.data()),
        method == 1 ? "discover_pool_both" : "discover_exact");
  return m;
}
}  // namespace detail

inline BlockScoreMap discover_pool_both(const SequenceBatch& q, const SequenceBatch& k,
                                        const BlockGrid& grid, float tau,
                                        float epsilon = kDefaultEpsilon) {
  return detail::discover_method(1, q, k, grid, tau, epsilon);
}
inline BlockScoreMap discover_exact(const SequenceBatch& q, const SequenceBatch& k,
                                    const BlockGrid& grid, float tau,
                                    float epsilon = kDefaultEpsilon) {
  return detail::discover_method(2, q, k, grid, tau, epsilon);
}

// ----------------------------------------------------------------------------- selection.hpp
inline ActiveMask max_threshold_mask(const Tensor<float>& score, const PipelineConfig& config,
                                     SelectionStats* stats = nullptr) {
  config.validate();
  if (score.ndim() != 4) throw ValidationError("score map must be Z x H x M x N");
  const std::uint64_t Z = score.dim(0), H = score.dim(1), M = score.dim(2), N = score.dim(3);
  if (M != N) throw ValidationError("score map must be square");
  auto p = detail::problem(Z, H, H, (M - 1) * config.block_size + 1, 128, config.block_size);
  p.alpha = config.alpha;
  p.sink_tokens = static_cast<int32_t>(config.sink_tokens);
  p.window_tokens = static_cast<int32_t>(config.window_tokens);
  p.epsilon = config.epsilon;
  ActiveMask mask{Tensor<std::uint8_t>({Z, M, N, H})};
  unsigned long long cmp = 0;
  detail::check(fpb_host_max_threshold_mask(&p, score.data(), mask.active.data(), &cmp),
                "max_threshold_mask");
  if (stats) stats->score_comparisons += cmp;
  return mask;
}
inline ActiveMask max_threshold_mask(const BlockScoreMap& scores, const PipelineConfig& config,
                                     SelectionStats* stats = nullptr) {
  return max_threshold_mask(scores.score, config, stats);
}

namespace detail {
inline ActiveMask sort_select(const Tensor<float>& score, int mode, std::uint32_t k, float top_p,
                              const PipelineConfig& config) {
  config.validate();
  if (score.ndim() != 4) throw ValidationError("score map must be Z x H x M x N");
  const std::uint64_t Z = score.dim(0), H = score.dim(1), M = score.dim(2), N = score.dim(3);
  auto p = problem(Z, H, H, (M - 1) * config.block_size + 1, 128, config.block_size);
  p.sink_tokens = static_cast<int32_t>(config.sink_tokens);
  p.window_tokens = static_cast<int32_t>(config.window_tokens);
  ActiveMask mask{Tensor<std::uint8_t>({Z, M, N, H})};
  const int rc = mode == 0 ? fpb_host_topk_select(&p, score.data(), static_cast<int32_t>(k),
                                                  mask.active.data())
                           : fpb_host_topp_select(&p, score.data(), top_p, mask.active.data());
  if (rc == FPB_EVALIDATION) throw ConfigError(fpb_last_error());
  check(rc, mode == 0 ? "topk_select" : "topp_select");
  return mask;
}
}  // namespace detail

// selection.hpp:96-123 / 127-159 (comparison baselines)
inline ActiveMask topk_select(const Tensor<float>& score, std::uint32_t k,
                              const PipelineConfig& config) {
  if (k < 1) throw ConfigError("top-k requires k >= 1");
  return detail::sort_select(score, 0, k, 0.0f, config);
}
inline ActiveMask topp_select(const Tensor<float>& score, float p, const PipelineConfig& config) {
  if (!(p > 0.0f) || p > 1.0f) throw ConfigError("top-p requires p in (0, 1]");
  return detail::sort_select(score, 1, 1, p, config);
}
inline ActiveMask topk_select(const BlockScoreMap& s, std::uint32_t k, const PipelineConfig& c) {
  return topk_select(s.score, k, c);
}
inline ActiveMask topp_select(const BlockScoreMap& s, float p, const PipelineConfig& c) {
  return topp_select(s.score, p, c);
}

inline SparseBlockPlan compress_indices(const ActiveMask& mask) {
  const std::uint64_t Z = mask.batch(), M = mask.query_blocks(), N = mask.key_blocks(),
                      H = mask.heads();
  if (M != N) throw ValidationError("mask must be square");
  auto p = detail::problem(Z, H, H, (M - 1) * 128 + 1, 128, 128);
  SparseBlockPlan plan{Tensor<std::int32_t>({Z, M, N, H}), Tensor<std::int32_t>({Z, M, H})};
  detail::check(fpb_host_compress_indices(&p, mask.active.data(), plan.indices.data(),
                                          plan.counts.data()),
                "compress_indices");
  return plan;
}

inline std::uint64_t visit_count(const SparseBlockPlan& plan) {
  std::uint64_t total = 0;
  for (std::size_t i = 0; i < plan.counts.numel(); ++i)
    total += static_cast<std::uint64_t>(plan.counts.data()[i]);
  return total;
}
inline double density(const SparseBlockPlan& plan, const BlockGrid& grid) {
  const double M = grid.num_query_blocks;
  return static_cast<double>(visit_count(plan)) /
         (static_cast<double>(plan.batch()) * static_cast<double>(plan.heads()) * (M * (M + 1) / 2.0));
}

// ----------------------------------------------------------------------------- attention.hpp
inline AttentionOutput block_sparse_attention(const SequenceBatch& q, const SequenceBatch& k,
                                              const SequenceBatch& v, const SparseBlockPlan& plan,
                                              const BlockGrid& grid, float tau,
                                              AttentionStats* stats = nullptr) {
  if (q.role != Role::kQuery || k.role != Role::kKey || v.role != Role::kValue)
    throw ValidationError("expected query/key/value roles");
  detail::require_qk(q, k);
  if (!k.data.same_shape(v.data)) throw ValidationError("key/value shape mismatch");
  if (plan.batch() != q.batch() || plan.heads() != q.heads() ||
      plan.query_blocks() != grid.num_query_blocks || plan.key_blocks() != grid.num_key_blocks)
    throw ValidationError("plan shape does not match grid/batch");
  auto p = detail::problem(q.batch(), q.heads(), k.heads(), q.seq_len(), q.head_dim(),
                           grid.block_size);
  p.scale = tau;
  AttentionOutput res{Tensor<float>(q.data.shape()),
                      Tensor<float>({q.batch(), q.heads(), q.seq_len()})};
  unsigned long long visits = 0;
  detail::check(fpb_host_block_sparse_attention(&p, FPB_F32, q.data.data(), k.data.data(),
                                                v.data.data(), plan.indices.data(),
                                                plan.counts.data(), FPB_F32, res.out.data(),
                                                res.lse.data(), &visits),
                "block_sparse_attention", /*plan=*/true);
  if (stats) stats->block_visits += visits;
  return res;
}

inline AttentionOutput dense_attention(const SequenceBatch& q, const SequenceBatch& k,
                                       const SequenceBatch& v, float tau) {
  if (q.role != Role::kQuery || k.role != Role::kKey || v.role != Role::kValue)
    throw ValidationError("expected query/key/value roles");
  detail::require_qk(q, k);
  if (!k.data.same_shape(v.data)) throw ValidationError("key/value shape mismatch");
  auto p = detail::problem(q.batch(), q.heads(), k.heads(), q.seq_len(), q.head_dim(), 128);
  p.scale = tau;
  AttentionOutput res{Tensor<float>(q.data.shape()),
                      Tensor<float>({q.batch(), q.heads(), q.seq_len()})};
  detail::check(fpb_host_dense_attention(&p, FPB_F32, q.data.data(), k.data.data(), v.data.data(),
                                         FPB_F32, res.out.data(), res.lse.data()),
                "dense_attention");
  return res;
}

inline SparseBlockPlan full_causal_plan(std::uint64_t batch, std::uint64_t heads,
                                        const BlockGrid& grid) {
  const std::uint64_t M = grid.num_query_blocks, N = grid.num_key_blocks;
  SparseBlockPlan plan{Tensor<std::int32_t>({batch, M, N, heads}, static_cast<std::int32_t>(N)),
                       Tensor<std::int32_t>({batch, M, heads}, 0)};
  for (std::uint64_t z = 0; z < batch; ++z)
    for (std::uint64_t i = 0; i < M; ++i)
      for (std::uint64_t h = 0; h < heads; ++h) {
        for (std::uint64_t j = 0; j <= i; ++j) plan.indices(z, i, j, h) = static_cast<std::int32_t>(j);
        plan.counts(z, i, h) = static_cast<std::int32_t>(i + 1);
      }
  return plan;
}

}  // namespace fpb200
