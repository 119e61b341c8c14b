// fpb200_cli — the reference's command-line harness (tools/bsattn_main.cpp) over the fpb200 C ABI.
//
// Same subcommands, flags, report schema and exit codes as the reference binary, so scripts and the
// reference's CLI tests (tests/test_cli.cpp) drive it unchanged:
//   gen       synthetic planted workload -> <out>.{q,k,v,gt}.fpt           (bsattn_main.cpp:246-273)
//   discover  block score map (approx | pool-both | exact)                  (bsattn_main.cpp:275-333)
//   select    score map -> sparse block plan (max | --topk | --topp)        (bsattn_main.cpp:335-366)
//   attend    block-sparse (or --dense) attention, --check vs dense         (bsattn_main.cpp:368-463)
//   sweep     alpha / top-k / top-p / length sweep, one report row per cell (bsattn_main.cpp:465-574)
// Exit codes (bsattn_main.cpp:671-692): 0 ok, 1 usage, 2 config/validation/plan, 3 format/io;
// 4 is ours: a CUDA failure inside the library.  All compute runs on the GPU through libfpb200.so;
// the generators and metrics are host-side evaluation helpers, as in the reference.
//
// The argument parser is a small table-driven replacement for CLI11 (not available here): options
// take "--opt value" or "--opt=value", lists are comma-delimited, unknown options / bad numbers /
// values outside a choice set are usage errors (exit 1), --help prints usage and exits 0.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "cli/json.hpp"
#include "cli/workloads.hpp"
#include "fpb200/bsattn.hpp"
#include "fpb200/fpt1.hpp"

namespace {

using namespace fpb200;
using cli::Json;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class Timer {
 public:
  double ms() const {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0_).count();
  }

 private:
  std::chrono::steady_clock::time_point t0_ = std::chrono::steady_clock::now();
};

// ------------------------------------------------------------------------------------- arguments
struct Args {
  std::string sub;
  // common (bsattn_main.cpp:64-80)
  PipelineConfig config;
  std::string format = "json", out;
  // workload (bsattn_main.cpp:82-97)
  std::string pattern, target;
  std::uint64_t Z = 1, H = 1, L = 2048, d = 64;
  float strength = 2.5f, noise = 0.5f, head_mass = 0.7f;
  // per-command
  std::string method = "approx", q, k, v, scores, plan;
  bool compare_exact = false, dense = false, check = false, lse_natural = false;
  std::optional<std::uint32_t> topk;
  std::optional<float> topp;
  std::vector<float> alphas, topps;
  std::vector<std::uint32_t> topks;
  std::vector<std::uint64_t> lengths;
};

template <typename T>
T parse_uint(const std::string& opt, const std::string& s) {
  if (s.empty() || s[0] == '-' || s[0] == '+') throw UsageError(opt + ": expected a non-negative integer, got '" + s + "'");
  std::size_t pos = 0;
  unsigned long long v = 0;
  try {
    v = std::stoull(s, &pos, 10);
  } catch (const std::exception&) {
    throw UsageError(opt + ": expected a non-negative integer, got '" + s + "'");
  }
  if (pos != s.size() || v > std::numeric_limits<T>::max())
    throw UsageError(opt + ": expected a non-negative integer, got '" + s + "'");
  return static_cast<T>(v);
}
float parse_float(const std::string& opt, const std::string& s) {
  std::size_t pos = 0;
  float v = 0.0f;
  try {
    v = std::stof(s, &pos);
  } catch (const std::exception&) {
    throw UsageError(opt + ": expected a number, got '" + s + "'");
  }
  if (pos != s.size()) throw UsageError(opt + ": expected a number, got '" + s + "'");
  return v;
}
std::vector<std::string> split_list(const std::string& s) {
  std::vector<std::string> out;
  std::string cur;
  std::stringstream ss(s);
  while (std::getline(ss, cur, ',')) out.push_back(cur);
  return out;
}
void choice(const std::string& opt, const std::string& v, std::initializer_list<const char*> allowed) {
  for (const char* a : allowed)
    if (v == a) return;
  std::string msg = opt + ": '" + v + "' not in {";
  bool first = true;
  for (const char* a : allowed) {
    msg += (first ? "" : ", ") + std::string(a);
    first = false;
  }
  throw UsageError(msg + "}");
}

const char* kUsage =
    "usage: fpb200_cli <gen|discover|select|attend|sweep> [options]\n"
    "  common:    --block-size/-B/--B N  --alpha A  --sink-tokens N  --window-tokens N  --scale S\n"
    "             --seed N  --format json|csv  --out PREFIX\n"
    "  workload:  --gen vertical|slash|block|needle|alt-slash[|heavy-tail (sweep)]  --L --Z --H --d\n"
    "             --strength S  --noise S  --target A[,B]  --head-mass M\n"
    "  discover:  --method approx|pool-both|exact  --q PATH  --k PATH  --compare-exact\n"
    "  select:    --scores PATH  [--topk K | --topp P]\n"
    "  attend:    --q --k --v PATH  --plan PREFIX  --method M  [--topk K | --topp P]\n"
    "             --dense  --check  --lse-natural\n"
    "  sweep:     --alphas a,b,..  --topks k,..  --topps p,..  --Ls L,..\n";

Args parse(int argc, char** argv) {
  Args a;
  if (argc < 2) throw UsageError("a subcommand is required");
  a.sub = argv[1];
  if (a.sub == "-h" || a.sub == "--help") {
    std::cout << kUsage;
    std::exit(0);
  }
  choice("subcommand", a.sub, {"gen", "discover", "select", "attend", "sweep"});
  const bool wl = a.sub != "select";
  using Setter = std::function<void(const std::string&, const std::string&)>;
  std::map<std::string, Setter> opts;
  std::map<std::string, bool*> flags;
  auto u32 = [](std::uint32_t& dst) { return [&dst](const std::string& o, const std::string& s) { dst = parse_uint<std::uint32_t>(o, s); }; };
  auto u64 = [](std::uint64_t& dst) { return [&dst](const std::string& o, const std::string& s) { dst = parse_uint<std::uint64_t>(o, s); }; };
  auto f32 = [](float& dst) { return [&dst](const std::string& o, const std::string& s) { dst = parse_float(o, s); }; };
  auto str = [](std::string& dst) { return [&dst](const std::string&, const std::string& s) { dst = s; }; };
  for (const char* n : {"--block-size", "-B", "--B"}) opts[n] = u32(a.config.block_size);
  opts["--alpha"] = f32(a.config.alpha);
  opts["--sink-tokens"] = u32(a.config.sink_tokens);
  opts["--window-tokens"] = u32(a.config.window_tokens);
  opts["--scale"] = f32(a.config.scale);
  opts["--seed"] = u64(a.config.rng_seed);
  opts["--format"] = [&a](const std::string& o, const std::string& s) {
    choice(o, s, {"json", "csv"});
    a.format = s;
  };
  opts["--out"] = str(a.out);
  if (wl) {
    const bool heavy = a.sub == "sweep";
    opts["--gen"] = [&a, heavy](const std::string& o, const std::string& s) {
      if (heavy)
        choice(o, s, {"vertical", "slash", "block", "needle", "alt-slash", "heavy-tail"});
      else
        choice(o, s, {"vertical", "slash", "block", "needle", "alt-slash"});
      a.pattern = s;
    };
    opts["--L"] = u64(a.L);
    opts["--Z"] = u64(a.Z);
    opts["--H"] = u64(a.H);
    opts["--d"] = u64(a.d);
    opts["--strength"] = f32(a.strength);
    opts["--noise"] = f32(a.noise);
    opts["--target"] = str(a.target);
    opts["--head-mass"] = f32(a.head_mass);
  }
  auto method = [&a](const std::string& o, const std::string& s) {
    choice(o, s, {"approx", "pool-both", "exact"});
    a.method = s;
  };
  auto topk = [&a](const std::string& o, const std::string& s) { a.topk = parse_uint<std::uint32_t>(o, s); };
  auto topp = [&a](const std::string& o, const std::string& s) { a.topp = parse_float(o, s); };
  if (a.sub == "discover") {
    opts["--method"] = method;
    opts["--q"] = str(a.q);
    opts["--k"] = str(a.k);
    flags["--compare-exact"] = &a.compare_exact;
  } else if (a.sub == "select") {
    opts["--scores"] = str(a.scores);
    opts["--topk"] = topk;
    opts["--topp"] = topp;
  } else if (a.sub == "attend") {
    opts["--q"] = str(a.q);
    opts["--k"] = str(a.k);
    opts["--v"] = str(a.v);
    opts["--plan"] = str(a.plan);
    opts["--method"] = method;
    opts["--topk"] = topk;
    opts["--topp"] = topp;
    flags["--dense"] = &a.dense;
    flags["--check"] = &a.check;
    flags["--lse-natural"] = &a.lse_natural;
  } else if (a.sub == "sweep") {
    opts["--alphas"] = [&a](const std::string& o, const std::string& s) {
      for (auto& t : split_list(s)) a.alphas.push_back(parse_float(o, t));
    };
    opts["--topks"] = [&a](const std::string& o, const std::string& s) {
      for (auto& t : split_list(s)) a.topks.push_back(parse_uint<std::uint32_t>(o, t));
    };
    opts["--topps"] = [&a](const std::string& o, const std::string& s) {
      for (auto& t : split_list(s)) a.topps.push_back(parse_float(o, t));
    };
    opts["--Ls"] = [&a](const std::string& o, const std::string& s) {
      for (auto& t : split_list(s)) a.lengths.push_back(parse_uint<std::uint64_t>(o, t));
    };
  }
  for (int i = 2; i < argc; ++i) {
    std::string tok = argv[i], val;
    bool inline_val = false;
    if (tok == "-h" || tok == "--help") {
      std::cout << kUsage;
      std::exit(0);
    }
    if (const auto eq = tok.find('='); tok.rfind("--", 0) == 0 && eq != std::string::npos) {
      val = tok.substr(eq + 1);
      tok = tok.substr(0, eq);
      inline_val = true;
    }
    if (auto f = flags.find(tok); f != flags.end()) {
      if (inline_val) throw UsageError(tok + " takes no value");
      *f->second = true;
      continue;
    }
    auto o = opts.find(tok);
    if (o == opts.end()) throw UsageError("unknown option for '" + a.sub + "': " + tok);
    if (!inline_val) {
      if (i + 1 >= argc) throw UsageError(tok + " requires a value");
      val = argv[++i];
    }
    o->second(tok, val);
  }
  return a;
}

// ------------------------------------------------------------------------------------- helpers
Json config_echo(const PipelineConfig& c) {  // report.hpp config_echo: same keys, same order
  Json j = Json::object();
  j["block_size"] = c.block_size;
  j["alpha"] = c.alpha;
  j["sink_tokens"] = c.sink_tokens;
  j["window_tokens"] = c.window_tokens;
  j["scale"] = c.scale;
  j["epsilon"] = c.epsilon;
  j["rng_seed"] = static_cast<unsigned long long>(c.rng_seed);
  return j;
}

Json base_report(const char* command, const Args& a) {
  Json r = Json::object();
  r["command"] = command;
  r["config"] = config_echo(a.config);
  r["config_hash"] = cli::fnv1a_hex(config_echo(a.config).dump());
  r["timings_ms"] = Json::object();
  r["metrics"] = Json::object();
  return r;
}

Json workload_echo(const Args& a) {
  Json j = Json::object();
  j["pattern"] = a.pattern;
  j["strength"] = a.strength;
  j["noise"] = a.noise;
  return j;
}

Json shape_echo(const SequenceBatch& b) {
  Json j = Json::object();
  j["Z"] = static_cast<unsigned long long>(b.batch());
  j["H"] = static_cast<unsigned long long>(b.heads());
  j["L"] = static_cast<unsigned long long>(b.seq_len());
  j["d"] = static_cast<unsigned long long>(b.head_dim());
  return j;
}

void emit(const Json& report, const Args& a, const char* suffix) {
  const std::string text = a.format == "csv" ? cli::to_csv(report) : report.dump(2) + "\n";
  std::cout << text;
  if (!a.out.empty()) {
    const std::string path = a.out + suffix + (a.format == "csv" ? ".csv" : ".json");
    std::ofstream f(path, std::ios::trunc);
    if (!f) throw IoError("cannot open for writing: " + path);
    f << text;
    if (!f.flush()) throw IoError("write failed: " + path);
  }
}

std::pair<std::int64_t, std::int64_t> parse_target(const std::string& t) {
  try {
    const auto comma = t.find(',');
    if (comma == std::string::npos) return {std::stoll(t), 0};
    return {std::stoll(t.substr(0, comma)), std::stoll(t.substr(comma + 1))};
  } catch (const std::exception&) {
    throw UsageError("--target: expected 'a' or 'a,b', got '" + t + "'");
  }
}

cli::Planted planted_spec(const Args& a, std::uint64_t L, const std::string& target) {
  cli::Planted s;
  s.strength = a.strength;
  s.noise = a.noise;
  s.seed = a.config.rng_seed;
  const std::uint32_t M = make_block_grid(L, a.config.block_size).num_query_blocks;
  if (a.pattern == "vertical") {
    s.kind = cli::Pattern::kVertical;
    s.a = target.empty() ? M / 4 : parse_target(target).first;
  } else if (a.pattern == "slash" || a.pattern == "alt-slash") {
    s.kind = cli::Pattern::kSlash;
    s.a = target.empty() ? 2 * static_cast<std::int64_t>(a.config.block_size) : parse_target(target).first;
  } else if (a.pattern == "block") {
    s.kind = cli::Pattern::kBlock;
    if (target.empty()) {
      s.a = M / 2;
      s.b = M / 4;
    } else {
      std::tie(s.a, s.b) = parse_target(target);
    }
  } else if (a.pattern == "needle") {
    s.kind = cli::Pattern::kNeedle;
    s.a = target.empty() ? static_cast<std::int64_t>(L / 3) : parse_target(target).first;
  } else {
    throw UsageError("pattern '" + a.pattern + "' cannot generate q/k/v tensors");
  }
  return s;
}

cli::Workload build_workload(const Args& a, std::uint64_t L, const std::string& target) {
  const cli::Planted s = planted_spec(a, L, target);
  const float tau = a.config.resolved_scale(a.d);
  if (a.pattern == "alt-slash")
    return cli::generate_alternating_slash(s, a.Z, a.H, L, a.d, a.config.block_size, tau);
  return cli::generate_planted(s, a.Z, a.H, L, a.d, a.config.block_size, tau);
}

void require_same_shape(const SequenceBatch& x, const SequenceBatch& y) {
  if (!x.data.same_shape(y.data)) throw ValidationError("q/k/v shapes must match (Z x H x L x d)");
}

SequenceBatch load_batch(const std::string& path, Role role) {
  return make_sequence_batch(load_tensor<float>(path), role);
}

Tensor<std::int32_t> mask_to_i32(const ActiveMask& m) {
  Tensor<std::int32_t> t(m.active.shape(), 0);
  for (std::size_t i = 0; i < t.numel(); ++i) t.data()[i] = m.active.data()[i];
  return t;
}

SparseBlockPlan load_plan(const std::string& prefix) {
  SparseBlockPlan plan{load_tensor<std::int32_t>(prefix + ".idx.fpt"),
                       load_tensor<std::int32_t>(prefix + ".cnt.fpt")};
  if (plan.indices.ndim() != 4 || plan.counts.ndim() != 3)
    throw ValidationError("plan tensors must be Z x M x N x H and Z x M x H");
  for (std::size_t ax = 0; ax < 3; ++ax)
    if (plan.indices.dim(ax == 2 ? 3 : ax) != plan.counts.dim(ax))
      throw ValidationError("plan index/count shapes disagree");
  return plan;
}

BlockScoreMap run_discover(const std::string& method, const SequenceBatch& q, const SequenceBatch& k,
                           const BlockGrid& g, float tau, float eps) {
  if (method == "pool-both") return discover_pool_both(q, k, g, tau, eps);
  if (method == "exact") return discover_exact(q, k, g, tau, eps);
  return discover(q, k, g, tau, eps);
}

struct Selector {
  std::string method = "max";
  std::uint32_t k = 8;
  float p = 0.9f;
};

Selector selector_of(const Args& a) {
  if (a.topk && a.topp) throw UsageError("choose one of --topk / --topp");
  Selector s;
  if (a.topk) {
    s.method = "topk";
    s.k = *a.topk;
  } else if (a.topp) {
    s.method = "topp";
    s.p = *a.topp;
  }
  return s;
}

ActiveMask run_selector(const Selector& s, const Tensor<float>& score, const PipelineConfig& c,
                        SelectionStats* stats = nullptr) {
  if (s.method == "topk") return topk_select(score, s.k, c);
  if (s.method == "topp") return topp_select(score, s.p, c);
  return max_threshold_mask(score, c, stats);
}

// ------------------------------------------------------------------------------------- commands
int cmd_gen(const Args& a) {
  if (a.pattern.empty()) throw UsageError("gen requires --gen <pattern>");
  if (a.out.empty()) throw UsageError("gen requires --out <prefix>");
  a.config.validate();
  Timer t;
  const cli::Workload w = build_workload(a, a.L, a.target);
  const double gen_ms = t.ms();
  save_tensor(w.q.data, a.out + ".q.fpt");
  save_tensor(w.k.data, a.out + ".k.fpt");
  save_tensor(w.v.data, a.out + ".v.fpt");
  save_tensor(mask_to_i32(w.gt), a.out + ".gt.fpt");
  Json r = base_report("gen", a);
  r["workload"] = workload_echo(a);
  r["shape"] = shape_echo(w.q);
  r["timings_ms"]["generate"] = gen_ms;
  Json outs = Json::object();
  outs["q"] = a.out + ".q.fpt";
  outs["k"] = a.out + ".k.fpt";
  outs["v"] = a.out + ".v.fpt";
  outs["gt"] = a.out + ".gt.fpt";
  r["outputs"] = outs;
  emit(r, a, ".report");
  return 0;
}

int cmd_discover(const Args& a) {
  a.config.validate();
  Json r = base_report("discover", a);
  r["method"] = a.method;
  SequenceBatch q, k;
  std::optional<ActiveMask> gt;
  if (!a.pattern.empty()) {
    Timer t;
    cli::Workload w = build_workload(a, a.L, a.target);
    r["timings_ms"]["generate"] = t.ms();
    r["workload"] = workload_echo(a);
    q = std::move(w.q);
    k = std::move(w.k);
    gt = std::move(w.gt);
  } else {
    if (a.q.empty() || a.k.empty()) throw UsageError("discover needs --q and --k, or --gen <pattern>");
    q = load_batch(a.q, Role::kQuery);
    k = load_batch(a.k, Role::kKey);
  }
  require_same_shape(q, k);
  r["shape"] = shape_echo(q);
  const BlockGrid g = make_block_grid(q.seq_len(), a.config.block_size);
  const float tau = a.config.resolved_scale(q.head_dim());
  Timer t;
  const BlockScoreMap map = run_discover(a.method, q, k, g, tau, a.config.epsilon);
  r["timings_ms"]["discover"] = t.ms();
  if (gt) {
    r["metrics"]["recall"] = cli::planted_score_recall(map.score, *gt, a.config.alpha);
    r["metrics"]["recall_top1"] = cli::planted_top1_recall(map.score, *gt);
  }
  if (a.compare_exact && a.method != "exact") {
    Timer te;
    const BlockScoreMap exact = discover_exact(q, k, g, tau, a.config.epsilon);
    r["timings_ms"]["discover_exact"] = te.ms();
    r["metrics"]["rank_corr_exact"] = cli::mean_row_spearman(map.score, exact.score, 5);
  }
  if (!a.out.empty()) {
    save_tensor(map.score, a.out + ".score.fpt");
    save_tensor(map.energy, a.out + ".energy.fpt");
    save_tensor(map.local_max, a.out + ".localmax.fpt");
    Json outs = Json::object();
    outs["score"] = a.out + ".score.fpt";
    outs["energy"] = a.out + ".energy.fpt";
    outs["local_max"] = a.out + ".localmax.fpt";
    r["outputs"] = outs;
  }
  emit(r, a, ".report");
  return 0;
}

int cmd_select(const Args& a) {
  a.config.validate();
  if (a.scores.empty()) throw UsageError("select requires --scores <score tensor>");
  const Selector sel = selector_of(a);
  const Tensor<float> score = load_tensor<float>(a.scores);
  if (score.ndim() != 4) throw ValidationError("score map must be Z x H x M x N");
  const BlockGrid g = make_block_grid(score.dim(2) * a.config.block_size, a.config.block_size);
  Json r = base_report("select", a);
  r["selector"] = sel.method;
  if (sel.method == "topk") r["selector_k"] = sel.k;
  if (sel.method == "topp") r["selector_p"] = sel.p;
  Timer t;
  SelectionStats stats;
  const ActiveMask mask = run_selector(sel, score, a.config, &stats);
  const SparseBlockPlan plan = compress_indices(mask);
  r["timings_ms"]["select"] = t.ms();
  r["metrics"]["density"] = density(plan, g);
  r["metrics"]["visit_count"] = static_cast<unsigned long long>(visit_count(plan));
  if (sel.method == "max")
    r["metrics"]["score_comparisons"] = static_cast<unsigned long long>(stats.score_comparisons);
  if (!a.out.empty()) {
    save_tensor(plan.indices, a.out + ".idx.fpt");
    save_tensor(plan.counts, a.out + ".cnt.fpt");
    Json outs = Json::object();
    outs["indices"] = a.out + ".idx.fpt";
    outs["counts"] = a.out + ".cnt.fpt";
    r["outputs"] = outs;
  }
  emit(r, a, ".report");
  return 0;
}

int cmd_attend(const Args& a) {
  a.config.validate();
  const Selector sel = selector_of(a);
  Json r = base_report("attend", a);
  SequenceBatch q, k, v;
  std::optional<ActiveMask> gt;
  if (!a.pattern.empty()) {
    Timer t;
    cli::Workload w = build_workload(a, a.L, a.target);
    r["timings_ms"]["generate"] = t.ms();
    q = std::move(w.q);
    k = std::move(w.k);
    v = std::move(w.v);
    gt = std::move(w.gt);
  } else {
    if (a.q.empty() || a.k.empty() || a.v.empty())
      throw UsageError("attend needs --q/--k/--v, or --gen <pattern>");
    q = load_batch(a.q, Role::kQuery);
    k = load_batch(a.k, Role::kKey);
    v = load_batch(a.v, Role::kValue);
  }
  require_same_shape(q, k);
  require_same_shape(q, v);
  r["shape"] = shape_echo(q);
  const BlockGrid g = make_block_grid(q.seq_len(), a.config.block_size);
  const float tau = a.config.resolved_scale(q.head_dim());

  AttentionOutput result;
  std::optional<AttentionOutput> dense;
  if (a.dense || a.check) {
    Timer t;
    dense = dense_attention(q, k, v, tau);
    r["timings_ms"]["attend_dense"] = t.ms();
  }
  if (a.dense) {
    result = std::move(*dense);
    dense.reset();
  } else {
    SparseBlockPlan plan;
    if (!a.plan.empty()) {
      plan = load_plan(a.plan);
    } else {
      Timer td;
      const BlockScoreMap map = run_discover(a.method, q, k, g, tau, a.config.epsilon);
      r["timings_ms"]["discover"] = td.ms();
      Timer ts;
      const ActiveMask mask = run_selector(sel, map.score, a.config);
      plan = compress_indices(mask);
      r["timings_ms"]["select"] = ts.ms();
      if (gt) {
        r["metrics"]["mask_recall"] = cli::mask_recall(mask, *gt);
        r["metrics"]["mask_precision"] = cli::mask_precision(mask, *gt);
      }
    }
    r["metrics"]["density"] = density(plan, g);
    r["metrics"]["visit_count"] = static_cast<unsigned long long>(visit_count(plan));
    Timer t;
    AttentionStats stats;
    result = block_sparse_attention(q, k, v, plan, g, tau, &stats);
    r["timings_ms"]["attend_sparse"] = t.ms();
    r["metrics"]["block_visits"] = static_cast<unsigned long long>(stats.block_visits);
  }
  if (a.check && dense) {
    const auto oe = cli::tensor_error(result.out, dense->out);
    const auto le = cli::tensor_error(result.lse, dense->lse);
    r["metrics"]["err_max_abs"] = oe.max_abs;
    r["metrics"]["err_mean_abs"] = oe.mean_abs;
    r["metrics"]["lse_err_max_abs"] = le.max_abs;
  }
  if (a.lse_natural) {  // base-2 log-sum-exp -> natural log (bsattn_main.cpp:446-453)
    for (std::size_t i = 0; i < result.lse.numel(); ++i) result.lse.data()[i] *= 0.6931471805599453f;
    r["lse_units"] = "nat";
  } else {
    r["lse_units"] = "log2";
  }
  if (!a.out.empty()) {
    save_tensor(result.out, a.out + ".out.fpt");
    save_tensor(result.lse, a.out + ".lse.fpt");
    Json outs = Json::object();
    outs["out"] = a.out + ".out.fpt";
    outs["lse"] = a.out + ".lse.fpt";
    r["outputs"] = outs;
  }
  emit(r, a, ".report");
  return 0;
}

int cmd_sweep(const Args& a) {
  a.config.validate();
  if (a.pattern.empty()) throw UsageError("sweep requires --gen <pattern>");
  if (a.alphas.empty() && a.topks.empty() && a.topps.empty())
    throw UsageError("sweep requires a nonempty --alphas, --topks, or --topps list");
  std::vector<std::uint64_t> lengths = a.lengths;
  if (lengths.empty()) lengths.push_back(a.L);
  Json r = base_report("sweep", a);
  r["workload"] = workload_echo(a);
  r["cells"] = Json::array();
  Json& cells = r["cells"];

  auto for_each_cell = [&](const std::function<void(const std::string&, double, const Selector&)>& run) {
    for (float al : a.alphas) run("max", al, Selector{"max", 0, 0.0f});
    for (std::uint32_t kk : a.topks) run("topk", kk, Selector{"topk", kk, 0.0f});
    for (float pp : a.topps) run("topp", pp, Selector{"topp", 0, pp});
  };

  for (const std::uint64_t L : lengths) {
    const BlockGrid g = make_block_grid(L, a.config.block_size);
    if (a.pattern == "heavy-tail") {  // selector-only sweep over synthetic score rows
      const auto map = cli::heavy_tail_sweep_map(g.num_query_blocks, a.head_mass, 0.2f, a.config.rng_seed);
      for_each_cell([&](const std::string& method, double param, const Selector& sel) {
        PipelineConfig c = a.config;
        if (method == "max") c.alpha = static_cast<float>(param);
        const ActiveMask mask = run_selector(sel, map.score, c);
        const SparseBlockPlan plan = compress_indices(mask);
        std::size_t heavy = 0, hits = 0;
        for (std::uint32_t i = 0; i < g.num_query_blocks; ++i) {
          if (map.head_index[i] < 0) continue;
          ++heavy;
          hits += mask.active(0, i, static_cast<std::uint64_t>(map.head_index[i]), 0) ? 1 : 0;
        }
        Json cell = Json::object();
        cell["method"] = method;
        cell["param"] = param;
        cell["L"] = static_cast<unsigned long long>(L);
        cell["density"] = density(plan, g);
        cell["visit_count"] = static_cast<unsigned long long>(visit_count(plan));
        cell["head_retention"] = heavy == 0 ? 1.0 : static_cast<double>(hits) / static_cast<double>(heavy);
        cells.push_back(cell);
      });
      continue;
    }
    Timer tg;
    const cli::Workload w = build_workload(a, L, "");  // per-length default targets stay in range
    const double gen_ms = tg.ms();
    const float tau = a.config.resolved_scale(w.q.head_dim());
    Timer td;
    const BlockScoreMap map = discover(w.q, w.k, g, tau, a.config.epsilon);
    const double disc_ms = td.ms();
    Timer tdn;
    const AttentionOutput dense = dense_attention(w.q, w.k, w.v, tau);
    const double dense_ms = tdn.ms();
    const double full = static_cast<double>(w.q.batch()) * static_cast<double>(w.q.heads()) *
                        g.num_query_blocks * (g.num_query_blocks + 1) / 2.0;
    for_each_cell([&](const std::string& method, double param, const Selector& sel) {
      PipelineConfig c = a.config;
      if (method == "max") c.alpha = static_cast<float>(param);
      Timer ts;
      const ActiveMask mask = run_selector(sel, map.score, c);
      const SparseBlockPlan plan = compress_indices(mask);
      const double sel_ms = ts.ms();
      Timer ta;
      AttentionStats st;
      const AttentionOutput sp = block_sparse_attention(w.q, w.k, w.v, plan, g, tau, &st);
      const double att_ms = ta.ms();
      const auto err = cli::tensor_error(sp.out, dense.out);
      Json tm = Json::object();
      tm["generate"] = gen_ms;
      tm["discover"] = disc_ms;
      tm["attend_dense"] = dense_ms;
      tm["select"] = sel_ms;
      tm["attend_sparse"] = att_ms;
      Json cell = Json::object();
      cell["method"] = method;
      cell["param"] = param;
      cell["L"] = static_cast<unsigned long long>(L);
      cell["density"] = density(plan, g);
      cell["visit_count"] = static_cast<unsigned long long>(visit_count(plan));
      cell["block_visits"] = static_cast<unsigned long long>(st.block_visits);
      cell["visit_fraction"] = static_cast<double>(st.block_visits) / full;
      cell["recall"] = cli::planted_score_recall(map.score, w.gt,
                                                 static_cast<float>(method == "max" ? param : c.alpha));
      cell["mask_recall"] = cli::mask_recall(mask, w.gt);
      cell["mask_precision"] = cli::mask_precision(mask, w.gt);
      cell["err_max_abs"] = err.max_abs;
      cell["err_mean_abs"] = err.mean_abs;
      cell["timings_ms"] = tm;
      cells.push_back(cell);
    });
  }
  emit(r, a, "");
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    if (a.sub == "gen") return cmd_gen(a);
    if (a.sub == "discover") return cmd_discover(a);
    if (a.sub == "select") return cmd_select(a);
    if (a.sub == "attend") return cmd_attend(a);
    return cmd_sweep(a);
  } catch (const UsageError& e) {
    std::cerr << "usage error: " << e.what() << "\n" << kUsage;
    return 1;
  } catch (const PlanError& e) {
    std::cerr << "plan error: " << e.what() << "\n";
    return 2;
  } catch (const ConfigError& e) {
    std::cerr << "config error: " << e.what() << "\n";
    return 2;
  } catch (const ValidationError& e) {
    std::cerr << "validation error: " << e.what() << "\n";
    return 2;
  } catch (const FormatError& e) {
    std::cerr << "format error: " << e.what() << "\n";
    return 3;
  } catch (const IoError& e) {
    std::cerr << "io error: " << e.what() << "\n";
    return 3;
  } catch (const CudaError& e) {
    std::cerr << "cuda error: " << e.what() << "\n";
    return 4;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
}
