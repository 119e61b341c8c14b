// abi.cu — the C ABI (include/fpb200.h): validation, workspace carving, tensor maps, launches,
// and the host-buffer entry points the C++ drop-in layer uses.
//
// Validation mirrors the reference's exceptions (return code 2 == ValidationError / ConfigError /
// PlanError):  PipelineConfig::validate (core.hpp:96-101), make_block_grid (core.hpp:31-41),
// require_same_shape / require_qkv (core.hpp:81-85, attention.hpp:25-30), plan shape
// (attention.hpp:47-49) and the per-visit block range check (attention.hpp:78-81).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fpb200.h"
#include "fp_kernels.h"

namespace fpb {

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(FPB_ECUDA, "%s: CUDA error %d (%s)", where, (int)e, cudaGetErrorString(e));
}

#define FPB_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);  \
  } while (0)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

size_t align_up(size_t x, size_t a = 1024) { return (x + a - 1) / a * a; }

// Resolves the problem into kernel dims; returns 0 or an error code.
int resolve(const fpb_problem* p, Dims* D) {
  if (!p) return fail(FPB_EUSAGE, "null problem");
  if (p->Z < 1 || p->Hq < 1 || p->Hkv < 1 || p->L < 1 || p->d < 1)
    return fail(FPB_EVALIDATION, "sequence batch dims must be >= 1");
  if (p->Hq % p->Hkv) return fail(FPB_EVALIDATION, "Hq must be a multiple of Hkv");
  if (p->block_size < 1) return fail(FPB_EVALIDATION, "block_size must be >= 1");
  if (!(p->alpha >= 0.0f)) return fail(FPB_EVALIDATION, "alpha must be >= 0");
  if (p->window_tokens < 1) return fail(FPB_EVALIDATION, "window_tokens must be >= 1");
  if (p->sink_tokens < 0) return fail(FPB_EVALIDATION, "sink_tokens must be >= 0");
  if (!(p->epsilon > 0.0f)) return fail(FPB_EVALIDATION, "epsilon must be > 0");
  if (p->d > 1024) return fail(FPB_EVALIDATION, "head_dim %lld too large (max 1024)", (long long)p->d);
  if (p->block_size > 4096)
    return fail(FPB_EVALIDATION, "block_size %d too large (max 4096)", p->block_size);
  if (p->L > (int64_t)1 << 30 || p->Z * p->Hq > (int64_t)1 << 24 ||
      (p->L + p->block_size - 1) / p->block_size > 65535)
    return fail(FPB_EVALIDATION, "problem too large");
  D->Z = (int)p->Z;
  D->Hq = (int)p->Hq;
  D->Hkv = (int)p->Hkv;
  D->L = (int)p->L;
  D->B = p->block_size;
  D->d = (int)p->d;
  D->M = (int)((p->L + D->B - 1) / D->B);
  D->group = D->Hq / D->Hkv;
  D->last_len = (int)(p->L - (int64_t)(D->M - 1) * D->B);
  const float tau = p->scale > 0.0f ? p->scale : 1.0f / sqrtf((float)p->d);  // core.hpp:109-111
  D->to_bits = tau * kLog2e;
  D->eps = p->epsilon;
  D->alpha = p->alpha;
  D->sink_blocks = (p->sink_tokens + D->B - 1) / D->B;      // core.hpp:103-105
  D->window_blocks = (p->window_tokens + D->B - 1) / D->B;  // core.hpp:106-108
  D->rb = 0;
  D->rs = 1;
  D->Mr = D->M;
  D->zz = D->zh_end = D->zh_n = D->zl_end = 0;
  return FPB_OK;
}

// Restrict a resolved problem to the query blocks I = row_begin + row_step * k.
int restrict_rows(Dims* D, int32_t row_begin, int32_t row_step) {
  if (row_step < 1 || row_begin < 0 || row_begin >= row_step)
    return fail(FPB_EVALIDATION, "row shard needs 0 <= row_begin < row_step");
  if (row_step > 1 && !(D->d == kHeadDim && D->B == kBlock))
    return fail(FPB_EVALIDATION, "row sharding needs d = block_size = 128");
  D->rb = row_begin;
  D->rs = row_step;
  D->Mr = row_begin < D->M ? (D->M - row_begin + row_step - 1) / row_step : 0;
  return FPB_OK;
}

// Restrict a resolved problem to rank's zigzag shard of world: chunks `rank` and
// `2 world - 1 - rank` of 2 world contiguous chunks of ceil(M / (2 world)) query blocks.
int restrict_zigzag(Dims* D, int32_t rank, int32_t world) {
  if (world < 1 || rank < 0 || rank >= world)
    return fail(FPB_EVALIDATION, "zigzag shard needs 0 <= rank < world");
  if (world > 1 && !(D->d == kHeadDim && D->B == kBlock))
    return fail(FPB_EVALIDATION, "row sharding needs d = block_size = 128");
  const int64_t c = (D->M + 2 * (int64_t)world - 1) / (2 * (int64_t)world);
  const int64_t hi0 = (2 * (int64_t)world - 1 - rank) * c, lo0 = rank * c;
  const int64_t hi1 = std::min<int64_t>(D->M, hi0 + c), lo1 = std::min<int64_t>(D->M, lo0 + c);
  D->zz = 1;
  D->zh_end = (int)hi1;
  D->zh_n = (int)std::max<int64_t>(0, hi1 - hi0);
  D->zl_end = (int)lo1;
  D->Mr = D->zh_n + (int)std::max<int64_t>(0, lo1 - lo0);
  return FPB_OK;
}

// The tcgen05/TMA kernels cover the tile shape d = B = 128; every other shape the reference
// accepts runs the SIMT kernels of generic.cu.
bool tc_path(const Dims& D) { return D.d == kHeadDim && D.B == kBlock; }

// The tcgen05 path moves Q / K / V / O with TMA tensor maps, bulk copies and 16-byte vector
// accesses: their base addresses must be 16-byte aligned (a misaligned view would fault).
int check_align16(std::initializer_list<const void*> ptrs) {
  for (const void* q : ptrs)
    if (reinterpret_cast<uintptr_t>(q) & 15u)
      return fail(FPB_EVALIDATION, "tensor base address %p is not 16-byte aligned", q);
  return FPB_OK;
}

int check_dtype(fpb_dtype t) {
  return (t == FPB_F32 || t == FPB_BF16) ? FPB_OK : fail(FPB_EUSAGE, "bad dtype %d", (int)t);
}

size_t q_elems(const Dims& D) { return (size_t)D.Z * D.Hq * D.L * D.d; }
size_t kv_elems(const Dims& D) { return (size_t)D.Z * D.Hkv * D.L * D.d; }
size_t map_elems(const Dims& D) { return (size_t)D.Z * D.Hq * D.M * D.M; }
size_t pooled_bytes(const Dims& D) { return (size_t)D.Z * D.Hkv * D.M * D.d * 4; }
size_t kbar_split_bytes(const Dims& D) { return 2ull * D.Z * D.Hkv * D.M * kHeadDim * 2; }

// Workspace layouts.  discover: [scheduler counter][kbar split][Q hi/lo planes if fp32]
//                     attention: [Q hi/lo][K hi/lo][V bf16] if fp32
//   generic discover: [pooled][energy][local_max][score][mask]
constexpr size_t kSchedBytes = 1024;
constexpr size_t kMaxSmemPerCta = 227 * 1024;  // sm_100 opt-in dynamic shared memory per CTA
size_t ws_discover(const Dims& D, fpb_dtype t) {
  if (!tc_path(D))
    return align_up(pooled_bytes(D)) + 3 * align_up(map_elems(D) * 4) + align_up(map_elems(D));
  size_t b = kSchedBytes + align_up(kbar_split_bytes(D)) + align_up(discover_scratch_bytes(D));
  if (t == FPB_F32) b += align_up(2 * q_elems(D) * 2);
  b += D.M < 1024 ? align_up(discover_rows_bytes(D)) : 0;  // two-pass plan-only mode
  return b + align_up(discover_pool_ctr_bytes(D));         // in-kernel pooling counters
}
struct DiscWs {
  int* sched;
  __nv_bfloat16* kbar;
  float* mscratch;         // long sequences only (discover_scratch_bytes)
  __nv_bfloat16* qplanes;  // fp32 inputs only
  float2* rows;            // two-pass plan-only mode (discover_rows_bytes)
  int* pool_ctr;           // in-kernel pooling (bf16 keys): claim + per-chunk counters
};
DiscWs disc_ws(const Dims& D, void* ws, fpb_dtype t = FPB_BF16) {
  uint8_t* w = static_cast<uint8_t*>(ws);
  const size_t o1 = kSchedBytes + align_up(kbar_split_bytes(D));
  const size_t sb = discover_scratch_bytes(D);
  const size_t o2 = o1 + align_up(sb);
  const size_t o3 = o2 + (t == FPB_F32 ? align_up(2 * q_elems(D) * 2) : 0);
  const size_t o4 = o3 + (D.M < 1024 ? align_up(discover_rows_bytes(D)) : 0);
  return {reinterpret_cast<int*>(w), reinterpret_cast<__nv_bfloat16*>(w + kSchedBytes),
          sb ? reinterpret_cast<float*>(w + o1) : nullptr,
          reinterpret_cast<__nv_bfloat16*>(w + o2), reinterpret_cast<float2*>(w + o3),
          // the counters share the work counter's zeroed block when they fit (one memset)
          discover_pool_ctr_bytes(D) + sizeof(int) <= kSchedBytes ? reinterpret_cast<int*>(w) + 1
                                                                  : reinterpret_cast<int*>(w + o4)};
}
// attention: [sched][plan-row scratch] + fp32: Q hi/lo, K hi/lo, V bf16
size_t ws_attention(const Dims& D, fpb_dtype t) {
  if (!tc_path(D)) return align_up(g_attention_scratch_bytes(D));
  return kSchedBytes + align_up(attention_list_bytes(D)) +
         (t == FPB_F32 ? align_up(2 * q_elems(D) * 2) + align_up(2 * kv_elems(D) * 2) +
                             align_up(kv_elems(D) * 2)
                       : align_up(attention_phase_bytes(D)));
}

cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#ifndef FPB_DISC_TWO_PASS
#define FPB_DISC_TWO_PASS 1  // plan-only discovery as kernel + warp-per-row select kernel
#endif

int need_ws(size_t have, size_t need, void* ws) {
  if (need && (!ws || have < need))
    return fail(FPB_EUSAGE, "workspace too small: need %zu bytes, have %zu", need, have);
  return FPB_OK;
}

// Discovery front half for fp32 inputs: pool k̄ (+split) and stage the Q planes; returns the Q
// plane pointer.  bf16 inputs need nothing: the discovery kernel pools K itself.
int discover_prepare(const Dims& D, fpb_dtype t, const void* Q, const void* K, float* pooled,
                     const DiscWs& w, cudaStream_t st, const __nv_bfloat16** q_planes) {
  if (t == FPB_F32) FPB_CUDA(launch_pool_keys(D, false, K, pooled, w.kbar, st));
  if (t == FPB_BF16) {
    *q_planes = static_cast<const __nv_bfloat16*>(Q);
  } else {
    FPB_CUDA(launch_f32_to_bf16(static_cast<const float*>(Q), w.qplanes, w.qplanes + q_elems(D),
                                q_elems(D), st));
    *q_planes = w.qplanes;
  }
  return FPB_OK;
}

}  // namespace

bool make_tmap_rows128(CUtensorMap* map, const void* base, uint64_t rows, uint64_t planes) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)kHeadDim, rows, planes};
  cuuint64_t strides[2] = {(cuuint64_t)kHeadDim * 2, rows * kHeadDim * 2};
  cuuint32_t box[3] = {64, 128, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Whole 128 x 128 bf16 tile in ONE TMA: the two 64-column SW128 halves become a third box
// dimension (dims: 64 columns, rows, 2 halves, planes; the half stride, 128 B, is below the row
// stride), so shared memory receives [half][row][64] exactly as two 3-D loads would.
bool make_tmap_tiles128(CUtensorMap* map, const void* base, uint64_t rows, uint64_t planes,
                        uint32_t box_halves) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {64, rows, 2, planes};
  cuuint64_t strides[3] = {(cuuint64_t)kHeadDim * 2, 128, rows * kHeadDim * 2};
  cuuint32_t box[4] = {64, 128, box_halves, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace fpb

using namespace fpb;

extern "C" {

void fpb_problem_init(fpb_problem* p, int64_t Z, int64_t Hq, int64_t Hkv, int64_t L, int64_t d) {
  p->Z = Z;
  p->Hq = Hq;
  p->Hkv = Hkv;
  p->L = L;
  p->d = d;
  p->block_size = 128;
  p->alpha = 0.12f;
  p->sink_tokens = 256;
  p->window_tokens = 512;
  p->scale = 0.0f;
  p->epsilon = 1e-10f;
}

int fpb_version(void) { return 1; }

const char* fpb_last_error(void) { return g_err.c_str(); }

int fpb_workspace_bytes(const fpb_problem* p, fpb_dtype dtype, size_t* bytes) {
  Dims D;
  int rc = resolve(p, &D);
  if (rc || (rc = check_dtype(dtype))) return rc;
  if (!bytes) return fail(FPB_EUSAGE, "null bytes");
  const size_t a = ws_discover(D, dtype), b = ws_attention(D, dtype);
  *bytes = a > b ? a : b;
  return FPB_OK;
}

int fpb_pool_keys(const fpb_problem* p, fpb_dtype dtype, const void* K, float* pooled,
                  void* stream) {
  Dims D;
  int rc = resolve(p, &D);
  if (rc || (rc = check_dtype(dtype))) return rc;
  if (!K || !pooled) return fail(FPB_EUSAGE, "null pointer");
  if (tc_path(D) && (rc = check_align16({K}))) return rc;
  if (tc_path(D))
    FPB_CUDA(launch_pool_keys(D, dtype == FPB_BF16, K, pooled, nullptr, S(stream)));
  else
    FPB_CUDA(g_launch_pool(D, dtype == FPB_BF16, K, pooled, S(stream)));
  return FPB_OK;
}

int fpb_approx_block_scores(const fpb_problem* p, fpb_dtype dtype, const void* Q,
                            const float* pooled, float* energy, float* local_max, void* workspace,
                            size_t workspace_bytes, void* stream) {
  Dims D;
  int rc = resolve(p, &D);
  if (rc || (rc = check_dtype(dtype))) return rc;
  if (!Q || !pooled || !energy || !local_max) return fail(FPB_EUSAGE, "null pointer");
  if (!tc_path(D)) {
    FPB_CUDA(g_launch_approx(D, dtype == FPB_BF16, Q, pooled, energy, local_max, S(stream)));
    return FPB_OK;
  }
  if ((rc = need_ws(workspace_bytes, ws_discover(D, dtype), workspace))) return rc;
  if ((rc = check_align16({Q}))) return rc;
  const DiscWs w = disc_ws(D, workspace, dtype);
  FPB_CUDA(launch_split_pooled(D, pooled, w.kbar, S(stream)));
  const __nv_bfloat16* qp = static_cast<const __nv_bfloat16*>(Q);
  if (dtype == FPB_F32) {
    FPB_CUDA(launch_f32_to_bf16(static_cast<const float*>(Q), w.qplanes, w.qplanes + q_elems(D),
                                q_elems(D), S(stream)));
    qp = w.qplanes;
  }
  DiscoverOut o;
  o.energy = energy;
  o.local_max = local_max;
  o.normalize = false;
  FPB_CUDA(launch_discover(D, dtype == FPB_F32 ? 2 : 1, qp, w.kbar, o, w.sched, w.mscratch,
                           S(stream)));
  return FPB_OK;
}

int fpb_normalize_block_scores(const fpb_problem* p, const float* energy, const float* local_max,
                               float* score, void* stream) {
  Dims D;
  int rc = resolve(p, &D);
  if (rc) return rc;
  if (!energy || !local_max || !score) return fail(FPB_EUSAGE, "null pointer");
  FPB_CUDA(launch_normalize(D, energy, local_max, score, S(stream)));
  return FPB_OK;
}

static int discover_select_rows(const fpb_problem* p, int32_t row_begin, int32_t row_step,
                                fpb_dtype dtype, const void* Q, const void* K, float* energy,
                                float* local_max, float* score, uint8_t* mask, int32_t* idx,
                                int32_t* counts, void* workspace, size_t workspace_bytes,
                                void* stream, bool zigzag = false) {
  Dims D;
  int rc = resolve(p, &D);
  if (rc || (rc = check_dtype(dtype)) ||
      (rc = zigzag ? restrict_zigzag(&D, row_begin, row_step)
                   : restrict_rows(&D, row_begin, row_step)))
    return rc;
  if (!Q || !K) return fail(FPB_EUSAGE, "null pointer");
  if ((idx == nullptr) != (counts == nullptr))
    return fail(FPB_EUSAGE, "idx and counts must be given together");
  if ((rc = need_ws(workspace_bytes, ws_discover(D, dtype), workspace))) return rc;
  if (!tc_path(D)) {  // pool -> approx -> normalize -> threshold -> compress, SIMT kernels
    uint8_t* w = static_cast<uint8_t*>(workspace);
    const size_t mb = align_up(map_elems(D) * 4);
    float* pooled = reinterpret_cast<float*>(w);
    float* en = reinterpret_cast<float*>(w + align_up(pooled_bytes(D)));
    float* lm = reinterpret_cast<float*>(w + align_up(pooled_bytes(D)) + mb);
    float* sc = reinterpret_cast<float*>(w + align_up(pooled_bytes(D)) + 2 * mb);
    uint8_t* mk = w + align_up(pooled_bytes(D)) + 3 * mb;
    en = energy ? energy : en;
    lm = local_max ? local_max : lm;
    sc = score ? score : sc;
    mk = mask ? mask : mk;
    FPB_CUDA(g_launch_pool(D, dtype == FPB_BF16, K, pooled, S(stream)));
    FPB_CUDA(g_launch_approx(D, dtype == FPB_BF16, Q, pooled, en, lm, S(stream)));
    FPB_CUDA(launch_normalize(D, en, lm, sc, S(stream)));
    if (idx || mask) {
      FPB_CUDA(launch_threshold(D, sc, mk, nullptr, S(stream)));
      if (idx) FPB_CUDA(launch_compress(D, mk, idx, counts, S(stream)));
    }
    return FPB_OK;
  }
  if (D.Mr == 0) return FPB_OK;  // this row shard owns no query block
  if ((rc = check_align16({Q, K}))) return rc;
  const DiscWs w = disc_ws(D, workspace, dtype);
  const __nv_bfloat16* qp;
  if ((rc = discover_prepare(D, dtype, Q, K, nullptr, w, S(stream), &qp))) return rc;
  DiscoverOut o;
  o.energy = energy;
  o.local_max = local_max;
  o.score = score;
  o.mask = mask;
  o.idx = idx;
  o.counts = counts;
  // plan-only calls (the hot path) up to 128K tokens: two passes, the discovery kernel keeps no
  // per-item tail (32K: 0.133 -> 0.126 ms; no gain for longer rows, profiles/r1_ab_disc_two_pass)
  if (FPB_DISC_TWO_PASS && D.M < 1024 && idx && !energy && !local_max && !score && !mask)
    o.rows = w.rows;
  const bool fused_pool = dtype == FPB_BF16;  // the discovery kernel pools the bf16 keys itself
  FPB_CUDA(launch_discover(D, dtype == FPB_F32 ? 2 : 1, qp, w.kbar, o, w.sched, w.mscratch,
                           S(stream), fused_pool ? static_cast<const __nv_bfloat16*>(K) : nullptr,
                           nullptr, w.pool_ctr));
  return FPB_OK;
}

int fpb_discover_select(const fpb_problem* p, fpb_dtype dtype, const void* Q, const void* K,
                        float* energy, float* local_max, float* score, uint8_t* mask, int32_t* idx,
                        int32_t* counts, void* workspace, size_t workspace_bytes, void* stream) {
  return discover_select_rows(p, 0, 1, dtype, Q, K, energy, local_max, score, mask, idx, counts,
                              workspace, workspace_bytes, stream);
}

int fpb_discover_select_rows(const fpb_problem* p, int32_t row_begin, int32_t row_step,
                             fpb_dtype dtype, const void* Q, const void* K, float* energy,
                             float* local_max, float* score, uint8_t* mask, int32_t* idx,
                             int32_t* counts, void* workspace, size_t workspace_bytes,
                             void* stream) {
  return discover_select_rows(p, row_begin, row_step, dtype, Q, K, energy, local_max, score, mask,
                              idx, counts, workspace, workspace_bytes, stream);
}

int fpb_discover_select_zigzag(const fpb_problem* p, int32_t rank, int32_t world,
                               fpb_dtype dtype, const void* Q, const void* K, float* energy,
                               float* local_max, float* score, uint8_t* mask, int32_t* idx,
                               int32_t* counts, void* workspace, size_t workspace_bytes,
                               void* stream) {
  return discover_select_rows(p, rank, world, dtype, Q, K, energy, local_max, score, mask, idx,
                              counts, workspace, workspace_bytes, stream, true);
}

int fpb_discover(const fpb_problem* p, fpb_dtype dtype, const void* Q, const void* K,
                 float* energy, float* local_max, float* score, void* workspace,
                 size_t workspace_bytes, void* stream) {
  if (!score) return fail(FPB_EUSAGE, "null score");
  return fpb_discover_select(p, dtype, Q, K, energy, local_max, score, nullptr, nullptr, nullptr,
                             workspace, workspace_bytes, stream);
}

static int sort_select(const fpb_problem* p, const float* score, int mode, int32_t k,
                       float top_p, uint8_t* mask, void* stream) {
  Dims D;
  int rc = resolve(p, &D);
  if (rc) return rc;
  if (!score || !mask) return fail(FPB_EUSAGE, "null pointer");
  if (mode == 0 && k < 1) return fail(FPB_EVALIDATION, "top-k requires k >= 1");
  if (mode == 1 && (!(top_p > 0.0f) || top_p > 1.0f))
    return fail(FPB_EVALIDATION, "top-p requires p in (0, 1]");
  if (D.M > 4096) return fail(FPB_EVALIDATION, "top-k/top-p rows limited to 4096 blocks");
  FPB_CUDA(launch_sort_select(D, score, mask, mode, k, top_p, S(stream)));
  return FPB_OK;
}

int fpb_topk_select(const fpb_problem* p, const float* score, int32_t k, uint8_t* mask,
                    void* stream) {
  return sort_select(p, score, 0, k, 0.f, mask, stream);
}

int fpb_topp_select(const fpb_problem* p, const float* score, float top_p, uint8_t* mask,
                    void* stream) {
  return sort_select(p, score, 1, 1, top_p, mask, stream);
}

int fpb_baseline_workspace_bytes(const fpb_problem* p, size_t* bytes) {
  Dims D;
  int rc = resolve(p, &D);
  if (rc) return rc;
  if (!bytes) return fail(FPB_EUSAGE, "null bytes");
  const size_t pq = (size_t)D.Z * D.Hq * D.M * D.d * 4;
  const size_t both = align_up(pq) + align_up(pooled_bytes(D));
  const size_t exact = align_up(pooled_bytes(D)) + align_up(exact_table_bytes(D));
  *bytes = both > exact ? both : exact;
  return FPB_OK;
}

int fpb_discover_pool_both(const fpb_problem* p, fpb_dtype dtype, const void* Q, const void* K,
                           float* energy, float* local_max, float* score, void* workspace,
                           size_t workspace_bytes, void* stream) {
  Dims D;
  int rc = resolve(p, &D);
  if (rc || (rc = check_dtype(dtype))) return rc;
  if (!Q || !K || !energy || !local_max || !score) return fail(FPB_EUSAGE, "null pointer");
  size_t need;
  fpb_baseline_workspace_bytes(p, &need);
  if ((rc = need_ws(workspace_bytes, need, workspace))) return rc;
  uint8_t* w = static_cast<uint8_t*>(workspace);
  float* pq = reinterpret_cast<float*>(w);
  float* pk = reinterpret_cast<float*>(w + align_up((size_t)D.Z * D.Hq * D.M * D.d * 4));
  FPB_CUDA(launch_pool_both(D, dtype == FPB_BF16, Q, K, pq, pk, energy, local_max, S(stream)));
  FPB_CUDA(launch_normalize(D, energy, local_max, score, S(stream)));
  return FPB_OK;
}

int fpb_discover_exact(const fpb_problem* p, fpb_dtype dtype, const void* Q, const void* K,
                       float* energy, float* local_max, float* score, void* workspace,
                       size_t workspace_bytes, void* stream) {
  Dims D;
  int rc = resolve(p, &D);
  if (rc || (rc = check_dtype(dtype))) return rc;
  if (!Q || !K || !energy || !local_max || !score) return fail(FPB_EUSAGE, "null pointer");
  size_t need;
  fpb_baseline_workspace_bytes(p, &need);
  if ((rc = need_ws(workspace_bytes, need, workspace))) return rc;
  uint8_t* w = static_cast<uint8_t*>(workspace);
  float* pk = reinterpret_cast<float*>(w);
  float* table = reinterpret_cast<float*>(w + align_up(pooled_bytes(D)));
  FPB_CUDA(launch_exact(D, dtype == FPB_BF16, Q, K, pk, table, energy, local_max, score,
                        S(stream)));
  return FPB_OK;
}

int fpb_max_threshold_mask(const fpb_problem* p, const float* score, uint8_t* mask,
                           unsigned long long* comparisons, void* stream) {
  Dims D;
  int rc = resolve(p, &D);
  if (rc) return rc;
  if (!score || !mask) return fail(FPB_EUSAGE, "null pointer");
  FPB_CUDA(launch_threshold(D, score, mask, comparisons, S(stream)));
  return FPB_OK;
}

int fpb_compress_indices(const fpb_problem* p, const uint8_t* mask, int32_t* idx, int32_t* counts,
                         void* stream) {
  Dims D;
  int rc = resolve(p, &D);
  if (rc) return rc;
  if (!mask || !idx || !counts) return fail(FPB_EUSAGE, "null pointer");
  FPB_CUDA(launch_compress(D, mask, idx, counts, S(stream)));
  return FPB_OK;
}

int fpb_visit_count(const fpb_problem* p, const int32_t* counts, unsigned long long* total,
                    void* stream) {
  Dims D;
  int rc = resolve(p, &D);
  if (rc) return rc;
  if (!counts || !total) return fail(FPB_EUSAGE, "null pointer");
  FPB_CUDA(launch_visit_count(D, counts, total, S(stream)));
  return FPB_OK;
}

int fpb_full_causal_plan(const fpb_problem* p, int32_t* idx, int32_t* counts, void* stream) {
  Dims D;
  int rc = resolve(p, &D);
  if (rc) return rc;
  if (!idx || !counts) return fail(FPB_EUSAGE, "null pointer");
  FPB_CUDA(launch_full_causal_plan(D, idx, counts, S(stream)));
  return FPB_OK;
}

}  // extern "C"

static int attention_common(const fpb_problem* p, fpb_dtype dtype, const void* Q, const void* K,
                            const void* V, const int32_t* idx, const int32_t* counts,
                            fpb_dtype out_dtype, void* out, float* lse,
                            unsigned long long* visits, int32_t* plan_error, void* workspace,
                            size_t workspace_bytes, void* stream, int32_t row_begin = 0,
                            int32_t row_step = 1, bool zigzag = false) {
  Dims D;
  int rc = resolve(p, &D);
  if (rc || (rc = check_dtype(dtype)) || (rc = check_dtype(out_dtype)) ||
      (rc = zigzag ? restrict_zigzag(&D, row_begin, row_step)
                   : restrict_rows(&D, row_begin, row_step)))
    return rc;
  if (!Q || !K || !V || !out || !lse) return fail(FPB_EUSAGE, "null pointer");
  if ((rc = need_ws(workspace_bytes, ws_attention(D, dtype), workspace))) return rc;
  if (D.Mr == 0) return FPB_OK;  // this row shard owns no query block
  if (!tc_path(D)) {
    FPB_CUDA(g_launch_attention(D, dtype == FPB_BF16, Q, K, V, idx, counts,
                                out_dtype == FPB_BF16, out, lse, visits, plan_error,
                                static_cast<float*>(workspace), S(stream)));
    return FPB_OK;
  }
  if ((rc = check_align16({Q, K, V, out}))) return rc;
  const __nv_bfloat16 *q = static_cast<const __nv_bfloat16*>(Q),
                      *k = static_cast<const __nv_bfloat16*>(K),
                      *v = static_cast<const __nv_bfloat16*>(V);
  if (dtype == FPB_F32) {
    // the split-precision one-tile kernel keeps its block list in shared memory
    if (attention_f32_smem_bytes(D) > kMaxSmemPerCta)
      return fail(FPB_EVALIDATION,
                  "fp32 inputs support at most %d key blocks (got %d); pass bf16 for longer "
                  "sequences",
                  (int)((kMaxSmemPerCta - attention_f32_smem_bytes(Dims{})) / sizeof(int)), D.M);
    uint8_t* w = static_cast<uint8_t*>(workspace) + kSchedBytes + align_up(attention_list_bytes(D));
    __nv_bfloat16* q2 = reinterpret_cast<__nv_bfloat16*>(w);
    __nv_bfloat16* k2 = reinterpret_cast<__nv_bfloat16*>(w + align_up(2 * q_elems(D) * 2));
    __nv_bfloat16* v2 = reinterpret_cast<__nv_bfloat16*>(w + align_up(2 * q_elems(D) * 2) +
                                                         align_up(2 * kv_elems(D) * 2));
    FPB_CUDA(launch_f32_to_bf16(static_cast<const float*>(Q), q2, q2 + q_elems(D), q_elems(D),
                                S(stream)));
    FPB_CUDA(launch_f32_to_bf16(static_cast<const float*>(K), k2, k2 + kv_elems(D), kv_elems(D),
                                S(stream)));
    FPB_CUDA(launch_f32_to_bf16(static_cast<const float*>(V), v2, nullptr, kv_elems(D), S(stream)));
    q = q2;
    k = k2;
    v = v2;
  }
  uint8_t* wsb = static_cast<uint8_t*>(workspace);
  FPB_CUDA(launch_attention(D, dtype == FPB_F32 ? 2 : 1, q, k, v, idx, counts,
                            out_dtype == FPB_BF16, out, lse, visits, plan_error,
                            reinterpret_cast<int*>(wsb),
                            reinterpret_cast<uint16_t*>(wsb + kSchedBytes),
                            wsb + kSchedBytes + align_up(attention_list_bytes(D)), S(stream)));
  return FPB_OK;
}

extern "C" {

int fpb_block_sparse_attention(const fpb_problem* p, fpb_dtype dtype, const void* Q, const void* K,
                               const void* V, const int32_t* idx, const int32_t* counts,
                               fpb_dtype out_dtype, void* out, float* lse,
                               unsigned long long* visits, int32_t* plan_error, void* workspace,
                               size_t workspace_bytes, void* stream) {
  if (!idx || !counts) return fail(FPB_EUSAGE, "null plan");
  return attention_common(p, dtype, Q, K, V, idx, counts, out_dtype, out, lse, visits, plan_error,
                          workspace, workspace_bytes, stream);
}

int fpb_block_sparse_attention_rows(const fpb_problem* p, int32_t row_begin, int32_t row_step,
                                    fpb_dtype dtype, const void* Q, const void* K, const void* V,
                                    const int32_t* idx, const int32_t* counts,
                                    fpb_dtype out_dtype, void* out, float* lse,
                                    unsigned long long* visits, int32_t* plan_error,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  if (!idx || !counts) return fail(FPB_EUSAGE, "null plan");
  return attention_common(p, dtype, Q, K, V, idx, counts, out_dtype, out, lse, visits, plan_error,
                          workspace, workspace_bytes, stream, row_begin, row_step);
}

int fpb_block_sparse_attention_zigzag(const fpb_problem* p, int32_t rank, int32_t world,
                                      fpb_dtype dtype, const void* Q, const void* K,
                                      const void* V, const int32_t* idx, const int32_t* counts,
                                      fpb_dtype out_dtype, void* out, float* lse,
                                      unsigned long long* visits, int32_t* plan_error,
                                      void* workspace, size_t workspace_bytes, void* stream) {
  if (!idx || !counts) return fail(FPB_EUSAGE, "null plan");
  return attention_common(p, dtype, Q, K, V, idx, counts, out_dtype, out, lse, visits, plan_error,
                          workspace, workspace_bytes, stream, rank, world, true);
}

int fpb_dense_attention(const fpb_problem* p, fpb_dtype dtype, const void* Q, const void* K,
                        const void* V, fpb_dtype out_dtype, void* out, float* lse, void* workspace,
                        size_t workspace_bytes, void* stream) {
  return attention_common(p, dtype, Q, K, V, nullptr, nullptr, out_dtype, out, lse, nullptr,
                          nullptr, workspace, workspace_bytes, stream);
}

}  // extern "C"

// ------------------------------------------------------------------ host-buffer entry points
namespace {

// Grow-only per-thread device arena for the host entry points (no allocation on repeat calls).
struct Arena {
  void* ptr = nullptr;
  size_t cap = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t s_in = nullptr, s_out = nullptr;  // copy streams of the pipelined prefill
  cudaStream_t s_c2 = nullptr;                     // second compute stream of the prefill
  std::vector<cudaEvent_t> events;                 // grow-only pool of the prefill's chunk events
  ~Arena() {
    for (cudaEvent_t e : events) cudaEventDestroy(e);
    if (ptr) cudaFree(ptr);
    if (stream) cudaStreamDestroy(stream);
    if (s_in) cudaStreamDestroy(s_in);
    if (s_out) cudaStreamDestroy(s_out);
    if (s_c2) cudaStreamDestroy(s_c2);
  }
};
thread_local Arena g_arena;

// Drains every arena stream when a host entry point returns, so no async copy of the caller's
// host buffers (or kernel on the arena) is still in flight after an error return; on the success
// path the streams are already idle and this is a no-op.
struct ArenaDrain {
  ~ArenaDrain() {
    for (cudaStream_t s : {g_arena.stream, g_arena.s_in, g_arena.s_out, g_arena.s_c2})
      if (s) cudaStreamSynchronize(s);
  }
};

// n timing-disabled events from the arena's pool (created once, reused by every call)
int arena_events(size_t n, cudaEvent_t** out) {
  while (g_arena.events.size() < n) {
    cudaEvent_t e;
    FPB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    g_arena.events.push_back(e);
  }
  *out = g_arena.events.data();
  return FPB_OK;
}

int arena_get(size_t bytes, uint8_t** out, cudaStream_t* st) {
  if (!g_arena.stream) FPB_CUDA(cudaStreamCreateWithFlags(&g_arena.stream, cudaStreamNonBlocking));
  if (bytes > g_arena.cap) {
    if (g_arena.ptr) FPB_CUDA(cudaFree(g_arena.ptr));
    g_arena.ptr = nullptr;
    g_arena.cap = 0;
    FPB_CUDA(cudaMalloc(&g_arena.ptr, bytes));
    g_arena.cap = bytes;
  }
  *out = static_cast<uint8_t*>(g_arena.ptr);
  *st = g_arena.stream;
  return FPB_OK;
}

struct Carve {
  uint8_t* base;
  size_t off = 0;
  template <typename T>
  T* take(size_t bytes) {
    T* p = reinterpret_cast<T*>(base + off);
    off += align_up(bytes ? bytes : 1);
    return p;
  }
};

size_t dsz(fpb_dtype t) { return t == FPB_F32 ? 4 : 2; }

}  // namespace

extern "C" {

int fpb_host_pool_keys(const fpb_problem* p, fpb_dtype dtype, const void* K, float* pooled) {
  Dims D;
  ArenaDrain drain;  // error returns leave nothing in flight
  int rc = resolve(p, &D);
  if (rc || (rc = check_dtype(dtype))) return rc;
  if (!K || !pooled) return fail(FPB_EUSAGE, "null pointer");
  const size_t kb = kv_elems(D) * dsz(dtype), pb = pooled_bytes(D);
  uint8_t* base;
  cudaStream_t st;
  if ((rc = arena_get(align_up(kb) + align_up(pb), &base, &st))) return rc;
  Carve c{base};
  void* dk = c.take<void>(kb);
  float* dp = c.take<float>(pb);
  FPB_CUDA(cudaMemcpyAsync(dk, K, kb, cudaMemcpyHostToDevice, st));
  if ((rc = fpb_pool_keys(p, dtype, dk, dp, st))) return rc;
  FPB_CUDA(cudaMemcpyAsync(pooled, dp, pb, cudaMemcpyDeviceToHost, st));
  FPB_CUDA(cudaStreamSynchronize(st));
  return FPB_OK;
}

int fpb_host_approx_block_scores(const fpb_problem* p, fpb_dtype dtype, const void* Q,
                                 const float* pooled, float* energy, float* local_max) {
  Dims D;
  ArenaDrain drain;  // error returns leave nothing in flight
  int rc = resolve(p, &D);
  if (rc || (rc = check_dtype(dtype))) return rc;
  if (!Q || !pooled || !energy || !local_max) return fail(FPB_EUSAGE, "null pointer");
  const size_t qb = q_elems(D) * dsz(dtype), pb = pooled_bytes(D),
               mb = map_elems(D) * 4, wsb = ws_discover(D, dtype);
  uint8_t* base;
  cudaStream_t st;
  if ((rc = arena_get(align_up(qb) + align_up(pb) + 2 * align_up(mb) + align_up(wsb), &base, &st)))
    return rc;
  Carve c{base};
  void* dq = c.take<void>(qb);
  float* dp = c.take<float>(pb);
  float* de = c.take<float>(mb);
  float* dl = c.take<float>(mb);
  void* ws = c.take<void>(wsb);
  FPB_CUDA(cudaMemcpyAsync(dq, Q, qb, cudaMemcpyHostToDevice, st));
  FPB_CUDA(cudaMemcpyAsync(dp, pooled, pb, cudaMemcpyHostToDevice, st));
  if ((rc = fpb_approx_block_scores(p, dtype, dq, dp, de, dl, ws, wsb, st))) return rc;
  FPB_CUDA(cudaMemcpyAsync(energy, de, mb, cudaMemcpyDeviceToHost, st));
  FPB_CUDA(cudaMemcpyAsync(local_max, dl, mb, cudaMemcpyDeviceToHost, st));
  FPB_CUDA(cudaStreamSynchronize(st));
  return FPB_OK;
}

int fpb_host_normalize_block_scores(const fpb_problem* p, const float* energy,
                                    const float* local_max, float* score) {
  Dims D;
  ArenaDrain drain;  // error returns leave nothing in flight
  int rc = resolve(p, &D);
  if (rc) return rc;
  if (!energy || !local_max || !score) return fail(FPB_EUSAGE, "null pointer");
  const size_t mb = map_elems(D) * 4;
  uint8_t* base;
  cudaStream_t st;
  if ((rc = arena_get(3 * align_up(mb), &base, &st))) return rc;
  Carve c{base};
  float* de = c.take<float>(mb);
  float* dl = c.take<float>(mb);
  float* ds = c.take<float>(mb);
  FPB_CUDA(cudaMemcpyAsync(de, energy, mb, cudaMemcpyHostToDevice, st));
  FPB_CUDA(cudaMemcpyAsync(dl, local_max, mb, cudaMemcpyHostToDevice, st));
  if ((rc = fpb_normalize_block_scores(p, de, dl, ds, st))) return rc;
  FPB_CUDA(cudaMemcpyAsync(score, ds, mb, cudaMemcpyDeviceToHost, st));
  FPB_CUDA(cudaStreamSynchronize(st));
  return FPB_OK;
}

int fpb_host_discover(const fpb_problem* p, fpb_dtype dtype, const void* Q, const void* K,
                      float* energy, float* local_max, float* score) {
  Dims D;
  ArenaDrain drain;  // error returns leave nothing in flight
  int rc = resolve(p, &D);
  if (rc || (rc = check_dtype(dtype))) return rc;
  if (!Q || !K || !score) return fail(FPB_EUSAGE, "null pointer");
  const size_t qb = q_elems(D) * dsz(dtype), kb = kv_elems(D) * dsz(dtype),
               mb = map_elems(D) * 4, wsb = ws_discover(D, dtype);
  const size_t need = align_up(qb) + align_up(kb) + 3 * align_up(mb) + align_up(wsb);
  uint8_t* base;
  cudaStream_t st;
  if ((rc = arena_get(need, &base, &st))) return rc;
  Carve c{base};
  void* dq = c.take<void>(qb);
  void* dk = c.take<void>(kb);
  float* de = c.take<float>(mb);
  float* dl = c.take<float>(mb);
  float* ds = c.take<float>(mb);
  void* ws = c.take<void>(wsb);
  FPB_CUDA(cudaMemcpyAsync(dq, Q, qb, cudaMemcpyHostToDevice, st));
  FPB_CUDA(cudaMemcpyAsync(dk, K, kb, cudaMemcpyHostToDevice, st));
  if ((rc = fpb_discover(p, dtype, dq, dk, energy ? de : nullptr, local_max ? dl : nullptr, ds, ws,
                         wsb, st)))
    return rc;
  if (energy) FPB_CUDA(cudaMemcpyAsync(energy, de, mb, cudaMemcpyDeviceToHost, st));
  if (local_max) FPB_CUDA(cudaMemcpyAsync(local_max, dl, mb, cudaMemcpyDeviceToHost, st));
  FPB_CUDA(cudaMemcpyAsync(score, ds, mb, cudaMemcpyDeviceToHost, st));
  FPB_CUDA(cudaStreamSynchronize(st));
  return FPB_OK;
}

int fpb_host_max_threshold_mask(const fpb_problem* p, const float* score, uint8_t* mask,
                                unsigned long long* comparisons) {
  Dims D;
  ArenaDrain drain;  // error returns leave nothing in flight
  int rc = resolve(p, &D);
  if (rc) return rc;
  if (!score || !mask) return fail(FPB_EUSAGE, "null pointer");
  const size_t sb = map_elems(D) * 4, mb = map_elems(D);
  uint8_t* base;
  cudaStream_t st;
  if ((rc = arena_get(align_up(sb) + align_up(mb) + 1024, &base, &st))) return rc;
  Carve c{base};
  float* ds = c.take<float>(sb);
  uint8_t* dm = c.take<uint8_t>(mb);
  unsigned long long* dc = c.take<unsigned long long>(8);
  FPB_CUDA(cudaMemcpyAsync(ds, score, sb, cudaMemcpyHostToDevice, st));
  FPB_CUDA(cudaMemsetAsync(dc, 0, 8, st));
  if ((rc = fpb_max_threshold_mask(p, ds, dm, dc, st))) return rc;
  FPB_CUDA(cudaMemcpyAsync(mask, dm, mb, cudaMemcpyDeviceToHost, st));
  unsigned long long cmp = 0;
  FPB_CUDA(cudaMemcpyAsync(&cmp, dc, 8, cudaMemcpyDeviceToHost, st));
  FPB_CUDA(cudaStreamSynchronize(st));
  if (comparisons) *comparisons += cmp;
  return FPB_OK;
}

static int host_sort_select(const fpb_problem* p, const float* score, int mode, int32_t k,
                            float top_p, uint8_t* mask) {
  Dims D;
  ArenaDrain drain;  // error returns leave nothing in flight
  int rc = resolve(p, &D);
  if (rc) return rc;
  if (!score || !mask) return fail(FPB_EUSAGE, "null pointer");
  const size_t sb = map_elems(D) * 4, mb = map_elems(D);
  uint8_t* base;
  cudaStream_t st;
  if ((rc = arena_get(align_up(sb) + align_up(mb), &base, &st))) return rc;
  Carve c{base};
  float* ds = c.take<float>(sb);
  uint8_t* dm = c.take<uint8_t>(mb);
  FPB_CUDA(cudaMemcpyAsync(ds, score, sb, cudaMemcpyHostToDevice, st));
  if ((rc = sort_select(p, ds, mode, k, top_p, dm, st))) return rc;
  FPB_CUDA(cudaMemcpyAsync(mask, dm, mb, cudaMemcpyDeviceToHost, st));
  FPB_CUDA(cudaStreamSynchronize(st));
  return FPB_OK;
}

int fpb_host_topk_select(const fpb_problem* p, const float* score, int32_t k, uint8_t* mask) {
  return host_sort_select(p, score, 0, k, 0.f, mask);
}

int fpb_host_topp_select(const fpb_problem* p, const float* score, float top_p, uint8_t* mask) {
  return host_sort_select(p, score, 1, 1, top_p, mask);
}

int fpb_host_discover_method(const fpb_problem* p, fpb_dtype dtype, int method, const void* Q,
                             const void* K, float* energy, float* local_max, float* score) {
  if (method == 0) return fpb_host_discover(p, dtype, Q, K, energy, local_max, score);
  if (method != 1 && method != 2) return fail(FPB_EUSAGE, "unknown discovery method %d", method);
  Dims D;
  ArenaDrain drain;  // error returns leave nothing in flight
  int rc = resolve(p, &D);
  if (rc || (rc = check_dtype(dtype))) return rc;
  if (!Q || !K || !energy || !local_max || !score) return fail(FPB_EUSAGE, "null pointer");
  size_t wsb;
  fpb_baseline_workspace_bytes(p, &wsb);
  const size_t qb = q_elems(D) * dsz(dtype), kb = kv_elems(D) * dsz(dtype), mb = map_elems(D) * 4;
  uint8_t* base;
  cudaStream_t st;
  if ((rc = arena_get(align_up(qb) + align_up(kb) + 3 * align_up(mb) + align_up(wsb), &base, &st)))
    return rc;
  Carve c{base};
  void* dq = c.take<void>(qb);
  void* dk = c.take<void>(kb);
  float* de = c.take<float>(mb);
  float* dl = c.take<float>(mb);
  float* ds = c.take<float>(mb);
  void* ws = c.take<void>(wsb);
  FPB_CUDA(cudaMemcpyAsync(dq, Q, qb, cudaMemcpyHostToDevice, st));
  FPB_CUDA(cudaMemcpyAsync(dk, K, kb, cudaMemcpyHostToDevice, st));
  rc = method == 1 ? fpb_discover_pool_both(p, dtype, dq, dk, de, dl, ds, ws, wsb, st)
                   : fpb_discover_exact(p, dtype, dq, dk, de, dl, ds, ws, wsb, st);
  if (rc) return rc;
  FPB_CUDA(cudaMemcpyAsync(energy, de, mb, cudaMemcpyDeviceToHost, st));
  FPB_CUDA(cudaMemcpyAsync(local_max, dl, mb, cudaMemcpyDeviceToHost, st));
  FPB_CUDA(cudaMemcpyAsync(score, ds, mb, cudaMemcpyDeviceToHost, st));
  FPB_CUDA(cudaStreamSynchronize(st));
  return FPB_OK;
}

int fpb_host_compress_indices(const fpb_problem* p, const uint8_t* mask, int32_t* idx,
                              int32_t* counts) {
  Dims D;
  ArenaDrain drain;  // error returns leave nothing in flight
  int rc = resolve(p, &D);
  if (rc) return rc;
  if (!mask || !idx || !counts) return fail(FPB_EUSAGE, "null pointer");
  const size_t mb = map_elems(D), ib = map_elems(D) * 4, cb = (size_t)D.Z * D.M * D.Hq * 4;
  uint8_t* base;
  cudaStream_t st;
  if ((rc = arena_get(align_up(mb) + align_up(ib) + align_up(cb), &base, &st))) return rc;
  Carve c{base};
  uint8_t* dm = c.take<uint8_t>(mb);
  int32_t* di = c.take<int32_t>(ib);
  int32_t* dc = c.take<int32_t>(cb);
  FPB_CUDA(cudaMemcpyAsync(dm, mask, mb, cudaMemcpyHostToDevice, st));
  if ((rc = fpb_compress_indices(p, dm, di, dc, st))) return rc;
  FPB_CUDA(cudaMemcpyAsync(idx, di, ib, cudaMemcpyDeviceToHost, st));
  FPB_CUDA(cudaMemcpyAsync(counts, dc, cb, cudaMemcpyDeviceToHost, st));
  FPB_CUDA(cudaStreamSynchronize(st));
  return FPB_OK;
}

}  // extern "C"

static int host_attention(const fpb_problem* p, fpb_dtype dtype, const void* Q, const void* K,
                          const void* V, const int32_t* idx, const int32_t* counts,
                          fpb_dtype out_dtype, void* out, float* lse,
                          unsigned long long* visits) {
  Dims D;
  ArenaDrain drain;  // error returns leave nothing in flight
  int rc = resolve(p, &D);
  if (rc || (rc = check_dtype(dtype)) || (rc = check_dtype(out_dtype))) return rc;
  if (!Q || !K || !V || !out || !lse) return fail(FPB_EUSAGE, "null pointer");
  const size_t qb = q_elems(D) * dsz(dtype), kb = kv_elems(D) * dsz(dtype),
               ob = q_elems(D) * dsz(out_dtype), lb = (size_t)D.Z * D.Hq * D.L * 4,
               ib = idx ? map_elems(D) * 4 : 0, cb = idx ? (size_t)D.Z * D.M * D.Hq * 4 : 0,
               wsb = ws_attention(D, dtype);
  const size_t need = align_up(qb) + 2 * align_up(kb) + align_up(ob) + align_up(lb) +
                      align_up(ib) + align_up(cb) + align_up(wsb) + 2048;
  uint8_t* base;
  cudaStream_t st;
  if ((rc = arena_get(need, &base, &st))) return rc;
  Carve c{base};
  void* dq = c.take<void>(qb);
  void* dk = c.take<void>(kb);
  void* dv = c.take<void>(kb);
  void* dout = c.take<void>(ob);
  float* dl = c.take<float>(lb);
  int32_t* di = c.take<int32_t>(ib);
  int32_t* dc = c.take<int32_t>(cb);
  unsigned long long* dvis = c.take<unsigned long long>(8);
  int32_t* derr = c.take<int32_t>(4);
  void* ws = c.take<void>(wsb);
  FPB_CUDA(cudaMemcpyAsync(dq, Q, qb, cudaMemcpyHostToDevice, st));
  FPB_CUDA(cudaMemcpyAsync(dk, K, kb, cudaMemcpyHostToDevice, st));
  FPB_CUDA(cudaMemcpyAsync(dv, V, kb, cudaMemcpyHostToDevice, st));
  FPB_CUDA(cudaMemsetAsync(dvis, 0, 8, st));
  FPB_CUDA(cudaMemsetAsync(derr, 0, 4, st));
  if (idx) {
    FPB_CUDA(cudaMemcpyAsync(di, idx, ib, cudaMemcpyHostToDevice, st));
    FPB_CUDA(cudaMemcpyAsync(dc, counts, cb, cudaMemcpyHostToDevice, st));
    rc = fpb_block_sparse_attention(p, dtype, dq, dk, dv, di, dc, out_dtype, dout, dl, dvis, derr,
                                    ws, wsb, st);
  } else {
    rc = fpb_dense_attention(p, dtype, dq, dk, dv, out_dtype, dout, dl, ws, wsb, st);
  }
  if (rc) return rc;
  FPB_CUDA(cudaMemcpyAsync(out, dout, ob, cudaMemcpyDeviceToHost, st));
  FPB_CUDA(cudaMemcpyAsync(lse, dl, lb, cudaMemcpyDeviceToHost, st));
  unsigned long long vis = 0;
  int32_t err = 0;
  FPB_CUDA(cudaMemcpyAsync(&vis, dvis, 8, cudaMemcpyDeviceToHost, st));
  FPB_CUDA(cudaMemcpyAsync(&err, derr, 4, cudaMemcpyDeviceToHost, st));
  FPB_CUDA(cudaStreamSynchronize(st));
  if (err) return fail(FPB_EVALIDATION, "plan row lists a block index outside [0, %d)", D.M);
  if (visits) *visits += vis;
  return FPB_OK;
}

extern "C" {

int fpb_host_block_sparse_attention(const fpb_problem* p, fpb_dtype dtype, const void* Q,
                                    const void* K, const void* V, const int32_t* idx,
                                    const int32_t* counts, fpb_dtype out_dtype, void* out,
                                    float* lse, unsigned long long* visits) {
  if (!idx || !counts) return fail(FPB_EUSAGE, "null plan");
  return host_attention(p, dtype, Q, K, V, idx, counts, out_dtype, out, lse, visits);
}

int fpb_host_dense_attention(const fpb_problem* p, fpb_dtype dtype, const void* Q, const void* K,
                             const void* V, fpb_dtype out_dtype, void* out, float* lse) {
  return host_attention(p, dtype, Q, K, V, nullptr, nullptr, out_dtype, out, lse, nullptr);
}

int fpb_host_prefill(const fpb_problem* p, fpb_dtype dtype, const void* Q, const void* K,
                     const void* V, fpb_dtype out_dtype, void* out, float* lse, int32_t* idx,
                     int32_t* counts, unsigned long long* visits) {
  // Pipelined over chunks of Q heads (each inside one KV group): H2D of chunk c+1, the kernels of
  // chunk c and the D2H of chunk c-1 run concurrently on three streams (PCIe is full duplex).
  Dims D;
  ArenaDrain drain;  // error returns leave nothing in flight
  int rc = resolve(p, &D);
  if (rc || (rc = check_dtype(dtype)) || (rc = check_dtype(out_dtype))) return rc;
  if (!Q || !K || !V || !out || !lse) return fail(FPB_EUSAGE, "null pointer");
  const int group = D.Hq / D.Hkv;
  int min_chunks = 16;  // Q heads per chunk: at least 16 chunks when the problem allows it
  if (const char* e = getenv("FPB_E2E_CHUNKS")) min_chunks = atoi(e);
  int cq = group;
  while (cq % 2 == 0 && (int64_t)D.Z * D.Hq / cq < min_chunks) cq /= 2;
  // chunk list (z, first Q head, heads); a chunk never spans KV groups.  The first and the last
  // chunk are halved (when cq is even) to shorten the pipeline fill (H2D before the first
  // kernel) and drain (last kernels + D2H after the last H2D).
  struct Chunk { int z, q0, nh; };
  std::vector<Chunk> ch;
  for (int z = 0; z < D.Z; ++z)
    for (int q0 = 0; q0 < D.Hq; q0 += cq) ch.push_back({z, q0, cq});
  if (cq % 2 == 0 && ch.size() >= 4) {
    const int h = cq / 2;
    const Chunk f = ch.front(), l = ch.back();
    ch.erase(ch.begin());
    ch.insert(ch.begin(), {{f.z, f.q0, h}, {f.z, f.q0 + h, h}});
    ch.pop_back();
    ch.push_back({l.z, l.q0, h});
    ch.push_back({l.z, l.q0 + h, h});
  }
  const int nch = (int)ch.size();
  const size_t es = dsz(dtype), eo = dsz(out_dtype), Ld = (size_t)D.L * D.d;
  const size_t qb = q_elems(D) * es, kb = kv_elems(D) * es, ob = q_elems(D) * eo,
               lb = (size_t)D.Z * D.Hq * D.L * 4;
  fpb_problem sub = *p;  // sized for the largest chunk (cq heads); sub.Hq is set per chunk
  sub.Z = 1;
  sub.Hq = cq;
  sub.Hkv = 1;
  Dims Ds;
  if ((rc = resolve(&sub, &Ds))) return rc;
  const size_t sib = map_elems(Ds) * 4, scb = (size_t)Ds.M * cq * 4;
  const size_t wsd = ws_discover(Ds, dtype), wsa = ws_attention(Ds, dtype);
  const size_t wsb = wsd > wsa ? wsd : wsa;
  const size_t need = align_up(qb) + 2 * align_up(kb) + align_up(ob) + align_up(lb) +
                      nch * (align_up(sib) + align_up(scb)) + align_up(8 * nch) +
                      2 * align_up(wsb);
  uint8_t* base;
  cudaStream_t st;
  if ((rc = arena_get(need, &base, &st))) return rc;
  if (!g_arena.s_in) FPB_CUDA(cudaStreamCreateWithFlags(&g_arena.s_in, cudaStreamNonBlocking));
  if (!g_arena.s_out) FPB_CUDA(cudaStreamCreateWithFlags(&g_arena.s_out, cudaStreamNonBlocking));
  if (!g_arena.s_c2) FPB_CUDA(cudaStreamCreateWithFlags(&g_arena.s_c2, cudaStreamNonBlocking));
  cudaStream_t s_in = g_arena.s_in, s_out = g_arena.s_out;
  // chunks alternate between two compute streams with their own workspaces, so the next chunk's
  // kernels fill the SMs that the current chunk's longest rows leave idle
  cudaStream_t sc[2] = {st, g_arena.s_c2};
  Carve c{base};
  uint8_t* dq = c.take<uint8_t>(qb);
  uint8_t* dk = c.take<uint8_t>(kb);
  uint8_t* dv = c.take<uint8_t>(kb);
  uint8_t* dout = c.take<uint8_t>(ob);
  float* dl = c.take<float>(lb);
  unsigned long long* dvis = c.take<unsigned long long>(8 * nch);
  void* wsc[2] = {c.take<void>(wsb), c.take<void>(wsb)};
  std::vector<int32_t*> di(nch), dc(nch);
  for (int i = 0; i < nch; ++i) {
    di[i] = c.take<int32_t>(sib);
    dc[i] = c.take<int32_t>(scb);
  }
  cudaEvent_t* evp;
  if ((rc = arena_events(2 * (size_t)nch + 1, &evp))) return rc;
  cudaEvent_t *ev_in = evp, *ev_done = evp + nch, e0 = evp[2 * nch];
  FPB_CUDA(cudaMemsetAsync(dvis, 0, 8 * nch, st));
  // the second compute stream starts after the memset (and any earlier use of the arena)
  FPB_CUDA(cudaEventRecord(e0, st));
  FPB_CUDA(cudaStreamWaitEvent(sc[1], e0, 0));
  // FPB_E2E_TRACE=1: per-chunk timeline (H2D done / kernels done / D2H done) on stderr
  static const bool trace = getenv("FPB_E2E_TRACE") != nullptr;
  std::vector<cudaEvent_t> tr_in, tr_k, tr_out;
  cudaEvent_t tr0 = nullptr;
  auto tr_mark = [&](std::vector<cudaEvent_t>& v, cudaStream_t s) -> int {
    if (!trace) return FPB_OK;
    cudaEvent_t e;
    FPB_CUDA(cudaEventCreate(&e));
    FPB_CUDA(cudaEventRecord(e, s));
    v.push_back(e);
    return FPB_OK;
  };
  if (trace) {
    FPB_CUDA(cudaEventCreate(&tr0));
    FPB_CUDA(cudaEventRecord(tr0, s_in));
  }
  const uint8_t* hq = static_cast<const uint8_t*>(Q);
  const uint8_t* hk = static_cast<const uint8_t*>(K);
  const uint8_t* hv = static_cast<const uint8_t*>(V);
  for (int i = 0; i < nch; ++i) {  // H2D: K/V of a group with its first chunk, then the Q slice
    const int z = ch[i].z, q0 = ch[i].q0, nh = ch[i].nh, kv = q0 / group;
    if (q0 % group == 0) {
      const size_t off = ((size_t)z * D.Hkv + kv) * Ld * es;
      FPB_CUDA(cudaMemcpyAsync(dk + off, hk + off, Ld * es, cudaMemcpyHostToDevice, s_in));
      FPB_CUDA(cudaMemcpyAsync(dv + off, hv + off, Ld * es, cudaMemcpyHostToDevice, s_in));
    }
    const size_t off = ((size_t)z * D.Hq + q0) * Ld * es;
    FPB_CUDA(cudaMemcpyAsync(dq + off, hq + off, nh * Ld * es, cudaMemcpyHostToDevice, s_in));
    FPB_CUDA(cudaEventRecord(ev_in[i], s_in));
    if ((rc = tr_mark(tr_in, s_in))) return rc;
  }
  for (int i = 0; i < nch; ++i) {  // kernels of each chunk on alternating compute streams
    const int z = ch[i].z, q0 = ch[i].q0, kv = q0 / group;
    sub.Hq = ch[i].nh;
    cudaStream_t cs = sc[i & 1];
    void* ws = wsc[i & 1];
    FPB_CUDA(cudaStreamWaitEvent(cs, ev_in[i], 0));
    const uint8_t* q = dq + ((size_t)z * D.Hq + q0) * Ld * es;
    const uint8_t* k = dk + ((size_t)z * D.Hkv + kv) * Ld * es;
    const uint8_t* v = dv + ((size_t)z * D.Hkv + kv) * Ld * es;
    uint8_t* o = dout + ((size_t)z * D.Hq + q0) * Ld * eo;
    float* l = dl + ((size_t)z * D.Hq + q0) * D.L;
    if ((rc = fpb_discover_select(&sub, dtype, q, k, nullptr, nullptr, nullptr, nullptr, di[i],
                                  dc[i], ws, wsb, cs)))
      return rc;
    if ((rc = fpb_block_sparse_attention(&sub, dtype, q, k, v, di[i], dc[i], out_dtype, o, l,
                                         dvis + i, nullptr, ws, wsb, cs)))
      return rc;
    FPB_CUDA(cudaEventRecord(ev_done[i], cs));
    if ((rc = tr_mark(tr_k, cs))) return rc;
  }
  uint8_t* ho = static_cast<uint8_t*>(out);
  for (int i = 0; i < nch; ++i) {  // D2H of each finished chunk
    const int z = ch[i].z, q0 = ch[i].q0, nh = ch[i].nh;
    FPB_CUDA(cudaStreamWaitEvent(s_out, ev_done[i], 0));
    const size_t oo = ((size_t)z * D.Hq + q0) * Ld * eo;
    FPB_CUDA(cudaMemcpyAsync(ho + oo, dout + oo, nh * Ld * eo, cudaMemcpyDeviceToHost, s_out));
    const size_t lo = ((size_t)z * D.Hq + q0) * D.L;
    FPB_CUDA(cudaMemcpyAsync(lse + lo, dl + lo, (size_t)nh * D.L * 4, cudaMemcpyDeviceToHost,
                             s_out));
    // plans are head-last: scatter the chunk's heads into the caller's Z x M x N x Hq layout
    if (idx)
      FPB_CUDA(cudaMemcpy2DAsync(idx + (size_t)z * D.M * D.M * D.Hq + q0, (size_t)D.Hq * 4, di[i],
                                 (size_t)nh * 4, (size_t)nh * 4, (size_t)D.M * D.M,
                                 cudaMemcpyDeviceToHost, s_out));
    if (counts)
      FPB_CUDA(cudaMemcpy2DAsync(counts + (size_t)z * D.M * D.Hq + q0, (size_t)D.Hq * 4, dc[i],
                                 (size_t)nh * 4, (size_t)nh * 4, (size_t)D.M,
                                 cudaMemcpyDeviceToHost, s_out));
    if ((rc = tr_mark(tr_out, s_out))) return rc;
  }
  std::vector<unsigned long long> vis(nch, 0);
  FPB_CUDA(cudaStreamSynchronize(st));
  FPB_CUDA(cudaStreamSynchronize(sc[1]));
  FPB_CUDA(cudaMemcpyAsync(vis.data(), dvis, 8 * nch, cudaMemcpyDeviceToHost, s_out));
  FPB_CUDA(cudaStreamSynchronize(s_out));
  if (trace) {
    for (int i = 0; i < nch; ++i) {
      float a = 0, b = 0, c2 = 0;
      cudaEventElapsedTime(&a, tr0, tr_in[i]);
      cudaEventElapsedTime(&b, tr0, tr_k[i]);
      cudaEventElapsedTime(&c2, tr0, tr_out[i]);
      fprintf(stderr, "e2e chunk %2d: h2d %.3f  kernels %.3f  d2h %.3f ms\n", i, a, b, c2);
      cudaEventDestroy(tr_in[i]);
      cudaEventDestroy(tr_k[i]);
      cudaEventDestroy(tr_out[i]);
    }
    cudaEventDestroy(tr0);
  }
  if (visits)
    for (auto x : vis) *visits += x;
  return FPB_OK;
}

}  // extern "C"
