// extern "C" boundary of libsampleattn (declared in include/sampleattn.h).
//
// Argument validation mirrors the reference's InputError checks
// (sampler.py:52-56 SparseConfig, filtering.py:37-43 find_k, core.py:30-37
// as_matrix); kernel dispatch picks the tcgen05 path for bf16 (d == blk == 128)
// and the exact SIMT path for fp32.  No allocation, no stream synchronisation.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <string>

#include "sa_internal.h"

namespace sa {

int launch_select(const double* col, const double* slash, int Hq, int cn, int nb, double ac,
                  double as, double eps, const double* bound, double bound_ref, int* flags, const int* only,
                  const int* k_in, int* k_out, int* idx_out, int* band, double band_eps, cudaStream_t st);
int launch_merge(const int* k_sel, const int* idx_sel, int Hq, int cn, int nb, int S, int blk,
                 int itv, int sink_blocks, int local_blocks, int* kv_cnt, int* kv_idx,
                 long long* ab, long long* ae, cudaStream_t st);
int launch_full(int Hq, int nb, int* kv_cnt, int* kv_idx, cudaStream_t st);
int launch_sched(const int* kv_cnt, const int* kv_idx, int Hq, int nb, int group, int q_head0, int* order,
                 int* scratch, cudaStream_t st);
int launch_check_finite(const void* x, int dtype, long long n, int* flag, cudaStream_t st);

namespace {
thread_local std::string g_err;
std::atomic<long long> g_launches{0};

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}
// cuMemGetAddressRange (driver API through the runtime's entry-point query, so
// the library needs no -lcuda): the allocation base a CUDA IPC handle refers to
typedef CUresult (*AddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
AddrRangeFn addr_range_fn() {
  static AddrRangeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<AddrRangeFn>(p);
  });
  return fn;
}
}  // namespace

void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return SA_OK;
}

__device__ unsigned g_status[4];

unsigned* status_ptr() {
  static std::mutex mu;
  static unsigned* ptr[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (!ptr[dev & 63]) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_status) != cudaSuccess) return nullptr;
    ptr[dev & 63] = static_cast<unsigned*>(p);
  }
  return ptr[dev & 63];
}

void set_smem_attr(const void* fn, int bytes) {
  // The opt-in is a ceiling: keep the largest size set per (kernel, device)
  // and only ever raise it, so a call with a smaller size cannot lower the
  // limit under a later, larger launch.
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> ceiling;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_pair(fn, dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = ceiling.find(key);
  if (it != ceiling.end() && it->second >= bytes) return;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess)
    ceiling[key] = bytes;
}

bool make_tmap_bf16_hsd(CUtensorMap* map, const void* base, int H, int S, int d, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)S, (cuuint64_t)H};
  const cuuint64_t strides[2] = {(cuuint64_t)d * 2, (cuuint64_t)S * d * 2};
  const cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

Workspace workspace_layout(int S, int Hq, int Hkv, int d, int blk, int cn, int dtype) {
  (void)d;
  Workspace L{};
  const int nb = ceil_div(S, blk);
  const size_t rows = (size_t)Hq * cn * blk;
  size_t off = 0;
  L.tc_part = off;
  if (dtype == SA_BF16) off = align_up(off + (size_t)3 * Hq * cn * 128 * nb * sizeof(float));
  L.rowstat = off;
  off = align_up(off + rows * 2 * sizeof(double));
  L.x_part = off;
  off = align_up(off + 3 * rows * nb * sizeof(double));
  L.part3 = off;
  off = align_up(off + (size_t)Hq * cn * nb * 4 * sizeof(double));
  L.flag_list = off;
  off = align_up(off + (size_t)(Hq * cn + 2) * sizeof(int));
  L.kmax2 = off;
  off = align_up(off + (size_t)Hkv * sizeof(unsigned));
  L.band_items = off;
  off = align_up(off + (1 + 2 * (size_t)Hq * cn * nb) * sizeof(int));  // each pair's key blocks at most once
  L.total = off;
  return L;
}

}  // namespace sa

using namespace sa;

namespace {
int check_geom(int S, int Hq, int Hkv, int d, int blk, int group, int q_head0, int dtype) {
  if (S < 1 || Hq < 1 || Hkv < 1 || d < 1 || blk < 1)
    return fail(SA_ERR_INVALID, "S, heads, d and blk must all be >= 1");
  if (group < 1 || q_head0 < 0) return fail(SA_ERR_INVALID, "group must be >= 1, q_head0 >= 0");
  if (kv_head_of(Hq - 1, group, q_head0) >= Hkv)
    return fail(SA_ERR_INVALID, "q heads map past the supplied kv heads");
  if (dtype == SA_BF16) {
    if (d != kHeadDim || blk != kBlk)
      return fail(SA_ERR_UNSUPPORTED, "bf16 tensor-core path needs d == 128 and blk == 128");
  } else if (dtype == SA_FP32) {
    if (d > kMaxSimtD || blk > kMaxSimtBlk)
      return fail(SA_ERR_UNSUPPORTED, "fp32 path supports d <= 128 and blk <= 128");
  } else {
    return fail(SA_ERR_INVALID, "dtype must be SA_BF16 or SA_FP32");
  }
  return SA_OK;
}
}  // namespace

extern "C" {

int sa_version(void) { return 100; }

const char* sa_last_error(void) { return g_err.c_str(); }

long long sa_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int sa_status(unsigned* status4, int reset) {
  if (!status4) return fail(SA_ERR_INVALID, "sa_status: null pointer");
  if (cudaMemcpyFromSymbol(status4, g_status, 4 * sizeof(unsigned)) != cudaSuccess)
    return fail(SA_ERR_CUDA, "sa_status: cannot read the device status word");
  if (reset) {
    const unsigned z[4] = {0, 0, 0, 0};
    if (cudaMemcpyToSymbol(g_status, z, sizeof(z)) != cudaSuccess)
      return fail(SA_ERR_CUDA, "sa_status: cannot reset the device status word");
  }
  return SA_OK;
}

size_t sa_workspace_bytes(int S, int Hq, int Hkv, int d, int blk, int chunk_n, int dtype) {
  if (S < 1 || Hq < 1 || blk < 1 || chunk_n < 1) return 0;
  return workspace_layout(S, Hq, Hkv, d, blk, chunk_n, dtype).total;
}

int sa_check_finite(const void* x, int dtype, int64_t n, int* flag_dev, void* stream) {
  if (!x || !flag_dev) return fail(SA_ERR_INVALID, "sa_check_finite: null pointer");
  return launch_check_finite(x, dtype, n, flag_dev, static_cast<cudaStream_t>(stream));
}

int sa_copy2d_async(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                    void* stream) {
  if (!dst || !src) return fail(SA_ERR_INVALID, "sa_copy2d_async: null pointer");
  if (width > dpitch || width > spitch) return fail(SA_ERR_INVALID, "sa_copy2d_async: width exceeds a pitch");
  if (!width || !height) return SA_OK;
  const cudaError_t e = cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDefault,
                                          static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(SA_ERR_CUDA, std::string("sa_copy2d_async: ") + cudaGetErrorString(e));
  return SA_OK;
}

int sa_stage1(const void* q, const void* k, int dtype, int S, int Hq, int Hkv, int d, int blk,
              int group, int q_head0, int chunk_n, int itv, double* col, double* slash,
              double* logit_bound, int mode, const int* only_flags, void* workspace,
              size_t workspace_bytes, void* stream) {
  if (int e = check_geom(S, Hq, Hkv, d, blk, group, q_head0, dtype)) return e;
  if (!q || !k || !col || !slash || !workspace) return fail(SA_ERR_INVALID, "sa_stage1: null pointer");
  if (chunk_n < 1 || itv < 1) return fail(SA_ERR_INVALID, "sa_stage1: chunk_n and itv must be >= 1");
  if (S >= blk && ((long long)chunk_n * itv > S || itv < blk))
    return fail(SA_ERR_INVALID, "sa_stage1: (chunk_n, itv) is not a plan_chunks layout");
  if (S < blk && (chunk_n != 1 || itv != S))
    return fail(SA_ERR_INVALID, "sa_stage1: S < blk needs chunk_n == 1, itv == S");
  const Workspace L = workspace_layout(S, Hq, Hkv, d, blk, chunk_n, dtype);
  if (workspace_bytes < L.total) return fail(SA_ERR_INVALID, "sa_stage1: workspace too small");
  Stage1Geom g{S, Hq, Hkv, d, blk, group, q_head0, chunk_n, itv, ceil_div(S, blk)};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(workspace);
  if (mode == SA_STAGE1_TENSOR) {
    if (dtype != SA_BF16) return fail(SA_ERR_UNSUPPORTED, "tensor-core stage 1 needs bf16 inputs");
    if (logit_bound && !only_flags)
      if (int e = launch_logit_bound(g, q, k, ws, L, logit_bound, st)) return e;
    return launch_stage1_tc(g, q, k, only_flags, ws, L, col, slash, st);
  }
  if (mode == SA_STAGE1_EXACT)
    return launch_stage1_exact(g, q, k, dtype, only_flags, ws, L, col, slash, st);
  return fail(SA_ERR_INVALID, "sa_stage1: unknown mode");
}

int sa_select(const double* col, const double* slash, int Hq, int chunk_n, int nb, double alpha_c,
              double alpha_s, double margin_eps, const double* logit_bound, double bound_ref, int* flags,
              const int* only_flags, const int* k_in, int* k_out, int* idx_out, int* band, double band_eps,
              void* stream) {
  if (!(alpha_c >= 0.0 && alpha_c <= 1.0))
    return fail(SA_ERR_INVALID, "alpha_c must be in [0, 1]");
  if (!(alpha_s >= 0.0 && alpha_s <= 1.0))
    return fail(SA_ERR_INVALID, "alpha_s must be in [0, 1]");
  if (Hq < 1 || chunk_n < 1 || nb < 1) return fail(SA_ERR_INVALID, "sa_select: empty geometry");
  if (!col || !slash || !k_out || !idx_out) return fail(SA_ERR_INVALID, "sa_select: null pointer");
  if (margin_eps > 0.0 && !flags) return fail(SA_ERR_INVALID, "sa_select: guard needs flags");
  if (logit_bound && !(bound_ref > 0.0)) return fail(SA_ERR_INVALID, "sa_select: bound_ref must be > 0");
  return launch_select(col, slash, Hq, chunk_n, nb, alpha_c, alpha_s, margin_eps, logit_bound, bound_ref, flags,
                       only_flags, k_in, k_out, idx_out, band, band_eps, static_cast<cudaStream_t>(stream));
}

int sa_band_table_len(int Hq, int chunk_n) {
  if (Hq < 1 || chunk_n < 1) return fail(SA_ERR_INVALID, "sa_band_table_len: bad args");
  return Hq * chunk_n * 2 * kBandEntry;
}

long long sa_workspace_offset(int S, int Hq, int Hkv, int d, int blk, int chunk_n, int dtype, int region) {
  if (S < 1 || Hq < 1 || Hkv < 1 || blk < 1 || chunk_n < 1) return fail(SA_ERR_INVALID, "sa_workspace_offset: bad args");
  const Workspace L = workspace_layout(S, Hq, Hkv, d, blk, chunk_n, dtype);
  if (region == SA_WS_ROW_STATS) return (long long)L.rowstat;
  return fail(SA_ERR_INVALID, "sa_workspace_offset: unknown region");
}

int sa_refine_bands(const void* q, const void* k, int dtype, int S, int Hq, int Hkv, int d, int blk, int group,
                    int q_head0, int chunk_n, int itv, const int* band, const int* flags, int* band_pairs,
                    const double* row_stats, double* col, double* slash, void* workspace, size_t workspace_bytes,
                    void* stream) {
  if (int e = check_geom(S, Hq, Hkv, d, blk, group, q_head0, dtype)) return e;
  if (!q || !k || !band || !flags || !band_pairs || !row_stats || !col || !slash || !workspace)
    return fail(SA_ERR_INVALID, "sa_refine_bands: null pointer");
  const Workspace L = workspace_layout(S, Hq, Hkv, d, blk, chunk_n, dtype);
  if (workspace_bytes < L.total) return fail(SA_ERR_INVALID, "sa_refine_bands: workspace too small");
  if (dtype != SA_BF16) return fail(SA_ERR_UNSUPPORTED, "sa_refine_bands: the band guard serves the bf16 path");
  Stage1Geom g{S, Hq, Hkv, d, blk, group, q_head0, chunk_n, itv, ceil_div(S, blk)};
  return launch_refine_bands(g, q, k, dtype, band, flags, band_pairs, row_stats, static_cast<char*>(workspace), L,
                             col, slash, static_cast<cudaStream_t>(stream));
}

int sa_certify_band_ties(int dtype, int S, int Hq, int Hkv, int d, int blk, int chunk_n, int itv, const int* band,
                         int* flags, const double* row_stats, const double* col, const double* slash,
                         const double* logit_bound, double bound_ref, double band_eps, void* workspace,
                         size_t workspace_bytes, void* stream) {
  if (Hkv < 1) return fail(SA_ERR_INVALID, "sa_certify_band_ties: Hkv must be >= 1");
  if (int e = check_geom(S, Hq, Hkv, d, blk, ceil_div(Hq, Hkv), 0, dtype)) return e;
  if (!band || !flags || !row_stats || !col || !slash || !workspace)
    return fail(SA_ERR_INVALID, "sa_certify_band_ties: null pointer");
  if (chunk_n < 1 || itv < 1 || !(band_eps > 0.0) || (logit_bound && !(bound_ref > 0.0)))
    return fail(SA_ERR_INVALID, "sa_certify_band_ties: bad chunk_n / itv / band_eps / bound_ref");
  const Workspace L = workspace_layout(S, Hq, Hkv, d, blk, chunk_n, dtype);
  if (workspace_bytes < L.total) return fail(SA_ERR_INVALID, "sa_certify_band_ties: workspace too small");
  if (dtype != SA_BF16) return fail(SA_ERR_UNSUPPORTED, "sa_certify_band_ties: the band guard serves the bf16 path");
  Stage1Geom g{S, Hq, Hkv, d, blk, 1, 0, chunk_n, itv, ceil_div(S, blk)};
  return launch_band_ties(g, band, flags, row_stats, col, slash, logit_bound, bound_ref, band_eps,
                          static_cast<char*>(workspace), L, static_cast<cudaStream_t>(stream));
}

int sa_merge(const int* k_sel, const int* idx_sel, int Hq, int chunk_n, int nb, int S, int blk,
             int itv, int sink_blocks, int local_blocks, int* kv_cnt, int* kv_idx,
             long long* active_blocks, long long* active_entries, void* stream) {
  if (Hq < 1 || chunk_n < 1 || S < 1 || blk < 1 || itv < 1 || nb != ceil_div(S, blk))
    return fail(SA_ERR_INVALID, "sa_merge: inconsistent geometry");
  if (sink_blocks < 0 || local_blocks < 1)
    return fail(SA_ERR_INVALID, "sa_merge: sink_blocks must be >= 0 and local_blocks >= 1");
  if (!k_sel || !idx_sel || !kv_cnt || !kv_idx) return fail(SA_ERR_INVALID, "sa_merge: null pointer");
  return launch_merge(k_sel, idx_sel, Hq, chunk_n, nb, S, blk, itv, sink_blocks, local_blocks, kv_cnt,
                      kv_idx, active_blocks, active_entries, static_cast<cudaStream_t>(stream));
}

int sa_sampled_retained(int dtype, int S, int Hq, int Hkv, int d, int blk, int chunk_n, int itv, int mode,
                        const int* rescored_flags, const int* kv_cnt, const int* kv_idx, const void* workspace,
                        size_t workspace_bytes, double* retained, void* stream) {
  if (S < 1 || Hq < 1 || Hkv < 1 || blk < 1 || blk > kMaxSimtBlk || chunk_n < 1 || itv < 1)
    return fail(SA_ERR_INVALID, "sa_sampled_retained: bad geometry");
  if (!kv_cnt || !kv_idx || !workspace || !retained) return fail(SA_ERR_INVALID, "sa_sampled_retained: null pointer");
  if (mode == SA_STAGE1_TENSOR && dtype != SA_BF16)
    return fail(SA_ERR_UNSUPPORTED, "sa_sampled_retained: tensor-mode partials exist for bf16 only");
  if (mode != SA_STAGE1_TENSOR && mode != SA_STAGE1_EXACT) return fail(SA_ERR_INVALID, "sa_sampled_retained: mode");
  const Workspace L = workspace_layout(S, Hq, Hkv, d, blk, chunk_n, dtype);
  if (workspace_bytes < L.total) return fail(SA_ERR_INVALID, "sa_sampled_retained: workspace too small");
  Stage1Geom g{S, Hq, Hkv, d, blk, 1, 0, chunk_n, itv, ceil_div(S, blk)};
  return launch_sampled_retained(g, mode == SA_STAGE1_EXACT, rescored_flags, kv_cnt, kv_idx,
                                 static_cast<const char*>(workspace), L, retained, static_cast<cudaStream_t>(stream));
}

int sa_full_mask(int Hq, int nb, int* kv_cnt, int* kv_idx, void* stream) {
  if (Hq < 1 || nb < 1 || !kv_cnt || !kv_idx) return fail(SA_ERR_INVALID, "sa_full_mask: bad args");
  return launch_full(Hq, nb, kv_cnt, kv_idx, static_cast<cudaStream_t>(stream));
}

int sa_schedule(const int* kv_cnt, const int* kv_idx, int Hq, int nb, int group, int q_head0, int* order,
                int* scratch, void* stream) {
  if (Hq < 1 || nb < 1 || !kv_cnt || !order) return fail(SA_ERR_INVALID, "sa_schedule: bad args");
  if (group < 1 || q_head0 < 0) return fail(SA_ERR_INVALID, "sa_schedule: bad group / q_head0");
  return launch_sched(kv_cnt, kv_idx, Hq, nb, group, q_head0, order, scratch, static_cast<cudaStream_t>(stream));
}

int sa_schedule_len(int Hq, int nb, int group, int q_head0) {
  if (Hq < 1 || nb < 1 || group < 1 || q_head0 < 0) return fail(SA_ERR_INVALID, "sa_schedule_len: bad args");
  return 2 * n_units(Hq, nb, group, q_head0);
}

int sa_sparse_forward(const void* q, const void* k, const void* v, int dtype, int S, int Hq, int Hkv,
                      int d, int blk, int group, int q_head0, const int* kv_cnt, const int* kv_idx,
                      const int* order, void* out, float* lse, long long* touched, void* stream) {
  if (int e = check_geom(S, Hq, Hkv, d, blk, group, q_head0, dtype)) return e;
  if (!q || !k || !v || !kv_cnt || !kv_idx || !out)
    return fail(SA_ERR_INVALID, "sa_sparse_forward: null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int n_order = order ? 2 * n_units(Hq, ceil_div(S, blk), group, q_head0) : 0;
  if (dtype == SA_BF16) {
    return launch_sparse_share(q, k, v, S, Hq, Hkv, group, q_head0, kv_cnt, kv_idx, order, out, lse, touched,
                               st);
  }
  return launch_sparse_simt(static_cast<const float*>(q), static_cast<const float*>(k),
                            static_cast<const float*>(v), S, Hq, Hkv, d, blk, group, q_head0, kv_cnt,
                            kv_idx, order, n_order, static_cast<float*>(out), lse, touched, st);
}

int sa_sparse_forward_peers(const void* q, const void* k, const void* v, int dtype, int S, int Hq, int Hkv,
                            int d, int blk, int group, int q_head0, const int* kv_cnt, const int* kv_idx,
                            const int* order, void* out, float* lse, long long* touched, void* const* peer_out,
                            int n_peer, void* stream) {
  if (int e = check_geom(S, Hq, Hkv, d, blk, group, q_head0, dtype)) return e;
  if (!q || !k || !v || !kv_cnt || !kv_idx || !out)
    return fail(SA_ERR_INVALID, "sa_sparse_forward_peers: null pointer");
  if (n_peer < 0 || n_peer > SA_MAX_PEERS || (n_peer > 0 && !peer_out))
    return fail(SA_ERR_INVALID, "sa_sparse_forward_peers: n_peer must be in [0, SA_MAX_PEERS] with peer_out set");
  for (int p = 0; p < n_peer; ++p)
    if (!peer_out[p]) return fail(SA_ERR_INVALID, "sa_sparse_forward_peers: null peer buffer");
  if (dtype != SA_BF16) return fail(SA_ERR_UNSUPPORTED, "sa_sparse_forward_peers: bf16 only");
  return launch_sparse_share(q, k, v, S, Hq, Hkv, group, q_head0, kv_cnt, kv_idx, order, out, lse, touched,
                             static_cast<cudaStream_t>(stream), peer_out, n_peer);
}

int sa_ipc_export(const void* ptr, void* handle, unsigned long long* offset) {
  if (!ptr || !handle || !offset) return fail(SA_ERR_INVALID, "sa_ipc_export: null pointer");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (!addr_range_fn() || addr_range_fn()(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
    return fail(SA_ERR_CUDA, "sa_ipc_export: cuMemGetAddressRange failed (not a device allocation?)");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return fail(SA_ERR_CUDA, std::string("sa_ipc_export: ") + cudaGetErrorString(e));
  std::memcpy(handle, &h, sizeof(h));
  *offset = reinterpret_cast<CUdeviceptr>(ptr) - base;
  return SA_OK;
}

int sa_ipc_open(const void* handle, void** base) {
  if (!handle || !base) return fail(SA_ERR_INVALID, "sa_ipc_open: null pointer");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(SA_ERR_CUDA, std::string("sa_ipc_open: ") + cudaGetErrorString(e));
  return SA_OK;
}

int sa_ipc_close(void* base) {
  if (!base) return fail(SA_ERR_INVALID, "sa_ipc_close: null pointer");
  cudaError_t e = cudaIpcCloseMemHandle(base);
  if (e != cudaSuccess) return fail(SA_ERR_CUDA, std::string("sa_ipc_close: ") + cudaGetErrorString(e));
  return SA_OK;
}

}  // extern "C"
