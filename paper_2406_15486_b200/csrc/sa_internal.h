// Internal declarations shared by the SampleAttention CUDA translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>

#include "sampleattn.h"

namespace sa {

// Thread-local error message behind sa_last_error().
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_launch(const char* what);
// Opt `fn` into at least `bytes` of dynamic shared memory on the CURRENT
// device.  The attribute is per device and a ceiling, so the largest size set
// is kept per (kernel, device) and only ever raised.
void set_smem_attr(const void* fn, int bytes);

// Device status word behind sa_status(): [0] OR of the SA_STATUS_* bits,
// [1] head and [2] query block of the first report, [3] number of reports
// (bits SA_STATUS_EMPTY_BLOCK / _MASK / _NORMALISER, include/sampleattn.h).
unsigned* status_ptr();  // this device's status word
__device__ __forceinline__ void report_status(unsigned* st, unsigned bits, int h, int qb) {
  if (!st) return;
  atomicOr(st, bits);
  if (atomicAdd(st + 3, 1u) == 0) {
    st[1] = (unsigned)h;
    st[2] = (unsigned)qb;
  }
}

constexpr int kBlk = 128;       // tensor-core tile (query rows == key rows == blk)
constexpr int kHeadDim = 128;   // tensor-core head dimension
constexpr int kMaxSimtD = 128;  // SIMT paths
constexpr int kMaxSimtBlk = 128;

__host__ __device__ inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }
__host__ __device__ inline long long tri(long long n) { return n * (n + 1) / 2; }

// Geometry of one stage-1 call.
struct Stage1Geom {
  int S, Hq, Hkv, d, blk, group, q_head0, cn, itv, nb;
};

// Workspace carve-up (byte offsets), identical for every call of a geometry.
struct Workspace {
  size_t tc_part;   // float  [3][Hq*cn*blk*nb]   (A, B, m) per (row, key block)
  size_t rowstat;   // double [Hq*cn*blk][2]      (log2 max, sum) per sampled row
  size_t x_part;    // double [3][Hq*cn*blk*nb]   exact (A, B, m) per (row, key block)
  size_t part3;     // double [Hq*cn*nb][4]       (col, slash X-1, X, X+1) per key block
  size_t flag_list; // int    [Hq*cn + 2]             compacted guard-flagged pairs: count, then indices
  size_t kmax2;     // uint   [Hkv]                 max ||k_j||^2 per KV head (guard logit bound)
  size_t band_items;// int    [1 + 2 * n_items]       band refinement work list: count, then (pair, key block)
  size_t total;
};
Workspace workspace_layout(int S, int Hq, int Hkv, int d, int blk, int cn, int dtype);

// Selection guard, band refinement: per (head, chunk, direction) the run of
// nearly tied blocks at the cut -- [count, first rank, tie a, tie b, block / bin
// indices]; tie a / b: the two refined blocks at the certified cut whose order
// the per-row test (k_band_ties) still has to settle, or -1.
// Bands of up to 512 blocks are refined (the reference's calibrated heads
// reach ~350 at 128K, where the refinement still touches about half the key
// blocks a full re-score does); a wider band sends the pair to the re-score.
constexpr int kBandMax = 512;
constexpr int kBandHdr = 4;
constexpr int kBandEntry = kBandHdr + kBandMax;

// Launchers (return SA_OK or an error code; all stream-ordered).
int launch_stage1_exact(const Stage1Geom& g, const void* q, const void* k, int dtype,
                        const int* only_flags, char* ws, const Workspace& L, double* col,
                        double* slash, cudaStream_t st);
// Per sampled row: the normalised probability mass inside the mask, from the
// stage-1 partials left in the workspace (exact planes for rescored pairs).
int launch_sampled_retained(const Stage1Geom& g, int exact_all, const int* rescored, const int* kv_cnt,
                            const int* kv_idx, const char* ws, const Workspace& L, double* retained,
                            cudaStream_t st);
// Guard logit bound per (head, chunk): max ||q_r|| * max ||k_j|| / sqrt(d) (bf16 inputs).
int launch_logit_bound(const Stage1Geom& g, const void* q, const void* k, char* ws, const Workspace& L,
                       double* bound, cudaStream_t st);
// Band refinement of the selection guard: exact (fp64) masses of the blocks in
// each recorded band, normalised with the tensor-core row statistics, written
// over those blocks' col / slash scores; marks band_pairs.
int launch_refine_bands(const Stage1Geom& g, const void* q, const void* k, int dtype, const int* band,
                        const int* flags, int* band_pairs, const double* row_stats, char* ws, const Workspace& L,
                        double* col, double* slash, cudaStream_t st);
// Per-row certificate of the tie left at a certified band cut (band slots 2, 3);
// flags the pair for the full re-score when it does not hold.
int launch_band_ties(const Stage1Geom& g, const int* band, int* flags, const double* row_stats, const double* col,
                     const double* slash, const double* bound, double bound_ref, double band_eps, char* ws,
                     const Workspace& L, cudaStream_t st);
int launch_stage1_tc(const Stage1Geom& g, const void* q, const void* k, const int* only_flags,
                     char* ws, const Workspace& L, double* col, double* slash, cudaStream_t st);
// rows' global max / sum, fold into part3, scatter into col / slash.  With
// `only` (guard re-score), the flagged (head, chunk) pairs are first compacted
// into ws + L.flag_list and every kernel loops over that list, so the grids
// scale with the flagged pairs, not with Hq * chunk_n.
template <typename TPlane, bool kLog2>
int launch_fold(const Stage1Geom& g, const int* only, const TPlane* pa, const TPlane* pb,
                const TPlane* pm, char* ws, const Workspace& L, double* col, double* slash,
                cudaStream_t st);
// compact the nonzero entries of only[0..n) into list = {count, i0, i1, ...}
int launch_flag_compact(const int* only, int n, int* list, cudaStream_t st);
// grid rows used for flagged-pair loops (enough to fill the GPU, bounded by the pair count)
inline int flagged_grid_rows(int n_pairs) { return n_pairs < 32 ? n_pairs : 32; }

int launch_sparse_simt(const float* q, const float* k, const float* v, int S, int Hq, int Hkv,
                       int d, int blk, int group, int q_head0, const int* kv_cnt,
                       const int* kv_idx, const int* order, int n_order, float* out, float* lse,
                       long long* touched, cudaStream_t st);

// TMA descriptor for a contiguous [H][S][d] bf16 tensor, box {64, box_rows, 1}, 128B swizzle.
bool make_tmap_bf16_hsd(CUtensorMap* map, const void* base, int H, int S, int d, int box_rows = 128);

__host__ __device__ inline int kv_head_of(int h, int group, int q_head0) {
  return (q_head0 + h) / group - q_head0 / group;
}

// ---- stage-3 work units: two (head, query block) items that read the same
// KV head, so one CTA loads each listed K/V tile once for both.  The local q
// heads of a KV group pair up (h_lo, h_lo+1), (h_lo+2, h_lo+3), ... at the same
// query block; an odd head out pairs adjacent query blocks (2j, 2j+1).
// Items are h * nb + qb; a missing partner is -1.
__host__ __device__ inline int n_local_kv(int Hq, int group, int q_head0) {
  return kv_head_of(Hq - 1, group, q_head0) + 1;
}
__host__ __device__ inline void kv_group_heads(int g, int Hq, int group, int q_head0, int& lo, int& hi) {
  const int g_first = q_head0 / group;
  lo = (g_first + g) * group - q_head0;
  hi = lo + group;
  if (lo < 0) lo = 0;
  if (hi > Hq) hi = Hq;
}
__host__ __device__ inline int units_of_group(int nh, int nb) {
  return (nh / 2) * nb + ((nh & 1) ? (nb + 1) / 2 : 0);
}
__host__ __device__ inline void unit_items(int u, int h_lo, int nh, int nb, int& a, int& b) {
  const int paired = (nh / 2) * nb;
  if (u < paired) {
    const int p = u / nb, qb = u - p * nb;
    a = (h_lo + 2 * p) * nb + qb;
    b = a + nb;
  } else {
    const int qb = 2 * (u - paired);
    a = (h_lo + nh - 1) * nb + qb;
    b = qb + 1 < nb ? a + 1 : -1;
  }
}
__host__ __device__ inline int n_units(int Hq, int nb, int group, int q_head0) {
  int total = 0;
  for (int g = 0, G = n_local_kv(Hq, group, q_head0); g < G; ++g) {
    int lo, hi;
    kv_group_heads(g, Hq, group, q_head0, lo, hi);
    total += units_of_group(hi - lo, nb);
  }
  return total;
}

int launch_sparse_share(const void* q, const void* k, const void* v, int S, int Hq, int Hkv, int group,
                        int q_head0, const int* kv_cnt, const int* kv_idx, const int* units, void* out,
                        float* lse, long long* touched, cudaStream_t st, void* const* peer_out = nullptr,
                        int n_peer = 0);

}  // namespace sa
