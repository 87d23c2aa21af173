// Stage 1, exact mode: fp64 SIMT re-statement of sample_scores + block_reduce
// (ref pkg/src/blocksift/sampler.py:135-191, math of core.py:110-154).
//
// Used (a) as the fp32-mode stage 1 and (b) as the selection guard's
// re-score of (head, chunk) pairs whose tensor-core scores are too close to a
// find_k / arg_topk decision to trust (sa_select margin flags).
//
// Three kernels, all deterministic (fixed reduction trees, no float atomics):
//   x_stats   : per (row, key split) online max / sum of exp(s - max)   [fp64]
//   x_rowfin  : per row, combine splits -> (M_r, L_r)
//   x_reduce  : per key block, p = exp(s - M_r) / L_r summed into the column
//               bin and the <= 3 slash bins the block feeds (part3)
// and the shared finalize that scatters part3 into col / slash [fp64].
//
// Slash binning: for sampled row r and key j = kb*blk + t, the offset block is
// (r - j) // blk = r//blk - kb - (t > r % blk); a window of <= blk
// consecutive rows spans at most two values of r//blk, so one key block feeds
// bins X-1, X, X+1 with X = b0 - kb, b0 = sample_start // blk.
#include <cuda_bf16.h>

#include "sa_internal.h"

namespace sa {
namespace {

constexpr int kTile = 64;       // rows x keys per register tile (16x16 threads, 4x4 each)
constexpr int kThreads = 256;

struct Win {
  int ss, se, nkb;  // sampled rows [ss, se); key blocks 0..nkb-1 hold keys < se
};

__device__ __forceinline__ Win window_of(int c, int S, int blk, int itv) {
  Win w;
  if (S < blk) {
    w.ss = 0;
    w.se = S;
  } else {
    w.se = (c + 1) * itv;
    w.ss = max(0, w.se - blk);
  }
  w.nkb = (w.se + blk - 1) / blk;
  return w;
}

template <typename T>
__device__ __forceinline__ float load_as_float(const T* p);
template <>
__device__ __forceinline__ float load_as_float<float>(const float* p) { return __ldg(p); }
template <>
__device__ __forceinline__ float load_as_float<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}

// Stage `n` rows of width d (row stride d) starting at `src` into smem [n][d+1].
template <typename T>
__device__ void stage_rows(float* dst, const T* src, int n, int d) {
  const int dp = d + 1;
  for (int i = threadIdx.x; i < n * d; i += blockDim.x) {
    int r = i / d, c = i - r * d;
    dst[r * dp + c] = load_as_float(src + (size_t)r * d + c);
  }
}

// 4x4 fp64 dot-product micro-tile: rows ty+16a (of the staged q tile), keys tx+16b.
__device__ __forceinline__ void tile_dots(const float* qs, const float* ks, int d, int ty, int tx,
                                          double (&acc)[4][4]) {
  const int dp = d + 1;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int i = 0; i < d; ++i) {
    double qv[4], kv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) qv[a] = (double)qs[(ty + 16 * a) * dp + i];
#pragma unroll
    for (int b = 0; b < 4; ++b) kv[b] = (double)ks[(tx + 16 * b) * dp + i];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fma(qv[a], kv[b], acc[a][b]);
  }
}

__device__ __forceinline__ void lse_merge(double& m, double& l, double m2, double l2) {
  if (m2 == -INFINITY) return;
  if (m == -INFINITY) {
    m = m2;
    l = l2;
    return;
  }
  if (m2 > m) {
    l = l * exp(m - m2) + l2;
    m = m2;
  } else {
    l = l + l2 * exp(m2 - m);
  }
}

// ---- pass 1: per (row, split) running max / sum  (core.py:150-153 in fp64)
template <typename T>
__global__ void __launch_bounds__(kThreads) x_stats(const T* __restrict__ q, const T* __restrict__ k,
                                                    Stage1Geom g, const int* __restrict__ only,
                                                    double* __restrict__ xpart, int nsx) {
  extern __shared__ float smem[];
  const int hc = blockIdx.y, split = blockIdx.x;
  if (only && only[hc] == 0) return;
  const int h = hc / g.cn, c = hc - h * g.cn;
  const Win w = window_of(c, g.S, g.blk, g.itv);
  const int kb0 = split * kExactKbPerCta;
  if (kb0 >= w.nkb) {
    // empty split: publish neutral stats
    for (int r = threadIdx.x; r < g.blk; r += blockDim.x) {
      size_t o = (((size_t)hc * g.blk + r) * nsx + split) * 2;
      xpart[o] = -INFINITY;
      xpart[o + 1] = 0.0;
    }
    return;
  }
  const int kb1 = min(w.nkb, kb0 + kExactKbPerCta);
  const int kvh = kv_head_of(h, g.group, g.q_head0);
  const int nr = w.se - w.ss, d = g.d, dp = d + 1;
  float* qs = smem;                   // [kTile][dp]
  float* ks = smem + kTile * dp;      // [kTile][dp]
  double* red = reinterpret_cast<double*>(ks + kTile * dp);  // [16][kTile][2]
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const T* qh = q + ((size_t)h * g.S + w.ss) * d;
  const T* kh = k + (size_t)kvh * g.S * d;
  const double scale = 1.0 / sqrt((double)d);
  const int key_lo = kb0 * g.blk, key_hi = min(kb1 * g.blk, w.se);

  for (int r0 = 0; r0 < nr; r0 += kTile) {
    const int rn = min(kTile, nr - r0);
    __syncthreads();
    stage_rows(qs, qh + (size_t)r0 * d, rn, d);
    double m[4], l[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      m[a] = -INFINITY;
      l[a] = 0.0;
    }
    for (int j0 = key_lo; j0 < key_hi; j0 += kTile) {
      const int jn = min(kTile, key_hi - j0);
      __syncthreads();
      stage_rows(ks, kh + (size_t)j0 * d, jn, d);
      __syncthreads();
      double acc[4][4];
      tile_dots(qs, ks, d, ty, tx, acc);
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int rl = ty + 16 * a;
        const int row = w.ss + r0 + rl;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int kl = tx + 16 * b;
          const int key = j0 + kl;
          if (rl < rn && kl < jn && key <= row) lse_merge(m[a], l[a], acc[a][b] * scale, 1.0);
        }
      }
    }
    // combine the 16 tx partials of each row in a fixed order
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int rl = ty + 16 * a;
      red[(tx * kTile + rl) * 2] = m[a];
      red[(tx * kTile + rl) * 2 + 1] = l[a];
    }
    __syncthreads();
    for (int rl = threadIdx.x; rl < rn; rl += blockDim.x) {
      double mm = -INFINITY, ll = 0.0;
      for (int t = 0; t < 16; ++t) lse_merge(mm, ll, red[(t * kTile + rl) * 2], red[(t * kTile + rl) * 2 + 1]);
      size_t o = (((size_t)hc * g.blk + r0 + rl) * nsx + split) * 2;
      xpart[o] = mm;
      xpart[o + 1] = ll;
    }
  }
}

// ---- combine splits -> (M_r, L_r)
__global__ void x_rowfin(Stage1Geom g, const int* __restrict__ only, const double* __restrict__ xpart,
                         int nsx, double* __restrict__ rowstat) {
  const int hc = blockIdx.x;
  if (only && only[hc] == 0) return;
  const int c = hc % g.cn;
  const Win w = window_of(c, g.S, g.blk, g.itv);
  const int nr = w.se - w.ss;
  const int used = (w.nkb + kExactKbPerCta - 1) / kExactKbPerCta;
  for (int r = threadIdx.x; r < nr; r += blockDim.x) {
    double m = -INFINITY, l = 0.0;
    const double* p = xpart + ((size_t)hc * g.blk + r) * nsx * 2;
    for (int s = 0; s < used; ++s) lse_merge(m, l, p[2 * s], p[2 * s + 1]);
    rowstat[((size_t)hc * g.blk + r) * 2] = m;
    rowstat[((size_t)hc * g.blk + r) * 2 + 1] = l;
  }
}

// ---- pass 2: per key block, normalised mass into col + 3 slash bins
template <typename T>
__global__ void __launch_bounds__(kThreads) x_reduce(const T* __restrict__ q, const T* __restrict__ k,
                                                     Stage1Geom g, const int* __restrict__ only,
                                                     const double* __restrict__ rowstat,
                                                     double* __restrict__ part3) {
  extern __shared__ float smem[];
  const int hc = blockIdx.y, kb = blockIdx.x;
  if (only && only[hc] == 0) return;
  const int h = hc / g.cn, c = hc - h * g.cn;
  const Win w = window_of(c, g.S, g.blk, g.itv);
  if (kb >= g.nb) return;
  double* out = part3 + ((size_t)hc * g.nb + kb) * 4;
  if (kb >= w.nkb) {
    if (threadIdx.x < 4) out[threadIdx.x] = 0.0;
    return;
  }
  const int kvh = kv_head_of(h, g.group, g.q_head0);
  const int nr = w.se - w.ss, d = g.d, dp = d + 1;
  float* qs = smem;
  float* ks = smem + kTile * dp;
  double* red = reinterpret_cast<double*>(ks + kTile * dp);  // [kThreads][4]
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const T* qh = q + ((size_t)h * g.S + w.ss) * d;
  const T* kh = k + (size_t)kvh * g.S * d;
  const double scale = 1.0 / sqrt((double)d);
  const int key_lo = kb * g.blk, key_hi = min(key_lo + g.blk, w.se);
  const int b0 = w.ss / g.blk;
  const double* rs = rowstat + (size_t)hc * g.blk * 2;
  double sums[4] = {0.0, 0.0, 0.0, 0.0};

  for (int r0 = 0; r0 < nr; r0 += kTile) {
    const int rn = min(kTile, nr - r0);
    __syncthreads();
    stage_rows(qs, qh + (size_t)r0 * d, rn, d);
    for (int j0 = key_lo; j0 < key_hi; j0 += kTile) {
      const int jn = min(kTile, key_hi - j0);
      __syncthreads();
      stage_rows(ks, kh + (size_t)j0 * d, jn, d);
      __syncthreads();
      double acc[4][4];
      tile_dots(qs, ks, d, ty, tx, acc);
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int rl = ty + 16 * a;
        if (rl >= rn) continue;
        const int row = w.ss + r0 + rl;
        const double M = rs[(r0 + rl) * 2], Linv = 1.0 / rs[(r0 + rl) * 2 + 1];
        const int rho = row % g.blk;
        const int base_slot = row / g.blk - b0 + 1;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int kl = tx + 16 * b;
          const int key = j0 + kl;
          if (kl < jn && key <= row) {
            const double p = exp(acc[a][b] * scale - M) * Linv;
            const int t = key - key_lo;
            const int slot = base_slot - (t > rho ? 1 : 0);
            sums[0] += p;
            sums[1 + slot] += p;
          }
        }
      }
    }
  }
  // deterministic block reduction of the 4 sums
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) red[threadIdx.x * 4 + i] = sums[i];
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
#pragma unroll
      for (int i = 0; i < 4; ++i) red[threadIdx.x * 4 + i] += red[(threadIdx.x + s) * 4 + i];
    __syncthreads();
  }
  if (threadIdx.x < 4) out[threadIdx.x] = red[threadIdx.x];
}

// ---- part3 -> col / slash (shared with the tensor-core path)
__global__ void s1_finalize(Stage1Geom g, const int* __restrict__ only,
                            const double* __restrict__ part3, double* __restrict__ col,
                            double* __restrict__ slash) {
  const int hc = blockIdx.x;
  if (only && only[hc] == 0) return;
  const int c = hc % g.cn;
  const Win w = window_of(c, g.S, g.blk, g.itv);
  const int b0 = w.ss / g.blk;
  const double* p3 = part3 + (size_t)hc * g.nb * 4;
  for (int i = threadIdx.x; i < g.nb; i += blockDim.x) {
    col[(size_t)hc * g.nb + i] = i < w.nkb ? p3[(size_t)i * 4] : 0.0;
    // offset block ob = i receives slot 0 of kb = b0-i-1, slot 1 of kb = b0-i, slot 2 of kb = b0-i+1
    double s = 0.0;
    int kb = b0 - i - 1;
    if (kb >= 0 && kb < w.nkb) s += p3[(size_t)kb * 4 + 1];
    kb = b0 - i;
    if (kb >= 0 && kb < w.nkb) s += p3[(size_t)kb * 4 + 2];
    kb = b0 - i + 1;
    if (kb >= 0 && kb < w.nkb) s += p3[(size_t)kb * 4 + 3];
    slash[(size_t)hc * g.nb + i] = s;
  }
}

template <typename T>
int run_exact(const Stage1Geom& g, const T* q, const T* k, const int* only, char* ws,
              const Workspace& L, cudaStream_t st) {
  const int dp = g.d + 1;
  const size_t smem_stats = (size_t)2 * kTile * dp * sizeof(float) + (size_t)16 * kTile * 2 * sizeof(double);
  const size_t smem_red = (size_t)2 * kTile * dp * sizeof(float) + (size_t)kThreads * 4 * sizeof(double);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(x_stats<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaFuncSetAttribute(x_reduce<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    attr_set = true;
  }
  double* xpart = reinterpret_cast<double*>(ws + L.x_part);
  double* rowstat = reinterpret_cast<double*>(ws + L.rowstat);
  double* part3 = reinterpret_cast<double*>(ws + L.part3);
  const int HC = g.Hq * g.cn;
  x_stats<T><<<dim3(L.nsx, HC), kThreads, smem_stats, st>>>(q, k, g, only, xpart, L.nsx);
  if (int e = check_launch("stage1 exact stats")) return e;
  x_rowfin<<<HC, 128, 0, st>>>(g, only, xpart, L.nsx, rowstat);
  if (int e = check_launch("stage1 exact rowfin")) return e;
  x_reduce<T><<<dim3(g.nb, HC), kThreads, smem_red, st>>>(q, k, g, only, rowstat, part3);
  return check_launch("stage1 exact reduce");
}

}  // namespace

int launch_stage1_finalize(const Stage1Geom& g, const int* only, const double* part3, double* col,
                           double* slash, cudaStream_t st) {
  s1_finalize<<<g.Hq * g.cn, 256, 0, st>>>(g, only, part3, col, slash);
  return check_launch("stage1 finalize");
}

int launch_stage1_exact(const Stage1Geom& g, const void* q, const void* k, int dtype,
                        const int* only, char* ws, const Workspace& L, double* col, double* slash,
                        cudaStream_t st) {
  int e;
  if (dtype == SA_FP32)
    e = run_exact(g, static_cast<const float*>(q), static_cast<const float*>(k), only, ws, L, st);
  else
    e = run_exact(g, static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k),
                  only, ws, L, st);
  if (e) return e;
  return launch_stage1_finalize(g, only, reinterpret_cast<const double*>(ws + L.part3), col, slash,
                                st);
}

}  // namespace sa
