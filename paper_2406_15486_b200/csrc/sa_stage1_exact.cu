// Stage 1, exact mode: fp64 re-statement of sample_scores + block_reduce
// (ref pkg/src/blocksift/sampler.py:135-191, math of core.py:110-154).
//
// Used (a) as the fp32-mode stage 1 and (b) as the selection guard's
// re-score of (head, chunk) pairs whose tensor-core scores sit too close to a
// find_k / arg_topk decision to trust (sa_select margin flags).
//
// Same single-pass structure as the tensor-core path, in fp64 on the SIMT
// pipes: one CTA per (head, chunk, key-block split) scores the window's rows
// against each key block (128 x 128 dot products, 8x8 fp64 register tiles),
// keeps a running per-row max m, and emits per (row, key block)
//     A = sum_{t <= r % blk} exp(s - m),  B = sum_{t > r % blk} exp(s - m)
// (causal keys only).  xf_rowfin / xf_fold then normalise with the rows'
// global max / sum and fold the rows into part3 (col + 3 slash bins per key
// block), deterministically (fixed reduction orders, no float atomics).
//
// Slash binning: for sampled row r and key j = kb*blk + t, the offset block is
// (r - j) // blk = r//blk - kb - (t > r % blk); a window of <= blk consecutive
// rows spans at most two values of r//blk, so one key block feeds bins
// X-1, X, X+1 with X = b0 - kb, b0 = sample_start // blk.
#include <cuda_bf16.h>

#include "sa_internal.h"

namespace sa {
namespace {

#ifndef SA_XF_DMMA
#define SA_XF_DMMA 1  // FP64 tensor-core inner products (0: the SIMT 8x8 register-tile version)
#endif
#ifndef SA_XF_W16
#define SA_XF_W16 1  // DMMA with 16 warps of one 8-row tile each (0: 8 warps of two tiles)
#endif
// SIMT: 16 x 16 threads, ty -> rows ty + 16a (a < 8), tx -> keys tx + 16b (b < 8).
// DMMA: warp w -> rows kMT*8*w .. +kMT*8 (kMT 8-row tiles) x all 128 keys.
constexpr int kThreads = (SA_XF_DMMA && SA_XF_W16) ? 512 : 256;
constexpr int kMT = (SA_XF_DMMA && SA_XF_W16) ? 1 : 2;
constexpr int kRows = 128;
constexpr int kKeys = 128;
constexpr int kDChunk = 64;    // head-dim slice staged per round

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
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

// stage rows [r0, r0+n) x dims [c0, c0+kDChunk) of a row-major [*, d] matrix into smem [kRows][kDChunk+1]
// (staged as fp64 so the inner product loop issues no conversions)
template <typename T>
__device__ void stage(double* dst, const T* src, int n, int d, int c0) {
  const int cn = min(kDChunk, d - c0);
  for (int e = threadIdx.x; e < kRows * kDChunk; e += kThreads) {
    const int r = e / kDChunk, c = e - r * kDChunk;
    dst[r * (kDChunk + 1) + c] = (r < n && c < cn) ? (double)to_f(src[(size_t)r * d + c0 + c]) : 0.0;
  }
}

// Work of one CTA: key blocks [kb0, kb1) of (head, chunk) hc.
template <typename T>
__device__ __forceinline__ void xf_work(const T* __restrict__ q, const T* __restrict__ k, const Stage1Geom& g,
                                        int hc, int kb0, int kb1, double* __restrict__ pa,
                                        double* __restrict__ pb, double* __restrict__ pm, double* qs,
                                        double* ks) {
  const int h = hc / g.cn, c = hc - h * g.cn;
  const Win w = window_of(c, g.S, g.blk, g.itv);
  kb1 = min(kb1, w.nkb);
  const int kvh = kv_head_of(h, g.group, g.q_head0);
  const int nr = w.se - w.ss, d = g.d, blk = g.blk;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const T* qh = q + ((size_t)h * g.S + w.ss) * d;
  const T* kh = k + (size_t)kvh * g.S * d;
  const double scale = 1.0 / sqrt((double)d);
  double m_run[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) m_run[a] = -INFINITY;

  for (int kb = kb0; kb < kb1; ++kb) {
    const int key0 = kb * blk;
    const int nk = min(blk, w.se - key0);  // keys of this block that any sampled row can see
    double acc[8][8];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
    for (int c0 = 0; c0 < d; c0 += kDChunk) {
      __syncthreads();
      stage(qs, qh, nr, d, c0);
      stage(ks, kh + (size_t)key0 * d, nk, d, c0);
      __syncthreads();
      const int cn = min(kDChunk, d - c0);
      for (int i = 0; i < cn; ++i) {
        double qv[8], kv[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) qv[a] = qs[(ty + 16 * a) * (kDChunk + 1) + i];
#pragma unroll
        for (int b = 0; b < 8; ++b) kv[b] = ks[(tx + 16 * b) * (kDChunk + 1) + i];
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
          for (int b = 0; b < 8; ++b) acc[a][b] = fma(qv[a], kv[b], acc[a][b]);
      }
    }
    // per row: block max over causal keys (16 tx lanes of the warp share a row set)
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int rl = ty + 16 * a;
      const int row = w.ss + rl;
      double mx = -INFINITY;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const int t = tx + 16 * b;
        acc[a][b] *= scale;
        if (t < nk && key0 + t <= row) mx = fmax(mx, acc[a][b]);
      }
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const double m_new = fmax(m_run[a], mx);
      const int rho = row % blk;
      double sa_ = 0.0, sb_ = 0.0;
      if (m_new != -INFINITY) {
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          const int t = tx + 16 * b;
          if (t < nk && key0 + t <= row) {
            const double p = exp(acc[a][b] - m_new);
            if (t <= rho) sa_ += p; else sb_ += p;
          }
        }
      }
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) {
        sa_ += __shfl_xor_sync(0xffffffffu, sa_, o);
        sb_ += __shfl_xor_sync(0xffffffffu, sb_, o);
      }
      m_run[a] = m_new;
      if (tx == 0 && rl < nr) {
        const size_t o = ((size_t)hc * blk + rl) * g.nb + kb;
        pa[o] = sa_;
        pb[o] = sb_;
        pm[o] = m_new;
      }
    }
  }
}


constexpr int kPitchD = 68;  // DMMA staging pitch (doubles): conflict-free fragment loads

template <typename T>
__device__ void stage_p(double* dst, const T* src, int n, int d, int c0) {
  const int cn = min(kDChunk, d - c0);
  for (int e = threadIdx.x; e < kRows * kDChunk; e += kThreads) {
    const int r = e / kDChunk, c = e - r * kDChunk;
    dst[r * kPitchD + c] = (r < n && c < cn) ? (double)to_f(src[(size_t)r * d + c0 + c]) : 0.0;
  }
}

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// xf_work on the FP64 tensor cores (mma.sync m8n8k4): warp w owns rows
// 16w..16w+15 (two 8-row tiles) x all 128 keys (sixteen 8-key tiles); lane
// (g = lane / 4, c = lane % 4) holds rows 16w + 8mt + g, keys 8nt + 2c + {0, 1}.
template <typename T>
__device__ __forceinline__ void xf_work_dmma(const T* __restrict__ q, const T* __restrict__ k, const Stage1Geom& g,
                                             int hc, int kb0, int kb1, double* __restrict__ pa,
                                             double* __restrict__ pb, double* __restrict__ pm, double* qs,
                                             double* ks) {
  const int h = hc / g.cn, c = hc - h * g.cn;
  const Win w = window_of(c, g.S, g.blk, g.itv);
  kb1 = min(kb1, w.nkb);
  const int kvh = kv_head_of(h, g.group, g.q_head0);
  const int nr = w.se - w.ss, d = g.d, blk = g.blk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, tg = lane & 3;
  const T* qh = q + ((size_t)h * g.S + w.ss) * d;
  const T* kh = k + (size_t)kvh * g.S * d;
  const double scale = 1.0 / sqrt((double)d);
  double m_run[kMT];
#pragma unroll
  for (int mt = 0; mt < kMT; ++mt) m_run[mt] = -INFINITY;
  for (int kb = kb0; kb < kb1; ++kb) {
    const int key0 = kb * blk;
    const int nk = min(blk, w.se - key0);
    double acc[kMT][16][2];
#pragma unroll
    for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
      for (int nt = 0; nt < 16; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    for (int c0 = 0; c0 < d; c0 += kDChunk) {
      __syncthreads();
      stage_p(qs, qh, nr, d, c0);
      stage_p(ks, kh + (size_t)key0 * d, nk, d, c0);
      __syncthreads();
      const int cn = min(kDChunk, d - c0);
      for (int kc = 0; kc < cn; kc += 4) {
        double a[kMT], b[16];
#pragma unroll
        for (int mt = 0; mt < kMT; ++mt) a[mt] = qs[(8 * kMT * warp + 8 * mt + gq) * kPitchD + kc + tg];
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) b[nt] = ks[(8 * nt + gq) * kPitchD + kc + tg];
#pragma unroll
        for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
          for (int nt = 0; nt < 16; ++nt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
      }
    }
#pragma unroll
    for (int mt = 0; mt < kMT; ++mt) {
      const int rl = 8 * kMT * warp + 8 * mt + gq;
      const int row = w.ss + rl;
      double mx = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 16; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int t = 8 * nt + 2 * tg + e;
          acc[mt][nt][e] *= scale;
          if (t < nk && key0 + t <= row) mx = fmax(mx, acc[mt][nt][e]);
        }
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const double m_new = fmax(m_run[mt], mx);
      const int rho = row % blk;
      double sa_ = 0.0, sb_ = 0.0;
      if (m_new != -INFINITY) {
#pragma unroll
        for (int nt = 0; nt < 16; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int t = 8 * nt + 2 * tg + e;
            if (t < nk && key0 + t <= row) {
              const double p = exp(acc[mt][nt][e] - m_new);
              if (t <= rho) sa_ += p; else sb_ += p;
            }
          }
      }
      sa_ += __shfl_xor_sync(0xffffffffu, sa_, 1);
      sb_ += __shfl_xor_sync(0xffffffffu, sb_, 1);
      sa_ += __shfl_xor_sync(0xffffffffu, sa_, 2);
      sb_ += __shfl_xor_sync(0xffffffffu, sb_, 2);
      m_run[mt] = m_new;
      if (tg == 0 && rl < nr) {
        const size_t o = ((size_t)hc * blk + rl) * g.nb + kb;
        pa[o] = sa_;
        pb[o] = sb_;
        pm[o] = m_new;
      }
    }
  }
}

// One CTA per (key-block split, pair slot).  For the guard's re-score every
// key block gets its own CTA so the few flagged pairs spread over all SMs, and
// the pair slots loop over the compacted flagged list (L.flag_list).
template <typename T>
__global__ void __launch_bounds__(kThreads, 1)
    xf_pass(const T* __restrict__ q, const T* __restrict__ k, Stage1Geom g, const int* __restrict__ list,
            int kb_per_cta, double* __restrict__ pa, double* __restrict__ pb, double* __restrict__ pm) {
  extern __shared__ double smem_d[];
  double* qs = smem_d;                                              // [kRows][pitch]
  double* ks = smem_d + kRows * (SA_XF_DMMA ? kPitchD : kDChunk + 1);  // [kKeys][pitch]
  const int n_pairs = list ? list[0] : g.Hq * g.cn;
  const int kb0 = blockIdx.x * kb_per_cta;
  for (int f = blockIdx.y; f < n_pairs; f += gridDim.y) {  // uniform per CTA
    const int hc = list ? list[1 + f] : f;
#if SA_XF_DMMA
    xf_work_dmma(q, k, g, hc, kb0, kb0 + kb_per_cta, pa, pb, pm, qs, ks);
#else
    xf_work(q, k, g, hc, kb0, kb0 + kb_per_cta, pa, pb, pm, qs, ks);
#endif
    __syncthreads();  // qs / ks are reused by the next pair
  }
}

}  // namespace

// Per sampled row: global max M and normaliser L over the row's key blocks.
// One warp per row, lanes stride the key blocks; fixed shuffle tree.
// TPlane = float with log2-domain maxima (tensor-core partials) or double
// with natural-log maxima (exact partials).
template <typename TPlane, bool kLog2>
__device__ __forceinline__ void rowfin_pair(Stage1Geom g, int hc, const TPlane* __restrict__ pa,
                                            const TPlane* __restrict__ pb, const TPlane* __restrict__ pm,
                                            double* __restrict__ rowstat) {
  const Win w = window_of(hc % g.cn, g.S, g.blk, g.itv);
  const int nr = w.se - w.ss;
  const int lane = threadIdx.x & 31, warps = blockDim.x >> 5;
  for (int rl = blockIdx.x * warps + (threadIdx.x >> 5); rl < nr; rl += gridDim.x * warps) {
    const size_t o = ((size_t)hc * g.blk + rl) * g.nb;
    double mx = -INFINITY;
    for (int kb = lane; kb < w.nkb; kb += 32) mx = fmax(mx, (double)pm[o + kb]);
    for (int s = 16; s > 0; s >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, s));
    double L = 0.0;
    for (int kb = lane; kb < w.nkb; kb += 32) {
      const double m = (double)pm[o + kb];
      if (m != -INFINITY) L += ((double)pa[o + kb] + (double)pb[o + kb]) * (kLog2 ? exp2(m - mx) : exp(m - mx));
    }
    for (int s = 16; s > 0; s >>= 1) L += __shfl_xor_sync(0xffffffffu, L, s);
    if (lane == 0) {
      rowstat[((size_t)hc * g.blk + rl) * 2] = mx;
      rowstat[((size_t)hc * g.blk + rl) * 2 + 1] = L;
    }
  }
}

template <typename TPlane, bool kLog2>
__global__ void s1_rowfin(Stage1Geom g, const int* __restrict__ list, const TPlane* __restrict__ pa,
                          const TPlane* __restrict__ pb, const TPlane* __restrict__ pm,
                          double* __restrict__ rowstat) {
  const int n_pairs = list ? list[0] : g.Hq * g.cn;
  for (int f = blockIdx.y; f < n_pairs; f += gridDim.y) {
    const int hc = list ? list[1 + f] : f;
    rowfin_pair<TPlane, kLog2>(g, hc, pa, pb, pm, rowstat);
  }
}

// Per key block: fold the rows' normalised partial masses into part3
// (col, slash X-1, X, X+1).  Thread per key block, rows in a fixed order.
template <typename TPlane, bool kLog2>
__device__ __forceinline__ void fold_pair(Stage1Geom g, int hc, const TPlane* __restrict__ pa,
                                          const TPlane* __restrict__ pb, const TPlane* __restrict__ pm,
                                          const double* __restrict__ rowstat, double* __restrict__ part3,
                                          double (*s_w)[2]) {
  const Win w = window_of(hc % g.cn, g.S, g.blk, g.itv);
  const int nr = w.se - w.ss;
  for (int r = threadIdx.x; r < nr; r += blockDim.x) {
    s_w[r][0] = rowstat[((size_t)hc * g.blk + r) * 2];
    s_w[r][1] = 1.0 / rowstat[((size_t)hc * g.blk + r) * 2 + 1];
  }
  __syncthreads();
  const int kb = blockIdx.x * blockDim.x + threadIdx.x;
  if (kb >= g.nb) return;
  double* out = part3 + ((size_t)hc * g.nb + kb) * 4;
  if (kb >= w.nkb) {
    out[0] = out[1] = out[2] = out[3] = 0.0;
    return;
  }
  const int b0 = w.ss / g.blk;
  double s4[4] = {0.0, 0.0, 0.0, 0.0};
  for (int r = 0; r < nr; ++r) {
    const size_t o = ((size_t)hc * g.blk + r) * g.nb + kb;
    const double m = (double)pm[o];
    if (m == -INFINITY) continue;
    const double wgt = (kLog2 ? exp2(m - s_w[r][0]) : exp(m - s_w[r][0])) * s_w[r][1];
    const double a = (double)pa[o] * wgt, b = (double)pb[o] * wgt;
    const int slot_a = (w.ss + r) / g.blk - b0 + 1;  // bin r//blk - kb, relative to X-1
    s4[0] += a + b;
    s4[1 + slot_a] += a;
    s4[slot_a] += b;  // bin r//blk - kb - 1
  }
  out[0] = s4[0];
  out[1] = s4[1];
  out[2] = s4[2];
  out[3] = s4[3];
}

template <typename TPlane, bool kLog2>
__global__ void s1_fold(Stage1Geom g, const int* __restrict__ list, const TPlane* __restrict__ pa,
                        const TPlane* __restrict__ pb, const TPlane* __restrict__ pm,
                        const double* __restrict__ rowstat, double* __restrict__ part3) {
  __shared__ double s_w[kMaxSimtBlk][2];  // (M, 1/L) per row
  const int n_pairs = list ? list[0] : g.Hq * g.cn;
  for (int f = blockIdx.y; f < n_pairs; f += gridDim.y) {
    fold_pair<TPlane, kLog2>(g, list ? list[1 + f] : f, pa, pb, pm, rowstat, part3, s_w);
    __syncthreads();  // s_w is reloaded for the next pair
  }
}

// part3 -> col / slash
__global__ void s1_finalize(Stage1Geom g, const int* __restrict__ list, const double* __restrict__ part3,
                            double* __restrict__ col, double* __restrict__ slash) {
  const int n_pairs = list ? list[0] : g.Hq * g.cn;
  if ((int)blockIdx.x >= n_pairs) return;
  const int hc = list ? list[1 + blockIdx.x] : (int)blockIdx.x;
  const Win w = window_of(hc % g.cn, g.S, g.blk, g.itv);
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

namespace {
__global__ void k_flag_compact(const int* __restrict__ only, int n, int* __restrict__ list) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (only[i]) list[1 + atomicAdd(&cnt, 1)] = i;  // order is irrelevant: pairs are independent
  __syncthreads();
  if (threadIdx.x == 0) list[0] = cnt;
}
}  // namespace

int launch_flag_compact(const int* only, int n, int* list, cudaStream_t st) {
  k_flag_compact<<<1, 1024, 0, st>>>(only, n, list);
  return check_launch("stage1 flag compaction");
}

template <typename TPlane, bool kLog2>
int launch_fold(const Stage1Geom& g, const int* only, const TPlane* pa, const TPlane* pb,
                const TPlane* pm, char* ws, const Workspace& L, double* col, double* slash,
                cudaStream_t st) {
  double* rowstat = reinterpret_cast<double*>(ws + L.rowstat);
  double* part3 = reinterpret_cast<double*>(ws + L.part3);
  const int n_all = g.Hq * g.cn;
  const int* list = nullptr;
  int rows = n_all;
  if (only) {  // the exact pass already compacted the flags for its own grid; rebuild (cheap) for the TC path
    int* fl = reinterpret_cast<int*>(ws + L.flag_list);
    if (int e = launch_flag_compact(only, n_all, fl, st)) return e;
    list = fl;
    rows = flagged_grid_rows(n_all);
  }
  s1_rowfin<TPlane, kLog2><<<dim3(16, rows), 256, 0, st>>>(g, list, pa, pb, pm, rowstat);
  if (int e = check_launch("stage1 rowfin")) return e;
  s1_fold<TPlane, kLog2><<<dim3(ceil_div(g.nb, 128), rows), 128, 0, st>>>(g, list, pa, pb, pm, rowstat, part3);
  if (int e = check_launch("stage1 fold")) return e;
  s1_finalize<<<only ? n_all : n_all, 256, 0, st>>>(g, list, part3, col, slash);
  return check_launch("stage1 finalize");
}

// ---- sampled-row retained mass from the stage-1 partials (ref pipeline.py:
// 37-58 _retained_by_block / _sampled_cra): for sampled row r of pair hc,
//   retained = sum over the key blocks kb active for query block r//blk of
//              (A + B)[r][kb] * exp(m[r][kb] - M_r) / L_r
// i.e. the row's normalised probability mass inside the mask, from the same
// partial planes and row statistics stage 1 folded into col / slash (tensor
// planes in the log2 domain, exact planes -- guard-rescored pairs or exact
// mode -- in the natural-log domain).  One CTA per pair, one thread per row.
__global__ void k_sampled_retained(Stage1Geom g, int exact_all, const int* __restrict__ rescored,
                                   const float* __restrict__ ta, const float* __restrict__ tb,
                                   const float* __restrict__ tm, const double* __restrict__ xa,
                                   const double* __restrict__ xb, const double* __restrict__ xm,
                                   const double* __restrict__ rowstat, const int* __restrict__ kv_cnt,
                                   const int* __restrict__ kv_idx, double* __restrict__ retained) {
  const int hc = blockIdx.x, h = hc / g.cn;
  const Win w = window_of(hc - h * g.cn, g.S, g.blk, g.itv);
  const bool exact = exact_all || (rescored && rescored[hc]);
  for (int r = threadIdx.x; r < g.blk; r += blockDim.x) {
    const size_t ro = (size_t)hc * g.blk + r;
    if (r >= w.se - w.ss) {
      retained[ro] = nan("");
      continue;
    }
    const int row = w.ss + r, qb = row / g.blk;
    const double M = rowstat[ro * 2], invL = 1.0 / rowstat[ro * 2 + 1];
    const int n = kv_cnt[(size_t)h * g.nb + qb];
    const int* list = kv_idx + (size_t)h * tri(g.nb) + tri(qb);
    double acc = 0.0;
    for (int j = 0; j < n; ++j) {
      const size_t o = ro * g.nb + list[j];
      if (exact) {
        const double m = xm[o];
        if (m != -INFINITY) acc += (xa[o] + xb[o]) * exp(m - M);
      } else {
        const double m = (double)tm[o];
        if (m != -INFINITY) acc += ((double)ta[o] + (double)tb[o]) * exp2(m - M);
      }
    }
    retained[ro] = acc * invL;
  }
}

int launch_sampled_retained(const Stage1Geom& g, int exact_all, const int* rescored, const int* kv_cnt,
                            const int* kv_idx, const char* ws, const Workspace& L, double* retained,
                            cudaStream_t st) {
  const size_t plane = (size_t)g.Hq * g.cn * g.blk * g.nb;
  const float* ta = reinterpret_cast<const float*>(ws + L.tc_part);
  const double* xa = reinterpret_cast<const double*>(ws + L.x_part);
  k_sampled_retained<<<g.Hq * g.cn, 128, 0, st>>>(g, exact_all, rescored, ta, ta + plane, ta + 2 * plane, xa,
                                                  xa + plane, xa + 2 * plane,
                                                  reinterpret_cast<const double*>(ws + L.rowstat), kv_cnt, kv_idx,
                                                  retained);
  return check_launch("sampled retained mass");
}

template int launch_fold<float, true>(const Stage1Geom&, const int*, const float*, const float*,
                                      const float*, char*, const Workspace&, double*, double*,
                                      cudaStream_t);

namespace {
template <typename T>
int run_exact(const Stage1Geom& g, const T* q, const T* k, const int* only, char* ws, const Workspace& L,
              double* col, double* slash, cudaStream_t st) {
  const size_t smem = (size_t)(kRows + kKeys) * (SA_XF_DMMA ? kPitchD : kDChunk + 1) * sizeof(double);
  set_smem_attr(reinterpret_cast<const void*>(&xf_pass<T>), (int)smem);
  const size_t plane = (size_t)g.Hq * g.cn * g.blk * g.nb;
  double* pa = reinterpret_cast<double*>(ws + L.x_part);
  double* pb = pa + plane;
  double* pm = pb + plane;
  const long long work = (long long)g.Hq * g.cn * g.nb;
  const int kpc = only ? 1 : (int)std::max<long long>(2, std::min<long long>(32, work / (148LL * 4)));
  const int n_all = g.Hq * g.cn;
  int* list = nullptr;
  if (only) {
    list = reinterpret_cast<int*>(ws + L.flag_list);
    if (int e = launch_flag_compact(only, n_all, list, st)) return e;
  }
  const int rows = only ? flagged_grid_rows(n_all) : n_all;
  xf_pass<T><<<dim3(ceil_div(g.nb, kpc), rows), kThreads, smem, st>>>(q, k, g, list, kpc, pa, pb, pm);
  if (int e = check_launch("stage1 exact pass")) return e;
  return launch_fold<double, false>(g, only, pa, pb, pm, ws, L, col, slash, st);
}
}  // namespace

int launch_stage1_exact(const Stage1Geom& g, const void* q, const void* k, int dtype, const int* only,
                        char* ws, const Workspace& L, double* col, double* slash, cudaStream_t st) {
  if (dtype == SA_FP32)
    return run_exact(g, static_cast<const float*>(q), static_cast<const float*>(k), only, ws, L, col, slash, st);
  return run_exact(g, static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k), only, ws, L,
                   col, slash, st);
}

}  // namespace sa
