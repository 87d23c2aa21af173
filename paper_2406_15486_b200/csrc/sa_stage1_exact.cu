// Stage 1, exact mode: fp64 re-statement of sample_scores + block_reduce
// (ref pkg/src/blocksift/sampler.py:135-191, math of core.py:110-154).
//
// Used (a) as the fp32-mode stage 1 and (b) as the selection guard's
// re-score of (head, chunk) pairs whose tensor-core scores sit too close to a
// find_k / arg_topk decision to trust (sa_select margin flags).
//
// Same single-pass structure as the tensor-core path, in fp64: one CTA per
// (head, chunk, key-block split) scores the window's rows against each key
// block (128 x 128 dot products on the FP64 tensor cores, mma.sync m8n8k4),
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

// 16 warps; warp w owns rows 8w..8w+7 of the window x all 128 keys of a block.
constexpr int kThreads = 512;
constexpr int kRows = 128;
constexpr int kKeys = 128;
constexpr int kDChunk = 64;      // head-dim slice of K staged per round (double-buffered, fp64)
constexpr int kPitchQ = 132;     // smem pitches: conflict-free m8n8k4 fragment loads (Q raw, K fp64 = 4 mod 32)
constexpr int kPitchK = 68;
template <typename T>
constexpr int xf_smem_bytes() {  // Q raw (T), then two fp64 K slices (8-byte aligned: kRows * kPitchQ * 2 % 8 == 0)
  return kRows * kPitchQ * (int)sizeof(T) + 2 * kKeys * kPitchK * 8;
}

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

// 16 consecutive elements of row r, dims [c, c+16), of a row-major [n, d]
// matrix, zero past n rows / d dims, held RAW (8 registers for bf16): 16-byte
// loads when d allows it; converted to fp64 only when stored into the smem slice.
template <typename T>
struct Slice16 {
  T v[16];
  __device__ __forceinline__ void load(const T* __restrict__ src, int r, int n, int c, int d) {
    if (r >= n || c >= d) {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = T(0.f);
      return;
    }
    const T* p = src + (size_t)r * d + c;
    if (c + 16 <= d && d % 8 == 0) {
#pragma unroll
      for (int i = 0; i < (int)(16 * sizeof(T) / 16); ++i)
        reinterpret_cast<uint4*>(v)[i] = reinterpret_cast<const uint4*>(p)[i];
      return;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = c + i < d ? p[i] : T(0.f);
  }
  __device__ __forceinline__ void store(double* dst) const {
#pragma unroll
    for (int i = 0; i < 16; i += 2)
      *reinterpret_cast<double2*>(dst + i) = make_double2((double)to_f(v[i]), (double)to_f(v[i + 1]));
  }
};

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Work of one CTA: the key blocks `kbs` of (head, chunk) hc.  The window's
// query rows are staged once, raw (converted to fp64 per MMA fragment: one
// conversion per 16 MMAs); K streams through two 64-dim fp64 smem slices, the
// next slice's global loads issued into registers before the current slice's
// MMAs so their latency hides under them.  Lane (gq = lane / 4, tg = lane % 4)
// of warp w holds rows 8w + gq, keys 8nt + 2tg + {0, 1}.
// The key blocks: a range (xf_pass: maxima run across the range, as the
// fold expects) or entries of the band work list (xf_items: each block's
// maximum its own, so a block listed twice is written with identical values).
struct KbRange {
  int kb0, n;
  static constexpr bool kRunning = true;
  __device__ __forceinline__ int operator()(int i) const { return kb0 + i; }
};
struct KbList {
  const int* items;  // [count, (pair, key block)...]
  int i0, n;
  static constexpr bool kRunning = false;
  __device__ __forceinline__ int operator()(int i) const { return items[2 + 2 * (i0 + i)]; }
};

template <typename T, typename KB>
__device__ __forceinline__ void xf_work(const T* __restrict__ q, const T* __restrict__ k, const Stage1Geom& g,
                                        int hc, KB kbs, double* __restrict__ pa, double* __restrict__ pb,
                                        double* __restrict__ pm, T* qs, double* ks) {
  const int h = hc / g.cn, c = hc - h * g.cn;
  const Win w = window_of(c, g.S, g.blk, g.itv);
  if (kbs.n <= 0) return;
  const int kvh = kv_head_of(h, g.group, g.q_head0);
  const int nr = w.se - w.ss, d = g.d, blk = g.blk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, tg = lane & 3;
  const T* qh = q + ((size_t)h * g.S + w.ss) * d;
  const T* kh = k + (size_t)kvh * g.S * d;
  const double scale = 1.0 / sqrt((double)d);
  const int nch = (d + kDChunk - 1) / kDChunk;  // K slices per key block
  for (int e = threadIdx.x; e < kRows * kPitchQ; e += kThreads) {  // Q once, all dims (zero pad)
    const int r = e / kPitchQ, cc = e - r * kPitchQ;
    qs[e] = (r < nr && cc < d) ? qh[(size_t)r * d + cc] : T(0.f);
  }
  // staging map: thread -> (row, 16 dims) of a 128 x 64 slice
  const int sr = threadIdx.x >> 2, sc = (threadIdx.x & 3) * 16;
  auto nk_of = [&](int kb) { return min(blk, w.se - kb * blk); };  // keys any sampled row can see
  Slice16<T> nxt;
  int kb = kbs(0);
  nxt.load(kh + (size_t)kb * blk * d, sr, nk_of(kb), sc, d);
  nxt.store(ks + sr * kPitchK + sc);
  __syncthreads();
  double m_run = -INFINITY;
  int buf = 0;
  for (int it = 0; it < kbs.n; ++it) {
    kb = kbs(it);
    const int kb_next = it + 1 < kbs.n ? kbs(it + 1) : -1;
    if (!KB::kRunning) m_run = -INFINITY;
    const int key0 = kb * blk;
    const int nk = nk_of(kb);
    double acc[16][2];
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
    for (int ch = 0; ch < nch; ++ch) {
      // prefetch the next slice (this block's next 64 dims, or the next block's first)
      const bool more = ch + 1 < nch || kb_next >= 0;
      if (more) {
        const int kbn = ch + 1 < nch ? kb : kb_next, chn = ch + 1 < nch ? ch + 1 : 0;
        nxt.load(kh + (size_t)kbn * blk * d, sr, nk_of(kbn), chn * kDChunk + sc, d);
      }
      const double* kq = ks + buf * (kKeys * kPitchK);
      const T* qq = qs + (8 * warp + gq) * kPitchQ + ch * kDChunk + tg;
#pragma unroll 4
      for (int kc = 0; kc < kDChunk; kc += 4) {
        const double a = (double)to_f(qq[kc]);
        double b[16];
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) b[nt] = kq[(8 * nt + gq) * kPitchK + kc + tg];
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) dmma_8x8x4(acc[nt][0], acc[nt][1], a, b[nt]);
      }
      if (more) nxt.store(ks + (buf ^ 1) * (kKeys * kPitchK) + sr * kPitchK + sc);
      buf ^= 1;
      __syncthreads();
    }
    const int rl = 8 * warp + gq;
    const int row = w.ss + rl;
    double mx = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 16; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int t = 8 * nt + 2 * tg + e;
        acc[nt][e] *= scale;
        if (t < nk && key0 + t <= row) mx = fmax(mx, acc[nt][e]);
      }
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const double m_new = fmax(m_run, mx);
    const int rho = row % blk;
    double sa_ = 0.0, sb_ = 0.0;
    if (m_new != -INFINITY) {
#pragma unroll
      for (int nt = 0; nt < 16; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int t = 8 * nt + 2 * tg + e;
          if (t < nk && key0 + t <= row) {
            const double p = exp(acc[nt][e] - m_new);
            if (t <= rho) sa_ += p; else sb_ += p;
          }
        }
    }
    sa_ += __shfl_xor_sync(0xffffffffu, sa_, 1);
    sb_ += __shfl_xor_sync(0xffffffffu, sb_, 1);
    sa_ += __shfl_xor_sync(0xffffffffu, sa_, 2);
    sb_ += __shfl_xor_sync(0xffffffffu, sb_, 2);
    m_run = m_new;
    if (tg == 0 && rl < nr) {
      const size_t o = ((size_t)hc * blk + rl) * g.nb + kb;
      pa[o] = sa_;
      pb[o] = sb_;
      pm[o] = m_new;
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
  T* qs = reinterpret_cast<T*>(smem_d);                                                  // [kRows][kPitchQ] raw
  double* ks = reinterpret_cast<double*>(reinterpret_cast<char*>(smem_d) + kRows * kPitchQ * sizeof(T));  // 2 x slice
  const int n_pairs = list ? list[0] : g.Hq * g.cn;
  const int kb0 = blockIdx.x * kb_per_cta;
  for (int f = blockIdx.y; f < n_pairs; f += gridDim.y) {  // uniform per CTA
    const int hc = list ? list[1 + f] : f;
    const int nkb = window_of(hc % g.cn, g.S, g.blk, g.itv).nkb;
    xf_work(q, k, g, hc, KbRange{kb0, min(kb0 + kb_per_cta, nkb) - kb0}, pa, pb, pm, qs, ks);
    __syncthreads();  // qs / ks are reused by the next pair
  }
}

// Exact partials of an explicit (pair, key block) work list (band
// refinement): CTA j takes the j-th run of ceil(n / gridDim.x) consecutive
// items and stages Q once per stretch of one pair (k_band_items writes each
// band entry's blocks contiguously, ascending).
template <typename T>
__global__ void __launch_bounds__(kThreads, 1)
    xf_items(const T* __restrict__ q, const T* __restrict__ k, Stage1Geom g, const int* __restrict__ items,
             double* __restrict__ pa, double* __restrict__ pb, double* __restrict__ pm) {
  extern __shared__ double smem_d[];
  T* qs = reinterpret_cast<T*>(smem_d);
  double* ks = reinterpret_cast<double*>(reinterpret_cast<char*>(smem_d) + kRows * kPitchQ * sizeof(T));
  const int n = items[0];
  const int per = (n + gridDim.x - 1) / gridDim.x;
  const int i1 = min(n, (int)(blockIdx.x + 1) * per);
  for (int i = blockIdx.x * per; i < i1;) {  // uniform per CTA
    const int hc = items[1 + 2 * i];
    int j = i + 1;
    while (j < i1 && items[1 + 2 * j] == hc) ++j;
    xf_work(q, k, g, hc, KbList{items, i, j - i}, pa, pb, pm, qs, ks);
    __syncthreads();
    i = j;
  }
}

// Band entries -> (pair, key block) work items: a col band lists key blocks,
// a slash band lists offset bins o, each read from key blocks X - o (keys at or
// below the row's own offset in its block) and X - o - 1 for the query
// block(s) X the sampled window spans.  Pairs already flagged for the full
// re-score are skipped.  One CTA per pair: the key blocks both of its entries
// need are marked in a shared bitmap (dynamic smem, one bit per key block) and
// written out once each, ascending, under one atomicAdd on the list's count.
constexpr int kItemThreads = 128;

__global__ void __launch_bounds__(kItemThreads)
    k_band_items(Stage1Geom g, const int* __restrict__ band, const int* __restrict__ flags,
                 int* __restrict__ band_pairs, int* __restrict__ items) {
  extern __shared__ unsigned bits[];
  __shared__ int s_warp[kItemThreads / 32], s_base;
  const int hc = blockIdx.x;
  const int* ent_c = band + (size_t)(2 * hc) * kBandEntry;
  const int* ent_s = ent_c + kBandEntry;
  const int nc = ent_c[0], ns = ent_s[0];
  if ((nc <= 0 && ns <= 0) || flags[hc]) return;
  if (threadIdx.x == 0) band_pairs[hc] = 1;
  const Win w = window_of(hc % g.cn, g.S, g.blk, g.itv);
  const int X0 = w.ss / g.blk, X1 = (w.se - 1) / g.blk;
  const int nw = (w.nkb + 31) >> 5;
  for (int i = threadIdx.x; i < nw; i += kItemThreads) bits[i] = 0u;
  __syncthreads();
  auto mark = [&](int kb) {
    if (kb >= 0 && kb < w.nkb) atomicOr(bits + (kb >> 5), 1u << (kb & 31));
  };
  for (int i = threadIdx.x; i < nc; i += kItemThreads) mark(ent_c[kBandHdr + i]);
  for (int i = threadIdx.x; i < ns; i += kItemThreads) {
    const int b = ent_s[kBandHdr + i];
    for (int X = X0; X <= X1; ++X) {
      mark(X - b);
      mark(X - b - 1);
    }
  }
  __syncthreads();
  // thread t owns words [t * per, (t + 1) * per): count, block exclusive scan, write ascending
  const int per = (nw + kItemThreads - 1) / kItemThreads;
  const int w0 = threadIdx.x * per, w1 = min(nw, w0 + per);
  int cnt = 0;
  for (int i = w0; i < w1; ++i) cnt += __popc(bits[i]);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int i = 0; i < kItemThreads / 32; ++i) tot += s_warp[i];
    s_base = atomicAdd(items, tot);
  }
  __syncthreads();
  int at = s_base + incl - cnt;
  for (int i = 0; i < wid; ++i) at += s_warp[i];
  for (int i = w0; i < w1; ++i)
    for (unsigned m = bits[i]; m; m &= m - 1) {
      const int kb = (i << 5) + __ffs(m) - 1;
      items[1 + 2 * at] = hc;
      items[2 + 2 * at] = kb;
      ++at;
    }
}

// Row r's normalised exact mass in band block / bin b of pair hc: the exact
// (fp64) partials of the key blocks it covers, scaled by the tensor-core row
// statistics (M in log2 units, L): part_r * exp(m_r - M_r ln2) / L_r.
struct BandRow {
  const double *xa, *xb, *xm;
  size_t row;  // (hc * blk + r) * nb: the row's partial-plane offset
  int nkb, X;  // key blocks of the window; query block of the row
  double M, invL;
  __device__ double plane(const double* pl, int kb) const {
    if (kb < 0 || kb >= nkb) return 0.0;
    const double m = xm[row + kb];
    return m == -INFINITY ? 0.0 : pl[row + kb] * exp(m - M) * invL;
  }
  __device__ double mass(int dir, int b) const {
    if (dir == 0) {  // both parts of key block b share its maximum
      if (b < 0 || b >= nkb) return 0.0;
      const double m = xm[row + b];
      return m == -INFINITY ? 0.0 : (xa[row + b] + xb[row + b]) * exp(m - M) * invL;
    }
    return plane(xa, X - b) + plane(xb, X - b - 1);
  }
};

__device__ __forceinline__ BandRow band_row(const Stage1Geom& g, int hc, int r, const Win& w, const double* xa,
                                            const double* xb, const double* xm, const double* rowstat) {
  const size_t ro = (size_t)hc * g.blk + r;
  return BandRow{xa, xb, xm, ro * g.nb, w.nkb, (w.ss + r) / g.blk, rowstat[ro * 2] * 0.6931471805599453,
                 1.0 / rowstat[ro * 2 + 1]};
}

// Fixed-order sum over the window's rows of f(row) by one warp: lane l adds
// rows l, l + 32, l + 64, l + 96 in that order, then a fixed xor-shuffle tree
// (deterministic).  Returns the sum on every lane.
template <typename F>
__device__ __forceinline__ double warp_rows_sum(int nr, F f) {
  double v[kRows / 32];
#pragma unroll
  for (int j = 0; j < kRows / 32; ++j) {  // unrolled: every row's loads in flight at once
    const int r = (threadIdx.x & 31) + 32 * j;
    v[j] = r < nr ? f(r) : 0.0;
  }
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < kRows / 32; ++j) acc += v[j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

constexpr int kBandWarps = 8;

// Refined band scores: per band block, the sum over the window's rows of the
// exact (fp64) mass in the block / bin, normalised with the tensor-core row
// statistics.  One CTA per band entry, its warps stride over the entry's
// blocks; rows are added in a fixed order (deterministic).  Overwrites col /
// slash.
__global__ void __launch_bounds__(kBandWarps * 32)
    k_band_scores(Stage1Geom g, const int* __restrict__ band, const int* __restrict__ flags,
                  const double* __restrict__ xa, const double* __restrict__ xb, const double* __restrict__ xm,
                  const double* __restrict__ rowstat, double* __restrict__ col, double* __restrict__ slash) {
  const int e = blockIdx.x, hc = e >> 1, dir = e & 1;
  const int* ent = band + (size_t)e * kBandEntry;
  const int n = ent[0];
  if (n <= 0 || flags[hc]) return;
  const Win w = window_of(hc % g.cn, g.S, g.blk, g.itv);
  const int nr = w.se - w.ss;
  double* out = (dir == 0 ? col : slash) + (size_t)hc * g.nb;
  for (int i = threadIdx.x >> 5; i < n; i += kBandWarps) {
    const int b = ent[kBandHdr + i];
    const double acc = warp_rows_sum(nr, [&](int r) { return band_row(g, hc, r, w, xa, xb, xm, rowstat).mass(dir, b); });
    if ((threadIdx.x & 31) == 0) out[b] = acc;
  }
}

// Per-row certificate of the order of the two refined blocks a, b at a
// certified cut (band entry slots 2, 3, left by sa_select's certify pass when
// band_eps * (s_a + s_b) could not settle it).  Row r's normaliser error d_r
// (|d_r| <= band_eps * scale) scales x_ra and x_rb alike, so the refined
// difference s_a - s_b = sum_r (x_ra - x_rb) / (1 + d_r) is off by at most
// band_eps * scale * sum_r |x_ra - x_rb|: a larger gap fixes the exact order;
// else the pair is flagged for the full re-score.
__global__ void k_band_ties(Stage1Geom g, const int* __restrict__ band, int* __restrict__ flags,
                            const double* __restrict__ xa, const double* __restrict__ xb,
                            const double* __restrict__ xm, const double* __restrict__ rowstat,
                            const double* __restrict__ col, const double* __restrict__ slash,
                            const double* __restrict__ bound, double bound_ref, double band_eps) {
  const int e = blockIdx.x, hc = e >> 1, dir = e & 1;
  const int* ent = band + (size_t)e * kBandEntry;
  if (ent[0] <= 0 || ent[2] < 0 || flags[hc]) return;
  const int a = ent[2], b = ent[3];
  const Win w = window_of(hc % g.cn, g.S, g.blk, g.itv);
  const double W = warp_rows_sum(w.se - w.ss, [&](int r) {
    const BandRow br = band_row(g, hc, r, w, xa, xb, xm, rowstat);
    return fabs(br.mass(dir, a) - br.mass(dir, b));
  });
  if (threadIdx.x == 0) {
    const double* s = (dir == 0 ? col : slash) + (size_t)hc * g.nb;
    const double scale = bound ? fmax(1.0, bound[hc] / bound_ref) : 1.0;
    if (!(s[a] - s[b] > band_eps * scale * W)) atomicOr(flags + hc, 1);
  }
}

}  // namespace

int launch_refine_bands(const Stage1Geom& g, const void* q, const void* k, int dtype, const int* band,
                        const int* flags, int* band_pairs, const double* row_stats, char* ws, const Workspace& L,
                        double* col, double* slash, cudaStream_t st) {
  int* items = reinterpret_cast<int*>(ws + L.band_items);
  const int n_ent = g.Hq * g.cn * 2;
  cudaMemsetAsync(items, 0, sizeof(int), st);
  cudaMemsetAsync(band_pairs, 0, sizeof(int) * g.Hq * g.cn, st);
  const int bitmap_bytes = ceil_div(g.nb, 32) * 4;
  if (bitmap_bytes > 48 * 1024) set_smem_attr(reinterpret_cast<const void*>(&k_band_items), bitmap_bytes);
  k_band_items<<<g.Hq * g.cn, kItemThreads, bitmap_bytes, st>>>(g, band, flags, band_pairs, items);
  if (int e = check_launch("band refinement: work list")) return e;
  const size_t plane = (size_t)g.Hq * g.cn * g.blk * g.nb;
  double* pa = reinterpret_cast<double*>(ws + L.x_part);
  double* pb = pa + plane;
  double* pm = pb + plane;
  if (dtype == SA_FP32) {
    set_smem_attr(reinterpret_cast<const void*>(&xf_items<float>), xf_smem_bytes<float>());
    xf_items<float><<<148, kThreads, xf_smem_bytes<float>(), st>>>(
        static_cast<const float*>(q), static_cast<const float*>(k), g, items, pa, pb, pm);
  } else {
    set_smem_attr(reinterpret_cast<const void*>(&xf_items<__nv_bfloat16>), xf_smem_bytes<__nv_bfloat16>());
    xf_items<__nv_bfloat16><<<148, kThreads, xf_smem_bytes<__nv_bfloat16>(), st>>>(
        static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k), g, items, pa, pb, pm);
  }
  if (int e = check_launch("band refinement: exact partials")) return e;
  k_band_scores<<<n_ent, kBandWarps * 32, 0, st>>>(g, band, flags, pa, pb, pm, row_stats, col, slash);
  return check_launch("band refinement: scores");
}

int launch_band_ties(const Stage1Geom& g, const int* band, int* flags, const double* row_stats, const double* col,
                     const double* slash, const double* bound, double bound_ref, double band_eps, char* ws,
                     const Workspace& L, cudaStream_t st) {
  const size_t plane = (size_t)g.Hq * g.cn * g.blk * g.nb;
  const double* pa = reinterpret_cast<const double*>(ws + L.x_part);
  k_band_ties<<<g.Hq * g.cn * 2, 32, 0, st>>>(g, band, flags, pa, pa + plane, pa + 2 * plane, row_stats, col,
                                                 slash, bound, bound_ref, band_eps);
  return check_launch("band refinement: per-row tie certificate");
}

// loads issued per batch in the fold / row-statistics kernels (4 beat 8 and 16
// in profiles/r2/s3/foldb_*.txt)
constexpr int kRowfinBatch = 4;
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
    // the lane's key blocks in batches of 4: loads first, then the sums in order
    for (int kb0 = lane; kb0 < w.nkb; kb0 += kRowfinBatch * 32) {
      TPlane m_[kRowfinBatch], ab_[kRowfinBatch][2];
#pragma unroll
      for (int u = 0; u < kRowfinBatch; ++u) {
        const int kb = kb0 + 32 * u;
        const bool in = kb < w.nkb;
        m_[u] = in ? pm[o + kb] : (TPlane)-INFINITY;
        ab_[u][0] = in ? pa[o + kb] : (TPlane)0;
        ab_[u][1] = in ? pb[o + kb] : (TPlane)0;
      }
#pragma unroll
      for (int u = 0; u < kRowfinBatch; ++u) {
        const double m = (double)m_[u];
        if (m != -INFINITY)
          L += ((double)ab_[u][0] + (double)ab_[u][1]) * (kLog2 ? exp2(m - mx) : exp(m - mx));
      }
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
// (col, slash X-1, X, X+1).  A CTA covers 32 key blocks of one pair with 8
// row groups of 16 rows (256 threads: lanes = key blocks, so every row's loads
// are coalesced); each thread folds its rows in order and the 8 partial sums
// are added in group order, so the result is deterministic.  (A thread per
// key block looping over all 128 rows left the fold latency-bound: ~140 us
// at C3 for 50 MB.)
constexpr int kFoldKb = 32, kFoldGroups = 8, kFoldBatch = 4;

template <typename TPlane, bool kLog2>
__device__ __forceinline__ void fold_pair(Stage1Geom g, int hc, const TPlane* __restrict__ pa,
                                          const TPlane* __restrict__ pb, const TPlane* __restrict__ pm,
                                          const double* __restrict__ rowstat, double* __restrict__ part3,
                                          double (*s_w)[2], double (*s_acc)[kFoldKb][4]) {
  const Win w = window_of(hc % g.cn, g.S, g.blk, g.itv);
  const int nr = w.se - w.ss;
  for (int r = threadIdx.x; r < nr; r += blockDim.x) {
    s_w[r][0] = rowstat[((size_t)hc * g.blk + r) * 2];
    s_w[r][1] = 1.0 / rowstat[((size_t)hc * g.blk + r) * 2 + 1];
  }
  __syncthreads();
  const int lane = threadIdx.x % kFoldKb, grp = threadIdx.x / kFoldKb;
  const int kb = blockIdx.x * kFoldKb + lane;
  const int b0 = w.ss / g.blk;
  const int per = (g.blk + kFoldGroups - 1) / kFoldGroups;
  double s4[4] = {0.0, 0.0, 0.0, 0.0};
  if (kb < w.nkb) {
    const int r1 = min(nr, (grp + 1) * per);
    // rows in batches of kFoldBatch: the batch's loads are issued before any of
    // its arithmetic (the fold is load-latency bound), rows still added in order
    for (int rb = grp * per; rb < r1; rb += kFoldBatch) {
      TPlane m_[kFoldBatch], a_[kFoldBatch], b_[kFoldBatch];
#pragma unroll
      for (int u = 0; u < kFoldBatch; ++u) {
        const size_t o = ((size_t)hc * g.blk + rb + u) * g.nb + kb;
        const bool in = rb + u < r1;
        m_[u] = in ? pm[o] : (TPlane)-INFINITY;
        a_[u] = in ? pa[o] : (TPlane)0;
        b_[u] = in ? pb[o] : (TPlane)0;
      }
#pragma unroll
      for (int u = 0; u < kFoldBatch; ++u) {
        const int r = rb + u;
        const double m = (double)m_[u];
        if (m == -INFINITY) continue;
        const double wgt = (kLog2 ? exp2(m - s_w[r][0]) : exp(m - s_w[r][0])) * s_w[r][1];
        const double a = (double)a_[u] * wgt, b = (double)b_[u] * wgt;
        const int slot_a = (w.ss + r) / g.blk - b0 + 1;  // bin r//blk - kb, relative to X-1
        s4[0] += a + b;
        s4[1 + slot_a] += a;
        s4[slot_a] += b;  // bin r//blk - kb - 1
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) s_acc[grp][lane][i] = s4[i];
  __syncthreads();
  if (grp == 0 && kb < g.nb) {
    double t4[4] = {0.0, 0.0, 0.0, 0.0};
    if (kb < w.nkb)
      for (int x = 0; x < kFoldGroups; ++x)
#pragma unroll
        for (int i = 0; i < 4; ++i) t4[i] += s_acc[x][lane][i];
    double* out = part3 + ((size_t)hc * g.nb + kb) * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) out[i] = t4[i];
  }
}

template <typename TPlane, bool kLog2>
__global__ void __launch_bounds__(kFoldKb * kFoldGroups)
    s1_fold(Stage1Geom g, const int* __restrict__ list, const TPlane* __restrict__ pa,
            const TPlane* __restrict__ pb, const TPlane* __restrict__ pm,
            const double* __restrict__ rowstat, double* __restrict__ part3) {
  __shared__ double s_w[kMaxSimtBlk][2];                  // (M, 1/L) per row
  __shared__ double s_acc[kFoldGroups][kFoldKb][4];       // per row group
  const int n_pairs = list ? list[0] : g.Hq * g.cn;
  for (int f = blockIdx.y; f < n_pairs; f += gridDim.y) {
    fold_pair<TPlane, kLog2>(g, list ? list[1 + f] : f, pa, pb, pm, rowstat, part3, s_w, s_acc);
    __syncthreads();  // s_w / s_acc are reloaded for the next pair
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
  s1_fold<TPlane, kLog2><<<dim3(ceil_div(g.nb, kFoldKb), rows), kFoldKb * kFoldGroups, 0, st>>>(
      g, list, pa, pb, pm, rowstat, part3);
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
  const size_t smem = xf_smem_bytes<T>();
  set_smem_attr(reinterpret_cast<const void*>(&xf_pass<T>), (int)smem);
  const size_t plane = (size_t)g.Hq * g.cn * g.blk * g.nb;
  double* pa = reinterpret_cast<double*>(ws + L.x_part);
  double* pb = pa + plane;
  double* pm = pb + plane;
  // key blocks per CTA: Q is staged once per CTA, so longer runs amortise it;
  // the flagged-pair grid (few pairs) keeps ~4+ waves on the SMs
  const long long work = (long long)g.Hq * g.cn * g.nb;
  const int kpc = only ? 8 : (int)std::max<long long>(2, std::min<long long>(32, work / (148LL * 4)));
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
