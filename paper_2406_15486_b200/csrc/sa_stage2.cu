// Stage 2: minimal-quota selection and block-mask assembly.
//
// k2_select  replaces find_k + arg_topk (ref pkg/src/blocksift/filtering.py:30-62)
//            for every (head, chunk, direction) of select_and_merge (:245-255):
//            block-wide bitonic sort on (score desc, index asc), the reference's
//            SEQUENTIAL fp64 cumulative sum (bit-exact with np.cumsum), first
//            index with cum >= alpha * cum[-1], then the picked index set
//            compacted in ascending order.  Optional selection guard: flags a
//            (head, chunk) whose alpha cut or boundary tie gap lies within
//            eps * total of a decision.
// k2_merge   replaces merge_index (:198-230): one warp per (head, query block)
//            builds the union of column picks (kb <= qb), slash picks
//            ({qb-ob-1, qb-ob} clipped to [0, qb]) of the 1-2 chunks whose
//            region covers qb, and the diagonal, as an ascending list.
// k2_full    dense causal mask (the dense comparison row).
// k2_units   stage-3 work units (two items of one KV head), longest-first.
#include <algorithm>

#include "sa_internal.h"

namespace sa {
namespace {

constexpr int kSelThreads = 1024;

__device__ __forceinline__ bool before(unsigned long long ka, int ia, unsigned long long kb_, int ib) {
  return ka > kb_ || (ka == kb_ && ia < ib);
}

__global__ void __launch_bounds__(kSelThreads)
    k2_select(const double* __restrict__ col, const double* __restrict__ slash, int cn, int nb,
              int npow2, double alpha_c, double alpha_s, double eps, const double* __restrict__ bound,
              double bound_ref, int* __restrict__ flags,
              const int* __restrict__ only, const int* __restrict__ k_in, int* __restrict__ k_out,
              int* __restrict__ idx_out, int* __restrict__ band, double band_eps) {
  extern __shared__ unsigned char smem_raw[];
  const int dir = blockIdx.x, hc = blockIdx.y;
  if (only && only[hc] == 0) return;
  unsigned long long* key = reinterpret_cast<unsigned long long*>(smem_raw);  // [npow2]
  double* cum = reinterpret_cast<double*>(key + npow2);                      // [npow2]
  int* idx = reinterpret_cast<int*>(cum + npow2);                            // [npow2]
  unsigned char* mark = reinterpret_cast<unsigned char*>(idx + npow2);       // [npow2]
  __shared__ int s_k;
  __shared__ int s_warp[32];

  const double* s = (dir == 0 ? col : slash) + (size_t)hc * nb;
  const double alpha = dir == 0 ? alpha_c : alpha_s;
  for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
    double v = i < nb ? s[i] : 0.0;
    // scores are nonnegative; fold -0.0 onto +0.0 so bit order == value order
    key[i] = v > 0.0 ? (unsigned long long)__double_as_longlong(v) : 0ull;
    idx[i] = i < nb ? i : 0x7fffffff;
    mark[i] = 0;
  }
  __syncthreads();
  // bitonic sort into "before" order (descending score, ascending index)
  for (int size = 2; size <= npow2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < (npow2 >> 1); t += blockDim.x) {
        const int lo = 2 * stride * (t / stride) + (t % stride);
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const unsigned long long ka = key[lo], kb_ = key[hi];
        const int ia = idx[lo], ib = idx[hi];
        const bool swap = up ? before(kb_, ib, ka, ia) : before(ka, ia, kb_, ib);
        if (swap) {
          key[lo] = kb_;
          key[hi] = ka;
          idx[lo] = ib;
          idx[hi] = ia;
        }
      }
      __syncthreads();
    }
  }
  if (eps > 0.0) {
    // guard / certify passes: a parallel prefix sum (contiguous runs per
    // thread, then a block scan of the run totals).  It differs from the
    // sequential sum by ~1e-16 relative, far below the guard's margin E, and
    // these passes keep a decision only when every margin exceeds E, so k and
    // the picks are those of the sequential sum.
    const int T = blockDim.x, per = (nb + T - 1) / T;
    const int a0 = threadIdx.x * per, a1 = min(nb, a0 + per);
    double run = 0.0;
    for (int i = a0; i < a1; ++i) {
      run += __longlong_as_double((long long)key[i]);
      cum[i] = run;
    }
    double incl = run;  // inclusive scan of the run totals: warps, then warp totals
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      const double v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    __shared__ double s_wsum[32];
    if (lane == 31) s_wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      double v = lane < (T >> 5) ? s_wsum[lane] : 0.0;
      for (int o = 1; o < 32; o <<= 1) {
        const double u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      s_wsum[lane] = v;
    }
    __syncthreads();
    const double base = (incl - run) + (wid > 0 ? s_wsum[wid - 1] : 0.0);
    for (int i = a0; i < a1; ++i) cum[i] += base;
  } else if (threadIdx.x == 0) {
    // the selection proper: sequential fp64 cumulative sum in sorted order
    // (np.cumsum semantics), 32 scores loaded ahead per round so only the
    // dependent adds are serial (adding the +0.0 tail leaves the sum bit-identical)
    double acc = 0.0;
    for (int i0 = 0; i0 < nb; i0 += 32) {
      double v[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) v[t] = i0 + t < nb ? __longlong_as_double((long long)key[i0 + t]) : 0.0;
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        acc += v[t];
        if (i0 + t < nb) cum[i0 + t] = acc;
      }
    }
  }
  __syncthreads();
  const double total = cum[nb - 1];
  const double target = alpha * total;
  // k = searchsorted(cum, target, 'left') + 1 = #(cum < target) + 1
  int cnt = 0;
  if (target > 0.0)
    for (int i = threadIdx.x; i < nb; i += blockDim.x) cnt += cum[i] < target ? 1 : 0;
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += s_warp[w];
    int k = target > 0.0 ? tot + 1 : 0;
    if (k_in) k = min(max(k_in[hc * 2 + dir], 0), nb);
    s_k = k;
    k_out[hc * 2 + dir] = k;
    const double scale_b = bound ? fmax(1.0, bound[hc] / bound_ref) : 1.0;
    auto sc = [&](int i) { return __longlong_as_double((long long)key[i]); };
    int* ent = band ? band + ((size_t)hc * 2 + dir) * kBandEntry : nullptr;
    const bool certify = band && only;  // re-select of refined pairs
    const double E = eps * total * scale_b;  // error bound of tensor-core scores (guard)
    if (ent && !certify) ent[0] = 0, ent[2] = ent[3] = -1;
    if (eps > 0.0 && k > 0 && flags && !k_in && !certify) {
      // guard pass: margin widened for large-logit pairs (bound: see k_pair_bound, sa_stage1_tc.cu)
      const double m1 = cum[k - 1] - target, m2 = k >= 2 ? target - cum[k - 2] : INFINITY;
      const bool cut = m1 < E || m2 < E;
      const bool tie = k < nb && sc(k - 1) - sc(k) < E;
      if (cut) {
        atomicOr(flags + hc, 1);
      } else if (tie) {
        // A boundary tie alone leaves only WHICH blocks make the cut in doubt.
        // With every score within E of its exact value, the exact k-th largest
        // score lies within E of hi = s(k-1): blocks above hi + 2E are in,
        // blocks below hi - 2E are out, and the band between (contiguous in
        // sorted order) goes to the refinement; else the pair is re-scored.
        const double hi = sc(k - 1);
        int a = k - 1, z = k - 1;
        while (a > 0 && sc(a - 1) <= hi + 2.0 * E) --a;
        while (z + 1 < nb && sc(z + 1) >= hi - 2.0 * E) ++z;
        if (!ent || z - a + 1 > kBandMax) {
          atomicOr(flags + hc, 1);
        } else {
          ent[0] = z - a + 1;
          ent[1] = a;
          for (int i = a; i <= z; ++i) ent[kBandHdr + i - a] = idx[i];
        }
      }
    } else if (certify && eps > 0.0 && k > 0 && flags && ent) {
      // certify a refined pair: band blocks now carry near-exact scores, the
      // others tensor-core ones (error <= E, which also bounds the prefix
      // sums), so k must clear the alpha cut by E on both sides, and the two
      // blocks at the cut must differ by more than their own error: E unless
      // both are refined; for two refined blocks band_eps * (s_a + s_b)
      // settles it here, and a closer pair is left to k_band_ties' per-row
      // bound (band_eps * sum_r |x_ra - x_rb| <= band_eps * (s_a + s_b))
      const double m1 = cum[k - 1] - target, m2 = k >= 2 ? target - cum[k - 2] : INFINITY;
      bool ok = m1 >= E && m2 >= E;
      ent[2] = ent[3] = -1;
      if (ok && k < nb) {
        const double sa = sc(k - 1), sb = sc(k);
        bool ra = false, rb = false;
        for (int i = 0; i < ent[0]; ++i) {
          ra |= ent[kBandHdr + i] == idx[k - 1];
          rb |= ent[kBandHdr + i] == idx[k];
        }
        if (!(ra && rb)) {
          ok = sa - sb >= E;
        } else if (!(sa - sb > band_eps * scale_b * (sa + sb))) {
          ent[2] = idx[k - 1];
          ent[3] = idx[k];
        }
      }
      if (!ok) atomicOr(flags + hc, 1);
    }
  }
  __syncthreads();
  const int k = s_k;
  for (int i = threadIdx.x; i < k; i += blockDim.x) mark[idx[i]] = 1;
  __syncthreads();
  // ascending compaction of the picked indices: each thread owns a contiguous run
  const int per = (nb + blockDim.x - 1) / blockDim.x;
  const int a0 = threadIdx.x * per, a1 = min(nb, a0 + per);
  int local = 0;
  for (int i = a0; i < a1; ++i) local += mark[i];
  // block exclusive scan of `local`
  int incl = local;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  __syncthreads();
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int v = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      int u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    s_warp[lane] = v;
  }
  __syncthreads();
  int pos = incl - local + (wid > 0 ? s_warp[wid - 1] : 0);
  int* dst = idx_out + ((size_t)hc * 2 + dir) * nb;
  for (int i = a0; i < a1; ++i)
    if (mark[i]) dst[pos++] = i;
}

constexpr int kMergeWarps = 8;

__global__ void __launch_bounds__(kMergeWarps * 32)
    k2_merge(const int* __restrict__ k_sel, const int* __restrict__ idx_sel, int Hq, int cn, int nb,
             int S, int blk, int itv, int sink_blocks, int local_blocks, int* __restrict__ kv_cnt,
             int* __restrict__ kv_idx, long long* __restrict__ active_blocks,
             long long* __restrict__ active_entries) {
  extern __shared__ unsigned int bits_all[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long item = (long long)blockIdx.x * kMergeWarps + wid;
  if (item >= (long long)Hq * nb) return;
  const int h = (int)(item / nb), qb = (int)(item - (long long)h * nb);
  const int nwords = (nb + 31) >> 5;
  unsigned int* bits = bits_all + wid * nwords;
  const int w_used = (qb >> 5) + 1;
  for (int w = lane; w < w_used; w += 32) bits[w] = 0u;
  __syncwarp();
  const int row0 = qb * blk, row1 = min(row0 + blk, S) - 1;
  const int c_first = min(cn - 1, row0 / itv), c_last = min(cn - 1, row1 / itv);
  for (int c = c_first; c <= c_last; ++c) {
    const int hc = h * cn + c;
    const int kc = k_sel[hc * 2], ks = k_sel[hc * 2 + 1];
    const int* ic = idx_sel + ((size_t)hc * 2) * nb;
    const int* is = ic + nb;
    for (int i = lane; i < kc; i += 32) {
      const int kb = ic[i];
      if (kb <= qb) atomicOr(bits + (kb >> 5), 1u << (kb & 31));
    }
    for (int i = lane; i < ks; i += 32) {
      const int ob = is[i];
      const int kb1 = qb - ob - 1, kb2 = qb - ob;
      if (kb1 >= 0) atomicOr(bits + (kb1 >> 5), 1u << (kb1 & 31));
      if (kb2 >= 0) atomicOr(bits + (kb2 >> 5), 1u << (kb2 & 31));
    }
  }
  if (lane == 0) atomicOr(bits + (qb >> 5), 1u << (qb & 31));
  // optional forced sink / local-window blocks (defaults 0 / 1 add nothing)
  for (int kb = lane; kb < min(sink_blocks, qb + 1); kb += 32) atomicOr(bits + (kb >> 5), 1u << (kb & 31));
  for (int kb = max(0, qb - local_blocks + 1) + lane; kb < qb; kb += 32)
    atomicOr(bits + (kb >> 5), 1u << (kb & 31));
  __syncwarp();
  int* dst = kv_idx + (size_t)h * tri(nb) + tri(qb);
  int off = 0;
  for (int w0 = 0; w0 < w_used; w0 += 32) {
    const int w = w0 + lane;
    unsigned int word = w < w_used ? bits[w] : 0u;
    const int pc = __popc(word);
    int incl = pc;
    for (int o = 1; o < 32; o <<= 1) {
      int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    int pos = off + incl - pc;
    while (word) {
      const int b = __ffs(word) - 1;
      dst[pos++] = (w << 5) + b;
      word &= word - 1;
    }
    off += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) {
    kv_cnt[(size_t)h * nb + qb] = off;
    if (active_blocks) atomicAdd(reinterpret_cast<unsigned long long*>(active_blocks + h), (unsigned long long)off);
    if (active_entries) {
      const long long m = min(blk, S - row0);
      const long long e = (long long)(off - 1) * m * blk + m * (m + 1) / 2;
      atomicAdd(reinterpret_cast<unsigned long long*>(active_entries + h), (unsigned long long)e);
    }
  }
}

__global__ void k2_full(int Hq, int nb, int* __restrict__ kv_cnt, int* __restrict__ kv_idx) {
  const long long item = blockIdx.x;
  const int h = (int)(item / nb), qb = (int)(item - (long long)h * nb);
  int* dst = kv_idx + (size_t)h * tri(nb) + tri(qb);
  for (int i = threadIdx.x; i <= qb; i += blockDim.x) dst[i] = i;
  if (threadIdx.x == 0) kv_cnt[item] = qb + 1;
}

// Stage-3 unit pairing by list overlap.  A unit's CTA walks the UNION of its two
// items' key-block lists, and a union step listed by only one item leaves the
// other item's softmax idle and its chain exposed.  The heads of one KV group
// at one query block have different lists (stage 2 selects per head), so which
// heads share a unit matters: one CTA per (query block, local KV group) builds
// the group's key-block bitmaps, the symmetric difference |A xor B| of every
// head pair, and matches the heads greedily (smallest difference first, ties
// by head index).  At C3 this halves the one-item steps (17.6 % -> 8.4 % of the
// union steps) against the fixed (2p, 2p+1) pairing.  An odd group keeps its
// last head for the adjacent-query-block units of unit_items.
constexpr int kPairMaxHeads = 64;

__global__ void __launch_bounds__(256) k2_pair(const int* __restrict__ kv_cnt, const int* __restrict__ kv_idx,
                                               int Hq, int nb, int group, int q_head0, int* __restrict__ pairs) {
  extern __shared__ unsigned bm[];  // [m][W] key-block bitmaps, [np] pair differences, [np] pair table
  const int qb = blockIdx.x, g = blockIdx.y;
  int lo, hi;
  kv_group_heads(g, Hq, group, q_head0, lo, hi);
  const int m = (hi - lo) & ~1;
  if (m < 2) return;
  int base = 0;
  for (int x = 0; x < g; ++x) {
    int l2, h2;
    kv_group_heads(x, Hq, group, q_head0, l2, h2);
    base += units_of_group(h2 - l2, nb);
  }
  const int W = (qb >> 5) + 1;
  const int np = m * (m - 1) / 2;
  unsigned* diff = bm + m * W;
  unsigned* pij = diff + np;  // pair t -> (i << 8) | j, i < j, row-major over the upper triangle
  for (int i = threadIdx.x; i < m * W; i += blockDim.x) bm[i] = 0u;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const int t0 = i * (2 * m - i - 1) / 2;
    for (int j = i + 1; j < m; ++j) pij[t0 + j - i - 1] = (unsigned)((i << 8) | j);
  }
  __syncthreads();
  for (int i = 0; i < m; ++i) {
    const int item = (lo + i) * nb + qb;
    const int n = min(max(__ldg(kv_cnt + item), 0), qb + 1);
    const int* list = kv_idx + (size_t)(lo + i) * tri(nb) + tri(qb);
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
      const int kb = __ldg(list + e);
      if (kb >= 0 && kb <= qb) atomicOr(bm + i * W + (kb >> 5), 1u << (kb & 31));
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int t = warp; t < np; t += nwarps) {
    const int i = pij[t] >> 8, j = pij[t] & 255;
    int c = 0;
    for (int w = lane; w < W; w += 32) c += __popc(bm[i * W + w] ^ bm[j * W + w]);
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) diff[t] = (unsigned)c;
  }
  __syncthreads();
  if (warp != 0) return;
  unsigned long long used = 0ull;
  for (int p = 0; p < m / 2; ++p) {
    // key = difference (<= nb < 2^20), then i, then j: the smallest key wins
    unsigned best = 0xffffffffu;
    for (int t = lane; t < np; t += 32) {
      const int i = pij[t] >> 8, j = pij[t] & 255;
      if (((used >> i) & 1ull) || ((used >> j) & 1ull)) continue;
      best = min(best, (diff[t] << 12) | (unsigned)(i << 6) | (unsigned)j);
    }
    best = __reduce_min_sync(0xffffffffu, best);
    const int i = (best >> 6) & 63, j = best & 63;
    used |= (1ull << i) | (1ull << j);
    if (lane == 0) {
      const size_t u = (size_t)base + (size_t)p * nb + qb;
      pairs[2 * u] = (lo + i) * nb + qb;
      pairs[2 * u + 1] = (lo + j) * nb + qb;
    }
  }
}

// Stage-3 work units (sa_internal.h: two items of one KV head per unit),
// counting-sorted by descending cost kv_cnt[a] + kv_cnt[b], one CTA per local
// KV group.  Group-major keeps one KV head's K/V (64 MiB at 128K) resident in
// L2 while its units run; longest-first inside a group evens out the tail.
// With `pairs` (k2_pair's matching) the paired units take their items from it.
__global__ void __launch_bounds__(1024) k2_units(const int* __restrict__ kv_cnt, int Hq, int nb, int group,
                                                 int q_head0, const int* __restrict__ pairs, int* __restrict__ units) {
  extern __shared__ int hist[];  // [2 * nb + 2]
  int h_lo, h_hi;
  kv_group_heads(blockIdx.x, Hq, group, q_head0, h_lo, h_hi);
  const int nh = h_hi - h_lo;
  if (nh <= 0) return;
  int base = 0;  // units of the groups before this one
  for (int g = 0; g < (int)blockIdx.x; ++g) {
    int lo, hi;
    kv_group_heads(g, Hq, group, q_head0, lo, hi);
    base += units_of_group(hi - lo, nb);
  }
  const int nu = units_of_group(nh, nb);
  const int paired = (nh / 2) * nb;
  const int nbins = 2 * nb + 2;
  for (int i = threadIdx.x; i < nbins; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  auto items = [&](int u, int& a, int& b) {
    if (pairs && u < paired) {
      a = __ldg(pairs + 2 * (base + u));
      b = __ldg(pairs + 2 * (base + u) + 1);
    } else {
      unit_items(u, h_lo, nh, nb, a, b);
    }
  };
  auto cost = [&](int u) {
    int a, b;
    items(u, a, b);
    const int c = max(kv_cnt[a], 0) + (b >= 0 ? max(kv_cnt[b], 0) : 0);
    return min(c, nbins - 1);
  };
  for (int u = threadIdx.x; u < nu; u += blockDim.x) atomicAdd(hist + cost(u), 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = base;  // descending cost
    for (int c = nbins - 1; c >= 0; --c) {
      const int v = hist[c];
      hist[c] = run;
      run += v;
    }
  }
  __syncthreads();
  for (int u = threadIdx.x; u < nu; u += blockDim.x) {
    const int slot = atomicAdd(hist + cost(u), 1);
    int a, b;
    items(u, a, b);
    units[2 * slot] = a;
    units[2 * slot + 1] = b;
  }
}

// NaN/Inf scan, 16-byte vector loads (any non-finite element sets *flag).
__device__ __forceinline__ bool bad_f32(uint32_t w) { return (w & 0x7f800000u) == 0x7f800000u; }
__device__ __forceinline__ bool bad_bf16x2(uint32_t w) {
  return (w & 0x7f80u) == 0x7f80u || (w & 0x7f800000u) == 0x7f800000u;
}
template <bool kBf16>
__global__ void k_check_finite(const uint32_t* __restrict__ x, long long nwords,
                               const unsigned short* __restrict__ tail16, int* flag) {
  const uint4* x4 = reinterpret_cast<const uint4*>(x);
  const long long n4 = nwords >> 2;
  bool bad = false;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const uint4 v = __ldg(x4 + i);
    if (kBf16)
      bad |= bad_bf16x2(v.x) | bad_bf16x2(v.y) | bad_bf16x2(v.z) | bad_bf16x2(v.w);
    else
      bad |= bad_f32(v.x) | bad_f32(v.y) | bad_f32(v.z) | bad_f32(v.w);
  }
  for (long long i = (n4 << 2) + blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += (long long)gridDim.x * blockDim.x)
    bad |= kBf16 ? bad_bf16x2(x[i]) : bad_f32(x[i]);
  if (tail16 && blockIdx.x == 0 && threadIdx.x == 0) bad |= (*tail16 & 0x7f80u) == 0x7f80u;
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *flag = 1;
}

}  // namespace

int launch_select(const double* col, const double* slash, int Hq, int cn, int nb, double ac,
                  double as, double eps, const double* bound, double bound_ref, int* flags, const int* only,
                  const int* k_in, int* k_out, int* idx_out, int* band, double band_eps, cudaStream_t st) {
  int npow2 = 1;
  while (npow2 < nb) npow2 <<= 1;
  const size_t smem = (size_t)npow2 * (8 + 8 + 4 + 1);
  if (smem > 220 * 1024) return fail(SA_ERR_UNSUPPORTED, "sa_select: too many blocks (nb > 8192)");
  cudaFuncSetAttribute(k2_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int threads = npow2 >= 2048 ? 1024 : (npow2 >= 64 ? npow2 / 2 : 32);
  k2_select<<<dim3(2, Hq * cn), threads, smem, st>>>(col, slash, cn, nb, npow2, ac, as, eps, bound, bound_ref, flags,
                                                     only, k_in, k_out, idx_out, band, band_eps);
  return check_launch("sa_select");
}

int launch_merge(const int* k_sel, const int* idx_sel, int Hq, int cn, int nb, int S, int blk,
                 int itv, int sink_blocks, int local_blocks, int* kv_cnt, int* kv_idx,
                 long long* ab, long long* ae, cudaStream_t st) {
  const long long items = (long long)Hq * nb;
  const int nwords = (nb + 31) / 32;
  const size_t smem = (size_t)kMergeWarps * nwords * 4;
  const int grid = (int)((items + kMergeWarps - 1) / kMergeWarps);
  if (ab) cudaMemsetAsync(ab, 0, sizeof(long long) * Hq, st);
  if (ae) cudaMemsetAsync(ae, 0, sizeof(long long) * Hq, st);
  k2_merge<<<grid, kMergeWarps * 32, smem, st>>>(k_sel, idx_sel, Hq, cn, nb, S, blk, itv,
                                                   sink_blocks, local_blocks, kv_cnt, kv_idx, ab, ae);
  return check_launch("sa_merge");
}

int launch_full(int Hq, int nb, int* kv_cnt, int* kv_idx, cudaStream_t st) {
  k2_full<<<Hq * nb, 128, 0, st>>>(Hq, nb, kv_cnt, kv_idx);
  return check_launch("sa_full_mask");
}

int launch_sched(const int* kv_cnt, const int* kv_idx, int Hq, int nb, int group, int q_head0, int* units,
                 int* scratch, cudaStream_t st) {
  const size_t smem = (size_t)(2 * nb + 2) * 4;
  if (smem > 200 * 1024) return fail(SA_ERR_UNSUPPORTED, "sa_schedule: nb too large");
  const int G = n_local_kv(Hq, group, q_head0);
  const int* pairs = nullptr;
  if (kv_idx && scratch) {
    int m = 0;  // largest matched head count of a local group
    for (int g = 0; g < G; ++g) {
      int lo, hi;
      kv_group_heads(g, Hq, group, q_head0, lo, hi);
      m = std::max(m, (hi - lo) & ~1);
    }
    const size_t psmem = ((size_t)m * ((nb + 31) / 32) + (size_t)m * (m - 1)) * 4;
    if (m >= 4 && m <= kPairMaxHeads && psmem <= 200 * 1024) {  // m == 2 has one possible pairing
      set_smem_attr(reinterpret_cast<const void*>(&k2_pair), (int)psmem);
      k2_pair<<<dim3(nb, G), 256, psmem, st>>>(kv_cnt, kv_idx, Hq, nb, group, q_head0, scratch);
      if (int e = check_launch("sa_schedule (pairing)")) return e;
      pairs = scratch;
    }
  }
  set_smem_attr(reinterpret_cast<const void*>(&k2_units), (int)smem);
  k2_units<<<G, 1024, smem, st>>>(kv_cnt, Hq, nb, group, q_head0, pairs, units);
  return check_launch("sa_schedule");
}

int launch_check_finite(const void* x, int dtype, long long n, int* flag, cudaStream_t st) {
  if (n <= 0) return SA_OK;
  const int esize = dtype == SA_FP32 ? 4 : 2;
  const long long bytes = n * esize;
  const long long nwords = bytes / 4;
  const int grid = (int)std::min<long long>(148LL * 16, std::max<long long>(1, (nwords / 4 + 255) / 256));
  // odd bf16 count: the last element sits alone in a half word
  const unsigned short* tail =
      (dtype != SA_FP32 && (n & 1)) ? static_cast<const unsigned short*>(x) + (n - 1) : nullptr;
  if (dtype == SA_FP32)
    k_check_finite<false><<<grid, 256, 0, st>>>(static_cast<const uint32_t*>(x), nwords, nullptr, flag);
  else
    k_check_finite<true><<<grid, 256, 0, st>>>(static_cast<const uint32_t*>(x), nwords, tail, flag);
  return check_launch("sa_check_finite");
}

}  // namespace sa
