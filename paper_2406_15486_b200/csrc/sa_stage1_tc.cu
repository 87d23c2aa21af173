// Stage 1, tensor-core mode: fused sampled-query attention + column / slash
// block reduction on sm_100a (replaces sample_scores + block_reduce,
// ref pkg/src/blocksift/sampler.py:135-191; math of core.py:110-154).
//
// One CTA = (q head h, chunk c, key-block split).  The chunk's 128 sampled
// query rows (a possibly UNALIGNED window, sampler.py:103-117) are TMA-loaded
// once; key tiles stream through TMA; S = Q K^T is computed by tcgen05.mma into
// a TMEM accumulator (128 columns); three CTAs share an SM, so one CTA's MMA
// and loads overlap the others' softmax.  Four softmax warps own
// one sampled row each per thread (TMEM lane == row) and, per key block, emit
// the row's running log2-max m and the two partial masses
//     A = sum_{t <= r%128} exp2(s - m),   B = sum_{t > r%128} exp2(s - m)
// (keys j = kb*128 + t, causal j <= r).  A lands in slash bin r//128 - kb and
// B in r//128 - kb - 1, both in column bin kb.  The score matrix never leaves
// TMEM/registers; the per-(row, block) partials (12 B per 128 keys) are the
// only HBM traffic, and two tiny deterministic kernels normalise them with
// the rows' global max / sum and fold the 128 rows into part3 (col + 3 slash
// bins per key block), finished by the shared s1_finalize.
#include <cuda_bf16.h>

#include "sa_internal.h"
#include "sa_ptx.cuh"

namespace sa {
namespace {

constexpr int kThreads = 192;  // warp 0 TMA, warp 1 MMA + TMEM owner, warps 2-5 softmax
// 3 CTAs per SM, each with a single K stage and a single TMEM S (smem 64 KB,
// 128 TMEM columns): the other CTAs' work fills the gaps of a CTA's
// load -> QK^T -> softmax chain (C3 stage-1 kernel -4 %, C4 -1.5 % against 2
// CTAs with a 2-stage ring and a double-buffered S, profiles/r2/k1_ctas_ab.txt)
constexpr int kCtasPerSm = 3;
constexpr int kStages = 1;  // K ring depth
constexpr int kSBuf = 1;    // TMEM S buffers
constexpr uint32_t kTileBytes = 128 * 128 * 2;  // one 128 x 128 bf16 tile (two 64-col boxes)
constexpr uint32_t kBoxBytes = kTileBytes / 2;
constexpr uint32_t kIdescQK = idesc_bf16_f32(128, 128, false);

struct __align__(8) K1Smem {
  uint64_t q_full;
  uint64_t k_full[kStages];
  uint64_t k_empty[kStages];
  uint64_t s_full[2];
  uint64_t s_empty[2];
  uint32_t tmem_base;
};

struct K1Params {
  Stage1Geom g;
  const int* only;
  int kb_per_cta;
  float* pa;  // [Hq*cn][128][nb]
  float* pb;
  float* pm;
};

__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    k1_tc(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
          const K1Params P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment for the 128B-swizzled tiles
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sQ = base;                 // 32 KB
  unsigned char* sK = base + kTileBytes;    // kStages x 32 KB
  K1Smem* sm = reinterpret_cast<K1Smem*>(base + kTileBytes * (1 + kStages));

  const Stage1Geom& g = P.g;
  const int hc = blockIdx.y;
  if (P.only && P.only[hc] == 0) return;
  const int h = hc / g.cn, c = hc - h * g.cn;
  int se, ss;
  if (g.S < 128) {
    ss = 0;
    se = g.S;
  } else {
    se = (c + 1) * g.itv;
    ss = se - 128;
  }
  const int nkb = (se + 127) / 128;
  const int kb0 = blockIdx.x * P.kb_per_cta;
  if (kb0 >= nkb) return;
  const int n = min(P.kb_per_cta, nkb - kb0);
  const int kvh = kv_head_of(h, g.group, g.q_head0);
  const int warp = warp_id();

  if (threadIdx.x == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    mbar_init(&sm->q_full, 1);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&sm->k_full[i], 1);
      mbar_init(&sm->k_empty[i], 1);
    }
    for (int i = 0; i < kSBuf; ++i) {
      mbar_init(&sm->s_full[i], 1);
      mbar_init(&sm->s_empty[i], 128);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(&sm->tmem_base, 128 * kSBuf);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm->tmem_base;

  if (warp == 0) {
    if (elect_one()) {
      mbar_expect_tx(&sm->q_full, kTileBytes);
      tma_load_3d(sQ, &tm_q, &sm->q_full, 0, ss, h);
      tma_load_3d(sQ + kBoxBytes, &tm_q, &sm->q_full, 64, ss, h);
      for (int j = 0; j < n; ++j) {
        const int st = j % kStages;
        if (j >= kStages) mbar_wait(&sm->k_empty[st], ((j / kStages) - 1) & 1);
        unsigned char* dst = sK + st * kTileBytes;
        const int key0 = (kb0 + j) * 128;
        mbar_expect_tx(&sm->k_full[st], kTileBytes);
        tma_load_3d(dst, &tm_k, &sm->k_full[st], 0, key0, kvh);
        tma_load_3d(dst + kBoxBytes, &tm_k, &sm->k_full[st], 64, key0, kvh);
      }
    }
  } else if (warp == 1) {
    mbar_wait(&sm->q_full, 0);
    const uint32_t q_addr = smem_u32(sQ);
    for (int j = 0; j < n; ++j) {
      const int st = j % kStages, buf = j % kSBuf;
      mbar_wait(&sm->k_full[st], (j / kStages) & 1);
      if (j >= kSBuf) mbar_wait(&sm->s_empty[buf], ((j / kSBuf) - 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t k_addr = smem_u32(sK + st * kTileBytes);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * kBoxBytes + (kk & 3) * 32;
          umma_ss(tmem + buf * 128, sdesc_sw128(q_addr + off, 16, 1024),
                  sdesc_sw128(k_addr + off, 16, 1024), kIdescQK, kk > 0 ? 1u : 0u);
        }
        umma_commit(&sm->s_full[buf]);
        umma_commit(&sm->k_empty[st]);
      }
      __syncwarp();
    }
  } else {
    // softmax warps: TMEM lane quadrant = warp % 4
    const int quad = warp & 3;
    const int rl = quad * 32 + lane_id();       // row within the window
    const int row = ss + rl;                    // global query position
    const bool valid = row < se;
    const int rho = row & 127;
    const float sl2 = 1.4426950408889634f / sqrtf((float)g.d);
    float m_run = -INFINITY;
    const size_t prow = ((size_t)hc * 128 + rl) * g.nb;
    for (int j = 0; j < n; ++j) {
      const int buf = j % kSBuf;
      const int kb = kb0 + j;
      mbar_wait(&sm->s_full[buf], (j / kSBuf) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + buf * 128;
      const int lim = row - kb * 128;  // keys t <= lim are causal
      // every key of the block is causal for every row of the window: no per-element mask (warp-uniform)
      const bool full = kb * 128 + 127 < ss;
      float mx = -INFINITY;
      uint32_t rb[2][32];  // TMEM loads double-buffered: chunk ch+1 in flight while ch is reduced
      tmem_ld32(taddr, rb[0]);
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        uint32_t(&r)[32] = rb[ch & 1];
        tmem_ld_wait_regs(r);
        if (ch < 3) tmem_ld32(taddr + (ch + 1) * 32, rb[(ch + 1) & 1]);
        if (full) {
          float mb = -INFINITY;
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            mx = fmax3(mx, __uint_as_float(r[i]), __uint_as_float(r[i + 1]));
            mb = fmax3(mb, __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]));
          }
          mx = fmaxf(mx, mb);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float x = __uint_as_float(r[i]);
            if (ch * 32 + i <= lim) mx = fmaxf(mx, x);
          }
        }
      }
      const float m_new = fmaxf(m_run, mx * sl2);
      // four independent add chains per sum (t & 3), so the adds do not serialise on their latency
      float ac[4] = {0.f, 0.f, 0.f, 0.f}, bc[4] = {0.f, 0.f, 0.f, 0.f};
      // warp-collective TMEM loads stay outside any per-row condition
      const int lim_e = m_new == -INFINITY ? -1 : lim;
      tmem_ld32(taddr, rb[0]);
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        uint32_t(&r)[32] = rb[ch & 1];
        tmem_ld_wait_regs(r);
        if (ch < 3) tmem_ld32(taddr + (ch + 1) * 32, rb[(ch + 1) & 1]);
        if (ch == 2) {
          // chunk 3 is waited for here too, so every S value of this block is in
          // registers and the next QK^T may overwrite S before the last 64
          // exponentials (stage 1 -3..5 %, profiles/r2/s3/k1er_*.txt, k1r2_*.txt)
          tmem_ld_wait_regs(rb[1]);
          tc_fence_before();
          mbar_arrive(&sm->s_empty[buf]);
        }
        if (full) {  // same values (FFMA2 = two fused FMAs) as the masked loop
          const uint64_t negm = f32x2(-m_new, -m_new), sl2x2 = f32x2(sl2, sl2);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            float y0, y1;
            unpack_f32x2(ffma2(f32x2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), sl2x2, negm), y0, y1);
            const float p0 = ex2(y0), p1 = ex2(y1);
            if (ch * 32 + i <= rho) ac[i & 3] += p0; else bc[i & 3] += p0;
            if (ch * 32 + i + 1 <= rho) ac[(i + 1) & 3] += p1; else bc[(i + 1) & 3] += p1;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int t = ch * 32 + i;
            const float p = t <= lim_e ? ex2(fmaf(__uint_as_float(r[i]), sl2, -m_new)) : 0.f;
            if (t <= rho) ac[i & 3] += p; else bc[i & 3] += p;
          }
        }
      }
      const float a = (ac[0] + ac[1]) + (ac[2] + ac[3]);
      const float b = (bc[0] + bc[1]) + (bc[2] + bc[3]);
      if (valid) {
        P.pa[prow + kb] = a;
        P.pb[prow + kb] = b;
        P.pm[prow + kb] = m_new;
      }
      m_run = m_new;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 128 * kSBuf);
  }
}

// ---- selection-guard logit bound.  The tensor-core scores carry the fp32
// accumulation error of q.k, which grows with sum_i |q_i k_i| <= ||q|| ||k||;
// the guard margin of a (head, chunk) is scaled by
//   bound = max_{sampled rows r} ||q_r|| * max_{keys j} ||k_j|| / sqrt(d)
// (Cauchy-Schwarz), so large-logit heads get a proportionally wider margin.
// Max ||k_j||^2 per KV head: 16 threads per key row (one 16-byte load each),
// four rows in flight per half-warp so the loads overlap (nonnegative floats
// order like their bit patterns, so atomicMax on the bits is a float max).
__global__ void k_key_norm(const __nv_bfloat16* __restrict__ k, int S, unsigned* __restrict__ kmax2) {
  const int kvh = blockIdx.y;
  const int sub = threadIdx.x & 15;  // 16-byte slice of the row
  const int half = (threadIdx.x >> 4) & 1;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // global warp: 8 rows per round
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const uint4* base = reinterpret_cast<const uint4*>(k + (size_t)kvh * S * 128);
  float best = 0.f;
  for (int w0 = gw * 8; w0 < S; w0 += nw * 8) {  // warp-uniform trip count (the shuffles below)
    const int j0 = w0 + half * 4;
    uint4 u[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) u[r] = j0 + r < S ? __ldg(base + (size_t)(j0 + r) * 16 + sub) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t w[4] = {u[r].x, u[r].y, u[r].z, u[r].w};
      float ss = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
        ss = fmaf(f.x, f.x, fmaf(f.y, f.y, ss));
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      best = fmaxf(best, ss);
    }
  }
  for (int o = 16; o > 0; o >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, o));
  __shared__ float s_best[32];
  if ((threadIdx.x & 31) == 0) s_best[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best = fmaxf(best, s_best[w]);
    atomicMax(kmax2 + kvh, __float_as_uint(best));
  }
}

// One CTA per (head, chunk); thread r = sampled row r of the window.
__global__ void k_pair_bound(const __nv_bfloat16* __restrict__ q, Stage1Geom g, const unsigned* __restrict__ kmax2,
                             double* __restrict__ bound) {
  const int hc = blockIdx.x, h = hc / g.cn, c = hc - h * g.cn;
  const int se = min(g.S, (c + 1) * g.itv), ss = max(0, se - g.blk);
  float qq = 0.f;
  for (int r = ss + (int)threadIdx.x; r < se; r += blockDim.x) {
    const uint4* row = reinterpret_cast<const uint4*>(q + ((size_t)h * g.S + r) * 128);
    float acc = 0.f;
#pragma unroll 4
    for (int t = 0; t < 16; ++t) {
      const uint4 u = __ldg(row + t);
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
        acc = fmaf(f.x, f.x, fmaf(f.y, f.y, acc));
      }
    }
    qq = fmaxf(qq, acc);
  }
  for (int o = 16; o > 0; o >>= 1) qq = fmaxf(qq, __shfl_xor_sync(0xffffffffu, qq, o));
  __shared__ float s_q[32];
  if ((threadIdx.x & 31) == 0) s_q[threadIdx.x >> 5] = qq;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) qq = fmaxf(qq, s_q[w]);
    const float kk = __uint_as_float(kmax2[kv_head_of(h, g.group, g.q_head0)]);
    bound[hc] = sqrt((double)qq * (double)kk) / sqrt((double)g.d);
  }
}

}  // namespace

int launch_logit_bound(const Stage1Geom& g, const void* q, const void* k, char* ws, const Workspace& L,
                       double* bound, cudaStream_t st) {
  unsigned* kmax2 = reinterpret_cast<unsigned*>(ws + L.kmax2);
  cudaMemsetAsync(kmax2, 0, sizeof(unsigned) * g.Hkv, st);
  const int per_kv = std::max(1, std::min(ceil_div(g.S, 64), 4 * 148 / std::max(1, g.Hkv) + 1));
  k_key_norm<<<dim3(per_kv, g.Hkv), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(k), g.S, kmax2);
  if (int e = check_launch("stage1 key norms")) return e;
  k_pair_bound<<<g.Hq * g.cn, 128, 0, st>>>(static_cast<const __nv_bfloat16*>(q), g, kmax2, bound);
  return check_launch("stage1 logit bound");
}

int launch_stage1_tc(const Stage1Geom& g, const void* q, const void* k, const int* only, char* ws,
                     const Workspace& L, double* col, double* slash, cudaStream_t st) {
  CUtensorMap tq, tk;
  if (!make_tmap_bf16_hsd(&tq, q, g.Hq, g.S, 128) || !make_tmap_bf16_hsd(&tk, k, g.Hkv, g.S, 128))
    return fail(SA_ERR_CUDA, "stage1: cuTensorMapEncodeTiled failed");
  const size_t plane = (size_t)g.Hq * g.cn * 128 * g.nb;
  K1Params P;
  P.g = g;
  P.only = only;
  P.pa = reinterpret_cast<float*>(ws + L.tc_part);
  P.pb = P.pa + plane;
  P.pm = P.pb + plane;
  // split the key range so the grid covers the SMs a few times over
  const long long total_kb = (long long)g.Hq * g.cn * g.nb;
  int kpc = (int)std::max<long long>(4, std::min<long long>(64, total_kb / (148LL * kCtasPerSm * 4)));
  P.kb_per_cta = kpc;
  const int nsplit = ceil_div(g.nb, kpc);
  const size_t smem = kTileBytes * (1 + kStages) + sizeof(K1Smem) + 1024;
  set_smem_attr(reinterpret_cast<const void*>(&k1_tc), (int)smem);
  k1_tc<<<dim3(nsplit, g.Hq * g.cn), kThreads, smem, st>>>(tq, tk, P);
  if (int e = check_launch("stage1 tcgen05")) return e;
  return launch_fold<float, true>(g, only, P.pa, P.pb, P.pm, ws, L, col, slash, st);
}

}  // namespace sa
