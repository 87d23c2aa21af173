// Stage 3, tensor-core mode, paired tiles: block-sparse causal attention
// prefill on sm_100a (replaces sparse_attention, ref
// pkg/src/blocksift/executor.py:104-158).
//
// One CTA (one per SM: 512 TMEM columns, 192 KB smem) runs TWO work items,
// A and B, adjacent in the longest-first order of sa_schedule (so their block
// counts are close).  Each tile keeps its own Q, K and V smem tiles, its own
// S/P (128 cols) and O (128 cols) TMEM accumulators and its own mbarriers;
// what the pairing buys is ONE tcgen05 issuer that alternates the tiles,
//     [PV_A(i-1), S_A(i)], [PV_B(i-1), S_B(i)], [PV_A(i), S_A(i+1)], ...
// so the softmax of A runs while the tensor core works on B and vice versa,
// and the two softmax warpgroups never compete for the MUFU unit (the exp
// pipe, which an unpaired CTA pair on one SM shares half of the time).
//   warp 0 / warp 2   TMA producers for A / B (Q once, then K, V per block)
//   warp 1            MMA issuer (and TMEM owner)
//   warps 4-7 / 8-11  softmax + epilogue of A / B, one query row per thread
// The softmax math is that of sa_sparse_tc.cu: diagonal-only causal mask,
// FMNMX3 row max, lazy O rescale (2^8), FFMA2/FADD2 packed math, a quarter of
// the off-diagonal exponentials as an FMA-pipe polynomial, bf16 P written
// over S in TMEM and consumed by the PV MMA straight from TMEM; the first 3/4
// of PV is issued as soon as that part of P has landed.
#include <cuda_bf16.h>

#include "sa_internal.h"
#include "sa_ptx.cuh"

namespace sa {
namespace {

constexpr int kWarps = 12;  // WG0: 0 TMA-A, 1 MMA, 2 TMA-B, 3 idle; WG1 (4-7) softmax A; WG2 (8-11) softmax B
constexpr int kThreads = kWarps * 32;
constexpr uint32_t kTileBytes = 128 * 128 * 2;
constexpr uint32_t kBoxBytes = kTileBytes / 2;
constexpr uint32_t kIdescQK = idesc_bf16_f32(128, 128, false);
constexpr uint32_t kIdescPV = idesc_bf16_f32(128, 128, true);
constexpr float kRescaleThreshold = 8.0f;  // log2 units

#ifndef SA_K3_PROF
#define SA_K3_PROF 0
#endif
__device__ unsigned long long g_k3p_prof[16];
#if SA_K3_PROF
#define PT0() const long long _pt0 = clock64()
#define PADD(slot) (lp[slot] += clock64() - _pt0)
#define PFLUSH() for (int _k = 0; _k < 8; ++_k) if (lp[_k]) atomicAdd(&g_k3p_prof[_k], (unsigned long long)lp[_k])
#else
#define PT0()
#define PADD(slot)
#define PFLUSH()
#endif

struct __align__(8) TileBars {
  uint64_t q_full, k_full, k_empty, v_full, v_empty, s_full, p_part, p_full, o_full;
};
struct __align__(8) PairSmem {
  TileBars bar[2];
  uint32_t tmem_base;
};

struct PairParams {
  int S, nb, group, q_head0, n_items;
  const int* kv_cnt;
  const int* kv_idx;
  const int* order;
  __nv_bfloat16* out;
  float* lse;
  long long* touched;
};

struct Tile {
  int n, h, qb, kvh;
  const int* list;
};

__device__ __forceinline__ Tile tile_of(const PairParams& P, int slot) {
  Tile t;
  const int pos = 2 * (int)blockIdx.x + slot;
  if (pos >= P.n_items) {
    t.n = 0;
    t.h = t.qb = t.kvh = 0;
    t.list = nullptr;
    return t;
  }
  const int item = P.order ? __ldg(P.order + pos) : pos;
  t.h = item / P.nb;
  t.qb = item - t.h * P.nb;
  t.n = __ldg(P.kv_cnt + item);
  t.list = P.kv_idx + (size_t)t.h * tri(P.nb) + tri(t.qb);
  t.kvh = kv_head_of(t.h, P.group, P.q_head0);
  return t;
}

// ---------------------------------------------------------------- roles
__device__ void produce(const Tile& T, TileBars& b, unsigned char* sQ, unsigned char* sK, unsigned char* sV,
                        const CUtensorMap* tq, const CUtensorMap* tk, const CUtensorMap* tv) {
  const uint64_t keep = policy_evict_last();
  mbar_expect_tx(&b.q_full, kTileBytes);
  tma_load_3d(sQ, tq, &b.q_full, 0, T.qb * 128, T.h);
  tma_load_3d(sQ + kBoxBytes, tq, &b.q_full, 64, T.qb * 128, T.h);
  for (int j = 0; j < T.n; ++j) {
    const int key0 = __ldg(T.list + j) * 128;
    if (j >= 1) mbar_wait(&b.k_empty, (j - 1) & 1);
    mbar_expect_tx(&b.k_full, kTileBytes);
    tma_load_3d_hint(sK, tk, &b.k_full, 0, key0, T.kvh, keep);
    tma_load_3d_hint(sK + kBoxBytes, tk, &b.k_full, 64, key0, T.kvh, keep);
    if (j >= 1) mbar_wait(&b.v_empty, (j - 1) & 1);
    mbar_expect_tx(&b.v_full, kTileBytes);
    tma_load_3d_hint(sV, tv, &b.v_full, 0, key0, T.kvh, keep);
    tma_load_3d_hint(sV + kBoxBytes, tv, &b.v_full, 64, key0, T.kvh, keep);
  }
}

// S_X(j) = Q_X K_X(j)^T into TMEM tS
__device__ __forceinline__ void issue_s(TileBars& b, int j, uint32_t tS, uint32_t q_addr, uint32_t k_addr,
                                        long long* lp) {
  {
    PT0();
    mbar_wait(&b.k_full, j & 1);
    PADD(6);
  }
  tc_fence_after();
  if (elect_one()) {
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const uint32_t off = (kk >> 2) * kBoxBytes + (kk & 3) * 32;
      umma_ss(tS, sdesc_sw128(q_addr + off, 16, 1024), sdesc_sw128(k_addr + off, 16, 1024), kIdescQK,
              kk > 0 ? 1u : 0u);
    }
    umma_commit(&b.s_full);
    umma_commit(&b.k_empty);
  }
  __syncwarp();
}

// O_X += P_X(j) V_X(j): K-steps 0..5 (keys 0..95) once that part of P is in
// TMEM, K-steps 6, 7 after the rest lands
__device__ __forceinline__ void issue_pv(TileBars& b, int j, bool last, uint32_t tS, uint32_t tO,
                                         uint32_t v_addr, long long* lp) {
  {
    PT0();
    mbar_wait(&b.p_part, j & 1);
    PADD(3);
  }
  {
    PT0();
    mbar_wait(&b.v_full, j & 1);
    PADD(4);
  }
  tc_fence_after();
  if (elect_one()) {
#pragma unroll
    for (int kk = 0; kk < 6; ++kk)
      umma_ts(tO, tS + kk * 8, sdesc_sw128(v_addr + kk * 2048, kBoxBytes, 1024), kIdescPV,
              (j > 0 || kk > 0) ? 1u : 0u);
  }
  __syncwarp();
  {
    PT0();
    mbar_wait(&b.p_full, j & 1);
    PADD(5);
  }
  tc_fence_after();
  if (elect_one()) {
#pragma unroll
    for (int kk = 6; kk < 8; ++kk)
      umma_ts(tO, tS + kk * 8, sdesc_sw128(v_addr + kk * 2048, kBoxBytes, 1024), kIdescPV, 1u);
    umma_commit(&b.v_empty);
    if (last) umma_commit(&b.o_full);
  }
  __syncwarp();
}

// Softmax of one tile: one query row per thread (= TMEM lane); S is read
// from TMEM twice (row max, then exponentials) with the loads double-buffered.
__device__ void softmax_tile(const PairParams& P, const Tile& T, TileBars& b, uint32_t tS0, uint32_t tO0,
                             int quad) {
  const int i = quad * 32 + lane_id();  // query row within the tile
  const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
  const uint32_t tS = tS0 + lane_off, tO = tO0 + lane_off;
  const float sl2 = 1.4426950408889634f * 0.08838834764831845f;  // log2(e) / sqrt(128)
  const uint64_t sl2x2 = f32x2(sl2, sl2);
  float m_ref = -INFINITY;
  uint64_t lacc0 = f32x2(0.f, 0.f), lacc1 = f32x2(0.f, 0.f);
#if SA_K3_PROF
  long long lp[8] = {0};
#endif
  for (int j = 0; j < T.n; ++j) {
    const int kb = __ldg(T.list + j);
    const bool diag = kb == T.qb;  // warp-uniform: only the diagonal block needs the causal mask
    {
      PT0();
      mbar_wait(&b.s_full, j & 1);
      PADD(0);
    }
#if SA_K3_PROF
    long long _p1 = clock64();
#endif
    tc_fence_after();
    // ---- pass 1: row max (four FMNMX3 chains)
    float ma = -INFINITY, mb = -INFINITY, mc = -INFINITY, md = -INFINITY;
    {
      uint32_t buf[2][32];
      tmem_ld32(tS, buf[0]);
      tmem_ld_wait_regs(buf[0]);
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        uint32_t(&r)[32] = buf[ch & 1];
        if (ch < 3) tmem_ld32(tS + (ch + 1) * 32, buf[(ch + 1) & 1]);
        if (diag) {
#pragma unroll
          for (int t = 0; t < 32; ++t)
            if (ch * 32 + t > i) r[t] = __float_as_uint(-INFINITY);
        }
#pragma unroll
        for (int t = 0; t < 32; t += 8) {
          ma = fmax3(ma, __uint_as_float(r[t]), __uint_as_float(r[t + 1]));
          mb = fmax3(mb, __uint_as_float(r[t + 2]), __uint_as_float(r[t + 3]));
          mc = fmax3(mc, __uint_as_float(r[t + 4]), __uint_as_float(r[t + 5]));
          md = fmax3(md, __uint_as_float(r[t + 6]), __uint_as_float(r[t + 7]));
        }
        if (ch < 3) tmem_ld_wait_regs(buf[(ch + 1) & 1]);
      }
    }
    const float mxs = fmax3(fmaxf(ma, mb), mc, md) * sl2;
#if SA_K3_PROF
    lp[1] += clock64() - _p1;
    _p1 = clock64();
#endif
    // tcgen05.ld/st are warp-collective: rescale decision per warp; O is
    // stable here (PV(j-1) completed before S(j) did, in-order tensor pipe)
    if (__any_sync(0xffffffffu, mxs > m_ref + kRescaleThreshold)) {
      const float m_new = fmaxf(m_ref, mxs);
      if (j > 0) {
        const float f = ex2(m_ref - m_new);
        const uint64_t f2 = f32x2(f, f);
        lacc0 = fmul2(lacc0, f2);
        lacc1 = fmul2(lacc1, f2);
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t r[32];
          tmem_ld32_sync(tO + ch * 32, r);
#pragma unroll
          for (int t = 0; t < 32; t += 2) {
            uint64_t v = fmul2(f32x2(__uint_as_float(r[t]), __uint_as_float(r[t + 1])), f2);
            float a, c;
            unpack_f32x2(v, a, c);
            r[t] = __float_as_uint(a);
            r[t + 1] = __float_as_uint(c);
          }
          tmem_st32(tO + ch * 32, r);
        }
      }
      m_ref = m_new;
    }
    // ---- pass 2: P = exp2(s*log2e/sqrt(d) - m) -> bf16 over S (cols [0,64)), row sum
    const uint64_t negm = f32x2(-m_ref, -m_ref);
    {
      uint32_t buf[2][32];
      tmem_ld32(tS, buf[0]);
      tmem_ld_wait_regs(buf[0]);
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        uint32_t(&r)[32] = buf[ch & 1];
        if (ch < 3) tmem_ld32(tS + (ch + 1) * 32, buf[(ch + 1) & 1]);
        uint32_t pk[16];
        if (diag) {
#pragma unroll
          for (int t = 0; t < 32; ++t)
            if (ch * 32 + t > i) r[t] = __float_as_uint(-INFINITY);
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            float y0, y1;
            unpack_f32x2(ffma2(f32x2(__uint_as_float(r[2 * t]), __uint_as_float(r[2 * t + 1])), sl2x2, negm), y0, y1);
            const float p0 = ex2(y0), p1 = ex2(y1);
            if (t & 1) lacc1 = fadd2(lacc1, f32x2(p0, p1));
            else lacc0 = fadd2(lacc0, f32x2(p0, p1));
            pk[t] = pack_bf16(p0, p1);
          }
        } else {
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            float y0, y1;
            unpack_f32x2(ffma2(f32x2(__uint_as_float(r[2 * t]), __uint_as_float(r[2 * t + 1])), sl2x2, negm), y0, y1);
            const uint64_t pp = ((t & 3) == 3) ? ex2_poly2(y0, y1) : f32x2(ex2(y0), ex2(y1));
            if (t & 1) lacc1 = fadd2(lacc1, pp);
            else lacc0 = fadd2(lacc0, pp);
            float p0, p1;
            unpack_f32x2(pp, p0, p1);
            pk[t] = pack_bf16(p0, p1);
          }
        }
        tmem_st16(tS + ch * 16, pk);
        if (ch == 2) {  // keys 0..95 of P are in TMEM: let the PV MMA start
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&b.p_part);
        }
        if (ch < 3) tmem_ld_wait_regs(buf[(ch + 1) & 1]);
      }
    }
    tmem_st_wait();
    tc_fence_before();
    mbar_arrive(&b.p_full);
#if SA_K3_PROF
    lp[2] += clock64() - _p1;
#endif
  }
#if SA_K3_PROF
  if (lane_id() == 0) PFLUSH();
#endif
  // ---- epilogue: O / l -> bf16
  float l;
  {
    float a0, a1, b0, b1;
    unpack_f32x2(lacc0, a0, a1);
    unpack_f32x2(lacc1, b0, b1);
    l = (a0 + a1) + (b0 + b1);
  }
  mbar_wait(&b.o_full, 0);
  tc_fence_after();
  const int row = T.qb * 128 + i;
  const bool valid = row < P.S;
  const float inv = 1.f / l;
  __nv_bfloat16* dst = P.out + ((size_t)T.h * P.S + row) * 128;
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) {
    uint32_t r[32];
    tmem_ld32_sync(tO + ch * 32, r);
    uint32_t pk[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) pk[t] = pack_bf16(__uint_as_float(r[2 * t]) * inv, __uint_as_float(r[2 * t + 1]) * inv);
    if (valid) {
      uint4* d4 = reinterpret_cast<uint4*>(dst + ch * 32);
#pragma unroll
      for (int t = 0; t < 4; ++t) d4[t] = make_uint4(pk[4 * t], pk[4 * t + 1], pk[4 * t + 2], pk[4 * t + 3]);
    }
  }
  if (valid && P.lse) P.lse[(size_t)T.h * P.S + row] = (m_ref + __log2f(l)) * 0.6931471805599453f;
  if (i == 0 && P.touched) atomicAdd(reinterpret_cast<unsigned long long*>(P.touched + T.h), (unsigned long long)T.n);
}

__global__ void __launch_bounds__(kThreads, 1)
    k3_pair(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
            const __grid_constant__ CUtensorMap tm_v, const PairParams P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // per tile: Q, K, V (32 KB each)
  unsigned char* sQ[2] = {base, base + 3 * kTileBytes};
  unsigned char* sK[2] = {base + kTileBytes, base + 4 * kTileBytes};
  unsigned char* sV[2] = {base + 2 * kTileBytes, base + 5 * kTileBytes};
  PairSmem* sm = reinterpret_cast<PairSmem*>(base + 6 * kTileBytes);
  const int warp = warp_id();
  const Tile T[2] = {tile_of(P, 0), tile_of(P, 1)};

  if (threadIdx.x == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    for (int x = 0; x < 2; ++x) {
      TileBars& b = sm->bar[x];
      mbar_init(&b.q_full, 1);
      mbar_init(&b.k_full, 1);
      mbar_init(&b.k_empty, 1);
      mbar_init(&b.v_full, 1);
      mbar_init(&b.v_empty, 1);
      mbar_init(&b.s_full, 1);
      mbar_init(&b.p_part, 128);
      mbar_init(&b.p_full, 128);
      mbar_init(&b.o_full, 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(&sm->tmem_base, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm->tmem_base;
  const uint32_t tS[2] = {tmem, tmem + 256};
  const uint32_t tO[2] = {tmem + 128, tmem + 384};

  if (warp < 4) {
    if (warp == 0 || warp == 2) {
      const int x = warp == 0 ? 0 : 1;
      if (T[x].n > 0 && elect_one()) produce(T[x], sm->bar[x], sQ[x], sK[x], sV[x], &tm_q, &tm_k, &tm_v);
    } else if (warp == 1) {
      long long lp[8] = {0};
      (void)lp;
      // ping-pong issue order across the two tiles
      uint32_t q_addr[2], k_addr[2], v_addr[2];
      for (int x = 0; x < 2; ++x) {
        q_addr[x] = smem_u32(sQ[x]);
        k_addr[x] = smem_u32(sK[x]);
        v_addr[x] = smem_u32(sV[x]);
      }
      for (int x = 0; x < 2; ++x)
        if (T[x].n > 0) {
          mbar_wait(&sm->bar[x].q_full, 0);
          issue_s(sm->bar[x], 0, tS[x], q_addr[x], k_addr[x], lp);
        }
      const int nmax = max(T[0].n, T[1].n);
      for (int j = 1; j <= nmax; ++j) {
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          if (j > T[x].n) continue;
          issue_pv(sm->bar[x], j - 1, j == T[x].n, tS[x], tO[x], v_addr[x], lp);
          if (j < T[x].n) issue_s(sm->bar[x], j, tS[x], q_addr[x], k_addr[x], lp);
        }
      }
      if (lane_id() == 0) PFLUSH();
    }
  } else {
    const int x = warp < 8 ? 0 : 1;
    if (T[x].n > 0) softmax_tile(P, T[x], sm->bar[x], tS[x], tO[x], warp & 3);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
#if SA_K3_PROF
    if (lane_id() == 0) {
      atomicAdd(&g_k3p_prof[12], (unsigned long long)(T[0].n + T[1].n));
    }
#endif
  }
}

}  // namespace

int launch_sparse_tc_pair(const void* q, const void* k, const void* v, int S, int Hq, int Hkv, int group,
                          int q_head0, const int* kv_cnt, const int* kv_idx, const int* order, void* out,
                          float* lse, long long* touched, cudaStream_t st) {
  CUtensorMap tq, tk, tv;
  if (!make_tmap_bf16_hsd(&tq, q, Hq, S, 128) || !make_tmap_bf16_hsd(&tk, k, Hkv, S, 128) ||
      !make_tmap_bf16_hsd(&tv, v, Hkv, S, 128))
    return fail(SA_ERR_CUDA, "sparse_forward: cuTensorMapEncodeTiled failed");
  PairParams P;
  P.S = S;
  P.nb = ceil_div(S, 128);
  P.group = group;
  P.q_head0 = q_head0;
  P.n_items = Hq * P.nb;
  P.kv_cnt = kv_cnt;
  P.kv_idx = kv_idx;
  P.order = order;
  P.out = static_cast<__nv_bfloat16*>(out);
  P.lse = lse;
  P.touched = touched;
  const size_t smem = 6 * (size_t)kTileBytes + sizeof(PairSmem) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k3_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  if (touched) cudaMemsetAsync(touched, 0, sizeof(long long) * Hq, st);
  k3_pair<<<ceil_div(P.n_items, 2), kThreads, smem, st>>>(tq, tk, tv, P);
  return check_launch("sparse_forward tcgen05 (paired)");
}

}  // namespace sa

extern "C" int sa_debug_k3p_profile(unsigned long long* out16, int reset) {
  cudaMemcpyFromSymbol(out16, sa::g_k3p_prof, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(sa::g_k3p_prof, z, sizeof(z));
  }
  return 0;
}
