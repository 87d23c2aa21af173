// Stage 3, tensor-core mode: block-sparse causal attention prefill on sm_100a
// (replaces sparse_attention, ref pkg/src/blocksift/executor.py:104-158).
//
// One CTA = one (q head, 128-row query block) work item, taken in the
// longest-first order produced by sa_schedule.  The item's ascending key-block
// list (the merged column + slash + diagonal mask of stage 2) drives:
//   warp 0   TMA producer: Q once, then K and V tiles of each listed block
//   warp 1   tcgen05 issuer: S = Q K^T into TMEM cols [0,128); after the
//            softmax has overwritten S with bf16 P (cols [0,64)), O += P V
//            with P read straight from TMEM (A-from-TMEM form) and V as an
//            MN-major smem operand; O lives in TMEM cols [128,256)
//   warps 2-5 softmax (one query row per thread = one TMEM lane): causal mask
//            on the diagonal block only, online max with lazy rescaling
//            (O is rescaled in TMEM only when the running max grows by more
//            than 2^8), P = exp2(s*log2e/sqrt(d) - m), running sum; epilogue
//            O / l -> bf16.
// Two CTAs share an SM (256 TMEM columns and ~97 KB smem each), so one CTA's
// softmax overlaps the other's MMAs.  GQA: q head h reads kv head h / group.
#include <cuda_bf16.h>

#include <cstdlib>

#include "sa_internal.h"
#include "sa_ptx.cuh"

namespace sa {
namespace {

constexpr int kThreads = 192;
constexpr uint32_t kTileBytes = 128 * 128 * 2;
constexpr uint32_t kBoxBytes = kTileBytes / 2;
constexpr uint32_t kIdescQK = idesc_bf16_f32(128, 128, false);
constexpr uint32_t kIdescPV = idesc_bf16_f32(128, 128, true);
constexpr float kRescaleThreshold = 8.0f;  // log2 units
#ifndef SA_PACK_P
#define SA_PACK_P pack_bf16
#endif
#ifndef SA_EMU_MASK
#define SA_EMU_MASK 3
#endif

#ifndef SA_K3_PROF
#define SA_K3_PROF 0
#endif
// Optional cycle accounting (build with -DSA_K3_PROF=1; read via
// sa_debug_k3_profile): where the softmax / MMA / TMA roles spend time.
__device__ unsigned long long g_k3_prof[16];
#if SA_K3_PROF
#define PROF_T0() const long long _pt0 = clock64()
#define PROF_ADD(slot) prof[slot] += clock64() - _pt0
#else
#define PROF_T0()
#define PROF_ADD(slot)
#endif

struct __align__(8) K3Smem {
  uint64_t q_full, k_full, k_empty, v_full, v_empty, s_full, p_part, p_full, o_full;
  uint32_t tmem_base;
};

struct K3Params {
  int S, Hq, nb, group, q_head0;
  const int* kv_cnt;
  const int* kv_idx;
  const int* order;
  __nv_bfloat16* out;
  float* lse;
  long long* touched;
};

// kExp: 0 = production; 1/2/3 = timing experiments (skip softmax math / skip
// MMAs / skip both) used only by tools/k3_experiments.py via SA_K3_EXP.
template <int kExp>
__global__ void __launch_bounds__(kThreads, 2)
    k3_tc(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
          const __grid_constant__ CUtensorMap tm_v, const K3Params P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sQ = base;
  unsigned char* sK = base + kTileBytes;
  unsigned char* sV = base + 2 * kTileBytes;
  K3Smem* sm = reinterpret_cast<K3Smem*>(base + 3 * kTileBytes);

  const int item = P.order ? P.order[blockIdx.x] : (int)blockIdx.x;  // flattened unit list
  if (item < 0) return;  // uniform per CTA, before any barrier or TMEM use
  const int h = item / P.nb, qb = item - h * P.nb;
  const int n = P.kv_cnt[item];
  const int* list = P.kv_idx + (size_t)h * tri(P.nb) + tri(qb);
  const int kvh = kv_head_of(h, P.group, P.q_head0);
  const int warp = warp_id();
#if SA_K3_PROF
  long long prof[16] = {0};
  const long long t_start = clock64();
#endif

  if (threadIdx.x == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    mbar_init(&sm->q_full, 1);
    mbar_init(&sm->k_full, 1);
    mbar_init(&sm->k_empty, 1);
    mbar_init(&sm->v_full, 1);
    mbar_init(&sm->v_empty, 1);
    mbar_init(&sm->s_full, 1);
    mbar_init(&sm->p_part, 128);
    mbar_init(&sm->p_full, 128);
    mbar_init(&sm->o_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(&sm->tmem_base, 256);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm->tmem_base;
  const uint32_t tS = tmem, tO = tmem + 128;

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t keep = policy_evict_last();
      mbar_expect_tx(&sm->q_full, kTileBytes);
      tma_load_3d(sQ, &tm_q, &sm->q_full, 0, qb * 128, h);
      tma_load_3d(sQ + kBoxBytes, &tm_q, &sm->q_full, 64, qb * 128, h);
      for (int j = 0; j < n; ++j) {
        const int key0 = __ldg(list + j) * 128;
        if (j >= 1) {
          PROF_T0();
          mbar_wait(&sm->k_empty, (j - 1) & 1);
          PROF_ADD(9);
        }
        mbar_expect_tx(&sm->k_full, kTileBytes);
        tma_load_3d_hint(sK, &tm_k, &sm->k_full, 0, key0, kvh, keep);
        tma_load_3d_hint(sK + kBoxBytes, &tm_k, &sm->k_full, 64, key0, kvh, keep);
        if (j >= 1) {
          PROF_T0();
          mbar_wait(&sm->v_empty, (j - 1) & 1);
          PROF_ADD(10);
        }
        mbar_expect_tx(&sm->v_full, kTileBytes);
        tma_load_3d_hint(sV, &tm_v, &sm->v_full, 0, key0, kvh, keep);
        tma_load_3d_hint(sV + kBoxBytes, &tm_v, &sm->v_full, 64, key0, kvh, keep);
      }
    }
  } else if (warp == 1) {
    const uint32_t q_addr = smem_u32(sQ), k_addr = smem_u32(sK), v_addr = smem_u32(sV);
    mbar_wait(&sm->q_full, 0);
    for (int j = 0; j <= n; ++j) {
      if (j >= 1) {
        // O += P_{j-1} V_{j-1}: the first 3/4 of the keys as soon as the softmax
        // has written that part of P, the last quarter after the rest lands
        {
          PROF_T0();
          mbar_wait(&sm->p_part, (j - 1) & 1);
          PROF_ADD(5);
        }
        {
          PROF_T0();
          mbar_wait(&sm->v_full, (j - 1) & 1);
          PROF_ADD(6);
        }
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 6; ++kk)
            if (kExp < 2) umma_ts(tO, tS + kk * 8, sdesc_sw128(v_addr + kk * 2048, kBoxBytes, 1024), kIdescPV,
                    (j > 1 || kk > 0) ? 1u : 0u);
        }
        __syncwarp();
        {
          PROF_T0();
          mbar_wait(&sm->p_full, (j - 1) & 1);
          PROF_ADD(7);
        }
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 6; kk < 8; ++kk)
            if (kExp < 2) umma_ts(tO, tS + kk * 8, sdesc_sw128(v_addr + kk * 2048, kBoxBytes, 1024), kIdescPV, 1u);
          umma_commit(&sm->v_empty);
          if (j == n) umma_commit(&sm->o_full);
        }
        __syncwarp();
      }
      if (j < n) {
        {
          PROF_T0();
          mbar_wait(&sm->k_full, j & 1);
          PROF_ADD(8);
        }
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * kBoxBytes + (kk & 3) * 32;
            if (kExp < 2) umma_ss(tS, sdesc_sw128(q_addr + off, 16, 1024), sdesc_sw128(k_addr + off, 16, 1024),
                    kIdescQK, kk > 0 ? 1u : 0u);
          }
          umma_commit(&sm->s_full);
          umma_commit(&sm->k_empty);
        }
        __syncwarp();
      }
    }
  } else {
    const int quad = warp & 3;
    const int i = quad * 32 + lane_id();  // query row within the block
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const float sl2 = 1.4426950408889634f * 0.08838834764831845f;  // log2(e) / sqrt(128)
    const uint64_t sl2x2 = f32x2(sl2, sl2);
    float m_ref = -INFINITY;
    uint64_t lacc0 = f32x2(0.f, 0.f), lacc1 = f32x2(0.f, 0.f);  // packed row-sum partials
    for (int j = 0; j < n; ++j) {
      const int kb = __ldg(list + j);
      const bool diag = kb == qb;  // warp-uniform: only the diagonal block needs the causal mask
      {
        PROF_T0();
        mbar_wait(&sm->s_full, j & 1);
        PROF_ADD(0);
      }
#if SA_K3_PROF
      long long _p1 = clock64();
#endif
      tc_fence_after();
      if (kExp == 1 || kExp == 3) {
        tc_fence_before();
        mbar_arrive(&sm->p_part);
        mbar_arrive(&sm->p_full);
        continue;
      }
      // ---- pass 1: row max of the raw scores (FMNMX3, two chains); TMEM loads
      // double-buffered so chunk c+1 is in flight while chunk c is reduced
      float ma = -INFINITY, mb = -INFINITY, mc = -INFINITY, md = -INFINITY;
      {
        uint32_t buf[2][32];
        tmem_ld32(tS + lane_off, buf[0]);
        tmem_ld_wait_regs(buf[0]);
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t(&r)[32] = buf[ch & 1];
          if (ch < 3) tmem_ld32(tS + lane_off + (ch + 1) * 32, buf[(ch + 1) & 1]);
          if (diag) {
#pragma unroll
            for (int t = 0; t < 32; ++t)
              if (ch * 32 + t > i) r[t] = __float_as_uint(-INFINITY);
          }
#pragma unroll
          for (int t = 0; t < 32; t += 8) {  // four independent FMNMX3 chains
            ma = fmax3(ma, __uint_as_float(r[t]), __uint_as_float(r[t + 1]));
            mb = fmax3(mb, __uint_as_float(r[t + 2]), __uint_as_float(r[t + 3]));
            mc = fmax3(mc, __uint_as_float(r[t + 4]), __uint_as_float(r[t + 5]));
            md = fmax3(md, __uint_as_float(r[t + 6]), __uint_as_float(r[t + 7]));
          }
          if (ch < 3) tmem_ld_wait_regs(buf[(ch + 1) & 1]);
        }
      }
#if SA_K3_PROF
      prof[1] += clock64() - _p1;
      _p1 = clock64();
#endif
      const float mxs = fmax3(fmaxf(ma, mb), mc, md) * sl2;
      // tcgen05.ld/st are warp-collective: take the rescale decision per warp
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
            tmem_ld32_sync(tO + lane_off + ch * 32, r);
#pragma unroll
            for (int t = 0; t < 32; t += 2) {
              uint64_t v = fmul2(f32x2(__uint_as_float(r[t]), __uint_as_float(r[t + 1])), f2);
              float a, b;
              unpack_f32x2(v, a, b);
              r[t] = __float_as_uint(a);
              r[t + 1] = __float_as_uint(b);
            }
            tmem_st32(tO + lane_off + ch * 32, r);
          }
        }
        m_ref = m_new;
      }
#if SA_K3_PROF
      prof[2] += clock64() - _p1;
      _p1 = clock64();
#endif
      // ---- pass 2: P = exp2(s * log2e/sqrt(d) - m) -> bf16 into TMEM (aliasing S), row sum.
      // Off the diagonal a quarter of the exponentials run as an FMA-pipe
      // polynomial so the MUFU unit stops pacing the tensor core.
      const uint64_t negm = f32x2(-m_ref, -m_ref);
      {
        uint32_t buf[2][32];
        tmem_ld32(tS + lane_off, buf[0]);
        tmem_ld_wait_regs(buf[0]);
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t(&r)[32] = buf[ch & 1];
          if (ch < 3) tmem_ld32(tS + lane_off + (ch + 1) * 32, buf[(ch + 1) & 1]);
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
              pk[t] = SA_PACK_P(p0, p1);
            }
          } else {
#pragma unroll
            for (int t = 0; t < 16; ++t) {
              float y0, y1;
              unpack_f32x2(ffma2(f32x2(__uint_as_float(r[2 * t]), __uint_as_float(r[2 * t + 1])), sl2x2, negm), y0, y1);
              uint64_t pp;
              if (kExp == 4)
                pp = f32x2(y0, y1);  // timing experiment: no exponentials at all
              else if ((t & 3) >= SA_EMU_MASK)
                pp = ex2_poly2(y0, y1);
              else
                pp = f32x2(ex2(y0), ex2(y1));
              if (t & 1) lacc1 = fadd2(lacc1, pp);
              else lacc0 = fadd2(lacc0, pp);
              float p0, p1;
              unpack_f32x2(pp, p0, p1);
              pk[t] = SA_PACK_P(p0, p1);
            }
          }
          tmem_st16(tS + lane_off + ch * 16, pk);
          if (ch == 2) {  // P columns for keys 0..95 are in TMEM: let the PV MMA start
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&sm->p_part);
          }
          if (ch < 3) tmem_ld_wait_regs(buf[(ch + 1) & 1]);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&sm->p_full);
#if SA_K3_PROF
      prof[3] += clock64() - _p1;
#endif
    }
    float l;
    {
      float a0, a1, b0, b1;
      unpack_f32x2(lacc0, a0, a1);
      unpack_f32x2(lacc1, b0, b1);
      l = (a0 + a1) + (b0 + b1);
    }
    // epilogue: O / l -> bf16
    {
      PROF_T0();
      mbar_wait(&sm->o_full, 0);
      PROF_ADD(4);
    }
    tc_fence_after();
    const int row = qb * 128 + i;
    const bool valid = row < P.S;
    const float inv = 1.f / l;
    __nv_bfloat16* dst = P.out + ((size_t)h * P.S + row) * 128;
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) {
      uint32_t r[32];
      tmem_ld32_sync(tO + lane_off + ch * 32, r);
      uint32_t pk[16];
#pragma unroll
      for (int t = 0; t < 16; ++t)
        pk[t] = pack_bf16(__uint_as_float(r[2 * t]) * inv, __uint_as_float(r[2 * t + 1]) * inv);
      if (valid) {
        uint4* d4 = reinterpret_cast<uint4*>(dst + ch * 32);
#pragma unroll
        for (int t = 0; t < 4; ++t) d4[t] = make_uint4(pk[4 * t], pk[4 * t + 1], pk[4 * t + 2], pk[4 * t + 3]);
      }
    }
    if (valid && P.lse) P.lse[(size_t)h * P.S + row] = (m_ref + __log2f(l)) * 0.6931471805599453f;
    if (threadIdx.x == 64 && P.touched)
      atomicAdd(reinterpret_cast<unsigned long long*>(P.touched + h), (unsigned long long)n);
  }
#if SA_K3_PROF
  if (lane_id() == 0 && warp != 0) {  // softmax warps (slots 0-4), MMA warp (5-8)
    for (int k = 0; k < 9; ++k)
      if (prof[k]) atomicAdd(&g_k3_prof[k], (unsigned long long)prof[k]);
    if (warp == 1) {
      atomicAdd(&g_k3_prof[11], (unsigned long long)(clock64() - t_start));
      atomicAdd(&g_k3_prof[12], (unsigned long long)n);
    }
  }
  if (warp == 0 && lane_id() == 0) {
    atomicAdd(&g_k3_prof[9], (unsigned long long)prof[9]);
    atomicAdd(&g_k3_prof[10], (unsigned long long)prof[10]);
  }
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

}  // namespace

int launch_sparse_tc(const void* q, const void* k, const void* v, int S, int Hq, int Hkv, int group,
                     int q_head0, const int* kv_cnt, const int* kv_idx, const int* order, int n_order, void* out,
                     float* lse, long long* touched, cudaStream_t st) {
  CUtensorMap tq, tk, tv;
  if (!make_tmap_bf16_hsd(&tq, q, Hq, S, 128) || !make_tmap_bf16_hsd(&tk, k, Hkv, S, 128) ||
      !make_tmap_bf16_hsd(&tv, v, Hkv, S, 128))
    return fail(SA_ERR_CUDA, "sparse_forward: cuTensorMapEncodeTiled failed");
  K3Params P;
  P.S = S;
  P.Hq = Hq;
  P.nb = ceil_div(S, 128);
  P.group = group;
  P.q_head0 = q_head0;
  P.kv_cnt = kv_cnt;
  P.kv_idx = kv_idx;
  P.order = order;
  P.out = static_cast<__nv_bfloat16*>(out);
  P.lse = lse;
  P.touched = touched;
  const size_t smem = 3 * kTileBytes + sizeof(K3Smem) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k3_tc<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k3_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k3_tc<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k3_tc<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k3_tc<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  static const int exp_mode = [] {
    const char* e = getenv("SA_K3_EXP");
    return e ? atoi(e) : 0;
  }();
  if (touched) cudaMemsetAsync(touched, 0, sizeof(long long) * Hq, st);
  const int grid = order ? n_order : Hq * P.nb;
  switch (exp_mode) {
    case 1: k3_tc<1><<<grid, kThreads, smem, st>>>(tq, tk, tv, P); break;
    case 2: k3_tc<2><<<grid, kThreads, smem, st>>>(tq, tk, tv, P); break;
    case 3: k3_tc<3><<<grid, kThreads, smem, st>>>(tq, tk, tv, P); break;
    case 4: k3_tc<4><<<grid, kThreads, smem, st>>>(tq, tk, tv, P); break;
    default: k3_tc<0><<<grid, kThreads, smem, st>>>(tq, tk, tv, P); break;
  }
  return check_launch("sparse_forward tcgen05");
}

}  // namespace sa

extern "C" int sa_debug_k3_profile(unsigned long long* out16, int reset) {
  cudaMemcpyFromSymbol(out16, sa::g_k3_prof, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(sa::g_k3_prof, z, sizeof(z));
  }
  return 0;
}
