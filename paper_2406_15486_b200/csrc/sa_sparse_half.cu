// Stage 3, tensor-core mode, K/V-sharing work units with HALF-BLOCK S
// buffers (experiment, SA_K3_IMPL=half): block-sparse causal attention
// prefill on sm_100a (replaces sparse_attention, ref
// pkg/src/blocksift/executor.py:104-158).
//
// Why: in k3_share, P aliases the item's single 128-column S buffer, so an
// item's next QK^T cannot start before its PV has read P: every item runs a
// serial S -> softmax -> PV -> S chain, and the delay experiments put that
// chain, not the tensor pipe, on the critical path.  Here
// each item owns TWO 64-column S buffers (keys 0..63 and 64..127 of a key
// block) plus its 128-column O: 2 x (64 + 64 + 128) = 512 TMEM columns for the
// unit's two items.  QK^T runs as two N=64 MMAs; while the softmax works on
// one half, the other half's S and the other item's MMAs run, and a half's
// PV is issued one union step later, right before its buffer is reused.
//
//   warp 0      TMA producer (as in k3_share: union of the two lists, 2-stage K/V ring)
//   warp 1      tcgen05 issuer; per union step t and half h:
//                 for each item: [PV(previous block, h) if pending], [S(t, h) if listed]
//   warps 4-7 / 8-11  softmax + epilogue of A / B: per key block, half 0 then
//               half 1 (64 keys per thread), single-read fast path against the
//               running max; the rare rescale waits for the item's previous PV
//               (pv_done) because, unlike k3_share, it may still be in flight.
#include <cuda_bf16.h>

#include <climits>

#include "sa_internal.h"
#include "sa_k3_softmax.cuh"
#include "sa_ptx.cuh"

namespace sa {
namespace {

constexpr int kWarps = 12;
constexpr int kThreads = kWarps * 32;
constexpr uint32_t kTileBytes = 128 * 128 * 2;
constexpr uint32_t kBoxBytes = kTileBytes / 2;
constexpr uint32_t kIdescQK = idesc_bf16_f32(128, 64, false);  // S half: 128 rows x 64 keys
constexpr uint32_t kIdescPV = idesc_bf16_f32(128, 128, true);

struct __align__(8) HalfSmem {
  uint64_t q_full[2], k_full[2], k_empty[2], v_full[2], v_empty[2];
  uint64_t s_full[2][2], p_full[2][2];  // [item][half]
  uint64_t pv_done[2], o_full[2];       // [item]
  uint32_t tmem_base;
};

struct HalfParams {
  int S, Hq, nb, group, q_head0;
  const int* kv_cnt;
  const int* kv_idx;
  const int* units;
  __nv_bfloat16* out;
  float* lse;
  long long* touched;
};

__device__ __forceinline__ K3Tile half_tile(const HalfParams& P, int item) {
  K3Tile t;
  if (item < 0) {
    t.n = 0;
    t.h = t.qb = t.kvh = 0;
    t.list = nullptr;
    return t;
  }
  t.h = item / P.nb;
  t.qb = item - t.h * P.nb;
  t.n = __ldg(P.kv_cnt + item);
  t.list = P.kv_idx + (size_t)t.h * tri(P.nb) + tri(t.qb);
  t.kvh = kv_head_of(t.h, P.group, P.q_head0);
  return t;
}

__device__ __forceinline__ void half_unit(const HalfParams& P, int u, int& a, int& b) {
  if (P.units) {
    a = __ldg(P.units + 2 * u);
    b = __ldg(P.units + 2 * u + 1);
    return;
  }
  for (int g = 0, G = n_local_kv(P.Hq, P.group, P.q_head0); g < G; ++g) {
    int lo, hi;
    kv_group_heads(g, P.Hq, P.group, P.q_head0, lo, hi);
    const int n = units_of_group(hi - lo, P.nb);
    if (u < n) {
      unit_items(u, lo, hi - lo, P.nb, a, b);
      return;
    }
    u -= n;
  }
  a = b = -1;
}

struct Walk2 {
  const int* la;
  const int* lb;
  int na, nb, ia, ib;
  __device__ __forceinline__ bool next(int& kb, bool& inA, bool& inB) {
    if (ia >= na && ib >= nb) return false;
    const int ka = ia < na ? __ldg(la + ia) : INT_MAX;
    const int kc = ib < nb ? __ldg(lb + ib) : INT_MAX;
    kb = min(ka, kc);
    inA = ka == kb;
    inB = kc == kb;
    ia += inA;
    ib += inB;
    return true;
  }
};

// Softmax of one item over its blocks, half-block granularity.
__device__ __forceinline__ void softmax_halves(const K3Tile& T, HalfSmem* sm, int x, uint32_t tSb0, uint32_t tO0,
                                               int quad, const HalfParams& P) {
  const int i = quad * 32 + lane_id();
  const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
  const uint32_t tO = tO0 + lane_off;
  const float sl2 = 1.4426950408889634f * 0.08838834764831845f;  // log2(e) / sqrt(128)
  const uint64_t sl2x2 = f32x2(sl2, sl2);
  float m_ref = -INFINITY;
  uint64_t lacc0 = f32x2(0.f, 0.f), lacc1 = f32x2(0.f, 0.f);
  for (int j = 0; j < T.n; ++j) {
    const int kb = __ldg(T.list + j);
    const bool diag = kb == T.qb;
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      const int u = 2 * j + h;
      const uint32_t tS = tSb0 + h * 64 + lane_off;
      const int c0 = h * 64;  // key offset of this half inside the block
      k3_wait(&sm->s_full[x][h], j & 1);
      tc_fence_after();
      uint32_t pk[32];
      bool ok = false;
      if (u > 0 && !diag) {  // fast path: exponentials against the running max
        const uint64_t negm = f32x2(-m_ref, -m_ref);
        uint64_t bacc0 = f32x2(0.f, 0.f), bacc1 = f32x2(0.f, 0.f);
        float ymax = -INFINITY;
        uint32_t buf[2][32];
        tmem_ld32(tS, buf[0]);
        tmem_ld32(tS + 32, buf[1]);
        tmem_ld_wait_regs(buf[0]);
        tmem_ld_wait_regs(buf[1]);
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            float y0, y1;
            unpack_f32x2(ffma2(f32x2(__uint_as_float(buf[ch][2 * t]), __uint_as_float(buf[ch][2 * t + 1])), sl2x2,
                               negm),
                         y0, y1);
            ymax = fmax3(ymax, y0, y1);
            const uint64_t pp = ((t & 3) >= 4 - SA_K3_POLY) ? ex2_poly2(y0, y1) : f32x2(ex2(y0), ex2(y1));
            if (t & 1)
              bacc1 = fadd2(bacc1, pp);
            else
              bacc0 = fadd2(bacc0, pp);
            float p0, p1;
            unpack_f32x2(pp, p0, p1);
            pk[ch * 16 + t] = pack_bf16(p0, p1);
          }
        }
        if (!__any_sync(0xffffffffu, ymax > kK3RescaleThreshold)) {
          ok = true;
          lacc0 = fadd2(lacc0, bacc0);
          lacc1 = fadd2(lacc1, bacc1);
        }
      }
      if (!ok) {
        float ma = -INFINITY, mb = -INFINITY;
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          uint32_t r[32];
          tmem_ld32_sync(tS + ch * 32, r);
          if (diag) {
#pragma unroll
            for (int t = 0; t < 32; ++t)
              if (c0 + ch * 32 + t > i) r[t] = __float_as_uint(-INFINITY);
          }
#pragma unroll
          for (int t = 0; t < 32; t += 4) {
            ma = fmax3(ma, __uint_as_float(r[t]), __uint_as_float(r[t + 1]));
            mb = fmax3(mb, __uint_as_float(r[t + 2]), __uint_as_float(r[t + 3]));
          }
        }
        const float mxs = fmaxf(ma, mb) * sl2;
        if (__any_sync(0xffffffffu, mxs > m_ref + kK3RescaleThreshold)) {
          const float m_new = fmaxf(m_ref, mxs);
          if (u > 0) {
            // every earlier PV of this item must have landed in O before O is rescaled
            k3_wait(&sm->pv_done[x], (u - 1) & 1);
            tc_fence_after();
            const float f = ex2(m_ref - m_new);
            const uint64_t f2 = f32x2(f, f);
            lacc0 = fmul2(lacc0, f2);
            lacc1 = fmul2(lacc1, f2);
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
              uint32_t o[32];
              tmem_ld32_sync(tO + ch * 32, o);
#pragma unroll
              for (int t = 0; t < 32; t += 2) {
                float a, c;
                unpack_f32x2(fmul2(f32x2(__uint_as_float(o[t]), __uint_as_float(o[t + 1])), f2), a, c);
                o[t] = __float_as_uint(a);
                o[t + 1] = __float_as_uint(c);
              }
              tmem_st32(tO + ch * 32, o);
            }
            tmem_st_wait();
          }
          m_ref = m_new;
        }
        const uint64_t negm = f32x2(-m_ref, -m_ref);
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          uint32_t r[32];
          tmem_ld32_sync(tS + ch * 32, r);
          if (diag) {
#pragma unroll
            for (int t = 0; t < 32; ++t)
              if (c0 + ch * 32 + t > i) r[t] = __float_as_uint(-INFINITY);
          }
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            float y0, y1;
            unpack_f32x2(ffma2(f32x2(__uint_as_float(r[2 * t]), __uint_as_float(r[2 * t + 1])), sl2x2, negm), y0, y1);
            const float p0 = ex2(y0), p1 = ex2(y1);
            if (t & 1)
              lacc1 = fadd2(lacc1, f32x2(p0, p1));
            else
              lacc0 = fadd2(lacc0, f32x2(p0, p1));
            pk[ch * 16 + t] = pack_bf16(p0, p1);
          }
        }
      }
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        uint32_t(&q)[16] = *reinterpret_cast<uint32_t(*)[16]>(&pk[ch * 16]);
        tmem_st16(tS + ch * 16, q);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&sm->p_full[x][h]);
    }
  }
  // ---- epilogue
  float l;
  {
    float a0, a1, b0, b1;
    unpack_f32x2(lacc0, a0, a1);
    unpack_f32x2(lacc1, b0, b1);
    l = (a0 + a1) + (b0 + b1);
  }
  k3_wait(&sm->o_full[x], 0);
  tc_fence_after();
  const int row = T.qb * 128 + i;
  const bool valid = row < P.S;
  const float inv = 1.f / l;
  __nv_bfloat16* dst = P.out + ((size_t)T.h * P.S + row) * 128;
  const uint64_t stream_out = policy_evict_first();
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) {
    uint32_t r[32];
    tmem_ld32_sync(tO + ch * 32, r);
    uint32_t o[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) o[t] = pack_bf16(__uint_as_float(r[2 * t]) * inv, __uint_as_float(r[2 * t + 1]) * inv);
    if (valid) {
      uint4* d4 = reinterpret_cast<uint4*>(dst + ch * 32);
#pragma unroll
      for (int t = 0; t < 4; ++t)
        st_global_v4_hint(d4 + t, make_uint4(o[4 * t], o[4 * t + 1], o[4 * t + 2], o[4 * t + 3]), stream_out);
    }
  }
  if (valid && P.lse) P.lse[(size_t)T.h * P.S + row] = (m_ref + __log2f(l)) * 0.6931471805599453f;
  if (i == 0 && P.touched) atomicAdd(reinterpret_cast<unsigned long long*>(P.touched + T.h), (unsigned long long)T.n);
}

__global__ void __launch_bounds__(kThreads, 1)
    k3_half(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
            const __grid_constant__ CUtensorMap tm_v, const HalfParams P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sQ[2] = {base, base + kTileBytes};
  unsigned char* const sK0 = base + 2 * kTileBytes;
  unsigned char* const sV0 = base + 4 * kTileBytes;
  HalfSmem* sm = reinterpret_cast<HalfSmem*>(base + 6 * kTileBytes);
  const int warp = warp_id();
  int ia, ib;
  half_unit(P, blockIdx.x, ia, ib);
  const K3Tile T[2] = {half_tile(P, ia), half_tile(P, ib)};

  if (threadIdx.x == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    for (int x = 0; x < 2; ++x) {
      mbar_init(&sm->q_full[x], 1);
      mbar_init(&sm->k_full[x], 1);
      mbar_init(&sm->k_empty[x], 1);
      mbar_init(&sm->v_full[x], 1);
      mbar_init(&sm->v_empty[x], 1);
      for (int h = 0; h < 2; ++h) {
        mbar_init(&sm->s_full[x][h], 1);
        mbar_init(&sm->p_full[x][h], 128);
      }
      mbar_init(&sm->pv_done[x], 1);
      mbar_init(&sm->o_full[x], 1);
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
  // item x: S half buffers at cols [256x, 256x+64) and [256x+64, 256x+128), O at [256x+128, 256x+256)
  const int kvh = T[0].n > 0 ? T[0].kvh : T[1].kvh;

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t keep = policy_evict_last(), once = policy_evict_first();
      for (int x = 0; x < 2; ++x)
        if (T[x].n > 0) {
          mbar_expect_tx(&sm->q_full[x], kTileBytes);
          tma_load_3d_hint(sQ[x], &tm_q, &sm->q_full[x], 0, T[x].qb * 128, T[x].h, once);
          tma_load_3d_hint(sQ[x] + kBoxBytes, &tm_q, &sm->q_full[x], 64, T[x].qb * 128, T[x].h, once);
        }
      Walk2 w{T[0].list, T[1].list, T[0].n, T[1].n, 0, 0};
      int kb;
      bool inA, inB;
      for (int t = 0; w.next(kb, inA, inB); ++t) {
        const int s = t & 1;
        const int key0 = kb * 128;
        if (t >= 2) k3_wait(&sm->k_empty[s], ((t - 2) >> 1) & 1);
        mbar_expect_tx(&sm->k_full[s], kTileBytes);
        unsigned char* sK = sK0 + s * kTileBytes;
        tma_load_3d_hint(sK, &tm_k, &sm->k_full[s], 0, key0, kvh, keep);
        tma_load_3d_hint(sK + kBoxBytes, &tm_k, &sm->k_full[s], 64, key0, kvh, keep);
        if (t >= 2) k3_wait(&sm->v_empty[s], ((t - 2) >> 1) & 1);
        mbar_expect_tx(&sm->v_full[s], kTileBytes);
        unsigned char* sV = sV0 + s * kTileBytes;
        tma_load_3d_hint(sV, &tm_v, &sm->v_full[s], 0, key0, kvh, keep);
        tma_load_3d_hint(sV + kBoxBytes, &tm_v, &sm->v_full[s], 64, key0, kvh, keep);
      }
    }
  } else if (warp == 1) {
    const uint64_t q_desc[2] = {sdesc_sw128(smem_u32(sQ[0]), 16, 1024), sdesc_sw128(smem_u32(sQ[1]), 16, 1024)};
    const uint64_t k_desc0 = sdesc_sw128(smem_u32(sK0), 16, 1024);
    const uint64_t v_desc0 = sdesc_sw128(smem_u32(sV0), kBoxBytes, 1024);
    int n_s[2] = {0, 0};                 // blocks whose S halves were issued, per item
    int n_pv[2] = {0, 0};                // PVs issued per item (half granularity)
    int pend[2][2] = {{-1, -1}, {-1, -1}};  // union step whose PV(half h) is still to be issued
    Walk2 w{T[0].list, T[1].list, T[0].n, T[1].n, 0, 0};
    int kb;
    bool in[2];
    int t = 0;
    auto issue_pv = [&](int x, int h, int step) {
      const int s = step & 1;
      const int jb = n_pv[x] >> 1;  // block index of this PV within the item
      k3_wait(&sm->p_full[x][h], jb & 1);
      k3_wait(&sm->v_full[s], (step >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t tSb = tmem + x * 256 + h * 64, tO = tmem + x * 256 + 128;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_ts(tO, tSb + kk * 8, v_desc0 + ((s * kTileBytes + (4 * h + kk) * 2048) >> 4), kIdescPV,
                  (n_pv[x] > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&sm->pv_done[x]);
        if (n_pv[x] == 2 * T[x].n - 1) umma_commit(&sm->o_full[x]);
      }
      __syncwarp();
      ++n_pv[x];
    };
    while (w.next(kb, in[0], in[1])) {
      const int s = t & 1;
      k3_wait(&sm->k_full[s], (t >> 1) & 1);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          if (pend[x][h] >= 0) {
            issue_pv(x, h, pend[x][h]);
            pend[x][h] = -1;
          }
          if (in[x]) {
            if (n_s[x] == 0 && h == 0) k3_wait(&sm->q_full[x], 0);
            tc_fence_after();
            if (elect_one()) {
              const uint32_t tSb = tmem + x * 256 + h * 64;
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) {
                const uint32_t qoff = (kk >> 2) * kBoxBytes + (kk & 3) * 32;
                const uint32_t koff = s * kTileBytes + (kk >> 2) * kBoxBytes + h * 8192 + (kk & 3) * 32;
                umma_ss(tSb, q_desc[x] + (qoff >> 4), k_desc0 + (koff >> 4), kIdescQK, kk > 0 ? 1u : 0u);
              }
              umma_commit(&sm->s_full[x][h]);
            }
            __syncwarp();
            pend[x][h] = t;
          }
        }
      }
#pragma unroll
      for (int x = 0; x < 2; ++x) n_s[x] += in[x];
      if (elect_one()) {
        umma_commit(&sm->k_empty[s]);
        if (t >= 1) umma_commit(&sm->v_empty[s ^ 1]);  // every PV of step t-1 is issued by now
      }
      __syncwarp();
      ++t;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int x = 0; x < 2; ++x)
        if (pend[x][h] >= 0) issue_pv(x, h, pend[x][h]);
  } else if (warp >= 4) {
    const int x = warp < 8 ? 0 : 1;
    const K3Tile Tx = x ? T[1] : T[0];
    if (Tx.n > 0) softmax_halves(Tx, sm, x, tmem + x * 256, tmem + x * 256 + 128, warp & 3, P);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace

int launch_sparse_half(const void* q, const void* k, const void* v, int S, int Hq, int Hkv, int group, int q_head0,
                       const int* kv_cnt, const int* kv_idx, const int* units, void* out, float* lse,
                       long long* touched, cudaStream_t st) {
  CUtensorMap tq, tk, tv;
  if (!make_tmap_bf16_hsd(&tq, q, Hq, S, 128) || !make_tmap_bf16_hsd(&tk, k, Hkv, S, 128) ||
      !make_tmap_bf16_hsd(&tv, v, Hkv, S, 128))
    return fail(SA_ERR_CUDA, "sparse_forward: cuTensorMapEncodeTiled failed");
  HalfParams P;
  P.S = S;
  P.Hq = Hq;
  P.nb = ceil_div(S, 128);
  P.group = group;
  P.q_head0 = q_head0;
  P.kv_cnt = kv_cnt;
  P.kv_idx = kv_idx;
  P.units = units;
  P.out = static_cast<__nv_bfloat16*>(out);
  P.lse = lse;
  P.touched = touched;
  const size_t smem = 6 * (size_t)kTileBytes + sizeof(HalfSmem) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k3_half, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  if (touched) cudaMemsetAsync(touched, 0, sizeof(long long) * Hq, st);
  k3_half<<<n_units(Hq, P.nb, group, q_head0), kThreads, smem, st>>>(tq, tk, tv, P);
  return check_launch("sparse_forward tcgen05 (half-block S buffers)");
}

}  // namespace sa
