// Stage 3, tensor-core mode over SM pairs (cta_group::2): block-sparse causal
// attention prefill on sm_100a (replaces sparse_attention, ref
// pkg/src/blocksift/executor.py:104-158).
//
// Why: with one SM per 128-row tile, QK^T reads Q and K from shared memory for
// every key block (64 KB per 128x128x128 product) on top of the PV read of V
// and the TMA writes of K/V, which puts the tensor core at the 128 B/clk
// shared-memory limit (profiles/r1_summary.md).  Here a CLUSTER of two CTAs on
// two SMs runs one work unit (sa_schedule: two (head, query block) items of
// one KV head, item A on rank 0 and item B on rank 1) with 256-row MMAs:
//   S  = [Q_A; Q_B] K^T   (M = 256, N = 128 keys; each SM holds its own Q and
//                          HALF of the key rows)
//   O += [P_A; P_B] V     (P from each SM's TMEM; each SM holds half of V's
//                          head-dim columns)
// so each SM reads 48 KB + 16 KB of operands per key block instead of 96 KB,
// and loads half of every K/V tile.  Both tiles walk the ascending UNION of
// their two block lists; on a step outside its own list a tile writes P = 0
// for its rows (sa_k3_softmax.cuh, pair mode).  Two clusters share each SM
// pair (256 TMEM columns, 97 KB smem per CTA), so one cluster's softmax
// overlaps the other's MMAs.
//
// Per CTA: warp 0 TMA producer (own Q, own halves of K and V; completion
// bytes are counted on the leader's barriers), warp 1 TMEM owner and, in the
// leader (rank 0) only, the tcgen05 issuer, warps 2-5 softmax + epilogue of
// the CTA's own tile.  TMEM: S [0,128), O [128,256) of the pair allocation.
#include <cuda_bf16.h>

#include <cstdio>

#include "sa_internal.h"
#include "sa_k3_softmax.cuh"
#include "sa_ptx.cuh"

namespace sa {
namespace {

constexpr int kThreads = 192;
constexpr uint32_t kQBytes = 128 * 128 * 2;      // own Q tile (2 boxes of 64 d)
constexpr uint32_t kQBox = kQBytes / 2;
constexpr uint32_t kKHalf = 64 * 128 * 2;        // 64 key rows x 128 d (2 boxes of 64 d)
constexpr uint32_t kKBox = kKHalf / 2;
constexpr uint32_t kVHalf = 128 * 64 * 2;        // 128 key rows x 64 d (1 box)
constexpr uint32_t kIdescQK = idesc_bf16_f32(256, 128, false);
constexpr uint32_t kIdescPV = idesc_bf16_f32(256, 128, true);

struct __align__(8) PairSmem {
  uint64_t q_full, k_full[2], v_full[2];   // leader's copies count both CTAs' bytes
  uint64_t k_empty[2], v_empty[2];         // multicast tcgen05.commit to both CTAs
  uint64_t s_full, p_part, p_full, o_full;
  uint32_t tmem_base;
};

struct PairParams {
  int S, Hq, nb, group, q_head0;
  const int* kv_cnt;
  const int* kv_idx;
  const int* units;
  __nv_bfloat16* out;
  float* lse;
  long long* touched;
};

__device__ __forceinline__ K3Tile item_tile(const PairParams& P, int item) {
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

__device__ __forceinline__ void unit_items_of(const PairParams& P, int u, int& a, int& b) {
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

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 2)
    k3_pair2(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k64,
             const __grid_constant__ CUtensorMap tm_v, const PairParams P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sQ = base;
  unsigned char* sK0 = base + kQBytes;                // stage s at sK0 + s * kKHalf
  unsigned char* sV0 = sK0 + 2 * kKHalf;              // stage s at sV0 + s * kVHalf
  PairSmem* sm = reinterpret_cast<PairSmem*>(sV0 + 2 * kVHalf);
  const int warp = warp_id();
  const uint32_t rank = cluster_rank();
  int ia, ib;
  unit_items_of(P, blockIdx.x >> 1, ia, ib);
  const K3Tile TA = item_tile(P, ia), TB = item_tile(P, ib);
  const K3Tile Tm = rank == 0 ? TA : TB;  // this CTA's tile (n == 0: no item, rows only pad the MMA)
  const K3Tile To = rank == 0 ? TB : TA;  // partner's tile
  const int kvh = TA.kvh;
#ifdef SA_PAIR_DEBUG
  if (threadIdx.x == 0 && blockIdx.x < 64) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    printf("cta %d rank %u smid %u\n", (int)blockIdx.x, rank, smid);
  }
#endif

  if (threadIdx.x == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k64);
    tma_prefetch(&tm_v);
    mbar_init(&sm->q_full, 1);
    for (int x = 0; x < 2; ++x) {
      mbar_init(&sm->k_full[x], 1);
      mbar_init(&sm->v_full[x], 1);
      mbar_init(&sm->k_empty[x], 1);
      mbar_init(&sm->v_empty[x], 1);
    }
    mbar_init(&sm->s_full, 1);
    mbar_init(&sm->p_part, 2);  // one arrival per CTA of the pair
    mbar_init(&sm->p_full, 2);
    mbar_init(&sm->o_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc_pair(&sm->tmem_base, 256);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the partner's barriers are initialised before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem = sm->tmem_base;
  const uint32_t tS = tmem, tO = tmem + 128;

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t keep = policy_evict_last();
      const uint64_t first = policy_evict_first();
      const uint32_t q_full_cl = mapa_shared(smem_u32(&sm->q_full), 0);
      // Q: a CTA without an item loads its partner's rows (finite filler; its P is always 0)
      const K3Tile& Tq = Tm.n > 0 ? Tm : To;
      if (rank == 0) mbar_expect_tx(&sm->q_full, 2 * kQBytes);
      tma_load_3d_pair(sQ, &tm_q, q_full_cl, 0, Tq.qb * 128, Tq.h, first);
      tma_load_3d_pair(sQ + kQBox, &tm_q, q_full_cl, 64, Tq.qb * 128, Tq.h, first);
      int a = 0, b = 0;
      for (int t = 0;; ++t) {
        if (a >= TA.n && b >= TB.n) break;
        const int ka = a < TA.n ? __ldg(TA.list + a) : 0x7fffffff;
        const int kc = b < TB.n ? __ldg(TB.list + b) : 0x7fffffff;
        const int kb = min(ka, kc);
        a += ka == kb;
        b += kc == kb;
        const int s = t & 1;
        unsigned char* sK = sK0 + s * kKHalf;
        unsigned char* sV = sV0 + s * kVHalf;
        if (t >= 2) k3_wait(&sm->k_empty[s], ((t - 2) >> 1) & 1);
        if (rank == 0) mbar_expect_tx(&sm->k_full[s], 2 * kKHalf);
        const uint32_t kf = mapa_shared(smem_u32(&sm->k_full[s]), 0);
        tma_load_3d_pair(sK, &tm_k64, kf, 0, kb * 128 + rank * 64, kvh, keep);
        tma_load_3d_pair(sK + kKBox, &tm_k64, kf, 64, kb * 128 + rank * 64, kvh, keep);
        if (t >= 2) k3_wait(&sm->v_empty[s], ((t - 2) >> 1) & 1);
        if (rank == 0) mbar_expect_tx(&sm->v_full[s], 2 * kVHalf);
        tma_load_3d_pair(sV, &tm_v, mapa_shared(smem_u32(&sm->v_full[s]), 0), rank * 64, kb * 128, kvh, keep);
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      const uint32_t q_addr = smem_u32(sQ), k_addr0 = smem_u32(sK0), v_addr0 = smem_u32(sV0);
      K3Prof pf;
#if SA_K3_PROF
      const long long t_loop = clock64();
#endif
      mbar_wait_cluster(&sm->q_full, 0);
      // O += P(t) V(t): keys 0..95 once that part of P is in both SMs' TMEM, 96..127 after
      auto issue_pv = [&](int t) {
        const int s = t & 1;
        const uint32_t v_addr = v_addr0 + s * kVHalf;
        pf.start();
        mbar_wait_cluster(&sm->p_part, t & 1);
        pf.stop(5);
        pf.start();
        mbar_wait_cluster(&sm->v_full[s], (t >> 1) & 1);
        pf.stop(7);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 6; ++kk)
            umma_ts_pair(tO, tS + kk * 8, sdesc_sw128(v_addr + kk * 2048, kVHalf, 1024), kIdescPV,
                         (t > 0 || kk > 0) ? 1u : 0u);
        }
        __syncwarp();
        pf.start();
        mbar_wait_cluster(&sm->p_full, t & 1);
        pf.stop(6);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 6; kk < 8; ++kk)
            umma_ts_pair(tO, tS + kk * 8, sdesc_sw128(v_addr + kk * 2048, kVHalf, 1024), kIdescPV, 1u);
          umma_commit_pair(&sm->v_empty[s]);
        }
        __syncwarp();
      };
      int a = 0, b = 0;
      int t = 0;
      for (;; ++t) {
        if (a >= TA.n && b >= TB.n) break;
        const int ka = a < TA.n ? __ldg(TA.list + a) : 0x7fffffff;
        const int kc = b < TB.n ? __ldg(TB.list + b) : 0x7fffffff;
        const int kb = min(ka, kc);
        a += ka == kb;
        b += kc == kb;
        const int s = t & 1;
        if (t >= 1) issue_pv(t - 1);  // PV(t-1) reads P from the columns S(t) overwrites: issue it first
        pf.start();
        mbar_wait_cluster(&sm->k_full[s], (t >> 1) & 1);
        pf.stop(8);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t k_addr = k_addr0 + s * kKHalf;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            umma_ss_pair(tS, sdesc_sw128(q_addr + (kk >> 2) * kQBox + (kk & 3) * 32, 16, 1024),
                         sdesc_sw128(k_addr + (kk >> 2) * kKBox + (kk & 3) * 32, 16, 1024), kIdescQK,
                         kk > 0 ? 1u : 0u);
          }
          umma_commit_pair(&sm->s_full);
          umma_commit_pair(&sm->k_empty[s]);
        }
        __syncwarp();
      }
      if (t >= 1) issue_pv(t - 1);
      if (elect_one()) umma_commit_pair(&sm->o_full);
      __syncwarp();
#if SA_K3_PROF
      pf.add(12, clock64() - t_loop);
      pf.add(13, t);
#endif
      pf.flush(lane_id() == 0);
    }
  } else {
    const K3TileBars bars{&sm->s_full, nullptr, &sm->p_part, &sm->p_full, &sm->o_full};
    const K3PairCtx pc{To.list, To.n, mapa_shared(smem_u32(&sm->p_part), 0), mapa_shared(smem_u32(&sm->p_full), 0),
                       rank != 0};
    k3_softmax_tile<true>(Tm, bars, tS, tO, warp & 3, P.S, P.out, P.lse, P.touched, pc);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no remote arrive / multicast commit is still in flight into either CTA
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 256);
  }
}

}  // namespace

int launch_sparse_pair(const void* q, const void* k, const void* v, int S, int Hq, int Hkv, int group,
                       int q_head0, const int* kv_cnt, const int* kv_idx, const int* units, void* out,
                       float* lse, long long* touched, cudaStream_t st) {
  CUtensorMap tq, tk64, tv;
  if (!make_tmap_bf16_hsd(&tq, q, Hq, S, 128, 128) || !make_tmap_bf16_hsd(&tk64, k, Hkv, S, 128, 64) ||
      !make_tmap_bf16_hsd(&tv, v, Hkv, S, 128, 128))
    return fail(SA_ERR_CUDA, "sparse_forward: cuTensorMapEncodeTiled failed");
  PairParams P;
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
#ifndef SA_PAIR_PAD
#define SA_PAIR_PAD 0
#endif
  const size_t smem = kQBytes + 2 * kKHalf + 2 * kVHalf + sizeof(PairSmem) + 1024 + SA_PAIR_PAD;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k3_pair2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  if (touched) cudaMemsetAsync(touched, 0, sizeof(long long) * Hq, st);
  const int nu = n_units(Hq, P.nb, group, q_head0);
  k3_pair2<<<2 * nu, kThreads, smem, st>>>(tq, tk64, tv, P);
  return check_launch("sparse_forward tcgen05 (SM-pair units)");
}

}  // namespace sa

extern "C" int sa_debug_k3p2_profile(unsigned long long* out16, int reset) {
  cudaMemcpyFromSymbol(out16, sa::g_k3s_prof, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(sa::g_k3s_prof, z, sizeof(z));
  }
  return 0;
}
