// Stage 3, tensor-core mode, K/V-sharing work units: block-sparse causal
// attention prefill on sm_100a (replaces sparse_attention, ref
// pkg/src/blocksift/executor.py:104-158).
//
// Why: with one (head, query block) per CTA every kept block pair pulls its own
// 64 KB of K+V through L2, and at C3 that is ~350 GB per launch: the kernel sits
// on the L2->SM throughput cap (profiles/r1_summary.md).  Here one CTA (one per
// SM, 512 TMEM columns) runs a work UNIT of two items A, B that read the same
// KV head (two q heads of a GQA group at one query block, or adjacent query
// blocks of one head; sa_schedule builds the units).  The producer walks the
// ascending UNION of the two key-block lists and loads each K/V tile once; each
// item runs its MMAs only on the blocks of its own list.  On the bench masks the
// union is 55 % of the summed lists (profiles/r1/overlap_stats.jsonl).
//
//   warp 0      TMA producer: Q_A, Q_B once, then K and V of each union step
//               into a 2-stage ring (K and V released separately)
//   warp 1      tcgen05 issuer (TMEM owner); per union step t:
//                 [PV_A(prev), S_A(t) if A lists t], [PV_B(prev), S_B(t) if B lists t]
//               so A's softmax overlaps B's MMAs and vice versa; a pending PV
//               is issued at the next step even when its item skips that step,
//               so a V stage is never held past the following step
//   warps 4-7   softmax + epilogue of A, warps 8-11 of B (sa_k3_softmax.cuh)
// TMEM: S_A [0,128), O_A [128,256), S_B [256,384), O_B [384,512).
#include <cuda_bf16.h>

#include <climits>

#include "sa_internal.h"
#include "sa_k3_softmax.cuh"
#include "sa_ptx.cuh"

namespace sa {
namespace {

// warp 0 TMA, warp 1 MMA, warps 2-3 idle (so each softmax warpgroup starts at
// TMEM lane quadrant 0), then the softmax warps: 4-7 for A and 8-11 for B.
constexpr int kWarps = 12;

constexpr int kThreads = kWarps * 32;
constexpr uint32_t kTileBytes = 128 * 128 * 2;
constexpr uint32_t kBoxBytes = kTileBytes / 2;
constexpr uint32_t kIdescQK = idesc_bf16_f32(128, 128, false);
constexpr uint32_t kIdescPV = idesc_bf16_f32(128, 128, true);

// K / V ring depths (K and V tiles are released separately).  A third K or V
// stage (224 KB of smem) measured the same at C3, C3 dense and C2
// (profiles/r2/s3/k3_ring_*.txt): the issuer waits ~45 / ~75 cycles per
// item-block on K / V, the loads are not what holds the MMAs back.
constexpr int kKSt = 2, kVSt = 2;
static_assert((2 + kKSt + kVSt) * 32768 + 1024 + 256 <= 232448, "K3 smem over the 227 KB opt-in limit");

struct __align__(8) ShareSmem {
  uint64_t q_full[2], k_full[kKSt], k_empty[kKSt], v_full[kVSt], v_empty[kVSt];
  uint64_t s_full[2], p_part[2], p_full[2], o_full[2];  // p_part/p_full = P of keys 0..63 / all keys
  uint64_t pv_half[2];                                    // PV over keys 0..63 of the current block done
  uint32_t tmem_base;
};

struct ShareParams {
  int S, Hq, nb, group, q_head0;
  const int* kv_cnt;
  const int* kv_idx;
  const int* units;  // [n_units][2] items, or null for the natural unit order
  __nv_bfloat16* out;
  K3PeerOut peers;  // gather fused into the epilogue (sa_sparse_forward_peers)
  float* lse;
  long long* touched;
  unsigned* status;
};

__device__ __forceinline__ K3Tile tile_of_item(const ShareParams& P, int item) {
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

__device__ __forceinline__ void unit_of(const ShareParams& P, int u, int& a, int& b) {
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

// Ascending merge of the two key-block lists (each ascending, no repeats).
struct UnionWalk {
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

__global__ void __launch_bounds__(kThreads, 1)
    k3_share(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
             const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ ShareParams P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sQ[2] = {base, base + kTileBytes};
  unsigned char* const sK0 = base + 2 * kTileBytes;           // K stage s at sK0 + s * kTileBytes
  unsigned char* const sV0 = base + (2 + kKSt) * kTileBytes;  // V stage s at sV0 + s * kTileBytes
  ShareSmem* sm = reinterpret_cast<ShareSmem*>(base + (2 + kKSt + kVSt) * kTileBytes);
  const int warp = warp_id();
  int ia, ib;
  unit_of(P, blockIdx.x, ia, ib);
  const K3Tile T[2] = {tile_of_item(P, ia), tile_of_item(P, ib)};

  if (threadIdx.x == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    for (int x = 0; x < kKSt; ++x) {
      mbar_init(&sm->k_full[x], 1);
      mbar_init(&sm->k_empty[x], 1);
    }
    for (int x = 0; x < kVSt; ++x) {
      mbar_init(&sm->v_full[x], 1);
      mbar_init(&sm->v_empty[x], 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&sm->q_full[x], 1);
      mbar_init(&sm->s_full[x], 1);
      mbar_init(&sm->p_part[x], 4);  // one arrive per softmax warp
      mbar_init(&sm->p_full[x], 4);
      mbar_init(&sm->o_full[x], 1);
      mbar_init(&sm->pv_half[x], 1);
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
  const int kvh = T[0].n > 0 ? T[0].kvh : T[1].kvh;

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t keep = policy_evict_last(), once = policy_evict_first();
      for (int x = 0; x < 2; ++x)
        if (T[x].n > 0) {  // Q is read once: evict-first, K/V are re-read by every unit of the KV head: evict-last
          mbar_expect_tx(&sm->q_full[x], kTileBytes);
          tma_load_3d_hint(sQ[x], &tm_q, &sm->q_full[x], 0, T[x].qb * 128, T[x].h, once);
          tma_load_3d_hint(sQ[x] + kBoxBytes, &tm_q, &sm->q_full[x], 64, T[x].qb * 128, T[x].h, once);
        }
      UnionWalk w{T[0].list, T[1].list, T[0].n, T[1].n, 0, 0};
      int kb;
      bool inA, inB;
      K3Prof pf;
      int sk = 0, pk = 0, sv = 0, pv = 0;  // ring slot and its wrap count (phase) for K and V
      for (int t = 0; w.next(kb, inA, inB); ++t) {
        const int key0 = kb * 128;
        pf.start();
        if (t >= kKSt) k3_wait(&sm->k_empty[sk], (pk - 1) & 1);
        pf.stop(10);
        mbar_expect_tx(&sm->k_full[sk], kTileBytes);
        unsigned char* sK = sK0 + sk * kTileBytes;
        tma_load_3d_hint(sK, &tm_k, &sm->k_full[sk], 0, key0, kvh, keep);
        tma_load_3d_hint(sK + kBoxBytes, &tm_k, &sm->k_full[sk], 64, key0, kvh, keep);
        pf.start();
        if (t >= kVSt) k3_wait(&sm->v_empty[sv], (pv - 1) & 1);
        pf.stop(11);
        mbar_expect_tx(&sm->v_full[sv], kTileBytes);
        unsigned char* sV = sV0 + sv * kTileBytes;
        tma_load_3d_hint(sV, &tm_v, &sm->v_full[sv], 0, key0, kvh, keep);
        tma_load_3d_hint(sV + kBoxBytes, &tm_v, &sm->v_full[sv], 64, key0, kvh, keep);
        if (++sk == kKSt) sk = 0, ++pk;
        if (++sv == kVSt) sv = 0, ++pv;
      }
      pf.flush(true);
    }
  } else if (warp == 1) {
    // Descriptors are linear in the smem address (start address >> 4 in the low
    // bits), so each operand is a precomputed base plus a constant: keeps the
    // issuer's per-MMA work to one add on a sub-partition shared with softmax warps.
    const uint64_t q_desc[2] = {sdesc_sw128(smem_u32(sQ[0]), 16, 1024), sdesc_sw128(smem_u32(sQ[1]), 16, 1024)};
    const uint64_t k_desc0 = sdesc_sw128(smem_u32(sK0), 16, 1024);
    const uint64_t v_desc0 = sdesc_sw128(smem_u32(sV0), kBoxBytes, 1024);
    int n_s[2] = {0, 0};      // S MMAs issued per item
    int n_pv[2] = {0, 0};     // PV MMAs issued per item
    int pend[2] = {-1, -1};   // union step whose PV is still to be issued
    K3Prof pf;
#if SA_K3_PROF
    const long long t_loop = clock64();
#endif
    UnionWalk w{T[0].list, T[1].list, T[0].n, T[1].n, 0, 0};
    int kb;
    bool in[2];
    int t = 0;
    // O_X += P_X V(step): keys 0..63 once that half of P is in TMEM, 64..127 after
    auto issue_pv = [&](int x, int step) {
      const int j = n_pv[x];
      const int s = step % kVSt;
      pf.start();
      k3_wait(&sm->p_part[x], j & 1);
      pf.stop(5);
      pf.start();
      k3_wait(&sm->v_full[s], (step / kVSt) & 1);
      pf.stop(7);
      tc_fence_after();
      if (elect_one()) {
        constexpr int kFirst = 4;  // K-steps (16 keys each) covered by p_part
#pragma unroll
        for (int kk = 0; kk < kFirst; ++kk)
          umma_ts(tO[x], tS[x] + kk * 8, v_desc0 + ((s * kTileBytes + kk * 2048) >> 4), kIdescPV,
                  (j > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&sm->pv_half[x]);  // the softmax's rare second-half rescale waits for this
      }
      __syncwarp();
      pf.start();
      k3_wait(&sm->p_full[x], j & 1);
      pf.stop(6);
      tc_fence_after();
      if (elect_one()) {
        constexpr int kFirst = 4;
#pragma unroll
        for (int kk = kFirst; kk < 8; ++kk)
          umma_ts(tO[x], tS[x] + kk * 8,
                  v_desc0 + ((s * kTileBytes + kk * 2048) >> 4), kIdescPV, 1u);
        if (j == T[x].n - 1) umma_commit(&sm->o_full[x]);
      }
      __syncwarp();
      n_pv[x] = j + 1;
    };
    // S_X(step) from K slot `slot`: 8 K-steps of 16 into TMEM S_X, then s_full[X]
    auto issue_s = [&](int x, int slot) {
      pf.start();
      if (n_s[x] == 0) k3_wait(&sm->q_full[x], 0);
      pf.stop(9);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * kBoxBytes + (kk & 3) * 32;
          umma_ss(tS[x], q_desc[x] + (off >> 4), k_desc0 + ((slot * kTileBytes + off) >> 4), kIdescQK,
                  kk > 0 ? 1u : 0u);
        }
        umma_commit(&sm->s_full[x]);
      }
      __syncwarp();
      ++n_s[x];
    };
    int sk = 0, pk = 0;  // K ring slot of step t and its wrap count
    while (w.next(kb, in[0], in[1])) {
      const int s = sk;
      pf.start();
      k3_wait(&sm->k_full[s], pk & 1);
      pf.stop(8);
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        if (pend[x] >= 0) {
          issue_pv(x, pend[x]);
          pend[x] = -1;
        }
        if (in[x]) {
          issue_s(x, s);
          pend[x] = t;
        }
      }
      if (elect_one()) {
        umma_commit(&sm->k_empty[s]);
        if (t >= 1) umma_commit(&sm->v_empty[(t - 1) % kVSt]);  // every PV of step t-1 is issued by now
      }
      __syncwarp();
      ++t;
      if (++sk == kKSt) sk = 0, ++pk;
    }
#pragma unroll
    for (int x = 0; x < 2; ++x)
      if (pend[x] >= 0) issue_pv(x, pend[x]);
#if SA_K3_PROF
    pf.add(12, clock64() - t_loop);
    pf.add(13, T[0].n + T[1].n);
#endif
    pf.flush(lane_id() == 0);
  } else if (warp >= 4) {
    const int x = warp < 8 ? 0 : 1;
    const K3Tile Tx = x ? T[1] : T[0];  // select, not a dynamically indexed (local-memory) array
    if (Tx.n > 0) {
      const K3TileBars b{&sm->s_full[x], &sm->pv_half[x], &sm->p_part[x], &sm->p_full[x], &sm->o_full[x]};
      k3_softmax_tile(Tx, b, x ? tS[1] : tS[0], x ? tO[1] : tO[0], warp & 3, P.S, P.out, P.peers, P.lse, P.touched,
                      P.status);
    } else if ((x ? ib : ia) >= 0 && warp == 4 + 4 * x && lane_id() == 0) {
      report_status(P.status, SA_STATUS_EMPTY_BLOCK, Tx.h, Tx.qb);  // ref executor.py:131-132
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace

int launch_sparse_share(const void* q, const void* k, const void* v, int S, int Hq, int Hkv, int group,
                        int q_head0, const int* kv_cnt, const int* kv_idx, const int* units, void* out,
                        float* lse, long long* touched, cudaStream_t st, void* const* peer_out, int n_peer) {
  CUtensorMap tq, tk, tv;
  if (!make_tmap_bf16_hsd(&tq, q, Hq, S, 128) || !make_tmap_bf16_hsd(&tk, k, Hkv, S, 128) ||
      !make_tmap_bf16_hsd(&tv, v, Hkv, S, 128))
    return fail(SA_ERR_CUDA, "sparse_forward: cuTensorMapEncodeTiled failed");
  ShareParams P;
  P.S = S;
  P.Hq = Hq;
  P.nb = ceil_div(S, 128);
  P.group = group;
  P.q_head0 = q_head0;
  P.kv_cnt = kv_cnt;
  P.kv_idx = kv_idx;
  P.units = units;
  P.out = static_cast<__nv_bfloat16*>(out);
  P.peers.n = n_peer;
  for (int p = 0; p < K3PeerOut::kMax; ++p)
    P.peers.ptr[p] = p < n_peer ? static_cast<__nv_bfloat16*>(peer_out[p]) : nullptr;
  P.lse = lse;
  P.touched = touched;
  P.status = status_ptr();
  const size_t smem = (2 + kKSt + kVSt) * (size_t)kTileBytes + sizeof(ShareSmem) + 1024;
  set_smem_attr(reinterpret_cast<const void*>(&k3_share), (int)smem);
  if (touched) cudaMemsetAsync(touched, 0, sizeof(long long) * Hq, st);
  const int nu = n_units(Hq, P.nb, group, q_head0);
  k3_share<<<nu, kThreads, smem, st>>>(tq, tk, tv, P);
  return check_launch("sparse_forward tcgen05 (K/V-sharing units)");
}

}  // namespace sa

extern "C" int sa_debug_k3s_profile(unsigned long long* out16, int reset) {
  cudaMemcpyFromSymbol(out16, sa::g_k3s_prof, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(sa::g_k3s_prof, z, sizeof(z));
  }
  return 0;
}
