// Stage-3 softmax warpgroup of one 128-row query tile (shared by the
// tensor-core stage-3 kernels).  ref executor.py:124-151: per listed key block
// s = (q/sqrt(d)) k^T, -inf above the diagonal only on the diagonal block,
// online max / sum, O = sum P V, out = O / l.
//
// One query row per thread (= TMEM lane).  S (fp32, 128 TMEM columns) is read
// twice, row max then exponentials, with the TMEM loads double-buffered; bf16 P
// is written over S (columns [0, 64)) for the A-from-TMEM PV MMA.  Part of P
// is published early (p_part) so the PV MMA starts before the rest lands.  An
// FMA-pipe polynomial can take a share of the exponentials (SA_K3_POLY).  O is
// rescaled in TMEM only when the running max grows by more than 2^8.
#pragma once
#include <cuda_bf16.h>

#include "sa_internal.h"
#include "sa_ptx.cuh"

namespace sa {

struct K3Tile {
  int n, h, qb, kvh;
  const int* list;  // ascending key blocks of (h, qb)
};

struct K3TileBars {
  uint64_t* s_full;  // S(j) landed in TMEM           (tcgen05.commit)
  uint64_t* pv_half; // PV(j) over keys 0..63 done    (tcgen05.commit; split fast path only, may be null)
  uint64_t* p_part;  // P(j) keys 0..63 (split fast path) / 0..95 in TMEM (128 arrivals; pair mode: 1 per CTA)
  uint64_t* p_full;  // P(j) complete                  (128 arrivals; pair mode: 1 per CTA)
  uint64_t* o_full;  // last PV done                   (tcgen05.commit)
};

// Lazy rescale: O is rescaled (and, on the single-read fast path, the block
// redone) only when a row's max grows by more than this many log2 units, so
// unnormalised P stays <= 2^threshold (bf16 / fp32 safe far beyond 2^16).
#ifndef SA_K3_RESCALE_LOG2
#define SA_K3_RESCALE_LOG2 8.0f
#endif
constexpr float kK3RescaleThreshold = SA_K3_RESCALE_LOG2;  // log2 units

__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Cycle accounting (build with -DSA_K3_PROF=1, read with sa_debug_k3s_profile):
// slots 0-3 softmax (wait S, pass 1, rescale, pass 2), 4 epilogue wait,
// 5-9 issuer (wait P part, P full, V, K, Q), 10-11 producer (wait K, V empty),
// 12 issuer loop total, 13 blocks processed.
#ifndef SA_K3_PROF
#define SA_K3_PROF 0
#endif
static __device__ unsigned long long g_k3s_prof[16];  // one copy per kernel translation unit
struct K3Prof {
#if SA_K3_PROF
  long long acc[16] = {0};
  long long t0 = 0;
  __device__ __forceinline__ void start() { t0 = clock64(); }
  __device__ __forceinline__ void stop(int slot) { acc[slot] += clock64() - t0; }
  __device__ __forceinline__ void add(int slot, long long v) { acc[slot] += v; }
  __device__ __forceinline__ void flush(bool leader) {
    if (leader)
      for (int k = 0; k < 16; ++k)
        if (acc[k]) atomicAdd(&g_k3s_prof[k], (unsigned long long)acc[k]);
  }
#else
  __device__ __forceinline__ void start() {}
  __device__ __forceinline__ void stop(int) {}
  __device__ __forceinline__ void add(int, long long) {}
  __device__ __forceinline__ void flush(bool) {}
#endif
};

// Fraction of off-diagonal exponentials computed by the FMA-pipe polynomial:
// SA_K3_POLY n -> n/4 (build-time knob; production 0: with P published in two
// halves, all-MUFU exponentials measured ~4 % faster than a 1/4 polynomial share).
#ifndef SA_K3_WARPARRIVE  // P-ready barriers: one arrive per softmax warp (count 4) instead of per thread (128)
#define SA_K3_WARPARRIVE 1
#endif
#ifndef SA_K3_PVDRAIN  // wait on every pv_half phase (compute-sanitizer synccheck clean); 0: rare path only
#define SA_K3_PVDRAIN 1
#endif
#ifndef SA_K3_PREF  // fast path: issue the second half's TMEM loads before the first half's check/store
#define SA_K3_PREF 0  // 1 measured 0.5 ms slower at C3
#endif
#ifndef SA_K3_POLY
#define SA_K3_POLY 0
#endif
// SA_K3_EXP (timing experiments only): 1 = no softmax math (arrive at once),
// 2 = no exponentials (P = the scaled score, finite garbage), 3 = no math but
// SA_K3_SPIN cycles of delay (separates the softmax's latency from its
// resource use), 4 = the softmax's TMEM reads and writes without the math.
#ifndef SA_K3_SPIN
#define SA_K3_SPIN 1300
#endif
#ifndef SA_K3_EXP
#define SA_K3_EXP 0
#endif
// Fast path exponentials as ex2.approx.f16x2 (one MUFU op per pair; experiment).
#ifndef SA_K3_EXPH
#define SA_K3_EXPH 0
#endif
// Single-SM kernels: the fast path publishes P in two halves (keys 0..63, then
// 64..127) so the PV MMA starts after half of the softmax (see k3_softmax_tile).
#ifndef SA_K3_FASTSPLIT
#define SA_K3_FASTSPLIT 1
#endif
// Single-read fast path for off-diagonal blocks (see k3_softmax_tile).
#ifndef SA_K3_FAST
#define SA_K3_FAST 1
#endif


// Pair mode (cta_group::2 kernel): the tile walks the ascending UNION of its own
// block list and its partner's (one 256-row MMA covers both tiles); on steps
// outside its own list it only writes P = 0 for its rows.  The P-ready
// arrivals go to the pair leader's barriers (cluster addresses).
struct K3PairCtx {
  const int* other_list;
  int other_n;
  uint32_t p_part_cl, p_full_cl;  // the leader's P barriers (cluster addresses)
  bool remote;                    // this CTA is the peer: arrive remotely
};

template <bool kPair>
__device__ __forceinline__ void k3_softmax_tile(const K3Tile& T, const K3TileBars& b, uint32_t tS0,
                                                uint32_t tO0, int quad, int S, __nv_bfloat16* out,
                                                float* lse, long long* touched, const K3PairCtx pc = {}) {
  const int i = quad * 32 + lane_id();  // query row within the tile
  const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
  const uint32_t tS = tS0 + lane_off, tO = tO0 + lane_off;
  const float sl2 = 1.4426950408889634f * 0.08838834764831845f;  // log2(e) / sqrt(128)
  const uint64_t sl2x2 = f32x2(sl2, sl2);
  float m_ref = -INFINITY;
  uint64_t lacc0 = f32x2(0.f, 0.f), lacc1 = f32x2(0.f, 0.f);
  K3Prof pf;
  // P-ready arrivals.  Single-SM kernels: every softmax thread arrives on the
  // CTA's own barrier (count 128).  Pair mode: the tile's 128 softmax threads
  // meet at a named barrier (each has waited for and fenced its own TMEM
  // stores first), then ONE thread arrives on the leader CTA's barrier (count
  // 2: one per CTA) -- a remote cluster-scope arrive per thread stalls every
  // warp, one per CTA does not.
  auto arrive_on = [&](uint64_t* local, uint32_t cl) {
    if (kPair) {
      named_bar_sync(1, 128);
      if (quad == 0 && lane_id() == 0) {
        if (pc.remote)
          mbar_arrive_cluster(cl);
        else
          mbar_arrive(local);
      }
    } else {
#if SA_K3_WARPARRIVE
      __syncwarp();  // every lane has waited for and fenced its TMEM stores
      if (lane_id() == 0) mbar_arrive(local);
#else
      mbar_arrive(local);
#endif
    }
  };
  auto arrive_part = [&]() { arrive_on(b.p_part, pc.p_part_cl); };
  auto arrive_full = [&]() { arrive_on(b.p_full, pc.p_full_cl); };
  // p_part covers keys 0..63 (chunks 0-1) with the split fast path, else keys 0..95
  constexpr int kPartCh = (!kPair && SA_K3_FASTSPLIT) ? 1 : 2;
  int ia = 0, ib = 0;  // union walk (pair mode)
  int jj = 0;          // own blocks processed so far
  int pv_seen = 0;     // pv_half phases consumed (split fast path)
  for (int j = 0;; ++j) {
    int kb;
    bool mine = true;
    if (kPair) {
      if (ia >= T.n && ib >= pc.other_n) break;
      const int ka = ia < T.n ? __ldg(T.list + ia) : 0x7fffffff;
      const int kc = ib < pc.other_n ? __ldg(pc.other_list + ib) : 0x7fffffff;
      kb = min(ka, kc);
      mine = ka == kb;
      ia += mine;
      ib += kc == kb;
    } else {
      if (j >= T.n) break;
      kb = __ldg(T.list + j);
    }
    const bool diag = kb == T.qb;  // warp-uniform
#if SA_K3_PVDRAIN
    if (!kPair && SA_K3_FASTSPLIT && pv_seen < jj) {
      // consume the previous block's pv_half phase so that every phase has a waiter;
      // it completes before this block's S (same tensor pipe), so the wait below hides it
      k3_wait(b.pv_half, pv_seen & 1);
      ++pv_seen;
    }
#endif
    pf.start();
    k3_wait(b.s_full, j & 1);
    pf.stop(0);
    pf.start();
    tc_fence_after();
    if (kPair && !mine) {  // not this tile's block: its rows contribute P = 0
      uint32_t z[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) z[t] = 0u;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) tmem_st16(tS + ch * 16, z);
      tmem_st_wait();
      tc_fence_before();
      arrive_part();
      arrive_full();
      continue;
    }
    const bool first = jj == 0;
    ++jj;
#if SA_K3_FAST
    // ---- fast path (off-diagonal blocks after the first): ONE read of S.
    // Exponentials are taken against the running max m_ref, which the lazy
    // rescale already allows to trail the true max by up to 2^8; the block's
    // max is checked on the way and the packed P is held in registers until
    // the check passes.  If any row's max exceeds m_ref + 8 (rare once the
    // heavy columns have been seen) S is still intact in TMEM and the block
    // falls through to the two-pass path below.
    if (!kPair && SA_K3_FASTSPLIT && !first && !diag && SA_K3_EXP == 0) {
      // Two halves of 64 keys: each is published (p_part, p_full) as soon as its
      // exponentials pass the 2^8 check, so the first half of PV overlaps the
      // softmax of the second.  A failure in the first half leaves S intact for
      // the two-pass path; a failure in the second half (rare) waits until the
      // first half's PV has landed in O, rescales O and the row sum to the new
      // max and redoes keys 64..127 (their scores are still intact).
      const int jb = jj - 1;  // own block index
      bool done = false;
      uint32_t pk[32];
      uint64_t bacc0, bacc1;
      uint32_t buf[2][32];
      auto load_half = [&](int h) {
        tmem_ld32(tS + h * 64, buf[0]);
        tmem_ld32(tS + h * 64 + 32, buf[1]);
      };
      // exponentials of the half whose loads load_half() issued
      auto half_exps = [&](float m, float& ymax) {
        const uint64_t negm = f32x2(-m, -m);
        bacc0 = f32x2(0.f, 0.f);
        bacc1 = f32x2(0.f, 0.f);
        ymax = -INFINITY;
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
      };
      auto store_half = [&](int h) {  // bf16 P of keys 64h..64h+63 -> cols 32h..32h+31
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          uint32_t(&q)[16] = *reinterpret_cast<uint32_t(*)[16]>(&pk[ch * 16]);
          tmem_st16(tS + h * 32 + ch * 16, q);
        }
        tmem_st_wait();
        tc_fence_before();
      };
      float ymax;
      load_half(0);
      half_exps(m_ref, ymax);
#if SA_K3_PREF
      load_half(1);  // keys 64..127 stream in while half 0 is checked and stored
#endif
      if (!__any_sync(0xffffffffu, ymax > kK3RescaleThreshold)) {
        store_half(0);
        arrive_part();
        lacc0 = fadd2(lacc0, bacc0);
        lacc1 = fadd2(lacc1, bacc1);
#if !SA_K3_PREF
        load_half(1);
#endif
        half_exps(m_ref, ymax);
        if (__any_sync(0xffffffffu, ymax > kK3RescaleThreshold)) {
          k3_wait(b.pv_half, jb & 1);  // O now holds every PV up to this block's keys 0..63
          pv_seen = jb + 1;
          tc_fence_after();
          float mx = -INFINITY;
#pragma unroll
          for (int ch = 0; ch < 2; ++ch) {
            uint32_t r[32];
            tmem_ld32_sync(tS + 64 + ch * 32, r);
#pragma unroll
            for (int t = 0; t < 32; t += 2) mx = fmax3(mx, __uint_as_float(r[t]), __uint_as_float(r[t + 1]));
          }
          const float m_new = fmaxf(m_ref, mx * sl2);
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
          m_ref = m_new;
          load_half(1);
          half_exps(m_ref, ymax);  // with the row max of keys 64..127 every exponent is <= 0
        }
        store_half(1);
        arrive_full();
        lacc0 = fadd2(lacc0, bacc0);
        lacc1 = fadd2(lacc1, bacc1);
        done = true;
      }
      if (done) {
        pf.stop(3);
        continue;
      }
    } else if (!first && !diag && SA_K3_EXP == 0) {
      const uint64_t negm = f32x2(-m_ref, -m_ref);
      uint32_t pk[64];
      uint64_t bacc0 = f32x2(0.f, 0.f), bacc1 = f32x2(0.f, 0.f);
      float ymax = -INFINITY;
      {
        uint32_t buf[2][32];
        tmem_ld32(tS, buf[0]);
        tmem_ld_wait_regs(buf[0]);
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t(&r)[32] = buf[ch & 1];
          if (ch < 3) tmem_ld32(tS + (ch + 1) * 32, buf[(ch + 1) & 1]);
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            float y0, y1;
            unpack_f32x2(ffma2(f32x2(__uint_as_float(r[2 * t]), __uint_as_float(r[2 * t + 1])), sl2x2, negm),
                         y0, y1);
            ymax = fmax3(ymax, y0, y1);
            const uint64_t pp = SA_K3_EXPH ? ex2_h2(y0, y1)
                                : ((t & 3) >= 4 - SA_K3_POLY) ? ex2_poly2(y0, y1)
                                                              : f32x2(ex2(y0), ex2(y1));
            if (t & 1)
              bacc1 = fadd2(bacc1, pp);
            else
              bacc0 = fadd2(bacc0, pp);
            float p0, p1;
            unpack_f32x2(pp, p0, p1);
            pk[ch * 16 + t] = pack_bf16(p0, p1);
          }
          if (ch < 3) tmem_ld_wait_regs(buf[(ch + 1) & 1]);
        }
      }
      if (!__any_sync(0xffffffffu, ymax > kK3RescaleThreshold)) {
        lacc0 = fadd2(lacc0, bacc0);
        lacc1 = fadd2(lacc1, bacc1);
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t(&q)[16] = *reinterpret_cast<uint32_t(*)[16]>(&pk[ch * 16]);
          tmem_st16(tS + ch * 16, q);
          if (ch == 2) {  // keys 0..95 of P are in TMEM: let the PV MMA start
            tmem_st_wait();
            tc_fence_before();
            arrive_part();
          }
        }
        tmem_st_wait();
        tc_fence_before();
        arrive_full();
        pf.stop(3);
        continue;
      }
    }
#endif
    if (SA_K3_EXP == 4) {  // timing experiment: the softmax's TMEM traffic only (read S, write P), no math
      uint32_t acc = 0;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        uint32_t r[32];
        tmem_ld32_sync(tS + ch * 32, r);
#pragma unroll
        for (int t = 0; t < 32; ++t) acc ^= r[t];
      }
      uint32_t pk[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) pk[t] = acc & 0x3c003c00u;  // small finite bf16 pairs
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) tmem_st16(tS + ch * 16, pk);
      tmem_st_wait();
      tc_fence_before();
      arrive_part();
      arrive_full();
      continue;
    }
    if (SA_K3_EXP == 1 || SA_K3_EXP == 3) {
      if (SA_K3_EXP == 3) {  // timing experiment: a softmax that only takes SA_K3_SPIN cycles
        const long long t0 = clock64();
        while (clock64() - t0 < SA_K3_SPIN) {
        }
      }
      tc_fence_before();
      arrive_part();
      arrive_full();
      continue;
    }
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
    pf.stop(1);
    pf.start();
    // tcgen05.ld/st are warp-collective: rescale decision per warp.  O is
    // stable here: PV(j-1) completed before S(j) did (in-order tensor pipe).
    if (__any_sync(0xffffffffu, mxs > m_ref + kK3RescaleThreshold)) {
      const float m_new = fmaxf(m_ref, mxs);
      if (!first) {
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
    pf.stop(2);
    pf.start();
    // ---- pass 2: P = exp2(s*log2e/sqrt(d) - m) -> bf16 over S, row sum
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
            unpack_f32x2(ffma2(f32x2(__uint_as_float(r[2 * t]), __uint_as_float(r[2 * t + 1])), sl2x2, negm),
                         y0, y1);
            const float p0 = ex2(y0), p1 = ex2(y1);
            if (t & 1)
              lacc1 = fadd2(lacc1, f32x2(p0, p1));
            else
              lacc0 = fadd2(lacc0, f32x2(p0, p1));
            pk[t] = pack_bf16(p0, p1);
          }
        } else {
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            float y0, y1;
            unpack_f32x2(ffma2(f32x2(__uint_as_float(r[2 * t]), __uint_as_float(r[2 * t + 1])), sl2x2, negm),
                         y0, y1);
            const uint64_t pp = SA_K3_EXP == 2 ? f32x2(y0, y1)
                                : ((t & 3) >= 4 - SA_K3_POLY) ? ex2_poly2(y0, y1)
                                                              : f32x2(ex2(y0), ex2(y1));
            if (t & 1)
              lacc1 = fadd2(lacc1, pp);
            else
              lacc0 = fadd2(lacc0, pp);
            float p0, p1;
            unpack_f32x2(pp, p0, p1);
            pk[t] = pack_bf16(p0, p1);
          }
        }
        tmem_st16(tS + ch * 16, pk);
        if (ch == kPartCh) {  // the first part of P is in TMEM: let the PV MMA start
          tmem_st_wait();
          tc_fence_before();
          arrive_part();
        }
        if (ch < 3) tmem_ld_wait_regs(buf[(ch + 1) & 1]);
      }
    }
    tmem_st_wait();
    tc_fence_before();
    arrive_full();
    pf.stop(3);
  }
  if (kPair && T.n == 0) return;  // CTA without an item: its rows only padded the pair MMA
  // ---- epilogue: O / l -> bf16
  float l;
  {
    float a0, a1, b0, b1;
    unpack_f32x2(lacc0, a0, a1);
    unpack_f32x2(lacc1, b0, b1);
    l = (a0 + a1) + (b0 + b1);
  }
  pf.start();
  k3_wait(b.o_full, 0);
  pf.stop(4);
  pf.flush(lane_id() == 0);
  tc_fence_after();
  const int row = T.qb * 128 + i;
  const bool valid = row < S;
  const float inv = 1.f / l;
  __nv_bfloat16* dst = out + ((size_t)T.h * S + row) * 128;
  // the output streams through L2 once: mark it evict-first so it does not push
  // out the K/V of the KV head the other units are still reading
  const uint64_t stream_out = policy_evict_first();
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) {
    uint32_t r[32];
    tmem_ld32_sync(tO + ch * 32, r);
    uint32_t pk[16];
#pragma unroll
    for (int t = 0; t < 16; ++t)
      pk[t] = pack_bf16(__uint_as_float(r[2 * t]) * inv, __uint_as_float(r[2 * t + 1]) * inv);
    if (valid) {
      uint4* d4 = reinterpret_cast<uint4*>(dst + ch * 32);
#pragma unroll
      for (int t = 0; t < 4; ++t)
        st_global_v4_hint(d4 + t, make_uint4(pk[4 * t], pk[4 * t + 1], pk[4 * t + 2], pk[4 * t + 3]), stream_out);
    }
  }
  if (valid && lse) lse[(size_t)T.h * S + row] = (m_ref + __log2f(l)) * 0.6931471805599453f;
  if (i == 0 && touched) atomicAdd(reinterpret_cast<unsigned long long*>(touched + T.h), (unsigned long long)T.n);
}

// ---------------------------------------------------------------------------
// Split-column softmax: EIGHT warps per tile, two per TMEM lane quadrant.
// Warp (quad, half) owns rows quad*32..+31 and keys half*64..+63, so the
// per-tile softmax latency -- which sits on the S -> softmax -> PV -> S chain
// of every item -- is about half that of one warp per row.
//   * Fast path (off-diagonal blocks after the first): one read of the warp's
//     64 scores, exponentials against the running max m_ref, packed P held in
//     registers.  The two halves of a row then meet at a named barrier
//     (64 threads) to learn whether either saw a score above m_ref + 8; if
//     not, P is stored and m_ref stays (the common case: no max exchange).
//   * Otherwise (first block, diagonal block, max growth) both halves re-read
//     their scores (still intact: P was not stored), exchange the half-row
//     maxima through shared memory, rescale their 64 columns of O and their
//     partial row sums, and store P.
// Half h writes its bf16 P over the start of its own score columns (keys
// 0..63 -> cols 0..31, keys 64..127 -> cols 64..95) and signals its own
// p barrier (4 warps x 32 threads).  Row sums are combined in the epilogue.
struct K3SplitBars {
  uint64_t* s_full;   // S(j) landed in TMEM                 (tcgen05.commit)
  uint64_t* p_half0;  // P(j) keys 0..63 in cols 0..31        (128 arrivals)
  uint64_t* p_half1;  // P(j) keys 64..127 in cols 64..95     (128 arrivals)
  uint64_t* o_full;   // last PV done                         (tcgen05.commit)
};

// xchg: float[3][2][128] per tile: [parity 0/1 | epilogue][half][row]; flags: int[2][2][4] per tile
__device__ __forceinline__ void k3_softmax_split(const K3Tile& T, const K3SplitBars& b, uint32_t tS0, uint32_t tO0,
                                                 int quad, int half, float* xchg, int* flags, int bar_id, int S,
                                                 __nv_bfloat16* out, float* lse, long long* touched) {
  const int i = quad * 32 + lane_id();  // query row within the tile
  const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
  const uint32_t tS = tS0 + lane_off, tO = tO0 + lane_off;
  const int c0 = half * 64;  // first key (= score column) of this warp
  const float sl2 = 1.4426950408889634f * 0.08838834764831845f;  // log2(e) / sqrt(128)
  const uint64_t sl2x2 = f32x2(sl2, sl2);
  float m_ref = -INFINITY;
  uint64_t lacc0 = f32x2(0.f, 0.f), lacc1 = f32x2(0.f, 0.f);
  uint64_t* p_mine = half ? b.p_half1 : b.p_half0;
  for (int j = 0; j < T.n; ++j) {
    const int kb = __ldg(T.list + j);
    const bool diag = kb == T.qb;  // warp-uniform
    k3_wait(b.s_full, j & 1);
    tc_fence_after();
    uint32_t pk[32];
    bool ok = false;
    if (j > 0 && !diag) {  // fast path
      const uint64_t negm = f32x2(-m_ref, -m_ref);
      uint64_t bacc0 = f32x2(0.f, 0.f), bacc1 = f32x2(0.f, 0.f);
      float ymax = -INFINITY;
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        uint32_t r[32];
        tmem_ld32_sync(tS + c0 + ch * 32, r);
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          float y0, y1;
          unpack_f32x2(ffma2(f32x2(__uint_as_float(r[2 * t]), __uint_as_float(r[2 * t + 1])), sl2x2, negm), y0, y1);
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
      const int bad = __any_sync(0xffffffffu, ymax > kK3RescaleThreshold);
      int* fl = flags + (j & 1) * 8;  // parity double-buffered: [half][quad]
      if (lane_id() == 0) fl[half * 4 + quad] = bad;
      named_bar_sync(bar_id, 64);
      ok = !(bad | fl[(half ^ 1) * 4 + quad]);
      if (ok) {
        lacc0 = fadd2(lacc0, bacc0);
        lacc1 = fadd2(lacc1, bacc1);
      }
    }
    if (!ok) {  // exact path: block max over the whole row (both halves), rescale, exponentials
      float ma = -INFINITY, mb = -INFINITY;
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        uint32_t r[32];
        tmem_ld32_sync(tS + c0 + ch * 32, r);
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
      float mxs = fmaxf(ma, mb) * sl2;
      {
        float* slot = xchg + (j & 1) * 256;
        slot[half * 128 + i] = mxs;
        named_bar_sync(bar_id, 64);
        mxs = fmaxf(mxs, slot[(half ^ 1) * 128 + i]);
      }
      // both halves hold the same row maxima: identical (warp-wide) decisions
      if (__any_sync(0xffffffffu, mxs > m_ref + kK3RescaleThreshold)) {
        const float m_new = fmaxf(m_ref, mxs);
        if (j > 0) {
          const float f = ex2(m_ref - m_new);
          const uint64_t f2 = f32x2(f, f);
          lacc0 = fmul2(lacc0, f2);
          lacc1 = fmul2(lacc1, f2);
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            uint32_t o[16];
            tmem_ld16_sync(tO + c0 + ch * 16, o);
#pragma unroll
            for (int t = 0; t < 16; t += 2) {
              float a, c;
              unpack_f32x2(fmul2(f32x2(__uint_as_float(o[t]), __uint_as_float(o[t + 1])), f2), a, c);
              o[t] = __float_as_uint(a);
              o[t + 1] = __float_as_uint(c);
            }
            tmem_st16(tO + c0 + ch * 16, o);
          }
        }
        m_ref = m_new;
      }
      const uint64_t negm = f32x2(-m_ref, -m_ref);
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        uint32_t r[32];
        tmem_ld32_sync(tS + c0 + ch * 32, r);
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
      tmem_st16(tS + c0 + ch * 16, q);
    }
    tmem_st_wait();
    tc_fence_before();
    mbar_arrive(p_mine);
  }
  // ---- epilogue: combine the half-row sums, O / l -> bf16 (this warp's 64 columns)
  float l;
  {
    float a0, a1, b0, b1;
    unpack_f32x2(lacc0, a0, a1);
    unpack_f32x2(lacc1, b0, b1);
    l = (a0 + a1) + (b0 + b1);
    float* slot = xchg + 2 * 256;
    slot[half * 128 + i] = l;
    named_bar_sync(bar_id, 64);
    l += slot[(half ^ 1) * 128 + i];
  }
  k3_wait(b.o_full, 0);
  tc_fence_after();
  const int row = T.qb * 128 + i;
  const bool valid = row < S;
  const float inv = 1.f / l;
  __nv_bfloat16* dst = out + ((size_t)T.h * S + row) * 128 + c0;
  const uint64_t stream_out = policy_evict_first();
#pragma unroll
  for (int ch = 0; ch < 2; ++ch) {
    uint32_t r[32];
    tmem_ld32_sync(tO + c0 + ch * 32, r);
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
  if (half == 0) {
    if (valid && lse) lse[(size_t)T.h * S + row] = (m_ref + __log2f(l)) * 0.6931471805599453f;
    if (i == 0 && touched) atomicAdd(reinterpret_cast<unsigned long long*>(touched + T.h), (unsigned long long)T.n);
  }
}

}  // namespace sa
