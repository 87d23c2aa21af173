// Stage-3 softmax warpgroup of one 128-row query tile (k3_share).
// ref executor.py:124-151: per listed key block s = (q/sqrt(d)) k^T, -inf
// above the diagonal only on the diagonal block, online max / sum,
// O = sum P V, out = O / l.
//
// One query row per thread (= TMEM lane).  bf16 P is written over S (columns
// [0, 64)) for the A-from-TMEM PV MMA.  O is rescaled in TMEM only when the
// running max grows by more than 2^8 (lazy rescale).
//   * fast path (off-diagonal blocks after the first): ONE read of S, the
//     exponentials taken against the running max; P is published in two
//     halves (keys 0..63 on p_part, 64..127 on p_full) so the first half of
//     the PV MMA overlaps the softmax of the second half;
//   * two-pass path (first block, diagonal block, or a max jump in the first
//     half): row max, optional O rescale, then exponentials.
// Mask invariants the reference enforces on BlockMask (filtering.py:97-106:
// kb <= qb, the diagonal kept, ascending lists) and the executor's empty-block
// / empty-normaliser errors (executor.py:131-132, 150-153) are checked on the
// device and reported through the status word (sa_status).
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
  uint64_t* s_full;   // S(j) landed in TMEM           (tcgen05.commit)
  uint64_t* pv_half;  // PV(j) over keys 0..63 done    (tcgen05.commit)
  uint64_t* p_part;   // P(j) keys 0..63 in TMEM       (one arrive per softmax warp)
  uint64_t* p_full;   // P(j) complete                 (one arrive per softmax warp)
  uint64_t* o_full;   // last PV done                  (tcgen05.commit)
};

// Output rows also stored into up to kMax peer gather buffers (peer-mapped
// device pointers at the same [Hq][S][d] rows), tile by tile over NVLink.
struct K3PeerOut {
  static constexpr int kMax = 7;  // SA_MAX_PEERS
  __nv_bfloat16* ptr[kMax];
  int n;
};

// Lazy rescale threshold (log2 units): unnormalised P stays <= 2^8.
constexpr float kK3RescaleThreshold = 8.0f;

// Cycle accounting (build with -DSA_K3_PROF=1, read with sa_debug_k3s_profile):
// slots 0-3 softmax (wait S, pass 1, rescale, pass 2 / fast path), 4 epilogue
// wait, 5-9 issuer (wait P part, P full, V, K, Q), 10-11 producer (wait K, V
// empty), 12 issuer loop total, 13 blocks processed.
#ifndef SA_K3_PROF
#define SA_K3_PROF 0
#endif
static __device__ unsigned long long g_k3s_prof[16];
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

// Exponentials moved from the MUFU pipe to the FMA pipe (ex2_poly2_floor):
// per 128-key block the two softmax warps of an SM sub-partition need 8192
// MUFU ex2 (2048 cycles at 4/clk), exactly the 2048 cycles of tensor work of
// the step, so a share of emulated pairs gives the MUFU slack.  A pair (t in
// 0..15) of 32-key fragment fr (0..3) is emulated when bit fr of
// SA_K3_EMU_FRAG and bit t of SA_K3_EMU_T are set.  Product: fragments 1 and 2,
// pairs 6, 7, 14, 15 = 1/8 of the exponentials (A/B in DESIGN.md §3.1).
#ifndef SA_K3_EMU_FRAG
#define SA_K3_EMU_FRAG 0x6
#endif
#ifndef SA_K3_EMU_T
#define SA_K3_EMU_T 0xC0C0
#endif

__device__ __forceinline__ uint64_t k3_exp_pair(float y0, float y1, int fr, int t) {
  return (((SA_K3_EMU_FRAG >> fr) & 1) && ((SA_K3_EMU_T >> t) & 1)) ? ex2_poly2_floor(y0, y1)
                                                                     : f32x2(ex2(y0), ex2(y1));
}

__device__ __forceinline__ void k3_softmax_tile(const K3Tile& T, const K3TileBars& b, uint32_t tS0,
                                                uint32_t tO0, int quad, int S, __nv_bfloat16* out,
                                                const K3PeerOut& peers, float* lse, long long* touched, unsigned* status) {
  const int i = quad * 32 + lane_id();  // query row within the tile
  const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
  const uint32_t tS = tS0 + lane_off, tO = tO0 + lane_off;
  const float sl2 = 1.4426950408889634f * 0.08838834764831845f;  // log2(e) / sqrt(128)
  const uint64_t sl2x2 = f32x2(sl2, sl2);
  float m_ref = -INFINITY;
  uint64_t lacc0 = f32x2(0.f, 0.f), lacc1 = f32x2(0.f, 0.f);
  K3Prof pf;
  // P-ready: every lane has waited for and fenced its own TMEM stores, then
  // one arrive per warp (barrier count 4)
  auto arrive = [&](uint64_t* bar) {
    __syncwarp();
    if (lane_id() == 0) mbar_arrive(bar);
  };
  int pv_seen = 0;  // pv_half phases consumed
  int prev_kb = -1;
  bool bad_list = false;
  for (int j = 0; j < T.n; ++j) {
    const int kb = __ldg(T.list + j);
    bad_list |= kb <= prev_kb || kb > T.qb;
    prev_kb = kb;
    const bool diag = kb == T.qb;  // warp-uniform
    if (pv_seen < j) {
      // consume the previous block's pv_half phase so that every phase has a
      // waiter (compute-sanitizer synccheck); it completes before this block's
      // S (same in-order tensor pipe), so the S wait below hides it
      k3_wait(b.pv_half, pv_seen & 1);
      ++pv_seen;
    }
    pf.start();
    k3_wait(b.s_full, j & 1);
    pf.stop(0);
    pf.start();
    tc_fence_after();
    if (j > 0 && !diag) {
      // ---- fast path.  If any row's max exceeds m_ref + 8 in the first half, S
      // is still intact and the block falls through to the two-pass path; a
      // jump in the second half (rare) waits until the first half's PV has
      // landed in O, rescales O and the row sum and redoes keys 64..127.
      bool done = false;
      uint32_t pk[32];
      uint64_t bacc0, bacc1;
      uint32_t buf[2][32];
      auto load_half = [&](int h) {
        tmem_ld32(tS + h * 64, buf[0]);
        tmem_ld32(tS + h * 64 + 32, buf[1]);
      };
      auto half_exps = [&](int h, float m, float& ymax) {
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
            const uint64_t pp = k3_exp_pair(y0, y1, 2 * h + ch, t);
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
      half_exps(0, m_ref, ymax);
      if (!__any_sync(0xffffffffu, ymax > kK3RescaleThreshold)) {
        store_half(0);
        arrive(b.p_part);
        lacc0 = fadd2(lacc0, bacc0);
        lacc1 = fadd2(lacc1, bacc1);
        load_half(1);
        half_exps(1, m_ref, ymax);
        if (__any_sync(0xffffffffu, ymax > kK3RescaleThreshold)) {
          k3_wait(b.pv_half, j & 1);  // O now holds every PV up to this block's keys 0..63
          pv_seen = j + 1;
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
          half_exps(1, m_ref, ymax);  // with the row max of keys 64..127 every exponent is <= 0
        }
        store_half(1);
        arrive(b.p_full);
        lacc0 = fadd2(lacc0, bacc0);
        lacc1 = fadd2(lacc1, bacc1);
        done = true;
      }
      if (done) {
        pf.stop(3);
        continue;
      }
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
            const uint64_t pp = k3_exp_pair(y0, y1, ch, t);
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
        if (ch == 1) {  // keys 0..63 of P are in TMEM: let the PV MMA start
          tmem_st_wait();
          tc_fence_before();
          arrive(b.p_part);
        }
        if (ch < 3) tmem_ld_wait_regs(buf[(ch + 1) & 1]);
      }
    }
    tmem_st_wait();
    tc_fence_before();
    arrive(b.p_full);
    pf.stop(3);
  }
  // ---- epilogue: O / l -> bf16
  float l;
  {
    float a0, a1, b0, b1;
    unpack_f32x2(lacc0, a0, a1);
    unpack_f32x2(lacc1, b0, b1);
    l = (a0 + a1) + (b0 + b1);
  }
  const int row = T.qb * 128 + i;
  const bool valid = row < S;
  {
    unsigned bits = 0;
    if (bad_list || prev_kb != T.qb) bits |= SA_STATUS_MASK;
    if (valid && !(l > 0.f && l < INFINITY)) bits |= SA_STATUS_NORMALISER;
    bits = __reduce_or_sync(0xffffffffu, bits);
    if (bits && lane_id() == 0) report_status(status, bits, T.h, T.qb);
  }
  pf.start();
  k3_wait(b.o_full, 0);
  pf.stop(4);
  pf.flush(lane_id() == 0);
  tc_fence_after();
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
      // the gather: the same row into every peer's buffer (remote stores over NVLink)
      for (int p = 0; p < peers.n; ++p) {
        uint4* r4 = reinterpret_cast<uint4*>(peers.ptr[p] + ((size_t)T.h * S + row) * 128 + ch * 32);
#pragma unroll
        for (int t = 0; t < 4; ++t) r4[t] = make_uint4(pk[4 * t], pk[4 * t + 1], pk[4 * t + 2], pk[4 * t + 3]);
      }
    }
  }
  if (valid && lse) lse[(size_t)T.h * S + row] = (m_ref + __log2f(l)) * 0.6931471805599453f;
  if (i == 0 && touched) atomicAdd(reinterpret_cast<unsigned long long*>(touched + T.h), (unsigned long long)T.n);
}

}  // namespace sa
