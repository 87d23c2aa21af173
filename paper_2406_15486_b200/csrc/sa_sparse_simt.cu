// Stage 3, fp32 mode: exact SIMT block-sparse causal attention (replaces
// sparse_attention, ref pkg/src/blocksift/executor.py:104-158, for the fp32
// configuration; tolerance 1e-4 against the fp64 reference).
//
// One CTA per (head, query block) work item, one thread per query row; the
// listed key blocks stream through shared memory 32 keys at a time; the
// online-softmax recurrence (running max m, normaliser l, weighted sum) is the
// reference's, with logits (q * 1/sqrt(d)) . k (executor.py:124,133,139) and
// entry-level causality only in the diagonal block.  Any d <= 128 and
// blk <= 128: rows are zero-padded to the DP template width in shared memory.
#include "sa_internal.h"

namespace sa {
namespace {

constexpr int kChunk = 32;

template <int DP>
__global__ void __launch_bounds__(128)
    k3_simt(const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
            int S, int d, int blk, int nb, int group, int q_head0, const int* __restrict__ kv_cnt,
            const int* __restrict__ kv_idx, const int* __restrict__ order, float* __restrict__ out,
            float* __restrict__ lse, long long* __restrict__ touched, unsigned* status) {
  extern __shared__ float sm_f[];
  float (*ks)[DP + 1] = reinterpret_cast<float (*)[DP + 1]>(sm_f);
  float (*vs)[DP + 1] = reinterpret_cast<float (*)[DP + 1]>(sm_f + kChunk * (DP + 1));
  float (*qs)[DP + 1] = reinterpret_cast<float (*)[DP + 1]>(sm_f + 2 * kChunk * (DP + 1));
  const int item = order ? order[blockIdx.x] : (int)blockIdx.x;  // flattened unit list
  if (item < 0) return;
  const int h = item / nb, qb = item - h * nb;
  const int n = kv_cnt[item];
  const int* list = kv_idx + (size_t)h * tri(nb) + tri(qb);
  const int kvh = kv_head_of(h, group, q_head0);
  const int i = threadIdx.x;
  const int row = qb * blk + i;
  const bool valid = i < blk && row < S;
  const float scale = 1.0f / sqrtf((float)d);
  float acc[DP];
  float* qr = qs[threadIdx.x];
#pragma unroll
  for (int c = 0; c < DP; ++c) {
    qr[c] = (valid && c < d) ? q[((size_t)h * S + row) * d + c] * scale : 0.f;
    acc[c] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  const float* kh = k + (size_t)kvh * S * d;
  const float* vh = v + (size_t)kvh * S * d;
  if (n == 0 && threadIdx.x == 0) report_status(status, SA_STATUS_EMPTY_BLOCK, h, qb);  // executor.py:131-132
  bool bad_list = n > 0 && list[n - 1] != qb;  // BlockMask invariants, filtering.py:97-106
  for (int j = 0; j < n; ++j) {
    const int kb = list[j];
    bad_list |= kb > qb || (j > 0 && kb <= list[j - 1]);
    const int k0 = kb * blk, k1 = min(k0 + blk, S);
    for (int c0 = k0; c0 < k1; c0 += kChunk) {
      const int cn = min(kChunk, k1 - c0);
      __syncthreads();
      for (int e = threadIdx.x; e < kChunk * DP; e += blockDim.x) {
        const int t = e / DP, c = e - t * DP;
        const bool ok = t < cn && c < d;
        ks[t][c] = ok ? kh[(size_t)(c0 + t) * d + c] : 0.f;
        vs[t][c] = ok ? vh[(size_t)(c0 + t) * d + c] : 0.f;
      }
      __syncthreads();
      if (!valid) continue;
      float s[kChunk];
      float mx = -INFINITY;
#pragma unroll
      for (int t = 0; t < kChunk; ++t) {
        float dot = 0.f;
#pragma unroll
        for (int c = 0; c < DP; ++c) dot = fmaf(qr[c], ks[t][c], dot);
        const bool live = t < cn && (kb != qb || c0 + t <= row);
        s[t] = live ? dot : -INFINITY;
        mx = fmaxf(mx, s[t]);
      }
      if (mx == -INFINITY) continue;
      const float m_new = fmaxf(m, mx);
      const float corr = expf(m - m_new);
      l *= corr;
#pragma unroll
      for (int c = 0; c < DP; ++c) acc[c] *= corr;
#pragma unroll
      for (int t = 0; t < kChunk; ++t) {
        const float p = expf(s[t] - m_new);
        l += p;
#pragma unroll
        for (int c = 0; c < DP; ++c) acc[c] = fmaf(p, vs[t][c], acc[c]);
      }
      m = m_new;
    }
  }
  if (threadIdx.x == 0 && bad_list) report_status(status, SA_STATUS_MASK, h, qb);
  if (valid && n > 0 && !(l > 0.f && l < INFINITY)) report_status(status, SA_STATUS_NORMALISER, h, qb);
  if (valid) {
    const float inv = 1.f / l;
    for (int c = 0; c < d; ++c) out[((size_t)h * S + row) * d + c] = acc[c] * inv;
    if (lse) lse[(size_t)h * S + row] = m + logf(l);
  }
  if (threadIdx.x == 0 && touched)
    atomicAdd(reinterpret_cast<unsigned long long*>(touched + h), (unsigned long long)n);
}

}  // namespace

int launch_sparse_simt(const float* q, const float* k, const float* v, int S, int Hq, int Hkv, int d,
                       int blk, int group, int q_head0, const int* kv_cnt, const int* kv_idx,
                       const int* order, int n_order, float* out, float* lse, long long* touched,
                       cudaStream_t st) {
  const int nb = ceil_div(S, blk);
  const int threads = blk < 32 ? 32 : blk;
  if (touched) cudaMemsetAsync(touched, 0, sizeof(long long) * Hq, st);
  const dim3 grid(order ? n_order : Hq * nb);
#define SA_SIMT_CASE(DPV)                                                                    \
  do {                                                                                       \
  cudaFuncSetAttribute(k3_simt<DPV>, cudaFuncAttributeMaxDynamicSharedMemorySize,               \
                       (int)((2 * kChunk + threads) * (DPV + 1) * sizeof(float)));               \
  k3_simt<DPV><<<grid, threads, (2 * kChunk + threads) * (DPV + 1) * sizeof(float), st>>>(q, k, v, S, d, blk, nb, group, q_head0, kv_cnt, kv_idx, \
                                         order, out, lse, touched, status_ptr()); \
  } while (0)
  if (d <= 8)
    SA_SIMT_CASE(8);
  else if (d <= 16)
    SA_SIMT_CASE(16);
  else if (d <= 32)
    SA_SIMT_CASE(32);
  else if (d <= 64)
    SA_SIMT_CASE(64);
  else
    SA_SIMT_CASE(128);
#undef SA_SIMT_CASE
  return check_launch("sparse_forward fp32");
}

}  // namespace sa
