/*
 * sampleattn.h — C ABI of the B200-native SampleAttention hot path.
 *
 * The reference (`blocksift`, pure Python/numpy) exposes the hot path as the
 * per-head body of run_pipeline (pkg/src/blocksift/pipeline.py:169-176):
 *
 *   sample_scores + block_reduce  -> sa_stage1          (stage 1, sampler.py:135-191)
 *   find_k + arg_topk             -> sa_select          (stage 2a, filtering.py:30-62, 245-255)
 *   merge_index                   -> sa_merge           (stage 2b, filtering.py:198-230)
 *   sparse_attention              -> sa_sparse_forward  (stage 3, executor.py:104-158)
 *
 * plus helpers the Python host layer needs (workspace sizing, the finite
 * check of core.py:30-37 / as_matrix, the LPT work order, a dense causal mask
 * for the dense comparison row).
 *
 * Conventions (all entry points):
 *   - plain device pointers and sizes; no framework types; the caller owns
 *     every buffer (inputs, outputs, workspace); the library never allocates
 *     device memory and never synchronises the stream;
 *   - q is [Hq][S][d], k and v are [Hkv][S][d], out is [Hq][S][d], all
 *     contiguous; q head h reads kv head (q_head0 + h)/group - q_head0/group
 *     (GQA/MQA: group = Hq_total / Hkv_total; q_head0 = global index of the
 *     first local q head, for head-sharded multi-GPU runs);
 *   - dtype: SA_BF16 (tensor-core path, d == 128 and blk == 128 only) or
 *     SA_FP32 (exact SIMT path, 1 <= d <= 128, 1 <= blk <= 128);
 *   - the return value is SA_OK or a negative status; sa_last_error() gives
 *     a thread-local message.  SA_ERR_INVALID / SA_ERR_UNSUPPORTED map to the
 *     reference's InputError (exceptions.py:4), SA_ERR_INTERNAL to
 *     InternalInvariantError (exceptions.py:16).
 *
 * Stage-1/2 block-score layout: col and slash are fp64 [Hq][cn][nb]
 * (nb = ceil(S/blk)), the ChunkScores.col_scores / slash_scores of
 * sampler.py:152-165.  Selections: k_out [Hq][cn][2] (k_c, k_s) and
 * idx_out [Hq][cn][2][nb] (ascending i_c, i_s — filtering.py:65-76).
 * Block mask (padded CSR): kv_cnt [Hq][nb] and kv_idx [Hq][nb*(nb+1)/2],
 * query block qb's ascending key blocks at kv_idx + h*nb*(nb+1)/2 + qb*(qb+1)/2
 * (BlockMask.active_for, filtering.py:128-130).
 */
#ifndef SAMPLEATTN_H_
#define SAMPLEATTN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SA_OK 0
#define SA_ERR_INVALID (-1)     /* bad argument (InputError) */
#define SA_ERR_UNSUPPORTED (-2) /* shape/dtype the kernels do not specialise (InputError) */
#define SA_ERR_INTERNAL (-3)    /* self-check failed (InternalInvariantError) */
#define SA_ERR_CUDA (-4)        /* CUDA launch / driver failure */

#define SA_BF16 0
#define SA_FP32 1

/* stage-1 precision modes */
#define SA_STAGE1_TENSOR 0 /* tcgen05 bf16 x bf16 -> fp32 (bf16 only) */
#define SA_STAGE1_EXACT 1  /* fp64 SIMT; bit-for-bit selection guard */

int sa_version(void);
const char* sa_last_error(void);
/* Number of kernels this library has launched in the calling process
 * (monotonic; the bench reports deltas as gpu_launches). */
long long sa_launch_count(void);

/* Device-side invariant status of the calling thread's current device,
 * accumulated by sa_sparse_forward since the last reset (synchronises the
 * device).  status4[0] is the OR of SA_STATUS_* bits, status4[1] / [2] the
 * head and query block of the first report, status4[3] the report count.
 * Replaces the executor's raises (executor.py:131-132 InputError for a query
 * block without active key blocks, :150-153 InternalInvariantError for an
 * empty normaliser) and the BlockMask invariants (filtering.py:97-106). */
#define SA_STATUS_EMPTY_BLOCK 1u  /* InputError */
#define SA_STATUS_MASK 2u         /* kb > qb, unsorted list or no diagonal: InternalInvariantError */
#define SA_STATUS_NORMALISER 4u   /* l <= 0 or not finite: InternalInvariantError */
int sa_status(unsigned* status4, int reset);

/* Bytes of scratch the stage-1/2/3 calls need for this geometry. */
size_t sa_workspace_bytes(int S, int Hq, int Hkv, int d, int blk, int chunk_n, int dtype);

/* Replaces the finite check of core.py:30-37 (as_matrix): *flag_dev is set
 * to 1 (never cleared) when any of the n elements is NaN or Inf. */
int sa_check_finite(const void* x, int dtype, int64_t n, int* flag_dev, void* stream);

/* Host-side helper of the host-buffer entry point: `height` rows of `width`
 * bytes from src (row pitch spitch) to dst (row pitch dpitch), host or device
 * pointers, stream-ordered (cudaMemcpy2DAsync).  Moves the sampled query
 * windows of every head in one copy engine transfer. */
int sa_copy2d_async(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                    void* stream);

/* Stage 1 — replaces sample_scores + block_reduce (sampler.py:135-191) for
 * every q head and every chunk of the plan (plan_chunks, sampler.py:88-118:
 * window i samples rows [max(0, (i+1)*itv - blk), (i+1)*itv)).
 * Writes col/slash [Hq][cn][nb] fp64.  mode: SA_STAGE1_TENSOR or
 * SA_STAGE1_EXACT.  When only_flags != NULL, only (h, c) pairs with
 * only_flags[h*cn + c] != 0 are (re)computed (the exact re-score of pairs
 * sa_select flagged as too close to call).  logit_bound (optional, tensor mode,
 * full calls only): [Hq][cn] doubles, max ||q_r|| * max ||k_j|| / sqrt(d) over
 * the pair's sampled rows and the KV head's keys -- the scale of the
 * tensor-core score error, which widens sa_select's guard margin. */
int sa_stage1(const void* q, const void* k, int dtype, int S, int Hq, int Hkv, int d, int blk,
              int group, int q_head0, int chunk_n, int itv, double* col, double* slash,
              double* logit_bound, int mode, const int* only_flags, void* workspace,
              size_t workspace_bytes, void* stream);

/* Stage 2a — replaces find_k + arg_topk per (head, chunk, direction)
 * (filtering.py:30-62, applied as in select_and_merge :245-255).
 * margin_eps > 0 enables the selection guard.  E = margin_eps *
 * max(1, logit_bound[hc] / bound_ref) * total is the error the tensor-core
 * scores of pair hc may carry (logit_bound from sa_stage1, may be NULL).
 * Guard pass (band != NULL or NULL, only_flags == NULL):
 *   - alpha cut within E of a decision (either side): flags[hc] = 1 (the
 *     pair needs its exact re-score);
 *   - only the boundary tie within E: the blocks whose scores lie within 2E
 *     of the k-th largest are recorded in band (sa_band_table_len ints: per
 *     (hc, dir) [count, first rank, tie a, tie b, block / bin indices]) for
 *     sa_refine_bands -- or flags[hc] = 1 when band is NULL or they are more
 *     than 512.
 * Certify pass (band != NULL and only_flags != NULL, after sa_refine_bands):
 * k is recomputed on the refined scores and flags[hc] = 1 unless the alpha
 * cut clears E on both sides and the two blocks at the cut differ by more
 * than band_eps * (scale) * (s_a + s_b) (both refined) or E (otherwise); two
 * refined blocks closer than that are left to sa_certify_band_ties.
 * only_flags != NULL recomputes the flagged pairs only.  k_in != NULL
 * ([Hq][cn][2]) skips find_k and takes the given k (the reference's
 * arg_topk(scores, k), filtering.py:51-62). */
int sa_select(const double* col, const double* slash, int Hq, int chunk_n, int nb,
              double alpha_c, double alpha_s, double margin_eps, const double* logit_bound,
              double bound_ref, int* flags, const int* only_flags, const int* k_in, int* k_out,
              int* idx_out, int* band, double band_eps, void* stream);

/* Selection guard, band refinement (no reference counterpart: it reproduces the
 * reference's fp64 ordering of the few nearly tied blocks at a cut).  For each
 * band recorded by sa_select whose pair is not flagged, the exact (fp64) mass
 * of every band block / bin over the pair's sampled rows is computed on the
 * FP64 tensor cores and normalised with stage 1's tensor-core row statistics
 * (row_stats, see sa_workspace_offset), and written over that block's col /
 * slash score; band_pairs[hc] = 1 marks the refined pairs (for the certifying
 * sa_select).  bf16 path only. */
int sa_band_table_len(int Hq, int chunk_n);
int sa_refine_bands(const void* q, const void* k, int dtype, int S, int Hq, int Hkv, int d, int blk, int group,
                    int q_head0, int chunk_n, int itv, const int* band, const int* flags, int* band_pairs,
                    const double* row_stats, double* col, double* slash, void* workspace, size_t workspace_bytes,
                    void* stream);

/* Selection guard, band refinement, last step (after the certifying
 * sa_select): when the two refined blocks a, b at a certified cut differ by no
 * more than band_eps * scale * (s_a + s_b), the certify pass leaves them in the
 * band entry and this call settles their order per row instead: row r's
 * normaliser error scales both blocks' masses x_ra, x_rb alike, so the refined
 * gap s_a - s_b is trusted when it exceeds band_eps * scale * sum_r |x_ra -
 * x_rb| (scale = max(1, logit_bound[hc] / bound_ref)); else flags[hc] = 1 (the
 * pair joins the exact re-score).  Reads the exact partials sa_refine_bands
 * left in the workspace.  bf16 path only. */
int sa_certify_band_ties(int dtype, int S, int Hq, int Hkv, int d, int blk, int chunk_n, int itv, const int* band,
                         int* flags, const double* row_stats, const double* col, const double* slash,
                         const double* logit_bound, double bound_ref, double band_eps, void* workspace,
                         size_t workspace_bytes, void* stream);

/* Byte offset of a workspace region of this geometry (< 0 on bad args).
 * SA_WS_ROW_STATS: stage 1's per-sampled-row statistics, double
 * [Hq*chunk_n*blk][2] (log2 max, sum) after a tensor-mode sa_stage1 -- copy
 * them out to keep them for sa_refine_bands's row_stats, since later stage-1
 * calls of the same geometry reuse the workspace. */
#define SA_WS_ROW_STATS 0
long long sa_workspace_offset(int S, int Hq, int Hkv, int d, int blk, int chunk_n, int dtype, int region);

/* Stage 2b — replaces merge_index (filtering.py:198-230): extends every
 * chunk's picks over its query region, unions straddling blocks, forces the
 * diagonal.  Writes the padded CSR and, when non-NULL, per-head totals:
 * active_blocks[Hq] (BlockMask.active_count, filtering.py:118-119) and
 * active_entries[Hq] (active_causal_entries, filtering.py:148-164).
 * sink_blocks / local_blocks: optional forced key blocks [0, sink_blocks) and
 * [qb - local_blocks + 1, qb] for every query block; the defaults (0, 1)
 * reproduce the reference exactly (only the diagonal is forced). */
int sa_merge(const int* k_sel, const int* idx_sel, int Hq, int chunk_n, int nb, int S, int blk,
             int itv, int sink_blocks, int local_blocks, int* kv_cnt, int* kv_idx,
             long long* active_blocks, long long* active_entries, void* stream);

/* Sampled-row CRA — replaces _retained_by_block over the sampled rows
 * (pipeline.py:37-58, the reference's cra_sampled) from the partials the last
 * sa_stage1 call of this geometry left in `workspace`: retained[hc*blk + r] is
 * the normalised probability mass sampled row r of pair hc (= h*cn + c) keeps
 * inside the mask (kv_cnt / kv_idx, sa_merge's layout); NaN past the window.
 * mode is the mode of that stage-1 call; rescored_flags (sa_select's guard
 * flags, may be NULL) marks pairs whose exact re-score replaced the tensor
 * partials. */
int sa_sampled_retained(int dtype, int S, int Hq, int Hkv, int d, int blk, int chunk_n, int itv, int mode,
                        const int* rescored_flags, const int* kv_cnt, const int* kv_idx,
                        const void* workspace, size_t workspace_bytes, double* retained, void* stream);

/* Full causal block mask (every kb <= qb): the dense-attention comparison row. */
int sa_full_mask(int Hq, int nb, int* kv_cnt, int* kv_idx, void* stream);

/* Stage-3 work units.  A unit is two (head, query block) items that read the
 * same KV head (two q heads of one GQA group at the same query block, or
 * adjacent query blocks of a group's odd head out), run by one CTA that loads
 * each K/V tile of the union of their block lists once.  sa_schedule writes
 * order[2*u], order[2*u+1] = h*nb + qb of unit u's items (-1: no partner),
 * grouped by KV head (one KV head's K/V stays L2-resident while its units run)
 * and longest-first (descending kv_cnt[a] + kv_cnt[b]) inside a group.
 * With kv_idx and scratch (sa_schedule_len ints) the q heads of a group are
 * paired per query block by list overlap (fewest key blocks listed by only one
 * of the two); with either NULL they pair as (h, h+1).
 * sa_schedule_len returns the entry count 2 * n_units (or < 0 on bad args). */
int sa_schedule_len(int Hq, int nb, int group, int q_head0);
int sa_schedule(const int* kv_cnt, const int* kv_idx, int Hq, int nb, int group, int q_head0, int* order,
                int* scratch, void* stream);

/* Stage 3 — replaces sparse_attention (executor.py:104-158): per (head,
 * query block) the online-softmax recurrence over the mask's ascending key
 * blocks, entry-level causality inside the diagonal block.  out is
 * [Hq][S][d] in the input dtype; lse [Hq][S] fp32 (natural log) and
 * touched[Hq] (blocks processed, FlopReport.active_blocks) are optional.
 * order is sa_schedule's unit list (sa_schedule_len entries) or NULL
 * (natural unit order). */
int sa_sparse_forward(const void* q, const void* k, const void* v, int dtype, int S, int Hq,
                      int Hkv, int d, int blk, int group, int q_head0, const int* kv_cnt,
                      const int* kv_idx, const int* order, void* out, float* lse,
                      long long* touched, void* stream);

/* Stage 3 with the output gather fused into its epilogue (the 1M-token
 * configuration, heads sharded over GPUs; replaces sa_sparse_forward followed
 * by an all-gather of the per-rank outputs, ref pipeline.py:169-176 loops the
 * heads of one process).  Same arguments and result as sa_sparse_forward
 * (bf16 only); in addition every output row is stored, as soon as its tile
 * finishes, into the n_peer buffers peer_out[0..n_peer) -- device pointers
 * (peer-mapped through sa_ipc_open) to the same [Hq][S][d] rows of the other
 * ranks' gather buffers -- so the NVLink transfer overlaps the attention tile
 * by tile.  peer_out is a HOST array; n_peer <= SA_MAX_PEERS.  Completion on a
 * peer is the caller's to signal (stream sync + barrier). */
#define SA_MAX_PEERS 7
int sa_sparse_forward_peers(const void* q, const void* k, const void* v, int dtype, int S, int Hq,
                            int Hkv, int d, int blk, int group, int q_head0, const int* kv_cnt,
                            const int* kv_idx, const int* order, void* out, float* lse,
                            long long* touched, void* const* peer_out, int n_peer, void* stream);

/* CUDA IPC of a gather buffer between the ranks of one node.  sa_ipc_export
 * writes the 64-byte handle of the allocation holding ptr and ptr's byte
 * offset inside it; a peer process passes both to sa_ipc_open, adds the
 * offset to the returned base, and closes the base with sa_ipc_close. */
#define SA_IPC_HANDLE_BYTES 64
int sa_ipc_export(const void* ptr, void* handle, unsigned long long* offset);
int sa_ipc_open(const void* handle, void** base);
int sa_ipc_close(void* base);

#ifdef __cplusplus
}
#endif
#endif /* SAMPLEATTN_H_ */
