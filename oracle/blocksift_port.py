"""CPU oracle: a numpy restatement of the reference's SampleAttention hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_2406_15486_b200/`) imports this module; only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU-baseline / `--impl reference`
legs use it, and only as the checker or as the timed CPU baseline.

It restates, in fp64 numpy, the per-head body of the reference's
`run_pipeline` (`pkg/src/blocksift/pipeline.py:169-176`):

    plan_chunks -> sample_scores -> block_reduce -> select_and_merge -> sparse_attention

Every function cites the reference file:line it follows ("ref" below means
`/root/reference/pkg/src/blocksift/`).  The restatement is pinned against the
reference's own outputs by `tests/golden/make_golden.py` (fixtures in
`tests/golden/*.npz`, checked by `tests/test_oracle_golden.py`).

Data model: plain numpy arrays instead of the reference's frozen dataclasses.
A "head" is a (q, k, v) triple of [S, d] arrays; a plan is a `Plan` tuple; a
selection is a list of (i_c, i_s) tuples per chunk; a mask is a dense
[nb, nb] bool array.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np

__all__ = [
    "Plan",
    "n_blocks",
    "plan_chunks",
    "sampled_probs",
    "block_reduce",
    "find_k",
    "arg_topk",
    "select",
    "merge_index",
    "select_and_merge",
    "sparse_attention",
    "dense_causal_attention",
    "flop_accounting",
    "serialize_mask",
    "sampled_cra",
    "run_head",
    "block_scores",
]


def n_blocks(s: int, blk: int) -> int:
    """ceil(s / blk); ref sampler.py:33-35."""
    return (s + blk - 1) // blk


class Plan(NamedTuple):
    """ChunkPlan (ref sampler.py:69-85) as plain tuples.

    windows[i] = (sample_start, sample_end, region_start, region_end)."""

    S: int
    blk: int
    requested_chunk_n: int
    chunk_n: int
    itv: int
    windows: tuple

    def sampled_rows(self) -> int:
        return sum(b - a for a, b, _, _ in self.windows)


def plan_chunks(S: int, chunk_n: int, blk: int) -> Plan:
    """Window layout; ref sampler.py:88-118.

    S < blk: one window covering [0, S).  Otherwise itv = S // chunk_n; when a
    segment would be shorter than blk the chunk count clamps to max(1, S//blk).
    Window i (1-based) samples [i*itv - blk, i*itv) and governs
    [(i-1)*itv, i*itv), the last region running to S.
    """
    if S < 1:
        raise ValueError("S must be >= 1")
    if S < blk:
        cn, itv = 1, S
    else:
        cn = chunk_n
        itv = S // cn
        if itv < blk:
            cn = max(1, S // blk)
            itv = S // cn
    wins = []
    for i in range(1, cn + 1):
        end = i * itv
        wins.append((max(0, end - blk), end, (i - 1) * itv, S if i == cn else end))
    return Plan(S, blk, chunk_n, cn, itv, tuple(wins))


def _scores(q_rows: np.ndarray, k: np.ndarray) -> np.ndarray:
    """(q k^T) / sqrt(d) in fp64; ref core.py:110-122."""
    d = k.shape[1]
    return (np.asarray(q_rows, np.float64) @ np.asarray(k, np.float64).T) / np.sqrt(d)


def _causal_softmax(s: np.ndarray, rows: np.ndarray) -> np.ndarray:
    """Row softmax over keys j <= row (global index), zeros elsewhere;
    ref core.py:125-154 (max-subtract, exp, divide by the row sum)."""
    m = s.shape[1]
    keep = np.arange(m)[None, :] <= rows[:, None]
    z = np.where(keep, s, -np.inf)
    z = np.exp(z - z.max(axis=1, keepdims=True))
    return z / z.sum(axis=1, keepdims=True)


def sampled_probs(q: np.ndarray, k: np.ndarray, plan: Plan) -> list:
    """Exact probability rows of every sampled window; ref sampler.py:135-149.

    Returns a list of (rows, probs[n_rows, S]) per chunk."""
    out = []
    for a, b, _, _ in plan.windows:
        rows = np.arange(a, b)
        out.append((rows, _causal_softmax(_scores(q[a:b], k), rows)))
    return out


def block_reduce(samples: list, S: int, blk: int):
    """Per-chunk column-block and slash-block mass; ref sampler.py:168-191.

    col[b]   = sum of p[r, j] over sampled rows r and keys j in block b.
    slash[o] = sum of p[r, j] over (r - j) // blk == o; acausal entries
               (p == 0 exactly) are routed to bin 0 (ref sampler.py:186-189).
    Returns lists col[c], slash[c] (fp64 arrays of length nb) and totals.
    """
    nb = n_blocks(S, blk)
    key = np.arange(S)
    cols, slashes, totals = [], [], []
    for rows, p in samples:
        col = np.add.reduceat(p.sum(axis=0), np.arange(0, S, blk))
        off = np.clip((rows[:, None] - key[None, :]) // blk, 0, nb - 1)
        slash = np.bincount(off.ravel(), weights=p.ravel(), minlength=nb)
        cols.append(col)
        slashes.append(slash)
        totals.append(float(p.sum()))
    return cols, slashes, totals


def find_k(scores, alpha: float) -> int:
    """Minimal quota; ref filtering.py:30-48.

    Descending sort, sequential fp64 cumsum, target = alpha * cum[-1];
    target <= 0 -> 0; else first index with cum >= target, plus one."""
    s = np.asarray(scores, dtype=np.float64)
    if not 0.0 <= alpha <= 1.0:
        raise ValueError("alpha out of range")
    if s.ndim != 1 or s.size == 0 or (s < 0).any():
        raise ValueError("scores must be a nonempty nonnegative 1-D vector")
    cum = np.cumsum(-np.sort(-s))
    target = alpha * cum[-1]
    if target <= 0.0:
        return 0
    return int(np.searchsorted(cum, target, side="left")) + 1


def arg_topk(scores, k: int) -> tuple:
    """k largest, ties toward the lower index, returned ascending;
    ref filtering.py:51-62 (stable argsort of -s)."""
    s = np.asarray(scores, dtype=np.float64)
    if not 0 <= k <= s.size:
        raise ValueError("k out of range")
    if k == 0:
        return ()
    idx = np.argsort(-s, kind="stable")[:k]
    return tuple(int(i) for i in np.sort(idx))


def select(cols: list, slashes: list, alpha_c: float, alpha_s: float) -> list:
    """Per-chunk (i_c, i_s) picks; ref filtering.py:245-255."""
    out = []
    for col, slash in zip(cols, slashes):
        out.append((arg_topk(col, find_k(col, alpha_c)), arg_topk(slash, find_k(slash, alpha_s))))
    return out


def merge_index(selection: list, plan: Plan) -> np.ndarray:
    """Dense [nb, nb] bool block mask; ref filtering.py:198-230.

    For every chunk and every query block qb its region touches
    ([region_start // blk, (region_end - 1) // blk]): column picks kb <= qb,
    slash picks ob -> key blocks {qb-ob-1, qb-ob} clipped to [0, qb], and the
    diagonal.  Straddling query blocks take the union; the whole diagonal is
    forced at the end (ref filtering.py:229)."""
    blk, S = plan.blk, plan.S
    nb = n_blocks(S, blk)
    grid = np.zeros((nb, nb), dtype=bool)
    for (i_c, i_s), (_, _, r0, r1) in zip(selection, plan.windows):
        qbs = np.arange(r0 // blk, (r1 - 1) // blk + 1)
        ic = np.asarray(i_c, dtype=np.int64)
        for qb in qbs:
            grid[qb, ic[ic <= qb]] = True
            for ob in i_s:
                for kb in (qb - ob - 1, qb - ob):
                    if 0 <= kb <= qb:
                        grid[qb, kb] = True
    grid[np.arange(nb), np.arange(nb)] = True
    return grid


def select_and_merge(cols, slashes, plan: Plan, alpha_c: float, alpha_s: float):
    """ref filtering.py:233-256; returns (selection, grid)."""
    sel = select(cols, slashes, alpha_c, alpha_s)
    return sel, merge_index(sel, plan)


def sparse_attention(q, k, v, grid: np.ndarray, blk: int, qblocks=None):
    """Block-sparse causal attention with the online softmax recurrence;
    ref executor.py:104-158.  Per query block, active key blocks ascend;
    entry-level causality only inside the diagonal block; the logits are
    (q * (1/sqrt(d))) @ k^T as in ref executor.py:124,133,139.
    qblocks: optional subset of query blocks to compute (the recurrence is
    per query block, so a subset is exactly those rows of the full result;
    other rows are NaN) -- for bounded CPU samples at full scale.
    Returns (out[S, d] fp64, touched_blocks)."""
    q = np.asarray(q, np.float64)
    k = np.asarray(k, np.float64)
    v = np.asarray(v, np.float64)
    S, d = q.shape
    nb = n_blocks(S, blk)
    scale = 1.0 / np.sqrt(d)
    out = np.full((S, d), np.nan) if qblocks is not None else np.empty((S, d))
    touched = 0
    for qb in (range(nb) if qblocks is None else sorted(qblocks)):
        a, b = qb * blk, min((qb + 1) * blk, S)
        qs = q[a:b] * scale
        m = np.full(b - a, -np.inf)
        l = np.zeros(b - a)
        acc = np.zeros((b - a, d))
        for kb in np.flatnonzero(grid[qb]):
            c0, c1 = kb * blk, min((kb + 1) * blk, S)
            z = qs @ k[c0:c1].T
            if kb == qb:
                z[np.arange(c0, c1)[None, :] > np.arange(a, b)[:, None]] = -np.inf
            m_new = np.maximum(m, z.max(axis=1))
            corr = np.exp(m - m_new)
            pz = np.exp(z - m_new[:, None])
            l = corr * l + pz.sum(axis=1)
            acc = acc * corr[:, None] + pz @ v[c0:c1]
            m = m_new
            touched += 1
        if not np.all(l > 0.0):
            raise AssertionError(f"empty normaliser in query block {qb}")
        out[a:b] = acc / l[:, None]
    return out, touched


def dense_causal_attention(q, k, v, row_block: int = 512) -> np.ndarray:
    """fp64 dense causal attention in row blocks; ref core.py:157-172."""
    q = np.asarray(q, np.float64)
    S, d = q.shape
    out = np.empty((S, d))
    for a in range(0, S, row_block):
        b = min(a + row_block, S)
        p = _causal_softmax(_scores(q[a:b], k), np.arange(a, b))
        out[a:b] = p @ np.asarray(v, np.float64)
    return out


def flop_accounting(grid: np.ndarray, S: int, d: int, blk: int) -> dict:
    """ref executor.py:51-73: 4*d*sum(m*n) over active / causal block pairs,
    trailing partial blocks pro-rated by true size."""
    nb = n_blocks(S, blk)
    sizes = np.minimum(blk, S - np.arange(nb) * blk).astype(np.int64)
    area = sizes[:, None] * sizes[None, :]
    causal = np.tril(np.ones((nb, nb), dtype=bool))
    active = int(grid.sum())
    return {
        "active_blocks": active,
        "causal_blocks": nb * (nb + 1) // 2,
        "block_density": active / (nb * (nb + 1) // 2),
        "estimated_flops_sparse": 4 * d * int(area[grid].sum()),
        "estimated_flops_dense": 4 * d * int(area[causal].sum()),
    }


def serialize_mask(grid: np.ndarray, blk: int) -> str:
    """BLOCKMASK v1 text; ref filtering.py:166-172."""
    nb = grid.shape[0]
    lines = [f"BLOCKMASK v1 {nb} {grid.shape[1]} {blk}"]
    lines += [" ".join(str(int(x)) for x in np.flatnonzero(grid[qb])) for qb in range(nb)]
    return "\n".join(lines) + "\n"


def sampled_cra(samples: list, grid: np.ndarray, S: int, blk: int):
    """(min, mean) retained mass over sampled rows; ref pipeline.py:37-58."""
    kept = []
    for rows, p in samples:
        bsum = np.add.reduceat(p, np.arange(0, S, blk), axis=1)
        kept.append((bsum * grid[rows // blk]).sum(axis=1))
    kept = np.concatenate(kept)
    return float(kept.min()), float(kept.mean())


def run_head(q, k, v, alpha_c: float, alpha_s: float, chunk_n: int, blk: int = 128,
             with_output: bool = True) -> dict:
    """One head through stage 1 -> 2 -> 3 (ref pipeline.py:169-176)."""
    S = q.shape[0]
    plan = plan_chunks(S, chunk_n, blk)
    samples = sampled_probs(q, k, plan)
    cols, slashes, totals = block_reduce(samples, S, blk)
    sel, grid = select_and_merge(cols, slashes, plan, alpha_c, alpha_s)
    res = {"plan": plan, "cols": cols, "slashes": slashes, "totals": totals,
           "selection": sel, "grid": grid}
    if with_output:
        out, touched = sparse_attention(q, k, v, grid, blk)
        res["out"] = out
        res["touched"] = touched
    return res


def block_scores(q, k, plan: Plan, blk: int, workers: int | None = None):
    """sampled_probs + block_reduce window by window, windows in parallel
    threads (numpy releases the GIL), each window's probability rows freed
    once reduced: the same arithmetic as the two functions above (same
    per-window code, so the same fp64 results), with memory bounded by
    `workers` windows instead of all of them (ref sampler.py:135-191 keeps
    every [rows x S] window alive; at 96K and 77 windows that is 7.7 GB).
    Returns (cols, slashes, totals) like block_reduce."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    S = q.shape[0]
    q = np.asarray(q, np.float64)
    k = np.asarray(k, np.float64)

    def one(w):
        a, b, _, _ = w
        rows = np.arange(a, b)
        cols, slashes, totals = block_reduce([(rows, _causal_softmax(_scores(q[a:b], k), rows))], S, blk)
        return cols[0], slashes[0], totals[0]

    n = workers or min(16, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else 4)
    with ThreadPoolExecutor(max_workers=max(1, n)) as ex:
        res = list(ex.map(one, plan.windows))
    return [r[0] for r in res], [r[1] for r in res], [r[2] for r in res]
