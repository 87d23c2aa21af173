"""Block masks and selection provenance.

Mirrors the reference's BlockMask / ChunkSelection / SelectedIndices
(pkg/src/blocksift/filtering.py:65-195) with a device-resident layout: a
batch of H per-head masks stored as a padded CSR (kv_cnt [H, nb] and
kv_idx [H, nb*(nb+1)/2]; query block qb's ascending key blocks start at
qb*(qb+1)/2).  Host views (dense grid, BLOCKMASK v1 text, provenance tuples)
are produced on demand and cached.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import InputError
from .heads import dcall

__all__ = ["ChunkSelection", "SelectedIndices", "BlockMask"]


@dataclass(frozen=True)
class ChunkSelection:
    """Block indices one chunk picked, per direction (filtering.py:65-76)."""

    i_c: tuple
    i_s: tuple
    k_c: int
    k_s: int

    def __post_init__(self):
        if len(self.i_c) != self.k_c or len(self.i_s) != self.k_s:
            raise InputError("selection sizes disagree with k_c/k_s")


@dataclass(frozen=True)
class SelectedIndices:
    chunks: tuple


def _tri(n: int) -> int:
    return n * (n + 1) // 2


class BlockMask:
    """H heads' block-level masks over the (query block x key block) grid.

    Invariants (filtering.py:97-108) hold by construction for masks built by
    sa_merge / sa_full_mask and are checked for user-supplied grids:
    kb <= qb and every query block keeps its diagonal.  Single-head masks
    expose the reference's per-head API (active_for, serialize, provenance...).
    """

    def __init__(self, blk: int, S: int, kv_cnt: torch.Tensor, kv_idx: torch.Tensor,
                 k_sel: torch.Tensor | None = None, idx_sel: torch.Tensor | None = None,
                 active_blocks: torch.Tensor | None = None, active_entries: torch.Tensor | None = None):
        self.blk, self.S = int(blk), int(S)
        self.kv_cnt, self.kv_idx = kv_cnt, kv_idx
        self.k_sel, self.idx_sel = k_sel, idx_sel
        self._active_blocks, self._active_entries = active_blocks, active_entries
        self._order = None
        self._host = None

    # ------------------------------------------------------------ geometry
    @property
    def n_heads(self) -> int:
        return int(self.kv_cnt.shape[0])

    @property
    def n_qblocks(self) -> int:
        return int(self.kv_cnt.shape[1])

    @property
    def n_kblocks(self) -> int:
        return self.n_qblocks

    @property
    def device(self):
        return self.kv_cnt.device

    def head(self, h: int) -> "BlockMask":
        return self.heads(h, h + 1)

    def heads(self, h0: int, h1: int) -> "BlockMask":
        """The mask of heads [h0, h1) (views of the same device arrays)."""
        sl = slice(h0, h1)
        return BlockMask(self.blk, self.S, self.kv_cnt[sl], self.kv_idx[sl],
                         None if self.k_sel is None else self.k_sel[sl],
                         None if self.idx_sel is None else self.idx_sel[sl],
                         None if self._active_blocks is None else self._active_blocks[sl],
                         None if self._active_entries is None else self._active_entries[sl])

    # ------------------------------------------------------------ counts
    def active_counts(self) -> np.ndarray:
        """Active blocks per head (int64 [H])."""
        if self._active_blocks is not None:
            return self._active_blocks.cpu().numpy()
        return self.kv_cnt.sum(dim=1, dtype=torch.int64).cpu().numpy()

    def active_count(self) -> int:
        return int(self.active_counts().sum())

    def causal_count(self) -> int:
        nb = self.n_qblocks
        return nb * (nb + 1) // 2

    def block_density(self) -> float:
        """Per-head density for single-head masks, mean over heads otherwise
        (filtering.py:125-126)."""
        return float(self.active_counts().mean() / self.causal_count())

    def block_densities(self) -> np.ndarray:
        return self.active_counts() / self.causal_count()

    def active_causal_entries(self, S: int | None = None) -> int:
        """Exact token-level causal entries kept (filtering.py:148-164), summed over heads."""
        S = self.S if S is None else S
        if -(-S // self.blk) != self.n_qblocks:
            raise InputError(f"mask has {self.n_qblocks} blocks of {self.blk}, cannot cover S={S}")
        if self._active_entries is not None and S == self.S:
            return int(self._active_entries.sum().item())
        cnt = self.kv_cnt.to(torch.int64)
        nb, blk = self.n_qblocks, self.blk
        m = torch.clamp(S - torch.arange(nb, device=cnt.device, dtype=torch.int64) * blk, max=blk)
        ent = (cnt - 1) * m * blk + m * (m + 1) // 2
        return int(ent.sum().item())

    # ------------------------------------------------------------ host views
    def _host_csr(self):
        """(kv_cnt, kv_idx) on the host.  Only the first kv_cnt entries of each
        row segment are copied (a device gather); the capacity tail, which the
        merge never writes, reads back as -1."""
        if self._host is None:
            cnt = self.kv_cnt
            nb, dev = self.n_qblocks, cnt.device
            ar = torch.arange(nb, device=dev)
            seg = torch.repeat_interleave(ar, ar + 1)                  # row of each slot
            off = torch.arange(seg.numel(), device=dev) - seg * (seg + 1) // 2
            valid = off[None, :] < cnt[:, seg]                          # [H, tri(nb)]
            idx = np.full(tuple(self.kv_idx.shape), -1, dtype=np.int32)
            idx[valid.cpu().numpy()] = self.kv_idx[valid].cpu().numpy()
            self._host = (cnt.cpu().numpy(), idx)
        return self._host

    def _single(self):
        if self.n_heads != 1:
            raise InputError("this view needs a single-head mask; use .head(h)")

    def active_for(self, qb: int) -> np.ndarray:
        """Ascending active key blocks of query block qb (filtering.py:128-130)."""
        self._single()
        cnt, idx = self._host_csr()
        o = _tri(qb)
        return idx[0, o: o + int(cnt[0, qb])].astype(np.int64)

    @property
    def active(self) -> np.ndarray:
        """Dense bool grid [nb, nb] (single head) as in the reference."""
        self._single()
        return self.to_dense()[0]

    def to_dense(self) -> np.ndarray:
        cnt, idx = self._host_csr()
        H, nb = cnt.shape
        grid = np.zeros((H, nb, nb), dtype=bool)
        for h in range(H):
            for qb in range(nb):
                o = _tri(qb)
                grid[h, qb, idx[h, o: o + cnt[h, qb]]] = True
        return grid

    def serialize(self) -> str:
        """BLOCKMASK v1 text (filtering.py:166-172)."""
        self._single()
        nb = self.n_qblocks
        lines = [f"BLOCKMASK v1 {nb} {nb} {self.blk}"]
        lines += [" ".join(str(int(kb)) for kb in self.active_for(qb)) for qb in range(nb)]
        return "\n".join(lines) + "\n"

    @property
    def provenance(self) -> SelectedIndices | None:
        self._single()
        sel = self.selections()
        return None if sel is None else sel[0]

    def selections(self):
        """Per-head SelectedIndices (k_c, k_s, ascending i_c, i_s per chunk)."""
        if self.k_sel is None:
            return None
        ks = self.k_sel.cpu().numpy()
        valid = torch.arange(self.idx_sel.shape[-1], device=self.k_sel.device) < self.k_sel[..., None]
        ix = np.full(tuple(self.idx_sel.shape), -1, dtype=np.int32)  # only the first k entries are written
        ix[valid.cpu().numpy()] = self.idx_sel[valid].cpu().numpy()
        out = []
        for h in range(ks.shape[0]):
            chunks = []
            for c in range(ks.shape[1]):
                kc, kss = int(ks[h, c, 0]), int(ks[h, c, 1])
                chunks.append(ChunkSelection(tuple(int(x) for x in ix[h, c, 0, :kc]),
                                             tuple(int(x) for x in ix[h, c, 1, :kss]), kc, kss))
            out.append(SelectedIndices(tuple(chunks)))
        return out

    # ------------------------------------------------------------ builders
    @classmethod
    def from_dense(cls, blk: int, active, S: int | None = None, device=None) -> "BlockMask":
        """Upload a bool grid [nb, nb] (or [H, nb, nb]) after the reference's
        invariant checks (filtering.py:97-108)."""
        a = np.asarray(active, dtype=bool)
        if a.ndim == 2:
            a = a[None]
        if a.ndim != 3 or a.shape[1] != a.shape[2]:
            raise InputError(f"block grid must be square, got shape {a.shape}")
        if blk < 1:
            raise InputError(f"blk must be >= 1, got {blk}")
        H, nb, _ = a.shape
        if np.triu(a, 1).any():
            raise InputError("block mask violates block-level causality (kb > qb)")
        if not a[:, np.arange(nb), np.arange(nb)].all():
            raise InputError("every query block must keep its diagonal block")
        S = nb * blk if S is None else S
        if -(-S // blk) != nb:
            raise InputError(f"mask has {nb} blocks of {blk}, cannot cover S={S}")
        cnt = a.sum(axis=2).astype(np.int32)
        idx = np.zeros((H, _tri(nb)), dtype=np.int32)
        for h in range(H):
            for qb in range(nb):
                sel = np.flatnonzero(a[h, qb])
                idx[h, _tri(qb): _tri(qb) + sel.size] = sel
        device = torch.device(device or "cuda")
        return cls(blk, S, torch.from_numpy(cnt).to(device), torch.from_numpy(idx).to(device))

    @classmethod
    def deserialize(cls, text: str, S: int | None = None, device=None) -> "BlockMask":
        """Parse BLOCKMASK v1 (filtering.py:174-195)."""
        lines = text.splitlines()
        if not lines:
            raise InputError("empty block mask document")
        head = lines[0].split()
        if len(head) != 5 or head[0] != "BLOCKMASK" or head[1] != "v1":
            raise InputError(f"bad block mask header: {lines[0]!r}")
        try:
            nq, nk, blk = int(head[2]), int(head[3]), int(head[4])
        except ValueError as e:
            raise InputError(f"bad block mask header: {lines[0]!r}") from e
        if len(lines) < nq + 1:
            raise InputError(f"expected {nq} query block lines, got {len(lines) - 1}")
        grid = np.zeros((nq, nk), dtype=bool)
        for qb in range(nq):
            for tok in lines[1 + qb].split():
                kb = int(tok)
                if not 0 <= kb < nk:
                    raise InputError(f"key block {kb} out of range on line {qb + 2}")
                grid[qb, kb] = True
        return cls.from_dense(blk, grid, S=S, device=device)

    @classmethod
    def full(cls, n_heads: int, S: int, blk: int, device=None) -> "BlockMask":
        """Every causal block (the dense comparison row), built on the device."""
        device = torch.device(device or "cuda")
        nb = -(-S // blk)
        cnt = torch.empty((n_heads, nb), dtype=torch.int32, device=device)
        idx = torch.empty((n_heads, _tri(nb)), dtype=torch.int32, device=device)
        dcall(device, "sa_full_mask", n_heads, nb, cnt.data_ptr(), idx.data_ptr(),
              torch.cuda.current_stream(device).cuda_stream)
        return cls(blk, S, cnt, idx)

    # ------------------------------------------------------------ scheduling
    def order(self, group: int = 1, q_head0: int = 0) -> torch.Tensor:
        """Stage-3 work units (sa_schedule): pairs of items sharing a KV head
        (q heads matched per query block by list overlap), KV-group-major and
        longest-first; cached per (group, q_head0)."""
        key = (group, q_head0)
        if self._order is None or self._order[0] != key:
            nb = self.n_qblocks
            n = _lib.load().sa_schedule_len(self.n_heads, nb, group, q_head0)
            if n < 0:
                raise InputError(f"bad schedule geometry (heads {self.n_heads}, group {group}, q_head0 {q_head0})")
            order = torch.empty(n, dtype=torch.int32, device=self.device)
            scratch = torch.empty(n, dtype=torch.int32, device=self.device)  # the overlap pairing
            dcall(self.device, "sa_schedule", self.kv_cnt.data_ptr(), self.kv_idx.data_ptr(), self.n_heads, nb,
                  group, q_head0, order.data_ptr(), scratch.data_ptr(),
                  torch.cuda.current_stream(self.device).cuda_stream)
            self._order = (key, order)
        return self._order[1]
