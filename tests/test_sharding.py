"""Multi-GPU head sharding, exercised on CPU: the partition / GQA mapping and
the chunked all-gather of sample_attention_sharded, with world_size 2 over
gloo and the CPU oracle standing in for the kernels (test infrastructure)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import blocksift_port as O
from paper_2406_15486_b200.parallel import sample_attention_sharded, shard_heads
from paper_2406_15486_b200.errors import InputError


def test_shard_partition_and_gqa_mapping():
    for Hq, Hkv, world in [(32, 2, 8), (32, 8, 8), (32, 2, 4), (4, 4, 2), (32, 32, 2)]:
        seen = []
        for r in range(world):
            s = shard_heads(Hq, Hkv, world, r)
            seen += list(s.q_heads)
            for h in s.q_heads:
                # the C ABI mapping (q_head0 + h_local)/group - q_head0/group names the right kv head
                h_local = h - s.q_head0
                kv_local = (s.q_head0 + h_local) // s.group - s.q_head0 // s.group
                assert s.kv_heads[kv_local] == h // (Hq // Hkv)
                assert s.local_kv(h) == kv_local
        assert seen == list(range(Hq))
    with pytest.raises(InputError):
        shard_heads(32, 2, 3, 0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(Hq, Hkv, S, d, seed=0):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((Hq, S, d)) * 1.5
    k = rng.standard_normal((Hkv, S, d)) * 1.5
    v = rng.standard_normal((Hkv, S, d))
    return q, k, v


def _oracle_compute(q, k, v, q_head0, group, out, alpha=0.9, chunk_n=2):
    for h in range(q.shape[0]):
        kv = (q_head0 + h) // group - q_head0 // group
        r = O.run_head(q[h].numpy(), k[kv].numpy(), v[kv].numpy(), alpha, alpha, chunk_n, 32)
        out[h] = torch.from_numpy(r["out"])


def _worker(rank, world, port, Hq, Hkv, S, d, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q, k, v = _inputs(Hq, Hkv, S, d)
    shard = shard_heads(Hq, Hkv, world, rank)
    ql = torch.from_numpy(q[list(shard.q_heads)])
    kl = torch.from_numpy(k[list(shard.kv_heads)])
    vl = torch.from_numpy(v[list(shard.kv_heads)])
    _, full = sample_attention_sharded(ql, kl, vl, shard, heads_per_chunk=1, compute_fn=_oracle_compute)
    if rank == 0:
        results.put(full.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("Hq,Hkv", [(4, 2), (4, 1)])
def test_sharded_gather_matches_single_process(Hq, Hkv):
    S, d, world = 256, 16, 2
    ctx = mp.get_context("spawn")
    results = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, Hq, Hkv, S, d, results)) for r in range(world)]
    for p in procs:
        p.start()
    full = results.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    q, k, v = _inputs(Hq, Hkv, S, d)
    group = Hq // Hkv
    for h in range(Hq):
        want = O.run_head(q[h], k[h // group], v[h // group], 0.9, 0.9, 2, 32)["out"]
        np.testing.assert_allclose(full[h], want, rtol=0, atol=1e-12)


def test_p2p_transport_needs_cuda_tensors():
    """The fused p2p gather maps CUDA allocations; CPU tensors must ask for the
    collective transport (the default picks it for them)."""
    shard = shard_heads(4, 2, 2, 0)
    q = torch.zeros((2, 64, 8))
    k = torch.zeros((1, 64, 8))
    with pytest.raises(InputError):
        sample_attention_sharded(q, k, k, shard, transport="p2p", compute_fn=lambda *a, **kw: None)
    with pytest.raises(InputError):
        sample_attention_sharded(q, k, k, shard, transport="nvshmem", compute_fn=lambda *a, **kw: None)
