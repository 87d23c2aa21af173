"""The output gather fused into stage 3 (sample_attention_sharded, transport
"p2p"): ranks map each other's gather buffers through CUDA IPC and the K3
epilogue stores every output row into all of them (sa_sparse_forward_peers).

This box has one GPU, so two processes share it: each owns half the q heads,
writes its rows into both buffers, and after the call each buffer must equal
the single-process result for every head, bit for bit (the per-head kernels
and their arithmetic are the same; only the destination list differs).  The
ranks never wait on each other's kernels, only on a host barrier at the end.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

S, HQ, HKV, ALPHA = 8192, 4, 2, 0.95


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, heads_per_chunk, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2406_15486_b200 as sa
        from paper_2406_15486_b200 import synth
        from paper_2406_15486_b200.parallel import sample_attention_sharded, shard_heads

        q, k, v, _ = synth.make_inputs(S, HQ, HKV, seed=3, device="cuda")
        shard = shard_heads(HQ, HKV, world, rank)
        kv = list(shard.kv_heads)
        # the single-process result of every head, computed here for the comparison
        want = torch.empty_like(q)
        group = HQ // HKV
        for h in range(HQ):
            sa.sample_attention(q[h:h + 1], k[h // group:h // group + 1], v[h // group:h // group + 1],
                                alpha=ALPHA, chunk_n=1, q_head0=h, group=group, out=want[h:h + 1])
        full = torch.full_like(q, float("nan"))
        for _ in range(2):  # the second call reuses the cached IPC mappings
            full.fill_(float("nan"))
            mine, got = sample_attention_sharded(q[list(shard.q_heads)], k[kv[0]:kv[-1] + 1], v[kv[0]:kv[-1] + 1],
                                                 shard, heads_per_chunk=heads_per_chunk, gather=True,
                                                 out=full, alpha=ALPHA, chunk_n=1)
        torch.cuda.synchronize()
        results[rank] = {"same": bool(torch.equal(got, want)), "nan": int(torch.isnan(got).sum().item()),
                         "diff": float((got.float() - want.float()).abs().max().item()),
                         "mine_is_view": mine.data_ptr() == got[rank * (HQ // world)].data_ptr()}
    finally:
        dist.barrier()
        dist.destroy_process_group()


@pytest.mark.parametrize("heads_per_chunk", [1, 2])
def test_p2p_gather_two_ranks_one_gpu(heads_per_chunk):
    world = 2
    mgr = mp.get_context("spawn").Manager()
    results = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), heads_per_chunk, results), nprocs=world,
                       start_method="spawn", join=True)
    assert len(results) == world
    for r in range(world):
        res = results[r]
        assert res["nan"] == 0, res            # every rank's rows arrived in every buffer
        assert res["same"], res                # and equal the single-process heads bit for bit
        assert res["mine_is_view"], res


def test_peers_entry_point_rejects_bad_arguments():
    import ctypes

    from paper_2406_15486_b200 import _lib
    from paper_2406_15486_b200.errors import InputError

    q = torch.zeros((1, 256, 128), dtype=torch.bfloat16, device="cuda")
    cnt = torch.ones((1, 2), dtype=torch.int32, device="cuda")
    idx = torch.zeros((1, 3), dtype=torch.int32, device="cuda")
    too_many = (ctypes.c_void_p * (_lib.SA_MAX_PEERS + 1))(*([q.data_ptr()] * (_lib.SA_MAX_PEERS + 1)))
    with pytest.raises(InputError):
        _lib.call("sa_sparse_forward_peers", q.data_ptr(), q.data_ptr(), q.data_ptr(), _lib.SA_BF16, 256, 1, 1, 128,
                  128, 1, 0, cnt.data_ptr(), idx.data_ptr(), None, q.data_ptr(), None, None, too_many,
                  _lib.SA_MAX_PEERS + 1, None)
    nulls = (ctypes.c_void_p * 1)(None)
    with pytest.raises(InputError):
        _lib.call("sa_sparse_forward_peers", q.data_ptr(), q.data_ptr(), q.data_ptr(), _lib.SA_BF16, 256, 1, 1, 128,
                  128, 1, 0, cnt.data_ptr(), idx.data_ptr(), None, q.data_ptr(), None, None, nulls, 1, None)
