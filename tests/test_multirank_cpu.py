"""Row sharding across ranks on CPU with torch.distributed/gloo, world size 2.

Each rank answers its contiguous row shard (rows [r n / W, (r+1) n / W), as bench.py
shards them), the partial inner products are summed by ONE collective, reduced mod q_i,
and rank 0 finalizes: the result must equal the single-process answer word for word.
This is the arithmetic the GPU path relies on (cwg_answer_partial -> NCCL sum ->
cwg_finish); the GPU-side partial/finish composition itself is covered by
tests/test_gpu_parity.py::test_sharded_partials_equal_single.
"""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_path):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2202_07569_b200 import Client, configs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N, t = 1024, 12289
    primes = configs.custom_chain(N, 3, 36)
    n, k, m, c, s = 30, 2, 9, 4, 2
    client = Client(N, primes, t, seed=9, galois_levels=c)
    keys = client.keys()
    pos = configs.perfect_map(np.arange(n), m, k)
    q = client.pack_query(configs.codeword_bits(pos[21], m), c)
    db = np.random.default_rng(4).integers(0, t, (n, s, N), dtype=np.uint64)
    lo, hi = rank * n // world, (rank + 1) * n // world
    be = oracle.RefBackend(oracle.RefLib(), N, t, np.array(primes, np.uint64), keys=(keys.relin, keys.galois))
    part = be.answer_partial(q, c, m, pos[lo:hi], db[lo:hi])
    ten = torch.from_numpy(part.view(np.int64).copy())
    dist.all_reduce(ten, op=dist.ReduceOp.SUM)  # sum < 2 * 2^36: no overflow
    total = ten.numpy().view(np.uint64).reshape(part.shape)
    qv = np.array(primes, np.uint64)[None, None, :, None]
    total = total % qv
    if rank == 0:
        got = np.stack([be.finalize(total[j]) for j in range(s)])
        want, _ = be.answer(q, c, m, pos, db)
        np.save(result_path, np.array([int(np.array_equal(got, want)),
                                       int(np.array_equal(client.decrypt(got[0]), db[21, 0]))]))
    dist.barrier()
    dist.destroy_process_group()


def test_row_shards_sum_to_full_answer_gloo(tmp_path, reflib):
    import torch.multiprocessing as mp

    res = str(tmp_path / "res.npy")
    mp.spawn(_worker, args=(2, _free_port(), res), nprocs=2, join=True)
    ok = np.load(res)
    assert ok[0] == 1, "sharded answer differs from the single-process answer"
    assert ok[1] == 1, "sharded answer does not decrypt to the selected row"


def _shard_worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c, wpe = 5, 3  # 2^c leaves, words per entry
    P = (1 << c) // world
    # rank r's cwg_expand_shard output: global leaves r, r + W, r + 2W, ... (each entry = wpe words)
    local = torch.tensor([[(rank + world * u) * 10 + w for w in range(wpe)] for u in range(P)], dtype=torch.int64)
    gathered = [torch.zeros_like(local) for _ in range(world)]
    dist.all_gather(gathered, local)  # rank-major, as bench.py's all_gather_into_tensor on NCCL
    shards = torch.cat(gathered).reshape(-1).numpy()
    m = (1 << c) - 3
    # k_unshard (kernels.cuh): entries[e][w] = shards[((e % W) * P + e / W) * wpe + w]
    ent = np.array([[shards[((e % world) * P + e // world) * wpe + w] for w in range(wpe)] for e in range(m)])
    ok = np.array_equal(ent, np.array([[e * 10 + w for w in range(wpe)] for e in range(m)]))
    if rank == 0:
        np.save(result_path, np.array([int(ok)]))
    dist.barrier()
    dist.destroy_process_group()


def test_expansion_shards_gather_rank_major(tmp_path):
    """bench.py's sharded expansion (N > 1): rank r holds global leaves r + W u; an all-gather
    concatenates the shards rank-major and k_unshard's index map restores global order."""
    import torch.multiprocessing as mp

    world = 2
    path = str(tmp_path / "shard.npy")
    mp.spawn(_shard_worker, args=(world, _free_port(), path), nprocs=world, join=True)
    assert np.load(path)[0] == 1
