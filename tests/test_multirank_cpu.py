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
