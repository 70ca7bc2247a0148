"""Worker for tests/test_multirank_gpu.py (launched by torchrun, 2 ranks sharing cuda:0 over gloo).

Drives the product path of one-process-per-GPU row sharding (paper_2202_07569_b200.rowshard:
cwg_expand_shard -> all-gather -> cwg_answer_partial_shards -> reduce -> cwg_finish, and the
replicated-expansion variant cwg_answer_partial -> reduce -> cwg_finish) through libcwgpu.so and
checks rank 0's response: C1 at full size against the reference answer's SHA-256
(tests/golden/answers.json), C4 parameters with 512 rows against a single-context cwg_answer."""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    import bench
    from paper_2202_07569_b200 import Context, configs
    from paper_2202_07569_b200.rowshard import RowShardStep

    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "answers.json")))
    for name, rows in (("C1", None), ("C4", 512)):
        cfg = configs.config(name)
        if rows:
            cfg.n = rows
        client, keys, query, positions, target, lo, hi = bench.make_inputs(cfg, rank, world)
        ctx = Context(cfg.N, cfg.primes, cfg.t)
        ctx.load_db(positions[lo:hi], configs.db_payload(cfg, 1, lo, hi), n_total=cfg.n, row_begin=lo, m=cfg.m)
        for shard in (True, False):
            rs = RowShardStep(ctx, cfg, rank, world, backend="gloo", shard_expansion=shard)
            assert rs.shard == shard
            got = rs.answer(query, keys=keys)
            if rank == 0:
                if rows is None:
                    assert hashlib.sha256(got.tobytes()).hexdigest() == gold[name]["sha256"], (name, shard)
                else:
                    one = Context(cfg.N, cfg.primes, cfg.t)
                    one.load_db(positions, configs.db_payload(cfg, 1, 0, cfg.n), m=cfg.m)
                    want = one.answer(query, cfg.c, cfg.m, keys=keys)
                    assert np.array_equal(got, want), (name, shard)
                    one.close()
                for j in range(cfg.s):
                    assert np.array_equal(client.decrypt(got[j]), configs.db_payload(cfg, 1, target, target + 1)[0, j])
            dist.barrier()
        ctx.close()
    if rank == 0:
        print("multirank ok")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
