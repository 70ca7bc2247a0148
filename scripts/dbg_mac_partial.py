"""Dump the MAC partial accumulators of a C4-parameter answer (debug helper); env selects the kernel."""
import os, sys, numpy as np
sys.path.insert(0, '/root/repo')
import bench
from paper_2202_07569_b200 import Context, configs
cfg = configs.config("C4")
cfg.n = int(sys.argv[1])
client, keys, query, positions, target, lo, hi = bench.make_inputs(cfg, 0, 1)
payload = configs.db_payload(cfg, 1, 0, cfg.n)
ctx = Context(cfg.N, cfg.primes, cfg.t)
ctx.load_db(positions, payload, n_total=cfg.n, m=cfg.m)
ctx.set_keys(keys)
import torch
parts = []
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    dp = torch.zeros(ctx.partial_words(), dtype=torch.int64, device="cuda")
    ctx.answer_partial(query, cfg.c, cfg.m, dp.data_ptr())
    torch.cuda.synchronize()
    parts.append(dp.cpu().numpy().view(np.uint64).reshape(cfg.s, 3, -1, cfg.N))
out = os.path.join("gpurun_out", f"partial_{os.environ.get('CWGPU_MAC','tma')}_{cfg.n}.npy")
np.save(out, np.stack(parts))
print(out, len(parts), "all-equal", all(np.array_equal(parts[0], q) for q in parts[1:]))
