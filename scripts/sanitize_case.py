"""Small answers through every TMA / mbarrier / tcgen05 kernel, for compute-sanitizer
(scripts/sanitize.sh): C1 parameters, 64 rows, checked against the C restatement's answer.
  s = 1: k_tensor_intt_r + k_round_tma (TMA ring, tcgen05) + k_ntt_mac
  s = 3: k_mac_tma (TMA ring) ; batch of 2 queries: k_mac_tma_q"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2202_07569_b200 import Client, Context, configs  # noqa: E402

cfg = configs.config("C1")
n, k, m, c = 64, 2, 12, 4
client = Client(cfg.N, cfg.primes, cfg.t, seed=2, galois_levels=c)
keys = client.keys()
pos = configs.perfect_map(np.arange(n), m, k)
for s in (1, 3):
    db = np.random.default_rng(s).integers(0, cfg.t, (n, s, cfg.N), dtype=np.uint64)
    ctx = Context(cfg.N, cfg.primes, cfg.t, options={"tile_rows": 16})
    ctx.load_db(pos, db, m=m)
    qs = np.stack([client.pack_query(configs.codeword_bits(pos[tg], m), c, first_index=1 + 5 * i)
                   for i, tg in enumerate((7, 40))])
    got = ctx.answer(qs[0], c, m, keys=keys)
    for j in range(s):
        assert np.array_equal(client.decrypt(got[j]), db[7, j]), (s, j)
    if s == 3:
        both = ctx.answer_batch(qs, c, m, keys=keys)
        assert np.array_equal(both[0], got)
        assert np.array_equal(client.decrypt(both[1][0]), db[40, 0])
    ctx.close()
print("sanitize case ok")
