"""Answer parity for the two payload-MAC kernels (debug helper): CWGPU_MAC from the environment."""
import os, sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from oracle import RefLib, RefBackend
from paper_2202_07569_b200 import Context, Keys, configs
ref = RefLib()
for N, L, bits, t, k, n, s in [(1024, 3, 36, 12289, 2, 10, 1), (2048, 3, 36, 12289, 2, 40, 1), (2048, 3, 36, 12289, 2, 40, 3),
                               (2048, 3, 36, 12289, 1, 40, 2)]:
    primes = configs.custom_chain(N, L, bits)
    m = configs.min_code_length(n, k) if k > 1 else n
    c = configs.default_compression(N, m)
    be = RefBackend(ref, N, t, np.array(primes, np.uint64), seed=3, galois_levels=c)
    rk, gk = be.export_keys()
    pos = configs.perfect_map(np.arange(n), m, k)
    q = be.pack_query(configs.codeword_bits(pos[4], m), c)
    db = np.random.default_rng(5).integers(0, t, (n, s, N), dtype=np.uint64)
    want, _ = be.answer(q, c, m, pos, db)
    ctx = Context(N, primes, t); ctx.load_db(pos, db, m=m)
    got = ctx.answer(q, c, m, keys=Keys(rk, gk))
    print(os.environ.get("CWGPU_MAC"), N, k, n, s, "ok", np.array_equal(got, want), flush=True)
