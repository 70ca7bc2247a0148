import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from oracle import RefLib, RefBackend
from paper_2202_07569_b200 import Context, Keys, configs
ref = RefLib()
S = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for N, L, bits, t, k, n in [(256, 2, 36, 12289, 2, 10), (256, 2, 36, 12289, 1, 10), (512, 2, 36, 12289, 2, 10),
                            (1024, 2, 36, 12289, 2, 10), (2048, 2, 36, 12289, 2, 10), (1024, 3, 36, 12289, 2, 10)]:
    primes = configs.custom_chain(N, L, bits)
    m = configs.min_code_length(n, k) if k > 1 else n
    c = configs.default_compression(N, m)
    be = RefBackend(ref, N, t, np.array(primes, np.uint64), seed=3, galois_levels=c)
    rk, gk = be.export_keys()
    pos = configs.perfect_map(np.arange(n), m, k)
    q = be.pack_query(configs.codeword_bits(pos[4], m), c)
    db = np.random.default_rng(5).integers(0, t, (n, S, N), dtype=np.uint64)
    want, _ = be.answer(q, c, m, pos, db)
    ctx = Context(N, primes, t); ctx.load_db(pos, db, m=m)
    got = ctx.answer(q, c, m, keys=Keys(rk, gk))
    i = ctx.info()
    print(N, L, k, "s", S, "J", i.J, "Mm", i.Mm, "ok", np.array_equal(got, want))
