"""Debug helper (round 2): isolate the GPU decrypt rounding and the forced-exact lift."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_07569_b200 import Client, Context, configs
import oracle

for name in ("C1", "C4", "C5"):
    cfg = configs.config(name)
    client = Client(cfg.N, cfg.primes, cfg.t, seed=7, galois_levels=1)
    sec = client.secret()
    ctx = Context(cfg.N, cfg.primes, cfg.t)
    # ct = (Delta m, 0): decrypt must give m
    Q = 1
    for p in cfg.primes: Q *= p
    delta = Q // cfg.t
    m = np.random.default_rng(1).integers(0, cfg.t, cfg.N)
    ct = np.zeros((2, cfg.L, cfg.N), np.uint64)
    for i, p in enumerate(cfg.primes):
        ct[0, i] = np.array([(delta % p) * int(x) % p for x in m], dtype=np.uint64)
    got = ctx.decrypt(sec, ct)
    print(name, "trivial ct decrypt ok:", np.array_equal(got, m.astype(np.uint64)), got[:4], m[:4])
    # a fresh encryption of m
    c2 = client.encrypt(m.astype(np.uint64), 5)
    print(name, "enc decrypt cpu ok:", np.array_equal(client.decrypt(c2), m.astype(np.uint64)),
          "gpu ok:", np.array_equal(ctx.decrypt(sec, c2), m.astype(np.uint64)))
# forced exact lift: mul_lazy with and without force_exact
N, t = 1024, 12289
primes = configs.custom_chain(N, 3, 36)
ref = oracle.RefLib()
be = oracle.RefBackend(ref, N, t, np.array(primes, np.uint64), seed=31, galois_levels=4)
r = np.random.default_rng(5)
a = np.stack([np.stack([r.integers(0, p, N, dtype=np.uint64) for p in primes]) for _ in range(2)])
b = np.stack([np.stack([r.integers(0, p, N, dtype=np.uint64) for p in primes]) for _ in range(2)])
want = be.mul_lazy(a, b)
for opts in ({}, {"force_exact": 1}, {"force_exact": 1, "round": 0}, {"round": 0}):
    ctx = Context(N, primes, t, options=opts)
    print(opts, "mul_lazy ok:", np.array_equal(ctx.mul_lazy(a, b), want))
