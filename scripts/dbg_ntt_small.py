"""Aux-prime NTT parity at every register-NTT degree (debug helper)."""
import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from oracle import RefLib
from paper_2202_07569_b200 import Context, configs
ref = RefLib()
for N in (256, 512, 1024, 2048, 4096, 8192, 16384):
    primes = configs.custom_chain(N, 2, 36)
    ctx = Context(N, primes, 12289)
    J = ctx.info().J
    aux = configs.find_ntt_primes_below((1 << 30) - 1, 2 * N, J)
    a = np.random.default_rng(1).integers(0, aux[0], (2, N), dtype=np.uint64)
    f = np.array_equal(ctx.ntt(a, 0, chain=False), ref.ntt(N, aux[0], a))
    i = np.array_equal(ctx.ntt(a, 0, chain=False, inverse=True), ref.ntt(N, aux[0], a, inverse=True))
    print(N, "fwd", f, "inv", i, flush=True)
