"""Time register-NTT variants (cwg_bench_kernel) at N = 8192; prints ns per polynomial."""
import ctypes
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_07569_b200 import Context, configs

cfg = configs.config("C4")
ctx = Context(cfg.N, cfg.primes, cfg.t)
lib = ctx.lib
lib.cwg_bench_kernel.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
names = ["W5 fwd NP1 MINB3 (production)", "W5 inv NP1 MINB3 (production)", "W5 fwd NP2 MINB2",
         "W5 inv NP2 MINB2", "W4 fwd NP1 MINB3", "W6 fwd NP2 MINB1",
         "W5 fwd NP1 MINB3 prime-major", "W5 inv NP1 MINB3 prime-major", "W5 fwd NP2 MINB2 prime-major",
         "W5 fwd NP1 MINB4 prime-major", "W5 fwd NP1 MINB3 register twiddles (diag)",
         "W5 fwd NP2 MINB2 register twiddles (diag)", "W5 fwd NP1 MINB3 no transposes (diag)",
         "W5 fwd NP1 MINB3 no global load/store (diag)", "W5 fwd NP1 MINB3 butterflies only (diag)",
         "W5 fwd NP2 MINB2 butterflies only (diag)", "W5 fwd persistent cp.async prefetch 3/SM",
         "W5 fwd persistent cp.async prefetch 2/SM", "W5 fwd NP1 MINB3 loads, no stores (diag)",
         "W5 fwd NP1 MINB3 smem + bulk-copy store", "W5 inv NP1 MINB3 smem + bulk-copy store"]
npolys = 36000
only = [int(a) for a in sys.argv[1:]]
for w, nm in enumerate(names):
    if only and w not in only:
        continue
    ms = ctypes.c_float()
    rc = lib.cwg_bench_kernel(ctx.h, w, npolys, 5, ctypes.byref(ms))
    if rc != 0:
        print(nm, "error", lib.cwg_last_error()); continue
    ns = ms.value * 1e6 / (npolys // 6 * 6)
    bfly = 8192 * 13 / 2
    print(f"{nm:32s} {ns:8.1f} ns/poly  {bfly / ns:6.1f} Gbfly/s  {bfly / ns / 148 / 1.965:5.2f} bfly/cyc/SM")
