"""CPU-only checks: the C ABI library loads and exports every declared symbol, the
host-side workload definitions and client match the reference, and the C oracle
restatement matches the reference (oracle pinning)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, small_params


def _declared_symbols(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"\b(cwg_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2202_07569_b200 import build
    from paper_2202_07569_b200.cwgpu import CLIENT_SYMBOLS, EXPORTED_SYMBOLS

    build.build()
    for path, header, listed in ((build.LIB, "cwgpu.h", EXPORTED_SYMBOLS),
                                 (build.CLIENT_LIB, "cwgpu_client.h", CLIENT_SYMBOLS)):
        lib = ctypes.CDLL(path)
        declared = _declared_symbols(header)
        assert declared, "no declarations parsed"
        for name in declared:
            assert hasattr(lib, name), name
        assert sorted(listed) == declared


def test_client_library_has_no_cuda_dependency():
    """The seeded client is CPU code in its own library: harness code that only needs keys and
    queries (the reference arm of bench.py, the golden-vector script) never maps libcwgpu.so."""
    import subprocess

    from paper_2202_07569_b200 import build

    out = subprocess.run(["ldd", build.build_client()], capture_output=True, text=True).stdout
    assert "cuda" not in out.lower() and "libcwgpu.so" not in out


def test_create_without_gpu_fails_loudly():
    from conftest import cuda_available

    if cuda_available():
        pytest.skip("GPU present")
    from paper_2202_07569_b200 import Context

    N, primes, t = small_params()
    with pytest.raises(Exception):
        Context(N, primes, t)


def test_config_parameters_match_survey():
    from paper_2202_07569_b200 import configs

    c1 = configs.config("C1")
    assert c1.primes == [68719403009, 68719230977, 68719206401] and (c1.m, c1.c) == (46, 6)
    c4 = configs.config("C4")
    assert c4.primes == [8796092858369, 8796092792833, 17592186028033, 17592185438209, 17592184717313]
    assert c4.t == 1032193 and (c4.m, c4.c) == (363, 9)
    c5 = configs.config("C5")
    assert c5.t == 786433 and len(c5.primes) == 8 and (c5.m, c5.c) == (569, 10)
    assert [configs.config(f"C2-k{k}").m for k in (1, 2, 4, 8, 16)] == [16384, 182, 27, 17, 21]
    assert configs.config("C3").m == 180


def test_perfect_map_matches_reference(reflib):
    from paper_2202_07569_b200 import configs

    for m, k in ((46, 2), (363, 2), (27, 4), (17, 8), (21, 16), (569, 4)):
        cap = configs.comb(m, k)
        xs = sorted({0, 1, 2, cap // 3, cap // 2, cap - 1})
        got = configs.perfect_map(xs, m, k)
        for x, p in zip(xs, got):
            assert np.array_equal(reflib.perfect_map(x, m, k), p), (m, k, x)
        assert configs.min_code_length(cap, k) == m or configs.comb(m - 1, k) >= cap
    assert reflib.lib.ref_min_code_length(65536, 2) == configs.min_code_length(65536, 2) == 363


def test_client_keys_and_queries_match_reference(reflib):
    """cwg_client reproduces bfv_keygen / pack_query_bits / decrypt bit for bit."""
    from oracle import RefBackend
    from paper_2202_07569_b200 import Client

    N, primes, t = small_params()
    for digits in ((16, 16), (0, 8)):
        cl = Client(N, primes, t, seed=5, galois_levels=3, relin_bits=digits[0], galois_bits=digits[1])
        be = RefBackend(reflib, N, t, np.array(primes, np.uint64), relin_bits=digits[0], galois_bits=digits[1],
                        seed=5, galois_levels=3)
        rk, gk = be.export_keys()
        k = cl.keys()
        assert np.array_equal(k.relin, rk) and np.array_equal(k.galois, gk)
        ct = cl.encrypt(np.arange(N, dtype=np.uint64) % t, index=77)
        assert np.array_equal(be.decrypt(ct), np.arange(N) % t)
        assert np.array_equal(cl.decrypt(ct), np.arange(N) % t)


def test_oracle_matches_reference(reflib):
    """The C restatement (oracle/cwpir_oracle.c) against the reference, stage by stage."""
    from oracle import Oracle, RefBackend
    from paper_2202_07569_b200 import configs

    N, primes, t = small_params()
    c = 4
    be = RefBackend(reflib, N, t, np.array(primes, np.uint64), seed=5, galois_levels=c)
    orc = Oracle(N, t, primes)
    relin, galois = be.export_keys()
    r = np.random.default_rng(1)
    for i, p in enumerate(primes):
        a = r.integers(0, p, N, dtype=np.uint64)
        assert np.array_equal(orc.ntt(i, a), reflib.ntt(N, p, a))
        assert np.array_equal(orc.ntt(i, a, inverse=True), reflib.ntt(N, p, a, inverse=True))
    m, k, n = 12, 2, 30
    pos = configs.perfect_map(np.arange(n), m, k)
    q = be.pack_query(configs.codeword_bits(pos[7], m), c)
    ex = be.expand(q, c, m)
    assert np.array_equal(orc.expand(q, c, m, galois), ex)
    assert np.array_equal(orc.substitute(q[0], N + 1, galois[0]), be.substitute(q[0], N + 1))
    assert np.array_equal(orc.mul_lazy(ex[3], ex[7], relin), be.mul_lazy(ex[3], ex[7]))
    ct3 = be.mul_lazy(ex[1], ex[2])
    assert np.array_equal(orc.relinearize(ct3, relin), be.finalize(ct3))
    db = r.integers(0, t, (n, 2, N), dtype=np.uint64)
    want, _ = be.answer(q, c, m, pos, db, tile_rows=8)
    assert np.array_equal(orc.answer(relin, galois, q, c, m, pos, db), want)
    # the composition equals the reference's own process_query on a setup() database
    m2 = configs.min_code_length(n, k)
    q2 = be.pack_query(configs.codeword_bits(configs.perfect_map([11], m2, k)[0], m2), c)
    payloads = r.integers(1, 256, (n, 200), dtype=np.uint8)
    out_p, chunks, pos2 = be.process_query_bytes(q2, c, m2, n, k, payloads)
    out_a, _ = be.answer(q2, c, m2, pos2, chunks, tile_rows=7)
    assert np.array_equal(out_p, out_a)


@pytest.mark.parametrize("k,op", [(3, 0), (4, 1)])
def test_oracle_trees_match_reference(reflib, k, op):
    from oracle import Oracle, RefBackend
    from paper_2202_07569_b200 import configs

    N, primes, t = small_params(1024, 4, 50, 12289)
    c, n = 4, 10
    m = configs.min_code_length(n, k)
    be = RefBackend(reflib, N, t, np.array(primes, np.uint64), seed=7, galois_levels=c)
    orc = Oracle(N, t, primes)
    relin, galois = be.export_keys()
    pos = configs.perfect_map(np.arange(n), m, k)
    q = be.pack_query(configs.codeword_bits(pos[3], m), c)
    db = np.random.default_rng(2).integers(0, t, (n, 1, N), dtype=np.uint64)
    want, _ = be.answer(q, c, m, pos, db, op=op)
    assert np.array_equal(orc.answer(relin, galois, q, c, m, pos, db, op=op), want)
    assert np.array_equal(be.decrypt(want[0]), db[3, 0])


def test_client_secret_export_and_reference_arm_inputs(reflib):
    """The client's exported secret key decrypts what the reference encrypts with the same seed
    (the GPU client calls take it), and the reference arm's own keys / query (oracle.RefBackend)
    are word for word the repo client's, so both arms answer the same inputs."""
    from oracle import RefBackend
    from paper_2202_07569_b200 import Client, configs

    import bench

    N, primes, t = small_params()
    cl = Client(N, primes, t, seed=9, galois_levels=2)
    s, seed = cl.secret()
    assert s.dtype == np.int8 and set(np.unique(s)) <= {-1, 0, 1}
    assert list(seed[:1]) == [9]  # Seed256::from_u64(9) = {9, golden-ratio words} (prf.hpp:18-22)
    be = RefBackend(reflib, N, t, np.array(primes, np.uint64), seed=9, galois_levels=2)
    ct = be.encrypt(np.arange(N, dtype=np.uint64) % t)
    assert np.array_equal(cl.decrypt(ct), np.arange(N) % t)
    # the reference's encryption index is a process-global counter starting at 1 (bfv.cpp:518):
    # the reference arm draws its query first thing in a fresh process, as here
    import hashlib
    import subprocess
    import sys

    code = ("import sys, hashlib; sys.path.insert(0, %r); import bench; from paper_2202_07569_b200 import configs; "
            "cfg = configs.config('C1'); ref, be, q, pos = bench.reference_inputs(cfg); rk, gk = be.export_keys(); "
            "print(hashlib.sha256(q.tobytes() + pos.tobytes() + rk.tobytes() + gk.tobytes()).hexdigest())") % ROOT
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    cfg = configs.config("C1")
    client, keys, query, positions, target, lo, hi = bench.make_inputs(cfg, 0, 1)
    want = hashlib.sha256(query.tobytes() + positions.tobytes() + keys.relin.tobytes() + keys.galois.tobytes())
    assert out.stdout.strip().splitlines()[-1] == want.hexdigest()
    assert bench.bench_config(cfg) == {"workload": bench.workload_desc(cfg), "db_bytes": cfg.db_bytes()}


def test_reference_sample_bounds():
    """Reference-arm samples: >= 4096 rows unless the whole run would pass ~8 minutes, <= 8192."""
    import bench
    from paper_2202_07569_b200 import configs

    c4, c5, c1 = configs.config("C4"), configs.config("C5"), configs.config("C1")
    assert bench.sample_rows_for(c4, 0.0027, 3) == 8192
    assert bench.sample_rows_for(c4, 0.0027, 20) == 4096
    assert 64 <= bench.sample_rows_for(c5, 0.035, 20) < 4096
    assert bench.sample_rows_for(c1, 0.001, 3) == 1024  # whole database
