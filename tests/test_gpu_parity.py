"""Parity of the CUDA path (through the C ABI) against the reference itself.

Every case feeds identical inputs (keys, queries, database) to the compiled
reference (oracle/_ref, via oracle/ref_harness.cpp) and to libcwgpu.so and requires
word-for-word equal outputs.  Sizes are chosen so the reference finishes in seconds;
full-size configurations are covered in test_gpu_configs.py.
"""
import numpy as np
import pytest

from conftest import small_params

pytestmark = pytest.mark.gpu


def _ctx(N, primes, t, **kw):
    from paper_2202_07569_b200 import Context

    return Context(N, primes, t, **kw)


def _ref_backend(reflib, N, primes, t, seed, levels, relin_bits=16, galois_bits=16):
    from oracle import RefBackend

    return RefBackend(reflib, N, t, np.array(primes, np.uint64), relin_bits=relin_bits,
                      galois_bits=galois_bits, seed=seed, galois_levels=levels)


def _keys(be):
    from paper_2202_07569_b200 import Keys

    r, g = be.export_keys()
    return Keys(r, g)


def _rand_ct(rng, primes, N, comps=2):
    return np.stack([np.stack([rng.integers(0, p, N, dtype=np.uint64) for p in primes]) for _ in range(comps)])


@pytest.mark.parametrize("N,L,bits", [(1024, 3, 36), (4096, 3, 36), (8192, 5, 44), (16384, 8, 50)])
def test_ntt_chain_matches_ringcontext(gpu, reflib, N, L, bits):
    """RingContext::ntt_forward / ntt_inverse (ring.cpp:78-144), element for element."""
    _, primes, _ = small_params(N, L, bits, 65537)
    ctx = _ctx(N, primes, 65537)
    r = np.random.default_rng(N)
    for i, p in enumerate(primes):
        a = r.integers(0, p, (3, N), dtype=np.uint64)
        assert np.array_equal(ctx.ntt(a, i, chain=True), reflib.ntt(N, p, a))
        assert np.array_equal(ctx.ntt(a, i, chain=True, inverse=True), reflib.ntt(N, p, a, inverse=True))


@pytest.mark.parametrize("N", [1024, 8192, 16384])
def test_ntt_aux_matches_ringcontext(gpu, reflib, N):
    """The 30-bit aux/MAC primes use the same negacyclic convention."""
    from paper_2202_07569_b200 import configs

    _, primes, t = small_params(N, 3, 40, 65537)
    ctx = _ctx(N, primes, t)
    J = ctx.info().J
    aux = configs.find_ntt_primes_below((1 << 30) - 1, 2 * N, J)
    r = np.random.default_rng(1)
    for j in (0, J - 1):
        a = r.integers(0, aux[j], (2, N), dtype=np.uint64)
        assert np.array_equal(ctx.ntt(a, j, chain=False), reflib.ntt(N, aux[j], a))
        assert np.array_equal(ctx.ntt(a, j, chain=False, inverse=True), reflib.ntt(N, aux[j], a, inverse=True))


def test_substitute(gpu, reflib):
    """BfvBackend::substitute (bfv.cpp:694-712) for every level's exponent."""
    N, primes, t = small_params()
    c = 5
    be = _ref_backend(reflib, N, primes, t, seed=3, levels=c)
    ctx = _ctx(N, primes, t)
    ctx.set_keys(_keys(be))
    r = np.random.default_rng(2)
    ct = _rand_ct(r, primes, N)
    for a in range(c):
        g = N // (1 << a) + 1
        assert np.array_equal(ctx.substitute(ct, g), be.substitute(ct, g)), a
    from paper_2202_07569_b200 import HeError

    with pytest.raises(HeError, match="missing Galois key"):
        ctx.substitute(ct, 3)


@pytest.mark.parametrize("digits", [(16, 16), (8, 20), (0, 0)])
def test_expand(gpu, reflib, digits):
    """expand_query (expansion.cpp:67-83), incl. RNS digits (digit_bits 0) and a surplus."""
    N, primes, t = small_params()
    c, m = 4, 21  # h = 2, surplus entries dropped
    be = _ref_backend(reflib, N, primes, t, seed=4, levels=c, relin_bits=digits[0], galois_bits=digits[1])
    ctx = _ctx(N, primes, t, relin_bits=digits[0], galois_bits=digits[1])
    ctx.set_keys(_keys(be))
    bits = (np.random.default_rng(5).random(m) < 0.5).astype(np.uint8)
    q = be.pack_query(bits, c)
    assert np.array_equal(ctx.expand(q, c, m), be.expand(q, c, m))


@pytest.mark.parametrize("N,L,bits,t", [(1024, 3, 36, 12289), (2048, 4, 50, 65537), (8192, 5, 44, 1032193)])
def test_mul_lazy_random(gpu, reflib, N, L, bits, t):
    """mul_lazy = tensor + exact t/q rounding (bfv.cpp:765-857) on uniform ciphertexts."""
    _, primes, _ = small_params(N, L, bits, t)
    be = _ref_backend(reflib, N, primes, t, seed=6, levels=0)
    ctx = _ctx(N, primes, t)
    r = np.random.default_rng(7)
    a = np.stack([_rand_ct(r, primes, N) for _ in range(3)])
    b = np.stack([_rand_ct(r, primes, N) for _ in range(3)])
    got = ctx.mul_lazy(a, b)
    for x in range(3):
        assert np.array_equal(got[x], be.mul_lazy(a[x], b[x])), x


def test_relinearize(gpu, reflib):
    N, primes, t = small_params()
    be = _ref_backend(reflib, N, primes, t, seed=8, levels=0)
    ctx = _ctx(N, primes, t)
    ctx.set_keys(_keys(be))
    r = np.random.default_rng(9)
    ct3 = _rand_ct(r, primes, N, comps=3)
    assert np.array_equal(ctx.relinearize(ct3), be.finalize(ct3))


def _answer_case(reflib, N, primes, t, n, k, m, c, s, op, seed, positions=None, target=None, tile=0, options=None):
    from paper_2202_07569_b200 import configs

    be = _ref_backend(reflib, N, primes, t, seed=seed, levels=c)
    keys = _keys(be)
    r = np.random.default_rng(seed)
    if positions is None:
        positions = configs.perfect_map(np.arange(n), m, k)
    target = int(r.integers(0, n)) if target is None else target
    q = be.pack_query(configs.codeword_bits(positions[target], m), c)
    db = r.integers(0, t, (n, s, N), dtype=np.uint64)
    want, _ = be.answer(q, c, m, positions, db, op=op, tile_rows=tile)
    ctx = _ctx(N, primes, t, options=options)
    ctx.load_db(positions, db, m=m)
    got = ctx.answer(q, c, m, op=op, keys=keys)
    return got, want, be, db[target]


@pytest.mark.parametrize("k,op", [(2, 0), (1, 0), (3, 0), (4, 0), (4, 1), (2, 1)])
def test_answer_small(gpu, reflib, k, op):
    """process_query composition (pir.cpp:337-347) for folklore k = 1..4 and the arithmetic operator."""
    from paper_2202_07569_b200 import configs

    N, primes, t = small_params(2048, 4, 50, 65537)
    n = 40
    m = configs.min_code_length(n, k)
    c = configs.default_compression(N, m)
    got, want, be, payload = _answer_case(reflib, N, primes, t, n, k, m, c, s=2, op=op, seed=10 + k)
    assert np.array_equal(got, want)
    for j in range(2):
        assert np.array_equal(be.decrypt(got[j]), payload[j])


def test_answer_duplicate_codewords_and_ragged_tiles(gpu, reflib):
    """Config-2 style duplicate codewords (bypassing PirDatabase::setup) and a row count that
    is not a multiple of any tile size."""
    from paper_2202_07569_b200 import configs

    N, primes, t = small_params()
    n, k, m, c = 37, 2, 10, 4
    r = np.random.default_rng(11)
    positions = configs.perfect_map(r.integers(0, configs.comb(m, k), n), m, k)
    positions[5] = positions[9]
    got, want, be, _ = _answer_case(reflib, N, primes, t, n, k, m, c, s=1, op=0, seed=12, positions=positions)
    assert np.array_equal(got, want)


def test_answer_C1_full(gpu, reflib):
    """Config 1 at full size (n = 1024, m = 46, N = 4096, 3 x 36-bit primes, t = 65537)."""
    from paper_2202_07569_b200 import configs

    cfg = configs.config("C1")
    got, want, be, payload = _answer_case(reflib, cfg.N, cfg.primes, cfg.t, cfg.n, cfg.k, cfg.m, cfg.c, cfg.s,
                                          cfg.op, seed=21)
    assert np.array_equal(got, want)
    assert np.array_equal(be.decrypt(got[0]), payload[0])


def test_sharded_partials_equal_single(gpu, reflib):
    """Row sharding: per-shard partial accumulators summed then finished equal the
    single-device answer.  Shards run sequentially on one device (no cross-kernel waits)."""
    import torch

    from paper_2202_07569_b200 import configs

    N, primes, t = small_params()
    n, k, m, c, s = 50, 2, 11, 4, 2
    be = _ref_backend(reflib, N, primes, t, seed=13, levels=c)
    keys = _keys(be)
    positions = configs.perfect_map(np.arange(n), m, k)
    q = be.pack_query(configs.codeword_bits(positions[17], m), c)
    db = np.random.default_rng(14).integers(0, t, (n, s, N), dtype=np.uint64)
    want, _ = be.answer(q, c, m, positions, db)
    parts = []
    ctxs = []
    for lo, hi in ((0, 23), (23, n)):
        ctx = _ctx(N, primes, t)
        ctx.load_db(positions[lo:hi], db[lo:hi], n_total=n, row_begin=lo, m=m)
        buf = torch.zeros(ctx.partial_words(), dtype=torch.int64, device="cuda")
        ctx.answer_partial(q, c, m, buf.data_ptr(), keys=keys)
        parts.append(buf)
        ctxs.append(ctx)
    total = parts[0] + parts[1]
    torch.cuda.synchronize()
    got = ctxs[0].finish(total.data_ptr())
    assert np.array_equal(got, want)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_expansion_equals_full(gpu, reflib, world):
    """Sharded expand_query (cwg_expand_shard): the W rank subtrees, gathered rank-major as an
    all-gather would, give the full answer (cwg_answer_partial_shards + cwg_finish) and the
    reference answer; each shard holds the global leaves r, r + W, ... of cwg_expand."""
    import torch

    from paper_2202_07569_b200 import configs

    N, primes, t = small_params()
    n, k, m, c, s = 40, 2, 10, 4, 1
    be = _ref_backend(reflib, N, primes, t, seed=23, levels=c)
    keys = _keys(be)
    positions = configs.perfect_map(np.arange(n), m, k)
    q = be.pack_query(configs.codeword_bits(positions[11], m), c)
    db = np.random.default_rng(24).integers(0, t, (n, s, N), dtype=np.uint64)
    want, _ = be.answer(q, c, m, positions, db)
    ctx = _ctx(N, primes, t)
    ctx.load_db(positions, db, n_total=n, m=m)
    ctx.set_keys(keys)
    L = len(primes)
    per = ctx.shard_entries(c, world) * 2 * L * N
    shards = torch.zeros(world * per, dtype=torch.int64, device="cuda")
    for r in range(world):  # ranks run one after another on this device
        ctx.expand_shard_ptr(q.ctypes.data, c, world, r, shards[r * per:].data_ptr())
    full = ctx.expand(q, c, 1 << c)  # cwg_expand: all leaves in global order
    sh = shards.cpu().numpy().view(np.uint64).reshape(world, (1 << c) // world, 2, L, N)
    for e in range(1 << c):
        assert np.array_equal(sh[e % world, e // world], full[e])
    part = torch.zeros(ctx.partial_words(), dtype=torch.int64, device="cuda")
    ctx.answer_partial_shards_ptr(shards.data_ptr(), world, c, m, 0, part.data_ptr())
    got = ctx.finish(part.data_ptr())
    assert np.array_equal(got, want)


def test_errors_match_reference_messages(gpu):
    from paper_2202_07569_b200 import configs

    N, primes, t = small_params()
    with pytest.raises(ValueError, match="chain prime not NTT friendly"):
        _ctx(N, [primes[0] + 2], t)
    ctx = _ctx(N, primes, t)
    pos = configs.perfect_map(np.arange(10), 5, 2)
    ctx.load_db(pos, np.zeros((10, 1, N), np.uint64), m=5)
    q = np.zeros((1, 2, 3, N), np.uint64)
    with pytest.raises(ValueError, match="query code length does not match the database"):
        ctx.answer(q, 3, 6)


@pytest.mark.parametrize("kind", ["tc", "int"])
def test_exact_fallback_paths_match(gpu, reflib, kind):
    """Every rounding / centring decision forced through the exact multiword path
    (round_exact, crt_round_exact; option force_exact) for each rounding engine (tensor-core
    k_round_tma, IMAD-only k_round_mac_t)."""
    from paper_2202_07569_b200 import Context, configs

    N, primes, t = small_params(1024, 3, 36, 12289)
    be = _ref_backend(reflib, N, primes, t, seed=31, levels=4)
    r = np.random.default_rng(5)
    a = np.stack([np.stack([r.integers(0, p, N, dtype=np.uint64) for p in primes]) for _ in range(2)])
    b = np.stack([np.stack([r.integers(0, p, N, dtype=np.uint64) for p in primes]) for _ in range(2)])
    opts = {"force_exact": 1, "round": 2 if kind == "tc" else 0}
    ctx = Context(N, primes, t, options=opts)
    assert np.array_equal(ctx.mul_lazy(a, b), be.mul_lazy(a, b))
    n, k, m, c = 20, 2, 7, 3
    pos = configs.perfect_map(np.arange(n), m, k)
    q = be.pack_query(configs.codeword_bits(pos[4], m), c)
    db = r.integers(0, t, (n, 1, N), dtype=np.uint64)
    want, _ = be.answer(q, c, m, pos, db)
    ctx.load_db(pos, db, m=m)
    ctx.set_profiling(True)
    got, tm = ctx.answer(q, c, m, keys=_keys(be), timings=True)
    assert np.array_equal(got, want)
    assert tm["exact_fallbacks"] > 0
    assert ("k_round_tma" if kind == "tc" else "k_round_mac") in ctx.kernel_stats()


@pytest.mark.parametrize("kind", ["tc", "int"])
@pytest.mark.parametrize("N,L,bits", [(2048, 4, 50), (4096, 3, 36), (1024, 8, 55)])
def test_rounding_engines(gpu, reflib, kind, N, L, bits):
    """The two implementations of the tensor rounding (bfv.cpp:811-849) -- tcgen05 int8 GEMM
    (k_round_tma) and IMAD only (k_round_mac_t) -- against the reference answer, across
    aux-basis widths (JM = 8, 16, 32)."""
    from paper_2202_07569_b200 import configs

    _, primes, t = small_params(N, L, bits, 65537)
    n, k = 30, 2
    m = configs.min_code_length(n, k)
    c = configs.default_compression(N, m)
    got, want, be, payload = _answer_case(reflib, N, primes, t, n, k, m, c, s=1, op=0, seed=70 + L,
                                          options={"round": 2 if kind == "tc" else 0})
    assert np.array_equal(got, want)
    assert np.array_equal(be.decrypt(got[0]), payload[0])


@pytest.mark.parametrize("k", [1, 2, 4, 8, 16])
def test_select_config2_style(gpu, reflib, k):
    """compute_selection_vector (pir.cpp:277-312) for config 2's operator sweep: random
    codewords of weight k (1 in 4 equal to the query's), folklore product tree of depth
    ceil(log2 k) with lazy root."""
    from paper_2202_07569_b200 import configs

    N, primes, t = small_params(2048, 4, 50, 65537)
    n = 12
    m = configs.min_code_length(64, k) if k > 1 else 40
    c = configs.default_compression(N, m)
    be = _ref_backend(reflib, N, primes, t, seed=40 + k, levels=c)
    keys = _keys(be)
    r = np.random.default_rng(k)
    pos = configs.perfect_map(r.integers(0, configs.comb(m, k), n), m, k)
    pos[r.random(n) < 0.25] = pos[3]
    q = be.pack_query(configs.codeword_bits(pos[3], m), c)
    want, wcomps = be.select(q, c, m, pos)
    ctx = _ctx(N, primes, t)
    ctx.load_db(pos, None, m=m)
    got, comps = ctx.select(q, c, m, keys=keys)
    assert np.array_equal(comps, wcomps)
    assert np.array_equal(got, want)
    # matching rows decrypt to 1 (the selection bit), others to 0
    for i in range(n):
        bit = int(np.array_equal(pos[i], pos[3]))
        assert be.decrypt(got[i][: comps[i]])[0] == bit


@pytest.mark.parametrize("N,k", [(256, 1), (256, 2), (512, 2)])
def test_answer_small_rings(gpu, reflib, N, k):
    """Small rings exercise partially filled coefficient blocks in the payload MAC grid."""
    from paper_2202_07569_b200 import configs

    primes = configs.custom_chain(N, 3, 36)  # k = 2 needs > 72 bits of q to decrypt at these N
    n = 10
    m = configs.min_code_length(n, k) if k > 1 else n
    c = configs.default_compression(N, m)
    got, want, be, payload = _answer_case(reflib, N, primes, 12289, n, k, m, c, s=2, op=0, seed=60 + N + k)
    assert np.array_equal(got, want)
    assert be.noise_budget(got[1]) > 0
    assert np.array_equal(be.decrypt(got[1]), payload[1])


@pytest.mark.parametrize("nbytes,s_rows", [(200, (0, 30)), (3000, (7, 23))])
def test_load_db_bytes_matches_reference_setup(gpu, reflib, nbytes, s_rows):
    """cwg_load_db_bytes (codewords by perfect_map and chunk_payload on the device) against the
    reference's own process_query on a PirDatabase::setup database built from the same bytes
    (pir.cpp:214-252): identical positions, plaintexts and response; also a row shard and a
    payload spanning several plaintexts (3000 B > N floor(log2 t) / 8)."""
    import torch

    from paper_2202_07569_b200 import configs

    N, primes, t = small_params()
    n, k, c = 30, 2, 4
    m = configs.min_code_length(n, k)
    be = _ref_backend(reflib, N, primes, t, seed=41, levels=c)
    keys = _keys(be)
    r = np.random.default_rng(42)
    payloads = r.integers(0, 256, (n, nbytes), dtype=np.uint8)
    payloads[:, 0] |= 1  # no all-zero row (reserved by the reference)
    q = be.pack_query(configs.codeword_bits(configs.perfect_map([13], m, k)[0], m), c)
    want, chunks, pos = be.process_query_bytes(q, c, m, n, k, payloads)
    lo, hi = s_rows
    ctx = _ctx(N, primes, t)
    if (lo, hi) == (0, n):
        ctx.load_db_bytes(payloads, k, m)
        got = ctx.answer(q, c, m, keys=keys)
        assert np.array_equal(got, want)
    else:  # shard [lo, hi) summed with the single-device partial of the rest
        parts = []
        for a, b_ in ((0, lo), (lo, hi), (hi, n)):
            cx = _ctx(N, primes, t)
            cx.load_db_bytes(payloads[a:b_], k, m, n_total=n, row_begin=a)
            buf = torch.zeros(cx.partial_words(), dtype=torch.int64, device="cuda")
            cx.answer_partial(q, c, m, buf.data_ptr(), keys=keys)
            parts.append((cx, buf))
        total = parts[0][1] + parts[1][1] + parts[2][1]
        torch.cuda.synchronize()
        assert np.array_equal(parts[0][0].finish(total.data_ptr()), want)
    # the same database through cwg_load_db with the reference's own positions and plaintexts
    ref_ctx = _ctx(N, primes, t)
    ref_ctx.load_db(pos, chunks, m=m)
    assert np.array_equal(ref_ctx.answer(q, c, m, keys=keys), want)


def _chunk_payload(payloads, N, t):
    """chunk_payload (pir.cpp:169-193) restated: floor(log2 t) bits per coefficient, LSB first."""
    b = int(t).bit_length() - 1
    nbytes = payloads.shape[1]
    s = max(1, -(-(nbytes * 8) // (N * b)))
    bits = np.unpackbits(payloads, axis=1, bitorder="little")
    bits = np.pad(bits, ((0, 0), (0, s * N * b - bits.shape[1])))
    w = (1 << np.arange(b, dtype=np.uint64)).astype(np.uint64)
    return (bits.reshape(len(payloads), s, N, b).astype(np.uint64) * w).sum(axis=3).astype(np.uint64)


def test_load_db_bytes_errors_and_keyword_ids(gpu, reflib):
    """Keyword mode (row ids = keyword values, perfect_map on the device; config 5's CW(569, 4))
    against the reference answer on its own perfect_map positions, and the reference errors of
    PirDatabase::setup: all-zero payload, duplicate identifier, id outside the code."""
    from paper_2202_07569_b200 import configs

    N, primes, t = small_params(2048, 4, 50, 65537)
    m, k, c = 569, 4, 10
    n = 24
    ids = np.random.default_rng(5).choice(1 << 32, n, replace=False).astype(np.uint64)
    pl = np.random.default_rng(6).integers(1, 256, (n, 40), dtype=np.uint8)
    pos_ref = np.stack([reflib.perfect_map(int(x), m, k) for x in ids])
    chunks = _chunk_payload(pl, N, t)
    be = _ref_backend(reflib, N, primes, t, seed=51, levels=c)
    keys = _keys(be)
    q = be.pack_query(configs.codeword_bits(pos_ref[7], m), c)
    want, _ = be.answer(q, c, m, pos_ref, chunks)
    ctx = _ctx(N, primes, t)
    ctx.load_db_bytes(pl, k, m, row_ids=ids)
    assert np.array_equal(ctx.answer(q, c, m, keys=keys), want)
    assert np.array_equal(be.decrypt(want[0])[: chunks.shape[2]], chunks[7, 0])
    with pytest.raises(ValueError, match="all-zero payloads"):
        bad = pl.copy()
        bad[5] = 0
        ctx.load_db_bytes(bad, k, m, row_ids=ids)
    with pytest.raises(ValueError, match="duplicate identifier"):
        dup = ids.copy()
        dup[3] = dup[9]
        ctx.load_db_bytes(pl, k, m, row_ids=dup)
    with pytest.raises(ValueError, match="perfect_map: input out of range"):
        ctx.load_db_bytes(pl, 2, 8, row_ids=np.arange(n, dtype=np.uint64) + 20)


@pytest.mark.parametrize("ndev", [1, 2])
def test_load_db_file_matches_reference(gpu, reflib, tmp_path, ndev):
    """The reference's own CWDB file (write_db_file, db_file.cpp:13-31) loaded by cwg_load_db_file
    (index mode, ragged payloads zero padded as chunk_payload does) answers exactly as the
    reference's process_query on PirDatabase::setup of the same rows; keyword mode equals the
    device setup from the decoded keyword values; the parse_db / setup errors come back as the
    reference's messages.  ndev = 2: two contexts on one GPU (cwg_create_multi, rows split)."""
    from paper_2202_07569_b200 import configs

    N, primes, t = small_params()
    n, k, c, pb = 30, 2, 4, 300
    m = configs.min_code_length(n, k)
    be = _ref_backend(reflib, N, primes, t, seed=61, levels=c)
    keys = _keys(be)
    r = np.random.default_rng(62)
    payloads = r.integers(0, 256, (n, pb), dtype=np.uint8)
    payloads[:, 0] |= 1
    path = str(tmp_path / "db.cwdb")
    reflib.write_db_file(path, payloads)
    q = be.pack_query(configs.codeword_bits(configs.perfect_map([17], m, k)[0], m), c)
    want, _, _ = be.process_query_bytes(q, c, m, n, k, payloads)
    ctx = _ctx(N, primes, t, device=[0] * ndev)
    ctx.load_db_file(path, k, m)
    assert np.array_equal(ctx.answer(q, c, m, keys=keys), want)
    # keyword mode: 4-byte little-endian keys -> keyword_value
    mk, kk = 569, 4
    ids = r.choice(1 << 32, n, replace=False).astype(np.uint64)
    kbytes = ids.astype("<u4").view(np.uint8).reshape(n, 4)
    kpath = str(tmp_path / "kw.cwdb")
    reflib.write_db_file(kpath, payloads, keys=kbytes, keyword_bits=32)
    ctx.load_db_file(kpath, kk, mk)
    be10 = _ref_backend(reflib, N, primes, t, seed=61, levels=10)
    k10 = _keys(be10)
    qk = be10.pack_query(configs.codeword_bits(configs.perfect_map([int(ids[5])], mk, kk)[0], mk), 10)
    got = ctx.answer(qk, 10, mk, keys=k10)
    ref_ctx = _ctx(N, primes, t)
    ref_ctx.load_db_bytes(payloads, kk, mk, row_ids=ids)
    assert np.array_equal(got, ref_ctx.answer(qk, 10, mk, keys=k10))
    # errors (parse_db / setup wording)
    data = open(path, "rb").read()
    with pytest.raises(ValueError, match="not a database file"):
        ctx.load_db_file(b"XXXX" + data[4:], k, m)
    with pytest.raises(ValueError, match="trailing bytes in database file"):
        ctx.load_db_file(data + b"\0", k, m)
    with pytest.raises(ValueError, match="truncated database file"):
        ctx.load_db_file(data[:-1], k, m)
    dup = kbytes.copy()
    dup[3] = dup[8]
    reflib.write_db_file(kpath, payloads, keys=dup, keyword_bits=32)
    with pytest.raises(ValueError, match="duplicate key in database file"):
        ctx.load_db_file(kpath, kk, mk)


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0]])
def test_multi_device_context_matches_single(gpu, reflib, devices):
    """cwg_create_multi (SURVEY 8b device_ids): rows split across contexts (here several on one
    GPU), sharded expansion all-gathered by peer copies (power-of-two counts) or replicated, partials
    summed on the root -- bit-identical to the reference answer; selection rows land in place; the
    per-process row-shard entry points refuse a multi-device context."""
    import torch

    from paper_2202_07569_b200 import StateError, configs

    N, primes, t = small_params(2048, 4, 50, 65537)
    for k, op, s in ((2, 0, 1), (4, 1, 2)):
        n = 41
        m = configs.min_code_length(n, k)
        c = configs.default_compression(N, m)
        be = _ref_backend(reflib, N, primes, t, seed=90 + k, levels=c)
        keys = _keys(be)
        r = np.random.default_rng(k)
        pos = configs.perfect_map(np.arange(n), m, k)
        target = 29
        q = be.pack_query(configs.codeword_bits(pos[target], m), c)
        db = r.integers(0, t, (n, s, N), dtype=np.uint64)
        want, _ = be.answer(q, c, m, pos, db, op=op)
        ctx = _ctx(N, primes, t, device=devices)
        ctx.load_db(pos, db, m=m)
        assert ctx.info().n_local == n
        got, tm = ctx.answer(q, c, m, op=op, keys=keys, timings=True)
        assert np.array_equal(got, want)
        assert tm["n_devices"] == len(devices)
        got2, tm2 = ctx.answer(q, c, m, op=op, keys=keys, timings=True)  # same keys again: device key cache
        assert np.array_equal(got2, want) and tm2["keys_cached"] == 1
        if op == 0:
            sel_want, comps_want = be.select(q, c, m, pos)
            sel, comps = ctx.select(q, c, m, keys=keys)
            assert np.array_equal(sel, sel_want) and np.array_equal(comps, comps_want)
        with pytest.raises(StateError):
            ctx.answer_partial(q, c, m, torch.zeros(8, dtype=torch.int64, device="cuda").data_ptr())


@pytest.mark.parametrize("name", ["C1", "C4", "C5"])
def test_gpu_client_matches_reference_client(gpu, reflib, name):
    """SURVEY 8f-f4 on the GPU: pack_query_bits + encrypt (ChaCha20 streams, rejection-sampled
    uniform_rns, centred-binomial noise) equal the CPU client's words (pinned to the reference's
    bfv_keygen / pack_query_bits by test_cpu_host.py), for h = 1 and h = 2 query ciphertexts; decrypt
    of 2- and 3-component ciphertexts equals the reference's BfvBackend::decrypt."""
    from paper_2202_07569_b200 import Client, Context, configs

    cfg = configs.config(name)
    client = Client(cfg.N, cfg.primes, cfg.t, seed=7, galois_levels=1)
    secret = client.secret()
    ctx = Context(cfg.N, cfg.primes, cfg.t)
    r = np.random.default_rng(8)
    for m, first in ((cfg.m, 1), ((1 << cfg.c) + 5, 40)):  # h = 1, then h = 2 with a later index
        bits = (r.random(m) < 0.3).astype(np.uint8)
        want = client.pack_query(bits, cfg.c, first_index=first)
        got = ctx.encrypt_query(secret, bits, cfg.c, first_index=first)
        assert np.array_equal(got, want)
    be = oracle_backend(reflib, cfg, seed=7)
    ct2 = want
    assert np.array_equal(ctx.decrypt(secret, ct2), np.stack([client.decrypt(x) for x in ct2]))
    a, b = ct2[0], ct2[1]
    ct3 = be.mul_lazy(a, b)
    assert np.array_equal(ctx.decrypt(secret, ct3), be.decrypt(ct3))


def oracle_backend(reflib, cfg, seed):
    from oracle import RefBackend

    return RefBackend(reflib, cfg.N, cfg.t, np.array(cfg.primes, np.uint64), seed=seed, galois_levels=1)


@pytest.mark.parametrize("k", [3, 4, 5])
def test_arith_factor_preparation_variants(gpu, reflib, k):
    """The arithmetic operator's factors prepared from k' once plus per-factor constants
    (default) and prepared one by one (option prep_factors = 0) both equal the reference."""
    from paper_2202_07569_b200 import configs

    N, primes, t = small_params(2048, 4, 50, 65537)
    n = 30
    m = configs.min_code_length(n, k)
    c = configs.default_compression(N, m)
    for mode, ltc in ((1, 1), (0, 1), (1, 0)):
        got, want, be, payload = _answer_case(reflib, N, primes, t, n, k, m, c, s=1, op=1, seed=80 + k,
                                              options={"prep_factors": mode, "tile_rows": 7, "lift_tc": ltc})
        assert np.array_equal(got, want), mode
        assert np.array_equal(be.decrypt(got[0]), payload[0])
