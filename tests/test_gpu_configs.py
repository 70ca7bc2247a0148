"""BASELINE.json configurations at their full cryptographic parameters (N, chain, t, k, m,
c, s, operator) against the reference, with the row count reduced so the reference
finishes in seconds.  Full row counts are checked by test_golden.py (reference answer
hashes) and by bench.py (decryption of the selected row)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(reflib, cfg, rows, seed=1, select_only=False, expect_kernel=None, options=None):
    from oracle import RefBackend
    from paper_2202_07569_b200 import Client, Context, configs

    client = Client(cfg.N, cfg.primes, cfg.t, seed=seed, galois_levels=cfg.c)
    keys = client.keys()
    pos = configs.db_positions(cfg, seed)[:rows]
    target = rows // 3
    q = client.pack_query(configs.codeword_bits(pos[target], cfg.m), cfg.c, first_index=1)
    be = RefBackend(reflib, cfg.N, cfg.t, np.array(cfg.primes, np.uint64), keys=(keys.relin, keys.galois))
    ctx = Context(cfg.N, cfg.primes, cfg.t, options=options)
    if select_only:
        want, wc = be.select(q, cfg.c, cfg.m, pos)
        ctx.load_db(pos, None, m=cfg.m)
        got, gc = ctx.select(q, cfg.c, cfg.m, keys=keys)
        assert np.array_equal(gc, wc)
        assert np.array_equal(got, want)
        return client, got, pos, target
    db = configs.db_payload(cfg, seed, 0, rows)
    want, _ = be.answer(q, cfg.c, cfg.m, pos, db, op=cfg.op)
    ctx.load_db(pos, db, n_total=rows, m=cfg.m)
    if expect_kernel:
        ctx.set_profiling(True)
    got = ctx.answer(q, cfg.c, cfg.m, op=cfg.op, keys=keys)
    if expect_kernel:
        assert expect_kernel in ctx.kernel_stats(), f"{expect_kernel} did not run"
    assert np.array_equal(got, want)
    for j in range(cfg.s):
        assert np.array_equal(client.decrypt(got[j]), db[target, j])
    return client, got, pos, target


@pytest.mark.parametrize("name,rows", [("C3", 12), ("C4", 40)])
def test_config_full_params_reduced_rows(gpu, reflib, name, rows):
    from paper_2202_07569_b200 import configs

    _run(reflib, configs.config(name), rows)


@pytest.mark.parametrize("opts", [{}, {"m2c_tc": 0, "lift_tc": 0, "ks_fixed": 0, "dec_tc": 0}], ids=["default", "cuda-core-conversions"])
def test_config5_keyword_arith_reduced_rows(gpu, reflib, opts):
    """Config 5: N = 16384, 8 x 50-bit primes (400-bit q), t = 786433, arithmetic operator
    k = 4 over CW(569, 4) keyword codewords, s = 2, c = 10 (1023 substitutions).  Default: the chain
    <-> aux / MAC basis conversions of the product tree on the tensor cores (k_lift_tc,
    k_mac_to_chain_tc: Mm = 17 -> K = 96 bytes); second run: the CUDA-core kernels."""
    from paper_2202_07569_b200 import configs

    _run(reflib, configs.config("C5"), 6, options=opts)


@pytest.mark.parametrize("k", [2, 16])
def test_config2_full_params_reduced_rows(gpu, reflib, k):
    from paper_2202_07569_b200 import configs

    cfg = configs.config(f"C2-k{k}")
    client, sel, pos, target = _run(reflib, cfg, 10, select_only=True)


def test_payload_mac_kernels_agree_under_repetition(gpu):
    """The TMA-fed payload MAC (k_mac_tma: 4-stage shared-memory ring refilled by cp.async.bulk)
    and the register-streaming MAC (k_mac2) produce the same partial accumulators, answer after
    answer, at C3 parameters (15 plaintexts per row: the TMA path) over several row tiles (a
    missing async-proxy fence once made the ring race under load)."""
    import torch

    import bench
    from paper_2202_07569_b200 import Context, configs

    cfg = configs.config("C3")
    cfg.n = 1024
    _, keys, query, positions, _, _, _ = bench.make_inputs(cfg, 0, 1)
    payload = configs.db_payload(cfg, 1, 0, cfg.n)
    parts = {}
    variants = {
        "v2": {"mac": 0},                                  # k_mac2 (register stream)
        "tma": {"mac_rows": 0},                            # k_mac_tma_q (3 slices per CTA)
        "rows": {},                                        # k_mac_rows (whole rows, persistent CTAs)
        "rows20": {"mac_item_rows": 20, "tile_rows": 100}, # ragged items: folds at rows 8 and 16, 5-row tail
        "rows8": {"mac_item_rows": 8, "streams": 1},       # an item ends exactly on a fold boundary
    }
    for mac, opts in variants.items():
        ctx = Context(cfg.N, cfg.primes, cfg.t, options=opts)
        ctx.load_db(positions, payload, n_total=cfg.n, m=cfg.m)
        ctx.set_keys(keys)
        runs = []
        for _ in range(1 if mac == "v2" else 4):
            dp = torch.zeros(ctx.partial_words(), dtype=torch.int64, device="cuda")
            ctx.answer_partial(query, cfg.c, cfg.m, dp.data_ptr())
            torch.cuda.synchronize()
            runs.append(dp.cpu().numpy())
        parts[mac] = runs
        del ctx
    for mac, runs in parts.items():
        for r in runs:
            assert np.array_equal(r, parts["v2"][0]), mac


@pytest.mark.parametrize("opts,kernel", [
    ({"fuse_mac": 0}, "k_round_tma"),                   # selection NTT + separate payload MAC kernels
    ({}, "k_round_tma"),                                # default: k_tensor_intt_r, k_round_tma, k_ntt_mac
    ({"streams": 1}, "k_round_tma"),                    # one tile stream
    ({"round_g2": 0}, "k_round_tma"),                   # one-GEMM rounding epilogue
    ({"round": 0}, "k_round_mac"),                      # IMAD-only rounding
    ({"ks32": 0}, "k_round_tma"),                       # 64-bit key switching in the expansion
    ({"lift_tc": 0}, "k_round_tma"),                    # centred lift on the CUDA cores (k_lift)
    ({"m2c_tc": 0}, "k_round_tma"),                     # MAC basis -> chain on the CUDA cores (k_mac_to_chain)
    ({"ks_fixed": 0}, "k_round_tma"),                   # run-time-shape key-switch MAC (k_ks_mac32s)
    ({"dec_tc": 0}, "k_round_tma"),                     # digit decomposition on the CUDA cores (k_decompose_t)
    ({"force_exact": 1}, "k_round_tma"),                # every rounding through round_exact
    ({"force_exact": 1, "fuse_mac": 0}, "k_round_tma"),
], ids=["unfused", "default", "one-stream", "one-gemm", "imad-round", "ks64", "lift-cuda", "m2c-cuda", "ks-runtime-shape", "decompose-cuda", "exact",
        "exact-unfused"])
def test_answer_path_variants_match_reference(gpu, reflib, opts, kernel):
    """Every kernel variant of the answer path (tensor/rounding/NTT/MAC fusions, TMA feeds, the
    exact multiword rounding) against the reference at full C4 parameters, over ragged 16-row
    tiles rotating over the tile streams."""
    from paper_2202_07569_b200 import configs

    _run(reflib, configs.config("C4"), 40, expect_kernel=kernel, options={"tile_rows": 16, **opts})


@pytest.mark.parametrize("name,rows,Q,opts", [
    ("C3", 24, 5, {}),                 # s = 15: one database pass per group of <= 4 queries (k_mac_tma_q)
    ("C3", 24, 2, {"mac": 0}),         # s = 15 through k_mac2 per query
    ("C4", 40, 3, {"tile_rows": 16}),  # s = 1: fused selection NTT + MAC per query, ragged tiles
])
def test_answer_batch_matches_single_answers(gpu, reflib, name, rows, Q, opts):
    """cwg_answer_batch (several queries of one client in one database pass) returns,
    for every query, exactly the single-query answer -- and the first equals the reference's."""
    from oracle import RefBackend
    from paper_2202_07569_b200 import Client, Context, configs

    cfg = configs.config(name)
    client = Client(cfg.N, cfg.primes, cfg.t, seed=3, galois_levels=cfg.c)
    keys = client.keys()
    pos = configs.db_positions(cfg, 3)[:rows]
    db = configs.db_payload(cfg, 3, 0, rows)
    targets = [(5 * q + 1) % rows for q in range(Q)]
    qs = np.stack([client.pack_query(configs.codeword_bits(pos[tg], cfg.m), cfg.c, first_index=1 + 10 * q)
                   for q, tg in enumerate(targets)])
    ctx = Context(cfg.N, cfg.primes, cfg.t, options=opts)
    ctx.load_db(pos, db, n_total=rows, m=cfg.m)
    got = ctx.answer_batch(qs, cfg.c, cfg.m, keys=keys)
    for q in range(Q):
        assert np.array_equal(got[q], ctx.answer(qs[q], cfg.c, cfg.m, keys=keys)), q
        for j in range(cfg.s):
            assert np.array_equal(client.decrypt(got[q, j]), db[targets[q], j])
    be = RefBackend(reflib, cfg.N, cfg.t, np.array(cfg.primes, np.uint64), keys=(keys.relin, keys.galois))
    want, _ = be.answer(qs[0], cfg.c, cfg.m, pos, db)
    assert np.array_equal(got[0], want)


def test_async_kernels_repeatable_and_exact(gpu, reflib):
    """Stand-in for compute-sanitizer (closed on this GPU pool): the kernels with asynchronous
    copies, mbarrier rings and tcgen05 (k_round_tma, k_mac_rows, k_mac_tma_q, k_mac_tma, k_ntt_mac) answer
    the same small databases many times over ragged 16-row tiles on 3 streams, every response equal
    to the reference's -- a missing fence or a ring race shows up as a differing word."""
    from oracle import RefBackend
    from paper_2202_07569_b200 import Client, Context, configs

    cfg = configs.config("C1")
    n, k, m, c = 64, 2, 12, 4
    client = Client(cfg.N, cfg.primes, cfg.t, seed=2, galois_levels=c)
    keys = client.keys()
    be = RefBackend(reflib, cfg.N, cfg.t, np.array(cfg.primes, np.uint64), keys=(keys.relin, keys.galois))
    pos = configs.perfect_map(np.arange(n), m, k)
    for s, opts in ((1, {}), (3, {}), (3, {"mac_rows": 0}), (3, {"mac_rows": 0, "mac_sg": 0}), (5, {}), (15, {}),
                    (15, {"mac_item_rows": 5}), (15, {"mac_rows": 0})):
        db = np.random.default_rng(s).integers(0, cfg.t, (n, s, cfg.N), dtype=np.uint64)
        qs = np.stack([client.pack_query(configs.codeword_bits(pos[tg], m), c, first_index=1 + 5 * i)
                       for i, tg in enumerate((7, 40))])
        want = be.answer(qs[0], c, m, pos, db)[0]
        ctx = Context(cfg.N, cfg.primes, cfg.t, options={"tile_rows": 16, "streams": 3, **opts})
        ctx.load_db(pos, db, m=m)
        ctx.set_keys(keys)
        for _ in range(8):
            assert np.array_equal(ctx.answer(qs[0], c, m), want)
        for _ in range(3):
            both = ctx.answer_batch(qs, c, m)
            assert np.array_equal(both[0], want)
            assert np.array_equal(client.decrypt(both[1][0]), db[40, 0])
