"""Golden fixtures generated from the reference (scripts/make_golden.py): they pin the C
oracle on CPU and the CUDA path on the GPU box, where /root/reference is absent."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import ROOT

GOLD = os.path.join(ROOT, "tests", "golden")


def _tiny():
    return np.load(os.path.join(GOLD, "tiny_answer.npz"))


def test_oracle_ntt_known_answers():
    """C restatement of RingContext::ntt_forward/inverse vs the reference's outputs."""
    from oracle import Oracle

    kat = np.load(os.path.join(GOLD, "ntt_kat.npz"))
    N = int(kat["N"][0])
    tags = sorted({k.rsplit("_", 1)[0] for k in kat.files if k.endswith("_p")})
    assert len(tags) >= 8
    for tag in tags:
        p = int(kat[f"{tag}_p"][0])
        orc = Oracle(N, 3, [p])  # t irrelevant for the transform
        assert np.array_equal(orc.ntt(0, kat[f"{tag}_in"]), kat[f"{tag}_fwd"]), tag
        assert np.array_equal(orc.ntt(0, kat[f"{tag}_in"], inverse=True), kat[f"{tag}_inv"]), tag


def test_oracle_tiny_answer_golden():
    """C restatement of expand_query + the full answer vs the reference's fixture."""
    from oracle import Oracle

    g = _tiny()
    N, t = int(g["N"][0]), int(g["t"][0])
    orc = Oracle(N, t, [int(x) for x in g["primes"]])
    c, m = int(g["c"][0]), int(g["m"][0])
    assert np.array_equal(orc.expand(g["query"], c, m, g["galois"]), g["expanded"])
    got = orc.answer(g["relin"], g["galois"], g["query"], c, m, g["positions"], g["db"])
    assert np.array_equal(got, g["response"])


@pytest.mark.gpu
def test_gpu_tiny_answer_golden(gpu):
    from paper_2202_07569_b200 import Context, Keys

    g = _tiny()
    N, t = int(g["N"][0]), int(g["t"][0])
    ctx = Context(N, [int(x) for x in g["primes"]], t)
    c, m = int(g["c"][0]), int(g["m"][0])
    ctx.set_keys(Keys(g["relin"], g["galois"]))
    assert np.array_equal(ctx.expand(g["query"], c, m), g["expanded"])
    ctx.load_db(g["positions"], g["db"], m=m)
    assert np.array_equal(ctx.answer(g["query"], c, m), g["response"])


@pytest.mark.gpu
def test_gpu_ntt_known_answers(gpu):
    from paper_2202_07569_b200 import Context, configs

    kat = np.load(os.path.join(GOLD, "ntt_kat.npz"))
    N = int(kat["N"][0])
    for tag in ("C1_0", "C4_0", "C4_4", "C5_1"):
        p = int(kat[f"{tag}_p"][0])
        ctx = Context(N, [p], 65537)
        assert np.array_equal(ctx.ntt(kat[f"{tag}_in"], 0), kat[f"{tag}_fwd"]), tag
        assert np.array_equal(ctx.ntt(kat[f"{tag}_in"], 0, inverse=True), kat[f"{tag}_inv"]), tag


def _golden_answers():
    path = os.path.join(GOLD, "answers.json")
    return json.load(open(path)) if os.path.exists(path) else {}


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C1", "C4", "C3", "C5"])
def test_gpu_full_size_answer_matches_reference_hash(gpu, name):
    """Full-size configurations: the GPU answer's SHA-256 equals the reference's (computed once
    by scripts/make_golden.py on identical seeded inputs) and decrypts to the selected row."""
    gold = _golden_answers()
    if name not in gold:
        pytest.skip(f"no golden answer recorded for {name}")
    from paper_2202_07569_b200 import Client, Context, configs

    cfg = configs.config(name)
    client = Client(cfg.N, cfg.primes, cfg.t, seed=1, galois_levels=cfg.c)
    keys = client.keys()
    pos = configs.db_positions(cfg, 1)
    target = configs.query_row(cfg, 1)
    assert target == gold[name]["target"]
    q = client.pack_query(configs.codeword_bits(pos[target], cfg.m), cfg.c, first_index=1)
    db = configs.db_payload(cfg, 1)
    ctx = Context(cfg.N, cfg.primes, cfg.t)
    ctx.load_db(pos, db, m=cfg.m)
    resp = ctx.answer(q, cfg.c, cfg.m, op=cfg.op, keys=keys)
    assert hashlib.sha256(resp.tobytes()).hexdigest() == gold[name]["sha256"]
    for j in range(cfg.s):
        assert np.array_equal(client.decrypt(resp[j]), db[target, j])
