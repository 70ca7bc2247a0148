#!/usr/bin/env python
"""Generate tests/golden/ fixtures from the REFERENCE itself (oracle/_ref, built from
/root/reference by oracle/build_ref.sh).  Run in the build container; the fixtures are
committed so the GPU box (which has no /root/reference) can check against them.

  python scripts/make_golden.py small        # ntt_kat.npz, tiny_answer.npz (seconds)
  python scripts/make_golden.py C1 C3 C4 ... # answers.json: SHA-256 of full-size answers

Full-size inputs are regenerated bit-identically on any machine from seeds:
keys and query by the client (cwg_client, pinned to the reference's bfv_keygen /
pack_query_bits by tests/test_cpu_host.py), rows and payloads by configs.py.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLD = os.path.join(ROOT, "tests", "golden")


def small():
    import oracle
    from paper_2202_07569_b200 import configs

    oracle.build_ref()
    ref = oracle.RefLib()
    os.makedirs(GOLD, exist_ok=True)
    # NTT known answers (RingContext::ntt_forward, ring.cpp:78-109) for chain primes of every config
    kat = {}
    rng = np.random.default_rng(2024)
    N = 1024
    for tag, primes in (("C1", configs.config("C1").primes), ("C4", configs.c2_chain()),
                        ("C5", configs.config("C5").primes[:2]), ("aux30", configs.find_ntt_primes_below((1 << 30) - 1, 2 * 16384, 2))):
        for i, p in enumerate(primes):
            a = rng.integers(0, p, N, dtype=np.uint64)
            kat[f"{tag}_{i}_p"] = np.array([p], np.uint64)
            kat[f"{tag}_{i}_in"] = a
            kat[f"{tag}_{i}_fwd"] = ref.ntt(N, p, a)
            kat[f"{tag}_{i}_inv"] = ref.ntt(N, p, a, inverse=True)
    np.savez_compressed(os.path.join(GOLD, "ntt_kat.npz"), N=np.array([N]), **kat)
    # a tiny full answer: N = 256, 2 x 36-bit primes, t = 12289, n = 10, k = 2, m = 5, c = 3, s = 2
    N, t = 256, 12289
    primes = configs.custom_chain(N, 2, 36)
    be = oracle.RefBackend(ref, N, t, np.array(primes, np.uint64), seed=77, galois_levels=3)
    relin, galois = be.export_keys()
    n, k, m, c, s = 10, 2, 5, 3, 2
    pos = configs.perfect_map(np.arange(n), m, k)
    target = 6
    q = be.pack_query(configs.codeword_bits(pos[target], m), c)
    db = np.random.default_rng(5).integers(0, t, (n, s, N), dtype=np.uint64)
    resp, _ = be.answer(q, c, m, pos, db)
    expanded = be.expand(q, c, m)
    np.savez_compressed(os.path.join(GOLD, "tiny_answer.npz"), N=np.array([N]), t=np.array([t]),
                        primes=np.array(primes, np.uint64), k=np.array([k]), m=np.array([m]), c=np.array([c]),
                        target=np.array([target]), relin=relin, galois=galois, query=q, positions=pos, db=db,
                        expanded=expanded, response=resp)
    print("wrote ntt_kat.npz, tiny_answer.npz")


def full(names):
    import oracle
    from paper_2202_07569_b200 import Client, configs

    ref = oracle.RefLib()
    path = os.path.join(GOLD, "answers.json")
    gold = json.load(open(path)) if os.path.exists(path) else {}
    for name in names:
        cfg = configs.config(name)
        t0 = time.time()
        client = Client(cfg.N, cfg.primes, cfg.t, seed=1, galois_levels=cfg.c)
        keys = client.keys()
        pos = configs.db_positions(cfg, 1)
        target = configs.query_row(cfg, 1)
        q = client.pack_query(configs.codeword_bits(pos[target], cfg.m), cfg.c, first_index=1)
        db = configs.db_payload(cfg, 1)
        be = oracle.RefBackend(ref, cfg.N, cfg.t, np.array(cfg.primes, np.uint64), keys=(keys.relin, keys.galois))
        tile = 2048 if cfg.N <= 8192 else 256
        resp, st = be.answer(q, cfg.c, cfg.m, pos, db, op=cfg.op, tile_rows=tile)
        dec_ok = all(np.array_equal(client.decrypt(resp[j]), db[target, j]) for j in range(cfg.s))
        gold[name] = {"sha256": hashlib.sha256(resp.tobytes()).hexdigest(), "seed": 1, "target": int(target),
                      "shape": list(resp.shape), "decrypts_to_target": bool(dec_ok),
                      "reference_seconds": round(time.time() - t0, 1), "reference_threads": ref.worker_threads(),
                      "tile_rows": tile, "stage_ms": [round(x, 1) for x in st]}
        json.dump(gold, open(path, "w"), indent=1, sort_keys=True)
        print(name, gold[name], flush=True)


C2_TILE = 1024  # rows per tile hash (GPU tests may check the selection tile by tile)


def c2(names):
    """Config 2 (equality microbenchmark): the reference's compute_selection_vector BFV branch
    (pir.cpp:287-302, via ref_select) over all 16384 seeded codewords for each k, hashed as
    SHA-256 of the [n][3][L][N] selection array (2-component rows zero padded) in C2_TILE-row
    tiles plus the whole array, and of comps[n]."""
    import oracle
    from paper_2202_07569_b200 import Client, configs

    ref = oracle.RefLib()
    path = os.path.join(GOLD, "answers.json")
    gold = json.load(open(path)) if os.path.exists(path) else {}
    for name in names:
        cfg = configs.config(name)
        t0 = time.time()
        client = Client(cfg.N, cfg.primes, cfg.t, seed=1, galois_levels=cfg.c)
        keys = client.keys()
        pos = configs.db_positions(cfg, 1)
        target = configs.query_row(cfg, 1)
        q = client.pack_query(configs.codeword_bits(pos[target], cfg.m), cfg.c, first_index=1)
        be = oracle.RefBackend(ref, cfg.N, cfg.t, np.array(cfg.primes, np.uint64), keys=(keys.relin, keys.galois))
        sel, comps = be.select(q, cfg.c, cfg.m, pos)
        secs = time.time() - t0
        whole = hashlib.sha256()
        tiles = []
        for r0 in range(0, cfg.n, C2_TILE):
            b = sel[r0:r0 + C2_TILE].tobytes()
            whole.update(b)
            tiles.append(hashlib.sha256(b).hexdigest())
        # decrypt spot check: matching rows decrypt to the constant 1, others to 0 (coefficient 0)
        match = np.all(pos == pos[target], axis=1)
        rows = [int(np.flatnonzero(match)[0]), int(np.flatnonzero(~match)[0])]
        dec = [int(client.decrypt(sel[r, :comps[r]])[0]) for r in rows]
        gold[name] = {"sha256": whole.hexdigest(), "tile_rows": C2_TILE, "tile_sha256": tiles,
                      "comps_sha256": hashlib.sha256(comps.astype(np.uint32).tobytes()).hexdigest(),
                      "comps": int(comps[0]), "seed": 1, "target": int(target), "shape": list(sel.shape),
                      "matches": int(match.sum()), "decrypt_match_nonmatch": dec,
                      "reference_seconds": round(secs, 1), "reference_threads": ref.worker_threads()}
        del sel
        json.dump(gold, open(path, "w"), indent=1, sort_keys=True)
        print(name, {k: v for k, v in gold[name].items() if k != "tile_sha256"}, flush=True)


if __name__ == "__main__":
    args = sys.argv[1:] or ["small"]
    if "small" in args:
        small()
        args = [a for a in args if a != "small"]
    c2_names = [a for a in args if a.startswith("C2")]
    if c2_names:
        c2(c2_names)
    args = [a for a in args if not a.startswith("C2")]
    if args:
        full(args)
