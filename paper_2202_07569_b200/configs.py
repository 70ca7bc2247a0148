"""The five BASELINE.json workloads and their seeded synthetic inputs.

Parameter derivations restate the reference's (numeric.cpp:63-84 prime search,
bfv.cpp:410-422 custom chains, cw_code.cpp:34-102 code length / perfect map,
pir.cpp:95-147 default compression).  No public dataset is involved: every input is
generated from a seed.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from math import comb

import numpy as np

# ----------------------------------------------------------------------------- primes

_W = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(n: int) -> bool:
    """numeric.cpp:35-61 (deterministic Miller-Rabin for 64-bit n)."""
    if n < 2:
        return False
    for p in _W:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in _W:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def find_ntt_prime_below(hint: int, step: int) -> int:
    """numeric.cpp:63-71."""
    p = hint - (hint % step) + 1
    if p > hint:
        p -= step
    while p > 3 * step:
        if is_prime(p):
            return p
        p -= step
    raise RuntimeError("find_ntt_prime_below: no prime in range")


def find_ntt_primes_below(hint: int, step: int, count: int, exclude=()) -> list[int]:
    """numeric.cpp:73-84."""
    out, p = [], hint + 1
    while len(out) < count:
        p = find_ntt_prime_below(p - 1, step)
        if p not in exclude:
            out.append(p)
    return out


def custom_chain(N: int, L: int, bits: int) -> list[int]:
    """bfv_custom_params chain (bfv.cpp:410-422)."""
    return find_ntt_primes_below((1 << bits) - 1, 2 * N, L)


# ----------------------------------------------------------------------------- codes

def ceil_log2(n: int) -> int:
    r = 0
    while (1 << r) < n:
        r += 1
    return r


def min_code_length(n: int, k: int) -> int:
    """Smallest m with C(m, k) >= n (cw_code.cpp:34-53)."""
    m = k
    while comb(m, k) < n:
        m += 1
    return m


def default_compression(N: int, m: int) -> int:
    """c = min(ceil(log2 m), log2 N) (pir.cpp:98-106)."""
    return min(ceil_log2(m), ceil_log2(N))


def perfect_map(x, m: int, k: int) -> np.ndarray:
    """perfect_map (cw_code.cpp:80-102): the x-th weight-k m-bit word in colex order.

    Vectorised over x (array of ints < C(m, k)); returns ascending positions [len(x), k].
    """
    x = np.atleast_1d(np.asarray(x, dtype=object))
    if any(int(v) >= comb(m, k) or int(v) < 0 for v in x):
        raise ValueError("perfect_map: input out of range")
    small = comb(m, k) < (1 << 62)
    r = x.astype(np.int64) if small else x.copy()
    out = np.zeros((len(x), k), dtype=np.uint32)
    for h in range(k, 0, -1):
        table = [comb(c, h) for c in range(m)]
        if small:
            tab = np.array(table, dtype=np.int64)
            c = np.searchsorted(tab, r, side="right") - 1
            r = r - tab[c]
        else:
            c = np.array([max(i for i, v in enumerate(table) if v <= int(rv)) for rv in r])
            r = np.array([int(rv) - table[ci] for rv, ci in zip(r, c)], dtype=object)
        out[:, h - 1] = c
    return out


def codeword_bits(positions, m: int) -> np.ndarray:
    bits = np.zeros(m, np.uint8)
    bits[np.asarray(positions, dtype=np.int64)] = 1
    return bits


# ----------------------------------------------------------------------------- configs

@dataclass
class Config:
    name: str
    N: int
    primes: list[int]
    t: int
    n: int          # rows
    k: int          # Hamming weight
    m: int          # code length
    c: int          # compression
    s: int          # plaintexts per row (0 = selection only)
    op: int = 0     # 0 folklore, 1 arithmetic
    relin_bits: int = 16
    galois_bits: int = 16
    keyword: bool = False
    note: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def L(self) -> int:
        return len(self.primes)

    @property
    def h(self) -> int:
        return -(-self.m // (1 << self.c))

    def db_bytes(self, mac_words: int | None = None) -> int:
        """Algorithmic DB bytes scanned: n * s * L * N * 8 (the reference's NTT-form DB)."""
        return self.n * self.s * self.L * self.N * 8


C2_PRIMES = None


def c2_chain() -> list[int]:
    a = find_ntt_primes_below((1 << 43) - 1, 16384, 2)
    b = find_ntt_primes_below((1 << 44) - 1, 16384, 3, exclude=a)
    return a + b


def config(name: str, **over) -> Config:
    """C1..C5 of BASELINE.json. Keyword overrides shrink a config for tests."""
    if name == "C1":
        N, t = 4096, 65537
        cfg = Config("C1", N, custom_chain(N, 3, 36), t, n=1024, k=2, m=46, c=6, s=1,
                     note="tiny index PIR (CPU-runnable oracle)")
    elif name.startswith("C2"):
        # C2-k<k>: equality microbenchmark, 16384 codewords, no payload
        k = int(name.split("k")[1]) if "k" in name else 2
        N = 8192
        m = min_code_length(16384, k)
        cfg = Config(name, N, c2_chain(), find_ntt_prime_below((1 << 20) - 1, 2 * N), n=16384, k=k, m=m,
                     c=default_compression(N, m), s=0, note="equality-operator microbenchmark")
    elif name == "C3":
        N = 8192
        cfg = Config("C3", N, c2_chain(), find_ntt_prime_below((1 << 20) - 1, 2 * N), n=16000, k=2, m=180, c=8,
                     s=15, note="large-payload index PIR")
    elif name == "C4":
        N = 8192
        cfg = Config("C4", N, c2_chain(), find_ntt_prime_below((1 << 20) - 1, 2 * N), n=65536, k=2, m=363, c=9,
                     s=1, note="row-sharded index PIR (21 GB DB)")
    elif name == "C5":
        N = 16384
        cfg = Config("C5", N, find_ntt_primes_below((1 << 50) - 1, 2 * N, 8),
                     find_ntt_prime_below((1 << 20) - 1, 2 * N), n=65536, k=4, m=569, c=10, s=2, op=1,
                     keyword=True, note="single-round keyword PIR, arithmetic operator")
    else:
        raise ValueError(f"unknown config {name}")
    for key, v in over.items():
        setattr(cfg, key, v)
    return cfg


def db_positions(cfg: Config, seed: int = 1) -> np.ndarray:
    """Row codewords: index PIR -> perfect_map(i); C2 -> seeded random codewords (1/64 match
    the query codeword, chosen by query_row); keyword -> perfect_map(id) of seeded distinct
    32-bit ids (map_keyword on 4-byte LE keys, pir.cpp:22-30,155-159)."""
    if cfg.name.startswith("C2"):
        rng = np.random.default_rng(seed)
        cap = comb(cfg.m, cfg.k)
        x = rng.integers(0, cap, cfg.n, dtype=np.int64) if cap < (1 << 62) else np.array(
            [int(v) % cap for v in rng.integers(0, 1 << 62, cfg.n, dtype=np.int64)], dtype=object)
        pos = perfect_map(x, cfg.m, cfg.k)
        q = query_row(cfg, seed)
        hit = rng.random(cfg.n) < 1.0 / 64
        pos[hit] = pos[q]
        return pos
    if cfg.keyword:
        return perfect_map(keyword_ids(cfg, seed), cfg.m, cfg.k)
    return perfect_map(np.arange(cfg.n), cfg.m, cfg.k)


def keyword_ids(cfg: Config, seed: int = 1) -> np.ndarray:
    rng = np.random.default_rng(seed + 1000)
    ids = np.unique(rng.integers(0, 1 << 32, 2 * cfg.n, dtype=np.int64))
    rng.shuffle(ids)
    ids = ids[: cfg.n]
    assert len(ids) == cfg.n
    return ids


def query_row(cfg: Config, seed: int = 1) -> int:
    return int(np.random.default_rng(seed + 7).integers(0, cfg.n))


PAYLOAD_BLOCK = 1024


def db_payload(cfg: Config, seed: int = 1, lo: int = 0, hi: int | None = None) -> np.ndarray:
    """Payloads of rows [lo, hi): s plaintexts of N coefficients uniform in [0, t) per row.

    Generated per 1024-row block from its own seeded stream, so any row shard is
    reproducible on its own (identical bytes however the rows are split across GPUs)."""
    hi = cfg.n if hi is None else hi
    out = np.empty((hi - lo, cfg.s, cfg.N), dtype=np.uint64)
    b0 = lo // PAYLOAD_BLOCK
    for b in range(b0, -(-hi // PAYLOAD_BLOCK)):
        r0, r1 = b * PAYLOAD_BLOCK, min((b + 1) * PAYLOAD_BLOCK, cfg.n)
        blk = np.random.default_rng([seed, 99, b]).integers(0, cfg.t, (r1 - r0, cfg.s, cfg.N), dtype=np.uint64)
        s0, s1 = max(r0, lo), min(r1, hi)
        out[s0 - lo:s1 - lo] = blk[s0 - r0:s1 - r0]
    return out
