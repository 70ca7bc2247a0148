"""Parity oracles for the constant-weight PIR server answer (TEST INFRASTRUCTURE).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this package.  The product path
(``paper_2202_07569_b200``) never does.

Two checkers live here:

* ``RefLib``  -- the reference C++ core itself (``/root/reference/proj/core``),
  compiled by ``oracle/build_ref.sh`` into ``oracle/_ref/libcwpir_ref.so`` together
  with ``oracle/ref_harness.cpp`` (extern "C" entry points over the reference's
  public API).
* ``Oracle``  -- ``oracle/cwpir_oracle.c``, a plain-C restatement of the reference
  algorithms (file:line cited per function), pinned against ``RefLib`` and the
  fixtures in ``tests/golden/``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libcwpir_ref.so")
ORACLE_SO = os.path.join(HERE, "libcwpir_oracle.so")
REFERENCE_SRC = "/root/reference/proj/core"

_u64p = ctypes.POINTER(ctypes.c_uint64)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u8p = ctypes.POINTER(ctypes.c_uint8)


def _p64(a):
    assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_u64p)


def _p32(a):
    assert a.dtype == np.uint32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_u32p)


def build_oracle(force: bool = False) -> str:
    """Compile the C restatement (gcc, seconds)."""
    src = os.path.join(HERE, "cwpir_oracle.c")
    if force or not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", ORACLE_SO, src])
    return ORACLE_SO


def build_ref(force: bool = False) -> str | None:
    """Compile the reference + harness when the reference sources are present."""
    if not os.path.isdir(REFERENCE_SRC):
        return REF_SO if os.path.exists(REF_SO) else None
    script = os.path.join(HERE, "build_ref.sh")
    inputs = [os.path.join(HERE, f) for f in ("ref_harness.cpp", "build_ref.sh", "dropin_test.cpp")]
    inputs.append(os.path.join(os.path.dirname(HERE), "integration", "cwgpu_process_query.cpp"))
    lib = os.path.join(os.path.dirname(HERE), "paper_2202_07569_b200", "libcwgpu.so")
    dropin = os.path.join(HERE, "_ref", "libcwgpu_dropin.so")
    newest = max(os.path.getmtime(f) for f in inputs)
    stale = not os.path.exists(REF_SO) or os.path.getmtime(REF_SO) < newest
    if os.path.exists(lib):  # the drop-in shim links the product library
        stale = stale or not os.path.exists(dropin) or os.path.getmtime(dropin) < max(newest, os.path.getmtime(lib))
    if force or stale:
        subprocess.check_call(["sh", script])
    return REF_SO


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class RefError(RuntimeError):
    pass


class RefLib:
    """ctypes view of oracle/_ref/libcwpir_ref.so (the reference itself)."""

    def __init__(self, path: str = REF_SO):
        self.lib = lib = ctypes.CDLL(path)
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_backend_new.restype = ctypes.c_void_p
        lib.ref_backend_new.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, _u64p,
                                        ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32]
        lib.ref_backend_from_keys.restype = ctypes.c_void_p
        lib.ref_backend_from_keys.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, _u64p,
                                              ctypes.c_uint32, ctypes.c_uint32, _u64p, ctypes.c_uint32,
                                              _u64p, _u64p]
        lib.ref_backend_free.argtypes = [ctypes.c_void_p]
        lib.ref_digits.restype = ctypes.c_uint32
        lib.ref_digits.argtypes = [ctypes.c_void_p, ctypes.c_int]
        lib.ref_export_keys.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_uint32, _u64p]
        lib.ref_pack_query.argtypes = [ctypes.c_void_p, _u8p, ctypes.c_uint32, ctypes.c_uint32, _u64p]
        lib.ref_encrypt.argtypes = [ctypes.c_void_p, _u64p, _u64p]
        lib.ref_decrypt.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_uint32, _u64p]
        lib.ref_noise_budget.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_uint32]
        lib.ref_substitute.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_uint64, _u64p]
        lib.ref_expand.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_uint32, ctypes.c_uint32,
                                   ctypes.c_uint32, _u64p]
        lib.ref_mul_lazy.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_uint32, _u64p, ctypes.c_uint32, _u64p]
        lib.ref_mul.argtypes = [ctypes.c_void_p, _u64p, _u64p, _u64p]
        lib.ref_finalize.argtypes = [ctypes.c_void_p, _u64p, _u64p]
        lib.ref_weighted_sum.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_uint32, ctypes.c_uint64,
                                         _u64p, _u64p]
        lib.ref_answer.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_uint32, ctypes.c_uint32,
                                   ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, _u32p,
                                   ctypes.c_uint32, _u64p, ctypes.c_uint32, ctypes.c_uint64, _u64p,
                                   ctypes.POINTER(ctypes.c_double)]
        lib.ref_write_db_file.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64,
                                          ctypes.c_uint32, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p]
        lib.ref_select.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                   ctypes.c_uint64, ctypes.c_uint32, _u32p, _u64p, _u32p,
                                   ctypes.POINTER(ctypes.c_double)]
        lib.ref_answer_partial.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_uint32, ctypes.c_uint32,
                                           ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, _u32p,
                                           ctypes.c_uint32, _u64p, ctypes.c_uint32, _u64p]
        lib.ref_process_query_bytes.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_uint32, ctypes.c_uint32,
                                                ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, _u8p,
                                                ctypes.c_uint64, _u64p, _u32p, _u64p, _u32p]
        lib.ref_ntt.argtypes = [ctypes.c_uint32, ctypes.c_uint64, _u64p, ctypes.c_uint32, ctypes.c_int]
        lib.ref_perfect_map.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, _u32p]
        lib.ref_min_code_length.restype = ctypes.c_uint32
        lib.ref_min_code_length.argtypes = [ctypes.c_uint64, ctypes.c_uint32]
        lib.ref_find_ntt_prime_below.restype = ctypes.c_uint64
        lib.ref_find_ntt_prime_below.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        lib.ref_find_ntt_primes_below.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32,
                                                  _u64p, ctypes.c_uint32, _u64p]
        lib.ref_primitive_root.restype = ctypes.c_uint64
        lib.ref_primitive_root.argtypes = [ctypes.c_uint64]
        lib.ref_worker_threads.restype = ctypes.c_uint64

    def _check(self, rc):
        if rc != 0:
            raise RefError(self.lib.ref_last_error().decode())

    def ntt(self, N, q, a, inverse=False):
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        self._check(self.lib.ref_ntt(N, q, _p64(a), a.size // N, int(inverse)))
        return a

    def perfect_map(self, x, m, k):
        out = np.zeros(k, np.uint32)
        self._check(self.lib.ref_perfect_map(x, m, k, _p32(out)))
        return out

    def write_db_file(self, path, payloads, keys=None, keyword_bits=0):
        """write_db_file (db_file.cpp): index mode when keys is None, else keyword mode."""
        payloads = np.ascontiguousarray(payloads, dtype=np.uint8)
        n, pb = payloads.shape
        kk = None if keys is None else np.ascontiguousarray(keys, dtype=np.uint8)
        self._check(self.lib.ref_write_db_file(path.encode(), 0 if kk is None else 1, keyword_bits, n,
                                               0 if kk is None else kk.shape[1],
                                               None if kk is None else kk.ctypes.data, pb, payloads.ctypes.data))

    def worker_threads(self) -> int:
        return int(self.lib.ref_worker_threads())


class RefBackend:
    """A reference BfvBackend (client: keygen from seed; or server: from keys)."""

    def __init__(self, ref: RefLib, N, t, primes, relin_bits=16, galois_bits=16, seed=None,
                 galois_levels=0, keys=None):
        self.ref, self.N, self.t = ref, N, t
        self.primes = np.ascontiguousarray(primes, dtype=np.uint64)
        self.L = len(self.primes)
        lib = ref.lib
        if keys is None:
            h = lib.ref_backend_new(N, t, self.L, _p64(self.primes), relin_bits, galois_bits, seed,
                                    galois_levels)
        else:
            relin, galois = keys
            gs = np.array([N // (1 << a) + 1 for a in range(galois.shape[0])], np.uint64)
            h = lib.ref_backend_from_keys(N, t, self.L, _p64(self.primes), relin_bits, galois_bits,
                                          _p64(np.ascontiguousarray(relin)), galois.shape[0], _p64(gs),
                                          _p64(np.ascontiguousarray(galois)))
        if not h:
            raise RefError(lib.ref_last_error().decode())
        self.h = h
        self.galois_levels = galois_levels
        self.Dr = lib.ref_digits(h, 0)
        self.Dg = lib.ref_digits(h, 1)

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_backend_free(self.h)
            self.h = None

    def ct_shape(self, comps=2):
        return (comps, self.L, self.N)

    def export_keys(self, n_galois=None):
        n_galois = self.galois_levels if n_galois is None else n_galois
        relin = np.zeros((self.Dr, 2, self.L, self.N), np.uint64)
        galois = np.zeros((n_galois, self.Dg, 2, self.L, self.N), np.uint64)
        self.ref._check(self.ref.lib.ref_export_keys(self.h, _p64(relin), n_galois, _p64(galois)))
        return relin, galois

    def pack_query(self, bits, c):
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        h = -(-len(bits) // (1 << c))
        out = np.zeros((h, 2, self.L, self.N), np.uint64)
        self.ref._check(self.ref.lib.ref_pack_query(self.h, bits.ctypes.data_as(_u8p), len(bits), c, _p64(out)))
        return out

    def encrypt(self, plain):
        plain = np.ascontiguousarray(plain, dtype=np.uint64)
        out = np.zeros((2, self.L, self.N), np.uint64)
        self.ref._check(self.ref.lib.ref_encrypt(self.h, _p64(plain), _p64(out)))
        return out

    def decrypt(self, ct):
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        out = np.zeros(self.N, np.uint64)
        self.ref._check(self.ref.lib.ref_decrypt(self.h, _p64(ct), ct.shape[0], _p64(out)))
        return out

    def noise_budget(self, ct):
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        return self.ref.lib.ref_noise_budget(self.h, _p64(ct), ct.shape[0])

    def substitute(self, ct, g):
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        out = np.zeros_like(ct)
        self.ref._check(self.ref.lib.ref_substitute(self.h, _p64(ct), g, _p64(out)))
        return out

    def expand(self, query, c, m):
        query = np.ascontiguousarray(query, dtype=np.uint64)
        out = np.zeros((m, 2, self.L, self.N), np.uint64)
        self.ref._check(self.ref.lib.ref_expand(self.h, _p64(query), query.shape[0], c, m, _p64(out)))
        return out

    def mul_lazy(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        b = np.ascontiguousarray(b, dtype=np.uint64)
        out = np.zeros((3, self.L, self.N), np.uint64)
        self.ref._check(self.ref.lib.ref_mul_lazy(self.h, _p64(a), a.shape[0], _p64(b), b.shape[0], _p64(out)))
        return out

    def mul(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        b = np.ascontiguousarray(b, dtype=np.uint64)
        out = np.zeros((2, self.L, self.N), np.uint64)
        self.ref._check(self.ref.lib.ref_mul(self.h, _p64(a), _p64(b), _p64(out)))
        return out

    def finalize(self, ct3):
        ct3 = np.ascontiguousarray(ct3, dtype=np.uint64)
        out = np.zeros((2, self.L, self.N), np.uint64)
        self.ref._check(self.ref.lib.ref_finalize(self.h, _p64(ct3), _p64(out)))
        return out

    def weighted_sum(self, cts, plains):
        cts = np.ascontiguousarray(cts, dtype=np.uint64)
        plains = np.ascontiguousarray(plains, dtype=np.uint64)
        out = np.zeros((cts.shape[1], self.L, self.N), np.uint64)
        self.ref._check(self.ref.lib.ref_weighted_sum(self.h, _p64(cts), cts.shape[1], cts.shape[0],
                                                      _p64(plains), _p64(out)))
        return out

    def answer(self, query, c, m, positions, db, op=0, tile_rows=0):
        """Server answer composed from the reference's public calls (see ref_harness.cpp)."""
        query = np.ascontiguousarray(query, dtype=np.uint64)
        positions = np.ascontiguousarray(positions, dtype=np.uint32)
        db = np.ascontiguousarray(db, dtype=np.uint64)
        n, k = positions.shape
        s = db.shape[1]
        out = np.zeros((s, 2, self.L, self.N), np.uint64)
        st = (ctypes.c_double * 6)()
        self.ref._check(self.ref.lib.ref_answer(self.h, _p64(query), query.shape[0], c, m, n, k,
                                                _p32(positions), s, _p64(db), op, tile_rows, _p64(out), st))
        return out, list(st)

    def select(self, query, c, m, positions, stages=False):
        """compute_selection_vector per row: ([n][3][L][N], comps[n]) (+ stage ms: expand,
        prepare_cipher, selection, with stages=True)."""
        query = np.ascontiguousarray(query, dtype=np.uint64)
        positions = np.ascontiguousarray(positions, dtype=np.uint32)
        n, k = positions.shape
        sel = np.zeros((n, 3, self.L, self.N), np.uint64)
        comps = np.zeros(n, np.uint32)
        st = (ctypes.c_double * 3)()
        self.ref._check(self.ref.lib.ref_select(self.h, _p64(query), query.shape[0], c, m, n, k, _p32(positions),
                                                _p64(sel), _p32(comps), st))
        return (sel, comps, list(st)) if stages else (sel, comps)

    def answer_partial(self, query, c, m, positions, db, op=0):
        """Un-finalized inner product of a row shard: [s][3][L][N]."""
        query = np.ascontiguousarray(query, dtype=np.uint64)
        positions = np.ascontiguousarray(positions, dtype=np.uint32)
        db = np.ascontiguousarray(db, dtype=np.uint64)
        n, k = positions.shape
        s = db.shape[1]
        out = np.zeros((s, 3, self.L, self.N), np.uint64)
        self.ref._check(self.ref.lib.ref_answer_partial(self.h, _p64(query), query.shape[0], c, m, n, k,
                                                        _p32(positions), s, _p64(db), op, _p64(out)))
        return out

    def process_query_bytes(self, query, c, m, n, k, payloads):
        """The reference's own process_query on a PirDatabase::setup database."""
        query = np.ascontiguousarray(query, dtype=np.uint64)
        payloads = np.ascontiguousarray(payloads, dtype=np.uint8)
        pb = payloads.shape[1]
        bits = 0
        while (1 << (bits + 1)) <= self.t:
            bits += 1
        s = max(1, -(-(pb * 8) // (self.N * bits)))
        out = np.zeros((s, 2, self.L, self.N), np.uint64)
        s_out = ctypes.c_uint32()
        chunks = np.zeros((n, s, self.N), np.uint64)
        pos = np.zeros((n, k), np.uint32)
        self.ref._check(self.ref.lib.ref_process_query_bytes(
            self.h, _p64(query), query.shape[0], c, m, n, k, payloads.ctypes.data_as(_u8p), pb,
            _p64(out), ctypes.byref(s_out), _p64(chunks), _p32(pos)))
        assert s_out.value == s
        return out, chunks, pos


class Oracle:
    """ctypes view of the C restatement (oracle/cwpir_oracle.c)."""

    def __init__(self, N, t, primes, relin_bits=16, galois_bits=16, path=None):
        path = path or build_oracle()
        self.lib = lib = ctypes.CDLL(path)
        lib.orc_create.restype = ctypes.c_void_p
        lib.orc_create.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, _u64p,
                                   ctypes.c_uint, ctypes.c_uint]
        lib.orc_free.argtypes = [ctypes.c_void_p]
        lib.orc_info.restype = ctypes.c_uint32
        lib.orc_info.argtypes = [ctypes.c_void_p, ctypes.c_int]
        lib.orc_aux_prime.restype = ctypes.c_uint64
        lib.orc_aux_prime.argtypes = [ctypes.c_void_p, ctypes.c_uint32]
        lib.orc_ntt.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32, _u64p, ctypes.c_int]
        lib.orc_substitute.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_uint64, _u64p, _u64p]
        lib.orc_expand.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_uint32, ctypes.c_uint32,
                                   ctypes.c_uint32, _u64p, _u64p]
        lib.orc_relinearize.argtypes = [ctypes.c_void_p, _u64p, _u64p, _u64p]
        lib.orc_mul_lazy.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_uint32, _u64p, ctypes.c_uint32,
                                     _u64p, _u64p]
        lib.orc_mul.argtypes = [ctypes.c_void_p, _u64p, _u64p, _u64p, _u64p]
        lib.orc_answer.argtypes = [ctypes.c_void_p, _u64p, _u64p, _u64p, ctypes.c_uint32, ctypes.c_uint32,
                                   ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, _u32p,
                                   ctypes.c_uint32, _u64p, ctypes.c_uint32, _u64p]
        lib.orc_select.argtypes = [ctypes.c_void_p, _u64p, _u64p, _u64p, ctypes.c_uint32, ctypes.c_uint32,
                                   ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, _u32p,
                                   ctypes.c_uint32, _u64p, _u32p]
        lib.orc_find_ntt_prime_below.restype = ctypes.c_uint64
        lib.orc_find_ntt_prime_below.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        lib.orc_primitive_root.restype = ctypes.c_uint64
        lib.orc_primitive_root.argtypes = [ctypes.c_uint64]
        self.N, self.t = N, t
        self.primes = np.ascontiguousarray(primes, dtype=np.uint64)
        self.L = len(self.primes)
        self.h = lib.orc_create(N, t, self.L, _p64(self.primes), relin_bits, galois_bits)
        if not self.h:
            raise RuntimeError("orc_create failed")
        self.J = lib.orc_info(self.h, 0)
        self.Dr = lib.orc_info(self.h, 1)
        self.Dg = lib.orc_info(self.h, 2)
        self.q_bits = lib.orc_info(self.h, 3)
        self.aux_primes = [lib.orc_aux_prime(self.h, j) for j in range(self.J)]

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.orc_free(self.h)
            self.h = None

    def ntt(self, idx, a, inverse=False, aux=False):
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        self.lib.orc_ntt(self.h, int(aux), idx, _p64(a), int(inverse))
        return a

    def substitute(self, ct, g, gkey):
        out = np.zeros((2, self.L, self.N), np.uint64)
        self.lib.orc_substitute(self.h, _p64(np.ascontiguousarray(ct)), g, _p64(np.ascontiguousarray(gkey)),
                                _p64(out))
        return out

    def expand(self, query, c, m, galois):
        out = np.zeros((m, 2, self.L, self.N), np.uint64)
        rc = self.lib.orc_expand(self.h, _p64(np.ascontiguousarray(query)), query.shape[0], c, m,
                                 _p64(np.ascontiguousarray(galois)), _p64(out))
        assert rc == 0
        return out

    def relinearize(self, ct3, relin):
        out = np.zeros((2, self.L, self.N), np.uint64)
        self.lib.orc_relinearize(self.h, _p64(np.ascontiguousarray(ct3)), _p64(np.ascontiguousarray(relin)),
                                 _p64(out))
        return out

    def mul_lazy(self, a, b, relin):
        a = np.ascontiguousarray(a)
        b = np.ascontiguousarray(b)
        out = np.zeros((3, self.L, self.N), np.uint64)
        self.lib.orc_mul_lazy(self.h, _p64(a), a.shape[0], _p64(b), b.shape[0],
                              _p64(np.ascontiguousarray(relin)), _p64(out))
        return out

    def mul(self, a, b, relin):
        out = np.zeros((2, self.L, self.N), np.uint64)
        self.lib.orc_mul(self.h, _p64(np.ascontiguousarray(a)), _p64(np.ascontiguousarray(b)),
                         _p64(np.ascontiguousarray(relin)), _p64(out))
        return out

    def answer(self, relin, galois, query, c, m, positions, db, op=0):
        positions = np.ascontiguousarray(positions, dtype=np.uint32)
        db = np.ascontiguousarray(db, dtype=np.uint64)
        n, k = positions.shape
        s = db.shape[1]
        out = np.zeros((s, 2, self.L, self.N), np.uint64)
        rc = self.lib.orc_answer(self.h, _p64(np.ascontiguousarray(relin)), _p64(np.ascontiguousarray(galois)),
                                 _p64(np.ascontiguousarray(query)), query.shape[0], c, m, n, k,
                                 _p32(positions), s, _p64(db), op, _p64(out))
        assert rc == 0
        return out

    def select(self, relin, galois, query, c, m, positions, op=0):
        positions = np.ascontiguousarray(positions, dtype=np.uint32)
        n, k = positions.shape
        sel = np.zeros((n, 3, self.L, self.N), np.uint64)
        comps = np.zeros(n, np.uint32)
        rc = self.lib.orc_select(self.h, _p64(np.ascontiguousarray(relin)), _p64(np.ascontiguousarray(galois)),
                                 _p64(np.ascontiguousarray(query)), query.shape[0], c, m, n, k,
                                 _p32(positions), op, _p64(sel), _p32(comps))
        assert rc == 0
        return sel, comps
