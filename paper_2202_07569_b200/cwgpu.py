"""ctypes binding of libcwgpu.so (include/cwgpu.h, include/cwgpu_client.h).

Mirrors the reference's server-side interface for the answer path:

* ``Context``  ~ ``BfvBackend`` + ``PirDatabase`` resident on one B200
  (``bfv.hpp:68-136``, ``pir.hpp:64-100``); ``Context.answer`` is
  ``process_query`` (``pir.cpp:337-347``), ``Context.select`` is
  ``compute_selection_vector`` (``pir.cpp:277-312``).
* ``Client``   ~ the reference client (keygen / ``pack_query_bits`` / decrypt), CPU code in its
  own library ``libcwgpu_client.so`` (no CUDA).

Errors raise the reference's exception types: ``ValueError`` for
``std::invalid_argument``, ``HeError`` for ``he_error``.  There is no CPU fallback:
a missing library or device raises ``RuntimeError``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcwgpu.so")
CLIENT_LIB_PATH = os.path.join(HERE, "libcwgpu_client.so")

_u64p = ctypes.POINTER(ctypes.c_uint64)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u8p = ctypes.POINTER(ctypes.c_uint8)

CWG_OK, CWG_EINVAL, CWG_EHE, CWG_ECUDA, CWG_ESTATE = 0, -1, -2, -3, -4
OP_FOLKLORE, OP_ARITH = 0, 1

# the symbols include/cwgpu.h (libcwgpu.so) and include/cwgpu_client.h (libcwgpu_client.so) declare
EXPORTED_SYMBOLS = [
    "cwg_last_error", "cwg_create", "cwg_destroy", "cwg_get_info", "cwg_load_db", "cwg_load_db_bytes", "cwg_set_keys",
    "cwg_answer", "cwg_partial_words", "cwg_answer_partial", "cwg_finish", "cwg_expand_shard",
    "cwg_answer_partial_shards", "cwg_select", "cwg_ntt",
    "cwg_expand", "cwg_mul_lazy", "cwg_relinearize", "cwg_substitute", "cwg_kernel_launches",
    "cwg_stream", "cwg_set_profiling", "cwg_kernel_stats", "cwg_kernel_units", "cwg_set_option",
    "cwg_create_multi", "cwg_device_count", "cwg_load_db_file", "cwg_answer_batch", "cwg_encrypt_query",
    "cwg_decrypt", "cwg_pinned_alloc", "cwg_pinned_free",
]
CLIENT_SYMBOLS = [
    "cwg_client_last_error", "cwg_client_create", "cwg_client_destroy", "cwg_client_digits",
    "cwg_client_export_keys", "cwg_client_encrypt", "cwg_client_pack_query", "cwg_client_decrypt",
    "cwg_client_export_secret",
]


class HeError(RuntimeError):
    """he_error (reference he.hpp:16-18)."""


class CudaError(RuntimeError):
    pass


class StateError(RuntimeError):
    pass


class CwgInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint32) for n in ("N", "L", "J", "Mm", "Dr", "Dg", "q_bits", "aux_bits")] + [
        (n, ctypes.c_uint64) for n in ("n_total", "row_begin", "n_local")] + [
        (n, ctypes.c_uint32) for n in ("s", "k", "m")]


class CwgTimings(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("total_ms", "h2d_ms", "expand_ms", "select_ms", "mac_ms",
                                               "finish_ms", "d2h_ms")] + [
        ("kernel_launches", ctypes.c_uint64), ("exact_fallbacks", ctypes.c_uint64), ("keys_cached", ctypes.c_uint32),
        ("n_devices", ctypes.c_uint32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_LIB = None


def load_library(path: str = LIB_PATH):
    """Load libcwgpu.so (built in-tree by paper_2202_07569_b200.build)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise RuntimeError(f"libcwgpu.so not built ({path}); run python -m paper_2202_07569_b200.build")
    lib = ctypes.CDLL(path)
    lib.cwg_last_error.restype = ctypes.c_char_p
    lib.cwg_create.restype = ctypes.c_void_p
    lib.cwg_create.argtypes = [ctypes.c_uint32, ctypes.c_uint32, _u64p, ctypes.c_uint64, ctypes.c_uint32,
                               ctypes.c_uint32, ctypes.c_int]
    lib.cwg_create_multi.restype = ctypes.c_void_p
    lib.cwg_create_multi.argtypes = [ctypes.c_uint32, ctypes.c_uint32, _u64p, ctypes.c_uint64, ctypes.c_uint32,
                                     ctypes.c_uint32, ctypes.POINTER(ctypes.c_int), ctypes.c_int]
    lib.cwg_device_count.restype = ctypes.c_int
    lib.cwg_pinned_alloc.restype = ctypes.c_void_p
    lib.cwg_pinned_alloc.argtypes = [ctypes.c_uint64]
    lib.cwg_pinned_free.argtypes = [ctypes.c_void_p]
    lib.cwg_destroy.argtypes = [ctypes.c_void_p]
    lib.cwg_get_info.argtypes = [ctypes.c_void_p, ctypes.POINTER(CwgInfo)]
    lib.cwg_load_db.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32,
                                ctypes.c_uint32, ctypes.c_uint32, _u32p, _u64p]
    lib.cwg_load_db_file.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32,
                                     ctypes.c_uint32]
    lib.cwg_set_keys.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_uint32, _u64p, _u64p]
    lib.cwg_load_db_bytes.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                      ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
    keyargs = [_u64p, ctypes.c_uint32, _u64p, _u64p]
    qargs = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_uint32]
    lib.cwg_answer.argtypes = [ctypes.c_void_p, *keyargs, *qargs, ctypes.c_void_p, ctypes.POINTER(CwgTimings)]
    lib.cwg_answer_batch.argtypes = [ctypes.c_void_p, *keyargs, ctypes.c_uint32, *qargs, ctypes.c_void_p,
                                     ctypes.POINTER(CwgTimings)]
    lib.cwg_encrypt_query.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32,
                                      ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p]
    lib.cwg_decrypt.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p,
                                ctypes.c_void_p]
    lib.cwg_answer_partial.argtypes = [ctypes.c_void_p, *keyargs, *qargs, ctypes.c_void_p,
                                       ctypes.POINTER(CwgTimings)]
    lib.cwg_partial_words.restype = ctypes.c_uint64
    lib.cwg_partial_words.argtypes = [ctypes.c_void_p]
    lib.cwg_finish.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p,
                               ctypes.POINTER(CwgTimings)]
    lib.cwg_select.argtypes = [ctypes.c_void_p, *keyargs, *qargs, _u64p, _u32p, ctypes.POINTER(CwgTimings)]
    lib.cwg_expand_shard.argtypes = [ctypes.c_void_p, *keyargs, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_uint32,
                                     ctypes.c_uint32, ctypes.c_void_p]
    lib.cwg_answer_partial_shards.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32,
                                              ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p,
                                              ctypes.POINTER(CwgTimings)]
    lib.cwg_ntt.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32, _u64p, ctypes.c_uint32, ctypes.c_int]
    lib.cwg_expand.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, _u64p, _u64p]
    lib.cwg_mul_lazy.argtypes = [ctypes.c_void_p, ctypes.c_uint32, _u64p, _u64p, _u64p]
    lib.cwg_relinearize.argtypes = [ctypes.c_void_p, ctypes.c_uint32, _u64p, _u64p]
    lib.cwg_substitute.argtypes = [ctypes.c_void_p, ctypes.c_uint32, _u64p, ctypes.c_uint64, _u64p]
    lib.cwg_kernel_launches.restype = ctypes.c_uint64
    lib.cwg_kernel_launches.argtypes = [ctypes.c_void_p]
    lib.cwg_stream.restype = ctypes.c_void_p
    lib.cwg_stream.argtypes = [ctypes.c_void_p]
    lib.cwg_set_profiling.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.cwg_kernel_stats.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_char_p, ctypes.c_uint32,
                                     ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64)]
    lib.cwg_kernel_units.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.POINTER(ctypes.c_double)]
    lib.cwg_set_option.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int64]
    _LIB = lib
    return lib


_CLIENT_LIB = None


def load_client_library(path: str = CLIENT_LIB_PATH):
    """Load libcwgpu_client.so (CPU only; built in-tree by paper_2202_07569_b200.build)."""
    global _CLIENT_LIB
    if _CLIENT_LIB is not None:
        return _CLIENT_LIB
    if not os.path.exists(path):
        raise RuntimeError(f"libcwgpu_client.so not built ({path}); run python -m paper_2202_07569_b200.build")
    lib = ctypes.CDLL(path)
    lib.cwg_client_last_error.restype = ctypes.c_char_p
    lib.cwg_client_create.restype = ctypes.c_void_p
    lib.cwg_client_create.argtypes = [ctypes.c_uint32, ctypes.c_uint32, _u64p, ctypes.c_uint64, ctypes.c_uint32,
                                      ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32]
    lib.cwg_client_destroy.argtypes = [ctypes.c_void_p]
    lib.cwg_client_digits.restype = ctypes.c_uint32
    lib.cwg_client_digits.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.cwg_client_export_keys.argtypes = [ctypes.c_void_p, _u64p, _u64p]
    lib.cwg_client_encrypt.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_uint64, _u64p]
    lib.cwg_client_pack_query.argtypes = [ctypes.c_void_p, _u8p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                          _u64p]
    lib.cwg_client_decrypt.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_uint32, _u64p]
    lib.cwg_client_export_secret.argtypes = [ctypes.c_void_p, ctypes.c_void_p, _u64p]
    _CLIENT_LIB = lib
    return lib


def _p64(a):
    if a is None:
        return None
    assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"], (a.dtype, a.flags)
    return a.ctypes.data_as(_u64p)


def _p32(a):
    assert a.dtype == np.uint32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_u32p)


def _raise(lib, rc):
    if rc == CWG_OK:
        return
    msg = lib.cwg_last_error().decode()
    if rc == CWG_EINVAL:
        raise ValueError(msg)
    if rc == CWG_EHE:
        raise HeError(msg)
    if rc == CWG_ECUDA:
        raise CudaError(msg)
    if rc == CWG_ESTATE:
        raise StateError(msg)
    raise RuntimeError(msg)


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


@dataclass
class Keys:
    """EvalKeySet (bfv.hpp:42-51): relin [Dr][2][L][N], galois [c][Dg][2][L][N] for g_a = N/2^a + 1."""
    relin: np.ndarray
    galois: np.ndarray

    def exponents(self, N: int) -> np.ndarray:
        return np.array([N // (1 << a) + 1 for a in range(self.galois.shape[0])], dtype=np.uint64)


class Context:
    """The B200 server for one parameter set on one device, or -- device=[ids] -- on several
    devices of this process (cwg_create_multi: rows split across them, one reduction)."""

    def __init__(self, N, primes, t, relin_bits=16, galois_bits=16, device=0, options=None):
        self.lib = lib = load_library()
        self.N, self.t = int(N), int(t)
        self.primes = _c64(primes)
        self.L = len(self.primes)
        if isinstance(device, (list, tuple)):
            ids = (ctypes.c_int * len(device))(*device)
            h = lib.cwg_create_multi(self.N, self.L, _p64(self.primes), self.t, relin_bits, galois_bits, ids,
                                     len(device))
        else:
            h = lib.cwg_create(self.N, self.L, _p64(self.primes), self.t, relin_bits, galois_bits, device)
        if not h:
            msg = lib.cwg_last_error().decode()
            if "CUDA" in msg or "cuda" in msg:
                raise CudaError(msg)
            raise ValueError(msg)
        self.h = h
        for key, value in (options or {}).items():
            self.set_option(key, value)

    def set_option(self, key: str, value: int):
        """cwg_set_option: tuning / test switches (see include/cwgpu.h)."""
        _raise(self.lib, self.lib.cwg_set_option(self.h, key.encode(), int(value)))

    def close(self):
        if getattr(self, "h", None):
            self.lib.cwg_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def info(self) -> CwgInfo:
        i = CwgInfo()
        _raise(self.lib, self.lib.cwg_get_info(self.h, ctypes.byref(i)))
        return i

    def load_db(self, positions, payload=None, n_total=None, row_begin=0, m=None):
        positions = np.ascontiguousarray(positions, dtype=np.uint32)
        n_local, k = positions.shape
        n_total = n_local if n_total is None else n_total
        if m is None:
            m = int(positions.max()) + 1
        if payload is None:
            s, pp = 0, None
        else:
            payload = _c64(payload)
            assert payload.shape[0] == n_local and payload.shape[2] == self.N
            s, pp = payload.shape[1], _p64(payload)
        _raise(self.lib, self.lib.cwg_load_db(self.h, n_total, row_begin, n_local, s, k, m, _p32(positions), pp))

    def load_db_bytes(self, payloads, k, m, n_total=None, row_begin=0, row_ids=None):
        """cwg_load_db_bytes: PirDatabase::setup from raw rows on the device.  payloads:
        [n_local][payload_bytes] uint8; row_ids: perfect_map inputs (keyword mode) or None
        (index mode: the global row index)."""
        payloads = np.ascontiguousarray(payloads, dtype=np.uint8)
        n_local, nbytes = payloads.shape
        n_total = n_local if n_total is None else n_total
        ids = None if row_ids is None else np.ascontiguousarray(row_ids, dtype=np.uint64)
        _raise(self.lib, self.lib.cwg_load_db_bytes(self.h, n_total, row_begin, n_local, k, m, nbytes,
                                                    payloads.ctypes.data, None if ids is None else ids.ctypes.data))

    def load_db_file(self, path_or_bytes, k, m):
        """cwg_load_db_file: the reference's CWDB database file (db_file.cpp) into the device."""
        data = path_or_bytes
        if isinstance(path_or_bytes, str):
            with open(path_or_bytes, "rb") as f:
                data = f.read()
        buf = np.frombuffer(data, dtype=np.uint8)
        _raise(self.lib, self.lib.cwg_load_db_file(self.h, buf.ctypes.data, buf.size, k, m))

    def set_keys(self, keys: Keys):
        relin, galois = _c64(keys.relin), _c64(keys.galois)
        gg = keys.exponents(self.N)
        _raise(self.lib, self.lib.cwg_set_keys(self.h, _p64(relin), galois.shape[0], _p64(gg), _p64(galois)))

    def _key_args(self, keys):
        if keys is None:
            return (None, 0, None, None), ()
        relin, galois = _c64(keys.relin), _c64(keys.galois)
        gg = keys.exponents(self.N)
        return (_p64(relin), galois.shape[0], _p64(gg), _p64(galois)), (relin, galois, gg)

    def answer(self, query, c, m, op=OP_FOLKLORE, keys=None, out=None, timings=False):
        """process_query (pir.cpp:337-347). query: [h][2][L][N]; returns [s][2][L][N]."""
        query = _c64(query)
        info = self.info()
        if out is None:
            out = np.zeros((info.s, 2, self.L, self.N), np.uint64)
        ka, keep = self._key_args(keys)
        tm = CwgTimings()
        rc = self.lib.cwg_answer(self.h, *ka, query.shape[0], c, m, query.ctypes.data, op, out.ctypes.data,
                                 ctypes.byref(tm) if timings else None)
        _raise(self.lib, rc)
        return (out, tm.as_dict()) if timings else out

    def answer_batch(self, queries, c, m, op=OP_FOLKLORE, keys=None, timings=False):
        """cwg_answer_batch: queries [Q][h][2][L][N] -> [Q][s][2][L][N] (one DB pass per tile)."""
        queries = _c64(queries)
        Q, h = queries.shape[0], queries.shape[1]
        info = self.info()
        out = np.zeros((Q, info.s, 2, self.L, self.N), np.uint64)
        ka, keep = self._key_args(keys)
        tm = CwgTimings()
        rc = self.lib.cwg_answer_batch(self.h, *ka, Q, h, c, m, queries.ctypes.data, op, out.ctypes.data,
                                       ctypes.byref(tm) if timings else None)
        _raise(self.lib, rc)
        return (out, tm.as_dict()) if timings else out

    def answer_ptr(self, query_ptr, h, c, m, op, out_ptr, keys_ptrs=(None, 0, None, None), timings=None):
        """Raw-pointer variant (pinned host buffers from torch) used by bench.py."""
        rc = self.lib.cwg_answer(self.h, *keys_ptrs, h, c, m, query_ptr, op, out_ptr,
                                 ctypes.byref(timings) if timings is not None else None)
        _raise(self.lib, rc)

    def answer_partial_ptr(self, query_ptr, h, c, m, op, dev_partial_ptr, keys_ptrs=(None, 0, None, None),
                           timings=None):
        rc = self.lib.cwg_answer_partial(self.h, *keys_ptrs, h, c, m, query_ptr, op, dev_partial_ptr,
                                         ctypes.byref(timings) if timings is not None else None)
        _raise(self.lib, rc)

    def partial_words(self) -> int:
        return int(self.lib.cwg_partial_words(self.h))

    def answer_partial(self, query, c, m, dev_partial_ptr, op=OP_FOLKLORE, keys=None, timings=None):
        query = _c64(query)
        ka, keep = self._key_args(keys)
        rc = self.lib.cwg_answer_partial(self.h, *ka, query.shape[0], c, m, query.ctypes.data, op, dev_partial_ptr,
                                         ctypes.byref(timings) if timings is not None else None)
        _raise(self.lib, rc)

    def shard_entries(self, c, world) -> int:
        """Expanded entries one rank of `world` produces (cwg_expand_shard): 2^c / world."""
        return (1 << c) // world

    def expand_shard_ptr(self, query_ptr, c, world, rank, out_ptr, keys_ptrs=(None, 0, None, None)):
        """cwg_expand_shard: this rank's subtree of expand_query (one query ciphertext) into the
        device buffer out_ptr ([2^c / world][2][L][N] u64)."""
        rc = self.lib.cwg_expand_shard(self.h, *keys_ptrs, c, query_ptr, world, rank, out_ptr)
        _raise(self.lib, rc)

    def answer_partial_shards_ptr(self, shards_ptr, world, c, m, op, dev_partial_ptr, timings=None):
        """cwg_answer_partial_shards: the partial answer from the rank-major gathered shards."""
        rc = self.lib.cwg_answer_partial_shards(self.h, shards_ptr, world, c, m, op, dev_partial_ptr,
                                                ctypes.byref(timings) if timings is not None else None)
        _raise(self.lib, rc)

    def finish(self, dev_partial_ptr, op=OP_FOLKLORE, out=None, timings=None):
        """cwg_finish; `out` may be an ndarray or a raw (host or device) pointer."""
        if out is None:
            info = self.info()
            out = np.zeros((info.s, 2, self.L, self.N), np.uint64)
        ptr = out.ctypes.data if isinstance(out, np.ndarray) else int(out)
        rc = self.lib.cwg_finish(self.h, dev_partial_ptr, op, ptr,
                                 ctypes.byref(timings) if timings is not None else None)
        _raise(self.lib, rc)
        return out

    def select_ptr(self, query, c, m, sel_ptr, op=OP_FOLKLORE, keys_ptrs=(None, 0, None, None), timings=None):
        """cwg_select into a raw (device or host) buffer of n_local x 3 x L x N words; returns comps."""
        query = _c64(query)
        comps = np.zeros(self.info().n_local, np.uint32)
        rc = self.lib.cwg_select(self.h, *keys_ptrs, query.shape[0], c, m, query.ctypes.data, op,
                                 ctypes.cast(sel_ptr, _u64p), _p32(comps),
                                 ctypes.byref(timings) if timings is not None else None)
        _raise(self.lib, rc)
        return comps

    def select(self, query, c, m, op=OP_FOLKLORE, keys=None, timings=False):
        """compute_selection_vector (pir.cpp:277-312): ([n][3][L][N], comps[n])."""
        query = _c64(query)
        info = self.info()
        sel = np.zeros((info.n_local, 3, self.L, self.N), np.uint64)
        comps = np.zeros(info.n_local, np.uint32)
        ka, keep = self._key_args(keys)
        tm = CwgTimings()
        rc = self.lib.cwg_select(self.h, *ka, query.shape[0], c, m, query.ctypes.data, op, _p64(sel), _p32(comps),
                                 ctypes.byref(tm) if timings else None)
        _raise(self.lib, rc)
        return (sel, comps, tm.as_dict()) if timings else (sel, comps)

    def encrypt_query(self, secret, bits, c, first_index=1):
        """cwg_encrypt_query: pack_query_bits + encrypt on the GPU.  secret = (s [N] int8, seed words [4])
        (Client.secret()); returns [h][2][L][N], equal to Client.pack_query for the same indices."""
        s, seed = secret
        s = np.ascontiguousarray(s, dtype=np.int8)
        seed = np.ascontiguousarray(seed, dtype=np.uint64)
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        h = -(-len(bits) // (1 << c))
        out = np.zeros((max(h, 1), 2, self.L, self.N), np.uint64)
        _raise(self.lib, self.lib.cwg_encrypt_query(self.h, _p64(seed), s.ctypes.data, bits.ctypes.data, len(bits), c,
                                                    first_index, out.ctypes.data))
        return out

    def decrypt(self, secret, cts):
        """cwg_decrypt: cts [count][comps][L][N] (or one [comps][L][N]) -> [count][N] (or [N])."""
        s = np.ascontiguousarray(secret[0], dtype=np.int8)
        cts = _c64(cts)
        single = cts.ndim == 3
        c4 = _c64(cts[None]) if single else cts
        out = np.zeros((c4.shape[0], self.N), np.uint64)
        _raise(self.lib, self.lib.cwg_decrypt(self.h, s.ctypes.data, c4.shape[0], c4.shape[1], c4.ctypes.data,
                                              out.ctypes.data))
        return out[0] if single else out

    def ntt(self, a, idx, chain=True, inverse=False):
        a = _c64(a).copy()
        count = a.size // self.N
        _raise(self.lib, self.lib.cwg_ntt(self.h, int(chain), idx, _p64(a), count, int(inverse)))
        return a

    def expand(self, query, c, m):
        query = _c64(query)
        out = np.zeros((m, 2, self.L, self.N), np.uint64)
        _raise(self.lib, self.lib.cwg_expand(self.h, query.shape[0], c, m, _p64(query), _p64(out)))
        return out

    def mul_lazy(self, a, b):
        a, b = _c64(a), _c64(b)
        single = a.ndim == 3
        a4, b4 = (a[None], b[None]) if single else (a, b)
        a4, b4 = _c64(a4), _c64(b4)
        out = np.zeros((a4.shape[0], 3, self.L, self.N), np.uint64)
        _raise(self.lib, self.lib.cwg_mul_lazy(self.h, a4.shape[0], _p64(a4), _p64(b4), _p64(out)))
        return out[0] if single else out

    def relinearize(self, ct3):
        ct3 = _c64(ct3)
        single = ct3.ndim == 3
        c4 = _c64(ct3[None]) if single else ct3
        out = np.zeros((c4.shape[0], 2, self.L, self.N), np.uint64)
        _raise(self.lib, self.lib.cwg_relinearize(self.h, c4.shape[0], _p64(c4), _p64(out)))
        return out[0] if single else out

    def substitute(self, ct, g):
        ct = _c64(ct)
        single = ct.ndim == 3
        c4 = _c64(ct[None]) if single else ct
        out = np.zeros_like(c4)
        _raise(self.lib, self.lib.cwg_substitute(self.h, c4.shape[0], _p64(c4), g, _p64(out)))
        return out[0] if single else out

    def kernel_launches(self) -> int:
        return int(self.lib.cwg_kernel_launches(self.h))

    def stream(self) -> int:
        """cudaStream_t of the context (for torch.cuda.ExternalStream / event timing)."""
        return int(self.lib.cwg_stream(self.h))

    def set_profiling(self, on: bool):
        _raise(self.lib, self.lib.cwg_set_profiling(self.h, int(on)))

    def kernel_stats(self, units: bool = False) -> dict:
        """{kernel: (total_ms, launches)} collected while profiling was on; with units=True
        {kernel: (total_ms, launches, algorithmic units)} (see cwg_kernel_units)."""
        out, i = {}, 0
        buf = ctypes.create_string_buffer(128)
        tot, cnt, u = ctypes.c_double(), ctypes.c_uint64(), ctypes.c_double()
        while self.lib.cwg_kernel_stats(self.h, i, buf, 128, ctypes.byref(tot), ctypes.byref(cnt)) == CWG_OK:
            if units:
                self.lib.cwg_kernel_units(self.h, i, ctypes.byref(u))
                out[buf.value.decode()] = (tot.value, cnt.value, u.value)
            else:
                out[buf.value.decode()] = (tot.value, cnt.value)
            i += 1
        return out


class Client:
    """Client side (keygen / query / decrypt) on the CPU; reproduces the reference's seeded keys."""

    def __init__(self, N, primes, t, seed, galois_levels, relin_bits=16, galois_bits=16):
        self.lib = lib = load_client_library()
        self.N, self.t = int(N), int(t)
        self.primes = _c64(primes)
        self.L = len(self.primes)
        self.levels = galois_levels
        h = lib.cwg_client_create(self.N, self.L, _p64(self.primes), self.t, relin_bits, galois_bits, seed,
                                  galois_levels)
        if not h:
            raise ValueError(lib.cwg_client_last_error().decode())
        self.h = h
        self.Dr = lib.cwg_client_digits(h, 0)
        self.Dg = lib.cwg_client_digits(h, 1)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.cwg_client_destroy(self.h)
            self.h = None

    def _check(self, rc):
        if rc != 0:
            raise ValueError(self.lib.cwg_client_last_error().decode())

    def keys(self) -> Keys:
        relin = np.zeros((self.Dr, 2, self.L, self.N), np.uint64)
        galois = np.zeros((self.levels, self.Dg, 2, self.L, self.N), np.uint64)
        self._check(self.lib.cwg_client_export_keys(self.h, _p64(relin), _p64(galois)))
        return Keys(relin, galois)

    def encrypt(self, plain, index):
        plain = _c64(plain)
        out = np.zeros((2, self.L, self.N), np.uint64)
        self._check(self.lib.cwg_client_encrypt(self.h, _p64(plain), index, _p64(out)))
        return out

    def pack_query(self, bits, c, first_index=1):
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        h = -(-len(bits) // (1 << c))
        out = np.zeros((h, 2, self.L, self.N), np.uint64)
        self._check(self.lib.cwg_client_pack_query(self.h, bits.ctypes.data_as(_u8p), len(bits), c, first_index,
                                                   _p64(out)))
        return out

    def secret(self):
        """(secret key coefficients [N] int8, Seed256 words [4]) for the GPU client calls."""
        s = np.zeros(self.N, np.int8)
        seed = np.zeros(4, np.uint64)
        self._check(self.lib.cwg_client_export_secret(self.h, s.ctypes.data, _p64(seed)))
        return s, seed

    def decrypt(self, ct):
        ct = _c64(ct)
        out = np.zeros(self.N, np.uint64)
        self._check(self.lib.cwg_client_decrypt(self.h, _p64(ct), ct.shape[0], _p64(out)))
        return out
