"""One process per GPU: the row-sharded server answer over torch.distributed.

Rank r holds rows [r n / W, (r + 1) n / W) (cwg_load_db with row_begin).  Per answer:

  expansion   one query ciphertext and W a power of two <= 2^c: rank r expands the subtree of
              leaves r, r + W, ... (cwg_expand_shard) and an all-gather hands every rank all
              entries rank-major (cwg_answer_partial_shards restores the order); otherwise
              every rank expands the whole query (cwg_answer_partial);
  rows        selection + payload MAC of the local rows into partial accumulators
              (s x 3 x Mm x N u64 words, each < 2^31);
  reduction   one sum of the partials to rank 0 (u64 adds, no overflow for W < 2^33);
  finish      rank 0: cwg_finish (mod a_k, INTT, MAC basis -> chain, relinearisation).

backend "nccl": collectives on device tensors (one GPU per rank).  backend "gloo": the same
collectives on host-staged copies -- for several ranks sharing one GPU in tests (NCCL refuses
two ranks on one device); the library calls are identical.
The in-process alternative for a C++ caller is cwg_create_multi (include/cwgpu.h).
"""
from __future__ import annotations

import numpy as np


class RowShardStep:
    def __init__(self, ctx, cfg, rank: int, world: int, backend: str = "nccl", shard_expansion: bool = True):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.ctx, self.cfg, self.rank, self.world = ctx, cfg, rank, world
        self.gloo = backend == "gloo"
        self.ext = torch.cuda.ExternalStream(ctx.stream())
        L, N = cfg.L, cfg.N
        self.h_q = -(-cfg.m // (1 << cfg.c))
        self.shard = shard_expansion and self.h_q == 1 and (world & (world - 1)) == 0 and world <= (1 << cfg.c)
        dev = "cuda"
        self.partial = torch.zeros(ctx.partial_words(), dtype=torch.int64, device=dev)
        if self.shard:
            words = ctx.shard_entries(cfg.c, world) * 2 * L * N
            self.shard_local = torch.zeros(words, dtype=torch.int64, device=dev)
            self.shards_all = torch.zeros(world * words, dtype=torch.int64, device=dev)
        self.collective_ms = 0.0

    def _after_collective(self):
        # the library runs on its own stream: order it after the collective on torch's stream
        self.ext.wait_stream(self.torch.cuda.current_stream())

    def _all_gather(self):
        if self.gloo:
            self.torch.cuda.synchronize()
            loc = self.shard_local.cpu()
            parts = [self.torch.empty_like(loc) for _ in range(self.world)]
            self.dist.all_gather(parts, loc)
            self.shards_all.copy_(self.torch.cat(parts))
        else:
            self.dist.all_gather_into_tensor(self.shards_all, self.shard_local)
        self._after_collective()

    def _reduce(self):
        if self.gloo:
            self.torch.cuda.synchronize()
            host = self.partial.cpu()
            self.dist.reduce(host, dst=0)
            if self.rank == 0:
                self.partial.copy_(host)
        else:
            self.dist.reduce(self.partial, dst=0)
        self._after_collective()

    def partial_step(self, q_ptr, keys_ptrs=(None, 0, None, None)):
        """Everything up to (and including) the reduction; rank 0's self.partial holds the sum."""
        cfg = self.cfg
        if self.shard:
            self.ctx.expand_shard_ptr(q_ptr, cfg.c, self.world, self.rank, self.shard_local.data_ptr(),
                                      keys_ptrs=keys_ptrs)
            self._all_gather()
            self.ctx.answer_partial_shards_ptr(self.shards_all.data_ptr(), self.world, cfg.c, cfg.m, cfg.op,
                                               self.partial.data_ptr())
        else:
            self.ctx.answer_partial_ptr(q_ptr, self.h_q, cfg.c, cfg.m, cfg.op, self.partial.data_ptr(),
                                        keys_ptrs=keys_ptrs)
        self._reduce()

    def phase_times(self, q_ptr, out_ptr):
        """One answer with the phases timed on this rank (host wall clock around synchronised
        phases; diagnostics outside the timed region): ms for expansion (shard), the all-gather,
        the rows (selection + MAC), the reduction and, on rank 0, the finish."""
        import time

        cfg, t, torch = self.cfg, {}, self.torch

        def mark(name, t0):
            torch.cuda.synchronize()
            t[name] = (time.perf_counter() - t0) * 1e3
            return time.perf_counter()

        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if self.shard:
            self.ctx.expand_shard_ptr(q_ptr, cfg.c, self.world, self.rank, self.shard_local.data_ptr())
            t0 = mark("expand_shard_ms", t0)
            self._all_gather()
            t0 = mark("all_gather_ms", t0)
            self.ctx.answer_partial_shards_ptr(self.shards_all.data_ptr(), self.world, cfg.c, cfg.m, cfg.op,
                                               self.partial.data_ptr())
            t0 = mark("rows_ms", t0)
        else:
            self.ctx.answer_partial_ptr(q_ptr, self.h_q, cfg.c, cfg.m, cfg.op, self.partial.data_ptr())
            t0 = mark("expand_and_rows_ms", t0)
        self._reduce()
        t0 = mark("reduce_ms", t0)
        if self.rank == 0:
            self.ctx.finish(self.partial.data_ptr(), cfg.op, out=out_ptr)
            mark("finish_ms", t0)
        info = self.ctx.info()
        return {"rank": self.rank, "rows": int(info.n_local), "row_begin": int(info.row_begin),
                **{k: round(v, 3) for k, v in t.items()}}

    def step(self, q_ptr, out_ptr, keys_ptrs=(None, 0, None, None)):
        """One whole answer; rank 0 writes the response to out_ptr (host or device)."""
        self.partial_step(q_ptr, keys_ptrs)
        if self.rank == 0:
            self.ctx.finish(self.partial.data_ptr(), self.cfg.op, out=out_ptr)

    def answer(self, query: np.ndarray, keys=None) -> np.ndarray | None:
        """Convenience wrapper: host query in, rank 0 gets the [s][2][L][N] response."""
        query = np.ascontiguousarray(query, dtype=np.uint64)
        out = np.zeros((self.cfg.s, 2, self.cfg.L, self.cfg.N), np.uint64)
        ka, keep = self.ctx._key_args(keys)
        self.step(query.ctypes.data, out.ctypes.data, ka)
        return out if self.rank == 0 else None
