#!/usr/bin/env python
"""Benchmark: constant-weight PIR server answer on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cwgpu|reference] [--config C4]

One step = one server answer (process_query, reference pir.cpp:337-347) over the
whole database of the workload.  Default workload: config 4 (n = 65536 rows,
N = 8192, 5 x 43/44-bit chain primes, t = 1032193, k = 2, m = 363, c = 9, s = 1;
21.5 GB of NTT-form database), the configuration BASELINE's "1/2/4/8 B200" metric is
quoted on.  Synthetic seeded inputs (no public dataset), keys and query from the
client that reproduces the reference's seeded key generation.

value       = database GB/s scanned (n*s*L*N*8 bytes / answer time), inputs resident
              in HBM (keys, query, DB), device-timed with CUDA events, max over ranks.
e2e         = the same metric through cwg_answer with host buffers: the query and the
              evaluation keys (which the reference server receives with every query,
              server.cpp:63-68) copied H2D and the response D2H inside the timed region.
N > 1       = rows sharded contiguously (strong scaling), one NCCL sum of the
              partial NTT-domain accumulators to rank 0, which finishes (cwg_finish).
--impl reference = the reference C++ CPU implementation (oracle/_ref) on all host
              cores, on a bounded row sample extrapolated to the full database.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6650.0


IMAD_FALLBACK = 17999.2  # G IMAD lane-ops/s, profiles/r01_int_pipe_peaks.json


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


def imad_peak():
    try:
        with open(os.path.join(ROOT, "profiles", "r01_int_pipe_peaks.json")) as f:
            return float(json.load(f)["imad_gops"]), "measured (scripts/imad_peak.cu)"
    except Exception:
        return IMAD_FALLBACK, "measured constant"


# ncu --set full captures of the default C4 command (dram read + write bytes per launch) and the
# algorithmic units of the same launch, so `traffic` can be scaled to any launch of the kernel
def ncu_traffic():
    try:
        for tag in ("r02", "r01"):
            path = os.path.join(ROOT, "profiles", f"{tag}_ncu_traffic_C4.json")
            if os.path.exists(path):
                with open(path) as f:
                    return json.load(f)
        return {}
    except Exception:
        return {}


def rooflines(kstats, cfg, info, hbm, hbm_kind):
    """Per-kernel roofline from the profiled device times and the algorithmic work the
    library counted (cwg_kernel_units):
      NTT kernels (k_tensor_intt, k_ntt32r_sel3, ...): IMAD-bound; N/2 log2 N Shoup butterflies
        per polynomial at 4 IMAD slots each (IMAD.HI = 2 slots) vs the measured IMAD rate;
      k_round_tc / k_round_*: HBM; (J + Mm) 32-bit words per coefficient (read J residue planes,
        write Mm MAC-basis planes);
      k_mac: HBM; payload + selection words streamed."""
    import math

    ip, ip_kind = imad_peak()
    tr = ncu_traffic()
    out = {}
    N = cfg.N
    for name, (ms, cnt, units) in kstats.items():
        if ms <= 0 or cnt == 0:
            continue
        per_launch_s = ms / cnt / 1e3
        if name.startswith("k_ntt32r") or name == "k_tensor_intt":
            bfly = units / cnt * (N // 2) * int(math.log2(N))
            ach = bfly * 4 / per_launch_s / 1e9
            r = {"bound": "imad", "achieved": ach, "peak": ip, "unit": "G IMAD-slots/s", "frac": ach / ip,
                 "peak_kind": ip_kind, "work_per_launch": f"{units / cnt:.0f} polynomials x {N // 2 * int(math.log2(N))} "
                 "butterflies x 4 IMAD slots"}
        elif name == "k_ntt_mac":
            # fused forward NTT of the selection planes + payload MAC: IMAD-bound on the transform;
            # the HBM view counts the selection + payload words it streams (Z and DB planes)
            polys = units / cnt
            bfly = polys * (N // 2) * int(math.log2(N))
            ach = bfly * 4 / per_launch_s / 1e9
            nc = 3 if (cfg.op == 0 and cfg.k >= 2) else 2
            sel_bytes = polys * N * 4             # coefficient-domain selection planes, read once
            db_bytes_l = polys / nc * cfg.s * N * 4  # the rows' MAC-basis database planes, read once
            r = {"bound": "imad", "achieved": ach, "peak": ip, "unit": "G IMAD-slots/s", "frac": ach / ip,
                 "peak_kind": ip_kind, "work_per_launch": f"{polys:.0f} polynomials x {N // 2 * int(math.log2(N))} "
                 "butterflies x 4 IMAD slots (+ pointwise MAC)",
                 "hbm_view": {"achieved": (sel_bytes + db_bytes_l) / per_launch_s / 1e9, "peak": hbm, "unit": "GB/s",
                              "frac": (sel_bytes + db_bytes_l) / per_launch_s / 1e9 / hbm,
                              "db_only_frac": db_bytes_l / per_launch_s / 1e9 / hbm,
                              "bytes_per_launch": sel_bytes + db_bytes_l,
                              "what": "selection planes + database planes, each read once (DRAM view)"}}
        elif name == "k_round_chain":
            # exact rounding into the chain (selection output): J residue words read, L u64 written
            byt = units / cnt * (info.J * 4 + cfg.L * 8)
            ach = byt / per_launch_s / 1e9
            r = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm, "peak_kind": hbm_kind,
                 "work_per_launch": f"{units / cnt:.0f} coefficients x (4 J + 8 L) B"}
        elif name.startswith("k_round"):
            byt = units / cnt * (info.J + info.Mm) * 4
            ach = byt / per_launch_s / 1e9
            r = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm, "peak_kind": hbm_kind,
                 "work_per_launch": f"{units / cnt:.0f} coefficients x (J + Mm) x 4 B"}
        elif name in ("k_ks_mac32", "k_lift", "k_mac_to_chain"):
            # IMAD-bound dot products of 30-bit residues: k_ks_mac32 one IMAD.WIDE per digit product
            # (units = products), k_lift 2 L per (coefficient, output prime), k_mac_to_chain 2 per
            # (coefficient, MAC prime, chain prime) -- IMAD.WIDE = 2.4 IMAD slots
            per = {"k_ks_mac32": 1, "k_lift": 2 * cfg.L, "k_mac_to_chain": 2}[name]
            ach = units / cnt * per * 2.4 / per_launch_s / 1e9
            r = {"bound": "imad", "achieved": ach, "peak": ip, "unit": "G IMAD-slots/s", "frac": ach / ip,
                 "peak_kind": ip_kind, "work_per_launch": f"{units / cnt:.3e} units x {per} IMAD.WIDE x 2.4 slots"}
        elif name == "k_mac":
            byt = units / cnt  # selection planes + database planes, each read once
            ach = byt / per_launch_s / 1e9
            r = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm, "peak_kind": hbm_kind,
                 "work_per_launch": f"{byt:.3e} B (payload + selection words)"}
        else:
            continue
        t = tr.get(name)
        r["traffic"] = t["dram_bytes_per_unit"] * units / cnt if t else None
        r["launch_ms"] = ms / cnt
        r["ms_per_answer"] = ms
        out[name] = r
    return out


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 8:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        load = [s for s in sm if s > 0.5 * (max(sm) if sm else 1)]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------- helpers
def make_inputs(cfg, rank, world, seed=1):
    from paper_2202_07569_b200 import Client, configs

    lo = rank * cfg.n // world
    hi = (rank + 1) * cfg.n // world
    positions = configs.db_positions(cfg, seed)
    target = configs.query_row(cfg, seed)
    client = Client(cfg.N, cfg.primes, cfg.t, seed=seed, galois_levels=cfg.c, relin_bits=cfg.relin_bits,
                    galois_bits=cfg.galois_bits)
    keys = client.keys()
    query = client.pack_query(configs.codeword_bits(positions[target], cfg.m), cfg.c, first_index=1)
    return client, keys, query, positions, target, lo, hi


def reference_inputs(cfg, seed=1):
    """Keys and query for the reference arm from the REFERENCE itself (oracle/_ref: bfv_keygen with
    Seed256::from_u64(seed), pack_query_bits from encryption index 1) -- the same words the repo's
    client produces (pinned by tests/test_cpu_host.py), without mapping any repo library."""
    import oracle
    from paper_2202_07569_b200 import configs

    ref = oracle.RefLib()
    be = oracle.RefBackend(ref, cfg.N, cfg.t, np.array(cfg.primes, np.uint64), relin_bits=cfg.relin_bits,
                           galois_bits=cfg.galois_bits, seed=seed, galois_levels=cfg.c)
    positions = configs.db_positions(cfg, seed)
    target = configs.query_row(cfg, seed)
    query = be.pack_query(configs.codeword_bits(positions[target], cfg.m), cfg.c)
    return ref, be, query, positions


def cpu_reference_sample(cfg, be, ref, query, positions, seed=1, sample_rows=None):
    """The reference's own CPU path (oracle/_ref: expand_query, prepare_cipher, the per-row
    equality, weighted_sum, finalize -- pir.cpp:337-347's composition) on a bounded row sample.

    The sample's plaintexts are prepared (NTT form, prepare_plain) outside the timed stages, as
    the reference does offline (PirDatabase::prepare_for, pir.cpp:255-264).  The full answer is
    extrapolated: fixed per-query stages (expansion, prepare_cipher, finalize) as measured, plus
    the sample's per-row selection + inner-product time times n."""
    from paper_2202_07569_b200 import configs

    R = min(cfg.n, sample_rows or 4096)
    db = configs.db_payload(cfg, seed, 0, R)
    t0 = time.perf_counter()
    _, st = be.answer(query, cfg.c, cfg.m, positions[:R], db, op=cfg.op, tile_rows=R)
    wall = time.perf_counter() - t0
    t_expand, t_select, t_inner, t_final, t_prep, t_plain = [x / 1e3 for x in st]
    per_row = (t_select - t_prep + t_inner) / R
    full = t_expand + t_prep + per_row * cfg.n + t_final
    return {"seconds_full": full, "sample_rows": R, "sample_wall_s": wall, "threads": ref.worker_threads(),
            "stages_s": {"expand": t_expand, "prepare_cipher": t_prep, "select_per_row": (t_select - t_prep) / R,
                         "inner_per_row": t_inner / R, "finalize": t_final,
                         "prepare_plain_untimed": t_plain}}


def sample_rows_for(cfg, per_row_s, steps, budget_s=150.0, min_rows=4096):
    """Rows per reference sample so that `steps` samples take about budget_s, at least min_rows
    (4096 for the reference arm) and at most 8192 or the whole database."""
    per_row_s = max(per_row_s, 1e-6)
    rows = int(budget_s / max(steps, 1) / per_row_s)
    # the floor yields when even that would run past ~8 minutes (C5: ~35 ms per row on 16 threads)
    floor = min(min_rows, int(480.0 / max(steps, 1) / per_row_s))
    return int(min(cfg.n, max(floor, 64, min(rows, 8192))))


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def workload_desc(cfg):
    return (f"{cfg.name}: n={cfg.n} rows, N={cfg.N}, L={cfg.L} chain primes ({cfg.primes[0].bit_length()}-"
            f"{cfg.primes[-1].bit_length()} bit), t={cfg.t}, k={cfg.k}, m={cfg.m}, c={cfg.c}, s={cfg.s}, "
            f"op={'arith' if cfg.op else 'folklore'}")


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, cfg):
    """--impl reference: the reference's CPU implementation (oracle/_ref) on all host cores,
    keys / query / rows generated by the reference itself (no repo library is loaded)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    ref, be, query, positions = reference_inputs(cfg)
    if cfg.s == 0:
        return run_reference_select(args, cfg, ref, be, query, positions)
    probe = cpu_reference_sample(cfg, be, ref, query, positions, sample_rows=min(cfg.n, 256))
    per_row = probe["stages_s"]["select_per_row"] + probe["stages_s"]["inner_per_row"]
    R = args.cpu_sample_rows or sample_rows_for(cfg, per_row, args.steps)
    for _ in range(max(0, args.warmup - 1)):
        cpu_reference_sample(cfg, be, ref, query, positions, sample_rows=min(R, 256))
    runs, walls = [], []
    for _ in range(args.steps):
        runs.append(cpu_reference_sample(cfg, be, ref, query, positions, sample_rows=R))
        walls.append(runs[-1]["sample_wall_s"])
    secs = statistics.median(r["seconds_full"] for r in runs)
    gbps = cfg.db_bytes() / secs / 1e9
    sample = (f"each step: expand_query + prepare_cipher of the full query, then selection + weighted_sum on "
              f"{R} of {cfg.n} rows (plaintexts prepared beforehand, as prepare_for does offline), finalize; "
              f"full answer extrapolated linearly in rows ({secs:.1f} s); {runs[0]['threads']} threads, CPU {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": gbps, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.median(walls) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded rows/keys/query)", "config": bench_config(cfg),
        "cpu_baseline": {"value": gbps, "unit": "GB/s", "cores": runs[0]["threads"], "kind": "reference",
                         "sample": sample, "stages_s": runs[0]["stages_s"]},
        "e2e": {"value": gbps, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "answer_ms": secs * 1e3,
        "note": "ms_per_step is the measured wall time of one sample step; value and answer_ms are the "
                "full-database answer extrapolated from it",
    }
    print(json.dumps(line))
    return 0


def reference_select_sample(cfg, be, ref, query, positions, rows):
    """Config 2 on the reference: expand_query + prepare_cipher of the full query, then
    compute_selection_vector's per-row equality on `rows` of the 16384 codewords; the full
    selection time is extrapolated linearly in rows."""
    R = min(cfg.n, rows)
    t0 = time.perf_counter()
    _, _, st = be.select(query, cfg.c, cfg.m, positions[:R], stages=True)
    wall = time.perf_counter() - t0
    t_expand, t_prep, t_sel = [x / 1e3 for x in st]
    full = t_expand + t_prep + t_sel / R * cfg.n
    return {"seconds_full": full, "sample_rows": R, "sample_wall_s": wall, "threads": ref.worker_threads(),
            "stages_s": {"expand": t_expand, "prepare_cipher": t_prep, "select_per_row": t_sel / R}}


def run_reference_select(args, cfg, ref, be, query, positions):
    probe = reference_select_sample(cfg, be, ref, query, positions, 64)
    R = args.cpu_sample_rows or sample_rows_for(cfg, probe["stages_s"]["select_per_row"], args.steps)
    runs = [reference_select_sample(cfg, be, ref, query, positions, R) for _ in range(args.steps)]
    secs = statistics.median(r["seconds_full"] for r in runs)
    eqs = cfg.n / secs
    line = {
        "impl": "reference", "metric": SELECT_METRIC, "value": eqs, "unit": "equalities/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(r["sample_wall_s"] for r in runs) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded codewords/keys/query)",
        "config": bench_config(cfg),
        "cpu_baseline": {"value": eqs, "unit": "equalities/s", "cores": runs[0]["threads"], "kind": "reference",
                         "sample": f"each step: expand_query + prepare_cipher of the full query, then the per-row "
                                   f"equality on {R} of {cfg.n} codewords; extrapolated linearly in rows "
                                   f"({secs:.1f} s for all); CPU {cpu_model()}", "stages_s": runs[0]["stages_s"]},
        "e2e": {"value": eqs, "unit": "equalities/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "select_ms": secs * 1e3,
        "note": "ms_per_step is the measured wall time of one sample step; value is the full 16384-codeword "
                "selection extrapolated from it",
    }
    print(json.dumps(line))
    return 0


def run_select_bench(args, cfg):
    """Config 2 (equality-operator microbenchmark): compute_selection_vector over the 16384
    seeded weight-k codewords, no payload.  value: equalities per second with the query and keys
    resident and the selection written to device memory (expansion included: it is part of the
    operator's cost, and at k = 1 it is all of it); e2e: the same through cwg_select with the
    query and keys from pinned host memory and the whole selection (n x 3 x L x N words) read back."""
    import ctypes

    import torch

    from paper_2202_07569_b200 import Context
    from paper_2202_07569_b200.cwgpu import CwgTimings

    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        raise SystemExit("the config-2 microbenchmark runs on one GPU")
    client, keys, query, positions, target, lo, hi = make_inputs(cfg, 0, 1)
    options = {kv.split("=", 1)[0]: int(kv.split("=", 1)[1]) for kv in args.opt}
    ctx = Context(cfg.N, cfg.primes, cfg.t, relin_bits=cfg.relin_bits, galois_bits=cfg.galois_bits, options=options)
    ctx.load_db(positions, None, m=cfg.m)
    ctx.set_keys(keys)
    info = ctx.info()
    LN = cfg.L * cfg.N
    sel = torch.empty(cfg.n * 3 * LN, dtype=torch.int64, device="cuda")
    ext = torch.cuda.ExternalStream(ctx.stream())
    u64p = ctypes.POINTER(ctypes.c_uint64)
    hrelin = torch.from_numpy(keys.relin.view(np.int64).reshape(-1).copy()).pin_memory()
    hgal = torch.from_numpy(keys.galois.view(np.int64).reshape(-1).copy()).pin_memory()
    hg = np.ascontiguousarray(keys.exponents(cfg.N))
    key_ptrs = (ctypes.cast(hrelin.data_ptr(), u64p), keys.galois.shape[0], hg.ctypes.data_as(u64p),
                ctypes.cast(hgal.data_ptr(), u64p))
    hq = np.ascontiguousarray(query)
    hsel = np.empty(cfg.n * 3 * LN, np.uint64)

    def timed(fn, steps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        for _ in range(steps):
            fn()
        e1.record(ext)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    step = lambda: ctx.select_ptr(hq, cfg.c, cfg.m, sel.data_ptr())
    for _ in range(args.warmup):
        step()
    l0 = ctx.kernel_launches()
    clk = ClockSampler(0)
    clk.start()
    ms = timed(step, args.steps)
    clocks = clk.stop()
    launches = (ctx.kernel_launches() - l0) // args.steps
    t0 = time.perf_counter()
    e2e_steps = max(1, min(args.steps, 3))
    for _ in range(e2e_steps):
        comps = ctx.select_ptr(hq, cfg.c, cfg.m, hsel.ctypes.data, keys_ptrs=key_ptrs)
    ms_e2e = (time.perf_counter() - t0) / e2e_steps * 1e3
    verified = None
    if not args.no_verify:  # matching rows decrypt to 1, the others to 0 (constant coefficient)
        dsel = sel.cpu().numpy().view(np.uint64).reshape(cfg.n, 3, cfg.L, cfg.N)
        match = np.all(positions == positions[target], axis=1)
        picks = list(np.flatnonzero(match)[:4]) + list(np.flatnonzero(~match)[:4])
        verified = bool(all(client.decrypt(dsel[r, :comps[r]])[0] == int(match[r]) for r in picks)) and bool(
            np.array_equal(hsel.reshape(dsel.shape), dsel))
        del dsel
    ctx.set_profiling(True)
    tm = CwgTimings()
    ctx.select_ptr(hq, cfg.c, cfg.m, sel.data_ptr(), timings=tm)
    kstats = ctx.kernel_stats(units=True)
    ctx.set_profiling(False)
    hbm, peak_kind = peaks()
    roof = rooflines(kstats, cfg, info, hbm, peak_kind)
    tot = sum(v[0] for v in kstats.values())
    dom = max(kstats.items(), key=lambda kv: kv[1][0]) if kstats else ("", (0, 0, 0))
    top = dict(roof.get(dom[0], {}))
    if top:
        top = {"kernel": dom[0], **top, "share_of_step": dom[1][0] / tot if tot else None}
    line = {
        "metric": SELECT_METRIC, "value": cfg.n / (ms / 1e3), "unit": "equalities/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded codewords/keys/query)",
        "config": bench_config(cfg),
        "layout": {"rows_per_gpu": cfg.n, "l2": "selection output 16 GB >> L2", "aux_primes": info.J},
        "select_ms": ms,
        "e2e": {"value": cfg.n / (ms_e2e / 1e3), "unit": "equalities/s", "select_ms": ms_e2e,
                "h2d_bytes_per_step": int(query.nbytes + keys.relin.nbytes + keys.galois.nbytes),
                "d2h_bytes_per_step": int(hsel.nbytes + 4 * cfg.n), "timing": "host wall clock (synchronous call)"},
        "gpu_launches": int(launches), "clocks": clocks, "roofline": top or None, "rooflines": roof,
        "kernels_ms_per_step": {k: round(v[0], 3) for k, v in sorted(kstats.items(), key=lambda kv: -kv[1][0])},
        "stages_ms": {k: getattr(tm, k) for k in ("expand_ms", "select_ms")},
        "exact_fallbacks": int(tm.exact_fallbacks), "verified_decrypt": verified,
    }
    if not args.no_cpu_baseline:
        try:
            import oracle

            ref = oracle.RefLib()
            be = oracle.RefBackend(ref, cfg.N, cfg.t, np.array(cfg.primes, np.uint64), keys=(keys.relin, keys.galois))
            probe = reference_select_sample(cfg, be, ref, query, positions, 64)
            R = args.cpu_sample_rows or sample_rows_for(cfg, probe["stages_s"]["select_per_row"], 1, budget_s=20.0,
                                                        min_rows=64)
            cb = reference_select_sample(cfg, be, ref, query, positions, R)
            line["cpu_baseline"] = {
                "value": cfg.n / cb["seconds_full"], "unit": "equalities/s", "cores": cb["threads"], "kind": "reference",
                "sample": f"reference compute_selection_vector (oracle/_ref): expand_query + prepare_cipher of the "
                          f"full query, per-row equality on {R} of {cfg.n} codewords, extrapolated linearly in rows "
                          f"({cb['seconds_full']:.1f} s for all); CPU {cpu_model()}",
                "select_s": cb["seconds_full"], "stages_s": cb["stages_s"]}
        except Exception as e:
            line["cpu_baseline"] = {"value": None, "unit": "equalities/s", "cores": os.cpu_count(),
                                    "kind": "reference", "sample": f"unavailable: {e}"}
    print(json.dumps(line))
    return 0


SELECT_METRIC = "equalities_per_s"
METRIC = "db_GBps_scanned"


def bench_config(cfg):
    """The `config` object, identical in both arms for the same workload."""
    return {"workload": workload_desc(cfg), "db_bytes": cfg.db_bytes()}


# ----------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cwgpu", choices=["cwgpu", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--rows", type=int, default=0, help="override n (quick runs only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-rows", type=int, default=0)
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--batch", type=int, default=0,
                    help="also time cwg_answer_batch with this many queries (SURVEY 8f-f1; reported under 'batch')")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="N > 1 collectives: nccl (one GPU per rank) or gloo (host-staged; ranks may share a GPU)")
    ap.add_argument("--opt", action="append", default=[], metavar="KEY=VALUE",
                    help="library option (cwg_set_option), e.g. --opt tile_rows=256 --opt streams=2")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "cwgpu" else args.warmup

    from paper_2202_07569_b200 import configs

    cfg = configs.config(args.config)
    if args.rows:
        cfg.n = args.rows
    if args.impl == "reference":
        return run_reference(args, cfg)
    if cfg.s == 0:
        return run_select_bench(args, cfg)

    import torch

    from paper_2202_07569_b200 import Context
    from paper_2202_07569_b200.cwgpu import CwgTimings as CwgTimings_type

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # --dist-backend gloo (harness only): ranks may share a GPU, collectives host-staged
    if args.dist_backend == "gloo":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.dist_backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    client, keys, query, positions, target, lo, hi = make_inputs(cfg, rank, world)
    payload = configs.db_payload(cfg, 1, lo, hi)
    options = {kv.split("=", 1)[0]: int(kv.split("=", 1)[1]) for kv in args.opt}
    ctx = Context(cfg.N, cfg.primes, cfg.t, relin_bits=cfg.relin_bits, galois_bits=cfg.galois_bits, device=local,
                  options=options)
    t_load = time.perf_counter()
    ctx.load_db(positions[lo:hi], payload, n_total=cfg.n, row_begin=lo, m=cfg.m)
    t_load = time.perf_counter() - t_load
    info = ctx.info()
    ctx.set_keys(keys)
    L, N = cfg.L, cfg.N
    resp_words = cfg.s * 2 * L * N
    ext = torch.cuda.ExternalStream(ctx.stream())

    # device-resident inputs for `value`; pinned host buffers for `e2e`
    dq = torch.from_numpy(query.view(np.int64)).cuda()
    dout = torch.zeros(resp_words, dtype=torch.int64, device="cuda")
    hq = torch.from_numpy(query.view(np.int64).copy()).pin_memory()
    hrelin = torch.from_numpy(keys.relin.view(np.int64).reshape(-1).copy()).pin_memory()
    hgal = torch.from_numpy(keys.galois.view(np.int64).reshape(-1).copy()).pin_memory()
    hg = np.ascontiguousarray(keys.exponents(N))
    hout = torch.zeros(resp_words, dtype=torch.int64).pin_memory()
    import ctypes

    u64p = ctypes.POINTER(ctypes.c_uint64)
    key_ptrs = (ctypes.cast(hrelin.data_ptr(), u64p), keys.galois.shape[0], hg.ctypes.data_as(u64p),
                ctypes.cast(hgal.data_ptr(), u64p))
    h_q = query.shape[0]
    rs = None
    if world > 1:
        from paper_2202_07569_b200.rowshard import RowShardStep

        rs = RowShardStep(ctx, cfg, rank, world, backend=args.dist_backend)
    shard = rs is not None and rs.shard

    def step_value():
        if world == 1:
            ctx.answer_ptr(dq.data_ptr(), h_q, cfg.c, cfg.m, cfg.op, dout.data_ptr())
        else:
            rs.step(dq.data_ptr(), dout.data_ptr())

    def step_e2e():
        if world == 1:
            ctx.answer_ptr(hq.data_ptr(), h_q, cfg.c, cfg.m, cfg.op, hout.data_ptr(), keys_ptrs=key_ptrs)
        else:
            rs.step(hq.data_ptr(), hout.data_ptr(), key_ptrs)

    def timed(fn, steps):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream = ext if world == 1 else torch.cuda.current_stream()
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        if dist:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms

    for _ in range(args.warmup):
        step_value()
    launches0 = ctx.kernel_launches()
    clk = ClockSampler(local)
    clk.start()
    ms = timed(step_value, args.steps)
    clocks = clk.stop()
    launches = (ctx.kernel_launches() - launches0) // args.steps
    for _ in range(1):
        step_e2e()
    ms_e2e = timed(step_e2e, args.steps)

    # correctness of the benchmarked answer: the response decrypts to the selected row
    verified = None
    verify_detail = None
    if rank == 0 and not args.no_verify:
        resp = dout.cpu().numpy().view(np.uint64).reshape(cfg.s, 2, L, N)
        trow = configs.db_payload(cfg, 1, target, target + 1)[0]
        dec_ok = all(np.array_equal(client.decrypt(resp[j]), trow[j]) for j in range(cfg.s))
        hresp = hout.numpy().view(np.uint64).reshape(cfg.s, 2, L, N)
        e2e_eq = bool(np.array_equal(hresp, resp))
        verified = bool(dec_ok and e2e_eq)
        verify_detail = {"decrypt_equals_row": bool(dec_ok), "e2e_response_equals_device_response": e2e_eq}

    # multi-query batch (f1): Q queries of one client per database pass, timed like `value`
    batch_line = None
    if args.batch > 1 and world == 1:
        qb = np.stack([client.pack_query(configs.codeword_bits(positions[(target + 97 * b) % cfg.n], cfg.m), cfg.c,
                                         first_index=100 + 10 * b) for b in range(args.batch)])
        qb = np.ascontiguousarray(qb)
        ctx.answer_batch(qb, cfg.c, cfg.m, op=cfg.op)
        bms = timed(lambda: ctx.answer_batch(qb, cfg.c, cfg.m, op=cfg.op), max(1, args.steps // 2))
        batch_line = {"queries": args.batch, "ms_per_batch": bms, "ms_per_query": bms / args.batch,
                      "value_per_query": cfg.db_bytes() / (bms / args.batch / 1e3) / 1e9, "unit": "GB/s",
                      "timing": "CUDA events around cwg_answer_batch (synchronous, host query buffers)"}

    # N > 1: per-rank phase times of one more answer (outside the timed region)
    rank_rows = None
    if world > 1:
        mine = rs.phase_times(dq.data_ptr(), dout.data_ptr())
        rank_rows = [None] * world
        dist.all_gather_object(rank_rows, mine)

    # per-kernel device times (profiling pass, outside the timed region)
    ctx.set_profiling(True)
    tm = CwgTimings_type()
    if world == 1:
        ctx.answer_ptr(dq.data_ptr(), h_q, cfg.c, cfg.m, cfg.op, dout.data_ptr(), timings=tm)
    else:
        ctx.answer_partial_ptr(dq.data_ptr(), h_q, cfg.c, cfg.m, cfg.op, rs.partial.data_ptr(), timings=tm)
    kstats = ctx.kernel_stats(units=True)
    ctx.set_profiling(False)

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0

    hbm, peak_kind = peaks()
    db_bytes = cfg.db_bytes()
    value = db_bytes / (ms / 1e3) / 1e9
    e2e = db_bytes / (ms_e2e / 1e3) / 1e9
    roof = rooflines(kstats, cfg, info, hbm, peak_kind)
    tot_prof = sum(v[0] for v in kstats.values())
    dom = max(kstats.items(), key=lambda kv: kv[1][0]) if kstats else ("", (0, 0, 0))
    local_rows = hi - lo
    top = dict(roof.get(dom[0], {}))
    if top:
        top = {"kernel": dom[0], **top, "share_of_step": dom[1][0] / tot_prof if tot_prof else None}
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded rows/keys/query)",
        "config": bench_config(cfg),
        "layout": {"rows_per_gpu": local_rows,
                   "parallelism": f"row-shard x{world}" + (" + expansion-shard (all-gather)" if shard else ""),
                   "l2": "no flush: DB >> 126 MB L2" if db_bytes > 2e9 else "inputs larger than L2" if db_bytes > 2e8
                   else "small (L2-resident)", "aux_primes": info.J, "mac_primes": info.Mm},
        "answer_ms": ms,
        "e2e": {"value": e2e, "unit": "GB/s", "answer_ms": ms_e2e,
                "h2d_bytes_per_step": int(query.nbytes + keys.relin.nbytes + keys.galois.nbytes),
                "d2h_bytes_per_step": int(resp_words * 8)},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "roofline": top or None,
        "rooflines": roof,
        "kernels_ms_per_answer": {k: round(v[0], 3) for k, v in sorted(kstats.items(), key=lambda kv: -kv[1][0])},
        "dominant_kernel": {"name": dom[0], "share_of_step": dom[1][0] / tot_prof if tot_prof else None},
        "stages_ms": {k: getattr(tm, k) for k in ("expand_ms", "select_ms", "mac_ms", "finish_ms")},
        "exact_fallbacks": int(tm.exact_fallbacks),
        "verified_decrypt": verified,
        "verify_detail": verify_detail,
        "db_load_s": t_load,
    }
    if "k_mac" in roof:  # north_star: the payload MAC against HBM bandwidth (separate kernel when s >= 3)
        pm = roof["k_mac"]
        line["payload_mac"] = {"kernel": "k_mac", "bound": "hbm", "achieved": pm["achieved"], "peak": pm["peak"],
                               "unit": "GB/s", "frac": pm["frac"], "ms_per_answer": pm["ms_per_answer"],
                               "what": "database planes + selection planes, each read once"}
    elif "k_ntt_mac" in roof and "hbm_view" in roof["k_ntt_mac"]:
        line["payload_mac"] = {"kernel": "k_ntt_mac (fused with the selection NTT, IMAD-bound)",
                               **roof["k_ntt_mac"]["hbm_view"]}
    if rank_rows:
        line["ranks"] = rank_rows
    if batch_line:
        line["batch"] = batch_line
    if world == 1 and not args.no_cpu_baseline:
        try:
            import oracle

            ref = oracle.RefLib()
            be = oracle.RefBackend(ref, cfg.N, cfg.t, np.array(cfg.primes, np.uint64), relin_bits=cfg.relin_bits,
                                   galois_bits=cfg.galois_bits, keys=(keys.relin, keys.galois))
            probe = cpu_reference_sample(cfg, be, ref, query, positions, sample_rows=min(cfg.n, 256))
            per_row = probe["stages_s"]["select_per_row"] + probe["stages_s"]["inner_per_row"]
            R = args.cpu_sample_rows or sample_rows_for(cfg, per_row, 1, budget_s=20.0, min_rows=256)
            cb = cpu_reference_sample(cfg, be, ref, query, positions, sample_rows=R)
            line["cpu_baseline"] = {
                "value": db_bytes / cb["seconds_full"] / 1e9, "unit": "GB/s", "cores": cb["threads"],
                "kind": "reference",
                "sample": f"reference process_query composition (oracle/_ref): expand_query + prepare_cipher of the "
                          f"full query, selection + weighted_sum on {cb['sample_rows']} of {cfg.n} rows (plaintexts "
                          f"prepared beforehand, as prepare_for does offline), finalize; extrapolated linearly in "
                          f"rows ({cb['seconds_full']:.1f} s full answer); CPU {cpu_model()}",
                "answer_s": cb["seconds_full"], "stages_s": cb["stages_s"]}
        except Exception as e:  # the baseline must not hide the GPU line
            line["cpu_baseline"] = {"value": None, "unit": "GB/s", "cores": os.cpu_count(), "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
