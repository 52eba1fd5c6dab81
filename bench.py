#!/usr/bin/env python
"""Benchmark of the hash-SpGEMM hot path (BASELINE.json metric: SpGEMM GFLOPS =
2 * flop / t, sorted and unsorted C, % of the HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME]
                    [--impl ours|reference]

A step is one full C = A*B (flop count, binning, symbolic, scan, allocation of
C, numeric, and the per-row sort when sorted) on synthetic inputs already
resident in HBM; L2 is flushed (256 MiB write) between timed steps, outside
the per-step CUDA events.  Multi-GPU (torchrun): A's rows are split by
balanced flop (Fig:load_balance, computed on the GPU), B is broadcast once
with NCCL, each rank multiplies its row block; time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# C of the large configs is >100 GB: avoid caching-allocator fragmentation
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

DEFAULT_CONFIG = "c3_rmat20"      # the largest single-GPU config (configs[2]); C2 etc. via --config
L2_FLUSH_BYTES = 256 << 20
FALLBACK_HBM_GBS = 6650.0          # B200_PROFILING.md fallback


METRIC = "SpGEMM GFLOPS (2*flop/s), sorted C (unsorted in variants)"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except ValueError:
                continue
            for n, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(mx)) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- workload
def make_workload(name: str):
    import synth
    A, B, extra = synth.workload(name)
    return A, B, extra


def bin_of_rows_num(nnz_c: np.ndarray) -> np.ndarray:
    """Numeric bin of each row (same rule as the library: T = max(32,
    pow2ceil(2 nnz)); bins W256 / W1024 / B2K..B16K / G).  Accounting only."""
    lg = np.zeros(len(nnz_c), np.int64)
    nz = nnz_c > 0
    lg[nz] = np.maximum(5, np.ceil(np.log2(2 * nnz_c[nz])).astype(np.int64))
    b = np.zeros(len(nnz_c), np.int64)
    b[nz & (lg <= 8)] = 1
    b[nz & (lg > 8) & (lg <= 10)] = 2
    mid = nz & (lg >= 11) & (lg <= 14)
    b[mid] = 3 + (lg[mid] - 11)
    b[nz & (lg > 14)] = 7
    return b


def bin_of_rows_sym(flop: np.ndarray, ncols: int) -> np.ndarray:
    """Symbolic bin of each row (library rule: T = max(32, lowest 2^n >
    min(flop, ncols)); W128 / W1024 / B2K..B8K; above: BM bitmap when ncols <=
    1.6M, else B16K / B32K / G).  Accounting only."""
    s = np.minimum(flop, ncols)
    lg = np.zeros(len(flop), np.int64)
    nz = flop > 0
    lg[nz] = np.floor(np.log2(np.maximum(s[nz], 1))).astype(np.int64) + 1
    lg[nz] = np.maximum(lg[nz], 5)
    b = np.zeros(len(flop), np.int64)
    b[nz & (lg <= 7)] = 1
    b[nz & (lg > 7) & (lg <= 10)] = 2
    mid = nz & (lg >= 11) & (lg <= 13)
    b[mid] = 3 + (lg[mid] - 11)
    big = nz & (lg >= 14)
    if ncols <= 200 * 1024 * 8:
        b[big] = 9
    else:
        b[big & (lg <= 15)] = 3 + (lg[big & (lg <= 15)] - 11)
        b[big & (lg > 15)] = 8
    return b


NUM_KERNEL_BIN = {"k_num_warp<256>": [1], "k_num_warp<1024>": [2],
                  "k_num_block<128>": [3], "k_num_block<512>": [4, 5], "k_num_block<1024>": [6],
                  "k_num_global<1024>": [7], "k_num_tpart<512>": [7]}
SYM_KERNEL_BIN = {"k_sym_warp<128>": [1], "k_sym_warp<1024>": [2],
                  "k_sym_block<128>": [3, 4], "k_sym_block<256>": [5], "k_sym_block<1024>": [6, 7],
                  "k_sym_bitmap<1024>": [9], "k_sym_global<1024>": [8]}


def kernel_bytes(name: str, a_nnz_row, flop_row, c_nnz_row, m, nnzA, ncols, krows):
    """Algorithmic bytes per launch of kernel `name`:
    numeric: A row read (8 + 12 nnz(a_i)), gathered B rows (12 flop_i), C row
    write (8 + 12 nnz(c_i)); symbolic: 8 + 4 nnz(a_i) + 4 flop_i + 8;
    flop kernel: row_ptr + A.col + flop[] write."""
    if name in NUM_KERNEL_BIN:
        sel = np.isin(bin_of_rows_num(c_nnz_row), NUM_KERNEL_BIN[name])
        return float((16 + 12 * a_nnz_row[sel] + 12 * flop_row[sel] + 12 * c_nnz_row[sel]).sum())
    if name in SYM_KERNEL_BIN:
        sel = np.isin(bin_of_rows_sym(flop_row, ncols), SYM_KERNEL_BIN[name])
        return float((16 + 4 * a_nnz_row[sel] + 4 * flop_row[sel]).sum())
    if name == "k_flop_nz":
        return float(8 * (m + 1) + 4 * nnzA + 8 * m + 8 * (krows + 1))
    return None


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(config: str, kernel: str):
    """dram read+write bytes per launch of `kernel` from a committed ncu --set
    full capture summary (profiles/traffic.json), else None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(p))
        return d.get(config, {}).get(kernel)
    except Exception:
        return None


# ----------------------------------------------------------------------------- oracle
def row_sample(A, of, frac: float, seed: int = 2024):
    """Sub-matrix of A made of a seeded uniform random sample of its rows
    (every row equally likely, so hub and empty rows appear in proportion):
    returns (sub-A, sampled flop).  Host-side input preparation only."""
    import synth
    rng = np.random.default_rng(seed)
    m = A.nrows
    k = max(1, min(m, int(round(m * frac))))
    rows = np.sort(rng.choice(m, size=k, replace=False))
    lens = np.diff(A.row_ptr)[rows]
    rp = np.zeros(k + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    idx = np.repeat(A.row_ptr[rows] - rp[:-1], lens) + np.arange(int(rp[-1]), dtype=np.int64)
    sub = synth.CSR(k, A.ncols, rp, A.col[idx].astype(np.int32), A.val[idx].astype(np.float64))
    return sub, int(of[rows].sum()), k


def oracle_sample(A, B, target_s: float = 12.0, nthreads: int = 0, reps_min_s: float = 3.0):
    """Time the oracle (as it stands) on a bounded, representative sample of
    the workload: a seeded uniform random sample of A's rows (times B), sized
    to ~target_s of CPU work from a calibration run."""
    import oracle
    of, tot = oracle.flop(A, B)
    nthreads = nthreads or (os.cpu_count() or 1)
    frac = 0.002
    sub, f, k = row_sample(A, of, frac)
    t0 = time.perf_counter()
    oracle.spgemm(sub, B, nthreads=nthreads)
    dt = max(time.perf_counter() - t0, 1e-6)
    rate = max(f, 1) / dt
    frac = min(1.0, frac * max(1.0, target_s * rate / max(f, 1)) if f else 1.0)
    sub, f, k = row_sample(A, of, frac)
    reps, dt = 0, 0.0
    while reps == 0 or (dt < reps_min_s and reps < 50):  # tiny workloads: repeat, average
        t0 = time.perf_counter()
        oracle.spgemm(sub, B, nthreads=nthreads)
        dt += time.perf_counter() - t0
        reps += 1
    dt /= reps
    return {"value": 2 * f / dt / 1e9, "unit": "GFLOPS", "cores": nthreads, "kind": "oracle",
            "sample": f"{k} of {A.nrows} rows drawn uniformly at random (seed 2024): {f} of {tot} flop "
                      f"({100.0 * f / max(tot, 1):.2f}%), {dt:.3f} s per run (mean of {reps}), "
                      f"OpenMP over rows"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        log(f"[rank {rank}] reference arm: rank 0 alone runs the oracle")
        return 0
    import oracle
    A, B, extra = make_workload(args.config)
    of, tot = oracle.flop(A, B)
    nthreads = os.cpu_count() or 1
    # each step = the oracle on a seeded random row sample sized to ~2 s of
    # CPU, so the whole run stays within minutes (calibrated: best of 3)
    frac = 0.002
    sub, f, k = row_sample(A, of, frac)
    cal = []
    for _ in range(3):
        t0 = time.perf_counter()
        oracle.spgemm(sub, B, nthreads=nthreads)
        cal.append(time.perf_counter() - t0)
    rate = max(f, 1) / max(min(cal), 1e-6)
    frac = min(1.0, frac * max(1.0, 2.0 * rate / max(f, 1)) if f else 1.0)
    sub, f, k = row_sample(A, of, frac)
    for _ in range(args.warmup):
        oracle.spgemm(sub, B, nthreads=nthreads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.spgemm(sub, B, nthreads=nthreads)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.mean(times))
    val = 2 * f / (ms * 1e-3) / 1e9
    sample = (f"{k} of {A.nrows} rows drawn uniformly at random (seed 2024): {f} of {tot} flop "
              f"per step, OpenMP over rows")
    out = {"impl": "reference", "metric": METRIC, "value": val,
           "unit": "GFLOPS", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": args.config, "sorted": True, "flop_total": tot},
           "cpu_baseline": {"value": val, "unit": "GFLOPS", "cores": nthreads, "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": val, "unit": "GFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# ----------------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    from paper_1804_01698_b200 import build as spg_build
    if rank == 0:
        spg_build.build()
    if world > 1:
        dist.barrier()
    import paper_1804_01698_b200 as spg
    from paper_1804_01698_b200 import _lib

    # ---- inputs (host, seeded) -> HBM; B broadcast from rank 0 over NCCL
    t0 = time.perf_counter()
    A = B = extra = None
    if rank == 0 or world == 1:
        A, B, extra = make_workload(args.config)
    log(f"[rank {rank}] workload {args.config} generated in {time.perf_counter() - t0:.1f}s")
    same = args.config in ("c1_er4096", "c2_stencil64", "c3_rmat20")

    tri = args.config == "c5_triangle"
    ctx = spg.Context(local)
    if world == 1:
        dA = spg.DeviceCSR.from_host(A)
        dB = dA if same else spg.DeviceCSR.from_host(B)
        dG = spg.DeviceCSR.from_host(extra["G"]) if tri else None
        # ---- a8: flop-balanced row split (RowsToThreads on the GPU)
        offs, flop_total = spg.rows_to_parts(dA, dB, world, ctx)
        Aloc = dA
    else:
        # inputs from rank 0 with the library's distribution (paper_1804_01698_b200/dist.py,
        # tested with gloo): B broadcast (row_ptr first, col / val async), A row-scattered by
        # the flop-balanced split computed on rank 0's GPU; C5's mask G broadcast whole (the
        # degree-order variant relabels all of G on every rank)
        from paper_1804_01698_b200 import dist as sdist
        hA = spg.DeviceCSR.from_host(A) if rank == 0 else None
        hB = (hA if same else spg.DeviceCSR.from_host(B)) if rank == 0 else None
        dB, works = sdist.broadcast_csr(hB, 0, dev, async_values=True)
        meta = torch.zeros(world + 2, dtype=torch.int64, device=dev)
        if rank == 0:
            o, t = spg.rows_to_parts(hA, hB, world, ctx)
            meta[:] = torch.tensor(o + [t], dtype=torch.int64)
        dist.broadcast(meta, 0)
        offs, flop_total = [int(x) for x in meta[:world + 1].tolist()], int(meta[world].item())
        for w_ in works:
            w_.wait()
        if same:
            dA = dB
            Aloc = dB.rows(offs[rank], offs[rank + 1])
        else:
            dA = None
            Aloc = sdist.scatter_rows(hA, offs, 0, dev)
        dG = sdist.broadcast_csr(spg.DeviceCSR.from_host(extra["G"]) if (tri and rank == 0) else None,
                                 0, dev) if tri else None
    r0, r1 = offs[rank], offs[rank + 1]

    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)

    deg = None
    if tri:
        # degree-ascending relabelling (untimed preprocessing as in the
        # paper), then a flop-balanced split of the reordered L'
        t_rl = time.perf_counter()
        _, L2, U2, G2 = spg.degree_relabel(dG, ctx=ctx)
        offs2, flop_deg = spg.rows_to_parts(L2, U2, world, ctx)
        q0, q1 = offs2[rank], offs2[rank + 1]
        deg = {"L": L2.rows(q0, q1), "U": U2, "G": G2, "q0": q0, "q1": q1, "flop": flop_deg,
               "relabel_s": time.perf_counter() - t_rl}

    # accumulator A/B: sorted output with every eligible row
    # hashed, or merged by the heap (the default runs the cost model, AUTO).
    # The variants switch the accumulator of the bench's own ctx (a second ctx
    # could not hold C3's tile records next to the first one's)
    acc_ctx = {mode: ctx for mode in ("hash", "heap")}

    def step(sorted_out):
        if isinstance(sorted_out, str) and sorted_out.startswith("acc_"):  # acc_<mode>[_deg]
            mode = sorted_out.split("_")[1]
            if sorted_out.endswith("_deg"):  # L'*U' formed (sorted) in the degree order + mask
                return (spg.triangle_count_rows(deg["L"], deg["U"], deg["G"], 0, deg["q1"] - deg["q0"],
                                                sorted=True, ctx=acc_ctx[mode], g_shift=deg["q0"])
                        if deg["q1"] > deg["q0"] else 0)
            return spg.spgemm(Aloc, dB, sorted=True, ctx=acc_ctx[mode])
        if isinstance(sorted_out, str) and sorted_out.startswith("onephase_"):  # one-phase A/B
            return spg.spgemm(Aloc, dB, sorted=sorted_out.endswith("sorted"), ctx=ctx, method="one_phase")
        if sorted_out == "deg_formed":  # the same with the default (AUTO) accumulator
            return (spg.triangle_count_rows(deg["L"], deg["U"], deg["G"], 0, deg["q1"] - deg["q0"],
                                            sorted=True, ctx=ctx, g_shift=deg["q0"])
                    if deg["q1"] > deg["q0"] else 0)
        if sorted_out == "fused":  # C5 variant: mask fused into the product (C never formed)
            return spg.masked_sum_int(Aloc, dB, dG, r0, ctx) if r1 > r0 else 0
        if sorted_out == "fused_deg":  # the same on the degree-ordered split
            return (spg.masked_sum_int(deg["L"], deg["U"], deg["G"], deg["q0"], ctx)
                    if deg["q1"] > deg["q0"] else 0)
        if tri:  # rows [r0, r1) of C = L*U, masked by the same rows of G, in row blocks
            return spg.triangle_count_rows(Aloc, dB, dG, 0, r1 - r0, sorted=sorted_out, ctx=ctx,
                                           g_shift=r0)
        C = spg.spgemm(Aloc, dB, sorted=sorted_out, ctx=ctx)
        return C

    def timed(sorted_out, k, profile=False, keep=False):
        s = torch.cuda.current_stream()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(k)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        out = step(sorted_out)  # one more untimed step of this variant (warm)
        del out
        torch.cuda.synchronize()
        l0 = ctx.launches
        if profile:
            _lib.spg_profile_reset(ctx.handle)
            _lib.spg_profile_enable(ctx.handle, True)
        last = None
        for i in range(k):
            flush.fill_(i)                       # L2 flush, outside the events
            ev[i][0].record(s)
            out = step(sorted_out)
            ev[i][1].record(s)
            if i == k - 1:
                if keep or out is None or isinstance(out, (int, float)):
                    last = out                   # the final C (parity check) or count
                else:
                    last = out.row_ptr           # keep only the final row_ptr (C can be >100 GB)
            del out
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        launches = ctx.launches - l0
        recs = []
        if profile:
            _lib.spg_profile_enable(ctx.handle, False)
            recs = _lib.spg_profile_records(ctx.handle)
            _lib.spg_profile_reset(ctx.handle)
        ms = [a.elapsed_time(b) for a, b in ev]
        tot = torch.tensor([float(np.sum(ms))], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        log(f"[rank {rank}] sorted={sorted_out} step ms: {[round(x, 3) for x in ms]}")
        return float(tot.item()) / k, launches, recs, last

    clocks = ClockSampler(local)
    if not os.environ.get("SPG_BENCH_NO_CLOCKS"):
        clocks.start()
    for _ in range(args.warmup):
        step(True)
        step(False)
    ms_sorted, launches, _, last_sorted = timed(True, args.steps, keep=True)
    # parity of the timed run's own output vs the oracle (outside the timed region)
    parity = (bench_parity(args, A, B, last_sorted, tri, world, rank, dev, r0, r1)
              if not args.no_parity else None)
    Cs = last_sorted.row_ptr if (last_sorted is not None and not tri) else None
    del last_sorted
    torch.cuda.empty_cache()
    ms_unsorted, _, _, last_unsorted = timed(False, args.steps)
    ms_fused = None
    if tri:
        step("fused")
        ms_fused, _, _, last_fused = timed("fused", args.steps)
        step("fused_deg")
        ms_fused_deg, _, _, last_fdeg = timed("fused_deg", args.steps)
    acc_ab, acc_counts = {}, []
    if not tri and not args.no_accum_ab:
        # one-phase path where every row fits its tiers
        # (min(flop_i, ncols) <= 8192) and flop x 12 B fits the workspace
        try:
            for kname in ("onephase_sorted", "onephase_unsorted"):
                step(kname)
                acc_ab[kname] = timed(kname, max(1, min(args.steps, 10)))[0]
        except _lib.SpgError as e:
            log(f"one-phase not applicable: {e}")
    if not args.no_accum_ab:
        kinds = (("deg_formed", "acc_hash_deg", "acc_heap_deg") if tri else ("acc_hash", "acc_heap"))
        for kname in kinds:
            mode = kname.split("_")[1]
            if mode in ("hash", "heap"):
                ctx.set_accumulator(mode)
            try:
                step(kname)
                ms_k, _, _, last_k = timed(kname, max(1, min(args.steps, 5)))
            finally:
                ctx.set_accumulator("auto")
            acc_ab[kname] = ms_k
            if tri:
                acc_counts.append(float(last_k))
    if tri:
        counts = torch.tensor([float(last_unsorted), float(last_fused), float(last_fdeg)] + acc_counts,
                              dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(counts)
        if parity is not None:
            parity["triangles_unsorted_fused_degree_and_ab"] = [int(round(x / 2)) for x in counts.tolist()]
            parity["ok"] = parity["ok"] and all(
                int(round(x / 2)) == parity["oracle_triangles"] for x in counts.tolist())
    clk = clocks.stop()
    acc_ctx.clear()
    torch.cuda.empty_cache()

    # ---- per-kernel attribution: a separate profiled pass (outside the timed
    # steps) on the bench's ctx (its grow-only workspaces -- C3's tile records
    # among them -- are the timed steps' ones) with its bins on one stream, so
    # each kernel's events bracket only that kernel
    recs = []
    if rank == 0:
        pctx = ctx
        _lib.spg_set_serial_bins(pctx.handle, True)

        def prof_step():
            if tri:  # the headline C5 step: row blocks of C = L*U, each masked by G
                return spg.triangle_count_rows(Aloc, dB, dG, 0, r1 - r0, sorted=True, ctx=pctx,
                                               g_shift=r0)
            return spg.spgemm(Aloc, dB, sorted=True, ctx=pctx)
        for _ in range(2):  # (warm: grow-only workspaces sized by the first calls)
            out = prof_step()
            del out
        nprof = max(1, min(args.steps, 3))
        torch.cuda.synchronize()
        _lib.spg_profile_reset(pctx.handle)
        _lib.spg_profile_enable(pctx.handle, True)
        for i in range(nprof):
            flush.fill_(i)
            out = prof_step()
            del out
        torch.cuda.synchronize()
        _lib.spg_profile_enable(pctx.handle, False)
        recs = _lib.spg_profile_records(pctx.handle)
        _lib.spg_profile_reset(pctx.handle)
        _lib.spg_set_serial_bins(pctx.handle, False)
        ctx_attr, prof_steps = pctx, nprof

    gflops = lambda ms: 2.0 * flop_total / (ms * 1e-3) / 1e9  # noqa: E731

    # ---- e2e: through the public API with HOST buffers (H2D of A,B from pinned
    # memory, the multiply, D2H of C) inside the timed region
    e2e = e2e_measure(args, spg, ctx, Aloc, dB, dG, same, dev, world, rank, r0, r1, tri, flop_total)

    # ---- roofline of the dominant kernel (live per-launch events, sorted run)
    roof = None
    nnz_rank0 = None
    if rank == 0 and recs:
        agg = {}
        for n, t in recs:
            a = agg.setdefault(n, [0.0, 0])
            a[0] += t
            a[1] += 1
        top = max(agg, key=lambda n: agg[n][0])
        tot_ms, cnt = agg[top]
        avg_ms = tot_ms / cnt
        a_nnz = np.diff(A.row_ptr)[r0:r1]
        # per-row flop and nnz(c_i) from the library's symbolic phase of the
        # rank's whole row range (C5: C itself is only formed in row blocks)
        rp_all, _, _ = spg.spg_symbolic(Aloc, dB, ctx_attr)
        f_row = spg.plan_export(ctx_attr, r1 - r0)[0].cpu().numpy()
        c_nnz = np.diff(rp_all.cpu().numpy())
        nnz_rank0 = int(c_nnz.sum())
        del rp_all
        byts = kernel_bytes(top, a_nnz, f_row, c_nnz, r1 - r0, int(a_nnz.sum()), dB.ncols, dB.nrows)
        launches_per_step = cnt / prof_steps
        if byts is not None:
            byts /= max(launches_per_step, 1)  # bins launched once per step
        peak, peak_src = measured_peak()
        step_ms_serial = sum(t for _, t in recs) / prof_steps
        step_share = tot_ms / prof_steps / step_ms_serial
        roof = {"bound": "hbm", "kernel": top,
                "bytes_model": "numeric kernels: sum over their rows of 16 + 12 nnz(a_i) + 12 flop_i "
                               "+ 12 nnz(c_i) (A row, gathered B rows, C row); DESIGN.md section 3", "achieved": (byts / (avg_ms * 1e-3) / 1e9) if byts else None,
                "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                "frac": (byts / (avg_ms * 1e-3) / 1e9 / peak) if byts else None,
                "traffic": ncu_traffic(args.config, top), "algorithmic_bytes_per_launch": byts,
                "avg_launch_ms": avg_ms, "launches_per_step": launches_per_step,
                "share_of_step": step_share,
                "attribution": f"separate profiled pass, {prof_steps} sorted steps, bins on one stream, "
                               "per-launch CUDA events on the launching stream "
                               "(share = kernel time / sum of the step's kernel times)",
                "kernels_ms_per_step": {n: v[0] / prof_steps for n, v in sorted(agg.items(), key=lambda x: -x[1][0])}}

    # nnz(C) of the whole job (each rank holds its row block's row_ptr)
    nnzC = None
    if Cs is not None and not tri:
        t = torch.tensor([int(Cs[-1].item()) - int(Cs[0].item())], dtype=torch.int64, device=dev)
        if world > 1:
            dist.all_reduce(t)
        nnzC = int(t.item())
    if tri and world == 1:
        nnzC = nnz_rank0  # (C5: from the symbolic phase; C is only formed in row blocks)
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = oracle_sample(A, B, target_s=args.cpu_seconds)
        mb = None
        if nnzC is not None:
            mb = (8 * (A.nrows + 1) + 12 * A.nnz + 8 * (B.nrows + 1) + 12 * flop_total
                  + 8 * (A.nrows + 1) + 12 * nnzC)
        out = {
            "metric": METRIC,
            "value": gflops(ms_sorted), "unit": "GFLOPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_sorted, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "sorted": True, "flop_total": flop_total,
                       "nnz_C": nnzC, "m": A.nrows, "nnz_A": A.nnz,
                       "parallelism": f"rows x {world} (flop-balanced, B broadcast)",
                       "l2": "flushed between steps (256 MiB write outside the step events)"},
            "variants": {"sorted": {"value": gflops(ms_sorted), "ms_per_step": ms_sorted},
                         "unsorted": {"value": gflops(ms_unsorted), "ms_per_step": ms_unsorted},
                         **({"fused_mask": {"value": gflops(ms_fused), "ms_per_step": ms_fused,
                                            "note": "sum(L*U o G) with the mask fused into the "
                                                    "product (SURVEY 8(f) row 1); C not formed"}}
                            if ms_fused is not None else {}),
                         **({k: {"ms_per_step": v,
                                 "note": "A/B variant: "
                                         + {"onephase_sorted": "one-phase path: flop-sized tables, no "
                                                               "symbolic pass, one host round trip (8(f) row 3)",
                                            "onephase_unsorted": "one-phase path, unsorted C",
                                            "acc_hash": "every row hashed + sorted",
                                            "acc_heap": "heap merge for every eligible row (P:340-352)",
                                            "deg_formed": "degree order, L'*U' formed sorted, cost model "
                                                          "(AUTO) accumulator, + mask",
                                            "acc_hash_deg": "degree order, L'*U' formed sorted, all hashed",
                                            "acc_heap_deg": "degree order, L'*U' formed sorted, heap where "
                                                            "eligible"}[k]}
                             for k, v in acc_ab.items()}),
                         **({"fused_mask_degree_order": {
                             "ms_per_step": ms_fused_deg, "flop": deg["flop"],
                             "gflops_own_flop": 2.0 * deg["flop"] / (ms_fused_deg * 1e-3) / 1e9,
                             "relabel_s_untimed": deg["relabel_s"],
                             "note": "fused mask on L', U' of the degree-ascending relabelling "
                                     "(P:604, SURVEY 8(f) row 1; relabel untimed as in the "
                                     "paper); same triangle count, fewer products"}}
                            if deg is not None else {})},
            "minimal_bytes_model": mb,
            "hbm_roofline_frac_step": (mb / (ms_sorted * 1e-3) / 1e9 / (world * measured_peak()[0]))
                                      if mb else None,
            "gpu_launches": launches,
            "parity": parity,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def bench_parity(args, A, B, out, tri, world, rank, dev, r0, r1):
    """Checks the timed run's own output against the oracle, outside the
    timed region.  C = A*B configs (rank 0's row block): sampled rows (the 8
    heaviest + 120 drawn at random, seeded) of the last sorted C vs the
    oracle's rows -- structure bit-exact, strictly increasing columns, values
    within 1e-12 relative.  C5: the job's triangle count (sum over ranks) vs
    the oracle's count in tests/golden/full_configs.json (written by
    tools/oracle_goldens.py, which calls only oracle/)."""
    import torch
    import torch.distributed as dist
    if tri:
        cnt = torch.tensor([float(out)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(cnt)
        if rank != 0:
            return None
        try:
            gold = json.load(open(os.path.join(ROOT, "tests", "golden", "full_configs.json")))
            want = int(gold[args.config]["triangles"])
        except Exception:
            want = None
        got = int(round(cnt.item() / 2))
        return {"what": "triangle count of the timed run (sum over ranks / 2) vs the oracle's "
                        "(tests/golden/full_configs.json)",
                "triangles": got, "oracle_triangles": want, "ok": want is not None and got == want}
    if rank != 0 or out is None:
        return None
    import oracle
    import synth
    of, _ = oracle.flop(A, B)
    m = r1 - r0
    rng = np.random.default_rng(77)
    f_loc = of[r0:r1]
    nz = np.nonzero(f_loc)[0]
    heavy = np.argsort(f_loc)[::-1][:8]
    rnd = rng.choice(nz, size=min(120, len(nz)), replace=False) if len(nz) else np.zeros(0, np.int64)
    rows = np.unique(np.r_[heavy, rnd]).astype(np.int64)
    rows = rows[rows < m]
    lens = np.diff(A.row_ptr)[r0 + rows]
    rp = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    idx = np.repeat(A.row_ptr[r0 + rows] - rp[:-1], lens) + np.arange(int(rp[-1]), dtype=np.int64)
    sub = synth.CSR(len(rows), A.ncols, rp, A.col[idx].astype(np.int32), A.val[idx])
    o_rp, o_col, o_val = oracle.spgemm(sub, B)
    g_rp = out.row_ptr.cpu().numpy()
    ok, worst, nent = True, 0.0, 0
    for q, r in enumerate(rows):
        s, e = int(g_rp[r]), int(g_rp[r + 1])
        os_, oe = int(o_rp[q]), int(o_rp[q + 1])
        gc = out.col[s:e].cpu().numpy()
        gv = out.val[s:e].cpu().numpy()
        oc, ov = o_col[os_:oe], o_val[os_:oe]
        if e - s != oe - os_ or not np.array_equal(gc, oc):
            ok = False
            continue
        if len(gc) > 1 and not (np.diff(gc.astype(np.int64)) > 0).all():
            ok = False
        rel = np.abs(gv - ov) / np.maximum(np.abs(ov), 1e-300)
        if len(rel):
            worst = max(worst, float(rel.max()))
        nent += len(gc)
    ok = ok and worst <= 1e-12
    return {"what": "sampled rows of the last timed sorted C (rank 0's block) vs the oracle",
            "rows_checked": int(len(rows)), "entries_checked": int(nent),
            "max_rel_err": worst, "ok": bool(ok)}


def e2e_measure(args, spg, ctx, Aloc, dB, dG, same, dev, world, rank, r0, r1, tri, flop_total):
    """Same metric through the public API with host (pinned) buffers: every
    rank uploads ITS inputs (rows [r0, r1) of A, all of B, and for C5 the same
    rows of G) from pinned host memory, multiplies (C5: counts), and reads its
    result back (rows [r0, r1) of C, chunked through a bounded pinned buffer;
    C5: the count).  Time = max over ranks of the per-step device events; the
    byte counts are summed over ranks (whole job)."""
    import torch
    import torch.distributed as dist

    def host_rows(M, a, b):  # pinned host copy of rows [a, b) of a device CSR, row_ptr rebased
        rp = M.row_ptr[a:b + 1]
        s, e = int(rp[0].item()), int(rp[-1].item())
        return ((rp - s).cpu().pin_memory(), M.col[s:e].cpu().pin_memory(),
                M.val[s:e].cpu().pin_memory(), M.ncols)

    hA = host_rows(Aloc, 0, Aloc.nrows)
    hB = host_rows(dB, 0, dB.nrows) if not (same and world == 1) else hA
    hG = host_rows(dG, r0, r1) if tri else None
    m = r1 - r0
    chunk = 1 << 28
    outbuf_c = torch.empty(chunk // 4, dtype=torch.int32).pin_memory()
    outbuf_v = torch.empty(chunk // 8, dtype=torch.float64).pin_memory()
    outbuf_r = torch.empty(m + 1, dtype=torch.int64).pin_memory()
    k = max(1, min(args.steps, args.e2e_steps))
    s = torch.cuda.current_stream()
    nbytes = lambda h: sum(t.numel() * t.element_size() for t in h[:3])  # noqa: E731
    h2d = d2h = 0
    times = []
    for it in range(k + 1):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)

        def up(h):
            n = h[0].numel() - 1
            return spg.DeviceCSR(n, h[3], h[0].to(dev, non_blocking=True),
                                 h[1].to(dev, non_blocking=True), h[2].to(dev, non_blocking=True))
        dAl = up(hA)
        dBl = dAl if hB is hA else up(hB)
        hb = nbytes(hA) + (0 if hB is hA else nbytes(hB))
        if tri:
            dGl = up(hG)
            hb += nbytes(hG)
            cnt = spg.triangle_count_rows(dAl, dBl, dGl, 0, m, sorted=True, ctx=ctx) if m else 0
            outbuf_r[:1].copy_(torch.tensor([cnt]))
            db = 8
        else:
            C = spg.spgemm(dAl, dBl, sorted=True, ctx=ctx)
            nnz = C.col.numel()
            outbuf_r.copy_(C.row_ptr, non_blocking=True)
            for o in range(0, nnz, chunk // 8):
                n = min(chunk // 8, nnz - o)
                outbuf_c[:n].copy_(C.col[o:o + n], non_blocking=True)
                outbuf_v[:n].copy_(C.val[o:o + n], non_blocking=True)
            db = (m + 1) * 8 + nnz * 12
            del C
        e1.record(s)
        torch.cuda.synchronize()
        if it > 0:  # first iteration is a warm-up
            times.append(e0.elapsed_time(e1))
        h2d, d2h = hb, db
        del dAl, dBl
    red = torch.tensor([float(np.mean(times)), float(h2d), float(d2h)], dtype=torch.float64, device=dev)
    if world > 1:
        mx = red[:1].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = red[1:].clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        red = torch.cat([mx, sm])
    ms, h2d, d2h = (float(x) for x in red.tolist())
    return {"value": 2.0 * flop_total / (ms * 1e-3) / 1e9, "unit": "GFLOPS", "ms_per_step": ms,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": len(times),
            "timing": "max over ranks of per-rank device events; bytes summed over ranks"}


def self_launch(n: int) -> int:
    """`bench.py --gpus N` without a torchrun environment: re-launch this
    script as N ranks (one process per GPU) with torch.distributed.run on
    127.0.0.1 and return its exit code (rank 0 prints the JSON line)."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__),
           *sys.argv[1:]]
    log("self-launch: " + " ".join(cmd))
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG,
                    choices=["c1_er4096", "c2_stencil64", "c3_rmat20", "c4_tallskinny", "c5_triangle"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-accum-ab", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup < 3 is not allowed by the timing rules; using 3")
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        log(f"--gpus {args.gpus} but WORLD_SIZE={world}: the job runs {world} rank(s)")
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
