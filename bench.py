#!/usr/bin/env python3
"""Benchmark: exhaustive minimal-Goldbach-prime verification of every even n in a
range on 1..8 B200s.  Default: [4, 1e12] (BASELINE.json configs[3], the metric's
workload).  One "step" = the whole hot path over the whole range: K-SIEVE +
inverted marking + fallback in the fused kernel for every strip, the result
finalize, and the NCCL reduction of the result vector.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c1|c2|c3|c4|c5]
                  [--N 1e13] [--mode bulk|pern|resident] [--impl ours|reference]

Prints ONE JSON line on rank 0.  Metric: even n verified per second, whole job,
device-timed (CUDA events on the launching stream, max over ranks), L2 flushed
between steps.  Strong scaling: the range is fixed and sharded over ranks.  The
line carries the result of the last step and the verdict of checking it against
the oracle-written golden of that range (tests/golden/verify_<tag>.json) when one
exists, else against the invariants every run must satisfy (unresolved == 0,
sum of the histogram == evens); the process exits 1 if that check fails.
`--impl reference` times the CPU oracle (oracle/, the paper's cpu_goldbach
definition) on the host cores on a bounded sample of the same
workload -- the reference arm of this tier.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE_METRIC = "even n verified/sec (whole box, device-timed) to N=1e12 at 1/2/4/8 B200; sieve GB/s"
UNIT = "even_n/s"
NSM = 148

# BASELINE.json configs: (lo, hi, origin, golden tag, description)
TOP = 4 * 10**18
WORKLOADS = {
    "c1": (4, 10**6 + 1, 0, "1e06", "C1: every even n in [4, 1e6]"),
    "c2": (4, 10**9 + 1, 0, "1e09", "C2: every even n in [4, 1e9]"),
    "c3": (4, 10**11 + 1, 0, "1e11", "C3: every even n in [4, 1e11]"),
    "c4": (4, 10**12 + 1, 0, "1e12", "C4: every even n in [4, 1e12]"),
    "c5": (TOP - 10**11, TOP, TOP - 10**11, "c5_4e18", "C5: every even n in the window [4e18 - 1e11, 4e18)"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--N", type=float, default=None, help="custom range [4, N] (overrides --workload)")
    ap.add_argument("--p-max", type=int, default=65521)
    ap.add_argument("--mode", default="bulk", choices=["bulk", "pern", "resident", "counts"],
                    help="bulk: the product path (inverted bulk marking); pern: the paper's per-n "
                         "gpu3 kernel (NEXT-1, PAPER.md:82-95); resident: the paper's gpu2 with the "
                         "whole odd bitset of [3, hi) sieved into HBM each step (NEXT-2, PAPER.md:41-59); "
                         "counts: Goldbach partition counts c(n) of the top --counts-window even n below N "
                         "(default N = 1e9; NEXT-4, PAPER.md:421)")
    ap.add_argument("--counts-window", type=int, default=16384, help="even n per step in --mode counts")
    ap.add_argument("--strips-per-rank", type=int, default=None,
                    help="default 8 (balances the growth of work with n), fewer when a strip would have "
                         "under 8 tiles per SM; 2 for c5 (the window's cost is flat; fewer partial "
                         "K-LARGE chunks)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sieve", action="store_true", help="skip the standalone sieve GB/s leg")
    ap.add_argument("--no-check", action="store_true", help="do not exit 1 on a failed result check")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    a = ap.parse_args()
    return a


def auto_strips(args, lo: int, hi: int, world: int) -> int:
    """Strips (one gb_verify_range each) per rank: 2 for the C5 window (flat cost, fewer
    partial K-LARGE chunks); else 8 (balances the growth of work with n), but never
    fewer than 8 tiles per SM in a strip: a small range ([4, 1e9] is 254 tiles) runs as
    one call, whose tiles libgb balances over the SMs."""
    if args.strips_per_rank is not None:
        return args.strips_per_rank
    if args.workload == "c5" and args.N is None:
        return 2
    tiles = (hi - lo) / (192 * 21376) / world          # 192 integers per class word, kTileWords
    return max(1, min(8, int(tiles // (8 * NSM))))


def workload(args):
    """(lo, hi, origin, golden tag or None, description)"""
    if args.N is not None:
        N = int(args.N)
        return 4, N + 1, 0, f"{N:.0e}".replace("+", ""), f"every even n in [4, {N:.0e}]"
    return WORKLOADS[args.workload]


def metric_name(args):
    if args.N is None and args.workload == "c4" and args.mode == "bulk":
        return BASELINE_METRIC
    _, _, _, _, desc = workload(args)
    return f"even n verified/sec (whole box, device-timed), {desc}" + (
        f" [{args.mode} mode]" if args.mode != "bulk" else "")


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------- CPU oracle legs
def oracle_sample(hi: int, target_s: float, lo_min: int = 4):
    """Time the CPU oracle (as it stands) on a top slice of [lo_min, hi), growing the
    slice until it has run for at least target_s seconds."""
    from oracle import oracle
    threads = oracle.default_threads()
    span = 1 << 22
    while True:
        lo = max(lo_min, hi - span)
        t0 = time.perf_counter()
        r, _ = oracle.verify(lo, hi, threads=threads)
        dt = time.perf_counter() - t0
        if dt >= target_s or lo == lo_min:
            return {"value": r["evens"] / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
                    "sample": f"even n in [{lo}, {hi}) ({r['evens']} evens, {dt:.2f} s, top of the range)",
                    "seconds": dt, "evens": r["evens"]}
        span = int(span * min(8.0, max(2.0, 1.2 * target_s / max(dt, 1e-3))))


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    lo, hi, _, _, desc = workload(args)
    per_step = max(1.0, args.cpu_seconds / 4)
    for _ in range(args.warmup):
        oracle_sample(hi, per_step / 4, lo)
    times, evens = [], 0
    first = oracle_sample(hi, per_step, lo)
    for i in range(args.steps):
        s = first if i == 0 else oracle_sample(hi, per_step, lo)
        times.append(s["seconds"])
        evens += s["evens"]
    value = evens / sum(times)
    line = {"metric": metric_name(args), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (deterministic number-theoretic range)", "impl": "reference",
            "config": {"workload": desc, "lo": lo, "hi": hi, "sample": first["sample"]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": first["cores"], "kind": "oracle",
                             "sample": f"{args.steps} top-of-range slices of [{lo}, {hi}), ~{per_step:.1f} s each"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- roofline yardsticks
def small_primes(limit: int):
    import numpy as np
    s = np.ones(limit + 1, dtype=bool)
    s[:2] = False
    for i in range(2, int(limit**0.5) + 1):
        if s[i]:
            s[i * i::i] = False
    return np.flatnonzero(s)


def recip_sum(a: int, b: int) -> float:
    """sum of 1/p over primes a < p <= b: exact to 1e7, Mertens' ln ln x beyond
    (the difference of two ln ln terms is accurate to ~1e-6 there)."""
    import numpy as np
    cut = 10**7
    ps = small_primes(min(b, cut))
    s = float(np.sum(1.0 / ps[(ps > a) & (ps <= b)]))
    if b > cut:
        s += math.log(math.log(b)) - math.log(math.log(max(a, cut)))
    return s


def mark_word_iters(hi: int) -> float:
    """SURVEY.md 8(d) "Algorithmic work per even n": 64-bit word-iterations per even
    n of the inverted loop with 64-even exit (the table's values at its N, log-linear
    in log10 N between them)."""
    pts = [(9, 0.74), (11, 0.92), (12, 1.01), (18.6, 1.63)]
    x = math.log10(hi)
    if x <= pts[0][0]:
        return pts[0][1]
    for (x0, y0), (x1, y1) in zip(pts, pts[1:]):
        if x <= x1:
            return y0 + (y1 - y0) * (x - x0) / (x1 - x0)
    return pts[-1][1]


def load_peaks():
    """MEASURED_PEAKS.json (driver) + profiles/peaks_int.json (scripts/micro/peaks_int.cu
    on a B200 of this pool); returns the per-SM lane rates and the SM clock."""
    peaks, pint = {}, None
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    try:
        pint = json.load(open(os.path.join(ROOT, "profiles", "peaks_int.json")))
    except Exception:
        pass
    return peaks, pint


def launch_shares(wl: str):
    """Per-kernel GPU-time shares from the newest committed ncu launch list of this
    workload (profiles/r<NN>_launches_<wl>.md, scripts/launch_list.py), or None."""
    import glob
    lists = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_launches_{wl}.md")))
    if not lists:
        return None, None
    ns = {}
    for line in open(lists[-1]):
        parts = [x.strip() for x in line.split("|")]
        if len(parts) > 4 and parts[3].isdigit():
            ns[parts[1]] = int(parts[3])
    return ns, os.path.relpath(lists[-1], ROOT)


# K-LARGE (gb_kernels.cu large_mark_wheel_kernel): a sieving prime p > 2^21 clears
# q = p k only for cofactors k coprime to every prime <= 19 (the others are cleared by
# the window's own sieve): density prod_{p <= 19} (1 - 1/p) of the integers k
KLARGE_DENSITY = 1.0
for _q in (2, 3, 5, 7, 11, 13, 17, 19):
    KLARGE_DENSITY *= 1 - 1 / _q
KLARGE_PRIME_MIN = 1 << 21          # kCarryPrimeMax (gb_internal.h)


def ncu_capture(kernel: str, wl: str, mode: str):
    """The committed ncu --set full summary of `kernel` on this workload
    (profiles/r<NN>_<kernel>_<workload>[_<mode>].json, newest round first), or None."""
    import glob
    suffix = f"_{wl}" + ("" if mode == "bulk" else f"_{mode}")
    caps = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_{kernel}{suffix}.json")))
    if not caps:
        return None, None
    return json.load(open(caps[-1])), os.path.relpath(caps[-1], ROOT)


# ----------------------------------------------------------------- result check
def check_result(res, lo, hi, tag):
    """Compare with the oracle golden of this range if one exists, else check the
    invariants.  Returns (ok, what)."""
    from oracle import oracle
    from oracle.oracle import AGG_FIELDS, NBINS
    evens = oracle.n_evens(lo, hi)
    inv = (res["evens"] == evens and res["verified"] == evens and res["unresolved"] == 0
           and sum(res["hist"]) == evens)
    path = os.path.join(ROOT, "tests", "golden", f"verify_{tag}.json") if tag else None
    if path and os.path.exists(path):
        g = json.load(open(path))
        if (g["lo"], g["hi"]) == (lo, hi):
            gr = g["result"]
            bad = [k for k in AGG_FIELDS if res[k] != gr[k]]
            hist = [0] * NBINS
            for i, c in gr["hist"].items():
                hist[int(i)] = c
            if list(res["hist"]) != hist:
                bad.append("hist")
            return inv and not bad, {"golden": os.path.relpath(path, ROOT), "mismatch": bad,
                                     "invariants": inv}
    return inv, {"golden": None, "invariants": inv,
                 "note": "no oracle golden for this range: invariants only (evens, all verified, "
                         "no unresolved, sum hist = evens)"}


# ----------------------------------------------------------------- NEXT-4 leg
def run_counts(args, rank: int, world: int, local: int):
    """Goldbach partition counts c(n) (section 4.5; R13) for the
    top W even n of [4, N] on one GPU: one step = gb_sieve_segment of the odd bitset of
    [3, N] + gb_partition_counts of the window.  Metric: c(n) values per second.
    Roofline: the POPC pipe (one SHF + AND + POPC per (n, 32 i-bit word) pair, ~n/128
    pairs per n; 16 POPC lanes/clk/SM measured, profiles/peaks_int.json).  Check: the
    CPU oracle's plain scan (oracle.partition_counts) on 4 n of the window."""
    import numpy as np
    import torch
    if world > 1 and rank != 0:
        return                                     # single-GPU leg: no data-path collective
    N = int(args.N) if args.N is not None else 10**9
    W = args.counts_window
    hi = N + 1
    lo = hi - 2 * W
    lo += lo & 1
    torch.cuda.set_device(local)
    import __graft_entry__
    __graft_entry__.build()
    from paper_2603_02621_b200 import gb
    from paper_2603_02621_b200.verifier import Verifier
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    V = Verifier(hi_max=hi + 128, device=local, stream=stream)
    n_words = (hi - 3 + 127) // 128
    bits = torch.empty(n_words, dtype=torch.int64, device=dev)
    out = torch.empty(W, dtype=torch.int64, device=dev)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(max(4 * l2, 1 << 28) // 4, dtype=torch.int32, device=dev)

    def step(ev=None):
        gb.gb_sieve_segment(V.ctx, 0, n_words, bits, stream)
        if ev is not None:
            ev[0].record(stream)
        gb.gb_partition_counts(V.ctx, lo, hi, bits, n_words, out, stream)
        if ev is not None:
            ev[1].record(stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    launches0 = gb.gb_launch_count()
    st, kt = [], []
    for _ in range(args.steps):
        flush.fill_(1)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        s0.record(stream)
        step(k)
        s1.record(stream)
        st.append((s0, s1))
        kt.append(k)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    launches = gb.gb_launch_count() - launches0
    step_ms = [a.elapsed_time(b) for a, b in st]
    kern_ms = [a.elapsed_time(b) for a, b in kt]
    value = W * args.steps / (sum(step_ms) / 1e3)
    # e2e: the same step through the binding + D2H of the counts to pinned host memory
    h = torch.empty(W, dtype=torch.int64).pin_memory()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2):
        step()
        h.copy_(out, non_blocking=True)
        stream.synchronize()
    e2e_s = (time.perf_counter() - t0) / 2
    got = out.cpu().numpy()
    from oracle import oracle
    picks = [0, W // 3, (2 * W) // 3, W - 1]
    want = [int(oracle.partition_counts(lo + 2 * i, lo + 2 * i + 1)[0]) for i in picks]
    ok = all(int(got[i]) == w for i, w in zip(picks, want))
    pint = load_peaks()[1] or {}
    popc = (pint.get("per_sm_lane_ops_per_clk") or {}).get("popc", 16.0)
    sm_mhz = load_peaks()[0].get("sm_max_mhz", 1965.0)
    peak = NSM * popc * sm_mhz * 1e6 / 1e12
    pairs = sum(((n - 6) // 2 // 2) // 32 + 1 for n in range(lo, hi, 2))   # i-words per n (i <= K/2)
    ach = pairs / (statistics.mean(kern_ms) / 1e3) / 1e12
    line = {"metric": f"Goldbach partition counts c(n) per second, the top {W} even n of [4, {N:.0e}] "
                      "(NEXT-4) [counts mode]",
            "value": value, "unit": "c(n)/s", "n_gpus": 1, "steps": args.steps, "warmup": max(3, args.warmup),
            "ms_per_step": statistics.mean(step_ms), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic (deterministic number-theoretic range)",
            "config": {"workload": f"c(n) for even n in [{lo}, {hi})", "lo": lo, "hi": hi, "mode": "counts",
                       "l2": "flushed between steps"},
            "gpu_launches": launches, "clocks": clocks,
            "e2e": {"value": W / e2e_s, "unit": "c(n)/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 8 * W,
                    "note": "gb_sieve_segment + gb_partition_counts + D2H of the counts (pinned)"},
            "roofline": {"bound": "popc", "achieved": ach, "peak": peak, "unit": "T popc/s", "frac": ach / peak,
                         "kernel": "counts_kernel (popcount-AND of the odd bitset against its reversed shifts)",
                         "ops_basis": f"{pairs / W:.4g} 32-bit i-words per n (i <= K/2, K = (n-6)/2), one POPC each",
                         "peak_basis": f"148 SM x {popc:.2f} POPC lanes/clk x {sm_mhz:.0f} MHz (profiles/peaks_int.json)",
                         "kernel_ms_per_launch": statistics.mean(kern_ms),
                         "sieve_ms_per_step": statistics.mean(step_ms) - statistics.mean(kern_ms)},
            "check": {"ok": ok, "oracle_points": {str(lo + 2 * i): w for i, w in zip(picks, want)}},
            "step_ms": step_ms}
    print(json.dumps(line), flush=True)
    V.close()
    if not ok and not args.no_check:
        sys.exit(1)


# ----------------------------------------------------------------- GPU arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    if args.mode == "counts":
        run_counts(args, rank, world, local)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    # one process per GPU; GB_DIST_BACKEND=gloo lets a multi-rank run share one GPU
    # (a functional check of the N > 1 path on a 1-GPU box; NCCL refuses that)
    backend = os.environ.get("GB_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    import __graft_entry__
    __graft_entry__.build() if rank == 0 else None
    if world > 1:
        dist.barrier()
    from paper_2603_02621_b200 import gb
    from paper_2603_02621_b200 import dist as gdist
    from paper_2603_02621_b200.verifier import Verifier

    lo, hi, origin, tag, desc = workload(args)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    n_bits_words = (hi - 3) // 128 + 1 if args.mode == "resident" else 0
    # resident mode sieves every word of [3, hi): the context must cover their top q
    hi_max = max(hi, 3 + 128 * n_bits_words) if n_bits_words else hi
    V = Verifier(hi_max=hi_max, p_max=args.p_max, origin=origin, device=local, stream=stream)
    args.strips_per_rank = auto_strips(args, lo, hi, world)
    strips = gdist.rank_strips(gdist.plan_strips(lo, hi, args.strips_per_rank * world), rank, world)
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(max(4 * l2_bytes, 1 << 28) // 4, dtype=torch.int32, device=dev)
    bits = torch.empty(n_bits_words, dtype=torch.int64, device=dev) if n_bits_words else None

    def step(k_events=None):
        r = V.new_result()
        if bits is not None:                         # gpu2: sieve [3, hi) into HBM, then per-n lookups
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            gb.gb_sieve_segment(V.ctx, 0, bits.numel(), bits, stream)
            for a, b in strips:
                gb.gb_verify_range_resident(V.ctx, a, b, args.p_max, bits, bits.numel(), r, None, stream)
            e1.record(stream)
            if k_events is not None:
                k_events.append((e0, e1))
        else:
            for a, b in strips:
                if k_events is not None:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                V.verify(a, b, r, p_max=args.p_max, mode=args.mode)
                if k_events is not None:
                    e1.record(stream)
                    k_events.append((e0, e1))
        V.finalize(r)
        gdist.reduce_result(r)
        return r

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    launches0 = gb.gb_launch_count()
    k_events, results = [], []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush.fill_(1)                               # L2 flush between steps (untimed)
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        r = step(k_events)
        s1.record(stream)
        results.append((s0, s1, r))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = gb.gb_launch_count() - launches0
    launches_per_step = launches / args.steps
    if world > 1:                                    # whole job: every rank's launches
        lt = torch.tensor([launches], dtype=torch.int64, device=dev)
        dist.all_reduce(lt, op=dist.ReduceOp.SUM)
        launches = int(lt[0])
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b, _ in results]
    kern_ms = [a.elapsed_time(b) for a, b in k_events]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms, sum(kern_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    box_ms, box_kern_ms = float(t[0]), float(t[1])
    res = V.decode(results[-1][2])
    evens = res["evens"]
    value = evens * args.steps / (box_ms / 1e3)

    # ---- end to end through the public API with host buffers
    h_res = torch.empty(gb.RESULT_WORDS, dtype=torch.int64).pin_memory()
    e2e_steps = max(1, min(args.steps, 3))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        if args.mode == "bulk":                      # the C-ABI host entry: init + verify + finalize + D2H
            acc = np.zeros(gb.RESULT_WORDS, dtype=np.int64)
            for a, b in strips:
                gb.gb_verify_range_host(V.ctx, a, b, args.p_max, h_res, None, stream)
                acc += h_res.numpy()
        else:                                        # Verifier API of the comparison modes + D2H
            r = step()
            h_res.copy_(r, non_blocking=True)
            stream.synchronize()
    if world > 1:
        tt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt[0])
    else:
        e2e_s = time.perf_counter() - t0
    e2e = {"value": evens * e2e_steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 0,
           "d2h_bytes_per_step": 8 * gb.RESULT_WORDS * (len(strips) if args.mode == "bulk" else 1),
           "note": ("gb_verify_range_host per strip (C ABI, host result buffer): init + verify + finalize + "
                    "D2H of the 52 KB result; the inputs are (lo, hi, p_max) scalars, so no array H2D"
                    if args.mode == "bulk" else
                    f"Verifier API ({args.mode} mode) + D2H of the 52 KB result; scalar inputs")}

    # ---- rooflines
    peaks, pint = load_peaks()
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    hbm = peaks.get("hbm_gbs") or 6545.9
    if pint:
        rates = pint["per_sm_lane_ops_per_clk"]
        alu_rate, red_rate = rates["lop3"], rates["red_shared_and"]
        peak_src = "profiles/peaks_int.json (scripts/micro/peaks_int.cu, measured on a B200 of this pool)"
    else:
        alu_rate, red_rate = 64.0, 16.0
        peak_src = "nominal (profiles/peaks_int.json absent): 64 ALU / 16 shared-RED lanes per clk per SM"
    alu_peak = NSM * alu_rate * sm_mhz * 1e6 / 1e12          # T int32 lane-ops/s
    red_peak = NSM * red_rate * sm_mhz * 1e6 / 1e12
    n_launch = len(kern_ms)
    avg_launch_s = (sum(kern_ms) / n_launch) / 1e3 if n_launch else float("nan")
    evens_per_launch = evens / max(1, n_launch // args.steps) / world
    sqrt_hi = math.isqrt(hi - 1)
    clears = recip_sum(2, sqrt_hi)                 # sieve bit-clears per odd (= per even n)
    clears_red = recip_sum(61, sqrt_hi)            # the part not done by word patterns (p > 61)
    w_iters = mark_word_iters(hi)
    ops_per_even = clears + 6 * w_iters            # 1 op per clear, 6 per 64-bit word-iteration
    wl_key = args.workload if args.N is None else f"N{tag}"
    cap, dram_src = ncu_capture("verify_kernel" if args.mode == "bulk" else "pern_kernel", wl_key, args.mode)
    dram_pe = cap.get("dram_bytes_per_even") if cap else None
    if args.mode == "bulk":
        achieved = ops_per_even * evens_per_launch / avg_launch_s / 1e12
        roofline = {"bound": "alu", "achieved": achieved, "peak": alu_peak, "unit": "Tops/s",
                    "frac": achieved / alu_peak,
                    "traffic": dram_pe * evens_per_launch if dram_pe is not None else None,
                    "traffic_note": (f"DRAM read+write bytes per launch, scaled per even n from {dram_src}"
                                     if dram_src else "no ncu capture of this workload in profiles/"),
                    "kernel": "verify_kernel (fused sieve + mark + fallback)",
                    "ops_per_even": round(ops_per_even, 4),
                    "ops_basis": (f"SURVEY 8(d): {clears:.3f} sieve bit-clears per odd (primes to isqrt(hi)) + "
                                  f"6 int32 ops x {w_iters:.3f} 64-bit mark word-iterations per even n"),
                    "peak_basis": f"148 SM x {alu_rate:.1f} LOP3 lanes/clk x {sm_mhz:.0f} MHz; {peak_src}",
                    "kernel_ms_per_launch": avg_launch_s * 1e3, "launches_timed": n_launch,
                    "kernel_share_of_step": box_kern_ms / box_ms if box_ms else None}
    else:
        # comparison modes (the paper's own designs): a bitset in HBM written once and read
        # by per-n lookups -- algorithmic bytes 1 bit written + 1 bit read per even n
        bytes_pe = 0.25
        achieved = bytes_pe * evens_per_launch / avg_launch_s / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                    "traffic": dram_pe * evens_per_launch if dram_pe is not None else None,
                    "kernel": f"{args.mode} mode (sieve to HBM/L2 + per-n lookups)",
                    "bytes_per_even": bytes_pe, "kernel_ms_per_launch": avg_launch_s * 1e3,
                    "launches_timed": n_launch}

    # ---- sieve GB/s (BASELINE.json metric, second half): standalone gb_sieve_segment
    # (K-SIEVE, the paper's odd-only layout PAPER.md:46-51) writing the bitset of the
    # top 2^34 integers of the range to HBM; bytes written / device time.  Its roofline
    # is the shared-memory RED pipe (the bit-clears), not HBM.
    sieve = None
    sieve_ms_per_int = None
    if not args.no_sieve and hi > 1 << 30:
        nwords = 1 << 27                                   # u64 words = 2^34 integers, 1 GiB
        w_hi = (hi - 3) // 128
        if math.isqrt(3 + 128 * w_hi + 126) > V.R:
            w_hi -= 1                                      # top word must stay within the base primes
        w_lo = max(0, w_hi - nwords)
        out = torch.empty(w_hi - w_lo, dtype=torch.int64, device=dev)
        for _ in range(2):
            gb.gb_sieve_segment(V.ctx, w_lo, w_hi - w_lo, out, stream)
        ev = []
        for _ in range(5):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            gb.gb_sieve_segment(V.ctx, w_lo, w_hi - w_lo, out, stream)
            e1.record(stream)
            ev.append((e0, e1))
        torch.cuda.synchronize()
        ms = statistics.median(a.elapsed_time(b) for a, b in ev)
        nbytes = 8 * (w_hi - w_lo)
        odds = 64 * (w_hi - w_lo)
        sieve_ms_per_int = ms / (2 * odds)
        red_achieved = clears_red * odds / (ms / 1e3) / 1e12
        sieve = {"value": nbytes / (ms / 1e3) / 1e9, "unit": "GB/s", "ms_per_launch": ms,
                 "odd_integers_per_s": odds / (ms / 1e3),
                 "window": f"odd q in [{3 + 128 * w_lo}, {3 + 128 * w_hi})",
                 "kernel": "sieve_out_kernel (gb_sieve_segment)",
                 "hbm_frac": nbytes / (ms / 1e3) / 1e9 / hbm, "hbm_peak_gbps": hbm,
                 "roofline": {"bound": "smem_red", "achieved": red_achieved, "peak": red_peak, "unit": "Tops/s",
                              "frac": red_achieved / red_peak,
                              "ops_basis": f"{clears_red:.3f} bit-clears per odd by primes 61 < p <= isqrt(hi) "
                                           "(SURVEY 8(d) 'excl. p <= 61': the clears no word pattern does)",
                              "peak_basis": f"148 SM x {red_rate:.2f} red.shared.and lanes/clk x {sm_mhz:.0f} MHz; "
                                            f"{peak_src}"}}
        del out
    share = (cap or {}).get("phase_share_samples")
    if args.mode == "bulk" and not share:
        roofline["split_note"] = ("no ncu capture of this workload with per-region samples in profiles/: "
                                  "no separate K-SIEVE / K-MARK fractions")
    if args.mode == "bulk" and share:
        # the fused kernel's two halves: the sieve share of the kernel's stall samples in
        # the committed ncu capture of this workload (scripts/ncu_regions.py: time per
        # source region); the rest (marking + bookkeeping) is the marking half
        t_sieve = max(share.get("sieve", 0.0) * avg_launch_s, 1e-12)
        split_basis = f"sieve share {share.get('sieve', 0.0):.3f} of the stall samples in {dram_src}"
        t_mark = max(avg_launch_s - t_sieve, 1e-12)
        mark_ach = 6 * w_iters * evens_per_launch / t_mark / 1e12
        sieve_ach = clears_red * evens_per_launch / t_sieve / 1e12
        roofline["sieve"] = {"bound": "smem_red", "achieved": sieve_ach, "peak": red_peak, "unit": "Tops/s",
                             "frac": sieve_ach / red_peak, "est_share_of_kernel": t_sieve / avg_launch_s,
                             "basis": split_basis + f"; {clears_red:.3f} clears per even by primes > 61"}
        roofline["mark"] = {"bound": "alu", "achieved": mark_ach, "peak": alu_peak, "unit": "Tops/s",
                            "frac": mark_ach / alu_peak, "est_share_of_kernel": t_mark / avg_launch_s,
                            "basis": "verify_kernel time minus the sieve share; 6 ops x SURVEY word-iterations"}

    # ---- K-LARGE (ranges above 2^42): no-return L2 REDs into the chunk mask.  Its
    # roofline is the L2 RED rate (profiles/r02b_red_sms.json, 64 MB L2-resident buffer,
    # all SMs); its time is the step time x its share of the GPU time in the committed
    # launch list of this workload (cold-cache / serialised: a share, not a time)
    if args.mode == "bulk" and sqrt_hi > KLARGE_PRIME_MIN:
        split = KLARGE_PRIME_MIN * KLARGE_PRIME_MIN
        frac_above = (hi - max(lo, split)) / (hi - lo)
        reds_per_even = 2 * KLARGE_DENSITY * recip_sum(KLARGE_PRIME_MIN, sqrt_hi)
        ns, ls_src = launch_shares(wl_key)
        red_peak_s = None
        try:
            rs = json.load(open(os.path.join(ROOT, "profiles", "r02b_red_sms.json")))
            red_peak_s = rs["reds_per_s"]["64MB"][str(NSM)]
        except Exception:
            pass
        if ns and red_peak_s:
            t_large = sum(v for k, v in ns.items() if "large_" in k)
            t_step = t_large + sum(v for k, v in ns.items() if "verify_kernel" in k)
            share_l = t_large / t_step
            reds = reds_per_even * evens * frac_above
            ach = reds / ((box_ms / args.steps) / 1e3 * share_l)
            roofline["klarge"] = {
                "bound": "l2_red", "achieved": ach / 1e9, "peak": red_peak_s / 1e9, "unit": "G red/s",
                "frac": ach / red_peak_s, "est_share_of_step": share_l,
                "kernel": "large_mark_wheel_kernel (+ large_fill_kernel)",
                "reds_per_even": round(reds_per_even, 5),
                "basis": (f"2 x {KLARGE_DENSITY:.4f} (cofactors coprime to 2..19) x sum 1/p over "
                          f"{KLARGE_PRIME_MIN} < p <= {sqrt_hi} red.global.and per even n above 2^42; share "
                          f"{share_l:.3f} of the step's GPU time from {ls_src}"),
                "peak_basis": "red.global.and into a 64 MB (L2-resident) buffer from all 148 SMs, "
                              "profiles/r02b_red_sms.json (scripts/micro/red_sms.cu; 96 MB: 1.28e11/s)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_sample(hi, args.cpu_seconds, lo)
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}

    ok, check = check_result(res, lo, hi, tag) if rank == 0 else (True, None)
    if rank == 0:
        line = {"metric": metric_name(args), "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": box_ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
                "data": "synthetic (deterministic number-theoretic range; no dataset)",
                "config": {"workload": desc, "lo": lo, "hi": hi, "p_max": args.p_max,
                           "strips_per_rank": args.strips_per_rank, "parallelism": f"range-sharded x{world}",
                           "l2": "flushed between steps", "mode": args.mode},
                "gpu_launches": launches, "gpu_launches_per_step_per_rank": launches_per_step,
                "clocks": clocks, "e2e": e2e, "roofline": roofline,
                "cpu_baseline": cpu, "sieve": sieve,
                "result": {k: res[k] for k in ("evens", "verified", "fastpath_unresolved", "unresolved",
                                                  "max_pmin", "max_pmin_n", "sum_pmin")},
                "check": dict(check, ok=ok),
                "step_ms": step_ms}
        print(json.dumps(line), flush=True)
    V.close()
    if world > 1:
        dist.destroy_process_group()
    if rank == 0 and not ok and not args.no_check:
        sys.exit(1)


if __name__ == "__main__":
    main()
