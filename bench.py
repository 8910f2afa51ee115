#!/usr/bin/env python3
"""Benchmark: exhaustive minimal-Goldbach-prime verification of every even n in
[4, N] (default N = 1e12, BASELINE.json configs[3], the metric's workload) on
1..8 B200s.  One "step" = the whole hot path over the whole range: K-SIEVE +
inverted marking + fallback in the fused kernel for every strip, the result
finalize, and the NCCL reduction of the result vector.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--N 1e12] [--impl ours|reference]

Prints ONE JSON line on rank 0.  Metric: even n verified per second, whole job,
device-timed (CUDA events on the launching stream, max over ranks), L2 flushed
between steps.  Strong scaling: the range is fixed and sharded over ranks.
`--impl reference` times the CPU oracle (oracle/, the paper's cpu_goldbach
definition) on the host cores on a bounded sample of the same
workload -- the reference arm of this tier.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "even n verified/sec (whole box, device-timed) to N=1e12"
UNIT = "even_n/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--N", type=float, default=1e12)
    ap.add_argument("--workload", default="c4", choices=["c4", "c5"],
                    help="c4: every even n in [4, N] (the metric's workload); c5: the window "
                         "[4e18 - 1e11, 4e18) of BASELINE.json configs[4]")
    ap.add_argument("--p-max", type=int, default=65521)
    ap.add_argument("--mode", default="bulk", choices=["bulk", "pern", "resident"],
                    help="bulk: the product path (inverted bulk marking); pern: the paper's per-n "
                         "gpu3 kernel (NEXT-1, PAPER.md:82-95); resident: the paper's gpu2 with the "
                         "whole odd bitset of [3, hi) sieved into HBM each step (NEXT-2, PAPER.md:41-59)")
    ap.add_argument("--strips-per-rank", type=int, default=None,
                    help="default 8 for c4 (balances the growth of work with n), 2 for c5 (the "
                         "window's cost is flat; fewer partial K-LARGE chunks)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sieve", action="store_true", help="skip the standalone sieve GB/s leg")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    a = ap.parse_args()
    if a.strips_per_rank is None:
        a.strips_per_rank = 2 if a.workload == "c5" else 8
    return a


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
def workload(args):
    """(lo, hi, origin, description, algorithmic int32 ops per even n) of the run."""
    if args.workload == "c5":
        top = 4 * 10**18
        return top - 10**11, top, top - 10**11, "C5 window: every even n in [4e18 - 1e11, 4e18)", C5_OPS_PER_EVEN
    N = int(args.N)
    return 4, N + 1, 0, f"N={N:.0e} exhaustive verification, even n in [4, N]", ALU_OPS_PER_EVEN


def oracle_sample(hi: int, target_s: float, lo_min: int = 4):
    """Time the CPU oracle (as it stands) on a top slice of [lo_min, hi), growing the
    slice until it has run for at least target_s seconds."""
    from oracle import oracle
    threads = oracle.default_threads()
    span = 1 << 27
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
    lo, hi, _, desc, _ = workload(args)
    per_step = max(1.0, args.cpu_seconds / 4)
    for _ in range(args.warmup):
        oracle_sample(hi, per_step / 4, lo)
    vals, times, evens = [], [], 0
    first = oracle_sample(hi, per_step, lo)
    for i in range(args.steps):
        s = first if i == 0 else oracle_sample(hi, per_step, lo)
        vals.append(s["value"])
        times.append(s["seconds"])
        evens += s["evens"]
    value = evens / sum(times)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (deterministic number-theoretic range)", "impl": "reference",
            "config": {"workload": desc, "lo": lo, "hi": hi, "sample": first["sample"]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": first["cores"], "kind": "oracle",
                             "sample": f"{args.steps} top-of-range slices of [{lo}, {hi}), ~{per_step:.1f} s each"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

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

    lo, hi, origin, desc, ops_per_even = workload(args)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    V = Verifier(hi_max=hi, p_max=args.p_max, origin=origin, device=local, stream=stream)
    strips = gdist.rank_strips(gdist.plan_strips(lo, hi, args.strips_per_rank * world), rank, world)
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(max(4 * l2_bytes, 1 << 28) // 4, dtype=torch.int32, device=dev)

    bits = None
    if args.mode == "resident":
        n_bits_words = (hi - 3) // 128 + 1
        bits = torch.empty(n_bits_words, dtype=torch.int64, device=dev)

    def step(k_events=None):
        r = V.new_result()
        if bits is not None:                         # gpu2: sieve [3, hi) into HBM, then per-n lookups
            gb.gb_sieve_segment(V.ctx, 0, bits.numel(), bits, stream)
            for a, b in strips:
                gb.gb_verify_range_resident(V.ctx, a, b, args.p_max, bits, bits.numel(), r, None, stream)
            V.finalize(r)
            gdist.reduce_result(r)
            return r
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
    step_ms, k_events, results = [], [], []
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

    # ---- end to end through the C-ABI host entry point (host result buffer)
    e2e = None
    import numpy as np
    h_res = torch.empty(gb.RESULT_WORDS, dtype=torch.int64).pin_memory()
    e2e_steps = max(1, min(args.steps, 3))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        acc = np.zeros(gb.RESULT_WORDS, dtype=np.int64)
        for a, b in strips:
            gb.gb_verify_range_host(V.ctx, a, b, args.p_max, h_res, None, stream)
            acc += h_res.numpy()
    if world > 1:
        tt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt[0])
    else:
        e2e_s = time.perf_counter() - t0
    e2e = {"value": evens * e2e_steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 0,
           "d2h_bytes_per_step": 8 * gb.RESULT_WORDS * len(strips),
           "note": "gb_verify_range_host per strip: init+verify+finalize+D2H of the 52 KB result; "
                   "inputs are (lo, hi, p_max) scalars, no array H2D; cross-rank sum not included"}

    # ---- roofline of the dominant kernel (the fused verify kernel)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    n_launch = len(kern_ms)
    avg_launch_s = (sum(kern_ms) / n_launch) / 1e3 if n_launch else float("nan")
    evens_per_launch = evens / max(1, len(strips) * world)
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    alu_peak = 148 * 64 * sm_mhz * 1e6 / 1e12           # T int32 lane-ops/s on the ALU pipe
    achieved = ops_per_even * evens_per_launch / avg_launch_s / 1e12 if n_launch else None
    traffic, traffic_src = None, None
    try:   # DRAM bytes per even n of verify_kernel from the latest committed ncu --set full capture
        import glob
        caps = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_verify_kernel_ncu.json")))
        if caps:
            cap = json.load(open(caps[-1]))
            traffic = cap["dram_bytes_per_even"] * evens_per_launch
            traffic_src = os.path.relpath(caps[-1], ROOT)
    except Exception:
        pass
    roofline = {"bound": "alu", "achieved": achieved, "peak": alu_peak, "unit": "Tops/s",
                "frac": achieved / alu_peak if achieved else None, "traffic": traffic,
                "traffic_note": (f"DRAM read+write bytes per launch, scaled per even n from {traffic_src}"
                                 if traffic_src else None),
                "kernel": "verify_kernel (fused sieve + mark + fallback)",
                "ops_per_even": ops_per_even,
                "peak_basis": f"148 SM x 64 int32 lanes/clk (ALU pipe) x {sm_mhz:.0f} MHz (MEASURED_PEAKS sm_max_mhz)",
                "kernel_ms_per_launch": avg_launch_s * 1e3 if n_launch else None, "launches_timed": n_launch,
                "kernel_share_of_step": box_kern_ms / box_ms if box_ms else None}

    # ---- sieve GB/s (BASELINE.json metric, second half): standalone gb_sieve_segment
    # (K-SIEVE, the paper's odd-only layout PAPER.md:46-51) writing the bitset of the
    # top 2^34 integers of the range to HBM; bytes written / device time
    sieve = None
    if not args.no_sieve:
        nwords = 1 << 27                                   # u64 words = 2^34 integers, 1 GiB
        w_hi = (hi - 3) // 128
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
        hbm = peaks.get("hbm_gbs") or 6545.9
        sieve = {"value": nbytes / (ms / 1e3) / 1e9, "unit": "GB/s", "ms_per_launch": ms,
                 "odd_integers_per_s": 64 * (w_hi - w_lo) / (ms / 1e3),
                 "window": f"odd q in [{3 + 128 * w_lo}, {3 + 128 * w_hi})",
                 "kernel": "sieve_out_kernel (gb_sieve_segment)",
                 "hbm_frac": nbytes / (ms / 1e3) / 1e9 / hbm, "hbm_peak_gbps": hbm}
        del out

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_sample(hi, args.cpu_seconds, lo)
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": box_ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "u64",
                "data": "synthetic (deterministic number-theoretic range; no dataset)",
                "config": {"workload": desc, "lo": lo, "hi": hi, "p_max": args.p_max, "strips_per_rank": args.strips_per_rank,
                           "parallelism": f"range-sharded x{world}", "l2": "flushed between steps",
                           "mode": args.mode},
                "gpu_launches": launches, "clocks": clocks, "e2e": e2e, "roofline": roofline,
                "cpu_baseline": cpu, "sieve": sieve,
                "result": {k: res[k] for k in ("evens", "verified", "fastpath_unresolved", "unresolved",
                                                  "max_pmin", "max_pmin_n", "sum_pmin", "chk")},
                "step_ms": step_ms}
        print(json.dumps(line), flush=True)
    V.close()
    if world > 1:
        dist.destroy_process_group()


# Algorithmic int32 ops per even n at N = 1e12 (SURVEY.md section 8d "Algorithmic
# work per even n"; derivation in DESIGN.md section "Roofline"):
#   sieve : 2.387 bit-clears per odd (= per even n), 1 op each
#   mark  : 1.01 64-bit word-iterations per even n (64-even exit) x 6 int32 ops
#           (2 funnel shifts, 2 AND, 2 XOR)
ALU_OPS_PER_EVEN = 2.387 + 1.01 * 6
# the same yardstick in the C5 window ("4e18 window" row)
C5_OPS_PER_EVEN = 2.826 + 1.63 * 6

if __name__ == "__main__":
    main()
