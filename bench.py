#!/usr/bin/env python3
"""Benchmark: LAD-LASSO solves/sec (n=30, p=5, fp64) on B200 -- BASELINE.json's metric.

Workload (BASELINE.json configs[2], the largest n=30/p=5 configuration): the
lambda path -- 2^20 datasets generated as config 0, each solved at a 16-point
log-spaced lambda grid 1e-2..1e1 (cold solves: the reference has no warm-start
knob), with both outer searches as the config states.  One bench
*step* = one block of datasets (default 2^14) x all 16 lambdas x {ternary,
quadrature} = 524,288 solves per GPU (two launches over the same resident
datasets); the whole config is 64 such steps.
Weak scaling: rank r of N solves block (step * N + r).

Timing: per-step CUDA events on the launching stream, L2 flushed (256 MiB
memset) between steps outside the events, barrier + synchronize around the
timed region, max over ranks.  ``e2e`` repeats the workload through the
host-buffer C ABI call (pinned host inputs, H2D + solve + D2H inside the
timed region).  ``cpu_baseline`` is the CPU oracle (a C restatement of the
reference's solve_locus, oracle/) on a bounded sample of the same problems,
all host threads.  ``--impl reference`` times that same CPU path as the
reference arm.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from types import SimpleNamespace

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LAD-LASSO solves/sec (n=30,p=5 fp64) at 1/2/4/8 B200; % of roofline"
N_ROWS, N_FEAT = 30, 5
LAMBDA_GRID = 10.0 ** np.linspace(-2.0, 1.0, 16)
TOTAL_DATASETS = 1 << 20
SEED = 15649 + 2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--block", type=int, default=1 << 14, help="datasets per step per GPU (x16 lambdas)")
    ap.add_argument("--variant", choices=["ternary", "quadrature", "both"], default=None,
                    help="outer search; default: both for config 2 (as BASELINE states), quadrature for "
                         "config 3, ternary otherwise")
    ap.add_argument("--cpu-sample", type=int, default=2048,
                    help="CPU baseline sample: datasets (x16 lambdas) for config 2, problems otherwise (~10 s of CPU)")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--config", type=int, default=2, choices=[0, 1, 2, 3, 4],
                    help="BASELINE config (2 = the metric's n=30/p=5 lambda path, the default)")
    ap.add_argument("--block4", type=int, default=1 << 16, help="config 4 problems per step per GPU")
    ap.add_argument("--solver", choices=["locus", "lp", "brute"], default="locus",
                    help="locus (the metric); lp = the simplex on config-2 problems; brute = the check on config 1")
    ap.add_argument("--warm-groups", type=int, default=2,
                    help="--warm: dataset groups walking their lambda stages on concurrent streams (path.py)")
    ap.add_argument("--warm", action="store_true",
                    help="config 2 warm-start lambda path (previous lambda's solution seeds the bracket)")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="torch.distributed backend for the barrier / max-reduce (gloo: the 1-GPU multi-rank test)")
    ap.add_argument("--dtype", choices=["f64", "f32"], default="f64",
                    help="f32: the fp32 mode (binary32 data and descents; config 4 runs in both)")
    return ap.parse_args()


def flops_per_solve(steps, descents, n=N_ROWS, p=N_FEAT):
    """Algorithmic FP64 flops: S*(8n+4) + D*(4np+4n+4p)."""
    return steps * (8 * n + 4) + descents * (4 * n * p + 4 * n + 4 * p)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        # nvidia-smi's start-up (driver attach, first query) can pause the GPU briefly: let it
        # finish before the timed region begins (sampling then continues through the region)
        t0 = time.time()
        while self.proc is not None and time.time() - t0 < 5.0:
            try:
                if os.path.getsize(self.path) > 0:
                    break
            except OSError:
                break
            time.sleep(0.05)
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 8:
                    rows.append(parts)
        except OSError:
            pass
        finally:
            if self.path and os.path.exists(self.path):
                os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        loaded = [r for r in rows if (num(r[7]) or 0) > 0] or rows
        sm = [num(r[0]) for r in loaded if num(r[0]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": num(rows[0][1]),
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(loaded),
                "power_w_max": max((num(r[2]) or 0) for r in rows)}


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def variants_of(a, config):
    """Outer searches one step runs (config 2 states both, config 3 quadrature)."""
    v = a.variant or {2: "both", 3: "quadrature"}.get(config, "ternary")
    return ["ternary", "quadrature"] if v == "both" else [v]


CPU_SAMPLE = {0: 256, 1: 1 << 16, 2: 128, 3: 2048, 4: 256}  # per step: solves (config 2: datasets x 16 lambdas)
SEEDS = {c: 15649 + c for c in range(5)}


def block_for_step(step, world, rank, nblocks):
    """Weak-scaling schedule (paper_2510_15649_b200.distributed.block_for_step, restated here so the
    reference arm imports nothing from the product package)."""
    return (step * world + rank) % nblocks


def shard_range(B, world, rank):
    """Contiguous shard of rank (paper_2510_15649_b200.distributed.shard_range)."""
    base, extra = divmod(B, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def step_first(config, a, s, world, rank):
    """First problem (config 2: first dataset) of bench step s on `rank` -- shared by both arms."""
    if config == 2:
        return block_for_step(s, world, rank, TOTAL_DATASETS // a.block) * a.block
    if config == 3:
        return shard_range(142506, world, rank)[0]
    return (s * world + rank) * {0: 256, 1: 1 << 20, 4: a.block4}[config]


def workload_config(config, a, world):
    """The workload description both arms print (identical dicts: the driver compares them)."""
    variants = variants_of(a, config)
    n, p = {0: (30, 5), 1: (10, 2), 2: (30, 5), 3: (25, 5), 4: (31, 8)}[config]
    if config == 2:
        desc = (f"config 2 lambda path: 2^20 datasets (n=30, p=5, config-0 distributions) x 16 lambdas 1e-2..1e1; "
                f"step = {a.block} datasets x 16 lambdas x {'+'.join(variants)}")
        solves = a.block * 16
    elif config == 3:
        s0, e0 = shard_range(142506, world, 0)
        desc = "config 3: C(30,25)=142506 row subsets of one dataset, lambda=0.5, quadrature"
        solves = e0 - s0
    else:
        solves = {0: 256, 1: 1 << 20, 4: a.block4}[config]
        desc = {0: "config 0: B=256, n=30, p=5, lambda=1, ternary",
                1: "config 1: B=2^20, n=10, p=2, lambda~U(0.1,2), thread-per-problem kernel",
                4: f"config 4: n=31, p=8, Student-t(3) X, Cauchy noise, lambda=1; step = {solves} of the 2^26 problems"}[config]
    cfg = {"workload": f"config{config}", "description": desc, "n": n, "p": p,
           "solves_per_step_per_gpu": solves * len(variants), "variant": "+".join(variants),
           "dtype": a.dtype, "parallelism": f"shard{world} (independent problems, no collective)",
           "inputs": f"seeded synthetic (Philox keyed by seed {SEEDS[config]} and problem index)"}
    if a.warm:
        cfg["warm"] = True
        cfg["description"] += ("; warm-started path: largest lambda first, then initial_bracket (-R, R), "
                               "R = max(1, 2 max|beta_prev|) (paper_2510_15649_b200/path.py), 16 dependent "
                               f"stages per variant, {a.warm_groups} dataset groups on concurrent streams")
    return cfg


def host_step_problems(config, a, s, world, rank, limit):
    """The first `limit` solves' inputs of bench step s, generated on the HOST by the oracle's
    restatement of the device generator (oracle/gen_host.c; byte-identical to lad_generate_f64,
    tests/test_gpu_generator.py) -- the reference arm never loads the product library."""
    from oracle import oracle as O

    first = step_first(config, a, s, world, rank)
    if config == 2:
        X, Y, _ = O.generate(2, limit, SEEDS[2], first)
        return np.repeat(X, 16, axis=0), np.repeat(Y, 16, axis=0), np.tile(LAMBDA_GRID, limit)
    if config == 3:
        X0, Y0 = O.config3_dataset(SEEDS[3])
        X, Y = O.subsets(X0, Y0, 25, first, limit)
        return X, Y, np.full(limit, 0.5)
    return O.generate(config, limit, SEEDS[config], first)


def run_reference(a, rank, world):
    """Reference arm: the reference's solve_locus restated on the CPU (the oracle, a C port pinned
    bit-exact to the reference) on all host threads, on a bounded sample of each bench step's
    problems generated on the host; rank 0 only.  Loads no product code (no torch either)."""
    if rank != 0:
        return
    from oracle import oracle as O

    O.build()
    config = a.config
    variants = variants_of(a, config)
    limit = CPU_SAMPLE[config] // (1 if config == 2 else len(variants))
    nth = cpu_threads()
    fp32 = a.dtype == "f32"
    times, solves = [], 0
    for s in range(a.warmup + a.steps):
        X, Y, L = host_step_problems(config, a, s, world, rank, limit)
        if fp32:
            X, Y, L = X.astype(np.float32), Y.astype(np.float32), L.astype(np.float32)
        t0 = time.perf_counter()
        for v in variants:
            if a.warm:  # the warm lambda path (paper_2510_15649_b200/path.py's rule) on the oracle
                O.solve_warm_path(X[::16], Y[::16], LAMBDA_GRID, outer_search=v, nthreads=nth)
            else:
                O.solve_locus_batch(X, Y, L, nthreads=nth, outer_search=v)
        dt = time.perf_counter() - t0
        if s >= a.warmup:
            times.append(dt)
            solves += X.shape[0] * len(variants)
    total = sum(times)
    value = solves / total
    per = solves // a.steps
    sample = (f"first {per // len(variants)} solves of each bench step "
              f"({limit} datasets x 16 lambdas)" if config == 2 else f"first {per // len(variants)} problems of each bench step")
    line = {"metric": metric_name(a), "impl": "reference", "value": value, "unit": "solves/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * total / a.steps, "higher_is_better": True,
            "scaling": "weak" if config != 3 else "strong", "vs_baseline": None, "dtype": a.dtype,
            "data": "synthetic (host restatement of the device Philox generator, BASELINE config distributions)",
            "config": workload_config(config, a, world),
            "cpu_baseline": {"value": value, "unit": "solves/s", "cores": nth, "kind": "port",
                             "sample": f"{sample} x {'+'.join(variants)}, {a.steps} timed steps after {a.warmup} "
                                       f"warm-up; CPU oracle (C restatement of solve_locus, pinned bit-exact to "
                                       f"the reference){', binary32 build' if fp32 else ''} on {nth} threads"},
            "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def metric_name(a):
    if a.config == 2 and a.dtype == "f64" and not a.warm:
        return METRIC
    n, p = {0: (30, 5), 1: (10, 2), 2: (30, 5), 3: (25, 5), 4: (31, 8)}[a.config]
    return f"LAD-LASSO solves/sec (config {a.config}{' warm' if a.warm else ''}, n={n},p={p} {a.dtype.replace('f', 'fp')})"


class Workload:
    """One bench step's device inputs for a BASELINE config (inputs resident before timing)."""

    def __init__(self, config, a, world, rank, dev):
        self._build(config, a, world, rank, dev)
        if a.dtype == "f32":  # generated in binary64, rounded once to binary32 on the device
            self.steps_inputs = [tuple(t.float() for t in inp) for inp in self.steps_inputs]
            if self.lam is not None:
                self.lam = self.lam.float()

    def _build(self, config, a, world, rank, dev):
        import torch
        from paper_2510_15649_b200 import configgen as G

        self.config = config
        self.variants = variants_of(a, config)
        self.n, self.p = G.CONFIG_SHAPES[config]
        self.dev = dev
        self.data_index = None
        self.steps_inputs = []
        nsteps = a.warmup + a.steps
        solves = workload_config(config, a, world)["solves_per_step_per_gpu"] // len(self.variants)
        if config == 2:
            blk = a.block
            for s in range(nsteps):
                X, Y, _ = G.generate(2, blk, seed=SEEDS[2], first=step_first(2, a, s, world, rank), device=dev)
                self.steps_inputs.append((X, Y))
            self.data_index = torch.arange(blk, device=dev, dtype=torch.int64).repeat_interleave(16)
            self.lam = torch.tensor(LAMBDA_GRID, device=dev, dtype=torch.float64).repeat(blk)
        elif config == 3:
            X0, Y0 = G.config3_dataset(seed=SEEDS[3], device=dev)
            s0, e0 = shard_range(G.CONFIG_BATCH[3], world, rank)
            Xs, Ys = G.subsets(X0, Y0, 25, s0, e0 - s0)
            self.steps_inputs = [(Xs, Ys)] * nsteps
            self.lam = torch.full((e0 - s0,), 0.5, device=dev, dtype=torch.float64)
            solves = e0 - s0
        else:
            for s in range(nsteps):
                X, Y, L = G.generate(config, solves, seed=SEEDS[config], first=step_first(config, a, s, world, rank),
                                     device=dev)
                self.steps_inputs.append((X, Y, L))
            self.lam = None
        self.solves = solves

    def inputs(self, s):
        t = self.steps_inputs[s]
        if len(t) == 3:
            return t[0], t[1], t[2]
        return t[0], t[1], self.lam

    def cpu_sample(self, s, max_solves):
        """Exact bytes of the first problems of step s, expanded to (X, Y, lam) per solve."""
        X, Y, L = self.inputs(s)
        if self.data_index is not None:
            nd = max(1, max_solves // 16)
            Xh = np.repeat(X[:nd].cpu().numpy(), 16, axis=0)
            Yh = np.repeat(Y[:nd].cpu().numpy(), 16, axis=0)
            Lh = np.tile(LAMBDA_GRID, nd)
            return Xh, Yh, Lh
        m = min(max_solves, X.shape[0])
        return X[:m].cpu().numpy(), Y[:m].cpu().numpy(), L[:m].cpu().numpy()


def lp_flops(pivots, m, d):
    """Algorithmic FP64 flops of the dense tableau simplex: per pivot (n+1) divisions for the pivot
    row + 2 (mul, sub) per entry of the other m rows; setup m*n products + (m+1)*n sums."""
    n = 2 * d + 2 * m
    return pivots * ((n + 1) + 2 * m * (n + 1)) + 2 * (m + 1) * n


def brute_flops(vertices, m, d):
    """Per nonsingular vertex: Gaussian elimination (2/3 d^3 + 2 d^2) and the objective (2md + 2m + 2d)."""
    return vertices * (2.0 / 3.0 * d ** 3 + 2 * d * d + 2 * m * d + 2 * m + 2 * d)


def ncu_lookup(key, solves_per_launch, units, elapsed, clocks, dev, unit):
    """`traffic` (DRAM bytes per launch) and `issue_roofline` of a bench line from the committed ncu
    --set full summary profiles/ncu_traffic.json[key]: bytes per solve x solves per launch, and warp
    instructions per work unit x the live work-unit rate against 4 warp instructions per SM per cycle
    at the sampled SM clock.  (None, None) without a capture of this workload."""
    import torch

    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(key)
    except (OSError, ValueError):
        return None, None
    if not tr:
        return None, None
    traffic = tr["bytes_per_solve"] * solves_per_launch if tr.get("bytes_per_solve") is not None else None
    issue = None
    ipu = tr.get("warp_instr_per_unit") or tr.get("warp_instr_per_coord_step")
    if ipu and clocks.get("sm_mhz") and elapsed > 0:
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        peak_issue = 4 * sms * clocks["sm_mhz"] * 1e6  # one warp instruction per SMSP per cycle
        ach = ipu * units / elapsed
        issue = {"bound": "issue", "achieved": ach / 1e9, "peak": peak_issue / 1e9, "unit": "G warp-instr/s",
                 "frac": ach / peak_issue, f"warp_instr_per_{unit.replace(' ', '_')}": ipu,
                 "ncu_issue_active_pct": tr.get("issue_active_pct"), "ncu_key": key,
                 "source": f"instr/{unit} from profiles/ncu_traffic.json x live {unit}s/s; "
                           "peak = 4 SMSPs x SMs x sampled SM clock"}
    return traffic, issue


def run_aux(a, world, rank, local):
    """--solver lp | brute: the widened rows (the check of §8a a17), same protocol."""
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    import paper_2510_15649_b200 as lad
    from paper_2510_15649_b200 import _lib, configgen as G
    from paper_2510_15649_b200.solver import fp64_peak_tflops

    if a.solver == "lp":
        config, B = 2, 1 << 16
        n, p = G.CONFIG_SHAPES[2]
        desc = f"simplex (lp.solve_lp) on config-2 problems: {B} (dataset, lambda) pairs per step, n=30, p=5"
        steps_inputs = []
        for s_ in range(a.warmup + a.steps):
            X, Y, _ = G.generate(2, B // 16, seed=SEED, first=((s_ * world + rank) * (B // 16)) % TOTAL_DATASETS,
                                 device=dev)
            idx = torch.arange(B // 16, device=dev).repeat_interleave(16)
            lam = torch.tensor(LAMBDA_GRID, device=dev, dtype=torch.float64).repeat(B // 16)
            steps_inputs.append((X[idx].contiguous(), Y[idx].contiguous(), lam))

        def solve(k):
            X, Y, L = steps_inputs[k]
            return lad.solve_lp_batched(X, Y, L)

        def flops(r):
            return lp_flops(float(r.pivots.double().sum()), n, p)
    else:
        config, B = 1, 1 << 20
        n, p = G.CONFIG_SHAPES[1]
        desc = f"brute-force vertex check (brute.solve_brute) on config 1: B={B}, n=10, p=2, C(12,2)=66 vertices"
        steps_inputs = [G.generate(1, B, seed=SEED - 2 + 1, first=(s_ * world + rank) * B, device=dev)
                        for s_ in range(a.warmup + a.steps)]

        def solve(k):
            X, Y, L = steps_inputs[k]
            return lad.solve_brute_batched(X, Y, L)

        def flops(r):
            return brute_flops(float(r[2].double().sum()), n, p)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    peak = fp64_peak_tflops()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for k in range(a.warmup):
        solve(k)
    barrier()
    stream = torch.cuda.current_stream(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    results = []
    launches0 = _lib.kernel_launches()
    with ClockSampler(local) as clk:
        barrier()
        # a step here is a few ms of GPU time, about what the host needs to enqueue it: a short spin
        # kernel first lets the host run ahead, so the events time the GPU and not the enqueue gaps
        if hasattr(torch.cuda, "_sleep") and not os.environ.get("LAD_BENCH_NO_SPIN"):
            torch.cuda._sleep(200_000_000)
        for k in range(a.steps):
            flush.zero_()
            evs[k][0].record(stream)
            results.append(solve(a.warmup + k))
            evs[k][1].record(stream)
        barrier()
    gpu_launches = _lib.kernel_launches() - launches0
    clocks = clk.summary()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    elapsed = sum(step_ms) / 1e3
    t = torch.tensor([elapsed], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    value = world * a.steps * B / float(t.item())
    fl = sum(flops(r) for r in results)
    achieved = fl / elapsed / 1e12
    # work units of the timed launches (pivots / nonsingular vertices) for the issue roofline
    units = sum(float(r.pivots.double().sum()) if a.solver == "lp" else float(r[2].double().sum()) for r in results)
    # e2e through the public API with host (pinned) inputs and host outputs, over the same number of
    # steps as the device-timed region (distinct host inputs within 2 GiB of pinned memory, cycled)
    step_bytes = sum(v.numel() * v.element_size() for v in steps_inputs[a.warmup])
    n_host = max(1, min(a.steps, (2 << 30) // max(1, step_bytes)))
    hosts = []
    for k in range(n_host):
        hx, hy, hl = (torch.empty(v.shape, dtype=v.dtype, pin_memory=True).copy_(v) for v in steps_inputs[a.warmup + k])
        hosts.append((hx.numpy(), hy.numpy(), hl.numpy()))
    run_host = (lambda h: lad.solve_lp_batched(*h)) if a.solver == "lp" else (lambda h: lad.solve_brute_batched(*h))
    run_host(hosts[0])  # untimed full-size warm-up (allocator and pool growth)
    barrier()
    t0 = time.perf_counter()
    for k in range(a.steps):
        run_host(hosts[k % n_host])
    barrier()
    e2e_value = world * a.steps * B / (time.perf_counter() - t0)
    h2d = sum(v.nbytes for v in hosts[0])
    d2h = B * (p * 8 + 8 + 4 + 1 + 1) if a.solver == "lp" else B * (p * 8 + 8 + 8)
    traffic, issue = ncu_lookup(f"{a.solver}_f64", B, units, elapsed, clocks, dev,
                                "pivot" if a.solver == "lp" else "nonsingular vertex")
    cpu = parity = None
    if rank == 0 and world == 1 and not a.no_cpu:
        from oracle import oracle as O

        O.build()
        Xh, Yh, Lh = (v.cpu().numpy() for v in steps_inputs[a.warmup])
        g = results[0]
        t0 = time.perf_counter()
        nsol = exact = 0
        while nsol < B and time.perf_counter() - t0 < 10.0:  # single-thread oracle, ~10 s sample
            lam_eff = max(float(Lh[nsol]), 1e-9)
            if a.solver == "lp":
                o = O.lp_solve(Xh[nsol], Yh[nsol], lam_eff)
                gb, go = g.beta[nsol].cpu().numpy(), float(g.objective[nsol])
                ok = np.array_equal(gb, o.beta) and go == o.objective and int(g.pivots[nsol]) == o.pivots
            else:
                ob, oo, ov = O.solve_brute(Xh[nsol], Yh[nsol], lam_eff)
                ok = np.array_equal(g[0][nsol].cpu().numpy(), ob) and float(g[1][nsol]) == oo
            exact += int(ok)
            nsol += 1
        dt = time.perf_counter() - t0
        what = "lp.solve_lp (oracle orc_lp_solve)" if a.solver == "lp" else "brute.solve_brute (oracle orc_solve_brute)"
        cpu = {"value": nsol / dt, "unit": "solves/s", "cores": 1, "kind": "port",
               "sample": f"first {nsol} problems of the first timed step, {what}, 1 thread, {dt:.1f} s "
                         "(includes the GPU-vs-oracle comparison)"}
        parity = {"sample": nsol, "bit_exact": exact}
    if rank == 0:
        metric = ("LP (dense simplex) solves/sec (n=30,p=5 fp64)" if a.solver == "lp"
                  else "brute-force vertex checks/sec (config 1: n=10,p=2 fp64)")
        print(json.dumps({
            "metric": metric, "value": value, "unit": "solves/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": float(t.item()) * 1e3 / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device Philox generator with the BASELINE config distributions)",
            "config": {"workload": f"{a.solver}_config{config}", "description": desc, "n": n, "p": p,
                       "solves_per_step_per_gpu": B, "parallelism": f"shard{world} (independent problems)",
                       "l2": "flushed between steps (256 MiB memset)"},
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": "profiles/ncu_traffic.json (dram__bytes_read+write per solve) x solves per launch",
                         "flops_model": "bench.lp_flops" if a.solver == "lp" else "bench.brute_flops"},
            "issue_roofline": issue,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "solves/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "steps": a.steps, "distinct_input_steps": n_host},
            "gpu_launches": gpu_launches, "clocks": clocks, "parity_sample": parity, "step_ms": step_ms}),
            flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.warm and a.config != 2:
        raise SystemExit("--warm is the config-2 lambda path mode")
    if a.impl == "reference":
        return run_reference(a, rank, world)
    if a.solver != "locus":
        return run_aux(a, world, rank, local)

    import torch
    import torch.distributed as dist

    dev = torch.device("cuda", local % torch.cuda.device_count())  # ranks > GPUs only in the gloo test
    torch.cuda.set_device(dev)
    backend = a.dist_backend
    if world > 1:
        dist.init_process_group(backend, **({"device_id": dev} if backend == "nccl" else {}))
    import paper_2510_15649_b200 as lad
    from paper_2510_15649_b200 import _lib
    from paper_2510_15649_b200.solver import fp32_peak_tflops, fp64_peak_tflops

    wl = Workload(a.config, a, world, rank, dev)
    cfgs = [lad.LocusConfig(outer_search=v) for v in wl.variants]
    solves_per_step = wl.solves * len(cfgs)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    peak = fp32_peak_tflops() if a.dtype == "f32" else fp64_peak_tflops()
    hdt = torch.float32 if a.dtype == "f32" else torch.float64

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def flat(path):
        """(datasets, lambdas, ...) path results as one flat per-solve record per variant"""
        return SimpleNamespace(**{k: v.reshape((-1,) + tuple(v.shape[2:])) for k, v in path.items()})

    def solve(s):
        X, Y, L = wl.inputs(s)
        if a.warm:  # 16 dependent launches per variant (path.py: largest lambda first, bracketed)
            return [flat(lad.solve_lambda_path_batched(X, Y, LAMBDA_GRID, c, warm=True, groups=a.warm_groups)) for c in cfgs]
        return [lad.solve_locus_batched(X, Y, L, c, data_index=wl.data_index) for c in cfgs]

    for s in range(a.warmup):
        solve(s)
    barrier()
    stream = torch.cuda.current_stream(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    results = []
    launches0 = _lib.kernel_launches()
    with ClockSampler(local) as clk:
        barrier()
        for k in range(a.steps):
            flush.zero_()
            evs[k][0].record(stream)
            r = solve(a.warmup + k)
            evs[k][1].record(stream)
            results.extend(r)
        barrier()
    gpu_launches = _lib.kernel_launches() - launches0
    clocks = clk.summary()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    elapsed = sum(step_ms) / 1e3
    t = torch.tensor([elapsed], device=dev if backend == "nccl" else "cpu", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_max = float(t.item())
    value = world * a.steps * solves_per_step / elapsed_max
    # algorithmic flops of the timed launches (exact per-problem counters)
    S = sum(float(r.steps.double().sum()) for r in results)
    D = sum(float(r.descents.double().sum()) for r in results)
    fl = flops_per_solve(S, D, wl.n, wl.p)
    achieved_tflops = fl / elapsed / 1e12
    status_ok = all(bool((r.status == 0).all()) for r in results)
    conv_frac = float(np.mean([float(r.converged.float().mean()) for r in results]))

    # ---- end to end through the host-buffer C ABI (pinned host memory, copies inside), over the
    # same number of steps as the device-timed region
    e2e_steps = a.e2e_steps if a.e2e_steps is not None else a.steps
    host = []
    step_bytes = sum(t.numel() * (4 if a.dtype == "f32" else 8) for t in wl.inputs(a.warmup))
    n_host = max(1, min(e2e_steps, (2 << 30) // max(1, step_bytes)))  # distinct steps within 2 GiB of pinned memory
    for k in range(n_host):
        bufs = []
        for v in wl.inputs(a.warmup + k):
            h = torch.empty(v.shape, dtype=hdt, pin_memory=True)
            h.copy_(v)
            bufs.append(h.numpy())
        host.append(tuple(bufs))
    hidx_np = None
    if wl.data_index is not None:
        hidx = torch.empty(wl.data_index.shape, dtype=torch.int64, pin_memory=True)
        hidx.copy_(wl.data_index)
        hidx_np = hidx.numpy()
    # untimed warm-up of the host-buffer path at full size (the device memory pool grows to the
    # step's buffers once; the device-side arm likewise runs its warm-up steps untimed)
    if a.warm:
        lad.solve_lambda_path_batched(host[0][0], host[0][1], LAMBDA_GRID, cfgs[0], warm=True, groups=a.warm_groups)
    else:
        lad.solve_locus_batched(host[0][0], host[0][1], host[0][2], cfgs[0], data_index=hidx_np)
    barrier()
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        h = host[k % n_host]
        for c in cfgs:  # each variant is one public-API call with its own H2D and D2H
            if a.warm:  # one public-API call per variant: X and Y cross once, every stage's results come back
                lad.solve_lambda_path_batched(h[0], h[1], LAMBDA_GRID, c, warm=True, groups=a.warm_groups)
            else:
                lad.solve_locus_batched(h[0], h[1], h[2], c, data_index=hidx_np)
    barrier()
    e2e_elapsed = time.perf_counter() - t0
    te = torch.tensor([e2e_elapsed], device=dev if backend == "nccl" else "cpu", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * e2e_steps * solves_per_step / float(te.item())
    h2d = len(cfgs) * (sum(x.nbytes for x in host[0]) + (hidx_np.nbytes if hidx_np is not None else 0))
    d2h = solves_per_step * (wl.p * 8 + 8 + 4 + 4 + 1 + 1 + 4 + 8)
    if a.warm:  # per variant: X and Y once (lambdas and brackets are made on the device)
        h2d = len(cfgs) * (host[0][0].nbytes + host[0][1].nbytes)

    # DRAM traffic per launch and warp instructions per coordinate step from the committed
    # ncu --set full capture of this workload (None otherwise)
    key = f"config{a.config}{'_warm' if a.warm else ''}_{a.dtype}"
    traffic, issue = ncu_lookup(key, wl.solves, S, elapsed, clocks, dev, "coordinate step")
    cpu = None
    parity = None
    fp32_dist = None
    if rank == 0 and world == 1 and not a.no_cpu:
        # ~10 s of CPU work per config on a 16-thread host (config 0 is the whole config)
        max_solves = {0: 256, 1: 1 << 20, 2: a.cpu_sample * 16, 3: 32768, 4: 8192}[a.config] // len(cfgs)
        Xh, Yh, Lh = wl.cpu_sample(a.warmup, max_solves)
        from oracle import oracle as O

        O.build()
        nth = cpu_threads()
        if a.dtype == "f32":  # the f32 workload's inputs are the fp64 problems rounded once
            X64, Y64, L64 = Xh.astype(np.float64), Yh.astype(np.float64), np.asarray(Lh, dtype=np.float64)
            Xh, Yh, Lh = Xh.astype(np.float32), Yh.astype(np.float32), np.asarray(Lh, dtype=np.float32)
        t0 = time.perf_counter()
        if a.warm:  # the oracle replay of the warm path on the sample's datasets (same rule, path.py)
            nd = Xh.shape[0] // 16
            ros = [{k: v.reshape((-1,) + v.shape[2:]) for k, v in
                    O.solve_warm_path(Xh[::16], Yh[::16], LAMBDA_GRID, outer_search=v, nthreads=nth).items()}
                   for v in wl.variants]
        else:
            ros = [O.solve_locus_batch(Xh, Yh, Lh, nthreads=nth, outer_search=v) for v in wl.variants]
        dt = time.perf_counter() - t0
        nsol = Xh.shape[0]
        cpu = {"value": nsol * len(ros) / dt, "unit": "solves/s", "cores": nth, "kind": "port",
               "sample": f"first {nsol} solves of the first timed step x {'+'.join(wl.variants)}, CPU oracle "
                         f"(C restatement of solve_locus{', binary32 build' if a.dtype == 'f32' else ''}) on "
                         f"{nth} threads, {dt:.1f} s"}
        exact = within = 0
        for g, ro in zip(results[:len(ros)], ros):  # the first timed step's launch per variant
            gb = g.beta[:nsol].cpu().numpy()
            go = g.objective[:nsol].cpu().numpy()
            gs = g.steps[:nsol].cpu().numpy()
            exact += int(np.sum(np.all(gb == ro["beta"], axis=1) & (go == ro["objective"]) & (gs == ro["steps"])))
            rel = np.abs(go - ro["objective"]) / np.abs(ro["objective"])
            within += int(np.sum(rel <= 1e-9))
        parity = {"sample": nsol * len(ros), "bit_exact": exact, "obj_within_1e-9": within,
                  "checker": "CPU oracle" + (" (binary32 build)" if a.dtype == "f32" else "")}
        if a.dtype == "f32":
            # the fp32 mode against the fp64 reference path (the oracle in binary64 = the reference
            # bit for bit) on the unrounded problems: a reported statistic, not a parity claim
            m = min(nsol, 1024)
            r64 = O.solve_locus_batch(X64[:m], Y64[:m], L64[:m], nthreads=nth, outer_search=wl.variants[0])
            g = results[0]
            go = g.objective[:m].cpu().numpy()
            rel = (go - r64["objective"]) / np.abs(r64["objective"])
            sup = np.all((np.abs(g.beta[:m].cpu().numpy()) > 1e-6) == (np.abs(r64["beta"]) > 1e-6), axis=1)
            fp32_dist = {"sample": m, "rel_obj_diff_max": float(np.max(np.abs(rel))),
                         "rel_obj_diff_median": float(np.median(rel)), "rel_obj_diff_p99": float(np.quantile(np.abs(rel), 0.99)),
                         "fp32_lower_frac": float(np.mean(rel < 0)), "support_equal_frac": float(np.mean(sup))}

    if rank == 0:
        line = {
            "metric": metric_name(a),
            "value": value, "unit": "solves/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": elapsed_max * 1e3 / a.steps, "higher_is_better": True,
            "scaling": "weak" if a.config != 3 else "strong", "vs_baseline": None, "dtype": a.dtype,
            "data": "synthetic (device Philox generator with the BASELINE config distributions)",
            "config": workload_config(a.config, a, world),
            "kernel": {1: "locus_kernel<10,2,1> thread-per-problem sm_100a"}.get(
                a.config, "locus_warp_kernel warp-per-problem sm_100a"),
            "l2": "flushed between steps (256 MiB memset, outside the events)",
            "roofline": {"bound": "fp64" if a.dtype == "f64" else "fp32", "achieved": achieved_tflops, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved_tflops / peak if peak else None, "traffic": traffic,
                         "traffic_source": "profiles/ncu_traffic.json (dram__bytes_read+write per solve) x solves per launch",
                         "peak_source": (f"measured {'DFMA' if a.dtype == 'f64' else 'FFMA'} loop on this GPU "
                                         f"(lad_{a.dtype.replace('f', 'fp')}_peak_tflops); "
                                         "MEASURED_PEAKS.json has no FP64/FP32 CUDA-core figure"),
                         "flops_per_solve": fl / (a.steps * solves_per_step),
                         "coord_steps_per_solve": S / (a.steps * solves_per_step),
                         "descents_per_solve": D / (a.steps * solves_per_step)},
            "issue_roofline": issue,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "solves/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "steps": e2e_steps, "distinct_input_steps": n_host},
            "fp32_vs_fp64_reference": fp32_dist,
            "gpu_launches": gpu_launches,
            "clocks": clocks,
            "status_ok": status_ok,
            "converged_frac": conv_frac,
            "parity_sample": parity,
            "step_ms": step_ms,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
