"""Markdown table of the round-2 bench lines (profiles/r02/final/bench_*.json) beside round 1's
(profiles/r01_final_bench_*.json).

usage: python scripts/bench_table_r02.py
"""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")
ROWS = [
    ("bench_default", "**config 2** (the metric: n=30, p=5, fp64, λ path, ternary + quadrature)"),
    ("bench_reference", "reference arm (`--impl reference`: CPU oracle, all host threads)"),
    ("bench_config2_ternary", "config 2, ternary only"),
    ("bench_config2_quadrature", "config 2, quadrature only"),
    ("bench_config2_warm", "config 2, warm-started λ path (`--warm`)"),
    ("bench_config0", "config 0 (B=256; latency-bound)"),
    ("bench_config1", "config 1 (B=2^20, n=10, p=2, thread per problem)"),
    ("bench_config3", "config 3 (142,506 subsets, quadrature)"),
    ("bench_config4", "config 4 fp64 (n=31, p=8)"),
    ("bench_config4_f32", "config 4 fp32 mode"),
    ("bench_lp", "LP simplex on config-2 problems"),
    ("bench_brute", "brute-force vertex check, config 1"),
]


def load(path):
    if not os.path.exists(path):
        return None
    return json.loads(open(path).read().strip().splitlines()[-1])


def main():
    print("| workload | round 1 | **round 2** (device) | e2e (host ABI) | CPU oracle | FP64 roofline | issue roofline | parity sample |")
    print("|---|---|---|---|---|---|---|---|")
    for f, label in ROWS:
        d = load(os.path.join(P, "r02", "final", f"{f}.json"))
        if d is None:
            continue
        r1 = load(os.path.join(P, f"r01_final_{f}.json"))
        r1v = f"{r1['value']:,.0f}" if r1 and "value" in r1 else "—"
        if d.get("impl") == "reference":
            print(f"| {label} | {r1v} | {d['value']:,.0f} | — | {d['cpu_baseline']['cores']} threads | — | — | — |")
            continue
        cpu = d.get("cpu_baseline") or {}
        rf = d.get("roofline") or {}
        iss = d.get("issue_roofline") or {}
        ps = d.get("parity_sample") or {}
        par = f"{ps.get('bit_exact'):,} / {ps.get('sample'):,}" if ps else "—"
        cpus = f"{cpu['value']:,.0f} ({cpu['cores']} thr)" if cpu else "—"
        issue = f"{100 * iss['frac']:.0f}%" if iss.get("frac") is not None else "—"
        print(f"| {label} | {r1v} | **{d['value']:,.0f}** | {d['e2e']['value']:,.0f} | {cpus} | "
              f"{100 * rf.get('frac', 0):.1f}% of {rf.get('peak', 0):.1f} TF/s | {issue} | {par} |")


if __name__ == "__main__":
    main()
