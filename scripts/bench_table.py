"""Markdown table of the committed round-end bench lines (profiles/r01_final_*.json).

usage: python scripts/bench_table.py [--write]   (--write replaces the table in profiles/r01_summary.md
between the <!-- bench-table --> markers)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")

ROWS = [
    ("bench_default", "**config 2** (the metric: n=30, p=5, fp64, λ path, ternary + quadrature, 524,288 solves/step)"),
    ("bench_reference", "reference arm (`--impl reference`: the CPU oracle, all host threads, both variants)"),
    ("bench_config2_ternary", "config 2, ternary only"),
    ("bench_config2_quadrature", "config 2, quadrature only"),
    ("bench_config0", "config 0 (B=256, ternary; latency-bound)"),
    ("bench_config1", "config 1 (B=2^20, n=10, p=2, thread-per-problem)"),
    ("bench_config3", "config 3 (C(30,25)=142,506 subsets, quadrature)"),
    ("bench_config4", "config 4 fp64 (n=31, p=8, 65,536 problems/step)"),
    ("bench_config4_f32", "config 4 fp32 (fp32 mode)"),
    ("bench_lp", "LP: dense tableau simplex (`lp.solve_lp`) on config-2 problems, 65,536/step"),
    ("bench_brute", "brute-force vertex check (`brute.solve_brute`) on config 1, 2^20/step"),
]


def n(x):
    return f"{x:,.0f}"


def table():
    out = ["| workload | solves/s (device) | e2e (host ABI) | CPU oracle | roofline | parity sample |",
           "|---|---|---|---|---|---|"]
    for f, label in ROWS:
        path = os.path.join(P, f"r01_final_{f}.json")
        if not os.path.exists(path):
            continue
        d = json.loads(open(path).read().strip().splitlines()[-1])
        if d.get("impl") == "reference":
            out.append(f"| {label} | {n(d['value'])} | — | — | — | — |")
            continue
        r = d.get("roofline") or {}
        iss = d.get("issue_roofline") or {}
        roof = f"{100 * r['frac']:.1f}% of {r['peak']:.1f} TF/s {'DFMA' if r['bound'] == 'fp64' else 'FFMA'}"
        if iss:
            roof += f"; issue {100 * iss['frac']:.0f}%"
        c = d.get("cpu_baseline")
        cpu = f"{n(c['value'])} ({c['cores']} thr)" if c else "—"
        par = d.get("parity_sample")
        ps = f"{par['bit_exact']:,} / {par['sample']:,}" if par else "—"
        label = label if not label.startswith("**") else label
        dev = f"**{n(d['value'])}**" if f == "bench_default" else n(d["value"])
        out.append(f"| {label} | {dev} | {n(d['e2e']['value'])} | {cpu} | {roof} | {ps} |")
    return "\n".join(out)


if __name__ == "__main__":
    t = table()
    if "--write" in sys.argv:
        sp = os.path.join(P, "r01_summary.md")
        s = open(sp).read()
        a, b = s.index("<!-- bench-table -->"), s.index("<!-- /bench-table -->")
        s = s[:a] + "<!-- bench-table -->\n" + t + "\n" + s[b:]
        open(sp, "w").write(s)
    print(t)
