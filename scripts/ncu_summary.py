"""Summarise ncu --set full captures of the library's kernels into profiles/ncu_traffic.json.

usage: python scripts/ncu_summary.py [--db OUT.json] OUTDIR WORKLOAD...   (reads OUTDIR/prof_WORKLOAD.ncu-rep and
OUTDIR/units_WORKLOAD.json written by scripts/gpurun/r2_profile_all.sh)
Per workload: kernel duration, warp instructions per work unit (coordinate step / vertex / pivot /
problem), issue-slot utilisation, resident warps, active threads per warp, FP64 / LSU / ALU pipe
utilisation, DRAM bytes (read + write) per launch and per solve, L2 hit rate, registers, and the
top stall reasons per issued instruction.  bench.py reads `bytes_per_solve` and
`warp_instr_per_unit` (the roofline `traffic` and `issue_roofline`).
"""
import csv
import io
import json
import os
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}
WANT = {
    "duration_s": "gpu__time_duration.sum",
    "warp_instr": "smsp__inst_executed.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_per_sm": "sm__warps_active.avg.per_cycle_active",
    "threads_per_warp_instr": "smsp__thread_inst_executed_per_inst_executed.ratio",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    kern = [r for r in rows[2:] if r]
    return h, u, kern[-1]  # the profiled launch (one per capture)


def num(v, unit):
    try:
        return float(v.replace(",", "")) * SCALE.get(unit, 1.0)
    except ValueError:
        return None


def summarise(rep, units):
    h, u, v = raw(rep)
    idx = {n: i for i, n in enumerate(h)}
    s = {}
    for key, name in WANT.items():
        if name in idx:
            s[key] = num(v[idx[name]], u[idx[name]])
    s["kernel"] = v[idx["Kernel Name"]] if "Kernel Name" in idx else None
    stalls = {}
    for n, i in idx.items():
        if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
            val = num(v[i], u[i])
            if val and val > 0.05:
                stalls[n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(val, 3)
    s["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:7])
    s.update({k: units[k] for k in ("unit", "units", "solves", "n", "p") if k in units})
    if units.get("units"):
        s["warp_instr_per_unit"] = s["warp_instr"] / units["units"]
    if s.get("dram_read_bytes") is not None:
        s["dram_bytes"] = s["dram_read_bytes"] + s["dram_write_bytes"]
        s["bytes_per_solve"] = s["dram_bytes"] / units["solves"]
    return s


def main():
    args = sys.argv[1:]
    path = os.path.join("profiles", "ncu_traffic.json")
    if "--db" in args:  # write elsewhere (on the GPU box: under gpurun_out/, merged here afterwards)
        i = args.index("--db")
        path = args[i + 1]
        del args[i:i + 2]
    out, works = args[0], args[1:]
    db = json.load(open(path)) if os.path.exists(path) else {}
    for w in works:
        rep = os.path.join(out, f"prof_{w}.ncu-rep")
        uj = os.path.join(out, f"units_{w}.json")
        if not (os.path.exists(rep) and os.path.exists(uj)):
            print(f"{w}: missing capture", file=sys.stderr)
            continue
        s = summarise(rep, json.load(open(uj)))
        s["source"] = f"ncu --set full --clock-control none, one launch of scripts/prof_kernels.py {w} (round 2)"
        db[f"r02_{w}"] = s
        print(w, json.dumps({k: (round(x, 3) if isinstance(x, float) else x) for k, x in s.items()}))
    json.dump(db, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
