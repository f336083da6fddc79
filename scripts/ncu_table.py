"""Markdown table of the round-2 ncu --set full captures in profiles/ncu_traffic.json (keys r02_*).

usage: python scripts/ncu_table.py [--keys k1,k2,...]
One row per capture: kernel, work unit, warp instructions per unit, issue-slot utilisation, resident
warps per SM, active threads per warp instruction, FP64 / LSU / ALU pipe utilisation, DRAM bytes per
solve, L2 hit rate, registers and the top three stall reasons per issued instruction.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
db = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
keys = sys.argv[sys.argv.index("--keys") + 1].split(",") if "--keys" in sys.argv else sorted(k for k in db if k.startswith("r02_"))


def f(v, fmt):
    return "-" if v is None else format(v, fmt)


print("| capture | kernel | unit | instr/unit | issue % | warps/SM | thr/warp-instr | FP64 % | LSU % | ALU % | "
      "DRAM B/solve | L2 hit % | regs | top stalls per issue |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for k in keys:
    v = db[k]
    stalls = sorted(((a, b) for a, b in v.get("stalls_per_issue", {}).items() if a != "selected"), key=lambda x: -x[1])
    st = ", ".join(f"{a} {b:.2f}" for a, b in stalls[:3])
    kern = (v.get("kernel") or "").replace("void ", "").replace("(LocusArgs)", "").replace("lad::", "")
    kern = kern.split("(")[0]
    print(f"| {k[4:]} | `{kern}` | {v.get('unit', '-')} | {f(v.get('warp_instr_per_unit'), '.1f')} | "
          f"{f(v.get('issue_active_pct'), '.1f')} | {f(v.get('warps_active_per_sm'), '.1f')} | "
          f"{f(v.get('threads_per_warp_instr'), '.1f')} | {f(v.get('fp64_pipe_pct'), '.1f')} | "
          f"{f(v.get('lsu_pipe_pct'), '.1f')} | {f(v.get('alu_pipe_pct'), '.1f')} | {f(v.get('bytes_per_solve'), '.0f')} | "
          f"{f(v.get('l2_hit_pct'), '.1f')} | {f(v.get('registers'), '.0f')} | {st} |")
