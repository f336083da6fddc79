"""Merge a fresh ncu summary database (gpurun_out/prof/ncu_r02.json, written on the GPU box by
ncu_summary.py --db) into profiles/ncu_traffic.json: the r02_* captures and the bench keys that
alias them (bench.py looks up config2_f64, config1_f64, ... for `traffic` and `issue_roofline`).

usage: python scripts/ncu_merge.py [gpurun_out/prof/ncu_r02.json]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ALIASES = {"config2_f64": "r02_bench2", "config1_f64": "r02_cfg1", "config0_f64": "r02_cfg0",
           "config2_warm_f64": "r02_warm2", "config3_f64": "r02_cfg3", "config4_f32": "r02_cfg4f32",
           "config4_f64": "r02_cfg4", "lp_f64": "r02_lp2", "brute_f64": "r02_brute1"}

src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "prof", "ncu_r02.json")
new = json.load(open(src))
path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
db = json.load(open(path))
for k, v in new.items():
    db[k] = v
for alias, k in ALIASES.items():
    if k in new:
        db[alias] = dict(new[k], alias_of=k)
json.dump(db, open(path, "w"), indent=1, sort_keys=True)
print(f"merged {len(new)} captures into {path}")
