#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --warm --steps 3 --warmup 3 > gpurun_out/r2_warm.json 2> gpurun_out/r2_warm.err; echo "warm rc=$?"
timeout 600 python bench.py --warm --impl reference --steps 3 --warmup 1 > gpurun_out/r2_warm_ref.json 2>&1; echo "ref rc=$?"
python3 - <<'PY'
import json
for f in ("gpurun_out/r2_warm.json", "gpurun_out/r2_warm_ref.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"]), "e2e", round(d["e2e"]["value"]), d.get("parity_sample"), d.get("ms_per_step"))
    except Exception as e:
        print(f, "ERR", e)
PY
tail -5 gpurun_out/r2_warm.err
