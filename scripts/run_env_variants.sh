#!/bin/bash
# GPU side: bench the default library under different environment settings.
# usage: scripts/run_env_variants.sh CONFIG "NAME=VAL ..." "NAME=VAL ..." ...  ("-" = no extra env)
cfg=$1; shift
i=0
for e in "$@"; do
  i=$((i+1))
  envs=""; [ "$e" != "-" ] && envs="$e"
  env $envs python bench.py --config $cfg --steps 6 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1 > gpurun_out/env_${cfg}_$i.json 2> gpurun_out/env_${cfg}_$i.err
  python - <<PY
import json
try:
    d=json.loads(open("gpurun_out/env_${cfg}_$i.json").read().strip().splitlines()[-1])
    print("[$e] $cfg", round(d["ms_per_step"],2), {k:round(x,2) for k,x in d["phases_ms"].items()}, "ht", round(d["roofline"].get("ms_per_launch",0)*d["roofline"].get("launches_per_step",0),2))
except Exception as ex:
    print("[$e] $cfg FAILED", ex)
PY
done
