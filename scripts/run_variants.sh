#!/bin/bash
# GPU side: bench each variant library (FG_LIB) on a config and print phases.
# usage: scripts/run_variants.sh CONFIG name1 name2 ...
cfg=$1; shift
for v in "$@"; do
  lib=paper_2204_00525_b200/lib_$v/libfigaro_cuda.so
  [ "$v" = base ] && lib=paper_2204_00525_b200/lib/libfigaro_cuda.so
  FG_LIB=$PWD/$lib python bench.py --config $cfg --steps 6 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1 > gpurun_out/var_${cfg}_$v.json 2> gpurun_out/var_${cfg}_$v.err
  python - <<PY
import json
try:
    d=json.loads(open("gpurun_out/var_${cfg}_$v.json").read().strip().splitlines()[-1])
    print("$v $cfg", round(d["ms_per_step"],2), {k:round(x,2) for k,x in d["phases_ms"].items()}, "ht", round(d["roofline"].get("ms_per_launch",0)*d["roofline"].get("launches_per_step",0),2))
except Exception as e:
    print("$v $cfg FAILED", e)
PY
done
