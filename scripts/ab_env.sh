#!/bin/bash
# dev helper: the D-grid proxy bench under different values of one environment variable,
# interleaved twice, on one box. usage: ab_env.sh tag VAR value1 value2 ...
tag=$1; var=$2; shift 2
for rep in 1 2; do
  for v in "$@"; do
    env $var=$v python bench.py --config D --nt 200 --steps 2 --warmup 1 --cpu-baseline 0 --e2e-steps 0 > gpurun_out/abenv_${tag}_${v}_$rep.json 2>&1
    python - "$var=$v.$rep" "gpurun_out/abenv_${tag}_${v}_$rep.json" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], "%.3f s/grad"%d["s_per_gradient"], d["clocks"]["sm_mhz"], {k:(round(v["ms_per_launch"],3), round(v["achieved_GBps"])) for k,v in d["kernels"].items()})
except Exception as e: print(sys.argv[1], "ERR", open(sys.argv[2]).read()[-800:])
PY
  done
done
