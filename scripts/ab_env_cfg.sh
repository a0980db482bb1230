#!/bin/bash
# dev helper: bench.py on one config under several environment settings, interleaved twice.
# usage: ab_env_cfg.sh tag CONFIG "ENV=a" "ENV=b" ...
tag=$1; cfg=$2; shift 2
for rep in 1 2; do
  i=0
  for v in "$@"; do
    i=$((i+1))
    env $v python bench.py --config $cfg --steps 3 --warmup 3 --cpu-baseline 0 --e2e-steps 0 > gpurun_out/abcfg_${tag}_${i}_$rep.json 2>&1
    python - "$cfg $v [$rep]" "gpurun_out/abcfg_${tag}_${i}_$rep.json" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], "%.4f s/grad"%d["s_per_gradient"], d["clocks"]["sm_mhz"], {k:(round(v["ms_per_launch"],4), round(v["achieved_GBps"])) for k,v in d["kernels"].items()})
except Exception as e: print(sys.argv[1], "ERR", open(sys.argv[2]).read()[-800:])
PY
  done
done
