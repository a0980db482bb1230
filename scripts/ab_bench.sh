#!/bin/bash
# dev helper: GPU tests, then the D-grid proxy bench under two environment variants
tag=$1; shift
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_$tag.log 2>&1; tail -2 gpurun_out/gpu_tests_$tag.log
for v in "$@"; do
  env $v python bench.py --config D --nt 200 --steps 2 --warmup 1 --cpu-baseline 0 --e2e-steps 0 > gpurun_out/ab_${tag}_${v//=/_}.json 2>&1
  python - "$v" "gpurun_out/ab_${tag}_${v//=/_}.json" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], "%.3f s/grad"%d["s_per_gradient"], {k:(round(v["ms_per_launch"],3), round(v["achieved_GBps"])) for k,v in d["kernels"].items()})
except Exception as e: print(sys.argv[1], "ERR", open(sys.argv[2]).read()[-800:])
PY
done
