#!/bin/bash
# dev helper: the D-grid proxy bench with alternative builds of the library swapped in
# (scratch_so/<name>.so), interleaved twice, on one box. usage: ab_so.sh tag name1 name2 ...
tag=$1; shift
lib=paper_2102_00755_b200/libustfwi_b200.so
cp $lib /tmp/orig_lib.so
for rep in 1 2; do
  for v in "$@"; do
    cp scratch_so/$v.so $lib
    python bench.py --config D --nt 200 --steps 2 --warmup 1 --cpu-baseline 0 --e2e-steps 0 > gpurun_out/abso_${tag}_${v}_$rep.json 2>&1
    python - "$v.$rep" "gpurun_out/abso_${tag}_${v}_$rep.json" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], "%.3f s/grad"%d["s_per_gradient"], d["clocks"]["sm_mhz"], {k:(round(v["ms_per_launch"],3), round(v["achieved_GBps"])) for k,v in d["kernels"].items()})
except Exception as e: print(sys.argv[1], "ERR", open(sys.argv[2]).read()[-800:])
PY
  done
done
cp /tmp/orig_lib.so $lib
