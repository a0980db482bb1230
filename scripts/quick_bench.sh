#!/bin/bash
# dev helper: GPU tests + short benches; summary printed at the end
tag=$1
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_$tag.log 2>&1; tail -3 gpurun_out/gpu_tests_$tag.log
for c in A B; do python bench.py --config $c --steps 3 --warmup 3 --cpu-baseline 0 --e2e-steps 0 > gpurun_out/bench_${tag}_$c.json 2>gpurun_out/bench_${tag}_$c.err; done
python bench.py --config D --nt 200 --steps 2 --warmup 1 --cpu-baseline 0 --e2e-steps 0 > gpurun_out/bench_${tag}_D200.json 2>gpurun_out/bench_${tag}_D200.err
python - <<PY
import json
for f in ["A","B","D200"]:
    try:
        d=json.loads(open("gpurun_out/bench_${tag}_%s.json"%f).read().strip().splitlines()[-1])
        print(f, "%.3f s/grad"%d["s_per_gradient"], "%.3g vu/s"%d["value"], {k:(round(v["ms_per_launch"],3), round(v["achieved_GBps"])) for k,v in d["kernels"].items()})
    except Exception as e: print(f, "ERR", e, open("gpurun_out/bench_${tag}_%s.err"%f).read()[-500:])
PY
