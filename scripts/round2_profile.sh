#!/bin/bash
# Round-2 evidence run (one GPU call): host/GPU info, the default bench line (config D) with
# clocks, the ncu launch list of the same command, one ncu --set full capture of every pass
# kernel of a short D-grid gradient, and the GPU test suite + smoke. Outputs into gpurun_out/.
tag=${1:-r2a}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$tag.txt
(nproc; lscpu | head -20; free -g) > gpurun_out/host_$tag.txt
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$tag.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; tail -1 gpurun_out/smoke_$tag.log
python bench.py > gpurun_out/bench_full_$tag.json 2> gpurun_out/bench_full_$tag.err
echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_full_$tag.json
python bench.py --cpu-baseline 0 --e2e-steps 0 --steps 1 --warmup 3 > gpurun_out/bench_short_$tag.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --cpu-baseline 0 --e2e-steps 0 --steps 1 --warmup 3 \
    > gpurun_out/ncu_list_$tag.log 2>&1
echo "ncu list rc=$?"
python scripts/prof_step.py --config D --nt 4 --grad > gpurun_out/prof_plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pencil_|zvel|zrho|zp2_kernel" -s 0 -c 9 \
    -o gpurun_out/prof_full_$tag python scripts/prof_step.py --config D --nt 4 --grad > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu full rc=$?"
# the adjoint's correlating pressure kernel (pair loop only)
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:zp2_kernel.*[(]bool[)]1, [(]bool[)]0" -s 0 -c 1 \
    -o gpurun_out/prof_corr_$tag python scripts/prof_step.py --config D --nt 4 --grad > gpurun_out/ncu_corr_$tag.log 2>&1
echo "ncu corr rc=$?"
