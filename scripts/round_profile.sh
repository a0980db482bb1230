#!/bin/bash
# Full default bench (config D) + clocks, the ncu launch list of the same command, and one
# full ncu capture of each pass kernel on a short D-grid run. Outputs into gpurun_out/.
tag=$1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$tag.txt
nproc > gpurun_out/host_$tag.txt; lscpu | head -20 >> gpurun_out/host_$tag.txt; free -g >> gpurun_out/host_$tag.txt
python bench.py > gpurun_out/bench_full_$tag.json 2> gpurun_out/bench_full_$tag.err
echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_full_$tag.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --cpu-baseline 0 --e2e-steps 0 --steps 1 --warmup 3 \
    > gpurun_out/ncu_list_$tag.log 2>&1
echo "ncu list rc=$?"
python scripts/prof_step.py --config D --nt 4 --grad > gpurun_out/prof_plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pencil_|zvel|zrho|zp_kernel|zp2_kernel" -s 0 -c 9 \
    -o gpurun_out/prof_full_$tag python scripts/prof_step.py --config D --nt 4 --grad > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu full rc=$?"
