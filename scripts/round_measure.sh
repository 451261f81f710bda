#!/bin/bash
# Round measurement bundle (run under gpurun): bench lines, launch list, full profile of the top kernel.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_fp32.json 2> gpurun_out/bench_fp32.err
timeout 900 python bench.py --dtype bf16 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "step/" --csv \
    --log-file gpurun_out/launches_fp32.csv python scripts/profile_step.py --ncu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step/" -k regex:attn_bwd -s 10 -c 1 \
    -o gpurun_out/attn_bwd_step python scripts/profile_step.py --ncu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step/" -k regex:lstm_bwd -s 20 -c 1 \
    -o gpurun_out/lstm_bwd_step python scripts/profile_step.py --ncu > /dev/null 2>&1
timeout 300 python scripts/kernel_bench.py > gpurun_out/kernels_fp32.txt 2>&1
timeout 300 python scripts/kernel_bench.py --batch 4096 --reps 10 > gpurun_out/kernels_fp32_b4096.txt 2>&1
ls -la gpurun_out
