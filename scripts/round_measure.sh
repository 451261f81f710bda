#!/bin/bash
# Round measurement bundle (run under gpurun): bench lines, in-graph kernel breakdown (CUPTI),
# serialized launch lists (ncu), full ncu captures of the dominant kernel (a6) fp32 and bf16.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_fp32.json 2> gpurun_out/bench_fp32.err
timeout 900 python bench.py --dtype bf16 --steps 20 --warmup 5 --no-cpu --legs "" > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err
for dt in fp32 bf16; do
  timeout 300 python scripts/profile_step.py --dtype $dt --graph > gpurun_out/cupti_c2_${dt}_recompute.txt 2>&1
  timeout 300 python scripts/profile_step.py --dtype $dt --graph --mode stash > gpurun_out/cupti_c2_${dt}_stash.txt 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "step/" --csv \
      --log-file gpurun_out/launches_${dt}.csv python scripts/profile_step.py --ncu --dtype $dt > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_tma -s 3 -c 1 \
      -o gpurun_out/a6_c2_${dt} python scripts/kernel_bench.py --only attn_bwd --reps 3 --dtype $dt > /dev/null 2>&1
done
timeout 300 python scripts/kernel_bench.py > gpurun_out/kernels_fp32.txt 2>&1
timeout 300 python scripts/kernel_bench.py --dtype bf16 > gpurun_out/kernels_bf16.txt 2>&1
timeout 300 python scripts/kernel_bench.py --batch 4096 --reps 10 > gpurun_out/kernels_fp32_b4096.txt 2>&1
ls -la gpurun_out
