#!/bin/bash
# Round-2 measurement bundle (run under gpurun): bench lines (fp32 with every leg + CPU baseline, bf16),
# in-graph kernel tables (CUPTI), serialized launch lists (ncu), per-kernel benches, the tcgen05 step
# bench, colsum, a 2-rank functional bench.  Everything lands in gpurun_out/r02m_*.
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/r02m_gpu.txt
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02m_bench_fp32.json 2> gpurun_out/r02m_bench_fp32.err
timeout 900 python bench.py --dtype bf16 --steps 20 --warmup 5 --no-cpu --legs "" > gpurun_out/r02m_bench_bf16.json 2> gpurun_out/r02m_bench_bf16.err
for dt in fp32 bf16; do
  timeout 300 python scripts/profile_step.py --dtype $dt --graph > gpurun_out/r02m_cupti_c2_${dt}_recompute.txt 2>&1
  timeout 300 python scripts/profile_step.py --dtype $dt --graph --mode stash > gpurun_out/r02m_cupti_c2_${dt}_stash.txt 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "step/" --csv \
      --log-file gpurun_out/r02m_launches_${dt}.csv python scripts/profile_step.py --ncu --dtype $dt > /dev/null 2>&1
  timeout 300 python scripts/kernel_bench.py --dtype $dt > gpurun_out/r02m_kernels_c2_${dt}.txt 2>&1
  timeout 300 python scripts/kernel_bench.py --batch 4096 --reps 10 --dtype $dt > gpurun_out/r02m_kernels_b4096_${dt}.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_tma -s 3 -c 1 \
    -o gpurun_out/r02m_a6_c2_bf16 python scripts/kernel_bench.py --only attn_bwd --reps 3 --dtype bf16 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lstm_cscan -s 3 -c 1 \
    -o gpurun_out/r02m_a2_b4096_bf16 python scripts/kernel_bench.py --only cscan --batch 4096 --reps 3 --dtype bf16 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:colsum_vec -s 2 -c 1 \
    -o gpurun_out/r02m_colsum python scripts/colsum_bench.py --reps 1 --only fp32 > /dev/null 2>&1
timeout 300 python scripts/colsum_bench.py > gpurun_out/r02m_colsum.txt 2>&1
timeout 300 python scripts/lstm_tc_bench.py > gpurun_out/r02m_tc_bench.txt 2>&1
timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --quick > gpurun_out/r02m_bench_gpus2.json 2> gpurun_out/r02m_bench_gpus2.err
ls -la gpurun_out | grep r02m
