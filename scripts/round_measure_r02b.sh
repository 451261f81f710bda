#!/bin/bash
# Round-2 closing bundle (run under gpurun): the full GPU suite at HEAD, bench lines (fp32 with every
# leg + CPU baseline, bf16), kernel benches at C2 and B = 4096 / 24576, ncu --set full of the a5 rows
# kernel (B = 4096 and 24576, bf16 and fp32) and of a6 at C2 fp32, the launch list of the bench step.
# Everything lands in gpurun_out/r02b_*.
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/r02b_gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02b_pytest.txt 2>&1
echo "pytest exit $?" >> gpurun_out/r02b_pytest.txt
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02b_bench_fp32.json 2> gpurun_out/r02b_bench_fp32.err
timeout 900 python bench.py --dtype bf16 --steps 20 --warmup 5 --no-cpu --legs "" > gpurun_out/r02b_bench_bf16.json 2> gpurun_out/r02b_bench_bf16.err
for dt in fp32 bf16; do
  timeout 300 python scripts/kernel_bench.py --dtype $dt > gpurun_out/r02b_kernels_c2_${dt}.txt 2>&1
  for b in 4096 24576; do
    timeout 300 python scripts/kernel_bench.py --only attn_fwd --batch $b --reps 10 --dtype $dt > gpurun_out/r02b_a5_${dt}_${b}.txt 2>&1
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_rows -s 3 -c 1 \
        -o gpurun_out/r02b_a5rows_${dt}_${b} python scripts/kernel_bench.py --only attn_fwd --batch $b --reps 3 --dtype $dt > /dev/null 2>&1
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_tma -s 3 -c 1 \
    -o gpurun_out/r02b_a6_c2_fp32 python scripts/kernel_bench.py --only attn_bwd --reps 3 --dtype fp32 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "step/" --csv \
    --log-file gpurun_out/r02b_launches_fp32.csv python scripts/profile_step.py --ncu --dtype fp32 > /dev/null 2>&1
ls -la gpurun_out | grep r02b
