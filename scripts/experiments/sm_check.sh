#!/bin/bash
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_nmt.py -x -q > gpurun_out/sm_pytest.txt 2>&1
for dt in fp32 bf16; do
  timeout 300 python scripts/kernel_bench.py --only attn --dtype $dt --reps 20 > gpurun_out/sm_k_$dt.txt 2>&1
  timeout 300 python scripts/kernel_bench.py --only attn --dtype $dt --batch 4096 --reps 10 > gpurun_out/sm_k4096_$dt.txt 2>&1
done
timeout 600 python scripts/profile_step.py --dtype bf16 --graph --batch 24576 > gpurun_out/cupti_c5_bf16_recompute.txt 2>&1
