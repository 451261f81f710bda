#!/bin/bash
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_nmt.py -x -q > gpurun_out/ho_pytest.txt 2>&1
for dt in fp32 bf16; do
  timeout 300 python scripts/kernel_bench.py --only attn --dtype $dt > gpurun_out/ho_k_$dt.txt 2>&1
  timeout 300 python scripts/kernel_bench.py --only attn --dtype $dt --batch 4096 --reps 10 > gpurun_out/ho_k4096_$dt.txt 2>&1
done
timeout 1500 python bench.py --dtype bf16 --steps 20 --warmup 5 --no-cpu --legs C5 > gpurun_out/ho_bench.json 2> gpurun_out/ho_bench.err
