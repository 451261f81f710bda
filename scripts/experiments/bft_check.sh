#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tanh_err scripts/micro/tanh_err.cu && /tmp/tanh_err > gpurun_out/bft_err.txt 2>&1
python -m paper_1805_08899_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_nmt.py -x -q > gpurun_out/bft_pytest.txt 2>&1
for b in 128 4096; do
  timeout 300 python scripts/kernel_bench.py --only attn --dtype bf16 --batch $b --reps 10 > gpurun_out/bft_k${b}.txt 2>&1
done
timeout 1500 python bench.py --dtype bf16 --steps 20 --warmup 5 --no-cpu --legs C5 > gpurun_out/bft_bench.json 2> gpurun_out/bft_bench.err
