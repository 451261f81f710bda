#!/bin/bash
# a5/a6: the four TMA chunks issued by four lanes of warp 0 instead of one thread
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_nmt.py -x -q > gpurun_out/ln_pytest.txt 2>&1
for dt in fp32 bf16; do
  timeout 300 python scripts/kernel_bench.py --only attn --dtype $dt --reps 30 > gpurun_out/ln_k_$dt.txt 2>&1
  timeout 300 python scripts/kernel_bench.py --only attn --dtype $dt --batch 4096 --reps 10 > gpurun_out/ln_k4096_$dt.txt 2>&1
  timeout 900 python bench.py --dtype $dt --steps 20 --warmup 5 --no-cpu --legs "" > gpurun_out/ln_bench_$dt.json 2> gpurun_out/ln_bench_$dt.err
done
