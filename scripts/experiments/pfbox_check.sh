#!/bin/bash
# a6: dKp / dH_s L2 prefetch as one whole-tile box per tensor (2 TMA prefetches instead of 8)
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_nmt.py -x -q > gpurun_out/pb_pytest.txt 2>&1
for dt in fp32 bf16; do
  timeout 300 python scripts/kernel_bench.py --only attn_bwd --dtype $dt --reps 30 > gpurun_out/pb_k_$dt.txt 2>&1
  timeout 300 python scripts/kernel_bench.py --only attn_bwd --dtype $dt --batch 4096 --reps 10 > gpurun_out/pb_k4096_$dt.txt 2>&1
  timeout 900 python bench.py --dtype $dt --steps 20 --warmup 5 --no-cpu --legs "" > gpurun_out/pb_bench_$dt.json 2> gpurun_out/pb_bench_$dt.err
done
