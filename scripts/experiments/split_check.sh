#!/bin/bash
# split a6 experiment (under gpurun): bitwise tests, step time with / without the side-stream accumulation
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_nmt.py -x -q -k deferred > gpurun_out/sp_pytest.txt 2>&1
for sp in 0 1; do
  for dt in fp32 bf16; do
    ECHO_A6_SPLIT=$sp timeout 600 python bench.py --dtype $dt --steps 20 --warmup 5 --no-cpu --legs "" --quick > gpurun_out/sp_bench_${dt}_$sp.json 2> gpurun_out/sp_bench_${dt}_$sp.err
  done
  ECHO_A6_SPLIT=$sp timeout 300 python scripts/profile_step.py --dtype bf16 --graph > gpurun_out/sp_cupti_bf16_$sp.txt 2>&1
done
ECHO_A6_SPLIT=1 timeout 900 python bench.py --dtype bf16 --batch 24576 --steps 3 --warmup 2 --no-cpu --legs "" --quick > gpurun_out/sp_bench_c5_1.json 2> gpurun_out/sp_bench_c5_1.err
ECHO_A6_SPLIT=0 timeout 900 python bench.py --dtype bf16 --batch 24576 --steps 3 --warmup 2 --no-cpu --legs "" --quick > gpurun_out/sp_bench_c5_0.json 2> gpurun_out/sp_bench_c5_0.err
