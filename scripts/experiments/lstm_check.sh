#!/bin/bash
# LSTM vector-width change (under gpurun): parity / bit-identity tests, kernel timings, bench, CUPTI
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_lstm.py tests/test_gpu_lstm_vec.py tests/test_gpu_ds2.py tests/test_gpu_nmt.py -x -q > gpurun_out/lc_pytest.txt 2>&1
for dt in fp32 bf16; do
  timeout 300 python scripts/kernel_bench.py --only lstm --dtype $dt > gpurun_out/lc_k_${dt}.txt 2>&1
  timeout 600 python bench.py --dtype $dt --steps 10 --warmup 3 --no-cpu --legs "" > gpurun_out/lc_bench_$dt.json 2> gpurun_out/lc_bench_$dt.err
  timeout 300 python scripts/profile_step.py --dtype $dt --graph > gpurun_out/lc_cupti_$dt.txt 2>&1
done
timeout 300 python scripts/kernel_bench.py --only lstm --batch 4096 --reps 10 > gpurun_out/lc_k4096_fp32.txt 2>&1
