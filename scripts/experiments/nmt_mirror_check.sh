#!/bin/bash
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 1500 python -m pytest tests/test_gpu_nmt.py tests/test_gpu_ds2.py tests/test_gpu_lstm.py -x -q > gpurun_out/nm_pytest.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --legs "" > gpurun_out/nm_bench_fp32.json 2> gpurun_out/nm_bench_fp32.err
timeout 900 python bench.py --dtype bf16 --steps 10 --warmup 3 --no-cpu --legs "" > gpurun_out/nm_bench_bf16.json 2> gpurun_out/nm_bench_bf16.err
