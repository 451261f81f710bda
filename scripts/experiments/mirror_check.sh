#!/bin/bash
# Mirror-plan check (under gpurun): kernel + model tests, C3/C4 legs with the three plans
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 1200 python -m pytest tests/test_gpu_lstm.py tests/test_gpu_ds2.py tests/test_gpu_transformer.py -x -q > gpurun_out/mi_pytest.txt 2>&1
timeout 1200 python bench.py --dtype bf16 --steps 5 --warmup 3 --no-cpu --legs C3,C4 > gpurun_out/mi_bench.json 2> gpurun_out/mi_bench.err
timeout 1200 python bench.py --dtype bf16 --steps 5 --warmup 3 --no-cpu --legs C3,C4 --leg-dtype fp32 > gpurun_out/mi_bench_fp32legs.json 2> gpurun_out/mi_bench_fp32legs.err
