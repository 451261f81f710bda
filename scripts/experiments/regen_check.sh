#!/bin/bash
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 1200 python -m pytest tests/test_gpu_transformer.py tests/test_gpu_attention.py -x -q > gpurun_out/rg_pytest.txt 2>&1
timeout 1200 python bench.py --dtype bf16 --steps 5 --warmup 3 --no-cpu --legs C4 > gpurun_out/rg_bench.json 2> gpurun_out/rg_bench.err
