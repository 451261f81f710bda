#!/bin/bash
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 1500 python -m pytest tests/test_gpu_nmt.py tests/test_gpu_attention.py tests/test_gpu_transformer.py -x -q > gpurun_out/dr_pytest.txt 2>&1
