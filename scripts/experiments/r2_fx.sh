mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 900 python -m pytest -q -rf tests/test_gpu_fx_pass.py > gpurun_out/r2_fx_tests.txt 2>&1
