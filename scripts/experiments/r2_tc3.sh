mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 600 python -m pytest -q tests/test_gpu_lstm_tc.py > gpurun_out/r2_tc3_tests.txt 2>&1
timeout 300 python scripts/lstm_tc_bench.py > gpurun_out/r2_tc3_bench.txt 2>&1
