mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 600 python -m pytest -q tests/test_gpu_lstm_tc.py > gpurun_out/r2_tc1_tests.txt 2>&1
timeout 300 python scripts/lstm_tc_bench.py > gpurun_out/r2_tc1_bench.txt 2>&1
timeout 2400 python -m pytest -q tests/test_gpu_sanitizer.py > gpurun_out/r2_tc1_sanitizer.txt 2>&1
bash scripts/run_sanitizers.sh > gpurun_out/r2_sanitizers2.txt 2>&1
