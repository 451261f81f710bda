mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 1200 python -m pytest -q -rf tests/test_gpu_dp_parity.py tests/test_gpu_nmt.py > gpurun_out/r2_retest.txt 2>&1
bash scripts/experiments/r2_prof1.sh
