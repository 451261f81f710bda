mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 900 python -m pytest -q tests/test_gpu_attention.py tests/test_gpu_xent.py tests/test_gpu_lstm.py tests/test_gpu_lstm_vec.py > gpurun_out/r2_v3_tests.txt 2>&1
for dt in fp32 bf16; do
timeout 300 python scripts/kernel_bench.py --batch 4096 --reps 10 --dtype $dt > gpurun_out/r2_v3_k4096_${dt}.txt 2>&1
timeout 300 python scripts/kernel_bench.py --batch 128 --reps 20 --dtype $dt > gpurun_out/r2_v3_k128_${dt}.txt 2>&1
done
timeout 300 python scripts/colsum_bench.py > gpurun_out/r2_colsum_v3.txt 2>&1
timeout 900 python -m pytest -q tests/test_gpu_nmt.py tests/test_gpu_ds2.py tests/test_gpu_transformer.py > gpurun_out/r2_v3_models.txt 2>&1
