mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 900 python -m pytest -q -x tests/test_gpu_attention.py > gpurun_out/r2_a6p_tests.txt 2>&1
for dt in fp32 bf16; do
timeout 300 python scripts/kernel_bench.py --only attn --batch 4096 --reps 10 --dtype $dt > gpurun_out/r2_a6p_k4096_${dt}.txt 2>&1
timeout 300 python scripts/kernel_bench.py --only attn --batch 128 --reps 20 --dtype $dt > gpurun_out/r2_a6p_k128_${dt}.txt 2>&1
done
timeout 900 python -m pytest -q tests/test_gpu_nmt.py > gpurun_out/r2_a6p_nmt.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --quick > gpurun_out/r2_a6p_bench.json 2> gpurun_out/r2_a6p_bench.err
bash scripts/run_sanitizers.sh > gpurun_out/r2_sanitizers.txt 2>&1
