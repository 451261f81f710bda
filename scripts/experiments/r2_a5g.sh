mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 900 python -m pytest -q -x tests/test_gpu_attention.py > gpurun_out/r2_a5g_tests.txt 2>&1
for dt in fp32 bf16; do
timeout 300 python scripts/kernel_bench.py --only attn_fwd --batch 4096 --reps 10 --dtype $dt > gpurun_out/r2_a5g_b4096_${dt}.txt 2>&1
timeout 300 python scripts/kernel_bench.py --only attn_fwd --batch 128 --reps 20 --dtype $dt > gpurun_out/r2_a5g_c2_${dt}.txt 2>&1
done
