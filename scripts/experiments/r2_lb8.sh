mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 900 python -m pytest -q -x tests/test_gpu_attention.py > gpurun_out/r2_lb8_tests.txt 2>&1
for dt in bf16 fp32; do
for b in 4096 24576; do
timeout 300 python scripts/kernel_bench.py --only attn_fwd --batch $b --reps 10 --dtype $dt > gpurun_out/r2_lb8_${b}_${dt}.txt 2>&1
done
timeout 300 python scripts/kernel_bench.py --only attn_fwd --batch 128 --reps 20 --dtype $dt > gpurun_out/r2_lb8_128_${dt}.txt 2>&1
done
