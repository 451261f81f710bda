mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 900 python -m pytest -q -x tests/test_gpu_attention.py > gpurun_out/r2_a5fast_tests.txt 2>&1
for dt in bf16 fp32; do
timeout 300 python scripts/kernel_bench.py --only attn_fwd --batch 4096 --reps 10 --dtype $dt > gpurun_out/r2_a5fast_b4096_${dt}.txt 2>&1
timeout 300 python scripts/kernel_bench.py --only attn_fwd --batch 128 --reps 20 --dtype $dt > gpurun_out/r2_a5fast_c2_${dt}.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_tma -s 3 -c 1 \
     -o gpurun_out/r2_a5fast_b4096_bf16 python scripts/kernel_bench.py --only attn_fwd --batch 4096 --reps 3 --dtype bf16 > /dev/null 2>&1
