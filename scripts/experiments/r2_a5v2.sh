mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 900 python -m pytest -q -x tests/test_gpu_attention.py tests/test_gpu_xent.py > gpurun_out/r2_a5v2_tests.txt 2>&1
for b in 4096 128; do for dt in fp32 bf16; do
timeout 300 python scripts/kernel_bench.py --only attn_fwd --batch $b --reps 10 --dtype $dt > gpurun_out/r2_a5v2_${b}_${dt}.txt 2>&1
done; done
timeout 300 python scripts/colsum_bench.py > gpurun_out/r2_colsum_v2.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_tma -s 3 -c 1 \
     -o gpurun_out/r2_a5v2_b4096_fp32 python scripts/kernel_bench.py --only attn_fwd --batch 4096 --reps 3 --dtype fp32 > /dev/null 2>&1
timeout 900 python -m pytest -q -x tests/test_gpu_nmt.py -k "c2 or small" > gpurun_out/r2_a5v2_nmt.txt 2>&1
