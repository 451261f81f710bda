# a6 rows kernel: parity (both a6 kernels) + timing vs the cluster kernel
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 1200 python -m pytest -q -x tests/test_gpu_attention.py -k "a6_rows or a5_rows or parity_and_bit" > gpurun_out/r2_rows6_tests.txt 2>&1
for dt in bf16 fp32; do
for b in 512 4096 24576; do
for r in 0 1; do
ECHO_A6_ROWS=$r timeout 300 python scripts/kernel_bench.py --only attn_bwd --batch $b --reps 10 --dtype $dt > gpurun_out/r2_rows6_${dt}_${b}_${r}.txt 2>&1
done
done
done
