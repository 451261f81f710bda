# a5 rows kernel v2 (explicit shared addressing, position pairs): parity + timing
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 1200 python -m pytest -q -x tests/test_gpu_attention.py -k "a5_rows or parity_and_bit" > gpurun_out/r2_rows5_tests.txt 2>&1
for dt in bf16 fp32; do
for b in 512 4096 24576; do
ECHO_A5_ROWS=1 timeout 300 python scripts/kernel_bench.py --only attn_fwd --batch $b --reps 10 --dtype $dt > gpurun_out/r2_rows5_${dt}_${b}.txt 2>&1
done
done
ECHO_A5_ROWS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_rows -s 3 -c 1 \
     -o gpurun_out/r2_rows5_b4096_bf16 python scripts/kernel_bench.py --only attn_fwd --batch 4096 --reps 3 --dtype bf16 > /dev/null 2>&1
