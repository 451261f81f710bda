mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
ECHO_A5_ROWS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_rows -s 3 -c 1 \
     -o gpurun_out/r2_rows_b4096_bf16 python scripts/kernel_bench.py --only attn_fwd --batch 4096 --reps 3 --dtype bf16 > /dev/null 2>&1
