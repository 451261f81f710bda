mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
for dt in bf16 fp32; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_tma -s 3 -c 1 \
     -o gpurun_out/r2_a5v3_b4096_$dt python scripts/kernel_bench.py --only attn_fwd --batch 4096 --reps 3 --dtype $dt > /dev/null 2>&1
done
