# round 2: fresh ncu captures of a5 (B=4096 fp32 / bf16), a2 bf16 (B=4096), colsum at a C5-like shape
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
for dt in fp32 bf16; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_tma -s 3 -c 1 \
     -o gpurun_out/r2_a5_b4096_$dt python scripts/kernel_bench.py --only attn_fwd --batch 4096 --reps 3 --dtype $dt > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lstm_cscan -s 3 -c 1 \
   -o gpurun_out/r2_a2_b4096_bf16 python scripts/kernel_bench.py --only lstm_cscan --batch 4096 --reps 3 --dtype bf16 > /dev/null 2>&1
timeout 600 python scripts/colsum_bench.py > gpurun_out/r2_colsum.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:colsum -s 2 -c 1 \
   -o gpurun_out/r2_colsum python scripts/colsum_bench.py --reps 1 --only fp32 > /dev/null 2>&1
ls -la gpurun_out
