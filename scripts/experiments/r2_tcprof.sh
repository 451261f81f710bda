mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lstm_fwd_tc -s 5 -c 1 \
   -o gpurun_out/r2_tc_step python scripts/lstm_tc_bench.py --T 4 --reps 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"lstm_fwd_kernel|nvjet" -s 10 -c 2 \
   -o gpurun_out/r2_perstep python scripts/lstm_tc_bench.py --T 4 --reps 2 > /dev/null 2>&1
