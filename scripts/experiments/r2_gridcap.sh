mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
for cap in 2368 4736 9472 100000; do
  ECHO_LSTM_GRIDCAP=$cap timeout 300 python scripts/kernel_bench.py --only lstm --batch 24576 --reps 10 --dtype bf16 > gpurun_out/r2_gridcap_${cap}_bf16.txt 2>&1
  ECHO_LSTM_GRIDCAP=$cap timeout 300 python scripts/kernel_bench.py --only lstm --batch 16384 --reps 10 --dtype fp32 > gpurun_out/r2_gridcap_${cap}_fp32.txt 2>&1
done
