#!/bin/bash
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
for c in 5 10 25; do
  ECHO_ENC_CHUNKS=$c timeout 600 python bench.py --dtype bf16 --steps 30 --warmup 5 --quick --no-cpu --legs "" > gpurun_out/ch2_bf16_$c.json 2>/dev/null
done
for c in 10 25 50; do
  ECHO_ENC_CHUNKS=$c timeout 600 python bench.py --steps 20 --warmup 5 --quick --no-cpu --legs "" > gpurun_out/ch2_fp32_$c.json 2>/dev/null
done
