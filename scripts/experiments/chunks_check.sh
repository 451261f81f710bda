#!/bin/bash
# encoder wavefront chunk count (ECHO_ENC_CHUNKS) after the LSTM vector-width change
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
for c in 1 2 5; do
  for r in 1 2; do
    ECHO_ENC_CHUNKS=$c timeout 600 python bench.py --dtype bf16 --steps 30 --warmup 5 --quick --no-cpu --legs "" > gpurun_out/ch_bf16_${c}_$r.json 2>/dev/null
  done
done
for c in 1 5 10; do
  ECHO_ENC_CHUNKS=$c timeout 600 python bench.py --steps 20 --warmup 5 --quick --no-cpu --legs "" > gpurun_out/ch_fp32_$c.json 2>/dev/null
done
