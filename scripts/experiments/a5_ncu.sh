#!/bin/bash
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_tma -s 3 -c 1 -o gpurun_out/a5_b4096_bf16 python scripts/kernel_bench.py --only attn_fwd --batch 4096 --reps 3 --dtype bf16 > /dev/null 2>&1
ls -la gpurun_out/a5_b4096_bf16.ncu-rep
