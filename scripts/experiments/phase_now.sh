#!/bin/bash
mkdir -p gpurun_out
cp paper_1805_08899_b200/libecho.so /tmp/libecho_keep.so 2>/dev/null
ECHO_NVCC_EXTRA=-DECHO_PHASE_TIMING python -m paper_1805_08899_b200.build --force > /dev/null
timeout 120 python scripts/phase_timing.py 128 > gpurun_out/pn_phase_128.txt 2>&1
timeout 120 python scripts/phase_timing.py 1024 > gpurun_out/pn_phase_1024.txt 2>&1
cp /tmp/libecho_keep.so paper_1805_08899_b200/libecho.so 2>/dev/null || python -m paper_1805_08899_b200.build --force > /dev/null
