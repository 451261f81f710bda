#!/bin/bash
# quick a6/a5 check (under gpurun): attention parity tests, C2 kernel timings, phase timing
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_nmt.py -x -q > gpurun_out/q_pytest.txt 2>&1
for dt in fp32 bf16; do
  timeout 300 python scripts/kernel_bench.py --only attn --dtype $dt > gpurun_out/q_k_${dt}.txt 2>&1
done
timeout 300 python scripts/kernel_bench.py --only attn --batch 4096 --reps 10 > gpurun_out/q_k4096_fp32.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --legs "" > gpurun_out/q_bench_fp32.json 2> gpurun_out/q_bench_fp32.err
timeout 600 python bench.py --dtype bf16 --steps 10 --warmup 3 --no-cpu --legs "" > gpurun_out/q_bench_bf16.json 2> gpurun_out/q_bench_bf16.err
cp paper_1805_08899_b200/libecho.so /tmp/libecho_keep.so
ECHO_NVCC_EXTRA=-DECHO_PHASE_TIMING python -m paper_1805_08899_b200.build --force > /dev/null
timeout 120 python scripts/phase_timing.py 128 > gpurun_out/q_phase.txt 2>&1
cp /tmp/libecho_keep.so paper_1805_08899_b200/libecho.so
