#!/bin/bash
# a6 experiments (run under gpurun): L2 prefetch modes of the dKp / dH_s tiles, standalone and in-step,
# plus per-phase cycle timing.  Output in gpurun_out/a6v_*.
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
for pf in 0 1 2; do
  for dt in fp32 bf16; do
    ECHO_A6_PREFETCH=$pf timeout 300 python scripts/kernel_bench.py --only attn_bwd --dtype $dt > gpurun_out/a6v_k_${dt}_pf$pf.txt 2>&1
    ECHO_A6_PREFETCH=$pf timeout 300 python scripts/kernel_bench.py --only attn_bwd --dtype $dt --batch 4096 --reps 10 > gpurun_out/a6v_k4096_${dt}_pf$pf.txt 2>&1
  done
done
for pf in 1 2; do
  ECHO_A6_PREFETCH=$pf timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --legs "" > gpurun_out/a6v_bench_fp32_pf$pf.json 2> gpurun_out/a6v_bench_fp32_pf$pf.err
  ECHO_A6_PREFETCH=$pf timeout 600 python bench.py --dtype bf16 --steps 10 --warmup 3 --no-cpu --legs "" > gpurun_out/a6v_bench_bf16_pf$pf.json 2> gpurun_out/a6v_bench_bf16_pf$pf.err
done
cp paper_1805_08899_b200/libecho.so /tmp/libecho_keep.so
ECHO_NVCC_EXTRA=-DECHO_PHASE_TIMING python -m paper_1805_08899_b200.build --force > /dev/null
for pf in 0 1 2; do
  ECHO_A6_PREFETCH=$pf timeout 120 python scripts/phase_timing.py 128 > gpurun_out/a6v_phase_pf$pf.txt 2>&1
done
cp /tmp/libecho_keep.so paper_1805_08899_b200/libecho.so
