# a6 L2-prefetch modes at C2 / B=4096 (standalone + in-step via the quick bench) and the packed-z a5
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 900 python -m pytest -q -x tests/test_gpu_attention.py > gpurun_out/r2_a6pf_tests.txt 2>&1
for pf in 1 3 2 0; do
  for dt in fp32 bf16; do
    ECHO_A6_PREFETCH=$pf timeout 300 python scripts/kernel_bench.py --only attn --batch 128 --reps 20 --dtype $dt > gpurun_out/r2_a6pf_${pf}_c2_${dt}.txt 2>&1
  done
  ECHO_A6_PREFETCH=$pf timeout 300 python scripts/kernel_bench.py --only attn --batch 4096 --reps 10 --dtype bf16 > gpurun_out/r2_a6pf_${pf}_b4096_bf16.txt 2>&1
  ECHO_A6_PREFETCH=$pf timeout 600 python bench.py --steps 20 --warmup 5 --legs "" --no-cpu > gpurun_out/r2_a6pf_${pf}_bench.json 2>/dev/null
done
