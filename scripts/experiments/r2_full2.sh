mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/r2_full2_gputest.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_full2_smoke.txt 2>&1
timeout 1500 python bench.py > gpurun_out/r2_full2_bench.json 2> gpurun_out/r2_full2_bench.err
timeout 900 python bench.py --dtype bf16 --no-cpu --legs "" > gpurun_out/r2_full2_bench_bf16.json 2> gpurun_out/r2_full2_bench_bf16.err
for dt in fp32 bf16; do
  timeout 300 python scripts/kernel_bench.py --batch 4096 --reps 10 --dtype $dt > gpurun_out/r2_full2_kernels_b4096_${dt}.txt 2>&1
  timeout 300 python scripts/kernel_bench.py --dtype $dt > gpurun_out/r2_full2_kernels_c2_${dt}.txt 2>&1
done
