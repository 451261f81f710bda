mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_fp32.json 2> gpurun_out/r2_bench_fp32.err
timeout 300 python scripts/kernel_bench.py --batch 4096 --reps 10 > gpurun_out/r2_kernels_fp32_b4096.txt 2>&1
timeout 300 python scripts/kernel_bench.py --batch 4096 --reps 10 --dtype bf16 > gpurun_out/r2_kernels_bf16_b4096.txt 2>&1
