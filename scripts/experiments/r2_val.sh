# round-2 re-entry: full GPU suite + bench lines at HEAD (after the a5 rows kernel)
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/v_gpu.txt
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/v_pytest.txt 2>&1
echo "pytest exit $?" >> gpurun_out/v_pytest.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/v_bench_fp32.json 2> gpurun_out/v_bench_fp32.err
timeout 600 python bench.py --dtype bf16 --steps 20 --warmup 5 --no-cpu --legs "" > gpurun_out/v_bench_bf16.json 2> gpurun_out/v_bench_bf16.err
timeout 300 python scripts/kernel_bench.py --dtype fp32 > gpurun_out/v_kernels_c2_fp32.txt 2>&1
timeout 300 python scripts/kernel_bench.py --dtype bf16 > gpurun_out/v_kernels_c2_bf16.txt 2>&1
