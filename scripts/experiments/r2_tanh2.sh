mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tanh_err scripts/micro/tanh_err.cu && /tmp/tanh_err > gpurun_out/r2_tanh_err.txt 2>&1
timeout 1200 python -m pytest -q -x tests/test_gpu_attention.py tests/test_gpu_nmt.py -k "bf16 or attention" > gpurun_out/r2_tanh2_tests.txt 2>&1
for b in 4096 128; do
timeout 300 python scripts/kernel_bench.py --only attn --batch $b --reps 10 --dtype bf16 > gpurun_out/r2_tanh2_k${b}.txt 2>&1
done
timeout 900 python bench.py --dtype bf16 --steps 20 --warmup 5 --no-cpu --legs "" > gpurun_out/r2_tanh2_bench.json 2>/dev/null
