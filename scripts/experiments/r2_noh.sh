# a5 fp32 with H_s read from L2 (not staged in shared memory): parity + per-kernel timing; conv fx test
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 900 python -m pytest -q -x tests/test_gpu_attention.py > gpurun_out/r2_noh_tests.txt 2>&1
timeout 600 python -m pytest -q -x tests/test_gpu_fx_pass.py > gpurun_out/r2_noh_fx.txt 2>&1
for b in 128 4096 24576; do
timeout 300 python scripts/kernel_bench.py --only attn_fwd --batch $b --reps 10 --dtype fp32 > gpurun_out/r2_noh_${b}_fp32.txt 2>&1
done
timeout 300 python scripts/kernel_bench.py --only attn_fwd --batch 4096 --reps 10 --dtype bf16 > gpurun_out/r2_noh_4096_bf16.txt 2>&1
