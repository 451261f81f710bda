#!/bin/bash
# L2-residency experiment for the attention tensors (under gpurun)
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 300 python -m pytest tests/test_gpu_attention.py -x -q > gpurun_out/l2_pytest.txt 2>&1
ECHO_ATTN_L2LAST=1 timeout 300 python -m pytest tests/test_gpu_attention.py -x -q >> gpurun_out/l2_pytest.txt 2>&1
for l2 in 0 1; do
  ECHO_ATTN_L2LAST=$l2 timeout 300 python scripts/kernel_bench.py --only attn --noflush > gpurun_out/l2_k_noflush_$l2.txt 2>&1
  ECHO_ATTN_L2LAST=$l2 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --legs "" > gpurun_out/l2_bench_fp32_$l2.json 2> gpurun_out/l2_bench_fp32_$l2.err
  ECHO_ATTN_L2LAST=$l2 timeout 600 python bench.py --dtype bf16 --steps 10 --warmup 3 --no-cpu --legs "" > gpurun_out/l2_bench_bf16_$l2.json 2> gpurun_out/l2_bench_bf16_$l2.err
  ECHO_ATTN_L2LAST=$l2 timeout 300 python scripts/profile_step.py --dtype fp32 --graph > gpurun_out/l2_cupti_fp32_$l2.txt 2>&1
  ECHO_ATTN_L2LAST=$l2 timeout 300 python scripts/profile_step.py --dtype bf16 --graph > gpurun_out/l2_cupti_bf16_$l2.txt 2>&1
done
