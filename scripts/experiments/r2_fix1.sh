mkdir -p gpurun_out/sanitizer
python -m paper_1805_08899_b200.build > /dev/null
timeout 600 python -m pytest -q -x tests/test_gpu_attention.py > gpurun_out/r2_fix1_tests.txt 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
for cfg in c1 small; do for dt in fp32 bf16; do
timeout 1200 $CS --tool memcheck --error-exitcode 9 --print-limit 20 python scripts/sanitize_step.py --cfg $cfg --dtype $dt > gpurun_out/sanitizer/memcheck_${cfg}_${dt}.txt 2>&1
echo "memcheck $cfg $dt rc=$? $(grep 'ERROR SUMMARY' gpurun_out/sanitizer/memcheck_${cfg}_${dt}.txt)" >> gpurun_out/r2_fix1_san.txt
done; done
timeout 600 $CS --tool initcheck --print-limit 5 python scripts/micro/initcheck_tma_store.py > gpurun_out/sanitizer/initcheck_tma_store_micro.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_tma -s 3 -c 1 \
     -o gpurun_out/r2_a6_c2_fp32 python scripts/kernel_bench.py --only attn_bwd --batch 128 --reps 3 --dtype fp32 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_tma -s 3 -c 1 \
     -o gpurun_out/r2_a5_b4096_bf16_v2 python scripts/kernel_bench.py --only attn_fwd --batch 4096 --reps 3 --dtype bf16 > /dev/null 2>&1
