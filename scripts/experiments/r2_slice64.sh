# a6 / a5 at C2 (B = 128) with 64-column slices (C = 8) vs 128 (C = 4): parity + timing + in-step probe
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
ECHO_ATTN_SLICE=64 timeout 900 python -m pytest -q -x tests/test_gpu_attention.py -k "parity_and_bit or a5_rows" > gpurun_out/r2_s64_tests.txt 2>&1
for sl in 128 64; do
for dt in fp32 bf16; do
ECHO_ATTN_SLICE=$sl timeout 300 python scripts/kernel_bench.py --only attn --batch 128 --reps 20 --dtype $dt > gpurun_out/r2_s64_${sl}_${dt}.txt 2>&1
ECHO_ATTN_SLICE=$sl timeout 300 python scripts/kernel_bench.py --only attn --batch 128 --reps 20 --dtype $dt --noflush > gpurun_out/r2_s64_${sl}_${dt}_nf.txt 2>&1
done
done
