#!/bin/bash
# After `gpurun -- bash scripts/round_measure_r02b.sh`: copy the closing bundle into profiles/ (bench
# lines, pytest summary, kernel benches) and summarise the ncu reports with scripts/ncu_summary.py.
set -u
cd "$(dirname "$0")/.."
out=gpurun_out
for f in bench_fp32.json bench_bf16.json kernels_c2_fp32.txt kernels_c2_bf16.txt gpu.txt; do
  [ -s "$out/r02b_$f" ] && cp "$out/r02b_$f" "profiles/r02b_$f"
done
[ -s "$out/r02b_pytest.txt" ] && tail -5 "$out/r02b_pytest.txt" > profiles/r02b_pytest_tail.txt
cat $out/r02b_a5_*.txt > profiles/r02b_a5_rows_kernel_bench.txt 2>/dev/null
for r in $out/r02b_a5rows_*.ncu-rep $out/r02b_a6_c2_fp32.ncu-rep; do
  [ -f "$r" ] || continue
  b=$(basename "$r" .ncu-rep)
  python scripts/ncu_summary.py "$r" > "profiles/${b}_ncu.txt" 2>&1
done
[ -s "$out/r02b_launches_fp32.csv" ] && python scripts/summarize_launches.py "$out/r02b_launches_fp32.csv" profiles/r02b_launches_c2_fp32_recompute.csv "C2 fp32 recompute, round 2 closing bundle"
ls -la profiles | grep r02b
