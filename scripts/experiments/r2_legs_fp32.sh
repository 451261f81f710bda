# the secondary BASELINE workloads in fp32 storage (C3, C4, C2d, C5 at B=16384), one bench line
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 2400 python bench.py --steps 10 --warmup 3 --no-cpu --legs C3,C4,C2d,C5 --leg-dtype fp32 > gpurun_out/r02m_bench_legs_fp32.json 2> gpurun_out/r02m_bench_legs_fp32.err
timeout 900 python scripts/profile_step.py --dtype bf16 --graph --batch 24576 > gpurun_out/r02m_cupti_c5_bf16_recompute.txt 2>&1
