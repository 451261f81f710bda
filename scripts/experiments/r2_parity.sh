# round 2: bf16 parity report + the GPU suite after the boundary rename (no -x: see every failure)
mkdir -p gpurun_out
timeout 1500 python scripts/bf16_parity_report.py > gpurun_out/r2_bf16_report.jsonl 2> gpurun_out/r2_bf16_report.err
timeout 2400 python -m pytest tests -m gpu -q -s -rf > gpurun_out/r2_gputest2.txt 2>&1
