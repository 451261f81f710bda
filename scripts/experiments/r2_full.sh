mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/r2_full_gputest.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_full_smoke.txt 2>&1
