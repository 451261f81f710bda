# reduced closing check (when little time is left): the full GPU suite and one fp32 bench line
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2f_pytest.txt 2>&1
echo "pytest exit $?" >> gpurun_out/r2f_pytest.txt
timeout 900 python bench.py --steps 20 --warmup 5 --legs "" --no-cpu > gpurun_out/r2f_bench_fp32.json 2> gpurun_out/r2f_bench_fp32.err
