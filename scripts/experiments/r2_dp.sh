# round 2: the new multi-rank / seed-guard / bf16-gate tests, then a --gpus 2 bench line
mkdir -p gpurun_out
python -m paper_1805_08899_b200.build > /dev/null
timeout 1800 python -m pytest -q -s -rf tests/test_gpu_dp_parity.py tests/test_gpu_dp_bench.py "tests/test_gpu_nmt.py::test_graph_refuses_new_dropout_seeds" "tests/test_gpu_nmt.py::test_nmt_step_parity_and_bit_identity" "tests/test_gpu_nmt.py::test_nmt_mirror_plan_parity_and_graph" "tests/test_gpu_nmt.py::test_nmt_embedding_dropout_plans" tests/test_gpu_lstm.py tests/test_gpu_attention.py > gpurun_out/r2_dp_tests.txt 2>&1
timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --quick > gpurun_out/r2_bench_gpus2.json 2> gpurun_out/r2_bench_gpus2.err
timeout 600 python bench.py --steps 20 --warmup 5 --quick > gpurun_out/r2_bench_quick.json 2> gpurun_out/r2_bench_quick.err
