cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -k "tail_wave or resident_kinds or determinism or c5 or two_rank" > gpurun_out/c_tests.txt 2>&1
echo "rc $?" >> gpurun_out/c_tests.txt
timeout 1200 python bench.py --no-e2e > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err
echo "bench rc $?" >> gpurun_out/c_bench.err
