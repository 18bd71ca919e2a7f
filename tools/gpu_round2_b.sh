cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "resident_kinds or temporal_blocking_max" > gpurun_out/b_tests.txt 2>&1
echo "rc $?" >> gpurun_out/b_tests.txt
timeout 1200 python bench.py > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err
echo "bench rc $?" >> gpurun_out/b_bench.err
bash tools/gpu_ncu_c5.sh ws0 296 60
