cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_adjoint.py tests/test_estimate.py -q > gpurun_out/adj_tests.txt 2>&1
echo "rc $?" >> gpurun_out/adj_tests.txt
bash tools/gpu_adj_cycles.sh
