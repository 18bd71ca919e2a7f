cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_adjoint.py tests/test_estimate.py tests/test_gpu_parity.py -q -x -k "adjoint or estimat or poly or long or determinism" > gpurun_out/ipow_tests.txt 2>&1
echo "rc $?" >> gpurun_out/ipow_tests.txt
timeout 300 python tools/adj_ab.py 1000 - PBE_ADJ_CLUSTER=0 > gpurun_out/ipow_ab.txt 2>&1
PBE_LIB=variants/libpbe_timing.so timeout 300 python tools/adjoint_cycles.py 1000 > gpurun_out/adj_cycles.txt 2>&1
