cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_adjoint.py -q -x > gpurun_out/cl_tests.txt 2>&1
echo "rc $?" >> gpurun_out/cl_tests.txt
timeout 300 python tools/adj_ab.py 1000 - PBE_ADJ_CLUSTER=0 PBE_ADJ_CLUSTER=8 > gpurun_out/cl_ab.txt 2>&1
PBE_LIB=variants/libpbe_timing.so timeout 300 python tools/adjoint_cycles.py 1000 > gpurun_out/adj_cycles.txt 2>&1
