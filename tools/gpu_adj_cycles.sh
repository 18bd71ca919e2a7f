cd $GRAFT_REPO_ROOT
PBE_LIB=variants/libpbe_timing.so timeout 300 python tools/adjoint_cycles.py 1000 > gpurun_out/adj_cycles.txt 2>&1
PBE_LIB=variants/libpbe_timing.so timeout 300 python tools/adjoint_cycles.py 8 >> gpurun_out/adj_cycles.txt 2>&1
timeout 300 python tools/next3_time.py > gpurun_out/next3_time.txt 2>&1
PBE_ADJ_K=8 timeout 300 python tools/prof_adj.py 1000 > gpurun_out/adj_k8.txt 2>&1
