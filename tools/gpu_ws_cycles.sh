cd $GRAFT_REPO_ROOT
PBE_LIB=variants/libpbe_timing.so timeout 300 python tools/ws_cycles.py 148 30 8 > gpurun_out/g2_ws_cycles.txt 2>&1
PBE_LIB=variants/libpbe_timing.so timeout 300 python tools/ws_cycles.py 1184 30 8 >> gpurun_out/g2_ws_cycles.txt 2>&1
