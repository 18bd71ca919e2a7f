cd $GRAFT_REPO_ROOT
timeout 600 python tools/cases_time.py > gpurun_out/cases_time.txt 2>&1
PBE_WS=0 timeout 300 python tools/ab_c5.py 1184 120 8 > gpurun_out/ab_lockstep.txt 2>&1
timeout 300 python tools/ab_c5.py 1184 120 8 >> gpurun_out/ab_lockstep.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q > gpurun_out/res_tests.txt 2>&1
echo "rc $?" >> gpurun_out/res_tests.txt
