cd $GRAFT_REPO_ROOT
timeout 300 python tools/dbg_tail.py > gpurun_out/dbg_tail.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -k "tail_wave or resident_kinds or determinism or c5" > gpurun_out/d_tests.txt 2>&1
echo "rc $?" >> gpurun_out/d_tests.txt
WS_VARIANTS="0" bash tools/gpu_ws_ab.sh
