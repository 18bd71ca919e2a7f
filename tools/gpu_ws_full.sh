cd $GRAFT_REPO_ROOT
timeout 300 python tools/ws_smoke.py > gpurun_out/ws_smoke.txt 2>&1
WS_VARIANTS="0 6" bash tools/gpu_ws_ab.sh
timeout 1800 python -m pytest tests/ -m gpu -x -q > gpurun_out/ws_gputests.txt 2>&1
echo "rc $?" >> gpurun_out/ws_gputests.txt
