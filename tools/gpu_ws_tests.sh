cd $GRAFT_REPO_ROOT
timeout 300 python tools/ws_smoke.py > gpurun_out/ws_smoke.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -k "resident_kinds or temporal_blocking or c5 or tangent or lognormal or extra_limiters or determinism or status" > gpurun_out/ws_tests2.txt 2>&1
echo "rc $?" >> gpurun_out/ws_tests2.txt
