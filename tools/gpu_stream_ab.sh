cd $GRAFT_REPO_ROOT
timeout 600 python tools/ab_c4.py 1000000 64 200 'PBE_TEMPORAL_BLOCK=0|PBE_TEMPORAL_BLOCK=0,PBE_STREAM_STATIC=1' > gpurun_out/st_ab.txt 2>&1
timeout 600 python tools/ab_c4.py 4000000 1 200 'PBE_TEMPORAL_BLOCK=0|PBE_TEMPORAL_BLOCK=0,PBE_STREAM_STATIC=1' >> gpurun_out/st_ab.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -k "stream or outflow or lognormal or extra_limiters_dissolution" > gpurun_out/st_tests.txt 2>&1
echo "rc $?" >> gpurun_out/st_tests.txt
