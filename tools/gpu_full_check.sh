# full validation: GPU parity suite, smoke, default bench, launch list of the bench command
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests/ -m gpu -q > gpurun_out/full_tests.txt 2>&1
echo "rc $?" >> gpurun_out/full_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.txt 2>&1
echo "rc $?" >> gpurun_out/full_smoke.txt
timeout 1500 python bench.py > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err
echo "rc $?" >> gpurun_out/full_bench.err
