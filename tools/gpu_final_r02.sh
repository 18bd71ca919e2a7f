# round-2 final: default bench, then its launch list under ncu (gpu__time_duration only)
cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
echo "rc $?" >> gpurun_out/final_bench.err
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/final_bench_s3.json 2>> gpurun_out/final_bench.err
echo "rc $?" >> gpurun_out/final_bench.err
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/final_launches.csv python bench.py --steps 3 --warmup 3 > gpurun_out/final_ncu.log 2>&1
echo "ncu rc $?" >> gpurun_out/final_ncu.log
