# ncu --set full of the adjoint kernel on the NEXT-3 workload; summaries come back as text/CSV
cd $GRAFT_REPO_ROOT
P=${1:-1000}
timeout 300 python tools/prof_adj.py $P > gpurun_out/ncu_adj_plain.txt 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_adjoint -c 1 \
    -o /tmp/adj python tools/prof_adj.py $P > gpurun_out/ncu_adj.log 2>&1
echo "ncu rc $?" >> gpurun_out/ncu_adj.log
ncu -i /tmp/adj.ncu-rep --page raw --csv > gpurun_out/ncu_adj_raw.csv 2>/dev/null
ncu -i /tmp/adj.ncu-rep --page details --csv > gpurun_out/ncu_adj_details.csv 2>/dev/null
python tools/ncu_lines.py /tmp/adj.ncu-rep 60 > gpurun_out/ncu_adj_lines.txt 2>&1
