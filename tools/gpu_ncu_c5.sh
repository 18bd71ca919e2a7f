# one ncu --set full capture of the resident kernel on a small C5-shaped run (default 296 sims,
# 60 min); the report stays on the box (/tmp), its raw/source/details pages come back as CSV
cd $GRAFT_REPO_ROOT
TAG=${1:-ws}
SIMS=${2:-296}
TMAX=${3:-60}
timeout 300 python tools/prof_c5.py $SIMS $TMAX > gpurun_out/ncu_${TAG}_plain.txt 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_resident -c 1 \
    -o /tmp/c5_${TAG} python tools/prof_c5.py $SIMS $TMAX > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu rc $?" >> gpurun_out/ncu_${TAG}.log
ncu -i /tmp/c5_${TAG}.ncu-rep --page raw --csv > gpurun_out/ncu_${TAG}_raw.csv 2>/dev/null
ncu -i /tmp/c5_${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_${TAG}_sass.csv 2>/dev/null
ncu -i /tmp/c5_${TAG}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_${TAG}_src.csv 2>/dev/null
ncu -i /tmp/c5_${TAG}.ncu-rep --page details --csv > gpurun_out/ncu_${TAG}_details.csv 2>/dev/null
ls -la /tmp/c5_${TAG}.ncu-rep >> gpurun_out/ncu_${TAG}.log
