# A/B of the k_resident_ws tuning variants (PBE_WS_VARIANT) and k_resident (PBE_WS=0) on C5
cd $GRAFT_REPO_ROOT
timeout 300 python tools/ws_smoke.py > gpurun_out/ws_smoke.txt 2>&1
PBE_WS_VARIANT=6 timeout 300 python tools/ws_smoke.py >> gpurun_out/ws_smoke.txt 2>&1
for v in ${WS_VARIANTS:-0 1 2 3 4 5 6}; do
  echo "== variant $v" >> gpurun_out/ab_ws.txt
  PBE_WS_VARIANT=$v timeout 300 python tools/ab_c5.py 1184 120 8 >> gpurun_out/ab_ws.txt 2>&1
done
echo "== k_resident" >> gpurun_out/ab_ws.txt
PBE_WS=0 timeout 300 python tools/ab_c5.py 1184 120 8 >> gpurun_out/ab_ws.txt 2>&1
