# A/B of the k_resident_ws tuning variants (PBE_WS_VARIANT) with the stencil tangent sweep, C5 1184 sims
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/ab_ws2.txt
for v in 0 1 2 3 4 5 6 0; do
  echo "== variant $v" >> gpurun_out/ab_ws2.txt
  PBE_WS_VARIANT=$v timeout 300 python tools/ab_c5.py 1184 120 8 >> gpurun_out/ab_ws2.txt 2>&1
done
