# A/B of plain-stream pipeline shapes (build variants) on C4 64 x 1e6, 200 steps
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/st_cfg.txt
for r in 1 2; do
for v in default m1s6 m1s4 m2s2; do
  lib=paper_2411_00742_b200/libpbe.so; [ $v != default ] && lib=variants/libpbe_$v.so
  echo "== $v" >> gpurun_out/st_cfg.txt
  PBE_LIB=$lib timeout 600 python tools/ab_c4.py 1000000 64 200 'PBE_TEMPORAL_BLOCK=0' >> gpurun_out/st_cfg.txt 2>&1
done
done
