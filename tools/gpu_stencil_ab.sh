# A/B: tangent sweep in stencil form (default build) vs flux form (variants/libpbe_fluxform.so), C5 1184 sims
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/ab_stencil.txt
for r in 1 2; do
  echo "== stencil" >> gpurun_out/ab_stencil.txt
  timeout 300 python tools/ab_c5.py 1184 120 8 >> gpurun_out/ab_stencil.txt 2>&1
  echo "== fluxform" >> gpurun_out/ab_stencil.txt
  PBE_LIB=variants/libpbe_fluxform.so timeout 300 python tools/ab_c5.py 1184 120 8 >> gpurun_out/ab_stencil.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/stencil_tests.txt 2>&1
echo "rc $?" >> gpurun_out/stencil_tests.txt
