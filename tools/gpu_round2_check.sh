cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_clock.txt
timeout 120 python -c "
import numpy as np, oracle, workloads as W, paper_2411_00742_b200 as pb
w = W.c5_ensemble(n_sims=4, N=200, t_max=5.0, M=5)
g = pb.run_workload(w)
o = oracle.run(w, mode=oracle.MODE_DUAL, threads=4)
print('info', g['info'])
print('status', g['status'], o['status'], 'steps', g['steps'], o['steps'])
print('samples maxrel', np.nanmax(np.abs(g['samples']-o['samples'])/np.abs(o['samples'])))
print('tsamples maxabs', np.nanmax(np.abs(g['tsamples']-o['tsamples'])), np.nanmax(np.abs(o['tsamples'])))
print('n maxabs', np.max(np.abs(g['n_final']-o['n_final'])), np.max(o['n_final']))
print('loss', g['loss'], o['loss'])
print('grad', g['grad'][0], o['grad'][0])
" > gpurun_out/g1_smoke.txt 2>&1
echo "smoke rc $?" >> gpurun_out/g1_smoke.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/g1_par.txt 2>&1
echo "par rc $?" >> gpurun_out/g1_par.txt
timeout 600 python tools/ab_c5.py 4096 600 8 PBE_WS=0 > gpurun_out/g1_ab.txt 2>&1
echo "ab rc $?" >> gpurun_out/g1_ab.txt
