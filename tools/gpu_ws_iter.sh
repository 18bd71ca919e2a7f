# iteration check of k_resident_ws: smoke parity, phase cycles, C5 A/B vs k_resident
cd $GRAFT_REPO_ROOT
timeout 120 python -c "
import numpy as np, oracle, workloads as W, paper_2411_00742_b200 as pb
for N in (200, 2000):
    w = W.c5_ensemble(n_sims=4, N=N, t_max=5.0, M=5)
    g = pb.run_workload(w)
    o = oracle.run(w, mode=oracle.MODE_DUAL, threads=4)
    print(N, 'info', g['info'])
    print(' status', g['status'], o['status'], 'steps', g['steps'], o['steps'])
    print(' samples maxrel', np.nanmax(np.abs(g['samples']-o['samples'])/np.abs(o['samples'])))
    print(' tsamples rel', np.nanmax(np.abs(g['tsamples']-o['tsamples']))/np.nanmax(np.abs(o['tsamples'])))
    print(' n maxrel', np.max(np.abs(g['n_final']-o['n_final']))/np.max(o['n_final']))
    print(' loss', g['loss'], o['loss'])
    print(' grad rel', np.max(np.abs(g['grad']-o['grad']))/np.max(np.abs(o['grad'])))
" > gpurun_out/it_smoke.txt 2>&1
echo "smoke rc $?" >> gpurun_out/it_smoke.txt
PBE_LIB=variants/libpbe_timing.so timeout 300 python tools/ws_cycles.py 148 30 8 > gpurun_out/it_cycles.txt 2>&1
timeout 600 python tools/ab_c5.py 4096 600 8 PBE_WS=0 > gpurun_out/it_ab.txt 2>&1
