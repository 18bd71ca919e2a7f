#!/usr/bin/env python
"""Benchmark of the batched PBE finite-volume march (BASELINE.json metric: bin-updates/s).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5|c4|c3|c2|c1|c2d]
                  [--scaling strong|weak] [--impl ours|reference] [--quick]

A bench "step" is one pass of the whole hot path (rows a1-a8: the complete time-march of
every simulation of this rank's batch, one pbe_run_batch) over one batch of synthetic
input.  Default workload = BASELINE config 5 as written (the one the metric is quoted on at
1/2/4/8 GPUs): 4096 kinetic parameter sets in total, sharded round-robin over the GPUs
(strong scaling; --scaling weak keeps 4096 per GPU), 2000 bins, 8 forward-mode tangent
lanes, 600 samples.

One JSON line on rank 0 (see DESIGN.md "Measurement" for every field's definition):
  value      bin-updates/s over all ranks, inputs resident in HBM, CUDA events on the
             launch stream, L2 flushed (512 MiB write) between timed iterations
  e2e        the same metric through the C ABI with pinned HOST buffers: the H2D copy of
             each step's inputs and the D2H read of its records (moments, status, steps,
             loss, gradient) inside the timed region
  roofline   the dominant kernel (k_resident_ws: the only kernel of the step): FP64 instructions
             of the method per bin-update x rate against the DFMA throughput measured in the
             same run (bound "alu"), or HBM for the streaming workloads (bound "hbm")
  cpu_baseline   the CPU oracle timed on a bounded sample on this host's cores
  --impl reference   the CPU oracle as the reference arm (the paper ships no code)
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "bin-updates/sec (bins x steps x sims)"
UNIT = "bin-updates/s"


# ----------------------------------------------------------------------------------------
# workloads
# ----------------------------------------------------------------------------------------
def make_workload(name: str, world: int, args):
    """The GLOBAL workload (all ranks) and a short description for config."""
    if name == "c5":
        strong = args.scaling == "strong"
        S = 4096 if strong else 4096 * world
        w = W.c5_ensemble(n_sims=S)
        desc = dict(workload="C5 ensemble + forward-mode tangents", global_sims=S,
                    sims_per_gpu=S // world if strong else 4096, bins=2000, tangent_lanes=8, samples=600,
                    t_max_min=600.0, dt_max=0.05, law="polynomial k=8", limiter="van Leer",
                    target="App. B method-of-moments traces (workloads/data/appb_targets.npy)")
    elif name == "c4":
        N = args.bins or 1_000_000
        b = args.batch or 64
        w = W.c4_sweep(N, batch=b * world, n_steps=args.march_steps or 1000)
        desc = dict(workload=f"C4 bin sweep N={N} batch {b}/GPU", sims_per_gpu=b, bins=N,
                    march_steps=w.n_steps, limiter="van Leer", cfl="uncapped (C = 0.9)")
    elif name == "c2d":
        N1 = args.bins or 6000
        N2 = args.bins2 or N1 // 2
        b = args.batch or 1
        w = W.c2d_base(N1, N2, n_sims=b * world)
        w.n_steps = args.march_steps or 200
        w.t_samples = np.array([1.0])
        desc = dict(workload=f"NEXT-1 2D base case {N1}x{N2} (Table 1 grid x {1200 // N1 if N1 <= 1200 else 'fine'}), "
                    f"Godunov splitting, {w.n_steps} uncapped CFL steps, {b} sim(s)/GPU", bins=N1 * N2,
                    sims_per_gpu=b, march_steps=w.n_steps, limiter="van Leer")
    elif name == "c3":
        w = W.c3_cycling()
        desc = dict(workload="C3 temperature cycling (single sim; replicas only)", bins=1000, march_steps=100000)
    elif name == "c2":
        w = W.c2_dissolution()
        desc = dict(workload="C2 dissolution (single sim; replicas only)", bins=1000, march_steps=6000)
    elif name == "c1":
        w = W.c1_growth(W.LIM_VANLEER, M=1000)
        desc = dict(workload="C1 growth, constant G (single sim; replicas only)", bins=100, march_steps=1000)
    else:
        raise SystemExit(f"unknown workload {name}")
    return w, desc


def replicate_single(w, world: int):
    """Single-simulation configs run as independent replicas (one per rank)."""
    return w.subset(np.zeros(world, dtype=np.int64)) if w.n_sims == 1 else w


# FP64 INSTRUCTIONS per bin-update of the method in the flux form the kernels implement
# (DESIGN.md §5 "Roofline"; each DFMA / DMUL / DADD is one instruction on the FP64 pipe, the
# reciprocal's MUFU seed runs on the XU pipe):
#   van Leer primal 15: a, b (2), ab (1), a + b (1), Newton reciprocal (4), h = ab r (1),
#       F = C n_up + kappa psi (2), update (2), mu3 (1), clip test (1)
#   tangent support per face 10: b r, a r (2), qa, qb (2), kappa qa, kappa qb (2),
#       g = n_up + beta psi (1), dg (1), w_mid (2)
#   per tangent lane 7: lane flux (3), update (2), Cdot dg (1), mu3dot (1)   [k_resident: flux form]
#   k_resident_ws (stencil form of the same update): per bin 3 (two coefficient sums), per lane 6:
#       stencil (1 DMUL + 3 DFMA), Cdot dg (1), mu3dot (1)
#   upwind: primal 6 (F 1, update 2, mu3 1, clip 1, n_up 1), lane 5 (flux 1, update 2, Cdot 1, mu3dot 1)
# SURVEY §8(d) estimated ~19 + 10 per lane before the kernels existed; the counts above are
# the implemented formulation's (its SASS executes 91.5 for C5: profiles/fp64_instr.json).
def fp64_instr_per_bin_update(limiter: int, P: int, stencil: bool = False) -> float:
    if limiter == W.LIM_UPWIND:
        return 6.0 + (1.0 if P else 0.0) + 5.0 * P
    if stencil and P:
        return 15.0 + 10.0 + 3.0 + 6.0 * P
    return 15.0 + (10.0 if P else 0.0) + 7.0 * P


# ----------------------------------------------------------------------------------------
# clocks sampling (nvidia-smi during the timed region)
# ----------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        rows = [r for r in self.rows if len(r) >= 8]
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return dict(sm_mhz=float(np.median(sm)) if sm else None, sm_max_mhz=max(mx) if mx else None,
                    reasons=reasons, samples=len(rows))


# ----------------------------------------------------------------------------------------
# CPU oracle legs
# ----------------------------------------------------------------------------------------
def oracle_sample(w, threads: int, seed_offset: int = 0):
    """A bounded sample of the workload: `threads` simulations (one per host thread),
    spread over the batch, full size.  Returns (bin_updates, seconds, description)."""
    import oracle
    S = w.n_sims
    k = min(threads, S)
    sims = (np.arange(k) * max(S // k, 1) + seed_offset) % S
    ws = w.subset(sims)
    mode = oracle.MODE_DUAL if w.n_tangents else oracle.MODE_DOUBLE
    t0 = time.perf_counter()
    r = oracle.run(ws, mode=mode, threads=threads, want_n=False)
    dt = time.perf_counter() - t0
    bu = float(w.N) * float(np.sum(r["steps"]))
    desc = f"{k} of {S} sims (full size: {w.N} bins, {w.n_tangents} tangent lanes), one per host thread"
    return bu, dt, desc


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ----------------------------------------------------------------------------------------
def run_reference(args, rank, world):
    """--impl reference: the CPU oracle as it stands, on this host's cores (rank 0 only)."""
    if rank != 0:
        return 0
    w, desc = make_workload(args.workload, 1, args)
    w = replicate_single(w, 1)
    th = host_threads()
    for i in range(args.warmup):
        oracle_sample(w, th, seed_offset=i)
    tot_bu, tot_s, sdesc = 0.0, 0.0, ""
    for i in range(args.steps):
        bu, s, sdesc = oracle_sample(w, th, seed_offset=args.warmup + i)
        tot_bu += bu; tot_s += s
    value = tot_bu / tot_s
    line = dict(metric=METRIC, value=value, unit=UNIT, n_gpus=world, steps=args.steps, warmup=args.warmup,
                ms_per_step=1e3 * tot_s / args.steps, higher_is_better=True,
                scaling=args.scaling if args.workload == "c5" else "weak", vs_baseline=None,
                dtype="f64", data="synthetic", impl="reference", config=desc,
                cpu_baseline=dict(value=value, unit=UNIT, cores=th, kind="oracle", sample=sdesc),
                e2e=dict(value=value, unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0),
                gpu_launches=0)
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c5", choices=["c1", "c2", "c3", "c4", "c5", "c2d"])
    ap.add_argument("--bins2", type=int, default=0, help="2D: bins along L2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--bins", type=int, default=0, help="C4: bins per simulation")
    ap.add_argument("--batch", type=int, default=0, help="C4: simulations per GPU")
    ap.add_argument("--march-steps", type=int, default=0, help="C4: time steps per simulation")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the C4 streaming entry")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="C5: 4096 simulations in total (strong) or per GPU (weak)")
    ap.add_argument("--quick", action="store_true", help="skip the per-config, sweep and 2D entries")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: WORLD_SIZE={world} != --gpus {args.gpus}", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import paper_2411_00742_b200 as pb
    from paper_2411_00742_b200 import dist as D

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    wg, desc = make_workload(args.workload, world, args)
    wg = replicate_single(wg, world)
    mine = D.shard(wg.n_sims, rank, world)
    w = wg.subset(mine)
    P = w.n_tangents
    ctx = pb.context_for(w, device=local_rank)
    n0_dev = torch.from_numpy(np.ascontiguousarray(w.n0)).to(dev)
    ts = w.t_samples if w.n_steps == 0 else None
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # 512 MiB > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def measure(ctx, w, n0_dev, ts, gather, clocks=None):
        """W warm-up + K timed steps (CUDA events per step on the launch stream, L2 flushed
        in between).  Returns (ms per step, max over ranks; this rank's bin-updates per
        step; mean main-kernel ms measured by libpbe's events on the same stream)."""
        P = w.n_tangents

        def step():
            ctx.run_batch(n0_dev, w.c0, ts, w.target, stream=stream)
            if gather and world > 1:
                out = ctx.moments(on_device=True)
                grad = (ctx.tangents(on_device=True, out=dict(grad=torch.empty((w.n_sims, P), dtype=torch.float64,
                                                                               device=dev)))["grad"] if P else None)
                rec = D.pack_records(out["status"], out["steps"], out["moments"], out["loss"], grad)
                D.allgather_records(rec, wg.n_sims)

        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize(dev)
        res = ctx.moments()
        assert np.all(res["status"] == 0), f"simulation failures: {np.unique(res['status'])}"
        bu = float(w.N) * max(getattr(w, "N2", 0), 1) * float(np.sum(res["steps"]))
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        barrier()
        torch.cuda.synchronize(dev)
        if clocks:
            clocks.start()
        kms = []
        for k in range(args.steps):
            flush.fill_(float(k))                              # evict L2 between timed iterations
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
            if world == 1:
                torch.cuda.synchronize(dev)
                kms.append(ctx.last_run_info()["main_ms"])
        torch.cuda.synchronize(dev)
        barrier()
        ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
        if not kms:
            ctx.moments()
            kms = [ctx.last_run_info()["main_ms"]]
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t[0])
        return ms, bu, float(np.mean(kms))

    def roofline(w, info, bu_local, kms, workload):
        P = w.n_tangents
        if info["kernel"] in (pb.KERNEL_STREAM, pb.KERNEL_2D):
            # 2D: the fused kernel reads + writes each cell once per split step (16 B); the unfused
            # one (PBE_2D_UNFUSED=1) does that once per sweep (32 B)
            unfused = info["kernel"] == pb.KERNEL_2D and os.environ.get("PBE_2D_UNFUSED", "0") not in ("", "0")
            spp = max(1, int(info.get("steps_per_pass", 1)))       # temporal blocking: 16 B per spp steps
            bytes_per = 16.0 * (1 + P) * (2.0 if unfused else 1.0) / spp
            achieved = bytes_per * bu_local / (kms * 1e-3) / 1e9
            hbm = float(peaks.get("hbm_gbs", 6650.0))
            kname = ("k_2d" if unfused else "k_2d_fused") if info["kernel"] == pb.KERNEL_2D else "k_stream"
            if spp > 1:
                kname = "k_stream_tb"
            r = dict(bound="hbm", achieved=achieved, peak=hbm, unit="GB/s", frac=achieved / hbm, traffic=None,
                     kernel=kname, bytes_per_bin_update=bytes_per,
                     peak_source="MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6.65 TB/s", kernel_ms=kms)
        else:
            f = fp64_instr_per_bin_update(w.limiter, P, stencil=bool(info.get("warp_specialized")))
            achieved = f * bu_local / (kms * 1e-3) / 1e12
            sm_max = float(peaks.get("sm_max_mhz", 1965.0))
            nominal = 148 * 64 * sm_max * 1e6 / 1e12      # FP64 lanes x SMs x max SM clock (instr/s)
            peak, src = nominal, f"derived: 148 SMs x 64 FP64 lanes/clk x {sm_max:.0f} MHz (no DFMA measurement)"
            if dfma_tflops and dfma_tflops > 0:
                peak, src = dfma_tflops / 2.0, "DFMA microbenchmark in this run (libpbe_mb.so), FMA = 1 instruction"
            kname = "k_cluster" if info["kernel"] == pb.KERNEL_CLUSTER else (
                "k_resident_ws" if info.get("warp_specialized") else "k_resident")
            r = dict(bound="alu", achieved=achieved, peak=peak, unit="FP64 Tinst/s", frac=achieved / peak, traffic=None,
                     kernel=kname, fp64_instr_per_bin_update=f, peak_source=src, peak_nominal=nominal, kernel_ms=kms)
            fi = os.path.join(ROOT, "profiles", "fp64_instr.json")
            if os.path.exists(fi):
                try:
                    e = json.load(open(fi)).get(kname)
                    if e:
                        r["sass_fp64_instr_per_bin_update"] = e["sass_fp64_instr_per_bin_update"]
                        r["frac_sass"] = e["sass_fp64_instr_per_bin_update"] * bu_local / (kms * 1e-3) / 1e12 / peak
                        r["ncu_fp64_pipe_active"] = e.get("ncu_fp64_pipe_active")
                        r["sass_source"] = e["source"]
                except Exception:
                    pass
        if r.get("kernel") == "k_stream_tb":
            # temporal blocking moves 16 B per bin per HBM pass of spp steps, so HBM is not its bound;
            # report where it stands against the plain-streaming ceiling as well
            r["note"] = "temporal blocking: traffic 16 B / steps_per_pass; latency/FP64-bound, not HBM-bound"
            r["frac_of_plain_stream_ceiling"] = bu_local / (kms * 1e-3) / (r["peak"] * 1e9 / 16.0)
        # DRAM bytes of the kernel from an ncu --set full capture (profiles/traffic.json), as
        # bytes per bin-update, scaled to this launch
        prof = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(prof):
            try:
                tr = json.load(open(prof)).get(r["kernel"])
                if tr is not None:
                    r["traffic"] = tr["dram_bytes_per_bin_update"] * bu_local
                    r["traffic_source"] = tr["source"]
            except Exception:
                pass
        return r

    # ---- FP64 roofline denominator, measured on this GPU first ---------------------------------------
    dfma_tflops = None
    try:
        import ctypes as C
        mbl = C.CDLL(os.path.join(ROOT, "paper_2411_00742_b200", "libpbe_mb.so"))
        mbl.pbe_mb_dfma_tflops.restype = C.c_double
        dfma_tflops = float(mbl.pbe_mb_dfma_tflops(local_rank, 5))
    except Exception:
        pass

    # ---- main measurement ----------------------------------------------------------------------------
    clocks = ClockSampler(local_rank)
    ms, bu_local, kms = measure(ctx, w, n0_dev, ts, gather=True, clocks=clocks)
    clk = clocks.stop()
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([bu_local], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        bu_total = float(t[0])
    else:
        bu_total = bu_local
    info = ctx.last_run_info()
    value = bu_total / (ms * 1e-3)
    roof = roofline(w, info, bu_local, kms, args.workload)
    roof["dfma_microbench_tflops"] = dfma_tflops

    # ---- e2e through the C ABI with pinned host buffers ------------------------------------------
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        n0_h, c0_h = pin(w.n0), pin(w.c0)
        ts_h = pin(ts) if ts is not None else None
        tg_h = pin(w.target) if w.target is not None else None
        S, M = w.n_sims, w.M
        outh = dict(moments=torch.empty((S, M, 6), dtype=torch.float64).pin_memory().numpy(),
                    status=torch.empty(S, dtype=torch.int32).pin_memory().numpy(),
                    steps=torch.empty(S, dtype=torch.int64).pin_memory().numpy(),
                    loss=torch.empty(S, dtype=torch.float64).pin_memory().numpy())
        grad_h = torch.empty((S, max(P, 1)), dtype=torch.float64).pin_memory().numpy()
        trec_h = torch.empty((S, M, max(P, 1), 5), dtype=torch.float64).pin_memory().numpy() if P else None
        h2d = n0_h.nbytes + c0_h.nbytes + (ts_h.nbytes if ts_h is not None else 0) + (tg_h.nbytes if tg_h is not None else 0)
        d2h = sum(v.nbytes for v in outh.values()) + (grad_h.nbytes + trec_h.nbytes if P else 0)

        def e2e_step():
            ctx.run_batch(n0_h, c0_h, ts_h, tg_h, stream=stream)
            ctx.moments(out=outh)
            if P:
                ctx.tangents(out=dict(grad=grad_h, tangents=trec_h))     # gradient + every tangent record
        e2e_step()
        barrier(); torch.cuda.synchronize(dev)
        ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for k in range(args.steps):
            flush.fill_(float(k))
            ev2[k][0].record(stream)
            e2e_step()
            ev2[k][1].record(stream)
        torch.cuda.synchronize(dev); barrier()
        ms2 = sum(a.elapsed_time(b) for a, b in ev2) / args.steps
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([ms2], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms2 = float(t[0])
        e2e = dict(value=bu_total / (ms2 * 1e-3), unit=UNIT, h2d_bytes_per_step=int(h2d), d2h_bytes_per_step=int(d2h),
                   ms_per_step=ms2, host_buffers="pinned",
                   api="C ABI pbe_run_batch(n0_on_device=0) + pbe_moments + pbe_tangents (records, loss, gradient, "
                       "tangent records)")

    # ---- secondary (1 GPU): the C4 10^6-bin batch through the HBM-streaming kernel ----------------
    secondary = None
    next4 = None
    if world == 1 and args.workload == "c5" and not args.no_secondary:
        w4 = W.c4_sweep(1_000_000, batch=64, n_steps=1000)
        n04 = torch.from_numpy(np.ascontiguousarray(w4.n0)).to(dev)
        old_tb = os.environ.get("PBE_TEMPORAL_BLOCK")
        os.environ["PBE_TEMPORAL_BLOCK"] = "0"                      # plain streaming: 16 B/update
        ctx4 = pb.context_for(w4, device=local_rank)
        ms4, bu4, kms4 = measure(ctx4, w4, n04, None, gather=False)
        info4 = ctx4.last_run_info()
        secondary = dict(workload="C4 bin sweep N=1e6, batch 64, 1000 uncapped CFL steps (plain streaming)",
                         value=bu4 / (ms4 * 1e-3), unit=UNIT, ms_per_step=ms4,
                         roofline=roofline(w4, info4, bu4, kms4, "c4"), kernel=info4,
                         gpu_launches=int(info4["launches"]) * args.steps)
        ctx4.close()
        # NEXT-4: the same workload with temporal blocking (the library default for uncapped-CFL
        # steps mode): 8 steps per HBM pass, 2 B/update of traffic
        os.environ["PBE_TEMPORAL_BLOCK"] = "1"
        ctx4 = pb.context_for(w4, device=local_rank)
        ms5, bu5, kms5 = measure(ctx4, w4, n04, None, gather=False)
        info5 = ctx4.last_run_info()
        ctx4.close()
        if old_tb is None:
            os.environ.pop("PBE_TEMPORAL_BLOCK", None)
        else:
            os.environ["PBE_TEMPORAL_BLOCK"] = old_tb
        hbm = float(peaks.get("hbm_gbs", 6650.0))
        v5 = bu5 / (ms5 * 1e-3)
        next4 = dict(workload="C4 bin sweep N=1e6, batch 64, 1000 uncapped CFL steps, temporal blocking (NEXT-4)",
                     value=v5, unit=UNIT, ms_per_step=ms5, kernel=info5, speedup_vs_plain_stream=v5 / (bu4 / (ms4 * 1e-3)),
                     bytes_per_bin_update=16.0 / max(1, info5["steps_per_pass"]),
                     plain_stream_hbm_ceiling=hbm * 1e9 / 16.0, frac_of_plain_stream_ceiling=v5 / (hbm * 1e9 / 16.0),
                     gpu_launches=int(info5["launches"]) * args.steps)
        del n04

    # ---- NEXT-3 (1 GPU): one reverse-mode gradient over 1000 parameters (9 App-B experiments) vs the
    #      batched forward-difference gradient (the paper's jax-ND analogue) --------
    next3 = None
    if world == 1 and args.workload == "c5" and not args.no_secondary:
        P3 = 1000
        w3 = W.next3_estimation(n_params=P3)
        n03 = torch.from_numpy(np.ascontiguousarray(w3.n0)).to(dev)
        ctx3 = pb.context_for(w3, device=local_rank)
        ta = []
        for it in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            ctx3.run_adjoint(n03, w3.c0, w3.t_samples, w3.target)
            g3 = ctx3.adjoint_gradient(P3)
            torch.cuda.synchronize(); ta.append(time.perf_counter() - t0)
        r3 = ctx3.moments()
        i3 = ctx3.last_run_info()
        ctx3.close()
        h = 1e-6
        th = np.repeat(w3.theta, P3 + 1, axis=0)
        for si in range(w3.n_sims):
            blk = th[si * (P3 + 1):(si + 1) * (P3 + 1)]
            blk[1 + np.arange(P3), np.arange(P3)] += h * np.maximum(np.abs(w3.theta[si]), 1e-3)
        wf = W.replace(w3, theta=th, c0=np.repeat(w3.c0, P3 + 1), knot_T=np.repeat(w3.knot_T, P3 + 1, axis=0),
                       target=np.repeat(w3.target, P3 + 1, axis=0))
        ctxf = pb.context_for(wf, device=local_rank)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        ctxf.run_batch(n03, wf.c0, wf.t_samples, wf.target)
        ctxf.moments()
        torch.cuda.synchronize(); tf = time.perf_counter() - t0
        ctxf.close()
        next3 = dict(workload=f"NEXT-3: d loss/d theta, {P3} POLY parameters, 9 App-B experiments, N={w3.N}, "
                              f"{int(r3['steps'].max())} steps", metric="ms per gradient (wall, incl. copies)",
                     adjoint_ms=1e3 * min(ta), fd_batched_ms=1e3 * tf, fd_sims=int(wf.n_sims),
                     speedup_vs_fd=tf / min(ta), finite=bool(np.isfinite(g3["grad"]).all()),
                     kernel_ms=i3["main_ms"], cluster=i3["cluster"], ctas=i3["ctas"],
                     note="k_adjoint in 16-CTA clusters (one per experiment) + k_adjoint_theta; forward-mode "
                          "tangents need 100 passes of 10 lanes (tools/next3_time.py: ~400x slower)")
        del n03

    # ---- strong scaling on one GPU: the rank-0 shard of W = 2, 4, 8 GPUs (BASELINE config 5 as written) --
    strong_pred = None
    if world == 1 and args.workload == "c5" and args.scaling == "strong" and not args.quick:
        rows = []
        for Wn in (2, 4, 8):
            wsh = wg.subset(D.shard(wg.n_sims, 0, Wn))
            ctxs = pb.context_for(wsh, device=local_rank)
            n0s = torch.from_numpy(np.ascontiguousarray(wsh.n0)).to(dev)
            ms_s, bu_s, kms_s = measure(ctxs, wsh, n0s, ts, gather=False)
            ctxs.close()
            rows.append(dict(gpus=Wn, sims_per_gpu=int(wsh.n_sims), ms_per_step=ms_s,
                             predicted_efficiency=ms / (Wn * ms_s)))
        strong_pred = dict(rows=rows, note="T(4096 sims, 1 GPU) / (W x T(4096/W sims, 1 GPU)): a shard runs no "
                                          "collective during the march (one allgather of per-sim records after it)")

    # ---- C1-C3 and the C4 bin sweep beside the oracle on one host core (same inputs) -------------------
    def oracle_1core(wo, steps_cap=None):
        import oracle
        if steps_cap:
            wo = W.replace(wo, n_steps=steps_cap)
        t0 = time.perf_counter()
        r = oracle.run(wo, threads=1, want_n=False)
        dt = time.perf_counter() - t0
        return float(wo.N) * float(np.sum(r["steps"])) / dt, dt, int(np.sum(r["steps"]))

    cases, sweep = None, None
    if world == 1 and rank == 0 and not args.quick:
        cases = {}
        for name, wc, what in (("c1", W.c1_growth(W.LIM_VANLEER, M=1000), "growth, constant G, fixed dt"),
                               ("c2", W.c2_dissolution(), "dissolution, polynomial c*, T ramp"),
                               ("c3", W.c3_cycling(), "temperature cycling, 10^5 steps")):
            ctxc = pb.context_for(wc, device=local_rank)
            n0c = torch.from_numpy(np.ascontiguousarray(wc.n0)).to(dev)
            msc, buc, kmsc = measure(ctxc, wc, n0c, wc.t_samples, gather=False)
            infoc = ctxc.last_run_info()
            ctxc.close()
            nst = buc / wc.N
            orate, osec, _ = oracle_1core(wc)
            cases[name] = dict(workload=what, bins=wc.N, sims=1, steps=int(round(nst)), ms=msc,
                               us_per_step=1e3 * msc / nst, value=buc / (msc * 1e-3), unit=UNIT,
                               kernel=infoc["kernel"], threads_per_cta=infoc["threads_per_cta"],
                               oracle_1core=orate, oracle_seconds=osec, speedup_vs_oracle_1core=buc / (msc * 1e-3) / orate,
                               note="latency-bound: one simulation is one CTA; us/step is the figure of merit")
        sweep = []
        for N in (1000, 10000, 100000, 1000000):
            orate = None
            for b in (1, 64):
                w4 = W.c4_sweep(N, batch=b, n_steps=1000)
                ctx4 = pb.context_for(w4, device=local_rank)
                n04 = torch.from_numpy(np.ascontiguousarray(w4.n0)).to(dev)
                ms4, bu4, _ = measure(ctx4, w4, n04, None, gather=False)
                i4 = ctx4.last_run_info()
                ctx4.close()
                if orate is None:
                    cap = int(min(1000, max(20, 2e7 // N)))
                    orate, _, osteps = oracle_1core(W.c4_sweep(N, batch=1, n_steps=1000), steps_cap=cap)
                sweep.append(dict(bins=N, sims=b, steps=1000, ms=ms4, us_per_step=1e3 * ms4 / 1000,
                                  value=bu4 / (ms4 * 1e-3), unit=UNIT, kernel=i4["kernel"],
                                  steps_per_pass=i4["steps_per_pass"], oracle_1core=orate,
                                  oracle_note=(f"one simulation, first {osteps} of the 1000 steps on one core "
                                               "(per-step cost is constant in steps mode: rate extrapolated)"
                                               if osteps < 1000 else "one simulation, all 1000 steps, one core")))

    # ---- NEXT-1 (1 GPU): the paper's 2D model, 6000 x 3000 grid, 4 simulations ------------------------
    next1 = None
    if world == 1 and args.workload == "c5" and not args.quick:
        w2 = W.c2d_base(6000, 3000, n_sims=4)
        w2.n_steps = 100
        w2.t_samples = np.array([1.0])
        ctx2 = pb.context_for(w2, device=local_rank)
        n02 = torch.from_numpy(np.ascontiguousarray(w2.n0)).to(dev)
        ms2d, bu2d, kms2d = measure(ctx2, w2, n02, None, gather=False)
        i2 = ctx2.last_run_info()
        ctx2.close()
        next1 = dict(workload="NEXT-1 2D base case 6000 x 3000 (Godunov splitting, van Leer), 4 sims, 100 uncapped "
                              "CFL steps", value=bu2d / (ms2d * 1e-3), unit="cell-updates/s", ms_per_step=ms2d,
                     roofline=roofline(w2, i2, bu2d, kms2d, "c2d"), kernel=i2)
        del n02

    # ---- CPU oracle baseline (rank 0, N = 1 only) -----------------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        th = host_threads()
        bu, s, sdesc = oracle_sample(w, th)
        cpu = dict(value=bu / s, unit=UNIT, cores=th, kind="oracle", sample=sdesc, seconds=s)

    if rank == 0:
        cfg = dict(desc)
        cfg.update(parallelism=(f"sims sharded round-robin over {world} GPUs; NCCL allgather of per-sim records"
                                if world > 1 else "1 GPU"), l2="flushed between timed iterations (512 MiB write)",
                   scaling=args.scaling,
                   steps_per_sim_mean=bu_local / (w.N * max(w.N2, 1)) / max(w.n_sims, 1), kernel=info)
        line = dict(metric=METRIC, value=value, unit=UNIT, n_gpus=world, steps=args.steps, warmup=args.warmup,
                    ms_per_step=ms, higher_is_better=True, scaling=args.scaling if args.workload == "c5" else "weak",
                    vs_baseline=None, dtype="f64",
                    data="synthetic (seeded; DESIGN.md input recipe)", config=cfg, roofline=roof,
                    cpu_baseline=cpu, e2e=e2e, gpu_launches=int(info["launches"]) * args.steps, clocks=clk,
                    secondary=secondary, next3=next3, next4=next4, next1=next1,
                    strong_scaling_prediction=strong_pred, cases=cases, c4_sweep=sweep)
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    ctx.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
