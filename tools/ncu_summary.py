"""Summarise an ncu report: key SOL metrics, pipe utilisation, stall reasons, opcode mix."""
import collections
import csv
import io
import re
import subprocess
import sys


def ncu(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main(rep, kernel_regex=None):
    raw = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    hdr, vals = raw[0], raw[2]
    d = dict(zip(hdr, vals))
    keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "smsp__warps_eligible.avg.per_cycle_active", "smsp__warps_active.avg.per_cycle_active",
            "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
            "smsp__inst_executed.sum"]
    for k in keys:
        if k in d:
            print(f"{k:75s} {d[k]}")
    stalls = {k: v for k, v in d.items() if k.startswith("smsp__average_warp_latency_issue_stalled_") or
              (k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"))}
    tot = 0.0
    items = []
    for k, v in stalls.items():
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            continue
        items.append((x, k)); tot += x
    items.sort(reverse=True)
    print("-- stall samples --")
    for x, k in items[:12]:
        print(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):50s} {100 * x / max(tot, 1):5.1f}%")
    src = list(csv.reader(io.StringIO(ncu([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    h = src[1]
    i_src, i_exec, i_samp = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    cnt, samp = collections.Counter(), collections.Counter()
    for r in src[2:]:
        if len(r) <= i_exec:
            continue
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[i_src].strip())
        if not m:
            continue
        try:
            cnt[m.group(2)] += int(r[i_exec]); samp[m.group(2)] += int(r[i_samp] or 0)
        except ValueError:
            pass
    tc, ts = sum(cnt.values()), sum(samp.values())
    print("-- opcode mix (executed warp instructions, share of stall samples) --")
    for op, n in cnt.most_common(22):
        print(f"  {op:10s} {n / 1e6:9.1f}M {100 * n / tc:5.1f}%   stalls {100 * samp[op] / max(ts, 1):5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
