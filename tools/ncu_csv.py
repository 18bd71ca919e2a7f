"""Summaries of ncu CSV exports (tools/gpu_ncu_c5.sh): key metrics + stall reasons from the raw
page, per-source-line stall/instruction shares from the source page.
usage: python tools/ncu_csv.py gpurun_out/ncu_TAG [top]"""
import collections
import csv
import io
import sys

base = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = list(csv.reader(open(base + "_raw.csv")))
hdr = raw[0]
row = [r for r in raw[2:] if len(r) == len(hdr)][0]
d = dict(zip(hdr, row))
keys = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active", "smsp__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smsp__sass_inst_executed_op_local_ld.sum", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fp64.sum", "smsp__inst_executed_pipe_fp64.sum"]
for k in keys:
    if k in d:
        print(f"{k:75s} {d[k]}")
st = {}
for k, v in d.items():
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            st[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v.replace(",", ""))
        except ValueError:
            pass
tot = sum(st.values()) or 1
print("-- stall samples --")
for k, v in sorted(st.items(), key=lambda x: -x[1])[:12]:
    print(f"  {k:40s} {100 * v / tot:5.1f}%")
# per source line (CUDA source rows of the mixed page)
rows = list(csv.reader(open(base + "_src.csv")))
fname, data = None, []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] and r[0].isdigit() and fname:
        try:
            data.append((int(r[7] or 0), int(r[4] or 0), fname, int(r[0]), r[1][:95]))
        except ValueError:
            pass
ti = sum(x[0] for x in data) or 1
ts = sum(x[1] for x in data) or 1
print(f"-- per line: instructions {ti}, stall samples {ts}")
for n, sm, f, l, src in sorted(data, key=lambda x: -x[1])[:top]:
    print(f"stall {100 * sm / ts:5.1f}%  inst {100 * n / ti:5.1f}%  {f}:{l:<4d} {src}")
