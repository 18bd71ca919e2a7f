"""SASS FP64 instructions per bin-update of a kernel from an ncu source-page CSV export
(tools/gpu_ncu_c5.sh writes gpurun_out/ncu_TAG_sass.csv and ncu_TAG_raw.csv), stored in
profiles/fp64_instr.json for bench.py's roofline entry (frac_sass).
usage: python tools/fp64_count.py gpurun_out/ncu_TAG KERNEL BIN_UPDATES"""
import collections
import csv
import json
import os
import sys

base, kname, bu = sys.argv[1], sys.argv[2], float(sys.argv[3])
rows = list(csv.reader(open(base + "_sass.csv")))
hdr = rows[1]
i_src, i_ti = hdr.index("Source"), hdr.index("Thread Instructions Executed")
cnt = collections.Counter()
for r in rows[2:]:
    if len(r) < len(hdr) or not r[i_ti].isdigit():
        continue
    op = r[i_src].split()
    if not op:
        continue
    o = (op[1] if op[0].startswith("@") else op[0]).split(".")[0]
    cnt[o] += int(r[i_ti])
fp = sum(cnt[k] for k in ("DFMA", "DADD", "DMUL", "DSETP", "DMNMX"))
raw = list(csv.reader(open(base + "_raw.csv")))
d = dict(zip(raw[0], [r for r in raw[2:] if len(r) == len(raw[0])][0]))
pipe = float(d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "nan").replace(",", "")) / 100
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "fp64_instr.json")
tab = json.load(open(out)) if os.path.exists(out) else {}
tab[kname] = dict(sass_fp64_instr_per_bin_update=round(fp / bu, 2), ncu_fp64_pipe_active=round(pipe, 4),
                  by_opcode={k: round(cnt[k] / bu, 2) for k in ("DFMA", "DADD", "DMUL", "DSETP", "DMNMX") if cnt[k]},
                  source=f"ncu --set full thread-instruction counts ({os.path.basename(base)}), {bu:.4g} bin-updates")
json.dump(tab, open(out, "w"), indent=1)
print(kname, tab[kname])
