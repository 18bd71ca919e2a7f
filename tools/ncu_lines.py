"""Per-source-line instruction and stall-sample shares of an ncu report (needs -lineinfo
and --import-source on)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
data, fname = [], None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] and r[0].isdigit():
        try:
            data.append((int(r[7] or 0), int(r[4] or 0), fname, int(r[0]), r[1][:95]))
        except ValueError:
            pass
tot = sum(d[0] for d in data) or 1
ts = sum(d[1] for d in data) or 1
print(f"instructions {tot}, stall samples {ts}")
for n, sm, f, l, src in sorted(data, key=lambda d: -d[1])[:top]:
    print(f"stall {100 * sm / ts:5.1f}%  inst {100 * n / tot:5.1f}%  {f}:{l:<4d} {src}")
