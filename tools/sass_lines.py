"""Static SASS profile of one kernel in libpbe.so: instructions per source line."""
import collections
import os
import re
import subprocess
import sys
import tempfile

lib = sys.argv[1]
pat = sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
parts = re.split(r"\n\s*\.section\s+\.text\.", txt)
part = [p for p in parts if re.match(pat, p)][0]
cur = None
cnt, ops, allops = collections.Counter(), collections.defaultdict(collections.Counter), collections.Counter()
for l in part.splitlines():
    if l.strip().startswith("//"):
        m = re.search(r"line (\d+)", l)
        f = re.search(r'"([^"]+)"', l)
        if m:
            cur = ((f.group(1).split("/")[-1] if f else "?"), int(m.group(1)))
        continue
    m2 = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", l)
    if m2:
        allops[m2.group(2)] += 1
        if cur:
            cnt[cur] += 1
            ops[cur][m2.group(2)] += 1
print("static instructions", sum(allops.values()))
print("opcodes:", dict(allops.most_common(25)))
for k, n in cnt.most_common(top):
    print(f"{n:6d} {k[0]}:{k[1]}  {dict(ops[k].most_common(5))}")
