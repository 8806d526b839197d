"""Per-kernel SASS instruction census of the built library (cuobjdump -sass):
DMMA (FP64 tensor MMA), UBLKCP (bulk-copy engine), SYNCS (mbarriers), LDGSTS
(cp.async), the proof that the hot kernels run on the FP64 tensor pipe and the
copy engine.  python scripts/sass_summary.py > profiles/<tag>_sass.md"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.path.join(ROOT, "paper_2502_08382_b200", "libfeti_b200.so")
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
cnt = collections.defaultdict(collections.Counter)
cur = None
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"/\*[0-9a-f]{4,6}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if cur and m:
        cnt[cur][m.group(1).split(".")[0]] += 1
names = subprocess.run(["c++filt"], input="\n".join(cnt), capture_output=True, text=True).stdout.split("\n")
rows = []
for (f, c), dn in zip(cnt.items(), names):
    rows.append((dn.split("(")[0].replace("feti::", ""), c["DMMA"], c["UBLKCP"], c["SYNCS"], c["LDGSTS"],
                 sum(c.values())))
rows.sort(key=lambda r: (-r[1], -r[2], r[0]))
print("| kernel | DMMA | UBLKCP | SYNCS | LDGSTS | instructions |")
print("|---|---|---|---|---|---|")
for r in rows:
    print("| " + " | ".join(str(x) for x in r) + " |")
