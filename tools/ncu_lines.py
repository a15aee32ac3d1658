"""Aggregate ncu source-page (SASS) stall samples by CUDA source line.

usage: python tools/ncu_lines.py <report.ncu-rep> <binary-or-cubin-sass> [N]
The SASS listing (nvdisasm -g -c) of the same build maps offsets to lines.
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, sass = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
S = "Warp Stall Sampling (All Samples)"
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][ix["Address"]], 16)
off2line = {}
cur = ("?", 0)
for l in open(sass):
    m = re.search(r'//## File "([^"]*)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m:
        off2line[int(m.group(1), 16)] = cur
agg = collections.Counter()
why = collections.defaultdict(collections.Counter)
tot = 0.0
for r in data:
    off = int(r[ix["Address"]], 16) - base
    v = float(r[ix[S]] or 0)
    tot += v
    key = off2line.get(off, ("?", 0))
    agg[key] += v
    for s in stalls:
        why[key][s] += float(r[ix[s]] or 0)
srcs = {}
for (f, l), v in agg.most_common(N):
    if f not in srcs:
        try:
            srcs[f] = open(subprocess.run(["bash", "-c", f"ls /root/repo/paper_0809_2407_b200/csrc/{f} 2>/dev/null || echo /dev/null"], capture_output=True, text=True).stdout.strip()).read().split("\n")
        except Exception:
            srcs[f] = []
    txt = srcs[f][l - 1].strip() if 0 < l <= len(srcs[f]) else ""
    top = ", ".join(f"{k[6:]} {c / v * 100:.0f}%" for k, c in why[(f, l)].most_common(2)) if v else ""
    print(f"{v / tot * 100:5.1f}% {f}:{l:<4} {txt[:60]:60s} [{top}]")
