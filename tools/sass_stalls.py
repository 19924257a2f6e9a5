"""Aggregate ncu warp-stall samples (source page, SASS) by the innermost line of
one of our .cu files, using nvdisasm -g line info of the same cubin.

  python tools/sass_stalls.py /tmp/sass.csv /tmp/ab.sass attn_bwd.cu
"""
import collections
import csv
import re
import sys

sass_csv, dis, target = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) >= len(hdr) - 1]
base = int(data[0]["Address"], 16)
lines = open(dis).read().split("\n")
kname = rows[0][1].split("(")[0].split("::")[-1]
start = [i for i, l in enumerate(lines) if l.strip().startswith(".text.") and kname in l][0]
# nvdisasm prints only the innermost file:line; attribute helper-header code to the
# last line of `target` seen above it in the listing (its call site, approximately)
mp, last = {}, -1
for l in lines[start:]:
    if "//## File" in l:
        m = re.search(r'File "([^"]+)", line (\d+)', l)
        if m and m.group(1).split("/")[-1] == target:
            last = int(m.group(2))
        continue
    a = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if a:
        mp[int(a.group(1), 16)] = last
agg = collections.Counter()
for d in data:
    agg[mp.get(int(d["Address"], 16) - base, -2)] += int(d["Warp Stall Sampling (All Samples)"] or 0)
src = open([p for p in sys.argv[4:5]][0] if len(sys.argv) > 4 else f"paper_2510_18830_b200/csrc/{target}").read().split("\n")
tot = sum(agg.values())
for ln, c in agg.most_common(30):
    print(f"{c:8d} {100 * c / tot:5.1f}% L{ln}: {src[ln - 1].strip()[:90] if ln > 0 else ''}")
