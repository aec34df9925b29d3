"""Instructions executed per fragment by source region (frame.cu line ranges)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
nfrag = float(sys.argv[2]) if len(sys.argv) > 2 else 66355200
regions = []
for a in sys.argv[3:]:
    lo, hi, name = a.split(":")
    regions.append((int(lo), int(hi), name))
hdr = None
cur = None
agg = {}
byline = {}
tot = 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        inst = float(d.get("Instructions Executed", 0) or 0)
    except ValueError:
        continue
    tot += inst
    key = cur
    if cur == "frame.cu":
        for lo, hi, name in regions:
            if lo <= int(r[0]) <= hi:
                key = name
    agg[key] = agg.get(key, 0) + inst
    byline[(cur, r[0], r[1][:60])] = inst
print(f"total {tot / nfrag:.2f} warp-instr/frag")
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"  {k:26s} {v / nfrag:6.2f}")
print("top lines:")
for k, v in sorted(byline.items(), key=lambda x: -x[1])[:30]:
    print(f"  {v / nfrag:6.3f} {k[0]}:{k[1]} {k[2]}")
