"""Per-phase instruction / stall breakdown of the frame kernel from an ncu cuda,sass csv."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
nfrag = float(sys.argv[2]) if len(sys.argv) > 2 else 66355200
src = open(sys.argv[3] if len(sys.argv) > 3 else "paper_2201_00094_b200/csrc/frame.cu").read().split("\n")
marks = [(i + 1, l.strip()[8:44]) for i, l in enumerate(src) if l.strip().startswith("// ---- ")]


def region(ln):
    name = "pre"
    for m, n in marks:
        if ln >= m:
            name = n
    return name


hdr = None
cur = None
agg, aggi, tot, lines = {}, {}, {}, []
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
        s = float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
        ins = float(d.get("Instructions Executed", 0) or 0)
    except ValueError:
        continue
    key = region(int(r[0])) if cur == "frame.cu" else cur
    agg[key] = agg.get(key, 0) + s
    aggi[key] = aggi.get(key, 0) + ins
    lines.append((s, ins, cur, r[0], r[1][:90]))
    for k, v in d.items():
        if k.startswith("stall_") and "(Not Issued)" not in k:
            try:
                tot[k] = tot.get(k, 0) + float(v or 0)
            except ValueError:
                pass
ts = sum(agg.values())
print(f"total {sum(aggi.values()) / nfrag:.2f} warp-instr/frag")
for k in sorted(agg, key=lambda k: -agg[k]):
    print(f"{100 * agg[k] / ts:5.1f}% samples  {aggi[k] / nfrag:5.2f} winst/frag  {k}")
s = sum(tot.values())
print("stalls:", ", ".join(f"{k[6:]} {100 * v / s:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:7]))
print("top lines by stall samples:")
for sm, ins, f, ln, txt in sorted(lines, key=lambda x: -x[0])[:int(sys.argv[4]) if len(sys.argv) > 4 else 15]:
    print(f"  {100 * sm / ts:5.1f}%  {ins / nfrag:5.2f}  {f}:{ln} {txt}")
