"""Aggregate an ncu 'cuda,sass' source page (csv) to per-source-line totals."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = []
cur_file = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    d = dict(zip(hdr[2:], r[2:]))
    # line rows have Line No filled and Address '-'
    try:
        samples = int(r[4] or 0)
    except ValueError:
        continue
    def num(k):
        try:
            return float(d.get(k, 0) or 0)
        except ValueError:
            return 0.0
    out.append((samples, num("Instructions Executed"), cur_file, r[0], r[1][:90]))
tot_s = sum(o[0] for o in out) or 1
tot_i = sum(o[1] for o in out) or 1
out.sort(reverse=True)
print(f"total samples {tot_s}, instructions {tot_i:.3e}")
for s, i, f, ln, src in out[:top]:
    print(f"{100*s/tot_s:5.1f}%  inst {100*i/tot_i:5.1f}%  {f}:{ln}  {src}")
