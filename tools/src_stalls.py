"""Aggregate an ncu source page (``ncu -i X --page source --csv --print-source cuda,sass``)
by CUDA source line: share of warp-stall samples and the top stall reasons.

    python tools/src_stalls.py gpurun_out/src.csv [--top 40]
"""
import argparse
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    cur = hdr = None
    out = []
    for r in csv.reader(open(a.csv)):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if not (hdr and cur):
            continue
        try:
            ln = int(r[0])
        except ValueError:
            continue
        d = dict(zip(hdr, r))
        try:
            s = float(d.get("Warp Stall Sampling (All Samples)") or 0)
        except ValueError:
            s = 0.0
        if s > 0:
            st = sorted(((float(v), k[6:]) for k, v in d.items()
                         if k.startswith("stall_") and "(Not" not in k and v not in ("0", "")), reverse=True)[:3]
            out.append((s, cur.split("/")[-1], ln, r[1].strip()[:90], st, d.get("Instructions Executed", "")))
    tot = sum(o[0] for o in out) or 1.0
    print(f"total samples {tot:.0f} over {len(out)} lines")
    for s, f, ln, src, st, ie in sorted(out, reverse=True)[:a.top]:
        print(f"{100 * s / tot:5.1f}% {f}:{ln} inst={ie} {src!r} " + " ".join(f"{k}={v:.0f}" for v, k in st))


if __name__ == "__main__":
    main()
