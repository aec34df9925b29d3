"""Summarise an ncu launch list (``ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv --log-file X ...``): one line per launch with its duration and
DRAM bytes, kernels filtered by a name substring.

    python tools/launch_list.py gpurun_out/binprof.csv [--filter bin::]
"""
import argparse
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--filter", default="bin::")
    a = ap.parse_args()
    hdr, agg = None, {}
    for r in csv.reader(open(a.csv)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            agg.setdefault((int(d["ID"]), d["Kernel Name"][:60]), {})[d["Metric Name"]] = float(
                d["Metric Value"].replace(",", ""))
    tot = 0.0
    for (i, name), v in sorted(agg.items()):
        if a.filter not in name:
            continue
        t = v.get("gpu__time_duration.sum", 0.0) / 1e3
        tot += t
        print(i, name, "%.1f us" % t, "R %.0f MB W %.0f MB" % (v.get("dram__bytes_read.sum", 0.0) / 1e6,
                                                             v.get("dram__bytes_write.sum", 0.0) / 1e6))
    print("total %.1f us" % tot)


if __name__ == "__main__":
    main()
