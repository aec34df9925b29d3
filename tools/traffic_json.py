"""profiles/traffic.json from ncu --set full captures: dram__bytes_read.sum +
dram__bytes_write.sum per launch of the frame kernel, keyed config<N>_rank<R>.

    python tools/traffic_json.py OUT.json key=report.ncu-rep [key=report.ncu-rep ...]
"""
import csv
import json
import os
import subprocess
import sys

out = {"_doc": "dram__bytes_read.sum + dram__bytes_write.sum per launch of the frame kernel (bytes), "
               "from one ncu --set full capture of the same configuration bench.py measures; "
               "source reports listed under _source (tools/refresh_profiles.sh)", "_source": {}}
for arg in sys.argv[2:]:
    key, rep = arg.split("=", 1)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) < 3:
        continue
    h, units = rows[0], rows[1]
    for v in rows[2:]:
        d = dict(zip(h, v))
        if "frame_kernel" not in d.get("Kernel Name", ""):
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(d[k].replace(",", "")) * scale.get(units[h.index(k)], 1)
        out[key] = int(round(tot))
        out["_source"][key] = os.path.basename(rep)
        break
with open(sys.argv[1], "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out))
