"""SASS opcode histogram of the hot frame-kernel instances (evidence that the shipped
code uses TMA bulk copies, mbarriers and the sm_100 paired fp32 ops).

    python tools/sass_hist.py [build/frame.o] > profiles/r02_sass_hist.txt
"""
import collections
import re
import subprocess
import sys

OBJ = sys.argv[1] if len(sys.argv) > 1 else "build/frame.o"
INSTANCES = {
    "frame_kernel<3, fast, plain> (configs 2, 4)": "_ZN4woit12frame_kernelILi3ELb0ELb1ELi0ELi0EEEvNS_7KParamsE",
    "frame_kernel<3, fast, thin> (shallow scenes)": "_ZN4woit12frame_kernelILi3ELb0ELb1ELi1ELi0EEEvNS_7KParamsE",
    "frame_kernel<3, fast, deep> (config 5)": "_ZN4woit12frame_kernelILi3ELb0ELb1ELi2ELi0EEEvNS_7KParamsE",
    "frame_kernel<3, fast, packed storage>": "_ZN4woit12frame_kernelILi3ELb0ELb1ELi0ELi16EEEvNS_7KParamsE",
    "frame_kernel<3, general, config-3 flags>": "_ZN4woit12frame_kernelILi3ELb1ELb1ELi1ELi7EEEvNS_7KParamsE",
}
KEYS = ("UBLKCP", "UTMACCTL", "SYNCS", "FFMA2", "FMUL2", "FADD2", "MUFU", "LDS", "STS", "SHFL", "MATCH", "DFMA",
        "DADD", "DMUL", "F2I", "ATOMS", "RED", "BAR", "FFMA", "FADD", "FMUL")
for label, sym in INSTANCES.items():
    out = subprocess.run(["cuobjdump", "-sass", "-fun", sym, OBJ], capture_output=True, text=True).stdout
    ops = collections.Counter()
    for ln in out.splitlines():
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", ln)
        if m:
            ops[m.group(1)] += 1
    total = sum(ops.values())
    print(f"{label}  [{sym}]  {total} SASS instructions")
    print("  " + "  ".join(f"{k}={ops.get(k, 0)}" for k in KEYS))
