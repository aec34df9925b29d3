"""Build and time tuning variants of libwoit on one config (run on the GPU box).

    python tools/variants.py build NAME=DEF1,DEF2 ...   # here: compile variants
    python tools/variants.py time                       # on the box: time each built variant
"""
import glob
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VDIR = os.path.join(REPO, "variants_lib")  # git-ignored, travels with gpurun (build/ does not)


def do_build(specs):
    sys.path.insert(0, REPO)
    from paper_2201_00094_b200 import build as B
    os.makedirs(VDIR, exist_ok=True)
    for spec in specs:
        name, defs = spec.split("=", 1) if "=" in spec else (spec, "")
        defines = tuple(d for d in defs.split(",") if d)
        out = os.path.join(VDIR, f"libwoit_{name}.so")
        B.build(defines=defines or ("WOIT_VARIANT_BASE=1",), out=out)
        print("built", out, defines)


def do_time(extra):
    res = {}
    for lib in sorted(glob.glob(os.path.join(VDIR, "libwoit_*.so"))):
        name = os.path.basename(lib)[len("libwoit_"):-3]
        env = dict(os.environ, WOIT_LIB=lib)
        r = subprocess.run([sys.executable, os.path.join(REPO, "tools", "profile_frame.py"), "--iters", "6", *extra],
                           env=env, capture_output=True, text=True)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("ms per frame")]
        res[name] = line[0] if line else (r.stderr[-400:] or "failed")
        print(name, res[name], flush=True)
    return res


if __name__ == "__main__":
    if sys.argv[1] == "build":
        do_build(sys.argv[2:])
    else:
        do_time(sys.argv[2:])
