"""Same-box A/B of woit_bin_frame (config 2, layer-major and random arrival, core
fields) over the libraries in variants_lib/ (WOIT_LIB selects one per child process).

    python tools/bin_ab.py [--rounds 3]
"""
import glob
import json
import os
import statistics
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child():
    sys.path.insert(0, REPO)
    import torch
    import paper_2201_00094_b200 as W
    frame = W.FrameFragments.synthetic("smoke", 1920, 1080, seed=1, layers=32)
    n = frame.nfrag
    run = frame.offsets[1:] - frame.offsets[:-1]
    L = int(run.max())
    lm = frame.offsets[:-1][None, :] + torch.arange(L, device="cuda")[:, None]
    lm = lm[torch.arange(L, device="cuda")[:, None] < run[None, :]].contiguous()
    rnd = torch.randperm(n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(5))
    out = {}
    for tag, od in (("layer_major", lm), ("random", rnd)):
        pix = W.pixel_ids(frame)[od].to(torch.int32).contiguous()
        ins = [frame.depth[od], frame.alpha[od], frame.trans[od], frame.radiance[od]]
        fb = W.FrameFragments.from_unbinned(1920, 1080, pix, *ins)
        ok = bool(torch.equal(fb.offsets, frame.offsets))
        if tag == "layer_major":  # arrival order within a pixel = the CSR order
            ok = ok and bool(torch.equal(fb.depth, frame.depth)) and bool(torch.equal(fb.radiance, frame.radiance))
        st = torch.cuda.current_stream()
        ts = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            for _ in range(5):
                W.FrameFragments.from_unbinned(1920, 1080, pix, *ins)
            b.record(st)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / 5)
        out[tag] = (statistics.median(ts), ok)
    print(json.dumps(out))


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        return child()
    rounds = int(sys.argv[sys.argv.index("--rounds") + 1]) if "--rounds" in sys.argv else 3
    libs = sorted(glob.glob(os.path.join(REPO, "variants_lib", "libwoit_*.so")))
    res = {}
    for r in range(rounds):
        for lib in libs:
            name = os.path.basename(lib)[8:-3]
            o = subprocess.run([sys.executable, __file__, "child"], env={**os.environ, "WOIT_LIB": lib},
                               capture_output=True, text=True)
            line = o.stdout.strip().splitlines()[-1] if o.stdout.strip() else o.stderr[-300:]
            print(f"round {r} {name}: {line}", flush=True)
            try:
                for k, (ms, ok) in json.loads(line).items():
                    res.setdefault((name, k), []).append(ms)
                    assert ok, (name, k)
            except ValueError:
                pass
    print("median:")
    for (name, k), v in sorted(res.items()):
        print(f"  {name:10s} {k:12s} {statistics.median(v):.3f} ms")


if __name__ == "__main__":
    main()
