"""Benchmark: Gfragments/s of the fused wavelet OIT frame (build + evaluate + composite).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2|4]

Workload (BASELINE.json configs[1], "config 2"): 1920x1080, 32 fragments/pixel
synthetic smoke volume, rank 3 (16 Haar slots), fp32 CSR stream generated on the
device (bit-identical to the numpy generator). One step = one full frame through
the fused kernel: bounds, closed-form Haar build, per-fragment transmittance v̂
(written, 12 B/fragment), visibility-weighted accumulation and composite (image
written). Inputs (2.1 GB) are larger than L2 (126 MB), so no flush is needed.

Multi-GPU (torchrun, one rank per GPU): config 2 scales weakly -- rank r renders
rows [1080 r, 1080 (r+1)) of a 1920 x 1080N frame; --config 4 (BASELINE configs[3],
4K x 128 particles) scales strongly -- the one 4K frame is split into N equal row
bands. Either way the fp32 image bands are all-gathered over NCCL inside the timed
step, and time = max over ranks.

--impl reference times the reference's CPU algorithm (the numpy port in oracle/,
a float64 restatement pinned against the reference's own outputs) on the host
cores, on a bounded row band of the same workload per step.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "Gfragments/s (build+eval+composite) and % HBM roofline at 1/2/4/8 B200 vs CPU"
UNIT = "Gfrag/s"
CPU_STEPS = 8        # cpu_baseline: 8 timed renders of the row band (~10 s of CPU work)
REF_BUDGET_S = 150.0  # --impl reference: wall-clock budget for all W + K steps
CONFIGS = {
    2: dict(workload="smoke", width=1920, height=1080, layers=32, rank=3, seed=1,
            name="config2: 1080p synthetic smoke, 32 frag/px, rank 3 (16 coeffs), 1 B200"),
    4: dict(workload="particles", width=3840, height=2160, layers=128, rank=3, seed=1, strong=True,
            name="config4: 4K particles, 128 frag/px, depth-varying alpha, rank 3, row bands over the GPUs"),
    # config 5: the 8K x 256 stress frame is 8.5 G fragments (272 GB of fp32 stream), so
    # it is the 8-GPU job: every GPU renders its 540-row eighth (1.06 G fragments);
    # N GPUs render the first N eighths, N = 8 the whole frame. --rank 2/3/4 sweeps
    # the coefficient count (8/16/32).
    5: dict(workload="particles", width=7680, height=4320, layers=256, rank=3, seed=1, share=8,
            name="config5: 8K stress, 256 frag/px, 540-row eighth of the frame per GPU"),
}


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def algorithmic_bytes(npix: int, nfrag: int, rank: int) -> int:
    """44 B/fragment (depth, alpha, T, L in; v̂ out) +
    (32 + 12 S) B/pixel (offsets, opaque RGB in; coefficients, image out)."""
    S = 1 << (rank + 1)
    return nfrag * 44 + npix * (32 + 12 * S)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_reference(cfg, rows: int, steps: int, warmup: int):
    """Time the reference algorithm (numpy port, all host threads) on `rows` rows."""
    from oracle import woit_oracle as O
    from paper_2201_00094_b200 import synth

    workers = O.default_workers()
    sf = synth.generate(cfg["workload"], cfg["width"], cfg["height"], seed=cfg["seed"], layers=cfg["layers"],
                        row0=0, rows=rows)
    frame = O.OFrame.from_synth(sf)
    ocfg = O.OConfig(rank=cfg["rank"], width=cfg["width"], height=rows, workers=workers)
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        O.render_frame(frame, ocfg, workers=workers)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    n = sf.nfrag
    return n / float(np.mean(times)) / 1e9, workers, f"{rows} rows x {cfg['width']} px x {cfg['layers']} frag/px " \
        f"= {n} fragments, float64 numpy port, {workers} threads", float(np.mean(times))


def run_reference(args, cfg):
    """The reference's CPU path (the pinned numpy port, all host threads) on this
    arm's config and metric. Every step renders a bounded row band of the frame;
    the band height is sized from a short pilot so that all W + K steps finish in
    about REF_BUDGET_S seconds. Rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    _, _, _, pilot_s = cpu_reference(cfg, 16, 1, 0)
    rate = 16 * cfg["width"] * cfg["layers"] / pilot_s  # fragments/s
    total = max(1, args.steps + args.warmup)
    rows = int(REF_BUDGET_S * rate / (total * cfg["width"] * cfg["layers"]))
    rows = max(4, min(args.ref_rows, rows))
    value, cores, sample, secs = cpu_reference(cfg, rows, args.steps, args.warmup)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg["name"], "width": cfg["width"], "height": cfg["height"],
                       "frag_per_px": cfg["layers"], "rank": cfg["rank"]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample + " per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, cfg):
    import torch

    import paper_2201_00094_b200 as W
    from paper_2201_00094_b200 import _lib

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    Wd = cfg["width"]
    strong = bool(cfg.get("strong"))
    if cfg.get("share"):
        # config 5: the GPU's fixed share of the frame (weak scaling up to the full frame)
        frame_h = cfg["height"]
        if world > cfg["share"]:
            raise SystemExit(f"--config {args.config} runs on at most {cfg['share']} GPUs")
        H1 = frame_h // cfg["share"]
    elif strong:
        # config 4: one frame, screen-sharded into equal row bands (strong scaling)
        frame_h = cfg["height"]
        if frame_h % world:
            raise SystemExit(f"--config 4 needs the GPU count to divide {frame_h} rows")
        H1 = frame_h // world
    else:
        # config 2: every GPU renders a 1080-row band of a 1920 x 1080N frame (weak scaling)
        H1 = cfg["height"]
        frame_h = H1 * world
    frame = W.FrameFragments.synthetic(cfg["workload"], Wd, frame_h, seed=cfg["seed"], layers=cfg["layers"],
                                       row0=H1 * rank, rows=H1, device=dev)
    rcfg = W.RenderConfig(rank=cfg["rank"], width=Wd, height=frame_h)
    lib = _lib.load()
    P, n = frame.npix, frame.nfrag
    S = 1 << (cfg["rank"] + 1)
    coeffs = torch.empty(P, S, 3, dtype=torch.float32, device=dev)
    vhat = torch.empty(n, 3, dtype=torch.float32, device=dev)
    out = torch.empty(P, 3, dtype=torch.float32, device=dev)
    image = torch.empty(P * world, 3, dtype=torch.float32, device=dev) if world > 1 else out
    wsn = lib.woit_frame_workspace_bytes(P, n)
    ws = torch.empty(wsn, dtype=torch.uint8, device=dev)
    fs = frame.c_struct()
    ps = W.pipeline._params(rcfg, cfg["rank"])
    bs = _lib.Bufs()
    bs.coeffs, bs.vhat, bs.output = coeffs.data_ptr(), vhat.data_ptr(), out.data_ptr()
    stream = torch.cuda.current_stream(dev)

    def step():
        _lib.check(lib.woit_render_band(fs, ps, bs, ws.data_ptr(), wsn, stream.cuda_stream), "render_band")
        if world > 1:
            pg.all_gather_into_tensor(image, out)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        pg.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        time.sleep(0.1)
        torch.cuda.synchronize()
        if world > 1:
            pg.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for i in range(args.steps):
            starts[i].record(stream)
            _lib.check(lib.woit_render_band(fs, ps, bs, ws.data_ptr(), wsn, stream.cuda_stream), "render_band")
            kends[i].record(stream)
            if world > 1:
                pg.all_gather_into_tensor(image, out)
            ends[i].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            pg.barrier()
    total_ms = t0.elapsed_time(t1)
    kern_ms = float(np.mean([s.elapsed_time(k) for s, k in zip(starts, kends)]))
    if world > 1:
        t = torch.tensor([total_ms, kern_ms], device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        total_ms, kern_ms = float(t[0]), float(t[1])
    ms = total_ms / args.steps
    frags_total = n
    if world > 1:
        tn = torch.tensor([n], dtype=torch.int64, device=dev)
        pg.all_reduce(tn)
        frags_total = int(tn.item())
    value = frags_total / (ms * 1e-3) / 1e9

    # end to end through the public API: pinned host stream -> device, render, image -> host
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, W, frame, rcfg, dev, world, pg, out)

    peak, peak_kind = peaks()
    if args.traffic is None:
        try:
            with open(os.path.join(REPO, "profiles", "traffic.json")) as f:
                args.traffic = json.load(f).get(f"config{args.config}")
        except Exception:
            args.traffic = None
    alg = algorithmic_bytes(P, n, cfg["rank"])
    frame_in_bytes = n * 32 + (P + 1) * 8 + P * 12  # depth, alpha, T, L + offsets + opaque RGB
    achieved = alg / (kern_ms * 1e-3) / 1e9
    clocks = clk.summary()
    if rank != 0:
        if pg is not None:
            pg.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        # a bounded sample: <= 14.7 M fragments (config 2: 240 rows)
        rows = max(1, min(args.ref_rows, 14745600 // (cfg["width"] * cfg["layers"])))
        v, cores, sample, secs = cpu_reference(cfg, rows, CPU_STEPS, 1)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{sample}, 1 warm-up + {CPU_STEPS} timed renders ({CPU_STEPS * secs:.1f} s)"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": "f32 (z, indices and per-pixel sums in f64)", "data": "synthetic",
        "config": {"workload": cfg["name"], "width": Wd, "height": frame_h, "frag_per_px": cfg["layers"],
                   "rank": cfg["rank"], "fragments": frags_total, "l2_flush": f"inputs {frame_in_bytes / 1e9:.1f} GB/GPU > 126 MB L2",
                   "parallelism": f"row bands x{world}, NCCL image all-gather" if world > 1 else "1 GPU"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": args.traffic,
                     "kernel": f"frame_kernel<{cfg['rank']}> (fused bounds+build+eval+composite)",
                     "kernel_ms": kern_ms, "algorithmic_bytes_per_launch": alg, "peak_kind": peak_kind},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": 2 * args.steps,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    if pg is not None:
        pg.destroy_process_group()


def run_e2e(args, W, frame, rcfg, dev, world, pg, ref_image=None):
    """Same metric through the public API with host buffers: every step copies the
    step's fragment stream host->device (pinned), renders, and reads the image back.
    Uploads are double-buffered on a copy stream, so step i+1's upload overlaps step
    i's render and read-back; the timed region still holds every step's copies."""
    import torch

    names = ("offsets", "depth", "alpha", "trans", "radiance", "opaque_color")
    host = {k: torch.empty_like(getattr(frame, k), device="cpu").pin_memory() for k in names}
    for k in names:
        host[k].copy_(getattr(frame, k))
    # two device copies of the stream: step i+1's upload (copy stream) overlaps step
    # i's render and image read-back (compute stream), as a frame-serving loop would
    devbufs = [{k: torch.empty_like(getattr(frame, k)) for k in names} for _ in range(2)]
    f2s = [W.FrameFragments(frame.width, frame.height, d["offsets"], d["depth"], d["alpha"],
                            d["trans"], d["radiance"], frame.normal, frame.ior, frame.backface,
                            frame.opaque_depth, d["opaque_color"], frame.pixel_base, frame.frag_base)
           for d in devbufs]
    bufs = W.FrameBuffers.allocate(f2s[0], rcfg.rank)
    img_host = torch.empty(frame.npix, 3, dtype=torch.float32).pin_memory()
    h2d = sum(host[k].numel() * host[k].element_size() for k in names)
    d2h = img_host.numel() * 4
    ws = W.Workspace()
    stream = torch.cuda.current_stream(dev)
    copy_stream = torch.cuda.Stream(dev)
    uploaded = [torch.cuda.Event(), torch.cuda.Event()]
    consumed = [torch.cuda.Event(), torch.cuda.Event()]

    def upload(i):
        b = i % 2
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(consumed[b])  # render i-2 has read this copy
            for k in names:
                devbufs[b][k].copy_(host[k], non_blocking=True)
            uploaded[b].record(copy_stream)

    def render(i):
        b = i % 2
        stream.wait_event(uploaded[b])
        W.render_band(f2s[b], rcfg, bufs=bufs, ws=ws)
        consumed[b].record(stream)
        img_host.copy_(bufs.output, non_blocking=True)

    def run(n):
        upload(0)
        for i in range(n):
            if i + 1 < n:
                upload(i + 1)
            render(i)

    for e in consumed:
        e.record(stream)
    run(max(1, min(args.warmup, 2)))
    torch.cuda.synchronize()
    if world > 1:
        pg.barrier()
    k = max(1, min(args.steps, 5))
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    copy_stream.wait_stream(stream)  # no upload starts before t0
    run(k)
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / k
    # the image read back to the host against the device-resident run's image
    diff = None
    if ref_image is not None:
        diff = float((img_host - ref_image.cpu()).abs().max()) if img_host.numel() else 0.0
    if world > 1:
        t = torch.tensor([ms], device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        ms = float(t[0])
    return {"value": frame.nfrag * world / (ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms, "steps": k,
            "image_max_abs_diff_vs_device_run": diff}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, choices=sorted(CONFIGS), default=2)
    ap.add_argument("--rank", type=int, default=None, help="override the config's rank (config 5 sweep)")
    ap.add_argument("--ref-rows", type=int, default=240, help="rows of the CPU sample")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per launch from an ncu --set full capture (profiles/)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    cfg = dict(CONFIGS[args.config])
    if args.rank is not None:
        if not 0 <= args.rank <= 6:
            raise SystemExit("--rank must be in 0..6")
        cfg["rank"] = args.rank
        cfg["name"] += f" (rank {args.rank}: {2 << args.rank} coefficients)"
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
