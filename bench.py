"""Benchmark: Gfragments/s of the fused wavelet OIT frame (build + evaluate + composite).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2|4|5]

Workload (BASELINE.json configs[1], "config 2"): 1920x1080, 32 fragments/pixel
synthetic smoke volume, rank 3 (16 Haar slots), fp32 CSR stream generated on the
device (bit-identical to the numpy generator). One step = one full frame through
the fused kernel: bounds, closed-form Haar build, per-fragment transmittance v̂
(written, 12 B/fragment), visibility-weighted accumulation and composite (image
written). Inputs (2.1 GB) are larger than L2 (126 MB), so no flush is needed.

Multi-GPU: one process per GPU over NCCL. ``--gpus N`` without a torchrun
environment re-launches itself under ``torch.distributed.run`` with N ranks.
Config 2 scales weakly -- rank r renders rows [1080 r, 1080 (r+1)) of a
1920 x 1080N frame; the fp32 image bands are all-gathered inside the timed step,
time = max over ranks. Every run (any N) also carries ``config4_strong``: BASELINE
configs[3] (4K x 128 particles) split into N equal row bands (strong scaling,
the north star's >= 6x-at-8-GPUs target), with its 1-GPU time measured in the same
job on rank 0, the speed-up, and a bitwise check of the gathered image against
that 1-GPU render.

--impl reference times the reference's own CPU implementation
(``woit.pipeline.render_frame`` from baseline/_ref, installed by
tools/install_ref.sh; the pinned numpy port in oracle/ when that is absent) on
the host cores, on a bounded row band of the same workload per step.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)
REF_DIR = os.path.join(REPO, "baseline", "_ref")

METRIC = "Gfragments/s (build+eval+composite) and % HBM roofline at 1/2/4/8 B200 vs CPU"
UNIT = "Gfrag/s"
CPU_STEPS = 8        # cpu_baseline: 8 timed renders of the row band (~10-30 s of CPU work)
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


def algorithmic_bytes(npix: int, nfrag: int, rank: int, packed: bool = False) -> int:
    """44 B/fragment (depth, alpha, T, L in; v̂ out) +
    (32 + 12 S) B/pixel (offsets, opaque RGB in; coefficients, image out); with packed
    storage the coefficients leave as S E5B9G9R9 words: (32 + 4 S) B/pixel."""
    S = 1 << (rank + 1)
    return nfrag * 44 + npix * (32 + (4 if packed else 12) * S)


def scaled(cfg: dict, tiny: bool) -> dict:
    """--tiny (tests only): the same workload on an 8x smaller frame (each side)."""
    if not tiny:
        return cfg
    c = dict(cfg)
    c["width"] //= 8
    c["height"] //= 8
    c["name"] += " [tiny: 1/8 frame side, test mode]"
    return c


def geometry(cfg: dict, world: int):
    """(frame height, rows per rank) of the job at `world` GPUs."""
    if cfg.get("share"):
        if world > cfg["share"]:
            raise SystemExit(f"this config runs on at most {cfg['share']} GPUs")
        return cfg["height"], cfg["height"] // cfg["share"]
    if cfg.get("strong"):
        if cfg["height"] % world:
            raise SystemExit(f"strong scaling needs the GPU count to divide {cfg['height']} rows")
        return cfg["height"], cfg["height"] // world
    return cfg["height"] * world, cfg["height"]


def job_fragments(cfg: dict, world: int) -> int:
    from paper_2201_00094_b200 import synth

    frame_h, h1 = geometry(cfg, world)
    return int(sum(synth.run_lengths(cfg["workload"], cfg["width"], frame_h, cfg["seed"], cfg["layers"],
                                     h1 * r, h1).sum() for r in range(world)))


def config_dict(cfg: dict, world: int) -> dict:
    """The `config` object of the JSON line -- identical for both arms."""
    frame_h, h1 = geometry(cfg, world)
    n1 = job_fragments(cfg, 1) if world == 1 else None
    total = job_fragments(cfg, world)
    per_gpu = n1 if n1 is not None else total // world
    p1 = h1 * cfg["width"]
    in_bytes = per_gpu * 32 + (p1 + 1) * 8 + p1 * 12
    return {"workload": cfg["name"], "width": cfg["width"], "height": frame_h, "frag_per_px": cfg["layers"],
            "rank": cfg["rank"], "fragments": total,
            "l2_flush": f"none needed: inputs {in_bytes / 1e9:.1f} GB/GPU > 126 MB L2",
            "parallelism": (f"row bands x{world}, NCCL image all-gather" if world > 1 else "1 GPU")}


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


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_cmd(argv, gpus: int, port: int):
    """`python bench.py --gpus N ...` outside torchrun -> the torchrun command line."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(REPO, "bench.py"), *argv]


# ---------------------------------------------------------------------------
# the reference's CPU path


def host_info() -> dict:
    model = platform.processor() or ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"cpu_model": model, "numpy": np.__version__, "host_threads": os.cpu_count()}


def reference_available() -> bool:
    return os.path.isfile(os.path.join(REF_DIR, "woit", "pipeline.py"))


def cpu_reference(cfg, rows: int, steps: int, warmup: int):
    """Time the reference's CPU path on `rows` rows of the workload with all host
    threads: the reference itself (baseline/_ref: ``woit.pipeline.render_frame`` with
    ``workers = os.cpu_count()``) when installed, else the pinned
    numpy port (oracle/woit_oracle.py). Returns (Gfrag/s, threads, sample, s/step, kind)."""
    from paper_2201_00094_b200 import synth

    sf = synth.generate(cfg["workload"], cfg["width"], cfg["height"], seed=cfg["seed"], layers=cfg["layers"],
                        row0=0, rows=rows)
    workers = os.cpu_count() or 1
    if reference_available():
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        from woit import pipeline as rp
        from woit.scene import Camera, FrameFragments, Scene

        f64 = lambda a: np.asarray(a, dtype=np.float64)
        frame = FrameFragments(sf.width, sf.rows, sf.pixel_ids(), f64(sf.depth), f64(sf.alpha), f64(sf.trans),
                               f64(sf.radiance), f64(sf.normal), f64(sf.ior), sf.backface.astype(bool),
                               sf.offsets.copy(), f64(sf.opaque_depth), f64(sf.opaque_color))
        rcfg = rp.RenderConfig(method="wavelet", rank=cfg["rank"], width=cfg["width"], height=rows, workers=workers)
        scene = Scene(Camera(), ())
        run = lambda: rp.render_frame(scene, rcfg, frame=frame)
        kind, what = "reference", "woit.pipeline.render_frame (the reference, baseline/_ref)"
    else:
        from oracle import woit_oracle as O

        workers = O.default_workers()
        frame = O.OFrame.from_synth(sf)
        ocfg = O.OConfig(rank=cfg["rank"], width=cfg["width"], height=rows, workers=workers)
        run = lambda: O.render_frame(frame, ocfg, workers=workers)
        kind, what = "port", "float64 numpy port of the reference (oracle/)"
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        run()
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    n = sf.nfrag
    sample = f"{rows} rows x {cfg['width']} px x {cfg['layers']} frag/px = {n} fragments, {what}, {workers} threads"
    return n / float(np.mean(times)) / 1e9, workers, sample, float(np.mean(times)), kind


def run_reference(args, cfg):
    """The reference's CPU path on this arm's config and metric (rank 0 only). Every
    step renders a bounded row band of the frame, sized from a short pilot so that
    all W + K steps finish in about REF_BUDGET_S seconds."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    _, _, _, pilot_s, _ = cpu_reference(cfg, 16, 1, 0)
    rate = 16 * cfg["width"] * cfg["layers"] / pilot_s  # fragments/s
    total = max(1, args.steps + args.warmup)
    rows = int(REF_BUDGET_S * rate / (total * cfg["width"] * cfg["layers"]))
    rows = max(4, min(args.ref_rows, rows))
    value, cores, sample, secs, kind = cpu_reference(cfg, rows, args.steps, args.warmup)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs * 1e3,
            "higher_is_better": True, "scaling": "strong" if cfg.get("strong") else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_dict(cfg, world), "sample_rows": rows,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": sample + " per step", **host_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm


class Comm:
    """The few collectives the bench needs, over NCCL (GPUs) or gloo (tests: CPU
    copies, since gloo does not gather CUDA tensors)."""

    def __init__(self, world: int, backend: str, dev):
        import torch.distributed as dist

        self.dist, self.world, self.dev = dist, world, dev
        self.backend = backend
        if world > 1:
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=dev)
            else:
                dist.init_process_group("gloo")

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def gather(self, image, band):
        """image[world * P1] <- every rank's band[P1] (equal bands)."""
        if self.world == 1:
            return
        if self.backend == "nccl":
            self.dist.all_gather_into_tensor(image, band)
        else:
            parts = [band.new_empty(band.shape, device="cpu") for _ in range(self.world)]
            self.dist.all_gather(parts, band.cpu())
            image.copy_(__import__("torch").cat(parts))

    def max(self, *vals):
        import torch

        if self.world == 1:
            return [float(v) for v in vals]
        t = torch.tensor(vals, dtype=torch.float64, device=self.dev if self.backend == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return [float(v) for v in t.cpu()]

    def sum_int(self, v: int) -> int:
        import torch

        if self.world == 1:
            return int(v)
        t = torch.tensor([v], dtype=torch.int64, device=self.dev if self.backend == "nccl" else "cpu")
        self.dist.all_reduce(t)
        return int(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


class Renderer:
    """One band's device buffers and its woit_render_band launch (the C ABI)."""

    def __init__(self, W, lib, frame, rank_n: int, height: int, packed: bool = False):
        import torch

        self.lib, self.frame = lib, frame
        P, n = frame.npix, frame.nfrag
        S = 1 << (rank_n + 1)
        dev = frame.device
        # packed storage: the coefficients leave only as E5B9G9R9 words (4 S B/px)
        self.coeffs = None if packed else torch.empty(P, S, 3, dtype=torch.float32, device=dev)
        self.words = torch.empty(P, S, dtype=torch.int32, device=dev) if packed else None
        self.vhat = torch.empty(n, 3, dtype=torch.float32, device=dev)
        self.out = torch.empty(P, 3, dtype=torch.float32, device=dev)
        self.wsn = lib.woit_frame_workspace_bytes(P, n)
        self.ws = torch.empty(self.wsn, dtype=torch.uint8, device=dev)
        self.fs = frame.c_struct()
        self.ps = W.pipeline._params(W.RenderConfig(rank=rank_n, width=frame.width, height=height,
                                                    packed_storage=packed), rank_n)
        from paper_2201_00094_b200 import _lib

        self._lib = _lib
        self.bs = _lib.Bufs()
        self.bs.coeffs = self.coeffs.data_ptr() if self.coeffs is not None else None
        self.bs.coeff_words = self.words.data_ptr() if self.words is not None else None
        self.bs.vhat, self.bs.output = self.vhat.data_ptr(), self.out.data_ptr()

    def launch(self, stream):
        self._lib.check(self.lib.woit_render_band(self.fs, self.ps, self.bs, self.ws.data_ptr(), self.wsn,
                                                  stream.cuda_stream), "render_band")


def timed_steps(r: Renderer, comm: Comm, image, steps: int, warmup: int, stream, gather: bool = True):
    """W untimed + K timed steps (render, then gather when world > 1); returns
    (ms per step, mean kernel ms) on this rank, CUDA events on the launching stream."""
    import torch

    for _ in range(warmup):
        r.launch(stream)
        if gather:
            comm.gather(image, r.out)
    torch.cuda.synchronize()
    comm.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    kends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(steps):
        starts[i].record(stream)
        r.launch(stream)
        kends[i].record(stream)
        if gather:
            comm.gather(image, r.out)
    t1.record(stream)
    torch.cuda.synchronize()
    comm.barrier()
    return t0.elapsed_time(t1) / steps, float(np.mean([s.elapsed_time(k) for s, k in zip(starts, kends)]))


def strong_config4(args, W, lib, comm: Comm, rank: int, world: int, dev, stream) -> dict:
    """BASELINE configs[3] (4K x 128 particles, rank 3) as one frame split into
    `world` equal row bands: ms/step (render + NCCL image gather) max over ranks, the
    1-GPU time of the whole frame on rank 0 in the same job, and the gathered image
    compared bitwise with that 1-GPU render."""
    import torch

    c4 = scaled(CONFIGS[4], args.tiny)
    Wd, H = c4["width"], c4["height"]
    if H % world:
        return {"skipped": f"{world} GPUs do not divide {H} rows"}
    steps, warm = args.c4_steps, 3
    peak, _ = peaks()
    ms1 = kern1 = None
    img1 = None
    if rank == 0:
        full = W.FrameFragments.synthetic(c4["workload"], Wd, H, seed=c4["seed"], layers=c4["layers"], device=dev)
        r1 = Renderer(W, lib, full, c4["rank"], H)
        ms1, kern1 = timed_steps(r1, comm, None, steps, warm, stream, gather=False) if world == 1 else \
            _solo(r1, steps, warm, stream)
        img1 = r1.out.clone()
        n_full, p_full = full.nfrag, full.npix
        del r1, full
        torch.cuda.empty_cache()
    comm.barrier()
    if world == 1:
        ms, kern, n_job = ms1, kern1, n_full
        alg_per_gpu = algorithmic_bytes(p_full, n_full, c4["rank"])
        equal = True
    else:
        rows = H // world
        band = W.FrameFragments.synthetic(c4["workload"], Wd, H, seed=c4["seed"], layers=c4["layers"],
                                          row0=rows * rank, rows=rows, device=dev)
        rb = Renderer(W, lib, band, c4["rank"], H)
        image = torch.empty(world * band.npix, 3, dtype=torch.float32, device=dev)
        ms, kern = timed_steps(rb, comm, image, steps, warm, stream)
        ms, kern = comm.max(ms, kern)
        n_job = comm.sum_int(band.nfrag)
        alg_per_gpu = algorithmic_bytes(band.npix, band.nfrag, c4["rank"])
        equal = bool(torch.equal(image, img1)) if rank == 0 else None
        del rb, band, image
        torch.cuda.empty_cache()
    ms1 = comm.max(ms1 if ms1 is not None else 0.0)[0]
    achieved = alg_per_gpu / (kern * 1e-3) / 1e9
    return {"workload": c4["name"], "n_gpus": world, "steps": steps, "warmup": warm, "fragments": n_job,
            "ms_per_step": ms, "kernel_ms": kern, "value": n_job / (ms * 1e-3) / 1e9, "unit": UNIT,
            "roofline_frac_per_gpu": achieved / peak, "ms_per_step_1gpu": ms1,
            "speedup_vs_1gpu": ms1 / ms, "gathered_image_bitwise_equal_1gpu": equal,
            "scaling": "strong"}


def _solo(r: Renderer, steps: int, warm: int, stream):
    """Rank 0 alone (the other ranks wait at the barrier that follows)."""
    import torch

    for _ in range(warm):
        r.launch(stream)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        r.launch(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    return ms, ms


def run_ours(args, cfg):
    import torch

    import paper_2201_00094_b200 as W
    from paper_2201_00094_b200 import _lib

    rank, world, local = dist_env()
    if os.environ.get("WOIT_BENCH_ONE_DEVICE"):
        local = 0  # tests: every rank on the one GPU (gloo backend)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = Comm(world, args.backend, dev)
    Wd = cfg["width"]
    frame_h, H1 = geometry(cfg, world)
    frame = W.FrameFragments.synthetic(cfg["workload"], Wd, frame_h, seed=cfg["seed"], layers=cfg["layers"],
                                       row0=H1 * rank, rows=H1, device=dev)
    lib = _lib.load()
    r = Renderer(W, lib, frame, cfg["rank"], frame_h, packed=args.packed)
    P, n = frame.npix, frame.nfrag
    image = torch.empty(P * world, 3, dtype=torch.float32, device=dev) if world > 1 else r.out
    stream = torch.cuda.current_stream(dev)

    with ClockSampler(local) as clk:
        time.sleep(0.1)
        ms, kern_ms = timed_steps(r, comm, image, args.steps, args.warmup, stream)
    ms, kern_ms = comm.max(ms, kern_ms)
    frags_total = comm.sum_int(n)
    value = frags_total / (ms * 1e-3) / 1e9

    # end to end through the public API: pinned host stream -> device, render, image -> host
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, W, frame, W.RenderConfig(rank=cfg["rank"], width=Wd, height=frame_h,
                                                     packed_storage=args.packed), dev, world, comm, r.out)
    del r, image
    torch.cuda.empty_cache()
    c4 = None
    if not args.no_c4:
        c4 = strong_config4(args, W, lib, comm, rank, world, dev, stream)

    peak, peak_kind = peaks()
    if args.traffic is None and not args.packed:
        try:
            with open(os.path.join(REPO, "profiles", "traffic.json")) as f:
                tj = json.load(f)
            args.traffic = tj.get(f"config{args.config}_rank{cfg['rank']}", tj.get(f"config{args.config}"))
        except Exception:
            args.traffic = None
    alg = algorithmic_bytes(P, n, cfg["rank"], args.packed)
    achieved = alg / (kern_ms * 1e-3) / 1e9
    clocks = clk.summary()
    if rank != 0:
        comm.close()
        return
    conf = config_dict(cfg, world)
    assert conf["fragments"] == frags_total, (conf["fragments"], frags_total)
    cpu = None
    if world == 1 and not args.no_cpu:
        # a bounded sample: <= 14.7 M fragments (config 2: 240 rows)
        rows = max(1, min(args.ref_rows, 14745600 // (cfg["width"] * cfg["layers"])))
        v, cores, sample, secs, kind = cpu_reference(cfg, rows, CPU_STEPS, 1)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
               "sample": f"{sample}, 1 warm-up + {CPU_STEPS} timed renders ({CPU_STEPS * secs:.1f} s)",
               **host_info()}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if cfg.get("strong") else "weak",
        "vs_baseline": None, "dtype": "f32 (z, indices and per-pixel sums in f64)", "data": "synthetic",
        "config": conf,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": args.traffic,
                     "kernel": f"frame_kernel<{cfg['rank']}> (fused bounds+build+eval+composite)",
                     "kernel_ms": kern_ms, "algorithmic_bytes_per_launch": alg, "peak_kind": peak_kind},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": 2 * args.steps,
        "clocks": clocks,
        "config4_strong": c4,
    }
    print(json.dumps(line), flush=True)
    comm.close()


def run_e2e(args, W, frame, rcfg, dev, world, comm: Comm, ref_image=None):
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
    comm.barrier()
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
    ms = comm.max(ms)[0]
    return {"value": frame.nfrag * world / (ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms, "steps": k,
            "image_max_abs_diff_vs_device_run": diff}


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
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
    ap.add_argument("--no-c4", action="store_true", help="skip the config4_strong sub-record")
    ap.add_argument("--c4-steps", type=int, default=20, help="timed steps of the config4_strong sub-record")
    ap.add_argument("--backend", choices=("nccl", "gloo"), default="nccl",
                    help="process-group backend (gloo: tests running ranks on one GPU)")
    ap.add_argument("--tiny", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--packed", action="store_true",
                    help="E5B9G9R9 packed coefficient storage (4 S B/px words instead of fp32 coefficients)")
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per launch from an ncu --set full capture (profiles/)")
    args = ap.parse_args(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (127.0.0.1 rendezvous)
        r = subprocess.run(relaunch_cmd(argv, args.gpus, free_port()))
        raise SystemExit(r.returncode)
    _, world, _ = dist_env()
    if "WORLD_SIZE" in os.environ and args.gpus not in (1, world):
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    cfg = scaled(dict(CONFIGS[args.config]), args.tiny)
    if args.packed:
        cfg["name"] += " [packed E5B9G9R9 storage: coefficients as 4 S B/px words]"
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
