"""GPU parity: the sm_100a path through the C ABI against the oracle and the
reference-generated golden fixtures.

Tolerances (BASELINE.json north star, fp32 I/O):
  * near / far, z, slot and cell indices: bit-exact;
  * coefficients and per-fragment transmittance v̂: |err| <= 1e-5;
  * image RGB: |err| <= 1e-4;
  * kernel-level float64 API (build_into binned, interp, cells, total, packing):
    bit-exact against the reference's own outputs.
"""

import math

import numpy as np
import pytest
import torch

from oracle import woit_oracle as O
from tests import fixtures

pytestmark = pytest.mark.gpu

COEF_TOL = 1e-5
VHAT_TOL = 1e-5
IMG_TOL = 1e-4


@pytest.fixture(scope="module")
def W():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2201_00094_b200 as w

    w._lib.load()
    return w


def gpu_cfg(W, meta, **over):
    c = dict(meta["cfg"])
    c.update(over)
    return W.RenderConfig(method="wavelet", **c)


def camera_of(W, meta):
    cam = meta.get("camera")
    return W.Camera(**cam) if cam else W.Camera()


def oracle_on(sf, meta, **over):
    cfg = dict(meta["cfg"])
    cfg.update(over)
    cam = meta.get("camera")
    return O.render_frame(O.OFrame.from_synth(sf), O.OConfig(**cfg), O.OCamera(**cam) if cam else O.OCamera())


def render(W, sf, meta, **over):
    frame = W.FrameFragments.from_synth(sf)
    cfg = gpu_cfg(W, meta, **over)
    rays = W.camera_rays(camera_of(W, meta), cfg.width, cfg.height)
    full = frame.opaque_color.reshape(cfg.height, cfg.width, 3)
    bufs = W.render_band(frame, cfg, rays, full_opaque_image=full, vhat=True)
    torch.cuda.synchronize()
    return frame, bufs


def h(t):
    return t.detach().double().cpu().numpy()


def assert_close_to(bufs, ref, tag, coef_tol=COEF_TOL, vhat_tol=VHAT_TOL, img_tol=IMG_TOL):
    np.testing.assert_array_equal(h(bufs.near), ref.near.astype(np.float32).astype(np.float64), tag)
    np.testing.assert_array_equal(h(bufs.far), ref.far.astype(np.float32).astype(np.float64), tag)
    ce = np.abs(h(bufs.coeffs) - ref.coeffs).max(initial=0.0)
    ve = np.abs(h(bufs.vhat) - ref.vhat).max(initial=0.0)
    ie = np.abs(h(bufs.output) - ref.output).max(initial=0.0)
    assert ce <= coef_tol, f"{tag}: coeffs {ce:.3e}"
    assert ve <= vhat_tol, f"{tag}: vhat {ve:.3e}"
    assert ie <= img_tol, f"{tag}: image {ie:.3e}"
    return ce, ve, ie


# ---------------------------------------------------------------------------
# generator


@pytest.mark.parametrize("workload,w,hgt,layers", [("plane4", 64, 64, 5), ("smoke", 40, 24, 32),
                                                    ("particles", 16, 8, 128), ("ragged", 24, 20, 40),
                                                    ("smoke", 17, 9, 24)])
def test_device_generator_matches_numpy(W, workload, w, hgt, layers):
    dev = W.FrameFragments.synthetic(workload, w, hgt, seed=3, layers=layers).to_synth()
    host = W.synth.generate(workload, w, hgt, seed=3, layers=layers)
    for name in ("offsets", "depth", "alpha", "trans", "radiance", "normal", "ior", "backface",
                 "opaque_depth", "opaque_color"):
        np.testing.assert_array_equal(getattr(dev, name), getattr(host, name), name)


def test_device_generator_bands(W):
    full = W.synth.generate("ragged", 16, 12, seed=5, layers=30)
    band = W.FrameFragments.synthetic("ragged", 16, 12, seed=5, layers=30, row0=4, rows=5)
    lo, hi = full.offsets[4 * 16], full.offsets[9 * 16]
    assert band.frag_base == lo
    np.testing.assert_array_equal(band.depth.cpu().numpy(), full.depth[lo:hi])


# ---------------------------------------------------------------------------
# the fused frame against the reference's own outputs


@pytest.mark.parametrize("name", fixtures.names())
def test_render_matches_reference_fixture(W, name):
    meta, d = fixtures.load(name)
    sf = fixtures.input_stream(meta, d)
    frame, bufs = render(W, sf, meta)
    # oracle on the identical fp32 inputs
    ref = oracle_on(sf, meta)
    assert_close_to(bufs, ref, name)
    # and the reference's golden outputs directly (f64 inputs; the fp32 input
    # rounding of scene fixtures is inside the tolerances)
    np.testing.assert_array_equal(h(bufs.near), d["near"].astype(np.float32).astype(np.float64))
    assert np.abs(h(bufs.coeffs) - d["coeffs"]).max(initial=0) <= COEF_TOL
    assert np.abs(h(bufs.vhat) - d["vhat"]).max(initial=0) <= VHAT_TOL
    assert np.abs(h(bufs.output) - d["output"]).max(initial=0) <= IMG_TOL
    assert np.abs(h(bufs.accum) - d["accum"]).max(initial=0) <= IMG_TOL
    assert np.abs(h(bufs.accum_weight) - d["weight"]).max(initial=0) <= IMG_TOL
    assert np.abs(h(bufs.refraction_offset) - d["refr"]).max(initial=0) <= 1e-3


# scene fixtures' inputs are f64 (their fp32 rounding moves z), so z is compared
# bitwise on the synthetic, fp32-exact fixtures only
@pytest.mark.parametrize("name", fixtures.exact_names())
def test_z_and_indices_bit_exact(W, name):
    """z equals the reference's f64 z bitwise; k_n and (c0, c1) equal the oracle's."""
    meta, d = fixtures.load(name)
    sf = fixtures.input_stream(meta, d)
    frame = W.FrameFragments.from_synth(sf)
    rank = meta["cfg"]["rank"]
    bufs = W.FrameBuffers.allocate(frame, rank)
    W.step1_depth_bounds(frame, bufs)
    lib = W._lib.load()
    n = frame.nfrag
    z = torch.empty(n, dtype=torch.float64, device="cuda")
    k = torch.empty(n, rank + 1, dtype=torch.int32, device="cuda")
    c = torch.empty(n, 2, dtype=torch.int32, device="cuda")
    W._lib.check(lib.woit_fragment_indices(frame.c_struct(), bufs.near.data_ptr(), bufs.far.data_ptr(), rank,
                                           z.data_ptr(), k.data_ptr(), c.data_ptr(),
                                           torch.cuda.current_stream().cuda_stream), "indices")
    torch.cuda.synchronize()
    np.testing.assert_array_equal(z.cpu().numpy(), d["z"])
    np.testing.assert_array_equal(k.cpu().numpy(), O.slot_indices(d["z"], rank))
    c0, c1, _ = O.cell_indices(d["z"], rank)
    np.testing.assert_array_equal(c.cpu().numpy(), np.stack([c0, c1], axis=1))


# ---------------------------------------------------------------------------
# step-wise drop-in API


@pytest.mark.parametrize("name", ["plane4_64", "ragged_r3", "wine33_refr_ca_cube", "glass9_packed",
                                  "ragged_r6", "particles_256"])
def test_steps_match_reference(W, name):
    meta, d = fixtures.load(name)
    sf = fixtures.input_stream(meta, d)
    frame = W.FrameFragments.from_synth(sf)
    cfg = gpu_cfg(W, meta)
    rays = W.camera_rays(camera_of(W, meta), cfg.width, cfg.height)
    bufs = W.FrameBuffers.allocate(frame, cfg.rank, vhat=True)
    c = W.TouchCounter()
    W.step1_depth_bounds(frame, bufs)
    W.step2_build(frame, bufs, cfg, c)
    W.step3_accumulate(rays, frame, bufs, cfg, c)
    W.step4_composite(bufs, cfg, c, full_opaque_image=frame.opaque_color.reshape(cfg.height, cfg.width, 3))
    torch.cuda.synchronize()
    ref = oracle_on(sf, meta)
    assert_close_to(bufs, ref, name)
    assert c.per_insert == cfg.rank + 2 and c.per_eval == cfg.rank + 2
    # step2 and the fused build use the same reduction: identical coefficients
    fused = W.render_band(frame, cfg, rays, vhat=True)
    torch.cuda.synchronize()
    assert torch.equal(fused.coeffs, bufs.coeffs)
    assert torch.equal(fused.near, bufs.near)


def test_step1_accumulates_with_existing_bounds(W):
    sf = W.synth.generate("ragged", 8, 4, seed=2, layers=10)
    frame = W.FrameFragments.from_synth(sf)
    bufs = W.FrameBuffers.allocate(frame, 3)
    bufs.near.fill_(1.5)
    bufs.far.fill_(1.6)
    W.step1_depth_bounds(frame, bufs)
    ref = O.OBuffers.allocate(O.OFrame.from_synth(sf), 3)
    ref.near[:] = np.float32(1.5)
    ref.far[:] = np.float32(1.6)
    O.step1_depth_bounds(O.OFrame.from_synth(sf), ref)
    np.testing.assert_array_equal(h(bufs.near), ref.near)
    np.testing.assert_array_equal(h(bufs.far), ref.far)


# ---------------------------------------------------------------------------
# determinism and order independence


def test_band_split_is_bit_identical(W):
    """workers=1 vs workers=3 (test_pipeline.py:361-365): bitwise equal images."""
    sf = W.synth.generate("ragged", 37, 23, seed=11, layers=60)
    frame = W.FrameFragments.from_synth(sf)
    a = W.render_frame(None, W.RenderConfig(rank=3, width=37, height=23, workers=1), frame=frame)
    b = W.render_frame(None, W.RenderConfig(rank=3, width=37, height=23, workers=3), frame=frame)
    c = W.render_frame(None, W.RenderConfig(rank=3, width=37, height=23, workers=7), frame=frame)
    assert torch.equal(a, b) and torch.equal(a, c)


@pytest.mark.parametrize("workload,layers", [("ragged", 40), ("smoke", 32), ("particles", 128), ("ragged", 6)])
def test_band_needs_only_pixel_base(W, workload, layers):
    """A band built from host arrays (from_synth / from_numpy: pixel_base set, the
    informational frag_base left at 0, as the reference-side binding does) renders
    bit-identically to the same rows of the whole frame."""
    w, hgt, r0, rows = 40, 24, 7, 11
    whole = W.synth.generate(workload, w, hgt, seed=17, layers=layers)
    band = W.synth.generate(workload, w, hgt, seed=17, layers=layers, row0=r0, rows=rows)
    cfg = W.RenderConfig(rank=3, width=w, height=hgt)
    fw = W.FrameFragments.from_synth(whole)
    fb = W.FrameFragments.from_synth(band)
    assert fb.frag_base == 0 and fb.pixel_base == r0 * w
    a = W.render_band(fw, cfg, vhat=True)
    b = W.render_band(fb, cfg, vhat=True)
    torch.cuda.synchronize()
    p0, p1 = r0 * w, (r0 + rows) * w
    f0, f1 = int(whole.offsets[p0]), int(whole.offsets[p1])
    for name in ("coeffs", "output", "accum", "accum_weight", "near"):
        assert torch.equal(getattr(a, name)[p0:p1], getattr(b, name)), name
    assert torch.equal(a.vhat[f0:f1], b.vhat)


def test_concurrent_streams_without_shared_workspace(W):
    """Launches on two streams at once, each without an explicit workspace: the
    per-launch window counter / long list are not shared, results are exact."""
    frames = [W.FrameFragments.synthetic("ragged", 96, 64, seed=s, layers=300) for s in (31, 32)]
    cfg = W.RenderConfig(rank=3, width=96, height=64)
    want = [W.render_band(f, cfg) for f in frames]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [[], []]
    for _ in range(8):
        for i in (0, 1):
            with torch.cuda.stream(streams[i]):
                outs[i].append(W.render_band(frames[i], cfg))
    torch.cuda.synchronize()
    for i in (0, 1):
        for o in outs[i]:
            assert torch.equal(o.output, want[i].output) and torch.equal(o.coeffs, want[i].coeffs)


@pytest.mark.parametrize("layers", [6, 12, 128, 256])
def test_tiling_is_bit_identical(W, layers):
    """Ragged runs: shallow ones (thin sub-tiles, one pixel per lane, whose extent
    depends on where the windows fall) and deep ones (sub-tiles of one or two
    pixels). Band splits move the windows; the images, coefficients and v̂ must not
    change, and they match the oracle."""
    sf = W.synth.generate("ragged", 37, 23, seed=13, layers=layers)
    frame = W.FrameFragments.from_synth(sf)
    outs = [W.render_frame(None, W.RenderConfig(rank=3, width=37, height=23, workers=k), frame=frame)
            for k in (1, 3, 7)]
    assert all(torch.equal(outs[0], o) for o in outs[1:])
    cfg = W.RenderConfig(rank=3, width=37, height=23)
    full = W.render_band(frame, cfg, vhat=True)
    bands = [W.render_band(frame.band(p0, p1), cfg, vhat=True) for p0, p1 in ((0, 37 * 5), (37 * 5, 37 * 23))]
    torch.cuda.synchronize()
    for name in ("coeffs", "vhat"):
        assert torch.equal(getattr(full, name), torch.cat([getattr(b, name) for b in bands])), name
    ref = O.render_frame(O.OFrame.from_synth(sf), O.OConfig(rank=3, width=37, height=23))
    assert np.abs(h(full.coeffs) - ref.coeffs).max() <= 1e-5
    assert np.abs(h(full.vhat) - ref.vhat).max() <= 1e-5
    assert np.abs(h(full.output) - ref.output).max() <= 1e-4


def test_thin_and_deep_kernels_agree_bitwise(W):
    """Shallow frames (<= 16 fragments per pixel on average) launch the fast kernel
    with thin sub-tiles, deeper ones the instance without: a shallow band rendered
    alone (thin) equals the same rows of a deep frame (no thin), bit for bit."""
    w = 40
    top = W.synth.generate("ragged", w, 24, seed=21, layers=8, row0=0, rows=12)
    bot = W.synth.generate("particles", w, 24, seed=21, layers=64, row0=12, rows=12)
    cat = lambda a, b: np.concatenate([a, b])
    offs = cat(top.offsets[:-1], bot.offsets + top.offsets[-1])
    sf = W.synth.SynthFrame(w, 24, 0, 24, offs, *(cat(getattr(top, k), getattr(bot, k)) for k in (
        "depth", "alpha", "trans", "radiance", "normal", "ior", "backface", "opaque_depth", "opaque_color")))
    frame = W.FrameFragments.from_synth(sf)
    assert frame.nfrag > 16 * frame.npix and top.nfrag <= 16 * 12 * w
    cfg = W.RenderConfig(rank=3, width=w, height=24)
    full = W.render_band(frame, cfg, vhat=True)
    band = W.render_band(W.FrameFragments.from_synth(top), cfg, vhat=True)
    torch.cuda.synchronize()
    P, n = 12 * w, top.nfrag
    assert torch.equal(full.coeffs[:P], band.coeffs) and torch.equal(full.vhat[:n], band.vhat)
    assert torch.equal(full.output[:P], band.output) and torch.equal(full.near[:P], band.near)


def test_deep_and_plain_kernels_agree_bitwise(W):
    """Frames of > 160 fragments per pixel on average launch the fast kernel with the
    deep-pixel combine: a band of 256-fragment pixels rendered alone (deep instance)
    equals the same rows of a shallower frame (plain instance), bit for bit."""
    w = 24
    top = W.synth.generate("particles", w, 16, seed=22, layers=256, row0=0, rows=8)
    bot = W.synth.generate("ragged", w, 16, seed=22, layers=8, row0=8, rows=8)
    cat = lambda a, b: np.concatenate([a, b])
    offs = cat(top.offsets[:-1], bot.offsets + top.offsets[-1])
    sf = W.synth.SynthFrame(w, 16, 0, 16, offs, *(cat(getattr(top, k), getattr(bot, k)) for k in (
        "depth", "alpha", "trans", "radiance", "normal", "ior", "backface", "opaque_depth", "opaque_color")))
    frame = W.FrameFragments.from_synth(sf)
    assert 16 * frame.npix < frame.nfrag <= 160 * frame.npix and top.nfrag > 160 * 8 * w
    cfg = W.RenderConfig(rank=3, width=w, height=16)
    full = W.render_band(frame, cfg, vhat=True)
    band = W.render_band(W.FrameFragments.from_synth(top), cfg, vhat=True)
    torch.cuda.synchronize()
    P, n = 8 * w, top.nfrag
    assert torch.equal(full.coeffs[:P], band.coeffs) and torch.equal(full.vhat[:n], band.vhat)
    assert torch.equal(full.output[:P], band.output)
    ref = O.render_frame(O.OFrame.from_synth(top), O.OConfig(rank=3, width=w, height=8))
    assert np.abs(h(band.coeffs) - ref.coeffs).max() <= 1e-5
    assert np.abs(h(band.output) - ref.output).max() <= 1e-4


def test_repeat_runs_bit_identical(W):
    frame = W.FrameFragments.synthetic("particles", 64, 32, seed=4, layers=128)
    cfg = W.RenderConfig(rank=3, width=64, height=32)
    a = W.render_band(frame, cfg, vhat=True)
    b = W.render_band(frame, cfg, vhat=True)
    torch.cuda.synchronize()
    for name in ("coeffs", "vhat", "output", "accum"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name


def test_order_independence(W):
    """Shuffled within-pixel order: RMSE < 1e-5 (acceptance 04, test_pipeline.py:609-616)."""
    m1, d1 = fixtures.load("smokefire24")
    m2, d2 = fixtures.load("smokefire24_shuf7")
    _, b1 = render(W, fixtures.input_stream(m1, d1), m1)
    _, b2 = render(W, fixtures.input_stream(m2, d2), m2)
    rmse = math.sqrt(float(((h(b1.output) - h(b2.output)) ** 2).mean()))
    assert rmse < 1e-5
    assert np.abs(h(b1.coeffs) - h(b2.coeffs)).max() < 1e-6


# ---------------------------------------------------------------------------
# edge cases


def test_empty_frame(W):
    offsets = np.zeros(8 * 8 + 1, np.int64)
    frame = W.FrameFragments.from_numpy(8, 8, offsets, np.zeros(0), np.zeros(0), np.zeros((0, 3)),
                                        np.zeros((0, 3)), opaque_color=np.full((64, 3), 0.5))
    bufs = W.render_band(frame, W.RenderConfig(rank=3, width=8, height=8), vhat=True)
    torch.cuda.synchronize()
    assert torch.all(bufs.coeffs == 0)
    assert torch.all(bufs.output == 0.5)
    assert torch.all(torch.isinf(bufs.near)) and torch.all(bufs.near > 0)


@pytest.mark.parametrize("case", ["sparse", "sparse_long", "all_empty"])
def test_general_kernel_sparse_frames(W, case):
    """Sparse frames in the general kernel (refraction + aberration + cubed transmission):
    fewer fragments than pixels, so its windows are claimed heaviest-first (the
    window-order pre-pass); with a pixel deeper than a sub-tile (long-pixel kernel) and
    with no fragments at all. Against the oracle on the same fp32 inputs."""
    rng = np.random.default_rng({"sparse": 1, "sparse_long": 2, "all_empty": 3}[case])
    wd, ht = 96, 40
    P = wd * ht
    runs = np.zeros(P, np.int64)
    if case != "all_empty":
        hit = rng.choice(P, P // 12, replace=False)
        runs[hit] = rng.integers(1, 9, hit.size)
        if case == "sparse_long":
            runs[rng.integers(0, P)] = 700
    offsets = np.concatenate([[0], np.cumsum(runs)])
    n = int(offsets[-1])
    f = lambda *s: rng.uniform(0, 1, s).astype(np.float32)
    depth = rng.uniform(0.5, 3.0, n).astype(np.float32)
    nrm = rng.normal(size=(n, 3))
    nrm[:, 2] = -np.abs(nrm[:, 2]) - 0.5
    nrm = (nrm / np.linalg.norm(nrm, axis=1, keepdims=True)).astype(np.float32)
    ior = np.where(rng.uniform(0, 1, n) < 0.7, 1.5, 1.0).astype(np.float32)
    bf = (rng.uniform(0, 1, n) < 0.5).astype(np.uint8)
    od = np.where(rng.uniform(0, 1, P) < 0.8, 4.0, np.inf).astype(np.float32)
    oc = f(P, 3)
    args = (wd, ht, offsets, depth, (f(n) * 0.6).astype(np.float32), f(n, 3), f(n, 3), nrm, ior, bf, od, oc)
    flags = dict(refraction=True, chromatic_aberration=True, cube_transmission=True)
    frame = W.FrameFragments.from_numpy(*args)
    cfg = W.RenderConfig(rank=3, width=wd, height=ht, **flags)
    rays = W.camera_rays(W.Camera(), wd, ht)
    bufs = W.render_band(frame, cfg, rays, full_opaque_image=frame.opaque_color.reshape(ht, wd, 3), vhat=True)
    torch.cuda.synchronize()
    ref = O.render_frame(O.OFrame.from_arrays(*args), O.OConfig(rank=3, width=wd, height=ht, **flags), O.OCamera())
    assert_close_to(bufs, ref, case)
    np.testing.assert_allclose(h(bufs.refraction_offset), ref.refraction_offset, atol=1e-3)


@pytest.mark.parametrize("run", [2049, 5000, 20000])
def test_long_pixel_path(W, run):
    """Pixels deeper than one sub-tile go through the long-pixel kernel."""
    rng = np.random.default_rng(run)
    runs = np.array([3, run, 0, 7, run // 2], np.int64)
    offsets = np.concatenate([[0], np.cumsum(runs)])
    n = int(offsets[-1])
    depth = rng.uniform(0.5, 4.0, n).astype(np.float32)
    alpha = (rng.uniform(0, 1, n) * 0.05).astype(np.float32)
    trans = rng.uniform(0, 1, (n, 3)).astype(np.float32)
    rad = rng.uniform(0, 1, (n, 3)).astype(np.float32)
    oc = rng.uniform(0, 1, (5, 3)).astype(np.float32)
    frame = W.FrameFragments.from_numpy(5, 1, offsets, depth, alpha, trans, rad, opaque_color=oc)
    for rank in (0, 3, 6):
        bufs = W.render_band(frame, W.RenderConfig(rank=rank, width=5, height=1), vhat=True)
        torch.cuda.synchronize()
        ref = O.render_frame(O.OFrame.from_arrays(5, 1, offsets, depth, alpha, trans, rad, opaque_color=oc),
                             O.OConfig(rank=rank, width=5, height=1))
        assert_close_to(bufs, ref, f"long run={run} rank={rank}")


def test_misaligned_views_take_the_scalar_path(W):
    """A band view whose arrays are not 16-B aligned still renders identically."""
    sf = W.synth.generate("ragged", 16, 10, seed=8, layers=33)
    frame = W.FrameFragments.from_synth(sf)
    cfg = W.RenderConfig(rank=3, width=16, height=10)
    whole = W.render_band(frame, cfg, vhat=True)
    p0 = 3 * 16
    band = frame.band(p0, 10 * 16)
    part = W.render_band(band, cfg, vhat=True)
    torch.cuda.synchronize()
    assert torch.equal(part.output, whole.output[p0:])
    lo = int(sf.offsets[p0])
    assert torch.equal(part.vhat, whole.vhat[lo:])


def test_missing_library_fails_loudly(W, monkeypatch, tmp_path):
    monkeypatch.setattr(W._lib, "_lib", None)
    monkeypatch.setattr(W._lib, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(ImportError, match="no CPU fallback"):
        W._lib.load()


# ---------------------------------------------------------------------------
# kernel-level float64 API: bit-exact against the reference


def test_kernel_api_bit_exact(W):
    d = dict(np.load(fixtures.GOLDEN + "/kernels.npz"))
    rank = int(d["rank"])
    coeffs = np.zeros_like(d["coeffs"])
    c = W.TouchCounter()
    W.build_into(coeffs, d["pix"], d["z"], d["a"], rank, c)
    np.testing.assert_array_equal(coeffs, d["coeffs"])
    assert c.per_insert == rank + 2
    atomic = np.zeros_like(d["coeffs"])
    W.build_into(atomic, d["pix"], d["z"], d["a"], rank, mode="atomic")
    np.testing.assert_allclose(atomic, d["coeffs"], rtol=0, atol=1e-12)
    np.testing.assert_array_equal(W.interp_absorbance_batch(coeffs, d["qpix"], d["qz"], rank), d["interp"])
    np.testing.assert_array_equal(W.cells_raw_batch(coeffs, d["qpix"], d["cells"], rank), d["raw"])
    np.testing.assert_array_equal(W.total_absorbance_batch(coeffs, rank), d["total"])
    np.testing.assert_array_equal(W.pack_rgb9e5(d["triples"]), d["words"])
    np.testing.assert_array_equal(W.roundtrip_coeff_array(d["coeffs"]), d["packed_rt"])
    assert np.array_equal(W.unpack_rgb9e5(W.pack_rgb9e5([0.5, 0.25, 0.125])), [0.5, 0.25, 0.125])


def test_binning_bit_exact(W):
    rng = np.random.default_rng(5)
    P = 1000
    pix = rng.integers(0, P, 50000)
    offsets, perm = W.bin_by_pixel(pix, P)
    want_off = np.concatenate([[0], np.cumsum(np.bincount(pix, minlength=P))])
    np.testing.assert_array_equal(offsets.cpu().numpy(), want_off)
    np.testing.assert_array_equal(perm.cpu().numpy(), np.argsort(pix, kind="stable"))


# ---------------------------------------------------------------------------
# BASELINE config 2 at full size: size-independent properties + sampled parity


def test_config2_full_size_properties(W):
    frame = W.FrameFragments.synthetic("smoke", 1920, 1080, seed=1, layers=32)
    cfg = W.RenderConfig(rank=3, width=1920, height=1080)
    bufs = W.render_band(frame, cfg, vhat=True)
    torch.cuda.synchronize()
    assert torch.isfinite(bufs.output).all() and torch.isfinite(bufs.vhat).all()
    assert bool((bufs.vhat > 0).all()) and bool((bufs.vhat <= 1).all())
    # telescoping: exp(-A_total) equals the product of fragment transmittances
    # (test_pipeline.py:593-605), evaluated through the f64 kernel API
    a = -torch.log(torch.clamp(frame.net_transmittance(), min=1e-6))
    per_pix = torch.zeros(frame.npix, 3, dtype=torch.float64, device="cuda").index_add_(0, frame.pixel, a)
    tot = W.total_absorbance_batch(bufs.coeffs.double(), 3)
    assert float((torch.exp(-tot) - torch.exp(-per_pix)).abs().max()) < 1e-3
    # sampled pixels against the oracle (runs extracted from the full stream)
    host = frame.to_synth()
    rows = np.random.default_rng(0).choice(1080, 3, replace=False)
    for r in rows:
        sub = W.synth.generate("smoke", 1920, 1080, seed=1, layers=32, row0=int(r), rows=1)
        ref = O.render_frame(O.OFrame.from_synth(sub), O.OConfig(rank=3, width=1920, height=1),
                             workers=1)
        p0, p1 = int(r) * 1920, (int(r) + 1) * 1920
        f0, f1 = int(host.offsets[p0]), int(host.offsets[p1])
        assert np.abs(h(bufs.coeffs[p0:p1]) - ref.coeffs).max() <= COEF_TOL
        assert np.abs(h(bufs.vhat[f0:f1]) - ref.vhat).max() <= VHAT_TOL
        assert np.abs(h(bufs.accum[p0:p1]) - ref.accum).max() <= IMG_TOL
        assert np.abs(h(bufs.output[p0:p1]) - ref.output).max() <= IMG_TOL


@pytest.mark.parametrize("workload,w,hgt,layers", [("ragged", 61, 37, 40), ("smoke", 96, 64, 32), ("plane4", 300, 1, 5)])
def test_bin_frame_is_the_reference_csr(W, workload, w, hgt, layers):
    """woit_bin_frame on a shuffled (unbinned) stream: offsets = cumsum(bincount), the
    fields of each pixel in arrival order (np.argsort(kind="stable"), scene.py:559-566),
    and the render of the binned stream equals the render of the original CSR stream."""
    sf = W.synth.generate(workload, w, hgt, seed=9, layers=layers)
    frame = W.FrameFragments.from_synth(sf)
    n, P = frame.nfrag, frame.npix
    order = torch.randperm(n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3))
    pix = W.pixel_ids(frame)[order].contiguous()
    fb, perm = W.FrameFragments.from_unbinned(w, hgt, pix, frame.depth[order], frame.alpha[order],
                                              frame.trans[order], frame.radiance[order], frame.normal[order],
                                              frame.ior[order], frame.backface[order], frame.opaque_depth,
                                              frame.opaque_color, return_perm=True)
    torch.cuda.synchronize()
    p_np = pix.cpu().numpy()
    want_perm = np.argsort(p_np, kind="stable")
    np.testing.assert_array_equal(perm.cpu().numpy(), want_perm)
    np.testing.assert_array_equal(fb.offsets.cpu().numpy(),
                                  np.concatenate([[0], np.cumsum(np.bincount(p_np, minlength=P))]))
    for name in ("depth", "alpha", "trans", "radiance", "normal", "ior", "backface"):
        np.testing.assert_array_equal(getattr(fb, name).cpu().numpy(),
                                      getattr(frame, name)[order].cpu().numpy()[want_perm], name)
    cfg = W.RenderConfig(rank=3, width=w, height=hgt)
    a = W.render_band(frame, cfg)
    b = W.render_band(fb, cfg)
    torch.cuda.synchronize()
    # same fragments per pixel, a different within-pixel order: order independence
    assert float((a.output - b.output).abs().max()) < 1e-5


@pytest.mark.parametrize("case", ["layer_major_core", "deep_pixel", "sparse"])
def test_bin_frame_gather_paths(W, case):
    """The field gather's paths: a layer-major arrival without refraction fields (core
    fields only; the absent ones come back as the frame kernels' constants), a pixel
    deeper than the transposed path takes (slot-by-slot copy) beside multi-chunk and
    empty pixels, and a sparse frame (mostly empty tiles)."""
    g = torch.Generator(device="cuda").manual_seed(11)
    if case == "layer_major_core":
        P, L = 3000, 37
        pix = torch.arange(P, device="cuda", dtype=torch.int32).repeat(L)  # layer by layer
    elif case == "deep_pixel":
        P = 300
        pix = torch.cat([torch.full((5000,), 7, device="cuda", dtype=torch.int32),
                         torch.randint(0, P, (20000,), device="cuda", generator=g, dtype=torch.int32)])
        pix = pix[torch.randperm(pix.numel(), device="cuda", generator=g)].contiguous()
    else:
        P = 100_000
        pix = torch.randint(0, P // 50, (3000,), device="cuda", generator=g, dtype=torch.int32) * 50
    n = pix.numel()
    rnd = lambda *s: torch.rand(*s, device="cuda", generator=g)
    depth, alpha, trans, rad = rnd(n), rnd(n), rnd(n, 3), rnd(n, 3)
    refr = case != "layer_major_core"
    normal, ior = (rnd(n, 3), 1.0 + rnd(n)) if refr else (None, None)
    bf = (rnd(n) > 0.5).to(torch.uint8) if refr else None
    fb, perm = W.FrameFragments.from_unbinned(P, 1, pix, depth, alpha, trans, rad, normal, ior, bf, return_perm=True)
    torch.cuda.synchronize()
    p_np = pix.cpu().numpy()
    want = np.argsort(p_np, kind="stable")
    np.testing.assert_array_equal(perm.cpu().numpy(), want)
    np.testing.assert_array_equal(fb.offsets.cpu().numpy(), np.concatenate([[0], np.cumsum(np.bincount(p_np, minlength=P))]))
    src = dict(depth=depth, alpha=alpha, trans=trans, radiance=rad)
    if refr:
        src.update(normal=normal, ior=ior, backface=bf)
    for name, t in src.items():
        np.testing.assert_array_equal(getattr(fb, name).cpu().numpy(), t.cpu().numpy()[want], name)
    if not refr:
        assert bool((fb.normal == torch.tensor([0.0, 0.0, -1.0], device="cuda")).all())
        assert bool((fb.ior == 1.0).all()) and bool((fb.backface == 0).all())


@pytest.mark.parametrize("P,n", [(1, 1000), (256, 3), (257, 100000), (70000, 1 << 20), (2_073_600, 3_000_000)])
def test_binning_sizes(W, P, n):
    """Key widths of 0-21 bits (1-3 radix passes), tiny and ragged tiles, empty pixels."""
    rng = np.random.default_rng(P + n)
    pix = rng.integers(0, P, n)
    offsets, perm = W.bin_by_pixel(pix, P)
    np.testing.assert_array_equal(offsets.cpu().numpy(), np.concatenate([[0], np.cumsum(np.bincount(pix, minlength=P))]))
    np.testing.assert_array_equal(perm.cpu().numpy(), np.argsort(pix, kind="stable"))
