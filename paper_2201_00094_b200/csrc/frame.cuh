// Frame-path kernels: the fused four-pass compositor (bounds -> build -> eval
// -> composite) over CSR pixel tiles staged in shared memory by TMA bulk copies,
// plus the long-pixel kernel and the standalone composite kernel.
//
// Reference: pipeline.py:131-308 (steps 1-4), wavelet.py:272-337 (batch math).
// Design notes, smem layout and the roofline argument: DESIGN.md.
#pragma once

#include "common.cuh"
#include "packing.cuh"

#ifndef WOIT_WPB
#define WOIT_WPB 1
#endif

namespace woit {

// which passes a launch performs (the step entry points use subsets)
enum : uint32_t {
    PH_BOUNDS = 1u,       // near/far from the fragments (else read bufs->near/far)
    PH_BOUNDS_ACC = 2u,   // ... combined with the existing bufs->near/far (step1)
    PH_BUILD = 4u,        // coefficients from the fragments (else read bufs->coeffs)
    PH_BUILD_ACC = 8u,    // ... added to the existing bufs->coeffs (step2)
    PH_EVAL = 16u,        // v̂, accum, weight, refraction offset
    PH_EVAL_ACC = 32u,    // ... added to the existing bufs accumulators (step3)
    PH_COMPOSITE = 64u,   // output
};

// Aberration taps tabulated on the host (pipeline.py:226-239, 258-281): the
// spectral weights and positions depend only on (i, k, literal), so the kernels
// read them instead of recomputing three f64 divisions per tap per pixel.
constexpr int kMaxTapTable = 65;
struct TapTable {
    int32_t n;  // taps tabulated; 0 (k > kMaxTapTable): computed in the kernel
    int32_t unit;  // every weight exactly 0 or 1: a zero-offset gather is the pixel itself
    double fac[kMaxTapTable];   // 2 i / (k - 1)
    double w[kMaxTapTable][3];  // spectral_weight(i, k)
};

struct KParams {
    woit_frags_t f;
    woit_params_t p;
    woit_bufs_t b;
    uint32_t phases;
    int32_t use_tma;
    int64_t* long_list;  // [0] = count, [1..] = band-local pixel ids
    int64_t long_cap;
    unsigned long long* win_counter;  // dynamic window claims (zeroed per launch)
    unsigned* order_cnt;              // [2] window-order fill counters (zeroed per launch)
    int32_t* win_order;               // [nwin] claim order of the windows (fused general kernel)
    TapTable taps;
};

// per-rank warp-tile geometry
template <int R>
struct WT {
    static constexpr int S = 1 << (R + 1);   // coefficient slots (== cells M)
    static constexpr int V = 3 * S;          // values per pixel
    static constexpr int CH = 8;             // fragments per chunk (max)
    static constexpr int FBW = 32 * CH;      // fragments per warp sub-tile (max)
    static constexpr int WIN = 32;           // pixels per warp window
    static constexpr int SUBP = 8;           // pixels per sub-tile (3 SUBP <= 32 (pixel, channel) tasks)
    static constexpr int WPB = R <= 3 ? WOIT_WPB : 1;  // warps per CTA
    static constexpr int VR = V + ((35 - V % 32) % 32);  // row stride == 3 (mod 32), >= V
};

#ifndef WOIT_NRM_GLOBAL  // refraction normals read from global memory in the evaluation (not staged)
#define WOIT_NRM_GLOBAL 1
#endif

struct WLayout {
    uint32_t offs, cb, lo, den, rcp, vtot;
    uint32_t depth, alpha, trans, rad, ior, normal, bf, zfix, part, cells, coef32, accp, words, opq, bar, total;
};

WOIT_HD uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }

// Rows of the chunk partials (per-cell differences D_c). For R >= 1 the padded depth
// map (eval_bounds, pipeline.py:110-128) puts every fragment's z strictly inside
// [1/M, 1 - 1/M), so j_f = floor(M z) lies in [1, M-2]: D_0 and D_M are never touched
// and only cells 1..M-1 get a row (row c-1); v_0 = 0. Rank 0 keeps all M rows.
// (The step-wise entry points take the caller's bounds, so they keep every row.)
template <int R>
struct PartRows {
    WOIT_HD static constexpr int row0(bool tight) { return tight && R >= 1 ? 1 : 0; }  // first cell with a row
    WOIT_HD static constexpr int n(bool tight) { return (2 << R) - row0(tight); }
};

// shared-memory slice of one warp (bytes); the CTA holds WPB slices. alias_z (the fast
// path): the fixed-point z overwrites the staged depth in place (the build computes z
// and nothing reads the depth afterwards), every chunk lane derives its own depth map
// (no per-pixel map arrays), and exp(-A_total) lives in the reused partials region.
template <int R>
WOIT_HD WLayout make_wlayout(uint32_t phases, int flags, bool alias_z, bool gen) {
    using G = WT<R>;
    const bool at = phases & (PH_BUILD | PH_EVAL);
    const bool ev = phases & PH_EVAL;
    const bool need_ior = at && (flags & (WOIT_CUBE_TRANSMISSION | WOIT_REFRACTION));
    const bool need_bf = at && (flags & WOIT_CUBE_TRANSMISSION) && (flags & WOIT_CUBE_BACKFACE_ONLY);
    const bool need_nrm = !WOIT_NRM_GLOBAL && ev && (flags & WOIT_REFRACTION);
    const bool packed = (phases & PH_BUILD) && (flags & WOIT_PACKED_STORAGE);
    const uint32_t FS = G::FBW + 4;  // staging window: [fa & ~3, fb)
    WLayout L;
    uint32_t o = 0;
    L.offs = o;  o = align16(o + 4u * (G::WIN + 1));  // int32, relative to the window's first fragment
    L.cb = o;    o = align16(o + 2u * (G::WIN + 1));  // int16 chunk prefix (chunks of q = cb[q+1] - cb[q])
    // per sub-tile pixel (<= SUBP): depth maps and exp(-A_total) [SUBP][3] (general path)
    L.lo = L.den = L.rcp = L.vtot = o;
    if (!alias_z) {
        L.lo = o;    o = align16(o + 8u * G::SUBP);
        L.den = o;   o = align16(o + 8u * G::SUBP);
        L.rcp = o;   o = align16(o + 8u * G::SUBP);
        L.vtot = o;  o = align16(o + 4u * 3 * G::SUBP);
    }
    L.depth = o; o = align16(o + 4u * FS);
    L.alpha = o; o = align16(o + (at ? 4u * FS : 0u));
    L.trans = o; o = align16(o + (at ? 12u * FS : 0u));
    L.rad = o;   o = align16(o + (ev ? 12u * FS : 0u));
    L.ior = o;   o = align16(o + (need_ior ? 4u * FS : 0u));
    L.normal = o; o = align16(o + (need_nrm ? 12u * FS : 0u));
    L.bf = o;    o = align16(o + (need_bf ? (uint32_t)G::FBW + 32u : 0u));
    L.zfix = alias_z ? L.depth : o;
    o = align16(o + (at && !alias_z ? 4u * G::FBW : 0u));
    // one region, reused: chunk partials [rows][3][32] (per-cell differences D) during
    // the build, then the sub-tile's coefficients [SUBP][V], cell staircase (frame.cu
    // CellTab), chunk accumulators [6 or 9][32] and, on the fast path, exp(-A_total)
    const bool tight = phases == (PH_BOUNDS | PH_BUILD | PH_EVAL | PH_COMPOSITE);  // the fused render's own bounds
    const uint32_t part_b = (phases & PH_BUILD) ? 4u * 3 * 32 * PartRows<R>::n(tight) : 0u;
    const uint32_t cells_b = (uint32_t)G::SUBP * (G::S + 1) * 24u;  // frame.cu CellTab
    // chunk accumulators: acc / weight (6 rows), + refraction offset (2) and diffusion
    // coverage (1) in the general kernel; rows of 33 (frame.cu AR)
    const uint32_t acc_rows = !gen ? 6u : (flags & WOIT_DIFFUSION) ? 9u : 8u;
    const uint32_t acc_b = ev ? align16(4u * acc_rows * 33) : 0u;
    const uint32_t vtot_b = alias_z ? align16(4u * 3 * G::SUBP) : 0u;
    const uint32_t words_b = packed ? align16(4u * G::SUBP * G::S) : 0u;  // E5B9G9R9 words of the sub-tile
    const uint32_t after_b = align16(4u * G::SUBP * G::V) + align16(cells_b) + acc_b + vtot_b + words_b;
    L.part = o;  o = align16(o + (part_b > after_b ? part_b : after_b));
    L.coef32 = L.part;
    L.cells = L.part + align16(4u * G::SUBP * G::V);
    L.accp = L.cells + align16(cells_b);
    if (alias_z) L.vtot = L.accp + acc_b;
    L.words = L.accp + acc_b + vtot_b;
    L.opq = o;   o = align16(o + (gen ? 0u : 12u * (G::SUBP + 4)));  // fast path: [pa & ~3, pb rounded up to 4)
    L.bar = o;   o = align16(o + 16u);
#ifdef WOIT_SMEM_PAD
    o += WOIT_SMEM_PAD;
#endif
    L.total = align16(o);
    return L;
}

// ---------------------------------------------------------------------------
// composite of one pixel (pipeline.py:242-308)

// smoothstep / spectral_weight (pipeline.py:220-239) with explicit round-to-nearest
// operations (no FMA contraction), i.e. exactly the reference's f64 arithmetic. The
// host tabulates the same formulas (abi.cu fill_taps); this is the k > 65 fallback.
WOIT_HD double smoothstep_d(double e0, double e1, double x) {
#ifdef __CUDA_ARCH__
    double u = ddiv(dsub(x, e0), dsub(e1, e0));
    u = fmin(1.0, fmax(0.0, u));
    return dmul(dmul(u, u), dsub(3.0, dmul(2.0, u)));
#else
    volatile double d = e1 - e0;  // volatile: keep every rounding step
    double u = (x - e0) / d;
    u = u < 0.0 ? 0.0 : u;
    u = u > 1.0 ? 1.0 : u;
    volatile double uu = u * u;
    volatile double r = 3.0 - 2.0 * u;
    return uu * r;
#endif
}

WOIT_HD void spectral_weight(int i, int k, bool literal, double w[3]) {
#ifdef __CUDA_ARCH__
    const double q = ddiv(dmul(2.0, (double)i), (double)(k - 1));
    const double t = literal ? dadd(0.5, q) : ddiv((double)i, (double)(k - 1));
    const double wr = smoothstep_d(0.5, 1.0 / 3.0, t);
    const double wb = smoothstep_d(0.5, 2.0 / 3.0, t);
    w[0] = wr;
    w[1] = dsub(dsub(1.0, wr), wb);
    w[2] = wb;
#else
    const double t = literal ? 0.5 + 2.0 * i / (double)(k - 1) : i / (double)(k - 1);
    const double wr = smoothstep_d(0.5, 1.0 / 3.0, t);
    const double wb = smoothstep_d(0.5, 2.0 / 3.0, t);
    volatile double g = 1.0 - wr;
    w[0] = wr;
    w[1] = g - wb;
    w[2] = wb;
#endif
}

// column / row of global pixel gp in an image W wide: 32-bit division when the id
// fits (every image the ABI accepts: width * height < 2^31), 64-bit otherwise
WOIT_D void pixel_xy(int64_t gp, int W, double& px, double& py) {
    if ((uint64_t)gp <= 0xffffffffull) {
        const uint32_t g = (uint32_t)gp, w = (uint32_t)W, y = g / w;
        px = (double)(g - y * w);
        py = (double)y;
    } else {
        px = (double)(gp % W);
        py = (double)(gp / W);
    }
}

// bilinear_sample (pipeline.py:242-255): edge clamped, in f64
WOIT_D void bilinear(const float* __restrict__ img, int W, int H, double x, double y,
                     double out[3]) {
    x = fmin(fmax(x, 0.0), (double)W - 1.0);
    y = fmin(fmax(y, 0.0), (double)H - 1.0);
    const double fx = floor(x), fy = floor(y);
    const int x0 = (int)fx, y0 = (int)fy;
    const int x1 = min(x0 + 1, W - 1), y1 = min(y0 + 1, H - 1);
    const double tx = x - fx, ty = y - fy;
    const float* a = img + ((int64_t)y0 * W + x0) * 3;
    const float* b = img + ((int64_t)y0 * W + x1) * 3;
    const float* c = img + ((int64_t)y1 * W + x0) * 3;
    const float* d = img + ((int64_t)y1 * W + x1) * 3;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        const double top = dadd(dmul((double)a[ch], 1.0 - tx), dmul((double)b[ch], tx));
        const double bot = dadd(dmul((double)c[ch], 1.0 - tx), dmul((double)d[ch], tx));
        out[ch] = dadd(dmul(top, 1.0 - ty), dmul(bot, ty));
    }
}

// one channel of bilinear(): the same operations for that channel
WOIT_D double bilinear_ch(const float* __restrict__ img, int W, int H, double x, double y, int ch) {
    x = fmin(fmax(x, 0.0), (double)W - 1.0);
    y = fmin(fmax(y, 0.0), (double)H - 1.0);
    const double fx = floor(x), fy = floor(y);
    const int x0 = (int)fx, y0 = (int)fy;
    const int x1 = min(x0 + 1, W - 1), y1 = min(y0 + 1, H - 1);
    const double tx = x - fx, ty = y - fy;
    const double a = img[((int64_t)y0 * W + x0) * 3 + ch], b = img[((int64_t)y0 * W + x1) * 3 + ch];
    const double c = img[((int64_t)y1 * W + x0) * 3 + ch], d = img[((int64_t)y1 * W + x1) * 3 + ch];
    const double top = dadd(dmul(a, 1.0 - tx), dmul(b, tx));
    const double bot = dadd(dmul(c, 1.0 - tx), dmul(d, tx));
    return dadd(dmul(top, 1.0 - ty), dmul(bot, ty));
}

WOIT_D void tap(const TapTable& tt, int i, int k, bool lit, double& fac, double w[3]) {
    if (tt.n == k) {
        fac = tt.fac[i];
        w[0] = tt.w[i][0];
        w[1] = tt.w[i][1];
        w[2] = tt.w[i][2];
    } else {
        spectral_weight(i, k, lit, w);
        fac = ddiv(dmul(2.0, (double)i), (double)(k - 1));
    }
}

// Channel `ch` of the background of one pixel (pipeline.py:290-303); see sample_background.
// `self`, when not null, holds img[gp * 3 + ch] already loaded (a register prefetch).
WOIT_D double sample_background_ch(const float* img, int W, int H, int64_t gp, int flags, int taps,
                                   const TapTable& tt, double ox, double oy, int ch,
                                   const float* self = nullptr) {
    if (flags & (WOIT_CHROMATIC_ABERRATION | WOIT_REFRACTION)) {
        if (ox == 0.0 && oy == 0.0) {
            // every tap lands on the pixel itself, where the bilinear weights are exactly
            // (1, 0) and the sample is exactly the pixel: same arithmetic, no gathers
            const double s0 = self ? (double)*self : (double)img[gp * 3 + ch];
            // with 0/1 weights (k = 3, 5, 7) the sum is m s0 exactly (s0 is fp32-valued)
            // and m s0 / m == s0: the pixel itself, bit for bit
            if (!(flags & WOIT_CHROMATIC_ABERRATION) || (tt.n == taps && tt.unit)) return s0;
            const bool lit = flags & WOIT_LITERAL_SPECTRAL_T;
            double num = 0.0, den = 0.0;
            for (int i = 0; i < taps; ++i) {
                double w[3], fac;
                tap(tt, i, taps, lit, fac, w);
                num = dadd(num, dmul(w[ch], s0));
                den = dadd(den, w[ch]);
            }
            return den > 0.0 ? ddiv(num, den) : s0;
        }
        double px, py;
        pixel_xy(gp, W, px, py);
        if (flags & WOIT_CHROMATIC_ABERRATION) {
            const bool lit = flags & WOIT_LITERAL_SPECTRAL_T;
            double num = 0.0, den = 0.0;
            for (int i = 0; i < taps; ++i) {
                double w[3], fac;
                tap(tt, i, taps, lit, fac, w);
                if (w[ch] != 0.0)  // w s adds exactly 0 otherwise (s is finite)
                    num = dadd(num, dmul(w[ch], bilinear_ch(img, W, H, dadd(px, dmul(ox, fac)),
                                                            dadd(py, dmul(oy, fac)), ch)));
                den = dadd(den, w[ch]);
            }
            return den > 0.0 ? ddiv(num, den) : bilinear_ch(img, W, H, dadd(px, ox), dadd(py, oy), ch);
        }
        return bilinear_ch(img, W, H, dadd(px, ox), dadd(py, oy), ch);
    }
    return self ? (double)*self : (double)img[gp * 3 + ch];
}

// Background of one pixel read from `img` (pipeline.py:290-303): the k-tap aberration
// gather, a bilinear sample at the refracted position, or the pixel itself. `img` is
// [H][W][3] addressed by the pixel id gp (global with a full image, else band-local).
WOIT_D void sample_background(const float* img, int W, int H, int64_t gp, int flags, int taps,
                              const TapTable& tt, double ox, double oy, double bg[3],
                              const float* self = nullptr) {
    if (flags & (WOIT_CHROMATIC_ABERRATION | WOIT_REFRACTION)) {
        double px, py;
        pixel_xy(gp, W, px, py);
        if (ox == 0.0 && oy == 0.0 && (!(flags & WOIT_CHROMATIC_ABERRATION) || (tt.n == taps && tt.unit))) {
            // exact bilinear weights (1, 0) at the pixel, 0/1 tap weights: the pixel itself
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) bg[ch] = self ? (double)self[ch] : (double)img[gp * 3 + ch];
            return;
        }
        if (flags & WOIT_CHROMATIC_ABERRATION) {
            const bool lit = flags & WOIT_LITERAL_SPECTRAL_T;
            double num[3] = {0.0, 0.0, 0.0}, den[3] = {0.0, 0.0, 0.0};
            for (int i = 0; i < taps; ++i) {
                double w[3], s[3], fac;
                tap(tt, i, taps, lit, fac, w);
                bilinear(img, W, H, dadd(px, dmul(ox, fac)), dadd(py, dmul(oy, fac)), s);
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    num[ch] = dadd(num[ch], dmul(w[ch], s[ch]));
                    den[ch] = dadd(den[ch], w[ch]);
                }
            }
            double ctr[3];
            bilinear(img, W, H, dadd(px, ox), dadd(py, oy), ctr);
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) bg[ch] = den[ch] > 0.0 ? ddiv(num[ch], den[ch]) : ctr[ch];
        } else {
            bilinear(img, W, H, dadd(px, ox), dadd(py, oy), bg);
        }
    } else {
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) bg[ch] = self ? (double)self[ch] : (double)img[gp * 3 + ch];
    }
}

// Diffusion weight w = min(1, diffusion * D_p), D_p = sum alpha (r + g + b) / 3 (woit.h)
WOIT_D double diffusion_weight(const KParams& kp, double dp) {
    return fmin(1.0, dmul(kp.p.diffusion, dp));
}

// step4_composite for pixel p (band-local). accum/weight/refr are the pixel's
// final accumulators, vtot = exp(-A_total), dp the diffusion coverage D_p
// (only read with WOIT_DIFFUSION).
WOIT_D void composite_pixel(const KParams& kp, int flags, int64_t p, const double acc[3],
                            const double wgt[3], double ox, double oy, const double vtot[3],
                            double dp, float out[3], const float* self = nullptr) {
    const int W = kp.f.width;
    // flags: kp.p.flags, or a compile-time copy of them (specialised kernel instances)
    double bg[3];
    const bool gather = flags & (WOIT_CHROMATIC_ABERRATION | WOIT_REFRACTION);
    const bool full = kp.b.full_opaque_image != nullptr;
    // with a full image pixels are addressed globally; else the band is the image
    const int H = full ? kp.f.height : (int)(kp.f.npix / W);
    const int64_t gp = full ? kp.f.pixel_base + p : p;
    if (gather) {
        sample_background(full ? kp.b.full_opaque_image : kp.f.opaque_color, W, H, gp, flags,
                          kp.p.aberration_taps, kp.taps, ox, oy, bg, self);
    } else {
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) bg[ch] = self ? (double)self[ch] : (double)kp.f.opaque_color[p * 3 + ch];
    }
    if (flags & WOIT_DIFFUSION) {
        // K_resolve: lerp towards the same sample of the blurred background
        double bb[3];
        sample_background(kp.b.blurred_image, W, H, gp, flags, kp.p.aberration_taps, kp.taps, ox, oy, bb);
        const double w = diffusion_weight(kp, dp);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) bg[ch] = dadd(bg[ch], dmul(w, dsub(bb[ch], bg[ch])));
    }
    if (flags & WOIT_NORMALIZE) {
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            const double avg = ddiv(acc[ch], fmax(kNormEps, wgt[ch]));
            out[ch] = (float)dadd(dmul(avg, 1.0 - vtot[ch]), dmul(bg[ch], vtot[ch]));
        }
    } else {
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) out[ch] = (float)dadd(acc[ch], dmul(bg[ch], vtot[ch]));
    }
}

// composite without refraction or aberration: background = the pixel's opaque colour
WOIT_D void composite_plain(int flags, const float bgc[3], const double acc[3], const double wgt[3],
                            const double vtot[3], float out[3]) {
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        const double bg = (double)bgc[ch];
        if (flags & WOIT_NORMALIZE) {
            const double avg = acc[ch] * rcp_refined(fmax(kNormEps, wgt[ch]));
            out[ch] = (float)dadd(dmul(avg, 1.0 - vtot[ch]), dmul(bg, vtot[ch]));
        } else {
            out[ch] = (float)dadd(acc[ch], dmul(bg, vtot[ch]));
        }
    }
}

// Channel `ch` of composite_pixel, for per-(pixel, channel) lanes: the same
// operations, so the result is bit-identical to composite_pixel's channel. `self`:
// as in sample_background_ch (the pixel's own background value, prefetched), or null.
WOIT_D float composite_channel(const KParams& kp, int flags, int64_t p, int ch, double acc, double wgt, double ox,
                               double oy, double vt, double dp, const float* self = nullptr) {
    const int W = kp.f.width;
    // flags as in composite_pixel
    const bool gather = flags & (WOIT_CHROMATIC_ABERRATION | WOIT_REFRACTION);
    const bool full = kp.b.full_opaque_image != nullptr;
    const int H = full ? kp.f.height : (int)(kp.f.npix / W);
    const int64_t gp = full ? kp.f.pixel_base + p : p;
    double bg = gather ? sample_background_ch(full ? kp.b.full_opaque_image : kp.f.opaque_color, W, H, gp,
                                              flags, kp.p.aberration_taps, kp.taps, ox, oy, ch, self)
                       : (self ? (double)*self : (double)kp.f.opaque_color[p * 3 + ch]);
    if (flags & WOIT_DIFFUSION) {
        const double bb = sample_background_ch(kp.b.blurred_image, W, H, gp, flags, kp.p.aberration_taps,
                                               kp.taps, ox, oy, ch);
        bg = dadd(bg, dmul(diffusion_weight(kp, dp), dsub(bb, bg)));
    }
    if (flags & WOIT_NORMALIZE) {
        const double avg = ddiv(acc, fmax(kNormEps, wgt));
        return (float)dadd(dmul(avg, 1.0 - vt), dmul(bg, vt));
    }
    return (float)dadd(acc, dmul(bg, vt));
}

// Primary ray direction of global pixel gp (scene.py:199-212), f64.
WOIT_D void ray_dir(const KParams& kp, int64_t gp, double d[3]) {
    const int W = kp.f.width, H = kp.f.height;
    double px, py;
    pixel_xy(gp, W, px, py);
    const double u = dmul(dmul(dsub(ddiv(dmul(2.0, dadd(px, 0.5)), (double)W), 1.0), kp.p.tan_half),
                          kp.p.aspect);
    const double v = dmul(dsub(1.0, ddiv(dmul(2.0, dadd(py, 0.5)), (double)H)), kp.p.tan_half);
#pragma unroll
    for (int i = 0; i < 3; ++i)
        d[i] = dadd(dadd(kp.p.cam_forward[i], dmul(u, kp.p.cam_right[i])), dmul(v, kp.p.cam_up[i]));
    const double nrm = sqrt(dadd(dadd(dmul(d[0], d[0]), dmul(d[1], d[1])), dmul(d[2], d[2])));
#pragma unroll
    for (int i = 0; i < 3; ++i) d[i] = ddiv(d[i], nrm);
}

// Screen-space refraction offset of one ior>1 fragment (pipeline.py:189-217).
WOIT_D void refraction_offset(const KParams& kp, const double d[3], double t_opq, float depth,
                              const float nrm[3], float ior, double off[2]) {
    off[0] = 0.0;
    off[1] = 0.0;
    const double n0 = nrm[0], n1 = nrm[1], n2 = nrm[2];
    const double ci = -dadd(dadd(dmul(d[0], n0), dmul(d[1], n1)), dmul(d[2], n2));
    const double eta = ddiv(1.0, (double)ior);
    const double s2 = dmul(dmul(eta, eta), dsub(1.0, dmul(ci, ci)));
    bool ok = (ci > kDirEps) && (s2 <= 1.0) && isfinite(t_opq);
    const double root = sqrt(fmax(dsub(1.0, s2), 0.0));
    const double g = dsub(dmul(eta, ci), root);
    const double td0 = dadd(dmul(eta, d[0]), dmul(g, n0));
    const double td1 = dadd(dmul(eta, d[1]), dmul(g, n1));
    const double td2 = dadd(dmul(eta, d[2]), dmul(g, n2));
    const double* F = kp.p.cam_forward;
    const double tdf = dadd(dadd(dmul(td0, F[0]), dmul(td1, F[1])), dmul(td2, F[2]));
    const double dirf = dadd(dadd(dmul(d[0], F[0]), dmul(d[1], F[1])), dmul(d[2], F[2]));
    ok = ok && (tdf > kDirEps);
    if (!ok) return;
    const double x = depth;
    const double s = ddiv(dsub(dmul(t_opq, dirf), dmul(x, dirf)), tdf);
    const double w0 = dsub(dadd(dmul(x, d[0]), dmul(s, td0)), dmul(t_opq, d[0]));
    const double w1 = dsub(dadd(dmul(x, d[1]), dmul(s, td1)), dmul(t_opq, d[1]));
    const double w2 = dsub(dadd(dmul(x, d[2]), dmul(s, td2)), dmul(t_opq, d[2]));
    const double* Rv = kp.p.cam_right;
    const double* U = kp.p.cam_up;
    // W / 512 == W * 2^-9 exactly (an integer times a power of two): no f64 division
    const double scale = dmul(kp.p.refraction_scale, dmul((double)kp.f.width, 0x1p-9));
    const double ox = dmul(dadd(dadd(dmul(w0, Rv[0]), dmul(w1, Rv[1])), dmul(w2, Rv[2])), scale);
    const double oy = dmul(-dadd(dadd(dmul(w0, U[0]), dmul(w1, U[1])), dmul(w2, U[2])), scale);
    if (isfinite(ox) && isfinite(oy)) {
        off[0] = ox;
        off[1] = oy;
    }
}

}  // namespace woit
