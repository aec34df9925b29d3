// Fused wavelet-OIT frame kernel (steps 1-4 of pipeline.py:131-308 in one pass
// over HBM) and its step-wise / long-pixel / composite companions.
//
// Work decomposition:
//   CTA      = a window of PB consecutive pixels of the band, split into
//              sub-tiles of <= FB fragments / <= T chunks;
//   chunk    = <= 8 consecutive fragments of ONE pixel, owned by one lane;
//   staging  = the sub-tile's fragment fields copied global->shared by TMA
//              bulk copies (cp.async.bulk + mbarrier), read once from HBM;
//   per-pixel reductions (bounds, coefficients, accumulators) combine the
//   chunk partials in a fixed order in fp64 -> deterministic for any tiling.
#include <mutex>
#include <utility>
#include <vector>

#include "frame.cuh"

#ifndef WOIT_UNROLL
#define WOIT_UNROLL 1
#endif
#ifndef WOIT_ZUNROLL
#define WOIT_ZUNROLL 8
#endif
#ifndef WOIT_ALIASZ  // fast path: fixed-point z stored over the staged depth
#define WOIT_ALIASZ 1
#endif
#ifndef WOIT_ZR_ON
#define WOIT_ZR_ON 1
#endif
#if WOIT_ZR_ON
#define WOIT_ZR __restrict__
#else
#define WOIT_ZR
#endif
#ifndef WOIT_DYN  // dynamic window claims
#define WOIT_DYN 1
#endif
#ifndef WOIT_EVPIPE  // software-pipelined evaluation loop (2: unrolled by two, no register copies)
#define WOIT_EVPIPE 2
#endif
#ifndef WOIT_MINB  // launch bound: minimum resident 1-warp CTAs per SM (14: <= 144 registers; ptxas then picks 127, measured best)
#define WOIT_MINB 14
#endif
#ifndef WOIT_THIN  // thin sub-tiles (one pixel per lane) for shallow pixel runs
#define WOIT_THIN 1
#endif
#ifndef WOIT_FLAG_INSTANCES  // general-kernel instances specialised for fixed flag sets
#define WOIT_FLAG_INSTANCES 1
#endif
#ifndef WOIT_GEN_FL_MINW  // resident warps per SM the flag-specialised general instances are compiled for
#define WOIT_GEN_FL_MINW 12
#endif
#ifndef WOIT_NRM_PREFETCH  // general kernel: L2 bulk prefetch of the sub-tile's normals
#define WOIT_NRM_PREFETCH 1
#endif
#ifndef WOIT_GEN_ORDER  // fused general kernel: windows with fragments claimed first
#define WOIT_GEN_ORDER 1
#endif
#ifndef WOIT_TAIL_SPLIT  // fast kernel: windows per warp claimed as half windows at the frame's end
#define WOIT_TAIL_SPLIT 2
#endif
#ifndef WOIT_GEN_ALIASZ  // fused general kernel: z over the staged depth (as the fast path)
#define WOIT_GEN_ALIASZ 1
#endif
#ifndef WOIT_GEN_DYN  // dynamic window claims in the general kernel
#define WOIT_GEN_DYN 1
#endif
#ifndef WOIT_GEN_PIPE  // pipelined window claims in the flag-specialised general instances
#define WOIT_GEN_PIPE 1
#endif
#ifndef WOIT_EMPTY_DIRECT  // empty pixels of the general kernel take the background directly
#define WOIT_EMPTY_DIRECT 1
#endif
#ifndef WOIT_PERSIST  // resident CTAs per SM slot multiplier for the persistent grid (0: one CTA per 2 windows)
#define WOIT_PERSIST 1
#endif
namespace woit {
// fast-kernel instances (frame_kernel VAR): plain, with thin sub-tiles, with the deep-pixel combine
constexpr int kVarPlain = 0, kVarThin = 1, kVarDeep = 2;
constexpr int kUnroll = WOIT_UNROLL;  // fragment-loop unroll (tuning knob)
constexpr int kZUnroll = WOIT_ZUNROLL;  // z-loop unroll
}

namespace woit {

// Within-chunk iteration starts at a rotation that depends only on the chunk's
// key = gpix * run + st (global pixel id, the pixel's run length, the chunk's first
// fragment within the pixel). For a uniform stream of L fragments per pixel the
// key is the global id of the chunk's first fragment, so lanes spread over the
// 32 smem banks; and as a function of (global pixel, run, chunk) only, the
// summation order -- hence every output bit -- is independent of the tiling and
// of how the frame is cut into bands (pixel_base is all a band needs to carry).
WOIT_D int chunk_rotation(int64_t key, int len) {
    const uint32_t g = (uint32_t)(key >> 5);
    return (int)(len == 8 ? (g & 7u) : g % (uint32_t)len);  // full chunks: no division
}
WOIT_D int64_t chunk_key(int64_t gpix, int run, int st) { return gpix * (int64_t)run + st; }


// ---------------------------------------------------------------------------
// staging: [fa, fb) of one array into shared memory at index (f - a), where a
// is fa rounded down to the array's 16-B granule. The 16-B aligned interior
// goes by one bulk copy (TMA); the < 1 granule tail at the end of the array,
// or everything when the base pointer is misaligned, goes by plain loads.

struct StageSpec {
    const void* g;    // global base (element 0)
    void* s;          // shared destination (element a)
    int esize;        // bytes per element
    int gran;         // elements per 16 B
};

WOIT_D int64_t stage_bulk_end(const StageSpec& sp, int64_t fa, int64_t fb, int64_t nalloc,
                              int use_tma, int64_t& a) {
    a = fa & ~(int64_t)(sp.gran - 1);
    if (!use_tma) return a;
    int64_t b = (fb + sp.gran - 1) & ~(int64_t)(sp.gran - 1);
    const int64_t bmax = nalloc & ~(int64_t)(sp.gran - 1);
    b = b < bmax ? b : bmax;
    return b > a ? b : a;
}

template <int T>
WOIT_D void stage_scalar(const StageSpec& sp, int64_t fa, int64_t fb, int64_t nalloc, int use_tma, int tid) {
    int64_t a;
    const int64_t e = stage_bulk_end(sp, fa, fb, nalloc, use_tma, a);
    const int64_t s0 = e > fa ? e : fa;
    const int words = sp.esize >= 4 ? sp.esize / 4 : 0;
    for (int64_t i = s0 + tid; i < fb; i += T) {
        if (words) {
            const float* g = static_cast<const float*>(sp.g) + i * words;
            float* d = static_cast<float*>(sp.s) + (i - a) * words;
            for (int w = 0; w < words; ++w) d[w] = g[w];
        } else {
            static_cast<uint8_t*>(sp.s)[i - a] = static_cast<const uint8_t*>(sp.g)[i];
        }
    }
}

// In-place inverse Haar synthesis of one channel: c[0..S) coefficients ->
// staircase value at each of the M = S cell centres (wavelet.py:221-239),
// level by level: cell(c) = c0 + sum_n 2^(n/2) (+/-) c[2^n + (c >> (N+1-n))].
template <int R>
WOIT_D void haar_cells(const double c[], double cell[]) {
    constexpr int S = 1 << (R + 1);
    cell[0] = c[0];
    int width = 1;  // number of distinct values after level n-1
#pragma unroll
    for (int n = 0; n <= R; ++n) {
        // each value splits into (v + s c, v - s c) with c = level-n offset k
#pragma unroll
        for (int k = (1 << n) - 1; k >= 0; --k) {
            const double v = cell[k];
            const double w = dmul(kSqrt2Pow[n], c[(1 << n) + k]);
            cell[2 * k] = dadd(v, w);
            cell[2 * k + 1] = dadd(v, -w);
        }
        width <<= 1;
    }
    (void)width;
    (void)S;
}

// cell table entry (v_c, v_{c+1} - v_c) for one (pixel, channel) of the sub-tile;
// pixel rows of CR float2 (CR == 3 mod 16) put the (pixel, channel) lanes on
// distinct banks
template <int M>
struct CellRow {
    static constexpr int CR = 3 * M + ((3 - 3 * M) % 16 + 16) % 16;
};

template <int M, typename TV>
WOIT_D void store_cells(float2* cells, int kq, int kch, const TV v[M]) {
#pragma unroll
    for (int c = 0; c < M; ++c) {
        const float vc = (float)v[c];
        const float dv = c + 1 < M ? (float)v[c + 1] - vc : 0.0f;
        cells[kq * CellRow<M>::CR + c * 3 + kch] = make_float2(vc, dv);
    }
}

// Fast-path chunk loops as functions with __restrict__ parameters: the compiler may
// then move the loads of later fragments above the shared-memory stores of earlier
// ones (the pointers provably do not alias), which it cannot do in the kernel body.
// Fragment part of the build: z (fused; stored for the evaluation over the staged
// depth), opacity alpha (1 - T) (stored in the T slot for the evaluation) and the
// absorbance a = -ln(max(1e-6, 1 - opacity)) per channel.
template <int R>
WOIT_D void build_prep(zfix_t* WOIT_ZR zf, const float* WOIT_ZR dep, const DepthMap& m,
                       const float* __restrict__ alp, float* __restrict__ trs, int fr, int si, zfix_t& zi,
                       float2& a01, float& a2) {
    zi = z_fixed_of(dep[si], m);
    zf[fr] = zi;
    const float al = alp[si];
    // channels 0 and 1 paired (bit-identical to the scalar sequence), channel 2 scalar
    const float2 one = make_float2(1.0f, 1.0f);
    const float2 T01 = make_float2(trs[3 * si], trs[3 * si + 1]);
    const float2 op01 = __fmul2_rn(make_float2(al, al), __fadd2_rn(one, make_float2(-T01.x, -T01.y)));
    const float op2 = opacity_ch(al, trs[3 * si + 2], false);
    trs[3 * si] = op01.x;  // the evaluation's weight 1 - t (pipeline.py:184)
    trs[3 * si + 1] = op01.y;
    trs[3 * si + 2] = op2;
    const float2 y01 = __fadd2_rn(one, make_float2(-op01.x, -op01.y));
    const float2 l01 = log_poly2(make_float2(fmaxf((float)kTransFloor, y01.x), fmaxf((float)kTransFloor, y01.y)));
    a01 = make_float2(-l01.x, -l01.y);
    a2 = -log_poly(fmaxf((float)kTransFloor, 1.0f - op2));
}

// Difference-array part: a (1 - w) to D_j, a w to D_{j+1} of this lane's partials
// column, j = floor(M z), w = M z - j. (Pairing red / green into FFMA2 updates
// measured 0.3% slower: same-box A/B.) Rows start at cell ROW0 (PartRows): with the
// fused render's own, tight bounds every j lies in [1, M-2] (the clamp changes
// nothing for finite depths and keeps NaN depths inside the region); the step-wise
// build (caller bounds, z may clip to 0 or 1 - 2^-24) keeps every row and drops D_M.
template <int R, int ROW0>
WOIT_D void d_update(float* __restrict__ part, int lane, zfix_t zi, float2 a01, float a2) {
    constexpr int M = 2 << R, WC = 32;
    int cell = (int)(zi >> (kZBits - (R + 1)));
    const float fr_ = u32_to_unit(zi << (R + 1), kZBits);  // M z - j_f
    const float w0 = 1.0f - fr_;
    if (ROW0) cell = min(max(cell, 1), M - 2);
    float* d = part + (cell - ROW0) * 3 * WC + lane;
    d[0] = fmaf(a01.x, w0, d[0]);
    d[WC] = fmaf(a01.y, w0, d[WC]);
    d[2 * WC] = fmaf(a2, w0, d[2 * WC]);
    if (ROW0 || cell + 1 < M) {
        float* d2 = d + 3 * WC;
        d2[0] = fmaf(a01.x, fr_, d2[0]);
        d2[WC] = fmaf(a01.y, fr_, d2[WC]);
        d2[2 * WC] = fmaf(a2, fr_, d2[2 * WC]);
    }
}

// The chunk loops visit fragment (crot + j) mod clen at step j. (Fully unrolled
// loops for full chunks measured 3.5% slower: code size. Software pipelining of
// this loop -- the next fragment's prep beside this one's updates -- measured 4%
// slower, and so did two fragments per step with paired fp32 ops across them
// (3%); the evaluation loop's pipelining pays.)
template <int R, int ROW0>
WOIT_D void build_chunk_fast(zfix_t* WOIT_ZR zf, const float* WOIT_ZR dep, const DepthMap m,
                             const float* __restrict__ alp, float* __restrict__ trs, float* __restrict__ part,
                             int lane, int cst, int clen, int crot, int sh4) {
    int jj = crot;
#pragma unroll kUnroll
    for (int j = 0; j < clen; ++j) {
        const int fr = cst + jj;
        jj = jj + 1 == clen ? 0 : jj + 1;
        zfix_t zi;
        float2 a01;
        float a2;
        build_prep<R>(zf, dep, m, alp, trs, fr, sh4 + fr, zi, a01, a2);
        d_update<R, ROW0>(part, lane, zi, a01, a2);
    }
}

// Cell pair (v_c, v_{c+1} - v_c) for the evaluation. CellsPair reads the per-sub-tile
// table store_cells wrote; CellsCol (thin sub-tiles) reads the lane's own staircase
// column in the partials region and forms the difference the same way (fp32 v_{c+1} -
// v_c; 0 for the last cell, where the evaluation's lerp weight is 0 anyway).
struct CellsPair {
    const float2* __restrict__ cq2;
    WOIT_D float2 get(int c0, int ch) const { return cq2[c0 * 3 + ch]; }
};
template <int M, int ROW0>
struct CellsCol {
    const float* __restrict__ col;  // part + lane: row stride 3 x 32 floats per cell, from cell ROW0
    WOIT_D float v(int c, int ch) const { return c < ROW0 ? 0.0f : col[(c - ROW0) * 96 + ch * 32]; }
    WOIT_D float2 get(int c0, int ch) const {
        const float v0 = v(c0, ch);
        const int c1 = c0 + 1 < M ? c0 + 1 : c0;
        return make_float2(v0, v(c1, ch) - v0);
    }
};

// t / n for 0 <= t < 32 and 1 <= n <= 8 (the (pixel, channel) lane split of a
// sub-tile) by a multiply-shift: with m = ceil(256 / n), t m / 256 exceeds t / n by
// less than 1/8, and t / n's fraction is at most 7/8, so the floor is exact.
__constant__ uint32_t kDivMagic8[9] = {0u, 256u, 128u, 86u, 64u, 52u, 43u, 37u, 32u};
WOIT_D int div_small(int t, int n) { return (int)(((uint32_t)t * kDivMagic8[n]) >> 8); }

// kSqrt2Pow[n] / 2^(R+1) as a compile-time constant (the same literals as kSqrt2Pow)
template <int R>
WOIT_D constexpr double kSqrt2PowOverM(int n) {
    return (n == 0 ? 1.0 : n == 1 ? 1.4142135623730951 : n == 2 ? 2.0 : n == 3 ? 2.8284271247461903
            : n == 4 ? 4.0 : n == 5 ? 5.656854249492381 : 8.0) / (double)(2 << R);
}

// Haar analysis of the staircase (cell averages T[0..M)) in f64, wavelet.py:3-9
// layout: c[2^n + k] = 2^(n/2)/M (sum left half - sum right half), c[0] = mean.
// T is consumed.
template <int R>
WOIT_D void haar_analysis(double T[], double c[]) {
    constexpr int M = 2 << R;
#pragma unroll
    for (int m = 0; m <= R; ++m) {
        const int half = M >> (m + 1);  // wavelets at level n = R - m
#pragma unroll
        for (int k = 0; k < half; ++k) {
            const double x = T[2 * k], y = T[2 * k + 1];
            // (x - y) 2^((R-m)/2) / M in one rounding: 1/M is a power of two, so
            // RN(RN(d s) / M) == RN(d (s / M)) (no underflow at these magnitudes)
            c[half + k] = dmul(dsub(x, y), kSqrt2PowOverM<R>(R - m));
            T[k] = dadd(x, y);
        }
    }
    c[0] = dmul(T[0], 1.0 / M);
}

// Composite of one channel on the fast path (no refraction / aberration: the
// background is the pixel's opaque colour), pipeline.py:284-308.
WOIT_D float composite_fast_ch(int flags, double acc, double wgt, double bg, double vt) {
    if (flags & WOIT_NORMALIZE) {
        const double avg = acc * rcp_refined(fmax(kNormEps, wgt));
        return (float)dadd(dmul(avg, 1.0 - vt), dmul(bg, vt));
    }
    return (float)dadd(acc, dmul(bg, vt));
}

template <int R>
WOIT_D void eval_frag(const zfix_t* __restrict__ zf, const float* __restrict__ alp, const float* __restrict__ opw,
                      const float2* __restrict__ cq2, float* __restrict__ rad, int fr, int si, float ac[3],
                      float wg[3]) {
    int c0;
    float t;
    eval_cell(zf[fr], R, c0, t);
    const float2* cv = cq2 + c0 * 3;
    const float al = alp[si];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        const float2 vd = cv[ch];
        const float A = fmaxf(fmaf(t, vd.y, vd.x), 0.0f);
        const float vh = exp_neg(A);
        ac[ch] += (rad[3 * si + ch] * al) * vh;
        wg[ch] += opw[3 * si + ch] * vh;
        rad[3 * si + ch] = vh;  // v̂ replaces radiance in place
    }
}

template <int R, typename CELLS>
WOIT_D void eval_chunk_fast(const zfix_t* __restrict__ zf, const float* __restrict__ alp,
                            const float* __restrict__ opw, const CELLS cq2,
                            float* __restrict__ rad, int cst, int clen, int crot, int sh4, float ac[3],
                            float wg[3]) {
#if WOIT_EVPIPE == 2
    // software-pipelined and unrolled by two: two operand sets alternate, so the
    // pipeline needs no register copies (same visiting and summation order)
    if (clen <= 0) return;
    struct Ops {
        float al, t, L[3], op[3];
        float2 vd[3];
        int si;
    };
    auto load = [&](int jj, Ops& o) {
        const int fr = cst + jj;
        o.si = sh4 + fr;
        o.al = alp[o.si];
        int c0;
        eval_cell(zf[fr], R, c0, o.t);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            o.L[ch] = rad[3 * o.si + ch];
            o.op[ch] = opw[3 * o.si + ch];
            o.vd[ch] = cq2.get(c0, ch);
        }
    };
    auto step = [&](const Ops& o) {
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            const float A = fmaxf(fmaf(o.t, o.vd[ch].y, o.vd[ch].x), 0.0f);
            const float vh = exp_neg(A);
            ac[ch] += (o.L[ch] * o.al) * vh;
            wg[ch] += o.op[ch] * vh;
            rad[3 * o.si + ch] = vh;  // v̂ replaces radiance in place
        }
    };
    auto nxt = [&](int jj) { return jj + 1 == clen ? 0 : jj + 1; };
    Ops a, b;
    int ja = crot;
    load(ja, a);
#pragma unroll 1
    for (int j = 0; j < clen; j += 2) {
        const int jb = nxt(ja);
        load(jb, b);  // wrap-around prefetch past the last fragment: discarded
        step(a);
        if (j + 1 >= clen) break;
        ja = nxt(jb);
        load(ja, a);
        step(b);
    }
#elif WOIT_EVPIPE
    // software-pipelined: the next fragment's operands -- and, at depth 2, its cell
    // pair -- are loaded before this fragment's v̂ stores (different fragments, so
    // no hazard; the wrap-around prefetch after the last fragment is discarded)
    if (clen <= 0) return;
    int jj = crot;
    int fr = cst + jj;
    float al = alp[sh4 + fr];
    float L[3], op[3];
    float2 vd[3];
    float t;
    {
        int c0;
        eval_cell(zf[fr], R, c0, t);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            L[ch] = rad[3 * (sh4 + fr) + ch];
            op[ch] = opw[3 * (sh4 + fr) + ch];
            vd[ch] = cq2.get(c0, ch);
        }
    }
#pragma unroll 1
    for (int j = 0; j < clen; ++j) {
        const int si = sh4 + fr;
        const int jn = jj + 1 == clen ? 0 : jj + 1;
        const int frn = cst + jn, sin = sh4 + frn;
        const float aln = alp[sin];
        float Ln[3], opn[3], tn;
        float2 vdn[3];
        int cn;
        eval_cell(zf[frn], R, cn, tn);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            Ln[ch] = rad[3 * sin + ch];
            opn[ch] = opw[3 * sin + ch];
            vdn[ch] = cq2.get(cn, ch);
        }
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            const float A = fmaxf(fmaf(t, vd[ch].y, vd[ch].x), 0.0f);
            const float vh = exp_neg(A);
            ac[ch] += (L[ch] * al) * vh;
            wg[ch] += op[ch] * vh;
            rad[3 * si + ch] = vh;  // v̂ replaces radiance in place
        }
        jj = jn;
        fr = frn;
        al = aln;
        t = tn;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            L[ch] = Ln[ch];
            op[ch] = opn[ch];
            vd[ch] = vdn[ch];
        }
    }
#else
    int jj = crot;
#pragma unroll kUnroll
    for (int j = 0; j < clen; ++j) {
        const int fr = cst + jj;
        jj = jj + 1 == clen ? 0 : jj + 1;
        eval_frag<R>(zf, alp, opw, cq2.cq2, rad, fr, sh4 + fr, ac, wg);
    }
#endif
}

// ---------------------------------------------------------------------------
// The fused frame kernel. Every warp owns a window of WIN consecutive pixels and
// processes it in sub-tiles of <= 32 chunks (<= 256 fragments) on its own slice
// of shared memory, synchronising only with __syncwarp and its own mbarrier, so
// warps never wait on each other. GEN=false is the compile-time fast path of the
// fused frame without refraction / aberration / cubed transmission / packed
// storage (the headline configuration); GEN=true covers every flag and the
// step-wise entry points.

// A run of `ne` fragment-free pixels starting at band pixel p0, in the fused frame:
// lane l finishes pixel p0 + l with the values the full phases would produce for
// an empty pixel -- bounds (+inf, -inf), zero coefficients (packed: slot 0 +0,
// the others -0, as the E5B9G9R9 round trip of 0), zero accumulators and offset,
// and the composite with acc = wgt = 0, v_tot = 1, offset 0, D = 0, i.e. the
// background itself -- without staging, chunks or the per-(pixel, channel) phases.
template <int R, bool GEN>
WOIT_D void empty_run(const KParams& kp, int flags, int64_t p0, int ne, int lane, const float* self = nullptr) {
    constexpr int V = 3 * (2 << R);
    if (kp.b.coeffs) {
        float* c = kp.b.coeffs + p0 * V;
        const bool packed = flags & WOIT_PACKED_STORAGE;
        if (V % 4 == 0 && (reinterpret_cast<uintptr_t>(c) & 15u) == 0) {
            constexpr int V4 = V / 4 > 0 ? V / 4 : 1;
            float4* c4 = reinterpret_cast<float4*>(c);
            if (packed) {
                for (int i = lane; i < ne * V4; i += 32) {
                    const float l0 = (i % V4) == 0 ? 0.0f : -0.0f;
                    c4[i] = make_float4(l0, l0, l0, -0.0f);
                }
            } else {
                for (int i = lane; i < ne * V4; i += 32) c4[i] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            }
        } else {
            for (int i = lane; i < ne * V; i += 32) c[i] = (packed && (i % V) >= 3) ? -0.0f : 0.0f;
        }
    }
    if ((flags & WOIT_PACKED_STORAGE) && kp.b.coeff_words) {
        constexpr int S = 2 << R;  // E5B9G9R9 of zeros: word 0
        for (int i = lane; i < ne * S; i += 32) kp.b.coeff_words[p0 * S + i] = 0u;
    }
    if (lane >= ne) return;
    const int64_t p = p0 + lane;
    if (kp.b.near) kp.b.near[p] = INFINITY;
    if (kp.b.far) kp.b.far[p] = -INFINITY;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        if (kp.b.accum) kp.b.accum[p * 3 + ch] = 0.0f;
        if (kp.b.weight) kp.b.weight[p * 3 + ch] = 0.0f;
    }
    if (kp.b.refraction_offset) {
        kp.b.refraction_offset[p * 2] = 0.0f;
        kp.b.refraction_offset[p * 2 + 1] = 0.0f;
    }
    if (GEN && (flags & WOIT_DIFFUSION) && kp.b.diffusion) kp.b.diffusion[p] = 0.0f;
    if (kp.b.output) {
        // no fragments: v_tot = 1, acc = wgt = 0 and a zero refraction offset, so the
        // composite returns the background sample exactly -- the pixel's own colour
        // (the full image's at its global id when refraction / aberration gather from
        // it, whose zero-offset sample is the pixel itself for 0/1 tap weights)
        const bool gather = flags & (WOIT_CHROMATIC_ABERRATION | WOIT_REFRACTION);
        const bool direct = !GEN || (WOIT_EMPTY_DIRECT && !(flags & WOIT_DIFFUSION) &&
                                     (!(flags & WOIT_CHROMATIC_ABERRATION) ||
                                      (kp.taps.n == kp.p.aberration_taps && kp.taps.unit)));
        if (direct) {
            const bool full = GEN && gather && kp.b.full_opaque_image;
            const float* img = full ? kp.b.full_opaque_image + (kp.f.pixel_base + p) * 3 : kp.f.opaque_color + p * 3;
            const float r = self ? self[0] : img[0], g = self ? self[1] : img[1], b = self ? self[2] : img[2];
            kp.b.output[p * 3] = r;
            kp.b.output[p * 3 + 1] = g;
            kp.b.output[p * 3 + 2] = b;
        } else {
#pragma unroll
            for (int ch = 0; ch < 3; ++ch)
                kp.b.output[p * 3 + ch] =
                    composite_channel(kp, flags, p, ch, 0.0, 0.0, 0.0, 0.0, 1.0, 0.0, self ? self + ch : nullptr);
        }
    }
}

template <int R, bool GEN>
struct WSmem {
    int32_t* offs;     // [WIN+1] window CSR offsets, relative to the window's first fragment
    int16_t* cb;       // [WIN+1] window chunk prefix (chunks per pixel capped at WC + 1)
    double* lo;        // [SUBP]  depth map (general path; fast-path chunk lanes keep theirs in registers)
    double* den;
    double* rcp;
    float* vtot;       // [SUBP][3] exp(-A_total) (an fp32 expf result, so fp32 holds it exactly)
    float* depth;      // staging [FBW+4] (granule-aligned window)
    float* alpha;
    float* trans;      // [FBW+4][3]
    float* rad;        // [FBW+4][3], v̂ written in place
    float* ior;
    float* normal;
    uint8_t* bf;
    zfix_t* zfix;      // [FBW] z in fixed point, by fragment
    float* part;       // [rows][3][32] chunk partials
    float2* cells;     // [SUBP][M][3] (v_c, v_{c+1} - v_c): staircase at cell centres
    float* coef32;     // [WIN][V] coefficients, bulk-stored to bufs->coeffs
    float* accp;       // [8][32] chunk accumulators
    uint32_t* words;   // [SUBP][S] E5B9G9R9 words of the sub-tile (packed storage)
    float* opq;        // [SUBP+4][3] staged opaque colours of the sub-tile (fast path)
    uint64_t* bar;
};

template <int R, bool GEN>
WOIT_D WSmem<R, GEN> wcarve(unsigned char* base, const WLayout& L) {
    WSmem<R, GEN> s;
    s.offs = reinterpret_cast<int32_t*>(base + L.offs);
    s.cb = reinterpret_cast<int16_t*>(base + L.cb);
    s.lo = reinterpret_cast<double*>(base + L.lo);
    s.den = reinterpret_cast<double*>(base + L.den);
    s.rcp = reinterpret_cast<double*>(base + L.rcp);
    s.vtot = reinterpret_cast<float*>(base + L.vtot);
    s.depth = reinterpret_cast<float*>(base + L.depth);
    s.alpha = reinterpret_cast<float*>(base + L.alpha);
    s.trans = reinterpret_cast<float*>(base + L.trans);
    s.rad = reinterpret_cast<float*>(base + L.rad);
    s.ior = reinterpret_cast<float*>(base + L.ior);
    s.normal = reinterpret_cast<float*>(base + L.normal);
    s.bf = reinterpret_cast<uint8_t*>(base + L.bf);
    s.zfix = reinterpret_cast<zfix_t*>(base + L.zfix);
    s.part = reinterpret_cast<float*>(base + L.part);
    s.cells = reinterpret_cast<float2*>(base + L.cells);
    s.coef32 = reinterpret_cast<float*>(base + L.coef32);
    s.accp = reinterpret_cast<float*>(base + L.accp);
    s.words = reinterpret_cast<uint32_t*>(base + L.words);
    s.opq = reinterpret_cast<float*>(base + L.opq);
    s.bar = reinterpret_cast<uint64_t*>(base + L.bar);
    return s;
}

// FUS: the phases are the fused render's (compile-time constant), so the
// step-wise accumulate / from-buffer branches compile out; GEN && !FUS serves the
// step1..step4 entry points.
// Minimum resident warps per SM the fast instances are compiled for (the register cap):
// rank <= 3 hold 15 warps by shared memory; ranks 4-6 fewer (their partials and cell
// tables are larger), so their register budget is looser and they do not spill.
template <int R>
constexpr int kMinWarps() { return R <= 3 ? WOIT_MINB : R == 4 ? 10 : R == 5 ? 6 : 4; }

template <int R, bool GEN, bool FUS, int VAR, int FL>
__global__ void __launch_bounds__(WT<R>::WPB * 32, (GEN ? (FL != 0 ? WOIT_GEN_FL_MINW : 12) : kMinWarps<R>()) / WT<R>::WPB) frame_kernel(const __grid_constant__ KParams kp) {
    using G = WT<R>;
    constexpr int S = G::S, V = G::V, CH = G::CH, WC = 32, FBW = G::FBW, WIN = G::WIN, SUBP = G::SUBP;
    constexpr int AR = WC + 1;  // chunk-accumulator row stride: the (pixel, channel) combine lanes hit distinct banks
    constexpr int M = S;       // cells
    constexpr uint32_t kFused = PH_BOUNDS | PH_BUILD | PH_EVAL | PH_COMPOSITE;
    // partials rows start at cell kRow0 (PartRows): 1 when the bounds are the fused
    // render's own (every j in [1, M-2]), 0 for the step-wise entry points
    constexpr int kRow0 = PartRows<R>::row0(FUS), kPRows = M - kRow0;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t ph = (GEN && !FUS) ? kp.phases : kFused;
    // FL != 0: an instance specialised for exactly these flags (all but NORMALIZE)
    // (the fast path's FL is WOIT_PACKED_STORAGE for its packed-storage instance, else 0)
    const int flags = GEN ? (FL ? (FL | (kp.p.flags & WOIT_NORMALIZE)) : kp.p.flags) : ((kp.p.flags & WOIT_NORMALIZE) | FL);
    // z in place of the staged depth: the fast path, and the fused general kernel (whose
    // refraction then reads the fragment's depth from global memory, next to its normal)
    constexpr bool kAliasZ = WOIT_ALIASZ && (!GEN || (FUS && WOIT_GEN_ALIASZ));
    const WLayout L = make_wlayout<R>(ph, flags, kAliasZ, GEN);
    const int lane = threadIdx.x & 31;
    WSmem<R, GEN> sm = wcarve<R, GEN>(smem_raw + (threadIdx.x >> 5) * L.total, L);

    // persistent warps: the first window is the warp id, later ones are claimed from
    // a global counter (dynamic: the SM sub-partitions hold unequal warp counts and
    // windows unequal work). The next window's CSR offsets are prefetched into
    // registers while the current one is processed.
    const int64_t nwin = (kp.f.npix + WIN - 1) / WIN;
    const int64_t nwarps = (int64_t)gridDim.x * G::WPB;
    // Fused general kernel: windows are claimed in the order of kp.win_order (those
    // with fragments first, window_order_kernel), so the frame ends on empty windows
    // instead of its heaviest ones
    const int32_t* worder = (GEN && FUS && WOIT_GEN_ORDER) ? kp.win_order : nullptr;
    auto wmap = [&](int64_t t) -> int64_t { return (worder && t < nwin) ? (int64_t)worder[t] : t; };
    // Tail split (fast kernel): the frame's last WOIT_TAIL_SPLIT windows per warp are
    // claimed as half windows (WIN / 2 pixels), so the warps' last units -- whose end
    // the frame waits for -- are half as long. A unit u < u1 is window u; the rest are
    // the half windows from pixel u1 WIN on. (Pixel results do not depend on the
    // tiling: chunk order is keyed on the global pixel.)
    constexpr int HALF = WIN / 2;
    const int64_t u1 = (!GEN && WOIT_TAIL_SPLIT > 0)
                           ? (nwin > WOIT_TAIL_SPLIT * nwarps ? nwin - WOIT_TAIL_SPLIT * nwarps : 0) : nwin;
    const int64_t nunit = u1 + (u1 < nwin ? (kp.f.npix - u1 * WIN + HALF - 1) / HALF : 0);
    auto ustart = [&](int64_t u) -> int64_t { return u < u1 ? u * WIN : u1 * WIN + (u - u1) * HALF; };
    auto uend = [&](int64_t u) -> int64_t {
        const int64_t e = ustart(u) + (u < u1 ? WIN : HALF);
        return e < kp.f.npix ? e : kp.f.npix;
    };
    int64_t win = (int64_t)blockIdx.x * G::WPB + (threadIdx.x >> 5);
    if (win >= nunit) return;  // warp-uniform
    win = wmap(win);
    // The claims are pipelined one window deep: the atomic for the window after next
    // is issued while the next window's id (claimed one window earlier) is consumed,
    // so its round trip is hidden behind a window of work. (Deeper -- two claims in
    // flight, or runs of 2-8 windows per claim, also after the ordering below --
    // measured slower on config 3.)
    // (Fast kernel only: in the general kernel it measured slower -- the extra live
    // register spills in the generic instance, costs occupancy in the specialised ones.)
#if WOIT_DYN
    unsigned long long claim_raw = 0;
    constexpr bool kPipeClaims = !GEN || (WOIT_GEN_PIPE && FL != 0);
    if (kPipeClaims && lane == 0) claim_raw = atomicAdd(kp.win_counter, 1ull);
#endif
    auto claim = [&]() -> int64_t {
#if WOIT_DYN
        if (GEN && !WOIT_GEN_DYN) return win + nwarps;
        if (!kPipeClaims) {
            unsigned long long c = 0;
            if (lane == 0) c = atomicAdd(kp.win_counter, 1ull);
            return wmap(nwarps + (int64_t)__shfl_sync(0xffffffffu, c, 0));
        }
        const int64_t c = nwarps + (int64_t)__shfl_sync(0xffffffffu, claim_raw, 0);
        if (lane == 0) claim_raw = atomicAdd(kp.win_counter, 1ull);
        return wmap(c);
#else
        return win + nwarps;
#endif
    };

    const bool do_at = ph & (PH_BUILD | PH_EVAL);
    const bool do_eval = ph & PH_EVAL;
    const bool refr_pf = GEN && (flags & WOIT_REFRACTION);
    const bool need_coef = ph & (PH_EVAL | PH_COMPOSITE);
    const bool refr = GEN && do_eval && (flags & WOIT_REFRACTION);
    const bool diffuse = GEN && (flags & WOIT_DIFFUSION);
    const bool cube = GEN && (flags & WOIT_CUBE_TRANSMISSION);
    const bool bfonly = cube && (flags & WOIT_CUBE_BACKFACE_ONLY);
    const bool need_ior = do_at && (cube || refr);
    const bool packed = flags & WOIT_PACKED_STORAGE;
    const int64_t nalloc = kp.f.nfrag;
    // thin sub-tiles: the fused render without packed storage, when the coefficient
    // transpose ([V][33] floats) fits over the depth / alpha / T / L staging arrays
    const bool kThinOK = VAR == kVarThin && FUS && !packed && V * 33 * 4 <= (int)(L.rad - L.depth) + 12 * (FBW + 4);

    if (lane == 0) mbar_init(sm.bar, 1);
    uint32_t parity = 0;
    int64_t off_lane = 0, off_last;  // this window's offsets[lane] and offsets[end]
    // General fused kernel: lane l's pixel of the next window -- its own background
    // value (what an empty or unrefracted pixel composites over: the full image's
    // pixel when refraction / aberration gather from it, else its opaque colour) and
    // its opaque depth -- is prefetched into registers with the window's offsets, so
    // empty pixels and the refraction setup do not wait on those loads.
    constexpr bool kPF = GEN && FUS;
    const float* bgimg = ((flags & (WOIT_CHROMATIC_ABERRATION | WOIT_REFRACTION)) && kp.b.full_opaque_image)
                             ? kp.b.full_opaque_image + kp.f.pixel_base * 3 : kp.f.opaque_color;
    float pf_bg[3] = {0.0f, 0.0f, 0.0f}, pf_od = INFINITY;
    auto prefetch_px = [&](int64_t px0, int64_t pend) {
        if (kPF && px0 + lane < pend) {
            const int64_t pp = px0 + lane;
            pf_bg[0] = bgimg[pp * 3];
            pf_bg[1] = bgimg[pp * 3 + 1];
            pf_bg[2] = bgimg[pp * 3 + 2];
            if (refr_pf && kp.f.opaque_depth) pf_od = kp.f.opaque_depth[pp];
        }
    };
    {
        const int64_t s0 = ustart(win), end = uend(win);
        if (s0 + lane < end) off_lane = kp.f.offsets[s0 + lane];
        off_last = kp.f.offsets[end];
        prefetch_px(s0, end);
    }
    // Fast path: a sub-tile's composite (phase 7) is deferred until the next
    // sub-tile's staging copies are in flight, so it hides part of their latency.
    // It only reads the per-window chunk prefix, the chunk accumulators, v_tot and
    // the staged opaque colours (taken into a register before the next copies).
    bool pend = false;
    int pq0 = 0, pnqs = 0;
    int64_t pw0 = 0;
    auto composite_fast = [&](int cq0, int cnqs, int64_t cw0, float bgr) {
        if (lane >= 3 * cnqs) return;
        const int kch = div_small(lane, cnqs), kq = lane - kch * cnqs;
        const int q = cq0 + kq;
        const int64_t p = cw0 + q;
        const int nc = (sm.cb[q + 1] - sm.cb[q]);
        const int cbq = sm.cb[q] - sm.cb[cq0];
        double acc = 0.0, wgt = 0.0;
        for (int i = 0; i < nc; ++i) {
            acc += (double)sm.accp[kch * AR + cbq + i];
            wgt += (double)sm.accp[(3 + kch) * AR + cbq + i];
        }
        if (kp.b.accum) kp.b.accum[p * 3 + kch] = (float)acc;
        if (kp.b.weight) kp.b.weight[p * 3 + kch] = (float)wgt;
        if (kp.b.output) kp.b.output[p * 3 + kch] = composite_fast_ch(flags, acc, wgt, (double)bgr, (double)sm.vtot[kq * 3 + kch]);
        if (kch == 0 && kp.b.refraction_offset) {
            kp.b.refraction_offset[p * 2] = 0.0f;
            kp.b.refraction_offset[p * 2 + 1] = 0.0f;
        }
    };
    // this lane's opaque colour of the pending composite, from the staged copy
    auto pending_bg = [&]() -> float {
        if (!pend || lane >= 3 * pnqs || !kp.b.output) return 0.0f;
        const int kch = div_small(lane, pnqs), kq = lane - kch * pnqs;
        const int si = (int)(pw0 + pq0 + kq - ((pw0 + pq0) & ~(int64_t)3));
        return sm.opq[3 * si + kch];
    };
    auto flush = [&]() {
        if (!GEN && pend) {
            composite_fast(pq0, pnqs, pw0, pending_bg());
            pend = false;
            __syncwarp();
        }
    };
    int64_t eg_fa = 0;  // the current sub-tile's first fragment (for eval_gen)
    // general-path evaluation of one chunk (step 3, pipeline.py:170-217): v̂, the
    // accumulators, the diffusion coverage and the refraction offsets; `cells` is the
    // sub-tile's cell table (CellsPair) or the lane's staircase column (CellsCol)
    auto eval_gen = [&](auto cells, int cst, int clen, int crot, const double d[3], double topq, float ac[3],
                        float wg[3], float& df, double ro[2]) {
        const int64_t fa_ = eg_fa;
        const int sh4 = (int)(fa_ - (fa_ & ~(int64_t)3)), shb = (int)(fa_ - (fa_ & ~(int64_t)15));
        const bool op_staged = ph & PH_BUILD;  // the build left alpha (1 - T') in the trans slot
        int jj = crot;
#pragma unroll kUnroll
        for (int j = 0; j < clen; ++j) {
            const int fr = cst + jj;
            jj = jj + 1 == clen ? 0 : jj + 1;
            const int si = sh4 + fr;
            int c0;
            float t;
            eval_cell(sm.zfix[(kAliasZ ? sh4 : 0) + fr], R, c0, t);
            const float al = sm.alpha[si];
            bool cb_ = false;
            float io = 1.0f;
            if (need_ior) {
                io = sm.ior[si];
                cb_ = cube && io > 1.0f && (!bfonly || sm.bf[shb + fr] != 0);
            }
            float vs = 0.0f;
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                // A = lerp of the two neighbouring cell centres, clamped >= 0 (wavelet.py:316-319)
                const float2 vd = cells.get(c0, ch);
                const float A = fmaxf(fmaf(t, vd.y, vd.x), 0.0f);
                const float vh = exp_neg(A);
                const float Lr = sm.rad[3 * si + ch];
                const float op = op_staged ? sm.trans[3 * si + ch] : opacity_ch(al, sm.trans[3 * si + ch], cb_);
                ac[ch] += (Lr * al) * vh;
                wg[ch] += op * vh;
                vs += vh;
                sm.rad[3 * si + ch] = vh;  // v̂ replaces radiance in place
            }
            if (diffuse) df += al * vs;  // diffusion coverage (woit.h WOIT_DIFFUSION)
            if (refr && io > 1.0f) {
#if WOIT_NRM_GLOBAL
                const float* gn = kp.f.normal + 3 * (fa_ + fr);
                const float nrm[3] = {gn[0], gn[1], gn[2]};
#else
                const float nrm[3] = {sm.normal[3 * si], sm.normal[3 * si + 1], sm.normal[3 * si + 2]};
#endif
                double off[2];
                // (with z over the staged depth, the depth comes from global memory)
                refraction_offset(kp, d, topq, kAliasZ ? kp.f.depth[fa_ + fr] : sm.depth[si], nrm, io, off);
                ro[0] += off[0];
                ro[1] += off[1];
            }
        }
    };
    int64_t next_win = nunit;
    for (; win < nunit; win = next_win) {
    flush();  // the pending composite reads this window's chunk prefix
    const int64_t w0 = ustart(win);
    const int nq = (int)(uend(win) - w0);
    // the window's offsets relative to its first fragment (int32: a window of WIN
    // pixels holds < 2^31 fragments, include/woit.h)
    const int64_t wbase = __shfl_sync(0xffffffffu, off_lane, 0);
    if (off_last - wbase > (int64_t)0x7fffffff) __trap();
    if (lane < nq) sm.offs[lane] = (int32_t)(off_lane - wbase);
    if (lane == 0) sm.offs[nq] = (int32_t)(off_last - wbase);
    // this window's prefetched per-pixel values (lane l: pixel w0 + l)
    const float cur_bg0 = pf_bg[0], cur_bg1 = pf_bg[1], cur_bg2 = pf_bg[2], cur_od = pf_od;
    {   // prefetch the next window's offsets (consumed one window later)
        const int64_t nw = claim();
        next_win = nw;
        if (nw < nunit) {
            const int64_t nw0 = ustart(nw);
            const int64_t nend = uend(nw);
            if (nw0 + lane < nend) off_lane = kp.f.offsets[nw0 + lane];
            off_last = kp.f.offsets[nend];
            prefetch_px(nw0, nend);
        }
    }
    // pixel q's prefetched values (all lanes take part in the shuffles)
    auto self_bg = [&](int q, float out[3]) {
        out[0] = __shfl_sync(0xffffffffu, cur_bg0, q & 31);
        out[1] = __shfl_sync(0xffffffffu, cur_bg1, q & 31);
        out[2] = __shfl_sync(0xffffffffu, cur_bg2, q & 31);
    };
    __syncwarp();
    // chunks per pixel, window prefix (warp scan) and combine rotation
    int my_nch = 0;
    // any fragment-free pixel in this window? (enables the empty-run shortcut below)
    const bool any_empty = __any_sync(0xffffffffu, lane < nq && sm.offs[lane + 1] == sm.offs[lane]);
    if (lane < nq) {
        const int run = sm.offs[lane + 1] - sm.offs[lane];
        const int nc = (int)(((unsigned)run + CH - 1) / CH);
        // a pixel of more than WC chunks never forms a sub-tile (long-pixel kernel), so
        // its count is capped at WC + 1: the window prefix fits 16 bits
        my_nch = nc > WC + 1 ? WC + 1 : nc;
    }
    int inc = my_nch;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane < nq) sm.cb[lane + 1] = (int16_t)inc;
    if (lane == 0) sm.cb[0] = 0;
    __syncwarp();

    int q0 = 0;
    while (q0 < nq) {
        if (ph == kFused && any_empty) {
            // leading fragment-free pixels: finished directly, 32 per pass
            const bool emp = q0 + lane < nq && sm.offs[q0 + lane + 1] == sm.offs[q0 + lane];
            const unsigned em = __ballot_sync(0xffffffffu, emp);
            const int ne = em == 0xffffffffu ? 32 : __ffs(~em) - 1;
            if (ne > 0) {
                float sb[3];
                if (kPF) self_bg(q0 + lane, sb);
                empty_run<R, GEN>(kp, flags, w0 + q0, ne, lane, kPF ? sb : nullptr);
                q0 += ne;
                continue;
            }
        }
        // sub-tile end: largest q1 with <= FBW fragments and <= 32 chunks
        const int cand = lane + 1;
        const bool fits = cand > q0 && cand <= nq && cand - q0 <= SUBP &&
                          (sm.offs[cand] - sm.offs[q0]) <= FBW && (sm.cb[cand] - sm.cb[q0]) <= WC;
        const int cnt = __popc(__ballot_sync(0xffffffffu, fits));
        if (cnt == 0) {
            // a single pixel deeper than FBW fragments: handled by long_pixel_kernel
            if (lane == 0) {
                const unsigned long long idx =
                    atomicAdd(reinterpret_cast<unsigned long long*>(kp.long_list), 1ull);
                if ((int64_t)idx < kp.long_cap) kp.long_list[1 + idx] = w0 + q0;
            }
            q0 += 1;
            continue;
        }
        // thin sub-tile: a run of > SUBP pixels from q0 with 1..CH fragments each (every
        // pixel one chunk) is taken whole, one pixel per lane (shallow scenes)
        bool thin = false;
        int q1 = q0 + cnt;
        if (kThinOK) {
            const int q = q0 + lane;
            const int run = q < nq ? sm.offs[q + 1] - sm.offs[q] : 0;
            const unsigned b = __ballot_sync(0xffffffffu, run >= 1 && run <= CH);
            const int tc = b == 0xffffffffu ? 32 : __ffs(~b) - 1;
            if (tc > SUBP) {
                thin = true;
                q1 = q0 + tc;
            }
        }
        const int nqs = q1 - q0;
        const int ofa = sm.offs[q0];  // window-relative first fragment of the sub-tile
        const int64_t fa = wbase + ofa, fb = wbase + sm.offs[q1];
        eg_fa = fa;
        const int C = sm.cb[q1] - sm.cb[q0];
        const int64_t a4 = fa & ~(int64_t)3, a16 = fa & ~(int64_t)15;
        const int sh4 = (int)(fa - a4);  // staging index of fragment fa (granule-4 arrays)
        const int shb = (int)(fa - a16);

        // the previous sub-tile's deferred composite: its opaque colours out of the
        // staging buffer before this sub-tile's copies overwrite it
        const float pbg = GEN ? 0.0f : pending_bg();
        if (!GEN) __syncwarp();

        // ---- 1. stage fragment fields (TMA bulk copies, one mbarrier per warp) ----
        // All 4-byte-element and 12-byte-element arrays share the 16-B granule
        // window [a4, b4): one bulk copy each; lanes load the < 4-fragment tail
        // that ends the arrays (or everything without TMA). Backface bytes have a
        // 16-fragment granule and their own window.
        {
            const bool w_ior = GEN && need_ior && kp.f.ior;
            const bool w_nrm = GEN && refr && !WOIT_NRM_GLOBAL;
            const bool w_bf = GEN && bfonly && kp.f.backface;
            int64_t b4 = (fb + 3) & ~(int64_t)3;
            b4 = b4 < (nalloc & ~(int64_t)3) ? b4 : (nalloc & ~(int64_t)3);
            if (!kp.use_tma || b4 < a4) b4 = a4;
            int64_t b16 = (fb + 15) & ~(int64_t)15;
            b16 = b16 < (nalloc & ~(int64_t)15) ? b16 : (nalloc & ~(int64_t)15);
            if (!kp.use_tma || b16 < a16) b16 = a16;
            // fast path: the sub-tile's opaque colours ride along (12 B/pixel, 4-pixel granule)
            const int64_t pa = w0 + q0, pb = w0 + q1, pa4 = pa & ~(int64_t)3;
            int64_t pb4 = (pb + 3) & ~(int64_t)3;
            pb4 = pb4 < (kp.f.npix & ~(int64_t)3) ? pb4 : (kp.f.npix & ~(int64_t)3);
            if (GEN || thin || !kp.use_tma || pb4 < pa4) pb4 = pa4;
            if (kp.use_tma && lane == 0) {
                bulk_wait_read_all();  // the previous sub-tile's stores have left smem
                const uint32_t n4 = (uint32_t)(b4 - a4);
                const uint32_t per = 4u + (do_at ? 16u : 0u) + (do_eval ? 12u : 0u) + (w_ior ? 4u : 0u) +
                                     (w_nrm ? 12u : 0u);
                const uint32_t tx = n4 * per + (w_bf ? (uint32_t)(b16 - a16) : 0u) + 12u * (uint32_t)(pb4 - pa4);
                if (pb4 > pa4) bulk_g2s(sm.opq, kp.f.opaque_color + 3 * pa4, 12u * (uint32_t)(pb4 - pa4), sm.bar);
                mbar_arrive_expect_tx(sm.bar, tx);
                if (n4) {
                    bulk_g2s(sm.depth, kp.f.depth + a4, 4u * n4, sm.bar);
                    if (do_at) {
                        bulk_g2s(sm.alpha, kp.f.alpha + a4, 4u * n4, sm.bar);
                        bulk_g2s(sm.trans, kp.f.trans + 3 * a4, 12u * n4, sm.bar);
                    }
                    if (do_eval) bulk_g2s(sm.rad, kp.f.radiance + 3 * a4, 12u * n4, sm.bar);
                    if (w_ior) bulk_g2s(sm.ior, kp.f.ior + a4, 4u * n4, sm.bar);
                    if (w_nrm) bulk_g2s(sm.normal, kp.f.normal + 3 * a4, 12u * n4, sm.bar);
                    // refraction normals are read from global memory by the evaluation:
                    // on their way into L2 while the sub-tile is built
                    if (GEN && refr && WOIT_NRM_GLOBAL && WOIT_NRM_PREFETCH && kp.f.normal)
                        bulk_prefetch_l2(kp.f.normal + 3 * a4, 12u * n4);
                }
                if (w_bf && b16 > a16) bulk_g2s(sm.bf, kp.f.backface + a16, (uint32_t)(b16 - a16), sm.bar);
            }
            for (int64_t i = (b4 > fa ? b4 : fa) + lane; i < fb; i += 32) {
                const int si = (int)(i - a4);
                sm.depth[si] = kp.f.depth[i];
                if (do_at) {
                    sm.alpha[si] = kp.f.alpha[i];
#pragma unroll
                    for (int c = 0; c < 3; ++c) sm.trans[3 * si + c] = kp.f.trans[3 * i + c];
                }
                if (do_eval)
#pragma unroll
                    for (int c = 0; c < 3; ++c) sm.rad[3 * si + c] = kp.f.radiance[3 * i + c];
                if (w_ior) sm.ior[si] = kp.f.ior[i];
                if (w_nrm)
#pragma unroll
                    for (int c = 0; c < 3; ++c) sm.normal[3 * si + c] = kp.f.normal[3 * i + c];
            }
            if (!GEN && !thin)
                for (int64_t p = (pb4 > pa ? pb4 : pa) + lane; p < pb; p += 32) {
                    const int si = (int)(p - pa4);
                    sm.opq[3 * si] = kp.f.opaque_color[3 * p];
                    sm.opq[3 * si + 1] = kp.f.opaque_color[3 * p + 1];
                    sm.opq[3 * si + 2] = kp.f.opaque_color[3 * p + 2];
                }
            if (w_bf)
                for (int64_t i = (b16 > fa ? b16 : fa) + lane; i < fb; i += 32) sm.bf[(int)(i - a16)] = kp.f.backface[i];
            if (GEN && need_ior && !kp.f.ior)
                for (int i = lane; i < (int)(fb - fa); i += 32) sm.ior[sh4 + i] = 1.0f;
            if (GEN && bfonly && !kp.f.backface)
                for (int i = lane; i < (int)(fb - fa); i += 32) sm.bf[shb + i] = 0;
        }

        if (!GEN && pend) {  // overlaps the copies just issued
            composite_fast(pq0, pnqs, pw0, pbg);
            pend = false;
            __syncwarp();
        }

        if (kThinOK && thin) {
            // ---- thin sub-tile: lane l owns pixel q0 + l, whose whole run is one chunk.
            // Same operations, in the same order, as the general sub-tile with one
            // chunk per pixel (bit-identical results), without the per-(pixel, channel)
            // passes: the lane's column of the partials region holds D, then the
            // staircase v in place, read back by its own evaluation.
            const bool act = lane < nqs;
            const int64_t p = w0 + q0 + lane;
            float tsb[3];
            float tod = INFINITY;
            if (kPF) {
                self_bg(q0 + lane, tsb);
                tod = __shfl_sync(0xffffffffu, cur_od, (q0 + lane) & 31);
            }
            int cst = 0, clen = 0, crot = 0;
            if (act) {
                const int oq = sm.offs[q0 + lane];
                clen = sm.offs[q0 + lane + 1] - oq;
                cst = oq - ofa;
                crot = chunk_rotation(chunk_key(kp.f.pixel_base + p, clen, 0), clen);
            }
            if (kp.use_tma) {
                mbar_wait(sm.bar, parity);
                parity ^= 1u;
            }
            __syncwarp();
            // bounds (step 1)
            float mn = INFINITY, mx = -INFINITY;
            int jj = crot;
            for (int j = 0; j < clen; ++j) {
                const float x = sm.depth[sh4 + cst + jj];
                jj = jj + 1 == clen ? 0 : jj + 1;
                mn = fminf(mn, x);
                mx = fmaxf(mx, x);
            }
            DepthMap m{0.0, 0.0, 0.0, 0.0};
            if (act) {
                if (kp.b.near) kp.b.near[p] = mn;
                if (kp.b.far) kp.b.far[p] = mx;
                m = depth_map(mn, mx, R);
            }
            // build (step 2) into the lane's column
            float* part = sm.part;
            {
                float4* pz = reinterpret_cast<float4*>(part);
                for (int i = lane; i < (kPRows * 3 * WC) / 4; i += 32) pz[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            if (GEN && act) {
                jj = crot;
                for (int j = 0; j < clen; ++j) {
                    const int fr = cst + jj;
                    jj = jj + 1 == clen ? 0 : jj + 1;
                    sm.zfix[(kAliasZ ? sh4 : 0) + fr] = z_fixed_of(sm.depth[sh4 + fr], m);
                }
            }
            __syncwarp();
            if (act) {
                if (!GEN) {
                    build_chunk_fast<R, kRow0>(sm.zfix + (WOIT_ALIASZ ? sh4 : 0), sm.depth, m, sm.alpha, sm.trans, part,
                                               lane, cst, clen, crot, sh4);
                } else {
                    jj = crot;
                    for (int j = 0; j < clen; ++j) {
                        const int fr = cst + jj;
                        jj = jj + 1 == clen ? 0 : jj + 1;
                        const int si = sh4 + fr;
                        const zfix_t zi = sm.zfix[(kAliasZ ? sh4 : 0) + fr];
                        const float al = sm.alpha[si];
                        bool cb_ = false;
                        if (cube) cb_ = sm.ior[si] > 1.0f && (!bfonly || sm.bf[shb + fr] != 0);
                        float a[3];
#pragma unroll
                        for (int ch = 0; ch < 3; ++ch) {
                            const float op = opacity_ch(al, sm.trans[3 * si + ch], cb_);
                            sm.trans[3 * si + ch] = op;
                            a[ch] = -log_poly(fmaxf((float)kTransFloor, 1.0f - op));
                        }
                        d_update<R, kRow0>(part, lane, zi, make_float2(a[0], a[1]), a[2]);
                    }
                }
            }
            // staircase v (prefix of D) in place, total transmittance exp(-v_{M-1})
            double vt[3] = {1.0, 1.0, 1.0};
            if (act) {
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    float r = 0.0f;  // v_c for c < kRow0 is 0
#pragma unroll
                    for (int k = kRow0; k < M; ++k) {
                        float* a = part + (k - kRow0) * 3 * WC + ch * WC + lane;
                        r += *a;
                        *a = r;
                    }
                    vt[ch] = (double)expf(-r);
                }
            }
            // evaluate (step 3)
            float ac[3] = {0.f, 0.f, 0.f}, wg[3] = {0.f, 0.f, 0.f}, df = 0.f;
            double ro[2] = {0.0, 0.0};
            if (act) {
                const CellsCol<M, kRow0> col{part + lane};
                if (!GEN) {
                    eval_chunk_fast<R>(sm.zfix + (WOIT_ALIASZ ? sh4 : 0), sm.alpha, sm.trans, col, sm.rad, cst, clen,
                                       crot, sh4, ac, wg);
                } else {
                    double d[3] = {0.0, 0.0, 0.0}, topq = INFINITY;
                    if (refr) {
                        ray_dir(kp, kp.f.pixel_base + p, d);
                        topq = kPF ? (double)tod : kp.f.opaque_depth ? (double)kp.f.opaque_depth[p] : INFINITY;
                    }
                    eval_gen(col, cst, clen, crot, d, topq, ac, wg, df, ro);
                }
            }
            fence_proxy_async();  // v̂ in smem becomes visible to the bulk store
            __syncwarp();
            if (kp.b.vhat) {
                const int64_t i0 = (fa + 3) & ~(int64_t)3, i1 = fb & ~(int64_t)3;
                const bool bulk = kp.use_tma && i1 > i0;
                if (bulk && lane == 0) {
                    bulk_s2g(kp.b.vhat + 3 * i0, sm.rad + 3 * (i0 - a4), (uint32_t)(12 * (i1 - i0)));
                    bulk_commit();
                }
                const int nhead = bulk ? (int)(i0 - fa) : (int)(fb - fa);
                const int ntail = bulk ? (int)(fb - i1) : 0;
                for (int i = lane; i < nhead + ntail; i += 32) {
                    const int64_t f = i < nhead ? fa + i : i1 + (i - nhead);
                    const int si = (int)(f - a4);
                    kp.b.vhat[3 * f] = sm.rad[3 * si];
                    kp.b.vhat[3 * f + 1] = sm.rad[3 * si + 1];
                    kp.b.vhat[3 * f + 2] = sm.rad[3 * si + 2];
                }
            }
            // accumulators and composite (step 4): the chunk sums of a one-chunk pixel
            if (act) {
                const double ro0 = 0.0 + (double)(float)ro[0], ro1 = 0.0 + (double)(float)ro[1];
                double dp = 0.0;
                if (diffuse) {
                    dp = dadd(dp, ddiv(0.0 + (double)df, 3.0));
                    if (kp.b.diffusion) kp.b.diffusion[p] = (float)dp;
                }
                if (kp.b.refraction_offset) {
                    kp.b.refraction_offset[p * 2] = GEN ? (float)ro0 : 0.0f;
                    kp.b.refraction_offset[p * 2 + 1] = GEN ? (float)ro1 : 0.0f;
                }
                double acc[3], wgt[3];
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    acc[ch] = 0.0 + (double)ac[ch];
                    wgt[ch] = 0.0 + (double)wg[ch];
                    if (kp.b.accum) kp.b.accum[p * 3 + ch] = (float)acc[ch];
                    if (kp.b.weight) kp.b.weight[p * 3 + ch] = (float)wgt[ch];
                }
                if (kp.b.output) {
                    if (GEN) {
                        // all three channels at once (composite_pixel: the same operations
                        // as composite_channel's, bit for bit), so every background gather
                        // of the pixel is in flight together
                        float o3[3];
                        composite_pixel(kp, flags, p, acc, wgt, ro0, ro1, vt, dp, o3, kPF ? tsb : nullptr);
#pragma unroll
                        for (int ch = 0; ch < 3; ++ch) kp.b.output[p * 3 + ch] = o3[ch];
                    } else {
#pragma unroll
                        for (int ch = 0; ch < 3; ++ch)
                            kp.b.output[p * 3 + ch] =
                                composite_fast_ch(flags, acc[ch], wgt[ch], (double)kp.f.opaque_color[p * 3 + ch], vt[ch]);
                    }
                }
            }
            // coefficients: Haar analysis of each channel's staircase in f64, transposed
            // through shared memory ([V][33] over the staging arrays, free once the v̂
            // store has read them) into coalesced stores
            if (kp.b.coeffs) {
                if (lane == 0) bulk_wait_read_all();
                __syncwarp();
                float* stg = sm.depth;
                if (act) {
#pragma unroll 1
                    for (int ch = 0; ch < 3; ++ch) {
                        double T[M], c[S];
#pragma unroll
                        for (int k = 0; k < M; ++k)
                            T[k] = k < kRow0 ? 0.0 : (double)part[(k - kRow0) * 3 * WC + ch * WC + lane];
                        haar_analysis<R>(T, c);
#pragma unroll
                        for (int sl = 0; sl < S; ++sl) stg[(3 * sl + ch) * 33 + lane] = (float)c[sl];
                    }
                }
                __syncwarp();
                float* g = kp.b.coeffs + (w0 + q0) * V;
                for (int o = lane; o < nqs * V; o += 32) {
                    const int pq = o / V, r = o - pq * V;
                    g[o] = stg[r * 33 + pq];
                }
            }
            __syncwarp();
            q0 = q1;
            continue;
        }

        // ---- 2. chunks + per-pixel init (overlaps the copies) -----------------------
        // lane l < C owns chunk l of the sub-tile: its pixel q is the number of sub-tile
        // pixels whose chunks end at or before l, and chunk i of a pixel is fragments
        // [CH i, min(CH (i+1), run)) -- a function of the run length only, so the
        // reduction order never depends on the tiling
        int cq = 0, cst = 0, clen = 0, crot = 0;
        const int cb0 = sm.cb[q0];
        {   // q = the last sub-tile pixel whose first chunk is at or before l: lane j
            // holds pixel j's first chunk (non-decreasing in j), binary search by shuffles
            static_assert((SUBP & (SUBP - 1)) == 0 && SUBP <= 32, "SUBP: power of two");
            const int sj = lane < nqs ? sm.cb[q0 + lane] - cb0 : 0x7fffffff;
#pragma unroll
            for (int step = SUBP / 2; step >= 1; step >>= 1) {
                const int v = __shfl_sync(0xffffffffu, sj, cq + step);
                if (v <= lane) cq += step;
            }
        }
        if (lane < C) {
            const int q = q0 + cq;
            const int st = (lane - (sm.cb[q] - cb0)) * CH;
            const int oq = sm.offs[q];
            const int run = sm.offs[q + 1] - oq;
            cst = oq - ofa + st;
            clen = run - st < CH ? run - st : CH;
            crot = chunk_rotation(chunk_key(kp.f.pixel_base + w0 + q, run, st), clen);
        }
        if (kp.use_tma) {
            mbar_wait(sm.bar, parity);
            parity ^= 1u;
        }
        __syncwarp();

        // ---- 3. bounds (step1) ------------------------------------------------------
        // chunk min / max, then a segmented reduction over each pixel's chunk lanes
        // (consecutive lanes) in order-preserving integers: the pixel's first chunk lane
        // ends up with the pixel's bounds (exact, so independent of the order)
        constexpr unsigned kAll = 0xffffffffu;
        uint32_t mnu = f2ord(INFINITY), mxu = f2ord(-INFINITY);
        if (ph & PH_BOUNDS) {
            if (lane < C) {
                float mn = INFINITY, mx = -INFINITY;
                if (clen == CH && ((sh4 + cst) & 3) == 0) {
                    // min / max do not depend on the order: two 16-B loads per full chunk,
                    // the halves swapped on lanes 4..7 of each quarter warp, so its eight
                    // 16-B accesses hit distinct banks
                    const float4* d4 = reinterpret_cast<const float4*>(sm.depth + sh4 + cst);
                    const int h = (lane >> 2) & 1;
                    const float4 u = d4[h], w = d4[h ^ 1];
                    mn = fminf(fminf(fminf(u.x, u.y), fminf(u.z, u.w)), fminf(fminf(w.x, w.y), fminf(w.z, w.w)));
                    mx = fmaxf(fmaxf(fmaxf(u.x, u.y), fmaxf(u.z, u.w)), fmaxf(fmaxf(w.x, w.y), fmaxf(w.z, w.w)));
                } else {
                    int jj = crot;  // rotated start: conflict-free banks across lanes
                    for (int j = 0; j < clen; ++j) {
                        const float x = sm.depth[sh4 + cst + jj];
                        jj = jj + 1 == clen ? 0 : jj + 1;
                        mn = fminf(mn, x);
                        mx = fmaxf(mx, x);
                    }
                }
                mnu = f2ord(mn);
                mxu = f2ord(mx);
            }
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t a = __shfl_down_sync(kAll, mnu, o), b = __shfl_down_sync(kAll, mxu, o);
                const int k = __shfl_down_sync(kAll, cq, o);
                if (lane + o < C && k == cq) {
                    mnu = min(mnu, a);
                    mxu = max(mxu, b);
                }
            }
        }
        float nf = INFINITY, ff = -INFINITY;
        {
            const int fc = lane < nqs ? sm.cb[q0 + lane] - cb0 : 0;  // the pixel's first chunk lane
            const uint32_t pmn = __shfl_sync(kAll, mnu, fc & 31), pmx = __shfl_sync(kAll, mxu, fc & 31);
            if (lane < nqs) {
                const int64_t p = w0 + q0 + lane;
                uint32_t n_ = f2ord(INFINITY), f_ = f2ord(-INFINITY);
                if ((ph & PH_BOUNDS) && sm.cb[q0 + lane + 1] > fc + cb0) {
                    n_ = pmn;
                    f_ = pmx;
                }
                if (!(ph & PH_BOUNDS) || (ph & PH_BOUNDS_ACC)) {  // combined with the buffers' bounds
                    n_ = min(n_, f2ord(kp.b.near[p]));
                    f_ = max(f_, f2ord(kp.b.far[p]));
                }
                nf = ord2f(n_);
                ff = ord2f(f_);
                if ((ph & PH_BOUNDS) && kp.b.near) kp.b.near[p] = nf;
                if ((ph & PH_BOUNDS) && kp.b.far) kp.b.far[p] = ff;
                if (GEN && !kAliasZ) {
                    const DepthMap m = depth_map(nf, ff, R);
                    sm.lo[lane] = m.lo;
                    sm.den[lane] = m.den;
                    sm.rcp[lane] = m.rs;  // fixed-point z scale (z_fixed_of)
                }
            }
        }
        // fast path: every chunk lane derives its pixel's depth map itself (the same
        // warp instructions as the pixel lanes computing it, no shared-memory round trip)
        DepthMap mq{0.0, 0.0, 0.0, 0.0};
        if (!GEN || kAliasZ) {
            const float cnf = __shfl_sync(kAll, nf, cq), cff = __shfl_sync(kAll, ff, cq);
            if (lane < C) mq = depth_map(cnf, cff, R);
        } else {
            __syncwarp();
        }

        // ---- 4. z (fixed point) and build (step2): chunk partials -> part[v][lane] ----
        float* part = sm.part;
        const bool fused_z = !GEN && (ph & PH_BUILD);  // the fast build computes z itself
        if (lane < C && do_at && !fused_z) {
            const DepthMap m = kAliasZ ? mq : DepthMap{sm.lo[cq], sm.den[cq], 0.0, sm.rcp[cq]};
#pragma unroll kZUnroll
            for (int j = 0; j < CH; ++j) {  // independent chains: unrolled for ILP
                if (j < clen) {
                    int jj = crot + j;
                    jj = jj >= clen ? jj - clen : jj;
                    const int fr = cst + jj;
                    sm.zfix[(kAliasZ ? sh4 : 0) + fr] = z_fixed_of(sm.depth[sh4 + fr], m);
                }
            }
        }
        // The rank-N Haar space (scaling + levels 0..N, M = 2^(N+1) slots) is exactly
        // the piecewise constants on M cells, so the projection of the absorbance
        // staircase is its cell averages: v_c = sum_{j_f < c} a_f + sum_{j_f = c} a_f w_f
        // with j_f = floor(M z_f) and w_f = (j_f + 1) - M z_f. In differences
        // D_c = v_c - v_{c-1} a fragment adds a w to D_j and a (1 - w) to D_{j+1}:
        // two updates per channel, all terms >= 0 (no cancellation), and v is the
        // prefix sum of D. The reference's coefficients are the Haar analysis of v
        // (phase 5) -- its closed form (wavelet.py:272-287) up to rounding.
        if (ph & PH_BUILD) {
            {   // zero the partials [kPRows][3][32] cooperatively, 16 B per store
                float4* pz = reinterpret_cast<float4*>(part);
                for (int i = lane; i < (kPRows * 3 * WC) / 4; i += 32) pz[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            __syncwarp();
            if (!GEN && lane < C) {
                build_chunk_fast<R, kRow0>(sm.zfix + (WOIT_ALIASZ ? sh4 : 0), sm.depth, mq, sm.alpha, sm.trans, part,
                                           lane, cst, clen, crot, sh4);
            } else if (lane < C) {
                int jj = crot;
#pragma unroll kUnroll
                for (int j = 0; j < clen; ++j) {
                    const int fr = cst + jj;   // fragment index relative to fa
                    jj = jj + 1 == clen ? 0 : jj + 1;
                    const int si = sh4 + fr;   // staging index
                    const zfix_t zi = sm.zfix[(kAliasZ ? sh4 : 0) + fr];
                    const float al = sm.alpha[si];
                    bool cb_ = false;
                    if (cube) cb_ = sm.ior[si] > 1.0f && (!bfonly || sm.bf[shb + fr] != 0);
                    float a[3];
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) {
                        const float op = opacity_ch(al, sm.trans[3 * si + ch], cb_);
                        sm.trans[3 * si + ch] = op;  // the evaluation's weight 1 - t (pipeline.py:184)
                        a[ch] = -log_poly(fmaxf((float)kTransFloor, 1.0f - op));
                    }
                    d_update<R, kRow0>(part, lane, zi, make_float2(a[0], a[1]), a[2]);
                }
            }
            __syncwarp();
        }

        // ---- 5. per (pixel, channel): combine chunks in f64, coefficients, total
        //         transmittance and the cell staircase --------------------------------
        if (ph & PH_BUILD) {
            // pixel fastest across lanes: the rotated chunk reads hit distinct banks.
            // nqs <= SUBP keeps this to one round, so every lane has read its partials
            // before the region is reused for coefficients and cells.
            const int t = lane;
            const int ntask = nqs * 3;
            const bool task = t < ntask;
            const int kch = task ? div_small(t, nqs) : 0, kq = task ? t - kch * nqs : 0;
            double c[S];
            float rc[M];
            // Few deep pixels (>= 64 fragments each, <= 4 per sub-tile): the (pixel,
            // channel, cell block) sums are spread over the warp -- KB cells per lane, the
            // cells k = blk + j B of a block, B = M / KB blocks per (pixel, channel) --
            // and gathered through shared memory. Each cell is summed in the general
            // combine's order (chunk order, 4-chunk groups), so neither the split -- a
            // function of the tiling -- nor the kernel instance changes a bit.
            constexpr int B = M >= 8 ? 8 : M, KB = M / B, NR = (12 * B + 31) / 32;
            if (VAR == kVarDeep && nqs <= 4 && B > 1) {
                constexpr int SR = M % 4 == 0 ? M + 4 : M + 1;  // [ntask][SR] scratch rows
                float rs[NR][KB];
                int nr = 0;
#pragma unroll
                for (int r = 0; r < NR; ++r) {  // ntask B <= 12 B lane tasks
                    const int u = lane + 32 * r;
                    const int tb = u / B, blk = u % B;
                    if (tb < ntask) {
                        ++nr;
                        const int kchb = tb / nqs, kqb = tb - kchb * nqs;
                        const int q = q0 + kqb;
                        const int nc = (sm.cb[q + 1] - sm.cb[q]);
                        const int cbq = sm.cb[q] - sm.cb[q0];
                        const float* pv = part + kchb * WC + cbq;
#pragma unroll
                        for (int j = 0; j < KB; ++j) rs[r][j] = 0.0f;
                        if ((nc & 3) == 0 && (cbq & 3) == 0) {
                            // chunk order in 4-chunk groups, like the general combine; lane
                            // blk runs blk steps behind lane 0, so at any step the lanes of
                            // a (pixel, channel) read different groups -- distinct banks
                            const int ng = nc >> 2;
#pragma unroll 1
                            for (int st = 0; st < ng + B - 1; ++st) {
                                const int g = st - blk;
                                if (g >= 0 && g < ng) {
#pragma unroll
                                    for (int j = 0; j < KB; ++j) {
                                        if (blk + j * B < kRow0) continue;  // D_0 (no row): 0
                                        const float4 p4 = *reinterpret_cast<const float4*>(
                                            pv + (blk + j * B - kRow0) * 3 * WC + 4 * g);
                                        rs[r][j] += p4.x;
                                        rs[r][j] += p4.y;
                                        rs[r][j] += p4.z;
                                        rs[r][j] += p4.w;
                                    }
                                }
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < KB; ++j) {
                                float x = 0.0f;
                                if (blk + j * B >= kRow0) {
                                    const float* pk = pv + (blk + j * B - kRow0) * 3 * WC;
#pragma unroll 1
                                    for (int i = 0; i < nc; ++i) x += pk[i];
                                }
                                rs[r][j] = x;
                            }
                        }
                    }
                }
                __syncwarp();  // every lane has read its partials: the region takes the sums
#pragma unroll
                for (int r = 0; r < NR; ++r) {
                    const int u = lane + 32 * r;
                    if (r < nr) {
#pragma unroll
                        for (int j = 0; j < KB; ++j) part[(u / B) * SR + u % B + j * B] = rs[r][j];
                    }
                }
                __syncwarp();
                if (task) {
                    if constexpr (M % 4 == 0) {
#pragma unroll
                        for (int k = 0; k < M; k += 4) {
                            const float4 v4 = *reinterpret_cast<const float4*>(part + t * SR + k);
                            rc[k] = v4.x;
                            rc[k + 1] = v4.y;
                            rc[k + 2] = v4.z;
                            rc[k + 3] = v4.w;
                        }
                    } else {
#pragma unroll
                        for (int k = 0; k < M; ++k) rc[k] = part[t * SR + k];
                    }
#pragma unroll
                    for (int k = 1; k < M; ++k) rc[k] += rc[k - 1];
                }
            } else if (task) {
                const int q = q0 + kq;
                const int nc = (sm.cb[q + 1] - sm.cb[q]);
                const int cbq = sm.cb[q] - sm.cb[q0];
                const float* pv = part + kch * WC + cbq;
#pragma unroll
                for (int k = 0; k < M; ++k) rc[k] = 0.0f;
                if (((cbq | nc) & 3) == 0) {
                    // chunks summed in chunk order (fixed by the pixel's run length only),
                    // all cells interleaved for ILP, 16-B vector loads
#pragma unroll 1
                    for (int i = 0; i < nc; i += 4) {
#pragma unroll
                        for (int k = kRow0; k < M; ++k) {  // D_c for c < kRow0 is 0
                            const float4 p4 = *reinterpret_cast<const float4*>(pv + (k - kRow0) * 3 * WC + i);
                            rc[k] += p4.x;
                            rc[k] += p4.y;
                            rc[k] += p4.z;
                            rc[k] += p4.w;
                        }
                    }
                } else {
#pragma unroll 1
                    for (int i = 0; i < nc; ++i) {
#pragma unroll
                        for (int k = kRow0; k < M; ++k) rc[k] += pv[(k - kRow0) * 3 * WC + i];
                    }
                }
                // cell averages v_c = D_0 + ... + D_c, all terms >= 0
#pragma unroll
                for (int k = 1; k < M; ++k) rc[k] += rc[k - 1];
            }
            // every lane has read its partials: the region now takes coefficients and cells
            __syncwarp();
            if (task) {
                const int q = q0 + kq;
                if (do_eval && !packed) store_cells<M>(sm.cells, kq, kch, rc);
                if (need_coef && !packed) sm.vtot[kq * 3 + kch] = expf(-rc[M - 1]);  // A(z -> 1) = v_{M-1}
                // coefficients: Haar analysis of v in f64 (wavelet.py:3-9 layout):
                // c[2^n + k] = 2^(n/2)/M (sum left half - sum right half), c[0] = mean
                double T[M];
#pragma unroll
                for (int k = 0; k < M; ++k) T[k] = (double)rc[k];
                haar_analysis<R>(T, c);
                if (GEN && (ph & PH_BUILD_ACC)) {
#pragma unroll
                    for (int s = 0; s < S; ++s) c[s] = dadd(c[s], (double)kp.b.coeffs[(w0 + q) * V + 3 * s + kch]);
                }
            }
            if (task) {
#pragma unroll
                for (int s = 0; s < S; ++s) sm.coef32[kq * V + 3 * s + kch] = (float)c[s];
            }
            if (packed) {
                // E5B9G9R9 storage (packing.py:46-111, pipeline.py:154-155): the shared
                // exponent couples the channels, so each (pixel, slot) task packs the three
                // fp32 coefficients just stored (fp32-valued inputs: every step of the
                // reference's pack is exact), keeps the word and writes back the unpacked
                // value m 2^(e-24) (exact in fp32) with the positional sign -- the values
                // the evaluation, v_tot and the coefficient output then use
                __syncwarp();
                for (int idx = lane; idx < nqs * S; idx += 32) {
                    const int pq = idx / S, sl = idx - pq * S;
                    float* t3 = sm.coef32 + pq * V + 3 * sl;
                    const uint32_t w = rgb9e5_pack_fp32(fabsf(t3[0]), fabsf(t3[1]), fabsf(t3[2]));
                    float rt[3];
                    rgb9e5_unpack_fp32(w, rt);
                    sm.words[idx] = w;
                    const float sg = sl == 0 ? 1.0f : -1.0f;
                    t3[0] = sg * rt[0];
                    t3[1] = sg * rt[1];
                    t3[2] = sg * rt[2];
                }
                __syncwarp();
                if (task) {
                    double cu[S];
#pragma unroll
                    for (int s = 0; s < S; ++s) cu[s] = (double)sm.coef32[kq * V + 3 * s + kch];
                    if (need_coef) {
                        double at = cu[0];
#pragma unroll
                        for (int n = 0; n <= R; ++n) at = dsub(at, dmul(kSqrt2Pow[n], cu[(2 << n) - 1]));
                        sm.vtot[kq * 3 + kch] = expf(-(float)fmax(at, 0.0));
                    }
                    if (do_eval) {
                        double cell[S];
                        haar_cells<R>(cu, cell);
                        store_cells<M>(sm.cells, kq, kch, cell);
                    }
                }
            }
        } else if (GEN && need_coef) {
            for (int t = lane; t < nqs * 3; t += 32) {
                const int kch = t / nqs, kq = t - kch * nqs;
                const int64_t p = w0 + q0 + kq;
                double c[S];
#pragma unroll
                for (int s = 0; s < S; ++s) c[s] = (double)kp.b.coeffs[p * V + 3 * s + kch];
                double at = c[0];
#pragma unroll
                for (int n = 0; n <= R; ++n) at = dsub(at, dmul(kSqrt2Pow[n], c[(2 << n) - 1]));
                sm.vtot[kq * 3 + kch] = expf(-(float)fmax(at, 0.0));
                double cell[S];
                haar_cells<R>(c, cell);
                store_cells<M>(sm.cells, kq, kch, cell);
            }
        }
        fence_proxy_async();  // coef32 / words become visible to the bulk stores
        __syncwarp();
        if (packed && (ph & PH_BUILD) && kp.b.coeff_words) {
            uint32_t* g = kp.b.coeff_words + (w0 + q0) * S;
            const uint32_t bytes = (uint32_t)(nqs * S * 4);
            if (kp.use_tma && ((reinterpret_cast<uintptr_t>(g) & 15u) == 0) && (bytes & 15u) == 0) {
                if (lane == 0) {
                    bulk_s2g(g, sm.words, bytes);
                    bulk_commit();
                }
            } else {
                for (int i = lane; i < nqs * S; i += 32) g[i] = sm.words[i];
            }
        }
        if ((ph & PH_BUILD) && kp.b.coeffs) {
            float* g = kp.b.coeffs + (w0 + q0) * V;
            const uint32_t bytes = (uint32_t)(nqs * V * 4);
            if (kp.use_tma && ((reinterpret_cast<uintptr_t>(g) & 15u) == 0) && (bytes & 15u) == 0) {
                if (lane == 0) {
                    bulk_s2g(g, sm.coef32, bytes);
                    bulk_commit();
                }
            } else {
                for (int i = lane; i < nqs * V; i += 32) g[i] = sm.coef32[i];
            }
        }

        // ---- 6. evaluate (step3): v̂ per fragment, chunk accumulators --------------
        if (do_eval) {
            const float cod = kPF ? __shfl_sync(0xffffffffu, cur_od, (q0 + cq) & 31) : INFINITY;
            if (lane < C) {
                const float2* cq2 = sm.cells + cq * CellRow<M>::CR;
                float ac[3] = {0.f, 0.f, 0.f}, wg[3] = {0.f, 0.f, 0.f}, df = 0.f;
                double ro[2] = {0.0, 0.0};
                double d[3] = {0.0, 0.0, 0.0}, topq = INFINITY;
                const int64_t p = w0 + q0 + cq;
                if (refr) {
                    ray_dir(kp, kp.f.pixel_base + p, d);
                    topq = kPF ? (double)cod : kp.f.opaque_depth ? (double)kp.f.opaque_depth[p] : INFINITY;
                }
                const bool op_staged = ph & PH_BUILD;  // the build left alpha (1 - T') in the trans slot
                if (!GEN) {
                    eval_chunk_fast<R>(sm.zfix + (WOIT_ALIASZ ? sh4 : 0), sm.alpha, sm.trans, CellsPair{cq2}, sm.rad, cst, clen, crot, sh4, ac, wg);
                } else {
                    eval_gen(CellsPair{cq2}, cst, clen, crot, d, topq, ac, wg, df, ro);
                }
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    sm.accp[ch * AR + lane] = ac[ch];
                    sm.accp[(3 + ch) * AR + lane] = wg[ch];
                }
                if (GEN) {  // the fast path's accumulators are ac / wg only (its v_tot follows them)
                    sm.accp[6 * AR + lane] = (float)ro[0];
                    sm.accp[7 * AR + lane] = (float)ro[1];
                }
                if (diffuse) sm.accp[8 * AR + lane] = df;  // (the row exists with diffusion only)
            }
            fence_proxy_async();  // v̂ in smem becomes visible to the bulk store
            __syncwarp();
            // v̂ store: aligned interior by one bulk copy, ragged ends by the lanes
            if (kp.b.vhat) {
                const int64_t i0 = (fa + 3) & ~(int64_t)3, i1 = fb & ~(int64_t)3;
                const bool bulk = kp.use_tma && i1 > i0;
                if (bulk && lane == 0) {
                    bulk_s2g(kp.b.vhat + 3 * i0, sm.rad + 3 * (i0 - a4), (uint32_t)(12 * (i1 - i0)));
                    bulk_commit();
                }
                // lanes cover the ragged head [fa, i0) and tail [i1, fb) (< 4 each), or
                // everything without TMA
                const int nhead = bulk ? (int)(i0 - fa) : (int)(fb - fa);
                const int ntail = bulk ? (int)(fb - i1) : 0;
                for (int i = lane; i < nhead + ntail; i += 32) {
                    const int64_t f = i < nhead ? fa + i : i1 + (i - nhead);
                    const int si = (int)(f - a4);
                    kp.b.vhat[3 * f] = sm.rad[3 * si];
                    kp.b.vhat[3 * f + 1] = sm.rad[3 * si + 1];
                    kp.b.vhat[3 * f + 2] = sm.rad[3 * si + 2];
                }
            }
        }

        // ---- 7. per-pixel accumulators + composite (step4) -------------------------
        float csb = 0.0f;  // lane (pixel kq, channel kch)'s prefetched background value
        if (kPF) {
            const int kch = lane / nqs, kq = lane - kch * nqs;
            float b[3];
            self_bg(q0 + kq, b);
            csb = kch == 0 ? b[0] : kch == 1 ? b[1] : b[2];
        }
        if (!GEN) {
            // fast path: deferred to the next sub-tile's staging (composite_fast)
            pend = true;
            pq0 = q0;
            pnqs = nqs;
            pw0 = w0;
        } else if (lane < 3 * nqs) {
            // general path: one lane per (pixel, channel) as well; the refraction and
            // diffusion sums are per pixel, and every channel lane forms them in the
            // same order (identical values); the channel-0 lane stores them
            const int kch = lane / nqs, kq = lane - kch * nqs;
            const int q = q0 + kq;
            const int64_t p = w0 + q;
            double acc = 0.0, wgt = 0.0, ro0 = 0.0, ro1 = 0.0, dsum = 0.0, dp = 0.0;
            const bool acc_in = (ph & PH_EVAL_ACC) || ((ph & PH_COMPOSITE) && !do_eval);
            if (acc_in) {
                acc = kp.b.accum[p * 3 + kch];
                wgt = kp.b.weight[p * 3 + kch];
                if (kp.b.refraction_offset) {
                    ro0 = kp.b.refraction_offset[p * 2];
                    ro1 = kp.b.refraction_offset[p * 2 + 1];
                }
                if (diffuse && kp.b.diffusion) dp = kp.b.diffusion[p];
            }
            if (do_eval) {
                const int nc = (sm.cb[q + 1] - sm.cb[q]);
                const int cbq = sm.cb[q] - sm.cb[q0];
                for (int i = 0; i < nc; ++i) {
                    const int cc = cbq + i;
                    acc += (double)sm.accp[kch * AR + cc];
                    wgt += (double)sm.accp[(3 + kch) * AR + cc];
                    if (refr) {
                        ro0 += (double)sm.accp[6 * AR + cc];
                        ro1 += (double)sm.accp[7 * AR + cc];
                    }
                    if (diffuse) dsum += (double)sm.accp[8 * AR + cc];
                }
                if (diffuse) dp = dadd(dp, ddiv(dsum, 3.0));
                if (kp.b.accum) kp.b.accum[p * 3 + kch] = (float)acc;
                if (kp.b.weight) kp.b.weight[p * 3 + kch] = (float)wgt;
                if (kch == 0) {
                    if (diffuse && kp.b.diffusion) kp.b.diffusion[p] = (float)dp;
                    if (kp.b.refraction_offset) {
                        kp.b.refraction_offset[p * 2] = (float)ro0;
                        kp.b.refraction_offset[p * 2 + 1] = (float)ro1;
                    }
                }
            }
            if ((ph & PH_COMPOSITE) && kp.b.output)
                kp.b.output[p * 3 + kch] = composite_channel(kp, flags, p, kch, acc, wgt, ro0, ro1,
                                                             (double)sm.vtot[kq * 3 + kch], dp, kPF ? &csb : nullptr);
        }
        fence_proxy_async();
        __syncwarp();
        q0 = q1;
    }
    }  // window loop
    flush();
    if (lane == 0) bulk_wait_all();
}

// ---------------------------------------------------------------------------
// pixels deeper than one sub-tile: one CTA per pixel, fragments streamed from
// global memory (coalesced), per-thread fp64 accumulators, fixed-order combine.

constexpr int kLongT = 256;

template <int R>
__global__ void __launch_bounds__(kLongT) long_pixel_kernel(const __grid_constant__ KParams kp) {
    constexpr int S = 1 << (R + 1), V = 3 * S, M = S;
    constexpr int TL = R <= 3 ? kLongT : (kLongT >> (R - 3));  // keep acc64 <= 96 KB
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* acc64 = reinterpret_cast<double*>(smem_raw);      // [V][TL]
    double* coef = acc64 + V * TL;                              // [V]
    float* cells = reinterpret_cast<float*>(coef + V);          // [V]
    __shared__ double red[9][kLongT];
    __shared__ double vt[3];
    __shared__ float nf_s, ff_s;
    const int tid = threadIdx.x;
    const uint32_t ph = kp.phases;
    const int flags = kp.p.flags;
    const bool cube = flags & WOIT_CUBE_TRANSMISSION;
    const bool bfonly = cube && (flags & WOIT_CUBE_BACKFACE_ONLY);
    const bool refr = (ph & PH_EVAL) && (flags & WOIT_REFRACTION);
    // launched as a programmatic dependent of the frame kernel: its CTAs may start
    // while the frame kernel's last warps finish; the list is read only after the
    // frame kernel has completed and its writes are visible
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int64_t count = kp.long_list[0] < kp.long_cap ? kp.long_list[0] : kp.long_cap;
    for (int64_t li = blockIdx.x; li < count; li += gridDim.x) {
        const int64_t p = kp.long_list[1 + li];
        const int64_t s = kp.f.offsets[p], e = kp.f.offsets[p + 1];
        // bounds
        float mn = INFINITY, mx = -INFINITY;
        if (ph & PH_BOUNDS) {
            for (int64_t f = s + tid; f < e; f += kLongT) {
                mn = fminf(mn, kp.f.depth[f]);
                mx = fmaxf(mx, kp.f.depth[f]);
            }
        }
        red[0][tid] = mn;
        red[1][tid] = mx;
        __syncthreads();
        for (int o = kLongT / 2; o > 0; o >>= 1) {
            if (tid < o) {
                red[0][tid] = fmin(red[0][tid], red[0][tid + o]);
                red[1][tid] = fmax(red[1][tid], red[1][tid + o]);
            }
            __syncthreads();
        }
        if (tid == 0) {
            float nf = (float)red[0][0], ff = (float)red[1][0];
            if (!(ph & PH_BOUNDS) || (ph & PH_BOUNDS_ACC)) {
                const float bn = kp.b.near[p], bfar = kp.b.far[p];
                nf = (ph & PH_BOUNDS) ? fminf(nf, bn) : bn;
                ff = (ph & PH_BOUNDS) ? fmaxf(ff, bfar) : bfar;
            }
            if ((ph & PH_BOUNDS) && kp.b.near) kp.b.near[p] = nf;
            if ((ph & PH_BOUNDS) && kp.b.far) kp.b.far[p] = ff;
            nf_s = nf;
            ff_s = ff;
        }
        __syncthreads();
        if (!(ph & (PH_BUILD | PH_EVAL | PH_COMPOSITE))) continue;  // step1 alone: bounds only
        const DepthMap m = depth_map(nf_s, ff_s, R);
        // build
        if (ph & PH_BUILD) {
            if (tid < TL) {
                for (int v = 0; v < V; ++v) acc64[v * TL + tid] = 0.0;
                for (int64_t f = s + tid; f < e; f += TL) {
                    const zfix_t zi = z_fixed_of(kp.f.depth[f], m);
                    const float al = kp.f.alpha[f];
                    bool cb_ = false;
                    if (cube) {
                        const float io = kp.f.ior ? kp.f.ior[f] : 1.0f;
                        cb_ = io > 1.0f && (!bfonly || (kp.f.backface && kp.f.backface[f]));
                    }
                    float a[3];
                    for (int ch = 0; ch < 3; ++ch) a[ch] = absorbance_ch(al, kp.f.trans[3 * f + ch], cb_);
                    const float one_m_z = one_minus_z(zi);
                    const float psi0 = level_psi(zi, 0);
                    for (int ch = 0; ch < 3; ++ch) {
                        acc64[ch * TL + tid] += (double)(a[ch] * one_m_z);
                        acc64[(3 + ch) * TL + tid] -= (double)(a[ch] * psi0);
                    }
                    for (int n = 1; n <= R; ++n) {
                        const int k = slot_offset(zi, n);
                        const float psi = level_psi(zi, n) * kInvSqrt2PowF[n];
                        for (int ch = 0; ch < 3; ++ch)
                            acc64[(((1 << n) + k) * 3 + ch) * TL + tid] -= (double)(a[ch] * psi);
                    }
                }
            }
            __syncthreads();
            for (int v = tid; v < V; v += kLongT) {
                double sum = (ph & PH_BUILD_ACC) ? (double)kp.b.coeffs[p * V + v] : 0.0;
                for (int t = 0; t < TL; ++t) sum += acc64[v * TL + t];
                coef[v] = sum;
            }
            __syncthreads();
            if (flags & WOIT_PACKED_STORAGE) {
                // the frame kernel's packing: the fp32 coefficients, packed and unpacked
                for (int sl = tid; sl < S; sl += kLongT) {
                    const uint32_t w = rgb9e5_pack_fp32(fabsf((float)coef[3 * sl]), fabsf((float)coef[3 * sl + 1]),
                                                        fabsf((float)coef[3 * sl + 2]));
                    float rt[3];
                    rgb9e5_unpack_fp32(w, rt);
                    if (kp.b.coeff_words) kp.b.coeff_words[p * S + sl] = w;
                    const double sg = sl == 0 ? 1.0 : -1.0;
                    for (int ch = 0; ch < 3; ++ch) coef[3 * sl + ch] = sg * (double)rt[ch];
                }
                __syncthreads();
            }
            if (kp.b.coeffs)
                for (int v = tid; v < V; v += kLongT) kp.b.coeffs[p * V + v] = (float)coef[v];
        } else {
            for (int v = tid; v < V; v += kLongT) coef[v] = kp.b.coeffs[p * V + v];
        }
        __syncthreads();
        if (tid < 3) {
            double at = coef[tid];
            for (int n = 0; n <= R; ++n) at = dsub(at, dmul(kSqrt2Pow[n], coef[((2 << n) - 1) * 3 + tid]));
            vt[tid] = exp(-fmax(at, 0.0));
        }
        for (int w = tid; w < V; w += kLongT) {
            const int cell = w / 3, ch = w - cell * 3;
            double val = coef[ch];
            for (int n = 0; n <= R; ++n) {
                const int mm = R + 1 - n;
                const double sg = ((cell >> (mm - 1)) & 1) ? -1.0 : 1.0;
                val = dadd(val, dmul(dmul(kSqrt2Pow[n], sg), coef[((1 << n) + (cell >> mm)) * 3 + ch]));
            }
            cells[w] = (float)val;
        }
        __syncthreads();
        // eval
        double lac[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        if (ph & PH_EVAL) {
            double d[3] = {0, 0, 0}, topq = INFINITY;
            if (refr) {
                ray_dir(kp, kp.f.pixel_base + p, d);
                topq = kp.f.opaque_depth ? (double)kp.f.opaque_depth[p] : INFINITY;
            }
            for (int64_t f = s + tid; f < e; f += kLongT) {
                const zfix_t zi = z_fixed_of(kp.f.depth[f], m);
                int c0, c1;
                float t;
                eval_cells(zi, R, c0, c1, t);
                const float al = kp.f.alpha[f];
                const float io = kp.f.ior ? kp.f.ior[f] : 1.0f;
                const bool cb_ = cube && io > 1.0f && (!bfonly || (kp.f.backface && kp.f.backface[f]));
                float vs = 0.0f;
                for (int ch = 0; ch < 3; ++ch) {
                    const float A = fmaxf((1.0f - t) * cells[c0 * 3 + ch] + t * cells[c1 * 3 + ch], 0.0f);
                    const float vh = expf(-A);
                    lac[ch] += (double)((kp.f.radiance[3 * f + ch] * al) * vh);
                    lac[3 + ch] += (double)(opacity_ch(al, kp.f.trans[3 * f + ch], cb_) * vh);
                    vs += vh;
                    if (kp.b.vhat) kp.b.vhat[3 * f + ch] = vh;
                }
                lac[8] += (double)(al * vs);
                if (refr && io > 1.0f) {
                    const float nrm[3] = {kp.f.normal[3 * f], kp.f.normal[3 * f + 1], kp.f.normal[3 * f + 2]};
                    double off[2];
                    refraction_offset(kp, d, topq, kp.f.depth[f], nrm, io, off);
                    lac[6] += off[0];
                    lac[7] += off[1];
                }
            }
        }
        for (int k = 0; k < 9; ++k) red[k][tid] = lac[k];
        __syncthreads();
        for (int o = kLongT / 2; o > 0; o >>= 1) {
            if (tid < o)
                for (int k = 0; k < 9; ++k) red[k][tid] += red[k][tid + o];
            __syncthreads();
        }
        if (tid == 0) {
            double acc[3], wgt[3], ro[2];
            const bool acc_in = (ph & PH_EVAL_ACC) || ((ph & PH_COMPOSITE) && !(ph & PH_EVAL));
            for (int ch = 0; ch < 3; ++ch) {
                acc[ch] = (acc_in ? (double)kp.b.accum[p * 3 + ch] : 0.0) + ((ph & PH_EVAL) ? red[ch][0] : 0.0);
                wgt[ch] = (acc_in ? (double)kp.b.weight[p * 3 + ch] : 0.0) + ((ph & PH_EVAL) ? red[3 + ch][0] : 0.0);
            }
            for (int k = 0; k < 2; ++k)
                ro[k] = (acc_in && kp.b.refraction_offset ? (double)kp.b.refraction_offset[p * 2 + k] : 0.0) +
                        ((ph & PH_EVAL) ? red[6 + k][0] : 0.0);
            double dp = (acc_in && kp.b.diffusion) ? (double)kp.b.diffusion[p] : 0.0;
            if (ph & PH_EVAL) dp = dadd(dp, ddiv(red[8][0], 3.0));
            if (ph & PH_EVAL) {
                if (kp.b.diffusion && (kp.p.flags & WOIT_DIFFUSION)) kp.b.diffusion[p] = (float)dp;
                if (kp.b.accum)
                    for (int ch = 0; ch < 3; ++ch) kp.b.accum[p * 3 + ch] = (float)acc[ch];
                if (kp.b.weight)
                    for (int ch = 0; ch < 3; ++ch) kp.b.weight[p * 3 + ch] = (float)wgt[ch];
                if (kp.b.refraction_offset) {
                    kp.b.refraction_offset[p * 2] = (float)ro[0];
                    kp.b.refraction_offset[p * 2 + 1] = (float)ro[1];
                }
            }
            if ((ph & PH_COMPOSITE) && kp.b.output) {
                float out[3];
                composite_pixel(kp, kp.p.flags, p, acc, wgt, ro[0], ro[1], vt, dp, out);
                for (int ch = 0; ch < 3; ++ch) kp.b.output[p * 3 + ch] = out[ch];
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// host side

template <int R>
size_t long_smem_bytes() {
    constexpr int S = 1 << (R + 1), V = 3 * S;
    constexpr int TL = R <= 3 ? kLongT : (kLongT >> (R - 3));
    return (size_t)V * TL * 8 + (size_t)V * 8 + (size_t)V * 4;
}

// Per-(kernel, device, dynamic smem size) launch configuration, computed once: the
// smem opt-in attribute and the occupancy query are host calls worth microseconds,
// which showed at short frames (config 3) and in the step-wise API. Errors of these
// calls are returned, never cleared (a pending error of an unrelated earlier launch
// stays visible to the caller).
struct LaunchKey {
    const void* fn;
    int dev, bytes;
    bool operator==(const LaunchKey& o) const { return fn == o.fn && dev == o.dev && bytes == o.bytes; }
};
struct LaunchVal {
    int sms, per_sm;
};
cudaError_t launch_config(const void* fn, int threads, int bytes, int& sms, int& per_sm) {
    static std::mutex mu;
    static std::vector<std::pair<LaunchKey, LaunchVal>> cache;
    // the smem opt-in attribute only ever grows (per kernel and device): a launch with
    // fewer bytes than the largest seen so far needs no new call, and lowering it would
    // break a later launch of a cached larger size
    static std::vector<std::pair<LaunchKey, int>> optin;
    int dev = 0;
    cudaError_t err = cudaGetDevice(&dev);
    if (err != cudaSuccess) return err;
    const LaunchKey key{fn, dev, bytes};
    std::lock_guard<std::mutex> lock(mu);
    for (const auto& e : cache)
        if (e.first == key) {
            sms = e.second.sms;
            per_sm = e.second.per_sm;
            return cudaSuccess;
        }
    int* cur = nullptr;
    for (auto& e : optin)
        if (e.first.fn == fn && e.first.dev == dev) cur = &e.second;
    if (!cur || *cur < bytes) {
        if ((err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes)) != cudaSuccess)
            return err;
        if (cur)
            *cur = bytes;
        else
            optin.push_back({LaunchKey{fn, dev, 0}, bytes});
    }
    if ((err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return err;
    if ((err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, bytes)) != cudaSuccess) return err;
    if (per_sm < 1) per_sm = 1;
    cache.push_back({key, LaunchVal{sms, per_sm}});
    return cudaSuccess;
}

template <int R, bool GEN, bool FUS, int VAR, int FL = 0>
cudaError_t launch_tiles(const KParams& kp, cudaStream_t st) {
    using G = WT<R>;
    const uint32_t ph = (GEN && !FUS) ? kp.phases : (PH_BOUNDS | PH_BUILD | PH_EVAL | PH_COMPOSITE);
    constexpr bool kAliasZ = WOIT_ALIASZ && (!GEN || (FUS && WOIT_GEN_ALIASZ));  // as frame_kernel
    const WLayout L = make_wlayout<R>(ph, GEN ? kp.p.flags : ((kp.p.flags & WOIT_NORMALIZE) | FL), kAliasZ, GEN);
    const int bytes = (int)(L.total * G::WPB);
    // persistent grid: as many CTAs as can be resident, each warp loops over windows
    const int64_t warps = (kp.f.npix + G::WIN - 1) / G::WIN;
    int64_t grid = (warps + G::WPB - 1) / G::WPB;
    int sms = 148, per_sm = 1;
    cudaError_t err = launch_config(reinterpret_cast<const void*>(frame_kernel<R, GEN, FUS, VAR, FL>), G::WPB * 32,
                                    bytes, sms, per_sm);
    if (err != cudaSuccess) return err;
    const int64_t resident = (int64_t)sms * per_sm * WOIT_PERSIST;
    if (WOIT_PERSIST > 0) grid = grid < resident ? grid : resident;
    if (grid > 0) {
        frame_kernel<R, GEN, FUS, VAR, FL><<<(unsigned)grid, G::WPB * 32, bytes, st>>>(kp);
        err = cudaGetLastError();
    }
    return err;
}

// Claim order of the fused general kernel's windows: the windows holding fragments
// first, the empty ones after them (in any order: the results do not depend on which
// warp takes a window, or when). One thread per window, warp-aggregated counters.
__global__ void window_order_kernel(const int64_t* __restrict__ offsets, int64_t npix, int64_t nwin,
                                    int32_t* __restrict__ order, unsigned* __restrict__ cnt) {
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool in = w < nwin;
    bool full = false;
    if (in) {
        const int64_t a = w * 32, b = a + 32 < npix ? a + 32 : npix;
        full = offsets[b] > offsets[a];
    }
    const unsigned mf = __ballot_sync(0xffffffffu, in && full), me = __ballot_sync(0xffffffffu, in && !full);
    unsigned bf = 0, be = 0;
    if (lane == 0) {
        if (mf) bf = atomicAdd(cnt, (unsigned)__popc(mf));
        if (me) be = atomicAdd(cnt + 1, (unsigned)__popc(me));
    }
    bf = __shfl_sync(0xffffffffu, bf, 0);
    be = __shfl_sync(0xffffffffu, be, 0);
    const unsigned lt = (1u << lane) - 1u;
    if (in) {
        if (full)
            order[bf + __popc(mf & lt)] = (int32_t)w;
        else
            order[nwin - 1 - (int64_t)(be + __popc(me & lt))] = (int32_t)w;
    }
}

// Sparse frames only (fewer fragments than pixels, so most windows are empty): in
// denser frames the claim's extra dependent load outweighs the shorter tail
// (glass-stack, 3.8 fragments per pixel: +6%).
cudaError_t launch_window_order(KParams& kp, cudaStream_t st) {
    if (!WOIT_GEN_ORDER || !kp.win_order || kp.f.nfrag >= kp.f.npix) {
        kp.win_order = nullptr;
        return cudaSuccess;
    }
    const int64_t nwin = (kp.f.npix + 31) / 32;
    window_order_kernel<<<(unsigned)((nwin + 255) / 256), 256, 0, st>>>(kp.f.offsets, kp.f.npix, nwin, kp.win_order,
                                                                         kp.order_cnt);
    return cudaGetLastError();
}

// The fused general kernel, with instances specialised (at rank 3) for the flag
// sets of the measured configurations: the flags fold to constants, so the code of
// the other features drops out (a smaller kernel: fewer instruction-cache misses,
// fewer registers). Identical operations, identical bits.
constexpr int kFlC3 = WOIT_REFRACTION | WOIT_CHROMATIC_ABERRATION | WOIT_CUBE_TRANSMISSION;  // config 3
constexpr int kFlC3D = kFlC3 | WOIT_DIFFUSION;                                              // + diffusion
constexpr int kFlRefr = WOIT_REFRACTION;                                                    // glass stacks
template <int R>
cudaError_t launch_general(const KParams& kp_in, cudaStream_t st) {
    constexpr int TV = WOIT_THIN ? kVarThin : kVarPlain;
    KParams kp = kp_in;
    const cudaError_t oerr = launch_window_order(kp, st);
    if (oerr != cudaSuccess) return oerr;
    if constexpr (R == 3 && WOIT_FLAG_INSTANCES) {
        const int fl = kp.p.flags & ~WOIT_NORMALIZE;
        if (fl == kFlC3) return launch_tiles<R, true, true, TV, kFlC3>(kp, st);
        if (fl == kFlC3D) return launch_tiles<R, true, true, TV, kFlC3D>(kp, st);
        if (fl == kFlRefr) return launch_tiles<R, true, true, TV, kFlRefr>(kp, st);
    }
    return launch_tiles<R, true, true, TV>(kp, st);
}

template <int R>
cudaError_t launch_rank(const KParams& kp, cudaStream_t st) {
    using G = WT<R>;
    constexpr uint32_t kFused = PH_BOUNDS | PH_BUILD | PH_EVAL | PH_COMPOSITE;
    const bool fused = kp.phases == kFused;
    const bool fast = fused && (kp.p.flags & ~WOIT_NORMALIZE) == 0;
    // packed storage alone: the fast kernel with the E5B9G9R9 epilogue (plain sub-tiles
    // at every depth); rank 0 (8-byte words per pixel pair) takes the general kernel
    const bool fast_packed = R >= 1 && fused && (kp.p.flags & ~WOIT_NORMALIZE) == WOIT_PACKED_STORAGE;
    // thin sub-tiles are compiled into a separate instance of the fast kernel: their
    // code measurably slows the deep-pixel instance even when no thin sub-tile forms
    // (the two give identical bits, so the choice is only a matter of speed)
    // Likewise the deep-pixel combine (few pixels of >= 64 fragments per sub-tile) is
    // compiled only into the instance for deep frames (> 160 fragments per pixel on
    // average): it pays at 256 fragments per pixel and costs the others codegen.
    const bool shallow = WOIT_THIN && kp.f.nfrag <= 16 * kp.f.npix;
    const bool deep = kp.f.nfrag > 160 * kp.f.npix;
    cudaError_t err = fast_packed ? launch_tiles<R, false, true, kVarPlain, WOIT_PACKED_STORAGE>(kp, st)
                      : fast ? (shallow ? launch_tiles<R, false, true, kVarThin>(kp, st)
                              : deep  ? launch_tiles<R, false, true, kVarDeep>(kp, st)
                                      : launch_tiles<R, false, true, kVarPlain>(kp, st))
                           : fused ? launch_general<R>(kp, st)
                                   : launch_tiles<R, true, false, kVarPlain>(kp, st);
    if (err != cudaSuccess) return err;
    const size_t ls = long_smem_bytes<R>();
    if (kp.f.nfrag > G::FBW) {  // a pixel deeper than FBW can only exist if nfrag > FBW
        int sms = 0, per_sm = 0;
        err = launch_config(reinterpret_cast<const void*>(long_pixel_kernel<R>), kLongT, (int)ls, sms, per_sm);
        if (err != cudaSuccess) return err;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(64);
        cfg.blockDim = dim3(kLongT);
        cfg.dynamicSmemBytes = ls;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        err = cudaLaunchKernelEx(&cfg, long_pixel_kernel<R>, kp);
    }
    return err;
}

cudaError_t launch_frame(const KParams& kp, cudaStream_t st) {
    switch (kp.p.rank) {
        case 0: return launch_rank<0>(kp, st);
        case 1: return launch_rank<1>(kp, st);
        case 2: return launch_rank<2>(kp, st);
        case 3: return launch_rank<3>(kp, st);
        case 4: return launch_rank<4>(kp, st);
        case 5: return launch_rank<5>(kp, st);
        case 6: return launch_rank<6>(kp, st);
        default: return cudaErrorInvalidValue;
    }
}

// step4 alone: per-pixel composite from the buffers
template <int R>
__global__ void composite_kernel(const __grid_constant__ KParams kp) {
    constexpr int S = 1 << (R + 1), V = 3 * S;
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= kp.f.npix) return;
    const float* c = kp.b.coeffs + p * V;
    double vt[3], acc[3], wgt[3];
    for (int ch = 0; ch < 3; ++ch) {
        double at = c[ch];
        for (int n = 0; n <= R; ++n) at = dsub(at, dmul(kSqrt2Pow[n], (double)c[((2 << n) - 1) * 3 + ch]));
        vt[ch] = exp(-fmax(at, 0.0));
        acc[ch] = kp.b.accum[p * 3 + ch];
        wgt[ch] = kp.b.weight[p * 3 + ch];
    }
    const double ox = kp.b.refraction_offset ? kp.b.refraction_offset[2 * p] : 0.0;
    const double oy = kp.b.refraction_offset ? kp.b.refraction_offset[2 * p + 1] : 0.0;
    const double dp = kp.b.diffusion ? (double)kp.b.diffusion[p] : 0.0;
    float out[3];
    composite_pixel(kp, kp.p.flags, p, acc, wgt, ox, oy, vt, dp, out);
    for (int ch = 0; ch < 3; ++ch) kp.b.output[p * 3 + ch] = out[ch];
}

// Per-fragment z and every index the kernels derive from it, through the same
// device functions (parity tests check these bit-exactly against the reference).
__global__ void indices_kernel(const KParams kp, double* z_out, int32_t* k_out, int32_t* cell_out) {
    const int rank = kp.p.rank;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < kp.f.npix;
         p += (int64_t)gridDim.x * blockDim.x) {
        const DepthMap m = depth_map(kp.b.near[p], kp.b.far[p], rank);
        for (int64_t f = kp.f.offsets[p]; f < kp.f.offsets[p + 1]; ++f) {
            const double z = normalized_z(kp.f.depth[f], m);
            const zfix_t zi = z_fixed_of(kp.f.depth[f], m);
            z_out[f] = z;
            for (int n = 0; n <= rank; ++n) k_out[f * (rank + 1) + n] = slot_offset(zi, n);
            int c0, c1;
            float t;
            eval_cells(zi, rank, c0, c1, t);
            cell_out[2 * f] = c0;
            cell_out[2 * f + 1] = c1;
        }
    }
}

cudaError_t launch_indices(const KParams& kp, double* z, int32_t* k, int32_t* cells, cudaStream_t st) {
    const int64_t g = (kp.f.npix + 127) / 128;
    if (g == 0) return cudaSuccess;
    indices_kernel<<<(unsigned)(g > 65535 ? 65535 : g), 128, 0, st>>>(kp, z, k, cells);
    return cudaGetLastError();
}

cudaError_t launch_composite(const KParams& kp, cudaStream_t st) {
    const unsigned grid = (unsigned)((kp.f.npix + 255) / 256);
    if (grid == 0) return cudaSuccess;
    switch (kp.p.rank) {
        case 0: composite_kernel<0><<<grid, 256, 0, st>>>(kp); break;
        case 1: composite_kernel<1><<<grid, 256, 0, st>>>(kp); break;
        case 2: composite_kernel<2><<<grid, 256, 0, st>>>(kp); break;
        case 3: composite_kernel<3><<<grid, 256, 0, st>>>(kp); break;
        case 4: composite_kernel<4><<<grid, 256, 0, st>>>(kp); break;
        case 5: composite_kernel<5><<<grid, 256, 0, st>>>(kp); break;
        case 6: composite_kernel<6><<<grid, 256, 0, st>>>(kp); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace woit
