// Fused wavelet-OIT frame kernel (steps 1-4 of pipeline.py:131-308 in one pass
// over HBM) and its step-wise / long-pixel / composite companions.
//
// Work decomposition:
//   CTA      = a window of PB consecutive pixels of the band, split into
//              sub-tiles of <= FB fragments / <= T chunks;
//   chunk    = <= 16 consecutive fragments of ONE pixel, owned by one thread;
//   staging  = the sub-tile's fragment fields copied global->shared by TMA
//              bulk copies (cp.async.bulk + mbarrier), read once from HBM;
//   per-pixel reductions (bounds, coefficients, accumulators) combine the
//   chunk partials in a fixed order in fp64 -> deterministic for any tiling.
#include "frame.cuh"

namespace woit {

template <int R>
struct Smem {
    int64_t* offs;
    int64_t* nch;
    int64_t* cb;
    uint32_t* nearu;
    uint32_t* faru;
    double* lo;
    double* den;
    double* vtot;
    uint32_t* chunk;
    float* depth;
    float* alpha;
    float* trans;
    float* rad;
    float* ior;
    float* normal;
    uint8_t* bf;
    int64_t* zfix;
    float* r1;
    unsigned char* r2;
    uint64_t* bar;
};

template <int R>
WOIT_D Smem<R> carve(unsigned char* base, const Layout& L) {
    Smem<R> s;
    s.offs = reinterpret_cast<int64_t*>(base + L.offs);
    s.nch = reinterpret_cast<int64_t*>(base + L.nch);
    s.cb = reinterpret_cast<int64_t*>(base + L.cb);
    s.nearu = reinterpret_cast<uint32_t*>(base + L.nearu);
    s.faru = reinterpret_cast<uint32_t*>(base + L.faru);
    s.lo = reinterpret_cast<double*>(base + L.lo);
    s.den = reinterpret_cast<double*>(base + L.den);
    s.vtot = reinterpret_cast<double*>(base + L.vtot);
    s.chunk = reinterpret_cast<uint32_t*>(base + L.chunk);
    s.depth = reinterpret_cast<float*>(base + L.depth);
    s.alpha = reinterpret_cast<float*>(base + L.alpha);
    s.trans = reinterpret_cast<float*>(base + L.trans);
    s.rad = reinterpret_cast<float*>(base + L.rad);
    s.ior = reinterpret_cast<float*>(base + L.ior);
    s.normal = reinterpret_cast<float*>(base + L.normal);
    s.bf = reinterpret_cast<uint8_t*>(base + L.bf);
    s.zfix = reinterpret_cast<int64_t*>(base + L.zfix);
    s.r1 = reinterpret_cast<float*>(base + L.r1);
    s.r2 = base + L.r2;
    s.bar = reinterpret_cast<uint64_t*>(base + L.bar);
    return s;
}

// chunk descriptor: pixel (7 bits), start within sub-tile (12 bits), length (5 bits)
WOIT_D uint32_t pack_chunk(int q, int start, int len) {
    return (uint32_t)q | ((uint32_t)start << 7) | ((uint32_t)len << 19);
}
WOIT_D void unpack_chunk(uint32_t c, int& q, int& start, int& len) {
    q = (int)(c & 127u);
    start = (int)((c >> 7) & 4095u);
    len = (int)(c >> 19);
}

// Within-chunk iteration starts at a rotation that depends only on the global
// fragment id of the chunk start: it spreads the lanes of a warp over the 32
// smem banks for uniform run lengths and keeps the summation order independent
// of the tiling (bit-identical results for any band split).
WOIT_D int chunk_rotation(int64_t gstart, int len) { return (int)((gstart >> 5) % len); }

// rotation of the chunk loop in the per-pixel combine (same purpose)
WOIT_D int combine_rotation(int64_t gpix, int64_t nch) { return (int)(((gpix * nch) >> 5) % nch); }

// exclusive scan of one int64 per thread across the CTA (T threads)
template <int T>
WOIT_D int64_t block_exclusive_scan(int64_t v, int64_t* warp_sums, int64_t& total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    int64_t base = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < T / 32; ++w) {
        const int64_t s = warp_sums[w];
        base += (w < wid) ? s : 0;
        tot += s;
    }
    total = tot;
    __syncthreads();
    return base + x - v;
}

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

WOIT_D uint32_t stage_issue(const StageSpec& sp, int64_t fa, int64_t fb, int64_t nalloc,
                            int use_tma, uint64_t* bar) {
    int64_t a;
    const int64_t e = stage_bulk_end(sp, fa, fb, nalloc, use_tma, a);
    if (e <= a) return 0;
    const uint32_t bytes = (uint32_t)((e - a) * sp.esize);
    bulk_g2s(sp.s, static_cast<const unsigned char*>(sp.g) + a * sp.esize, bytes, bar);
    return bytes;
}

template <int T>
WOIT_D void stage_scalar(const StageSpec& sp, int64_t fa, int64_t fb, int64_t nalloc, int use_tma) {
    int64_t a;
    const int64_t e = stage_bulk_end(sp, fa, fb, nalloc, use_tma, a);
    const int64_t s0 = e > fa ? e : fa;
    const int words = sp.esize >= 4 ? sp.esize / 4 : 0;
    for (int64_t i = s0 + threadIdx.x; i < fb; i += T) {
        if (words) {
            const float* g = static_cast<const float*>(sp.g) + i * words;
            float* d = static_cast<float*>(sp.s) + (i - a) * words;
            for (int w = 0; w < words; ++w) d[w] = g[w];
        } else {
            static_cast<uint8_t*>(sp.s)[i - a] = static_cast<const uint8_t*>(sp.g)[i];
        }
    }
}

// ---------------------------------------------------------------------------

template <int R>
__global__ void __launch_bounds__(RT<R>::T, 1) frame_kernel(const KParams kp) {
    using G = RT<R>;
    constexpr int T = G::T, PB = G::PB, FB = G::FB, V = G::V, S = G::S, CH = G::CH, VP = G::VP;
    constexpr int M = S;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t ph = kp.phases;
    const int flags = kp.p.flags;
    const Layout L = make_layout<R>(ph, flags);
    Smem<R> sm = carve<R>(smem_raw, L);
    __shared__ int64_t warp_sums[T / 32];

    const int tid = threadIdx.x;
    const int64_t w0 = (int64_t)blockIdx.x * PB;
    const int nq = (int)((kp.f.npix - w0) < PB ? (kp.f.npix - w0) : PB);
    if (nq <= 0) return;

    const bool do_frag = ph & (PH_BOUNDS | PH_BUILD | PH_EVAL);
    const bool do_at = ph & (PH_BUILD | PH_EVAL);
    const bool do_eval = ph & PH_EVAL;
    const bool refr = do_eval && (flags & WOIT_REFRACTION);
    const bool cube = flags & WOIT_CUBE_TRANSMISSION;
    const bool bfonly = cube && (flags & WOIT_CUBE_BACKFACE_ONLY);
    const bool need_ior = do_at && (cube || refr);
    const bool keep_z = (ph & PH_BUILD) && do_eval;
    const int64_t nalloc = kp.f.nfrag;

    if (tid == 0) mbar_init(sm.bar, 1);
    for (int q = tid; q <= nq; q += T) sm.offs[q] = kp.f.offsets[w0 + q];
    __syncthreads();
    // chunks per pixel and their window prefix
    int64_t my_nch = 0;
    if (tid < nq) {
        const int64_t run = sm.offs[tid + 1] - sm.offs[tid];
        my_nch = (run + CH - 1) / CH;
        sm.nch[tid] = my_nch;
    }
    int64_t tot;
    const int64_t ex = block_exclusive_scan<T>(my_nch, warp_sums, tot);
    if (tid < nq) sm.cb[tid] = ex;
    if (tid == 0) sm.cb[nq] = tot;
    __syncthreads();

    uint32_t parity = 0;
    int q0 = 0;
    while (q0 < nq) {
        // sub-tile end: largest q1 with <= FB fragments and <= T chunks
        const int cand = tid + 1;
        const bool fits = cand > q0 && cand <= nq && (sm.offs[cand] - sm.offs[q0]) <= FB &&
                          (sm.cb[cand] - sm.cb[q0]) <= T;
        const int cnt = __syncthreads_count(fits);
        if (cnt == 0) {
            // a single pixel deeper than FB fragments: handled by long_pixel_kernel
            if (tid == 0) {
                const unsigned long long idx =
                    atomicAdd(reinterpret_cast<unsigned long long*>(kp.long_list), 1ull);
                if ((int64_t)idx < kp.long_cap) kp.long_list[1 + idx] = w0 + q0;
            }
            q0 += 1;
            continue;
        }
        const int q1 = q0 + cnt;
        const int nqs = q1 - q0;
        const int64_t fa = sm.offs[q0], fb = sm.offs[q1];
        const int C = (int)(sm.cb[q1] - sm.cb[q0]);
        const int64_t a4 = fa & ~(int64_t)3, a16 = fa & ~(int64_t)15;
        const int sh4 = (int)(fa - a4);  // staging index of fragment fa (granule-4 arrays)

        // ---- 1. stage fragment fields (TMA bulk) ---------------------------------
        StageSpec specs[7];
        int nspec = 0;
        if (do_frag) specs[nspec++] = {kp.f.depth, sm.depth, 4, 4};
        if (do_at) specs[nspec++] = {kp.f.alpha, sm.alpha, 4, 4};
        if (do_at) specs[nspec++] = {kp.f.trans, sm.trans, 12, 4};
        if (do_eval) specs[nspec++] = {kp.f.radiance, sm.rad, 12, 4};
        if (need_ior && kp.f.ior) specs[nspec++] = {kp.f.ior, sm.ior, 4, 4};
        if (refr) specs[nspec++] = {kp.f.normal, sm.normal, 12, 4};
        if (bfonly && kp.f.backface) specs[nspec++] = {kp.f.backface, sm.bf, 1, 16};
        if (kp.use_tma && nspec > 0 && tid == 0) {
            bulk_wait_read_all();  // previous sub-tile's v̂ store has left smem
            fence_proxy_async();
            uint32_t tx = 0;
            for (int i = 0; i < nspec; ++i) {
                int64_t a;
                const int64_t e = stage_bulk_end(specs[i], fa, fb, nalloc, 1, a);
                if (e > a) tx += (uint32_t)((e - a) * specs[i].esize);
            }
            mbar_arrive_expect_tx(sm.bar, tx);
            for (int i = 0; i < nspec; ++i) stage_issue(specs[i], fa, fb, nalloc, 1, sm.bar);
        }
        for (int i = 0; i < nspec; ++i) stage_scalar<T>(specs[i], fa, fb, nalloc, kp.use_tma);
        if (need_ior && !kp.f.ior)
            for (int i = tid; i < (int)(fb - fa); i += T) sm.ior[sh4 + i] = 1.0f;
        if (bfonly && !kp.f.backface)
            for (int i = tid; i < (int)(fb - fa); i += T) sm.bf[(int)(fa - a16) + i] = 0;

        // ---- 2. chunk table + per-pixel init (overlaps the copies) -----------------
        if (tid < nqs) {
            const int q = q0 + tid;
            const int64_t run = sm.offs[q + 1] - sm.offs[q];
            const int nc = (int)sm.nch[q];
            const int base = (int)(sm.cb[q] - sm.cb[q0]);
            const int rel = (int)(sm.offs[q] - fa);
            if (nc > 0) {
                const int len0 = (int)(run / nc), extra = (int)(run % nc);
                int st = rel;
                for (int i = 0; i < nc; ++i) {
                    const int len = len0 + (i < extra ? 1 : 0);
                    sm.chunk[base + i] = pack_chunk(tid, st, len);
                    st += len;
                }
            }
            const int64_t p = w0 + q;
            if (ph & PH_BOUNDS) {
                if (ph & PH_BOUNDS_ACC) {
                    sm.nearu[tid] = f2ord(kp.b.near[p]);
                    sm.faru[tid] = f2ord(kp.b.far[p]);
                } else {
                    sm.nearu[tid] = f2ord(INFINITY);
                    sm.faru[tid] = f2ord(-INFINITY);
                }
            } else {
                sm.nearu[tid] = f2ord(kp.b.near[p]);
                sm.faru[tid] = f2ord(kp.b.far[p]);
            }
        }
        if (kp.use_tma && nspec > 0) {
            mbar_wait(sm.bar, parity);
            parity ^= 1u;
        }
        __syncthreads();

        // ---- 3. bounds (step1) ------------------------------------------------------
        if (ph & PH_BOUNDS) {
            if (tid < C) {
                int q, st, len;
                unpack_chunk(sm.chunk[tid], q, st, len);
                float mn = INFINITY, mx = -INFINITY;
                for (int j = 0; j < len; ++j) {
                    const float x = sm.depth[sh4 + st + j];
                    mn = fminf(mn, x);
                    mx = fmaxf(mx, x);
                }
                atomicMin(&sm.nearu[q], f2ord(mn));
                atomicMax(&sm.faru[q], f2ord(mx));
            }
            __syncthreads();
        }
        if (tid < nqs) {
            const float nf = ord2f(sm.nearu[tid]), ff = ord2f(sm.faru[tid]);
            const int64_t p = w0 + q0 + tid;
            if ((ph & PH_BOUNDS) && kp.b.near) kp.b.near[p] = nf;
            if ((ph & PH_BOUNDS) && kp.b.far) kp.b.far[p] = ff;
            const DepthMap m = depth_map(nf, ff, R);
            sm.lo[tid] = m.lo;
            sm.den[tid] = m.den;
        }
        __syncthreads();

        // ---- 4. build (step2): chunk partials -> r1[v][c] --------------------------
        float* part = sm.r1;
        double* coef64 = reinterpret_cast<double*>(sm.r2);
        if (ph & PH_BUILD) {
            if (tid < C) {
                int q, st, len;
                unpack_chunk(sm.chunk[tid], q, st, len);
                const DepthMap m{sm.lo[q], sm.den[q]};
                for (int v = 6; v < V; ++v) part[v * T + tid] = 0.0f;
                float s0[3] = {0.f, 0.f, 0.f}, s1[3] = {0.f, 0.f, 0.f};
                const int rot = chunk_rotation(kp.f.frag_base + fa + st, len);
                for (int j = 0; j < len; ++j) {
                    int jj = j + rot;
                    if (jj >= len) jj -= len;
                    const int fr = st + jj;          // fragment index relative to fa
                    const int si = sh4 + fr;         // staging index
                    const double z = normalized_z(sm.depth[si], m);
                    const int64_t zi = z_fixed(z);
                    if (keep_z) sm.zfix[fr] = zi;
                    const float al = sm.alpha[si];
                    bool cb_ = false;
                    if (cube) {
                        const float io = sm.ior[si];
                        cb_ = io > 1.0f && (!bfonly || sm.bf[(int)(fa - a16) + fr] != 0);
                    }
                    float a[3];
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) a[ch] = absorbance_ch(al, sm.trans[3 * si + ch], cb_);
                    const float one_m_z = fixed_to_unit((int64_t(1) << kZBits) - zi, kZBits);
                    const float psi0 = level_psi(zi, 0);
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) {
                        s0[ch] += a[ch] * one_m_z;
                        s1[ch] -= a[ch] * psi0;
                    }
#pragma unroll
                    for (int n = 1; n <= R; ++n) {
                        const int k = slot_offset(zi, n);
                        const float psi = level_psi(zi, n) * kInvSqrt2PowF[n];
                        float* col = part + ((1 << n) + k) * 3 * T + tid;
#pragma unroll
                        for (int ch = 0; ch < 3; ++ch) col[ch * T] -= a[ch] * psi;
                    }
                }
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    part[ch * T + tid] = s0[ch];
                    part[(3 + ch) * T + tid] = s1[ch];
                }
            }
            __syncthreads();
            // combine chunk partials per (pixel, value) in fp64, fixed order
            for (int idx = tid; idx < nqs * V; idx += T) {
                const int v = idx / nqs, ql = idx - v * nqs;
                const int q = q0 + ql;
                const int64_t nc = sm.nch[q];
                const int cbq = (int)(sm.cb[q] - sm.cb[q0]);
                double acc = (ph & PH_BUILD_ACC) ? (double)kp.b.coeffs[(w0 + q) * V + v] : 0.0;
                if (nc > 0) {
                    const int r = combine_rotation(kp.f.pixel_base + w0 + q, nc);
                    const float* pv = part + v * T + cbq;
                    for (int i = 0; i < nc; ++i) {
                        int ii = i + r;
                        if (ii >= nc) ii -= (int)nc;
                        acc += (double)pv[ii];
                    }
                }
                coef64[ql * VP + v] = acc;
            }
            __syncthreads();
            if (flags & WOIT_PACKED_STORAGE) {
                for (int idx = tid; idx < nqs * S; idx += T) {
                    const int ql = idx / S, s = idx - ql * S;
                    double* c = coef64 + ql * VP + 3 * s;
                    double mag[3] = {fabs(c[0]), fabs(c[1]), fabs(c[2])}, rt[3];
                    rgb9e5_unpack_impl(rgb9e5_pack_impl(mag), rt);
                    const double sg = s == 0 ? 1.0 : -1.0;
                    c[0] = sg * rt[0];
                    c[1] = sg * rt[1];
                    c[2] = sg * rt[2];
                }
                __syncthreads();
            }
            if (kp.b.coeffs) {
                for (int idx = tid; idx < nqs * V; idx += T) {
                    const int ql = idx / V, v = idx - ql * V;
                    kp.b.coeffs[(w0 + q0) * V + idx] = (float)coef64[ql * VP + v];
                }
            }
        } else if (ph & (PH_EVAL | PH_COMPOSITE)) {
            for (int idx = tid; idx < nqs * V; idx += T) {
                const int ql = idx / V, v = idx - ql * V;
                coef64[ql * VP + v] = (double)kp.b.coeffs[(w0 + q0) * V + idx];
            }
            __syncthreads();
        }

        // ---- 5. per-pixel total transmittance and cell staircase ------------------
        float* cells = sm.r1;  // r1 is free again (partials consumed)
        if (ph & (PH_EVAL | PH_COMPOSITE)) {
            for (int idx = tid; idx < nqs * 3; idx += T) {
                const int ql = idx / 3, ch = idx - ql * 3;
                const double* c = coef64 + ql * VP;
                double at = c[ch];
#pragma unroll
                for (int n = 0; n <= R; ++n) at = dsub(at, dmul(kSqrt2Pow[n], c[((2 << n) - 1) * 3 + ch]));
                sm.vtot[idx] = exp(-fmax(at, 0.0));
            }
            if (do_eval) {
                for (int idx = tid; idx < nqs * V; idx += T) {
                    const int ql = idx / V, w = idx - ql * V;
                    const int cell = w / 3, ch = w - cell * 3;
                    const double* c = coef64 + ql * VP;
                    double val = c[ch];
#pragma unroll
                    for (int n = 0; n <= R; ++n) {
                        const int mm = R + 1 - n;
                        const double sg = ((cell >> (mm - 1)) & 1) ? -1.0 : 1.0;
                        val = dadd(val, dmul(dmul(kSqrt2Pow[n], sg), c[((1 << n) + (cell >> mm)) * 3 + ch]));
                    }
                    cells[idx] = (float)val;
                }
            }
            __syncthreads();
        }

        // ---- 6. evaluate (step3): v̂ per fragment, chunk accumulators --------------
        float* accp = reinterpret_cast<float*>(sm.r2);  // [8][T], coef64 consumed
        if (do_eval) {
            if (tid < C) {
                int q, st, len;
                unpack_chunk(sm.chunk[tid], q, st, len);
                const DepthMap m{sm.lo[q], sm.den[q]};
                const float* cq = cells + q * V;
                float ac[3] = {0.f, 0.f, 0.f}, wg[3] = {0.f, 0.f, 0.f};
                double ro[2] = {0.0, 0.0};
                double d[3] = {0.0, 0.0, 0.0}, topq = INFINITY;
                const int64_t p = w0 + q0 + q;
                if (refr) {
                    ray_dir(kp, kp.f.pixel_base + p, d);
                    topq = kp.f.opaque_depth ? (double)kp.f.opaque_depth[p] : INFINITY;
                }
                const int rot = chunk_rotation(kp.f.frag_base + fa + st, len);
                for (int j = 0; j < len; ++j) {
                    int jj = j + rot;
                    if (jj >= len) jj -= len;
                    const int fr = st + jj;
                    const int si = sh4 + fr;
                    const int64_t zi = keep_z ? sm.zfix[fr] : z_fixed(normalized_z(sm.depth[si], m));
                    int c0, c1;
                    float t;
                    eval_cells(zi, R, c0, c1, t);
                    const float al = sm.alpha[si];
                    bool cb_ = false;
                    float io = 1.0f;
                    if (need_ior) {
                        io = sm.ior[si];
                        cb_ = cube && io > 1.0f && (!bfonly || sm.bf[(int)(fa - a16) + fr] != 0);
                    }
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) {
                        const float A = fmaxf((1.0f - t) * cq[c0 * 3 + ch] + t * cq[c1 * 3 + ch], 0.0f);
                        const float vh = expf(-A);
                        const float L = sm.rad[3 * si + ch];
                        ac[ch] += (L * al) * vh;
                        wg[ch] += opacity_ch(al, sm.trans[3 * si + ch], cb_) * vh;
                        sm.rad[3 * si + ch] = vh;  // v̂ replaces radiance in place
                    }
                    if (refr && io > 1.0f) {
                        const float nrm[3] = {sm.normal[3 * si], sm.normal[3 * si + 1], sm.normal[3 * si + 2]};
                        double off[2];
                        refraction_offset(kp, d, topq, sm.depth[si], nrm, io, off);
                        ro[0] += off[0];
                        ro[1] += off[1];
                    }
                }
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    accp[ch * T + tid] = ac[ch];
                    accp[(3 + ch) * T + tid] = wg[ch];
                }
                accp[6 * T + tid] = (float)ro[0];
                accp[7 * T + tid] = (float)ro[1];
            }
            fence_proxy_async();  // v̂ in smem becomes visible to the bulk store
            __syncthreads();
            // v̂ store: aligned interior by one bulk copy, ragged ends by threads
            if (kp.b.vhat) {
                const int64_t i0 = (fa + 3) & ~(int64_t)3, i1 = fb & ~(int64_t)3;
                const bool bulk = kp.use_tma && i1 > i0;
                if (bulk && tid == 0) {
                    bulk_s2g(kp.b.vhat + 3 * i0, sm.rad + 3 * (i0 - a4), (uint32_t)(12 * (i1 - i0)));
                    bulk_commit();
                }
                for (int64_t f = fa + tid; f < fb; f += T) {
                    if (bulk && f >= i0 && f < i1) continue;
                    const int si = (int)(f - a4);
                    kp.b.vhat[3 * f] = sm.rad[3 * si];
                    kp.b.vhat[3 * f + 1] = sm.rad[3 * si + 1];
                    kp.b.vhat[3 * f + 2] = sm.rad[3 * si + 2];
                }
            }
        }

        // ---- 7. per-pixel accumulators + composite (step4) -------------------------
        if (tid < nqs) {
            const int q = q0 + tid;
            const int64_t p = w0 + q;
            double acc[3] = {0, 0, 0}, wgt[3] = {0, 0, 0}, ro[2] = {0, 0};
            const bool acc_in = (ph & PH_EVAL_ACC) || ((ph & PH_COMPOSITE) && !do_eval);
            if (acc_in) {
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    acc[ch] = kp.b.accum[p * 3 + ch];
                    wgt[ch] = kp.b.weight[p * 3 + ch];
                }
                if (kp.b.refraction_offset) {
                    ro[0] = kp.b.refraction_offset[p * 2];
                    ro[1] = kp.b.refraction_offset[p * 2 + 1];
                }
            }
            if (do_eval) {
                const int64_t nc = sm.nch[q];
                const int cbq = (int)(sm.cb[q] - sm.cb[q0]);
                for (int i = 0; i < nc; ++i) {
                    const int c = cbq + i;
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) {
                        acc[ch] += (double)accp[ch * T + c];
                        wgt[ch] += (double)accp[(3 + ch) * T + c];
                    }
                    ro[0] += (double)accp[6 * T + c];
                    ro[1] += (double)accp[7 * T + c];
                }
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
                composite_pixel(kp, p, acc, wgt, ro[0], ro[1], sm.vtot + 3 * tid, out);
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) kp.b.output[p * 3 + ch] = out[ch];
            }
        }
        __syncthreads();
        q0 = q1;
    }
    if (tid == 0) bulk_wait_all();
}

// ---------------------------------------------------------------------------
// pixels deeper than one sub-tile: one CTA per pixel, fragments streamed from
// global memory (coalesced), per-thread fp64 accumulators, fixed-order combine.

constexpr int kLongT = 256;

template <int R>
__global__ void __launch_bounds__(kLongT) long_pixel_kernel(const KParams kp) {
    constexpr int S = 1 << (R + 1), V = 3 * S, M = S;
    constexpr int TL = R <= 3 ? kLongT : (kLongT >> (R - 3));  // keep acc64 <= 96 KB
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* acc64 = reinterpret_cast<double*>(smem_raw);      // [V][TL]
    double* coef = acc64 + V * TL;                              // [V]
    float* cells = reinterpret_cast<float*>(coef + V);          // [V]
    __shared__ double red[8][kLongT];
    __shared__ double vt[3];
    __shared__ float nf_s, ff_s;
    const int tid = threadIdx.x;
    const uint32_t ph = kp.phases;
    const int flags = kp.p.flags;
    const bool cube = flags & WOIT_CUBE_TRANSMISSION;
    const bool bfonly = cube && (flags & WOIT_CUBE_BACKFACE_ONLY);
    const bool refr = (ph & PH_EVAL) && (flags & WOIT_REFRACTION);
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
        const DepthMap m = depth_map(nf_s, ff_s, R);
        // build
        if (ph & PH_BUILD) {
            if (tid < TL) {
                for (int v = 0; v < V; ++v) acc64[v * TL + tid] = 0.0;
                for (int64_t f = s + tid; f < e; f += TL) {
                    const double z = normalized_z(kp.f.depth[f], m);
                    const int64_t zi = z_fixed(z);
                    const float al = kp.f.alpha[f];
                    bool cb_ = false;
                    if (cube) {
                        const float io = kp.f.ior ? kp.f.ior[f] : 1.0f;
                        cb_ = io > 1.0f && (!bfonly || (kp.f.backface && kp.f.backface[f]));
                    }
                    float a[3];
                    for (int ch = 0; ch < 3; ++ch) a[ch] = absorbance_ch(al, kp.f.trans[3 * f + ch], cb_);
                    const float one_m_z = fixed_to_unit((int64_t(1) << kZBits) - zi, kZBits);
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
                for (int sl = tid; sl < S; sl += kLongT) {
                    double mag[3] = {fabs(coef[3 * sl]), fabs(coef[3 * sl + 1]), fabs(coef[3 * sl + 2])}, rt[3];
                    rgb9e5_unpack_impl(rgb9e5_pack_impl(mag), rt);
                    const double sg = sl == 0 ? 1.0 : -1.0;
                    for (int ch = 0; ch < 3; ++ch) coef[3 * sl + ch] = sg * rt[ch];
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
        double lac[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (ph & PH_EVAL) {
            double d[3] = {0, 0, 0}, topq = INFINITY;
            if (refr) {
                ray_dir(kp, kp.f.pixel_base + p, d);
                topq = kp.f.opaque_depth ? (double)kp.f.opaque_depth[p] : INFINITY;
            }
            for (int64_t f = s + tid; f < e; f += kLongT) {
                const int64_t zi = z_fixed(normalized_z(kp.f.depth[f], m));
                int c0, c1;
                float t;
                eval_cells(zi, R, c0, c1, t);
                const float al = kp.f.alpha[f];
                const float io = kp.f.ior ? kp.f.ior[f] : 1.0f;
                const bool cb_ = cube && io > 1.0f && (!bfonly || (kp.f.backface && kp.f.backface[f]));
                for (int ch = 0; ch < 3; ++ch) {
                    const float A = fmaxf((1.0f - t) * cells[c0 * 3 + ch] + t * cells[c1 * 3 + ch], 0.0f);
                    const float vh = expf(-A);
                    lac[ch] += (double)((kp.f.radiance[3 * f + ch] * al) * vh);
                    lac[3 + ch] += (double)(opacity_ch(al, kp.f.trans[3 * f + ch], cb_) * vh);
                    if (kp.b.vhat) kp.b.vhat[3 * f + ch] = vh;
                }
                if (refr && io > 1.0f) {
                    const float nrm[3] = {kp.f.normal[3 * f], kp.f.normal[3 * f + 1], kp.f.normal[3 * f + 2]};
                    double off[2];
                    refraction_offset(kp, d, topq, kp.f.depth[f], nrm, io, off);
                    lac[6] += off[0];
                    lac[7] += off[1];
                }
            }
        }
        for (int k = 0; k < 8; ++k) red[k][tid] = lac[k];
        __syncthreads();
        for (int o = kLongT / 2; o > 0; o >>= 1) {
            if (tid < o)
                for (int k = 0; k < 8; ++k) red[k][tid] += red[k][tid + o];
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
            if (ph & PH_EVAL) {
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
                composite_pixel(kp, p, acc, wgt, ro[0], ro[1], vt, out);
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

template <int R>
cudaError_t launch_rank(const KParams& kp, cudaStream_t st) {
    using G = RT<R>;
    const Layout L = make_layout<R>(kp.phases, kp.p.flags);
    cudaError_t err = cudaFuncSetAttribute(frame_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)L.total);
    if (err != cudaSuccess) return err;
    const int64_t grid = (kp.f.npix + G::PB - 1) / G::PB;
    if (grid > 0) {
        frame_kernel<R><<<(unsigned)grid, G::T, L.total, st>>>(kp);
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
    }
    const size_t ls = long_smem_bytes<R>();
    err = cudaFuncSetAttribute(long_pixel_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ls);
    if (err != cudaSuccess) return err;
    if (kp.f.nfrag > G::FB) {  // a pixel deeper than FB can only exist if nfrag > FB
        long_pixel_kernel<R><<<64, kLongT, ls, st>>>(kp);
        err = cudaGetLastError();
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
__global__ void composite_kernel(const KParams kp) {
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
    float out[3];
    composite_pixel(kp, p, acc, wgt, ox, oy, vt, out);
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
            const int64_t zi = z_fixed(z);
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
