// On-device fragment producer: the reference's vectorised caster cast_frame
// (scene.py:430-630) for planes / panes, spheres (entry + exit), fog slabs
// (sliced), particle clouds (camera-facing discs) and opaque backdrops, emitting
// the CSR stream the frame kernels read -- SURVEY.md §8(f) rank 3.
//
// One thread per pixel casts its primary ray (the reference's camera_rays
// arithmetic, f64) against the primitives in scene order; a pixel's fragments come
// out in (primitive, sub-index) order, which is cast_frame's lexsort((sub, prim,
// pixel)) order. Two passes: count -> CUB exclusive scan -> fill. All geometry is
// float64 and rounded to fp32 once on output. Particle discs are tested only in
// the conservative screen box the reference derives per particle (computed on the
// host with its arithmetic and passed in), so culling matches cast_frame exactly.
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "internal.cuh"

namespace woit {
namespace {

constexpr double kRayEps = 1e-9;  // scene.py:41

WOIT_D double dot3(const double a[3], const double b[3]) { return dadd(dadd(dmul(a[0], b[0]), dmul(a[1], b[1])), dmul(a[2], b[2])); }

// camera_rays (scene.py:199-212) for pixel (px, py)
WOIT_D void primary_ray(const woit_scene_t& s, int W, int H, int px, int py, double d[3]) {
    const double u = dmul(dmul(dsub(ddiv(dmul(2.0, dadd((double)px, 0.5)), (double)W), 1.0), s.tan_half), s.aspect);
    const double v = dmul(dsub(1.0, ddiv(dmul(2.0, dadd((double)py, 0.5)), (double)H)), s.tan_half);
#pragma unroll
    for (int i = 0; i < 3; ++i) d[i] = dadd(dadd(s.forward[i], dmul(u, s.right[i])), dmul(v, s.up[i]));
    const double nrm = sqrt(dadd(dadd(dmul(d[0], d[0]), dmul(d[1], d[1])), dmul(d[2], d[2])));
#pragma unroll
    for (int i = 0; i < 3; ++i) d[i] = ddiv(d[i], nrm);
}

struct Out {
    float *depth, *alpha, *trans, *rad, *normal, *ior;
    uint8_t* bf;
};

template <bool FILL>
struct Emitter {
    int64_t k;
    Out o;
    bool live;  // false: a lane past the last pixel (emits nothing)
    WOIT_D void emit(double depth, double alpha, const double tr[3], const double rd[3], const double nr[3], double ior,
                     bool backface) {
        if (!live) return;
        if (FILL) {
            o.depth[k] = (float)depth;
            o.alpha[k] = (float)alpha;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                o.trans[3 * k + c] = (float)tr[c];
                o.rad[3 * k + c] = (float)rd[c];
                o.normal[3 * k + c] = (float)nr[c];
            }
            o.ior[k] = (float)ior;
            o.bf[k] = backface ? 1 : 0;
        }
        ++k;
    }
};

// _particle_alpha (scene.py:250-254)
WOIT_D double particle_alpha(int profile, double peak, double x) {
    if (profile == 0) return dmul(peak, exp(dmul(dmul(-4.0, x), x)));
    double u = ddiv(dsub(1.0, x), 0.25);
    u = fmin(fmax(u, 0.0), 1.0);
    return dmul(dmul(dmul(peak, u), u), dsub(3.0, dmul(2.0, u)));
}

template <bool FILL>
__global__ void __launch_bounds__(128) cast_kernel(const woit_scene_t s, int W, int H, int64_t* counts,
                                                   const int64_t* __restrict__ offsets, Out o, float* opaque_depth,
                                                   float* opaque_color) {
    const int64_t npix = (int64_t)W * H;
    const int lane = threadIdx.x & 31;
    // warp-uniform trip count (the fog slabs are written by the whole warp); lanes past
    // the end run the geometry of the last pixel and emit nothing
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t pw = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); pw < npix; pw += stride) {
        const bool live = pw + lane < npix;
        const int64_t p = live ? pw + lane : npix - 1;
        const int px = (int)(p % W), py = (int)(p / W);
        double d[3];
        primary_ray(s, W, H, px, py, d);
        const double dirf = dot3(d, s.forward);
        // nearest opaque backdrop (_opaque_frame, scene.py:430-458), else the background
        double ot = INFINITY;
        double oc[3];
        const bool bodd = s.bg_has_checker && (((px / s.bg_cell) + (py / s.bg_cell)) % 2 == 1);
#pragma unroll
        for (int c = 0; c < 3; ++c) oc[c] = bodd ? s.bg_checker[c] : s.bg_color[c];
        for (int i = 0; i < s.nprims; ++i) {
            const woit_prim_t& pr = s.prims[i];
            if (pr.kind != WOIT_PRIM_BACKDROP) continue;
            const double t = dirf > 0.0 ? ddiv(pr.d, dirf) : INFINITY;
            if (!(t > kRayEps && t < ot)) continue;
            bool odd = false;
            if (pr.flags & 2) {
                const double rel[3] = {dmul(t, d[0]), dmul(t, d[1]), dmul(t, d[2])};
                const double cx = floor(ddiv(dot3(rel, s.right), pr.cell));
                const double cy = floor(ddiv(dot3(rel, s.up), pr.cell));
                odd = fmod(dadd(cx, cy), 2.0) != 0.0;  // (cx + cy) % 2 == 1 for integral floats
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) oc[c] = odd ? pr.checker[c] : pr.color[c];
            ot = t;
        }
        if (FILL && live) {
            opaque_depth[p] = (float)ot;
#pragma unroll
            for (int c = 0; c < 3; ++c) opaque_color[3 * p + c] = (float)oc[c];
        }
        Emitter<FILL> em{FILL && live ? offsets[p] : 0, o, live};
        const double nf[3] = {-s.forward[0], -s.forward[1], -s.forward[2]};
        for (int i = 0; i < s.nprims; ++i) {
            const woit_prim_t& pr = s.prims[i];
            if (pr.kind == WOIT_PRIM_PLANE) {
                const double t = dirf > 0.0 ? ddiv(pr.d, dirf) : INFINITY;
                if (!(t > kRayEps && t < ot)) continue;
                if (pr.flags & 1) {
                    const double rel[3] = {dmul(t, d[0]), dmul(t, d[1]), dmul(t, d[2])};
                    const double lx = dsub(dot3(rel, s.right), pr.pcenter[0]);
                    const double ly = dsub(dot3(rel, s.up), pr.pcenter[1]);
                    if (!(fabs(lx) <= pr.extent[0] && fabs(ly) <= pr.extent[1])) continue;
                }
                em.emit(t, pr.alpha, pr.trans, pr.radiance, nf, pr.ior, false);
            } else if (pr.kind == WOIT_PRIM_SPHERE) {
                const double L[3] = {dsub(pr.center[0], s.origin[0]), dsub(pr.center[1], s.origin[1]),
                                     dsub(pr.center[2], s.origin[2])};
                const double tca = dot3(d, L);
                const double d2 = dsub(dot3(L, L), dmul(tca, tca));
                const double r2 = dmul(pr.radius, pr.radius);
                if (!(d2 < r2)) continue;
                const double thc = sqrt(dsub(r2, d2));
                for (int sub = 0; sub < 2; ++sub) {
                    const bool back = sub == 1;
                    const double t = back ? dadd(tca, thc) : dsub(tca, thc);
                    if (!(t > kRayEps && t < ot)) continue;
                    double n[3];
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const double q = dadd(s.origin[c], dmul(t, d[c]));
                        n[c] = ddiv(back ? dsub(pr.center[c], q) : dsub(q, pr.center[c]), pr.radius);
                    }
                    const double nn = sqrt(dadd(dadd(dmul(n[0], n[0]), dmul(n[1], n[1])), dmul(n[2], n[2])));
#pragma unroll
                    for (int c = 0; c < 3; ++c) n[c] = ddiv(n[c], nn);
                    em.emit(t, pr.alpha, pr.trans, pr.radiance, n, pr.ior, back);
                }
            } else if (pr.kind == WOIT_PRIM_FOG) {
                double ta = dirf > 0.0 ? ddiv(pr.near, dirf) : INFINITY;
                double tb = dirf > 0.0 ? ddiv(pr.far, dirf) : INFINITY;
                ta = fmax(ta, kRayEps);
                tb = fmin(tb, ot);
                const int cnt = (em.live && tb > ta) ? pr.count : 0;
                if (!FILL) {
                    em.k += cnt;
                    continue;
                }
                double delta = 0.0;
                float trf[3] = {0.f, 0.f, 0.f}, rdf[3] = {0.f, 0.f, 0.f};
                if (cnt) {
                    delta = ddiv(dsub(tb, ta), (double)pr.count);
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const double tr = exp(dmul(-pr.sigma[c], delta));
                        trf[c] = (float)tr;
                        rdf[c] = (float)dmul(pr.color[c], dsub(1.0, tr));
                    }
                }
                // The slices of every lane's slab are written by the whole warp, one lane's
                // run at a time: consecutive threads store consecutive fragments (coalesced).
                // Slice j's depth is ta + (j + 1/2) delta, as the per-lane loop computed it.
                for (int L = 0; L < 32; ++L) {
                    const int n = __shfl_sync(0xffffffffu, cnt, L);
                    if (n == 0) continue;
                    const int64_t k0 = __shfl_sync(0xffffffffu, em.k, L);
                    const double ta_ = __shfl_sync(0xffffffffu, ta, L), de = __shfl_sync(0xffffffffu, delta, L);
                    float t3[3], r3[3];
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        t3[c] = __shfl_sync(0xffffffffu, trf[c], L);
                        r3[c] = __shfl_sync(0xffffffffu, rdf[c], L);
                    }
                    for (int j = lane; j < n; j += 32) {
                        const int64_t k = k0 + j;
                        o.depth[k] = (float)dadd(ta_, dmul(dadd((double)j, 0.5), de));
                        o.alpha[k] = 1.0f;
                        o.ior[k] = 1.0f;
                        o.bf[k] = 0;
                    }
                    float* tr3 = o.trans + 3 * k0;
                    float* rd3 = o.rad + 3 * k0;
                    float* nr3 = o.normal + 3 * k0;
                    for (int e = lane; e < 3 * n; e += 32) {
                        const int c = e % 3;
                        tr3[e] = t3[c];
                        rd3[e] = r3[c];
                        nr3[e] = c == 2 ? -1.0f : 0.0f;
                    }
                }
                em.k += cnt;
            } else if (pr.kind == WOIT_PRIM_PARTICLES) {
                const double pr2 = dmul(pr.particle_radius, pr.particle_radius);
                for (int k = 0; k < pr.count; ++k) {
                    const int32_t* b = pr.box + 4 * k;
                    if (px < b[0] || px > b[1] || py < b[2] || py > b[3]) continue;
                    const double P[3] = {pr.positions[3 * k], pr.positions[3 * k + 1], pr.positions[3 * k + 2]};
                    double n[3] = {dsub(s.origin[0], P[0]), dsub(s.origin[1], P[1]), dsub(s.origin[2], P[2])};
                    const double nn = sqrt(dot3(n, n));
                    if (nn <= kRayEps) continue;
#pragma unroll
                    for (int c = 0; c < 3; ++c) n[c] = ddiv(n[c], nn);
                    const double den = dot3(d, n);
                    if (!(den < -kRayEps)) continue;
                    const double po[3] = {dsub(P[0], s.origin[0]), dsub(P[1], s.origin[1]), dsub(P[2], s.origin[2])};
                    const double t = ddiv(dot3(po, n), den);
                    double qp[3];
#pragma unroll
                    for (int c = 0; c < 3; ++c) qp[c] = dsub(dadd(s.origin[c], dmul(t, d[c])), P[c]);
                    const double rho2 = dadd(dadd(dmul(qp[0], qp[0]), dmul(qp[1], qp[1])), dmul(qp[2], qp[2]));
                    if (!(t > kRayEps && t < ot && rho2 < pr2)) continue;
                    const double a = particle_alpha(pr.profile, pr.alpha, ddiv(sqrt(rho2), pr.particle_radius));
                    const double sc = pr.radiance_scale[k];
                    const double rd[3] = {dmul(pr.radiance[0], sc), dmul(pr.radiance[1], sc), dmul(pr.radiance[2], sc)};
                    em.emit(t, a, pr.trans, rd, n, pr.ior, false);
                }
            }
        }
        if (!FILL && live) counts[p] = em.k;
    }
}

unsigned cast_grid(int64_t n) {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t g = (n + 127) / 128;
    return (unsigned)(g < 32 * sms ? (g > 0 ? g : 1) : 32 * sms);
}

size_t scan_temp(int64_t npix) {
    size_t t = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, t, (const int64_t*)nullptr, (int64_t*)nullptr, (int)(npix + 1));
    return t;
}

}  // namespace

size_t cast_workspace(int64_t npix) { return (size_t)(npix + 1) * 8 + scan_temp(npix) + 256; }

cudaError_t cast_count(const woit_scene_t& s, int W, int H, int64_t* offsets, void* ws, cudaStream_t st) {
    const int64_t npix = (int64_t)W * H;
    int64_t* counts = reinterpret_cast<int64_t*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
    void* temp = counts + npix + 1;
    cudaError_t e = cudaMemsetAsync(counts + npix, 0, sizeof(int64_t), st);
    if (e != cudaSuccess) return e;
    cast_kernel<false><<<cast_grid(npix), 128, 0, st>>>(s, W, H, counts, nullptr, Out{}, nullptr, nullptr);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    size_t tb = scan_temp(npix);
    return cub::DeviceScan::ExclusiveSum(temp, tb, counts, offsets, (int)(npix + 1), st);
}

cudaError_t cast_fill(const woit_scene_t& s, int W, int H, const int64_t* offsets, float* depth, float* alpha,
                      float* trans, float* rad, float* normal, float* ior, uint8_t* bf, float* od, float* oc,
                      cudaStream_t st) {
    const int64_t npix = (int64_t)W * H;
    Out o{depth, alpha, trans, rad, normal, ior, bf};
    cast_kernel<true><<<cast_grid(npix), 128, 0, st>>>(s, W, H, nullptr, offsets, o, od, oc);
    return cudaGetLastError();
}

}  // namespace woit
