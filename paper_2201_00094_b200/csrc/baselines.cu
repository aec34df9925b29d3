// The reference's comparison methods (RenderConfig.method = "abuffer" / "wboit" /
// "mlab4"; baselines.py:135-220) as frame kernels -- SURVEY.md §8(f) rank 2: the
// exact A-buffer is the image oracle of the quality criteria (acceptance 07), at
// sizes where the CPU path takes minutes.
//
// One thread per pixel walks the pixel's CSR run in float64 with the reference's
// arithmetic order, so outputs match the reference up to the final fp32 rounding:
//   abuffer  fragments in (depth, index) order -- a stable segmented sort by depth
//            (CUB DeviceSegmentedSort, library code) -- front to back:
//            acc += (L alpha) vis, vis *= t; out = acc + bg vis      (:135-148)
//   wboit    per-pixel bounds, weights clip(g / (1e-5 + z^2 + z^6), lo, hi),
//            accum / weight / reveal in fragment order               (:151-167)
//   mlab4    k = 4 depth-sorted nodes built in arrival order; an overflow merges
//            the last two nodes (over operator); then front to back  (:170-220)
// t = 1 - alpha (1 - T'), T' = T^3 on ior > 1 fragments with cube transmission
// (scene.py:394-402; the baselines never apply cube_backface_only).
#include <cub/device/device_segmented_sort.cuh>

#include "common.cuh"
#include "internal.cuh"

namespace woit {
namespace {

struct Frag64 {
    double c[3];  // L alpha
    double t[3];  // net transmittance
};

__device__ Frag64 load_frag(const woit_frags_t& f, int64_t i, bool cube) {
    Frag64 g;
    const double al = f.alpha[i];
    const bool cb = cube && f.ior && f.ior[i] > 1.0f;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        g.c[ch] = dmul((double)f.radiance[3 * i + ch], al);
        double T = f.trans[3 * i + ch];
        if (cb) T = dmul(dmul(T, T), T);
        g.t[ch] = dsub(1.0, dmul(al, dsub(1.0, T)));
    }
    return g;
}

__global__ void iota_kernel(int32_t* v, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (int32_t)i;
}

__global__ void abuffer_kernel(const woit_frags_t f, const int32_t* __restrict__ order, bool cube,
                               float* __restrict__ out) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < f.npix;
         p += (int64_t)gridDim.x * blockDim.x) {
        double acc[3] = {0.0, 0.0, 0.0}, vis[3] = {1.0, 1.0, 1.0};
        for (int64_t j = f.offsets[p]; j < f.offsets[p + 1]; ++j) {
            const Frag64 g = load_frag(f, order[j], cube);
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                acc[ch] = dadd(acc[ch], dmul(g.c[ch], vis[ch]));
                vis[ch] = dmul(vis[ch], g.t[ch]);
            }
        }
#pragma unroll
        for (int ch = 0; ch < 3; ++ch)
            out[p * 3 + ch] = (float)dadd(acc[ch], dmul((double)f.opaque_color[p * 3 + ch], vis[ch]));
    }
}

__global__ void wboit_kernel(const woit_frags_t f, bool cube, double gain, double lo, double hi,
                             float* __restrict__ out) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < f.npix;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = f.offsets[p], e = f.offsets[p + 1];
        double near = INFINITY, far = -INFINITY;
        for (int64_t i = s; i < e; ++i) {
            near = fmin(near, (double)f.depth[i]);
            far = fmax(far, (double)f.depth[i]);
        }
        const double rng = dsub(far, near);
        double acc[3] = {0.0, 0.0, 0.0}, rev[3] = {1.0, 1.0, 1.0}, wsum = 0.0;
        for (int64_t i = s; i < e; ++i) {
            double z = rng > 0.0 ? ddiv(dsub((double)f.depth[i], near), rng) : 0.5;
            z = fmin(fmax(z, 0.0), 1.0);
            const double z2 = dmul(z, z);
            const double z6 = dmul(dmul(z2, z2), z2);  // z**6 (the reference's libm pow: <= 1 ulp apart)
            const double w = fmin(fmax(ddiv(gain, dadd(dadd(1e-5, z2), z6)), lo), hi);
            const Frag64 g = load_frag(f, i, cube);
            const double wa = dmul(w, (double)f.alpha[i]);
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                acc[ch] = dadd(acc[ch], dmul(wa, (double)f.radiance[3 * i + ch]));
                rev[ch] = dmul(rev[ch], g.t[ch]);
            }
            wsum = dadd(wsum, wa);
        }
        const double den = fmax(1e-6, wsum);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            const double avg = ddiv(acc[ch], den);
            out[p * 3 + ch] = (float)dadd(dmul(avg, dsub(1.0, rev[ch])),
                                          dmul((double)f.opaque_color[p * 3 + ch], rev[ch]));
        }
    }
}

constexpr int kMlab = 4;

__global__ void mlab_kernel(const woit_frags_t f, bool cube, float* __restrict__ out) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < f.npix;
         p += (int64_t)gridDim.x * blockDim.x) {
        double nd[kMlab], nc[kMlab][3], nt[kMlab][3];
#pragma unroll
        for (int j = 0; j < kMlab; ++j) {
            nd[j] = INFINITY;
            nc[j][0] = nc[j][1] = nc[j][2] = 0.0;
            nt[j][0] = nt[j][1] = nt[j][2] = 1.0;
        }
        for (int64_t i = f.offsets[p]; i < f.offsets[p + 1]; ++i) {
            const double d = f.depth[i];
            const Frag64 g = load_frag(f, i, cube);
            int pos = 0;  // after every node with depth <= d
#pragma unroll
            for (int j = 0; j < kMlab; ++j) pos += nd[j] <= d ? 1 : 0;
            // the (k+1)-th node after insertion: the displaced last node, or the new one
            const bool over = pos == kMlab ? true : isfinite(nd[kMlab - 1]);
            double xd, xc[3], xt[3];
            if (pos == kMlab) {
                xd = d;
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    xc[ch] = g.c[ch];
                    xt[ch] = g.t[ch];
                }
            } else {
                xd = nd[kMlab - 1];
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    xc[ch] = nc[kMlab - 1][ch];
                    xt[ch] = nt[kMlab - 1][ch];
                }
#pragma unroll
                for (int j = kMlab - 1; j > 0; --j) {
                    if (j > pos) {
                        nd[j] = nd[j - 1];
#pragma unroll
                        for (int ch = 0; ch < 3; ++ch) {
                            nc[j][ch] = nc[j - 1][ch];
                            nt[j][ch] = nt[j - 1][ch];
                        }
                    }
                }
#pragma unroll
                for (int j = 0; j < kMlab; ++j) {
                    if (j == pos) {
                        nd[j] = d;
#pragma unroll
                        for (int ch = 0; ch < 3; ++ch) {
                            nc[j][ch] = g.c[ch];
                            nt[j][ch] = g.t[ch];
                        }
                    }
                }
            }
            (void)xd;
            if (over) {  // merge nodes k-1 and k: c = c_{k-1} + t_{k-1} c_k, t = t_{k-1} t_k
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    nc[kMlab - 1][ch] = dadd(nc[kMlab - 1][ch], dmul(nt[kMlab - 1][ch], xc[ch]));
                    nt[kMlab - 1][ch] = dmul(nt[kMlab - 1][ch], xt[ch]);
                }
            }
        }
        double acc[3] = {0.0, 0.0, 0.0}, vis[3] = {1.0, 1.0, 1.0};
#pragma unroll
        for (int j = 0; j < kMlab; ++j)
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                acc[ch] = dadd(acc[ch], dmul(nc[j][ch], vis[ch]));
                vis[ch] = dmul(vis[ch], nt[j][ch]);
            }
#pragma unroll
        for (int ch = 0; ch < 3; ++ch)
            out[p * 3 + ch] = (float)dadd(acc[ch], dmul((double)f.opaque_color[p * 3 + ch], vis[ch]));
    }
}

unsigned grid_for(int64_t n) {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t g = (n + 127) / 128;
    return (unsigned)(g < 16 * sms ? (g > 0 ? g : 1) : 16 * sms);
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

size_t sort_temp_bytes(int64_t n, int64_t npix) {
    size_t temp = 0;
    cub::DeviceSegmentedSort::StableSortPairs(nullptr, temp, (const float*)nullptr, (float*)nullptr,
                                              (const int32_t*)nullptr, (int32_t*)nullptr, (int)n, (int)npix,
                                              (const int64_t*)nullptr, (const int64_t*)nullptr);
    return temp;
}

}  // namespace

size_t baseline_workspace(int method, int64_t npix, int64_t nfrag) {
    if (method != 1) return 16;
    return align256(4 * (size_t)nfrag) * 3 + align256(sort_temp_bytes(nfrag, npix)) + 256;
}

cudaError_t render_baseline(const woit_frags_t& f, int method, bool cube, const double wboit[3], float* out,
                            void* ws, cudaStream_t st) {
    if (f.npix == 0) return cudaSuccess;
    const unsigned grid = grid_for(f.npix);
    if (method == 1) {
        char* w = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
        const size_t a = align256(4 * (size_t)f.nfrag);
        float* keys_out = reinterpret_cast<float*>(w);
        int32_t* ids = reinterpret_cast<int32_t*>(w + a);
        int32_t* order = reinterpret_cast<int32_t*>(w + 2 * a);
        void* temp = w + 3 * a;
        size_t temp_bytes = sort_temp_bytes(f.nfrag, f.npix);
        if (f.nfrag > 0) {
            iota_kernel<<<grid_for(f.nfrag), 128, 0, st>>>(ids, f.nfrag);
            cudaError_t e = cub::DeviceSegmentedSort::StableSortPairs(temp, temp_bytes, f.depth, keys_out, ids, order,
                                                                      (int)f.nfrag, (int)f.npix, f.offsets,
                                                                      f.offsets + 1, st);
            if (e != cudaSuccess) return e;
        }
        abuffer_kernel<<<grid, 128, 0, st>>>(f, order, cube, out);
    } else if (method == 2) {
        wboit_kernel<<<grid, 128, 0, st>>>(f, cube, wboit[0], wboit[1], wboit[2], out);
    } else {
        mlab_kernel<<<grid, 128, 0, st>>>(f, cube, out);
    }
    return cudaGetLastError();
}

}  // namespace woit
