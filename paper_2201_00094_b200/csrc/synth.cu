// Device twin of paper_2201_00094_b200/synth.py: bit-identical synthetic CSR
// fragment streams generated directly in HBM. Every fp32
// operation is an explicit round-to-nearest intrinsic so no FMA contraction can
// change a bit relative to the numpy generator.
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "internal.cuh"

namespace woit {
namespace synth {

constexpr uint32_t kPixelLayer = 0xFFFFu;
enum { F_DEPTH = 0, F_ALPHA, F_T0, F_T1, F_T2, F_L0, F_L1, F_L2 };
enum { P_NEAR = 0, P_SPAN = 1, P_RUN = 2 };

WOIT_D uint32_t mix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7FEB352Du;
    x ^= x >> 15;
    x *= 0x846CA68Bu;
    x ^= x >> 16;
    return x;
}

WOIT_D float uniform(uint32_t seed, uint32_t pixel, uint32_t layer, uint32_t field) {
    const uint32_t s = mix32(seed ^ 0x9E3779B9u);
    uint32_t h = mix32(pixel ^ s);
    const uint32_t key = (layer << 4) | field;
    h = mix32(h + key * 0x85EBCA6Bu);
    return __fmul_rn((float)(h >> 8), 5.9604644775390625e-08f);
}

WOIT_D float fma_free(float a, float b, float c) { return __fadd_rn(__fmul_rn(a, b), c); }

WOIT_D float gauss_profile(float r) {
    const float x = __fmul_rn(__fmul_rn(r, r), -4.0f);
    const float y = __fmul_rn(x, 0.125f);
    const float c[8] = {(float)(1.0 / 1), (float)(1.0 / 1), (float)(1.0 / 2), (float)(1.0 / 6),
                        (float)(1.0 / 24), (float)(1.0 / 120), (float)(1.0 / 720), (float)(1.0 / 5040)};
    float p = c[7];
    for (int k = 6; k >= 0; --k) p = fma_free(p, y, c[k]);
    p = __fmul_rn(p, p);
    p = __fmul_rn(p, p);
    p = __fmul_rn(p, p);
    return p;
}

WOIT_D int64_t run_length(int workload, uint32_t seed, int32_t layers, uint32_t gp) {
    if (workload == WOIT_SYNTH_PLANE4) return 5;
    if (workload == WOIT_SYNTH_RAGGED) {
        const float u = uniform(seed, gp, kPixelLayer, P_RUN);
        int64_t run = (int64_t)__fmul_rn(u, (float)(layers + 1));
        return run < layers ? run : layers;
    }
    return layers;
}

__global__ void runs_kernel(int workload, int32_t width, uint32_t seed, int32_t layers, int32_t row0,
                            int64_t npix, int64_t* offsets) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npix;
         p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t gp = (uint32_t)((int64_t)row0 * width + p);
        offsets[p + 1] = run_length(workload, seed, layers, gp);
        if (p == 0) offsets[0] = 0;
    }
}

WOIT_D void fragment(int workload, uint32_t seed, int32_t layers, uint32_t gp, int64_t j, int64_t i,
                     const Out& o) {
    const uint32_t lj = (uint32_t)j;
    auto u = [&](uint32_t f) { return uniform(seed, gp, lj, f); };
    float depth, alpha, T[3], L[3];
    if (workload == WOIT_SYNTH_PLANE4) {
        if (j == 0) {
            depth = 1.0f;
            alpha = 0.25f;
            T[0] = T[1] = T[2] = 0.0f;
            L[0] = (float)0.18;
            L[1] = (float)0.18;
            L[2] = (float)0.20;
        } else {
            depth = fma_free(u(F_DEPTH), (float)1.7, (float)0.25);
            alpha = u(F_ALPHA);
            for (int c = 0; c < 3; ++c) {
                T[c] = u(F_T0 + c);
                L[c] = u(F_L0 + c);
            }
        }
    } else if (workload == WOIT_SYNTH_SMOKE) {
        const float near = fma_free(uniform(seed, gp, kPixelLayer, P_NEAR), 0.5f, 0.5f);
        const float span = fma_free(uniform(seed, gp, kPixelLayer, P_SPAN), 2.0f, 1.0f);
        float frac = __fadd_rn((float)j, u(F_DEPTH));
        if ((layers & (layers - 1)) == 0)
            frac = __fmul_rn(frac, (float)(1.0 / layers));
        else
            frac = __fdiv_rn(frac, (float)layers);
        depth = fma_free(frac, span, near);
        alpha = __fmul_rn((float)0.4, gauss_profile(u(F_ALPHA)));
        const float tg = fma_free(u(F_T0), (float)0.3, (float)0.2);
        const float lg = fma_free(u(F_L0), (float)0.15, (float)0.3);
        T[0] = T[1] = T[2] = tg;
        L[0] = L[1] = L[2] = lg;
    } else {  // particles, ragged
        depth = fma_free(u(F_DEPTH), (float)2.2, 1.0f);
        const float fade = __fsub_rn(1.0f, __fmul_rn(__fdiv_rn(__fsub_rn(depth, 1.0f), (float)2.2), 0.5f));
        alpha = __fmul_rn(__fmul_rn(0.5f, gauss_profile(u(F_ALPHA))), fade);
        for (int c = 0; c < 3; ++c) {
            T[c] = fma_free(u(F_T0 + c), (float)0.31, (float)0.02);
            L[c] = __fmul_rn(u(F_L0 + c), (float)1.3);
        }
    }
    o.depth[i] = depth;
    o.alpha[i] = alpha;
    for (int c = 0; c < 3; ++c) {
        o.trans[3 * i + c] = T[c];
        o.rad[3 * i + c] = L[c];
    }
    o.normal[3 * i] = 0.0f;
    o.normal[3 * i + 1] = 0.0f;
    o.normal[3 * i + 2] = -1.0f;
    o.ior[i] = 1.0f;
    o.bf[i] = 0;
}

// uniform run length: one thread per fragment (coalesced stores)
__global__ void fill_uniform_kernel(int workload, int32_t width, uint32_t seed, int32_t layers, int32_t row0,
                                    int64_t nfrag, int64_t run, Out o) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nfrag;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = i / run, j = i - p * run;
        fragment(workload, seed, layers, (uint32_t)((int64_t)row0 * width + p), j, i, o);
    }
}

// ragged: one thread per pixel
__global__ void fill_ragged_kernel(int workload, int32_t width, uint32_t seed, int32_t layers, int32_t row0,
                                   int64_t npix, const int64_t* offsets, Out o) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npix;
         p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t gp = (uint32_t)((int64_t)row0 * width + p);
        for (int64_t i = offsets[p]; i < offsets[p + 1]; ++i) fragment(workload, seed, layers, gp, i - offsets[p], i, o);
    }
}

__global__ void opaque_kernel(int workload, int32_t width, int32_t row0, int64_t npix, float* od, float* oc) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npix;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t gp = (int64_t)row0 * width + p;
        if (workload == WOIT_SYNTH_PLANE4) {
            od[p] = 2.0f;
            oc[3 * p] = (float)0.85;
            oc[3 * p + 1] = (float)0.45;
            oc[3 * p + 2] = (float)0.12;
        } else {
            od[p] = INFINITY;
            const int64_t px = gp % width, py = gp / width;
            const bool odd = (((px >> 4) + (py >> 4)) & 1) != 0;
            oc[3 * p] = odd ? (float)0.25 : (float)0.85;
            oc[3 * p + 1] = odd ? (float)0.22 : (float)0.80;
            oc[3 * p + 2] = odd ? (float)0.20 : (float)0.72;
        }
    }
}

static unsigned grid_for(int64_t n) {
    const int64_t g = (n + 255) / 256;
    return (unsigned)(g < 1 ? 1 : (g > 16384 ? 16384 : g));
}

size_t workspace(int64_t npix) {
    size_t temp = 0;
    cub::DeviceScan::InclusiveSum(nullptr, temp, (int64_t*)nullptr, (int64_t*)nullptr, (int)(npix + 1));
    return temp + 256;
}

cudaError_t offsets(int workload, int32_t width, uint32_t seed, int32_t layers, int32_t row0, int32_t rows,
                    int64_t* off, void* ws, size_t ws_bytes, cudaStream_t st) {
    const int64_t npix = (int64_t)rows * width;
    if (npix == 0) return cudaMemsetAsync(off, 0, 8, st);
    runs_kernel<<<grid_for(npix), 256, 0, st>>>(workload, width, seed, layers, row0, npix, off);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    size_t temp = ws_bytes;
    return cub::DeviceScan::InclusiveSum(ws, temp, off, off, (int)(npix + 1), st);
}

cudaError_t fill(int workload, int32_t width, uint32_t seed, int32_t layers, int32_t row0, int32_t rows,
                 const int64_t* off, int64_t nfrag_uniform, Out o, float* od, float* oc, cudaStream_t st) {
    const int64_t npix = (int64_t)rows * width;
    if (npix == 0) return cudaSuccess;
    if (workload == WOIT_SYNTH_RAGGED) {
        fill_ragged_kernel<<<grid_for(npix), 128, 0, st>>>(workload, width, seed, layers, row0, npix, off, o);
    } else {
        const int64_t run = workload == WOIT_SYNTH_PLANE4 ? 5 : layers;
        if (npix * run > 0)
            fill_uniform_kernel<<<grid_for(npix * run), 256, 0, st>>>(workload, width, seed, layers, row0,
                                                                      npix * run, run, o);
    }
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    opaque_kernel<<<grid_for(npix), 256, 0, st>>>(workload, width, row0, npix, od, oc);
    (void)nfrag_uniform;
    return cudaGetLastError();
}

}  // namespace synth
}  // namespace woit
