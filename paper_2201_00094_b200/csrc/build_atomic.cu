// The north star's other build strategy, kept for the measured comparison
// (BASELINE.json north star (1): "bins fragments by pixel ... or uses fp32
// red.global atomics into a pixel-major SoA coefficient buffer, whichever ncu
// shows is faster"; DESIGN.md §3.6 has the numbers).
//
// One thread per fragment of an UNBINNED stream (explicit pixel ids): z from the
// pixel's depth map (f64 / fixed point, bit-exact like every other path), the
// absorbance per channel, and the closed-form Haar projection of wavelet.py:272-287
// scattered as (N + 2) x 3 `red.global.add.f32` into coeffs[P][S][3]. Results
// depend on the atomic arrival order (not bit-reproducible) and on fp32
// cancellation across levels; the fused CSR tile build is both deterministic and
// faster, so this path is not used by render_band.
#include "common.cuh"
#include "internal.cuh"

namespace woit {
namespace {

// per-pixel depth map (lo, den, rs) once, instead of two f64 divisions per fragment
__global__ void depth_map_kernel(const float* __restrict__ near, const float* __restrict__ far, int64_t npix,
                                 int rank, double* __restrict__ dm) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npix;
         p += (int64_t)gridDim.x * blockDim.x) {
        const DepthMap m = depth_map(near[p], far[p], rank);
        dm[p] = m.lo;
        dm[npix + p] = m.den;
        dm[2 * npix + p] = m.rs;
    }
}

template <int R>
__global__ void __launch_bounds__(256) build_atomic_kernel(const int32_t* __restrict__ pix,
                                                           const float* __restrict__ depth,
                                                           const float* __restrict__ alpha,
                                                           const float* __restrict__ trans,
                                                           const float* __restrict__ ior,
                                                           const uint8_t* __restrict__ backface, int64_t n,
                                                           int64_t npix, int flags, const double* __restrict__ dm,
                                                           float* __restrict__ coeffs) {
    constexpr int S = 2 << R;
    const bool cube = flags & WOIT_CUBE_TRANSMISSION;
    const bool bfonly = flags & WOIT_CUBE_BACKFACE_ONLY;
    for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < n; f += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = pix[f];
        DepthMap m;
        m.lo = dm[p];
        m.den = dm[npix + p];
        m.rcp = 0.0;
        m.rs = dm[2 * npix + p];
        const zfix_t zi = z_fixed_of(depth[f], m);
        const float al = alpha[f];
        bool cb = false;
        if (cube) {
            const float io = ior ? ior[f] : 1.0f;
            cb = io > 1.0f && (!bfonly || (backface && backface[f]));
        }
        float a[3];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) a[ch] = absorbance_ch(al, trans[3 * f + ch], cb);
        float* c = coeffs + p * (S * 3);
        const float omz = one_minus_z(zi);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) atomicAdd(c + ch, a[ch] * omz);  // slot 0 += a (1 - z)
#pragma unroll
        for (int lv = 0; lv <= R; ++lv) {  // slot 2^n + k -= a 2^(-n/2) min(u, 1 - u)
            const int slot = (1 << lv) + slot_offset(zi, lv);
            const float w = level_psi(zi, lv) * kInvSqrt2PowF[lv];
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) atomicAdd(c + slot * 3 + ch, -(a[ch] * w));
        }
    }
}

}  // namespace

size_t build_atomic_workspace(int64_t npix) { return (size_t)npix * 3 * sizeof(double); }

cudaError_t build_atomic(const int32_t* pix, const woit_frags_t& f, int rank, int flags, const float* near,
                         const float* far, float* coeffs, void* ws, cudaStream_t st) {
    double* dm = static_cast<double*>(ws);
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (f.npix > 0) {
        const int64_t g = (f.npix + 255) / 256;
        depth_map_kernel<<<(unsigned)(g < 8 * sms ? g : 8 * sms), 256, 0, st>>>(near, far, f.npix, rank, dm);
    }
    if (f.nfrag == 0) return cudaGetLastError();
    const int64_t g = (f.nfrag + 255) / 256;
    const unsigned grid = (unsigned)(g < 16 * sms ? g : 16 * sms);
#define WOIT_ATOMIC_CASE(RR)                                                                                     \
    case RR:                                                                                                     \
        build_atomic_kernel<RR><<<grid, 256, 0, st>>>(pix, f.depth, f.alpha, f.trans, f.ior, f.backface, f.nfrag, \
                                                      f.npix, flags, dm, coeffs);                                \
        break;
    switch (rank) {
        WOIT_ATOMIC_CASE(0)
        WOIT_ATOMIC_CASE(1)
        WOIT_ATOMIC_CASE(2)
        WOIT_ATOMIC_CASE(3)
        WOIT_ATOMIC_CASE(4)
        WOIT_ATOMIC_CASE(5)
        WOIT_ATOMIC_CASE(6)
        default: return cudaErrorInvalidValue;
    }
#undef WOIT_ATOMIC_CASE
    return cudaGetLastError();
}

}  // namespace woit
