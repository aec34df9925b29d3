// Kernel-level batch entry points (wavelet.py:272-337), fragment binning, and
// E5B9G9R9 packing (packing.py:46-111). float64 like the reference; the binned
// build reproduces np.add.at's per-slot addition order exactly.
#include "common.cuh"
#include "internal.cuh"
#include "packing.cuh"

namespace woit {

// --- binning: csrc/binning.cu (bin_by_pixel, bin_workspace) ---

// --- build_into ----------------------------------------------------------------

// Contribution of one fragment to slot s, exactly as wavelet.py:277-284 in f64.
// Slot 0: a (1 - z); slot 2^n + k_n: -(a psi_n).
struct Contrib {
    double w0;        // 1 - z
    double psi[7];    // 2^(-n/2) min(u, 1-u)
    int k[7];         // level offsets
};

WOIT_D void contrib(double z, int rank, Contrib& c) {
    c.w0 = dsub(1.0, z);
    for (int n = 0; n <= rank; ++n) {
        const int s = 1 << n;
        const double sz = dmul((double)s, z);
        int64_t k = (int64_t)sz;  // astype(int64): truncation
        if (k > s - 1) k = s - 1;
        const double u = dsub(sz, (double)k);
        c.psi[n] = dmul(kInvSqrt2Pow64[n], fmin(u, dsub(1.0, u)));
        c.k[n] = (int)k;
    }
}

// binned: one thread per pixel walks its fragments in original order
__global__ void build_binned_kernel(double* coeffs, int64_t npix, const int64_t* offsets,
                                    const int64_t* perm, const double* z, const double* a, int rank) {
    const int S = 1 << (rank + 1);
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npix;
         p += (int64_t)gridDim.x * blockDim.x) {
        double* cp = coeffs + p * S * 3;
        for (int64_t j = offsets[p]; j < offsets[p + 1]; ++j) {
            const int64_t i = perm[j];
            Contrib c;
            contrib(z[i], rank, c);
            const double a0 = a[3 * i], a1 = a[3 * i + 1], a2 = a[3 * i + 2];
            cp[0] = dadd(cp[0], dmul(a0, c.w0));
            cp[1] = dadd(cp[1], dmul(a1, c.w0));
            cp[2] = dadd(cp[2], dmul(a2, c.w0));
            for (int n = 0; n <= rank; ++n) {
                double* sl = cp + ((1 << n) + c.k[n]) * 3;
                sl[0] = dadd(sl[0], -dmul(a0, c.psi[n]));
                sl[1] = dadd(sl[1], -dmul(a1, c.psi[n]));
                sl[2] = dadd(sl[2], -dmul(a2, c.psi[n]));
            }
        }
    }
}

// atomic: one thread per fragment, red.global.add.f64 per slot and channel
__global__ void build_atomic_kernel(double* coeffs, const int64_t* pix, const double* z,
                                    const double* a, int64_t n, int rank) {
    const int S = 1 << (rank + 1);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        Contrib c;
        contrib(z[i], rank, c);
        double* cp = coeffs + pix[i] * S * 3;
        for (int ch = 0; ch < 3; ++ch) atomicAdd(cp + ch, dmul(a[3 * i + ch], c.w0));
        for (int nn = 0; nn <= rank; ++nn) {
            double* sl = cp + ((1 << nn) + c.k[nn]) * 3;
            for (int ch = 0; ch < 3; ++ch) atomicAdd(sl + ch, -dmul(a[3 * i + ch], c.psi[nn]));
        }
    }
}

// --- evaluation --------------------------------------------------------------

WOIT_D double cell_raw(const double* cp, int cell, int rank, int ch) {
    double val = cp[ch];
    for (int n = 0; n <= rank; ++n) {
        const int m = rank + 1 - n;
        const double sign = 1.0 - 2.0 * (double)((cell >> (m - 1)) & 1);
        val = dadd(val, dmul(dmul(kSqrt2Pow[n], sign), cp[((1 << n) + (cell >> m)) * 3 + ch]));
    }
    return val;
}

__global__ void interp_kernel(const double* coeffs, const int64_t* pix, const double* z, int64_t n,
                              int rank, double* out) {
    const int S = 1 << (rank + 1), M = S;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double u = dsub(dmul(z[i], (double)M), 0.5);
        const double fl = floor(u);
        int64_t c0 = (int64_t)fl;
        double t = dsub(u, (double)c0);
        if (c0 < 0 || c0 >= M - 1) t = 0.0;
        c0 = c0 < 0 ? 0 : (c0 > M - 1 ? M - 1 : c0);
        const int64_t c1 = c0 + 1 < M - 1 ? c0 + 1 : M - 1;
        const double* cp = coeffs + pix[i] * S * 3;
        for (int ch = 0; ch < 3; ++ch) {
            const double l = cell_raw(cp, (int)c0, rank, ch), r = cell_raw(cp, (int)c1, rank, ch);
            out[3 * i + ch] = fmax(dadd(dmul(dsub(1.0, t), l), dmul(t, r)), 0.0);
        }
    }
}

__global__ void cells_kernel(const double* coeffs, const int64_t* pix, const int64_t* cells, int64_t n,
                             int rank, double* out) {
    const int S = 1 << (rank + 1);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double* cp = coeffs + pix[i] * S * 3;
        for (int ch = 0; ch < 3; ++ch) out[3 * i + ch] = cell_raw(cp, (int)cells[i], rank, ch);
    }
}

__global__ void total_kernel(const double* coeffs, int64_t npix, int rank, double* out) {
    const int S = 1 << (rank + 1);
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npix;
         p += (int64_t)gridDim.x * blockDim.x) {
        const double* cp = coeffs + p * S * 3;
        for (int ch = 0; ch < 3; ++ch) {
            double val = cp[ch];
            for (int n = 0; n <= rank; ++n)
                val = dsub(val, dmul(kSqrt2Pow[n], cp[((1 << (n + 1)) - 1) * 3 + ch]));
            out[3 * p + ch] = fmax(val, 0.0);
        }
    }
}

// --- packing -----------------------------------------------------------------

__global__ void pack_kernel(const double* v, int64_t n, uint32_t* words) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double t[3] = {fabs(v[3 * i]), fabs(v[3 * i + 1]), fabs(v[3 * i + 2])};
        words[i] = rgb9e5_pack_impl(t);
    }
}

__global__ void unpack_kernel(const uint32_t* words, int64_t n, double* out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double t[3];
        rgb9e5_unpack_impl(words[i], t);
        out[3 * i] = t[0];
        out[3 * i + 1] = t[1];
        out[3 * i + 2] = t[2];
    }
}

static unsigned grid_for(int64_t n) {
    const int64_t g = (n + 255) / 256;
    return (unsigned)(g < 1 ? 1 : (g > 8192 ? 8192 : g));
}

cudaError_t build_into(double* coeffs, int64_t npix, const int64_t* pix, const double* z, const double* a,
                       int64_t n, int rank, int mode, void* ws, size_t ws_bytes, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    if (mode == WOIT_BUILD_ATOMIC) {
        build_atomic_kernel<<<grid_for(n), 256, 0, st>>>(coeffs, pix, z, a, n, rank);
        return cudaGetLastError();
    }
    unsigned char* w = static_cast<unsigned char*>(ws);
    int64_t* offsets = reinterpret_cast<int64_t*>(w);
    int64_t* perm = offsets + (npix + 1);
    unsigned char* rest = reinterpret_cast<unsigned char*>(perm + n);
    rest = reinterpret_cast<unsigned char*>(((uintptr_t)rest + 255) & ~(uintptr_t)255);
    cudaError_t err = bin_by_pixel(pix, n, npix, offsets, perm, rest, ws_bytes, st);
    if (err != cudaSuccess) return err;
    build_binned_kernel<<<grid_for(npix), 256, 0, st>>>(coeffs, npix, offsets, perm, z, a, rank);
    return cudaGetLastError();
}

size_t build_into_workspace(int64_t n, int64_t npix) {
    return (size_t)(npix + 1) * 8 + (size_t)(n > 0 ? n : 1) * 8 + 256 + bin_workspace(n, npix);
}

cudaError_t interp(const double* coeffs, const int64_t* pix, const double* z, int64_t n, int rank,
                   double* out, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    interp_kernel<<<grid_for(n), 256, 0, st>>>(coeffs, pix, z, n, rank, out);
    return cudaGetLastError();
}

cudaError_t cells_raw(const double* coeffs, const int64_t* pix, const int64_t* cells, int64_t n, int rank,
                      double* out, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    cells_kernel<<<grid_for(n), 256, 0, st>>>(coeffs, pix, cells, n, rank, out);
    return cudaGetLastError();
}

cudaError_t total(const double* coeffs, int64_t npix, int rank, double* out, cudaStream_t st) {
    if (npix == 0) return cudaSuccess;
    total_kernel<<<grid_for(npix), 256, 0, st>>>(coeffs, npix, rank, out);
    return cudaGetLastError();
}

cudaError_t pack(const double* v, int64_t n, uint32_t* words, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    pack_kernel<<<grid_for(n), 256, 0, st>>>(v, n, words);
    return cudaGetLastError();
}

cudaError_t unpack(const uint32_t* words, int64_t n, double* out, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    unpack_kernel<<<grid_for(n), 256, 0, st>>>(words, n, out);
    return cudaGetLastError();
}

}  // namespace woit
