// K_resolve: the diffusion blur of the background image (woit.h WOIT_DIFFUSION).
//
// The reference has no diffusion pass (SURVEY.md §8 row GAP), so
// this is the in-repo definition: a separable, edge-clamped Gaussian with `radius`
// taps each side and sigma = radius / 2, horizontal pass then vertical pass, fp32
// accumulation in tap order -radius..radius. Both passes stage a tile plus its
// halo in shared memory with 128-bit coalesced loads and write 128-bit stores, so
// each pass moves the image through HBM once in and once out (24 B/px total).
#include <cmath>

#include "common.cuh"
#include "internal.cuh"

namespace woit {
namespace {

constexpr int kMaxBlurRadius = 64;
constexpr int kRowTile = 512;  // pixels per horizontal-pass CTA
constexpr int kColTileY = 64;  // rows per vertical-pass CTA
constexpr int kColTileX = 32;  // float4 columns per vertical-pass CTA

struct Taps {
    float w[2 * kMaxBlurRadius + 1];
};

Taps gaussian_taps(int r) {
    // f64 weights exp(-i^2 / (2 sigma^2)) normalised to sum 1, then rounded to fp32
    // (oracle/woit_oracle.py gaussian_taps is the twin)
    const double sigma = 0.5 * r;
    double g[2 * kMaxBlurRadius + 1], sum = 0.0;
    for (int i = -r; i <= r; ++i) {
        g[i + r] = std::exp(-(double)(i * i) / (2.0 * sigma * sigma));
        sum += g[i + r];
    }
    Taps t{};
    for (int i = 0; i <= 2 * r; ++i) t.w[i] = (float)(g[i] / sum);
    return t;
}

// Horizontal pass over one row segment [x0, x0 + kRowTile): the floats of pixels
// [x0 - r, x0 + kRowTile + r) (clipped to the row) are staged, 16-B loads for the
// aligned body; every output float j (pixel j / 3, channel j % 3) sums its taps
// from the staged row with the pixel index clamped to [0, W).
__global__ void __launch_bounds__(256) blur_rows_kernel(const float* __restrict__ in, float* __restrict__ out,
                                                        int W, int H, int r, bool vec, const Taps taps) {
    extern __shared__ __align__(16) float srow[];
    const int y = blockIdx.y;
    const int x0 = blockIdx.x * kRowTile;
    const int x1 = min(W, x0 + kRowTile);
    const int lo = max(0, x0 - r), hi = min(W, x1 + r);  // staged pixels
    const int64_t row = (int64_t)y * W * 3;
    const int64_t g0 = row + 3 * (int64_t)lo, g1 = row + 3 * (int64_t)hi;  // staged floats [g0, g1)
    const int64_t a0 = g0 & ~(int64_t)3;                                     // smem float 0 <-> global a0
    const int64_t v0 = vec ? (g0 + 3) & ~(int64_t)3 : g1, v1 = vec ? g1 & ~(int64_t)3 : g1;  // 16-B body
    for (int64_t g = g0 + threadIdx.x; g < min(v0, g1); g += blockDim.x) srow[g - a0] = in[g];
    for (int64_t g = v0 + 4 * (int64_t)threadIdx.x; g < v1; g += 4 * (int64_t)blockDim.x)
        *reinterpret_cast<float4*>(srow + (g - a0)) = *reinterpret_cast<const float4*>(in + g);
    for (int64_t g = max(v1, v0) + threadIdx.x; g < g1; g += blockDim.x) srow[g - a0] = in[g];
    __syncthreads();
    const int off = (int)(row - a0);  // smem index of pixel x, channel c: off + 3 x + c
    auto tap_sum = [&](int j) {  // j = 3 x + c within the row
        const int x = j / 3, c = j - 3 * x;
        float s = 0.0f;
        for (int k = -r; k <= r; ++k) {
            const int xx = min(max(x + k, 0), W - 1);
            s = fmaf(taps.w[k + r], srow[off + 3 * xx + c], s);
        }
        return s;
    };
    const int64_t o0 = row + 3 * (int64_t)x0, o1 = row + 3 * (int64_t)x1;  // output floats
    const int64_t b0 = vec ? (o0 + 3) & ~(int64_t)3 : o1, b1 = vec ? o1 & ~(int64_t)3 : o1;
    for (int64_t g = o0 + threadIdx.x; g < min(b0, o1); g += blockDim.x) out[g] = tap_sum((int)(g - row));
    for (int64_t g = b0 + 4 * (int64_t)threadIdx.x; g < b1; g += 4 * (int64_t)blockDim.x) {
        const int j = (int)(g - row);
        *reinterpret_cast<float4*>(out + g) = make_float4(tap_sum(j), tap_sum(j + 1), tap_sum(j + 2), tap_sum(j + 3));
    }
    for (int64_t g = max(b1, b0) + threadIdx.x; g < o1; g += blockDim.x) out[g] = tap_sum((int)(g - row));
}

// Vertical pass: elementwise over the 3W floats of a row. A CTA owns kColTileX
// float4 columns x kColTileY rows and stages rows [y0 - r, y0 + kColTileY + r)
// (clamped) of those columns; 16-B loads/stores (VEC, when 3W % 4 == 0).
template <bool VEC>
__global__ void __launch_bounds__(256) blur_cols_kernel(const float* __restrict__ in, float* __restrict__ out,
                                                        int W, int H, int r, const Taps taps) {
    extern __shared__ __align__(16) float4 stile[];  // [kColTileY + 2r][kColTileX]
    const int RW = 3 * W;                             // floats per row
    const int ncol4 = (RW + 3) / 4;
    const int c4 = blockIdx.x * kColTileX + threadIdx.x;  // float4 column
    const int y0 = blockIdx.y * kColTileY;
    const int rows = kColTileY + 2 * r;
    const bool col_ok = c4 < ncol4;
    for (int i = threadIdx.y; i < rows; i += blockDim.y) {
        const int yy = min(max(y0 - r + i, 0), H - 1);
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (col_ok) {
            const float* src = in + (int64_t)yy * RW + 4 * c4;
            if (VEC) {
                v = *reinterpret_cast<const float4*>(src);
            } else {
                const int n = min(4, RW - 4 * c4);
                v.x = src[0];
                if (n > 1) v.y = src[1];
                if (n > 2) v.z = src[2];
                if (n > 3) v.w = src[3];
            }
        }
        stile[i * kColTileX + threadIdx.x] = v;
    }
    __syncthreads();
    if (!col_ok) return;
    for (int i = threadIdx.y; i < kColTileY && y0 + i < H; i += blockDim.y) {
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int k = 0; k <= 2 * r; ++k) {
            const float4 v = stile[(i + k) * kColTileX + threadIdx.x];
            const float w = taps.w[k];
            s.x = fmaf(w, v.x, s.x);
            s.y = fmaf(w, v.y, s.y);
            s.z = fmaf(w, v.z, s.z);
            s.w = fmaf(w, v.w, s.w);
        }
        float* dst = out + (int64_t)(y0 + i) * RW + 4 * c4;
        if (VEC) {
            *reinterpret_cast<float4*>(dst) = s;
        } else {
            const int n = min(4, RW - 4 * c4);
            dst[0] = s.x;
            if (n > 1) dst[1] = s.y;
            if (n > 2) dst[2] = s.z;
            if (n > 3) dst[3] = s.w;
        }
    }
}

}  // namespace

size_t blur_workspace(int32_t width, int32_t height) {
    return (size_t)width * (size_t)height * 3 * sizeof(float) + 16;
}

cudaError_t resolve_blur(const float* image, int32_t W, int32_t H, int32_t r, float* out, void* ws,
                         cudaStream_t st) {
    const Taps taps = gaussian_taps(r);
    float* tmp = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(ws) + 15) & ~uintptr_t(15));
    // horizontal: image -> tmp
    {
        const int maxpx = kRowTile + 2 * r;
        const size_t smem = (size_t)(3 * maxpx + 8) * sizeof(float);
        cudaError_t e = cudaFuncSetAttribute(blur_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        dim3 grid((W + kRowTile - 1) / kRowTile, H);
        const bool vec = (reinterpret_cast<uintptr_t>(image) & 15u) == 0;  // tmp is 16-B aligned
        blur_rows_kernel<<<grid, 256, smem, st>>>(image, tmp, W, H, r, vec, taps);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    // vertical: tmp -> out
    {
        const int ncol4 = (3 * W + 3) / 4;
        const size_t smem = (size_t)(kColTileY + 2 * r) * kColTileX * sizeof(float4);
        const bool vec = (3 * W) % 4 == 0 && ((reinterpret_cast<uintptr_t>(out) & 15u) == 0);
        dim3 grid((ncol4 + kColTileX - 1) / kColTileX, (H + kColTileY - 1) / kColTileY);
        dim3 block(kColTileX, 8);
        cudaError_t e;
        if (vec) {
            e = cudaFuncSetAttribute(blur_cols_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            blur_cols_kernel<true><<<grid, block, smem, st>>>(tmp, out, W, H, r, taps);
        } else {
            e = cudaFuncSetAttribute(blur_cols_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            blur_cols_kernel<false><<<grid, block, smem, st>>>(tmp, out, W, H, r, taps);
        }
        return cudaGetLastError();
    }
}

}  // namespace woit
