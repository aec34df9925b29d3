// E5B9G9R9 shared-exponent words (packing.py:1-111), f64 in / f64 out.
#pragma once

#include "common.cuh"

namespace woit {

constexpr int kMantBits = 9;
constexpr int kExpBias = 15;
constexpr uint32_t kMantMax = (1u << kMantBits) - 1u;
constexpr double kPackedMax = 65408.0;  // (511/512) * 2^16

// pack_rgb9e5 for one non-negative triple (packing.py:46-77)
WOIT_D uint32_t rgb9e5_pack_impl(const double v_in[3]) {
    double v[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) v[c] = fmin(fmax(v_in[c], 0.0), kPackedMax);
    const double mx = fmax(fmax(v[0], v[1]), v[2]);
    const double fl = mx > 0.0 ? floor(log2(mx)) : -INFINITY;
    double e = fmax(fmax(-kExpBias - 1.0, fl) + 1.0 + kExpBias, 0.0);
    double scale = ldexp(1.0, (int)e - kExpBias - kMantBits);
    if (floor(mx / scale + 0.5) >= (double)(1 << kMantBits)) {
        e += 1.0;
        scale *= 2.0;
    }
    uint32_t w = ((uint32_t)e) << 27;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        double m = floor(v[c] / scale + 0.5);
        uint32_t mi = m >= (double)kMantMax ? kMantMax : (uint32_t)m;
        w |= mi << (9 * c);
    }
    return w;
}

// unpack_rgb9e5 (packing.py:80-88)
WOIT_D void rgb9e5_unpack_impl(uint32_t w, double out[3]) {
    const int e = (int)((w >> 27) & 31u);
    const double scale = ldexp(1.0, e - kExpBias - kMantBits);
#pragma unroll
    for (int c = 0; c < 3; ++c) out[c] = (double)((w >> (9 * c)) & kMantMax) * scale;
}

}  // namespace woit
