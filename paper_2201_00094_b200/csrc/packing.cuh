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

// pack_rgb9e5 of an fp32-valued non-negative triple, without log2 or divisions: for an
// fp32 value floor(log2 x) is its exponent field (the largest fp32 below 2^k has
// log2 = k - 8.6e-8, which f64 resolves), the scale 2^(e-24) is a power of two, so
// v / scale is exact, and floor(y + 0.5) is exact in f64 -- every step equals the
// reference's (packing.py:46-77) on these inputs, bit for bit.
WOIT_D uint32_t rgb9e5_pack_fp32(float a, float b, float c) {
    const float v[3] = {fminf(fmaxf(a, 0.0f), (float)kPackedMax), fminf(fmaxf(b, 0.0f), (float)kPackedMax),
                        fminf(fmaxf(c, 0.0f), (float)kPackedMax)};
    const float mx = fmaxf(fmaxf(v[0], v[1]), v[2]);
    int e = 0;
    if (mx > 0.0f) {
        const int fl = ((__float_as_int(mx) >> 23) & 0xff) - 127;  // subnormals: -127, clamped below
        e = max(max(-kExpBias - 1, fl) + 1 + kExpBias, 0);
    }
    double inv = __hiloint2double((1023 + kExpBias + kMantBits - e) << 20, 0);  // 2^(24 - e)
    if (floor((double)mx * inv + 0.5) >= (double)(1 << kMantBits)) {
        e += 1;
        inv *= 0.5;
    }
    uint32_t w = ((uint32_t)e) << 27;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        const double m = floor((double)v[ch] * inv + 0.5);
        w |= (m >= (double)kMantMax ? kMantMax : (uint32_t)m) << (9 * ch);
    }
    return w;
}

// unpack_rgb9e5 into fp32 (m 2^(e-24) with m < 2^9 is exact in fp32)
WOIT_D void rgb9e5_unpack_fp32(uint32_t w, float out[3]) {
    const float scale = __int_as_float((int)(((w >> 27) & 31u) + 127 - kExpBias - kMantBits) << 23);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) out[ch] = (float)((w >> (9 * ch)) & kMantMax) * scale;
}

}  // namespace woit
