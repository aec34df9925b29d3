// Fragment binning (scene.py:559-566 contract): an unbinned stream with a pixel id
// per fragment -> the CSR stream, stable (the fragments of a pixel keep their
// arrival order), offsets = [0, cumsum(bincount(pix, minlength=npix))],
// perm = argsort(pix, kind="stable"), and optionally the fragment fields
// gathered into CSR order in the same pass that places them.
//
// Hand-written LSD radix sort = one stable counting sort per 8-bit digit of the
// pixel id, over only ceil(log2 npix) key bits (3 passes at 1080p, 4 at 8K):
//   histogram  per tile of 4096 ids, the tile's digit counts (shared-memory atomics),
//              written digit-major [256][tiles];
//   scan       per digit, the exclusive scan of its counts over the tiles (one CTA
//              per digit, contiguous rows), plus the digit totals;
//   scatter    per tile: stable local ranks -- each warp walks its 512 ids in
//              rounds of 32 consecutive ids, __match_any_sync groups a round's equal
//              digits (rank = lanes before in the group + the warp's running count),
//              warps are ordered by a per-digit scan over the warps -- then the tile
//              is reordered in shared memory and written out as one contiguous run
//              per digit (coalesced). The last pass writes perm and, fused, gathers
//              each fragment's fields from its original index into its CSR slot
//              (a separate full-occupancy gather kernel after the sort measured 0.9 ms
//              slower at config 2: its reads, 32 scattered sectors per warp load,
//              multiply L2 traffic; the fused pass issues all of a thread's loads first).
// Bit-exact to the reference's numpy binning (tests/test_gpu_parity.py).
#include "common.cuh"
#include "internal.cuh"

namespace woit {
namespace bin {

constexpr int kThreads = 256, kWarps = kThreads / 32, kPerThread = 16;
constexpr int kTile = kThreads * kPerThread;  // 4096 ids per tile
constexpr int kRadix = 256;

int key_bits(int64_t npix) {
    int b = 1;
    while (b < 31 && (int64_t(1) << b) < npix) ++b;
    return b;
}

struct Plan {
    int64_t n, npix, tiles;
    int passes;
    // workspace carving
    int32_t *keys[2], *vals[2], *counts, *totals;
    size_t bytes;
};

Plan plan(int64_t n, int64_t npix, void* ws) {
    Plan p;
    p.n = n;
    p.npix = npix;
    p.tiles = (n + kTile - 1) / kTile;
    p.passes = (key_bits(npix) + 7) / 8;
    unsigned char* w = static_cast<unsigned char*>(ws);
    size_t o = 0;
    auto take = [&](size_t b) {
        unsigned char* q = w ? w + o : nullptr;
        o += (b + 255) & ~(size_t)255;
        return q;
    };
    const size_t nn = (size_t)(n > 0 ? n : 1);
    for (int i = 0; i < 2; ++i) {
        p.keys[i] = reinterpret_cast<int32_t*>(take(4 * nn));
        p.vals[i] = reinterpret_cast<int32_t*>(take(4 * nn));
    }
    p.counts = reinterpret_cast<int32_t*>(take(4 * (size_t)kRadix * (size_t)(p.tiles > 0 ? p.tiles : 1)));
    p.totals = reinterpret_cast<int32_t*>(take(4 * kRadix));
    p.bytes = o;
    return p;
}

template <typename K>
WOIT_D int key_at(const K* k, int64_t i) { return (int)k[i]; }

// tile digit histograms, digit-major: counts[d * tiles + t]
template <typename K>
__global__ void __launch_bounds__(kThreads) histogram_kernel(const K* __restrict__ keys, int64_t n, int shift,
                                                             int64_t tiles, int32_t* __restrict__ counts) {
    __shared__ int h[kRadix];
    const int64_t t = blockIdx.x;
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = t * kTile;
    if (sizeof(K) == 4 && base + kTile <= n && (reinterpret_cast<uintptr_t>(keys) & 15u) == 0) {
        // full 32-bit tile: 16-B loads, all issued before the counter updates
        const int4* k4 = reinterpret_cast<const int4*>(keys + base);
        int4 v[kPerThread / 4];
#pragma unroll
        for (int j = 0; j < kPerThread / 4; ++j) v[j] = __ldg(k4 + j * kThreads + threadIdx.x);
#pragma unroll
        for (int j = 0; j < kPerThread / 4; ++j) {
            atomicAdd(&h[(v[j].x >> shift) & (kRadix - 1)], 1);
            atomicAdd(&h[(v[j].y >> shift) & (kRadix - 1)], 1);
            atomicAdd(&h[(v[j].z >> shift) & (kRadix - 1)], 1);
            atomicAdd(&h[(v[j].w >> shift) & (kRadix - 1)], 1);
        }
    } else {
        int kv[kPerThread];
#pragma unroll
        for (int i = 0; i < kPerThread; ++i) {
            const int64_t e = base + i * kThreads + threadIdx.x;
            kv[i] = e < n ? key_at(keys, e) : -1;
        }
#pragma unroll
        for (int i = 0; i < kPerThread; ++i)
            if (kv[i] >= 0) atomicAdd(&h[(kv[i] >> shift) & (kRadix - 1)], 1);
    }
    __syncthreads();
    counts[(int64_t)threadIdx.x * tiles + t] = h[threadIdx.x];
}

// per digit (one CTA per digit): exclusive scan of its row over the tiles, and the total
__global__ void __launch_bounds__(1024) scan_rows_kernel(int32_t* __restrict__ counts, int64_t tiles,
                                                         int32_t* __restrict__ totals) {
    __shared__ int warp_sums[32];
    __shared__ int carry;
    int32_t* row = counts + (int64_t)blockIdx.x * tiles;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < tiles; c0 += 1024) {
        const int64_t i = c0 + threadIdx.x;
        const int v = i < tiles ? row[i] : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[wid] = x;
        __syncthreads();
        if (wid == 0) {
            int s = warp_sums[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            warp_sums[lane] = s;  // inclusive over warps
        }
        __syncthreads();
        const int excl = carry + (wid ? warp_sums[wid - 1] : 0) + x - v;
        if (i < tiles) row[i] = excl;
        __syncthreads();
        if (threadIdx.x == 0) carry += warp_sums[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) totals[blockIdx.x] = carry;
}

struct Gather {
    // fused field gather of the last pass (null `in.depth`: none)
    woit_frags_t in;
    woit_frags_t out;
    int64_t* perm;  // argsort(pix, stable); may be null
};

// one stable counting-sort pass over digit (key >> shift) & 255; GATHER (last pass
// only) scatters the fragment fields instead of the ids
template <typename K, bool FIRST, bool LAST, bool GATHER>
__global__ void __launch_bounds__(kThreads, GATHER ? 1 : 4) scatter_kernel(const K* __restrict__ keys_in,
                                                           const int32_t* __restrict__ vals_in, int64_t n,
                                                           int shift, int64_t tiles,
                                                           const int32_t* __restrict__ counts,
                                                           const int32_t* __restrict__ totals,
                                                           int32_t* __restrict__ keys_out,
                                                           int32_t* __restrict__ vals_out, const Gather g) {
    __shared__ int warp_cnt[kWarps][kRadix];  // running, then per-warp base of each digit
    __shared__ int tile_start[kRadix];        // digit's first slot in the reordered tile
    __shared__ int gbase[kRadix];             // digit's first global slot for this tile
    __shared__ int skey[kTile];
    __shared__ int sval[kTile];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t t = blockIdx.x;
    const int64_t base = t * kTile;
    const int tn = (int)((n - base) < kTile ? (n - base) : kTile);
    for (int i = threadIdx.x; i < kWarps * kRadix; i += kThreads) (&warp_cnt[0][0])[i] = 0;
    {   // the digit's global base: digits before it (exclusive scan of the totals) plus
        // the same digit in earlier tiles
        const int d = threadIdx.x;
        int x = totals[d];
        const int v = x;
        __shared__ int ws_[kWarps];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) ws_[w] = x;
        __syncthreads();
        int before = 0;
        for (int j = 0; j < w; ++j) before += ws_[j];
        gbase[d] = before + x - v + counts[(int64_t)d * tiles + t];
    }
    __syncthreads();
    // stable ranks within the warp's 512 consecutive ids, rounds of 32
    int kk[kPerThread], vv[kPerThread], rk[kPerThread];
#pragma unroll
    for (int r = 0; r < kPerThread; ++r) {
        const int le = w * (kPerThread * 32) + r * 32 + lane;  // tile-local element
        const bool act = le < tn;
        const int64_t e = base + le;
        const int key = act ? key_at(keys_in, e) : 0;
        const int val = act ? (FIRST ? (int)e : vals_in[e]) : 0;
        const int d = act ? (key >> shift) & (kRadix - 1) : kRadix;  // inactive lanes: their own group
        const unsigned grp = __match_any_sync(0xffffffffu, d);
        const int before = __popc(grp & ((1u << lane) - 1u));
        int run = 0;
        if (act) run = warp_cnt[w][d];
        __syncwarp();
        if (act && before == 0) warp_cnt[w][d] = run + __popc(grp);
        __syncwarp();
        kk[r] = key;
        vv[r] = val;
        rk[r] = act ? run + before : -1;
    }
    __syncthreads();
    {   // per digit: warps in order, then the tile's digit order
        const int d = threadIdx.x;
        int s = 0;
#pragma unroll
        for (int j = 0; j < kWarps; ++j) {
            const int c = warp_cnt[j][d];
            warp_cnt[j][d] = s;
            s += c;
        }
        int x = s;
        const int v = s;
        __shared__ int ws2[kWarps];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) ws2[w] = x;
        __syncthreads();
        int before = 0;
        for (int j = 0; j < w; ++j) before += ws2[j];
        tile_start[d] = before + x - v;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kPerThread; ++r) {
        if (rk[r] < 0) continue;
        const int d = (kk[r] >> shift) & (kRadix - 1);
        const int pos = tile_start[d] + warp_cnt[w][d] + rk[r];
        skey[pos] = kk[r];
        sval[pos] = vv[r];
    }
    __syncthreads();
    // out: one contiguous run per digit
    if (!GATHER) {
        for (int i = threadIdx.x; i < tn; i += kThreads) {
            const int key = skey[i], val = sval[i];
            const int d = (key >> shift) & (kRadix - 1);
            const int64_t gp = (int64_t)gbase[d] + (i - tile_start[d]);
            keys_out[gp] = key;
            if (!LAST) vals_out[gp] = val;
            if (LAST && g.perm) g.perm[gp] = val;
        }
    } else {
        // last pass with the fused gather: every fragment's fields from its arrival slot
        // into its CSR slot. The reads are random, so each thread first issues the
        // loads of all its fragments (memory-level parallelism), then stores them.
        const woit_frags_t a = g.in, b = g.out;
        constexpr int kG = kPerThread;
        float dep[kG], alp[kG], tr[kG][3], ra[kG][3];
        int64_t gps[kG];
        int vals[kG];
#pragma unroll
        for (int j = 0; j < kG; ++j) {
            const int i = threadIdx.x + j * kThreads;
            gps[j] = -1;
            if (i < tn) {
                const int key = skey[i], val = sval[i];
                const int d = (key >> shift) & (kRadix - 1);
                gps[j] = (int64_t)gbase[d] + (i - tile_start[d]);
                vals[j] = val;
                keys_out[gps[j]] = key;
                const int64_t v = val;
                dep[j] = __ldg(a.depth + v);
                alp[j] = a.alpha ? __ldg(a.alpha + v) : 0.0f;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    tr[j][c] = a.trans ? __ldg(a.trans + 3 * v + c) : 0.0f;
                    ra[j][c] = a.radiance ? __ldg(a.radiance + 3 * v + c) : 0.0f;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < kG; ++j) {
            if (gps[j] < 0) continue;
            const int64_t gp = gps[j], v = vals[j];
            if (g.perm) g.perm[gp] = v;
            const_cast<float*>(b.depth)[gp] = dep[j];
            if (a.alpha) const_cast<float*>(b.alpha)[gp] = alp[j];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (a.trans) const_cast<float*>(b.trans)[3 * gp + c] = tr[j][c];
                if (a.radiance) const_cast<float*>(b.radiance)[3 * gp + c] = ra[j][c];
            }
            if (a.normal)
#pragma unroll
                for (int c = 0; c < 3; ++c) const_cast<float*>(b.normal)[3 * gp + c] = __ldg(a.normal + 3 * v + c);
            if (a.ior) const_cast<float*>(b.ior)[gp] = __ldg(a.ior + v);
            if (a.backface) const_cast<uint8_t*>(b.backface)[gp] = __ldg(a.backface + v);
        }
    }
}

// offsets[p] = lower_bound(sorted keys, p): at every key change (and the ends) the
// thread writes the boundaries of the pixels in between (empty pixels included)
__global__ void offsets_kernel(const int32_t* __restrict__ keys, int64_t n, int64_t npix, int64_t* __restrict__ offsets) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = i == 0 ? 0 : (int64_t)keys[i - 1] + 1;  // pixels whose run starts at i
        const int64_t hi = i == n ? npix : (int64_t)keys[i];
        for (int64_t p = lo; p <= hi; ++p) offsets[p] = i;
    }
}

template <typename K>
cudaError_t run(const K* pix, int64_t n, int64_t npix, int64_t* offsets, const Gather& g, void* ws,
                cudaStream_t st) {
    if (n == 0) return cudaMemsetAsync(offsets, 0, (size_t)(npix + 1) * 8, st);
    Plan p = plan(n, npix, ws);
    const unsigned tiles = (unsigned)p.tiles;
    const int32_t* kin = nullptr;
    const int32_t* vin = nullptr;
    int cur = 0;
    for (int pass = 0; pass < p.passes; ++pass) {
        const int shift = 8 * pass;
        const bool first = pass == 0, last = pass == p.passes - 1;
        if (first)
            histogram_kernel<K><<<tiles, kThreads, 0, st>>>(pix, n, shift, p.tiles, p.counts);
        else
            histogram_kernel<int32_t><<<tiles, kThreads, 0, st>>>(kin, n, shift, p.tiles, p.counts);
        scan_rows_kernel<<<kRadix, 1024, 0, st>>>(p.counts, p.tiles, p.totals);
        int32_t* ko = p.keys[cur];
        int32_t* vo = p.vals[cur];
        const bool gather = last && g.in.depth;
        const dim3 gr(tiles), bl(kThreads);
        if (first && last)
            gather ? scatter_kernel<K, true, true, true><<<gr, bl, 0, st>>>(pix, nullptr, n, shift, p.tiles, p.counts,
                                                                              p.totals, ko, vo, g)
                   : scatter_kernel<K, true, true, false><<<gr, bl, 0, st>>>(pix, nullptr, n, shift, p.tiles,
                                                                               p.counts, p.totals, ko, vo, g);
        else if (first)
            scatter_kernel<K, true, false, false><<<gr, bl, 0, st>>>(pix, nullptr, n, shift, p.tiles, p.counts,
                                                                       p.totals, ko, vo, g);
        else if (last)
            gather ? scatter_kernel<int32_t, false, true, true><<<gr, bl, 0, st>>>(kin, vin, n, shift, p.tiles,
                                                                                    p.counts, p.totals, ko, vo, g)
                   : scatter_kernel<int32_t, false, true, false><<<gr, bl, 0, st>>>(kin, vin, n, shift, p.tiles,
                                                                                     p.counts, p.totals, ko, vo, g);
        else
            scatter_kernel<int32_t, false, false, false><<<gr, bl, 0, st>>>(kin, vin, n, shift, p.tiles, p.counts,
                                                                              p.totals, ko, vo, g);
        cudaError_t err = cudaGetLastError();
        if (err != cudaSuccess) return err;
        kin = ko;
        vin = vo;
        cur ^= 1;
    }
    const int64_t g2 = (n + 256) / 256;
    offsets_kernel<<<(unsigned)(g2 < 8192 ? g2 : 8192), 256, 0, st>>>(kin, n, npix, offsets);
    return cudaGetLastError();
}

}  // namespace bin

size_t bin_workspace(int64_t n, int64_t npix) { return bin::plan(n, npix, nullptr).bytes; }

cudaError_t bin_by_pixel(const int64_t* pix, int64_t n, int64_t npix, int64_t* offsets, int64_t* perm, void* ws,
                         size_t ws_bytes, cudaStream_t st) {
    (void)ws_bytes;
    bin::Gather g = {};
    g.perm = perm;
    // perm is int64 in the ABI; the sort carries int32 ids and widens in the last pass
    return bin::run<int64_t>(pix, n, npix, offsets, g, ws, st);
}

cudaError_t bin_frame(const int32_t* pix, int64_t n, int64_t npix, const woit_frags_t& in, const woit_frags_t& out,
                      int64_t* offsets, int64_t* perm, void* ws, cudaStream_t st) {
    bin::Gather g = {};
    g.in = in;
    g.out = out;
    g.perm = perm;
    return bin::run<int32_t>(pix, n, npix, offsets, g, ws, st);
}

}  // namespace woit
