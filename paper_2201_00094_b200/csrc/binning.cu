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
//              rounds of 32 consecutive ids, eight ballots group a round's equal
//              digits (rank = lanes before in the group + the warp's running count),
//              warps are ordered by a per-digit scan over the warps -- then the tile
//              is reordered in shared memory and written out as one contiguous run
//              per digit (coalesced). The last pass writes perm.
// The fields of bin_frame then move in CSR order by gather_kernel: a tile of 32
// pixels at a time, lanes = pixels and warps = each pixel's k-th fragments, so a warp
// load reads the k-th fragments of 32 consecutive pixels -- consecutive arrival slots
// when the producer emits the frame layer by layer -- and the tile leaves through
// shared memory as contiguous runs. (It replaced a gather fused into the last pass,
// whose reads from the arrival slots of pixel-sorted ids scattered over 32 sectors
// per warp load: 4 ms of the 6.1 ms at config 2.)
// Bit-exact to the reference's numpy binning (tests/test_gpu_parity.py).
#include "common.cuh"
#include "internal.cuh"

namespace woit {
namespace bin {

#ifndef WOIT_BIN_PER_THREAD  // ids per thread of a radix tile
#define WOIT_BIN_PER_THREAD 16  // 4,096-id tiles (8 with 6 CTAs per SM: faster scatters, slower histograms and scans, the same total)
#endif
constexpr int kThreads = 256, kWarps = kThreads / 32, kPerThread = WOIT_BIN_PER_THREAD;
constexpr int kTile = kThreads * kPerThread;  // ids per tile
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
    // fields moved into CSR order after the sort (null `in.depth`: none)
    woit_frags_t in;
    woit_frags_t out;
    int64_t* perm;  // argsort(pix, stable); may be null
};

// one stable counting-sort pass over digit (key >> shift) & 255; the last pass writes
// perm (int64, if asked) and, for the field gather, the int32 ids (`vals_out` non-null)
#ifndef WOIT_BIN_MINB
#define WOIT_BIN_MINB 4
#endif
template <typename K, bool FIRST, bool LAST>
__global__ void __launch_bounds__(kThreads, WOIT_BIN_MINB) scatter_kernel(const K* __restrict__ keys_in,
                                                              const int32_t* __restrict__ vals_in, int64_t n,
                                                              int shift, int dbits, int64_t tiles,
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
    // stable ranks within the warp's 512 consecutive ids, rounds of 32; every key and
    // id is loaded first (the rounds' __syncwarp would otherwise serialise the loads)
    int kk[kPerThread], vv[kPerThread], rk[kPerThread];
#pragma unroll
    for (int r = 0; r < kPerThread; ++r) {
        const int le = w * (kPerThread * 32) + r * 32 + lane;  // tile-local element
        const int64_t e = base + le;
        kk[r] = le < tn ? key_at(keys_in, e) : 0;
        vv[r] = le < tn ? (FIRST ? (int)e : vals_in[e]) : 0;
    }
#pragma unroll
    for (int r = 0; r < kPerThread; ++r) {
        const int le = w * (kPerThread * 32) + r * 32 + lane;  // tile-local element
        const bool act = le < tn;
        const int key = kk[r];
        const int d = act ? (key >> shift) & (kRadix - 1) : kRadix;  // inactive lanes: their own group
        // lanes with the same digit: one ballot per digit bit (a warp multisplit; the
        // hardware match instruction measured 35% of this kernel's stalls)
        unsigned grp = __ballot_sync(0xffffffffu, act);
        grp = act ? grp : ~grp;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            if (b < dbits) {  // the digit's significant bits only (the top pass has fewer)
                const bool bit = (d >> b) & 1;
                const unsigned m = __ballot_sync(0xffffffffu, bit);
                grp &= bit ? m : ~m;
            }
        }
        const int before = __popc(grp & ((1u << lane) - 1u));
        // the group's leader advances the warp's running count of the digit (shared
        // atomics of one warp to one address apply in program order, so the rounds
        // need no barrier between them) and hands the old count to its group
        const int leader = __ffs(grp) - 1;
        int run = 0;
        if (act && before == 0) run = atomicAdd(&warp_cnt[w][d], __popc(grp));
        run = __shfl_sync(0xffffffffu, run, leader);
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
    for (int i = threadIdx.x; i < tn; i += kThreads) {
        const int key = skey[i], val = sval[i];
        const int d = (key >> shift) & (kRadix - 1);
        const int64_t gp = (int64_t)gbase[d] + (i - tile_start[d]);
        keys_out[gp] = key;
        if (!LAST || vals_out) vals_out[gp] = val;
        if (LAST && g.perm) g.perm[gp] = val;
    }
}

// offsets[p] = lower_bound(sorted keys, p): at every key change (and the ends) the
// thread writes the boundaries of the pixels in between (empty pixels included).
// Four keys per thread (one 16-B load; `keys` is 16-B aligned) plus the one before.
__global__ void offsets_kernel(const int32_t* __restrict__ keys, int64_t n, int64_t npix, int64_t* __restrict__ offsets) {
    const int64_t n4 = n / 4;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= n4; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = 4 * j;
        int k[4];
        int cnt = 4;
        if (j < n4) {
            const int4 v = __ldg(reinterpret_cast<const int4*>(keys) + j);
            k[0] = v.x, k[1] = v.y, k[2] = v.z, k[3] = v.w;
        } else {  // the tail (< 4 keys) and the end i == n
            cnt = (int)(n - i0);
#pragma unroll
            for (int m = 0; m < 4; ++m) k[m] = m < cnt ? keys[i0 + m] : 0;
        }
        int64_t prev = i0 == 0 ? -1 : (int64_t)keys[i0 - 1];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            if (m < cnt) {
                for (int64_t p = prev + 1; p <= k[m]; ++p) offsets[p] = i0 + m;  // pixels whose run starts here
                prev = k[m];
            }
        }
        if (j == n4)  // the last thread: the pixels after the last key end at n
            for (int64_t p = prev + 1; p <= npix; ++p) offsets[p] = n;
    }
}

// Fields into CSR order: out[s] = in[perm[s]] for every field present. One tile of
// kGP = 32 pixels per iteration: lane = pixel, warp w takes the pixel's fragments
// k = kc + w, kc + w + 8, ... of the chunk [kc, kc + kGK); a thread issues all its
// id and field loads before staging them in shared memory ([field][k][pixel], rows of
// 33: conflict-free both ways); the chunk then leaves as each pixel's run of slots,
// consecutive threads on consecutive slots. Tiles with a pixel deeper than kGDeep
// copy slot by slot instead (a pixel's k-th fragments have no neighbours to share
// sectors with).
constexpr int kGT = 256, kGW = kGT / 32, kGP = 32, kGK = 32, kGDeep = 4096;
constexpr int kGPlane = kGK * (kGP + 1);  // floats per staged field

template <bool REFR>
__global__ void __launch_bounds__(kGT) gather_kernel(const int64_t* __restrict__ offsets,
                                                     const int32_t* __restrict__ perm, int64_t npix,
                                                     const woit_frags_t in, const woit_frags_t out) {
    extern __shared__ float gst[];  // [planes][kGK][kGP + 1] (+ backface bytes)
    constexpr int NPL = REFR ? 12 : 8;  // depth, alpha, trans 3, radiance 3 (+ normal 3, ior)
    uint8_t* gbf = reinterpret_cast<uint8_t*>(gst + NPL * kGPlane);
    __shared__ int s_len[kGP];          // chunk run-length prefix over the tile's pixels
    __shared__ int64_t s_slot[kGP];     // first slot of the pixel's chunk run
    __shared__ uint8_t s_own[kGP * kGK];  // chunk output position -> pixel
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const bool has_a = in.alpha, has_t = in.trans, has_r = in.radiance;
    const bool has_n = REFR && in.normal, has_i = REFR && in.ior, has_b = REFR && in.backface;
    float* od = const_cast<float*>(out.depth);
    float* oa = const_cast<float*>(out.alpha);
    float* ot = const_cast<float*>(out.trans);
    float* orad = const_cast<float*>(out.radiance);
    float* on = const_cast<float*>(out.normal);
    float* oi = const_cast<float*>(out.ior);
    uint8_t* ob_ = const_cast<uint8_t*>(out.backface);
    const int64_t ntile = (npix + kGP - 1) / kGP;
    for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
        const int64_t p0 = tile * kGP;
        const int np = (int)((npix - p0) < kGP ? (npix - p0) : kGP);
        const int64_t o_p = offsets[p0 + (lane < np ? lane : np)];
        const int c_p = lane < np ? (int)(offsets[p0 + lane + 1] - o_p) : 0;
        const int cmax = __reduce_max_sync(0xffffffffu, c_p);
        if (cmax > kGDeep) {  // slot by slot
            const int64_t s0 = __shfl_sync(0xffffffffu, o_p, 0), s1 = offsets[p0 + np];
            for (int64_t s = s0 + threadIdx.x; s < s1; s += kGT) {
                const int64_t a = perm[s];
                od[s] = in.depth[a];
                if (has_a) oa[s] = in.alpha[a];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    if (has_t) ot[3 * s + c] = in.trans[3 * a + c];
                    if (has_r) orad[3 * s + c] = in.radiance[3 * a + c];
                    if (has_n) on[3 * s + c] = in.normal[3 * a + c];
                }
                if (has_i) oi[s] = in.ior[a];
                if (has_b) ob_[s] = in.backface[a];
            }
            continue;
        }
        for (int kc = 0; kc < cmax; kc += kGK) {
            // read: ids, then the fields of this thread's (pixel, k) pairs
            constexpr int KPW = kGK / kGW;  // pairs per thread
            int64_t a[KPW];
#pragma unroll
            for (int j = 0; j < KPW; ++j) {
                const int k = kc + w + kGW * j;
                a[j] = k < c_p ? (int64_t)perm[o_p + k] : -1;
            }
            float f[KPW][NPL];
            uint8_t fb[KPW];
#pragma unroll
            for (int j = 0; j < KPW; ++j) {
                if (a[j] < 0) continue;
                const int64_t x = a[j];
                f[j][0] = __ldg(in.depth + x);
                f[j][1] = has_a ? __ldg(in.alpha + x) : 0.0f;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    f[j][2 + c] = has_t ? __ldg(in.trans + 3 * x + c) : 0.0f;
                    f[j][5 + c] = has_r ? __ldg(in.radiance + 3 * x + c) : 0.0f;
                    if (REFR) f[j][8 + c] = has_n ? __ldg(in.normal + 3 * x + c) : 0.0f;
                }
                if (REFR) f[j][NPL - 1] = has_i ? __ldg(in.ior + x) : 0.0f;
                fb[j] = has_b ? __ldg(in.backface + x) : 0;
            }
            // the chunk's run per pixel and its prefix over the tile (every warp forms it)
            const int len = c_p - kc < 0 ? 0 : (c_p - kc < kGK ? c_p - kc : kGK);
            int incl = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int excl = incl - len;
            if (w == 0) {
                s_len[lane] = excl;
                s_slot[lane] = o_p + kc;
            }
#pragma unroll
            for (int j = 0; j < KPW; ++j) {
                if (a[j] < 0) continue;
                const int kk = w + kGW * j;
                const int r = kk * (kGP + 1) + lane;
#pragma unroll
                for (int q = 0; q < NPL; ++q) gst[q * kGPlane + r] = f[j][q];
                if (has_b) gbf[r] = fb[j];
                s_own[excl + kk] = (uint8_t)lane;  // output position -> its pixel
            }
            __syncthreads();
            // write: the runs, consecutive threads on consecutive slots
            const int tot = __shfl_sync(0xffffffffu, incl, 31);
            for (int e = threadIdx.x; e < tot; e += kGT) {
                const int q = s_own[e], kk = e - s_len[q];
                const int64_t s = s_slot[q] + kk;
                const int r = kk * (kGP + 1) + q;
                od[s] = gst[r];
                if (has_a) oa[s] = gst[kGPlane + r];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    if (has_t) ot[3 * s + c] = gst[(2 + c) * kGPlane + r];
                    if (has_r) orad[3 * s + c] = gst[(5 + c) * kGPlane + r];
                    if (has_n) on[3 * s + c] = gst[(8 + c) * kGPlane + r];
                }
                if (has_i) oi[s] = gst[(NPL - 1) * kGPlane + r];
                if (has_b) ob_[s] = gbf[r];
            }
            __syncthreads();
        }
    }
}

template <bool REFR>
constexpr size_t gather_smem() { return (REFR ? 12 : 8) * kGPlane * sizeof(float) + kGPlane; }

template <bool REFR>
cudaError_t launch_gather(const int64_t* offsets, const int32_t* perm, int64_t npix, const Gather& g,
                          cudaStream_t st) {
    const size_t smem = gather_smem<REFR>();
    // the opt-in attribute and the occupancy: frame.cu's cached, thread-safe query
    int sms = 148, per = 1;
    cudaError_t err = launch_config(reinterpret_cast<const void*>(gather_kernel<REFR>), kGT, (int)smem, sms, per);
    if (err != cudaSuccess) return err;
    const int64_t ntile = (npix + kGP - 1) / kGP;
    int64_t grid = (int64_t)sms * (per > 0 ? per : 1);
    grid = grid < ntile ? grid : ntile;
    gather_kernel<REFR><<<(unsigned)grid, kGT, smem, st>>>(offsets, perm, npix, g.in, g.out);
    return cudaGetLastError();
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
        const int kb = key_bits(npix), dbits = kb - shift < 8 ? kb - shift : 8;
        const bool first = pass == 0, last = pass == p.passes - 1;
        if (first)
            histogram_kernel<K><<<tiles, kThreads, 0, st>>>(pix, n, shift, p.tiles, p.counts);
        else
            histogram_kernel<int32_t><<<tiles, kThreads, 0, st>>>(kin, n, shift, p.tiles, p.counts);
        scan_rows_kernel<<<kRadix, 1024, 0, st>>>(p.counts, p.tiles, p.totals);
        int32_t* ko = p.keys[cur];
        int32_t* vo = p.vals[cur];
        // the field gather needs the int32 ids of the last pass
        int32_t* vlast = g.in.depth ? vo : nullptr;
        const dim3 gr(tiles), bl(kThreads);
        if (first && last)
            scatter_kernel<K, true, true><<<gr, bl, 0, st>>>(pix, nullptr, n, shift, dbits, p.tiles, p.counts, p.totals, ko,
                                                             vlast, g);
        else if (first)
            scatter_kernel<K, true, false><<<gr, bl, 0, st>>>(pix, nullptr, n, shift, dbits, p.tiles, p.counts, p.totals, ko,
                                                              vo, g);
        else if (last)
            scatter_kernel<int32_t, false, true><<<gr, bl, 0, st>>>(kin, vin, n, shift, dbits, p.tiles, p.counts, p.totals,
                                                                    ko, vlast, g);
        else
            scatter_kernel<int32_t, false, false><<<gr, bl, 0, st>>>(kin, vin, n, shift, dbits, p.tiles, p.counts, p.totals,
                                                                     ko, vo, g);
        cudaError_t err = cudaGetLastError();
        if (err != cudaSuccess) return err;
        kin = ko;
        vin = vo;
        cur ^= 1;
    }
    const int64_t g2 = (n / 4 + 256) / 256;
    offsets_kernel<<<(unsigned)(g2 < 8192 ? g2 : 8192), 256, 0, st>>>(kin, n, npix, offsets);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess || !g.in.depth) return err;
    const bool refr = g.in.normal || g.in.ior || g.in.backface;
    return refr ? launch_gather<true>(offsets, vin, npix, g, st) : launch_gather<false>(offsets, vin, npix, g, st);
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
