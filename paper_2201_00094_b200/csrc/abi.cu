// extern "C" entry points of libwoit.so (declared in include/woit.h): argument
// validation, workspace carving and launch. No allocation, no global state.
#include <cmath>

#include "frame.cuh"
#include "internal.cuh"

using namespace woit;

namespace {

constexpr int64_t kMinFB = 256;
constexpr int kMaxDiffusionRadius = 64;  // smallest sub-tile (rank 6): bounds the long-pixel list

int64_t long_cap(int64_t nfrag) { return nfrag / (kMinFB + 1) + 2; }

inline int cuda_status(cudaError_t e) { return e == cudaSuccess ? WOIT_OK : WOIT_ECUDA; }

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int check_params(const woit_params_t* p) {
    if (!p) return WOIT_EINVAL;
    if (p->rank < 0 || p->rank > kMaxRank) return WOIT_ERANK;
    if (p->aberration_taps < 3 || (p->aberration_taps % 2) == 0) return WOIT_ETAPS;
    if ((p->flags & WOIT_DIFFUSION) &&
        (!(p->diffusion >= 0.0) || !std::isfinite(p->diffusion) || p->diffusion_radius < 1 ||
         p->diffusion_radius > kMaxDiffusionRadius))
        return WOIT_EINVAL;
    return WOIT_OK;
}

int check_frags(const woit_frags_t* f, bool need_frag_arrays) {
    if (!f) return WOIT_EINVAL;
    if (f->width < 1 || f->height < 1 || f->npix < 0 || f->nfrag < 0) return WOIT_EINVAL;
    if (!f->offsets) return WOIT_EINVAL;
    if (need_frag_arrays && f->nfrag > 0 && (!f->depth || !f->alpha || !f->trans || !f->radiance))
        return WOIT_EINVAL;
    return WOIT_OK;
}

// aberration taps for the kernels (frame.cuh TapTable), with the reference's f64
// operation order (spectral_weight's host branch keeps every rounding)
void fill_taps(KParams& kp) {
    const int k = kp.p.aberration_taps;
    kp.taps.n = 0;
    kp.taps.unit = 0;
    if (!(kp.p.flags & WOIT_CHROMATIC_ABERRATION) || k < 3 || k > kMaxTapTable) return;
    const bool lit = kp.p.flags & WOIT_LITERAL_SPECTRAL_T;
    for (int i = 0; i < k; ++i) {
        spectral_weight(i, k, lit, kp.taps.w[i]);
        volatile double two_i = 2.0 * i;
        kp.taps.fac[i] = two_i / (double)(k - 1);
    }
    kp.taps.n = k;
    int unit = 1;
    for (int i = 0; i < k; ++i)
        for (int c = 0; c < 3; ++c) unit &= (kp.taps.w[i][c] == 0.0 || kp.taps.w[i][c] == 1.0) ? 1 : 0;
    kp.taps.unit = unit;
}

int run_frame(const woit_frags_t* f, const woit_params_t* p, woit_bufs_t* b, uint32_t phases, void* ws,
              size_t ws_bytes, void* stream) {
    if (!b) return WOIT_EINVAL;
    if (f->npix == 0) return WOIT_OK;
    if (ws_bytes < woit_frame_workspace_bytes(f->npix, f->nfrag) || !ws) return WOIT_EWORKSPACE;
    if ((phases & PH_COMPOSITE) && (!b->output || !f->opaque_color)) return WOIT_EINVAL;
    if ((phases & PH_COMPOSITE) && (p->flags & WOIT_DIFFUSION) && !b->blurred_image) return WOIT_EINVAL;
    if ((phases & (PH_BOUNDS_ACC)) && (!b->near || !b->far)) return WOIT_EINVAL;
    if (!(phases & PH_BOUNDS) && (!b->near || !b->far)) return WOIT_EINVAL;
    if ((phases & PH_BUILD_ACC) && !b->coeffs) return WOIT_EINVAL;
    if (!(phases & PH_BUILD) && (phases & (PH_EVAL | PH_COMPOSITE)) && !b->coeffs) return WOIT_EINVAL;
    if ((phases & PH_EVAL_ACC) && (!b->accum || !b->weight)) return WOIT_EINVAL;
    if ((phases & PH_EVAL) && (p->flags & WOIT_REFRACTION) && f->nfrag > 0 && !f->normal) return WOIT_EINVAL;
    KParams kp;
    kp.f = *f;
    kp.p = *p;
    kp.b = *b;
    kp.phases = phases;
    fill_taps(kp);
    const void* ptrs[] = {f->depth, f->alpha, f->trans, f->radiance, f->normal, f->ior, f->backface, b->vhat,
                          f->opaque_color};
    bool al = true;
    for (const void* q : ptrs) al = al && (q == nullptr || aligned16(q));
    kp.use_tma = al ? 1 : 0;
    // workspace: [0] window counter, [1] window-order counters, [2] long-pixel count,
    // [3 .. 3 + long_cap) long-pixel list, then the window order (int32 per window)
    kp.win_counter = static_cast<unsigned long long*>(ws);
    kp.order_cnt = reinterpret_cast<unsigned*>(static_cast<int64_t*>(ws) + 1);
    kp.long_list = static_cast<int64_t*>(ws) + 2;
    kp.long_cap = long_cap(f->nfrag);
    kp.win_order = reinterpret_cast<int32_t*>(static_cast<int64_t*>(ws) + 3 + kp.long_cap);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t err = cudaMemsetAsync(ws, 0, 3 * sizeof(int64_t), st);
    if (err != cudaSuccess) return WOIT_ECUDA;
    return cuda_status(launch_frame(kp, st));
}

}  // namespace

extern "C" {

int woit_abi_version(void) { return WOIT_ABI_VERSION; }

const char* woit_status_string(int status) {
    switch (status) {
        case WOIT_OK: return "ok";
        case WOIT_EINVAL: return "invalid argument";
        case WOIT_EWORKSPACE: return "workspace too small";
        case WOIT_ECUDA: return "CUDA error";
        case WOIT_ERANK: return "rank must lie in [0, 6]";
        case WOIT_ETAPS: return "aberration taps must be odd and >= 3";
        default: return "unknown status";
    }
}

size_t woit_frame_workspace_bytes(int64_t npix, int64_t nfrag) {
    // counters, long-pixel list, window order (run_frame)
    return (size_t)(3 + long_cap(nfrag)) * sizeof(int64_t) + (size_t)((npix + 31) / 32) * sizeof(int32_t);
}

int woit_render_band(const woit_frags_t* frags, const woit_params_t* params, woit_bufs_t* bufs, void* ws,
                     size_t ws_bytes, void* stream) {
    int s = check_params(params);
    if (s) return s;
    if ((s = check_frags(frags, true))) return s;
    return run_frame(frags, params, bufs, PH_BOUNDS | PH_BUILD | PH_EVAL | PH_COMPOSITE, ws, ws_bytes, stream);
}

int woit_step1_depth_bounds(const woit_frags_t* frags, woit_bufs_t* bufs, void* ws, size_t ws_bytes,
                            void* stream) {
    int s = check_frags(frags, false);
    if (s) return s;
    if (frags->nfrag > 0 && !frags->depth) return WOIT_EINVAL;
    woit_params_t p = {};
    p.rank = 0;
    p.aberration_taps = 5;
    woit_bufs_t b = {};
    if (!bufs) return WOIT_EINVAL;
    b.near = bufs->near;
    b.far = bufs->far;
    return run_frame(frags, &p, &b, PH_BOUNDS | PH_BOUNDS_ACC, ws, ws_bytes, stream);
}

int woit_step2_build(const woit_frags_t* frags, const woit_params_t* params, woit_bufs_t* bufs, void* ws,
                     size_t ws_bytes, void* stream) {
    int s = check_params(params);
    if (s) return s;
    if ((s = check_frags(frags, false))) return s;
    if (frags->nfrag > 0 && (!frags->depth || !frags->alpha || !frags->trans)) return WOIT_EINVAL;
    if (!bufs || !bufs->coeffs) return WOIT_EINVAL;
    woit_bufs_t b = {};
    b.near = bufs->near;
    b.far = bufs->far;
    b.coeffs = bufs->coeffs;
    b.coeff_words = bufs->coeff_words;  // packed storage: the words of the accumulated coefficients
    return run_frame(frags, params, &b, PH_BUILD | PH_BUILD_ACC, ws, ws_bytes, stream);
}

int woit_step3_accumulate(const woit_frags_t* frags, const woit_params_t* params, woit_bufs_t* bufs,
                          void* ws, size_t ws_bytes, void* stream) {
    int s = check_params(params);
    if (s) return s;
    if ((s = check_frags(frags, true))) return s;
    if (!bufs) return WOIT_EINVAL;
    woit_bufs_t b = *bufs;
    b.output = nullptr;
    return run_frame(frags, params, &b, PH_EVAL | PH_EVAL_ACC, ws, ws_bytes, stream);
}

int woit_step4_composite(const woit_frags_t* frags, const woit_params_t* params, woit_bufs_t* bufs,
                         void* stream) {
    int s = check_params(params);
    if (s) return s;
    if (!frags || frags->width < 1 || frags->height < 1 || frags->npix < 0) return WOIT_EINVAL;
    if (!bufs || !bufs->coeffs || !bufs->accum || !bufs->weight || !bufs->output || !frags->opaque_color)
        return WOIT_EINVAL;
    if ((params->flags & WOIT_DIFFUSION) && (!bufs->blurred_image || !bufs->diffusion)) return WOIT_EINVAL;
    KParams kp;
    kp.f = *frags;
    kp.p = *params;
    kp.b = *bufs;
    kp.phases = PH_COMPOSITE;
    fill_taps(kp);
    kp.use_tma = 0;
    kp.long_list = nullptr;
    kp.long_cap = 0;
    kp.win_counter = nullptr;
    kp.order_cnt = nullptr;
    kp.win_order = nullptr;
    return cuda_status(launch_composite(kp, static_cast<cudaStream_t>(stream)));
}

int woit_fragment_indices(const woit_frags_t* frags, const float* near, const float* far, int rank, double* z,
                          int32_t* slots, int32_t* cells, void* stream) {
    if (rank < 0 || rank > kMaxRank) return WOIT_ERANK;
    if (!frags || !frags->offsets || !near || !far || frags->npix < 0) return WOIT_EINVAL;
    if (frags->nfrag > 0 && (!frags->depth || !z || !slots || !cells)) return WOIT_EINVAL;
    KParams kp = {};
    kp.f = *frags;
    kp.p.rank = rank;
    kp.b.near = const_cast<float*>(near);
    kp.b.far = const_cast<float*>(far);
    return cuda_status(launch_indices(kp, z, slots, cells, static_cast<cudaStream_t>(stream)));
}

size_t woit_cast_workspace_bytes(int64_t npix) { return npix < 0 ? 0 : cast_workspace(npix); }

static int check_scene(const woit_scene_t* s, int32_t W, int32_t H) {
    if (!s || W < 1 || H < 1 || s->nprims < 0 || (s->nprims > 0 && !s->prims)) return WOIT_EINVAL;
    if (s->bg_has_checker && s->bg_cell < 1) return WOIT_EINVAL;
    if ((int64_t)W * H >= ((int64_t)1 << 31)) return WOIT_EINVAL;  // CUB scan item count
    return WOIT_OK;
}

int woit_cast_offsets(const woit_scene_t* scene, int32_t width, int32_t height, int64_t* offsets, void* ws,
                      size_t ws_bytes, void* stream) {
    int s = check_scene(scene, width, height);
    if (s) return s;
    if (!offsets) return WOIT_EINVAL;
    if (!ws || ws_bytes < cast_workspace((int64_t)width * height)) return WOIT_EWORKSPACE;
    return cuda_status(cast_count(*scene, width, height, offsets, ws, static_cast<cudaStream_t>(stream)));
}

int woit_cast_fill(const woit_scene_t* scene, int32_t width, int32_t height, const int64_t* offsets, float* depth,
                   float* alpha, float* trans, float* radiance, float* normal, float* ior, uint8_t* backface,
                   float* opaque_depth, float* opaque_color, void* stream) {
    int s = check_scene(scene, width, height);
    if (s) return s;
    if (!offsets || !depth || !alpha || !trans || !radiance || !normal || !ior || !backface || !opaque_depth ||
        !opaque_color)
        return WOIT_EINVAL;
    return cuda_status(cast_fill(*scene, width, height, offsets, depth, alpha, trans, radiance, normal, ior, backface,
                                 opaque_depth, opaque_color, static_cast<cudaStream_t>(stream)));
}

size_t woit_baseline_workspace_bytes(int method, int64_t npix, int64_t nfrag) {
    if (method < WOIT_METHOD_ABUFFER || method > WOIT_METHOD_MLAB4 || npix < 0 || nfrag < 0) return 0;
    return baseline_workspace(method, npix, nfrag);
}

int woit_render_baseline(const woit_frags_t* frags, int method, int flags, const double* wboit_weight, float* output,
                         void* ws, size_t ws_bytes, void* stream) {
    if (method < WOIT_METHOD_ABUFFER || method > WOIT_METHOD_MLAB4) return WOIT_EINVAL;
    int s = check_frags(frags, true);
    if (s) return s;
    if (!output || !frags->opaque_color || (method == WOIT_METHOD_WBOIT && !wboit_weight)) return WOIT_EINVAL;
    if (method == WOIT_METHOD_ABUFFER && frags->nfrag >= ((int64_t)1 << 31)) return WOIT_EINVAL;
    if (!ws || ws_bytes < baseline_workspace(method, frags->npix, frags->nfrag)) return WOIT_EWORKSPACE;
    const double zero[3] = {0.0, 0.0, 0.0};
    return cuda_status(render_baseline(*frags, method, (flags & WOIT_CUBE_TRANSMISSION) != 0,
                                       wboit_weight ? wboit_weight : zero, output, ws,
                                       static_cast<cudaStream_t>(stream)));
}

size_t woit_build_atomic_workspace_bytes(int64_t npix) { return npix < 0 ? 0 : build_atomic_workspace(npix); }

int woit_build_atomic(const woit_frags_t* frags, const int32_t* pix, const woit_params_t* params, woit_bufs_t* bufs,
                      void* ws, size_t ws_bytes, void* stream) {
    int s = check_params(params);
    if (s) return s;
    if (!frags || frags->npix < 0 || frags->nfrag < 0 || !bufs) return WOIT_EINVAL;
    if (params->flags & WOIT_PACKED_STORAGE) return WOIT_EINVAL;
    if (!bufs->near || !bufs->far || !bufs->coeffs) return WOIT_EINVAL;
    if (frags->nfrag > 0 && (!pix || !frags->depth || !frags->alpha || !frags->trans)) return WOIT_EINVAL;
    if (frags->npix == 0) return WOIT_OK;
    if (!ws || ws_bytes < build_atomic_workspace(frags->npix)) return WOIT_EWORKSPACE;
    return cuda_status(build_atomic(pix, *frags, params->rank, params->flags, bufs->near, bufs->far, bufs->coeffs, ws,
                                    static_cast<cudaStream_t>(stream)));
}

size_t woit_blur_workspace_bytes(int32_t width, int32_t height) {
    return width < 1 || height < 1 ? 0 : blur_workspace(width, height);
}

int woit_resolve_blur(const float* image, int32_t width, int32_t height, int32_t radius, float* out, void* ws,
                      size_t ws_bytes, void* stream) {
    if (!image || !out || width < 1 || height < 1) return WOIT_EINVAL;
    if (radius < 1 || radius > kMaxDiffusionRadius) return WOIT_EINVAL;
    if (!ws || ws_bytes < blur_workspace(width, height)) return WOIT_EWORKSPACE;
    return cuda_status(resolve_blur(image, width, height, radius, out, ws, static_cast<cudaStream_t>(stream)));
}

size_t woit_build_into_workspace_bytes(int64_t n, int64_t npix) { return build_into_workspace(n, npix); }

int woit_build_into(double* coeffs, int64_t npix, const int64_t* pix, const double* z, const double* a,
                    int64_t n, int rank, int mode, void* ws, size_t ws_bytes, void* stream) {
    if (rank < 0 || rank > kMaxRank) return WOIT_ERANK;
    if (n < 0 || npix < 0 || (n > 0 && (!coeffs || !pix || !z || !a))) return WOIT_EINVAL;
    if (mode != WOIT_BUILD_BINNED && mode != WOIT_BUILD_ATOMIC) return WOIT_EINVAL;
    if (mode == WOIT_BUILD_BINNED && n > 0 && (!ws || ws_bytes < build_into_workspace(n, npix)))
        return WOIT_EWORKSPACE;
    return cuda_status(build_into(coeffs, npix, pix, z, a, n, rank, mode, ws, ws_bytes,
                                  static_cast<cudaStream_t>(stream)));
}

int woit_interp_absorbance(const double* coeffs, int64_t npix, const int64_t* pix, const double* z, int64_t n,
                           int rank, double* out, void* stream) {
    if (rank < 0 || rank > kMaxRank) return WOIT_ERANK;
    if (n < 0 || npix < 0 || (n > 0 && (!coeffs || !pix || !z || !out))) return WOIT_EINVAL;
    return cuda_status(interp(coeffs, pix, z, n, rank, out, static_cast<cudaStream_t>(stream)));
}

int woit_cells_raw(const double* coeffs, int64_t npix, const int64_t* pix, const int64_t* cells, int64_t n,
                   int rank, double* out, void* stream) {
    if (rank < 0 || rank > kMaxRank) return WOIT_ERANK;
    if (n < 0 || npix < 0 || (n > 0 && (!coeffs || !pix || !cells || !out))) return WOIT_EINVAL;
    return cuda_status(cells_raw(coeffs, pix, cells, n, rank, out, static_cast<cudaStream_t>(stream)));
}

int woit_total_absorbance(const double* coeffs, int64_t npix, int rank, double* out, void* stream) {
    if (rank < 0 || rank > kMaxRank) return WOIT_ERANK;
    if (npix < 0 || (npix > 0 && (!coeffs || !out))) return WOIT_EINVAL;
    return cuda_status(total(coeffs, npix, rank, out, static_cast<cudaStream_t>(stream)));
}

size_t woit_bin_workspace_bytes(int64_t n, int64_t npix) { return bin_workspace(n, npix); }

int woit_bin_by_pixel(const int64_t* pix, int64_t n, int64_t npix, int64_t* offsets, int64_t* perm, void* ws,
                      size_t ws_bytes, void* stream) {
    if (n < 0 || npix < 0 || !offsets || (n > 0 && (!pix || !perm))) return WOIT_EINVAL;
    if (n >= ((int64_t)1 << 31) || npix >= ((int64_t)1 << 31)) return WOIT_EINVAL;
    if (n > 0 && (!ws || ws_bytes < bin_workspace(n, npix))) return WOIT_EWORKSPACE;
    return cuda_status(bin_by_pixel(pix, n, npix, offsets, perm, ws, ws_bytes, static_cast<cudaStream_t>(stream)));
}

size_t woit_bin_frame_workspace_bytes(int64_t n, int64_t npix) { return n < 0 || npix < 0 ? 0 : bin_workspace(n, npix); }

int woit_bin_frame(const int32_t* pix, const woit_frags_t* unbinned, woit_frags_t* binned, int64_t* offsets,
                   int64_t* perm, void* ws, size_t ws_bytes, void* stream) {
    if (!unbinned || !binned || !offsets) return WOIT_EINVAL;
    const int64_t n = unbinned->nfrag, npix = unbinned->npix;
    if (n < 0 || npix < 1 || n >= ((int64_t)1 << 31) || npix >= ((int64_t)1 << 31)) return WOIT_EINVAL;
    if (n > 0 && (!pix || !unbinned->depth || !binned->depth)) return WOIT_EINVAL;
    // every optional field travels iff both sides have it
    const void* pairs[][2] = {{unbinned->alpha, binned->alpha}, {unbinned->trans, binned->trans},
                              {unbinned->radiance, binned->radiance}, {unbinned->normal, binned->normal},
                              {unbinned->ior, binned->ior}, {unbinned->backface, binned->backface}};
    for (auto& pr : pairs)
        if ((pr[0] == nullptr) != (pr[1] == nullptr)) return WOIT_EINVAL;
    if (n > 0 && (!ws || ws_bytes < bin_workspace(n, npix))) return WOIT_EWORKSPACE;
    return cuda_status(bin_frame(pix, n, npix, *unbinned, *binned, offsets, perm, ws, static_cast<cudaStream_t>(stream)));
}

int woit_pack_rgb9e5(const double* v, int64_t n, uint32_t* words, void* stream) {
    if (n < 0 || (n > 0 && (!v || !words))) return WOIT_EINVAL;
    return cuda_status(pack(v, n, words, static_cast<cudaStream_t>(stream)));
}

int woit_unpack_rgb9e5(const uint32_t* words, int64_t n, double* out, void* stream) {
    if (n < 0 || (n > 0 && (!words || !out))) return WOIT_EINVAL;
    return cuda_status(unpack(words, n, out, static_cast<cudaStream_t>(stream)));
}

size_t woit_synth_workspace_bytes(int64_t npix) { return synth::workspace(npix); }

int woit_synth_offsets(int workload, int32_t width, int32_t height, uint32_t seed, int32_t layers, int32_t row0,
                       int32_t rows, int64_t* offsets, void* ws, size_t ws_bytes, void* stream) {
    if (workload < 0 || workload > WOIT_SYNTH_RAGGED || width < 1 || height < 1 || layers < 1 || row0 < 0 ||
        rows < 0 || row0 + rows > height || !offsets)
        return WOIT_EINVAL;
    if (!ws || ws_bytes < synth::workspace((int64_t)rows * width)) return WOIT_EWORKSPACE;
    return cuda_status(synth::offsets(workload, width, seed, layers, row0, rows, offsets, ws, ws_bytes,
                                      static_cast<cudaStream_t>(stream)));
}

int woit_synth_fill(int workload, int32_t width, int32_t height, uint32_t seed, int32_t layers, int32_t row0,
                    int32_t rows, const int64_t* offsets, float* depth, float* alpha, float* trans, float* radiance,
                    float* normal, float* ior, uint8_t* backface, float* opaque_depth, float* opaque_color,
                    void* stream) {
    if (workload < 0 || workload > WOIT_SYNTH_RAGGED || width < 1 || height < 1 || layers < 1 || row0 < 0 ||
        rows < 0 || row0 + rows > height || !offsets || !depth || !alpha || !trans || !radiance || !normal ||
        !ior || !backface || !opaque_depth || !opaque_color)
        return WOIT_EINVAL;
    synth::Out o{depth, alpha, trans, radiance, normal, ior, backface};
    return cuda_status(synth::fill(workload, width, seed, layers, row0, rows, offsets, 0, o, opaque_depth,
                                   opaque_color, static_cast<cudaStream_t>(stream)));
}

}  // extern "C"
