/*
 * woit.h — C ABI of the B200-native wavelet OIT hot path (libwoit.so).
 *
 * The reference (`woit`, pure Python/numpy) has no FFI; its boundary for this
 * path is a set of Python functions over numpy arrays. Each entry point below
 * replaces one of them; the Python shim `paper_2201_00094_b200` binds them with
 * ctypes exactly as INTEGRATION.md shows.
 *
 * Conventions
 *  - every pointer argument is a DEVICE pointer unless stated otherwise;
 *  - `stream` is a cudaStream_t (passed as void* so this header needs no CUDA
 *    headers); 0 is the legacy default stream;
 *  - the library never allocates or frees memory and keeps no global mutable
 *    state: scratch is passed in as `ws`/`ws_bytes`, sized by the matching
 *    *_workspace_bytes() query;
 *  - calls are asynchronous and stream-ordered; the return value reports
 *    argument validation and launch errors only (negative = error).
 *  - results are deterministic: per-pixel reductions run in an order fixed by
 *    the global pixel id (pixel_base + band-local id), the pixel's run length
 *    and the fragment's position in its run, so any row-band split yields
 *    bit-identical outputs as long as every band carries its pixel_base;
 *  - a workspace `ws` carries per-launch state (the frame kernels' window-claim
 *    counter, window claim order and long-pixel list, reset by each call):
 *    launches that may run concurrently (different streams or host threads) must
 *    not share one.
 *
 * Data layout (SoA, CSR by pixel — the reference's FrameFragments contract,
 * scene.py:367-392, in fp32 instead of f64):
 *   offsets  int64 [npix+1]          fragments of pixel p are [offsets[p], offsets[p+1])
 *   depth, alpha, ior   float [n]
 *   trans, radiance, normal float [n][3]
 *   backface uint8 [n]
 *   opaque_depth float [npix] (+inf = no opaque hit), opaque_color float [npix][3]
 * Per-pixel buffers (FrameBuffers, pipeline.py:76-104):
 *   near, far float [npix]; coeffs float [npix][S][3] with S = 2^(rank+1)
 *   (slot 0 = scaling coefficient, slot 2^n+k = level n offset k,
 *   wavelet.py:3-9); accum, weight, output float [npix][3];
 *   refraction_offset float [npix][2]; vhat float [n][3].
 */
#ifndef WOIT_H
#define WOIT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WOIT_ABI_VERSION 3

/* status codes */
#define WOIT_OK 0
#define WOIT_EINVAL (-1)      /* bad argument (null pointer, size, rank, flags) */
#define WOIT_EWORKSPACE (-2)  /* ws_bytes smaller than the *_workspace_bytes query */
#define WOIT_ECUDA (-3)       /* a CUDA launch / API call failed */
#define WOIT_ERANK (-4)       /* rank outside [0, 6] (pipeline.py:66-67) */
#define WOIT_ETAPS (-5)       /* aberration taps even or < 3 (pipeline.py:68-69) */

/* RenderConfig booleans (pipeline.py:45-61) */
#define WOIT_REFRACTION 0x01
#define WOIT_CHROMATIC_ABERRATION 0x02
#define WOIT_CUBE_TRANSMISSION 0x04
#define WOIT_NORMALIZE 0x08
#define WOIT_PACKED_STORAGE 0x10
#define WOIT_LITERAL_SPECTRAL_T 0x20
#define WOIT_CUBE_BACKFACE_ONLY 0x40
/* Diffusion ("resolve and blur", BASELINE north star (3)-(4)). The reference has no
 * such pass, so this is the IN-REPO definition, parity unpinned:
 *   step3 also accumulates the pixel's visibility-weighted coverage
 *       D_p = sum_f alpha_f * (vhat_f.r + vhat_f.g + vhat_f.b) / 3      (bufs->diffusion)
 *   K_resolve blurs the background image with a separable, edge-clamped Gaussian of
 *       `diffusion_radius` taps each side, sigma = radius / 2 (woit_resolve_blur);
 *   step4 replaces the background bg by bg + w (bg_blurred - bg), w = min(1, diffusion * D_p),
 *       bg_blurred sampled from the blurred image exactly as bg is from the sharp one.
 * Off by default; with the flag clear every output is bit-identical to a build
 * without this feature. */
#define WOIT_DIFFUSION 0x80

typedef struct woit_frags {
    int32_t width;        /* full frame width  (RenderConfig.width)  */
    int32_t height;       /* full frame height (RenderConfig.height) */
    int64_t npix;         /* pixels in this band = len(offsets) - 1   */
    int64_t nfrag;        /* element count of the fragment arrays (>= offsets[npix]) */
    int64_t pixel_base;   /* global id of the band's first pixel (pipeline.py:321-330) */
    int64_t frag_base;    /* informational only (global id of fragment 0 of the band); the
                             kernels do not read it: outputs depend on pixel_base alone */
    const int64_t* offsets;
    const float* depth;
    const float* alpha;
    const float* trans;
    const float* radiance;
    const float* normal;        /* may be NULL unless WOIT_REFRACTION */
    const float* ior;           /* may be NULL: all 1.0 */
    const uint8_t* backface;    /* may be NULL: all false */
    const float* opaque_depth;  /* may be NULL: all +inf */
    const float* opaque_color;  /* band-local [npix][3] */
} woit_frags_t;

typedef struct woit_params {
    int32_t rank;            /* N, 0..6 */
    int32_t flags;           /* WOIT_* booleans */
    int32_t aberration_taps; /* odd, >= 3 */
    int32_t diffusion_radius; /* WOIT_DIFFUSION: blur taps each side, 1..64 */
    double refraction_scale; /* pixels per world unit at width 512 */
    double cam_forward[3];   /* Camera.basis() (scene.py:141-150) */
    double cam_right[3];
    double cam_up[3];
    double tan_half;         /* tan(fov/2) (scene.py:201) */
    double aspect;           /* width / height */
    double diffusion;        /* WOIT_DIFFUSION: strength (>= 0), w = min(1, diffusion * D_p) */
} woit_params_t;

typedef struct woit_bufs {
    float* near;               /* NULL: not written */
    float* far;
    float* coeffs;
    float* accum;
    float* weight;
    float* refraction_offset;
    float* output;
    float* vhat;               /* per-fragment transmittance; NULL: not written */
    const float* full_opaque_image; /* [height][width][3] for refraction / aberration gathers;
                                       NULL: the band's opaque_color with pixel_base 0 */
    float* diffusion;          /* [npix] coverage D_p (WOIT_DIFFUSION); NULL: not written */
    const float* blurred_image; /* WOIT_DIFFUSION: woit_resolve_blur of the background image,
                                   same extent/indexing as the image bg is read from */
    uint32_t* coeff_words;     /* WOIT_PACKED_STORAGE: [npix][S] E5B9G9R9 words (packing.py:46-77),
                                  word s = pack(|coefficients of slot s|), the paper's 4 S B/px
                                  storage; NULL: not written (ABI 3) */
} woit_bufs_t;

/* ---- version / errors ---------------------------------------------------- */
int woit_abi_version(void);
const char* woit_status_string(int status);

/* ---- frame path (pipeline.py) -------------------------------------------- */

/* Scratch for the frame and step entry points: counters, the long-pixel list and
 * the claim order of the 32-pixel windows (sparse frames in the general kernel). */
size_t woit_frame_workspace_bytes(int64_t npix, int64_t nfrag);

/* All four passes fused over one row band, fragments read from HBM once.
 * Replaces pipeline._wavelet_band (pipeline.py:321-330) on freshly allocated
 * FrameBuffers: every non-NULL buffer in `bufs` is overwritten. */
int woit_render_band(const woit_frags_t* frags, const woit_params_t* params, woit_bufs_t* bufs,
                     void* ws, size_t ws_bytes, void* stream);

/* step1_depth_bounds (pipeline.py:131-134): near = min(near, depth), far = max(far, depth). */
int woit_step1_depth_bounds(const woit_frags_t* frags, woit_bufs_t* bufs, void* ws,
                            size_t ws_bytes, void* stream);

/* step2_build (pipeline.py:148-155): coeffs += closed-form Haar projection of every
 * fragment's absorbance step, using bufs->near/far; packed storage if flagged. */
int woit_step2_build(const woit_frags_t* frags, const woit_params_t* params, woit_bufs_t* bufs,
                     void* ws, size_t ws_bytes, void* stream);

/* step3_accumulate (pipeline.py:170-217): accum/weight/refraction_offset += ... from
 * bufs->coeffs, near, far; writes vhat if non-NULL. */
int woit_step3_accumulate(const woit_frags_t* frags, const woit_params_t* params,
                          woit_bufs_t* bufs, void* ws, size_t ws_bytes, void* stream);

/* step4_composite (pipeline.py:284-308): output from coeffs, accum, weight,
 * refraction_offset and the background. Only width/height/npix/pixel_base and
 * opaque_color of `frags` are read. */
int woit_step4_composite(const woit_frags_t* frags, const woit_params_t* params,
                         woit_bufs_t* bufs, void* stream);

/* The north star's alternative build, kept for the measured comparison (DESIGN.md
 * §3.6): step2_build on an UNBINNED stream with explicit pixel ids pix[nfrag]
 * (frags->offsets unused), one thread per fragment scattering the closed-form
 * projection (wavelet.py:272-287) with fp32 red.global.add into coeffs (which the
 * caller zeroes). Not bit-reproducible (atomic order); no packed storage. */
size_t woit_build_atomic_workspace_bytes(int64_t npix);
int woit_build_atomic(const woit_frags_t* frags, const int32_t* pix, const woit_params_t* params,
                      woit_bufs_t* bufs, void* ws, size_t ws_bytes, void* stream);

/* Per-fragment normalised depth z (double[n]), level slot offsets k_n
 * (int32[n][rank+1], wavelet.py:281) and interpolation cells c0, c1
 * (int32[n][2], wavelet.py:309-315), computed by the same device functions the
 * frame kernels use, from bufs near/far. For bit-exact index parity checks. */
int woit_fragment_indices(const woit_frags_t* frags, const float* near, const float* far, int rank,
                          double* z, int32_t* slots, int32_t* cells, void* stream);

/* ---- on-device fragment producer (scene.py:430-630 cast_frame) ---------------
 * Casts every pixel's primary ray against an analytic scene and writes the CSR
 * stream (fp32, the layout above) in cast_frame's row order: per pixel, primitives
 * in scene order, sub-index order inside a primitive (sphere entry then exit, fog
 * slices front to back, particles by index). Geometry in float64. */
#define WOIT_PRIM_PLANE 0
#define WOIT_PRIM_SPHERE 1
#define WOIT_PRIM_FOG 2
#define WOIT_PRIM_PARTICLES 3
#define WOIT_PRIM_BACKDROP 4

typedef struct woit_prim {
    int32_t kind;           /* WOIT_PRIM_* */
    int32_t count;          /* fog: slices; particles: particle count */
    int32_t profile;        /* particles: 0 gauss, 1 mask */
    int32_t flags;          /* bit 0: plane has an extent (pane); bit 1: backdrop checker */
    double d;               /* plane / backdrop forward distance */
    double center[3];       /* sphere / particle-cloud centre */
    double radius;          /* sphere radius */
    double particle_radius; /* particle disc radius */
    double extent[2];       /* pane half extents */
    double pcenter[2];      /* pane centre (right, up) */
    double alpha, ior;      /* material */
    double trans[3], radiance[3];
    double sigma[3];        /* fog extinction */
    double color[3];        /* fog in-scatter colour; backdrop colour */
    double checker[3];      /* backdrop checker colour */
    double near, far;       /* fog slab */
    double cell;            /* backdrop checker cell (world units) */
    const double* positions;      /* particles: device [count][3] */
    const double* radiance_scale; /* particles: device [count] */
    const int32_t* box;           /* particles: device [count][4] screen box x0, x1, y0, y1
                                     (cast_frame's conservative bound; x0 > x1 = culled) */
} woit_prim_t;

typedef struct woit_scene {
    int32_t nprims;
    int32_t bg_cell;          /* background checker cell in pixels */
    int32_t bg_has_checker;
    int32_t reserved;
    const woit_prim_t* prims; /* DEVICE array [nprims] */
    double origin[3], forward[3], right[3], up[3];  /* Camera.basis() */
    double tan_half, aspect;
    double bg_color[3], bg_checker[3];
} woit_scene_t;

size_t woit_cast_workspace_bytes(int64_t npix);
/* offsets[W*H+1] of the frame's CSR stream (pass 1). */
int woit_cast_offsets(const woit_scene_t* scene, int32_t width, int32_t height, int64_t* offsets, void* ws,
                      size_t ws_bytes, void* stream);
/* the fragment arrays (sized by offsets[W*H]) and the opaque depth / colour (pass 2). */
int woit_cast_fill(const woit_scene_t* scene, int32_t width, int32_t height, const int64_t* offsets,
                   float* depth, float* alpha, float* trans, float* radiance, float* normal, float* ior,
                   uint8_t* backface, float* opaque_depth, float* opaque_color, void* stream);

/* ---- comparison methods (RenderConfig.method, baselines.py:135-220) ---------
 * The reference's non-wavelet methods over the same CSR stream, in float64 with the
 * reference's operation order (one thread per pixel), output fp32 [npix][3] over the
 * opaque colour. WOIT_METHOD_ABUFFER is the exact sorted oracle (stable per-pixel sort
 * by depth, then front to back); WBOIT uses wboit_weight = (gain, clamp lo, clamp hi);
 * MLAB4 is the 4-node streaming blend. flags: WOIT_CUBE_TRANSMISSION only.
 * wboit_weight is a HOST pointer to 3 doubles (read during the call).
 * ABUFFER needs nfrag < 2^31 (segmented sort). */
#define WOIT_METHOD_ABUFFER 1
#define WOIT_METHOD_WBOIT 2
#define WOIT_METHOD_MLAB4 3

size_t woit_baseline_workspace_bytes(int method, int64_t npix, int64_t nfrag);
int woit_render_baseline(const woit_frags_t* frags, int method, int flags, const double* wboit_weight,
                         float* output, void* ws, size_t ws_bytes, void* stream);

/* ---- K_resolve: the diffusion blur (in-repo definition, see WOIT_DIFFUSION) ----- */

size_t woit_blur_workspace_bytes(int32_t width, int32_t height);

/* out = separable Gaussian blur of image (float [height][width][3]), edge clamped,
 * taps -radius..radius with weights exp(-i^2 / (2 sigma^2)) / sum, sigma = radius / 2:
 * a horizontal then a vertical pass, both with 128-bit coalesced loads/stores. */
int woit_resolve_blur(const float* image, int32_t width, int32_t height, int32_t radius,
                      float* out, void* ws, size_t ws_bytes, void* stream);

/* ---- batch kernels (wavelet.py:272-337) ------------------------------------
 * Same dtypes as the reference (float64 throughout). With WOIT_BUILD_BINNED the
 * per-slot additions happen in fragment order in f64 with no FMA contraction,
 * i.e. in exactly the order np.add.at performs them, so results are
 * bit-identical to the reference's. coeffs is double[npix][2^(rank+1)][3]. */

#define WOIT_BUILD_BINNED 0   /* stable sort by pixel, per-pixel ordered f64 sums */
#define WOIT_BUILD_ATOMIC 1   /* red.global.add.f64 straight into coeffs (unordered) */

size_t woit_build_into_workspace_bytes(int64_t n, int64_t npix);

/* build_into (wavelet.py:272-287): coeffs[pix[i]] += projection of (z[i], a[i]) for
 * arbitrary (unbinned) pixel ids. z: double[n], a: double[n][3]. */
int woit_build_into(double* coeffs, int64_t npix, const int64_t* pix, const double* z,
                    const double* a, int64_t n, int rank, int mode, void* ws, size_t ws_bytes,
                    void* stream);

/* interp_absorbance_batch (wavelet.py:306-319) -> out double[n][3] */
int woit_interp_absorbance(const double* coeffs, int64_t npix, const int64_t* pix,
                           const double* z, int64_t n, int rank, double* out, void* stream);

/* cells_raw_batch (wavelet.py:290-303) -> out double[n][3] */
int woit_cells_raw(const double* coeffs, int64_t npix, const int64_t* pix, const int64_t* cells,
                   int64_t n, int rank, double* out, void* stream);

/* total_absorbance_batch (wavelet.py:322-337) -> out double[npix][3] */
int woit_total_absorbance(const double* coeffs, int64_t npix, int rank, double* out,
                          void* stream);

/* ---- fragment binning (scene.py:559-566 contract) ------------------------ */

size_t woit_bin_workspace_bytes(int64_t n, int64_t npix);

/* Stable sort of fragment ids by pixel (an LSD radix sort: one stable counting sort --
 * digit histogram per tile, scan, stable scatter -- per 8 bits of the pixel id, over
 * ceil(log2 npix) bits): offsets[npix+1] equals concatenate([0], cumsum(bincount(pix,
 * minlength=npix))) and perm lists the fragment ids of each pixel in their original
 * order (np.argsort(pix, kind="stable")). pix in [0, npix); n, npix < 2^31. */
int woit_bin_by_pixel(const int64_t* pix, int64_t n, int64_t npix, int64_t* offsets,
                      int64_t* perm, void* ws, size_t ws_bytes, void* stream);

/* An unbinned stream -> the CSR stream the frame kernels take (scene.py:559-566): the
 * same stable sort, then every fragment's fields (depth, alpha, trans, radiance,
 * normal, ior, backface -- each present on both sides or neither) move from its
 * arrival slot into its CSR slot, 32 pixels at a time (reads coalesce when the
 * arrival is layer by layer). unbinned->nfrag / npix
 * give the sizes (unbinned->offsets unused); binned's field pointers are the outputs
 * (its const qualifiers notwithstanding); offsets int64[npix+1]; perm int64[n] or NULL. */
size_t woit_bin_frame_workspace_bytes(int64_t n, int64_t npix);
int woit_bin_frame(const int32_t* pix, const woit_frags_t* unbinned, woit_frags_t* binned, int64_t* offsets,
                   int64_t* perm, void* ws, size_t ws_bytes, void* stream);

/* ---- E5B9G9R9 packing (packing.py:46-111) --------------------------------- */

/* words[i] = pack(|v[i][0..2]|) ; v is double[n][3] */
int woit_pack_rgb9e5(const double* v, int64_t n, uint32_t* words, void* stream);
/* out[i][0..2] = unpack(words[i]) */
int woit_unpack_rgb9e5(const uint32_t* words, int64_t n, double* out, void* stream);

/* ---- synthetic streams (paper_2201_00094_b200/synth.py twin) ------------- */

#define WOIT_SYNTH_PLANE4 0
#define WOIT_SYNTH_SMOKE 1
#define WOIT_SYNTH_PARTICLES 2
#define WOIT_SYNTH_RAGGED 3

size_t woit_synth_workspace_bytes(int64_t npix);

/* CSR offsets[rows*width+1] of band [row0, row0+rows): per-pixel run lengths and
 * their scan (offsets[0] = 0). */
int woit_synth_offsets(int workload, int32_t width, int32_t height, uint32_t seed, int32_t layers,
                       int32_t row0, int32_t rows, int64_t* offsets, void* ws, size_t ws_bytes,
                       void* stream);

/* Fill the fragment arrays of the band from its offsets (all arrays non-NULL). */
int woit_synth_fill(int workload, int32_t width, int32_t height, uint32_t seed, int32_t layers,
                    int32_t row0, int32_t rows, const int64_t* offsets, float* depth,
                    float* alpha, float* trans, float* radiance, float* normal, float* ior,
                    uint8_t* backface, float* opaque_depth, float* opaque_color, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* WOIT_H */
