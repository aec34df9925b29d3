// Internal (C++) entry points shared between the .cu translation units.
#pragma once

#include "common.cuh"

namespace woit {
struct KParams;
cudaError_t launch_frame(const KParams& kp, cudaStream_t st);
cudaError_t launch_composite(const KParams& kp, cudaStream_t st);
cudaError_t launch_indices(const KParams& kp, double* z, int32_t* k, int32_t* cells, cudaStream_t st);
size_t bin_workspace(int64_t n, int64_t npix);
cudaError_t bin_by_pixel(const int64_t* pix, int64_t n, int64_t npix, int64_t* offsets, int64_t* perm,
                         void* ws, size_t ws_bytes, cudaStream_t st);
cudaError_t bin_frame(const int32_t* pix, int64_t n, int64_t npix, const woit_frags_t& in, const woit_frags_t& out,
                      int64_t* offsets, int64_t* perm, void* ws, cudaStream_t st);
size_t build_into_workspace(int64_t n, int64_t npix);
cudaError_t build_into(double* coeffs, int64_t npix, const int64_t* pix, const double* z, const double* a,
                       int64_t n, int rank, int mode, void* ws, size_t ws_bytes, cudaStream_t st);
cudaError_t interp(const double* coeffs, const int64_t* pix, const double* z, int64_t n, int rank,
                   double* out, cudaStream_t st);
cudaError_t cells_raw(const double* coeffs, const int64_t* pix, const int64_t* cells, int64_t n, int rank,
                      double* out, cudaStream_t st);
cudaError_t total(const double* coeffs, int64_t npix, int rank, double* out, cudaStream_t st);
cudaError_t pack(const double* v, int64_t n, uint32_t* words, cudaStream_t st);
cudaError_t unpack(const uint32_t* words, int64_t n, double* out, cudaStream_t st);
size_t blur_workspace(int32_t width, int32_t height);
size_t build_atomic_workspace(int64_t npix);
size_t baseline_workspace(int method, int64_t npix, int64_t nfrag);
size_t cast_workspace(int64_t npix);
cudaError_t cast_count(const woit_scene_t& s, int W, int H, int64_t* offsets, void* ws, cudaStream_t st);
cudaError_t cast_fill(const woit_scene_t& s, int W, int H, const int64_t* offsets, float* depth, float* alpha,
                      float* trans, float* rad, float* normal, float* ior, uint8_t* bf, float* od, float* oc,
                      cudaStream_t st);
cudaError_t render_baseline(const woit_frags_t& f, int method, bool cube, const double wboit[3], float* out,
                            void* ws, cudaStream_t st);
cudaError_t build_atomic(const int32_t* pix, const woit_frags_t& f, int rank, int flags, const float* near,
                         const float* far, float* coeffs, void* ws, cudaStream_t st);
cudaError_t resolve_blur(const float* image, int32_t W, int32_t H, int32_t r, float* out, void* ws,
                         cudaStream_t st);
// kernel launch geometry (frame.cu): sets the smem opt-in attribute as needed and
// returns the SM count and resident blocks per SM, cached per (kernel, device, bytes)
cudaError_t launch_config(const void* fn, int threads, int bytes, int& sms, int& per_sm);
namespace synth {
struct Out {
    float *depth, *alpha, *trans, *rad, *normal, *ior;
    uint8_t* bf;
};
size_t workspace(int64_t npix);
cudaError_t offsets(int workload, int32_t width, uint32_t seed, int32_t layers, int32_t row0, int32_t rows,
                    int64_t* off, void* ws, size_t ws_bytes, cudaStream_t st);
cudaError_t fill(int workload, int32_t width, uint32_t seed, int32_t layers, int32_t row0, int32_t rows,
                 const int64_t* off, int64_t nfrag_uniform, Out o, float* od, float* oc, cudaStream_t st);
}  // namespace synth
}  // namespace woit

