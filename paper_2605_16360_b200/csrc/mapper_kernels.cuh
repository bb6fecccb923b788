#pragma once
#include <cuda_fp16.h>

#include "internal.h"

namespace pkv {

// Where the windows of a batch of "units" (one unit = one [H_s, N] proxy score
// slab, i.e. one (batch, proxy layer)) live in the caller's input.
// FP16F8 correction planes (gemm.cuh): written instead of the fp16 lo plane
// when lo8 is set: lo8 = e4m3((v − hi)·lo_mul), hi8 = e4m3(hi·hi_mul).
struct F8Out {
    uint8_t* lo8 = nullptr;
    uint8_t* hi8 = nullptr;
    float lo_mul = 1.0f, hi_mul = 1.0f;
};

struct MapperSrc {
    const float* x = nullptr;
    const int64_t* unit_off = nullptr;  // device [units]: element offset of (head 0, token 0)
    const int64_t* win_off = nullptr;   // device [W]: token offset of each window
    int64_t head_stride = 0;            // elements between heads (= N)
    int units = 0, W = 0, Lw = 0, hs = 0;
};

void launch_window_mean(const MapperSrc& s, float* mean_out, cudaStream_t st);
// rinv [rows]: inverse power-of-two scale of each panel row (GemmEpiParams::row_scale)
void launch_conv1_im2col(const MapperSrc& s, const float* mean, const float* w1, const float* b1, int mid,
                         __half* col_h, __half* col_l, float* rinv, cudaStream_t st, F8Out f8 = {});
void launch_split_rows_scaled(const float* z, int64_t rows, int D, __half* hi, __half* lo, float* rinv,
                              cudaStream_t st);
void launch_bypass_stem(const MapperSrc& s, const float* mean, const float* w, const float* b, const float* pe, int D,
                        float* z, cudaStream_t st);
void launch_layernorm(const float* z, int64_t rows, int D, const float* g, const float* b, __half* hi, __half* lo,
                      cudaStream_t st, F8Out f8 = {});
void launch_window_colmean_add(float* z, int64_t nwin, int Lw, int D, cudaStream_t st);
void launch_stage3(const float* s3, int64_t rows, int ld, int hl, int syn, bool cross_active, float out_b, int Lw,
                   float* logitsT, float* attn, cudaStream_t st);
void launch_window_average(const float* logitsT, const int* out_unit, int n_out, int hl, int W, int Lw, int stride,
                           int n_regular, int tail_off, int64_t N, float* y, cudaStream_t st);

}  // namespace pkv
