// mapper_kernels.cu — the HybridAxialMapper's non-GEMM kernels
// (proj/src/mapper.cpp:274-377 over proj/src/ops.cpp):
//   window_mean_kernel  normalize_input per-window mean (mapper.cpp:288-292)
//   conv1_im2col_kernel Stage 1a: Conv1D(H_s->mid,k3,pad1)+BN(eval)+GELU along
//                       the token axis, shared-memory staged, writing the
//                       im2col panel of Stage 1b (conv2 runs as a tcgen05 GEMM)
//   bypass_stem_kernel  stage_conv = bypass: 1x1 projection (mapper.cpp:302)
//   layernorm_kernel    pre-norm LN (ops.cpp:721-754) -> fp16 hi/lo planes
//   split_rows_scaled   Stage-3 input: residual stream -> row-scaled fp16 hi/lo
//   window_colmean_add  stage_encoder = bypass: z += mean_N z (mapper.cpp:318)
//   stage3_kernel       Stage 3 on the folded projection: per token, H_l
//                       softmaxes over the synthetic heads and the value·out_w
//                       dot (mapper.cpp:321-341)
//   window_average_kernel sliding_forward's overlap average (mapper.cpp:356-375)
#include <cuda_fp8.h>

#include "mapper_kernels.cuh"
#include "sm100.cuh"

namespace pkv {
namespace {

__device__ __forceinline__ uint32_t e4m3x2(float a, float b) {
    return (uint32_t)__nv_cvt_float2_to_fp8x2(make_float2(a, b), __NV_SATFINITE, __NV_E4M3);
}

// Power of two s with max_abs·s in [2^13, 2^14) (1 for an all-zero row); the
// GEMM epilogue multiplies by 1/s (GemmEpiParams::row_scale). Exact: scaling by
// 2^e only moves the exponent, and 2^14 leaves fp16 headroom for the hi plane's
// round-up.
__device__ __forceinline__ float row_pow2_scale(float max_abs) {
    if (!(max_abs > 0.0f)) return 1.0f;
    int e;
    frexpf(max_abs, &e);  // max_abs = m·2^e, m in [0.5, 1)
    int sh = 14 - e;
    sh = sh > 100 ? 100 : (sh < -100 ? -100 : sh);
    return __int_as_float((127 + sh) << 23);
}

// Source pointer of (unit, window): x + unit_off[unit] + off_w, rows of H_s
// with token stride tok_stride (= N) and head stride head_stride.
struct WinSrc {
    const float* x;
    const int64_t* unit_off;  // [units] element offset of x for the unit (head 0, token 0)
    const int64_t* win_off;   // [W] token offset of each window
    int64_t head_stride;
    int W;
    int Lw;
    int hs;
};

__global__ void window_mean_kernel(WinSrc src, float* __restrict__ mean_out) {
    // one block per (unit, window, head)
    const int idx = blockIdx.x;
    const int h = idx % src.hs, uw = idx / src.hs;
    const int u = uw / src.W, w = uw % src.W;
    const float* row = src.x + src.unit_off[u] + h * src.head_stride + src.win_off[w];
    float s = 0.0f;
    for (int t = threadIdx.x; t < src.Lw; t += blockDim.x) s += row[t];
    __shared__ float red[32];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) mean_out[idx] = fmaxf(s / (float)src.Lw, 1e-12f);
    }
}

constexpr int kConvTok = 64;  // tokens per block (amortises the per-block weight staging)

// z1[c, t] = gelu(b1'[c] + Σ_ci Σ_tap W1'[c, ci, tap] · x_pad[ci, t + tap - 1]) (BN folded)
// im2col row t = [z1[t-1] | z1[t] | z1[t+1]] with zero padding at the window edges.
// Each panel row is stored pre-scaled by row_pow2_scale(max |row|) and the
// inverse goes to rinv[row]: sum-pooled X (up to g·N_q) drives z1 far past the
// fp16 maximum, max-pooled X (<= 1) leaves it tiny; both keep the hi/lo split's
// full 22-bit precision this way.
__global__ void conv1_im2col_kernel(WinSrc src, const float* __restrict__ inv_mean, const float* __restrict__ w1,
                                    const float* __restrict__ b1, int mid, __half* __restrict__ col_h,
                                    __half* __restrict__ col_l, float* __restrict__ rinv, F8Out f8) {
    extern __shared__ float sm[];
    const int hs = src.hs, kw = hs * 3, kws = kw + 1;
    float* sw = sm;                            // [mid][kws]
    float* sx = sw + mid * kws;                // [hs][kConvTok + 4]
    float* sz = sx + hs * (kConvTok + 4);      // [kConvTok + 2][mid]
    float* smax = sz + (kConvTok + 2) * mid;   // [kConvTok + 2] max |z1| per token
    float* sscale = smax + (kConvTok + 2);     // [kConvTok] per panel row
    const int uw = blockIdx.y;
    const int u = uw / src.W, w = uw % src.W;
    const int t0 = blockIdx.x * kConvTok;
    const int tid = threadIdx.x;
    for (int i = tid; i < mid * kw; i += blockDim.x) sw[(i / kw) * kws + (i % kw)] = w1[i];
    const float* xb = src.x + src.unit_off[u] + src.win_off[w];
    for (int i = tid; i < hs * (kConvTok + 4); i += blockDim.x) {
        const int ci = i / (kConvTok + 4), j = i % (kConvTok + 4);
        const int t = t0 - 2 + j;
        float v = (t >= 0 && t < src.Lw) ? xb[ci * src.head_stride + t] : 0.0f;
        if (inv_mean) v = v / inv_mean[(uw)*hs + ci];
        sx[i] = v;
    }
    __syncthreads();
    for (int c = tid; c < mid; c += blockDim.x) {
        const float* wr = sw + c * kws;
        const float bias = b1[c];
        for (int tt = 0; tt < kConvTok + 2; ++tt) {
            const int t = t0 - 1 + tt;
            float acc = bias;
            for (int ci = 0; ci < hs; ++ci) {
                const float* xr = sx + ci * (kConvTok + 4) + tt;  // x at t-1 .. t+1
                acc = fmaf(wr[ci * 3 + 0], xr[0], acc);
                acc = fmaf(wr[ci * 3 + 1], xr[1], acc);
                acc = fmaf(wr[ci * 3 + 2], xr[2], acc);
            }
            sz[tt * mid + c] = (t >= 0 && t < src.Lw) ? sm100::gelu_fast(acc) : 0.0f;
        }
    }
    __syncthreads();
    {  // per-token max |z1| (one warp per token), then the per-row scale
        const int warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
        for (int tt = warp; tt < kConvTok + 2; tt += nwarps) {
            float m = 0.0f;
            for (int c = lane; c < mid; c += 32) m = fmaxf(m, fabsf(sz[tt * mid + c]));
            for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) smax[tt] = m;
        }
    }
    __syncthreads();
    const int ntok = min(kConvTok, src.Lw - t0);
    for (int tt = tid; tt < ntok; tt += blockDim.x) {
        const float s = row_pow2_scale(fmaxf(fmaxf(smax[tt], smax[tt + 1]), smax[tt + 2]));
        sscale[tt] = s;
        rinv[(int64_t)uw * src.Lw + t0 + tt] = 1.0f / s;
    }
    __syncthreads();
    const int64_t K = 3 * (int64_t)mid;
    // 16-byte stores: 8 consecutive panel columns (never straddling a tap: mid % 8 == 0)
    const int chunks = (3 * mid) / 8;
    for (int i = tid; i < ntok * chunks; i += blockDim.x) {
        const int tt = i / chunks, col = (i % chunks) * 8;
        const int tap = col / mid, c = col % mid;
        const float* zr = sz + (tt + tap) * mid + c;
        const float s = sscale[tt];
        __align__(16) __half hi[8];
        __align__(16) __half lo[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const float v = zr[e] * s;
            hi[e] = __float2half_rn(v);
            lo[e] = __float2half_rn(v - __half2float(hi[e]));
        }
        const int64_t off = ((int64_t)uw * src.Lw + t0 + tt) * K + col;
        *reinterpret_cast<uint4*>(col_h + off) = *reinterpret_cast<const uint4*>(hi);
        if (f8.lo8) {  // lo[e] holds v − hi exactly enough (fp16 of the residual) for an e4m3 rounding
            uint32_t l8[2], h8[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int e = 4 * q;
                l8[q] = e4m3x2(__half2float(lo[e]) * f8.lo_mul, __half2float(lo[e + 1]) * f8.lo_mul) |
                        (e4m3x2(__half2float(lo[e + 2]) * f8.lo_mul, __half2float(lo[e + 3]) * f8.lo_mul) << 16);
                h8[q] = e4m3x2(__half2float(hi[e]) * f8.hi_mul, __half2float(hi[e + 1]) * f8.hi_mul) |
                        (e4m3x2(__half2float(hi[e + 2]) * f8.hi_mul, __half2float(hi[e + 3]) * f8.hi_mul) << 16);
            }
            *reinterpret_cast<uint2*>(f8.lo8 + off) = make_uint2(l8[0], l8[1]);
            *reinterpret_cast<uint2*>(f8.hi8 + off) = make_uint2(h8[0], h8[1]);
        } else if (col_l) {
            *reinterpret_cast<uint4*>(col_l + off) = *reinterpret_cast<const uint4*>(lo);
        }
    }
}

// z[row, d] = Σ_ci W[d, ci] x[ci, t] + b[d] (+ pe[t, d])
__global__ void bypass_stem_kernel(WinSrc src, const float* __restrict__ inv_mean, const float* __restrict__ w,
                                   const float* __restrict__ b, const float* __restrict__ pe, int D,
                                   float* __restrict__ z) {
    const int uw = blockIdx.y, t = blockIdx.x;
    const int u = uw / src.W, win = uw % src.W;
    const float* xb = src.x + src.unit_off[u] + src.win_off[win];
    const int64_t row = (int64_t)uw * src.Lw + t;
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
        float acc = b[d];
        for (int ci = 0; ci < src.hs; ++ci) {
            float v = xb[ci * src.head_stride + t];
            if (inv_mean) v = v / inv_mean[uw * src.hs + ci];
            acc = fmaf(w[d * src.hs + ci], v, acc);
        }
        if (pe) acc += pe[(int64_t)t * D + d];
        z[row * D + d] = acc;
    }
}

// One warp per row of D = 128·V floats.
template <int V>
__global__ void layernorm_kernel(const float* __restrict__ z, int64_t rows, const float* __restrict__ g,
                                 const float* __restrict__ b, __half* __restrict__ hi, __half* __restrict__ lo,
                                 F8Out f8) {
    constexpr int D = 128 * V;
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const float4* zr = reinterpret_cast<const float4*>(z + row * D);
    float4 v[V];
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < V; ++i) {
        v[i] = zr[lane + 32 * i];
        s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mu = s / (float)D;
    float q = 0.0f;
#pragma unroll
    for (int i = 0; i < V; ++i) {
        const float a = v[i].x - mu, bb = v[i].y - mu, c = v[i].z - mu, d = v[i].w - mu;
        q += (a * a + bb * bb) + (c * c + d * d);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    const float inv = rsqrtf(q / (float)D + 1e-5f);
#pragma unroll
    for (int i = 0; i < V; ++i) {
        const int c0 = 4 * (lane + 32 * i);
        const float x[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
        __align__(8) __half h4[4];
        __align__(8) __half l4[4];
        float r4[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const float y = g[c0 + t] * ((x[t] - mu) * inv) + b[c0 + t];
            h4[t] = __float2half_rn(y);
            r4[t] = y - __half2float(h4[t]);
            l4[t] = __float2half_rn(r4[t]);
        }
        *reinterpret_cast<uint2*>(hi + row * D + c0) = *reinterpret_cast<const uint2*>(h4);
        if (f8.lo8) {
            *reinterpret_cast<uint32_t*>(f8.lo8 + row * D + c0) =
                e4m3x2(r4[0] * f8.lo_mul, r4[1] * f8.lo_mul) | (e4m3x2(r4[2] * f8.lo_mul, r4[3] * f8.lo_mul) << 16);
            *reinterpret_cast<uint32_t*>(f8.hi8 + row * D + c0) =
                e4m3x2(__half2float(h4[0]) * f8.hi_mul, __half2float(h4[1]) * f8.hi_mul) |
                (e4m3x2(__half2float(h4[2]) * f8.hi_mul, __half2float(h4[3]) * f8.hi_mul) << 16);
        } else if (lo) {
            *reinterpret_cast<uint2*>(lo + row * D + c0) = *reinterpret_cast<const uint2*>(l4);
        }
    }
}

// Stage-3 A operand: the raw fp32 residual stream z (no final LN,
// mapper.cpp:316-324) split into fp16 hi/lo planes, one warp per row, each row
// pre-scaled by row_pow2_scale(max |row|) with the inverse in rinv[row].
__global__ void split_rows_scaled_kernel(const float* __restrict__ z, int64_t rows, int D, __half* __restrict__ hi,
                                         __half* __restrict__ lo, float* __restrict__ rinv) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const float* zr = z + row * D;
    float m = 0.0f;
    if ((D & 3) == 0) {
        for (int c = 4 * lane; c < D; c += 128) {
            const float4 v = *reinterpret_cast<const float4*>(zr + c);
            m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
        }
    } else {
        for (int c = lane; c < D; c += 32) m = fmaxf(m, fabsf(zr[c]));
    }
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const float s = row_pow2_scale(m);
    if (lane == 0) rinv[row] = 1.0f / s;
    if ((D & 3) == 0) {
        for (int c = 4 * lane; c < D; c += 128) {
            const float4 v = *reinterpret_cast<const float4*>(zr + c);
            const float x[4] = {v.x * s, v.y * s, v.z * s, v.w * s};
            __align__(8) __half h4[4];
            __align__(8) __half l4[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                h4[t] = __float2half_rn(x[t]);
                l4[t] = __float2half_rn(x[t] - __half2float(h4[t]));
            }
            *reinterpret_cast<uint2*>(hi + row * D + c) = *reinterpret_cast<const uint2*>(h4);
            if (lo) *reinterpret_cast<uint2*>(lo + row * D + c) = *reinterpret_cast<const uint2*>(l4);
        }
    } else {
        for (int c = lane; c < D; c += 32) {
            const float x = zr[c] * s;
            const __half h = __float2half_rn(x);
            hi[row * D + c] = h;
            if (lo) lo[row * D + c] = __float2half_rn(x - __half2float(h));
        }
    }
}

// stage_encoder = bypass: z[w, t, :] += mean_t z[w, :, :]
__global__ void window_colmean_add_kernel(float* __restrict__ z, int Lw, int D) {
    const int w = blockIdx.y;
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= D) return;
    float* base = z + (int64_t)w * Lw * D + d;
    float s = 0.0f;
    for (int t = 0; t < Lw; ++t) s += base[(int64_t)t * D];
    const float m = s / (float)Lw;
    for (int t = 0; t < Lw; ++t) base[(int64_t)t * D] += m;
}

// s3 row = [scores (H_l x syn, already q·k/√dh incl. bias) | v'_s (syn)].
// attn (nullable, StageTrace, mapper.hpp:111-114): [row, H_l, syn] softmax weights.
__global__ void stage3_kernel(const float* __restrict__ s3, int64_t rows, int ld, int hl, int syn, int cross_active,
                              float out_b, int Lw, float* __restrict__ logitsT, float* __restrict__ attn) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= rows) return;
    const float* r = s3 + row * ld;
    const float* vp = r + (cross_active ? hl * syn : 0);
    const int64_t uw = row / Lw, t = row % Lw;
    for (int h = 0; h < hl; ++h) {
        float logit;
        if (cross_active) {
            const float* sc = r + h * syn;
            float m = -INFINITY;
            for (int s = 0; s < syn; ++s) m = fmaxf(m, sc[s]);
            float z = 0.0f, acc = 0.0f;
            for (int s = 0; s < syn; ++s) {
                const float e = __expf(sc[s] - m);
                z += e;
                acc = fmaf(e, vp[s], acc);
            }
            logit = acc / z + out_b;
            if (attn) {
                const float iz = 1.0f / z;
                for (int s = 0; s < syn; ++s) attn[(row * hl + h) * syn + s] = __expf(sc[s] - m) * iz;
            }
        } else {
            float acc = 0.0f;
            for (int s = 0; s < syn; ++s) acc += vp[s];
            logit = acc / (float)syn + out_b;
        }
        logitsT[(uw * hl + h) * Lw + t] = logit;
    }
}

// y[o, h, n] = mean over windows w covering n (ascending offsets) of
// logitsT[(unit(o)·W + w)·H_l + h, n - off_w]
__global__ void window_average_kernel(const float* __restrict__ logitsT, const int* __restrict__ out_unit,
                                      int hl, int W, int Lw, int stride, int n_regular, int tail_off, int64_t N,
                                      float* __restrict__ y) {
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int oh = blockIdx.y;
    if (n >= N) return;
    const int o = oh / hl, h = oh % hl;
    const int u = out_unit[o];
    float acc = 0.0f;
    int cnt = 0;
    int64_t w_lo = (n - Lw + 1 + stride - 1) / stride;  // first regular window with off + Lw > n
    if (n - Lw + 1 <= 0) w_lo = 0;
    int64_t w_hi = n / stride;
    if (w_hi > n_regular - 1) w_hi = n_regular - 1;
    for (int64_t w = w_lo; w <= w_hi; ++w) {
        acc += logitsT[(((int64_t)u * W + w) * hl + h) * Lw + (n - w * stride)];
        ++cnt;
    }
    if (tail_off >= 0 && n >= tail_off) {
        acc += logitsT[(((int64_t)u * W + (W - 1)) * hl + h) * Lw + (n - tail_off)];
        ++cnt;
    }
    y[(int64_t)oh * N + n] = acc / (float)cnt;
}

}  // namespace

void launch_window_mean(const MapperSrc& s, float* mean_out, cudaStream_t st) {
    WinSrc w{s.x, s.unit_off, s.win_off, s.head_stride, s.W, s.Lw, s.hs};
    window_mean_kernel<<<(unsigned)(s.units * s.W * s.hs), 256, 0, st>>>(w, mean_out);
    check_launch("window_mean_kernel");
}

void launch_conv1_im2col(const MapperSrc& s, const float* inv_mean, const float* w1, const float* b1, int mid,
                         __half* col_h, __half* col_l, float* rinv, cudaStream_t st, F8Out f8) {
    WinSrc w{s.x, s.unit_off, s.win_off, s.head_stride, s.W, s.Lw, s.hs};
    const size_t smem = sizeof(float) * ((size_t)mid * (s.hs * 3 + 1) + (size_t)s.hs * (kConvTok + 4) +
                                         (size_t)(kConvTok + 2) * mid + (kConvTok + 2) + kConvTok);
    static std::atomic<size_t> attr[64];  // per device (the limit is a per-device function attribute)
    int dev = 0;
    PKV_CUDA(cudaGetDevice(&dev));
    if (smem > 48 * 1024 && smem > attr[dev & 63].load()) {
        PKV_CUDA(cudaFuncSetAttribute(conv1_im2col_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr[dev & 63] = smem;
    }
    const dim3 grid((unsigned)((s.Lw + kConvTok - 1) / kConvTok), (unsigned)(s.units * s.W));
    conv1_im2col_kernel<<<grid, 256, smem, st>>>(w, inv_mean, w1, b1, mid, col_h, col_l, rinv, f8);
    check_launch("conv1_im2col_kernel");
}

void launch_bypass_stem(const MapperSrc& s, const float* inv_mean, const float* w, const float* b, const float* pe,
                        int D, float* z, cudaStream_t st) {
    WinSrc ws{s.x, s.unit_off, s.win_off, s.head_stride, s.W, s.Lw, s.hs};
    const dim3 grid((unsigned)s.Lw, (unsigned)(s.units * s.W));
    bypass_stem_kernel<<<grid, 128, 0, st>>>(ws, inv_mean, w, b, pe, D, z);
    check_launch("bypass_stem_kernel");
}

void launch_layernorm(const float* z, int64_t rows, int D, const float* g, const float* b, __half* hi, __half* lo,
                      cudaStream_t st, F8Out f8) {
    const unsigned blocks = (unsigned)((rows + 7) / 8);
    switch (D) {
        case 128: layernorm_kernel<1><<<blocks, 256, 0, st>>>(z, rows, g, b, hi, lo, f8); break;
        case 256: layernorm_kernel<2><<<blocks, 256, 0, st>>>(z, rows, g, b, hi, lo, f8); break;
        case 512: layernorm_kernel<4><<<blocks, 256, 0, st>>>(z, rows, g, b, hi, lo, f8); break;
        case 1024: layernorm_kernel<8><<<blocks, 256, 0, st>>>(z, rows, g, b, hi, lo, f8); break;
        default: throw Error{PKV_ECONFIG, cat("GPU layernorm supports d_time in {128,256,512,1024}, got ", D)};
    }
    check_launch("layernorm_kernel");
}

void launch_split_rows_scaled(const float* z, int64_t rows, int D, __half* hi, __half* lo, float* rinv,
                              cudaStream_t st) {
    if (rows == 0) return;
    split_rows_scaled_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(z, rows, D, hi, lo, rinv);
    check_launch("split_rows_scaled_kernel");
}

void launch_window_colmean_add(float* z, int64_t nwin, int Lw, int D, cudaStream_t st) {
    const dim3 grid((unsigned)((D + 127) / 128), (unsigned)nwin);
    window_colmean_add_kernel<<<grid, 128, 0, st>>>(z, Lw, D);
    check_launch("window_colmean_add_kernel");
}

void launch_stage3(const float* s3, int64_t rows, int ld, int hl, int syn, bool cross_active, float out_b, int Lw,
                   float* logitsT, float* attn, cudaStream_t st) {
    stage3_kernel<<<(unsigned)((rows + 127) / 128), 128, 0, st>>>(s3, rows, ld, hl, syn, cross_active ? 1 : 0, out_b,
                                                                 Lw, logitsT, attn);
    check_launch("stage3_kernel");
}

void launch_window_average(const float* logitsT, const int* out_unit, int n_out, int hl, int W, int Lw, int stride,
                           int n_regular, int tail_off, int64_t N, float* y, cudaStream_t st) {
    const dim3 grid((unsigned)((N + 255) / 256), (unsigned)(n_out * hl));
    window_average_kernel<<<grid, 256, 0, st>>>(logitsT, out_unit, hl, W, Lw, stride, n_regular, tail_off, N, y);
    check_launch("window_average_kernel");
}

}  // namespace pkv
