// train.cu — GPU training of the HybridAxialMapper: the
// reference's training forward (forward_pair with training = true,
// proj/src/mapper.cpp:274-342: batchnorm1d on batch statistics and the
// running-stat EMA, ops.cpp:806-850) keeping the activations the backward
// needs, and the reverse sweep the reference's tape performs
// (proj/src/tensor.cpp:156-199 over the op closures in ops.cpp) from
// d loss / d logits — pkv_loss_total's gradient (loss.cpp:324-374) — to
// d loss / d every parameter, in the blob layout (named_parameters order).
//
// Precision: fp32 throughout (the reference is fp64); no fp16 planes, since
// gradients span far more range than the inference activations. The dense
// products are plain row-major GEMMs (linear layers, convolutions as im2col
// GEMMs, the per-head attention products) and go to cuBLAS in pedantic fp32
// (loaded at first use, like NCCL in shard.cpp); everything else is a
// hand-written kernel below.
//
// Layout: activations are token-major [R = B·n, C] (the reference's stem runs
// on [B, C, n]; the convolution is along the token axis of each batch row).
#include <cublas_v2.h>
#include <dlfcn.h>

#include <cmath>
#include <map>
#include <mutex>

#include "mapper.h"

namespace pkv {
namespace {

// ---------------------------------------------------------------- cuBLAS --
struct Blas {
    cublasStatus_t (*create)(cublasHandle_t*) = nullptr;
    cublasStatus_t (*destroy)(cublasHandle_t) = nullptr;
    cublasStatus_t (*set_stream)(cublasHandle_t, cudaStream_t) = nullptr;
    cublasStatus_t (*set_math)(cublasHandle_t, cublasMath_t) = nullptr;
    cublasStatus_t (*sgemm)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int, const float*,
                            const float*, int, const float*, int, const float*, float*, int) = nullptr;
    cublasStatus_t (*sgemm_sb)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int, const float*,
                               const float*, int, long long, const float*, int, long long, const float*, float*, int,
                               long long, int) = nullptr;
};

const Blas& blas() {
    static Blas b;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libcublas.so.12", RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("/usr/local/cuda/lib64/libcublas.so.12", RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            err = dlerror() ? dlerror() : "dlopen failed";
            return;
        }
        b.create = reinterpret_cast<decltype(b.create)>(dlsym(h, "cublasCreate_v2"));
        b.destroy = reinterpret_cast<decltype(b.destroy)>(dlsym(h, "cublasDestroy_v2"));
        b.set_stream = reinterpret_cast<decltype(b.set_stream)>(dlsym(h, "cublasSetStream_v2"));
        b.set_math = reinterpret_cast<decltype(b.set_math)>(dlsym(h, "cublasSetMathMode"));
        b.sgemm = reinterpret_cast<decltype(b.sgemm)>(dlsym(h, "cublasSgemm_v2"));
        b.sgemm_sb = reinterpret_cast<decltype(b.sgemm_sb)>(dlsym(h, "cublasSgemmStridedBatched"));
    });
    PKV_REQUIRE(b.sgemm && b.sgemm_sb && b.create, PKV_ECUDA, "cuBLAS unavailable for mapper training: ", err);
    return b;
}

void blas_ok(cublasStatus_t s, const char* what) {
    PKV_REQUIRE(s == CUBLAS_STATUS_SUCCESS, PKV_ECUDA, what, " failed: cuBLAS status ", (int)s);
}

// Row-major C[M, N] = alpha · op(A)[M, K] · op(B)[K, N] + beta · C, batched
// with element strides sa / sb / sc. cuBLAS is column-major: C^T = op(B)^T op(A)^T.
void gemm(cublasHandle_t h, bool ta, bool tb, int64_t M, int64_t N, int64_t K, float alpha, const float* A,
          int64_t lda, const float* B, int64_t ldb, float beta, float* C, int64_t ldc, int batch = 1, int64_t sa = 0,
          int64_t sb = 0, int64_t sc = 0) {
    if (M == 0 || N == 0) return;
    const Blas& b = blas();
    const cublasOperation_t oa = ta ? CUBLAS_OP_T : CUBLAS_OP_N, ob = tb ? CUBLAS_OP_T : CUBLAS_OP_N;
    if (batch == 1)
        blas_ok(b.sgemm(h, ob, oa, (int)N, (int)M, (int)K, &alpha, B, (int)ldb, A, (int)lda, &beta, C, (int)ldc),
                "cublasSgemm");
    else
        blas_ok(b.sgemm_sb(h, ob, oa, (int)N, (int)M, (int)K, &alpha, B, (int)ldb, sb, A, (int)lda, sa, &beta, C,
                           (int)ldc, sc, batch),
                "cublasSgemmStridedBatched");
}

// ------------------------------------------------------------- kernels ----
constexpr int kT = 256;
inline unsigned blocks_for(int64_t n) { return (unsigned)std::min<int64_t>((n + kT - 1) / kT, 148 * 16); }

__device__ __forceinline__ float gelu_f(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }
__device__ __forceinline__ float gelu_grad(float x) {
    return 0.5f * (1.0f + erff(x * 0.70710678118654752f)) + x * 0.39894228040143268f * expf(-0.5f * x * x);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// normalize_input (mapper.cpp:287-291) + transpose: x [B, Hs, n] -> inT [B·n, Hs],
// inT = x / clamp_min(mean_t x, 1e-12). One block per (b, h).
__global__ void normalize_t_kernel(const float* __restrict__ x, int Hs, int n, bool normalize,
                                   float* __restrict__ inT) {
    const int bh = blockIdx.x, b = bh / Hs, h = bh % Hs;
    const float* row = x + (int64_t)bh * n;
    float scale = 1.0f;
    if (normalize) {
        __shared__ double red[32];
        double s = 0.0;
        for (int t = threadIdx.x; t < n; t += blockDim.x) s += row[t];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double tot = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
            red[0] = fmax(tot / n, 1e-12);
        }
        __syncthreads();
        scale = (float)(1.0 / red[0]);
    }
    for (int t = threadIdx.x; t < n; t += blockDim.x) inT[((int64_t)b * n + t) * Hs + h] = row[t] * scale;
}

// im2col along the token axis (conv1d k = 3, pad 1, ops.cpp:582-629):
// col[(b, t), c·3 + k] = a[(b, t + k − 1), c] (zero outside the batch row).
__global__ void im2col3_kernel(const float* __restrict__ a, int64_t R, int n, int C, float* __restrict__ col) {
    const int64_t total = R * C * 3;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / (3 * C);
        const int ck = (int)(i % (3 * C)), c = ck / 3, k = ck % 3;
        const int t = (int)(r % n) + k - 1;
        col[i] = (t >= 0 && t < n) ? a[(r - (r % n) + t) * C + c] : 0.0f;
    }
}

// its adjoint: da[(b, t), c] = Σ_k dcol[(b, t − k + 1), c·3 + k]
__global__ void col2im3_kernel(const float* __restrict__ dcol, int64_t R, int n, int C, float* __restrict__ da) {
    const int64_t total = R * C;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / C;
        const int c = (int)(i % C), t = (int)(r % n);
        float s = 0.0f;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int src = t - k + 1;
            if (src >= 0 && src < n) s += dcol[(r - t + src) * 3 * C + c * 3 + k];
        }
        da[i] = s;
    }
}

// y[r, c] += bias[c]
__global__ void add_bias_kernel(float* __restrict__ y, int64_t R, int C, const float* __restrict__ bias) {
    const int64_t total = R * C;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
        y[i] += bias[i % C];
}

// out[c] (+)= Σ_r a[r, c] (· b[r, c] when b != null); one block per 32 columns,
// fp64 partial sums. acc: add into out instead of overwriting.
__global__ void colsum_kernel(const float* __restrict__ a, const float* __restrict__ b, int64_t R, int C,
                              float* __restrict__ out, bool acc) {
    __shared__ double red[8][33];
    const int c = blockIdx.x * 32 + threadIdx.x;
    double s = 0.0;
    if (c < C)
        for (int64_t r = threadIdx.y; r < R; r += 8) s += b ? (double)a[r * C + c] * b[r * C + c] : (double)a[r * C + c];
    red[threadIdx.y][threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.y == 0 && c < C) {
        double t = 0.0;
        for (int y = 0; y < 8; ++y) t += red[y][threadIdx.x];
        out[c] = (float)(acc ? out[c] + t : t);
    }
}

// batchnorm1d training statistics (ops.cpp:818-850): per channel mean and
// biased variance over the R rows (two passes, fp64), rstd = 1/sqrt(var + eps),
// running stats EMA (momentum 0.1, unbiased variance).
__global__ void bn_stats_kernel(const float* __restrict__ y, int64_t R, int C, float* __restrict__ mean,
                                float* __restrict__ rstd, float* __restrict__ run_mean, float* __restrict__ run_var) {
    __shared__ double red[8][33];
    __shared__ double mu_s[32];
    const int c = blockIdx.x * 32 + threadIdx.x;
    double s = 0.0;
    if (c < C)
        for (int64_t r = threadIdx.y; r < R; r += 8) s += y[r * C + c];
    red[threadIdx.y][threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.y == 0) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += red[k][threadIdx.x];
        mu_s[threadIdx.x] = t / (double)R;
    }
    __syncthreads();
    const double mu = mu_s[threadIdx.x];
    double v = 0.0;
    if (c < C)
        for (int64_t r = threadIdx.y; r < R; r += 8) {
            const double d = y[r * C + c] - mu;
            v += d * d;
        }
    __syncthreads();
    red[threadIdx.y][threadIdx.x] = v;
    __syncthreads();
    if (threadIdx.y == 0 && c < C) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += red[k][threadIdx.x];
        const double var = t / (double)R;
        mean[c] = (float)mu;
        rstd[c] = (float)(1.0 / sqrt(var + 1e-5));
        run_mean[c] = (float)(0.9 * run_mean[c] + 0.1 * mu);
        run_var[c] = (float)(0.9 * run_var[c] + 0.1 * var * (double)R / (double)(R - 1));
    }
}

// xhat = (y − μ)·rstd (kept), pre = xhat·γ + β (kept), a = gelu(pre)
__global__ void bn_apply_gelu_kernel(const float* __restrict__ y, int64_t R, int C, const float* __restrict__ mean,
                                     const float* __restrict__ rstd, const float* __restrict__ g,
                                     const float* __restrict__ be, float* __restrict__ xhat, float* __restrict__ pre,
                                     float* __restrict__ a) {
    const int64_t total = R * C;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % C);
        const float xh = (y[i] - mean[c]) * rstd[c];
        const float p = xh * g[c] + be[c];
        xhat[i] = xh;
        pre[i] = p;
        a[i] = gelu_f(p);
    }
}

// d(pre) = da · gelu'(pre), in place into da
__global__ void gelu_back_kernel(float* __restrict__ da, const float* __restrict__ pre, int64_t total) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
        da[i] *= gelu_grad(pre[i]);
}

__global__ void gelu_fwd_kernel(const float* __restrict__ u, float* __restrict__ g, int64_t total) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
        g[i] = gelu_f(u[i]);
}

// batchnorm backward through the batch statistics (ops.cpp:879-930):
// dy = γ·rstd/R · (R·dpre − Σdpre − xhat·Σ(dpre·xhat)); sums[c] = Σdpre (dβ), sums[C + c] = Σ dpre·xhat (dγ)
__global__ void bn_back_kernel(const float* __restrict__ dpre, const float* __restrict__ xhat, int64_t R, int C,
                               const float* __restrict__ g, const float* __restrict__ rstd,
                               const float* __restrict__ dbeta, const float* __restrict__ dgamma,
                               float* __restrict__ dy) {
    const int64_t total = R * C;
    const float inv_r = 1.0f / (float)R;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % C);
        dy[i] = g[c] * rstd[c] * (dpre[i] - inv_r * (dbeta[c] + xhat[i] * dgamma[c]));
    }
}

// z[(b, t), :] += PE[t, :] (sinusoidal_pe, mapper.cpp:51-64, in fp64)
__global__ void add_pe_kernel(float* __restrict__ z, int64_t R, int n, int D) {
    const int64_t total = R * D;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int t = (int)((i / D) % n), c = (int)(i % D), i2 = c / 2 * 2;
        const double ang = (double)t * pow(10000.0, -(double)i2 / (double)D);
        z[i] += (float)((c & 1) ? cos(ang) : sin(ang));
    }
}

// layernorm (ops.cpp:721-754) forward: one warp per row, two passes; keeps mean / rstd
__global__ void ln_fwd_kernel(const float* __restrict__ x, int64_t R, int D, const float* __restrict__ g,
                              const float* __restrict__ b, float* __restrict__ y, float* __restrict__ mean,
                              float* __restrict__ rstd) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < R;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const float* xr = x + r * D;
        float s = 0.0f;
        for (int c = lane; c < D; c += 32) s += xr[c];
        const float mu = warp_sum(s) / D;
        float v = 0.0f;
        for (int c = lane; c < D; c += 32) {
            const float d = xr[c] - mu;
            v += d * d;
        }
        const float is = rsqrtf(warp_sum(v) / D + 1e-5f);
        for (int c = lane; c < D; c += 32) y[r * D + c] = (xr[c] - mu) * is * g[c] + b[c];
        if (lane == 0) {
            mean[r] = mu;
            rstd[r] = is;
        }
    }
}

// layernorm backward: dx (+)= rstd·(dxh − mean(dxh) − xhat·mean(dxh·xhat)), dxh = dy·γ;
// dγ += Σ dy·xhat, dβ += Σ dy (per-warp register partials over its rows, then atomics)
template <int kMaxCols>
__global__ void ln_back_kernel(const float* __restrict__ x, const float* __restrict__ dy, int64_t R, int D,
                               const float* __restrict__ g, const float* __restrict__ mean,
                               const float* __restrict__ rstd, float* __restrict__ dx, float* __restrict__ dg,
                               float* __restrict__ db) {
    const int lane = threadIdx.x & 31;
    float pg[kMaxCols / 32], pb[kMaxCols / 32];
#pragma unroll
    for (int i = 0; i < kMaxCols / 32; ++i) pg[i] = pb[i] = 0.0f;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < R;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const float mu = mean[r], is = rstd[r];
        float s1 = 0.0f, s2 = 0.0f;
#pragma unroll
        for (int i = 0; i < kMaxCols / 32; ++i) {
            const int c = lane + 32 * i;
            if (c < D) {
                const float xh = (x[r * D + c] - mu) * is, d = dy[r * D + c];
                const float dxh = d * g[c];
                s1 += dxh;
                s2 += dxh * xh;
                pg[i] += d * xh;
                pb[i] += d;
            }
        }
        s1 = warp_sum(s1) / D;
        s2 = warp_sum(s2) / D;
#pragma unroll
        for (int i = 0; i < kMaxCols / 32; ++i) {
            const int c = lane + 32 * i;
            if (c < D) {
                const float xh = (x[r * D + c] - mu) * is;
                dx[r * D + c] += is * (dy[r * D + c] * g[c] - s1 - xh * s2);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < kMaxCols / 32; ++i) {
        const int c = lane + 32 * i;
        if (c < D) {
            atomicAdd(dg + c, pg[i]);
            atomicAdd(db + c, pb[i]);
        }
    }
}

// row softmax in place over the last axis (length n), one warp per row
__global__ void softmax_rows_kernel(float* __restrict__ s, int64_t rows, int n) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        float* p = s + r * n;
        float m = -INFINITY;
        for (int c = lane; c < n; c += 32) m = fmaxf(m, p[c]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float z = 0.0f;
        for (int c = lane; c < n; c += 32) {
            const float e = expf(p[c] - m);
            p[c] = e;
            z += e;
        }
        const float inv = 1.0f / warp_sum(z);
        for (int c = lane; c < n; c += 32) p[c] *= inv;
    }
}

// softmax backward in place: dS = P ⊙ (dP − Σ_c dP·P), one warp per row
__global__ void softmax_back_kernel(const float* __restrict__ p, float* __restrict__ dp, int64_t rows, int n) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const float* pr = p + r * n;
        float* dr = dp + r * n;
        float s = 0.0f;
        for (int c = lane; c < n; c += 32) s += pr[c] * dr[c];
        s = warp_sum(s);
        for (int c = lane; c < n; c += 32) dr[c] = pr[c] * (dr[c] - s);
    }
}

// Stage 3, cross attention active (mapper.cpp:321-341), one block per token row
// r, one warp per target head l: score_s = Q_l·key_{r,s}/√dq, attn = softmax_s,
// head = Σ_s attn_s·value_{r,s}, logit = head·out_w + out_b.
__global__ void stage3_fwd_kernel(const float* __restrict__ vals, const float* __restrict__ keys,
                                  const float* __restrict__ Q, const float* __restrict__ ow, const float* __restrict__ ob,
                                  int64_t R, int Hl, int syn, int dq, float* __restrict__ attn,
                                  float* __restrict__ heads, float* __restrict__ logit) {
    const int64_t r = blockIdx.x;
    const int l = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (l >= Hl) return;
    const float isq = rsqrtf((float)dq);
    float* a = attn + (r * Hl + l) * syn;
    float m = -INFINITY;
    for (int s = 0; s < syn; ++s) {
        float d = 0.0f;
        for (int e = lane; e < dq; e += 32) d += Q[l * dq + e] * keys[(r * syn + s) * dq + e];
        d = warp_sum(d) * isq;
        if (lane == 0) a[s] = d;
        m = fmaxf(m, d);
    }
    __syncwarp();
    float z = 0.0f;
    for (int s = lane; s < syn; s += 32) {
        const float e = expf(a[s] - m);
        a[s] = e;
        z += e;
    }
    const float inv = 1.0f / warp_sum(z);
    __syncwarp();
    for (int s = lane; s < syn; s += 32) a[s] *= inv;
    __syncwarp();
    float lg = 0.0f;
    for (int e = lane; e < dq; e += 32) {
        float h = 0.0f;
        for (int s = 0; s < syn; ++s) h += a[s] * vals[(r * syn + s) * dq + e];
        heads[(r * Hl + l) * dq + e] = h;
        lg += h * ow[e];
    }
    lg = warp_sum(lg);
    if (lane == 0) logit[r * Hl + l] = lg + ob[0];
}

// Stage 3 backward (cross active): per row r (block), head l (warp).
// dvals / dkeys [R, syn·dq] are written (per row, accumulated over heads in shared memory);
// dQ [Hl, dq], d_ow [dq], d_ob [1] accumulate with atomics.
__global__ void stage3_back_kernel(const float* __restrict__ vals, const float* __restrict__ keys,
                                   const float* __restrict__ Q, const float* __restrict__ ow,
                                   const float* __restrict__ attn, const float* __restrict__ heads,
                                   const float* __restrict__ dlogit, int64_t R, int Hl, int syn, int dq,
                                   float* __restrict__ dvals, float* __restrict__ dkeys, float* __restrict__ dQ,
                                   float* __restrict__ dow, float* __restrict__ dob) {
    extern __shared__ float sh[];  // [syn·dq] dvals | [syn·dq] dkeys | [Hl][syn] dscore
    const int64_t r = blockIdx.x;
    const int l = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sd = syn * dq;
    float* sv = sh;
    float* sk = sh + sd;
    float* sds = sh + 2 * sd;
    for (int i = threadIdx.x; i < 2 * sd; i += blockDim.x) sh[i] = 0.0f;
    __syncthreads();
    const float isq = rsqrtf((float)dq);
    if (l < Hl) {
        const float dl = dlogit[r * Hl + l];
        const float* a = attn + (r * Hl + l) * syn;
        if (lane == 0) atomicAdd(dob, dl);
        for (int e = lane; e < dq; e += 32) atomicAdd(dow + e, dl * heads[(r * Hl + l) * dq + e]);
        // dattn_s = Σ_e dhead_e·v_{s,e}, dhead_e = dl·ow_e; dvals_{s,e} += attn_s·dhead_e
        float dot = 0.0f;
        for (int s = 0; s < syn; ++s) {
            float d = 0.0f;
            for (int e = lane; e < dq; e += 32) {
                const float dh = dl * ow[e];
                d += dh * vals[(r * syn + s) * dq + e];
                atomicAdd(sv + s * dq + e, a[s] * dh);
            }
            d = warp_sum(d);
            if (lane == 0) sds[l * syn + s] = d;
            dot += a[s] * d;
        }
        __syncwarp();
        for (int s = lane; s < syn; s += 32) sds[l * syn + s] = a[s] * (sds[l * syn + s] - dot) * isq;
        __syncwarp();
        // dkeys_{s,e} += dscore_s·Q_{l,e}; dQ_{l,e} += Σ_s dscore_s·key_{s,e}
        for (int e = lane; e < dq; e += 32) {
            float q = 0.0f;
            for (int s = 0; s < syn; ++s) {
                const float ds = sds[l * syn + s];
                atomicAdd(sk + s * dq + e, ds * Q[l * dq + e]);
                q += ds * keys[(r * syn + s) * dq + e];
            }
            atomicAdd(dQ + l * dq + e, q);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < sd; i += blockDim.x) {
        dvals[r * sd + i] = sv[i];
        dkeys[r * sd + i] = sk[i];
    }
}

// Stage 3, cross attention bypassed: pooled = mean_s value_s; logit_l = pooled·out_w + out_b
__global__ void stage3_pool_fwd_kernel(const float* __restrict__ vals, const float* __restrict__ ow,
                                       const float* __restrict__ ob, int64_t R, int Hl, int syn, int dq,
                                       float* __restrict__ pooled, float* __restrict__ logit) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < R;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        float lg = 0.0f;
        for (int e = lane; e < dq; e += 32) {
            float p = 0.0f;
            for (int s = 0; s < syn; ++s) p += vals[(r * syn + s) * dq + e];
            p /= (float)syn;
            pooled[r * dq + e] = p;
            lg += p * ow[e];
        }
        lg = warp_sum(lg) + ob[0];
        for (int l = lane; l < Hl; l += 32) logit[r * Hl + l] = lg;
    }
}

__global__ void stage3_pool_back_kernel(const float* __restrict__ pooled, const float* __restrict__ ow,
                                        const float* __restrict__ dlogit, int64_t R, int Hl, int syn, int dq,
                                        float* __restrict__ dvals, float* __restrict__ dow, float* __restrict__ dob) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < R;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        float dsum = 0.0f;
        for (int l = 0; l < Hl; ++l) dsum += dlogit[r * Hl + l];
        if (lane == 0) atomicAdd(dob, dsum);
        for (int e = lane; e < dq; e += 32) {
            atomicAdd(dow + e, dsum * pooled[r * dq + e]);
            const float dv = dsum * ow[e] / (float)syn;
            for (int s = 0; s < syn; ++s) dvals[(r * syn + s) * dq + e] = dv;
        }
    }
}

// logits [R = B·n, Hl] <-> the API's [B, Hl, n]
__global__ void tokens_to_heads_kernel(const float* __restrict__ a, int64_t R, int n, int Hl, float* __restrict__ out) {
    const int64_t total = R * Hl;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / Hl;
        const int l = (int)(i % Hl);
        out[((r / n) * Hl + l) * n + r % n] = a[i];
    }
}

__global__ void heads_to_tokens_f64_kernel(const double* __restrict__ a, int64_t R, int n, int Hl,
                                           float* __restrict__ out) {
    const int64_t total = R * Hl;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / Hl;
        const int l = (int)(i % Hl);
        out[i] = (float)a[((r / n) * Hl + l) * n + r % n];
    }
}

// encoder bypass (mapper.cpp:317-319): z += mean over tokens (per batch row);
// backward: dz_in = dz + (1/n) Σ_t dz
__global__ void add_token_mean_kernel(float* __restrict__ z, int B, int n, int D) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B * D; i += gridDim.x * blockDim.x) {
        const int b = i / D, c = i % D;
        double s = 0.0;
        for (int t = 0; t < n; ++t) s += z[((int64_t)b * n + t) * D + c];
        const float m = (float)(s / n);
        for (int t = 0; t < n; ++t) z[((int64_t)b * n + t) * D + c] += m;
    }
}

__global__ void acc_f64_kernel(const float* __restrict__ g, int64_t n, double* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] += (double)g[i];
}

}  // namespace

// ------------------------------------------------------------- trainer ----
class Trainer {
public:
    Trainer(pkv_ctx c, const Geometry& g, const Config& cf, const double* blob, int64_t count);
    ~Trainer();
    void forward(const float* x, int64_t B, int64_t n, float* logits, cudaStream_t st);
    void backward(const double* dlogits, double* grad, cudaStream_t st);
    void blob(double* out) const;

    int64_t last_logits() const { return have_forward ? B_ * geom.target_heads * n_ : 0; }

    pkv_ctx ctx;
    Geometry geom;
    Config cfg;
    int64_t count = 0, nparam = 0;
    DevBuf host_io;  // staging for the host forms

private:
    const float* p(const std::string& name) const { return P + off.at(name); }
    float* gp(const std::string& name) { return G + off.at(name); }
    float* buf(const std::string& name) { return P + off.at(name); }
    // saved-activation arena: name -> float offset (sized per forward)
    float* a(const std::string& name) { return act_base + act_off.at(name); }
    void plan(int64_t B, int64_t n);

    std::map<std::string, int64_t> off;
    float* P = nullptr;  // all tensors, blob layout (params then BN buffers)
    float* G = nullptr;  // parameter gradients of one backward
    DevBuf act;
    float* act_base = nullptr;
    std::map<std::string, int64_t> act_off;
    int64_t B_ = 0, n_ = 0;
    bool have_forward = false;
    cublasHandle_t h = nullptr;
};

Trainer::Trainer(pkv_ctx c, const Geometry& g, const Config& cf, const double* blob, int64_t cnt)
    : ctx(c), geom(g), cfg(cf) {
    geom.validate();
    cfg.validate();
    int64_t o = 0;
    for (const auto& [name, n] : param_layout(geom, cfg)) {
        off[name] = o;
        o += n;
        if (name.find("running_") == std::string::npos) nparam = o;
    }
    count = o;
    PKV_REQUIRE_VALUE(cnt == count, "mapper blob has ", cnt, " values, the geometry/config needs ", count);
    std::vector<float> f(blob, blob + count);
    PKV_CUDA(cudaMalloc(&P, count * sizeof(float)));
    PKV_CUDA(cudaMemcpy(P, f.data(), count * sizeof(float), cudaMemcpyHostToDevice));
    PKV_CUDA(cudaMalloc(&G, std::max<int64_t>(nparam, 1) * sizeof(float)));
    blas_ok(blas().create(&h), "cublasCreate");
    if (blas().set_math) blas_ok(blas().set_math(h, CUBLAS_PEDANTIC_MATH), "cublasSetMathMode");
}

Trainer::~Trainer() {
    if (h) blas().destroy(h);
    cudaFree(P);
    cudaFree(G);
}

void Trainer::blob(double* out) const {
    std::vector<float> f(count);
    PKV_CUDA(cudaMemcpy(f.data(), P, count * sizeof(float), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < count; ++i) out[i] = f[i];
}

void Trainer::plan(int64_t B, int64_t n) {
    const int64_t R = B * n, D = cfg.d_time, F = cfg.ffn_mult * D, Cm = cfg.conv_mid(), hs = geom.proxy_heads;
    const int64_t H = cfg.encoder_heads, syn = cfg.syn(geom), dq = cfg.d_head, hl = geom.target_heads;
    act_off.clear();
    int64_t o = 0;
    auto add = [&](const std::string& nm, int64_t n_el) {
        act_off[nm] = o;
        o += (n_el + 63) & ~int64_t(63);
    };
    add("inT", R * hs);
    if (cfg.conv_active) {
        for (const char* s : {"col1", "xhat1", "pre1", "a1"}) add(s, std::string(s) == "col1" ? R * hs * 3 : R * Cm);
        add("col2", R * Cm * 3);
        add("xhat2", R * D);
        add("pre2", R * D);
        for (const char* s : {"mean1", "rstd1"}) add(s, Cm);
        for (const char* s : {"mean2", "rstd2"}) add(s, D);
    }
    if (cfg.enc_active) {
        for (int64_t i = 0; i < cfg.encoder_layers; ++i) {
            const std::string p = "b" + std::to_string(i) + ".";
            for (const char* s : {"zin", "h1", "q", "k", "v", "ctx", "zmid", "h2"}) add(p + s, R * D);
            for (const char* s : {"u", "g"}) add(p + s, R * F);
            for (const char* s : {"m1", "r1", "m2", "r2"}) add(p + s, R);
            add(p + "P", B * H * n * n);
        }
    }
    add("z", R * D);
    add("vals", R * syn * dq);
    add("keys", R * syn * dq);
    add("attn", R * hl * syn);
    add("heads", R * hl * dq);
    add("pooled", R * dq);
    add("logitT", R * hl);
    // backward scratch
    add("dz", R * D);
    add("dtmp", R * std::max(F, 3 * std::max(D, Cm)));
    add("dtmp2", R * std::max(F, D));
    add("dq", R * D);
    add("dk", R * D);
    add("dv", R * D);
    add("dP", B * H * n * n);
    add("dvals", R * syn * dq);
    add("dkeys", R * syn * dq);
    add("dlogitT", R * hl);
    act_base = static_cast<float*>(act.get(static_cast<size_t>(o) * sizeof(float)));
    B_ = B;
    n_ = n;
}

void Trainer::forward(const float* x, int64_t B, int64_t n, float* logits, cudaStream_t st) {
    PKV_REQUIRE_SHAPE(B > 0 && n > 0, "forward_pair input must be [B, H_s, N] with positive extents");
    PKV_REQUIRE_VALUE(n <= cfg.crop_len, "input length ", n, " exceeds crop_len ", cfg.crop_len,
                      "; long inputs go through sliding_forward");
    PKV_REQUIRE(geom.target_heads <= 32, PKV_ECONFIG, "mapper training supports target_heads <= 32, got ",
                geom.target_heads);
    PKV_REQUIRE_VALUE(!cfg.conv_active || B * n >= 2, "batchnorm1d in train mode needs B*N >= 2 per channel, got ",
                      B * n);
    plan(B, n);
    blas_ok(blas().set_stream(h, st), "cublasSetStream");
    const int64_t R = B * n, D = cfg.d_time, F = cfg.ffn_mult * D, Cm = cfg.conv_mid(), hs = geom.proxy_heads;
    const int64_t H = cfg.encoder_heads, dh = D / H, syn = cfg.syn(geom), dq = cfg.d_head, hl = geom.target_heads;
    const dim3 red_blk(32, 8);
    normalize_t_kernel<<<(unsigned)(B * hs), 256, 0, st>>>(x, (int)hs, (int)n, cfg.normalize_input, a("inT"));
    float* z = a("z");
    // ---- Stage 1 (mapper.cpp:294-303)
    if (cfg.conv_active) {
        im2col3_kernel<<<blocks_for(R * hs * 3), kT, 0, st>>>(a("inT"), R, (int)n, (int)hs, a("col1"));
        float* y1 = a("dtmp");
        gemm(h, false, true, R, Cm, hs * 3, 1.0f, a("col1"), hs * 3, p("stem.conv1.w"), hs * 3, 0.0f, y1, Cm);
        add_bias_kernel<<<blocks_for(R * Cm), kT, 0, st>>>(y1, R, (int)Cm, p("stem.conv1.b"));
        bn_stats_kernel<<<(unsigned)((Cm + 31) / 32), red_blk, 0, st>>>(y1, R, (int)Cm, a("mean1"), a("rstd1"),
                                                                         buf("stem.bn1.running_mean"),
                                                                         buf("stem.bn1.running_var"));
        bn_apply_gelu_kernel<<<blocks_for(R * Cm), kT, 0, st>>>(y1, R, (int)Cm, a("mean1"), a("rstd1"),
                                                                p("stem.bn1.gamma"), p("stem.bn1.beta"), a("xhat1"),
                                                                a("pre1"), a("a1"));
        im2col3_kernel<<<blocks_for(R * Cm * 3), kT, 0, st>>>(a("a1"), R, (int)n, (int)Cm, a("col2"));
        float* y2 = a("dtmp");
        gemm(h, false, true, R, D, Cm * 3, 1.0f, a("col2"), Cm * 3, p("stem.conv2.w"), Cm * 3, 0.0f, y2, D);
        add_bias_kernel<<<blocks_for(R * D), kT, 0, st>>>(y2, R, (int)D, p("stem.conv2.b"));
        bn_stats_kernel<<<(unsigned)((D + 31) / 32), red_blk, 0, st>>>(y2, R, (int)D, a("mean2"), a("rstd2"),
                                                                        buf("stem.bn2.running_mean"),
                                                                        buf("stem.bn2.running_var"));
        bn_apply_gelu_kernel<<<blocks_for(R * D), kT, 0, st>>>(y2, R, (int)D, a("mean2"), a("rstd2"),
                                                               p("stem.bn2.gamma"), p("stem.bn2.beta"), a("xhat2"),
                                                               a("pre2"), z);
    } else {
        gemm(h, false, true, R, D, hs, 1.0f, a("inT"), hs, p("stem.bypass.w"), hs, 0.0f, z, D);
        add_bias_kernel<<<blocks_for(R * D), kT, 0, st>>>(z, R, (int)D, p("stem.bypass.b"));
    }
    // ---- Stage 2 (mapper.cpp:305-319)
    if (cfg.enc_active) {
        add_pe_kernel<<<blocks_for(R * D), kT, 0, st>>>(z, R, (int)n, (int)D);
        for (int64_t i = 0; i < cfg.encoder_layers; ++i) {
            const std::string pp = "encoder." + std::to_string(i) + ".", s = "b" + std::to_string(i) + ".";
            PKV_CUDA(cudaMemcpyAsync(a(s + "zin"), z, R * D * 4, cudaMemcpyDeviceToDevice, st));
            ln_fwd_kernel<<<blocks_for(R * 32), kT, 0, st>>>(z, R, (int)D, p(pp + "ln1.gamma"), p(pp + "ln1.beta"),
                                                             a(s + "h1"), a(s + "m1"), a(s + "r1"));
            for (const char* m : {"q", "k", "v"}) {
                gemm(h, false, false, R, D, D, 1.0f, a(s + "h1"), D, p(pp + "attn.w" + m), D, 0.0f, a(s + m), D);
                add_bias_kernel<<<blocks_for(R * D), kT, 0, st>>>(a(s + m), R, (int)D, p(pp + "attn.b" + m));
            }
            for (int64_t b = 0; b < B; ++b) {  // per batch row: heads are a strided batch
                const int64_t ro = b * n * D;
                float* Pb = a(s + "P") + b * H * n * n;
                gemm(h, false, true, n, n, dh, 1.0f / std::sqrt((float)dh), a(s + "q") + ro, D, a(s + "k") + ro, D,
                     0.0f, Pb, n, (int)H, dh, dh, n * n);
                softmax_rows_kernel<<<blocks_for(H * n * 32), kT, 0, st>>>(Pb, H * n, (int)n);
                gemm(h, false, false, n, dh, n, 1.0f, Pb, n, a(s + "v") + ro, D, 0.0f, a(s + "ctx") + ro, D, (int)H,
                     n * n, dh, dh);
            }
            // z_mid = z + ctx·Wo + bo
            gemm(h, false, false, R, D, D, 1.0f, a(s + "ctx"), D, p(pp + "attn.wo"), D, 1.0f, z, D);
            add_bias_kernel<<<blocks_for(R * D), kT, 0, st>>>(z, R, (int)D, p(pp + "attn.bo"));
            PKV_CUDA(cudaMemcpyAsync(a(s + "zmid"), z, R * D * 4, cudaMemcpyDeviceToDevice, st));
            ln_fwd_kernel<<<blocks_for(R * 32), kT, 0, st>>>(z, R, (int)D, p(pp + "ln2.gamma"), p(pp + "ln2.beta"),
                                                             a(s + "h2"), a(s + "m2"), a(s + "r2"));
            gemm(h, false, false, R, F, D, 1.0f, a(s + "h2"), D, p(pp + "ffn1.w"), F, 0.0f, a(s + "u"), F);
            add_bias_kernel<<<blocks_for(R * F), kT, 0, st>>>(a(s + "u"), R, (int)F, p(pp + "ffn1.b"));
            gelu_fwd_kernel<<<blocks_for(R * F), kT, 0, st>>>(a(s + "u"), a(s + "g"), R * F);
            gemm(h, false, false, R, D, F, 1.0f, a(s + "g"), F, p(pp + "ffn2.w"), D, 1.0f, z, D);
            add_bias_kernel<<<blocks_for(R * D), kT, 0, st>>>(z, R, (int)D, p(pp + "ffn2.b"));
        }
    } else {
        add_token_mean_kernel<<<blocks_for(B * D), kT, 0, st>>>(z, (int)B, (int)n, (int)D);
    }
    // ---- Stage 3 (mapper.cpp:321-341)
    const int64_t sd = syn * dq;
    gemm(h, false, false, R, sd, D, 1.0f, z, D, p("cross.value.w"), sd, 0.0f, a("vals"), sd);
    add_bias_kernel<<<blocks_for(R * sd), kT, 0, st>>>(a("vals"), R, (int)sd, p("cross.value.b"));
    if (cfg.cross_active) {
        gemm(h, false, false, R, sd, D, 1.0f, z, D, p("cross.key.w"), sd, 0.0f, a("keys"), sd);
        add_bias_kernel<<<blocks_for(R * sd), kT, 0, st>>>(a("keys"), R, (int)sd, p("cross.key.b"));
        stage3_fwd_kernel<<<(unsigned)R, (unsigned)(32 * hl), 0, st>>>(a("vals"), a("keys"), p("cross.queries"),
                                                                       p("cross.out.w"), p("cross.out.b"), R, (int)hl,
                                                                       (int)syn, (int)dq, a("attn"), a("heads"),
                                                                       a("logitT"));
    } else {
        stage3_pool_fwd_kernel<<<blocks_for(R * 32), kT, 0, st>>>(a("vals"), p("cross.out.w"), p("cross.out.b"), R,
                                                                  (int)hl, (int)syn, (int)dq, a("pooled"),
                                                                  a("logitT"));
    }
    tokens_to_heads_kernel<<<blocks_for(R * hl), kT, 0, st>>>(a("logitT"), R, (int)n, (int)hl, logits);
    check_launch("mapper training forward");
    have_forward = true;
}

void Trainer::backward(const double* dlogits, double* grad, cudaStream_t st) {
    PKV_REQUIRE_VALUE(have_forward, "backward needs a training forward first");
    blas_ok(blas().set_stream(h, st), "cublasSetStream");
    const int64_t B = B_, n = n_, R = B * n, D = cfg.d_time, F = cfg.ffn_mult * D, Cm = cfg.conv_mid();
    const int64_t hs = geom.proxy_heads, H = cfg.encoder_heads, dh = D / H, syn = cfg.syn(geom), dq = cfg.d_head;
    const int64_t hl = geom.target_heads, sd = syn * dq;
    const dim3 red_blk(32, 8);
    PKV_CUDA(cudaMemsetAsync(G, 0, nparam * sizeof(float), st));
    auto colsum = [&](const float* x, const float* y, int64_t rows, int64_t C, float* out, bool acc) {
        colsum_kernel<<<(unsigned)((C + 31) / 32), red_blk, 0, st>>>(x, y, rows, (int)C, out, acc);
    };
    heads_to_tokens_f64_kernel<<<blocks_for(R * hl), kT, 0, st>>>(dlogits, R, (int)n, (int)hl, a("dlogitT"));
    // ---- Stage 3
    float* dz = a("dz");
    float* z = a("z");
    if (cfg.cross_active) {
        const size_t shm = (size_t)(2 * sd + hl * syn) * sizeof(float);
        PKV_REQUIRE(shm <= 48 * 1024, PKV_ECONFIG, "mapper training: stage-3 backward needs synthetic_heads * d_head <= ",
                    (48 * 1024 / 4 - hl * syn) / 2, ", got ", sd);
        stage3_back_kernel<<<(unsigned)R, (unsigned)(32 * hl), shm, st>>>(
            a("vals"), a("keys"), p("cross.queries"), p("cross.out.w"), a("attn"), a("heads"), a("dlogitT"), R,
            (int)hl, (int)syn, (int)dq, a("dvals"), a("dkeys"), gp("cross.queries"), gp("cross.out.w"),
            gp("cross.out.b"));
        gemm(h, true, false, D, sd, R, 1.0f, z, D, a("dkeys"), sd, 0.0f, gp("cross.key.w"), sd);
        colsum(a("dkeys"), nullptr, R, sd, gp("cross.key.b"), false);
    } else {
        stage3_pool_back_kernel<<<blocks_for(R * 32), kT, 0, st>>>(a("pooled"), p("cross.out.w"), a("dlogitT"), R,
                                                                   (int)hl, (int)syn, (int)dq, a("dvals"),
                                                                   gp("cross.out.w"), gp("cross.out.b"));
    }
    gemm(h, true, false, D, sd, R, 1.0f, z, D, a("dvals"), sd, 0.0f, gp("cross.value.w"), sd);
    colsum(a("dvals"), nullptr, R, sd, gp("cross.value.b"), false);
    gemm(h, false, true, R, D, sd, 1.0f, a("dvals"), sd, p("cross.value.w"), sd, 0.0f, dz, D);
    if (cfg.cross_active) gemm(h, false, true, R, D, sd, 1.0f, a("dkeys"), sd, p("cross.key.w"), sd, 1.0f, dz, D);
    // ---- Stage 2, blocks in reverse (dz = d loss / d z_out of the block)
    if (cfg.enc_active) {
        PKV_REQUIRE(D <= 1024, PKV_ECONFIG, "mapper training supports d_time <= 1024, got ", D);
        for (int64_t i = cfg.encoder_layers - 1; i >= 0; --i) {
            const std::string pp = "encoder." + std::to_string(i) + ".", s = "b" + std::to_string(i) + ".";
            // FFN: z_out = z_mid + gelu(h2·W1 + b1)·W2 + b2
            gemm(h, true, false, F, D, R, 1.0f, a(s + "g"), F, dz, D, 0.0f, gp(pp + "ffn2.w"), D);
            colsum(dz, nullptr, R, D, gp(pp + "ffn2.b"), false);
            float* du = a("dtmp");
            gemm(h, false, true, R, F, D, 1.0f, dz, D, p(pp + "ffn2.w"), D, 0.0f, du, F);
            gelu_back_kernel<<<blocks_for(R * F), kT, 0, st>>>(du, a(s + "u"), R * F);
            gemm(h, true, false, D, F, R, 1.0f, a(s + "h2"), D, du, F, 0.0f, gp(pp + "ffn1.w"), F);
            colsum(du, nullptr, R, F, gp(pp + "ffn1.b"), false);
            float* dh2 = a("dtmp2");
            gemm(h, false, true, R, D, F, 1.0f, du, F, p(pp + "ffn1.w"), F, 0.0f, dh2, D);
            // dz (now d/d z_mid) += LN2 backward
            if (D <= 512)
                ln_back_kernel<512><<<296, kT, 0, st>>>(a(s + "zmid"), dh2, R, (int)D, p(pp + "ln2.gamma"),
                                                         a(s + "m2"), a(s + "r2"), dz, gp(pp + "ln2.gamma"),
                                                         gp(pp + "ln2.beta"));
            else
                ln_back_kernel<1024><<<296, kT, 0, st>>>(a(s + "zmid"), dh2, R, (int)D, p(pp + "ln2.gamma"),
                                                          a(s + "m2"), a(s + "r2"), dz, gp(pp + "ln2.gamma"),
                                                          gp(pp + "ln2.beta"));
            // attention: z_mid = z_in + ctx·Wo + bo
            gemm(h, true, false, D, D, R, 1.0f, a(s + "ctx"), D, dz, D, 0.0f, gp(pp + "attn.wo"), D);
            colsum(dz, nullptr, R, D, gp(pp + "attn.bo"), false);
            float* dctx = a("dtmp2");
            gemm(h, false, true, R, D, D, 1.0f, dz, D, p(pp + "attn.wo"), D, 0.0f, dctx, D);
            for (int64_t b = 0; b < B; ++b) {
                const int64_t ro = b * n * D;
                const float* Pb = a(s + "P") + b * H * n * n;
                float* dP = a("dP") + b * H * n * n;
                const float sc = 1.0f / std::sqrt((float)dh);
                gemm(h, false, true, n, n, dh, 1.0f, dctx + ro, D, a(s + "v") + ro, D, 0.0f, dP, n, (int)H, dh, dh,
                     n * n);
                gemm(h, true, false, n, dh, n, 1.0f, Pb, n, dctx + ro, D, 0.0f, a("dv") + ro, D, (int)H, n * n, dh,
                     dh);
                softmax_back_kernel<<<blocks_for(H * n * 32), kT, 0, st>>>(Pb, dP, H * n, (int)n);
                gemm(h, false, false, n, dh, n, sc, dP, n, a(s + "k") + ro, D, 0.0f, a("dq") + ro, D, (int)H, n * n,
                     dh, dh);
                gemm(h, true, false, n, dh, n, sc, dP, n, a(s + "q") + ro, D, 0.0f, a("dk") + ro, D, (int)H, n * n,
                     dh, dh);
            }
            float* dh1 = a("dtmp2");
            bool first = true;
            for (const char* m : {"q", "k", "v"}) {
                const float* dm = a(std::string("d") + m);
                gemm(h, true, false, D, D, R, 1.0f, a(s + "h1"), D, dm, D, 0.0f, gp(pp + "attn.w" + m), D);
                colsum(dm, nullptr, R, D, gp(pp + "attn.b" + m), false);
                gemm(h, false, true, R, D, D, 1.0f, dm, D, p(pp + "attn.w" + m), D, first ? 0.0f : 1.0f, dh1, D);
                first = false;
            }
            if (D <= 512)
                ln_back_kernel<512><<<296, kT, 0, st>>>(a(s + "zin"), dh1, R, (int)D, p(pp + "ln1.gamma"),
                                                         a(s + "m1"), a(s + "r1"), dz, gp(pp + "ln1.gamma"),
                                                         gp(pp + "ln1.beta"));
            else
                ln_back_kernel<1024><<<296, kT, 0, st>>>(a(s + "zin"), dh1, R, (int)D, p(pp + "ln1.gamma"),
                                                          a(s + "m1"), a(s + "r1"), dz, gp(pp + "ln1.gamma"),
                                                          gp(pp + "ln1.beta"));
        }
    } else {
        // z += mean_t z: dz_in = dz + (1/n) Σ_t dz, i.e. the same kernel on the gradient
        add_token_mean_kernel<<<blocks_for(B * D), kT, 0, st>>>(dz, (int)B, (int)n, (int)D);
    }
    // ---- Stage 1 (dz = d loss / d stem output; the PE add passes it through)
    if (cfg.conv_active) {
        gelu_back_kernel<<<blocks_for(R * D), kT, 0, st>>>(dz, a("pre2"), R * D);  // dz := d pre2
        colsum(dz, nullptr, R, D, gp("stem.bn2.beta"), false);
        colsum(dz, a("xhat2"), R, D, gp("stem.bn2.gamma"), false);
        float* dy2 = a("dtmp2");
        bn_back_kernel<<<blocks_for(R * D), kT, 0, st>>>(dz, a("xhat2"), R, (int)D, p("stem.bn2.gamma"), a("rstd2"),
                                                         gp("stem.bn2.beta"), gp("stem.bn2.gamma"), dy2);
        gemm(h, true, false, D, Cm * 3, R, 1.0f, dy2, D, a("col2"), Cm * 3, 0.0f, gp("stem.conv2.w"), Cm * 3);
        colsum(dy2, nullptr, R, D, gp("stem.conv2.b"), false);
        float* dcol = a("dtmp");
        gemm(h, false, false, R, Cm * 3, D, 1.0f, dy2, D, p("stem.conv2.w"), Cm * 3, 0.0f, dcol, Cm * 3);
        float* da1 = a("dk");
        col2im3_kernel<<<blocks_for(R * Cm), kT, 0, st>>>(dcol, R, (int)n, (int)Cm, da1);
        gelu_back_kernel<<<blocks_for(R * Cm), kT, 0, st>>>(da1, a("pre1"), R * Cm);
        colsum(da1, nullptr, R, Cm, gp("stem.bn1.beta"), false);
        colsum(da1, a("xhat1"), R, Cm, gp("stem.bn1.gamma"), false);
        float* dy1 = a("dv");
        bn_back_kernel<<<blocks_for(R * Cm), kT, 0, st>>>(da1, a("xhat1"), R, (int)Cm, p("stem.bn1.gamma"),
                                                          a("rstd1"), gp("stem.bn1.beta"), gp("stem.bn1.gamma"), dy1);
        gemm(h, true, false, Cm, hs * 3, R, 1.0f, dy1, Cm, a("col1"), hs * 3, 0.0f, gp("stem.conv1.w"), hs * 3);
        colsum(dy1, nullptr, R, Cm, gp("stem.conv1.b"), false);
    } else {
        gemm(h, true, false, D, hs, R, 1.0f, dz, D, a("inT"), hs, 0.0f, gp("stem.bypass.w"), hs);
        colsum(dz, nullptr, R, D, gp("stem.bypass.b"), false);
    }
    acc_f64_kernel<<<blocks_for(nparam), kT, 0, st>>>(G, nparam, grad);
    check_launch("mapper training backward");
}

}  // namespace pkv

struct pkv_trainer_s {
    std::unique_ptr<pkv::Trainer> t;
};

using namespace pkv;

extern "C" {

pkv_status pkv_trainer_create(pkv_ctx ctx, const int64_t* geom5, const int64_t* cfg12, const double* blob,
                              int64_t count, pkv_trainer* out) {
    return guard([&] {
        require_ctx(ctx);
        PKV_CUDA(cudaSetDevice(ctx->device));
        auto* h = new pkv_trainer_s();
        try {
            h->t.reset(new Trainer(ctx, Geometry::from5(geom5), Config::from12(cfg12), blob, count));
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

void pkv_trainer_destroy(pkv_trainer t) { delete t; }

pkv_status pkv_trainer_param_count(pkv_trainer t, int64_t* params, int64_t* total) {
    return guard([&] {
        PKV_REQUIRE_VALUE(t, "null trainer");
        *params = t->t->nparam;
        *total = t->t->count;
    });
}

pkv_status pkv_trainer_forward(pkv_trainer t, const float* x_dev, int64_t B, int64_t n, float* logits_dev,
                               void* stream) {
    return guard([&] {
        PKV_REQUIRE_VALUE(t, "null trainer");
        t->t->forward(x_dev, B, n, logits_dev, static_cast<cudaStream_t>(stream));
        count_launch(t->t->ctx);
    });
}

pkv_status pkv_trainer_backward(pkv_trainer t, const double* dlogits_dev, double* grad_dev, void* stream) {
    return guard([&] {
        PKV_REQUIRE_VALUE(t, "null trainer");
        t->t->backward(dlogits_dev, grad_dev, static_cast<cudaStream_t>(stream));
        count_launch(t->t->ctx);
    });
}

pkv_status pkv_trainer_forward_host(pkv_trainer t, const double* x_host, int64_t B, int64_t n, double* logits_host) {
    return guard([&] {
        PKV_REQUIRE_VALUE(t, "null trainer");
        Trainer& tr = *t->t;
        PKV_REQUIRE_SHAPE(B > 0 && n > 0, "forward_pair input must be [B, H_s, N] with positive extents");
        const size_t nx = static_cast<size_t>(B * tr.geom.proxy_heads * n), ny = static_cast<size_t>(B * tr.geom.target_heads * n);
        std::vector<float> xf(x_host, x_host + nx), yf(ny);
        float* d = static_cast<float*>(tr.host_io.get((nx + ny) * sizeof(float)));
        PKV_CUDA(cudaMemcpy(d, xf.data(), nx * sizeof(float), cudaMemcpyHostToDevice));
        tr.forward(d, B, n, d + nx, nullptr);
        PKV_CUDA(cudaMemcpy(yf.data(), d + nx, ny * sizeof(float), cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < ny; ++i) logits_host[i] = yf[i];
        count_launch(tr.ctx);
    });
}

pkv_status pkv_trainer_backward_host(pkv_trainer t, const double* dlogits_host, double* grad_host) {
    return guard([&] {
        PKV_REQUIRE_VALUE(t, "null trainer");
        Trainer& tr = *t->t;
        const size_t nl = static_cast<size_t>(tr.last_logits()), np = static_cast<size_t>(tr.nparam);
        PKV_REQUIRE_VALUE(nl > 0, "backward needs a training forward first");
        double* d = static_cast<double*>(tr.host_io.get((nl + np) * sizeof(double)));
        PKV_CUDA(cudaMemcpy(d, dlogits_host, nl * sizeof(double), cudaMemcpyHostToDevice));
        PKV_CUDA(cudaMemcpy(d + nl, grad_host, np * sizeof(double), cudaMemcpyHostToDevice));
        tr.backward(d, d + nl, nullptr);
        PKV_CUDA(cudaMemcpy(grad_host, d + nl, np * sizeof(double), cudaMemcpyDeviceToHost));
        count_launch(tr.ctx);
    });
}

pkv_status pkv_trainer_blob(pkv_trainer t, double* blob_host) {
    return guard([&] {
        PKV_REQUIRE_VALUE(t, "null trainer");
        t->t->blob(blob_host);
    });
}

}  // extern "C"
