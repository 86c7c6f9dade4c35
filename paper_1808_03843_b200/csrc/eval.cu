// Evaluation kernels: squared error over triples or a CSR
// view (als.objective data term, als.rmse), the weighted regulariser
// (als.py:86-93), predict_pairs (factors.py:41-54), and the float32->binary16
// store (gram.pack_half, gram.py:132-146).
//
// Reductions are deterministic: a fixed grid writes one float64 partial per
// block into out[1..nblocks], then one block sums them in index order into
// out[0].  `out` must hold CMF_REDUCE_SLOTS doubles.
#include "common.cuh"

namespace cmf {

constexpr int kRedBlocks = 592;  // 4 x 148 SMs
constexpr int kRedThreads = 256;

__device__ __forceinline__ double block_reduce_store(double v, double *slot) {
    __shared__ double red[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
        *slot = s;
    }
    return v;
}

// The reference's predict_pairs is numpy's float32 einsum "ij,ij->i"
// (factors.py:41-54), which this image's numpy runs on its SSE baseline
// (einsum_sumprod, no FMA): four lanes; each 16-element block adds its four
// vectors in the order 3, 2, 1, 0; the tail adds zero-padded vectors one at a
// time; the lanes then reduce as (l0 + l1) + (l2 + l3).  Restating that order
// with separate round-to-nearest multiplies and adds makes every predicted
// rating bit-identical to the reference's -- and to the ratings gen_synthetic
// wrote, so noiseless data round-trips to an RMSE of exactly zero.
__device__ __forceinline__ float dotf(const float *a, const float *b, int f) {
    float l0 = 0.0f, l1 = 0.0f, l2 = 0.0f, l3 = 0.0f;
    int c = 0;
    for (; c + 16 <= f; c += 16) {
#pragma unroll
        for (int k = 12; k >= 0; k -= 4) {
            l0 = __fadd_rn(__fmul_rn(a[c + k], b[c + k]), l0);
            l1 = __fadd_rn(__fmul_rn(a[c + k + 1], b[c + k + 1]), l1);
            l2 = __fadd_rn(__fmul_rn(a[c + k + 2], b[c + k + 2]), l2);
            l3 = __fadd_rn(__fmul_rn(a[c + k + 3], b[c + k + 3]), l3);
        }
    }
    for (; c < f; c += 4) {
        l0 = __fadd_rn(__fmul_rn(a[c], b[c]), l0);
        if (c + 1 < f) l1 = __fadd_rn(__fmul_rn(a[c + 1], b[c + 1]), l1);
        if (c + 2 < f) l2 = __fadd_rn(__fmul_rn(a[c + 2], b[c + 2]), l2);
        if (c + 3 < f) l3 = __fadd_rn(__fmul_rn(a[c + 3], b[c + 3]), l3);
    }
    return __fadd_rn(__fadd_rn(l0, l1), __fadd_rn(l2, l3));
}

// als.objective predicts in float64 (als.py:84-87)
__device__ __forceinline__ double dotd(const float *a, const float *b, int f) {
    double acc = 0.0;
    for (int c = 0; c < f; ++c) acc = fma(static_cast<double>(a[c]), static_cast<double>(b[c]), acc);
    return acc;
}

template <typename I>
__global__ void sq_error_kernel(const I *users, const I *items, const float *r, int64_t count,
                                const float *x, const float *theta, int f, double *out) {
    double acc = 0.0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < count; k += stride) {
        const float pred = dotf(x + static_cast<int64_t>(users[k]) * f, theta + static_cast<int64_t>(items[k]) * f, f);
        const double d = static_cast<double>(r[k]) - static_cast<double>(pred);
        acc = fma(d, d, acc);
    }
    block_reduce_store(acc, out + 1 + blockIdx.x);
}

__global__ void sq_error_csr_kernel(const int64_t *indptr, const int32_t *indices, const float *vals,
                                    int64_t nrows, const float *x, const float *theta, int f,
                                    double *out) {
    double acc = 0.0;
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t u = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < nrows; u += warps) {
        const float *xu = x + u * f;
        for (int64_t p = indptr[u] + lane; p < indptr[u + 1]; p += 32) {
            const double pred = dotd(xu, theta + static_cast<int64_t>(indices[p]) * f, f);
            const double d = static_cast<double>(vals[p]) - pred;
            acc = fma(d, d, acc);
        }
    }
    block_reduce_store(acc, out + 1 + blockIdx.x);
}

__global__ void wsqnorm_kernel(const int64_t *indptr, const float *x, int64_t nrows, int f, double *out) {
    double acc = 0.0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < nrows; u += stride) {
        double s = 0.0;
        for (int c = 0; c < f; ++c) {
            const double v = static_cast<double>(x[u * f + c]);
            s = fma(v, v, s);
        }
        const double w = indptr ? static_cast<double>(indptr[u + 1] - indptr[u]) : 1.0;
        acc = fma(w, s, acc);
    }
    block_reduce_store(acc, out + 1 + blockIdx.x);
}

__global__ void finish_reduce_kernel(double *out, int n) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += out[1 + i];
        out[0] = s;
    }
}

template <typename I>
__global__ void predict_kernel(const I *users, const I *items, int64_t count, const float *x,
                               const float *theta, int f, float *pred) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k < count) pred[k] = dotf(x + static_cast<int64_t>(users[k]) * f, theta + static_cast<int64_t>(items[k]) * f, f);
}

__global__ void pack_half_kernel(const float *in, __half *out, int64_t n, int32_t *ovf) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    int flag = 0;
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += stride) {
        const float v = in[k];
        const __half h = __float2half_rn(v);
        if (isfinite(v) && __hisinf(h)) flag = 1;
        out[k] = h;
    }
    if (flag && ovf) atomicOr(ovf, 1);
}

int sq_error_launch(const void *users, const void *items, bool idx64, const float *r, int64_t count,
                    const float *x, const float *theta, int f, double *out, cudaStream_t st) {
    if (idx64)
        sq_error_kernel<int64_t><<<kRedBlocks, kRedThreads, 0, st>>>(
            static_cast<const int64_t *>(users), static_cast<const int64_t *>(items), r, count, x, theta, f, out);
    else
        sq_error_kernel<int32_t><<<kRedBlocks, kRedThreads, 0, st>>>(
            static_cast<const int32_t *>(users), static_cast<const int32_t *>(items), r, count, x, theta, f, out);
    finish_reduce_kernel<<<1, 32, 0, st>>>(out, kRedBlocks);
    return check_launch("sq_error_kernel");
}

int sq_error_csr_launch(const int64_t *indptr, const int32_t *indices, const float *vals, int64_t nrows,
                        const float *x, const float *theta, int f, double *out, cudaStream_t st) {
    sq_error_csr_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(indptr, indices, vals, nrows, x, theta, f, out);
    finish_reduce_kernel<<<1, 32, 0, st>>>(out, kRedBlocks);
    return check_launch("sq_error_csr_kernel");
}

int wsqnorm_launch(const int64_t *indptr, const float *x, int64_t nrows, int f, double *out, cudaStream_t st) {
    wsqnorm_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(indptr, x, nrows, f, out);
    finish_reduce_kernel<<<1, 32, 0, st>>>(out, kRedBlocks);
    return check_launch("wsqnorm_kernel");
}

int predict_launch(const void *users, const void *items, bool idx64, int64_t count, const float *x,
                   const float *theta, int f, float *pred, cudaStream_t st) {
    if (count == 0) return CMF_OK;
    const unsigned blocks = static_cast<unsigned>((count + 255) / 256);
    if (idx64)
        predict_kernel<int64_t><<<blocks, 256, 0, st>>>(static_cast<const int64_t *>(users),
                                                         static_cast<const int64_t *>(items), count, x, theta, f, pred);
    else
        predict_kernel<int32_t><<<blocks, 256, 0, st>>>(static_cast<const int32_t *>(users),
                                                         static_cast<const int32_t *>(items), count, x, theta, f, pred);
    return check_launch("predict_kernel");
}

int pack_half_launch(const float *in, void *out, int64_t n, int32_t *ovf, cudaStream_t st) {
    if (n == 0) return CMF_OK;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    pack_half_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(in, static_cast<__half *>(out), n, ovf);
    return check_launch("pack_half_kernel");
}

}  // namespace cmf
