// K4: batched exact solve -- Cholesky factorisation + two triangular solves.
//
// Replaces solvers.exact_solve (solvers.py:148-164; scipy cho_factor(lower=
// True) + cho_solve = LAPACK dpotrf/dpotrs) and the per-system Python loop of
// batch_solve (solvers.py:221-237).
//
// One CTA (4 warps) per system.  The packed lower triangle is expanded into a
// shared-memory square (leading dimension f+1, conflict-free column access).
// Right-looking factorisation with ONE barrier per column: at step k every
// thread reads the (already updated, unscaled) column k, computes the pivot
// d = A[k][k] itself, and applies A[i][j] -= A[i][k]*A[j][k]/d to the trailing
// triangle.  The columns are scaled to the Cholesky factor in one pass at the
// end.  A non-positive pivot aborts the system with
// info = k+1 (LAPACK's convention).  Warp 0 then runs forward/back
// substitution with the right-hand side distributed over lanes (shuffles, no
// block barriers).
#include <cstdlib>

#include "common.cuh"

namespace cmf {

template <typename Acc>
__global__ void __launch_bounds__(128) chol_kernel(const float *A, int64_t a_stride, const float *B,
                                                   const int64_t *nu, int64_t nsys, int f,
                                                   float *X, int32_t *info, int32_t *nbad) {
    extern __shared__ __align__(16) unsigned char smraw[];
    Acc *L = reinterpret_cast<Acc *>(smraw);
    const int ld = f + 1;
    const int64_t s = blockIdx.x;
    if (nu && nu[s] == 0) return;
    const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5, NW = NT >> 5;
    const float *src = A + static_cast<size_t>(s) * a_stride;
    const int64_t P = packed_size(f);
    // expand packed lower: k -> (i, j)
    for (int64_t k = tid; k < P; k += NT) {
        int i = static_cast<int>((sqrt(8.0 * static_cast<double>(k) + 1.0) - 1.0) * 0.5);
        while (static_cast<int64_t>(i + 1) * (i + 2) / 2 <= k) ++i;
        while (static_cast<int64_t>(i) * (i + 1) / 2 > k) --i;
        const int j = static_cast<int>(k - static_cast<int64_t>(i) * (i + 1) / 2);
        L[i * ld + j] = static_cast<Acc>(src[k]);
    }
    __syncthreads();
    int bad = 0;
    for (int k = 0; k < f; ++k) {
        const Acc d = L[k * ld + k];
        if (!(d > Acc(0))) {
            bad = k + 1;
            break;
        }
        const Acc inv_d = Acc(1) / d;
        // trailing update with the unscaled column k (Gaussian elimination on
        // the symmetric matrix; column k is frozen from here on)
        for (int i = k + 1 + warp; i < f; i += NW) {
            const Acc lik = L[i * ld + k] * inv_d;
            for (int j = k + 1 + lane; j <= i; j += 32) L[i * ld + j] -= lik * L[j * ld + k];
        }
        __syncthreads();
    }
    // a block-uniform decision: every thread evaluated the same pivots
    if (bad) {
        if (tid == 0) {
            if (info) info[s] = bad;
            if (nbad) atomicAdd(nbad, 1);
        }
        return;
    }
    // Cholesky factor from the frozen columns: L[i][k] = A[i][k] / sqrt(d_k),
    // L[k][k] = sqrt(d_k)
    for (int64_t e = tid; e < static_cast<int64_t>(f) * f; e += NT) {
        const int i = static_cast<int>(e / f), k = static_cast<int>(e - static_cast<int64_t>(i) * f);
        if (k < i) L[i * ld + k] = L[i * ld + k] / sqrt(L[k * ld + k]);
    }
    __syncthreads();
    for (int i = tid; i < f; i += NT) L[i * ld + i] = sqrt(L[i * ld + i]);
    __syncthreads();
    if (warp != 0) return;
    // forward / back substitution on warp 0; y_t owned by lane t % 32
    constexpr int MQ = 8;  // f <= 256
    Acc y[MQ];
#pragma unroll
    for (int q = 0; q < MQ; ++q) {
        const int t = lane + 32 * q;
        y[q] = t < f ? static_cast<Acc>(B[s * f + t]) : Acc(0);
    }
    for (int i = 0; i < f; ++i) {  // L y = b
        const int oq = i >> 5, ol = i & 31;
        Acc yi = Acc(0);
#pragma unroll
        for (int q = 0; q < MQ; ++q)
            if (q == oq) yi = y[q];
        yi = __shfl_sync(0xffffffffu, yi, ol) / L[i * ld + i];
#pragma unroll
        for (int q = 0; q < MQ; ++q) {
            const int t = lane + 32 * q;
            if (t == i) y[q] = yi;
            else if (t > i && t < f) y[q] -= L[t * ld + i] * yi;
        }
    }
    for (int i = f - 1; i >= 0; --i) {  // L^T x = y
        const int oq = i >> 5, ol = i & 31;
        Acc xi = Acc(0);
#pragma unroll
        for (int q = 0; q < MQ; ++q)
            if (q == oq) xi = y[q];
        xi = __shfl_sync(0xffffffffu, xi, ol) / L[i * ld + i];
#pragma unroll
        for (int q = 0; q < MQ; ++q) {
            const int t = lane + 32 * q;
            if (t == i) y[q] = xi;
            else if (t < i) y[q] -= L[i * ld + t] * xi;
        }
    }
#pragma unroll
    for (int q = 0; q < MQ; ++q) {
        const int t = lane + 32 * q;
        if (t < f) X[s * f + t] = static_cast<float>(y[q]);
    }
    if (lane == 0 && info) info[s] = 0;
}

int chol_smem_launch(const float *, int64_t, const float *, const int64_t *, int64_t, int, float *, int32_t *,
                     int32_t *, cudaStream_t);

int chol_launch(const float *a, int64_t a_stride, const float *b, const int64_t *nu, int64_t nsys,
                int f, bool fp64, float *x, int32_t *info, int32_t *nbad, cudaStream_t st) {
    if (nsys == 0) return CMF_OK;
    // fp32 production path: 4x4 tiles in shared memory (chol_smem.cu); this
    // file's one-barrier-per-column kernel serves fp64 and f > 128
    if (!fp64 && f <= 128) return chol_smem_launch(a, a_stride, b, nu, nsys, f, x, info, nbad, st);
    if (f > 256) return set_error(CMF_EINVAL, "f=%d too large for the Cholesky kernel", f);
    const size_t es = fp64 ? 8 : 4;
    const size_t smem = static_cast<size_t>(f) * (f + 1) * es;
    if (smem > 227 * 1024)
        return set_error(CMF_EINVAL, "f=%d does not fit the shared-memory Cholesky (%s)", f,
                         fp64 ? "fp64" : "fp32");
    if (fp64) {
        auto k = chol_kernel<double>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<static_cast<unsigned>(nsys), 128, smem, st>>>(a, a_stride, b, nu, nsys, f, x, info, nbad);
    } else {
        auto k = chol_kernel<float>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<static_cast<unsigned>(nsys), 128, smem, st>>>(a, a_stride, b, nu, nsys, f, x, info, nbad);
    }
    return check_launch("chol_kernel");
}

}  // namespace cmf
