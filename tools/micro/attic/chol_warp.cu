// K4, exact route: batched Cholesky solve, one WARP per system (f <= 124).
//
// Replaces solvers.exact_solve / the exact branch of batch_solve
// (solvers.py:148-164, :221-237; LAPACK dpotrf + dpotrs in the reference).
//
// The system lives in shared memory as the packed lower triangle with every row
// padded to a 16-byte boundary (row i at off(i), ~21 KB at f = 100), plus a
// border row f holding b^T: factorising [[A, 0], [b^T, *]] leaves y = L^-1 b in
// that row, so the forward substitution is part of the factorisation.  A CTA is
// one warp (no block barriers at all), ~10 systems per SM.
//
// Left-looking with 8-column panels (13 at f = 100).  Lane l owns rows
// c0 + l + 32q (q = 0..3) of panel p (c0 = 8p) and accumulates their 8 panel
// entries in registers:
//   (1) s[q][c] = A[i][c0+c] - sum_{k < c0} L[i][k] L[c0+c][k]: its own row read as
//       float4, the 8 panel rows broadcast (all lanes read the same address);
//   (2) the 8x8 diagonal block is factorised right-looking inside the panel,
//       the pivots and the scaled column values broadcast by shuffles, which
//       also applies L_pp^-T to every row below (the panel TRSM);
//   (3) the panel is written back.
// Back substitution x = L^-T y walks the panels in reverse: lanes form the
// L_kp^T x_k partial sums of rows below the panel, a butterfly reduces them,
// and every lane solves the 8x8 triangle redundantly.  Operation order is
// fixed, so results are deterministic.  A non-positive pivot marks the system
// singular: info = column + 1 (LAPACK convention), X is not written.
#include "common.cuh"

namespace cmf {

constexpr int CW_P = 8;  // panel width

// offset (floats) of padded row i: rows of length i+1 rounded up to 4
__device__ __forceinline__ int crow_off(int i) {
    const int a = i >> 2, b = i & 3;
    return 4 * (i + 2 * a * (a - 1) + a * b);
}

__global__ void __launch_bounds__(32) chol_warp_kernel(const float *A, int64_t a_stride, const float *B,
                                                       const int64_t *nu, int64_t nsys, int f, float *X,
                                                       int32_t *info, int32_t *nbad) {
    const int64_t s = blockIdx.x;
    if (nu && nu[s] == 0) return;
    extern __shared__ __align__(16) float Ls[];  // padded packed rows 0..f (row f = b^T)
    float *xs = Ls + crow_off(f + 1);             // x, 128 floats
    const int lane = threadIdx.x;

    // ---- stage the packed system and b (4-byte async copies: rows are unaligned in HBM)
    const float *src = A + static_cast<size_t>(s) * a_stride;
    for (int i = 0; i < f; ++i) {
        const int64_t g0 = static_cast<int64_t>(i) * (i + 1) / 2;
        float *dst = Ls + crow_off(i);
        for (int j = lane; j <= i; j += 32) cp_async4(dst + j, src + g0 + j, 4);
    }
    for (int j = lane; j < f; j += 32) cp_async4(Ls + crow_off(f) + j, B + s * f + j, 4);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();

    const int TB = (f + CW_P - 1) / CW_P;
    int bad = 0;
    for (int p = 0; p < TB && !bad; ++p) {
        const int c0 = CW_P * p;
        const int nc = min(CW_P, f - c0);
        float sv[4][CW_P];
        int roff[4];
        bool rv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int i = c0 + lane + 32 * q;
            rv[q] = i <= f;  // rows c0..f-1 and the border row f
            roff[q] = rv[q] ? crow_off(i) : 0;
#pragma unroll
            for (int c = 0; c < CW_P; ++c)
                sv[q][c] = (rv[q] && c < nc && c0 + c <= i) ? Ls[roff[q] + c0 + c] : 0.0f;
        }
        // (1) left-looking update from the finished columns k < c0
        int poff[CW_P];
#pragma unroll
        for (int c = 0; c < CW_P; ++c) poff[c] = crow_off(c0 + min(c, nc - 1));
        for (int k = 0; k < c0; k += 4) {
            float4 pr[CW_P];
#pragma unroll
            for (int c = 0; c < CW_P; ++c) pr[c] = *reinterpret_cast<const float4 *>(Ls + poff[c] + k);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (!rv[q]) continue;
                const float4 o = *reinterpret_cast<const float4 *>(Ls + roff[q] + k);
#pragma unroll
                for (int c = 0; c < CW_P; ++c) {
                    float v = sv[q][c];
                    v = fmaf(-o.x, pr[c].x, v);
                    v = fmaf(-o.y, pr[c].y, v);
                    v = fmaf(-o.z, pr[c].z, v);
                    v = fmaf(-o.w, pr[c].w, v);
                    sv[q][c] = v;
                }
            }
        }
        // (2) factorise the diagonal block; rows below get L_pp^-T on the way
#pragma unroll
        for (int j = 0; j < CW_P; ++j) {
            if (j >= nc) break;
            const float d = __shfl_sync(0xffffffffu, sv[0][j], j);
            if (!(d > 0.0f)) {
                bad = c0 + j + 1;
                break;
            }
            const float rd = rsqrtf(d);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int i = c0 + lane + 32 * q;
                if (i == c0 + j) sv[q][j] = d * rd;
                else if (i > c0 + j) sv[q][j] *= rd;
            }
#pragma unroll
            for (int m = j + 1; m < CW_P; ++m) {
                if (m >= nc) break;
                const float lmj = __shfl_sync(0xffffffffu, sv[0][j], m);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int i = c0 + lane + 32 * q;
                    if (i >= c0 + m) sv[q][m] = fmaf(-sv[q][j], lmj, sv[q][m]);
                }
            }
        }
        if (bad) break;
        // (3) write the panel back
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int i = c0 + lane + 32 * q;
            if (!rv[q]) continue;
#pragma unroll
            for (int c = 0; c < CW_P; ++c)
                if (c < nc && c0 + c <= i) Ls[roff[q] + c0 + c] = sv[q][c];
        }
        __syncwarp();
    }
    if (bad) {
        if (lane == 0) {
            if (info) info[s] = bad;
            if (nbad) atomicAdd(nbad, 1);
        }
        return;
    }

    // ---- back substitution x = L^-T y, y = row f
    const float *y = Ls + crow_off(f);
    for (int p = TB - 1; p >= 0; --p) {
        const int c0 = CW_P * p;
        const int nc = min(CW_P, f - c0);
        float t[CW_P];
#pragma unroll
        for (int c = 0; c < CW_P; ++c) t[c] = 0.0f;
        for (int k = c0 + CW_P + lane; k < f; k += 32) {
            const float xk = xs[k];
            const float4 l0 = *reinterpret_cast<const float4 *>(Ls + crow_off(k) + c0);
            const float4 l1 = *reinterpret_cast<const float4 *>(Ls + crow_off(k) + c0 + 4);
            t[0] = fmaf(l0.x, xk, t[0]);
            t[1] = fmaf(l0.y, xk, t[1]);
            t[2] = fmaf(l0.z, xk, t[2]);
            t[3] = fmaf(l0.w, xk, t[3]);
            t[4] = fmaf(l1.x, xk, t[4]);
            t[5] = fmaf(l1.y, xk, t[5]);
            t[6] = fmaf(l1.z, xk, t[6]);
            t[7] = fmaf(l1.w, xk, t[7]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int c = 0; c < CW_P; ++c) t[c] += __shfl_xor_sync(0xffffffffu, t[c], o);
        float xv[CW_P];
#pragma unroll
        for (int j = CW_P - 1; j >= 0; --j) {
            if (j >= nc) {
                xv[j] = 0.0f;
                continue;
            }
            float v = y[c0 + j] - t[j];
#pragma unroll
            for (int m = j + 1; m < CW_P; ++m)
                if (m < nc) v = fmaf(-Ls[crow_off(c0 + m) + c0 + j], xv[m], v);
            xv[j] = v / Ls[crow_off(c0 + j) + c0 + j];
        }
        if (lane < nc) {
#pragma unroll
            for (int c = 0; c < CW_P; ++c)
                if (c == lane) xs[c0 + c] = xv[c];
        }
        __syncwarp();
    }
    for (int k = lane; k < f; k += 32) X[s * f + k] = xs[k];
    if (lane == 0 && info) info[s] = 0;
}

int chol_warp_launch(const float *a, int64_t a_stride, const float *b, const int64_t *nu, int64_t nsys, int f,
                     float *x, int32_t *info, int32_t *nbad, cudaStream_t st) {
    if (nsys == 0) return CMF_OK;
    if (f > 124) return set_error(CMF_EINVAL, "warp Cholesky supports f <= 124 (got %d)", f);
    const int a_ = (f + 1) >> 2, b_ = (f + 1) & 3;
    const size_t rows = 4 * ((f + 1) + 2 * a_ * (a_ - 1) + a_ * b_);  // crow_off(f + 1)
    const size_t smem = (rows + 128) * sizeof(float);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(chol_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return set_error(CMF_ECUDA, "chol_warp smem attr: %s", cudaGetErrorString(e));
    }
    chol_warp_kernel<<<static_cast<unsigned>(nsys), 32, smem, st>>>(a, a_stride, b, nu, nsys, f, x, info, nbad);
    return check_launch("chol_warp_kernel");
}

}  // namespace cmf
