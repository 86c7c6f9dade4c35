// Implicit-feedback side kernels (implicit.py:57-131):
//   dense_gram:   F^T F of a factor matrix (precompute_gram, implicit.py:57-60),
//                 fp32 or fp64 accumulation, packed lower triangle out.  Per-block
//                 partial Grams over row chunks (4x4 register tiles of the
//                 triangle, rows staged in shared memory), then an in-order sum
//                 over the partials: deterministic.
//   implicit_loss: sum_{r_uv > 0} c (1 - pred)^2 - pred^2, c = 1 + alpha r, in
//                 float64 over a CSR view (the data term of implicit_objective,
//                 implicit.py:87-104; the dense part is <X^T X, Theta^T Theta>).
//   mpr:          mean percentile rank numerators (implicit.py:115-131): for
//                 each held-out positive (u, v), 2 #{items scoring above v} +
//                 #{items tying with v} - 1, summed as an exact int64.  Scores
//                 are float32 x_u . theta_i (sequential FMA over features, the
//                 same chain for the positive's own score, so ties are exact);
//                 a CTA scores a tile of 32 users against 128-item tiles
//                 (4 users x 4 items per lane, operands in shared memory) and
//                 each warp counts its users' positives with a warp reduction.
#include "common.cuh"

namespace cmf {

namespace ie {

constexpr int GT = 256;       // dense_gram threads
constexpr int GROWS = 64;     // rows staged per step
constexpr int GMAXF = 128;    // f <= 128

template <typename T>
__global__ void __launch_bounds__(GT) gram_partial_kernel(const float *F, int64_t rows, int f, int64_t rows_per_block,
                                                          T *partial) {
    __shared__ float fs[GROWS][GMAXF + 4];
    const int fp = (f + 3) & ~3, TB = fp / 4, ntile = TB * (TB + 1) / 2;
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * rows_per_block;
    const int64_t r1 = min(rows, r0 + rows_per_block);
    // this thread's 4x4 tiles (I, J <= I) of the lower triangle: t = tid, tid + GT
    T acc[2][16];
    int ti[2], tj[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int t = threadIdx.x + q * GT;
        int I = 0, rem = t;
        while (I < TB && rem > I) {
            rem -= I + 1;
            ++I;
        }
        ti[q] = t < ntile ? I : -1;
        tj[q] = rem;
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[q][e] = T(0);
    }
    for (int64_t base = r0; base < r1; base += GROWS) {
        const int nr = static_cast<int>(min(static_cast<int64_t>(GROWS), r1 - base));
        __syncthreads();
        for (int k = threadIdx.x; k < GROWS * fp; k += GT) {
            const int r = k / fp, c = k % fp;
            fs[r][c] = (r < nr && c < f) ? F[(base + r) * f + c] : 0.0f;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            if (ti[q] < 0) continue;
            for (int r = 0; r < nr; ++r) {
                const float4 a = *reinterpret_cast<const float4 *>(&fs[r][4 * ti[q]]);
                const float4 b = *reinterpret_cast<const float4 *>(&fs[r][4 * tj[q]]);
                const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                for (int x = 0; x < 4; ++x)
#pragma unroll
                    for (int y = 0; y < 4; ++y) acc[q][4 * x + y] = fma(T(av[x]), T(bv[y]), acc[q][4 * x + y]);
            }
        }
    }
    const int64_t P = static_cast<int64_t>(f) * (f + 1) / 2;
    T *out = partial + static_cast<int64_t>(blockIdx.x) * P;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        if (ti[q] < 0) continue;
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) {
                const int i = 4 * ti[q] + x, j = 4 * tj[q] + y;
                if (i < f && j <= i) out[static_cast<int64_t>(i) * (i + 1) / 2 + j] = acc[q][4 * x + y];
            }
    }
}

// out[e] = sum_b partial[b][e] in block order (float64 running sum), as T_out
template <typename T, typename TO>
__global__ void gram_reduce_kernel(const T *partial, int nb, int64_t P, TO *out) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < P;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < nb; ++b) s += static_cast<double>(partial[static_cast<int64_t>(b) * P + e]);
        out[e] = static_cast<TO>(s);
    }
}

constexpr int kRedBlocks = 592;

__global__ void implicit_loss_kernel(const int64_t *indptr, const int32_t *indices, const float *vals, int64_t nrows,
                                     const float *x, const float *theta, int f, double alpha, double *out) {
    double acc = 0.0;
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t u = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < nrows; u += warps) {
        const float *xu = x + u * f;
        for (int64_t p = indptr[u] + lane; p < indptr[u + 1]; p += 32) {
            const float *tv = theta + static_cast<int64_t>(indices[p]) * f;
            double pred = 0.0;
            for (int c = 0; c < f; ++c) pred = fma(static_cast<double>(xu[c]), static_cast<double>(tv[c]), pred);
            const double cw = 1.0 + alpha * static_cast<double>(vals[p]);
            const double d = 1.0 - pred;
            acc += cw * d * d - pred * pred;
        }
    }
    __shared__ double red[32];
    acc = warp_sum(acc);
    if (lane == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += red[w];
        out[1 + blockIdx.x] = s;
    }
}

__global__ void finish_kernel(double *out, int n) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += out[1 + i];
        out[0] = s;
    }
}

// ---------------------------------------------------------------- MPR
constexpr int UT = 32;     // users per CTA tile (8 warps x 4)
constexpr int IT = 128;    // items per tile (32 lanes x 4, item = lane + 32 j)
constexpr int PMAX = 1024; // positives per pass
constexpr int MT = 256;

// f-stride of the shared tiles: >= roundup4(f), == 4 (mod 32) (conflict-free float4 rows across lanes)
__host__ __device__ inline int mpr_stride(int f) {
    const int fp = (f + 3) & ~3;
    return fp + ((4 - fp) % 32 + 32) % 32;
}

__device__ __forceinline__ float score(const float *a, const float *b, int f) {
    float acc = 0.0f;
    for (int k = 0; k < f; ++k) acc = fmaf(a[k], b[k], acc);
    return acc;
}

__global__ void __launch_bounds__(MT) mpr_kernel(const int64_t *pos_ptr, const int32_t *pos_item, int64_t m,
                                                 const float *x, const float *theta, int64_t n, int f,
                                                 unsigned long long *out) {
    extern __shared__ __align__(16) float msm[];
    const int S = mpr_stride(f);
    float *xs = msm;                // UT x S
    float *ts = xs + UT * S;        // IT x S
    float *psc = ts + IT * S;       // PMAX positive scores
    int *pcnt = reinterpret_cast<int *>(psc + PMAX);  // PMAX counts
    __shared__ int64_t pbeg[UT + 1];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    unsigned long long total = 0;
    for (int64_t u0 = static_cast<int64_t>(blockIdx.x) * UT; u0 < m; u0 += static_cast<int64_t>(gridDim.x) * UT) {
        const int nu = static_cast<int>(min(static_cast<int64_t>(UT), m - u0));
        __syncthreads();
        if (tid <= UT) pbeg[tid] = pos_ptr[u0 + min(tid, nu)];
        for (int k = tid; k < UT * S; k += MT) {
            const int r = k / S, c = k % S;
            xs[k] = (r < nu && c < f) ? x[(u0 + r) * f + c] : 0.0f;
        }
        __syncthreads();
        const int64_t P0 = pbeg[0], P1 = pbeg[UT];
        if (P1 == P0) continue;
        for (int64_t c0 = P0; c0 < P1; c0 += PMAX) {  // positives of this user tile, PMAX at a time
            const int np = static_cast<int>(min(static_cast<int64_t>(PMAX), P1 - c0));
            __syncthreads();
            for (int p = tid; p < np; p += MT) {
                // owner user of positive c0 + p
                int r = 0;
                while (pbeg[r + 1] <= c0 + p) ++r;
                psc[p] = score(xs + r * S, theta + static_cast<int64_t>(pos_item[c0 + p]) * f, f);
                pcnt[p] = 0;
            }
            for (int64_t i0 = 0; i0 < n; i0 += IT) {
                const int ni = static_cast<int>(min(static_cast<int64_t>(IT), n - i0));
                __syncthreads();
                for (int k = tid; k < IT * S; k += MT) {
                    const int r = k / S, c = k % S;
                    ts[k] = (r < ni && c < f) ? theta[(i0 + r) * f + c] : 0.0f;
                }
                __syncthreads();
                // 4 users (4w .. 4w+3) x 4 items (lane + 32 j): sequential FMA over features
                float s[4][4];
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int j = 0; j < 4; ++j) s[a][j] = 0.0f;
                for (int k = 0; k < f; k += 4) {
                    float4 xv[4], tv[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) xv[a] = *reinterpret_cast<const float4 *>(xs + (4 * w + a) * S + k);
#pragma unroll
                    for (int j = 0; j < 4; ++j) tv[j] = *reinterpret_cast<const float4 *>(ts + (lane + 32 * j) * S + k);
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            s[a][j] = fmaf(xv[a].x, tv[j].x, s[a][j]);
                            if (k + 1 < f) s[a][j] = fmaf(xv[a].y, tv[j].y, s[a][j]);
                            if (k + 2 < f) s[a][j] = fmaf(xv[a].z, tv[j].z, s[a][j]);
                            if (k + 3 < f) s[a][j] = fmaf(xv[a].w, tv[j].w, s[a][j]);
                        }
                }
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const int r = 4 * w + a;
                    if (r >= nu) break;
                    const int64_t pb = max(pbeg[r], c0), pe = min(pbeg[r + 1], c0 + np);
                    for (int64_t p = pb; p < pe; ++p) {
                        const float sp = psc[p - c0];
                        int cnt = 0;
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            if (lane + 32 * j < ni) cnt += (s[a][j] > sp ? 2 : 0) + (s[a][j] == sp ? 1 : 0);
                        cnt = __reduce_add_sync(0xffffffffu, cnt);
                        if (lane == 0) pcnt[p - c0] += cnt;  // this warp owns user r's positives
                    }
                }
            }
            __syncthreads();
            for (int p = tid; p < np; p += MT) total += static_cast<unsigned long long>(pcnt[p] - 1);  // minus itself
        }
    }
    total = warp_sum(total);
    if (lane == 0 && total) atomicAdd(out, total);
}

}  // namespace ie

int64_t dense_gram_workspace_bytes(int64_t rows, int f, bool fp64) {
    (void)rows;
    return static_cast<int64_t>(4 * 148) * (static_cast<int64_t>(f) * (f + 1) / 2) * (fp64 ? 8 : 4);
}

int dense_gram_launch(const float *F, int64_t rows, int f, bool fp64, void *out, void *ws, int64_t ws_bytes,
                      cudaStream_t st) {
    if (f > ie::GMAXF) return set_error(CMF_EINVAL, "dense_gram supports f <= %d", ie::GMAXF);
    const int fp = (f + 3) & ~3, TB = fp / 4;
    if (TB * (TB + 1) / 2 > 2 * ie::GT) return set_error(CMF_EINVAL, "dense_gram tile plan");
    int64_t nb = 4 * 148;
    if (nb * ie::GROWS > rows) nb = (rows + ie::GROWS - 1) / ie::GROWS;
    if (nb < 1) nb = 1;
    const int64_t rpb = (rows + nb - 1) / nb;
    const int64_t P = static_cast<int64_t>(f) * (f + 1) / 2;
    if (ws_bytes < nb * P * (fp64 ? 8 : 4)) return set_error(CMF_EINVAL, "dense_gram workspace too small");
    const unsigned rb = static_cast<unsigned>((P + 255) / 256);
    if (fp64) {
        ie::gram_partial_kernel<double><<<static_cast<unsigned>(nb), ie::GT, 0, st>>>(F, rows, f, rpb,
                                                                                     static_cast<double *>(ws));
        ie::gram_reduce_kernel<double, double><<<rb, 256, 0, st>>>(static_cast<double *>(ws), static_cast<int>(nb), P,
                                                                   static_cast<double *>(out));
    } else {
        ie::gram_partial_kernel<float><<<static_cast<unsigned>(nb), ie::GT, 0, st>>>(F, rows, f, rpb,
                                                                                   static_cast<float *>(ws));
        ie::gram_reduce_kernel<float, float><<<rb, 256, 0, st>>>(static_cast<float *>(ws), static_cast<int>(nb), P,
                                                                 static_cast<float *>(out));
    }
    return check_launch("dense_gram");
}

int implicit_loss_launch(const int64_t *indptr, const int32_t *indices, const float *vals, int64_t nrows,
                         const float *x, const float *theta, int f, double alpha, double *out, cudaStream_t st) {
    ie::implicit_loss_kernel<<<ie::kRedBlocks, 256, 0, st>>>(indptr, indices, vals, nrows, x, theta, f, alpha, out);
    ie::finish_kernel<<<1, 32, 0, st>>>(out, ie::kRedBlocks);
    return check_launch("implicit_loss");
}

int mpr_launch(const int64_t *pos_ptr, const int32_t *pos_item, int64_t m, const float *x, const float *theta,
               int64_t n, int f, unsigned long long *out, cudaStream_t st) {
    const int S = ie::mpr_stride(f);
    const size_t smem = static_cast<size_t>((ie::UT + ie::IT) * S + ie::PMAX) * 4 + ie::PMAX * 4;
    cudaError_t e = cudaFuncSetAttribute(ie::mpr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return set_error(CMF_ECUDA, "mpr smem attr: %s", cudaGetErrorString(e));
    int64_t grid = (m + ie::UT - 1) / ie::UT;
    if (grid > 148 * 4) grid = 148 * 4;
    if (grid < 1) grid = 1;
    e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return set_error(CMF_ECUDA, "mpr: %s", cudaGetErrorString(e));
    ie::mpr_kernel<<<static_cast<unsigned>(grid), ie::MT, smem, st>>>(pos_ptr, pos_item, m, x, theta, n, f, out);
    return check_launch("mpr_kernel");
}

}  // namespace cmf
