// K4, shared-memory tile variant: batched Cholesky + solve (fp32, f <= 128).
//
// Replaces solvers.exact_solve / the exact branch of batch_solve
// (solvers.py:148-164, :221-237; LAPACK dpotrf + dpotrs in the reference).
// One 128-thread CTA per system.  The register-tiled kernel (chol_tiled.cu)
// keeps 3 fixed tiles per thread and executes every tile's update code each
// panel, active or not; here the lower triangle lives in shared memory as 4x4
// tiles numbered column-major (tile (I, J), I >= J, at cs(J) + I - J), so the
// tiles still active after panel p are exactly the suffix [cs(p+1), T) and the
// threads stride over that suffix with no idle work:
//   TRSM:   rows of panel p below the diagonal, L_Ip = A_Ip L_pp^-T (one row
//           per thread), and the forward-substitution block y_p = L_pp^-1 z_p
//   update: A_IJ -= L_Ip L_Jp^T over the active tiles (rows of L_Ip, columns
//           of L_Jp from a transposed copy of the panel so that FFMA2 pairs
//           come straight from float4 loads: 12 LDS.128, 32 FFMA2, 4 STS.128
//           per tile), z_I -= L_Ip y_p, and the owner of the next
//           diagonal tile factorises it right after updating it (look-ahead).
// Two barriers per 4-column panel.  The backward solve L^T x = y runs on warp
// 0 (lanes own rows l + 32q, shuffles, no block barriers).  Padding rows
// (i >= f) are the identity.  A non-positive pivot marks the system singular
// (info = column + 1, LAPACK convention) and nothing is written for it.
#include "common.cuh"

namespace cmf {

namespace {

__device__ __forceinline__ int col_start(int J, int TR) { return J * TR - J * (J - 1) / 2; }

// 4x4 Cholesky of a tile whose rows are tl[0], tl[T], tl[2T], tl[3T], in
// place; reciprocal pivots to rd[0..3]; returns 0 or the failing column + 1
__device__ __forceinline__ int factor_tile(float4 *tl, int T, float *rd) {
    float l[4][4];
#pragma unroll
    for (int x = 0; x < 4; ++x) {
        const float4 v = tl[x * T];
        l[x][0] = v.x;
        l[x][1] = v.y;
        l[x][2] = v.z;
        l[x][3] = v.w;
    }
    int fail = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const float d0 = l[c][c];
        if (!(d0 > 0.0f) && !fail) fail = c + 1;
        const float dd = fmaxf(d0, 1e-30f);
        const float r = rsqrtf(dd);  // 1/sqrt(d); sqrt(d) = d * r
        l[c][c] = dd * r;
        rd[c] = r;
#pragma unroll
        for (int x = c + 1; x < 4; ++x) l[x][c] *= r;
#pragma unroll
        for (int x = c + 1; x < 4; ++x)
#pragma unroll
            for (int y = c + 1; y <= x; ++y) l[x][y] = fmaf(-l[x][c], l[y][c], l[x][y]);
    }
#pragma unroll
    for (int x = 0; x < 4; ++x)
        tl[x * T] = make_float4(l[x][0], x >= 1 ? l[x][1] : 0.0f, x >= 2 ? l[x][2] : 0.0f, x >= 3 ? l[x][3] : 0.0f);
    return fail;
}

}  // namespace

#ifndef CMF_CHOL_NT
#define CMF_CHOL_NT 128
#endif
__global__ void __launch_bounds__(CMF_CHOL_NT, 1024 / CMF_CHOL_NT) chol_smem_kernel(const float *A, int64_t a_stride, const float *B,
                                                          const int64_t *nu, int64_t nsys, int f, float *X,
                                                          int32_t *info, int32_t *nbad) {
    extern __shared__ __align__(16) float csm[];
    const int64_t s = blockIdx.x;
    if (nu && nu[s] == 0) return;
    constexpr int NT = CMF_CHOL_NT;
    const int tid = threadIdx.x;
    const int fp = (f + 3) & ~3, TR = fp >> 2, T = TR * (TR + 1) / 2;
    // shared: tiles | z / y (fp) | 1/L_ii (fp) | panel^T (4 fp) | tile rows I, cols J | flag.
    // Row x of tile t is the float4 tiles[x * T + t]: threads working on
    // consecutive tiles touch consecutive float4s (no bank conflicts).
    float4 *tiles = reinterpret_cast<float4 *>(csm);
    float *zy = csm + 16 * T;
    float *rdiag = zy + fp;
    float *pt = rdiag + fp;  // panel p transposed: pt[c * fp + r] = L[r][4p + c]
    unsigned char *tI = reinterpret_cast<unsigned char *>(pt + 4 * fp);
    const int T4 = (T + 3) & ~3;
    unsigned char *tJ = tI + T4;
    int *flag = reinterpret_cast<int *>(tJ + T4);

    // zero the tiles, identity on the padding diagonal, the tile map
    for (int k = tid; k < 4 * T; k += NT) tiles[k] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    for (int t = tid; t < T; t += NT) {
        int J = 0, rem = t;
        while (rem >= TR - J) {
            rem -= TR - J;
            ++J;
        }
        tI[t] = static_cast<unsigned char>(J + rem);
        tJ[t] = static_cast<unsigned char>(J);
    }
    for (int k = tid; k < fp; k += NT) zy[k] = k < f ? B[s * f + k] : 0.0f;
    if (tid == 0) *flag = 0;
    __syncthreads();
    if (tid < fp - f) {
        const int i = f + tid;
        csm[4 * ((i & 3) * T + col_start(i >> 2, TR)) + (i & 3)] = 1.0f;
    }
    // scatter the packed lower triangle (row-major, k = i(i+1)/2 + j), 14 loads
    // in flight per thread; row of k from an approximate square root + fix-up
    {
        const float *src = A + s * a_stride;
        const int P = static_cast<int>(packed_size(f));
        for (int k0 = tid; k0 < P; k0 += 14 * NT) {
            float v[14];
            int off[14];
#pragma unroll
            for (int u = 0; u < 14; ++u) {
                const int k = k0 + u * NT;
                off[u] = -1;
                if (k < P) {
                    const float q = 8.0f * static_cast<float>(k) + 1.0f;
                    int i = static_cast<int>((q * rsqrtf(q) - 1.0f) * 0.5f);
                    if ((i + 1) * (i + 2) / 2 <= k) ++i;
                    if (i * (i + 1) / 2 > k) --i;
                    const int j = k - i * (i + 1) / 2;
                    v[u] = __ldg(src + k);
                    off[u] = 4 * ((i & 3) * T + col_start(j >> 2, TR) + (i >> 2) - (j >> 2)) + (j & 3);
                }
            }
#pragma unroll
            for (int u = 0; u < 14; ++u)
                if (off[u] >= 0) csm[off[u]] = v[u];
        }
    }
    __syncthreads();
    if (tid == 0) {
        const int fail = factor_tile(tiles, T, rdiag);
        if (fail) *flag = fail;
    }
    __syncthreads();

    int bad = 0;
    for (int p = 0; p < TR; ++p) {
        if (*flag) {
            bad = *flag;
            break;
        }
        const int cp = col_start(p, TR);
        const float4 *Lpp = tiles + cp;  // rows Lpp[x * T]
        // (1) panel TRSM, one row per thread; thread NT-1 solves the rhs block y_p
        for (int r = 4 * p + 4 + tid; r < fp; r += NT) {
            float4 *row = tiles + (r & 3) * T + cp + (r >> 2) - p;
            const float4 a = *row;
            const float4 l1 = Lpp[T], l2 = Lpp[2 * T], l3 = Lpp[3 * T];
            const float y0 = a.x * rdiag[4 * p];
            const float y1 = fmaf(-y0, l1.x, a.y) * rdiag[4 * p + 1];
            const float y2 = fmaf(-y1, l2.y, fmaf(-y0, l2.x, a.z)) * rdiag[4 * p + 2];
            const float y3 = fmaf(-y2, l3.z, fmaf(-y1, l3.y, fmaf(-y0, l3.x, a.w))) * rdiag[4 * p + 3];
            *row = make_float4(y0, y1, y2, y3);
            pt[r] = y0;
            pt[fp + r] = y1;
            pt[2 * fp + r] = y2;
            pt[3 * fp + r] = y3;
        }
        if (tid == NT - 1) {
            const float4 l1 = Lpp[T], l2 = Lpp[2 * T], l3 = Lpp[3 * T];
            float *z = zy + 4 * p;
            const float y0 = z[0] * rdiag[4 * p];
            const float y1 = fmaf(-y0, l1.x, z[1]) * rdiag[4 * p + 1];
            const float y2 = fmaf(-y1, l2.y, fmaf(-y0, l2.x, z[2])) * rdiag[4 * p + 2];
            const float y3 = fmaf(-y2, l3.z, fmaf(-y1, l3.y, fmaf(-y0, l3.x, z[3]))) * rdiag[4 * p + 3];
            z[0] = y0;
            z[1] = y1;
            z[2] = y2;
            z[3] = y3;
        }
        __syncthreads();
        if (p + 1 == TR) break;
        // (2) trailing update over the active suffix; z_I -= L_Ip y_p
        // thread 0 takes only the next diagonal tile (it factorises it right
        // after the update); threads 1..NT-1 share the rest
        const int start = col_start(p + 1, TR);
        const int tstep = tid == 0 ? T : NT - 1;
        for (int t = start + tid; t < T; t += tstep) {
            const int I = tI[t], J = tJ[t];
            const float4 *LI = tiles + cp + I - p;
            // columns c of L_Jp (rows 4J..4J+3) from the transposed panel
            float4 lj[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) lj[c] = *reinterpret_cast<const float4 *>(pt + c * fp + 4 * J);
            float4 *at = tiles + t;
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                const float4 li = LI[x * T];
                const float4 a = at[x * T];
                float2 a01 = make_float2(a.x, a.y), a23 = make_float2(a.z, a.w);
                const float lic[4] = {li.x, li.y, li.z, li.w};
#pragma unroll
                for (int c = 0; c < 4; ++c) {  // a[x][y] -= L[4I+x][c] * L[4J+y][c]
                    const float2 m = make_float2(-lic[c], -lic[c]);
                    a01 = __ffma2_rn(m, make_float2(lj[c].x, lj[c].y), a01);
                    a23 = __ffma2_rn(m, make_float2(lj[c].z, lj[c].w), a23);
                }
                at[x * T] = make_float4(a01.x, a01.y, a23.x, a23.y);
            }
            if (t == start) {  // tile (p+1, p+1): factorise now (look-ahead)
                const int fail = factor_tile(at, T, rdiag + 4 * (p + 1));
                if (fail) *flag = 4 * (p + 1) + fail;
            }
        }
        for (int r = 4 * p + 4 + tid; r < fp; r += NT) {
            const float4 l = tiles[(r & 3) * T + cp + (r >> 2) - p];
            const float *y = zy + 4 * p;
            zy[r] = fmaf(-l.w, y[3], fmaf(-l.z, y[2], fmaf(-l.y, y[1], fmaf(-l.x, y[0], zy[r]))));
        }
        __syncthreads();
    }
    if (bad) {
        if (tid == 0) {
            if (info) info[s] = bad;
            if (nbad) atomicAdd(nbad, 1);
        }
        return;
    }
    if (tid >= 32) return;
    // backward solve L^T x = y on warp 0: lane l owns rows l + 32q
    const int lane = tid;
    float xv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) xv[q] = (lane + 32 * q < fp) ? zy[lane + 32 * q] : 0.0f;
    for (int p = TR - 1; p >= 0; --p) {
        // x_p = L_pp^-T z_p, every lane redundantly
        float zp[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int r = 4 * p + c;
            const int q = r >> 5;
            const float mine = q == 0 ? xv[0] : q == 1 ? xv[1] : q == 2 ? xv[2] : xv[3];
            zp[c] = __shfl_sync(0xffffffffu, mine, r & 31);
        }
        const float4 *Lpp = tiles + col_start(p, TR);
        const float4 l1 = Lpp[T], l2 = Lpp[2 * T], l3 = Lpp[3 * T];
        const float x3 = zp[3] * rdiag[4 * p + 3];
        const float x2 = fmaf(-l3.z, x3, zp[2]) * rdiag[4 * p + 2];
        const float x1 = fmaf(-l3.y, x3, fmaf(-l2.y, x2, zp[1])) * rdiag[4 * p + 1];
        const float x0 = fmaf(-l3.x, x3, fmaf(-l2.x, x2, fmaf(-l1.x, x1, zp[0]))) * rdiag[4 * p];
        // rows of block p take the solution; rows k < 4p: z_k -= sum_x L[4p+x][k] x_x
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int k = lane + 32 * q;
            if ((k >> 2) == p) {
                const int c = k & 3;
                xv[q] = c == 0 ? x0 : c == 1 ? x1 : c == 2 ? x2 : x3;
            } else if (k < 4 * p) {
                const float *tp = csm + 4 * (col_start(k >> 2, TR) + p - (k >> 2)) + (k & 3);  // row x at tp[4xT]
                xv[q] = fmaf(-tp[12 * T], x3, fmaf(-tp[8 * T], x2, fmaf(-tp[4 * T], x1, fmaf(-tp[0], x0, xv[q]))));
            }
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
        if (lane + 32 * q < f) X[s * f + lane + 32 * q] = xv[q];
    if (lane == 0 && info) info[s] = 0;
}

int chol_smem_launch(const float *a, int64_t a_stride, const float *b, const int64_t *nu, int64_t nsys, int f,
                     float *x, int32_t *info, int32_t *nbad, cudaStream_t st) {
    if (nsys == 0) return CMF_OK;
    if (f > 128) return set_error(CMF_EINVAL, "f=%d too large for the tile Cholesky", f);
    const int fp = (f + 3) & ~3, TR = fp / 4, T = TR * (TR + 1) / 2;
    const size_t smem = static_cast<size_t>(16 * T + 6 * fp) * sizeof(float) + 2 * ((T + 3) & ~3) + 16;
    if (smem > 48 * 1024) {
        cudaError_t e =
            cudaFuncSetAttribute(chol_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return set_error(CMF_ECUDA, "chol_smem smem attr: %s", cudaGetErrorString(e));
    }
    chol_smem_kernel<<<static_cast<unsigned>(nsys), CMF_CHOL_NT, smem, st>>>(a, a_stride, b, nu, nsys, f, x, info, nbad);
    return check_launch("chol_smem_kernel");
}

}  // namespace cmf
