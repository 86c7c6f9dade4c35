// K4 fast path: register-tiled batched Cholesky (fp32, f <= 128).
//
// Replaces solvers.exact_solve / the exact branch of batch_solve
// (solvers.py:148-164, :221-237; LAPACK dpotrf + dpotrs in the reference) for
// the production exact route.  One CTA per system.  The packed lower
// triangle is split into the same 4x4 register tiles as the SIMT Gram kernel
// (gram_simt.cu), TPT tiles per thread, and factorised right-looking one
// 4-column panel at a time:
//   (1) the owner of diagonal tile (p,p) factorises it in registers and
//       publishes L_pp (+ reciprocal diagonal) to shared memory;
//   (2) the panel TRSM L_ip = A_ip L_pp^-T runs row-parallel over all threads
//       from the raw panel the tile owners published (full SIMT efficiency);
//   (3) every thread applies A_ij -= L_ip L_jp^T to its trailing tiles
//       (32 FFMA2 per tile from two 16-float panel reads), and the owners of
//       the next column block publish its raw values.
// Two barriers per panel (50 for f=100) instead of three per column, and the
// next diagonal block is factorised by its owner as soon as its own update is
// done (look-ahead).  Padding rows (i >= f) are the identity, so they never
// touch real rows.  A non-positive pivot marks the system singular
// (info = column+1, LAPACK convention) and it is not written.  Forward/back
// substitution runs on warp 0 in 4-row blocks (shuffles, no block barriers).
#include "common.cuh"

namespace cmf {

__device__ __forceinline__ int tri_row_unused(int t) {
    int r = static_cast<int>((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
    while ((r + 1) * (r + 2) / 2 <= t) ++r;
    while (r * (r + 1) / 2 > t) --r;
    return r;
}

template <int TPT>
__global__ void __launch_bounds__(128, 7) chol_tiled_kernel(const float *A, int64_t a_stride, const float *B,
                                                         const int64_t *nu, int64_t nsys, int f, float *X,
                                                         int32_t *info, int32_t *nbad) {
    extern __shared__ __align__(16) float csm[];
    const int64_t s = blockIdx.x;
    if (nu && nu[s] == 0) return;
    const int tid = threadIdx.x, NT = blockDim.x;
    const int fp = (f + 3) & ~3, TR = fp >> 2, T = TR * (TR + 1) / 2;
    const int64_t P = packed_size(f);
    // shared: packed A / L (P floats, rounded to 4) | panel x2 (4*fp each, column-major) |
    //         diag block (16) + recip (4) | flag
    float *Ls = csm;
    const int Pr = static_cast<int>((P + 3) & ~3ll);
    float *panel = Ls + Pr;
    float *dblk = panel + 2 * 4 * fp;
    float *rdiag = dblk + 20;  // 1 / L_ii, for the substitution
    int *flag = reinterpret_cast<int *>(rdiag + fp);

    // stage the packed system with async copies (all loads in flight at once)
    const float *src = A + static_cast<size_t>(s) * a_stride;
    if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        const int64_t n16 = P >> 2;
        for (int64_t k = tid; k < n16; k += NT) cp_async16(Ls + 4 * k, src + 4 * k);
        for (int64_t k = 4 * n16 + tid; k < P; k += NT) cp_async4(Ls + k, src + k, 4);
    } else {
        for (int64_t k = tid; k < P; k += NT) cp_async4(Ls + k, src + k, 4);
    }
    cp_async_commit();
    if (tid == 0) *flag = 0;
    cp_async_wait<0>();
    __syncthreads();

    int ti[TPT], tj[TPT];
    bool valid[TPT];
    float a[TPT][4][4];
    // Tiles are numbered column-major (by tj, then ti) and dealt round-robin:
    // the tiles still active at panel p (tj > p) are then a contiguous suffix
    // of the numbering, so whole warps drop out as the trailing matrix
    // shrinks instead of every warp carrying a few active lanes.
#pragma unroll
    for (int q = 0; q < TPT; ++q) {
        const int t = tid + q * NT;
        valid[q] = t < T;
        int c = 0, rem = valid[q] ? t : 0;
        while (rem >= TR - c) {
            rem -= TR - c;
            ++c;
        }
        tj[q] = c;
        ti[q] = c + rem;
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) {
                const int i = 4 * ti[q] + x, j = 4 * tj[q] + y;
                float v = 0.0f;
                if (valid[q] && j <= i) v = (i < f) ? Ls[i * (i + 1) / 2 + j] : (i == j ? 1.0f : 0.0f);
                a[q][x][y] = v;
            }
    }

    // (1) for panel p is done by the owner of tile (p,p) right after it applied
    // panel p-1's update to that tile (look-ahead), so the serial 4x4
    // factorisation overlaps the other threads' trailing updates.
    auto factor_diag = [&](int q, int p) {
        float l[4][4];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) l[x][y] = a[q][x][y];
        int fail = 0;
        float *pan = panel + (p & 1) * 4 * fp;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const float d0 = l[c][c];
            if (!(d0 > 0.0f) && !fail) fail = 4 * p + c + 1;
            // one MUFU.RSQ gives both 1/sqrt(d) and sqrt(d) = d / sqrt(d) (serial chain)
            const float dd = fmaxf(d0, 1e-30f);
            const float rd = rsqrtf(dd);
            l[c][c] = dd * rd;
#pragma unroll
            for (int r = c + 1; r < 4; ++r) l[r][c] *= rd;
#pragma unroll
            for (int r = c + 1; r < 4; ++r)
#pragma unroll
                for (int t2 = c + 1; t2 <= r; ++t2) l[r][t2] = fmaf(-l[r][c], l[t2][c], l[r][t2]);
            dblk[16 + c] = rd;
            rdiag[4 * p + c] = rd;
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) {
                a[q][x][y] = y <= x ? l[x][y] : 0.0f;
                dblk[x * 4 + y] = y <= x ? l[x][y] : 0.0f;
                pan[y * fp + 4 * p + x] = y <= x ? l[x][y] : 0.0f;
            }
        if (fail) *flag = fail;
    };
#pragma unroll
    for (int q = 0; q < TPT; ++q)
        if (valid[q] && ti[q] == 0 && tj[q] == 0) factor_diag(q, 0);
    __syncthreads();

    // raw A values of panel column 0 for the row-parallel TRSM of panel 0
#pragma unroll
    for (int q = 0; q < TPT; ++q)
        if (valid[q] && tj[q] == 0 && ti[q] > 0)
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
                for (int y = 0; y < 4; ++y) panel[y * fp + 4 * ti[q] + x] = a[q][x][y];
    __syncthreads();

    int bad = 0;
    for (int p = 0; p < TR; ++p) {
        float *pan = panel + (p & 1) * 4 * fp;  // column-major: pan[c * fp + row]
        float *nxt = panel + ((p + 1) & 1) * 4 * fp;
        if (*flag) {
            bad = *flag;
            break;
        }
        // (2) panel TRSM, one matrix row per thread: L_r = A_r L_pp^-T for rows
        //     below the diagonal block (raw values were published to `pan`)
        for (int r = 4 * p + 4 + tid; r < fp; r += NT) {
            const float a0 = pan[r], a1 = pan[fp + r], a2 = pan[2 * fp + r], a3 = pan[3 * fp + r];
            const float y0 = a0 * dblk[16];
            const float y1 = fmaf(-y0, dblk[4], a1) * dblk[17];
            const float y2 = fmaf(-y1, dblk[9], fmaf(-y0, dblk[8], a2)) * dblk[18];
            const float y3 = fmaf(-y2, dblk[14], fmaf(-y1, dblk[13], fmaf(-y0, dblk[12], a3))) * dblk[19];
            pan[r] = y0;
            pan[fp + r] = y1;
            pan[2 * fp + r] = y2;
            pan[3 * fp + r] = y3;
        }
        __syncthreads();
        // (3) tiles (i, p): take the finished L_ip back into registers.  Tiles
        //     (i, j), i >= j > p: A_ij -= L_ip L_jp^T (FFMA2).  Tiles of column
        //     block p+1 publish their updated raw values for the next TRSM, and
        //     the owner of (p+1, p+1) factorises it right away (look-ahead).
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
            for (int q = 0; q < TPT; ++q) {
                if (!valid[q]) continue;
                const bool next_diag = ti[q] == p + 1 && tj[q] == p + 1;
                if (pass == 0 && tj[q] == p && ti[q] > p) {
#pragma unroll
                    for (int x = 0; x < 4; ++x)
#pragma unroll
                        for (int y = 0; y < 4; ++y) a[q][x][y] = pan[y * fp + 4 * ti[q] + x];
                }
                if (tj[q] > p && (pass == 0) == next_diag) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const float4 li = *reinterpret_cast<const float4 *>(pan + c * fp + 4 * ti[q]);
                        const float4 lj = *reinterpret_cast<const float4 *>(pan + c * fp + 4 * tj[q]);
                        const float lv[4] = {li.x, li.y, li.z, li.w};
                        const float2 n01 = make_float2(-lj.x, -lj.y), n23 = make_float2(-lj.z, -lj.w);
#pragma unroll
                        for (int x = 0; x < 4; ++x) {
                            float2 r01 = make_float2(a[q][x][0], a[q][x][1]);
                            float2 r23 = make_float2(a[q][x][2], a[q][x][3]);
                            r01 = __ffma2_rn(make_float2(lv[x], lv[x]), n01, r01);
                            r23 = __ffma2_rn(make_float2(lv[x], lv[x]), n23, r23);
                            a[q][x][0] = r01.x;
                            a[q][x][1] = r01.y;
                            a[q][x][2] = r23.x;
                            a[q][x][3] = r23.y;
                        }
                    }
                    if (next_diag) {
                        factor_diag(q, p + 1);
                    } else if (tj[q] == p + 1) {
#pragma unroll
                        for (int x = 0; x < 4; ++x)
#pragma unroll
                            for (int y = 0; y < 4; ++y) nxt[y * fp + 4 * ti[q] + x] = a[q][x][y];
                    }
                }
            }
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
    // publish L (packed) for the substitution
#pragma unroll
    for (int q = 0; q < TPT; ++q) {
        if (!valid[q]) continue;
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            const int i = 4 * ti[q] + x;
            if (i >= f) continue;
#pragma unroll
            for (int y = 0; y < 4; ++y) {
                const int j = 4 * tj[q] + y;
                if (j <= i) Ls[i * (i + 1) / 2 + j] = a[q][x][y];
            }
        }
    }
    __syncthreads();
    if (threadIdx.x >= 32) return;
    // Blocked substitution on warp 0: unknowns in blocks of 4 (the diagonal
    // tiles); lane l owns rows l, l+32, l+64, l+96.  Per block: gather the 4
    // right-hand sides by shuffle, solve the 4x4 triangle redundantly on every
    // lane, update the owned rows with one 4-wide FMA per row.
    const int lane = threadIdx.x;
    float y0 = lane < f ? B[s * f + lane] : 0.0f;
    float y1 = lane + 32 < f ? B[s * f + lane + 32] : 0.0f;
    float y2 = lane + 64 < f ? B[s * f + lane + 64] : 0.0f;
    float y3 = lane + 96 < f ? B[s * f + lane + 96] : 0.0f;
    auto get = [&](int t) {  // value of row t (held by lane t & 31)
        const int q = t >> 5;
        const float v = q == 0 ? y0 : q == 1 ? y1 : q == 2 ? y2 : y3;
        return __shfl_sync(0xffffffffu, v, t & 31);
    };
    auto L = [&](int i, int j) { return (i < f && j <= i) ? Ls[i * (i + 1) / 2 + j] : (i == j ? 1.0f : 0.0f); };
    auto R = [&](int i) { return i < f ? rdiag[i] : 1.0f; };
    for (int p = 0; p < TR; ++p) {  // L y = b
        const int r0 = 4 * p;
        float v0 = get(r0), v1 = get(r0 + 1), v2 = get(r0 + 2), v3 = get(r0 + 3);
        v0 *= R(r0);
        v1 = (v1 - L(r0 + 1, r0) * v0) * R(r0 + 1);
        v2 = (v2 - L(r0 + 2, r0) * v0 - L(r0 + 2, r0 + 1) * v1) * R(r0 + 2);
        v3 = (v3 - L(r0 + 3, r0) * v0 - L(r0 + 3, r0 + 1) * v1 - L(r0 + 3, r0 + 2) * v2) * R(r0 + 3);
        auto upd = [&](float &y, int t) {
            if (t >= r0 && t < r0 + 4) {
                y = t == r0 ? v0 : t == r0 + 1 ? v1 : t == r0 + 2 ? v2 : v3;
            } else if (t >= r0 + 4 && t < f) {
                const float *row = Ls + t * (t + 1) / 2 + r0;
                y = fmaf(-row[0], v0, fmaf(-row[1], v1, fmaf(-row[2], v2, fmaf(-row[3], v3, y))));
            }
        };
        upd(y0, lane);
        upd(y1, lane + 32);
        upd(y2, lane + 64);
        upd(y3, lane + 96);
    }
    for (int p = TR - 1; p >= 0; --p) {  // L^T x = y
        const int r0 = 4 * p;
        float v0 = get(r0), v1 = get(r0 + 1), v2 = get(r0 + 2), v3 = get(r0 + 3);
        v3 *= R(r0 + 3);
        v2 = (v2 - L(r0 + 3, r0 + 2) * v3) * R(r0 + 2);
        v1 = (v1 - L(r0 + 2, r0 + 1) * v2 - L(r0 + 3, r0 + 1) * v3) * R(r0 + 1);
        v0 = (v0 - L(r0 + 1, r0) * v1 - L(r0 + 2, r0) * v2 - L(r0 + 3, r0) * v3) * R(r0);
        auto upd = [&](float &y, int t) {
            if (t >= r0 && t < r0 + 4) {
                y = t == r0 ? v0 : t == r0 + 1 ? v1 : t == r0 + 2 ? v2 : v3;
            } else if (t < r0) {
                y = fmaf(-L(r0, t), v0, fmaf(-L(r0 + 1, t), v1, fmaf(-L(r0 + 2, t), v2, fmaf(-L(r0 + 3, t), v3, y))));
            }
        };
        upd(y0, lane);
        upd(y1, lane + 32);
        upd(y2, lane + 64);
        upd(y3, lane + 96);
    }
    if (lane < f) X[s * f + lane] = y0;
    if (lane + 32 < f) X[s * f + lane + 32] = y1;
    if (lane + 64 < f) X[s * f + lane + 64] = y2;
    if (lane + 96 < f) X[s * f + lane + 96] = y3;
    if (lane == 0 && info) info[s] = 0;
}

template <int TPT>
static int launch_chol_tiled(const float *a, int64_t a_stride, const float *b, const int64_t *nu, int64_t nsys,
                             int f, float *x, int32_t *info, int32_t *nbad, cudaStream_t st) {
    const int fp = (f + 3) & ~3;
    const int64_t P = packed_size(f);
    const size_t smem = (((P + 3) & ~3ll) + 2 * 4 * fp + 20 + fp + 4) * sizeof(float) + 16;
    auto k = chol_tiled_kernel<TPT>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return set_error(CMF_ECUDA, "chol_tiled smem attr: %s", cudaGetErrorString(e));
    }
    k<<<static_cast<unsigned>(nsys), 128, smem, st>>>(a, a_stride, b, nu, nsys, f, x, info, nbad);
    return check_launch("chol_tiled_kernel");
}

// f <= 128: TPT = ceil(tiles / 128)
int chol_tiled_launch(const float *a, int64_t a_stride, const float *b, const int64_t *nu, int64_t nsys, int f,
                      float *x, int32_t *info, int32_t *nbad, cudaStream_t st) {
    if (nsys == 0) return CMF_OK;
    const int TR = ((f + 3) & ~3) / 4, T = TR * (TR + 1) / 2;
    const int tpt = (T + 127) / 128;
    switch (tpt) {
        case 1: return launch_chol_tiled<1>(a, a_stride, b, nu, nsys, f, x, info, nbad, st);
        case 2: return launch_chol_tiled<2>(a, a_stride, b, nu, nsys, f, x, info, nbad, st);
        case 3: return launch_chol_tiled<3>(a, a_stride, b, nu, nsys, f, x, info, nbad, st);
        case 4: return launch_chol_tiled<4>(a, a_stride, b, nu, nsys, f, x, info, nbad, st);
        case 5: return launch_chol_tiled<5>(a, a_stride, b, nu, nsys, f, x, info, nbad, st);
        default: return set_error(CMF_EINVAL, "f=%d too large for the tiled Cholesky", f);
    }
}

}  // namespace cmf
