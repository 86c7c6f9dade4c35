// K1 + K2: per-row Gram matrix and right-hand side on the FP32 SIMT pipes.
//
// Replaces gram._accumulate_chunk / _accumulate_row (gram.py:149-206),
// gram.pack_half (gram.py:132-146) and gram._bias_chunk (gram.py:209-220) as
// driven by assemble_side (gram.py:236-314), in ONE pass over each row's
// gathered factor rows:
//
//   * one CTA per row u; the packed lower triangle (f padded to fp = 4k) is
//     split into 4x4 register tiles, TPT tiles per thread;
//   * the row's gathered factor rows are staged into shared memory
//     SR rows at a time with cp.async, double buffered;
//   * every staged row updates every tile in CSR order.  BITWISE mode does
//     fl(acc + fl(c_i * theta_j)) with c_i = fl(w * theta_i) -- the reference's
//     exact float32 operation sequence (numba fastmath=False), so the packed
//     result is bit-identical to gram.py; FMA mode fuses it (one rounding).
//     FMA mode issues the sm_100 paired FFMA2 (one instruction per 2 MACs);
//   * the bias b_u = sum_p w_p theta_p accumulates in float64 per column (one
//     thread per column), bit-identical to _bias_chunk since a float32 x
//     float32 product is exact in float64;
//   * epilogue: + float32(lam*n_u) on the diagonal, packed lower triangle
//     staged through shared memory and written coalesced, float32 or binary16
//     (RNE, overflow flag).
#include "common.cuh"

namespace cmf {

struct GramArgs {
    const int64_t *indptr;
    const int32_t *indices;
    const float *a_w;
    const float *b_w;
    int64_t nrows;
    const float *fixed;
    int f, fp;
    double lam;
    int weighted;
    const float *base;
    void *a_out;
    int64_t a_stride;
    float *b_out;
    int64_t *nu_out;
    int32_t *overflow;
    int stage_rows;
    int stage_out;
    int vec16;
};

__device__ __forceinline__ int tri_row(int t) {
    int r = static_cast<int>((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
    while ((r + 1) * (r + 2) / 2 <= t) ++r;
    while (r * (r + 1) / 2 > t) --r;
    return r;
}

template <int TPT, bool BITWISE, bool HALF, bool HAS_AW>
__global__ void gram_simt_kernel(GramArgs g) {
    extern __shared__ __align__(16) float smem[];
    const int NT = blockDim.x, tid = threadIdx.x;
    const int64_t u = blockIdx.x;
    const int f = g.f, fp = g.fp, SR = g.stage_rows;
    const int TR = fp >> 2, T = TR * (TR + 1) / 2;

    // [stage0 | stage1 | wa0 | wa1 | wb0 | wb1]; buffers selected arithmetically
    // (a pointer array indexed by a runtime value would live on the stack)
    float *const wbase = smem + 2 * SR * fp;
    auto stage = [&](int buf) { return smem + buf * SR * fp; };
    auto wa = [&](int buf) { return wbase + buf * SR; };
    auto wb = [&](int buf) { return wbase + (2 + buf) * SR; };

    int ti[TPT], tj[TPT];
    bool valid[TPT];
    float2 acc[TPT][4][2];
#pragma unroll
    for (int s = 0; s < TPT; ++s) {
        const int t = tid + s * NT;
        valid[s] = t < T;
        const int r = valid[s] ? tri_row(t) : 0;
        ti[s] = r;
        tj[s] = valid[s] ? t - r * (r + 1) / 2 : 0;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            float v[4];
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int i = 4 * ti[s] + a, j = 4 * tj[s] + b;
                v[b] = (g.base && valid[s] && i < f && j <= i) ? g.base[i * (i + 1) / 2 + j] : 0.0f;
            }
            acc[s][a][0] = make_float2(v[0], v[1]);
            acc[s][a][1] = make_float2(v[2], v[3]);
        }
    }

    const int64_t p0 = g.indptr[u], p1 = g.indptr[u + 1];
    const int64_t n_u = p1 - p0;
    const bool do_bias = g.b_w != nullptr;
    double bacc = 0.0;

    auto issue = [&](int64_t k, int buf) {
        const int64_t q0 = p0 + k * SR;
        const int nb = static_cast<int>(min(static_cast<int64_t>(SR), p1 - q0));
        float *st = stage(buf);
        if (g.vec16) {
            const int per = fp >> 2;
            for (int e = tid; e < nb * per; e += NT) {
                const int r = e / per, c = e - r * per;
                const int64_t idx = g.indices[q0 + r];
                cp_async16(st + r * fp + 4 * c, g.fixed + idx * f + 4 * c);
            }
        } else {
            for (int e = tid; e < nb * fp; e += NT) {
                const int r = e / fp, c = e - r * fp;
                const int64_t idx = g.indices[q0 + r];
                const bool in = c < f;
                cp_async4(st + r * fp + c, g.fixed + idx * f + (in ? c : 0), in ? 4 : 0);
            }
        }
        for (int r = tid; r < nb; r += NT) {
            if (HAS_AW) cp_async4(wa(buf) + r, g.a_w + q0 + r, 4);
            if (do_bias) cp_async4(wb(buf) + r, g.b_w + q0 + r, 4);
        }
        cp_async_commit();
    };

    const int64_t nbatch = (n_u + SR - 1) / SR;
    if (nbatch > 0) issue(0, 0);
    for (int64_t k = 0; k < nbatch; ++k) {
        const int buf = static_cast<int>(k & 1);
        if (k + 1 < nbatch) {
            issue(k + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const int nb = static_cast<int>(min(static_cast<int64_t>(SR), n_u - k * SR));
        const float *st = stage(buf);
        for (int r = 0; r < nb; ++r) {
            const float *th = st + r * fp;
            const float w = HAS_AW ? wa(buf)[r] : 1.0f;
#pragma unroll
            for (int s = 0; s < TPT; ++s) {
                if (!valid[s]) continue;
                const float4 xi = *reinterpret_cast<const float4 *>(th + 4 * ti[s]);
                const float4 xj = *reinterpret_cast<const float4 *>(th + 4 * tj[s]);
                float ci[4] = {xi.x, xi.y, xi.z, xi.w};
                if (HAS_AW) {
#pragma unroll
                    for (int a = 0; a < 4; ++a) ci[a] = __fmul_rn(w, ci[a]);
                }
                const float2 j01 = make_float2(xj.x, xj.y), j23 = make_float2(xj.z, xj.w);
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const float2 c2 = make_float2(ci[a], ci[a]);
                    if (BITWISE) {
                        // scalar FMUL + FADD: ptxas 12.9 contracts mul.rn.f32x2 followed
                        // by add.rn.f32x2 into FFMA2 (even with -fmad=false), which
                        // would break bit-parity; the scalar .rn pair is kept apart.
                        acc[s][a][0].x = __fadd_rn(acc[s][a][0].x, __fmul_rn(ci[a], xj.x));
                        acc[s][a][0].y = __fadd_rn(acc[s][a][0].y, __fmul_rn(ci[a], xj.y));
                        acc[s][a][1].x = __fadd_rn(acc[s][a][1].x, __fmul_rn(ci[a], xj.z));
                        acc[s][a][1].y = __fadd_rn(acc[s][a][1].y, __fmul_rn(ci[a], xj.w));
                    } else {
                        acc[s][a][0] = __ffma2_rn(c2, j01, acc[s][a][0]);
                        acc[s][a][1] = __ffma2_rn(c2, j23, acc[s][a][1]);
                    }
                }
            }
        }
        if (do_bias && tid < f) {
            for (int r = 0; r < nb; ++r)
                bacc = fma(static_cast<double>(wb(buf)[r]), static_cast<double>(st[r * fp + tid]), bacc);
        }
        __syncthreads();
    }

    // regulariser on the diagonal (gram.py:183-186)
    const float reg = g.weighted ? __double2float_rn(g.lam * static_cast<double>(n_u))
                                 : __double2float_rn(g.lam);
#pragma unroll
    for (int s = 0; s < TPT; ++s) {
        if (valid[s] && ti[s] == tj[s]) {
            acc[s][0][0].x = __fadd_rn(acc[s][0][0].x, reg);
            acc[s][1][0].y = __fadd_rn(acc[s][1][0].y, reg);
            acc[s][2][1].x = __fadd_rn(acc[s][2][1].x, reg);
            acc[s][3][1].y = __fadd_rn(acc[s][3][1].y, reg);
        }
    }

    const int64_t P = packed_size(f);
    const size_t esize = HALF ? 2 : 4;
    char *row_out = static_cast<char *>(g.a_out) + static_cast<size_t>(u) * g.a_stride * esize;
    int ovf = 0;
    auto emit = [&](int64_t k, float v) {
        if (HALF) {
            const __half h = __float2half_rn(v);
            if (isfinite(v) && __hisinf(h)) ovf = 1;
            reinterpret_cast<__half *>(row_out)[k] = h;
        } else {
            reinterpret_cast<float *>(row_out)[k] = v;
        }
    };
    if (g.stage_out) {
        float *outs = smem;  // staging buffers are free after the last barrier
#pragma unroll
        for (int s = 0; s < TPT; ++s) {
            if (!valid[s]) continue;
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int i = 4 * ti[s] + a;
                if (i >= f) continue;
                const float v[4] = {acc[s][a][0].x, acc[s][a][0].y, acc[s][a][1].x, acc[s][a][1].y};
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int j = 4 * tj[s] + b;
                    if (j <= i) outs[i * (i + 1) / 2 + j] = v[b];
                }
            }
        }
        __syncthreads();
        for (int64_t k = tid; k < P; k += NT) emit(k, outs[k]);
    } else {
#pragma unroll
        for (int s = 0; s < TPT; ++s) {
            if (!valid[s]) continue;
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int i = 4 * ti[s] + a;
                if (i >= f) continue;
                const float v[4] = {acc[s][a][0].x, acc[s][a][0].y, acc[s][a][1].x, acc[s][a][1].y};
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int j = 4 * tj[s] + b;
                    if (j <= i) emit(static_cast<int64_t>(i) * (i + 1) / 2 + j, v[b]);
                }
            }
        }
    }
    if (HALF && ovf && g.overflow) atomicOr(g.overflow, 1);
    if (do_bias && g.b_out && tid < f) g.b_out[u * f + tid] = __double2float_rn(bacc);
    if (tid == 0 && g.nu_out) g.nu_out[u] = n_u;
}

// K2 alone (get_bias / bias-only callers): one warp per row, 4 float64
// accumulators per lane, columns in passes of 128.
__global__ void spmm_bias_kernel(const int64_t *indptr, const int32_t *indices, const float *bw,
                                 int64_t nrows, const float *fixed, int f, float *b_out) {
    const int64_t u = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (u >= nrows) return;
    const int64_t p0 = indptr[u], p1 = indptr[u + 1];
    for (int c0 = 0; c0 < f; c0 += 128) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int64_t p = p0; p < p1; ++p) {
            const double w = static_cast<double>(bw[p]);
            const float *th = fixed + static_cast<int64_t>(indices[p]) * f;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int c = c0 + lane + 32 * q;
                if (c < f) acc[q] = fma(w, static_cast<double>(th[c]), acc[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int c = c0 + lane + 32 * q;
            if (c < f) b_out[u * f + c] = __double2float_rn(acc[q]);
        }
    }
}

template <int TPT, bool BITWISE, bool HALF, bool HAS_AW>
static int launch_t(const GramArgs &g, int nt, size_t smem, cudaStream_t st) {
    auto k = gram_simt_kernel<TPT, BITWISE, HALF, HAS_AW>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return set_error(CMF_ECUDA, "gram smem attr: %s", cudaGetErrorString(e));
    }
    k<<<static_cast<unsigned>(g.nrows), nt, smem, st>>>(g);
    return check_launch("gram_simt_kernel");
}

template <int TPT>
static int launch_tpt(const GramArgs &g, bool bitwise, bool half, bool aw, int nt, size_t smem,
                      cudaStream_t st) {
    if (bitwise) {
        if (half) return aw ? launch_t<TPT, true, true, true>(g, nt, smem, st)
                            : launch_t<TPT, true, true, false>(g, nt, smem, st);
        return aw ? launch_t<TPT, true, false, true>(g, nt, smem, st)
                  : launch_t<TPT, true, false, false>(g, nt, smem, st);
    }
    if (half) return aw ? launch_t<TPT, false, true, true>(g, nt, smem, st)
                        : launch_t<TPT, false, true, false>(g, nt, smem, st);
    return aw ? launch_t<TPT, false, false, true>(g, nt, smem, st)
              : launch_t<TPT, false, false, false>(g, nt, smem, st);
}

int gram_simt_launch(const int64_t *indptr, const int32_t *indices, const float *a_w,
                     const float *b_w, int64_t nrows, const float *fixed, int f, double lam,
                     int weighted, const float *base, bool half, bool bitwise, void *a_out,
                     int64_t a_stride, float *b_out, int64_t *nu_out, int32_t *overflow,
                     cudaStream_t st) {
    if (nrows == 0) return CMF_OK;
    const int fp = (f + 3) & ~3;
    const int TR = fp / 4, T = TR * (TR + 1) / 2;
    int tpt = (T + 127) / 128;
    if (tpt < 1) tpt = 1;
    if (tpt > 4) tpt = 4;
    int nt = (T + tpt - 1) / tpt;
    nt = (nt + 31) & ~31;
    const int fneed = (f + 31) & ~31;
    if (nt < fneed) nt = fneed;
    if (nt > 1024)
        return set_error(CMF_EINVAL, "f=%d exceeds the SIMT Gram kernel's register tiling", f);
    GramArgs g{};
    g.indptr = indptr;
    g.indices = indices;
    g.a_w = a_w;
    g.b_w = b_w;
    g.nrows = nrows;
    g.fixed = fixed;
    g.f = f;
    g.fp = fp;
    g.lam = lam;
    g.weighted = weighted;
    g.base = base;
    g.a_out = a_out;
    g.a_stride = a_stride;
    g.b_out = b_out;
    g.nu_out = nu_out;
    g.overflow = overflow;
    int sr = 6144 / fp;
    if (sr > 32) sr = 32;
    if (sr < 4) sr = 4;
    g.stage_rows = sr;
    g.vec16 = (f % 4 == 0) && ((reinterpret_cast<uintptr_t>(fixed) & 15) == 0);
    size_t stage_bytes = (static_cast<size_t>(2 * sr * fp) + 4 * sr) * sizeof(float);
    const size_t out_bytes = static_cast<size_t>(packed_size(f)) * sizeof(float);
    size_t smem = stage_bytes;
    g.stage_out = out_bytes <= 100 * 1024;
    if (g.stage_out && out_bytes > smem) smem = out_bytes;
    switch (tpt) {
        case 1: return launch_tpt<1>(g, bitwise, half, a_w != nullptr, nt, smem, st);
        case 2: return launch_tpt<2>(g, bitwise, half, a_w != nullptr, nt, smem, st);
        case 3: return launch_tpt<3>(g, bitwise, half, a_w != nullptr, nt, smem, st);
        default: return launch_tpt<4>(g, bitwise, half, a_w != nullptr, nt, smem, st);
    }
}

int spmm_bias_launch(const int64_t *indptr, const int32_t *indices, const float *bw, int64_t nrows,
                     const float *fixed, int f, float *b_out, cudaStream_t st) {
    if (nrows == 0) return CMF_OK;
    const int64_t threads = nrows * 32;
    const unsigned blocks = static_cast<unsigned>((threads + 255) / 256);
    spmm_bias_kernel<<<blocks, 256, 0, st>>>(indptr, indices, bw, nrows, fixed, f, b_out);
    return check_launch("spmm_bias_kernel");
}

}  // namespace cmf
