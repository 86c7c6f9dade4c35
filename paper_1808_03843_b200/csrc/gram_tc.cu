// K1 + K2 on the 5th-generation tensor cores (tcgen05 + TMEM), CG route.
//
// Replaces gram._accumulate_chunk + _bias_chunk + pack_half (gram.py:149-220,
// :132-146) for the approximate-computing path: the paper's get_hermitian is
// a dense contraction per row, A_u = Theta_S^T Theta_S, so each row's gathered
// factor rows are the K dimension of one M=128 x N x K MMA chain.
//
// Operand trick (tc_common.cuh): the gathered rows are staged ONCE per
// K-chunk by cp.async as an MN-major, 128-byte-swizzled UMMA operand
// and the SAME shared buffer is passed as both A (M = 128 feature rows) and B
// (N = roundup16(W + 2) rows).  Operand rows W, W+1 carry the row's ratings
// (fp16 hi + lo), so accumulator columns W, W+1 give b_u = sum_p r_p theta_p:
// the bias rides along in the same MMAs (fp32 accumulation in TMEM).
//
// The fixed factor matrix is read from a binary16 shadow (cmf_factors_to_half,
// row width W = roundup8(f) halves, zero padded): every 16-byte chunk of a
// gathered row is one cp.async with no SIMT conversion, and the shadow of X
// (Netflix: 100 MB) stays resident in the 126 MB L2 (loads carry an L2
// evict_last hint).
//
// Warp roles (288 threads, 2 CTAs per SM, persistent over rows):
//   warps 0-3  epilogue: tcgen05.ld the accumulator (thread i <-> TMEM lane i
//              <-> matrix row i) into a square staging tile (+ lambda*n_u on the
//              diagonal), then all 128 threads write the packed lower triangle
//              to HBM through an offset table; b_u straight to global.
//   warps 4-7  producers: cp.async gather of K-chunks (64 gathered rows) into
//              a 4-stage ring, one warp per stage slot;
//              cp.async.mbarrier.arrive.noinc completes full[s].
//   warp 8     TMEM allocator + single-thread MMA issuer (kind::f16, fp32
//              accumulate), tcgen05.commit -> empty[s] / tmem_full[b].
// Two TMEM accumulators (2 x 128 columns) let the epilogue of row u overlap
// the MMAs of row u+1.
#include <climits>
#include <cstdlib>
#include <type_traits>

#include "tc_common.cuh"

namespace cmf {
namespace tc {

constexpr int STAGES = 4;
constexpr int NUM_THREADS = 288;
constexpr int EPI_THREADS = 128;

struct Args {
    GatherArgs gather;
    const __half *fixed16, *fixed16_lo;  // binary16 shadow (+ split residual), (ncols, W)
    float gram_scale, bias_scale;  // undo the split shadow's power-of-two scaling
    int N, tmem_cols;  // accumulator width (Gram + rating columns W, W+1), TMEM allocation
    double lam;
    int weighted;
    const float *base;
    void *a_out;
    int64_t a_stride;
    float *b_out;
    int64_t *nu_out;
    int32_t *overflow;
    // multi-pass (gather.pass 3): add this pass's Gram / bias to a_out / b_out
    // (fp32 only), and lambda*n_u on the diagonal only in the last pass
    int accumulate, add_reg;
};

__device__ __forceinline__ void bar_epi() { named_bar(1, EPI_THREADS); }

// Packed-offset table: tab[k] = i*W + j for packed entry k = i*(i+1)/2 + j.
// Built once per CTA; the epilogue copy-out walks the packed row with it.
// SYM (split operands, long rows): the MMAs build H H^T and S = H^T L in two
// accumulators (two operand reads per K-step instead of three: the tensor core's
// shared-memory operand reads set the split Gram's pace); the staging keeps
// H H^T + S in the lower triangle and S in the upper one, and the copy-out adds
// the transposed entry (tabT), so A = H H^T + S + S^T.  The staging row stride is
// W + 1 (odd: the transposed reads spread over the banks).
template <int NCH, bool HALF_OUT, bool SPLIT, bool SYM = false>
__global__ void __launch_bounds__(NUM_THREADS, 1) gram_tc_kernel(const __grid_constant__ Args g) {
    static_assert(!SYM || (SPLIT && !HALF_OUT), "SYM: split fp32 Gram only");
    using PipeT = Pipe<STAGES, SPLIT, 2>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    constexpr int W = NCH * 8;
    // staging row stride: SYM odd (transposed reads); plain fp32 == 4 (mod 32) words,
    // so that a warp's float4 row stores (rows i = lanes) are conflict-free
    constexpr int WS = SYM ? W + 1 : (HALF_OUT ? W : W + ((4 - W) % 32 + 32) % 32);
    using SqT = typename std::conditional<HALF_OUT, __half, float>::type;
    const GatherArgs &ga = g.gather;
    const int f = ga.f;
    const int64_t P = packed_size(f);
    // layout: [stages (1024-aligned) | square staging (f x WS, SqT; SYM: + a zero slot) | offset table |
    //          SYM: transposed offset table, S rows W, W+1 (2f floats) | barriers | tmem slot]
    unsigned char *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    unsigned char *stage_mem = smem;
    SqT *sq = reinterpret_cast<SqT *>(smem + STAGES * PipeT::kStageBytes);
    const size_t sq_bytes = ((static_cast<size_t>(f) * WS * sizeof(SqT) + (SYM ? 4 : 0)) + 15) & ~static_cast<size_t>(15);
    uint16_t *tab = reinterpret_cast<uint16_t *>(smem + STAGES * PipeT::kStageBytes + sq_bytes);
    const size_t tab_bytes = ((static_cast<size_t>(P) * 2) + 15) & ~static_cast<size_t>(15);
    uint16_t *tabT = tab + tab_bytes / 2;
    float *sbias = reinterpret_cast<float *>(tabT + (SYM ? tab_bytes / 2 : 0));
    const size_t sym_bytes = SYM ? tab_bytes + ((static_cast<size_t>(f) * 8 + 15) & ~static_cast<size_t>(15)) : 0;
    uint64_t *bars =
        reinterpret_cast<uint64_t *>(smem + STAGES * PipeT::kStageBytes + sq_bytes + tab_bytes + sym_bytes);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + PipeT::kBars);
    PipeT pp{smem_u32(stage_mem), smem_u32(bars)};

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    pipe_init(pp, stage_mem, NUM_THREADS, 33, EPI_THREADS);
    for (int i = tid; i < f; i += NUM_THREADS) {
        const int base = i * (i + 1) / 2;
        for (int j = 0; j <= i; ++j) {
            tab[base + j] = static_cast<uint16_t>(i * WS + j);
            if (SYM) tabT[base + j] = static_cast<uint16_t>(j < i ? j * WS + i : f * WS);  // diagonal: zero slot
        }
    }
    if (SYM && tid == 0) sq[f * WS] = SqT(0.0f);
    if (warp == 8) tmem_alloc(smem_u32(tmem_slot), g.tmem_cols);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int64_t G = gridDim.x;
    if (warp >= 4 && warp < 8) {
        produce<STAGES, SPLIT, 2>(ga, g.fixed16, g.fixed16_lo, W, pp, warp - 4, 4, lane, blockIdx.x, G);
    } else if (warp == 8) {
        issue_mma<STAGES, SPLIT, 2, false, SYM>(ga, pp, tmem_base, g.N, blockIdx.x, G);
    } else {
        // ------------------------------------------------------------ epilogue
        // (1) thread i (= TMEM lane = matrix row) drains its accumulator row into
        //     the square staging as fp16/fp32, then overwrites its diagonal with
        //     fl(A_ii + lambda*n_u) (one rounding, as the reference); the bias is
        //     read from accumulator columns f, f+1 in fp32.  (2) all 128 threads
        //     walk the packed triangle with the offset table and write it
        //     coalesced to HBM, four entries per step.
        const int i = warp * 32 + lane;
        const int nchunk = (g.N + 31) >> 5;
        const int bias_cc = W >> 5, bias_cc1 = (W + 1) >> 5;
        float ovf_max = 0.0f;
        uint32_t rowc = 0;
        SqT *sq_row = sq + static_cast<size_t>(i) * WS;
        // SYM: float scale of this lane's S row (rows W, W+1 carry the ratings: bias terms)
        const float s_scale = (i == W || i == W + 1) ? g.bias_scale : g.gram_scale;
        for (int64_t u = blockIdx.x; u < ga.nrows; u += G) {
            const int64_t p0 = ga.indptr[u], p1 = ga.indptr[u + 1];
            const int64_t n_u = p1 - p0;
            const float reg = !g.add_reg ? 0.0f
                              : g.weighted ? __double2float_rn(g.lam * static_cast<double>(n_u))
                                           : __double2float_rn(g.lam);
            float bias = 0.0f, diag = 0.0f;
            if (n_u == 0) {
                if (i < f)
                    for (int j = 0; j < W; ++j) sq_row[j] = static_cast<SqT>(0.0f);
                if (SYM && (i == W || i == W + 1))
                    for (int j = 0; j < f; ++j) sbias[(i - W) * f + j] = 0.0f;
            } else {
                const int b = rowc & 1;
                mbar_wait(pp.tfull(b), (rowc >> 1) & 1);
                tc_fence_after();
                const uint32_t tbase = tmem_base + (static_cast<uint32_t>(warp * 32) << 16) + b * g.N * (SYM ? 2 : 1);
                // a pass whose segment of this row is empty: the MMA warp committed
                // the buffer untouched (stale), so its contribution is zero
                bool seg_acc = true;
                if (ga.pass) {
                    int64_t s0, s1;
                    row_segment(ga, u, s0, s1);
                    seg_acc = s1 > s0;
                }
                for (int cc = 0; cc < nchunk; ++cc) {
                    uint32_t v[32], w[SYM ? 32 : 1];
                    tmem_ld32(tbase + cc * 32, v);
                    if constexpr (SYM) tmem_ld32(tbase + g.N + cc * 32, w);
                    tmem_ld_wait();
                    if (!seg_acc) {
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj) v[jj] = 0u;
                        if constexpr (SYM) {
#pragma unroll
                            for (int jj = 0; jj < 32; ++jj) w[jj] = 0u;
                        }
                    }
                    const int c0 = cc * 32;
                    if constexpr (SYM) {
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj) w[jj] = __float_as_uint(__uint_as_float(w[jj]) * s_scale);
                        if (i == W || i == W + 1) {  // (L^T r)_j, the bias half that S carries
#pragma unroll
                            for (int jj = 0; jj < 32; ++jj)
                                if (c0 + jj < f) sbias[(i - W) * f + c0 + jj] = __uint_as_float(w[jj]);
                        }
                    }
                    if (SPLIT) {
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj) {
                            const int j = c0 + jj;
                            const float sc = (j == W || j == W + 1) ? g.bias_scale : g.gram_scale;
                            v[jj] = __float_as_uint(__uint_as_float(v[jj]) * sc);
                        }
                    }
                    if (cc == warp) {  // warp-uniform: this chunk holds every lane's diagonal
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj)
                            if (jj == lane)
                                diag = __uint_as_float(v[jj]) + (SYM ? 2.0f * __uint_as_float(w[SYM ? jj : 0]) : 0.0f);
                    }
                    if (cc == bias_cc || cc == bias_cc1) {  // warp-uniform
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj)
                            if (c0 + jj == W || c0 + jj == W + 1) bias += __uint_as_float(v[jj]);
                    }
                    if (SYM && i < f) {
                        // lower triangle: H H^T + S; upper: S (read transposed by the copy-out)
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj) {
                            const int j = c0 + jj;
                            if (j >= W) break;
                            const float s_ij = __uint_as_float(w[SYM ? jj : 0]);
                            sq_row[j] = static_cast<SqT>(j <= i ? __uint_as_float(v[jj]) + s_ij : s_ij);
                        }
                    } else if (i < f) {
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            if (c0 + 8 * q >= W) break;
                            const float *x = reinterpret_cast<const float *>(v) + 8 * q;
                            if (HALF_OUT) {
                                __half2 h[4];
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    h[e] = __floats2half2_rn(x[2 * e], x[2 * e + 1]);
                                    ovf_max = fmaxf(ovf_max, fmaxf(fabsf(x[2 * e]), fabsf(x[2 * e + 1])));
                                }
                                *reinterpret_cast<uint4 *>(sq_row + c0 + 8 * q) = *reinterpret_cast<uint4 *>(h);
                            } else {
                                float4 *d = reinterpret_cast<float4 *>(sq_row + c0 + 8 * q);
                                d[0] = make_float4(x[0], x[1], x[2], x[3]);
                                d[1] = make_float4(x[4], x[5], x[6], x[7]);
                            }
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive(pp.tempty(b));
                ++rowc;
            }
            if (i < f) {
                const float dv = diag + reg;
                sq_row[i] = static_cast<SqT>(dv);
                if (HALF_OUT) ovf_max = fmaxf(ovf_max, fabsf(dv));
            }
            if (tid == 0 && g.nu_out) g.nu_out[u] = n_u;
            bar_epi();
            if (SYM && i < f) bias += sbias[i] + sbias[f + i];
            if (g.b_out && i < f) g.b_out[u * f + i] = g.accumulate ? g.b_out[u * f + i] + bias : bias;
            // packed copy-out: entries k..k+3 per step (k % 4 == 0)
            const size_t row_off = static_cast<size_t>(u) * g.a_stride;
            if (!g.base && !HALF_OUT && !SYM) {
                // plain fp32 (short rows on the exact route): one packed entry per lane
                // per step -- consecutive lanes read consecutive staging words (no bank
                // conflicts) and store 128 contiguous bytes per warp
                float *dstf = reinterpret_cast<float *>(g.a_out) + row_off;
                for (int64_t k = tid; k < P; k += EPI_THREADS) {
                    const float e = static_cast<float>(sq[tab[k]]);
                    dstf[k] = g.accumulate ? dstf[k] + e : e;
                }
            } else if (!g.base) {
                for (int64_t k = 4 * tid; k < P; k += 4 * EPI_THREADS) {
                    const uint2 o = *reinterpret_cast<const uint2 *>(tab + k);
                    const int64_t nk = P - k;
                    SqT e0 = sq[o.x & 0xFFFF];
                    SqT e1 = nk > 1 ? sq[o.x >> 16] : SqT(0.0f);
                    SqT e2 = nk > 2 ? sq[o.y & 0xFFFF] : SqT(0.0f);
                    SqT e3 = nk > 3 ? sq[o.y >> 16] : SqT(0.0f);
                    if constexpr (SYM) {  // + S^T (the diagonal reads the zero slot)
                        const uint2 t = *reinterpret_cast<const uint2 *>(tabT + k);
                        e0 += sq[t.x & 0xFFFF];
                        if (nk > 1) e1 += sq[t.x >> 16];
                        if (nk > 2) e2 += sq[t.y & 0xFFFF];
                        if (nk > 3) e3 += sq[t.y >> 16];
                    }
                    SqT *dst = static_cast<SqT *>(g.a_out) + row_off + k;
                    if (nk >= 4 && (reinterpret_cast<uintptr_t>(dst) & (4 * sizeof(SqT) - 1)) == 0) {
                        if (HALF_OUT) {
                            __half2 a = __halves2half2(e0, e1), c = __halves2half2(e2, e3);
                            uint2 w;
                            w.x = *reinterpret_cast<uint32_t *>(&a);
                            w.y = *reinterpret_cast<uint32_t *>(&c);
                            *reinterpret_cast<uint2 *>(dst) = w;
                        } else {
                            float4 o = make_float4(static_cast<float>(e0), static_cast<float>(e1),
                                                   static_cast<float>(e2), static_cast<float>(e3));
                            if (g.accumulate) {
                                const float4 q = *reinterpret_cast<const float4 *>(dst);
                                o = make_float4(q.x + static_cast<float>(e0), q.y + static_cast<float>(e1),
                                                q.z + static_cast<float>(e2), q.w + static_cast<float>(e3));
                            }
                            *reinterpret_cast<float4 *>(dst) = o;
                        }
                    } else if (g.accumulate) {
                        dst[0] = static_cast<SqT>(static_cast<float>(dst[0]) + static_cast<float>(e0));
                        if (nk > 1) dst[1] = static_cast<SqT>(static_cast<float>(dst[1]) + static_cast<float>(e1));
                        if (nk > 2) dst[2] = static_cast<SqT>(static_cast<float>(dst[2]) + static_cast<float>(e2));
                        if (nk > 3) dst[3] = static_cast<SqT>(static_cast<float>(dst[3]) + static_cast<float>(e3));
                    } else {
                        dst[0] = e0;
                        if (nk > 1) dst[1] = e1;
                        if (nk > 2) dst[2] = e2;
                        if (nk > 3) dst[3] = e3;
                    }
                }
            } else {  // implicit-style base matrix: add in fp32, round once more
                for (int64_t k = tid; k < P; k += EPI_THREADS) {
                    const float a = static_cast<float>(sq[tab[k]]) + g.base[k];
                    static_cast<SqT *>(g.a_out)[row_off + k] = static_cast<SqT>(a);
                    if (HALF_OUT) ovf_max = fmaxf(ovf_max, fabsf(a));
                }
            }
            bar_epi();  // staging free for the next row
        }
        if (HALF_OUT && ovf_max >= 65520.0f && isfinite(ovf_max) && g.overflow) atomicOr(g.overflow, 1);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 8) {
        tc_fence_after();
        tmem_dealloc(tmem_base, g.tmem_cols);
    }
}

// fp32 (rows, f) -> binary16 (rows + 1, W), zero padded, RNE; row `rows` is the
// all-zero row the gather reads for padding positions.
// One warp per shadow row (rows + 1 of them, the last all zero), 4 halves per
// lane: 16-byte coalesced loads, 8-byte stores, no per-element index division.
// A finite factor whose binary16 rounding overflows (|x| >= 65520) sets *ovf:
// the fp16 Gram built from it would overflow as the reference's pack_half does
// (gram.py:132-146), so the caller raises NumericalError.
__global__ void factors_to_half_kernel(const float *x, int64_t rows, int f, __half *out, int W, int32_t *ovf) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    float amax = 0.0f;
    for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r <= rows; r += nw) {
        const float *src = x + r * f;
        for (int c = 4 * lane; c < W; c += 128) {
            float v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                v[k] = (r < rows && c + k < f) ? src[c + k] : 0.0f;
                amax = fmaxf(amax, fabsf(v[k]));  // NaN is dropped by fmaxf, inf is kept
            }
            const __half2 h01 = __floats2half2_rn(v[0], v[1]), h23 = __floats2half2_rn(v[2], v[3]);
            *reinterpret_cast<uint2 *>(out + r * W + c) =
                make_uint2(*reinterpret_cast<const uint32_t *>(&h01), *reinterpret_cast<const uint32_t *>(&h23));
        }
    }
    if (ovf && amax >= 65520.0f && amax <= 3.402823466e38f) atomicOr(ovf, 1);
}

// Split shadow: hi = fp16(scale*x), lo = fp16(scale*x - hi); scale is a power of
// two that keeps lo out of the binary16 subnormal range for |x| >= 2^-9.
__global__ void factors_to_half_split_kernel(const float *x, int64_t rows, int f, __half *hi, __half *lo, int W,
                                             float scale, int32_t *ovf) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    int bad = 0;
    for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r <= rows; r += nw) {
        const float *src = x + r * f;
        for (int c = 4 * lane; c < W; c += 128) {
            __align__(8) __half h[4];
            __align__(8) __half l[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float v = (r < rows && c + k < f) ? src[c + k] * scale : 0.0f;
                h[k] = __float2half_rn(v);
                if (isfinite(v) && __hisinf(h[k])) bad = 1;
                l[k] = __float2half_rn(v - __half2float(h[k]));
            }
            *reinterpret_cast<uint2 *>(hi + r * W + c) = *reinterpret_cast<const uint2 *>(h);
            *reinterpret_cast<uint2 *>(lo + r * W + c) = *reinterpret_cast<const uint2 *>(l);
        }
    }
    if (bad && ovf) atomicOr(ovf, 1);
}

}  // namespace tc

int factors_to_half_split_launch(const float *x, int64_t rows, int f, void *hi, void *lo, int W, float scale,
                                 int32_t *ovf, cudaStream_t st) {
    if (rows == 0) return CMF_OK;
    int64_t blocks = (rows + 1 + 7) / 8;  // 8 rows (warps) per 256-thread block
    if (blocks > 148 * 16) blocks = 148 * 16;
    tc::factors_to_half_split_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(
        x, rows, f, static_cast<__half *>(hi), static_cast<__half *>(lo), W, scale, ovf);
    return check_launch("factors_to_half_split_kernel");
}

int gram_tc_trace(void *buf) { return tc::set_trace_buf(buf); }

int gram_tc_width(int f) { return ((f + 7) / 8) * 8; }

int factors_to_half_launch(const float *x, int64_t rows, int f, void *out, int W, int32_t *ovf, cudaStream_t st) {
    if (rows == 0) return CMF_OK;
    int64_t blocks = (rows + 1 + 7) / 8;
    if (blocks > 148 * 16) blocks = 148 * 16;
    tc::factors_to_half_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(x, rows, f,
                                                                             static_cast<__half *>(out), W, ovf);
    return check_launch("factors_to_half_kernel");
}

template <int NCH, bool H, bool SPLIT, bool SYM>
static int launch_nch(const tc::Args &g, size_t smem, int64_t nrows, cudaStream_t st) {
    auto k = tc::gram_tc_kernel<NCH, H, SPLIT, SYM>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return set_error(CMF_ECUDA, "gram_tc smem attr: %s", cudaGetErrorString(e));
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    // two CTAs per SM when their shared memory and TMEM (2 x 256 columns) fit
    per_sm = (2 * (smem + 1024) <= 227 * 1024 && g.tmem_cols <= 256) ? 2 : 1;
    int64_t grid = static_cast<int64_t>(per_sm) * sms;
    if (grid > nrows) grid = nrows;
    k<<<static_cast<unsigned>(grid), tc::NUM_THREADS, smem, st>>>(g);
    return check_launch("gram_tc_kernel");
}

template <bool H, bool SPLIT, bool SYM = false>
static int dispatch_nch(int nch, const tc::Args &g, size_t smem, int64_t nrows, cudaStream_t st) {
    switch (nch) {
        case 1: return launch_nch<1, H, SPLIT, SYM>(g, smem, nrows, st);
        case 2: return launch_nch<2, H, SPLIT, SYM>(g, smem, nrows, st);
        case 3: return launch_nch<3, H, SPLIT, SYM>(g, smem, nrows, st);
        case 4: return launch_nch<4, H, SPLIT, SYM>(g, smem, nrows, st);
        case 5: return launch_nch<5, H, SPLIT, SYM>(g, smem, nrows, st);
        case 6: return launch_nch<6, H, SPLIT, SYM>(g, smem, nrows, st);
        case 7: return launch_nch<7, H, SPLIT, SYM>(g, smem, nrows, st);
        case 8: return launch_nch<8, H, SPLIT, SYM>(g, smem, nrows, st);
        case 9: return launch_nch<9, H, SPLIT, SYM>(g, smem, nrows, st);
        case 10: return launch_nch<10, H, SPLIT, SYM>(g, smem, nrows, st);
        case 11: return launch_nch<11, H, SPLIT, SYM>(g, smem, nrows, st);
        case 12: return launch_nch<12, H, SPLIT, SYM>(g, smem, nrows, st);
        case 13: return launch_nch<13, H, SPLIT, SYM>(g, smem, nrows, st);
        case 14: return launch_nch<14, H, SPLIT, SYM>(g, smem, nrows, st);
        case 15: return launch_nch<15, H, SPLIT, SYM>(g, smem, nrows, st);
        default: return launch_nch<16, H, SPLIT, SYM>(g, smem, nrows, st);
    }
}

int gram_tc_launch(const int64_t *indptr, const int32_t *indices, const float *values, int64_t nrows,
                   const void *fixed16, const void *fixed16_lo, int64_t ncols, float split_scale, int W, int f,
                   double lam,
                   int weighted, const float *base, bool half, void *a_out, int64_t a_stride, float *b_out,
                   int64_t *nu_out, int32_t *overflow, cudaStream_t st, const int64_t *seg,
                   const int64_t *seg_end, int accumulate, int add_reg, int sym) {
    if (nrows == 0) return CMF_OK;
    if (W + 2 > tc::M)
        return set_error(CMF_EINVAL, "tensor-core Gram supports f <= %d (got %d)", tc::M - 8, f);
    if (W != gram_tc_width(f)) return set_error(CMF_EINVAL, "fixed16 width must be %d", gram_tc_width(f));
    const int esz = half ? 2 : 4;
    if ((a_stride % 2) != 0 || (reinterpret_cast<uintptr_t>(a_out) & 15) != 0)
        return set_error(CMF_EINVAL, "tensor-core Gram needs an even a_stride and a 16-byte aligned a_out");
    tc::Args g{};
    const bool split = fixed16_lo != nullptr;
    if ((reinterpret_cast<uintptr_t>(fixed16) & 15) != 0 || (reinterpret_cast<uintptr_t>(fixed16_lo) & 15) != 0)
        return set_error(CMF_EINVAL, "fixed16 / fixed16_lo must be 16-byte aligned");
    if (ncols < 1 || ncols >= (int64_t(1) << 31)) return set_error(CMF_EINVAL, "bad shadow row count");
    g.fixed16 = static_cast<const __half *>(fixed16);
    g.fixed16_lo = static_cast<const __half *>(fixed16_lo);
    g.gather.indptr = indptr;
    g.gather.indices = indices;
    g.gather.values = values;
    g.gather.nrows = nrows;
    g.gather.f = f;
    g.gather.ncols = static_cast<int>(ncols);
    g.gather.trace = tc::g_trace_buf;
    g.gram_scale = split ? 1.0f / (split_scale * split_scale) : 1.0f;
    g.bias_scale = split ? 1.0f / split_scale : 1.0f;
    g.N = ((W + 2 + 15) / 16) * 16;
    if (sym && (!split || half || base)) sym = 0;
    g.tmem_cols = (sym || 2 * g.N > 256) ? 512 : 256;  // SYM: 2 buffers x (H H^T, S)
    g.lam = lam;
    g.weighted = weighted;
    g.base = base;
    g.a_out = a_out;
    g.a_stride = a_stride;
    g.b_out = b_out;
    g.nu_out = nu_out;
    g.overflow = overflow;
    g.gather.overflow = overflow;
    if (seg) {
        if (!split || half || base) return set_error(CMF_EINVAL, "multi-pass Gram: split fp32 output only");
        g.gather.pass = 3;
        g.gather.seg = seg;
        g.gather.seg_end = seg_end;
    }
    g.accumulate = accumulate;
    g.add_reg = add_reg;
    const int64_t P = packed_size(f);
    const size_t ws_row = sym ? W + 1 : (half ? W : W + ((4 - W) % 32 + 32) % 32);  // as the kernel's WS
    const size_t sq_bytes = ((static_cast<size_t>(f) * ws_row * esz + (sym ? 4 : 0)) + 15) & ~static_cast<size_t>(15);
    const size_t tab_bytes = ((static_cast<size_t>(P) * 2) + 15) & ~static_cast<size_t>(15);
    const size_t sym_bytes = sym ? tab_bytes + ((static_cast<size_t>(f) * 8 + 15) & ~static_cast<size_t>(15)) : 0;
    const size_t stage_bytes = split ? tc::Pipe<tc::STAGES, true, 2>::kStageBytes
                                     : tc::Pipe<tc::STAGES, false, 2>::kStageBytes;
    const size_t smem =
        1024 + tc::STAGES * stage_bytes + sq_bytes + tab_bytes + sym_bytes + tc::Pipe<tc::STAGES>::kBars * 8 + 16;
    const int nch = W / 8;
    if (split) {
        if (half) return set_error(CMF_EINVAL, "the split-precision Gram stores fp32");
        return sym ? dispatch_nch<false, true, true>(nch, g, smem, nrows, st)
                   : dispatch_nch<false, true>(nch, g, smem, nrows, st);
    }
    return half ? dispatch_nch<true, false>(nch, g, smem, nrows, st)
                : dispatch_nch<false, false>(nch, g, smem, nrows, st);
}

}  // namespace cmf

namespace cmf {

int segment_split_launch(const int64_t *indptr, const int32_t *indices, int64_t nrows, int32_t split, int64_t *seg,
                         cudaStream_t st);

// Split-precision (fp32) Gram over long rows whose fixed side's hi + lo shadow
// is larger than L2 keeps (the Netflix item side of the exact route: 200 MB of X
// shadow, 51% L2 hits and 28.5 GB of DRAM reads in one pass): P passes over
// equal user-id ranges, each gathering from a ~1/P slice of the shadow; pass 1
// writes A / b, later passes add to them, the last adds lambda*n_u.  The
// per-row segment bounds (P - 1 arrays of nrows int64) live in ws.
int64_t gram_tc_passes(int64_t nrows, int64_t nnz, int64_t ncols, int W, bool split) {
    if (const char *e = getenv("CMF_GRAM_PASSES"))  // A/B and tests (empty: automatic)
        if (*e) return atoi(e) > 1 ? (atoi(e) < 16 ? atoi(e) : 16) : 1;
    const int64_t shadow = ncols * W * 2 * (split ? 2 : 1);
    if (!split || nnz < 1024 * nrows || shadow <= (int64_t(72) << 20)) return 1;
    const int64_t p = (shadow + (int64_t(72) << 20) - 1) / (int64_t(72) << 20);
    return p < 8 ? p : 8;
}

int gram_tc_ws_launch(const int64_t *indptr, const int32_t *indices, const float *values, int64_t nrows,
                      const void *fixed16, const void *fixed16_lo, int64_t ncols, float split_scale, int W, int f,
                      double lam, int weighted, bool half, void *a_out, int64_t a_stride, float *b_out,
                      int64_t *nu_out, int32_t *overflow, int64_t nnz, void *ws, int64_t ws_bytes, cudaStream_t st) {
    const int64_t P = gram_tc_passes(nrows, nnz, ncols, W, fixed16_lo != nullptr);
    // long rows: the split Gram's K-steps dominate and the SYM copy-out's extra
    // transposed reads are amortised over ~80 stages per row (short rows: ~3)
    int sym = nnz >= 1024 * nrows;
    if (const char *e = getenv("CMF_GRAM_SYM"))  // A/B and tests (empty: automatic)
        if (*e) sym = atoi(e);
    if (P <= 1 || half || !fixed16_lo || !ws || ws_bytes < (P - 1) * nrows * 8 || ncols > INT32_MAX)
        return gram_tc_launch(indptr, indices, values, nrows, fixed16, fixed16_lo, ncols, split_scale, W, f, lam,
                              weighted, nullptr, half, a_out, a_stride, b_out, nu_out, overflow, st, nullptr,
                              nullptr, 0, 1, sym);
    int64_t *segs = static_cast<int64_t *>(ws);
    for (int64_t k = 1; k < P; ++k) {
        const int rc = segment_split_launch(indptr, indices, nrows, static_cast<int32_t>(ncols * k / P),
                                            segs + (k - 1) * nrows, st);
        if (rc != CMF_OK) return rc;
    }
    for (int64_t k = 1; k <= P; ++k) {
        const int64_t *b = k == 1 ? indptr : segs + (k - 2) * nrows;
        const int64_t *e = k == P ? indptr + 1 : segs + (k - 1) * nrows;
        const int rc = gram_tc_launch(indptr, indices, values, nrows, fixed16, fixed16_lo, ncols, split_scale, W, f,
                                      lam, weighted, nullptr, half, a_out, a_stride, b_out, nu_out, overflow, st, b,
                                      e, k > 1, k == P, sym);
        if (rc != CMF_OK) return rc;
    }
    return CMF_OK;
}

}  // namespace cmf
