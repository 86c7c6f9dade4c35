// Fused half-update for the CG route: tensor-core Gram -> TMEM -> truncated
// CG in registers -> x, without ever writing A_u to HBM.
//
// Replaces, for als.update_side with SolverConfig(method="cg") (als.py:54-74),
// the pair assemble_side (gram.py:236-314) + batch_solve/_cg_batch
// (solvers.py:121-145, 205-247).  The two-step scheme of the paper (materialise
// every A_u, then solve) is kept for the reference-facing assemble_side /
// batch_solve API; here the accumulator a tcgen05.mma chain leaves in TMEM is
// exactly the register-resident row layout the CG matvec wants (thread i <->
// TMEM lane i <-> row i of A_u), so the solve runs straight out of TMEM:
//
//   producers   cp.async gather of binary16 factor rows (+ the rating rows)
//               into a 12-stage swizzled operand ring (7 warps; 11 for long rows)
//   MMA warp    tcgen05.mma kind::f16 chain per row into one of 2 (3) fp32 TMEM
//               accumulators; tcgen05.commit -> stage empty / accumulator full
//   CG groups   4 (2 for long rows) groups of 4 warps; group r % NG takes row r:
//               reads b_u from the accumulator's rating columns, repacks A_u to
//               binary16 into its own TMEM slot (the tcgen05 A-operand layout)
//               and frees the accumulator, then runs Algorithm 1 (PAPER.md:
//               272-293, corrected r -= alpha*A p) in its pipelined form (one
//               barrier per iteration carries both dot products and the next
//               matvec's vector) with fp32 vectors; every matvec is 7
//               tensor-core MMAs with A read from TMEM; deterministic
//               reductions; x_u written in place (warm start = previous x_u).
// The kernel template lives in fused_cg.cuh (shared with the implicit-feedback
// instances, fused_implicit.cu); this file holds the launchers, the two-pass
// driver for long rows and the two-step route's batched CG (cg_tc_kernel).
//
// Semantics vs the reference: the diagonal gets lambda*n_u (weighted) or
// lambda; rows with n_u == 0 are left untouched; eps = cg_tol * ||b_u||;
// breakdown (p^T A p <= 0) keeps the current iterate and is counted.  A_u is
// rounded from the fp32 accumulator to binary16 (RNE) in TMEM -- the
// reference's precision="fp16" Hermitian storage (gram.py:132-146) -- and an
// entry that overflows binary16 sets the overflow flag, which the caller
// raises as NumericalError like pack_half does.  The CG vectors are fp32
// (split into fp16 hi/lo halves as the matvec's B operand).
#include "fused_cg.cuh"

namespace cmf {
namespace tc {

// ---------------------------------------------------------------------------
// Batched CG over packed binary16 systems (the two-step route's K3: replaces
// solvers._cg_batch for precision="fp16", solvers.py:121-145, 205-247).
// One CTA per SM with as many 128-thread groups as TMEM (a KP/2-column binary16
// slot + a 16-column result block each) and shared memory allow: 7 at f = 100
// (6 systems in flight per SM with the earlier 2 x 3 shape: 3.17 -> 2.96 ms on
// the Netflix user side, same box); each group double-buffers
// its systems' packed lower triangles HBM -> shared memory with cp.async
// (the only large read), expands row i of the symmetric matrix into its TMEM
// slot in the tcgen05 A-operand layout (the stored binary16 values, no
// rounding), and runs TmemCg (tensor-core matvecs, one barrier per iteration).
struct CgTcArgs {
    const __half *a;
    int64_t a_stride;  // halves, 8-aligned
    const float *b, *x0;
    const double *eps;
    double tol;
    const int64_t *nu;
    int64_t nsys;
    int f, f_s;
    float *x_out;
    int32_t *iters, *broke, *breakdowns;
    int pipelined;  // CMF_CG_PIPELINED=1: one barrier per iteration (pipelined recurrence)
};

// CTA shape: CGT_GROUPS systems in flight per CTA, CGT_PER_SM CTAs per SM, each
// CTA owning 512 / CGT_PER_SM TMEM columns (a 56-column binary16 slot and a
// 16-column matvec result block per group at f = 100)
#ifndef CMF_CGT_GROUPS
#define CMF_CGT_GROUPS 7
#endif
constexpr int CGT_PER_SM = CMF_CGT_GROUPS <= 3 ? 2 : 1;
constexpr int CGT_TMEM = 512 / CGT_PER_SM;
template <int KP>  // per-group shared memory: matvec operand + double-buffered staging
constexpr int cgt_group_bytes() {
    return (MVB_BYTES + 2 * ((((KP * (KP - 1) / 2 + 128) * 2) + 127) & ~127) + 1023) & ~1023;
}
template <int KP>  // groups whose slots + result blocks fit the CTA's TMEM and whose scratch fits smem
constexpr int cgt_groups() {
    constexpr int by_tmem = 512 / (KP / 2 + 16), by_smem = (227 * 1024 - 2048) / cgt_group_bytes<KP>();
    constexpr int g = CMF_CGT_GROUPS < by_tmem ? CMF_CGT_GROUPS : by_tmem;
    return CGT_PER_SM == 2 ? CMF_CGT_GROUPS : (g < by_smem ? g : by_smem);
}

template <int KP>
__global__ void __launch_bounds__(128 * cgt_groups<KP>(), CGT_PER_SM) cg_tc_kernel(const __grid_constant__ CgTcArgs g) {
    constexpr int CGT_GROUPS = cgt_groups<KP>(), CGT_THREADS = 128 * CGT_GROUPS;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    const int f = g.f;
    const int64_t P = packed_size(f);
    // staging bytes per system: every packed index a KP-wide expansion can touch
    // (j(j+1)/2 + i for j < KP, i < 128), the part past P zero (columns j >= f)
    constexpr int SB = (((KP * (KP - 1) / 2 + 128) * 2) + 127) & ~127;
    // per-group scratch: the matvec operand must sit on a 1024-byte swizzle atom
    const int GS = (MVB_BYTES + 2 * SB + 1023) & ~1023;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, grp = warp >> 2;
    unsigned char *scr = smem + grp * GS;
    unsigned char *stg = scr + MVB_BYTES;
    uint64_t *mvbars = reinterpret_cast<uint64_t *>(smem + CGT_GROUPS * GS);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(mvbars + CGT_GROUPS);
    for (int k = tid; k < CGT_GROUPS * GS / 16; k += CGT_THREADS)
        reinterpret_cast<int4 *>(smem)[k] = make_int4(0, 0, 0, 0);
    if (tid == 0) {
        for (int q = 0; q < CGT_GROUPS; ++q) mbar_init(smem_u32(mvbars + q), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(smem_u32(tmem_slot), CGT_TMEM);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    TmemCg<KP> cg(scr, smem_u32(mvbars + grp), 1 + grp, warp, lane, f);
    const int i = cg.i, gt = tid & 127;
    // TMEM: 16-column aligned slots (KP/2 packed columns each), then the 16-column
    // matvec results from a 32-column boundary
    constexpr uint32_t SLOT = CGT_PER_SM == 1 ? KP / 2 : (KP / 2 + 15) / 16 * 16;
    constexpr uint32_t DBASE = (CGT_GROUPS * SLOT + 15) / 16 * 16;
    static_assert(DBASE + 16 * CGT_GROUPS <= CGT_TMEM, "cg_tc TMEM plan");
    const uint32_t a_tmem = tmem_base + grp * SLOT;
    const uint32_t dcol = tmem_base + DBASE + 16 * grp;
    const uint32_t slot_t = a_tmem + cg.lane_base;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * CGT_GROUPS;
    const int nchunk = static_cast<int>((P * 2 + 15) / 16);  // within a_stride (8-aligned) of each system
    auto stage = [&](int64_t sys, int buf) {
        if (sys < g.nsys && !(g.nu && g.nu[sys] == 0)) {
            const char *src = reinterpret_cast<const char *>(g.a + sys * g.a_stride);
            unsigned char *dst = stg + buf * SB;
            for (int k = gt; k < nchunk; k += 128) cp_async16(dst + 16 * k, src + 16 * k);
        }
        cp_async_commit();
    };
    int32_t brk = 0;
    int buf = 0;
    int64_t sys = static_cast<int64_t>(blockIdx.x) * CGT_GROUPS + grp;
    stage(sys, 0);
    for (; sys < g.nsys; sys += stride, buf ^= 1) {
        stage(sys + stride, buf ^ 1);  // next system in flight while this one is solved
        if (g.nu && g.nu[sys] == 0) continue;
        const bool act = cg.act;
        float xi = act ? g.x0[sys * f + i] : 0.0f;
        const float bi = act ? g.b[sys * f + i] : 0.0f;
        cp_async_wait<1>();
        if (gt == (nchunk - 1) % 128)  // the last 16-byte chunk may carry stride padding past P
            for (int k = static_cast<int>(P); k < 8 * nchunk; ++k)
                reinterpret_cast<unsigned short *>(stg + buf * SB)[k] = 0;
        named_bar(1 + grp, CG_THREADS);
        // row i of the symmetric matrix -> binary16 pairs in TMEM
        const __half *A = reinterpret_cast<const __half *>(stg + buf * SB);
        // element (i, j): row i of the packed lower triangle for j <= i, column i
        // (row j, position i) above the diagonal.  Warp q holds rows 32q .. 32q+31,
        // so a 32-column chunk c is, for the whole warp, either below the diagonal
        // (c < q: a contiguous segment of row i, read as realigned 32-bit words),
        // above it (c > q: column i of rows j -- consecutive lanes read consecutive
        // halves, offsets j(j+1)/2 are immediates) or the diagonal chunk (per
        // element select).  Columns j >= f read the zero tail of the staging
        // buffer; lanes i >= f read row 0 (their rows only feed their own, unused
        // outputs).
        const int ri = act ? i * (i + 1) / 2 : 0;
        const int ci = act ? i : 0;
        const int wq = warp & 3;
        const unsigned short *Au = reinterpret_cast<const unsigned short *>(A);
        const uint32_t *Aw = reinterpret_cast<const uint32_t *>(A);
        const uint32_t sel = (ri & 1) ? 0x5432u : 0x3210u;
#pragma unroll
        for (int c = 0; c < (KP + 31) / 32; ++c) {  // fully unrolled: j, j(j+1)/2 are immediates
            uint32_t h[16];
            if (c < wq) {
                const int wb = (ri + 32 * c) >> 1;
                uint32_t wv[17];
#pragma unroll
                for (int k = 0; k < 17; ++k) wv[k] = Aw[wb + k];
#pragma unroll
                for (int q = 0; q < 16; ++q) h[q] = __byte_perm(wv[q], wv[q + 1], sel);
            } else if (c > wq) {
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const int j = 32 * c + 2 * q;
                    if (j >= KP) break;
                    h[q] = static_cast<uint32_t>(Au[j * (j + 1) / 2 + ci]) |
                           (static_cast<uint32_t>(Au[(j + 1) * (j + 2) / 2 + ci]) << 16);
                }
            } else {
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    uint32_t e[2];
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        const int j = 32 * c + 2 * q + t;
                        e[t] = j < KP ? Au[j <= ci ? ri + j : j * (j + 1) / 2 + ci] : 0u;
                    }
                    h[q] = e[0] | (e[1] << 16);
                }
            }
            if (16 * c + 16 <= KP / 2) tmem_st16(slot_t + 16 * c, h);
            else if (16 * c < KP / 2) tmem_st8(slot_t + 16 * c, h);
        }
        tmem_st_wait();
        tc_fence_before();
        int bd = 0, nit = 0;
        if (g.pipelined)
            cg.solve(a_tmem, dcol, 0.0f, bi, g.eps ? g.eps[sys] : -1.0, static_cast<float>(g.tol), g.f_s, xi, bd,
                     nit);
        else
            cg.solve_standard(a_tmem, dcol, bi, g.eps ? g.eps[sys] : -1.0, static_cast<float>(g.tol), g.f_s, xi,
                              bd, nit);
        if (act) g.x_out[sys * f + i] = xi;
        if (gt == 0) {
            if (g.iters) g.iters[sys] = nit;
            if (g.broke) g.broke[sys] = bd;
        }
        brk += bd;
        tc_fence_before();  // the next system's repack overwrites the slot the MMAs read
    }
    cp_async_wait<0>();
    if (gt == 0 && brk && g.breakdowns) atomicAdd(g.breakdowns, brk);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem_base, CGT_TMEM);
    }
}

}  // namespace tc

int gram_tc_width(int f);
int fused_cg_trace(void *buf) { return tc::set_trace_buf(buf); }

// seg[u] = first position of row u whose index is >= split (rows sorted by index,
// as build() leaves them; for unsorted rows the split is still a valid partition)
__global__ void segment_split_kernel(const int64_t *indptr, const int32_t *indices, int64_t nrows, int32_t split,
                                     int64_t *seg) {
    for (int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; u < nrows;
         u += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int64_t lo = indptr[u], hi = indptr[u + 1];
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (indices[mid] < split) lo = mid + 1;
            else hi = mid;
        }
        seg[u] = lo;
    }
}

int segment_split_launch(const int64_t *indptr, const int32_t *indices, int64_t nrows, int32_t split, int64_t *seg,
                         cudaStream_t st) {
    if (nrows == 0) return CMF_OK;
    const int64_t blocks = (nrows + 255) / 256;
    segment_split_kernel<<<static_cast<unsigned>(blocks < 4096 ? blocks : 4096), 256, 0, st>>>(indptr, indices, nrows,
                                                                                               split, seg);
    return check_launch("segment_split_kernel");
}

// Two passes pay when the rows are long (the partial accumulator's HBM round
// trip, ~2 x 43 KB per row at f = 100, is small against the row's gather) and
// the fixed side's binary16 shadow is too large to stay in L2 across the
// sweep (Netflix Theta side: 100 MB of X shadow, 67% L2 hits in one pass).
constexpr int64_t kTwoPassShadowBytes = int64_t(48) << 20;
int64_t fused_cg_workspace_bytes(int64_t nrows, int W) {
    const int64_t pws = (W + 2 + 3) / 4 * 4;
    return ((nrows * 8 + 255) & ~int64_t(255)) + nrows * 128 * pws * 4;  // (f <= 128 lanes per row)
}
int64_t fused_cg_partial_floats(int64_t nrows, int f) { return nrows * f * ((gram_tc_width(f) + 2 + 3) / 4 * 4); }

int fused_dispatch_implicit(tc::FusedArgs g, int f, bool long_rows, cudaStream_t st);

int fused_cg_launch(const int64_t *indptr, const int32_t *indices, const float *values, int64_t nrows,
                    const void *fixed16, int64_t ncols, int W, int f, double lam, int weighted, float *target,
                    float *const *peers, int npeers, int64_t nnz, int f_s, double cg_tol, int32_t *breakdowns,
                    int32_t *overflow, void *ws, int64_t ws_bytes, const float *base, float alpha, bool implicit,
                    const int64_t *ext_seg, float *ext_partial, int ext_pass, cudaStream_t st) {
    if (nrows == 0) return CMF_OK;
    if (npeers < 0 || (npeers > 0 && peers == nullptr)) return set_error(CMF_EINVAL, "bad peer replica list");
    if (nnz < 0) return set_error(CMF_EINVAL, "negative rating count");
    const bool long_rows = nnz >= tc::LONG_ROW_NNZ * nrows;
    if (W + 2 > tc::M) return set_error(CMF_EINVAL, "fused CG supports f <= %d (got %d)", tc::M - 8, f);
    if (W != gram_tc_width(f)) return set_error(CMF_EINVAL, "fixed16 width must be %d", gram_tc_width(f));
    if ((reinterpret_cast<uintptr_t>(fixed16) & 15) != 0) return set_error(CMF_EINVAL, "fixed16 must be 16-byte aligned");
    if (ncols < 1 || ncols >= (int64_t(1) << 31)) return set_error(CMF_EINVAL, "bad shadow row count");
    tc::FusedArgs g{};
    g.fixed16 = static_cast<const __half *>(fixed16);
    g.W = W;
    g.gather.indptr = indptr;
    g.gather.indices = indices;
    g.gather.values = values;
    g.gather.nrows = nrows;
    g.gather.f = f;
    g.gather.ncols = static_cast<int>(ncols);
    g.gather.trace = tc::g_trace_buf;
    g.N = ((W + 2 + 15) / 16) * 16;
    g.lam = lam;
    g.weighted = weighted;
    g.target = target;
    g.peers = peers;
    g.npeers = npeers;
    g.f_s = f_s;
    {
        // every producer warp of the shape (same-box A/B, tools/ab_probe.sh: with 4
        // CG groups the user side runs 5.48 ms with 7 producers, 5.65 with 5)
        const char *e = getenv("CMF_FUSED_PROD");
        g.nprod = e ? atoi(e) : 0;
    }
    g.tol = static_cast<float>(cg_tol);
    g.breakdowns = breakdowns;
    g.overflow = overflow;
    g.gather.overflow = overflow;
    g.base = base;
    g.alpha = alpha;
    // implicit systems (F^T F + plain lambda) are far worse conditioned than the
    // explicit ones (lambda n_u): the WEIGHTED kernels run the standard CG
    // recurrence, the pipelined one drifts there (tools/diag_implicit3.py)
    auto dispatch = [&](const tc::FusedArgs &a) {
        return implicit ? fused_dispatch_implicit(a, f, long_rows, st) : fused_dispatch_t<false>(a, f, long_rows, st);
    };
    if (ext_pass == 1 || ext_pass == 2) {
        // one pass of the two-pass scheme with the caller's segment split and
        // partial buffer (multi-GPU reduce-scatter of partial Grams, distributed.py)
        if (!ext_seg || !ext_partial) return set_error(CMF_EINVAL, "pass %d needs seg and partial", ext_pass);
        if (f > 104) return set_error(CMF_EINVAL, "partial passes support f <= 104");
        g.partial = ext_partial;
        g.pws = (W + 2 + 3) / 4 * 4;
        g.gather.seg = ext_seg;
        g.gather.pass = ext_pass;
        return dispatch(g);
    }
    {
        const char *e = getenv("CMF_TWO_PASS");
        const bool want = e ? atoi(e) != 0
                            : long_rows && static_cast<int64_t>(ncols) * W * 2 > kTwoPassShadowBytes;
        if (want && ws && ws_bytes >= fused_cg_workspace_bytes(nrows, W) && f <= 104) {
            int64_t *seg = static_cast<int64_t *>(ws);
            g.partial = reinterpret_cast<float *>(static_cast<char *>(ws) + ((nrows * 8 + 255) & ~int64_t(255)));
            g.pws = (W + 2 + 3) / 4 * 4;
            g.gather.seg = seg;
            const int64_t blocks = (nrows + 255) / 256;
            segment_split_kernel<<<static_cast<unsigned>(blocks < 4096 ? blocks : 4096), 256, 0, st>>>(
                indptr, indices, nrows, static_cast<int32_t>(ncols / 2), seg);
            int rc = check_launch("segment_split_kernel");
            if (rc != CMF_OK) return rc;
            for (int pass = 1; pass <= 2; ++pass) {
                g.gather.pass = pass;
                rc = dispatch(g);
                if (rc != CMF_OK) return rc;
            }
            return CMF_OK;
        }
    }
    return dispatch(g);
}


template <int KP>
static int launch_cg_tc(const tc::CgTcArgs &g, cudaStream_t st) {
    const int64_t P = packed_size(g.f);
    (void)P;
    constexpr size_t SB = (((KP * (KP - 1) / 2 + 128) * 2) + 127) & ~127;  // as in cg_tc_kernel
    const size_t GS = (tc::MVB_BYTES + 2 * SB + 1023) & ~static_cast<size_t>(1023);
    constexpr int G = tc::cgt_groups<KP>();
    const size_t smem = 1024 + G * GS + G * 8 + 16;
    auto k = tc::cg_tc_kernel<KP>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return set_error(CMF_ECUDA, "cg_tc smem attr: %s", cudaGetErrorString(e));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t grid = tc::CGT_PER_SM * static_cast<int64_t>(sms);
    const int64_t need = (g.nsys + G - 1) / G;
    if (grid > need) grid = need;
    k<<<static_cast<unsigned>(grid), 128 * G, smem, st>>>(g);
    return check_launch("cg_tc_kernel");
}

// fp16 batched CG on the tensor cores; returns -1 when the shape is not covered
// (the caller then uses the SIMT kernel): f <= 120, 16-byte aligned rows.
int cg_tc_launch(const void *a, int64_t a_stride, const float *b, const float *x0, const double *eps, double tol,
                 const int64_t *nu, int64_t nsys, int f, int f_s, float *x_out, int32_t *iters, int32_t *broke,
                 int32_t *breakdowns, cudaStream_t st) {
    if (f > 120 || (a_stride % 8) != 0 || (reinterpret_cast<uintptr_t>(a) & 15) != 0) return -1;
    if (nsys == 0) return CMF_OK;
    const char *pe = getenv("CMF_CG_PIPELINED");
    tc::CgTcArgs g{static_cast<const __half *>(a), a_stride, b, x0, eps, tol, nu, nsys, f, f_s, x_out, iters,
                   broke, breakdowns, pe ? atoi(pe) : 0};
    const int kp = (f + 15) / 16 * 16;
    switch (kp) {
        case 16: return launch_cg_tc<16>(g, st);
        case 32: return launch_cg_tc<32>(g, st);
        case 48: return launch_cg_tc<48>(g, st);
        case 64: return launch_cg_tc<64>(g, st);
        case 80: return launch_cg_tc<80>(g, st);
        case 96: return launch_cg_tc<96>(g, st);
        case 112: return launch_cg_tc<112>(g, st);
        default: return launch_cg_tc<128>(g, st);
    }
}

}  // namespace cmf
