// Shared pieces of the tcgen05 Gram kernels (gram_tc.cu, fused_cg.cu):
// PTX wrappers, the swizzled UMMA operand layout, the TMA gather producer and
// the single-thread MMA issuer.
//
// Operand layout (one pipeline stage = KS = 64 gathered factor rows):
//   the stage holds the K x 128 operand "Theta_S^T" (feature rows, gathered
//   columns) as an MN-major, 128-byte-swizzled UMMA operand:
//     MN-block mb (features 64mb .. 64mb+63)          stride LBO = 8192 B
//     K-block  kb (gathered rows 8kb .. 8kb+7)        stride SBO = 1024 B
//     inside the 1024 B atom: gathered row r = k%8 at r*128 B, and the 16-byte
//     chunk cb (features 8cb .. 8cb+7 of the block) at ((cb ^ r) << 4).
//   A gathered binary16 factor row is W/8 contiguous 16-byte chunks in global
//   memory that land in one 128-byte atom row per MN-block; the cp.async
//   gather maps consecutive lanes to consecutive chunks of the same row, so a
//   warp instruction reads two whole rows (coalesced) and writes them
//   conflict-free.  (A TMA tile::gather4 writes the same layout, but measured
//   on B200 its per-request cost caps a 128-byte-row gather near 3 TB/s;
//   the LSU path is faster for this access pattern.)
//   The SAME stage is the A operand (M = 128 feature rows) and the B operand
//   (N = roundup16(W + 2) rows) of kind::f16 MMAs with fp32 TMEM
//   accumulation: D = Theta_S^T Theta_S.  Operand rows W and W+1 (just past
//   the shadow's zero-padded width W = roundup8(f)) carry the row's ratings as
//   fp16 hi/lo, so accumulator columns W, W+1 hold the two halves of
//   b_u = Theta_S^T r: the bias rides in the same MMAs.  Those rows sit in a
//   16-byte chunk no cp.async writes, so the producer stores them directly.
//   (Accumulator ROWS W, W+1 hold rating-weighted sums too and are ignored.)
#pragma once

#include "common.cuh"

namespace cmf {
namespace tc {

constexpr int KS = 64;
constexpr int M = 128;
constexpr int MNBLK_BYTES = 8192;  // LBO
constexpr int KBLK_BYTES = 1024;   // SBO
constexpr int STAGE_BYTES = 2 * MNBLK_BYTES;

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
// try_wait with a suspend-time hint: the warp sleeps in hardware until the
// phase flips (or the hint expires) instead of spinning on issue slots.
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity), "r"(0x989680u)
            : "memory");
    } while (!ok);
}
// Same, but spinning with plain try_wait and a nanosleep backoff: for waiters
// that are not latency critical (producers facing a full ring; CG groups
// waiting for long rows use a longer cap so idle warps stay off the issue slots).
template <uint32_t NS0 = 32, uint32_t NSMAX = 512>
__device__ __forceinline__ void mbar_wait_backoff(uint32_t a, uint32_t parity) {
    uint32_t ok = 0, ns = NS0;
    while (true) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
        if (ok) return;
        __nanosleep(ns);
        if (ns < NSMAX) ns <<= 1;
    }
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(0), "r"(0), "r"(0), "r"(0)
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ int lane_id() { return static_cast<int>(threadIdx.x & 31); }
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t slot_s, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot_s), "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t base, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols) : "memory");
}

// ------------------------------------------------------------------ async copies
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// byte address of (gathered row k, 16-byte feature chunk c) inside a stage
__device__ __forceinline__ uint32_t operand_addr(uint32_t stage, int k, int c) {
    return stage + (c >> 3) * MNBLK_BYTES + (k >> 3) * KBLK_BYTES + (k & 7) * 128 + (((c & 7) ^ (k & 7)) << 4);
}

// UMMA shared-memory descriptor, MN-major, 128-byte swizzle (cute make_umma_desc:
// LBO = MN-block stride, SBO = K-block stride for swizzled MN-major layouts).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((MNBLK_BYTES >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((KBLK_BYTES >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;  // version (sm100)
    d |= static_cast<uint64_t>(2) << 61;  // SWIZZLE_128B
    return d;
}
// kind::f16 instruction descriptor: F16 x F16 -> F32, A and B MN-major.
__host__ __device__ constexpr uint32_t make_idesc(int m, int n) {
    return (1u << 4) | (0u << 7) | (0u << 10) | (1u << 15) | (1u << 16) | (static_cast<uint32_t>(n >> 3) << 17) |
           (static_cast<uint32_t>(m >> 4) << 24);
}


struct GatherArgs {
    const int64_t *indptr;
    const int32_t *indices;
    const float *values;   // ratings (b weights); nullptr -> zero bias
    int64_t nrows;
    int f;
    int ncols;             // rows of the fixed factors; the shadow's row ncols is all zeros
    long long *trace;      // debug timeline (CMF_TRACE builds), else unused
    int32_t *overflow;     // set when a rating does not fit its binary16 hi half (nullable)
    // Segmented gather (two passes over the fixed side, fused_cg.cu): pass 1
    // gathers positions [indptr[u], seg[u]) of each row, pass 2 [seg[u],
    // indptr[u+1]); pass 0 (default) the whole row.
    const int64_t *seg;
    int pass;
    // pass 3 (multi-pass split Gram, gram_tc.cu): positions [seg[u], seg_end[u])
    const int64_t *seg_end;
};

// Gather range of row u in the current pass.
__device__ __forceinline__ void row_segment(const GatherArgs &g, int64_t u, int64_t &b, int64_t &e) {
    b = g.indptr[u];
    e = g.indptr[u + 1];
    if (g.pass == 1) e = g.seg[u];
    else if (g.pass == 2) b = g.seg[u];
    else if (g.pass == 3) {
        b = g.seg[u];
        e = g.seg_end[u];
    }
}

// Operand ring of NST stages + NBUF TMEM accumulator hand-offs (mbarriers:
// full[NST], empty[NST], tfull[NBUF], tempty[NBUF]).
// Stage = [hi operand 16 KB | lo operand 16 KB (SPLIT only)].
// SPLIT: hi/lo binary16 halves of the factors (split-fp16 Gram,
// D = H H^T + H L^T + L H^T; the ratings live in H only, so b = (H + L)^T r).
template <int NST, bool SPLIT = false, int NBUF = 2>
struct Pipe {
    static constexpr int kStages = NST;
    static constexpr int kBufs = NBUF;
    static constexpr int kBars = 2 * NST + 2 * NBUF;
    static constexpr int kStageBytes = (SPLIT ? 2 : 1) * STAGE_BYTES;
    uint32_t stage_s, bar_s;
    __device__ uint32_t full(int s) const { return bar_s + 8u * s; }
    __device__ uint32_t empty(int s) const { return bar_s + 8u * (NST + s); }
    __device__ uint32_t tfull(int b) const { return bar_s + 8u * (2 * NST + b); }
    __device__ uint32_t tempty(int b) const { return bar_s + 8u * (2 * NST + NBUF + b); }
    __device__ uint32_t stage(int s) const { return stage_s + s * kStageBytes; }
};

// Walk over pipeline stages: (row u, first position q0 of the K-chunk) pairs
// in the order every role visits them.
struct StageIter {
    int64_t u, q0, p1;
    int64_t nrows, rstride;
    const GatherArgs *g;
    __device__ bool valid() const { return u < nrows; }
    __device__ void first(int64_t row0) {
        for (u = row0; u < nrows; u += rstride) {
            row_segment(*g, u, q0, p1);
            if (p1 > q0) return;
        }
    }
    __device__ void next() {
        q0 += KS;
        if (q0 < p1) return;
        for (u += rstride; u < nrows; u += rstride) {
            row_segment(*g, u, q0, p1);
            if (p1 > q0) return;
        }
    }
    // k stages on: jumps within a row, visits only the rows it crosses
    __device__ void advance(int k) {
        while (k > 0 && valid()) {
            const int64_t left = (p1 - q0 + KS - 1) / KS;  // stages of this row from q0 on
            if (k < left) {
                q0 += static_cast<int64_t>(k) * KS;
                return;
            }
            k -= static_cast<int>(left);
            q0 = p1;  // past the row's last stage:
            next();   // the first stage of the next non-empty row
        }
    }
};

// (index, rating) of positions q0 + lane and q0 + 32 + lane of a stage; positions past
// the row (and ids outside the shadow) read as index ncols: the shadow's zero
// padding row.
struct StagePairs {
    int idx[2];
    float val[2];
    __device__ void load(const GatherArgs &g, const StageIter &st, int lane) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t q = st.q0 + 32 * h + lane;
            const bool ok = st.valid() && q < st.p1;
            // no use of the loaded value here: the loads stay in flight until the
            // stage is produced (clamp_ids), two stages later
            idx[h] = g.ncols;
            val[h] = 0.0f;
            if (ok) {
                idx[h] = __ldcs(g.indices + q);
                if (g.values) val[h] = __ldcs(g.values + q);
            }
        }
    }
    // ids outside [0, ncols) gather the zero row (memory safety for bad input)
    __device__ void clamp_ids(int ncols) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
            idx[h] = static_cast<int>(min(static_cast<unsigned>(idx[h]), static_cast<unsigned>(ncols)));
    }
};

// Debug timeline (cmf_debug_trace, compiled in only with -DCMF_TRACE): CTA 0
// records clock64 per pipeline stage it < TRACE_STAGES: [8*it + 0] producer
// starts waiting for the slot, +1 slot free, +2 copies issued, +3 MMA sees
// full, +4 MMA committed; and per consumer row r < 2048 at [32768 + 4r + k].
// The buffer pointer travels in GatherArgs::trace (kernel parameter), so a
// stamp costs one clock read and one store.
constexpr int TRACE_STAGES = 4096;
static long long *g_trace_buf = nullptr;  // host side, set by cmf_debug_trace
static inline int set_trace_buf(void *buf) {
    g_trace_buf = static_cast<long long *>(buf);
    return CMF_OK;
}
__device__ __forceinline__ void trace_at(long long *t, uint32_t idx) {
#ifdef CMF_TRACE
    if (t != nullptr && blockIdx.x == 0) t[idx] = clock64();
#else
    (void)t;
    (void)idx;
#endif
}

// base + ix * stride as one IMAD.WIDE.U32 (keeps the compiler from splitting
// the 64-bit add and re-loading the base every row)
__device__ __forceinline__ uint64_t row_addr(uint64_t base, uint32_t ix, uint32_t stride) {
    uint64_t a;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(a) : "r"(ix), "r"(stride), "l"(base));
    return a;
}

// Producer warp `pw` of `nprod`: fills every stage `it` with it % nprod == pw.
// The (index, rating) pairs are loaded two of the warp's stages ahead, so the
// index-load latency stays off the ring.  Per stage: each lane stores the
// fp16 hi/lo ratings of positions lane, lane+32 into operand rows W, W+1 (one
// 32-bit store each), then the warp gathers the 64 factor rows with cp.async:
// lanes 0-15 / 16-31 take rows 2t / 2t+1, lane c%16
// copies 16-byte chunk c of the row (a warp instruction reads two whole rows,
// coalesced, and writes them conflict-free into the swizzled operand).  Rows
// past the end of the CSR row up to the next 16-row K-step copy the shadow's
// zero row; rows beyond are never read by the MMA and are skipped.  L2
// evict_last keeps the fixed factors' shadow resident.  Completion: 32
// cp.async.mbarrier.arrive.noinc (one per lane) + one release arrive by lane 0
// after the rating stores, so full[s] expects 33 arrivals per stage.
template <int NST, bool SPLIT, int NBUF>
__device__ void produce(const GatherArgs &g, const __half *fixed16, const __half *fixed16_lo, int W,
                        const Pipe<NST, SPLIT, NBUF> &pp, int pw, int nprod, int lane, int64_t row0,
                        int64_t rstride) {
    const uint64_t pol = policy_evict_last();
    StageIter cur{0, 0, 0, g.nrows, rstride, &g};
    cur.first(row0);
    cur.advance(pw);
    // three in-flight stages in a static ring: slot k always holds its own
    // registers (no register moves), so the index/rating loads issued for a
    // stage are not waited on until that stage is produced
    StageIter st[3];
    st[0] = cur;
    st[1] = st[0];
    st[1].advance(nprod);
    st[2] = st[1];
    st[2].advance(nprod);
    StagePairs q[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) q[k].load(g, st[k], lane);
    const int c = lane & 15, hrow = lane >> 4;
    const bool live = c < (W >> 3);
    const uint32_t W2 = static_cast<uint32_t>(W) * 2;
    const uint64_t src_hi = reinterpret_cast<uint64_t>(fixed16) + c * 16;
    const uint64_t src_lo = reinterpret_cast<uint64_t>(fixed16_lo) + c * 16;
    // swizzled destination of (row 2t + hrow, chunk c): depends on t only via
    // t & 3 (row within the 8-row atom) and t >> 2 (K-block, +1024 B)
    uint32_t dst_off[4];
#pragma unroll
    for (int t4 = 0; t4 < 4; ++t4) dst_off[t4] = operand_addr(0, 2 * t4 + hrow, c);
    // rating slots: operand row k, chunk W/8 (halves 0, 1 = features W, W+1)
    uint32_t r_off[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) r_off[h] = operand_addr(0, 32 * h + lane, W >> 3);
    uint32_t it = pw;
    auto stage_out = [&](const StageIter &cs, StagePairs &c0) {
        const int s = it % NST;
        const int nrem16 = static_cast<int>(min(static_cast<int64_t>(KS), cs.p1 - cs.q0) + 15) & ~15;
        c0.clamp_ids(g.ncols);
        if (lane == 0 && it < TRACE_STAGES) trace_at(g.trace, 8 * it + 0);
        mbar_wait_backoff(pp.empty(s), ((it / NST) & 1) ^ 1);
        if (lane == 0 && it < TRACE_STAGES) trace_at(g.trace, 8 * it + 1);
        const uint32_t stg = pp.stage(s);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const __half hi = __float2half_rn(c0.val[h]);
            if (fabsf(c0.val[h]) >= 65520.0f && g.overflow) *g.overflow = 1;
            const __half lo = __float2half_rn(c0.val[h] - __half2float(hi));
            const uint32_t v = static_cast<uint32_t>(__half_as_ushort(hi)) |
                               (static_cast<uint32_t>(__half_as_ushort(lo)) << 16);
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(stg + r_off[h]), "r"(v) : "memory");
        }
        fence_proxy_async();  // generic-proxy rating stores -> tensor-core reads
        __syncwarp();
        if (lane == 0) mbar_arrive(pp.full(s));  // release: the rating stores
#pragma unroll
        for (int t = 0; t < KS / 2; ++t) {
            if ((t & 7) == 0 && 2 * t >= nrem16) break;  // whole K-steps only (warp-uniform)
            // row 2t + hrow: position (2t + hrow) & 31 of register half t >> 4
            const uint32_t ix = static_cast<uint32_t>(__shfl_sync(0xffffffffu, c0.idx[t >> 4], (2 * t + hrow) & 31));
            const uint32_t dst = stg + dst_off[t & 3] + (t >> 2) * KBLK_BYTES;
            if (live) {
                asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst),
                             "l"(row_addr(src_hi, ix, W2)), "l"(pol)
                             : "memory");
                if (SPLIT)
                    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(
                                     dst + STAGE_BYTES),
                                 "l"(row_addr(src_lo, ix, W2)), "l"(pol)
                                 : "memory");
            }
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(pp.full(s)) : "memory");
        if (lane == 0 && it < TRACE_STAGES) trace_at(g.trace, 8 * it + 2);
        it += nprod;
    };
    // slot k's next stage is three of this warp's stages on: the stage after slot (k+2)'s
    while (true) {
        if (!st[0].valid()) break;
        stage_out(st[0], q[0]);
        st[0] = st[2];
        st[0].advance(nprod);
        q[0].load(g, st[0], lane);
        if (!st[1].valid()) break;
        stage_out(st[1], q[1]);
        st[1] = st[0];
        st[1].advance(nprod);
        q[1].load(g, st[1], lane);
        if (!st[2].valid()) break;
        stage_out(st[2], q[2]);
        st[2] = st[1];
        st[2].advance(nprod);
        q[2].load(g, st[2], lane);
    }
}

// Implicit-feedback producers (Pipe<NST, true, NBUF> stages = [gathered rows |
// weighted copy]), two decoupled roles so that no warp waits on its own copies:
//   gather_weighted (warp pw of ngath): stage it = pw, pw + ngath, ...: wait for
//     the slot, gather the 64 factor rows with cp.async into the first half
//     exactly as produce() does, and let the copies arrive on landed[s] (32
//     noinc arrivals, one per lane);
//   scale_weighted (warp pw of nscal): stage it = pw, pw + nscal, ...: load the
//     stage's ratings, wait for landed[s], write the weighted copy
//     w_k theta_k (w = alpha r_k, binary16 HMUL2) and the confidence rows
//     c_k = 1 + alpha r_k (fp16 hi/lo, operand rows W, W+1) into the second
//     half, fence, and arrive on full[s] (count 1).
// The MMA then reads gathered x weighted: D = sum_k theta_k (alpha r_k theta_k)^T
// and D[:, W] + D[:, W+1] = sum_k c_k theta_k (implicit.py:63-84).
template <int NST, int NBUF>
__device__ void gather_weighted(const GatherArgs &g, const __half *fixed16, int W, const Pipe<NST, true, NBUF> &pp,
                                uint32_t landed, int pw, int ngath, int lane, int64_t row0, int64_t rstride) {
    const uint64_t pol = policy_evict_last();
    StageIter cur{0, 0, 0, g.nrows, rstride, &g};
    cur.first(row0);
    cur.advance(pw);
    const int c = lane & 15, hrow = lane >> 4;
    const bool live = c < (W >> 3);
    const uint32_t W2 = static_cast<uint32_t>(W) * 2;
    const uint64_t src_hi = reinterpret_cast<uint64_t>(fixed16) + c * 16;
    uint32_t dst_off[4];
#pragma unroll
    for (int t4 = 0; t4 < 4; ++t4) dst_off[t4] = operand_addr(0, 2 * t4 + hrow, c);
    uint32_t it = pw;
    StagePairs qn;  // the next stage's pairs, loaded one stage ahead
    qn.load(g, cur, lane);
    while (cur.valid()) {
        StagePairs q = qn;
        const int nrem16 = static_cast<int>(min(static_cast<int64_t>(KS), cur.p1 - cur.q0) + 15) & ~15;
        cur.advance(ngath);
        qn.load(g, cur, lane);
        const int s = it % NST;
        q.clamp_ids(g.ncols);
        if (lane == 0 && it < TRACE_STAGES) trace_at(g.trace, 8 * it + 0);
        mbar_wait_backoff(pp.empty(s), ((it / NST) & 1) ^ 1);
        if (lane == 0 && it < TRACE_STAGES) trace_at(g.trace, 8 * it + 1);
        const uint32_t stg = pp.stage(s);
#pragma unroll
        for (int t = 0; t < KS / 2; ++t) {
            if ((t & 7) == 0 && 2 * t >= nrem16) break;
            const uint32_t ix = static_cast<uint32_t>(__shfl_sync(0xffffffffu, q.idx[t >> 4], (2 * t + hrow) & 31));
            const uint32_t dst = stg + dst_off[t & 3] + (t >> 2) * KBLK_BYTES;
            if (live)
                asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst),
                             "l"(row_addr(src_hi, ix, W2)), "l"(pol)
                             : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(landed + 8u * s) : "memory");
        if (lane == 0 && it < TRACE_STAGES) trace_at(g.trace, 8 * it + 2);
        it += ngath;
    }
}

#ifndef CMF_SCALE_BATCH
#define CMF_SCALE_BATCH 4
#endif
template <int NST, int NBUF>
__device__ void scale_weighted(const GatherArgs &g, int W, float alpha, const Pipe<NST, true, NBUF> &pp,
                               uint32_t landed, int pw, int nscal, int lane, int64_t row0, int64_t rstride) {
    constexpr int SB = CMF_SCALE_BATCH;
    StageIter cur{0, 0, 0, g.nrows, rstride, &g};
    cur.first(row0);
    cur.advance(pw);
    const int c = lane & 15, hrow = lane >> 4;
    uint32_t dst_off[4];
#pragma unroll
    for (int t4 = 0; t4 < 4; ++t4) dst_off[t4] = operand_addr(0, 2 * t4 + hrow, c);
    uint32_t r_off[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) r_off[h] = operand_addr(0, 32 * h + lane, W >> 3);
    uint32_t it = pw;
    StagePairs qn;
    qn.load(g, cur, lane);
    while (cur.valid()) {
        const float pv0 = qn.val[0], pv1 = qn.val[1];
        const int n16 = static_cast<int>(min(static_cast<int64_t>(KS), cur.p1 - cur.q0) + 15) & ~15;
        cur.advance(nscal);
        qn.load(g, cur, lane);
        const int s = it % NST;
        const uint32_t stg = pp.stage(s), wst = stg + STAGE_BYTES;
        // the slot's previous stage (it - NST) consumed first: then landed[s] is at
        // most one phase ahead of this wait (parity waits alias two phases apart;
        // valid while nscal <= NST, see the caller)
        mbar_wait_backoff(pp.empty(s), ((it / NST) & 1) ^ 1);
        mbar_wait(landed + 8u * s, (it / NST) & 1);  // the gathered rows of stage it are in
        if (lane == 0 && it < TRACE_STAGES) trace_at(g.trace, 8 * it + 5);
        // the weights as replicated binary16 pairs, one conversion per rating
        const __half2 hw0 = __float2half2_rn(alpha * pv0), hw1 = __float2half2_rn(alpha * pv1);
        const uint32_t w0 = *reinterpret_cast<const uint32_t *>(&hw0), w1 = *reinterpret_cast<const uint32_t *>(&hw1);
        // SB row pairs at a time, all loads first.  No lane predicate: the lanes
        // past the shadow width (chunks c >= W/8) scale stale chunks into operand
        // rows >= W that feed only accumulator columns the repack discards (rows
        // W, W+1 are rewritten below), which keeps the loop free of branches.
#pragma unroll
        for (int t0 = 0; t0 < KS / 2; t0 += SB) {
            if ((t0 & 7) == 0 && 2 * t0 >= n16) break;
            uint4 v[SB];
#pragma unroll
            for (int k = 0; k < SB; ++k) {
                const uint32_t off = dst_off[(t0 + k) & 3] + ((t0 + k) >> 2) * KBLK_BYTES;
                asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w)
                             : "r"(stg + off));
            }
#pragma unroll
            for (int k = 0; k < SB; ++k) {
                const int t = t0 + k;
                const uint32_t w = __shfl_sync(0xffffffffu, t < 16 ? w0 : w1, (2 * t + hrow) & 31);
                const uint32_t off = dst_off[t & 3] + (t >> 2) * KBLK_BYTES;
                auto mul = [&](uint32_t x) {
                    __half2 y = __hmul2(*reinterpret_cast<const __half2 *>(&x), *reinterpret_cast<const __half2 *>(&w));
                    return *reinterpret_cast<const uint32_t *>(&y);
                };
                asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(wst + off), "r"(mul(v[k].x)),
                             "r"(mul(v[k].y)), "r"(mul(v[k].z)), "r"(mul(v[k].w))
                             : "memory");
            }
        }
        __syncwarp();  // the stale-chunk stores above land before the rating rows
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float wv = alpha * (h ? pv1 : pv0);
            const float cv = 1.0f + wv;
            if ((fabsf(wv) >= 65520.0f || fabsf(cv) >= 65520.0f) && g.overflow) *g.overflow = 1;
            const __half hi = __float2half_rn(cv);
            const __half lo = __float2half_rn(cv - __half2float(hi));
            const uint32_t v = static_cast<uint32_t>(__half_as_ushort(hi)) |
                               (static_cast<uint32_t>(__half_as_ushort(lo)) << 16);
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(wst + r_off[h]), "r"(v) : "memory");
        }
        fence_proxy_async();  // generic-proxy stores -> tensor-core reads
        __syncwarp();
        if (lane == 0) mbar_arrive(pp.full(s));
        if (lane == 0 && it < TRACE_STAGES) trace_at(g.trace, 8 * it + 6);
        it += nscal;
    }
}

__device__ __forceinline__ uint32_t elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(pred));
    return pred;
}

// MMA issuer, run by a whole warp (warp-uniform control flow keeps the
// descriptors in uniform registers; one elected lane issues): one accumulator
// chain per non-empty row into TMEM buffer (row counter % NBUF), one 128 x N
// MMA per 16-row K-step; releases stages with tcgen05.commit.  Buffer b
// occupies columns [b*N, (b+1)*N).  The next row's extent is loaded one row
// ahead so the indptr latency stays off the issue loop.
// SYM (split operands only): two chains per row, H H^T into [2bN, 2bN + N) and
// S = H^T L into [2bN + N, 2bN + 2N); the epilogue adds S^T (= the L H^T term),
// so each K-step reads its operands from shared memory twice instead of three times.
template <int NST, bool SPLIT, int NBUF, bool WEIGHTED = false, bool SYM = false>
__device__ __forceinline__ void issue_mma(const GatherArgs &g, const Pipe<NST, SPLIT, NBUF> &pp, uint32_t tmem_base,
                                          int N, int64_t row0, int64_t rstride, uint32_t cons_full = 0,
                                          int ncons = 0) {
    const uint32_t idesc = make_idesc(M, N);
    const uint64_t desc0 = make_desc(pp.stage(0));
    // descriptor start address field is (addr >> 4): stage s, K-step kk adds
    // (s * kStageBytes + kk * 2048) >> 4; the lo operand adds STAGE_BYTES >> 4
    constexpr uint32_t kStageStep = Pipe<NST, SPLIT, NBUF>::kStageBytes >> 4;
    constexpr uint32_t kKStep = (2 * KBLK_BYTES) >> 4;
    constexpr uint32_t kLoStep = STAGE_BYTES >> 4;
    uint32_t it = 0, rowc = 0;
    int64_t u = row0;
    // rows with ratings get an accumulator hand-off (p0 < p1); in a segmented
    // pass the MMAs cover the row's segment [s0, s1) only, which may be empty
    // (then the commit announces an untouched buffer; the consumer knows)
    int64_t p0 = u < g.nrows ? g.indptr[u] : 0, p1 = u < g.nrows ? g.indptr[u + 1] : 0;
    int64_t s0 = p0, s1 = p1;
    if (g.pass && u < g.nrows) row_segment(g, u, s0, s1);
    while (u < g.nrows) {
        const int64_t un = u + rstride;
        const int64_t q0n = un < g.nrows ? g.indptr[un] : 0, q1n = un < g.nrows ? g.indptr[un + 1] : 0;
        int64_t t0n = q0n, t1n = q1n;
        if (g.pass && un < g.nrows) row_segment(g, un, t0n, t1n);
        if (p1 > p0) {
            const int b = rowc % NBUF;
            mbar_wait(pp.tempty(b), ((rowc / NBUF) & 1) ^ 1);
            tc_fence_after();
            const uint32_t tmem_d = tmem_base + b * N * (SYM ? 2 : 1);
            uint32_t acc = 0;
            for (int64_t q0 = s0; q0 < s1; q0 += KS, ++it) {
                const int s = it % NST;
                mbar_wait(pp.full(s), (it / NST) & 1);
                if (lane_id() == 0 && it < TRACE_STAGES) trace_at(g.trace, 8 * it + 3);
                tc_fence_after();
                const int nk = static_cast<int>(min(static_cast<int64_t>(KS), s1 - q0) + 15) >> 4;
                const uint64_t ds = desc0 + s * kStageStep;
                if (elect_one()) {
                    for (int kk = 0; kk < nk; ++kk) {
                        const uint64_t d = ds + kk * kKStep;
                        if (WEIGHTED) {  // gathered rows x weighted copy (+ the confidence rows)
                            tc_mma(tmem_d, d, d + kLoStep, idesc, acc | kk);
                            continue;
                        }
                        tc_mma(tmem_d, d, d, idesc, acc | kk);
                        if (SPLIT && SYM) {  // S = H^T L in the second accumulator
                            tc_mma(tmem_d + N, d, d + kLoStep, idesc, acc | kk);
                        } else if (SPLIT) {  // + H L^T + L H^T
                            tc_mma(tmem_d, d, d + kLoStep, idesc, 1);
                            tc_mma(tmem_d, d + kLoStep, d, idesc, 1);
                        }
                    }
                    tc_commit(pp.empty(s));
                }
                __syncwarp();
                acc = 1;
                if (lane_id() == 0 && it < TRACE_STAGES) trace_at(g.trace, 8 * it + 4);
            }
            // announce the accumulator: on the buffer's barrier, or (ncons > 0) on
            // the barrier of the consumer that owns row rowc (rowc % ncons), so that
            // each consumer waits on its own phase sequence
            if (elect_one()) tc_commit(ncons ? cons_full + 8u * (rowc % ncons) : pp.tfull(b));
            __syncwarp();
            ++rowc;
        }
        u = un;
        p0 = q0n;
        p1 = q1n;
        s0 = t0n;
        s1 = t1n;
    }
}

// Zero-initialise the operand ring (chunks past the rating slots are never
// written again) and the barriers; call from all threads, then sync.
template <int NST, bool SPLIT, int NBUF>
__device__ void pipe_init(const Pipe<NST, SPLIT, NBUF> &pp, unsigned char *stage_mem, int nthreads,
                          uint32_t full_count, uint32_t tempty_count) {
    for (int i = threadIdx.x; i < NST * Pipe<NST, SPLIT, NBUF>::kStageBytes / 16; i += nthreads)
        reinterpret_cast<int4 *>(stage_mem)[i] = make_int4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(pp.full(s), full_count);
            mbar_init(pp.empty(s), 1);
        }
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(pp.tfull(b), 1);
            mbar_init(pp.tempty(b), tempty_count);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
}

}  // namespace tc
}  // namespace cmf
