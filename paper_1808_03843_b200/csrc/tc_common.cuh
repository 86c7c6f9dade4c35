// Shared pieces of the tcgen05 Gram kernels (gram_tc.cu, fused_cg.cu):
// PTX wrappers, the swizzled UMMA operand layout, the cp.async gather producer
// and the single-thread MMA issuer.
//
// Operand layout (one pipeline stage = KS = 64 gathered factor rows):
//   the stage holds the K x 128 operand "Theta_S^T" (feature rows, gathered
//   columns) as an MN-major, 128-byte-swizzled UMMA operand:
//     MN-block mb (features 64mb .. 64mb+63)          stride LBO = 8192 B
//     K-block  kb (gathered rows 8kb .. 8kb+7)        stride SBO = 1024 B
//     inside the 1024 B atom: gathered row r = k%8 at r*128 B, and the 16-byte
//     chunk cb (features 8cb .. 8cb+7 of the block) at ((cb ^ r) << 4).
//   A gathered binary16 factor row is therefore 13 contiguous 16-byte chunks in
//   global memory that land in one 128-byte atom row per MN-block; the gather
//   maps consecutive lanes to consecutive chunks of the same row, so a warp
//   instruction reads two whole rows (coalesced) and writes conflict-free.
//   The SAME stage is the A operand (M = 128 feature rows) and the B operand
//   (N = roundup16(f+2) feature rows) of kind::f16 MMAs with fp32 TMEM
//   accumulation: D = Theta_S^T Theta_S.  Rows f and f+1 of the operand carry
//   the row's ratings (fp16 hi + lo), so D[:, f] + D[:, f+1] = b_u.
#pragma once

#include "common.cuh"

namespace cmf {
namespace tc {

constexpr int KS = 64;
constexpr int M = 128;
constexpr int MNBLK_BYTES = 8192;  // LBO
constexpr int KBLK_BYTES = 1024;   // SBO
constexpr int STAGE_BYTES = 2 * MNBLK_BYTES;
constexpr int TMEM_COLS = 256;

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
// that are not latency critical (producers facing a full ring).
__device__ __forceinline__ void mbar_wait_backoff(uint32_t a, uint32_t parity) {
    uint32_t ok = 0, ns = 32;
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
        if (ns < 512) ns <<= 1;
    }
}
__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint32_t bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
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

// v.{x,y,z,w} as 8 halves; set half `pos` (runtime) without a local array
__device__ __forceinline__ void set_half(uint4 &v, int pos, uint16_t h) {
    const uint32_t sh = (pos & 1) * 16, keep = ~(0xFFFFu << sh), val = static_cast<uint32_t>(h) << sh;
    const int w = pos >> 1;
    v.x = w == 0 ? (v.x & keep) | val : v.x;
    v.y = w == 1 ? (v.y & keep) | val : v.y;
    v.z = w == 2 ? (v.z & keep) | val : v.z;
    v.w = w == 3 ? (v.w & keep) | val : v.w;
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
    const float *values;   // ratings (b weights); nullptr -> zero bias rows
    const __half *fixed16; // (ncols, W) binary16 shadow, W = NCH * 8
    const __half *fixed16_lo;  // split mode: binary16 residual shadow (same layout)
    int64_t nrows;
    int f;
};

// Operand ring of NST stages + 2 TMEM accumulator hand-offs (mbarriers:
// full[NST], empty[NST], tfull[2], tempty[2]).
// SPLIT: every stage holds two operands, hi then lo (split-fp16 Gram,
// D = H H^T + H L^T + L H^T), so the stage stride doubles.
template <int NST, bool SPLIT = false>
struct Pipe {
    static constexpr int kStages = NST;
    static constexpr int kBars = 2 * NST + 4;
    static constexpr int kStageBytes = (SPLIT ? 2 : 1) * STAGE_BYTES;
    uint32_t stage_s, bar_s;
    __device__ uint32_t full(int s) const { return bar_s + 8u * s; }
    __device__ uint32_t empty(int s) const { return bar_s + 8u * (NST + s); }
    __device__ uint32_t tfull(int b) const { return bar_s + 8u * (2 * NST + b); }
    __device__ uint32_t tempty(int b) const { return bar_s + 8u * (2 * NST + 2 + b); }
    __device__ uint32_t stage(int s) const { return stage_s + s * kStageBytes; }
};

// Walk over pipeline stages: (row u, first position q0 of the K-chunk) pairs
// in the order every role visits them.
struct StageIter {
    int64_t u, q0, p1;
    int64_t nrows, rstride;
    const int64_t *indptr;
    __device__ bool valid() const { return u < nrows; }
    __device__ void first(int64_t row0) {
        for (u = row0; u < nrows; u += rstride) {
            q0 = indptr[u];
            p1 = indptr[u + 1];
            if (p1 > q0) return;
        }
    }
    __device__ void next() {
        q0 += KS;
        if (q0 < p1) return;
        for (u += rstride; u < nrows; u += rstride) {
            q0 = indptr[u];
            p1 = indptr[u + 1];
            if (p1 > q0) return;
        }
    }
};

// Producer warp `pw` of `nprod`: fills every stage `it` with it % nprod == pw.
// The (index, rating) pairs of the warp's NEXT stage are loaded while the
// current one is being gathered, so index-load latency stays off the ring.
template <int NCH, int NST, bool SPLIT>
__device__ void produce(const GatherArgs &g, const Pipe<NST, SPLIT> &pp, int pw, int nprod, int lane,
                        int64_t row0, int64_t rstride) {
    constexpr int W = NCH * 8;
    const int pf = g.f, pf1 = g.f + 1;
    const int pc0 = pf >> 3, pc1 = pf1 >> 3;
    const int c = lane & 15, hrow = lane >> 4;
    StageIter cur{0, 0, 0, g.nrows, rstride, g.indptr};
    cur.first(row0);
    for (int k = 0; k < pw && cur.valid(); ++k) cur.next();
    uint32_t it = pw;
    int idx[2] = {0, 0};
    float rv[2] = {0.0f, 0.0f};
    auto load_pairs = [&](const StageIter &st, int (&ix)[2], float (&r)[2]) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t q = st.q0 + h * 32 + lane;
            const bool ok = st.valid() && q < st.p1;
            ix[h] = ok ? g.indices[q] : 0;
            r[h] = (ok && g.values) ? g.values[q] : 0.0f;
        }
    };
    load_pairs(cur, idx, rv);
    // lanes with a plain (non-rating) chunk: 16-lane halves own rows 2t and 2t+1
    const bool c_live = c < NCH && c != pc0 && c != pc1;
    // swizzled destination of (row 2t + hrow, chunk c) minus its K-block part,
    // which depends only on t & 3 (operand_addr with k = 2t + hrow)
    uint32_t dst_off[4];
#pragma unroll
    for (int t4 = 0; t4 < 4; ++t4) dst_off[t4] = operand_addr(0, 2 * t4 + hrow, c);
    while (cur.valid()) {
        StageIter nxt = cur;
        for (int k = 0; k < nprod && nxt.valid(); ++k) nxt.next();
        int idx_n[2];
        float rv_n[2];
        load_pairs(nxt, idx_n, rv_n);
        const int64_t q0 = cur.q0, p1 = cur.p1;
        const int s = it % NST;
        // rating chunk(s) of rows lane, lane+32: loads issued before the wait
        uint4 pv[2][2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const bool ok = q0 + h * 32 + lane < p1;
            const __half *row = g.fixed16 + static_cast<int64_t>(idx[h]) * W;
            pv[h][0] = ok ? __ldg(reinterpret_cast<const uint4 *>(row + 8 * pc0)) : make_uint4(0, 0, 0, 0);
            pv[h][1] = (ok && pc1 != pc0) ? __ldg(reinterpret_cast<const uint4 *>(row + 8 * pc1))
                                          : make_uint4(0, 0, 0, 0);
        }
        mbar_wait_backoff(pp.empty(s), ((it / NST) & 1) ^ 1);
        const uint32_t stg = pp.stage(s);
        const int nrem = static_cast<int>(min(static_cast<int64_t>(KS), p1 - q0));
#pragma unroll
        for (int t = 0; t < KS / 2; ++t) {
            const int k = 2 * t + hrow;
            // every lane holds (index) pairs for rows lane and lane + 32: full-warp shuffle
            const int ix = __shfl_sync(0xffffffffu, t < 16 ? idx[0] : idx[1], k & 31);
            const bool valid = k < nrem;
            const int64_t off = static_cast<int64_t>(ix) * W + 8 * c;
            const __half *src = valid ? g.fixed16 + off : g.fixed16;
            const uint32_t dst = stg + dst_off[t & 3] + (t >> 2) * KBLK_BYTES;
            if (c_live) cp_async16_zfill(dst, src, valid ? 16u : 0u);
            if (SPLIT && c < NCH)  // residual operand: every chunk (its rating slots stay zero)
                cp_async16_zfill(dst + STAGE_BYTES, valid ? g.fixed16_lo + off : g.fixed16_lo, valid ? 16u : 0u);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int k = h * 32 + lane;
            const bool ok = q0 + k < p1;
            const __half hi = __float2half_rn(rv[h]);
            const __half lo = __float2half_rn(rv[h] - __half2float(hi));
            uint4 v0 = pv[h][0], v1 = pv[h][1];
            if (ok) {
                set_half(v0, pf & 7, __half_as_ushort(hi));
                if (pc1 == pc0) set_half(v0, pf1 & 7, __half_as_ushort(lo));
                else set_half(v1, pf1 & 7, __half_as_ushort(lo));
            }
            const uint32_t d0 = operand_addr(stg, k, pc0);
            asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(d0), "r"(v0.x), "r"(v0.y), "r"(v0.z),
                         "r"(v0.w)
                         : "memory");
            if (pc1 != pc0) {
                const uint32_t d1 = operand_addr(stg, k, pc1);
                asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(d1), "r"(v1.x), "r"(v1.y), "r"(v1.z),
                             "r"(v1.w)
                             : "memory");
            }
        }
        fence_proxy_async();
        cp_async_arrive_noinc(pp.full(s));
        cur = nxt;
        idx[0] = idx_n[0];
        idx[1] = idx_n[1];
        rv[0] = rv_n[0];
        rv[1] = rv_n[1];
        it += nprod;
    }
}

// Single-thread MMA issuer: one accumulator chain per non-empty row into TMEM
// buffer (row counter & 1); releases stages with tcgen05.commit.
template <int NST, bool SPLIT>
__device__ __forceinline__ void issue_mma(const GatherArgs &g, const Pipe<NST, SPLIT> &pp, uint32_t tmem_base,
                                          int N, int64_t row0, int64_t rstride) {
    const uint32_t idesc = make_idesc(M, N);
    uint32_t it = 0, rowc = 0;
    for (int64_t u = row0; u < g.nrows; u += rstride) {
        const int64_t p0 = g.indptr[u], p1 = g.indptr[u + 1];
        if (p1 == p0) continue;
        const int b = rowc & 1;
        mbar_wait(pp.tempty(b), ((rowc >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + b * 128;
        uint32_t acc = 0;
        for (int64_t q0 = p0; q0 < p1; q0 += KS, ++it) {
            const int s = it % NST;
            mbar_wait(pp.full(s), (it / NST) & 1);
            tc_fence_after();
            const int nb = static_cast<int>(min(static_cast<int64_t>(KS), p1 - q0));
            const uint32_t sbase = pp.stage(s);
            for (int kk = 0; kk < (nb + 15) / 16; ++kk) {
                const uint64_t d = make_desc(sbase + kk * 2 * KBLK_BYTES);
                tc_mma(tmem_d, d, d, idesc, acc);
                acc = 1;
                if (SPLIT) {  // + H L^T + L H^T into the same accumulator
                    const uint64_t dl = make_desc(sbase + STAGE_BYTES + kk * 2 * KBLK_BYTES);
                    tc_mma(tmem_d, d, dl, idesc, 1);
                    tc_mma(tmem_d, dl, d, idesc, 1);
                }
            }
            tc_commit(pp.empty(s));
        }
        tc_commit(pp.tfull(b));
        ++rowc;
    }
}

}  // namespace tc
}  // namespace cmf
