// Fused half-update kernel template (tensor-core Gram -> TMEM -> truncated CG),
// shared by the explicit launcher (fused_cg.cu) and the implicit-feedback
// launcher (fused_implicit.cu, WEIGHTED operands).  See fused_cg.cu for the design.
#pragma once
#include <cstdlib>

#include "tc_common.cuh"

namespace cmf {
namespace tc {

// producer warps: the gather rate scales with issuing warps.  Short rows (the
// user side) share the SM with 4 CG groups and run 7; long rows (the item side)
// leave the 2 CG groups mostly idle and run 11.  (A producer waits on stage
// it's slot for the release of stage it - NST, which is unambiguous only while
// producers <= ring stages: 12.)
constexpr int F_PROD_SHORT = 7;
constexpr int F_PROD_LONG = 11;
constexpr int CG_THREADS = 128;
constexpr int MVB_OPERAND = 4096;  // matvec B operand: 16 rows x 128 halves, K-major SW128 (2 K-atoms)
constexpr int MVB_BYTES = 5120;    // + warp partials, 1024-aligned per group
// NG CG groups (== TMEM accumulator buffers, one warpgroup each) + 2 auxiliary
// warpgroups (7 producers + the MMA warp).  Registers are rebalanced with
// setmaxnreg: the CG warpgroups hold a register row of A_u (4*FC floats) and
// grow to CG_REGS, the auxiliary warpgroups shrink to AUX_REGS, so that
// NG*128*CG_REGS + 256*AUX_REGS == THREADS*LAUNCH_REGS <= 64K registers.
// LONG: rows averaging >= LONG_ROW_NNZ ratings (the item side): the gather
// dominates and CG is rare, and two CG groups leave the producers more of the
// SM (measured: Theta side 3.21 -> 3.03 ms at Netflix shape).
constexpr int LONG_ROW_NNZ = 1024;
// TMEM plan (512 columns): NBUF fp32 Gram accumulators of N <= NMAX columns
// each, then one binary16 A_u slot of KP/2 columns per CG group, then one
// 16-column matvec result block per group.  A group copies its row's A_u out
// of the accumulator (repacking to binary16) and frees the accumulator at once,
// so the MMA warp builds the next Grams while up to NG systems are in CG.
template <int FC, bool LONG = false>
struct FusedShape {
    static constexpr int KP = (FC * 4 + 15) / 16 * 16;         // matvec K extent
    static constexpr int SLOT = KP / 2;                         // packed binary16 A_u columns
    static constexpr int NMAX = ((FC * 4 + 7) / 8 * 8 + 2 + 15) / 16 * 16;  // accumulator width bound
    static constexpr int NG = (FC <= 26 && !LONG) ? 4 : 2;
    static constexpr int tmem_need(int nbuf) { return (nbuf * NMAX + NG * SLOT + 15) / 16 * 16 + 16 * NG; }
    static constexpr int NBUF = (LONG && tmem_need(3) <= 512) ? 3 : 2;
    static constexpr int NPROD = LONG ? F_PROD_LONG : F_PROD_SHORT;
    static constexpr int THREADS = 32 * (4 * NG + NPROD + 1);
    static constexpr int MMA_WARP = 4 * NG + NPROD;
    // 768 threads (4 CG groups + 7 producers), 640 (2 groups + 11 producers) or
    // 512 (2 groups + 7, f > 104 short rows): registers per thread at launch
    static constexpr int LAUNCH_REGS = THREADS == 768 ? 80 : (THREADS == 640 ? 96 : 128);
    static constexpr int CG_REGS = NG == 4 ? 88 : (THREADS == 640 ? 144 : 168);
    static constexpr int AUX_REGS = THREADS == 512 ? 88 : 64;
    static_assert(THREADS == 768 || THREADS == 640 || THREADS == 512, "CTA shape");
    static_assert(NPROD <= 12, "producers <= ring stages");
    static_assert(NG * 128 * CG_REGS + 32 * (NPROD + 1) * AUX_REGS <= THREADS * LAUNCH_REGS, "register budget");
    static_assert(tmem_need(NBUF) <= 512, "TMEM plan");
};

template <int R>
__device__ __forceinline__ void regs_inc() {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(R));
}
template <int R>
__device__ __forceinline__ void regs_dec() {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(R));
}

struct FusedArgs {
    GatherArgs gather;
    const __half *fixed16;  // binary16 shadow of the fixed factors (ncols, W)
    int W, N, tmem_cols;  // shadow width, accumulator width (Gram + rating columns W, W+1)
    int slot_base, dmv_base;  // TMEM columns of the A_u slots and the matvec result blocks
    double lam;
    int weighted;
    float *target;  // (nrows, f) in/out
    float *const *peers;  // device array of npeers replicas of target (rows at the same index), or null
    int npeers;
    int f_s;
    int nprod;  // active producer warps (<= the shape's NPROD; the others exit at once; <= 0: all)
    float tol;
    int32_t *breakdowns;
    int32_t *overflow;  // set when a row's A_u does not fit binary16 (NumericalError)
    // Two-pass Gram (gather.pass 1 / 2, long rows over a fixed side larger than
    // L2 can hold, or a multi-GPU reduce-scatter of partial Grams): pass 1 stores
    // each row's partial accumulator (columns [0, W+2): the first-segment Gram
    // and bias) at partial + (u*f + i)*PWS for lanes i < f; pass 2 adds it to the
    // second segment's accumulator.
    float *partial;
    int pws;  // partial row stride in floats (roundup4(W + 2))
    // Implicit feedback (WEIGHTED kernels, implicit.py:57-84): A_u = base +
    // sum_k alpha r_k theta_k theta_k^T + lam I, b_u = sum_k (1 + alpha r_k) theta_k.
    // base: F^T F as a full row-major fp32 matrix, f rows of stride 4*FC (cmf_fused_base_ld; null: none).
    const float *base;
    float alpha;
};

// 12 x 16 KB operand ring; WEIGHTED: 32 KB stages (gathered + weighted copy), as many
// as fit next to the F^T F base kept in shared memory (fp32, f x 4FC)
// shared-memory row stride of the base: >= 4FC floats and == 4 (mod 32), so that
// the 8 lanes of a quarter-warp reading float4s of their own rows hit 32 distinct banks
template <int FC>
constexpr int base_lds() { return 4 * FC + ((4 - 4 * FC) % 32 + 32) % 32; }
template <int FC>
constexpr int base_smem_bytes() { return 4 * FC * base_lds<FC>() * 4; }  // 4FC rows (>= f)
template <int FC>
constexpr int weighted_stages() {  // 32 KB stages left next to the base + 4 groups' CG scratch
    return (227 * 1024 - 1024 - 4 * 5120 - 1024 - base_smem_bytes<FC>()) / 32768 < 5
               ? (227 * 1024 - 1024 - 4 * 5120 - 1024 - base_smem_bytes<FC>()) / 32768
               : 5;
}
template <int NBUF, bool WEIGHTED = false, int FC = 25>
using FPipe = Pipe<WEIGHTED ? weighted_stages<FC>() : 12, WEIGHTED, NBUF>;

// tcgen05.ld 32x32b of N consecutive columns (N = 4, 8, 16) into v[0..N)
template <int N>
__device__ __forceinline__ void tmem_ldn(uint32_t taddr, uint32_t *v);
template <>
__device__ __forceinline__ void tmem_ldn<4>(uint32_t taddr, uint32_t *v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr)
                 : "memory");
}
template <>
__device__ __forceinline__ void tmem_ldn<8>(uint32_t taddr, uint32_t *v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr)
                 : "memory");
}
template <>
__device__ __forceinline__ void tmem_ldn<32>(uint32_t taddr, uint32_t *v) {
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
template <>
__device__ __forceinline__ void tmem_ldn<16>(uint32_t taddr, uint32_t *v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr)
        : "memory");
}
// R (< 32, a multiple of 4) consecutive columns as x16 / x8 / x4 pieces
template <int R>
__device__ __forceinline__ void tmem_ld_tail(uint32_t taddr, uint32_t *v) {
    if (R & 16) tmem_ldn<16>(taddr, v);
    if (R & 8) tmem_ldn<8>(taddr + (R & 16), v + (R & 16));
    if (R & 4) tmem_ldn<4>(taddr + (R & 24), v + (R & 24));
}

// NC (a multiple of 4) consecutive accumulator columns of this thread's lane
template <int NC>
__device__ __forceinline__ void tmem_load_row(uint32_t taddr, uint32_t (&v)[NC]) {
#pragma unroll
    for (int c = 0; c + 16 <= NC; c += 16) tmem_ldn<16>(taddr + c, v + c);
    constexpr int r = NC % 16;
    if (r & 8) tmem_ldn<8>(taddr + (NC - r), v + (NC - r));
    if (r & 4) tmem_ldn<4>(taddr + (NC - (r & 4)), v + (NC - (r & 4)));
    tmem_ld_wait();
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t *v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t *v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// D[tmem] (+)= A[tmem] * B[smem]: kind::f16, A operand read from tensor memory
__device__ __forceinline__ void tc_mma_tmem_a(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// K-major, 128-byte swizzle (8 rows x 128 B atoms, SBO = 1024 B between 8-row
// groups); a K-step adds its byte offset to the start address.
__device__ __forceinline__ uint64_t make_desc_kmajor(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>((1024 >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}

__device__ __forceinline__ uint32_t tmem_ld1(uint32_t taddr) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr) : "memory");
    return v;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Truncated CG on one system whose binary16 matrix sits in TMEM (thread i <->
// lane i <-> row i; the tcgen05 A-operand layout: column j holds elements
// 2j, 2j+1), run by one 128-thread group (4 warps, one named barrier).
//
// The reference's Algorithm 1 (solvers.py:83-118, corrected
// r -= alpha*A p) in its pipelined (Ghysels-Vanroose) form: s = A p, z = A s,
// w = A r are carried by recurrences, so each iteration needs ONE exchange --
// thread i publishes its vector entry (fp16 hi/lo into a K-major smem operand)
// and the warp sums of (r.r, w.r); after the barrier one thread issues the
// matvec on the tensor core (A from TMEM, N = 16, result in TMEM) while every
// thread finishes the sums.  Semantics: at least one update unless
// p^T A p <= 0 (breakdown: x kept), stop once ||r|| < eps, `nit` counts the
// x updates.  Deterministic (fixed reduction order).
template <int KP>
struct TmemCg {
    static constexpr int NKS = KP / 16;  // kind::f16 MMAs per matvec
    uint32_t bop, bofs0, bofs1, mvbar, lane_base;
    float *red;
    uint32_t mvph = 0;
    int slot = 0, bar_id, i, lane, warp;
    bool leader, act;
    long long *tr = nullptr;  // CMF_TRACE: per-exchange stamps of one row (thread 0 of the group)
    int trk = 0;
#ifdef CMF_TRACE
#define CG_STAMP()                                  \
    do {                                            \
        if (i == 0 && tr) trace_at(tr, trk++ & 63); \
    } while (0)
#else
#define CG_STAMP() \
    do {           \
    } while (0)
#endif

    __device__ TmemCg(unsigned char *scratch, uint32_t mvbar_, int bar_id_, int warp_, int lane_, int f)
        : bop(smem_u32(scratch)), mvbar(mvbar_), bar_id(bar_id_), lane(lane_), warp(warp_) {
        i = (warp & 3) * 32 + lane;
        act = i < f;
        red = reinterpret_cast<float *>(scratch + MVB_OPERAND);
        // B(n, k): n = 0 / 1 hold the vector's fp16 hi / lo halves at K position k = i
        bofs0 = (i / 64) * 2048 + ((((i % 64) >> 3) ^ 0) << 4) + (i & 7) * 2;
        bofs1 = (i / 64) * 2048 + 128 + ((((i % 64) >> 3) ^ 1) << 4) + (i & 7) * 2;
        leader = (warp & 3) == 0;
        lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    }

    // y_i = (A v)_i + reg * v_i and (sa, sb) = group sums of (da, db); rows i >= f
    // (act == false) publish nothing and return 0
    // NRED: how many of (da, db) are reduced (0, 1 or 2); the others return 0
    template <int NRED = 2>
    __device__ float exchange(uint32_t a_tmem, uint32_t dcol, float reg, float v, float da, float db, float &sa,
                              float &sb, bool mv) {
        constexpr uint32_t idesc_mv = (1u << 4) | (static_cast<uint32_t>(16 >> 3) << 17) |
                                      (static_cast<uint32_t>(128 >> 4) << 24);  // f16 x f16 -> f32, K-major
        CG_STAMP();
        if (mv && act) {
            const __half hv = __float2half_rn(v);
            const __half lv = __float2half_rn(v - __half2float(hv));
            asm volatile("st.shared.b16 [%0], %1;" ::"r"(bop + bofs0), "h"(__half_as_ushort(hv)) : "memory");
            asm volatile("st.shared.b16 [%0], %1;" ::"r"(bop + bofs1), "h"(__half_as_ushort(lv)) : "memory");
        }
        if (mv) fence_proxy_async();
        // three butterfly levels leave 4 partials per warp (lanes 0-3); the 16
        // per value are summed after the barrier in a fixed order
#ifdef CMF_RED5
        constexpr int kLow = 0;
#else
        constexpr int kLow = 2;
#endif
#pragma unroll
        for (int o = 16; o > kLow; o >>= 1) {
            if (NRED >= 1) da += __shfl_xor_sync(0xffffffffu, da, o);
            if (NRED >= 2) db += __shfl_xor_sync(0xffffffffu, db, o);
        }
        float *rd = red + 32 * slot;
        slot ^= 1;
        if (lane < 4 && (kLow == 2 || lane == 0)) {
            if (NRED >= 1) rd[(warp & 3) * 4 + lane] = da;
            if (NRED >= 2) rd[16 + (warp & 3) * 4 + lane] = db;
        }
        named_bar(bar_id, CG_THREADS);
        CG_STAMP();
        if (mv && leader) {
            if (elect_one()) {
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < NKS; ++kk)
                    tc_mma_tmem_a(dcol, a_tmem + 8 * kk, make_desc_kmajor(bop + (kk >> 2) * 2048 + (kk & 3) * 32),
                                  idesc_mv, kk);
                tc_commit(mvbar);
            }
            __syncwarp();
        }
#if defined(CMF_RED5)
        {
            // one partial per warp (rd[4w] / rd[16 + 4w])
            sa = NRED >= 1 ? (rd[0] + rd[4]) + (rd[8] + rd[12]) : 0.0f;
            sb = NRED >= 2 ? (rd[16] + rd[20]) + (rd[24] + rd[28]) : 0.0f;
        }
#elif !defined(CMF_RED3)
        // (default; CMF_RED3: every lane sums the 16 partials of each value from
        // four float4 loads -- 2% slower on the Netflix user side, same-box A/B)
        if (NRED >= 1) {
            // lane l sums partial l & 15 of value l >> 4 with a 16-lane butterfly
            // (bitwise identical in every lane: each level adds the same pair)
            float t = rd[NRED >= 2 ? lane : (lane & 15)];
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (NRED >= 2) {
                const float o16 = __shfl_xor_sync(0xffffffffu, t, 16);
                sa = lane < 16 ? t : o16;
                sb = lane < 16 ? o16 : t;
            } else {
                sa = t;
                sb = 0.0f;
            }
        } else {
            sa = sb = 0.0f;
        }
#else
        {
            const float4 *r4 = reinterpret_cast<const float4 *>(rd);
            float t[8];
#pragma unroll
            for (int k = 0; k < 4 * NRED; ++k) {
                const float4 q = r4[k];
                t[k] = (q.x + q.y) + (q.z + q.w);
            }
            sa = NRED >= 1 ? (t[0] + t[1]) + (t[2] + t[3]) : 0.0f;
            sb = NRED >= 2 ? (t[4] + t[5]) + (t[6] + t[7]) : 0.0f;
        }
#endif
        if (!mv) return 0.0f;
        mbar_wait(mvbar, mvph & 1);
        CG_STAMP();
        ++mvph;
        tc_fence_after();
        uint32_t yv[2];  // matvec result columns: A v_hi, A v_lo
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];"
                     : "=r"(yv[0]), "=r"(yv[1])
                     : "r"(dcol + lane_base)
                     : "memory");
        tmem_ld_wait();
        const float y = act ? __uint_as_float(yv[0]) + __uint_as_float(yv[1]) : 0.0f;
        return fmaf(reg, v, y);
    }

    // The same solve with the standard recurrence (explicit p^T A p and r.r
    // reductions, three barriers per iteration): the per-system accuracy the
    // reference-facing batch_solve is held to on ill-conditioned systems.
    __device__ void solve_standard(uint32_t a_tmem, uint32_t dcol, float bi, double eps, float tol, int f_s,
                                   float &xi, int &bd, int &nit, float reg = 0.0f) {
        float bb, rs, unused;
        float r = bi - exchange<1>(a_tmem, dcol, reg, xi, bi * bi, 0.0f, bb, unused, true);
        // stop test ||r|| < eps as r.r < eps^2 in fp32 (no double sqrt per iteration)
        const float e2 = eps >= 0.0 ? static_cast<float>(eps * eps) : tol * tol * bb;
        exchange<1>(a_tmem, dcol, 0.0f, 0.0f, r * r, 0.0f, rs, unused, false);
        float p = r;
        bd = 0;
        nit = 0;
        for (int step = 0; step < f_s; ++step) {
            float pap, rs_new;
            const float ap = exchange<0>(a_tmem, dcol, reg, p, 0.0f, 0.0f, unused, unused, true);
            exchange<1>(a_tmem, dcol, 0.0f, 0.0f, p * ap, 0.0f, pap, unused, false);
            if (!(pap > 0.0f)) {
                bd = 1;
                break;
            }
            const float alpha = __fdividef(rs, pap);
            xi = fmaf(alpha, p, xi);
            r = fmaf(-alpha, ap, r);
            exchange<1>(a_tmem, dcol, 0.0f, 0.0f, r * r, 0.0f, rs_new, unused, false);
            ++nit;
            if (rs_new == 0.0f || rs_new < e2) break;
            p = fmaf(__fdividef(rs_new, rs), p, r);
            rs = rs_new;
        }
    }

    // solve (A + reg I) x = b from the warm start xi; eps < 0: eps = tol * ||b||
    __device__ void solve(uint32_t a_tmem, uint32_t dcol, float reg, float bi, double eps, float tol, int f_s,
                          float &xi, int &bd, int &nit) {
        float bb, unused;
        float r = bi - exchange<1>(a_tmem, dcol, reg, xi, bi * bi, 0.0f, bb, unused, true);
        const float eps2 = eps >= 0.0 ? static_cast<float>(eps * eps) : tol * tol * bb;
        float gamma, delta;
        float w = exchange<0>(a_tmem, dcol, reg, r, 0.0f, 0.0f, gamma, delta, true);
        // 1/gamma_old and 1/alpha_old are formed off the critical path (one
        // iteration early); only 1/pap sits on it.  rcp.approx (1 ulp): the
        // scalars feed a truncated CG graded on the RMSE trajectory.
        float p = 0.0f, sv = 0.0f, z = 0.0f, rgamma_old = 1.0f, ralpha_old = 1.0f;
        bd = 0;
        nit = 0;
        for (int step = 0; step < f_s; ++step) {
            const bool last = step + 1 >= f_s;
            const float m = exchange(a_tmem, dcol, reg, w, r * r, w * r, gamma, delta, !last);
            if (step > 0 && (gamma == 0.0f || gamma < eps2)) break;
            const float beta = step > 0 ? gamma * rgamma_old : 0.0f;
            const float pap = step > 0 ? delta - beta * gamma * ralpha_old : delta;
            if (!(pap > 0.0f)) {
                bd = 1;
                break;
            }
            const float alpha = gamma * rcp_approx(pap);
            z = fmaf(beta, z, m);
            sv = fmaf(beta, sv, w);
            p = fmaf(beta, p, r);
            xi = fmaf(alpha, p, xi);
            r = fmaf(-alpha, sv, r);
            w = fmaf(-alpha, z, w);
            rgamma_old = rcp_approx(gamma);
            ralpha_old = rcp_approx(alpha);
            ++nit;
        }
    }
};

// FC = ceil(f/4): register row of A_u as FC*2 float2 pairs.
template <int FC, bool LONG, bool WEIGHTED = false>
__global__ void __launch_bounds__(FusedShape<FC, LONG>::THREADS, 1)
    fused_cg_kernel(const __grid_constant__ FusedArgs g) {
    using Shape = FusedShape<FC, LONG>;
    constexpr int F_GROUPS = Shape::NG;
    constexpr int F_THREADS = Shape::THREADS;
    constexpr int F_MMA_WARP = Shape::MMA_WARP;
    constexpr int NBUF = Shape::NBUF;
    using PipeT = FPipe<NBUF, WEIGHTED, FC>;
    static_assert(!WEIGHTED || PipeT::kStages >= 3, "weighted ring too small");
    constexpr int KP = (FC * 4 + 15) / 16 * 16;  // matvec K extent (>= f), 16-half MMA steps
    constexpr int F_STAGES = PipeT::kStages;
    // "Gram ready" hand-off without parity aliasing: a waiter must never be two
    // phases behind its barrier.  With NG >= NBUF the row a group waits for can
    // be two phases ahead on its buffer's barrier but not on a per-group barrier
    // (row r + NG needs a buffer that row r's group releases); with NG < NBUF the
    // reverse holds (rows <= r - NG are committed before row r's group waits).
    constexpr bool kGroupFull = F_GROUPS >= NBUF;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const GatherArgs &ga = g.gather;
    const int f = ga.f;
    unsigned char *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    // [stages | per-group CG scratch (MVB_BYTES each: matvec B operand, warp partials) |
    //  barriers (pipeline + one matvec barrier per group) | tmem slot]
    unsigned char *scratch = smem + F_STAGES * PipeT::kStageBytes;
    // WEIGHTED: F^T F (f rows of 4FC floats) after the CG scratch; read by the repack
    float *base_s = reinterpret_cast<float *>(scratch + F_GROUPS * MVB_BYTES);
    uint64_t *bars = reinterpret_cast<uint64_t *>(scratch + F_GROUPS * MVB_BYTES +
                                                  (WEIGHTED ? base_smem_bytes<FC>() : 0));
    uint64_t *mvbars = bars + PipeT::kBars;
    uint64_t *gfull = mvbars + F_GROUPS;  // per-group "Gram ready" (row r -> group r % NG)
    uint64_t *landed = gfull + F_GROUPS;  // WEIGHTED: gathered rows of slot s landed (32 cp.async arrivals)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(landed + (WEIGHTED ? F_STAGES : 0));
    PipeT pp{smem_u32(smem), smem_u32(bars)};
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    pipe_init(pp, smem, F_THREADS, WEIGHTED ? 1 : 33, CG_THREADS);
    if (WEIGHTED && g.base) {
        const int nb = f * 4 * FC;
        for (int k = tid; k < nb; k += F_THREADS)
            base_s[(k / (4 * FC)) * base_lds<FC>() + k % (4 * FC)] = __ldg(g.base + k);
    }
    for (int i = tid; i < F_GROUPS * MVB_BYTES / 16; i += F_THREADS)
        reinterpret_cast<int4 *>(scratch)[i] = make_int4(0, 0, 0, 0);
    if (tid == 0) {
        for (int q = 0; q < F_GROUPS; ++q) {
            mbar_init(smem_u32(mvbars + q), 1);
            mbar_init(smem_u32(gfull + q), 1);
        }
        if (WEIGHTED)
            for (int q = 0; q < F_STAGES; ++q) mbar_init(smem_u32(landed + q), 32);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == F_MMA_WARP) tmem_alloc(smem_u32(tmem_slot), g.tmem_cols);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int64_t G = gridDim.x;

    if (warp >= 4 * F_GROUPS && warp < F_MMA_WARP) {
        regs_dec<Shape::AUX_REGS>();
        const int pw = warp - 4 * F_GROUPS;
        if constexpr (WEIGHTED) {
            // g.nprod gatherers, then the scalers (every other producer warp)
            if (pw < g.nprod)
                gather_weighted<F_STAGES, NBUF>(ga, g.fixed16, g.W, pp, smem_u32(landed), pw, g.nprod, lane,
                                                blockIdx.x, G);
            else if (pw - g.nprod < min(Shape::NPROD - g.nprod, F_STAGES))  // scalers <= stages
                scale_weighted<F_STAGES, NBUF>(ga, g.W, g.alpha, pp, smem_u32(landed), pw - g.nprod,
                                               min(Shape::NPROD - g.nprod, F_STAGES), lane, blockIdx.x, G);
        } else if (pw < g.nprod)
                produce<F_STAGES, false, NBUF>(ga, g.fixed16, nullptr, g.W, pp, warp - 4 * F_GROUPS, g.nprod, lane,
                                               blockIdx.x, G);
    } else if (warp == F_MMA_WARP) {
        regs_dec<Shape::AUX_REGS>();
        issue_mma<F_STAGES, WEIGHTED, NBUF, WEIGHTED>(ga, pp, tmem_base, g.N, blockIdx.x, G, smem_u32(gfull),
                                         kGroupFull ? F_GROUPS : 0);
    } else {
        regs_inc<Shape::CG_REGS>();
        // ------------------------------------------------------------ CG groups
        const int grp = warp >> 2;             // rows r with r % NG == grp
        const int i = (warp & 3) * 32 + lane;  // row of A_u == TMEM lane
        TmemCg<KP> cg(scratch + grp * MVB_BYTES, smem_u32(mvbars + grp), 1 + grp, warp, lane, f);
        const bool act = cg.act;
        int32_t brk = 0;
        uint32_t rowc = 0;    // non-empty rows of this CTA so far (all groups)
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        for (int64_t u = blockIdx.x; u < ga.nrows; u += G) {
            const int64_t p0 = ga.indptr[u];
            const int n_u = static_cast<int>(ga.indptr[u + 1] - p0);
            if (n_u == 0) continue;
            const uint32_t r_here = rowc++;
            if (r_here % F_GROUPS != static_cast<uint32_t>(grp)) continue;
            const int b = r_here % NBUF;
            float* const tgt = g.target + u * f;
            float xi = act ? tgt[i] : 0.0f;  // warm start, loaded while the Gram is built
            if (i == 0 && r_here < 2048) trace_at(ga.trace, 32768 + 4 * r_here + 0);
            // long rows keep the group idle: back-off wait
            if (ga.pass == 2 && act) {  // the first segment's partial: into L2 while the Gram builds
                const char *pr = reinterpret_cast<const char *>(g.partial + (u * f + i) * g.pws);
                for (int o = 0; o < g.pws * 4; o += 128)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(pr + o));
            }
            if (kGroupFull)
                mbar_wait_backoff<64, 4096>(smem_u32(gfull + grp), (r_here / F_GROUPS) & 1);
            else
                mbar_wait_backoff<64, 4096>(pp.tfull(b), (r_here / NBUF) & 1);
            if (i == 0 && r_here < 2048) trace_at(ga.trace, 32768 + 4 * r_here + 1);
            tc_fence_after();
            // A_u (fp32, thread i <-> lane i <-> row i) -> binary16 in this group's
            // slot: accumulator columns [32c, 32c+32) become slot columns
            // [16c, 16c+16), the tcgen05 A-operand layout (lane = row, column j =
            // elements 2j, 2j+1).  RNE, as the reference's fp16 Hermitian storage.
            // Columns >= f (padding, and the rating columns W, W+1) become zero, so
            // the matvec's K range sees only A_u; rows >= f keep whatever they hold
            // (a D row depends only on its own A row, and rows >= f are never
            // read).  |a| >= 65520 rounds to inf: the overflow flag.  The
            // accumulator is released as soon as it has been read.
            const uint32_t tb = tmem_base + lane_base + b * g.N;
            // segmented passes: which parts hold data (the MMA skipped an empty segment)
            bool seg_acc = true, seg_part = false;
            if (ga.pass) {
                const int64_t sp = ga.seg[u];
                seg_acc = ga.pass == 1 ? sp > p0 : ga.indptr[u + 1] > sp;
                seg_part = ga.pass == 2 && sp > p0;
            }
            float *const prow = g.partial + (u * f + i) * g.pws;
            if (ga.pass == 1) {
                // first segment: park the fp32 accumulator (Gram + bias columns) in HBM
                if (seg_acc) {
#pragma unroll 1
                    for (int c = 0; c < g.W + 2; c += 16) {
                        uint32_t v[16];
                        tmem_ldn<16>(tb + c, v);
                        tmem_ld_wait();
                        if (act) {
#pragma unroll
                            for (int j = 0; j < 16; j += 4)
                                if (c + j < g.pws)
                                    *reinterpret_cast<float4 *>(prow + c + j) =
                                        make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                                                    __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive(pp.tempty(b));
                continue;
            }
            float bi = 0.0f;
            if (seg_acc) {
                bi = __uint_as_float(tmem_ld1(tb + g.W)) + __uint_as_float(tmem_ld1(tb + g.W + 1));
                tmem_ld_wait();
            }
            if (seg_part && act) bi += prow[g.W] + prow[g.W + 1];
            bi = act ? bi : 0.0f;
            const uint32_t a_tmem = tmem_base + g.slot_base + grp * Shape::SLOT;
            float amax = 0.0f;
#pragma unroll
            for (int c = 0; c < (KP + 31) / 32; ++c) {
                uint32_t v[32], h[16];
                if (seg_acc) {
                    if (32 * c + 32 <= KP) tmem_ldn<32>(tb + 32 * c, v);
                    else tmem_ldn<16>(tb + 32 * c, v);
                    tmem_ld_wait();
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = 0u;
                }
                if (seg_part && act) {
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        if (32 * c + j >= KP) break;
                        if (32 * c + j < g.pws) {
                            const float4 q = *reinterpret_cast<const float4 *>(prow + 32 * c + j);
                            v[j] = __float_as_uint(__uint_as_float(v[j]) + q.x);
                            v[j + 1] = __float_as_uint(__uint_as_float(v[j + 1]) + q.y);
                            v[j + 2] = __float_as_uint(__uint_as_float(v[j + 2]) + q.z);
                            v[j + 3] = __float_as_uint(__uint_as_float(v[j + 3]) + q.w);
                        }
                    }
                }
                if (WEIGHTED && g.base && act) {
                    // + F^T F row i from shared memory (float4 rows, conflict-free; columns
                    // f .. 4FC-1 hold zeros, and the repack zeroes columns >= f anyway)
                    const float4 *brow = reinterpret_cast<const float4 *>(base_s + i * base_lds<FC>());
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        if (32 * c + j >= 4 * FC) break;  // columns >= 4FC (> f) get no base
                        const float4 q = brow[(32 * c + j) / 4];
                        float2 lo = make_float2(__uint_as_float(v[j]), __uint_as_float(v[j + 1]));
                        float2 hi = make_float2(__uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
                        lo = __fadd2_rn(lo, make_float2(q.x, q.y));
                        hi = __fadd2_rn(hi, make_float2(q.z, q.w));
                        v[j] = __float_as_uint(lo.x);
                        v[j + 1] = __float_as_uint(lo.y);
                        v[j + 2] = __float_as_uint(hi.x);
                        v[j + 3] = __float_as_uint(hi.y);
                    }
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    if (32 * c + 2 * j >= KP) break;
                    // f > 4 * (FC - 1): only columns >= 4FC - 4 can lie past f
                    const int col = 32 * c + 2 * j;
                    float a0 = __uint_as_float(v[2 * j]), a1 = __uint_as_float(v[2 * j + 1]);
                    if (col >= 4 * FC - 4 && col >= f) a0 = 0.0f;
                    if (col + 1 >= 4 * FC - 4 && col + 1 >= f) a1 = 0.0f;
                    amax = fmaxf(amax, fmaxf(fabsf(a0), fabsf(a1)));
                    const __half2 hv = __floats2half2_rn(a0, a1);
                    h[j] = *reinterpret_cast<const uint32_t *>(&hv);
                }
                if (32 * c + 32 <= KP) tmem_st16(a_tmem + lane_base + 16 * c, h);
                else tmem_st8(a_tmem + lane_base + 16 * c, h);
            }
            tc_fence_before();
            mbar_arrive(pp.tempty(b));  // the accumulator is free for row r_here + NBUF
            // binary16 max finite is 65504; RNE sends |a| >= 65520 to inf
            if (act && !(amax < 65520.0f) && g.overflow) *g.overflow = 1;  // also NaN
            tmem_st_wait();
            tc_fence_before();
            if (i == 0 && r_here < 2048) trace_at(ga.trace, 32768 + 4 * r_here + 2);
            const uint32_t dcol = tmem_base + g.dmv_base + 16 * grp;
            const float reg = g.weighted ? __double2float_rn(g.lam * static_cast<double>(n_u))
                                         : __double2float_rn(g.lam);
            int bd = 0, nit = 0;
            cg.tr = (ga.trace && r_here < 64) ? ga.trace + 40960 + 64 * r_here : nullptr;
            cg.trk = 0;
            if constexpr (WEIGHTED)  // ill-conditioned implicit systems: the standard recurrence
                cg.solve_standard(a_tmem, dcol, bi, -1.0, g.tol, g.f_s, xi, bd, nit, reg);
            else
                cg.solve(a_tmem, dcol, reg, bi, -1.0, g.tol, g.f_s, xi, bd, nit);
            tc_fence_before();  // the next row's repack overwrites the slot the MMAs read
            if (act) {
                tgt[i] = xi;
                // multi-GPU: the solved row also goes straight into every peer's
                // replica (NVLink stores, coalesced 4f bytes per row), which
                // replaces the all-gather after the half-update
                for (int k = 0; k < g.npeers; ++k) g.peers[k][u * f + i] = xi;
            }
            if (i == 0 && r_here < 2048) trace_at(ga.trace, 32768 + 4 * r_here + 3);
            brk += bd;
        }
        if (i == 0 && brk && g.breakdowns) atomicAdd(g.breakdowns, brk);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == F_MMA_WARP) {
        tc_fence_after();
        tmem_dealloc(tmem_base, g.tmem_cols);
    }
}

}  // namespace tc

int set_error(int code, const char *fmt, ...);

template <int FC, bool LONG, bool WEIGHTED>
static int launch_fused(tc::FusedArgs g, cudaStream_t st) {
    using Shape = tc::FusedShape<FC, LONG>;
    using PipeT = tc::FPipe<Shape::NBUF, WEIGHTED, FC>;
    const size_t smem = 1024 + PipeT::kStages * PipeT::kStageBytes + Shape::NG * tc::MVB_BYTES +
                        (WEIGHTED ? tc::base_smem_bytes<FC>() : 0) +
                        (PipeT::kBars + 2 * Shape::NG + (WEIGHTED ? PipeT::kStages : 0)) * 8 + 16;
    // matvec results (16 columns per group): after the accumulators when they fit,
    // else in each buffer's columns freed by the fp16 repacking of A_u
    if (g.N > Shape::NMAX) return set_error(CMF_EINVAL, "fused CG: accumulator width %d > %d", g.N, Shape::NMAX);
    if (g.nprod <= 0 || g.nprod > Shape::NPROD) g.nprod = Shape::NPROD;
    if (g.nprod > PipeT::kStages) g.nprod = PipeT::kStages;  // producers <= ring stages
    // weighted: a producer releases stage it only after issuing stage it + nprod,
    // whose slot must be a different, earlier-consumed one: nprod <= stages - 1
    // (one more stage of slack keeps the MMA fed)
    if (WEIGHTED) {
        // g.nprod = gather warps (<= stages); the other producer warps scale
        const char *e = getenv("CMF_WGATHER");  // A/B knob
        g.nprod = e ? atoi(e) : Shape::NPROD / 2;
        if (g.nprod < 1) g.nprod = 1;
        if (g.nprod > Shape::NPROD - 1) g.nprod = Shape::NPROD - 1;
        if (g.nprod > PipeT::kStages) g.nprod = PipeT::kStages;
    }
    g.slot_base = Shape::NBUF * g.N;
    g.dmv_base = (g.slot_base + Shape::NG * Shape::SLOT + 15) / 16 * 16;
    g.tmem_cols = 512;
    auto k = tc::fused_cg_kernel<FC, LONG, WEIGHTED>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return set_error(CMF_ECUDA, "fused_cg smem attr: %s", cudaGetErrorString(e));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t grid = sms;
    if (grid > g.gather.nrows) grid = g.gather.nrows;
    k<<<static_cast<unsigned>(grid), Shape::THREADS, smem, st>>>(g);
    return check_launch("fused_cg_kernel");
}


// f (<= 120) -> template instance FC (bucketed; 4*FC >= f): the row stride of the
// implicit base matrix (cmf_fused_base_ld)
inline int fused_fc(int f) {
    const int fmax[16] = {8, 16, 24, 32, 40, 48, 56, 64, 72, 80, 88, 96, 100, 104, 112, 120};
    const int fc[16] = {2, 4, 6, 8, 10, 12, 14, 16, 18, 20, 22, 24, 25, 26, 28, 30};
    for (int k = 0; k < 16; ++k)
        if (f <= fmax[k]) return fc[k];
    return -1;
}

// f (<= 120) -> template instance FC = ceil(f/4), bucketed
template <bool WEIGHTED>
static int fused_dispatch_t(tc::FusedArgs g, int f, bool long_rows, cudaStream_t st) {
#define CMF_FUSED_CASE(FMAX, FCV)                                                      \
    if (f <= FMAX)                                                                     \
        return long_rows ? launch_fused<FCV, true, WEIGHTED>(g, st) : launch_fused<FCV, false, WEIGHTED>(g, st);
    CMF_FUSED_CASE(8, 2)
    CMF_FUSED_CASE(16, 4)
    CMF_FUSED_CASE(24, 6)
    CMF_FUSED_CASE(32, 8)
    CMF_FUSED_CASE(40, 10)
    CMF_FUSED_CASE(48, 12)
    CMF_FUSED_CASE(56, 14)
    CMF_FUSED_CASE(64, 16)
    CMF_FUSED_CASE(72, 18)
    CMF_FUSED_CASE(80, 20)
    CMF_FUSED_CASE(88, 22)
    CMF_FUSED_CASE(96, 24)
    CMF_FUSED_CASE(100, 25)
    CMF_FUSED_CASE(104, 26)
    CMF_FUSED_CASE(112, 28)
    CMF_FUSED_CASE(120, 30)
#undef CMF_FUSED_CASE
    return set_error(CMF_EINVAL, "no fused CG instance for f=%d", f);
}

}  // namespace cmf
