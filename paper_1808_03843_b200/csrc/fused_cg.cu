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
//   warps 12-18 producers  cp.async gather of binary16 factor rows (+ the rating
//                          rows) into a 12-stage swizzled operand ring
//   warp 19     MMA        tcgen05.mma kind::f16 chain per row into TMEM buffer
//                          (row % 3); tcgen05.commit -> stage empty / tmem full
//   warps 0-11  CG         three groups of 4 warps, one per TMEM buffer: read
//                          b_u from the accumulator's rating columns, repack
//                          A_u to binary16 in place (the tcgen05 A-operand
//                          layout), run Algorithm 1 (PAPER.md:272-293,
//                          corrected r -= alpha*A p) in its pipelined form (one
//                          barrier per iteration carries both dot products and
//                          the next matvec's vector) with fp32 vectors; every
//                          matvec is 7 tensor-core MMAs with A read from TMEM;
//                          deterministic reductions; write x_u in place (warm
//                          start = previous x_u), then free the buffer.
//
// Semantics vs the reference: the diagonal gets lambda*n_u (weighted) or
// lambda; rows with n_u == 0 are left untouched; eps = cg_tol * ||b_u||;
// breakdown (p^T A p <= 0) keeps the current iterate and is counted.  A_u is
// rounded from the fp32 accumulator to binary16 (RNE) in TMEM -- the
// reference's precision="fp16" Hermitian storage (gram.py:132-146) -- and an
// entry that overflows binary16 sets the overflow flag, which the caller
// raises as NumericalError like pack_half does.  The CG vectors are fp32
// (split into fp16 hi/lo halves as the matvec's B operand).
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
    // L2 can hold): pass 1 stores each row's partial accumulator (columns
    // [0, W+2): the first-segment Gram and bias) at partial + (u*128 + i)*PWS
    // for lanes i < f; pass 2 adds it to the second segment's accumulator.
    float *partial;
    int pws;  // partial row stride in floats (roundup4(W + 2))
};

template <int NBUF>
using FPipe = Pipe<12, false, NBUF>;  // 12 x 18 KB operand ring: bytes in flight for the gather

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
#elif defined(CMF_RED16)
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
                                   float &xi, int &bd, int &nit) {
        float bb, rs, unused;
        float r = bi - exchange<1>(a_tmem, dcol, 0.0f, xi, bi * bi, 0.0f, bb, unused, true);
        // stop test ||r|| < eps as r.r < eps^2 in fp32 (no double sqrt per iteration)
        const float e2 = eps >= 0.0 ? static_cast<float>(eps * eps) : tol * tol * bb;
        exchange<1>(a_tmem, dcol, 0.0f, 0.0f, r * r, 0.0f, rs, unused, false);
        float p = r;
        bd = 0;
        nit = 0;
        for (int step = 0; step < f_s; ++step) {
            float pap, rs_new;
            const float ap = exchange<0>(a_tmem, dcol, 0.0f, p, 0.0f, 0.0f, unused, unused, true);
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
template <int FC, bool LONG>
__global__ void __launch_bounds__(FusedShape<FC, LONG>::THREADS, 1)
    fused_cg_kernel(const __grid_constant__ FusedArgs g) {
    using Shape = FusedShape<FC, LONG>;
    constexpr int F_GROUPS = Shape::NG;
    constexpr int F_THREADS = Shape::THREADS;
    constexpr int F_MMA_WARP = Shape::MMA_WARP;
    constexpr int NBUF = Shape::NBUF;
    using PipeT = FPipe<NBUF>;
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
    uint64_t *bars = reinterpret_cast<uint64_t *>(scratch + F_GROUPS * MVB_BYTES);
    uint64_t *mvbars = bars + PipeT::kBars;
    uint64_t *gfull = mvbars + F_GROUPS;  // per-group "Gram ready" (row r -> group r % NG)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(gfull + F_GROUPS);
    PipeT pp{smem_u32(smem), smem_u32(bars)};
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    pipe_init(pp, smem, F_THREADS, 33, CG_THREADS);
    for (int i = tid; i < F_GROUPS * MVB_BYTES / 16; i += F_THREADS)
        reinterpret_cast<int4 *>(scratch)[i] = make_int4(0, 0, 0, 0);
    if (tid == 0) {
        for (int q = 0; q < F_GROUPS; ++q) {
            mbar_init(smem_u32(mvbars + q), 1);
            mbar_init(smem_u32(gfull + q), 1);
        }
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
        if (warp - 4 * F_GROUPS < g.nprod)
            produce<F_STAGES, false, NBUF>(ga, g.fixed16, nullptr, g.W, pp, warp - 4 * F_GROUPS, g.nprod, lane,
                                           blockIdx.x, G);
    } else if (warp == F_MMA_WARP) {
        regs_dec<Shape::AUX_REGS>();
        issue_mma<F_STAGES, false, NBUF>(ga, pp, tmem_base, g.N, blockIdx.x, G, smem_u32(gfull),
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
                const char *pr = reinterpret_cast<const char *>(g.partial + (u * 128 + i) * g.pws);
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
            float *const prow = g.partial + (u * 128 + i) * g.pws;
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

// ---------------------------------------------------------------------------
// Batched CG over packed binary16 systems (the two-step route's K3: replaces
// solvers._cg_batch for precision="fp16", solvers.py:121-145, 205-247).
// Three 128-thread groups per CTA, two CTAs per SM; each group double-buffers
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

constexpr int CGT_GROUPS = 3;
constexpr int CGT_THREADS = 128 * CGT_GROUPS;

template <int KP>
__global__ void __launch_bounds__(CGT_THREADS, 2) cg_tc_kernel(const __grid_constant__ CgTcArgs g) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    const int f = g.f;
    const int64_t P = packed_size(f);
    const int SB = static_cast<int>((P * 2 + 127) & ~127ll);  // staging bytes per system
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
    if (warp == 0) tmem_alloc(smem_u32(tmem_slot), 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    TmemCg<KP> cg(scr, smem_u32(mvbars + grp), 1 + grp, warp, lane, f);
    const int i = cg.i, gt = tid & 127;
    // TMEM: 16-column aligned slots (KP/2 packed columns each), then the 16-column
    // matvec results from a 32-column boundary
    constexpr uint32_t SLOT = (KP / 2 + 15) / 16 * 16;
    constexpr uint32_t DBASE = (CGT_GROUPS * SLOT + 31) / 32 * 32;
    static_assert(DBASE + 16 * CGT_GROUPS <= 256, "cg_tc TMEM plan");
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
        named_bar(1 + grp, CG_THREADS);
        // row i of the symmetric matrix -> binary16 pairs in TMEM
        const __half *A = reinterpret_cast<const __half *>(stg + buf * SB);
        // element (i, j): row i of the packed lower triangle for j <= i, column i
        // (row j, position i) above the diagonal; j is warp-uniform, so the
        // column reads of a warp are consecutive halves.  32-bit offsets; lanes
        // i >= f read element 0 (their rows only feed their own, unused outputs)
        const int ri = act ? i * (i + 1) / 2 : 0;
        const int ci = act ? i : 0;
        const unsigned short *Au = reinterpret_cast<const unsigned short *>(A);
#pragma unroll
        for (int c = 0; c < (KP + 31) / 32; ++c) {  // fully unrolled: j, j(j+1)/2 are immediates
            uint32_t h[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                uint32_t e[2];
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const int j = 32 * c + 2 * q + t;
                    e[t] = 0u;
                    if (j < f) e[t] = Au[j <= ci ? ri + j : j * (j + 1) / 2 + ci];
                }
                h[q] = e[0] | (e[1] << 16);
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
        tmem_dealloc(tmem_base, 256);
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

// Two passes pay when the rows are long (the partial accumulator's HBM round
// trip, ~2 x 43 KB per row at f = 100, is small against the row's gather) and
// the fixed side's binary16 shadow is too large to stay in L2 across the
// sweep (Netflix Theta side: 100 MB of X shadow, 67% L2 hits in one pass).
constexpr int64_t kTwoPassShadowBytes = int64_t(48) << 20;
int64_t fused_cg_workspace_bytes(int64_t nrows, int W) {
    const int64_t pws = (W + 2 + 3) / 4 * 4;
    return ((nrows * 8 + 255) & ~int64_t(255)) + nrows * 128 * pws * 4;
}

template <int FC, bool LONG>
static int launch_fused(tc::FusedArgs g, cudaStream_t st) {
    using Shape = tc::FusedShape<FC, LONG>;
    using PipeT = tc::FPipe<Shape::NBUF>;
    const size_t smem = 1024 + PipeT::kStages * PipeT::kStageBytes + Shape::NG * tc::MVB_BYTES +
                        (PipeT::kBars + 2 * Shape::NG) * 8 + 16;
    // matvec results (16 columns per group): after the accumulators when they fit,
    // else in each buffer's columns freed by the fp16 repacking of A_u
    if (g.N > Shape::NMAX) return set_error(CMF_EINVAL, "fused CG: accumulator width %d > %d", g.N, Shape::NMAX);
    if (g.nprod <= 0 || g.nprod > Shape::NPROD) g.nprod = Shape::NPROD;
    g.slot_base = Shape::NBUF * g.N;
    g.dmv_base = (g.slot_base + Shape::NG * Shape::SLOT + 15) / 16 * 16;
    g.tmem_cols = 512;
    auto k = tc::fused_cg_kernel<FC, LONG>;
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

static int fused_dispatch(tc::FusedArgs g, int f, bool long_rows, cudaStream_t st);

// f (<= 120) -> template instance FC = ceil(f/4), bucketed
#define CMF_FUSED_CASE(FMAX, FCV) \
    if (f <= FMAX) return long_rows ? launch_fused<FCV, true>(g, st) : launch_fused<FCV, false>(g, st);

int fused_cg_launch(const int64_t *indptr, const int32_t *indices, const float *values, int64_t nrows,
                    const void *fixed16, int64_t ncols, int W, int f, double lam, int weighted, float *target,
                    float *const *peers, int npeers, int64_t nnz, int f_s, double cg_tol, int32_t *breakdowns,
                    int32_t *overflow, void *ws, int64_t ws_bytes, cudaStream_t st) {
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
                rc = fused_dispatch(g, f, long_rows, st);
                if (rc != CMF_OK) return rc;
            }
            return CMF_OK;
        }
    }
    return fused_dispatch(g, f, long_rows, st);
}

static int fused_dispatch(tc::FusedArgs g, int f, bool long_rows, cudaStream_t st) {
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
    return set_error(CMF_EINVAL, "no fused CG instance for f=%d", f);
}
#undef CMF_FUSED_CASE

template <int KP>
static int launch_cg_tc(const tc::CgTcArgs &g, cudaStream_t st) {
    const int64_t P = packed_size(g.f);
    const size_t SB = (P * 2 + 127) & ~127ll;
    const size_t GS = (tc::MVB_BYTES + 2 * SB + 1023) & ~static_cast<size_t>(1023);
    const size_t smem = 1024 + tc::CGT_GROUPS * GS + tc::CGT_GROUPS * 8 + 16;
    auto k = tc::cg_tc_kernel<KP>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return set_error(CMF_ECUDA, "cg_tc smem attr: %s", cudaGetErrorString(e));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t grid = 2 * static_cast<int64_t>(sms);
    const int64_t need = (g.nsys + tc::CGT_GROUPS - 1) / tc::CGT_GROUPS;
    if (grid > need) grid = need;
    k<<<static_cast<unsigned>(grid), tc::CGT_THREADS, smem, st>>>(g);
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
