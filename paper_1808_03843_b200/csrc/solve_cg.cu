// K3: batched truncated conjugate gradient (Algorithm 1, PAPER.md:272-293,
// with the corrected residual update r -= alpha * A p).
//
// Replaces solvers._cg_batch / _cg_system / _symv (solvers.py:70-145).
//
// cg_rowreg_kernel (CMF_CG_FP32, f <= 128) -- the production path:
//   one CTA per system; the packed lower triangle (fp16 or fp32, the only
//   large operand: 2 or 4 bytes x f(f+1)/2) is streamed once from HBM into
//   shared memory, then each thread i < f expands row i of the symmetric
//   matrix into registers.  Every matvec is then register FFMA2 against the
//   search direction broadcast from shared memory; dot products are
//   deterministic block reductions.  HBM traffic per system = A + b + x0 + x.
//
// cg_ref64_kernel (CMF_CG_FP64, any f): the reference's float64 recurrence
//   operation for operation (column-sweep matvec order, sequential dot
//   products, no fused multiply-add) -- bitwise equal to solvers.py.
#include "common.cuh"

namespace cmf {

struct CgArgs {
    const void *a;
    int64_t a_stride;
    const float *b;
    const float *x0;
    const double *eps;
    double tol;
    const int64_t *nu;
    int64_t nsys;
    int f, f_s;
    float *x_out;
    int32_t *iters;
    int32_t *broke;
    int32_t *breakdowns;
    int vec16;
};

// Stage one packed system into shared memory with async copies (every load in
// flight at once; the caller commits and waits).
template <bool HALF_A>
__device__ __forceinline__ void load_packed(const CgArgs &g, int64_t s, void *dst, int64_t P) {
    const size_t es = HALF_A ? 2 : 4;
    const char *src = static_cast<const char *>(g.a) + static_cast<size_t>(s) * g.a_stride * es;
    const int64_t bytes = P * es;
    char *d = static_cast<char *>(dst);
    if (g.vec16) {
        for (int64_t k = threadIdx.x; k < (bytes >> 4); k += blockDim.x) cp_async16(d + 16 * k, src + 16 * k);
        // tail (< 16 bytes): 4-byte pieces (P*es is even for fp16 when P is even; else 2-byte below)
        for (int64_t k = (bytes & ~15ll) + 4 * threadIdx.x; k + 4 <= bytes; k += 4 * blockDim.x)
            cp_async4(d + k, src + k, 4);
        if ((bytes & 3) && threadIdx.x == 0)
            *reinterpret_cast<uint16_t *>(d + bytes - 2) = *reinterpret_cast<const uint16_t *>(src + bytes - 2);
    } else if (HALF_A) {
        const uint16_t *s2 = reinterpret_cast<const uint16_t *>(src);
        uint16_t *d2 = reinterpret_cast<uint16_t *>(d);
        for (int64_t k = threadIdx.x; k < P; k += blockDim.x) d2[k] = s2[k];
    } else {
        for (int64_t k = threadIdx.x; k < P; k += blockDim.x) cp_async4(d + 4 * k, src + 4 * k, 4);
    }
    cp_async_commit();
}

template <bool HALF_A>
__device__ __forceinline__ float sm_a(const void *sA, int64_t k) {
    if (HALF_A) return half_bits_to_float(static_cast<const uint16_t *>(sA)[k]);
    return static_cast<const float *>(sA)[k];
}

template <int NC4, bool HALF_A>
__global__ void __launch_bounds__(128) cg_rowreg_kernel(CgArgs g) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const int64_t s = blockIdx.x;
    if (g.nu && g.nu[s] == 0) return;
    const int f = g.f, tid = threadIdx.x;
    const int64_t P = packed_size(f);
    const size_t abytes = ((P * (HALF_A ? 2 : 4)) + 15) & ~static_cast<size_t>(15);
    void *sA = smraw;
    float *pv = reinterpret_cast<float *>(smraw + abytes);  // NC4*4 floats
    float *red = pv + NC4 * 4;                               // 2 x 32 floats
    double *redd = reinterpret_cast<double *>(red + 64);     // 32 doubles

    load_packed<HALF_A>(g, s, sA, P);
    for (int k = tid; k < NC4 * 4; k += blockDim.x) pv[k] = 0.0f;
    const bool act = tid < f;
    float xi = act ? g.x0[s * f + tid] : 0.0f;
    const float bi = act ? g.b[s * f + tid] : 0.0f;
    cp_async_wait<0>();
    __syncthreads();

    // expand row `tid` of the symmetric matrix into registers
    float2 a2[NC4 * 2];
    const int64_t rbase = static_cast<int64_t>(tid) * (tid + 1) / 2;
#pragma unroll
    for (int k = 0; k < NC4 * 2; ++k) {
        float v[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = 2 * k + h;
            v[h] = 0.0f;
            if (act && j < f) v[h] = (j <= tid) ? sm_a<HALF_A>(sA, rbase + j)
                                                : sm_a<HALF_A>(sA, static_cast<int64_t>(j) * (j + 1) / 2 + tid);
        }
        a2[k] = make_float2(v[0], v[1]);
    }

    double eps;
    if (g.eps) {
        eps = g.eps[s];
    } else {
        const double bn = block_sum<double>(static_cast<double>(bi) * bi, redd);
        eps = g.tol * sqrt(bn);
    }

    const float eps2 = static_cast<float>(eps * eps);
    int slot = 0;
    auto bsum = [&](float v) {
        float r = block_sum<float>(v, red + 32 * slot);
        slot ^= 1;
        return r;
    };
    auto matvec = [&](float v) {
        if (act) pv[tid] = v;
        __syncthreads();
        float2 y2 = make_float2(0.0f, 0.0f);
        const float4 *p4 = reinterpret_cast<const float4 *>(pv);
#pragma unroll
        for (int c = 0; c < NC4; ++c) {
            const float4 q = p4[c];
            y2 = __ffma2_rn(a2[2 * c], make_float2(q.x, q.y), y2);
            y2 = __ffma2_rn(a2[2 * c + 1], make_float2(q.z, q.w), y2);
        }
        return y2.x + y2.y;
    };

    float ap = matvec(xi);
    float r = bi - ap;
    float p = r;
    float rs_old = bsum(r * r);
    int it = 0, bd = 0;
    for (int step = 0; step < g.f_s; ++step) {
        ap = matvec(p);
        const float pap = bsum(p * ap);
        if (!(pap > 0.0f)) {
            bd = 1;
            break;
        }
        const float alpha = __fdividef(rs_old, pap);
        xi = fmaf(alpha, p, xi);
        r = fmaf(-alpha, ap, r);
        const float rs_new = bsum(r * r);
        ++it;
        if (rs_new == 0.0f || rs_new < eps2) break;  // ||r|| < eps, squared in fp32
        const float beta = __fdividef(rs_new, rs_old);
        p = fmaf(beta, p, r);
        rs_old = rs_new;
    }
    if (act) g.x_out[s * f + tid] = xi;
    if (tid == 0) {
        if (g.iters) g.iters[s] = it;
        if (g.broke) g.broke[s] = bd;
        if (bd && g.breakdowns) atomicAdd(g.breakdowns, 1);
    }
}

// Reference-exact float64 CG.  Thread i owns row i; the matrix lives in
// shared memory as float64 (full square when it fits, else packed from
// global).  Dot products are summed sequentially by thread 0, exactly as
// solvers.py:91-108 does.
template <bool HALF_A, bool SQ>
__global__ void cg_ref64_kernel(CgArgs g) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const int64_t s = blockIdx.x;
    if (g.nu && g.nu[s] == 0) return;
    const int f = g.f, tid = threadIdx.x, NT = blockDim.x;
    const int64_t P = packed_size(f);
    double *vp = reinterpret_cast<double *>(smraw);  // p
    double *vap = vp + f;                              // ap
    double *vr = vap + f;                              // r
    double *sc = vr + f;                               // scalars
    double *sq = sc + 8;                               // f*f when SQ
    const size_t es = HALF_A ? 2 : 4;
    const char *ga = static_cast<const char *>(g.a) + static_cast<size_t>(s) * g.a_stride * es;
    auto aval = [&](int64_t k) -> double {
        return HALF_A ? static_cast<double>(half_bits_to_float(reinterpret_cast<const uint16_t *>(ga)[k]))
                      : static_cast<double>(reinterpret_cast<const float *>(ga)[k]);
    };
    if (SQ) {
        for (int64_t k = tid; k < static_cast<int64_t>(f) * f; k += NT) {
            const int i = static_cast<int>(k / f), j = static_cast<int>(k - static_cast<int64_t>(i) * f);
            const int hi = i > j ? i : j, lo = i > j ? j : i;
            sq[k] = aval(static_cast<int64_t>(hi) * (hi + 1) / 2 + lo);
        }
    }
    auto elem = [&](int i, int j) -> double {  // sq[j, i]
        if (SQ) return sq[static_cast<int64_t>(j) * f + i];
        const int hi = i > j ? i : j, lo = i > j ? j : i;
        return aval(static_cast<int64_t>(hi) * (hi + 1) / 2 + lo);
    };
    (void)P;
    // per-thread rows i = tid, tid+NT, ... ; keep x, b in registers (<= 8 rows per thread)
    constexpr int MR = 8;
    double x[MR], b[MR];
#pragma unroll
    for (int q = 0; q < MR; ++q) {
        const int i = tid + q * NT;
        x[q] = i < f ? static_cast<double>(g.x0[s * f + i]) : 0.0;
        b[q] = i < f ? static_cast<double>(g.b[s * f + i]) : 0.0;
    }
    __syncthreads();
    auto symv = [&](const double *v, double *y) {  // y[i] = sum_j sq[j,i]*v[j], j ascending
#pragma unroll
        for (int q = 0; q < MR; ++q) {
            const int i = tid + q * NT;
            if (i >= f) continue;
            double acc = 0.0;
            for (int j = 0; j < f; ++j) acc = __dadd_rn(acc, __dmul_rn(elem(i, j), v[j]));
            y[i] = acc;
        }
        __syncthreads();
    };
    auto seqdot = [&](const double *u, const double *v, int slot) {
        if (tid == 0) {
            double acc = 0.0;
            for (int i = 0; i < f; ++i) acc = __dadd_rn(acc, __dmul_rn(u[i], v[i]));
            sc[slot] = acc;
        }
        __syncthreads();
        return sc[slot];
    };
    // ap = A x
#pragma unroll
    for (int q = 0; q < MR; ++q) {
        const int i = tid + q * NT;
        if (i < f) vr[i] = x[q];  // borrow r as the x buffer for the first matvec
    }
    __syncthreads();
    symv(vr, vap);
#pragma unroll
    for (int q = 0; q < MR; ++q) {
        const int i = tid + q * NT;
        if (i < f) {
            const double ri = __dsub_rn(b[q], vap[i]);
            vr[i] = ri;
            vp[i] = ri;
        }
    }
    __syncthreads();
    double eps;
    if (g.eps) {
        eps = g.eps[s];
    } else {
        if (tid == 0) {
            double acc = 0.0;
            for (int i = 0; i < f; ++i) {
                const double bi = static_cast<double>(g.b[s * f + i]);
                acc = __dadd_rn(acc, __dmul_rn(bi, bi));
            }
            sc[7] = acc;
        }
        __syncthreads();
        eps = g.tol * sqrt(sc[7]);
    }
    double rs_old = seqdot(vr, vr, 0);
    int it = 0, bd = 0;
    for (int step = 0; step < g.f_s; ++step) {
        symv(vp, vap);
        const double pap = seqdot(vp, vap, 1 + (step & 1));
        if (pap <= 0.0) {
            bd = 1;
            break;
        }
        const double alpha = rs_old / pap;
#pragma unroll
        for (int q = 0; q < MR; ++q) {
            const int i = tid + q * NT;
            if (i < f) {
                x[q] = __dadd_rn(x[q], __dmul_rn(alpha, vp[i]));
                vr[i] = __dsub_rn(vr[i], __dmul_rn(alpha, vap[i]));
            }
        }
        __syncthreads();
        const double rs_new = seqdot(vr, vr, 3 + (step & 1));
        ++it;
        if (rs_new == 0.0 || sqrt(rs_new) < eps) break;
        const double beta = rs_new / rs_old;
#pragma unroll
        for (int q = 0; q < MR; ++q) {
            const int i = tid + q * NT;
            if (i < f) vp[i] = __dadd_rn(vr[i], __dmul_rn(beta, vp[i]));
        }
        __syncthreads();
        rs_old = rs_new;
    }
#pragma unroll
    for (int q = 0; q < MR; ++q) {
        const int i = tid + q * NT;
        if (i < f) g.x_out[s * f + i] = __double2float_rn(x[q]);
    }
    if (tid == 0) {
        if (g.iters) g.iters[s] = it;
        if (g.broke) g.broke[s] = bd;
        if (bd && g.breakdowns) atomicAdd(g.breakdowns, 1);
    }
}

template <typename K>
static int set_smem(K k, size_t smem) {
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return set_error(CMF_ECUDA, "smem attr: %s", cudaGetErrorString(e));
    }
    return CMF_OK;
}

template <int NC4, bool H>
static int launch_rowreg(const CgArgs &g, cudaStream_t st) {
    const int64_t P = packed_size(g.f);
    const size_t abytes = ((P * (H ? 2 : 4)) + 15) & ~static_cast<size_t>(15);
    const size_t smem = abytes + (NC4 * 4 + 64) * sizeof(float) + 32 * sizeof(double);
    auto k = cg_rowreg_kernel<NC4, H>;
    int rc = set_smem(k, smem);
    if (rc) return rc;
    const int nt = ((g.f + 31) / 32) * 32;
    k<<<static_cast<unsigned>(g.nsys), nt, smem, st>>>(g);
    return check_launch("cg_rowreg_kernel");
}

template <bool H>
static int dispatch_rowreg(const CgArgs &g, cudaStream_t st) {
    const int nc4 = (g.f + 3) / 4;
    if (nc4 <= 1) return launch_rowreg<1, H>(g, st);
    if (nc4 <= 2) return launch_rowreg<2, H>(g, st);
    if (nc4 <= 4) return launch_rowreg<4, H>(g, st);
    if (nc4 <= 8) return launch_rowreg<8, H>(g, st);
    if (nc4 <= 12) return launch_rowreg<12, H>(g, st);
    if (nc4 <= 16) return launch_rowreg<16, H>(g, st);
    if (nc4 <= 20) return launch_rowreg<20, H>(g, st);
    if (nc4 <= 25) return launch_rowreg<25, H>(g, st);
    return launch_rowreg<32, H>(g, st);
}

int cg_tc_launch(const void *, int64_t, const float *, const float *, const double *, double, const int64_t *,
                 int64_t, int, int, float *, int32_t *, int32_t *, int32_t *, cudaStream_t);

int cg_launch(const void *a, bool half, int64_t a_stride, const float *b, const float *x0,
              const double *eps, double tol, const int64_t *nu, int64_t nsys, int f, int f_s,
              bool fp64, float *x_out, int32_t *iters, int32_t *broke, int32_t *breakdowns,
              cudaStream_t st) {
    if (nsys == 0) return CMF_OK;
    CgArgs g{};
    g.a = a;
    g.a_stride = a_stride;
    g.b = b;
    g.x0 = x0;
    g.eps = eps;
    g.tol = tol;
    g.nu = nu;
    g.nsys = nsys;
    g.f = f;
    g.f_s = f_s;
    g.x_out = x_out;
    g.iters = iters;
    g.broke = broke;
    g.breakdowns = breakdowns;
    const size_t es = half ? 2 : 4;
    g.vec16 = ((reinterpret_cast<uintptr_t>(a) & 15) == 0) && ((a_stride * es) % 16 == 0);
    if (half && !fp64) {  // fp16 storage: tensor-core CG (A in TMEM) when the shape allows
        const int rc = cg_tc_launch(a, a_stride, b, x0, eps, tol, nu, nsys, f, f_s, x_out, iters, broke,
                                    breakdowns, st);
        if (rc >= 0) return rc;
    }
    if (!fp64 && f <= 128) return half ? dispatch_rowreg<true>(g, st) : dispatch_rowreg<false>(g, st);
    // float64 (reference-exact) path, also the fallback for f > 128
    int nt = ((f + 31) / 32) * 32;
    if (nt > 256) nt = 256;
    if (f > 8 * nt) return set_error(CMF_EINVAL, "f=%d too large for the CG kernel", f);
    const size_t base = (3 * static_cast<size_t>(f) + 8) * sizeof(double);
    const size_t sqb = static_cast<size_t>(f) * f * sizeof(double);
    const bool sq = base + sqb <= 200 * 1024;
    const size_t smem = base + (sq ? sqb : 0);
    int rc;
    if (half) {
        if (sq) {
            rc = set_smem(cg_ref64_kernel<true, true>, smem);
            if (rc) return rc;
            cg_ref64_kernel<true, true><<<static_cast<unsigned>(nsys), nt, smem, st>>>(g);
        } else {
            cg_ref64_kernel<true, false><<<static_cast<unsigned>(nsys), nt, smem, st>>>(g);
        }
    } else {
        if (sq) {
            rc = set_smem(cg_ref64_kernel<false, true>, smem);
            if (rc) return rc;
            cg_ref64_kernel<false, true><<<static_cast<unsigned>(nsys), nt, smem, st>>>(g);
        } else {
            cg_ref64_kernel<false, false><<<static_cast<unsigned>(nsys), nt, smem, st>>>(g);
        }
    }
    return check_launch("cg_ref64_kernel");
}

}  // namespace cmf
