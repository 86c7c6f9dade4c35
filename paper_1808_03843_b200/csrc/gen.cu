// Streaming synthetic generator: any rank produces the CSR rows
// of its user range and the CSC rows of its item range of a low-rank-plus-noise
// rating matrix directly in build() order, without materialising the triples
// (Hugewiki shape: 3.1B ratings would not fit one host, nor the reference's
// gen_synthetic, data.py:270-302, which draws positions from a materialised
// range of size m*n).
//
// Every quantity is a pure function of (seed, cell), counter-based, so a shard
// needs no communication and the shards of all ranks tile the global matrix:
//   cell (u, v) present   iff  H(s_cell, u, v) < p 2^64      (Bernoulli(p))
//   ... held out (test)   iff  H(s_test, u, v) < q 2^64      (Bernoulli(q))
//   truth  X[u][k] = (H(s_x, u, k) >> 40) 2^-24 - 1/2,  Theta[v][k] likewise
//   rating = fl(dot(X[u], Theta[v]) + noise), dot = sequential non-fused fp32
//            (round after every multiply and add), noise = ((a+b)+(c+d) - 2)
//            * fl32(sigma sqrt 3) with a..d = (16-bit fields of H(s_noise, u, v)
//            + 1/2) 2^-16 -- Irwin-Hall(4) scaled to variance sigma^2, every
//            step exact or one IEEE rounding, so numpy restates it bit for bit
// with H(s, u, v) = mix64((u << 32 | v) ^ s) (splitmix64 finaliser).  The
// oracle (oracle/oracle.py: gen_stream_triples) writes the same triples, and
// tests/test_gpu_gen.py checks the device CSR/CSC against oracle.build of them.
//
// Kernels: a warp per major index (user for CSR, item for CSC) walks the minor
// range 32 cells at a time; a count pass (ballot + popc) sizes the rows, an
// int64 scan makes the pointers, a fill pass writes the minor ids (ascending,
// so the rows are in build() order) and the ratings.
#include "common.cuh"

namespace cmf {
namespace gen {

struct Params {
    uint64_t s_cell, s_test, s_noise, s_x, s_t;
    uint64_t thr_cell, thr_test;  // Bernoulli thresholds (p 2^64, q 2^64)
    int64_t m, n;
    int f;
    float noise_scale;  // fl32(sigma sqrt 3)
};

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t H(uint64_t s, uint64_t a, uint64_t b) { return mix64(((a << 32) | b) ^ s); }

__global__ void truth_kernel(uint64_t salt, int64_t rows, int f, float *out) {
    const int64_t total = rows * f;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = static_cast<uint64_t>(i / f), k = static_cast<uint64_t>(i % f);
        out[i] = static_cast<float>(H(salt, r, k) >> 40) * 5.9604644775390625e-08f - 0.5f;
    }
}

__device__ __forceinline__ float rating(const Params &p, const float *xu, const float *tv, uint64_t u, uint64_t v) {
    float acc = 0.0f;
    for (int k = 0; k < p.f; ++k) acc = __fadd_rn(acc, __fmul_rn(xu[k], tv[k]));
    const uint64_t h = H(p.s_noise, u, v);
    const float a = (static_cast<float>(h & 0xffff) + 0.5f) * 1.52587890625e-05f;
    const float b = (static_cast<float>((h >> 16) & 0xffff) + 0.5f) * 1.52587890625e-05f;
    const float c = (static_cast<float>((h >> 32) & 0xffff) + 0.5f) * 1.52587890625e-05f;
    const float d = (static_cast<float>(h >> 48) + 0.5f) * 1.52587890625e-05f;
    const float s = __fadd_rn(__fadd_rn(a, b), __fadd_rn(c, d)) - 2.0f;
    return __fadd_rn(acc, __fmul_rn(s, p.noise_scale));
}

// by_user: majors = users [lo, hi) (CSR), minors = items; else majors = items (CSC)
// minors restricted to [mlo, mhi) (e.g. a rank's own users for the local CSC of
// the reduce-scatter exchange); minor ids are written relative to mlo
__global__ void count_kernel(Params p, bool by_user, int64_t lo, int64_t hi, int64_t mlo, int64_t mhi,
                             int64_t *cnt_train, int64_t *cnt_test) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    const int64_t minors = mhi;
    for (int64_t r = lo + ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5); r < hi; r += warps) {
        int64_t ctr = 0, cte = 0;
        for (int64_t c0 = mlo; c0 < minors; c0 += 32) {
            const int64_t c = c0 + lane;
            bool in = false, te = false;
            if (c < minors) {
                const uint64_t u = by_user ? r : c, v = by_user ? c : r;
                in = H(p.s_cell, u, v) < p.thr_cell;
                te = in && H(p.s_test, u, v) < p.thr_test;
            }
            ctr += __popc(__ballot_sync(0xffffffffu, in && !te));
            cte += __popc(__ballot_sync(0xffffffffu, te));
        }
        if (lane == 0) {
            cnt_train[r - lo] = ctr;
            if (cnt_test) cnt_test[r - lo] = cte;
        }
    }
}

// fill: train cells of major r at ptr[r - lo] .. (minor ids ascending), test
// cells (CSR pass only) at tptr[r - lo] .. as (user, item, rating) triples
__global__ void fill_kernel(Params p, bool by_user, int64_t lo, int64_t hi, int64_t mlo, int64_t mhi,
                            const float *X, const float *T, const int64_t *ptr, int32_t *minor_out, float *val_out,
                            const int64_t *tptr, int64_t *tu, int64_t *tv, float *tr) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    const int64_t minors = mhi;
    const uint32_t below = (1u << lane) - 1u;
    for (int64_t r = lo + ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5); r < hi; r += warps) {
        int64_t pos = ptr[r - lo], tpos = tptr ? tptr[r - lo] : 0;
        for (int64_t c0 = mlo; c0 < minors; c0 += 32) {
            const int64_t c = c0 + lane;
            bool in = false, te = false;
            const uint64_t u = by_user ? r : c, v = by_user ? c : r;
            if (c < minors) {
                in = H(p.s_cell, u, v) < p.thr_cell;
                te = in && H(p.s_test, u, v) < p.thr_test;
            }
            const uint32_t mtr = __ballot_sync(0xffffffffu, in && !te);
            const uint32_t mte = __ballot_sync(0xffffffffu, te);
            if (in) {
                const float rv = rating(p, X + u * p.f, T + v * p.f, u, v);
                if (!te) {
                    const int64_t q = pos + __popc(mtr & below);
                    minor_out[q] = static_cast<int32_t>(c - mlo);
                    val_out[q] = rv;
                } else if (tptr) {
                    const int64_t q = tpos + __popc(mte & below);
                    tu[q] = static_cast<int64_t>(u);
                    tv[q] = static_cast<int64_t>(v);
                    tr[q] = rv;
                }
            }
            pos += __popc(mtr);
            tpos += __popc(mte);
        }
    }
}

// int64 exclusive scan, one CTA (counts of a shard's rows; fine for <= ~1e8 rows)
__global__ void scan_i64_kernel(const int64_t *in, int64_t nr, int64_t *out) {
    __shared__ int64_t wsum[32];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
    int64_t carry = 0;
    for (int64_t b0 = 0; b0 < nr; b0 += blockDim.x) {
        const int64_t i = b0 + tid;
        const int64_t v = i < nr ? in[i] : 0;
        int64_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        int64_t before = 0, total = 0;
        for (int k = 0; k < nw; ++k) {
            if (k < w) before += wsum[k];
            total += wsum[k];
        }
        if (i < nr) out[i] = carry + before + x - v;
        carry += total;
        __syncthreads();
    }
    if (tid == 0) out[nr] = carry;
}

}  // namespace gen

static gen::Params make_params(uint64_t seed, int64_t m, int64_t n, int f, uint64_t thr_cell, uint64_t thr_test,
                               float noise_scale) {
    gen::Params p{};
    const uint64_t base = seed * 0x9E3779B97F4A7C15ull;
    p.s_cell = gen::mix64(base + 1);
    p.s_test = gen::mix64(base + 2);
    p.s_noise = gen::mix64(base + 3);
    p.s_x = gen::mix64(base + 4);
    p.s_t = gen::mix64(base + 5);
    p.thr_cell = thr_cell;
    p.thr_test = thr_test;
    p.m = m;
    p.n = n;
    p.f = f;
    p.noise_scale = noise_scale;
    return p;
}

static int grid_warps(int64_t rows) {
    int64_t b = (rows + 7) / 8;  // 8 warps per block
    if (b > 148 * 16) b = 148 * 16;
    if (b < 1) b = 1;
    return static_cast<int>(b);
}

int gen_truth_launch(uint64_t seed, int which, int64_t rows, int f, float *out, cudaStream_t st) {
    const gen::Params p = make_params(seed, 0, 0, f, 0, 0, 0.0f);
    int64_t b = (rows * f + 255) / 256;
    if (b > 148 * 32) b = 148 * 32;
    if (b < 1) b = 1;
    gen::truth_kernel<<<static_cast<unsigned>(b), 256, 0, st>>>(which == 0 ? p.s_x : p.s_t, rows, f, out);
    return check_launch("gen truth");
}

int gen_count_launch(uint64_t seed, int64_t m, int64_t n, uint64_t thr_cell, uint64_t thr_test, int by_user,
                     int64_t lo, int64_t hi, int64_t mlo, int64_t mhi, int64_t *ptr, int64_t *tptr, int64_t *scratch,
                     cudaStream_t st) {
    const gen::Params p = make_params(seed, m, n, 1, thr_cell, thr_test, 0.0f);
    const int64_t nr = hi - lo;
    if (nr <= 0) {
        cudaError_t e = cudaMemsetAsync(ptr, 0, 8, st);
        if (e == cudaSuccess && tptr) e = cudaMemsetAsync(tptr, 0, 8, st);
        return e == cudaSuccess ? CMF_OK : set_error(CMF_ECUDA, "gen: %s", cudaGetErrorString(e));
    }
    int64_t *cte = tptr ? scratch + nr : nullptr;
    gen::count_kernel<<<grid_warps(nr), 256, 0, st>>>(p, by_user != 0, lo, hi, mlo, mhi, scratch, cte);
    gen::scan_i64_kernel<<<1, 1024, 0, st>>>(scratch, nr, ptr);
    if (tptr) gen::scan_i64_kernel<<<1, 1024, 0, st>>>(cte, nr, tptr);
    return check_launch("gen count");
}

int gen_fill_launch(uint64_t seed, int64_t m, int64_t n, int f, uint64_t thr_cell, uint64_t thr_test,
                    float noise_scale, int by_user, int64_t lo, int64_t hi, int64_t mlo, int64_t mhi, const float *X,
                    const float *T,
                    const int64_t *ptr, int32_t *minor_out, float *val_out, const int64_t *tptr, int64_t *tu,
                    int64_t *tv, float *tr, cudaStream_t st) {
    const gen::Params p = make_params(seed, m, n, f, thr_cell, thr_test, noise_scale);
    if (hi <= lo) return CMF_OK;
    gen::fill_kernel<<<grid_warps(hi - lo), 256, 0, st>>>(p, by_user != 0, lo, hi, mlo, mhi, X, T, ptr, minor_out,
                                                          val_out, tptr, tu, tv, tr);
    return check_launch("gen fill");
}

}  // namespace cmf
