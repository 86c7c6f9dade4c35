// CSR + CSC construction on the device: replaces data.build (data.py:205-249).
//
// The reference sorts the triples by (user, item, file position) with
// np.lexsort, keeps the last element of each duplicate (user, item) run, and
// orders the CSC by (item, user).  Here both orders come from a stable LSD
// radix sort written for this layout:
//   CSR:  key = user * n + item (u64, ceil(log2(m n)) bits), payload = the
//         triple's file position t (u32).  Stability keeps file order inside a
//         duplicate run, so "last of run" is the reference's last occurrence.
//   dedup: keep[p] = last of its key run; an exclusive scan gives the CSR slot.
//   CSC:  key = item (u32, ceil(log2 n) bits) of every CSR entry, payload =
//         its CSR slot.  The CSR order is (user, item), so a stable sort by
//         item alone yields (item, user) -- the reference's lexsort((su, si)).
//   row_ptr / col_ptr come from the run boundaries of the sorted ids (empty
//   rows included), not from atomics: the whole build is deterministic.
//
// One radix pass (<= 8 bits) = histogram kernel (per-tile digit counts in
// shared memory, digit-major in HBM) + exclusive scan of the counts + scatter
// kernel.  The scatter ranks a tile of 4096 keys stably (each warp ranks its
// 512 consecutive keys with __match_any_sync and a per-warp running count per
// digit; a prefix over the 8 warps orders them), stages the tile in shared
// memory in digit order and writes each digit run contiguously (coalesced).
// HBM traffic per pass: read key+payload twice (histogram + scatter), write
// once: ~36 B per CSR entry (u64 keys), ~20 B per CSC entry.
#include "common.cuh"

namespace cmf {
namespace bld {

constexpr int TB = 256;           // threads per tile (== RADIX: one thread per digit)
constexpr int IPT = 16;           // keys per thread
constexpr int TILE = TB * IPT;    // 4096 keys per tile
constexpr int NW = TB / 32;       // 8 warps; warp w ranks tile positions [512 w, 512 w + 512)
constexpr int WCHUNK = TILE / NW; // 512
constexpr int RADIX = 256;
static_assert(TB == RADIX, "one thread per digit in the offset scan");

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// exclusive block scan of one uint32 per thread (TB threads); returns the total
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t &excl, uint32_t *wsum) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    uint32_t before = 0, total = 0;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
        const uint32_t s = wsum[k];
        if (k < w) before += s;
        total += s;
    }
    excl = before + x - v;
    __syncthreads();  // wsum is reused by the caller's next scan
    return total;
}

// ------------------------------------------------------------ validation
template <typename I>
__global__ void max_ids_kernel(const I *user, const I *item, int64_t k, long long *mx) {
    long long mu = -1, mi = -1;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < k;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        mu = max(mu, static_cast<long long>(user[t]));
        mi = max(mi, static_cast<long long>(item[t]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mu = max(mu, __shfl_xor_sync(0xffffffffu, mu, o));
        mi = max(mi, __shfl_xor_sync(0xffffffffu, mi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(mx, mu);
        atomicMax(mx + 1, mi);
    }
}

// first t whose (user, item) lies outside [0, m) x [0, n) (the reference names it)
template <typename I>
__global__ void first_bad_kernel(const I *user, const I *item, int64_t k, int64_t m, int64_t n,
                                 unsigned long long *first) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < k;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t u = static_cast<int64_t>(user[t]), v = static_cast<int64_t>(item[t]);
        if (u < 0 || u >= m || v < 0 || v >= n) atomicMin(first, static_cast<unsigned long long>(t));
    }
}

template <typename I>
__global__ void make_keys_kernel(const I *user, const I *item, int64_t k, uint64_t n, uint64_t *key,
                                 uint32_t *pay) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < k;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        key[t] = static_cast<uint64_t>(user[t]) * n + static_cast<uint64_t>(item[t]);
        pay[t] = static_cast<uint32_t>(t);
    }
}

// ------------------------------------------------------------ radix pass
template <typename K>
__global__ void __launch_bounds__(TB) radix_hist_kernel(const K *keys, int64_t count, int shift, int bits,
                                                        uint32_t *hist, int64_t ntiles) {
    __shared__ uint32_t h[RADIX];
    const int tid = threadIdx.x;
    h[tid] = 0;
    __syncthreads();
    const int64_t base = static_cast<int64_t>(blockIdx.x) * TILE;
    const uint32_t mask = (1u << bits) - 1u;
#pragma unroll 4
    for (int r = 0; r < IPT; ++r) {
        const int64_t idx = base + r * TB + tid;
        if (idx < count) atomicAdd(&h[static_cast<uint32_t>(keys[idx] >> shift) & mask], 1u);
    }
    __syncthreads();
    if (tid < (1 << bits)) hist[tid * ntiles + blockIdx.x] = h[tid];
}

template <typename K>
__global__ void __launch_bounds__(TB) radix_scatter_kernel(const K *__restrict__ kin, const uint32_t *__restrict__ pin,
                                                           K *__restrict__ kout, uint32_t *__restrict__ pout,
                                                           int64_t count, int shift, int bits,
                                                           const uint32_t *__restrict__ off, int64_t ntiles) {
    extern __shared__ __align__(16) unsigned char smem[];
    K *skey = reinterpret_cast<K *>(smem);
    uint32_t *spay = reinterpret_cast<uint32_t *>(skey + TILE);
    uint32_t *wrun = spay + TILE;     // [NW][RADIX] running counts, then prefix over warps
    uint32_t *loff = wrun + NW * RADIX;  // tile-local exclusive offset per digit
    uint32_t *gbase = loff + RADIX;      // global offset of this tile's run per digit
    uint32_t *wsum = gbase + RADIX;      // NW scan partials
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t base = static_cast<int64_t>(blockIdx.x) * TILE;
    const int nh = static_cast<int>(min(static_cast<int64_t>(TILE), count - base));
    const uint32_t mask = (1u << bits) - 1u;
    for (int i = tid; i < NW * RADIX; i += TB) wrun[i] = 0;
    __syncthreads();
    K key[IPT];
    uint32_t pay[IPT], rk[IPT];
    int dg[IPT];
    uint32_t *myrun = wrun + w * RADIX;
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
        const int pos = w * WCHUNK + r * 32 + lane;
        const bool ok = pos < nh;
        int d = RADIX;  // sentinel: past the end (grouped together, never counted)
        if (ok) {
            key[r] = kin[base + pos];
            pay[r] = pin[base + pos];
            d = static_cast<int>(static_cast<uint32_t>(key[r] >> shift) & mask);
        }
        dg[r] = d;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t below = __popc(peers & lanemask_lt());
        if (ok) rk[r] = myrun[d] + below;
        __syncwarp();
        if (ok && below == 0) myrun[d] += __popc(peers);  // the lowest peer updates the run
        __syncwarp();
    }
    __syncthreads();
    // thread d: prefix of digit d over the warps, then the tile-local digit offsets
    {
        const int d = tid;
        uint32_t s = 0;
#pragma unroll
        for (int k = 0; k < NW; ++k) {
            const uint32_t c = wrun[k * RADIX + d];
            wrun[k * RADIX + d] = s;
            s += c;
        }
        uint32_t ex;
        block_excl_scan(s, ex, wsum);
        loff[d] = ex;
        gbase[d] = d <= static_cast<int>(mask) ? off[d * ntiles + blockIdx.x] : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
        if (dg[r] < RADIX) {
            const uint32_t p = loff[dg[r]] + myrun[dg[r]] + rk[r];
            skey[p] = key[r];
            spay[p] = pay[r];
        }
    }
    __syncthreads();
    for (int i = tid; i < nh; i += TB) {
        const K kk = skey[i];
        const uint32_t d = static_cast<uint32_t>(kk >> shift) & mask;
        const uint32_t g = gbase[d] + (static_cast<uint32_t>(i) - loff[d]);
        kout[g] = kk;
        pout[g] = spay[i];
    }
}

template <typename K>
constexpr size_t scatter_smem() {
    return TILE * (sizeof(K) + 4) + (NW * RADIX + 2 * RADIX + NW) * 4;
}

// ------------------------------------------------------------ exclusive scan (uint32, in place allowed)
__global__ void __launch_bounds__(TB) scan_reduce_kernel(const uint32_t *in, int64_t L, uint32_t *part) {
    __shared__ uint32_t wsum[NW];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * TILE;
    uint32_t s = 0;
#pragma unroll 4
    for (int r = 0; r < IPT; ++r) {
        const int64_t i = base + r * TB + threadIdx.x;
        if (i < L) s += in[i];
    }
    uint32_t ex;
    const uint32_t tot = block_excl_scan(s, ex, wsum);
    if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

// one CTA: exclusive scan of the nb tile sums, in place; *total = the sum
__global__ void __launch_bounds__(TB) scan_part_kernel(uint32_t *part, int64_t nb, uint32_t *total) {
    __shared__ uint32_t wsum[NW];
    uint32_t carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += TB) {
        const int64_t i = b0 + threadIdx.x;
        const uint32_t v = i < nb ? part[i] : 0u;
        uint32_t ex;
        const uint32_t tot = block_excl_scan(v, ex, wsum);
        if (i < nb) part[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0 && total) *total = carry;
}

// tile b: thread t owns IPT consecutive elements
__global__ void __launch_bounds__(TB) scan_down_kernel(const uint32_t *in, uint32_t *out, int64_t L,
                                                       const uint32_t *part) {
    __shared__ uint32_t wsum[NW];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * TILE + threadIdx.x * IPT;
    uint32_t v[IPT], s = 0;
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        v[j] = base + j < L ? in[base + j] : 0u;
        s += v[j];
    }
    uint32_t ex;
    block_excl_scan(s, ex, wsum);
    uint32_t run = part[blockIdx.x] + ex;
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        if (base + j < L) out[base + j] = run;
        run += v[j];
    }
}

// ------------------------------------------------------------ dedup, outputs
// keep[p] = 1 if p is the last element of its key run (the reference's "last occurrence")
__global__ void keep_flags_kernel(const uint64_t *key, int64_t k, uint32_t *keep) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < k;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x)
        keep[p] = (p + 1 == k || key[p] != key[p + 1]) ? 1u : 0u;
}

// CSR slot q = slot[p] of every kept entry: col_idx, csr_val (from the file
// position), and the row id (u32) for the boundaries and the CSC
__global__ void csr_out_kernel(const uint64_t *key, const uint32_t *pay, const uint32_t *slot, int64_t k,
                               uint64_t n, const float *rating, int32_t *col_idx, float *csr_val,
                               uint32_t *row_of, uint32_t *item_key, uint32_t *item_pay) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < k;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t kk = key[p];
        if (p + 1 < k && kk == key[p + 1]) continue;  // an earlier duplicate
        const uint32_t q = slot[p];
        const uint64_t u = kk / n;
        const uint32_t v = static_cast<uint32_t>(kk - u * n);
        col_idx[q] = static_cast<int32_t>(v);
        csr_val[q] = rating[pay[p]];
        row_of[q] = static_cast<uint32_t>(u);
        item_key[q] = v;
        item_pay[q] = q;
    }
}

__global__ void csc_out_kernel(const uint32_t *pay, int64_t nnz, const uint32_t *row_of, const float *csr_val,
                               int32_t *row_idx, float *csc_val) {
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < nnz;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t q = pay[j];
        row_idx[j] = static_cast<int32_t>(row_of[q]);
        csc_val[j] = csr_val[q];
    }
}

// ptr[v] = first position whose sorted id is >= v, for v in [0, nrows]
__global__ void bounds_kernel(const uint32_t *ids, int64_t cnt, int64_t nrows, int64_t *ptr) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p <= cnt;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t lo = p == 0 ? 0 : static_cast<int64_t>(ids[p - 1]) + 1;
        const int64_t hi = p == cnt ? nrows : static_cast<int64_t>(ids[p]);
        for (int64_t v = lo; v <= hi; ++v) ptr[v] = p;
    }
}

__global__ void fill_i64_kernel(int64_t *p, int64_t count, int64_t v) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = v;
}

}  // namespace bld

static inline int grid_for(int64_t count, int per_block = 256) {
    int64_t g = (count + per_block - 1) / per_block;
    if (g < 1) g = 1;
    return static_cast<int>(g < 148 * 32 ? g : 148 * 32);
}

static inline int bit_length(uint64_t x) { return x == 0 ? 0 : 64 - __builtin_clzll(x); }

static inline int64_t align256(int64_t b) { return (b + 255) & ~int64_t(255); }

// workspace carve-up for k triples (see cmf_build_workspace_bytes)
struct BuildWs {
    uint64_t *keyA, *keyB;
    uint32_t *payA, *payB, *slot, *row_of, *hist, *part;
    unsigned long long *scal;  // [0] first bad, [1..2] max ids (long long), [3] u32 total
    int64_t bytes;
};

static BuildWs carve(void *ws, int64_t k) {
    BuildWs w{};
    const int64_t ntiles = (k + bld::TILE - 1) / bld::TILE;
    const int64_t hist_len = bld::RADIX * (ntiles > 0 ? ntiles : 1);
    const int64_t part_len = (hist_len > k ? hist_len : k) / bld::TILE + 2;
    char *p = static_cast<char *>(ws);
    int64_t o = 0;
    auto take = [&](int64_t b) {
        char *r = p ? p + o : nullptr;
        o += align256(b);
        return r;
    };
    w.scal = reinterpret_cast<unsigned long long *>(take(64));
    w.keyA = reinterpret_cast<uint64_t *>(take(8 * k));
    w.keyB = reinterpret_cast<uint64_t *>(take(8 * k));
    w.payA = reinterpret_cast<uint32_t *>(take(4 * k));
    w.payB = reinterpret_cast<uint32_t *>(take(4 * k));
    w.slot = reinterpret_cast<uint32_t *>(take(4 * k));
    w.row_of = reinterpret_cast<uint32_t *>(take(4 * k));
    w.hist = reinterpret_cast<uint32_t *>(take(4 * hist_len));
    w.part = reinterpret_cast<uint32_t *>(take(4 * part_len));
    w.bytes = o;
    return w;
}

int64_t build_workspace_bytes(int64_t k) { return carve(nullptr, k).bytes; }

// exclusive scan of L uint32 (in -> out, may alias); *total (device) = the sum
static int excl_scan(const uint32_t *in, uint32_t *out, int64_t L, uint32_t *part, uint32_t *total,
                     cudaStream_t st) {
    const int64_t nb = (L + bld::TILE - 1) / bld::TILE;
    if (nb == 0) return CMF_OK;
    bld::scan_reduce_kernel<<<static_cast<unsigned>(nb), bld::TB, 0, st>>>(in, L, part);
    bld::scan_part_kernel<<<1, bld::TB, 0, st>>>(part, nb, total);
    bld::scan_down_kernel<<<static_cast<unsigned>(nb), bld::TB, 0, st>>>(in, out, L, part);
    return check_launch("build scan");
}

// stable LSD radix sort of (key, payload) over the low `bits` bits; the result
// ends in (*k0, *p0) (buffers swap as passes complete)
template <typename K>
static int radix_sort(K *&k0, uint32_t *&p0, K *&k1, uint32_t *&p1, int64_t count, int bits, uint32_t *hist,
                      uint32_t *part, cudaStream_t st) {
    if (count <= 1 || bits <= 0) return CMF_OK;
    const int npass = (bits + 7) / 8;
    const int width = (bits + npass - 1) / npass;
    const int64_t ntiles = (count + bld::TILE - 1) / bld::TILE;
    constexpr size_t smem = bld::scatter_smem<K>();
    cudaError_t e = cudaFuncSetAttribute(bld::radix_scatter_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return set_error(CMF_ECUDA, "radix smem attr: %s", cudaGetErrorString(e));
    for (int pass = 0, shift = 0; pass < npass; ++pass, shift += width) {
        const int b = bits - shift < width ? bits - shift : width;
        bld::radix_hist_kernel<K><<<static_cast<unsigned>(ntiles), bld::TB, 0, st>>>(k0, count, shift, b, hist, ntiles);
        int rc = excl_scan(hist, hist, (int64_t(1) << b) * ntiles, part, nullptr, st);
        if (rc != CMF_OK) return rc;
        bld::radix_scatter_kernel<K><<<static_cast<unsigned>(ntiles), bld::TB, smem, st>>>(k0, p0, k1, p1, count, shift,
                                                                                          b, hist, ntiles);
        rc = check_launch("radix pass");
        if (rc != CMF_OK) return rc;
        K *tk = k0;
        k0 = k1;
        k1 = tk;
        uint32_t *tp = p0;
        p0 = p1;
        p1 = tp;
    }
    return CMF_OK;
}

template <typename I>
static int build_impl(const I *user, const I *item, const float *rating, int64_t k, int64_t *mn, int64_t *row_ptr,
                      int32_t *col_idx, float *csr_val, int64_t *col_ptr, int32_t *row_idx, float *csc_val,
                      void *ws, int64_t ws_bytes, int64_t *nnz_host, int64_t *bad_host, cudaStream_t st) {
    *bad_host = -1;
    *nnz_host = 0;
    if (k >= (int64_t(1) << 32) - 1) return set_error(CMF_EINVAL, "build supports < 2^32 - 1 triples per call");
    BuildWs w = carve(ws, k);
    if (ws == nullptr || ws_bytes < w.bytes)
        return set_error(CMF_EINVAL, "build workspace too small: %lld < %lld bytes", (long long)ws_bytes,
                         (long long)w.bytes);
    cudaError_t e;
    if (mn[0] < 0 || mn[1] < 0) {  // m, n default to max id + 1 (0 for no triples)
        long long init[2] = {-1, -1};
        e = cudaMemcpyAsync(w.scal + 1, init, sizeof(init), cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return set_error(CMF_ECUDA, "build: %s", cudaGetErrorString(e));
        if (k) bld::max_ids_kernel<I><<<grid_for(k), 256, 0, st>>>(user, item, k, reinterpret_cast<long long *>(w.scal + 1));
        long long mx[2];
        e = cudaMemcpyAsync(mx, w.scal + 1, sizeof(mx), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return set_error(CMF_ECUDA, "build: %s", cudaGetErrorString(e));
        if (mn[0] < 0) mn[0] = mx[0] + 1;
        if (mn[1] < 0) mn[1] = mx[1] + 1;
    }
    if (row_ptr == nullptr) return CMF_OK;  // query: resolve m, n only
    const int64_t m = mn[0], n = mn[1];
    if (m >= (int64_t(1) << 32) || n >= (int64_t(1) << 31))
        return set_error(CMF_EINVAL, "build: %lld x %lld exceeds 32-bit row / 31-bit column ids", (long long)m,
                         (long long)n);
    if (k) {
        const unsigned long long none = ~0ull;
        e = cudaMemcpyAsync(w.scal, &none, sizeof(none), cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return set_error(CMF_ECUDA, "build: %s", cudaGetErrorString(e));
        bld::first_bad_kernel<I><<<grid_for(k), 256, 0, st>>>(user, item, k, m, n, w.scal);
        unsigned long long first = 0;
        e = cudaMemcpyAsync(&first, w.scal, sizeof(first), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return set_error(CMF_ECUDA, "build: %s", cudaGetErrorString(e));
        if (first != none) {
            *bad_host = static_cast<int64_t>(first);
            return set_error(CMF_EINVAL, "triple %lld out of range for a %lld x %lld matrix", (long long)first,
                             (long long)m, (long long)n);
        }
    }
    if (k == 0) {
        bld::fill_i64_kernel<<<grid_for(m + 1), 256, 0, st>>>(row_ptr, m + 1, 0);
        bld::fill_i64_kernel<<<grid_for(n + 1), 256, 0, st>>>(col_ptr, n + 1, 0);
        return check_launch("build (empty)");
    }
    // CSR order: stable sort by user * n + item
    bld::make_keys_kernel<I><<<grid_for(k), 256, 0, st>>>(user, item, k, static_cast<uint64_t>(n), w.keyA, w.payA);
    uint64_t *k0 = w.keyA, *k1 = w.keyB;
    uint32_t *p0 = w.payA, *p1 = w.payB;
    const uint64_t cells = static_cast<uint64_t>(m) * static_cast<uint64_t>(n);
    int rc = radix_sort<uint64_t>(k0, p0, k1, p1, k, bit_length(cells - 1), w.hist, w.part, st);
    if (rc != CMF_OK) return rc;
    // dedup: slot = exclusive scan of the "last of run" flags
    uint32_t *total = reinterpret_cast<uint32_t *>(w.scal + 3);
    bld::keep_flags_kernel<<<grid_for(k), 256, 0, st>>>(k0, k, w.slot);
    rc = excl_scan(w.slot, w.slot, k, w.part, total, st);
    if (rc != CMF_OK) return rc;
    uint32_t nnz32 = 0;
    e = cudaMemcpyAsync(&nnz32, total, sizeof(nnz32), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return set_error(CMF_ECUDA, "build: %s", cudaGetErrorString(e));
    const int64_t nnz = nnz32;
    *nnz_host = nnz;
    // CSR outputs; the CSC keys (item of every CSR slot, payload = the slot) go
    // into the 32-bit halves of the free key buffer
    uint32_t *ik0 = reinterpret_cast<uint32_t *>(k1), *ik1 = ik0 + k;
    uint32_t *ip0 = p1, *ip1 = p0;  // p0 (file positions) is dead once csr_out_kernel ran
    bld::csr_out_kernel<<<grid_for(k), 256, 0, st>>>(k0, p0, w.slot, k, static_cast<uint64_t>(n), rating, col_idx,
                                                     csr_val, w.row_of, ik0, ip0);
    bld::bounds_kernel<<<grid_for(nnz + 1), 256, 0, st>>>(w.row_of, nnz, m, row_ptr);
    rc = check_launch("build csr");
    if (rc != CMF_OK) return rc;
    // CSC order: stable sort of the CSR entries by item
    rc = radix_sort<uint32_t>(ik0, ip0, ik1, ip1, nnz, bit_length(static_cast<uint64_t>(n) - 1), w.hist, w.part, st);
    if (rc != CMF_OK) return rc;
    bld::csc_out_kernel<<<grid_for(nnz), 256, 0, st>>>(ip0, nnz, w.row_of, csr_val, row_idx, csc_val);
    bld::bounds_kernel<<<grid_for(nnz + 1), 256, 0, st>>>(ik0, nnz, n, col_ptr);
    return check_launch("build csc");
}

int build_launch(const void *user, const void *item, bool idx64, const float *rating, int64_t k, int64_t *mn,
                 int64_t *row_ptr, int32_t *col_idx, float *csr_val, int64_t *col_ptr, int32_t *row_idx,
                 float *csc_val, void *ws, int64_t ws_bytes, int64_t *nnz_host, int64_t *bad_host, cudaStream_t st) {
    if (idx64)
        return build_impl(static_cast<const int64_t *>(user), static_cast<const int64_t *>(item), rating, k, mn,
                          row_ptr, col_idx, csr_val, col_ptr, row_idx, csc_val, ws, ws_bytes, nnz_host, bad_host, st);
    return build_impl(static_cast<const int32_t *>(user), static_cast<const int32_t *>(item), rating, k, mn, row_ptr,
                      col_idx, csr_val, col_ptr, row_idx, csc_val, ws, ws_bytes, nnz_host, bad_host, st);
}

}  // namespace cmf

// ------------------------------------------------------------ grouping without dedup
namespace cmf {
namespace bld {
template <typename I>
__global__ void group_keys_kernel(const I *rows, const I *cols, int64_t k, uint32_t *key, uint32_t *pay) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < k;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        key[t] = static_cast<uint32_t>(rows[t]);
        pay[t] = static_cast<uint32_t>(cols[t]);
    }
}
}  // namespace bld

int64_t group_workspace_bytes(int64_t k) {
    const int64_t ntiles = (k + bld::TILE - 1) / bld::TILE;
    const int64_t hist = bld::RADIX * (ntiles > 0 ? ntiles : 1);
    return 4 * align256(4 * k) + align256(4 * hist) + align256(4 * (hist / bld::TILE + 2));
}

// (row, col) pairs -> indptr[nrows+1] + cols in stable row order (file order kept
// inside a row, duplicates kept): the positives' grouping for mean_percentile_rank
template <typename I>
static int group_impl(const I *rows, const I *cols, int64_t k, int64_t nrows, int64_t *indptr, int32_t *cols_out,
                      void *ws, int64_t ws_bytes, cudaStream_t st) {
    if (ws_bytes < group_workspace_bytes(k)) return set_error(CMF_EINVAL, "group workspace too small");
    char *p = static_cast<char *>(ws);
    uint32_t *k0 = reinterpret_cast<uint32_t *>(p);
    uint32_t *k1 = reinterpret_cast<uint32_t *>(p + align256(4 * k));
    uint32_t *p0 = reinterpret_cast<uint32_t *>(p + 2 * align256(4 * k));
    uint32_t *p1 = reinterpret_cast<uint32_t *>(p + 3 * align256(4 * k));
    const int64_t ntiles = (k + bld::TILE - 1) / bld::TILE;
    uint32_t *hist = reinterpret_cast<uint32_t *>(p + 4 * align256(4 * k));
    uint32_t *part = reinterpret_cast<uint32_t *>(p + 4 * align256(4 * k) +
                                                  align256(4 * bld::RADIX * (ntiles > 0 ? ntiles : 1)));
    if (k == 0) {
        bld::fill_i64_kernel<<<grid_for(nrows + 1), 256, 0, st>>>(indptr, nrows + 1, 0);
        return check_launch("group (empty)");
    }
    bld::group_keys_kernel<I><<<grid_for(k), 256, 0, st>>>(rows, cols, k, k0, p0);
    int rc = radix_sort<uint32_t>(k0, p0, k1, p1, k, bit_length(static_cast<uint64_t>(nrows > 1 ? nrows - 1 : 1)),
                                  hist, part, st);
    if (rc != CMF_OK) return rc;
    bld::bounds_kernel<<<grid_for(k + 1), 256, 0, st>>>(k0, k, nrows, indptr);
    cudaError_t e = cudaMemcpyAsync(cols_out, p0, 4 * k, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return set_error(CMF_ECUDA, "group: %s", cudaGetErrorString(e));
    return check_launch("group");
}

int group_launch(const void *rows, const void *cols, bool idx64, int64_t k, int64_t nrows, int64_t *indptr,
                 int32_t *cols_out, void *ws, int64_t ws_bytes, cudaStream_t st) {
    if (idx64)
        return group_impl(static_cast<const int64_t *>(rows), static_cast<const int64_t *>(cols), k, nrows, indptr,
                          cols_out, ws, ws_bytes, st);
    return group_impl(static_cast<const int32_t *>(rows), static_cast<const int32_t *>(cols), k, nrows, indptr,
                      cols_out, ws, ws_bytes, st);
}

}  // namespace cmf
