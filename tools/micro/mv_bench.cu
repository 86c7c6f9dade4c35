// Cost of the CG matvec's small MMAs on one SM: back-to-back tcgen05.mma
// kind::f16 with M x N x 16, A from shared memory or from TMEM, one D or
// alternating D, to find the per-instruction floor the fused X side pays
// 49 times per system.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_1808_03843_b200/csrc -I ../../include -o mv_bench mv_bench.cu
#include <cstdio>
#include "tc_common.cuh"
using namespace cmf;
using namespace cmf::tc;

int cmf::set_error(int code, const char *, ...) { return code; }

__device__ __forceinline__ uint64_t desc_k(uint32_t saddr) {  // K-major SW128
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
__host__ __device__ constexpr uint32_t idesc_k(int m, int n) { return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24); }

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a_tmem), "l"(b),
                 "r"(idesc), "r"(acc)
                 : "memory");
}

__device__ __forceinline__ uint64_t desc_sw(uint32_t saddr, uint32_t layout, uint32_t sbo) {  // K-major, given swizzle
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

// Compile-time variants, descriptors hoisted out of the timed loop, one elect
// per 7-MMA group (the matvec's issue pattern).
// ATM: A from TMEM; WAIT: commit + wait after every group (a matvec round trip)
template <bool ATM, bool WAIT, int M, int N>
__global__ void bench(int iters, long long *out) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    __shared__ uint32_t slot;
    __shared__ uint64_t bar;
    for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<int4 *>(smem)[i] = make_int4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (threadIdx.x < 32) tmem_alloc(smem_u32(&slot), 512);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = slot;
    if (threadIdx.x < 32) {
        const uint32_t base = smem_u32(smem);
        constexpr uint32_t idesc = idesc_k(M, N);
        uint64_t a[7], b[7];
#pragma unroll
        for (int kk = 0; kk < 7; ++kk) {
            a[kk] = desc_k(base + (kk >> 2) * 16384 + (kk & 3) * 32);
            b[kk] = desc_k(base + 32768 + (kk >> 2) * 2048 + (kk & 3) * 32);
        }
        const uint32_t d = tm + 256;
        uint32_t ph = 0;
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 7; ++kk) {
                    if constexpr (ATM)
                        mma_ts(d, tm + 8 * kk, b[kk], idesc, kk);
                    else
                        tc_mma(d, a[kk], b[kk], idesc, kk);
                }
                if constexpr (WAIT) tc_commit(smem_u32(&bar));
            }
            __syncwarp();
            if constexpr (WAIT) {
                mbar_wait(smem_u32(&bar), ph & 1);
                ++ph;
                tc_fence_after();
            }
        }
        if (elect_one()) tc_commit(smem_u32(&bar));
        __syncwarp();
        mbar_wait(smem_u32(&bar), ph & 1);
        long long t1 = clock64();
        if (threadIdx.x == 0) out[0] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc(tm, 512);
    }
}

template <bool ATM, bool WAIT, int M, int N>
void run(long long *d) {
    const int iters = 2048;
    auto k = bench<ATM, WAIT, M, N>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
    long long cyc = 0;
    for (int rep = 0; rep < 2; ++rep) {
        k<<<148, 128, 70 * 1024>>>(iters, d);
        cudaDeviceSynchronize();
    }
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    printf("A %s %-13s M=%3d N=%3d: %6.1f cycles per MMA, %6.1f per 7-MMA group (%s)\n", ATM ? "tmem" : "smem",
           WAIT ? "commit+wait" : "streamed", M, N, (double)cyc / (iters * 7), (double)cyc / iters,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    long long *d;
    cudaMalloc(&d, 8);
    run<false, false, 128, 16>(d);
    run<false, false, 128, 32>(d);
    run<false, false, 128, 64>(d);
    run<false, false, 128, 112>(d);
    run<false, false, 128, 256>(d);
    run<false, false, 64, 8>(d);
    run<false, false, 64, 16>(d);
    run<true, false, 128, 16>(d);
    run<true, false, 128, 112>(d);
    run<false, true, 128, 16>(d);
    run<true, true, 128, 16>(d);
    run<true, true, 128, 32>(d);
    return 0;
}
