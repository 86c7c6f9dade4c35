// UMMA (tcgen05.mma kind::f16) throughput from shared memory: back-to-back
// 128 x N x 16 MMAs on one SM, operands MN-major vs K-major (SWIZZLE_128B).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_1808_03843_b200/csrc -I ../../include -o umma_bench umma_bench.cu
#include <cstdio>
#include <vector>
#include "tc_common.cuh"
using namespace cmf;
using namespace cmf::tc;

int cmf::set_error(int code, const char *, ...) { return code; }

__device__ __forceinline__ uint64_t desc_k(uint32_t saddr) {  // K-major SW128: SBO 1024, LBO 1
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
constexpr uint32_t idesc_k(int m, int n) {  // both K-major
    return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

template <bool KMAJ>
__global__ void bench(int N, int iters, long long *out, int mode, const uint4 *tab, const int *idx) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    __shared__ uint32_t slot;
    __shared__ uint64_t bar, bar2;
    __shared__ int slot_done;
    if (threadIdx.x == 0) slot_done = 0;
    for (int i = threadIdx.x; i < 200 * 1024 / 16; i += blockDim.x) reinterpret_cast<int4 *>(smem)[i] = make_int4(0, 0, 0, 0);
    if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); mbar_init(smem_u32(&bar2), 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    if (threadIdx.x < 32) tmem_alloc(smem_u32(&slot), 256);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    uint32_t tm = slot;
    if (threadIdx.x < 32) {
        const uint32_t base = smem_u32(smem);
        const uint32_t idesc = KMAJ ? idesc_k(128, N) : make_idesc(128, N);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            // 4 K-steps over a 64-row stage, like the Gram
            for (int kk = 0; kk < 4; ++kk) {
                uint64_t a, b;
                if (KMAJ) { a = desc_k(base + kk * 32); b = desc_k(base + 16384 + kk * 32); }
                else { a = make_desc(base + (mode & 4 ? (i % 12) * 16384 : 0) + kk * 2048); b = a; }
                if (elect_one()) tc_mma(tm, a, b, idesc, 1);
                __syncwarp();
            }
            if (mode & 1) {  // commit per stage, like the pipeline's empty barrier
                if (elect_one()) tc_commit(smem_u32(&bar2));
                __syncwarp();
            }
        }
        if (elect_one()) tc_commit(smem_u32(&bar));
        __syncwarp();
        mbar_wait(smem_u32(&bar), 0);
        long long t1 = clock64();
        if (threadIdx.x == 0) { out[0] = t1 - t0; *(volatile int *)&slot_done = 1; }
    }
    else if ((mode & 2) && threadIdx.x >= 64) {  // concurrent cp.async gather traffic (2 warps... blockDim-64 threads)
        const int lane = threadIdx.x & 31, c = lane & 15, hrow = lane >> 4;
        const int wid = (threadIdx.x - 64) >> 5;
        const uint32_t dst0 = smem_u32(smem) + (wid % 12) * 16384;
        for (int rep = 0; *(volatile int *)&slot_done == 0; ++rep) {
            int myidx = idx[(rep * 64 + lane + wid * 977) & 1048575];
#pragma unroll
            for (int t = 0; t < 32; ++t) {
                int ix = __shfl_sync(0xffffffffu, myidx, t);
                if (c < 13) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst0 + ((2 * t + hrow) * 16 + c) * 16 % 16384), "l"(tab + (long)ix * 13 + c));
            }
            asm volatile("cp.async.commit_group;");
            asm volatile("cp.async.wait_group 6;");
        }
        asm volatile("cp.async.wait_group 0;");
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tm, 256); }
}

int main() {
    long long *d;
    cudaMalloc(&d, 8);
    uint4 *tab; int *idx;
    cudaMalloc(&tab, 17770L * 208);
    cudaMalloc(&idx, 1048576 * 4);
    { std::vector<int> h(1048576); uint64_t s = 1; for (auto &v : h) { s = s * 6364136223846793005ull + 1; v = (int)((s >> 33) % 17770); }
      cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice); }
    int iters = 4096;
    for (int mode : {0, 4, 5, 7})
    for (int kmaj = 0; kmaj < 1; ++kmaj)
        for (int N : {112}) {
            long long cyc = 0;
            auto k = kmaj ? bench<true> : bench<false>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
            for (int rep = 0; rep < 2; ++rep) {
                k<<<148, (mode & 2) ? 512 : 128, 220 * 1024>>>(N, iters, d, mode, tab, idx);
                cudaDeviceSynchronize();
            }
            cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
            double per = (double)cyc / (iters * 4);
            printf("mode %d (commit/stage %d, gather traffic %d) %s N=%3d: %.1f cycles per 128x%dx16 MMA -> %.0f flops/clk (%s)\n", kmaj ? "K-major " : "MN-major", N,
                   per, N, 2.0 * 128 * N * 16 / per, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
