// B200 latency microbenchmarks for the CG consumer's primitives (one CTA, 128
// threads = one CG group; clock64 deltas averaged over many repetitions):
// shuffle butterfly, named barrier, tcgen05.ld x1 + wait, and a 7-MMA
// (128x16x16 kind::f16, A in TMEM, B in smem) + commit + mbarrier round trip.
#include <cstdio>
#include "tc_common.cuh"
using namespace cmf;
using namespace cmf::tc;
int cmf::set_error(int code, const char *, ...) { return code; }

__device__ __forceinline__ uint32_t tld1(uint32_t taddr) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr) : "memory");
    return v;
}
__device__ __forceinline__ void mma_ta(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(a), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ uint64_t desc_k(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF); d |= (uint64_t)1 << 16; d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61;
    return d;
}

__global__ void bench(long long *out, int reps) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    __shared__ uint32_t slot;
    __shared__ uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 8192 / 16; i += blockDim.x) reinterpret_cast<int4 *>(smem)[i] = make_int4(0, 0, 0, 0);
    if (tid == 0) { mbar_init(smem_u32(&bar), 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    if (warp == 0) tmem_alloc(smem_u32(&slot), 256);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = slot, lb = (uint32_t)(warp * 32) << 16;
    float x = tid * 0.001f;
    long long t0, t1;
    // 1) shuffle butterfly of 2 values
    t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        float a = x, b = x * 2;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) { a += __shfl_xor_sync(~0u, a, o); b += __shfl_xor_sync(~0u, b, o); }
        x = a * 1e-9f + b * 1e-9f;
    }
    t1 = clock64();
    if (tid == 0) out[0] = (t1 - t0) / reps;
    // 2) named barrier (128 threads)
    t0 = clock64();
    for (int r = 0; r < reps; ++r) named_bar(1, 128);
    t1 = clock64();
    if (tid == 0) out[1] = (t1 - t0) / reps;
    // 3) tcgen05.ld x1 + wait (dependent)
    uint32_t acc = 0;
    t0 = clock64();
    for (int r = 0; r < reps; ++r) { acc += tld1(tm + lb + (acc & 1)); tmem_ld_wait(); }
    t1 = clock64();
    if (tid == 0) out[2] = (t1 - t0) / reps;
    // 4) 7 MMAs (A in TMEM cols 0..55, B in smem, D in cols 64..79) + commit + wait, then ld
    const uint32_t idesc = (1u << 4) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t bop = smem_u32(smem);
    uint32_t ph = 0;
    t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        named_bar(1, 128);
        if (warp == 0) {
            if (elect_one()) {
                tc_fence_after();
                for (int kk = 0; kk < 7; ++kk) mma_ta(tm + 64, tm + 8 * kk, desc_k(bop + (kk >> 2) * 2048 + (kk & 3) * 32), idesc, kk);
                tc_commit(smem_u32(&bar));
            }
            __syncwarp();
        }
        mbar_wait(smem_u32(&bar), ph & 1);
        ++ph;
        tc_fence_after();
        acc += tld1(tm + lb + 64);
        tmem_ld_wait();
    }
    t1 = clock64();
    if (tid == 0) out[3] = (t1 - t0) / reps;
    // 5) same with 1 MMA
    t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        named_bar(1, 128);
        if (warp == 0) {
            if (elect_one()) { tc_fence_after(); mma_ta(tm + 64, tm, desc_k(bop), idesc, 0); tc_commit(smem_u32(&bar)); }
            __syncwarp();
        }
        mbar_wait(smem_u32(&bar), ph & 1);
        ++ph;
        tc_fence_after();
        acc += tld1(tm + lb + 64);
        tmem_ld_wait();
    }
    t1 = clock64();
    if (tid == 0) out[4] = (t1 - t0) / reps;
    // 6) sts + bar + lds round trip
    float *sf = reinterpret_cast<float *>(smem + 4096);
    t0 = clock64();
    for (int r = 0; r < reps; ++r) { sf[tid] = x; named_bar(1, 128); x += sf[(tid + 33) & 127] * 1e-9f; named_bar(1, 128); }
    t1 = clock64();
    if (tid == 0) out[5] = (t1 - t0) / reps;
    if (tid == 0) out[7] = acc + (long long)x;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tm, 256); }
}

int main() {
    long long *d, h[8];
    cudaMalloc(&d, 64);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 1024);
    for (int it = 0; it < 2; ++it) bench<<<1, 128, 16 * 1024>>>(d, 1000);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    printf("shfl butterfly (5 levels x 2 values): %lld cycles\n", h[0]);
    printf("named barrier (128 thr):              %lld cycles\n", h[1]);
    printf("tcgen05.ld x1 + wait (dependent):     %lld cycles\n", h[2]);
    printf("bar + 7 MMA + commit + wait + ld:     %lld cycles\n", h[3]);
    printf("bar + 1 MMA + commit + wait + ld:     %lld cycles\n", h[4]);
    printf("sts + bar + lds + bar:                %lld cycles\n", h[5]);
    return 0;
}
