// Which shared-memory layout does tcgen05.cp.128x256b read?  A 128 x 112 fp32
// matrix M[r][c] = r * 1000 + c is stored as no-swizzle core matrices (8 rows x
// 16 bytes, 128 contiguous bytes): chunk cc (4 columns) of row group rg at
// cc * 2048 + rg * 128 + (r % 8) * 16.  Fourteen copies (8 columns each) with
// (LBO, SBO) = (2048, 128) and then (128, 2048) land in TMEM columns 0..111;
// every thread checks its lane and the mismatch counts are printed.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --expt-relaxed-constexpr -I ../../paper_1808_03843_b200/csrc -I ../../include -o cp_probe cp_probe.cu
#include <cstdio>
#include "tc_common.cuh"
using namespace cmf;
using namespace cmf::tc;

int cmf::set_error(int code, const char *, ...) { return code; }

__device__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;  // version (sm100); layout type 0 = SWIZZLE_NONE
    return d;
}

__global__ void probe(int mode, int *bad, float *sample) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    __shared__ uint32_t slot;
    __shared__ uint64_t bar;
    const int tid = threadIdx.x;
    float *m = reinterpret_cast<float *>(smem);
    for (int k = tid; k < 128 * 112; k += blockDim.x) {
        const int r = k / 112, c = k % 112;
        const int off = (c >> 2) * 2048 + (r >> 3) * 128 + (r & 7) * 16 + (c & 3) * 4;
        m[off / 4] = static_cast<float>(r * 1000 + c);
    }
    if (tid == 0) {
        mbar_init(smem_u32(&bar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (tid < 32) tmem_alloc(smem_u32(&slot), 128);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = slot;
    if (tid == 0) {
        const uint32_t lbo = mode == 0 ? 2048 : 128, sbo = mode == 0 ? 128 : 2048;
        for (int j = 0; j < 14; ++j) {
            const uint64_t d = desc_none(smem_u32(smem) + j * 2 * 2048, lbo, sbo);
            asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tm + 8 * j), "l"(d) : "memory");
        }
        tc_commit(smem_u32(&bar));
    }
    mbar_wait(smem_u32(&bar), 0);
    tc_fence_after();
    int nb = 0;
    const uint32_t lb = static_cast<uint32_t>((tid >> 5) * 32) << 16;
    for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tm + lb + c0, v);
        tmem_ld_wait();
        for (int k = 0; k < 32; ++k) {
            const int c = c0 + k;
            if (c < 112 && __uint_as_float(v[k]) != static_cast<float>(tid * 1000 + c)) ++nb;
            if (tid == 9 && c < 16) sample[c] = __uint_as_float(v[k]);
        }
    }
    atomicAdd(bad, nb);
    tc_fence_before();
    __syncthreads();
    if (tid < 32) {
        tc_fence_after();
        tmem_dealloc(tm, 128);
    }
}

int main() {
    int *bad;
    float *sample;
    cudaMallocManaged(&bad, sizeof(int));
    cudaMallocManaged(&sample, 16 * sizeof(float));
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 60 * 1024 + 1024);
    for (int mode = 0; mode < 2; ++mode) {
        *bad = 0;
        probe<<<1, 128, 60 * 1024 + 1024>>>(mode, bad, sample);
        cudaError_t e = cudaDeviceSynchronize();
        printf("mode %d (LBO %d, SBO %d): %s, mismatches %d / %d; lane 9 cols 0..15:", mode, mode == 0 ? 2048 : 128,
               mode == 0 ? 128 : 2048, cudaGetErrorString(e), *bad, 128 * 112);
        for (int c = 0; c < 16; ++c) printf(" %.0f", sample[c]);
        printf("\n");
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
