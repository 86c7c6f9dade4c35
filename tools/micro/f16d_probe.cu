// Where does a kind::f16 MMA with an F16 accumulator (instruction descriptor
// D type 0) put D[m][n] in TMEM?  A = B = one stage (MN-major SW128, the Gram
// kernels' layout) with stage[f][k=0] = f + 1, so D[m][n] = (m+1)(n+1); lane 0
// then loads 16 columns and prints the raw words for F16 and F32 accumulators.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_1808_03843_b200/csrc -I ../../include -o f16d_probe f16d_probe.cu
#include <cstdio>
#include "tc_common.cuh"
using namespace cmf;
using namespace cmf::tc;

int cmf::set_error(int code, const char *, ...) { return code; }

__global__ void probe(int f16acc, uint32_t *out) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    __shared__ uint32_t slot;
    __shared__ uint64_t bar;
    for (int i = threadIdx.x; i < STAGE_BYTES / 16; i += blockDim.x) reinterpret_cast<int4 *>(smem)[i] = make_int4(0, 0, 0, 0);
    __syncthreads();
    if (threadIdx.x < 128) {  // feature f = tid: element (f, k = 0)
        const int fe = threadIdx.x;
        const uint32_t a = operand_addr(smem_u32(smem), 0, fe >> 3) + (fe & 7) * 2;
        const __half h = __float2half_rn(static_cast<float>(fe + 1));
        asm volatile("st.shared.b16 [%0], %1;" ::"r"(a), "h"(__half_as_ushort(h)));
    }
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (threadIdx.x < 32) tmem_alloc(smem_u32(&slot), 64);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = slot;
    // fill the 32 columns with a marker first so untouched columns show
    if (threadIdx.x < 128) {
        uint32_t v[16];
        for (int k = 0; k < 16; ++k) v[k] = 0xDEADBEEFu;
        const uint32_t lb = static_cast<uint32_t>((threadIdx.x >> 5) * 32) << 16;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                     ::"r"(tm + lb), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
                     "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
                     "r"(v[15]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        uint32_t idesc = make_idesc(128, 16);
        if (f16acc) idesc &= ~(3u << 4);  // D type F16
        const uint64_t d = make_desc(smem_u32(smem));
        tc_mma(tm, d, d, idesc, 0);
        tc_commit(smem_u32(&bar));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    tc_fence_after();
    if (threadIdx.x < 32) {
        uint32_t v[16];

        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(tm) : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (threadIdx.x < 2)
            for (int k = 0; k < 16; ++k) out[threadIdx.x * 16 + k] = v[k];
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc(tm, 64);
    }
}

int main() {
    uint32_t *d, h[32];
    cudaMalloc(&d, 32 * 4);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
    for (int f16 = 0; f16 < 2; ++f16) {
        probe<<<1, 128, 40 * 1024>>>(f16, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("%s accumulator (%s): lane 0 / lane 1 columns 0..15\n", f16 ? "F16" : "F32", cudaGetErrorString(e));
        for (int l = 0; l < 2; ++l) {
            for (int k = 0; k < 16; ++k) printf(" %08x", h[l * 16 + k]);
            printf("\n");
        }
    }
    return 0;
}
