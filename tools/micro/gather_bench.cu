// Microbenchmark: random-row gather bandwidth on B200 for W-half rows
// (208 B at f=100) from a table of R rows, into shared memory.
//   mode 0: cp.async 16 B, lanes over chunks (2 rows / warp instruction)
//   mode 1: ld.global.nc.v4 into registers (same mapping), accumulate (no smem)
//   mode 2: cp.async 16 B, lane per row (13 instructions per row, L1-cached .ca)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gb gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void k_cpasync(const uint4 *tab, int W16, const int *idx, long n, uint4 *sink, int nwarps_per_cta) {
    extern __shared__ uint4 sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c = lane & 15, hrow = lane >> 4;
    uint4 *mys = sm + (warp & 7) * 64 * 16;  // 64 rows x 16 chunks (shared by warps w, w+8: bandwidth only)
    long w = (long)blockIdx.x * nwarps_per_cta + warp, nw = (long)gridDim.x * nwarps_per_cta;
    for (long base = w * 64; base < n; base += nw * 64) {
        int myidx = idx[base + lane], myidx2 = idx[base + 32 + lane];
#pragma unroll
        for (int t = 0; t < 32; ++t) {
            int ix = __shfl_sync(0xffffffffu, t < 16 ? myidx : myidx2, (2 * t + hrow) & 31);
            if (c < W16) {
                unsigned dst = (unsigned)__cvta_generic_to_shared(mys + (2 * t + hrow) * 16 + c);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(tab + (long)ix * W16 + c));
            }
        }
        asm volatile("cp.async.commit_group;");
        asm volatile("cp.async.wait_group 4;");
    }
    asm volatile("cp.async.wait_group 0;");
    if (threadIdx.x == 0 && sm[0].x == 12345) sink[0] = sm[1];
}

__global__ void k_ldg(const uint4 *tab, int W16, const int *idx, long n, uint4 *sink, int nwarps_per_cta) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c = lane & 15, hrow = lane >> 4;
    long w = (long)blockIdx.x * nwarps_per_cta + warp, nw = (long)gridDim.x * nwarps_per_cta;
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (long base = w * 64; base < n; base += nw * 64) {
        int myidx = idx[base + lane], myidx2 = idx[base + 32 + lane];
#pragma unroll
        for (int t = 0; t < 32; ++t) {
            int ix = __shfl_sync(0xffffffffu, t < 16 ? myidx : myidx2, (2 * t + hrow) & 31);
            if (c < W16) {
                uint4 v = __ldg(tab + (long)ix * W16 + c);
                acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
            }
        }
    }
    if (acc.x == 0x12345678) sink[0] = acc;
}

int main(int argc, char **argv) {
    long R = argc > 1 ? atol(argv[1]) : 17770;
    int W = 104, W16 = W / 8;
    long n = 99000000;  // gathered rows
    size_t tab_bytes = (size_t)R * W * 2;
    uint4 *tab, *sink;
    int *idx;
    cudaMalloc(&tab, tab_bytes);
    cudaMemset(tab, 1, tab_bytes);
    cudaMalloc(&idx, n * 4 + 256);
    cudaMalloc(&sink, 64);
    std::vector<int> h(n);
    uint64_t s = 88172645463325252ull;
    for (long i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (int)(s % R); }
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    int sms = 148;
    for (int mode = 0; mode < 2; ++mode)
        for (int wpc : {4, 8, 12, 16, 24, 32}) {
            size_t smem = (size_t)(wpc < 8 ? wpc : 8) * 64 * 16 * 16;
            if (mode == 0 && smem > 220 * 1024) continue;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(e0);
                if (mode == 0) {
                    cudaFuncSetAttribute(k_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    k_cpasync<<<sms, wpc * 32, smem>>>(tab, W16, idx, n, sink, wpc);
                } else {
                    k_ldg<<<sms, wpc * 32>>>(tab, W16, idx, n, sink, wpc);
                }
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep == 2)
                    printf("R=%ld mode=%s warps/cta=%d: %.3f ms, %.2f TB/s gathered (%.1f B/clk/SM @1.9GHz) err=%s\n", R,
                           mode == 0 ? "cp.async" : "ldg.v4", wpc, ms, n * 208.0 / ms / 1e9,
                           n * 208.0 / (ms * 1e-3) / 148 / 1.9e9, cudaGetErrorString(cudaGetLastError()));
            }
        }
    return 0;
}
