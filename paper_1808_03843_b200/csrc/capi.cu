// extern "C" boundary (include/cmf_b200.h): argument validation, status codes,
// thread-local error text, and dispatch to the sm_100a kernels.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include "common.cuh"

namespace cmf {

static thread_local char g_err[512] = "";

int set_error(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int gram_simt_launch(const int64_t *, const int32_t *, const float *, const float *, int64_t,
                     const float *, int, double, int, const float *, bool, bool, void *, int64_t,
                     float *, int64_t *, int32_t *, cudaStream_t);
int gram_tc_launch(const int64_t *, const int32_t *, const float *, int64_t, const void *, const void *, int64_t,
                   float, int, int, double, int, const float *, bool, void *, int64_t, float *, int64_t *, int32_t *,
                   cudaStream_t, const int64_t * = nullptr, const int64_t * = nullptr, int = 0, int = 1, int = 0);
int gram_tc_ws_launch(const int64_t *, const int32_t *, const float *, int64_t, const void *, const void *, int64_t,
                      float, int, int, double, int, bool, void *, int64_t, float *, int64_t *, int32_t *, int64_t,
                      void *, int64_t, cudaStream_t);
int64_t gram_tc_passes(int64_t nrows, int64_t nnz, int64_t ncols, int W, bool split);
int factors_to_half_split_launch(const float *, int64_t, int, void *, void *, int, float, int32_t *, cudaStream_t);
int gram_tc_width(int f);
int fused_cg_launch(const int64_t *, const int32_t *, const float *, int64_t, const void *, int64_t, int, int, double,
                    int, float *, float *const *, int, int64_t, int, double, int32_t *, int32_t *, void *, int64_t,
                    const float *, float, bool, const int64_t *, float *, int, cudaStream_t);
int64_t fused_cg_partial_floats(int64_t nrows, int f);
int64_t fused_cg_workspace_bytes(int64_t nrows, int W);
int factors_to_half_launch(const float *, int64_t, int, void *, int, int32_t *, cudaStream_t);
int spmm_bias_launch(const int64_t *, const int32_t *, const float *, int64_t, const float *, int,
                     float *, cudaStream_t);
int cg_launch(const void *, bool, int64_t, const float *, const float *, const double *, double,
              const int64_t *, int64_t, int, int, bool, float *, int32_t *, int32_t *, int32_t *,
              cudaStream_t);
int chol_launch(const float *, int64_t, const float *, const int64_t *, int64_t, int, bool, float *,
                int32_t *, int32_t *, cudaStream_t);
int sq_error_launch(const void *, const void *, bool, const float *, int64_t, const float *,
                    const float *, int, double *, cudaStream_t);
int sq_error_csr_launch(const int64_t *, const int32_t *, const float *, int64_t, const float *,
                        const float *, int, double *, cudaStream_t);
int wsqnorm_launch(const int64_t *, const float *, int64_t, int, double *, cudaStream_t);
int predict_launch(const void *, const void *, bool, int64_t, const float *, const float *, int,
                   float *, cudaStream_t);
int pack_half_launch(const float *, void *, int64_t, int32_t *, cudaStream_t);
int build_launch(const void *, const void *, bool, const float *, int64_t, int64_t *, int64_t *, int32_t *, float *,
                 int64_t *, int32_t *, float *, void *, int64_t, int64_t *, int64_t *, cudaStream_t);
int64_t build_workspace_bytes(int64_t k);
int fused_base_ld(int f);
int gen_truth_launch(uint64_t, int, int64_t, int, float *, cudaStream_t);
int gen_count_launch(uint64_t, int64_t, int64_t, uint64_t, uint64_t, int, int64_t, int64_t, int64_t, int64_t,
                     int64_t *, int64_t *, int64_t *, cudaStream_t);
int gen_fill_launch(uint64_t, int64_t, int64_t, int, uint64_t, uint64_t, float, int, int64_t, int64_t, int64_t,
                    int64_t, const float *, const float *, const int64_t *, int32_t *, float *, const int64_t *,
                    int64_t *, int64_t *, float *, cudaStream_t);
int64_t group_workspace_bytes(int64_t k);
int group_launch(const void *, const void *, bool, int64_t, int64_t, int64_t *, int32_t *, void *, int64_t,
                 cudaStream_t);
int64_t dense_gram_workspace_bytes(int64_t rows, int f, bool fp64);
int dense_gram_launch(const float *, int64_t, int, bool, void *, void *, int64_t, cudaStream_t);
int implicit_loss_launch(const int64_t *, const int32_t *, const float *, int64_t, const float *, const float *, int,
                         double, double *, cudaStream_t);
int mpr_launch(const int64_t *, const int32_t *, int64_t, const float *, const float *, int64_t, int,
               unsigned long long *, cudaStream_t);

int gram_tc_trace(void *buf);
int fused_cg_trace(void *buf);
}  // namespace cmf

using namespace cmf;

#define REQUIRE(cond, ...)                                  \
    do {                                                    \
        if (!(cond)) return set_error(CMF_EINVAL, __VA_ARGS__); \
    } while (0)

static inline cudaStream_t S(void *s) { return static_cast<cudaStream_t>(s); }

extern "C" {

const char *cmf_last_error(void) { return g_err; }

int cmf_version(void) { return 1; }

int cmf_device_info(int *sm_count, int *cc_major, int *cc_minor) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess && sm_count) e = cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess && cc_major) e = cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev);
    if (e == cudaSuccess && cc_minor) e = cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (e != cudaSuccess) return set_error(CMF_ECUDA, "device query: %s", cudaGetErrorString(e));
    return CMF_OK;
}

static int gram_dispatch(const int64_t *indptr, const int32_t *indices, const float *a_w,
                         const float *b_w, int64_t nrows, const float *fixed, int32_t f, double lam,
                         int32_t weighted, const float *base, int32_t precision, int32_t kernel,
                         void *a_out, int64_t a_stride, float *b_out, int64_t *nu_out,
                         int32_t *ovf, cudaStream_t st) {
    const bool half = precision == CMF_PREC_FP16;
    if (kernel == CMF_GRAM_TC)
        return set_error(CMF_EINVAL, "use cmf_gram_assemble_tc for the tensor-core kernel");
    return gram_simt_launch(indptr, indices, a_w, b_w, nrows, fixed, f, lam, weighted, base, half,
                            kernel == CMF_GRAM_BITWISE, a_out, a_stride, b_out, nu_out, ovf, st);
}

int cmf_gram_assemble(const int64_t *indptr, const int32_t *indices, const float *a_weights,
                      const float *b_weights, int64_t nrows, const float *fixed, int64_t ncols,
                      int32_t f, double lam, int32_t weighted_reg, const float *base_packed,
                      int32_t precision, int32_t kernel, void *a_out, int64_t a_stride,
                      float *b_out, int64_t *nu_out, int32_t *overflow_flag, void *stream) {
    REQUIRE(nrows >= 0 && ncols >= 0, "negative dimensions");
    REQUIRE(f >= 1, "f must be >= 1");
    REQUIRE(precision == CMF_PREC_FP32 || precision == CMF_PREC_FP16, "unknown precision %d", precision);
    REQUIRE(kernel >= CMF_GRAM_BITWISE && kernel <= CMF_GRAM_TC, "unknown gram kernel %d", kernel);
    REQUIRE(a_stride >= f * (int64_t)(f + 1) / 2, "a_stride smaller than f*(f+1)/2");
    if (nrows == 0) return CMF_OK;
    REQUIRE(indptr && a_out, "null indptr / a_out");
    REQUIRE(fixed || ncols == 0, "null fixed factors");
    REQUIRE(!b_weights || b_out, "b_weights given without b_out");
    return gram_dispatch(indptr, indices, a_weights, b_weights, nrows, fixed, f, lam, weighted_reg,
                         base_packed, precision, kernel, a_out, a_stride, b_out, nu_out, overflow_flag,
                         S(stream));
}

int cmf_tc_width(int32_t f) { return gram_tc_width(f); }

int cmf_ipc_export(const void *ptr, void *handle64, int64_t *offset) {
    REQUIRE(ptr && handle64 && offset, "null argument");
    // cudaIpcGetMemHandle wants the allocation's base; the range comes from the
    // driver (fetched through the runtime, no libcuda link dependency)
    typedef int (*GetRange)(unsigned long long *, size_t *, unsigned long long);
    static GetRange range = nullptr;
    if (!range) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return set_error(CMF_ECUDA, "cuMemGetAddressRange unavailable");
        range = reinterpret_cast<GetRange>(fn);
    }
    unsigned long long base = 0;
    size_t size = 0;
    if (range(&base, &size, reinterpret_cast<unsigned long long>(ptr)) != 0)
        return set_error(CMF_EINVAL, "not a device allocation");
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base));
    if (e != cudaSuccess) return set_error(CMF_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    static_assert(sizeof(h) == 64, "IPC handle size");
    memcpy(handle64, &h, sizeof(h));
    *offset = static_cast<int64_t>(reinterpret_cast<unsigned long long>(ptr) - base);
    return CMF_OK;
}

int cmf_ipc_open(const void *handle64, int64_t offset, void **ptr_out) {
    REQUIRE(handle64 && ptr_out && offset >= 0, "bad argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof(h));
    void *base = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return set_error(CMF_ECUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    *ptr_out = static_cast<char *>(base) + offset;
    return CMF_OK;
}

int cmf_ipc_close(void *ptr, int64_t offset) {
    REQUIRE(ptr && offset >= 0, "bad argument");
    const cudaError_t e = cudaIpcCloseMemHandle(static_cast<char *>(ptr) - offset);
    if (e != cudaSuccess) return set_error(CMF_ECUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
    return CMF_OK;
}

int cmf_debug_trace(void *buf) {
    int rc = gram_tc_trace(buf);
    return rc ? rc : fused_cg_trace(buf);
}

int cmf_factors_to_half(const float *x, int64_t rows, int32_t f, void *out16, int32_t w16,
                        int32_t *overflow_flag, void *stream) {
    REQUIRE(rows >= 0 && f >= 1 && w16 >= f, "bad dimensions");
    if (rows == 0) return CMF_OK;
    REQUIRE(x && out16, "null argument");
    return factors_to_half_launch(x, rows, f, out16, w16, overflow_flag, S(stream));
}

int cmf_factors_to_half_split(const float *x, int64_t rows, int32_t f, void *hi16, void *lo16, int32_t w16,
                              float scale, int32_t *overflow_flag, void *stream) {
    REQUIRE(rows >= 0 && f >= 1 && w16 >= f && scale > 0.0f, "bad arguments");
    if (rows == 0) return CMF_OK;
    REQUIRE(x && hi16 && lo16, "null argument");
    return factors_to_half_split_launch(x, rows, f, hi16, lo16, w16, scale, overflow_flag, S(stream));
}

int cmf_gram_assemble_tc(const int64_t *indptr, const int32_t *indices, const float *b_weights,
                         int64_t nrows, const void *fixed16, const void *fixed16_lo, int64_t ncols,
                         float split_scale,
                         int32_t w16, int32_t f, double lam, int32_t weighted_reg, const float *base_packed,
                         int32_t precision, void *a_out, int64_t a_stride, float *b_out, int64_t *nu_out,
                         int32_t *overflow_flag, void *stream) {
    REQUIRE(nrows >= 0 && f >= 1, "bad dimensions");
    REQUIRE(precision == CMF_PREC_FP32 || precision == CMF_PREC_FP16, "unknown precision %d", precision);
    REQUIRE(a_stride >= f * (int64_t)(f + 1) / 2, "a_stride smaller than f*(f+1)/2");
    if (nrows == 0) return CMF_OK;
    REQUIRE(indptr && a_out && fixed16, "null argument");
    REQUIRE(!fixed16_lo || split_scale > 0.0f, "split_scale must be > 0");
    REQUIRE(ncols >= 1, "ncols must be >= 1");
    return gram_tc_launch(indptr, indices, b_weights, nrows, fixed16, fixed16_lo, ncols, split_scale, w16, f, lam,
                          weighted_reg, base_packed, precision == CMF_PREC_FP16, a_out, a_stride, b_out, nu_out,
                          overflow_flag, S(stream));
}

int cmf_gram_assemble_tc_ws(const int64_t *indptr, const int32_t *indices, const float *b_weights,
                            int64_t nrows, int64_t nnz, const void *fixed16, const void *fixed16_lo, int64_t ncols,
                            float split_scale, int32_t w16, int32_t f, double lam, int32_t weighted_reg,
                            int32_t precision, void *a_out, int64_t a_stride, float *b_out, int64_t *nu_out,
                            int32_t *overflow_flag, void *ws, int64_t ws_bytes, void *stream) {
    REQUIRE(nrows >= 0 && f >= 1 && nnz >= 0, "bad dimensions");
    REQUIRE(precision == CMF_PREC_FP32 || precision == CMF_PREC_FP16, "unknown precision %d", precision);
    REQUIRE(a_stride >= f * (int64_t)(f + 1) / 2, "a_stride smaller than f*(f+1)/2");
    if (nrows == 0) return CMF_OK;
    REQUIRE(indptr && a_out && fixed16, "null argument");
    REQUIRE(!fixed16_lo || split_scale > 0.0f, "split_scale must be > 0");
    REQUIRE(ncols >= 1, "ncols must be >= 1");
    REQUIRE(ws_bytes >= 0, "negative workspace size");
    return gram_tc_ws_launch(indptr, indices, b_weights, nrows, fixed16, fixed16_lo, ncols, split_scale, w16, f, lam,
                             weighted_reg, precision == CMF_PREC_FP16, a_out, a_stride, b_out, nu_out, overflow_flag,
                             nnz, ws, ws_bytes, S(stream));
}

int64_t cmf_gram_tc_workspace_bytes(int64_t nrows, int64_t nnz, int64_t ncols, int32_t f, int32_t split) {
    if (nrows <= 0) return 0;
    return (gram_tc_passes(nrows, nnz, ncols, gram_tc_width(f), split != 0) - 1) * nrows * 8;
}

int cmf_fused_cg_update(const int64_t *indptr, const int32_t *indices, const float *values,
                        int64_t nrows, int64_t nnz, const void *fixed16, int64_t ncols, int32_t w16, int32_t f, double lam,
                        int32_t weighted_reg, float *target, int32_t f_s, double cg_tol,
                        int32_t *breakdowns, int32_t *overflow_flag, void *stream) {
    REQUIRE(nrows >= 0 && f >= 1, "bad dimensions");
    REQUIRE(f_s >= 1, "cg_iters must be >= 1");
    REQUIRE(cg_tol >= 0.0, "cg_tol must be >= 0");
    if (nrows == 0) return CMF_OK;
    REQUIRE(indptr && fixed16 && target, "null argument");
    REQUIRE(ncols >= 1, "ncols must be >= 1");
    return fused_cg_launch(indptr, indices, values, nrows, fixed16, ncols, w16, f, lam, weighted_reg, target, nullptr,
                           0, nnz, f_s, cg_tol, breakdowns, overflow_flag, nullptr, 0, nullptr, 0.0f, false,
                           nullptr, nullptr, 0, S(stream));
}

int cmf_fused_cg_update_peers(const int64_t *indptr, const int32_t *indices, const float *values,
                              int64_t nrows, int64_t nnz, const void *fixed16, int64_t ncols, int32_t w16,
                              int32_t f, double lam, int32_t weighted_reg, float *target,
                              float *const *peer_targets, int32_t npeers, int32_t f_s, double cg_tol,
                              int32_t *breakdowns, int32_t *overflow_flag, void *stream) {
    REQUIRE(nrows >= 0 && f >= 1, "bad dimensions");
    REQUIRE(f_s >= 1, "cg_iters must be >= 1");
    REQUIRE(cg_tol >= 0.0, "cg_tol must be >= 0");
    REQUIRE(npeers >= 0 && npeers <= 64, "npeers must be in [0, 64]");
    if (nrows == 0) return CMF_OK;
    REQUIRE(indptr && fixed16 && target, "null argument");
    REQUIRE(npeers == 0 || peer_targets, "null peer list");
    REQUIRE(ncols >= 1, "ncols must be >= 1");
    return fused_cg_launch(indptr, indices, values, nrows, fixed16, ncols, w16, f, lam, weighted_reg, target,
                           peer_targets, npeers, nnz, f_s, cg_tol, breakdowns, overflow_flag, nullptr, 0, nullptr, 0.0f,
                           false, nullptr, nullptr, 0, S(stream));
}

int cmf_fused_cg_update_ws(const int64_t *indptr, const int32_t *indices, const float *values,
                           int64_t nrows, int64_t nnz, const void *fixed16, int64_t ncols, int32_t w16,
                           int32_t f, double lam, int32_t weighted_reg, float *target,
                           float *const *peer_targets, int32_t npeers, int32_t f_s, double cg_tol,
                           int32_t *breakdowns, int32_t *overflow_flag, void *workspace,
                           int64_t workspace_bytes, void *stream) {
    REQUIRE(nrows >= 0 && f >= 1, "bad dimensions");
    REQUIRE(f_s >= 1, "cg_iters must be >= 1");
    REQUIRE(cg_tol >= 0.0, "cg_tol must be >= 0");
    REQUIRE(npeers >= 0 && npeers <= 64, "npeers must be in [0, 64]");
    REQUIRE(workspace_bytes >= 0, "negative workspace size");
    if (nrows == 0) return CMF_OK;
    REQUIRE(indptr && fixed16 && target, "null argument");
    REQUIRE(npeers == 0 || peer_targets, "null peer list");
    REQUIRE(ncols >= 1, "ncols must be >= 1");
    REQUIRE((reinterpret_cast<uintptr_t>(workspace) & 255) == 0, "workspace must be 256-byte aligned");
    return fused_cg_launch(indptr, indices, values, nrows, fixed16, ncols, w16, f, lam, weighted_reg, target,
                           peer_targets, npeers, nnz, f_s, cg_tol, breakdowns, overflow_flag, workspace,
                           workspace_bytes, nullptr, 0.0f, false, nullptr, nullptr, 0, S(stream));
}

int cmf_fused_cg_update_implicit(const int64_t *indptr, const int32_t *indices, const float *values,
                                 int64_t nrows, int64_t nnz, const void *fixed16, int64_t ncols, int32_t w16,
                                 int32_t f, double alpha, double lam, const float *gram_full, float *target,
                                 float *const *peer_targets, int32_t npeers, int32_t f_s, double cg_tol,
                                 int32_t *breakdowns, int32_t *overflow_flag, void *workspace,
                                 int64_t workspace_bytes, void *stream) {
    REQUIRE(nrows >= 0 && f >= 1, "bad dimensions");
    REQUIRE(f_s >= 1, "cg_iters must be >= 1");
    REQUIRE(cg_tol >= 0.0, "cg_tol must be >= 0");
    REQUIRE(alpha > 0.0, "alpha must be > 0");
    REQUIRE(npeers >= 0 && npeers <= 64, "npeers must be in [0, 64]");
    REQUIRE(workspace_bytes >= 0, "negative workspace size");
    if (nrows == 0) return CMF_OK;
    REQUIRE(indptr && fixed16 && target && values, "null argument");
    REQUIRE(npeers == 0 || peer_targets, "null peer list");
    REQUIRE(ncols >= 1, "ncols must be >= 1");
    REQUIRE((reinterpret_cast<uintptr_t>(workspace) & 255) == 0, "workspace must be 256-byte aligned");
    return fused_cg_launch(indptr, indices, values, nrows, fixed16, ncols, w16, f, lam, 0, target, peer_targets,
                           npeers, nnz, f_s, cg_tol, breakdowns, overflow_flag, workspace, workspace_bytes, gram_full,
                           static_cast<float>(alpha), true, nullptr, nullptr, 0, S(stream));
}

int cmf_fused_cg_pass(const int64_t *indptr, const int32_t *indices, const float *values, int64_t nrows,
                      int64_t nnz, const void *fixed16, int64_t ncols, int32_t w16, int32_t f, double lam,
                      int32_t weighted_reg, float *target, float *const *peer_targets, int32_t npeers,
                      const int64_t *seg, float *partial, int32_t pass, int32_t f_s, double cg_tol,
                      int32_t *breakdowns, int32_t *overflow_flag, void *stream) {
    REQUIRE(nrows >= 0 && f >= 1, "bad dimensions");
    REQUIRE(pass == 1 || pass == 2, "pass must be 1 or 2");
    REQUIRE(f_s >= 1, "cg_iters must be >= 1");
    REQUIRE(cg_tol >= 0.0, "cg_tol must be >= 0");
    REQUIRE(npeers >= 0 && npeers <= 64, "npeers must be in [0, 64]");
    if (nrows == 0) return CMF_OK;
    REQUIRE(indptr && fixed16 && target && seg && partial, "null argument");
    REQUIRE(npeers == 0 || peer_targets, "null peer list");
    REQUIRE(ncols >= 1, "ncols must be >= 1");
    return fused_cg_launch(indptr, indices, values, nrows, fixed16, ncols, w16, f, lam, weighted_reg, target,
                           peer_targets, npeers, nnz, f_s, cg_tol, breakdowns, overflow_flag, nullptr, 0, nullptr,
                           0.0f, false, seg, partial, pass, S(stream));
}

int64_t cmf_fused_cg_partial_floats(int64_t nrows, int32_t f) {
    return (nrows < 0 || f < 1) ? -1 : fused_cg_partial_floats(nrows, f);
}

int32_t cmf_fused_base_ld(int32_t f) { return f < 1 ? -1 : fused_base_ld(f); }

int64_t cmf_fused_cg_workspace_bytes(int64_t nrows, int32_t f) {
    if (nrows < 0 || f < 1) return 0;
    return fused_cg_workspace_bytes(nrows, gram_tc_width(f));
}

int cmf_spmm_bias(const int64_t *indptr, const int32_t *indices, const float *b_weights,
                  int64_t nrows, const float *fixed, int64_t ncols, int32_t f, float *b_out,
                  void *stream) {
    REQUIRE(nrows >= 0 && ncols >= 0 && f >= 1, "bad dimensions");
    if (nrows == 0) return CMF_OK;
    REQUIRE(indptr && b_out, "null argument");
    return spmm_bias_launch(indptr, indices, b_weights, nrows, fixed, f, b_out, S(stream));
}

int cmf_batch_cg(const void *a, int32_t a_precision, int64_t a_stride, const float *b,
                 const float *x0, const double *eps, double cg_tol, const int64_t *nu,
                 int64_t nsys, int32_t f, int32_t f_s, int32_t accum, float *x_out,
                 int32_t *iters, int32_t *broke, int32_t *breakdowns, void *stream) {
    REQUIRE(nsys >= 0 && f >= 1, "bad dimensions");
    REQUIRE(f_s >= 1, "cg_iters must be >= 1");
    REQUIRE(cg_tol >= 0.0, "cg_tol must be >= 0");
    REQUIRE(a_precision == CMF_PREC_FP32 || a_precision == CMF_PREC_FP16, "unknown precision");
    REQUIRE(accum == CMF_CG_FP32 || accum == CMF_CG_FP64, "unknown accumulation mode");
    REQUIRE(a_stride == 0 || a_stride >= f * (int64_t)(f + 1) / 2,
            "a_stride must be 0 (one shared matrix) or >= f*(f+1)/2");
    if (nsys == 0) return CMF_OK;
    REQUIRE(a && b && x0 && x_out, "null argument");
    return cg_launch(a, a_precision == CMF_PREC_FP16, a_stride, b, x0, eps, cg_tol, nu, nsys, f, f_s,
                     accum == CMF_CG_FP64, x_out, iters, broke, breakdowns, S(stream));
}

int cmf_batch_cholesky(const float *a, int64_t a_stride, const float *b, const int64_t *nu,
                       int64_t nsys, int32_t f, int32_t accum, float *x_out, int32_t *info,
                       int32_t *nbad, void *stream) {
    REQUIRE(nsys >= 0 && f >= 1, "bad dimensions");
    REQUIRE(accum == CMF_CG_FP32 || accum == CMF_CG_FP64, "unknown accumulation mode");
    REQUIRE(a_stride >= f * (int64_t)(f + 1) / 2, "a_stride smaller than f*(f+1)/2");
    if (nsys == 0) return CMF_OK;
    REQUIRE(a && b && x_out, "null argument");
    return chol_launch(a, a_stride, b, nu, nsys, f, accum == CMF_CG_FP64, x_out, info, nbad, S(stream));
}

int cmf_half_update(const int64_t *indptr, const int32_t *indices, const float *values,
                    int64_t nrows, const float *fixed, int64_t ncols, float *target, int32_t f,
                    double lam, int32_t weighted_reg, int32_t method, int32_t precision,
                    int32_t kernel, int32_t f_s, double cg_tol, int32_t accum, void *ws_a,
                    int64_t a_stride, float *ws_b, int64_t *ws_nu, int64_t ws_rows, void *ws16,
                    int32_t *flags, void *stream) {
    REQUIRE(nrows >= 0 && ncols >= 0 && f >= 1, "bad dimensions");
    REQUIRE(method == 0 || method == 1, "unknown method %d", method);
    REQUIRE(!(method == 1 && precision == CMF_PREC_FP16),
            "half-precision Gram storage requires the cg solver");
    REQUIRE(ws_rows >= 1 || nrows == 0, "empty workspace");
    REQUIRE(flags, "null flags");
    if (nrows == 0) return CMF_OK;
    cudaStream_t st = S(stream);
    const int w16 = gram_tc_width(f);
    if (kernel == CMF_GRAM_TC) {
        REQUIRE(ws16, "CMF_GRAM_TC needs the ws16 shadow buffer");
        int rc = factors_to_half_launch(fixed, ncols, f, ws16, w16, flags + 0, st);
        if (rc) return rc;
    }
    for (int64_t r0 = 0; r0 < nrows; r0 += ws_rows) {
        const int64_t nb = nrows - r0 < ws_rows ? nrows - r0 : ws_rows;
        int rc = kernel == CMF_GRAM_TC
                     ? cmf_gram_assemble_tc(indptr + r0, indices, values, nb, ws16, nullptr, ncols, 1.0f, w16, f, lam,
                                            weighted_reg, nullptr, precision, ws_a, a_stride, ws_b,
                                            ws_nu, flags + 0, stream)
                     : cmf_gram_assemble(indptr + r0, indices, nullptr, values, nb, fixed, ncols, f,
                                         lam, weighted_reg, nullptr, precision, kernel, ws_a,
                                         a_stride, ws_b, ws_nu, flags + 0, stream);
        if (rc) return rc;
        float *tgt = target + r0 * f;
        if (method == 0)
            rc = cg_launch(ws_a, precision == CMF_PREC_FP16, a_stride, ws_b, tgt, nullptr, cg_tol, ws_nu,
                           nb, f, f_s, accum == CMF_CG_FP64, tgt, nullptr, nullptr, flags + 1, st);
        else
            rc = chol_launch(static_cast<const float *>(ws_a), a_stride, ws_b, ws_nu, nb, f,
                             accum == CMF_CG_FP64, tgt, nullptr, flags + 2, st);
        if (rc) return rc;
    }
    return CMF_OK;
}

int cmf_pack_half(const float *in, void *out, int64_t n, int32_t *overflow_flag, void *stream) {
    REQUIRE(n >= 0, "negative size");
    if (n == 0) return CMF_OK;
    REQUIRE(in && out, "null argument");
    return pack_half_launch(in, out, n, overflow_flag, S(stream));
}

int cmf_sq_error(const void *users, const void *items, int32_t idx64, const float *ratings,
                 int64_t count, const float *x, const float *theta, int32_t f, double *out,
                 void *stream) {
    REQUIRE(count >= 0 && f >= 1 && out, "bad arguments");
    return sq_error_launch(users, items, idx64 != 0, ratings, count, x, theta, f, out, S(stream));
}

int cmf_sq_error_csr(const int64_t *indptr, const int32_t *indices, const float *values,
                     int64_t nrows, const float *x, const float *theta, int32_t f, double *out,
                     void *stream) {
    REQUIRE(nrows >= 0 && f >= 1 && out, "bad arguments");
    return sq_error_csr_launch(indptr, indices, values, nrows, x, theta, f, out, S(stream));
}

int cmf_weighted_sqnorm(const int64_t *indptr, const float *x, int64_t nrows, int32_t f,
                        double *out, void *stream) {
    REQUIRE(nrows >= 0 && f >= 1 && out, "bad arguments");
    return wsqnorm_launch(indptr, x, nrows, f, out, S(stream));
}

int cmf_predict_pairs(const void *users, const void *items, int32_t idx64, int64_t count,
                      const float *x, const float *theta, int32_t f, float *pred, void *stream) {
    REQUIRE(count >= 0 && f >= 1, "bad arguments");
    return predict_launch(users, items, idx64 != 0, count, x, theta, f, pred, S(stream));
}

int cmf_build(const void *user, const void *item, int32_t idx64, const float *rating, int64_t k, int64_t *mn,
              int64_t *row_ptr, int32_t *col_idx, float *csr_val, int64_t *col_ptr, int32_t *row_idx, float *csc_val,
              void *ws, int64_t ws_bytes, int64_t *nnz_host, int64_t *bad_host, void *stream) {
    REQUIRE(k >= 0 && mn != nullptr && nnz_host != nullptr && bad_host != nullptr, "bad build arguments");
    REQUIRE(k == 0 || (user && item && rating), "null triple arrays");
    return build_launch(user, item, idx64 != 0, rating, k, mn, row_ptr, col_idx, csr_val, col_ptr, row_idx, csc_val,
                        ws, ws_bytes, nnz_host, bad_host, S(stream));
}

int64_t cmf_build_workspace_bytes(int64_t k) { return k < 0 ? -1 : build_workspace_bytes(k); }

int cmf_gen_truth(uint64_t seed, int32_t which, int64_t rows, int32_t f, float *out, void *stream) {
    REQUIRE(rows >= 0 && f >= 1 && (which == 0 || which == 1) && (rows == 0 || out), "bad gen_truth arguments");
    REQUIRE(rows < (int64_t(1) << 32), "gen: 32-bit row ids");
    return gen_truth_launch(seed, which, rows, f, out, S(stream));
}

int cmf_gen_count(uint64_t seed, int64_t m, int64_t n, uint64_t thr_cell, uint64_t thr_test, int32_t by_user,
                  int64_t lo, int64_t hi, int64_t minor_lo, int64_t minor_hi, int64_t *ptr, int64_t *tptr,
                  int64_t *scratch, void *stream) {
    REQUIRE(m >= 0 && n >= 0 && m < (int64_t(1) << 32) && n < (int64_t(1) << 31), "gen: bad extents");
    REQUIRE(lo >= 0 && hi >= lo && hi <= (by_user ? m : n), "gen: bad major range");
    REQUIRE(minor_lo >= 0 && minor_hi >= minor_lo && minor_hi <= (by_user ? n : m), "gen: bad minor range");
    REQUIRE(ptr && (hi == lo || scratch), "null argument");
    return gen_count_launch(seed, m, n, thr_cell, thr_test, by_user, lo, hi, minor_lo, minor_hi, ptr, tptr, scratch,
                            S(stream));
}

int cmf_gen_fill(uint64_t seed, int64_t m, int64_t n, int32_t f, uint64_t thr_cell, uint64_t thr_test,
                 float noise_scale, int32_t by_user, int64_t lo, int64_t hi, int64_t minor_lo, int64_t minor_hi,
                 const float *X, const float *T, const int64_t *ptr, int32_t *minor_out, float *val_out,
                 const int64_t *tptr, int64_t *test_u, int64_t *test_v, float *test_r, void *stream) {
    REQUIRE(m >= 0 && n >= 0 && m < (int64_t(1) << 32) && n < (int64_t(1) << 31) && f >= 1, "gen: bad extents");
    REQUIRE(lo >= 0 && hi >= lo && hi <= (by_user ? m : n), "gen: bad major range");
    REQUIRE(minor_lo >= 0 && minor_hi >= minor_lo && minor_hi <= (by_user ? n : m), "gen: bad minor range");
    REQUIRE(X && T && ptr, "null argument");
    REQUIRE(!tptr || (by_user && test_u && test_v && test_r), "test triples come from the user pass");
    return gen_fill_launch(seed, m, n, f, thr_cell, thr_test, noise_scale, by_user, lo, hi, minor_lo, minor_hi, X, T,
                           ptr, minor_out, val_out, tptr, test_u, test_v, test_r, S(stream));
}

int64_t cmf_group_workspace_bytes(int64_t k) { return k < 0 ? -1 : group_workspace_bytes(k); }

int cmf_group_rows(const void *rows, const void *cols, int32_t idx64, int64_t k, int64_t nrows, int64_t *indptr,
                   int32_t *cols_out, void *ws, int64_t ws_bytes, void *stream) {
    REQUIRE(k >= 0 && nrows >= 0 && indptr && (k == 0 || (rows && cols && cols_out && ws)), "bad group arguments");
    REQUIRE(nrows < (int64_t(1) << 32) && k < (int64_t(1) << 32), "group: 32-bit row ids and counts");
    return group_launch(rows, cols, idx64 != 0, k, nrows, indptr, cols_out, ws, ws_bytes, S(stream));
}

int64_t cmf_dense_gram_workspace_bytes(int64_t rows, int32_t f, int32_t fp64) {
    return (rows < 0 || f < 1) ? -1 : dense_gram_workspace_bytes(rows, f, fp64 != 0);
}

int cmf_dense_gram(const float *F, int64_t rows, int32_t f, int32_t fp64, void *out_packed, void *ws,
                   int64_t ws_bytes, void *stream) {
    REQUIRE(rows >= 0 && f >= 1 && F && out_packed && ws, "bad dense_gram arguments");
    return dense_gram_launch(F, rows, f, fp64 != 0, out_packed, ws, ws_bytes, S(stream));
}

int cmf_implicit_loss_csr(const int64_t *indptr, const int32_t *indices, const float *values, int64_t nrows,
                          const float *x, const float *theta, int32_t f, double alpha, double *out, void *stream) {
    REQUIRE(nrows >= 0 && f >= 1 && out, "bad arguments");
    return implicit_loss_launch(indptr, indices, values, nrows, x, theta, f, alpha, out, S(stream));
}

int cmf_mpr_count(const int64_t *pos_ptr, const int32_t *pos_item, int64_t m, const float *x, const float *theta,
                  int64_t n, int32_t f, uint64_t *out, void *stream) {
    REQUIRE(m >= 0 && n >= 1 && f >= 1 && pos_ptr && out && x && theta, "bad mpr arguments");
    return mpr_launch(pos_ptr, pos_item, m, x, theta, n, f, reinterpret_cast<unsigned long long *>(out), S(stream));
}

}  // extern "C"
