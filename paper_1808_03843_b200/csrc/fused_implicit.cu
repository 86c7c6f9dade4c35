// Implicit-feedback instances of the fused half-update (WEIGHTED operands,
// fused_cg.cuh): A_u = F^T F + sum_k alpha r_k theta_k theta_k^T + lam I,
// b_u = sum_k (1 + alpha r_k) theta_k (implicit.py:57-84), Gram on tcgen05
// (gathered rows x weighted copy), CG from TMEM.  A separate translation unit
// so the 32 extra kernel instances compile in parallel with fused_cg.cu.
#include "fused_cg.cuh"

namespace cmf {

int fused_base_ld(int f) {
    const int fc = fused_fc(f);
    return fc < 0 ? -1 : 4 * fc;
}

int fused_dispatch_implicit(tc::FusedArgs g, int f, bool long_rows, cudaStream_t st) {
    return fused_dispatch_t<true>(g, f, long_rows, st);
}

}  // namespace cmf
