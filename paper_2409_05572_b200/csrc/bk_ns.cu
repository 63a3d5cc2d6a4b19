// Newton-Schulz step coefficients for re-orthonormalising a nearly orthonormal
// block W (G = W^T W = I + E):  W (3I - G)/2 has W^T W = I - (3/4)E^2 + O(E^3).
// Used where the reference's CGS2 second pass only polishes orthogonality
// (kernel.cpp:71-86, pass 2): after the drop-deciding Cholesky pass, and for
// the eigenvector block of K5.  One elementwise kernel; the products are K2/K3.
#include "bk_common.cuh"

namespace bk {
namespace {
__global__ void ns_coeff_kernel(int a, const double* __restrict__ g, int ldg, double* __restrict__ m, int ldm) {
    const int total = a * a;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        const int i = e / a, j = e - i * a;
        const double gij = 0.5 * (g[static_cast<size_t>(i) * ldg + j] + g[static_cast<size_t>(j) * ldg + i]);
        m[static_cast<size_t>(i) * ldm + j] = (i == j ? 1.5 : 0.0) - 0.5 * gij;
    }
}
}  // namespace
}  // namespace bk

using namespace bk;

extern "C" int bk_ns_coeff_d(int a, const double* g, int ldg, double* m, int ldm, void* stream) {
    if (a <= 0) return 0;
    ns_coeff_kernel<<<max(1, min(ceil_div(a * a, 256), 4 * kSMs)), 256, 0, as_stream(stream)>>>(a, g, ldg, m, ldm);
    BK_LAUNCHED();
}
