// complex128 (Hermitian) variants of the dense block kernels — config 5.
//
// The reference is real-only (complex128 is new).  Complex
// n x k blocks are stored as interleaved (re, im) row-major, i.e. a REAL
// n x 2k block (the "real view").  Every tall-skinny contraction is then run
// on the real views by the FP64 DMMA kernels of bk_dense.cu, and only small
// matrices are rearranged:
//
//  * Gram  C = X^H Y: real-view Gram G' = Xr^T Yr (2a x 2b), then
//      C[p][q] = (G'[2p][2q] + G'[2p+1][2q+1]) + i (G'[2p][2q+1] - G'[2p+1][2q])
//    (8 n a b real flops = the complex count, on the tensor pipe);
//  * update Y = X C: Y_r = X_r E with E (2d x 2k) the block expansion
//      E[2p][2q] = E[2p+1][2q+1] = Re C,  E[2p][2q+1] = Im C,  E[2p+1][2q] = -Im C;
//  * Cholesky with the drop rule: the real 2a x 2a matrix
//      Emb(conj G) (blocks [[Re g, Im g], [-Im g, Re g]])
//    has the real Cholesky factor Emb(conj R) when G = R^H R, so the real
//    skip-pivot routine runs on it with index pairs (2c, 2c+1) locked together
//    and R^{-1} is read back from the even rows;
//  * column norms / residual norms: sums over the (re, im) column pairs.
#include "bk_chol.cuh"

namespace bk {
namespace {

constexpr size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

// C (a x b complex, ldc complex) from the real-view Gram G' (2a x 2b, ld 2b)
__global__ void gram_combine_kernel(int a, int b, const double* __restrict__ gp, double* __restrict__ c, int ldc) {
    const int total = a * b;
    const int ld = 2 * b;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        const int p = e / b, q = e - p * b;
        const double* r0 = gp + static_cast<size_t>(2 * p) * ld + 2 * q;
        const double* r1 = r0 + ld;
        double* o = c + 2 * (static_cast<size_t>(p) * ldc + q);
        o[0] = r0[0] + r1[1];
        o[1] = r0[1] - r1[0];
    }
}

// E (2d x 2k, ld 2k) from C (d x k complex, ldc complex)
__global__ void expand_kernel(int d, int k, const double* __restrict__ c, int ldc, double* __restrict__ e) {
    const int total = d * k;
    const int ld = 2 * k;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int p = t / k, q = t - p * k;
        const double re = c[2 * (static_cast<size_t>(p) * ldc + q)];
        const double im = c[2 * (static_cast<size_t>(p) * ldc + q) + 1];
        double* r0 = e + static_cast<size_t>(2 * p) * ld + 2 * q;
        double* r1 = r0 + ld;
        r0[0] = re;
        r0[1] = im;
        r1[0] = -im;
        r1[1] = re;
    }
}

// out[c] = in[2c] + in[2c+1]
__global__ void pairsum_kernel(int k, const double* __restrict__ in, double* __restrict__ out) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x)
        out[c] = in[2 * c] + in[2 * c + 1];
}

// out[2c] = out[2c+1] = in[c]
__global__ void dup_kernel(int k, const double* __restrict__ in, double* __restrict__ out) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x) {
        const double v = in[c];
        out[2 * c] = v;
        out[2 * c + 1] = v;
    }
}

// Emb(conj G) (2a x 2a, ld 2a) from a complex Gram G (a x a, ldg complex)
__global__ void emb_kernel(int a, const double* __restrict__ g, int ldg, double* __restrict__ e) {
    const int total = a * a;
    const int ld = 2 * a;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int p = t / a, q = t - p * a;
        const double re = g[2 * (static_cast<size_t>(p) * ldg + q)];
        const double im = g[2 * (static_cast<size_t>(p) * ldg + q) + 1];
        double* r0 = e + static_cast<size_t>(2 * p) * ld + 2 * q;
        double* r1 = r0 + ld;
        r0[0] = re;
        r0[1] = im;
        r1[0] = -im;
        r1[1] = re;
    }
}

// complex m (a x a, ldm complex) from the real chol output mr (2a x 2a, ld 2a):
// m[p][q] = mr[2p][2q] + i mr[2p][2q+1]; info[0] (kept) halved
__global__ void chol_extract_kernel(int a, const double* __restrict__ mr, double* __restrict__ m, int ldm,
                                    int* __restrict__ info) {
    const int total = a * a;
    const int ld = 2 * a;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int p = t / a, q = t - p * a;
        const double* r0 = mr + static_cast<size_t>(2 * p) * ld + 2 * q;
        double* o = m + 2 * (static_cast<size_t>(p) * ldm + q);
        o[0] = r0[0];
        o[1] = r0[1];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) info[0] >>= 1;
}

// m = (3I - (g + g^H)/2) / 2, complex a x a
__global__ void ns_coeff_z_kernel(int a, const double* __restrict__ g, int ldg, double* __restrict__ m, int ldm) {
    const int total = a * a;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        const int i = e / a, j = e - i * a;
        const double* gij = g + 2 * (static_cast<size_t>(i) * ldg + j);
        const double* gji = g + 2 * (static_cast<size_t>(j) * ldg + i);
        const double hr = 0.5 * (gij[0] + gji[0]);
        const double hi = 0.5 * (gij[1] - gji[1]);
        double* o = m + 2 * (static_cast<size_t>(i) * ldm + j);
        o[0] = (i == j ? 1.5 : 0.0) - 0.5 * hr;
        o[1] = -0.5 * hi;
    }
}

// complex transposes between the column-major host layout and row-major device blocks
__global__ void cm_to_rm_z_kernel(int n, int k, const double2* __restrict__ cm, int ldcm, double2* __restrict__ rm,
                                  int ldrm) {
    const int64_t total = static_cast<int64_t>(n) * k;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(e / k), c = static_cast<int>(e % k);
        rm[static_cast<size_t>(i) * ldrm + c] = cm[static_cast<size_t>(c) * ldcm + i];
    }
}
__global__ void rm_to_cm_z_kernel(int n, int k, const double2* __restrict__ rm, int ldrm, double2* __restrict__ cm,
                                  int ldcm) {
    const int64_t total = static_cast<int64_t>(n) * k;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(e / n), i = static_cast<int>(e % n);
        cm[static_cast<size_t>(c) * ldcm + i] = rm[static_cast<size_t>(i) * ldrm + c];
    }
}

int small_grid(int64_t total) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 8 * kSMs))); }

}  // namespace
}  // namespace bk

using namespace bk;

// long contractions (n > 512 rows) take the 3M DMMA kernels of bk_zdense.cu
extern "C" int bk_z3m_enabled();
extern "C" int bk_gram_z3m(int n, const double* x, int ldx, int a, const double* y, int ldy, int b, double* c, int ldc,
                           void* work, const int* run_if, void* stream);
extern "C" int bk_gram_sym_z3m(int n, const double* x, int ldx, const double* y, int ldy, int d, double* c, int ldc,
                               void* work, void* stream);
extern "C" int bk_gemm_z3m(int n, const double* x, int ldx, int d, const double* c, int ldc, int k, double alpha,
                           double beta, double* y, int ldy, const int* run_if, void* stream);
namespace {
inline bool use3m(int n) { return n > 512 && bk_z3m_enabled(); }
}  // namespace

extern "C" size_t bk_gram_z_work_bytes(int n, int a, int b) {
    return align256(bk_gram_work_bytes(n, 2 * a, 2 * b)) + align256(4 * static_cast<size_t>(a) * b * sizeof(double));
}

extern "C" int bk_gram_z(int n, const double* x, int ldx, int a, const double* y, int ldy, int b, double* c, int ldc,
                         void* work, void* stream) {
    if (a <= 0 || b <= 0) return 0;
    if (use3m(n)) return bk_gram_z3m(n, x, ldx, a, y, ldy, b, c, ldc, work, nullptr, stream);
    const cudaStream_t s = as_stream(stream);
    double* gp = reinterpret_cast<double*>(static_cast<char*>(work) + align256(bk_gram_work_bytes(n, 2 * a, 2 * b)));
    int rc = bk_gram_d(n, x, 2 * ldx, 2 * a, y, 2 * ldy, 2 * b, gp, 2 * b, work, stream);
    if (rc) return rc;
    gram_combine_kernel<<<small_grid(static_cast<int64_t>(a) * b), 256, 0, s>>>(a, b, gp, c, ldc);
    BK_LAUNCHED();
}

// Hermitian Rayleigh-Ritz matrix H = S^H (A S): the real symmetric-tile Gram
// of the real views computes only the 96 x 96 tiles on and above the diagonal
// and mirrors the rest by transposition; the combine step then yields exactly
// C[p][q] = conj(C[q][p]) below the diagonal tiles (4 n d (d+1)-class flops)
extern "C" int bk_gram_sym_z(int n, const double* x, int ldx, const double* y, int ldy, int d, double* c, int ldc,
                             void* work, void* stream) {
    if (d <= 0) return 0;
    if (use3m(n)) return bk_gram_sym_z3m(n, x, ldx, y, ldy, d, c, ldc, work, stream);
    const cudaStream_t s = as_stream(stream);
    double* gp = reinterpret_cast<double*>(static_cast<char*>(work) + align256(bk_gram_work_bytes(n, 2 * d, 2 * d)));
    int rc = bk_gram_sym_d(n, x, 2 * ldx, y, 2 * ldy, 2 * d, gp, 2 * d, work, stream);
    if (rc) return rc;
    gram_combine_kernel<<<small_grid(static_cast<int64_t>(d) * d), 256, 0, s>>>(d, d, gp, c, ldc);
    BK_LAUNCHED();
}

// predicated (device flag) variants for the second Gram-Schmidt pass
extern "C" int bk_gram_if_z(int n, const double* x, int ldx, int a, const double* y, int ldy, int b, double* c,
                            int ldc, void* work, const int* run_if, void* stream) {
    if (a <= 0 || b <= 0 || n <= 0) return 0;
    if (use3m(n)) return bk_gram_z3m(n, x, ldx, a, y, ldy, b, c, ldc, work, run_if, stream);
    const cudaStream_t s = as_stream(stream);
    double* gp = reinterpret_cast<double*>(static_cast<char*>(work) + align256(bk_gram_work_bytes(n, 2 * a, 2 * b)));
    int rc = bk_gram_if_d(n, x, 2 * ldx, 2 * a, y, 2 * ldy, 2 * b, gp, 2 * b, work, run_if, stream);
    if (rc) return rc;
    gram_combine_kernel<<<small_grid(static_cast<int64_t>(a) * b), 256, 0, s>>>(a, b, gp, c, ldc);  // harmless if skipped
    BK_LAUNCHED();
}

extern "C" int bk_gemm_if_z(int n, const double* x, int ldx, int d, const double* c, int ldc, int k, double alpha,
                            double beta, double* y, int ldy, void* work, const int* run_if, void* stream) {
    if (n <= 0 || k <= 0 || d <= 0) return 0;
    if (use3m(n)) return bk_gemm_z3m(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, run_if, stream);
    const cudaStream_t s = as_stream(stream);
    double* e = static_cast<double*>(work);
    expand_kernel<<<small_grid(static_cast<int64_t>(d) * k), 256, 0, s>>>(d, k, c, ldc, e);
    const int rc = static_cast<int>(cudaGetLastError());
    if (rc) return rc;
    return bk_gemm_if_d(n, x, 2 * ldx, 2 * d, e, 2 * k, 2 * k, alpha, beta, y, 2 * ldy, run_if, stream);
}

extern "C" size_t bk_gemm_z_work_bytes(int d, int k) { return 4 * static_cast<size_t>(d > 0 ? d : 1) * (k > 0 ? k : 1) * sizeof(double); }

extern "C" int bk_gemm_z(int n, const double* x, int ldx, int d, const double* c, int ldc, int k, double alpha,
                         double beta, double* y, int ldy, void* work, void* stream) {
    if (n <= 0 || k <= 0) return 0;
    if (d > 0 && use3m(n)) return bk_gemm_z3m(n, x, ldx, d, c, ldc, k, alpha, beta, y, ldy, nullptr, stream);
    const cudaStream_t s = as_stream(stream);
    double* e = static_cast<double*>(work);
    if (d > 0) expand_kernel<<<small_grid(static_cast<int64_t>(d) * k), 256, 0, s>>>(d, k, c, ldc, e);
    const int rc = static_cast<int>(cudaGetLastError());
    if (rc) return rc;
    return bk_gemm_d(n, x, 2 * ldx, 2 * d, e, 2 * k, 2 * k, alpha, beta, y, 2 * ldy, stream);
}

extern "C" size_t bk_colnorm2_z_work_bytes(int n, int k) {
    return align256(bk_colnorm2_work_bytes(n, 2 * k)) + align256(2 * static_cast<size_t>(k > 0 ? k : 1) * sizeof(double));
}

extern "C" int bk_colnorm2_z(int n, const double* x, int ldx, int k, double* out, void* work, void* stream) {
    if (k <= 0) return 0;
    double* tmp = reinterpret_cast<double*>(static_cast<char*>(work) + align256(bk_colnorm2_work_bytes(n, 2 * k)));
    int rc = bk_colnorm2_d(n, x, 2 * ldx, 2 * k, tmp, work, stream);
    if (rc) return rc;
    pairsum_kernel<<<ceil_div(k, 256), 256, 0, as_stream(stream)>>>(k, tmp, out);
    BK_LAUNCHED();
}

extern "C" size_t bk_coldot_z_work_bytes(int n, int k) { return bk_colnorm2_z_work_bytes(n, k); }

extern "C" int bk_coldot_z(int n, const double* x, int ldx, const double* y, int ldy, int k, double* out, void* work,
                           void* stream) {
    if (k <= 0) return 0;
    double* tmp = reinterpret_cast<double*>(static_cast<char*>(work) + align256(bk_colnorm2_work_bytes(n, 2 * k)));
    int rc = bk_coldot_d(n, x, 2 * ldx, y, 2 * ldy, 2 * k, tmp, work, stream);
    if (rc) return rc;
    pairsum_kernel<<<ceil_div(k, 256), 256, 0, as_stream(stream)>>>(k, tmp, out);
    BK_LAUNCHED();
}

extern "C" size_t bk_residual_z_work_bytes(int n, int k) {
    return align256(bk_residual_work_bytes(n, 2 * k)) + align256(8 * static_cast<size_t>(k > 0 ? k : 1) * sizeof(double));
}

extern "C" int bk_residual_w_z(int n, const double* v, int ldv, const double* av, int ldav, const double* lambda,
                               int k, double* r, int ldr, const double* t, double* w, int ldw, int w_from,
                               double* rn2, double* vn2, double* wn2, void* work, void* stream) {
    if (k <= 0) return 0;
    const cudaStream_t s = as_stream(stream);
    double* lam2 = reinterpret_cast<double*>(static_cast<char*>(work) + align256(bk_residual_work_bytes(n, 2 * k)));
    double* rn2r = lam2 + 2 * k;
    double* vn2r = rn2r + 2 * k;
    double* wn2r = vn2r + 2 * k;
    dup_kernel<<<ceil_div(k, 256), 256, 0, s>>>(k, lambda, lam2);
    int rc = bk_residual_w_d(n, v, 2 * ldv, av, 2 * ldav, lam2, 2 * k, r, 2 * ldr, t, w, 2 * ldw, 2 * w_from, rn2r,
                             vn2r, wn2 ? wn2r : nullptr, work, stream);
    if (rc) return rc;
    pairsum_kernel<<<ceil_div(k, 256), 256, 0, s>>>(k, rn2r, rn2);
    pairsum_kernel<<<ceil_div(k, 256), 256, 0, s>>>(k, vn2r, vn2);
    if (wn2 && w && k > w_from) pairsum_kernel<<<ceil_div(k - w_from, 256), 256, 0, s>>>(k - w_from, wn2r, wn2);
    BK_LAUNCHED();
}

extern "C" int bk_residual_z(int n, const double* v, int ldv, const double* av, int ldav, const double* lambda, int k,
                             double* r, int ldr, const double* t, double* w, int ldw, int w_from, double* rn2,
                             double* vn2, void* work, void* stream) {
    return bk_residual_w_z(n, v, ldv, av, ldav, lambda, k, r, ldr, t, w, ldw, w_from, rn2, vn2, nullptr, work,
                           stream);
}

extern "C" int bk_ns_coeff_z(int a, const double* g, int ldg, double* m, int ldm, void* stream) {
    if (a <= 0) return 0;
    ns_coeff_z_kernel<<<small_grid(static_cast<int64_t>(a) * a), 256, 0, as_stream(stream)>>>(a, g, ldg, m, ldm);
    BK_LAUNCHED();
}

extern "C" size_t bk_chol_z_work_bytes(int a) {
    const size_t a2 = 2 * static_cast<size_t>(a > 0 ? a : 1);
    return align256(bk_chol_work_bytes(static_cast<int>(a2))) + 2 * align256(a2 * a2 * sizeof(double)) +
           align256(a2 * sizeof(double));
}

extern "C" int bk_chol_drop_cond_z(int a, const double* g, int ldg, const double* ref2, double drop, double* m,
                                   int ldm, int* info, int* cond, void* work, void* stream) {
    const cudaStream_t s = as_stream(stream);
    if (a <= 0) {
        BK_RET(cudaMemsetAsync(info, 0, 3 * sizeof(int), s));
        if (cond) BK_RET(cudaMemsetAsync(cond, 0, 2 * sizeof(int), s));
        return 0;
    }
    const size_t a2 = 2 * static_cast<size_t>(a);
    char* p = static_cast<char*>(work);
    void* cw = p;
    p += align256(bk_chol_work_bytes(static_cast<int>(a2)));
    double* e = reinterpret_cast<double*>(p);
    p += align256(a2 * a2 * sizeof(double));
    double* mr = reinterpret_cast<double*>(p);
    p += align256(a2 * a2 * sizeof(double));
    double* r2 = reinterpret_cast<double*>(p);
    emb_kernel<<<small_grid(static_cast<int64_t>(a) * a), 256, 0, s>>>(a, g, ldg, e);
    if (ref2) dup_kernel<<<ceil_div(a, 256), 256, 0, s>>>(a, ref2, r2);
    int rc = chol_launch(static_cast<int>(a2), e, static_cast<int>(a2), ref2 ? r2 : nullptr, drop, mr,
                         static_cast<int>(a2), info, cw, s, true, cond);
    if (rc) return rc;
    chol_extract_kernel<<<small_grid(static_cast<int64_t>(a) * a), 256, 0, s>>>(a, mr, m, ldm, info);
    BK_LAUNCHED();
}

extern "C" int bk_chol_drop_z(int a, const double* g, int ldg, const double* ref2, double drop, double* m, int ldm,
                              int* info, void* work, void* stream) {
    return bk_chol_drop_cond_z(a, g, ldg, ref2, drop, m, ldm, info, nullptr, work, stream);
}

extern "C" int bk_cm_to_rm_z(int n, int k, const double* cm, int ldcm, double* rm, int ldrm, void* stream) {
    if (n <= 0 || k <= 0) return 0;
    cm_to_rm_z_kernel<<<small_grid(static_cast<int64_t>(n) * k), 256, 0, as_stream(stream)>>>(
        n, k, reinterpret_cast<const double2*>(cm), ldcm, reinterpret_cast<double2*>(rm), ldrm);
    BK_LAUNCHED();
}

extern "C" int bk_rm_to_cm_z(int n, int k, const double* rm, int ldrm, double* cm, int ldcm, void* stream) {
    if (n <= 0 || k <= 0) return 0;
    rm_to_cm_z_kernel<<<small_grid(static_cast<int64_t>(n) * k), 256, 0, as_stream(stream)>>>(
        n, k, reinterpret_cast<const double2*>(rm), ldrm, reinterpret_cast<double2*>(cm), ldcm);
    BK_LAUNCHED();
}
