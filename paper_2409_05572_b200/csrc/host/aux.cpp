// Auxiliary entry points of the C ABI that sit beside the hot path:
//   beig_matrix_lambda_min — dense decomposition on the device with the K5
//   Jacobi kernel (reference: sym_eig_small(to_dense(a)), proj/src/capi.cpp:97-103);
//   the analysis checks (reference proj/src/theory.cpp) are outside the scope of
//   this build (they verify the paper's theorems, not the
//   solver iteration) and report BEIG_ERR_INVALID with an explicit message.
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "../../../include/blockeig.h"
#include "host.hpp"

struct beig_matrix {
    b2::SparseSym m;
};

// beig_last_error lives in capi.cpp; errors from here are reported through
// the same thread-local slot by a small shim exported there.
extern "C" void bk_internal_set_error(const char* msg);

namespace {
int fail(int code, const char* msg) {
    bk_internal_set_error(msg);
    return code;
}
}  // namespace

extern "C" {

int beig_matrix_lambda_min(const beig_matrix* a, double* out) {
    if (!a || !out) return fail(BEIG_ERR_INVALID, "beig_matrix_lambda_min: null argument");
    try {
        const auto& m = a->m;
        const int n = m.rows();
        if (m.is_complex()) return fail(BEIG_ERR_INVALID, "lambda_min: real matrices only");
        if (n < 1) return fail(BEIG_ERR_INVALID, "lambda_min: empty matrix");
        if (n > 2048) return fail(BEIG_ERR_INVALID, "lambda_min: dense decomposition limited to n <= 2048");
        const size_t nn = static_cast<size_t>(n) * n;
        std::vector<double> dense(nn, 0.0);
        for (int r = 0; r < n; ++r)
            for (int64_t p = m.row_ptr()[r]; p < m.row_ptr()[r + 1]; ++p) {
                dense[static_cast<size_t>(r) * n + m.col()[p]] = m.val()[p];
                dense[static_cast<size_t>(m.col()[p]) * n + r] = m.val()[p];
            }
        b2::DevMem h(nn * sizeof(double)), z(nn * sizeof(double)), vals(n * sizeof(double)),
            work(bk_syev_work_bytes(n)), info(4 * sizeof(int));
        b2::cuda_check(cudaMemcpy(h.p(), dense.data(), nn * sizeof(double), cudaMemcpyHostToDevice), "upload");
        b2::cuda_check(bk_syev_d(n, h.d(), n, 1, vals.d(), z.d(), n, work.p(), info.as<int>(), nullptr), "bk_syev_d");
        int hinfo[2] = {0, 0};
        double v0 = 0.0;
        b2::cuda_check(cudaMemcpy(hinfo, info.p(), 2 * sizeof(int), cudaMemcpyDeviceToHost), "download");
        b2::cuda_check(cudaMemcpy(&v0, vals.p(), sizeof(double), cudaMemcpyDeviceToHost), "download");
        if (hinfo[1]) return fail(BEIG_ERR_NUMERIC, "sym_eig_small: eigensolver failed");
        *out = v0;
        bk_internal_set_error("");
        return BEIG_OK;
    } catch (const std::exception& e) {
        return fail(BEIG_ERR_INTERNAL, e.what());
    }
}

static const char* kTheory =
    "analysis checks (reference proj/src/theory.cpp) are outside the hot-path scope of this build";

int beig_theory_example3x3(beig_example3x3* out) {
    if (!out) return fail(BEIG_ERR_INVALID, "beig_theory_example3x3: null argument");
    return fail(BEIG_ERR_INVALID, kTheory);
}
int beig_theory_rate_suite(beig_suite_outcome* out, int trials, uint64_t, char*, size_t) {
    if (!out || trials < 1) return fail(BEIG_ERR_INVALID, "beig_theory_rate_suite: bad arguments");
    return fail(BEIG_ERR_INVALID, kTheory);
}
int beig_theory_decomp_suite(beig_suite_outcome* out, int trials, uint64_t, char*, size_t) {
    if (!out || trials < 1) return fail(BEIG_ERR_INVALID, "beig_theory_decomp_suite: bad arguments");
    return fail(BEIG_ERR_INVALID, kTheory);
}
int beig_theory_perturb_suite(beig_suite_outcome* out, int trials, uint64_t, char*, size_t) {
    if (!out || trials < 1) return fail(BEIG_ERR_INVALID, "beig_theory_perturb_suite: bad arguments");
    return fail(BEIG_ERR_INVALID, kTheory);
}
int beig_theory_scaling(beig_scaling_outcome* out, uint64_t) {
    if (!out) return fail(BEIG_ERR_INVALID, "beig_theory_scaling: null argument");
    return fail(BEIG_ERR_INVALID, kTheory);
}

}  // extern "C"
