// Sparse shift-and-invert factor (reference SpdFactor sparse path,
// proj/src/kernel.cpp:110-134: Eigen SimplicialLLT of A - zeta I with its
// default AMD ordering, for n > kDenseThreshold = 2000).
//
// Host: the one-time symbolic analysis — AMD ordering (cuSOLVER's
// cusolverSpXcsrsymamdHost, the same approximate-minimum-degree family as
// Eigen's AMDOrdering), the elimination tree (Liu), the row patterns of L by
// etree reach, the column structure, and the etree level sets that schedule
// the device work.  Device: the numeric factorisation and every solve
// (bk_spchol.cu).  The factor equals the reference's to rounding (a different
// summation order), so solves agree to rounding.
#include <cusolverSp.h>
#include <cusparse.h>

#include <algorithm>
#include <numeric>
#include <stdexcept>
#include <string>

#include "host.hpp"

namespace b2 {

namespace {
void sp_check(int status, const char* what) {
    if (status != 0) throw CudaError(std::string(what) + " failed with status " + std::to_string(status));
}

// AMD permutation of the full symmetric pattern (p[new] = old)
std::vector<int> amd_order(int n, const std::vector<int>& rp, const std::vector<int>& col) {
    std::vector<int> p(n);
    cusolverSpHandle_t h = nullptr;
    cusparseMatDescr_t d = nullptr;
    sp_check(cusolverSpCreate(&h), "cusolverSpCreate");
    const int st1 = cusparseCreateMatDescr(&d);
    if (st1 != 0) {
        cusolverSpDestroy(h);
        sp_check(st1, "cusparseCreateMatDescr");
    }
    cusparseSetMatType(d, CUSPARSE_MATRIX_TYPE_GENERAL);
    cusparseSetMatIndexBase(d, CUSPARSE_INDEX_BASE_ZERO);
    const int st = cusolverSpXcsrsymamdHost(h, n, static_cast<int>(col.size()), d, rp.data(), col.data(), p.data());
    cusparseDestroyMatDescr(d);
    cusolverSpDestroy(h);
    sp_check(st, "cusolverSpXcsrsymamdHost");
    return p;
}
}  // namespace

SpChol::SpChol(const SparseSym& a, double sgn, double shift, void* stream) : n_(a.rows()) {
    if (a.is_complex()) throw std::invalid_argument("shift-and-invert: complex matrices need the shifted operator mode");
    const int n = n_;
    // full symmetric pattern of B = sgn A - shift I (diagonal always present)
    const auto& f = a.full_csr();
    std::vector<int> rp(n + 1, 0), col;
    std::vector<double> val;
    col.reserve(f.col.size() + n);
    val.reserve(f.col.size() + n);
    for (int r = 0; r < n; ++r) {
        bool diag = false;
        std::vector<std::pair<int, double>> row;
        for (int p = f.rp[r]; p < f.rp[r + 1]; ++p) {
            double v = sgn * f.val[p];
            if (f.col[p] == r) {
                v -= shift;
                diag = true;
            }
            row.emplace_back(f.col[p], v);
        }
        if (!diag) row.emplace_back(r, -shift);
        std::sort(row.begin(), row.end(), [](auto& x, auto& y) { return x.first < y.first; });
        for (auto& e : row) {
            col.push_back(e.first);
            val.push_back(e.second);
        }
        rp[r + 1] = static_cast<int>(col.size());
    }
    perm_h_ = amd_order(n, rp, col);
    std::vector<int> pinv(n);
    for (int i = 0; i < n; ++i) pinv[perm_h_[i]] = i;

    // lower CSR of C = P B P^T: row i holds (j, v) for j <= i, ascending
    std::vector<int64_t> crp(n + 1, 0);
    std::vector<int> ccol;
    std::vector<double> cval;
    ccol.reserve(col.size() / 2 + n);
    cval.reserve(col.size() / 2 + n);
    {
        std::vector<std::pair<int, double>> row;
        for (int i = 0; i < n; ++i) {
            const int old = perm_h_[i];
            row.clear();
            for (int p = rp[old]; p < rp[old + 1]; ++p) {
                const int j = pinv[col[p]];
                if (j <= i) row.emplace_back(j, val[p]);
            }
            std::sort(row.begin(), row.end(), [](auto& x, auto& y) { return x.first < y.first; });
            for (auto& e : row) {
                ccol.push_back(e.first);
                cval.push_back(e.second);
            }
            crp[i + 1] = static_cast<int64_t>(ccol.size());
        }
    }
    // elimination tree (Liu, path compression)
    std::vector<int> parent(n, -1), anc(n, -1);
    for (int k = 0; k < n; ++k)
        for (int64_t p = crp[k]; p < crp[k + 1]; ++p) {
            int i = ccol[p];
            while (i != -1 && i < k) {
                const int next = anc[i];
                anc[i] = k;
                if (next == -1) parent[i] = k;
                i = next;
            }
        }
    // row patterns of L (etree reach of each row's lower entries), ascending
    std::vector<int64_t> rptr(n + 1, 0);
    std::vector<int> rk;
    std::vector<int> mark(n, -1), stack;
    for (int i = 0; i < n; ++i) {
        stack.clear();
        mark[i] = i;
        for (int64_t p = crp[i]; p < crp[i + 1]; ++p)
            for (int x = ccol[p]; x != -1 && x < i && mark[x] != i; x = parent[x]) {
                mark[x] = i;
                stack.push_back(x);
            }
        std::sort(stack.begin(), stack.end());
        rk.insert(rk.end(), stack.begin(), stack.end());
        rptr[i + 1] = static_cast<int64_t>(rk.size());
    }
    // column structure: diagonal first, then the rows ascending
    std::vector<int64_t> colptr(n + 1, 0);
    for (int j = 0; j < n; ++j) colptr[j + 1] = 1;
    for (int k : rk) colptr[k + 1] += 1;
    for (int j = 0; j < n; ++j) colptr[j + 1] += colptr[j];
    nnz_l_ = colptr[n];
    std::vector<int> rowind(static_cast<size_t>(nnz_l_));
    std::vector<int64_t> next(colptr.begin(), colptr.end() - 1), rpos(rk.size());
    for (int j = 0; j < n; ++j) rowind[next[j]++] = j;
    for (int i = 0; i < n; ++i)
        for (int64_t e = rptr[i]; e < rptr[i + 1]; ++e) {
            const int j = rk[e];
            rpos[e] = next[j];
            rowind[next[j]++] = i;
        }
    // where each entry of C lands in L's values
    std::vector<int64_t> aidx(ccol.size());
    for (int i = 0; i < n; ++i)
        for (int64_t p = crp[i]; p < crp[i + 1]; ++p) {
            const int j = ccol[p];
            const auto b = rowind.begin() + colptr[j], e = rowind.begin() + colptr[j + 1];
            aidx[p] = static_cast<int64_t>(std::lower_bound(b, e, i) - rowind.begin());
        }
    // etree levels from the leaves: level(parent) > level(child)
    std::vector<int> level(n, 0);
    int nlev = 0;
    for (int j = 0; j < n; ++j) {
        nlev = std::max(nlev, level[j] + 1);
        if (parent[j] != -1) level[parent[j]] = std::max(level[parent[j]], level[j] + 1);
    }
    lvlptr_h_.assign(nlev + 1, 0);
    for (int j = 0; j < n; ++j) lvlptr_h_[level[j] + 1] += 1;
    for (int l = 0; l < nlev; ++l) lvlptr_h_[l + 1] += lvlptr_h_[l];
    std::vector<int> order(n), fill(lvlptr_h_.begin(), lvlptr_h_.end() - 1);
    for (int j = 0; j < n; ++j) order[fill[level[j]]++] = j;
    nlev_ = nlev;

    // upload and factor on the device
    auto up = [&](DevMem& m, const void* src, size_t bytes) {
        m.alloc(std::max<size_t>(bytes, 8));
        if (bytes) cuda_check(cudaMemcpyAsync(m.p(), src, bytes, cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)),
                              "spchol upload");
    };
    up(colptr_, colptr.data(), colptr.size() * sizeof(int64_t));
    up(rowind_, rowind.data(), rowind.size() * sizeof(int));
    up(rptr_, rptr.data(), rptr.size() * sizeof(int64_t));
    up(rk_, rk.data(), rk.size() * sizeof(int));
    up(rpos_, rpos.data(), rpos.size() * sizeof(int64_t));
    up(order_, order.data(), order.size() * sizeof(int));
    up(lvlptr_, lvlptr_h_.data(), lvlptr_h_.size() * sizeof(int));
    up(perm_, perm_h_.data(), perm_h_.size() * sizeof(int));
    DevMem aidx_d, aval_d;
    up(aidx_d, aidx.data(), aidx.size() * sizeof(int64_t));
    up(aval_d, cval.data(), cval.size() * sizeof(double));
    val_.alloc(static_cast<size_t>(nnz_l_) * sizeof(double));
    fail_.alloc(sizeof(int));
    cuda_check(bk_spchol_factor_d(n, nlev_, lvlptr_h_.data(), order_.as<int>(), colptr_.as<int64_t>(),
                                  rowind_.as<int>(), val_.d(), nnz_l_, rptr_.as<int64_t>(), rk_.as<int>(),
                                  rpos_.as<int64_t>(), static_cast<int64_t>(aidx.size()), aidx_d.as<int64_t>(),
                                  aval_d.d(), fail_.as<int>(), stream),
               "bk_spchol_factor_d");
    int fail = 0;
    cuda_check(cudaMemcpyAsync(&fail, fail_.p(), sizeof(int), cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)),
               "spchol info");
    cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "spchol sync");
    if (fail) throw std::runtime_error("SpdFactor: matrix is not positive definite");
}

void SpChol::solve(const double* x, int ldx, int m, double* y, int ldy, void* stream) {
    if (m <= 0) return;
    const int ldt = (m + 7) / 8 * 8;
    const size_t need = static_cast<size_t>(n_) * ldt * sizeof(double);
    if (t_.bytes() < need) t_.alloc(need);
    cuda_check(bk_spchol_solve_d(n_, m, x, ldx, y, ldy, t_.d(), ldt, perm_.as<int>(), nlev_, lvlptr_.as<int>(),
                                 order_.as<int>(), colptr_.as<int64_t>(), rowind_.as<int>(), val_.d(),
                                 rptr_.as<int64_t>(), rk_.as<int>(), rpos_.as<int64_t>(), stream),
               "bk_spchol_solve_d");
}

}  // namespace b2
