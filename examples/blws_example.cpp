// Uses the reference-named C++ shim (include/blws/blws.hpp) the way a caller of
// the reference (proj/include/blws) does: no context argument (the default
// context on device 0), SvdBackend::blws(Options) / exact_full(), blws_svd on a
// DenseOperator, rpca_adm(RpcaProblem, ...) with the sparse E of the
// reference, and mc_svt(McProblem, ...).
#include <cmath>
#include <cstdio>

#include "blws/blws.hpp"

int main() {
    using namespace blws;
    std::setvbuf(stdout, nullptr, _IONBF, 0);
    Rng rng(7);
    const Index m = 300, n = 240, r = 12;
    // W = L R^T (rank 20)
    Matrix l = rng.split(1).gaussian_matrix(m, 20), rr = rng.split(2).gaussian_matrix(n, 20);
    Matrix w(m, n);
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < m; ++i) {
            double s = 0;
            for (Index k = 0; k < 20; ++k) s += l(i, k) * rr(j, k);
            w(i, j) = s;
        }
    DenseOperator op(w);
    WarmStart warm = adapt_subspace(default_context(), std::nullopt, r, m, n, rng);
    for (int it = 0; it < 3; ++it) warm = blws_svd(op, warm, 2, r, rng).warm;
    std::printf("blws_svd sigma[0..2] = %.6f %.6f %.6f, applications %lld\n", warm.sigma[0], warm.sigma[1],
                warm.sigma[2], static_cast<long long>(op.application_count()));

    // RPCA on a square low-rank + sparse D (solvers.hpp:72-157)
    const Index q = 200;
    Matrix lq = rng.split(3).gaussian_matrix(q, 10), rq = rng.split(4).gaussian_matrix(q, 10);
    RpcaProblem prob;
    prob.d = Matrix(q, q);
    Index planted = 0;
    for (Index j = 0; j < q; ++j)
        for (Index i = 0; i < q; ++i) {
            double s = 0;
            for (Index k = 0; k < 10; ++k) s += lq(i, k) * rq(j, k);
            const bool corrupt = (i * 7 + j * 13) % 41 == 0;
            planted += corrupt;
            prob.d(i, j) = s + (corrupt ? 300.0 : 0.0);
        }
    SvdBackend::Options bo;
    bo.seed = 6;
    auto backend = SvdBackend::blws(bo);
    RpcaSolution sol = rpca_adm(prob, backend);
    std::printf("rpca_adm: converged %d iterations %lld rank %lld, E nonzeros %lld (planted %lld), e_l0 %lld\n",
                sol.stats.converged ? 1 : 0, static_cast<long long>(sol.stats.iterations),
                static_cast<long long>(sol.stats.rank_hat), static_cast<long long>(sol.e.nonZeros()),
                static_cast<long long>(planted), static_cast<long long>(sol.stats.e_l0));

    // the dense exact backend (svt.hpp:108-116) on the same problem
    auto exact = SvdBackend::exact_full();
    RpcaSolution sx = rpca_adm(prob, exact);
    std::printf("rpca_adm exact_full: converged %d rank %lld\n", sx.stats.converged ? 1 : 0,
                static_cast<long long>(sx.stats.rank_hat));

    // MC on a sampled rank-4 product (solvers.hpp:202-270), CSC observation
    const Index mm = 150;
    Matrix ml = rng.split(5).gaussian_matrix(mm, 4), mr = rng.split(6).gaussian_matrix(mm, 4);
    McProblem mc;
    mc.observed.rows = mc.observed.cols = mm;
    mc.observed.colptr.assign(static_cast<size_t>(mm + 1), 0);
    Rng pick = rng.split(7);
    for (Index j = 0; j < mm; ++j) {
        for (Index i = 0; i < mm; ++i)
            if (pick.uniform() < 0.3) {  // ~30 % of the entries, uniformly at random
                double s = 0;
                for (Index k = 0; k < 4; ++k) s += ml(i, k) * mr(j, k);
                mc.observed.rowidx.push_back(static_cast<std::int32_t>(i));
                mc.observed.values.push_back(s);
            }
        mc.observed.colptr[static_cast<size_t>(j + 1)] = static_cast<std::int64_t>(mc.observed.values.size());
    }
    auto mb = SvdBackend::blws(bo);
    McSolution ms = mc_svt(mc, mb);
    std::printf("mc_svt: converged %d iterations %lld rank %lld\n", ms.stats.converged ? 1 : 0,
                static_cast<long long>(ms.stats.iterations), static_cast<long long>(ms.stats.rank_hat));
    return sol.stats.converged && sx.stats.converged && ms.stats.converged ? 0 : 1;
}
