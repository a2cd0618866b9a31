// Uses the reference-named C++ shim (include/blws/blws.hpp): a warm-started
// BLWS partial SVD and an RPCA solve, the two entry points a caller of the
// reference (proj/include/blws) would switch over.
#include <cmath>
#include <cstdio>

#include "blws/blws.hpp"

int main() {
    using namespace blws;
    Context ctx(0);
    Rng rng(7);
    const Index m = 300, n = 240, r = 12;
    // W = L R^T (rank 20) + small noise
    Matrix l = rng.split(1).gaussian_matrix(m, 20), rr = rng.split(2).gaussian_matrix(n, 20);
    Matrix w(m, n);
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < m; ++i) {
            double s = 0;
            for (Index k = 0; k < 20; ++k) s += l(i, k) * rr(j, k);
            w(i, j) = s;
        }
    DenseOperator op(ctx, w);
    WarmStart warm = adapt_subspace(ctx, std::nullopt, r, m, n, rng);
    for (int it = 0; it < 3; ++it) warm = blws_svd(op, warm, 2, r, rng).warm;
    std::setvbuf(stdout, nullptr, _IONBF, 0);
    std::printf("blws_svd sigma[0..2] = %.6f %.6f %.6f, applications %lld\n", warm.sigma[0], warm.sigma[1],
                warm.sigma[2], static_cast<long long>(op.application_count()));

    // RPCA on a square low-rank + sparse D (solvers.hpp:72-157)
    const Index q = 200;
    Matrix lq = rng.split(3).gaussian_matrix(q, 10), rq = rng.split(4).gaussian_matrix(q, 10);
    Matrix d(q, q);
    for (Index j = 0; j < q; ++j)
        for (Index i = 0; i < q; ++i) {
            double s = 0;
            for (Index k = 0; k < 10; ++k) s += lq(i, k) * rq(j, k);
            d(i, j) = s + ((i * 7 + j * 13) % 41 == 0 ? 300.0 : 0.0);
        }
    auto backend = SvdBackend::blws(ctx);
    RpcaSolution sol = rpca_adm(d, 0.0, backend);
    std::printf("rpca_adm: converged %d iterations %lld rank %lld\n", sol.stats.converged ? 1 : 0,
                static_cast<long long>(sol.stats.iterations), static_cast<long long>(sol.stats.rank_hat));
    return sol.stats.converged ? 0 : 1;
}
