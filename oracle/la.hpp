// TEST INFRASTRUCTURE ONLY — part of the CPU oracle (see oracle/README.md).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg may load this code. It is never on the product path.
//
// Minimal column-major dense matrix + BLAS/LAPACK bindings against the
// OpenBLAS 0.3.30 ILP64 build bundled with numpy (symbols scipy_*_64_).
// Stands in for Eigen 3.4, which the reference uses
// (/root/reference/proj/include/blws/core/types.hpp:11-23) but which is absent
// from this image.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

using Index = std::int64_t;

struct Mat {
    Index r = 0, c = 0;
    std::vector<double> a;
    Mat() = default;
    Mat(Index rows, Index cols) : r(rows), c(cols), a(static_cast<size_t>(rows * cols), 0.0) {}
    double& operator()(Index i, Index j) { return a[static_cast<size_t>(i + j * r)]; }
    double operator()(Index i, Index j) const { return a[static_cast<size_t>(i + j * r)]; }
    double* col(Index j) { return a.data() + j * r; }
    const double* col(Index j) const { return a.data() + j * r; }
    double* data() { return a.data(); }
    const double* data() const { return a.data(); }
    static Mat zeros(Index rows, Index cols) { return Mat(rows, cols); }
    static Mat identity(Index n) {
        Mat m(n, n);
        for (Index i = 0; i < n; ++i) m(i, i) = 1.0;
        return m;
    }
    Mat left_cols(Index k) const {
        Mat o(r, k);
        std::memcpy(o.a.data(), a.data(), sizeof(double) * static_cast<size_t>(r * k));
        return o;
    }
    Mat top_rows(Index k) const {
        Mat o(k, c);
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < k; ++i) o(i, j) = (*this)(i, j);
        return o;
    }
    Mat bottom_rows(Index k) const {
        Mat o(k, c);
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < k; ++i) o(i, j) = (*this)(r - k + i, j);
        return o;
    }
    Mat transpose() const {
        Mat o(c, r);
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) o(j, i) = (*this)(i, j);
        return o;
    }
};

using Vec = std::vector<double>;

inline double norm_sq(const double* x, Index n) {
    double s = 0;
    for (Index i = 0; i < n; ++i) s += x[i] * x[i];
    return s;
}
inline double fro(const Mat& m) { return std::sqrt(norm_sq(m.data(), m.r * m.c)); }
inline double vnorm(const Vec& v) { return std::sqrt(norm_sq(v.data(), static_cast<Index>(v.size()))); }
inline double dot(const double* x, const double* y, Index n) {
    double s = 0;
    for (Index i = 0; i < n; ++i) s += x[i] * y[i];
    return s;
}
inline bool all_finite(const double* x, Index n) {
    for (Index i = 0; i < n; ++i)
        if (!std::isfinite(x[i])) return false;
    return true;
}
inline bool all_finite(const Mat& m) { return all_finite(m.data(), m.r * m.c); }

// ---- BLAS / LAPACK (ILP64, gfortran hidden string lengths appended) ----
extern "C" {
void scipy_dgemm_64_(const char*, const char*, const Index*, const Index*, const Index*,
                     const double*, const double*, const Index*, const double*, const Index*,
                     const double*, double*, const Index*, size_t, size_t);
void scipy_dgeqrf_64_(const Index*, const Index*, double*, const Index*, double*, double*,
                      const Index*, Index*);
void scipy_dorgqr_64_(const Index*, const Index*, const Index*, double*, const Index*,
                      const double*, double*, const Index*, Index*);
void scipy_dsyevd_64_(const char*, const char*, const Index*, double*, const Index*, double*,
                      double*, const Index*, Index*, const Index*, Index*, size_t, size_t);
void scipy_dsteqr_64_(const char*, const Index*, double*, double*, double*, const Index*,
                      double*, Index*, size_t);
void scipy_dgesdd_64_(const char*, const Index*, const Index*, double*, const Index*, double*,
                      double*, const Index*, double*, const Index*, double*, const Index*,
                      Index*, Index*, size_t);
void scipy_openblas_set_num_threads64_(int);
}

/// C = alpha * op(A) * op(B) + beta * C (all column-major).
inline void gemm(char ta, char tb, Index m, Index n, Index k, double alpha, const double* A,
                 Index lda, const double* B, Index ldb, double beta, double* C, Index ldc) {
    if (m == 0 || n == 0) return;
    if (k == 0) {
        for (Index j = 0; j < n; ++j)
            for (Index i = 0; i < m; ++i) C[i + j * ldc] = beta == 0.0 ? 0.0 : beta * C[i + j * ldc];
        return;
    }
    scipy_dgemm_64_(&ta, &tb, &m, &n, &k, &alpha, A, &lda, B, &ldb, &beta, C, &ldc, 1, 1);
}

/// op(A) * op(B) as a new matrix.
inline Mat mul(const Mat& A, const Mat& B, char ta = 'N', char tb = 'N') {
    const Index m = ta == 'N' ? A.r : A.c;
    const Index k = ta == 'N' ? A.c : A.r;
    const Index n = tb == 'N' ? B.c : B.r;
    const Index kb = tb == 'N' ? B.r : B.c;
    if (k != kb) throw std::logic_error("mul: inner dimension mismatch");
    Mat C(m, n);
    gemm(ta, tb, m, n, k, 1.0, A.data(), std::max<Index>(A.r, 1), B.data(),
         std::max<Index>(B.r, 1), 0.0, C.data(), std::max<Index>(m, 1));
    return C;
}

/// Host threads for the oracle's own loops (sparse products, sampled
/// evaluation); set together with OpenBLAS's count. Each output element is
/// still accumulated by one thread in the serial order, so results are
/// bitwise independent of the thread count.
inline int& loop_threads() {
    static int n = std::max(1u, std::thread::hardware_concurrency());
    return n;
}

inline void set_threads(int n) {
    scipy_openblas_set_num_threads64_(n);
    loop_threads() = std::max(1, n);
}

/// Runs f(t, T) for t in [0, T) on T = min(loop_threads(), tasks) threads.
template <typename F>
inline void parallel_tasks(Index tasks, F&& f) {
    const Index T = std::max<Index>(1, std::min<Index>(loop_threads(), tasks));
    if (T == 1) {
        for (Index t = 0; t < tasks; ++t) f(t);
        return;
    }
    std::vector<std::thread> pool;
    for (Index w = 0; w < T; ++w)
        pool.emplace_back([&, w] {
            for (Index t = w; t < tasks; t += T) f(t);
        });
    for (auto& th : pool) th.join();
}

}  // namespace orc
