// Per-phase time (block 0's %globaltimer view between grid barriers) of the two
// cooperative Lanczos kernels over one uninterrupted run of `steps` steps on a
// dense m x m operator, and the agreement of their alpha / beta sequences.
// Links the library for the Context; the kernels come from this TU (built with
// -DCOOP_PROBE). Build: tools/probes/coop_probe.sh
#include <cmath>
#include <cstdio>
#include <memory>
#include <random>
#include <vector>

#include "../../paper_1012_0365_b200/csrc/lanczos_coop.cu"
#include "../../paper_1012_0365_b200/csrc/lanczos_rows.cu"
#include "blws_cuda.h"

struct blws_context {
    std::shared_ptr<blws::Context> ctx;
};

int main(int argc, char** argv) {
    const long m = argc > 1 ? atol(argv[1]) : 2000, n = m, steps = argc > 2 ? atol(argv[2]) : 1500;
    const long mp = m, ld = m + n, cap = steps + 1;
    blws_context* h = nullptr;
    blws_context_create(0, &h);
    blws::Context& ctx = *h->ctx;
    std::mt19937_64 g(1);
    std::normal_distribution<double> nd;
    std::vector<double> w(m * n), q0(ld, 0.0);
    for (auto& x : w) x = nd(g);
    double s = 0;
    for (long i = 0; i < m; ++i) s += (q0[i] = nd(g)) * q0[i];
    for (long i = 0; i < m; ++i) q0[i] /= std::sqrt(s);
    double *dw, *q, *r, *alpha, *lb, *coup, *state, *coef;
    unsigned long long* probe;
    cudaMalloc(&dw, sizeof(double) * m * n);
    cudaMalloc(&q, sizeof(double) * ld * cap);
    cudaMalloc(&r, sizeof(double) * ld);
    cudaMalloc(&alpha, sizeof(double) * cap);
    cudaMalloc(&lb, sizeof(double) * cap);
    cudaMalloc(&coup, sizeof(double) * (cap + 1));
    cudaMalloc(&state, sizeof(double) * 2);
    cudaMalloc(&coef, sizeof(double) * cap);
    cudaMalloc(&probe, sizeof(unsigned long long) * 8);
    cudaMemcpy(dw, w.data(), sizeof(double) * m * n, cudaMemcpyHostToDevice);
    blws::g_coop_probe = probe;
    blws::g_rows_probe = probe;
    const char* cols_names[8] = {"[1] apply", "[2] r_top sum", "[3] three-term", "[4] Q^T r #1", "[5] r -= Qc #1",
                                 "[6] Q^T r #2", "[7] r -= Qc #2", "[8] beta/next"};
    const char* rows_names[8] = {"[A] apply", "[B] r sums", "[C] 3-term+QtR", "[D] coef sums", "[E] r-=Qc+QtR",
                                 "[F] coef sums", "[G] r-=Qc,norm", "beta/next"};
    std::vector<double> ref_a, ref_b;
    for (int variant = 0; variant < 2; ++variant) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(q, 0, sizeof(double) * ld * cap);
            cudaMemcpy(q, q0.data(), sizeof(double) * ld, cudaMemcpyHostToDevice);
            cudaMemset(coup, 0, sizeof(double) * (cap + 1));
            const double st[2] = {-1.0, 0.0};
            cudaMemcpy(state, st, sizeof st, cudaMemcpyHostToDevice);
            cudaMemset(probe, 0, sizeof(unsigned long long) * 8);
            cudaDeviceSynchronize();
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0, ctx.stream());
            bool ok = variant == 0 ? blws::lanczos_coop_steps(ctx, dw, m, m, n, mp, q, ld, r, alpha, lb, coup, state,
                                                              coef, cap, m + n, 0, steps)
                                   : blws::lanczos_rows_steps(ctx, dw, m, m, n, mp, q, ld, r, alpha, lb, coup, state,
                                                              coef, cap, m + n, 0, steps);
            cudaEventRecord(e1, ctx.stream());
            cudaError_t err = cudaDeviceSynchronize();
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            unsigned long long p[8];
            cudaMemcpy(p, probe, sizeof p, cudaMemcpyDeviceToHost);
            std::vector<double> ha(steps), hb(steps);
            cudaMemcpy(ha.data(), alpha, sizeof(double) * steps, cudaMemcpyDeviceToHost);
            cudaMemcpy(hb.data(), lb, sizeof(double) * steps, cudaMemcpyDeviceToHost);
            double da = 0, db = 0, am = 0;
            if (variant == 0 && rep == 0) {
                ref_a = ha;
                ref_b = hb;
            }
            for (long k = 0; k < steps; ++k) {
                da = std::max(da, std::fabs(ha[k] - ref_a[k]));
                db = std::max(db, std::fabs(hb[k] - ref_b[k]));
                am = std::max(am, std::fabs(ref_a[k]));
            }
            std::printf("%s rep %d: m=%ld steps=%ld launched=%d: %.2f ms = %.1f us/step (%s); max|d alpha|=%.2e "
                        "max|d beta|=%.2e (|alpha|max %.2e)\n",
                        variant ? "rows" : "cols", rep, m, steps, ok, ms, 1e3 * ms / steps, cudaGetErrorString(err),
                        da, db, am);
            if (rep == 1)
                for (int k = 0; k < 8; ++k)
                    std::printf("  %-16s %8.2f us/step\n", variant ? rows_names[k] : cols_names[k],
                                1e-3 * static_cast<double>(p[k]) / steps);
        }
    }
    return 0;
}
