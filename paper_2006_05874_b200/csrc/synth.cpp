// synth.cpp — seeded synthetic instances for the BASELINE configs
// (SURVEY.md §8(d)): A = G diag(sigma), G drawn block-wise from
// make_stream(data_seed, 1000 + j*nb + q) with fill_gaussian (rng.hpp:30-40),
// sigma_j = decay^j or 1/j for j = 1..d (datasets.hpp:52-58 convention),
// optional outlier rows from sample_without_replacement(n, n*frac,
// make_stream(data_seed, 14)) scaled before b is formed, x_true from tag 12,
// noise from tag 13, b = A x_true + noise accumulated in column order.
// Host code, threaded over columns; the CPU oracle restates the same recipe
// (oracle/ihs_oracle.cpp synth_generate) and the tests check both agree bit
// for bit.
#include "host_rng.h"
#include "common.cuh"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <random>
#include <thread>
#include <vector>

namespace ihs_b200 {

namespace {
std::mt19937_64 make_stream(uint64_t seed, uint64_t tag) { return std::mt19937_64(derive_seed(seed, tag)); }
}  // namespace

void synth_generate(const ihs_synth_spec& s, int64_t row0, int64_t rows, double* A, int64_t lda, double* b,
                    double* x_true) {
    const int64_t n = s.n, d = s.d;
    if (n < 1 || d < 1 || row0 < 0 || rows < 0 || row0 + rows > n || lda < rows)
        fail(IHS_INVALID_INPUT, "synth_generate: bad shape");
    int64_t n_pad = 1;
    while (n_pad < n) n_pad <<= 1;
    const int64_t B = std::min<int64_t>(int64_t{1} << 16, n_pad);
    const int64_t nb = (n + B - 1) / B;
    const int64_t q0 = row0 / B, q1 = rows > 0 ? (row0 + rows - 1) / B : q0 - 1;

    // outlier mask over the requested rows
    std::vector<uint8_t> outlier;
    if (s.outlier_frac > 0.0 && rows > 0) {
        outlier.assign((size_t)rows, 0);
        const int64_t k = (int64_t)((double)n * s.outlier_frac);
        std::vector<int64_t> idx((size_t)k);
        sample_without_replacement(derive_seed(s.data_seed, 14), n, k, idx.data());
        for (int64_t r : idx)
            if (r >= row0 && r < row0 + rows) outlier[(size_t)(r - row0)] = 1;
    }

    int nthreads = s.threads > 0 ? s.threads : (int)std::max(1u, std::thread::hardware_concurrency());
    nthreads = (int)std::min<int64_t>(nthreads, d);
    std::atomic<int64_t> next{0};
    auto worker = [&] {
        std::vector<double> buf((size_t)B);
        for (;;) {
            const int64_t j = next.fetch_add(1);
            if (j >= d) break;
            const double sigma = s.spectrum == 0 ? std::pow(s.decay, (double)(j + 1)) : 1.0 / (double)(j + 1);
            for (int64_t q = q0; q <= q1; ++q) {
                std::mt19937_64 gen = make_stream(s.data_seed, (uint64_t)(1000 + j * nb + q));
                std::normal_distribution<double> dist(0.0, 1.0);
                const int64_t r0 = q * B, r1 = std::min(n, r0 + B);
                for (int64_t i = r0; i < r1; ++i) buf[(size_t)(i - r0)] = dist(gen);
                const int64_t lo = std::max(r0, row0), hi = std::min(r1, row0 + rows);
                for (int64_t i = lo; i < hi; ++i) {
                    double v = buf[(size_t)(i - r0)] * sigma;
                    if (!outlier.empty() && outlier[(size_t)(i - row0)]) v *= s.outlier_scale;
                    A[(i - row0) + j * lda] = v;
                }
            }
        }
    };
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; ++t) th.emplace_back(worker);
    for (auto& t : th) t.join();

    std::vector<double> xt((size_t)d);
    {
        std::mt19937_64 gen = make_stream(s.data_seed, 12);
        std::normal_distribution<double> dist(0.0, 1.0);
        for (int64_t j = 0; j < d; ++j) xt[(size_t)j] = dist(gen);
    }
    if (x_true) std::copy(xt.begin(), xt.end(), x_true);
    if (b) {
        std::vector<double> noise((size_t)(row0 + rows));
        {
            std::mt19937_64 gen = make_stream(s.data_seed, 13);
            std::normal_distribution<double> dist(0.0, s.noise_std);
            for (int64_t i = 0; i < row0 + rows; ++i) noise[(size_t)i] = dist(gen);
        }
        // b_i = (sum_j A_ij x_j, j ascending) + noise_i, rows split over threads
        std::vector<std::thread> tb;
        const int64_t chunk = std::max<int64_t>(1, (rows + nthreads - 1) / std::max(1, nthreads));
        for (int64_t c0 = 0; c0 < rows; c0 += chunk) {
            tb.emplace_back([&, c0] {
                const int64_t c1 = std::min(rows, c0 + chunk);
                std::vector<double> acc((size_t)(c1 - c0), 0.0);
                for (int64_t j = 0; j < d; ++j) {
                    const double xj = xt[(size_t)j];
                    const double* col = A + j * lda;
                    for (int64_t i = c0; i < c1; ++i) acc[(size_t)(i - c0)] += col[i] * xj;
                }
                for (int64_t i = c0; i < c1; ++i) b[i] = acc[(size_t)(i - c0)] + noise[(size_t)(row0 + i)];
            });
        }
        for (auto& t : tb) t.join();
    }
}

}  // namespace ihs_b200
