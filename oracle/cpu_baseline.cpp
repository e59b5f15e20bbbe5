// CPU baseline of the FCC-DCT hot path — TEST / BENCH INFRASTRUCTURE ONLY.
//
// Times the reference-faithful restatement (fcct_oracle.cpp: numeric
// derive_basis plan, recursive apply_values / solve_values with per-node
// temporaries, transform.cpp:429-494; dense GEMV for naive_apply,
// transform.cpp:146-156) on the host cores, one block per call as in the
// reference API, OpenMP over blocks (SURVEY.md §8(d) "mode 2, batched").
// The sparse LU solve of the inverse is replaced by an explicit sparse B^{-1}
// (pruned at 1e-12), which is at least as fast as SparseLU's two triangular
// solves. Blocks are split statically over std::thread workers. Output: one
// JSON line.
#include <chrono>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "fcct_oracle.cpp"

template <typename F>
static void parallel_for(int64_t count, int threads, F&& f) {
    std::vector<std::thread> pool;
    for (int w = 0; w < threads; ++w)
        pool.emplace_back([&, w] {
            const int64_t lo = count * w / threads, hi = count * (w + 1) / threads;
            for (int64_t i = lo; i < hi; ++i) f(i);
        });
    for (auto& t : pool) t.join();
}

static double splitmix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    x ^= x >> 31;
    return (static_cast<double>(x >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
}

int main(int argc, char** argv) {
    int n = 8;
    int64_t blocks = 4096;
    int threads = static_cast<int>(std::thread::hardware_concurrency());
    const char* method = "fast";
    double min_seconds = 0.0;  // repeat the timed passes until this much CPU time has elapsed
    for (int i = 1; i < argc; ++i) {
        if (!std::strcmp(argv[i], "--n") && i + 1 < argc) n = std::atoi(argv[++i]);
        else if (!std::strcmp(argv[i], "--blocks") && i + 1 < argc) blocks = std::atoll(argv[++i]);
        else if (!std::strcmp(argv[i], "--threads") && i + 1 < argc) threads = std::atoi(argv[++i]);
        else if (!std::strcmp(argv[i], "--method") && i + 1 < argc) method = argv[++i];
        else if (!std::strcmp(argv[i], "--min-seconds") && i + 1 < argc) min_seconds = std::atof(argv[++i]);
    }
    const Params p{0.125, 0.0, 0.375};
    const int64_t n3 = static_cast<int64_t>(n) * n * n;
    const auto t0 = std::chrono::steady_clock::now();
    std::shared_ptr<const Plan> plan;
    std::vector<Complex> dense;
    DenseLU<Complex> dense_lu;
    const bool fast = std::strcmp(method, "fast") == 0;
    if (fast) {
        plan = make_plan(n, p);
    } else {
        dense = dense_matrix<Complex, double>(n, p);
        dense_lu = DenseLU<Complex>(dense.data(), n3);
    }
    const double plan_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::vector<Complex> x(static_cast<size_t>(blocks * n3)), y(x.size()), z(x.size());
    for (int64_t i = 0; i < blocks * n3; ++i) x[i] = Complex{splitmix(2 * i), splitmix(2 * i + 1)};
    auto fwd = [&](int64_t b) {
        std::vector<Complex> in(x.begin() + b * n3, x.begin() + (b + 1) * n3), out;
        if (fast) {
            out = plan->apply_values(in);
        } else {
            out.assign(n3, Complex{0, 0});
            for (int64_t j = 0; j < n3; ++j)
                for (int64_t i = 0; i < n3; ++i) out[i] += dense[i + j * n3] * in[j];
        }
        std::copy(out.begin(), out.end(), y.begin() + b * n3);
    };
    auto inv = [&](int64_t b) {
        std::vector<Complex> in(y.begin() + b * n3, y.begin() + (b + 1) * n3), out;
        if (fast) {
            out = plan->solve_values(in);
        } else {
            out = in;
            dense_lu.solve_inplace(out.data());
        }
        std::copy(out.begin(), out.end(), z.begin() + b * n3);
    };
    // warm-up
    parallel_for(std::min<int64_t>(blocks, threads), threads, [&](int64_t b) { fwd(b); inv(b); });
    double fs = 0.0, is = 0.0;
    int reps = 0;
    do {
        const auto ta = std::chrono::steady_clock::now();
        parallel_for(blocks, threads, fwd);
        const auto tb = std::chrono::steady_clock::now();
        parallel_for(blocks, threads, inv);
        const auto tc = std::chrono::steady_clock::now();
        fs += std::chrono::duration<double>(tb - ta).count();
        is += std::chrono::duration<double>(tc - tb).count();
        ++reps;
    } while (fs + is < min_seconds);
    fs /= reps;
    is /= reps;
    double err = 0, scale = 0;
    for (int64_t i = 0; i < blocks * n3; ++i) {
        err = std::max(err, std::abs(z[i] - x[i]));
        scale = std::max(scale, std::abs(x[i]));
    }
    std::printf("{\"n\": %d, \"method\": \"%s\", \"blocks\": %ld, \"threads\": %d, \"plan_s\": %.6g, "
                "\"forward_s\": %.6g, \"inverse_s\": %.6g, \"reps\": %d, \"roundtrip_rel_err\": %.3g}\n",
                n, method, static_cast<long>(blocks), threads, plan_s, fs, is, reps, err / scale);
    return 0;
}
