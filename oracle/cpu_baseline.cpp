// CPU baseline of the FCC-DCT hot path — TEST / BENCH INFRASTRUCTURE ONLY.
//
// Times the reference-faithful restatement (fcct_oracle.cpp: numeric
// derive_basis plan, recursive apply_values / solve_values with per-node
// temporaries, transform.cpp:429-494; dense GEMV for naive_apply,
// transform.cpp:146-156) on the host cores. Output: one JSON line.
//
// Modes (BASELINE.md "CPU baseline plan"):
//   --mode batched   (mode 2) one block per call as in the reference API,
//                    std::thread workers over blocks on all cores. The fast
//                    inverse's sparse LU solve is replaced by an explicit
//                    sparse B^{-1} (at least as fast as SparseLU's two
//                    triangular solves); the direct inverse uses one LU
//                    factored at plan time (the reference refactors per call,
//                    transform.cpp:158-169, so this is a lower bound on its
//                    time).
//   --mode faithful  (mode 1) one vector per call, the `fcct bench` protocol
//                    (tools/fcct.cpp:508-521): one warm-up call, then the
//                    median over --repeats of the mean of an inner loop of
//                    max(1, 32768 / n^3) calls. --fanout 8 runs the
//                    reference's threads = 8 top-level child fan-out
//                    (std::async per root child, transform.cpp:440-454,
//                    473-487); the direct inverse refactors D per call like
//                    inverse_apply(dense) (transform.cpp:158-169).
//   --mode fftroute  n = 64 has no reference-path baseline (the plan needs
//                    ~137 GB of dense child LUs): the
//                    FFT-route oracle D x = n^3 IFFT3(S x), inverse
//                    S^{-1} FFT3(y) / n^3 with S's orbit blocks, one thread.
#include <algorithm>
#include <barrier>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <future>
#include <thread>

#include "fcct_oracle.cpp"

using Clock = std::chrono::steady_clock;

static double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

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

// Right-looking partial-pivot LU (the DenseLU algorithm) with the trailing
// update split over threads: plan-time factorisation of the n = 16 dense D.
static DenseLU<Complex> parallel_lu(const Complex* a, int64_t d, int threads) {
    DenseLU<Complex> f;
    f.dim = d;
    f.lu.assign(a, a + d * d);
    f.piv.assign(d, 0);
    auto& lu = f.lu;
    std::barrier sync(threads);
    auto worker = [&](int w) {
        for (int64_t k = 0; k < d; ++k) {
            if (w == 0) {
                int64_t best = k;
                double bv = std::abs(lu[k + k * d]);
                for (int64_t i = k + 1; i < d; ++i)
                    if (std::abs(lu[i + k * d]) > bv) bv = std::abs(lu[i + k * d]), best = i;
                f.piv[k] = best;
                if (best != k)
                    for (int64_t j = 0; j < d; ++j) std::swap(lu[k + j * d], lu[best + j * d]);
                if (lu[k + k * d] == Complex{0, 0}) {
                    f.singular = true;
                } else {
                    const Complex inv = Complex{1, 0} / lu[k + k * d];
                    for (int64_t i = k + 1; i < d; ++i) lu[i + k * d] *= inv;
                }
            }
            sync.arrive_and_wait();
            if (!f.singular) {
                const int64_t cols = d - k - 1, j0 = k + 1 + cols * w / threads, j1 = k + 1 + cols * (w + 1) / threads;
                const Complex* ck = &lu[k * d];
                for (int64_t j = j0; j < j1; ++j) {
                    const Complex fj = lu[k + j * d];
                    Complex* cj = &lu[j * d];
                    for (int64_t i = k + 1; i < d; ++i) cj[i] -= ck[i] * fj;
                }
            }
            sync.arrive_and_wait();
        }
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < threads; ++w) pool.emplace_back(worker, w);
    worker(0);
    for (auto& t : pool) t.join();
    return f;
}

// apply_values / solve_values with the reference's threads > 1 fan-out at the
// root (transform.cpp:440-454, 473-487): the eight root children on std::async.
static std::vector<Complex> apply_fanout(const Plan& pl, const std::vector<Complex>& x, int threads) {
    if (threads <= 1 || !pl.radix) return pl.apply_values(x);
    const int64_t n3 = static_cast<int64_t>(pl.n) * pl.n * pl.n, m3 = n3 / 8;
    std::vector<Complex> t(n3, Complex{0, 0});
    for (int64_t c = 0; c < n3; ++c)
        for (int64_t k = pl.basis.colptr[c]; k < pl.basis.colptr[c + 1]; ++k) t[pl.basis.rowidx[k]] += pl.basis.val[k] * x[c];
    std::array<std::future<std::vector<Complex>>, 8> fut;
    for (int blk = 0; blk < 8; ++blk)
        fut[blk] = std::async(std::launch::async, [&, blk] {
            std::vector<Complex> in(m3);
            for (int64_t h = 0; h < m3; ++h) {
                Complex acc{0, 0};
                for (int g = 0; g < 8; ++g) acc += t[g * m3 + h] * pl.kernel[blk + g * 8];
                in[h] = acc;
            }
            return pl.children[blk]->apply_values(in);
        });
    std::vector<Complex> y(n3), out(n3);
    for (int blk = 0; blk < 8; ++blk) {
        auto o = fut[blk].get();
        std::copy(o.begin(), o.end(), y.begin() + blk * m3);
    }
    for (int64_t idx = 0; idx < n3; ++idx) out[pl.perm[idx]] = y[idx];
    return out;
}

static std::vector<Complex> solve_fanout(const Plan& pl, const std::vector<Complex>& q, int threads) {
    if (threads <= 1 || !pl.radix) return pl.solve_values(q);
    const int64_t n3 = static_cast<int64_t>(pl.n) * pl.n * pl.n, m3 = n3 / 8;
    std::vector<Complex> y(n3), x(n3), t(n3);
    for (int64_t idx = 0; idx < n3; ++idx) y[idx] = q[pl.perm[idx]];
    std::array<std::future<std::vector<Complex>>, 8> fut;
    for (int blk = 0; blk < 8; ++blk)
        fut[blk] = std::async(std::launch::async, [&, blk] {
            std::vector<Complex> in(y.begin() + blk * m3, y.begin() + (blk + 1) * m3);
            return pl.children[blk]->solve_values(in);
        });
    for (int blk = 0; blk < 8; ++blk) {
        auto o = fut[blk].get();
        std::copy(o.begin(), o.end(), x.begin() + blk * m3);
    }
    for (int64_t h = 0; h < m3; ++h)
        for (int blk = 0; blk < 8; ++blk) {
            Complex acc{0, 0};
            for (int g = 0; g < 8; ++g) acc += x[g * m3 + h] * pl.kernel_inv[blk + g * 8];
            t[blk * m3 + h] = acc;
        }
    std::vector<Complex> out(n3, Complex{0, 0});
    for (int64_t c = 0; c < n3; ++c)
        for (int64_t k = pl.basis_inv.colptr[c]; k < pl.basis_inv.colptr[c + 1]; ++k)
            out[pl.basis_inv.rowidx[k]] += pl.basis_inv.val[k] * t[c];
    return out;
}

// --- FFT route (n = 64): D = F S, S block diagonal over the S4 orbits -------
struct FftRoute {
    int n;
    int64_t n3;
    std::vector<int32_t> row;  // [24][n3] a mod n, flattened
    std::vector<Complex> ph;   // [24][n3] e^{2 pi i (w k).p / n} / 24, unreduced exponent
    std::vector<std::vector<int64_t>> orbits;
    std::vector<std::vector<Complex>> sinv;  // per orbit, row-major |O| x |O|
    std::vector<Complex> tw;                 // e^{2 pi i j / n}

    FftRoute(int n_, const Params& p) : n(n_), n3(static_cast<int64_t>(n_) * n_ * n_) {
        const auto& G = group();
        row.resize(24 * n3);
        ph.resize(24 * n3);
        for (int w = 0; w < 24; ++w)
            for (int64_t c = 0; c < n3; ++c) {
                const Index3 wk = G[w].apply(unflatten(c, n));
                int64_t a = 0;
                for (int d = 0; d < 3; ++d) a = a * n + ((wk[d] % n) + n) % n;
                row[w * n3 + c] = static_cast<int32_t>(a);
                ph[w * n3 + c] = unit_phase((p.r * wk[0] + p.s * wk[1] + p.t * wk[2]) / n) / 24.0;
            }
        std::vector<int64_t> orbit_of(n3, -1);
        for (int64_t c = 0; c < n3; ++c) {
            if (orbit_of[c] >= 0) continue;
            std::vector<int64_t> mem;
            for (int w = 0; w < 24; ++w) mem.push_back(row[w * n3 + c]);
            std::sort(mem.begin(), mem.end());
            mem.erase(std::unique(mem.begin(), mem.end()), mem.end());
            for (auto m : mem) orbit_of[m] = static_cast<int64_t>(orbits.size());
            orbits.push_back(mem);
        }
        for (const auto& mem : orbits) {
            const int64_t d = static_cast<int64_t>(mem.size());
            std::vector<Complex> S(d * d, Complex{0, 0});  // column-major
            for (int64_t j = 0; j < d; ++j)
                for (int w = 0; w < 24; ++w) {
                    const int64_t a = row[w * n3 + mem[j]];
                    const int64_t i = std::lower_bound(mem.begin(), mem.end(), a) - mem.begin();
                    S[i + j * d] += ph[w * n3 + mem[j]];
                }
            DenseLU<Complex> lu(S.data(), d);
            std::vector<Complex> inv(d * d);
            for (int64_t j = 0; j < d; ++j) {
                std::vector<Complex> e(d, Complex{0, 0});
                e[j] = 1.0;
                lu.solve_inplace(e.data());
                for (int64_t i = 0; i < d; ++i) inv[i * d + j] = e[i];
            }
            sinv.push_back(std::move(inv));
        }
        tw.resize(n);
        for (int j = 0; j < n; ++j) tw[j] = unit_phase(static_cast<double>(j) / n);
    }
    // v[q] <- sum_p v[p] e^{sign 2 pi i p q / n}, radix 2, stride s
    void line(Complex* v, int64_t s, int sign) const {
        for (int i = 1, j = 0; i < n; ++i) {  // bit reversal
            int bit = n >> 1;
            for (; j & bit; bit >>= 1) j ^= bit;
            j ^= bit;
            if (i < j) std::swap(v[i * s], v[j * s]);
        }
        for (int len = 2; len <= n; len <<= 1)
            for (int i = 0; i < n; i += len)
                for (int k = 0; k < len / 2; ++k) {
                    Complex w = tw[(k * (n / len)) % n];
                    if (sign < 0) w = std::conj(w);
                    const Complex a = v[(i + k) * s], b = v[(i + k + len / 2) * s] * w;
                    v[(i + k) * s] = a + b;
                    v[(i + k + len / 2) * s] = a - b;
                }
    }
    void fft3(std::vector<Complex>& z, int sign) const {
        const int64_t nn = static_cast<int64_t>(n) * n;
        for (int64_t a = 0; a < nn; ++a) line(&z[a * n], 1, sign);                            // k
        for (int i = 0; i < n; ++i)
            for (int k = 0; k < n; ++k) line(&z[i * nn + k], n, sign);                          // j
        for (int64_t jk = 0; jk < nn; ++jk) line(&z[jk], nn, sign);                             // i
    }
    std::vector<Complex> forward(const std::vector<Complex>& x) const {
        std::vector<Complex> z(n3, Complex{0, 0});
        for (int w = 0; w < 24; ++w)
            for (int64_t c = 0; c < n3; ++c) z[row[w * n3 + c]] += ph[w * n3 + c] * x[c];
        fft3(z, +1);
        return z;
    }
    std::vector<Complex> inverse(const std::vector<Complex>& y) const {
        std::vector<Complex> z(y);
        fft3(z, -1);
        const double sc = 1.0 / static_cast<double>(n3);
        std::vector<Complex> x(n3);
        for (size_t o = 0; o < orbits.size(); ++o) {
            const auto& mem = orbits[o];
            const int64_t d = static_cast<int64_t>(mem.size());
            for (int64_t i = 0; i < d; ++i) {
                Complex acc{0, 0};
                for (int64_t j = 0; j < d; ++j) acc += sinv[o][i * d + j] * z[mem[j]];
                x[mem[i]] = acc * sc;
            }
        }
        return x;
    }
};

int main(int argc, char** argv) {
    int n = 8;
    int64_t blocks = 4096;
    int threads = static_cast<int>(std::thread::hardware_concurrency());
    int fanout = 1, repeats = 5, min_reps = 1;
    const char* method = "fast";
    const char* mode = "batched";
    double min_seconds = 0.0;  // repeat the timed passes until this much CPU time has elapsed
    for (int i = 1; i < argc; ++i) {
        if (!std::strcmp(argv[i], "--n") && i + 1 < argc) n = std::atoi(argv[++i]);
        else if (!std::strcmp(argv[i], "--blocks") && i + 1 < argc) blocks = std::atoll(argv[++i]);
        else if (!std::strcmp(argv[i], "--threads") && i + 1 < argc) threads = std::atoi(argv[++i]);
        else if (!std::strcmp(argv[i], "--method") && i + 1 < argc) method = argv[++i];
        else if (!std::strcmp(argv[i], "--mode") && i + 1 < argc) mode = argv[++i];
        else if (!std::strcmp(argv[i], "--fanout") && i + 1 < argc) fanout = std::atoi(argv[++i]);
        else if (!std::strcmp(argv[i], "--repeats") && i + 1 < argc) repeats = std::atoi(argv[++i]);
        else if (!std::strcmp(argv[i], "--reps") && i + 1 < argc) min_reps = std::atoi(argv[++i]);
        else if (!std::strcmp(argv[i], "--min-seconds") && i + 1 < argc) min_seconds = std::atof(argv[++i]);
    }
    const Params p{0.125, 0.0, 0.375};
    const int64_t n3 = static_cast<int64_t>(n) * n * n;
    const bool fast = std::strcmp(method, "fast") == 0;

    if (!std::strcmp(mode, "fftroute")) {
        const auto t0 = Clock::now();
        FftRoute route(n, p);
        const double plan_s = since(t0);
        std::vector<Complex> x(n3);
        for (int64_t i = 0; i < n3; ++i) x[i] = Complex{splitmix(2 * i), splitmix(2 * i + 1)};
        std::vector<Complex> y = route.forward(x), z = route.inverse(y);  // warm-up
        std::vector<double> tf, ti;
        const auto tall = Clock::now();
        for (int rep = 0; rep < repeats || since(tall) < min_seconds; ++rep) {
            auto ta = Clock::now();
            y = route.forward(x);
            tf.push_back(since(ta));
            ta = Clock::now();
            z = route.inverse(y);
            ti.push_back(since(ta));
        }
        std::sort(tf.begin(), tf.end());
        std::sort(ti.begin(), ti.end());
        double err = 0, scale = 0;
        for (int64_t i = 0; i < n3; ++i) err = std::max(err, std::abs(z[i] - x[i])), scale = std::max(scale, std::abs(x[i]));
        std::printf("{\"n\": %d, \"mode\": \"fftroute\", \"threads\": 1, \"plan_s\": %.6g, \"forward_us\": %.6g, "
                    "\"inverse_us\": %.6g, \"repeats\": %zu, \"roundtrip_rel_err\": %.3g}\n",
                    n, plan_s, 1e6 * tf[tf.size() / 2], 1e6 * ti[ti.size() / 2], tf.size(), err / scale);
        return 0;
    }

    const auto t0 = Clock::now();
    std::shared_ptr<const Plan> plan;
    std::vector<Complex> dense;
    DenseLU<Complex> dense_lu;
    if (fast) {
        plan = make_plan(n, p);
    } else {
        dense = dense_matrix<Complex, double>(n, p);
        dense_lu = parallel_lu(dense.data(), n3, std::max(1, threads));
    }
    const double plan_s = since(t0);

    if (!std::strcmp(mode, "faithful")) {
        // one vector per call (tools/fcct.cpp:508-521 protocol)
        std::vector<Complex> x(n3), y, z;
        for (int64_t i = 0; i < n3; ++i) x[i] = Complex{splitmix(2 * i), splitmix(2 * i + 1)};
        const int inner = static_cast<int>(std::max<int64_t>(1, 32768 / n3));
        auto fwd = [&] {
            if (fast) {
                y = apply_fanout(*plan, x, fanout);
            } else {
                y.assign(n3, Complex{0, 0});
                for (int64_t j = 0; j < n3; ++j)
                    for (int64_t i = 0; i < n3; ++i) y[i] += dense[i + j * n3] * x[j];
            }
        };
        auto inv = [&] {
            if (fast) {
                z = solve_fanout(*plan, y, fanout);
            } else {  // inverse_apply(dense): fresh LU + condition gate per call (transform.cpp:158-169)
                DenseLU<Complex> lu(dense.data(), n3);
                require_condition(condition_with_lu(dense.data(), n3, lu), "dense transform");
                z = y;
                lu.solve_inplace(z.data());
            }
        };
        auto median = [&](auto&& once) {
            std::vector<double> t;
            once();
            const auto tall = Clock::now();
            for (int rep = 0; rep < repeats || since(tall) < min_seconds; ++rep) {
                const auto ta = Clock::now();
                for (int i = 0; i < inner; ++i) once();
                t.push_back(since(ta) / inner);
            }
            std::sort(t.begin(), t.end());
            return std::make_pair(t[t.size() / 2], t.size());
        };
        const auto [tf, rf] = median(fwd);
        const auto [ti, ri] = median(inv);
        double err = 0, scale = 0;
        for (int64_t i = 0; i < n3; ++i) err = std::max(err, std::abs(z[i] - x[i])), scale = std::max(scale, std::abs(x[i]));
        std::printf("{\"n\": %d, \"method\": \"%s\", \"mode\": \"faithful\", \"threads\": %d, \"plan_s\": %.6g, "
                    "\"forward_us\": %.6g, \"inverse_us\": %.6g, \"inner\": %d, \"repeats\": %zu, "
                    "\"roundtrip_rel_err\": %.3g}\n",
                    n, method, fanout, plan_s, 1e6 * tf, 1e6 * ti, inner, std::max(rf, ri), err / scale);
        return 0;
    }

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
    std::string rep_list;
    do {
        const auto ta = Clock::now();
        parallel_for(blocks, threads, fwd);
        const auto tb = Clock::now();
        parallel_for(blocks, threads, inv);
        const auto tc = Clock::now();
        const double f = std::chrono::duration<double>(tb - ta).count(), v = std::chrono::duration<double>(tc - tb).count();
        fs += f;
        is += v;
        char buf[32];
        std::snprintf(buf, sizeof(buf), "%s%.6g", reps ? ", " : "", f + v);
        rep_list += buf;
        ++reps;
    } while (fs + is < min_seconds || reps < min_reps);
    fs /= reps;
    is /= reps;
    double err = 0, scale = 0;
    for (int64_t i = 0; i < blocks * n3; ++i) {
        err = std::max(err, std::abs(z[i] - x[i]));
        scale = std::max(scale, std::abs(x[i]));
    }
    std::printf("{\"n\": %d, \"method\": \"%s\", \"mode\": \"batched\", \"blocks\": %ld, \"threads\": %d, "
                "\"plan_s\": %.6g, \"forward_s\": %.6g, \"inverse_s\": %.6g, \"reps\": %d, \"rep_s\": [%s], "
                "\"roundtrip_rel_err\": %.3g}\n",
                n, method, static_cast<long>(blocks), threads, plan_s, fs, is, reps, rep_list.c_str(), err / scale);
    return 0;
}
