// Host side of the large-n orbit-FFT executor (orbit_big.hpp): the orbit blocks
// of S_n(p) / S_n(p)^{-1} as column-major coefficient blocks, one row per
// natural position.
#include <cmath>

#include "orbit_big.hpp"
#include "plan.hpp"

namespace fcct {

bool compile_orbit_big(int n, const Params& p, bool inverse, OrbitBigHost& h) {
    if (n != 32 && n != 64) return false;
    const int N = static_cast<int>(cube(n));
    OrbitBlocks ob = orbit_blocks(n, p);
    if (!(ob.worst_condition <= 1e12))
        throw FcctError(ST_ILL_CONDITIONED, "orbit-FFT plan: orbit block condition exceeds 1e12");
    const Orbits& orb = *ob.orb;
    h = OrbitBigHost{};
    h.n = n;
    h.N = N;
    h.dir = inverse ? 1 : 0;
    const int norb = static_cast<int>(orb.members.size());
    h.orbit_off.resize(norb + 1);
    h.coef_off.resize(norb);
    h.row_orbit.resize(N);
    h.row_index.resize(N);
    h.members.resize(N);
    int64_t slots = 0, coefs = 0;
    for (int o = 0; o < norb; ++o) {
        const int s = static_cast<int>(orb.members[o].size());
        h.orbit_off[o] = static_cast<int32_t>(slots);
        h.coef_off[o] = coefs;
        for (int m = 0; m < s; ++m) {
            h.members[slots + m] = orb.members[o][m];
            h.row_orbit[slots + m] = o;
            h.row_index[slots + m] = m;
        }
        slots += s;
        coefs += static_cast<int64_t>(s) * s;
    }
    h.orbit_off[norb] = static_cast<int32_t>(slots);
    h.coef.resize(2 * static_cast<size_t>(coefs));
    const long double scale = inverse ? 1.0L / N : 1.0L;
    for (int o = 0; o < norb; ++o) {
        const int s = static_cast<int>(orb.members[o].size());
        const std::vector<cld>& M = inverse ? ob.Sinv[o] : ob.S[o];  // [row][col]
        for (int r = 0; r < s; ++r)
            for (int c = 0; c < s; ++c) {
                const cld v = M[static_cast<size_t>(r) * s + c] * scale;
                const size_t e = static_cast<size_t>(h.coef_off[o] + static_cast<int64_t>(c) * s + r);
                h.coef[2 * e] = static_cast<double>(v.real());
                h.coef[2 * e + 1] = static_cast<double>(v.imag());
            }
    }
    return true;
}

double OrbitBigHost::exec_flops() const {
    // 8 flops per complex MAC of the orbit blocks, plus the radix-2 lines
    const double cmacs = static_cast<double>(coef.size() / 2);
    int lg = 0;
    while ((1 << lg) < n) ++lg;
    double twiddles = 0;
    for (int half = n / 2; half >= 1; half /= 2)
        for (int j = 0; j < half; ++j) {
            const int e = j * (n / (2 * half));
            if (e != 0 && 4 * e != n) twiddles += n / (2 * half);
        }
    return 8.0 * cmacs + 3.0 * n * n * ((n / 2.0) * lg * 4.0 + 6.0 * twiddles);
}

}  // namespace fcct
