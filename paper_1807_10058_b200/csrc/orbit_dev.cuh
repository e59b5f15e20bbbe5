// Device helpers shared by the n = 16 orbit-FFT kernels (orbit16.cu, orbit_pat.cu):
// element load / store by I/O mode, cp.async of 4 / 8 / 16 bytes, and the
// in-register radix-2 line FFT with compile-time twiddles.
#pragma once

#include "device.cuh"
#include "orbit_fft.hpp"

namespace fcct {
namespace odev {

using namespace dev;

__host__ __device__ constexpr int eb_of(int m) { return m == OF_C128 ? 16 : (m == OF_R32 ? 4 : 8); }

template <int M>
__device__ __forceinline__ void ld_el(const char* base, int idx, double& re, double& im) {
    if constexpr (M == OF_C128) {
        const double2 v = *reinterpret_cast<const double2*>(base + static_cast<size_t>(idx) * 16);
        re = v.x;
        im = v.y;
    } else if constexpr (M == OF_C64) {
        const float2 v = *reinterpret_cast<const float2*>(base + static_cast<size_t>(idx) * 8);
        re = v.x;
        im = v.y;
    } else if constexpr (M == OF_R64) {
        re = *reinterpret_cast<const double*>(base + static_cast<size_t>(idx) * 8);
        im = 0.0;
    } else {
        re = *reinterpret_cast<const float*>(base + static_cast<size_t>(idx) * 4);
        im = 0.0;
    }
}

template <int M>
__device__ __forceinline__ void st_el(char* base, int idx, double re, double im) {
    if constexpr (M == OF_C128) {
        *reinterpret_cast<double2*>(base + static_cast<size_t>(idx) * 16) = make_double2(re, im);
    } else if constexpr (M == OF_C64) {
        *reinterpret_cast<float2*>(base + static_cast<size_t>(idx) * 8) =
            make_float2(static_cast<float>(re), static_cast<float>(im));
    } else if constexpr (M == OF_R64) {
        *reinterpret_cast<double*>(base + static_cast<size_t>(idx) * 8) = re;
    } else {
        *reinterpret_cast<float*>(base + static_cast<size_t>(idx) * 4) = static_cast<float>(re);
    }
}

__device__ __forceinline__ double neg_hi16(double v) {
    return __hiloint2double(__double2hiint(v) ^ static_cast<int>(0x80000000u), __double2loint(v));
}

// cp.async of 4, 8 or 16 bytes with zero fill when !valid
template <int BYTES>
__device__ __forceinline__ void cp_async_n(void* dst, const void* src, bool valid) {
    const int sz = valid ? BYTES : 0;
    if constexpr (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(sz) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(smem_u32(dst)), "l"(src), "n"(BYTES), "r"(sz)
                     : "memory");
}

__host__ __device__ constexpr double c16(int e) {
    switch (e & 15) {
        case 0: return 1.0;
        case 1: return 0.92387953251128675613;
        case 2: return 0.70710678118654752440;
        case 3: return 0.38268343236508977173;
        case 4: return 0.0;
        case 5: return -0.38268343236508977173;
        case 6: return -0.70710678118654752440;
        case 7: return -0.92387953251128675613;
        case 8: return -1.0;
        case 9: return -0.92387953251128675613;
        case 10: return -0.70710678118654752440;
        case 11: return -0.38268343236508977173;
        case 12: return 0.0;
        case 13: return 0.38268343236508977173;
        case 14: return 0.70710678118654752440;
        default: return 0.92387953251128675613;
    }
}
__host__ __device__ constexpr int brev(int q, int nn) {
    int r = 0;
    for (int b = 1; b < nn; b <<= 1) {
        r = (r << 1) | (q & 1);
        q >>= 1;
    }
    return r;
}
template <int NN, int SIGN>
__device__ __forceinline__ double2 twid(double2 d, int e) {
    if (e == 0) return d;
    if (4 * e == NN) return SIGN > 0 ? make_double2(-d.y, d.x) : make_double2(d.y, -d.x);
    const double c = c16(e * (16 / NN)), s = SIGN * c16(e * (16 / NN) - 4);
    return make_double2(fma(d.x, c, -d.y * s), fma(d.x, s, d.y * c));
}
template <int NN, int SIGN>
__device__ __forceinline__ void fft_line16(double2 (&v)[NN]) {
#pragma unroll
    for (int half = NN / 2; half >= 1; half >>= 1) {
#pragma unroll
        for (int st = 0; st < NN; st += 2 * half) {
#pragma unroll
            for (int j = 0; j < half; ++j) {
                const double2 a = v[st + j], b = v[st + j + half];
                v[st + j] = make_double2(a.x + b.x, a.y + b.y);
                v[st + j + half] = twid<NN, SIGN>(make_double2(a.x - b.x, a.y - b.y), j * (NN / (2 * half)));
            }
        }
    }
    double2 t[NN];
#pragma unroll
    for (int q = 0; q < NN; ++q) t[q] = v[brev(q, NN)];
#pragma unroll
    for (int q = 0; q < NN; ++q) v[q] = t[q];
}

}  // namespace odev
}  // namespace fcct
