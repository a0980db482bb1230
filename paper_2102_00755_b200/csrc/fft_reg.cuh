// Register-resident mixed-radix DFT codelets, generated at compile time (sm_100a).
//
// RDft<N, INV>::run(v) transforms N complex values held in registers (natural order in
// and out). Composite N recurse as N = R * M (decimation in time): M-point sub-DFTs on the
// R strided subsets, inter-factor twiddles, then R-point butterflies. All twiddles are
// constexpr (evaluated in double at compile time, rounded to fp32) and fold into FMUL/
// FFMA immediates, so the codelets have no memory traffic and no transcendental calls.
#pragma once

#include <utility>

#include "fft_smem.cuh"

namespace ustfwi_dev {

// ---- constexpr trigonometry (double, compile time) --------------------------------------
constexpr double kPi = 3.14159265358979323846264338327950288;

constexpr double cx_sin_small(double x) {
    double x2 = x * x, term = x, sum = x;
    for (int k = 1; k < 14; ++k) {
        term *= -x2 / ((2.0 * k) * (2.0 * k + 1.0));
        sum += term;
    }
    return sum;
}
constexpr double cx_cos_small(double x) {
    double x2 = x * x, term = 1.0, sum = 1.0;
    for (int k = 1; k < 14; ++k) {
        term *= -x2 / ((2.0 * k - 1.0) * (2.0 * k));
        sum += term;
    }
    return sum;
}
// cos(2*pi*q/n), reduced exactly on integers to one octant
constexpr double cx_cos2pi(long q, long n) {
    q %= n;
    if (q < 0) q += n;
    const long e = 8 * q;
    const long oct = e / n;
    const double a = static_cast<double>(e - oct * n) / static_cast<double>(n) * kPi / 4.0;
    const double c = cx_cos_small(a), s = cx_sin_small(a);
    const double cb = cx_cos_small(kPi / 4.0 - a), sb = cx_sin_small(kPi / 4.0 - a);
    switch (oct) {
        case 0: return c;
        case 1: return sb;
        case 2: return -s;
        case 3: return -cb;
        case 4: return -c;
        case 5: return -sb;
        case 6: return s;
        default: return cb;
    }
}
constexpr double cx_sin2pi(long q, long n) { return cx_cos2pi(4 * q - n, 4 * n); }

// exp(sign * 2*pi*i*Q/N), sign = -1 forward, +1 inverse
template <int N, int Q, bool INV>
__host__ __device__ __forceinline__ float2 ctw() {
    constexpr float c = static_cast<float>(cx_cos2pi(Q, N));
    constexpr float s = static_cast<float>(INV ? cx_sin2pi(Q, N) : -cx_sin2pi(Q, N));
    return make_float2(c, s);
}

template <int B, int E, class F>
__host__ __device__ __forceinline__ void static_for(F&& f) {
    if constexpr (B < E) {
        f(std::integral_constant<int, B>{});
        static_for<B + 1, E>(f);
    }
}

// ---- radix choice -----------------------------------------------------------------------
constexpr bool is_base(int n) { return n == 1 || n == 2 || n == 3 || n == 4 || n == 5 || n == 7 || n == 8 || n == 16; }
constexpr int pick_radix(int n) {
    if (n % 16 == 0 && n / 16 > 1) return 16;
    if (n % 8 == 0 && n / 8 > 1) return 8;
    if (n % 4 == 0 && n / 4 > 1) return 4;
    for (int f = 2; f <= n; ++f)
        if (n % f == 0) return f;
    return n;
}

template <int N, bool INV, bool BASE = is_base(N)>
struct RDft;

template <bool INV>
struct RDft<1, INV, true> {
    __host__ __device__ __forceinline__ static void run(float2*) {}
};

template <int N, bool INV>
struct RDft<N, INV, true> {
    __host__ __device__ __forceinline__ static void run(float2* v) { Dft<N, INV>::run(v); }
};

template <int N, bool INV>
struct RDft<N, INV, false> {
    static constexpr int R = pick_radix(N);
    static constexpr int M = N / R;
    static_assert(R > 1 && M > 1, "unsupported length");
    __host__ __device__ __forceinline__ static void run(float2* v) {
        float2 t[R][M];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int m = 0; m < M; ++m) t[r][m] = v[r + R * m];
#pragma unroll
        for (int r = 0; r < R; ++r) RDft<M, INV>::run(t[r]);
        static_for<1, R>([&](auto rr) {
            constexpr int r = decltype(rr)::value;
            static_for<1, M>([&](auto kk) {
                constexpr int k = decltype(kk)::value;
                t[r][k] = cmul(t[r][k], ctw<N, r * k, INV>());
            });
        });
#pragma unroll
        for (int k = 0; k < M; ++k) {
            float2 u[R];
#pragma unroll
            for (int r = 0; r < R; ++r) u[r] = t[r][k];
            RDft<R, INV>::run(u);
#pragma unroll
            for (int q = 0; q < R; ++q) v[k + M * q] = u[q];
        }
    }
};

}  // namespace ustfwi_dev
