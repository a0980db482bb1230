// Register-resident mixed-radix DFT codelets, generated at compile time (sm_100a).
//
// RDft<N, INV>::run(v) transforms N complex values held in registers (natural order in
// and out). Composite N recurse either as a prime-factor (Good-Thomas) split N = R*M with
// gcd(R, M) = 1 (pure register permutation, no twiddles) or as a Cooley-Tukey decimation in
// time (M-point sub-DFTs on the R strided subsets, inter-factor twiddles, R-point
// butterflies). Twiddles are constexpr (evaluated in double at compile time, rounded to
// fp32) and fold into FMUL/FFMA immediates; multiples of pi/4 become adds/swaps. The
// codelets have no memory traffic and no transcendental calls.
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

// a * exp(sign*2*pi*i*Q/N) with the trivial angles (multiples of pi/4) special-cased
template <int N, int Q, bool INV>
__host__ __device__ __forceinline__ float2 twmul(float2 a) {
    constexpr int q8 = (8 * Q) % N == 0 ? ((8 * Q) / N) % 8 : -1;  // octant index if exact
    constexpr float h = 0.70710678118654752440f;
    if constexpr (q8 < 0) {
        return cmul(a, ctw<N, Q, INV>());
    } else {
        // angle = sign * q8 * pi/4
        constexpr int o = INV ? q8 : (8 - q8) % 8;
        if constexpr (o == 0) return a;
        else if constexpr (o == 2) return make_float2(-a.y, a.x);    // * i
        else if constexpr (o == 4) return make_float2(-a.x, -a.y);   // * -1
        else if constexpr (o == 6) return make_float2(a.y, -a.x);    // * -i
        else if constexpr (o == 1) return make_float2(h * (a.x - a.y), h * (a.x + a.y));
        else if constexpr (o == 3) return make_float2(-h * (a.x + a.y), h * (a.x - a.y));
        else if constexpr (o == 5) return make_float2(h * (a.y - a.x), -h * (a.x + a.y));
        else return make_float2(h * (a.x + a.y), h * (a.y - a.x));   // o == 7
    }
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

constexpr int cx_gcd(int a, int b) { return b == 0 ? a : cx_gcd(b, a % b); }
// modular inverse of a mod m (gcd(a, m) == 1), by search (compile time, small m)
constexpr int cx_inv_mod(int a, int m) {
    for (int x = 1; x < m; ++x)
        if ((a * x) % m == 1) return x;
    return m == 1 ? 0 : -1;
}
// Good-Thomas split N = R * M with gcd(R, M) == 1 and both > 1 (prefer the smallest R)
constexpr int pick_coprime(int n) {
    for (int r = 2; r * r <= n; ++r)
        if (n % r == 0 && cx_gcd(r, n / r) == 1) return r;
    return 0;
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

// Prime-factor (Good-Thomas) codelet for N = R * M, gcd(R, M) == 1: input index
// n = (M*r + R*m) mod N, output index k = (kr*M*(M^-1 mod R) + km*R*(R^-1 mod M)) mod N;
// the 2-D DFT needs no twiddle multiplications (pure register permutation).
template <int N, bool INV>
struct PfaDft {
    static constexpr int R = pick_coprime(N);
    static constexpr int M = N / R;
    static constexpr int CR = (M * cx_inv_mod(M % R, R)) % N;  // = 1 mod R, 0 mod M
    static constexpr int CM = (R * cx_inv_mod(R % M, M)) % N;  // = 0 mod R, 1 mod M
    __host__ __device__ __forceinline__ static void run(float2* v) {
        float2 t[R][M];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int m = 0; m < M; ++m) t[r][m] = v[(M * r + R * m) % N];
#pragma unroll
        for (int r = 0; r < R; ++r) RDft<M, INV>::run(t[r]);
#pragma unroll
        for (int km = 0; km < M; ++km) {
            float2 u[R];
#pragma unroll
            for (int r = 0; r < R; ++r) u[r] = t[r][km];
            RDft<R, INV>::run(u);
#pragma unroll
            for (int kr = 0; kr < R; ++kr) v[(kr * CR + km * CM) % N] = u[kr];
        }
    }
};

template <int N, bool INV>
struct CtDft;

template <int N, bool INV>
struct RDft<N, INV, false> {
    __host__ __device__ __forceinline__ static void run(float2* v) {
        if constexpr (pick_coprime(N) != 0 && N % 8 != 0) PfaDft<N, INV>::run(v);
        else CtDft<N, INV>::run(v);
    }
};

// Cooley-Tukey (decimation in time) codelet N = R * M with constexpr twiddles
template <int N, bool INV>
struct CtDft {
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
                t[r][k] = twmul<N, r * k, INV>(t[r][k]);
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
