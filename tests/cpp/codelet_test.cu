// Host-side check of the register DFT codelets (fft_reg.cuh) against a direct fp64 DFT.
#include <cmath>
#include <complex>
#include <cstdio>
#include <random>

#include "../../paper_2102_00755_b200/csrc/fft_reg.cuh"

using namespace ustfwi_dev;

template <int N, bool INV>
double check() {
    std::mt19937 rng(N * 7 + INV);
    std::normal_distribution<double> d;
    float2 v[N];
    std::complex<double> x[N];
    for (int i = 0; i < N; ++i) {
        x[i] = {d(rng), d(rng)};
        v[i] = make_float2(static_cast<float>(x[i].real()), static_cast<float>(x[i].imag()));
    }
    RDft<N, INV>::run(v);
    double err = 0, nrm = 0;
    const double s = INV ? 1.0 : -1.0;
    for (int k = 0; k < N; ++k) {
        std::complex<double> acc = 0;
        for (int n = 0; n < N; ++n) acc += x[n] * std::polar(1.0, s * 2 * M_PI * ((long)n * k % N) / N);
        err = std::max(err, std::abs(acc - std::complex<double>(v[k].x, v[k].y)));
        nrm = std::max(nrm, std::abs(acc));
    }
    return err / nrm;
}

#define T(N)                                                                                   \
    {                                                                                          \
        double a = check<N, false>(), b = check<N, true>();                                    \
        std::printf("N=%4d fwd %.2e inv %.2e %s\n", N, a, b, (a < 1e-6 && b < 1e-6) ? "ok" : "FAIL"); \
        bad |= !(a < 1e-6 && b < 1e-6);                                                        \
    }

int main() {
    bool bad = false;
    T(2) T(3) T(4) T(5) T(6) T(7) T(8) T(9) T(10) T(12) T(15) T(16) T(18) T(20) T(24) T(30) T(32) T(36) T(48)
    T(60) T(64) T(72) T(96)
    return bad ? 1 : 0;
}
