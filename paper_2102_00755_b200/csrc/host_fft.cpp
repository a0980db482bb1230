// fp64 multi-dimensional complex FFT on the host, for the drop-in's fp64 setup utilities
// (the reference's core/fft.hpp ComplexFft / RealFft and the grid/spectral.hpp operators built
// on them: spectral_derivative, fourier_shift, apply_isotropic_multiplier, make_kvectors).
// The reference links FFTW for these (fft.hpp:30-42); FFTW is not in this image, so the
// library carries its own mixed-radix transform. NOT on the hot path: the device engine
// runs its own sm_100a kernels; these utilities serve setup-time calls whose reference
// tolerances (1e-11 .. 1e-14) are fp64 statements.
//
// Algorithm: recursive decimation in time over the prime factorisation (radix 4 first, then
// 2, 3, 5, ...) with a generic radix-p butterfly X[k] = sum_q s[q] W_N^(q k stride), twiddles
// W_N^i = exp(-+2 pi i / N) evaluated in long double once per plan; multi-dimensional
// transforms apply the 1-D plan along every axis (gather, transform, scatter).
#include <cmath>
#include <complex>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "../../include/ustfwi_capi.h"
#include "host_setup.hpp"

namespace {

using cplx = std::complex<double>;

struct Plan1d {
    int n = 1;
    std::vector<int> fac;  // (p, m) pairs, m = remaining length after this radix
    std::vector<cplx> tw;  // W_n^i, i < n, for the plan's direction
    std::vector<cplx> scratch;

    Plan1d(int len, bool inverse) : n(len) {
        int m = n;
        auto take = [&](int p) {
            while (m % p == 0 && m > 1) {
                m /= p;
                fac.push_back(p);
                fac.push_back(m);
            }
        };
        take(4);
        take(2);
        for (int p = 3; m > 1; p += 2) take(p);
        if (n == 1) {
            fac = {1, 1};
        }
        tw.resize(static_cast<size_t>(n));
        const long double two_pi = 6.283185307179586476925286766559005768L;
        for (int i = 0; i < n; ++i) {
            const long double a = two_pi * static_cast<long double>(i) / static_cast<long double>(n);
            const double c = static_cast<double>(std::cos(a)), s = static_cast<double>(std::sin(a));
            tw[static_cast<size_t>(i)] = inverse ? cplx(c, s) : cplx(c, -s);
        }
        int pmax = 1;
        for (size_t i = 0; i < fac.size(); i += 2) pmax = std::max(pmax, fac[i]);
        scratch.resize(static_cast<size_t>(pmax));
    }

    void butterfly(cplx* out, size_t fstride, int m, int p) {
        for (int u = 0; u < m; ++u) {
            for (int q = 0, k = u; q < p; ++q, k += m) scratch[static_cast<size_t>(q)] = out[k];
            for (int q1 = 0, k = u; q1 < p; ++q1, k += m) {
                size_t idx = 0;
                const size_t step = fstride * static_cast<size_t>(k) % static_cast<size_t>(n);
                cplx acc = scratch[0];
                for (int q = 1; q < p; ++q) {
                    idx += step;
                    if (idx >= static_cast<size_t>(n)) idx -= static_cast<size_t>(n);
                    acc += scratch[static_cast<size_t>(q)] * tw[idx];
                }
                out[k] = acc;
            }
        }
    }

    void work(cplx* out, const cplx* in, size_t fstride, const int* f) {
        const int p = f[0], m = f[1];
        cplx* const beg = out;
        if (m == 1) {
            for (int q = 0; q < p; ++q) out[q] = in[static_cast<size_t>(q) * fstride];
        } else {
            for (int q = 0; q < p; ++q) work(out + static_cast<size_t>(q) * m, in + static_cast<size_t>(q) * fstride,
                                             fstride * static_cast<size_t>(p), f + 2);
        }
        if (p > 1) butterfly(beg, fstride, m, p);
    }

    // out = DFT(in), contiguous, out != in
    void run(const cplx* in, cplx* out) {
        if (n == 1) {
            out[0] = in[0];
            return;
        }
        work(out, in, 1, fac.data());
    }
};

void fft_nd(int ndim, const int* dims, cplx* data, bool inverse) {
    size_t total = 1;
    for (int a = 0; a < ndim; ++a) {
        if (dims[a] < 1) ustfwi_host::fail(USTFWI_ERR_INVALID, "fft dims must be positive");
        total *= static_cast<size_t>(dims[a]);
    }
    for (int a = 0; a < ndim; ++a) {
        const int n = dims[a];
        if (n == 1) continue;
        size_t post = 1;
        for (int b = a + 1; b < ndim; ++b) post *= static_cast<size_t>(dims[b]);
        const size_t pre = total / (post * static_cast<size_t>(n));
        Plan1d plan(n, inverse);
        std::vector<cplx> line(static_cast<size_t>(n)), res(static_cast<size_t>(n));
        for (size_t i = 0; i < pre; ++i)
            for (size_t j = 0; j < post; ++j) {
                cplx* base = data + i * static_cast<size_t>(n) * post + j;
                for (int k = 0; k < n; ++k) line[static_cast<size_t>(k)] = base[static_cast<size_t>(k) * post];
                plan.run(line.data(), res.data());
                for (int k = 0; k < n; ++k) base[static_cast<size_t>(k) * post] = res[static_cast<size_t>(k)];
            }
    }
}

}  // namespace

extern "C" int ustfwi_host_fft(int ndim, const int* dims, double* data, int inverse, int normalize) {
    try {
        if (ndim < 1 || ndim > 8 || !dims || !data) ustfwi_host::fail(USTFWI_ERR_INVALID, "bad fft arguments");
        auto* c = reinterpret_cast<cplx*>(data);
        fft_nd(ndim, dims, c, inverse != 0);
        if (inverse && normalize) {
            size_t total = 1;
            for (int a = 0; a < ndim; ++a) total *= static_cast<size_t>(dims[a]);
            const double s = 1.0 / static_cast<double>(total);
            for (size_t i = 0; i < total; ++i) c[i] *= s;
        }
        return USTFWI_OK;
    } catch (const ustfwi_host::Error& e) {
        ustfwi_host::set_last_error(e.msg);
        return e.code;
    } catch (const std::exception& e) {
        ustfwi_host::set_last_error(e.what());
        return USTFWI_ERR_INVALID;
    }
}
