// ustfwi drop-in (B200): the reference's fp64 spectral SETUP utilities — core/fft.hpp
// (RealFft, ComplexFft, fft_wavenumbers), grid/grid.hpp (sinc, KVectors, make_kvectors,
// largest_prime_factor) and grid/spectral.hpp (spectral_derivative, apply_isotropic_multiplier,
// fourier_shift), grid/filter.hpp (design_kaiser_lowpass, fft_convolve).
//
// These are setup / diagnostic operators whose reference contracts are fp64 statements
// (test_grid.cpp: 1e-9 .. 1e-12). They run on the host in fp64 over the library's own
// mixed-radix FFT (ustfwi_host_fft, csrc/host_fft.cpp; the reference links FFTW for them).
// The hot path — every leapfrog step of forward, adjoint and time-reversal simulations —
// never calls them: it runs on the device (SpectralEngine / WaveStepper, solver.hpp).
#pragma once

#include <complex>
#include <cstring>

#include "core.hpp"

namespace ustfwi {

enum class Stagger { none, plus, minus };

/// core/fft.hpp:75-118 — complex-to-complex transform of one shape; inverse normalised by 1/N.
class ComplexFft {
public:
    explicit ComplexFft(Dims dims) : dims_(std::move(dims)), n_(total_size(dims_)) {
        for (int d : dims_)
            if (d < 1) throw std::invalid_argument("fft dims must be positive");
    }
    std::size_t size() const { return n_; }
    void forward_inplace(std::complex<double>* data) {
        detail::check(ustfwi_host_fft(static_cast<int>(dims_.size()), dims_.data(), reinterpret_cast<double*>(data), 0, 0));
    }
    void inverse_inplace(std::complex<double>* data) {
        detail::check(ustfwi_host_fft(static_cast<int>(dims_.size()), dims_.data(), reinterpret_cast<double*>(data), 1, 1));
    }

private:
    Dims dims_;
    std::size_t n_ = 0;
};

/// core/fft.hpp:23-71 — real-to-complex pair (last axis halved to n/2+1 bins); inverse
/// normalised so inverse(forward(x)) == x. The inverse treats the half spectrum as Hermitian.
class RealFft {
public:
    explicit RealFft(Dims dims) : dims_(std::move(dims)), full_(dims_) {
        n_real_ = total_size(dims_);
        Dims half = dims_;
        half.back() = dims_.back() / 2 + 1;
        n_spec_ = total_size(half);
    }
    const Dims& dims() const { return dims_; }
    std::size_t real_size() const { return n_real_; }
    std::size_t spectrum_size() const { return n_spec_; }

    void forward(const double* in, std::complex<double>* out) {
        std::vector<std::complex<double>> buf(n_real_);
        for (std::size_t i = 0; i < n_real_; ++i) buf[i] = in[i];
        full_.forward_inplace(buf.data());
        const std::size_t nl = static_cast<std::size_t>(dims_.back()), nh = nl / 2 + 1;
        for (std::size_t r = 0; r < n_real_ / nl; ++r)
            for (std::size_t k = 0; k < nh; ++k) out[r * nh + k] = buf[r * nl + k];
    }

    void inverse(const std::complex<double>* in, double* out) {
        // rebuild the full spectrum: X[k] = conj(X[-k]) for the upper half of the last axis
        const std::size_t nl = static_cast<std::size_t>(dims_.back()), nh = nl / 2 + 1;
        const std::size_t rows = n_real_ / nl;
        std::vector<std::complex<double>> buf(n_real_);
        std::vector<std::size_t> neg(rows);  // row index of the negated leading coordinates
        {
            const int nd = static_cast<int>(dims_.size());
            Coord c(static_cast<std::size_t>(std::max(nd - 1, 0)), 0);
            for (std::size_t r = 0; r < rows; ++r) {
                std::size_t q = 0;
                for (int a = 0; a < nd - 1; ++a) {
                    const int n = dims_[static_cast<std::size_t>(a)];
                    const int ca = c[static_cast<std::size_t>(a)];
                    q = q * static_cast<std::size_t>(n) + static_cast<std::size_t>((n - ca) % n);
                }
                neg[r] = q;
                for (int a = nd - 2; a >= 0; --a) {
                    if (++c[static_cast<std::size_t>(a)] < dims_[static_cast<std::size_t>(a)]) break;
                    c[static_cast<std::size_t>(a)] = 0;
                }
            }
        }
        for (std::size_t r = 0; r < rows; ++r) {
            for (std::size_t k = 0; k < nh; ++k) buf[r * nl + k] = in[r * nh + k];
            for (std::size_t k = nh; k < nl; ++k) buf[r * nl + k] = std::conj(in[neg[r] * nh + (nl - k)]);
        }
        full_.inverse_inplace(buf.data());
        for (std::size_t i = 0; i < n_real_; ++i) out[i] = buf[i].real();
    }

private:
    Dims dims_;
    ComplexFft full_;
    std::size_t n_real_ = 0, n_spec_ = 0;
};

/// core/fft.hpp:121-130 — FFT-ordered angular wavenumbers; the Nyquist bin is negative.
inline std::vector<double> fft_wavenumbers(int n, double dx) {
    std::vector<double> k(static_cast<std::size_t>(n));
    const double dk = 2.0 * M_PI / (static_cast<double>(n) * dx);
    for (int m = 0; m < n; ++m) {
        const int signed_m = (2 * m < n) ? m : m - n;  // m == n/2 maps to -n/2
        k[static_cast<std::size_t>(m)] = dk * signed_m;
    }
    return k;
}

/// grid/grid.hpp:106-109 — sin(x)/x with the series 1 - x^2/6 near zero.
inline double sinc(double x) { return std::abs(x) < 1e-8 ? 1.0 - x * x / 6.0 : std::sin(x) / x; }

namespace detail {
/// grid/grid.hpp:55-67
inline long largest_prime_factor(long n) {
    long best = 1;
    for (long p = 2; p * p <= n; ++p)
        while (n % p == 0) {
            best = p;
            n /= p;
        }
    return n > 1 ? std::max(best, n) : best;
}

/// grid/spectral.hpp:16-31 — row-major multi-index walk
template <typename Fn>
void for_each_index(const Dims& dims, Fn&& fn) {
    Coord c(dims.size(), 0);
    const std::size_t n = total_size(dims);
    for (std::size_t idx = 0; idx < n; ++idx) {
        fn(idx, c);
        for (int a = static_cast<int>(dims.size()) - 1; a >= 0; --a) {
            if (++c[static_cast<std::size_t>(a)] < dims[static_cast<std::size_t>(a)]) break;
            c[static_cast<std::size_t>(a)] = 0;
        }
    }
}

inline std::vector<std::complex<double>> to_complex(const Field& f) {
    std::vector<std::complex<double>> s(f.size());
    for (std::size_t i = 0; i < f.size(); ++i) s[i] = f[i];
    return s;
}
inline Field real_part(const Dims& dims, const std::vector<std::complex<double>>& s) {
    Field out(dims);
    for (std::size_t i = 0; i < out.size(); ++i) out[i] = s[i].real();
    return out;
}
}  // namespace detail

/// grid/grid.hpp:113-143 — per-axis wavenumbers and kappa = sinc(c_ref dt |k| / 2) over the
/// full spectrum grid.
struct KVectors {
    std::vector<std::vector<double>> k;
    Field kappa;
    std::vector<double> dx;
};

inline KVectors make_kvectors(const Grid& g) {
    g.validate();
    KVectors kv;
    kv.dx = g.dx;
    for (std::size_t a = 0; a < g.dims.size(); ++a) kv.k.push_back(fft_wavenumbers(g.dims[a], g.dx[a]));
    kv.kappa = Field(g.dims);
    const double h = 0.5 * g.c_ref * g.dt;
    detail::for_each_index(g.dims, [&](std::size_t idx, const Coord& c) {
        double k2 = 0.0;
        for (std::size_t a = 0; a < c.size(); ++a) {
            const double ka = kv.k[a][static_cast<std::size_t>(c[a])];
            k2 += ka * ka;
        }
        kv.kappa[idx] = sinc(h * std::sqrt(k2));
    });
    return kv;
}

/// grid/spectral.hpp:36-66 — ifft(i k_a kappa e^{+-i k_a dx/2} fft(f)), real part; the
/// unstaggered operator vanishes on the Nyquist bin of the axis.
inline Field spectral_derivative(const Field& field, int axis, Stagger stagger, const KVectors& kvecs) {
    if (field.dims() != kvecs.kappa.dims()) throw std::invalid_argument("field dims do not match the k-vector grid");
    const Dims& dims = field.dims();
    const auto ua = static_cast<std::size_t>(axis);
    auto spec = detail::to_complex(field);
    ComplexFft fft(dims);
    fft.forward_inplace(spec.data());
    const double hdx = 0.5 * kvecs.dx[ua];
    detail::for_each_index(dims, [&](std::size_t idx, const Coord& c) {
        const double ka = kvecs.k[ua][static_cast<std::size_t>(c[ua])];
        std::complex<double> m(0.0, ka * kvecs.kappa[idx]);
        if (stagger == Stagger::none) {
            if (c[ua] == dims[ua] / 2) m = 0.0;
        } else {
            m *= std::polar(1.0, stagger == Stagger::plus ? ka * hdx : -ka * hdx);
        }
        spec[idx] *= m;
    });
    fft.inverse_inplace(spec.data());
    return detail::real_part(dims, spec);
}

/// grid/spectral.hpp:71-89 — multiplier m(|k|^2) per spectral index, real part.
template <typename MultFn>
Field apply_isotropic_multiplier(const Field& field, const KVectors& kvecs, MultFn&& mult) {
    const Dims& dims = field.dims();
    auto spec = detail::to_complex(field);
    ComplexFft fft(dims);
    fft.forward_inplace(spec.data());
    detail::for_each_index(dims, [&](std::size_t idx, const Coord& c) {
        double k2 = 0.0;
        for (std::size_t a = 0; a < dims.size(); ++a) {
            const double ka = kvecs.k[a][static_cast<std::size_t>(c[a])];
            k2 += ka * ka;
        }
        spec[idx] *= mult(k2);
    });
    fft.inverse_inplace(spec.data());
    return detail::real_part(dims, spec);
}

/// grid/spectral.hpp:94-112 — band-limited shift by shift_cells along axis (e^{i k s}, the
/// Nyquist bin keeps its real part).
inline Field fourier_shift(const Field& field, int axis, double shift_cells, const KVectors& kvecs) {
    const Dims& dims = field.dims();
    const auto ua = static_cast<std::size_t>(axis);
    auto spec = detail::to_complex(field);
    ComplexFft fft(dims);
    fft.forward_inplace(spec.data());
    const double s = shift_cells * kvecs.dx[ua];
    detail::for_each_index(dims, [&](std::size_t idx, const Coord& c) {
        const double ka = kvecs.k[ua][static_cast<std::size_t>(c[ua])];
        std::complex<double> m = std::polar(1.0, ka * s);
        if (c[ua] == dims[ua] / 2) m = m.real();
        spec[idx] *= m;
    });
    fft.inverse_inplace(spec.data());
    return detail::real_part(dims, spec);
}

/// grid/filter.hpp:38-66 — Kaiser-window FIR low-pass taps (odd length, unit DC gain).
inline std::vector<double> design_kaiser_lowpass(double dt, double cutoff_hz, double transition = 0.1,
                                                 double atten_db = 60.0) {
    int len = 0;
    detail::check(ustfwi_design_kaiser_lowpass(dt, cutoff_hz, transition, atten_db, nullptr, &len));
    std::vector<double> h(static_cast<std::size_t>(len));
    detail::check(ustfwi_design_kaiser_lowpass(dt, cutoff_hz, transition, atten_db, h.data(), &len));
    return h;
}

/// grid/filter.hpp:69-88 — linear convolution through a power-of-two FFT.
inline std::vector<double> fft_convolve(const std::vector<double>& a, const std::vector<double>& b) {
    if (a.empty() || b.empty()) return {};
    const std::size_t n = a.size() + b.size() - 1;
    std::size_t nfft = 1;
    while (nfft < n) nfft <<= 1;
    std::vector<std::complex<double>> fa(nfft), fb(nfft);
    for (std::size_t i = 0; i < a.size(); ++i) fa[i] = a[i];
    for (std::size_t i = 0; i < b.size(); ++i) fb[i] = b[i];
    ComplexFft fft({static_cast<int>(nfft)});
    fft.forward_inplace(fa.data());
    fft.forward_inplace(fb.data());
    for (std::size_t i = 0; i < nfft; ++i) fa[i] *= fb[i];
    fft.inverse_inplace(fa.data());
    std::vector<double> out(n);
    for (std::size_t i = 0; i < n; ++i) out[i] = fa[i].real();
    return out;
}

}  // namespace ustfwi
