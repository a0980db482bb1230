// Host-side setup of the engine: grid construction, PML profiles, wavenumbers, shell
// erosion, source pulse synthesis and the encoding RNG. These are the non-hot-path
// pieces of the reference API the hot path depends on; they are restated here (fp64,
// same formulas as the cited reference lines) so the product has no dependency on the
// reference or on FFTW.
#include "host_setup.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>

namespace ustfwi_host {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }
[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }

std::string dims_str(const int* dims, int ndim) {
    std::string s = "(";
    for (int a = 0; a < ndim; ++a) {
        if (a) s += ", ";
        s += std::to_string(dims[a]);
    }
    return s + ")";
}

void validate_grid(const ustfwi_grid& g) {
    if (g.ndim < 1 || g.ndim > 3) fail(USTFWI_ERR_INVALID, "grid must be 1-, 2- or 3-dimensional");
    for (int a = 0; a < g.ndim; ++a) {
        if (g.dims[a] < 4 || (g.dims[a] & 1))
            fail(USTFWI_ERR_INVALID, "grid dims must be even and >= 4, got " + dims_str(g.dims, g.ndim));
        if (!(g.dx[a] > 0.0)) fail(USTFWI_ERR_INVALID, "grid spacing must be positive");
        if (g.pml_size[a] < 0 || 2 * g.pml_size[a] >= g.dims[a])
            fail(USTFWI_ERR_INVALID, "pml thickness does not fit the grid");
    }
    if (!(g.dt > 0.0)) fail(USTFWI_ERR_INVALID, "time step must be positive");
    if (g.nt < 2) fail(USTFWI_ERR_INVALID, "need at least two time samples");
    if (!(g.c_ref > 0.0)) fail(USTFWI_ERR_INVALID, "reference sound speed must be positive");
}

long largest_prime_factor(long n) {
    long best = 1;
    for (long f = 2; f * f <= n; ++f)
        for (; n % f == 0; n /= f) best = f;
    return n > 1 ? n : best;
}

std::vector<int> choose_pml_size(const std::vector<int>& interior) {
    std::vector<int> out;
    for (int n : interior) {
        if (n < 4) fail(USTFWI_ERR_INVALID, "interior dims must be >= 4");
        // thinnest layer in [10, 20] whose padded size has the smallest largest prime
        int t_best = 10;
        long p_best = largest_prime_factor(n + 20L);
        for (int t = 11; t <= 20; ++t) {
            const long p = largest_prime_factor(n + 2L * t);
            if (p < p_best) {
                p_best = p;
                t_best = t;
            }
        }
        out.push_back(t_best);
    }
    return out;
}

ustfwi_grid make_grid(const std::vector<int>& interior, double dx, double c_max, double duration,
                      double cfl) {
    ustfwi_grid g;
    std::memset(&g, 0, sizeof(g));
    g.ndim = static_cast<int>(interior.size());
    if (g.ndim < 1 || g.ndim > 3) fail(USTFWI_ERR_INVALID, "grid must be 1-, 2- or 3-dimensional");
    const auto pml = choose_pml_size(interior);
    for (int a = 0; a < g.ndim; ++a) {
        g.pml_size[a] = pml[static_cast<size_t>(a)];
        g.dims[a] = interior[static_cast<size_t>(a)] + 2 * g.pml_size[a];
        g.dx[a] = dx;
    }
    g.c_ref = c_max;
    g.dt = cfl * dx / c_max;
    g.nt = static_cast<int>(std::ceil(duration / g.dt)) + 1;
    validate_grid(g);
    return g;
}

std::vector<double> wavenumbers(int n, double dx) {
    std::vector<double> k(static_cast<size_t>(n));
    const double dk = 2.0 * M_PI / (static_cast<double>(n) * dx);
    for (int m = 0; m < n; ++m) {
        // bins 0..n/2-1 positive, n/2..n-1 negative; the Nyquist bin n/2 is -n/2, which
        // also makes the single bin of a length-1 (padded singleton) axis zero
        const int signed_m = (m < n / 2) ? m : (m == n / 2 ? -(n / 2) : m - n);
        k[static_cast<size_t>(m)] = dk * signed_m;
    }
    return k;
}

double sinc(double x) { return std::abs(x) < 1e-8 ? 1.0 - x * x / 6.0 : std::sin(x) / x; }

void pml_profiles(const ustfwi_grid& g, int axis, double alpha, std::vector<double>& regular,
                  std::vector<double>& staggered) {
    const int n = g.dims[axis];
    const int layer = g.pml_size[axis];
    const double edge = static_cast<double>(layer - 1);  // ramp reaches zero here
    auto mult = [&](double u) {
        if (layer < 2) return 1.0;
        const double from_left = edge - u;
        const double from_right = edge - (static_cast<double>(n - 1) - u);
        double ramp = 0.0;
        if (from_left > 0.0) ramp = from_left / edge;
        if (from_right > 0.0) ramp = std::max(ramp, from_right / edge);
        const double sigma = alpha * (g.c_ref / g.dx[axis]) * std::pow(ramp, 4);
        return std::exp(-0.5 * sigma * g.dt);
    };
    regular.resize(static_cast<size_t>(n));
    staggered.resize(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
        regular[static_cast<size_t>(i)] = mult(static_cast<double>(i));
        staggered[static_cast<size_t>(i)] = mult(i + 0.5);
    }
}

std::vector<uint8_t> erode(const std::vector<uint8_t>& mask, const std::vector<int>& dims) {
    const int nd = static_cast<int>(dims.size());
    std::vector<size_t> stride(static_cast<size_t>(nd), 1);
    for (int a = nd - 2; a >= 0; --a) stride[static_cast<size_t>(a)] = stride[static_cast<size_t>(a) + 1] * dims[static_cast<size_t>(a) + 1];
    std::vector<uint8_t> out(mask.size(), 0);
    std::vector<int> c(static_cast<size_t>(nd), 0);
    for (size_t i = 0; i < mask.size(); ++i) {
        if (mask[i]) {
            bool interior = true;
            for (int a = 0; a < nd && interior; ++a) {
                const int ca = c[static_cast<size_t>(a)];
                if (ca == 0 || ca == dims[static_cast<size_t>(a)] - 1) interior = false;
                else if (!mask[i - stride[static_cast<size_t>(a)]] || !mask[i + stride[static_cast<size_t>(a)]])
                    interior = false;
            }
            out[i] = interior ? 1 : 0;
        }
        for (int a = nd - 1; a >= 0; --a) {
            if (++c[static_cast<size_t>(a)] < dims[static_cast<size_t>(a)]) break;
            c[static_cast<size_t>(a)] = 0;
        }
    }
    return out;
}

std::vector<size_t> shell_indices(const std::vector<uint8_t>& mask, const std::vector<int>& dims,
                                  int thickness) {
    if (thickness < 1) fail(USTFWI_ERR_INVALID, "shell thickness must be >= 1");
    std::vector<uint8_t> core = mask;
    for (int t = 0; t < thickness; ++t) core = erode(core, dims);
    const bool core_empty = std::none_of(core.begin(), core.end(), [](uint8_t v) { return v != 0; });
    if (core_empty && thickness > 1) fail(USTFWI_ERR_INVALID, "shell thickness exceeds the mask extent");
    std::vector<size_t> out;
    for (size_t i = 0; i < mask.size(); ++i)
        if (mask[i] && !core[i]) out.push_back(i);
    return out;
}

// ---- source pulse (simulate.hpp:124-148 with the Kaiser design of filter.hpp:14-101) ----
namespace {

double bessel_i0(double x) {
    const double q = 0.25 * x * x;
    double term = 1.0, sum = 1.0;
    for (int k = 1; k < 64; ++k) {
        term *= q / (static_cast<double>(k) * k);
        sum += term;
        if (term < 1e-18 * sum) break;
    }
    return sum;
}

double kaiser_beta(double atten_db) {
    if (atten_db > 50.0) return 0.1102 * (atten_db - 8.7);
    if (atten_db >= 21.0) return 0.5842 * std::pow(atten_db - 21.0, 0.4) + 0.07886 * (atten_db - 21.0);
    return 0.0;
}

std::vector<double> kaiser_lowpass(double dt, double cutoff, double transition, double atten_db) {
    if (!(cutoff > 0.0) || cutoff > 0.5 / dt) fail(USTFWI_ERR_INVALID, "cutoff must lie in (0, Nyquist]");
    const double width = transition * cutoff;
    const double dw = 2.0 * M_PI * width * dt;
    const int half = std::max(4, static_cast<int>(std::ceil((atten_db - 7.95) / (2.285 * dw) / 2.0)));
    const double beta = kaiser_beta(atten_db);
    const double norm = bessel_i0(beta);
    const double wc = 2.0 * M_PI * (cutoff + 0.5 * width) * dt;
    std::vector<double> h(static_cast<size_t>(2 * half + 1));
    double dc = 0.0;
    for (int i = -half; i <= half; ++i) {
        const double m = static_cast<double>(i);
        const double ideal = (i == 0) ? wc / M_PI : std::sin(wc * m) / (M_PI * m);
        const double r = m / half;
        const double win = bessel_i0(beta * std::sqrt(std::max(0.0, 1.0 - r * r))) / norm;
        h[static_cast<size_t>(i + half)] = ideal * win;
        dc += ideal * win;
    }
    for (double& v : h) v /= dc;
    return h;
}

}  // namespace

std::vector<double> synth_source_pulse(const ustfwi_grid& g, double frac, double c0_min) {
    if (!(frac > 0.0) || frac > 1.0) fail(USTFWI_ERR_INVALID, "frequency fraction must lie in (0, 1]");
    double min_dx = g.dx[0];
    for (int a = 1; a < g.ndim; ++a) min_dx = std::min(min_dx, g.dx[a]);
    const double cutoff = frac * c0_min / (2.0 * min_dx);
    const auto h = kaiser_lowpass(g.dt, cutoff, 0.1, 60.0);
    const int half = static_cast<int>(h.size() / 2);
    // zero-phase FIR of a centred impulse = the taps themselves, embedded in 4*half+1
    // samples (the impulse sits at 2*half; out-of-range taps are zero)
    const int n = 4 * half + 1;
    std::vector<double> pulse(static_cast<size_t>(n), 0.0);
    for (int i = 0; i < n; ++i) {
        const int k = i - 2 * half + half;  // tap index for output i
        if (k >= 0 && k < static_cast<int>(h.size())) pulse[static_cast<size_t>(i)] = h[static_cast<size_t>(k)];
    }
    double peak = 0.0;
    for (double v : pulse) peak = std::max(peak, std::abs(v));
    size_t first = 0, last = pulse.size() - 1;
    while (first < pulse.size() && std::abs(pulse[first]) < 1e-6 * peak) ++first;
    while (last > first && std::abs(pulse[last]) < 1e-6 * peak) --last;
    std::vector<double> out(pulse.begin() + static_cast<long>(first), pulse.begin() + static_cast<long>(last) + 1);
    for (double& v : out) v /= peak;
    if (out.size() > static_cast<size_t>(g.nt)) out.resize(static_cast<size_t>(g.nt));
    return out;
}

uint64_t stream_word(uint64_t master_seed, uint64_t iteration, uint64_t index, uint64_t counter) {
    auto mix = [](uint64_t z) {
        z += 0x9E3779B97F4A7C15ULL;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    };
    uint64_t k = mix(master_seed);
    k = mix(k ^ iteration);
    k = mix(k ^ index);
    return mix(k ^ counter);
}

}  // namespace ustfwi_host

// =====================================================================================
// C ABI: host setup
// =====================================================================================
using namespace ustfwi_host;

template <class Fn>
static int guarded(Fn&& fn) {
    try {
        fn();
        return USTFWI_OK;
    } catch (const Error& e) {
        set_last_error(e.msg);
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return USTFWI_ERR_OOM;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return USTFWI_ERR_INVALID;
    }
}

extern "C" {

const char* ustfwi_last_error(void) { return g_last_error.c_str(); }
const char* ustfwi_version(void) { return "ustfwi-b200 0.1 (sm_100a)"; }

int ustfwi_grid_validate(const ustfwi_grid* grid) {
    return guarded([&] {
        if (!grid) fail(USTFWI_ERR_INVALID, "null grid");
        validate_grid(*grid);
    });
}

int ustfwi_choose_pml_size(int ndim, const int* interior, int* pml_out) {
    return guarded([&] {
        const auto t = choose_pml_size(std::vector<int>(interior, interior + ndim));
        std::copy(t.begin(), t.end(), pml_out);
    });
}

int ustfwi_make_grid(int ndim, const int* interior, double dx, double c_max, double duration, double cfl,
                     ustfwi_grid* out) {
    return guarded([&] { *out = make_grid(std::vector<int>(interior, interior + ndim), dx, c_max, duration, cfl); });
}

int ustfwi_make_pml(const ustfwi_grid* grid, double alpha, double* regular, double* staggered) {
    return guarded([&] {
        validate_grid(*grid);
        size_t off = 0;
        for (int a = 0; a < grid->ndim; ++a) {
            std::vector<double> r, s;
            pml_profiles(*grid, a, alpha, r, s);
            std::copy(r.begin(), r.end(), regular + off);
            std::copy(s.begin(), s.end(), staggered + off);
            off += r.size();
        }
    });
}

int ustfwi_shell_indices(int ndim, const int* dims, const uint8_t* mask, int thickness, size_t* out,
                         size_t* count) {
    return guarded([&] {
        std::vector<int> d(dims, dims + ndim);
        size_t n = 1;
        for (int v : d) n *= static_cast<size_t>(v);
        const auto idx = shell_indices(std::vector<uint8_t>(mask, mask + n), d, thickness);
        if (out) std::copy(idx.begin(), idx.begin() + static_cast<long>(std::min(idx.size(), *count)), out);
        *count = idx.size();
    });
}

int ustfwi_ball_mask(int ndim, const int* dims, const double* center, double radius_points, uint8_t* out) {
    return guarded([&] {
        size_t n = 1;
        for (int a = 0; a < ndim; ++a) n *= static_cast<size_t>(dims[a]);
        std::vector<int> c(static_cast<size_t>(ndim), 0);
        const double r2max = radius_points * radius_points;
        for (size_t i = 0; i < n; ++i) {
            double r2 = 0.0;
            for (int a = 0; a < ndim; ++a) {
                const double d = c[static_cast<size_t>(a)] - center[a];
                r2 += d * d;
            }
            out[i] = r2 <= r2max ? 1 : 0;
            for (int a = ndim - 1; a >= 0; --a) {
                if (++c[static_cast<size_t>(a)] < dims[a]) break;
                c[static_cast<size_t>(a)] = 0;
            }
        }
    });
}

int ustfwi_synth_source_pulse(const ustfwi_grid* grid, double frac, double c0_min, double* out, int* len) {
    return guarded([&] {
        const auto p = synth_source_pulse(*grid, frac, c0_min);
        if (out) std::copy(p.begin(), p.begin() + std::min<long>(static_cast<long>(p.size()), *len), out);
        *len = static_cast<int>(p.size());
    });
}

int ustfwi_design_kaiser_lowpass(double dt, double cutoff_hz, double transition, double atten_db, double* out,
                                 int* len) {
    return guarded([&] {
        if (!len) fail(USTFWI_ERR_INVALID, "null length");
        const auto h = kaiser_lowpass(dt, cutoff_hz, transition, atten_db);
        if (out) std::copy(h.begin(), h.begin() + std::min<long>(static_cast<long>(h.size()), *len), out);
        *len = static_cast<int>(h.size());
    });
}

int ustfwi_draw_realization(size_t n_src, double tau, double dt, uint64_t master_seed, uint64_t iteration,
                            uint64_t index, int8_t* weights, int32_t* delay_steps, double* delays_unit) {
    return guarded([&] {
        if (tau < 0.0) fail(USTFWI_ERR_INVALID, "tau must be non-negative");
        if (!(dt > 0.0)) fail(USTFWI_ERR_INVALID, "dt must be positive");
        for (size_t i = 0; i < n_src; ++i) {
            const uint64_t hw = stream_word(master_seed, iteration, index, 2 * i);
            const uint64_t hd = stream_word(master_seed, iteration, index, 2 * i + 1);
            const double d = static_cast<double>(hd >> 11) * (1.0 / 9007199254740992.0);  // [0,1)
            if (weights) weights[i] = (hw >> 63) ? int8_t{1} : int8_t{-1};
            if (delays_unit) delays_unit[i] = d;
            if (delay_steps) delay_steps[i] = static_cast<int32_t>(std::llround(d * tau / dt));
        }
    });
}

}  // extern "C"
