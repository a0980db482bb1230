// Drop-in for the reference's grid/spectral.hpp resampling and grid/filter.hpp time-series
// filter (the multigrid transfer), plus the SPEC's restrict_data /
// prolong_model, on the device engine (csrc/resample.cu via the C ABI).
#pragma once

#include <cmath>
#include <stdexcept>
#include <vector>

#include "core.hpp"
#include "solver.hpp"

namespace ustfwi {

enum class SpectralWindow { none, blackman };

/// grid/spectral.hpp:166-212: trigonometric resampling to new_dims (all even, >= 4) by
/// zero-padding / truncating the spectrum, optional separable Blackman taper.
inline Field fourier_interpolate(const Field& field, const Dims& new_dims, SpectralWindow window = SpectralWindow::none,
                                 int device = 0) {
    if (static_cast<int>(new_dims.size()) != field.ndim()) throw std::invalid_argument("target dimensionality mismatch");
    Field out(new_dims);
    detail::check(ustfwi_fourier_interpolate(device, field.ndim(), field.dims().data(), field.data(), new_dims.data(),
                                             window == SpectralWindow::blackman ? 1 : 0, out.data()));
    return out;
}

/// grid/filter.hpp:88-101: zero-phase Kaiser-window FIR low-pass of a sampled series.
inline std::vector<double> lowpass_filter_timeseries(const std::vector<double>& signal, double dt, double cutoff_hz,
                                                     double transition = 0.1, double atten_db = 60.0, int device = 0) {
    if (signal.empty()) return {};
    std::vector<double> out(signal.size());
    detail::check(ustfwi_lowpass_timeseries(device, 1, signal.size(), signal.data(), dt, cutoff_hz, transition,
                                            atten_db, out.data()));
    return out;
}

/// SPEC.md:463-470 prolong_model: Blackman-windowed Fourier interpolation of a coarse model.
inline Field prolong_model(const Field& u_coarse, const Dims& fine_dims, int device = 0) {
    return fourier_interpolate(u_coarse, fine_dims, SpectralWindow::blackman, device);
}

/// SPEC.md:463-470 restrict_data for recorded traces: ceil(nt/eta) samples per sensor,
/// Kaiser low-passed at cutoff_hz, scaled by eta^(ndim-1) (Appendix C).
inline SensorData restrict_data(const SensorData& data, int eta, int ndim, double cutoff_hz, int device = 0) {
    std::size_t ntc = 0;
    detail::check(ustfwi_restrict_traces(device, static_cast<std::size_t>(data.n_sensors),
                                         static_cast<std::size_t>(data.nt), data.samples.data(), eta, ndim, data.dt,
                                         cutoff_hz, nullptr, &ntc));
    SensorData out;
    out.n_sensors = data.n_sensors;
    out.nt = static_cast<int>(ntc);
    out.dt = data.dt * eta;
    out.samples.assign(static_cast<std::size_t>(data.n_sensors) * ntc, 0.0);
    detail::check(ustfwi_restrict_traces(device, static_cast<std::size_t>(data.n_sensors),
                                         static_cast<std::size_t>(data.nt), data.samples.data(), eta, ndim, data.dt,
                                         cutoff_hz, out.samples.data(), &ntc));
    return out;
}

/// SPEC.md optimizer LbfgsState / two_loop_recursion (Algorithm 2) with the
/// curvature history in HBM (fp64).
class LbfgsState {
public:
    LbfgsState(std::size_t n, int history = 64, int device = 0, double reject_tol = 1e-10) : n_(n), tol_(reject_tol) {
        detail::check(ustfwi_lbfgs_create(device, n, history, &h_));
    }
    ~LbfgsState() { ustfwi_lbfgs_destroy(h_); }
    LbfgsState(const LbfgsState&) = delete;
    LbfgsState& operator=(const LbfgsState&) = delete;
    /// updateBuffer(s, S), updateBuffer(y, Y); false when the curvature pair is rejected
    bool push(const std::vector<double>& s, const std::vector<double>& y) {
        if (s.size() != n_ || y.size() != n_) throw std::invalid_argument("pair length does not match the state");
        int ok = 0;
        detail::check(ustfwi_lbfgs_push(h_, s.data(), y.data(), tol_, &ok));
        return ok != 0;
    }
    /// H_k g (twoLoopRecursion)
    std::vector<double> apply(const std::vector<double>& g) {
        if (g.size() != n_) throw std::invalid_argument("vector length does not match the state");
        std::vector<double> out(n_);
        detail::check(ustfwi_lbfgs_apply(h_, g.data(), out.data()));
        return out;
    }
    void reset() { detail::check(ustfwi_lbfgs_reset(h_)); }

private:
    ustfwi_lbfgs* h_ = nullptr;
    std::size_t n_;
    double tol_;
};

}  // namespace ustfwi
