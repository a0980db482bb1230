// ustfwi drop-in (B200): the gradient API of adjoint/gradient.hpp and the source-encoding
// estimators of SPEC.md (stochastic_estimators) on top of libustfwi_b200.so.
#pragma once

#include "solver.hpp"

namespace ustfwi {

enum class GradientParam { c0, rho0, alpha0, y };
enum class GradientMethod { full_storage, time_reversal };

inline const char* to_string(GradientParam p) {
    switch (p) {
        case GradientParam::c0: return "c0";
        case GradientParam::rho0: return "rho0";
        case GradientParam::alpha0: return "alpha0";
        default: return "y";
    }
}

/// adjoint/gradient.hpp:22-32, same defaults (method = full_storage). The device engine
/// implements the time-reversal method; full_storage (defective in the reference, SURVEY.md
/// F4, and 98 GB of snapshots at the paper's grid) is rejected with std::invalid_argument,
/// so a caller relying on the default gets an error, never a different method.
struct GradientOptions {
    GradientMethod method = GradientMethod::full_storage;
    int boundary_thickness = 8;
    int snapshot_decimation = 1;
    bool source_integration_correction = true;
    std::size_t storage_limit = std::size_t{12} << 30;
    bool dispersion_enabled = true;
};

struct GradientResult {
    double loss = 0.0;
    Field grad;
    GradientParam param = GradientParam::c0;
    GradientMethod method = GradientMethod::time_reversal;
    int boundary_thickness = 0;
    std::size_t bytes_forward_storage = 0;
    int n_simulations = 0;
};

/// adjoint/gradient.hpp:333-464 (time-reversal branch, GradientParam c0 / alpha0 / y)
inline GradientResult compute_gradient(const Medium& medium, const SourceSet& source, const SensorArray& sensors,
                                       const SensorData& observed, const Grid& grid, GradientParam param,
                                       const GradientOptions& opt = {}, SpectralEngine* engine = nullptr) {
    grid.validate();
    if (medium.gamma.empty()) throw std::invalid_argument("gradient computation requires a gamma mask");
    if (observed.nt != grid.nt) throw std::invalid_argument("observed data length does not match the grid");
    if (observed.n_sensors != static_cast<int>(sensors.count()))
        throw std::invalid_argument("observed data dimensions do not match the simulation");
    if (opt.method != GradientMethod::time_reversal)
        throw std::invalid_argument(
            "the device engine implements the time-reversal gradient method (set GradientOptions::method)");
    if (!opt.source_integration_correction)
        throw std::invalid_argument("the device engine always integrates the adjoint source");
    std::optional<SpectralEngine> local;
    if (!engine) {
        local.emplace(grid);
        engine = &*local;
    }
    engine->use_nt(grid.nt);
    engine->bind(medium);
    engine->bind(source);
    engine->bind(sensors);
    GradientResult r;
    r.grad = Field(grid.dims);
    detail::check(ustfwi_gpu_set_gradient_options(engine->ctx(), opt.dispersion_enabled ? 1 : 0));
    detail::check(ustfwi_gpu_set_gradient_param(
        engine->ctx(), param == GradientParam::alpha0 ? USTFWI_PARAM_ALPHA0
                       : param == GradientParam::y    ? USTFWI_PARAM_Y
                       : param == GradientParam::rho0 ? USTFWI_PARAM_RHO0
                                                      : USTFWI_PARAM_C0));
    detail::check(ustfwi_gpu_gradient_tr(engine->ctx(), observed.samples.data(), opt.boundary_thickness, r.grad.data(),
                                         &r.loss));
    r.param = param;
    r.method = GradientMethod::time_reversal;
    r.boundary_thickness = opt.boundary_thickness;
    r.bytes_forward_storage = ustfwi_gpu_shell_size(engine->ctx()) * static_cast<std::size_t>(grid.nt) * sizeof(float);
    r.n_simulations = 3;
    return r;
}

/// adjoint/gradient.hpp:466-476: kept for source compatibility; the full-storage method is not
/// provided by the device engine (see GradientOptions) and throws std::invalid_argument.
inline GradientResult gradient_full_storage(const Medium& medium, const SourceSet& source, const SensorArray& sensors,
                                            const SensorData& observed, const Grid& grid,
                                            GradientParam param = GradientParam::c0, int snapshot_decimation = 1,
                                            SpectralEngine* engine = nullptr) {
    GradientOptions opt;
    opt.method = GradientMethod::full_storage;
    opt.snapshot_decimation = snapshot_decimation;
    return compute_gradient(medium, source, sensors, observed, grid, param, opt, engine);
}

/// adjoint/gradient.hpp:478-488
inline GradientResult gradient_time_reversal(const Medium& medium, const SourceSet& source, const SensorArray& sensors,
                                             const SensorData& observed, const Grid& grid, int boundary_thickness,
                                             GradientParam param = GradientParam::c0, SpectralEngine* engine = nullptr) {
    GradientOptions opt;
    opt.method = GradientMethod::time_reversal;
    opt.boundary_thickness = boundary_thickness;
    return compute_gradient(medium, source, sensors, observed, grid, param, opt, engine);
}

/// adjoint/gradient.hpp:491-505
inline double evaluate_loss(const Medium& medium, const SourceSet& source, const SensorArray& sensors,
                            const SensorData& observed, const Grid& grid, SpectralEngine* engine = nullptr) {
    std::optional<SpectralEngine> local;
    if (!engine) {
        local.emplace(grid);
        engine = &*local;
    }
    engine->use_nt(grid.nt);
    engine->bind(medium);
    engine->bind(source);
    engine->bind(sensors);
    double loss = 0.0;
    detail::check(ustfwi_gpu_evaluate_loss(engine->ctx(), observed.samples.data(), &loss));
    return loss;
}

// ---- stochastic estimators ---------------------------------------------

/// SPEC.md:277-280
struct EncodingRealization {
    std::vector<double> weights;      // w_i in {-1, +1}
    std::vector<double> delays;       // d_i in [0, 1)
    std::vector<int> delay_steps;     // round(d_i * tau / dt)
    double tau = 0.0;
    double dt = 0.0;                  // time step the delays are quantized to
    std::uint64_t master_seed = 0, iteration = 0, index = 0;
};

/// Counter-based, reproducible draw keyed by (master_seed, iteration, index).
inline EncodingRealization draw_realization(std::size_t n_src, double tau, double dt, std::uint64_t master_seed,
                                            std::uint64_t iteration, std::uint64_t index) {
    std::vector<std::int8_t> w(n_src);
    std::vector<std::int32_t> d(n_src);
    EncodingRealization r;
    r.delays.resize(n_src);
    detail::check(ustfwi_draw_realization(n_src, tau, dt, master_seed, iteration, index, w.data(), d.data(), r.delays.data()));
    r.weights.assign(w.begin(), w.end());
    r.delay_steps.assign(d.begin(), d.end());
    r.tau = tau;
    r.dt = dt;
    r.master_seed = master_seed;
    r.iteration = iteration;
    r.index = index;
    return r;
}

/// ceil(tau / dt), robust to tau being a multiple of dt up to rounding.
inline int extension_steps(double tau, double dt) {
    if (tau <= 0.0) return 0;
    if (!(dt > 0.0)) throw std::invalid_argument("dt must be positive");
    return static_cast<int>(std::ceil(tau / dt - 1e-9));
}

/// super-source s^ = sum w_i s_i(t - d_i tau) and data f^ = sum w_i f_i(t - d_i tau),
/// zero-padded to nt_ext = nt + ceil(tau/dt). `data` may be empty (synthetic data from a forward
/// run); otherwise one SensorData per source, each with n_sensors equal to data[0]'s and nt <= nt.
struct Encoded {
    SourceSet source;
    SensorData data;
    int nt_ext = 0;
};

inline Encoded encode(const SourceSet& sources, const std::vector<SensorData>& data, const EncodingRealization& r,
                      int nt) {
    if (r.tau < 0.0) throw std::invalid_argument("tau must be non-negative");
    if (r.weights.size() != sources.count()) throw std::invalid_argument("realization size does not match the sources");
    Encoded e;
    e.source = sources;
    e.source.weights = r.weights;
    e.source.delays = r.delay_steps;
    if (r.delay_steps.size() != sources.count()) throw std::invalid_argument("realization size does not match the sources");
    const int ext = extension_steps(r.tau, r.dt);
    for (int d : r.delay_steps)
        if (d < 0 || d > ext) throw std::invalid_argument("delay outside [0, ceil(tau/dt)]");
    e.nt_ext = nt + ext;
    if (!data.empty()) {
        if (data.size() != sources.count()) throw std::invalid_argument("one SensorData per source is required");
        const int ns = data[0].n_sensors;
        for (const auto& d : data) {
            if (d.n_sensors != ns) throw std::invalid_argument("per-source data must share the sensor array");
            if (d.nt > nt || d.nt < 0) throw std::invalid_argument("per-source data longer than nt");
            if (d.samples.size() != static_cast<std::size_t>(d.n_sensors) * static_cast<std::size_t>(d.nt))
                throw std::invalid_argument("per-source data size does not match n_sensors * nt");
        }
        e.data.n_sensors = ns;
        e.data.nt = e.nt_ext;
        e.data.dt = data[0].dt;
        e.data.samples.assign(static_cast<std::size_t>(ns) * e.nt_ext, 0.0);
        for (std::size_t i = 0; i < data.size(); ++i)
            for (int s = 0; s < ns; ++s)
                for (int n = 0; n < data[i].nt; ++n)
                    e.data.at(s, n + r.delay_steps[i]) += r.weights[i] * data[i].at(s, n);
    }
    return e;
}

/// SPEC.md:305-313 encoded_gradient: one TR gradient of the encoded super-source over the
/// extended duration T + tau (the grid's nt is replaced by e.nt_ext; e.data is f^).
inline GradientResult encoded_gradient(const Medium& medium, const Encoded& e, const SensorArray& sensors,
                                       const Grid& grid, int boundary_thickness, SpectralEngine* engine = nullptr) {
    Grid ext = grid;
    ext.nt = e.nt_ext;
    return gradient_time_reversal(medium, e.source, sensors, e.data, ext, boundary_thickness, GradientParam::c0, engine);
}

/// arithmetic mean of gradients and losses (fixed order).
inline GradientResult average_estimates(const std::vector<GradientResult>& rs) {
    if (rs.empty()) throw std::invalid_argument("nothing to average");
    GradientResult out = rs[0];
    out.grad = Field(rs[0].grad.dims());
    out.loss = 0.0;
    for (const auto& r : rs) {
        out.grad += r.grad;
        out.loss += r.loss;
    }
    out.grad *= 1.0 / static_cast<double>(rs.size());
    out.loss /= static_cast<double>(rs.size());
    return out;
}

}  // namespace ustfwi
