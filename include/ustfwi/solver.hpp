// ustfwi drop-in (B200): medium / geometry types, the device SpectralEngine and
// simulate_forward — the reference's solver/medium.hpp, solver/engine.hpp and
// solver/simulate.hpp API on top of libustfwi_b200.so.
#pragma once

#include <memory>
#include <optional>

#include "core.hpp"

namespace ustfwi {

enum class Stagger { none, plus, minus };

/// solver/medium.hpp:15-21
inline double db2neper(double alpha_db, double y) {
    return 100.0 * alpha_db * (std::log(10.0) / 20.0) / std::pow(2.0 * M_PI * 1e6, y);
}

/// solver/medium.hpp:26-58 (validation happens on the device upload, same messages).
struct Medium {
    Field c0;
    Field rho0;
    Field alpha0;
    double y = 1.5;
    Mask gamma;
    double c0_min = 1350.0;
    double c0_max = 1800.0;

    bool absorbing() const {
        for (std::size_t i = 0; i < alpha0.size(); ++i)
            if (alpha0[i] != 0.0) return true;
        return false;
    }
};

inline Medium make_homogeneous_medium(const Grid& grid, double c0 = 1500.0, double rho0 = 1000.0,
                                      double alpha0 = 0.0, double y = 1.5) {
    Medium m;
    m.c0 = Field(grid.dims, c0);
    m.rho0 = Field(grid.dims, rho0);
    m.alpha0 = Field(grid.dims, alpha0);
    m.y = y;
    m.c0_min = std::min(1350.0, c0);
    m.c0_max = std::max(1800.0, c0);
    return m;
}

/// solver/medium.hpp:74-85, plus the encoded-source fields: sample(i, n) =
/// weight_i * signals[i][n - delay_i]; empty weights / delays mean 1 / 0.
struct SourceSet {
    std::vector<std::size_t> positions;
    std::vector<std::vector<double>> signals;
    double support_duration = 0.0;
    std::vector<double> weights;
    std::vector<int> delays;

    std::size_t count() const { return positions.size(); }
    double sample(std::size_t i, int n) const {
        const int d = delays.empty() ? 0 : delays[i];
        const double w = weights.empty() ? 1.0 : weights[i];
        const auto& s = signals[i];
        const int k = n - d;
        return (k >= 0 && static_cast<std::size_t>(k) < s.size()) ? w * s[static_cast<std::size_t>(k)] : 0.0;
    }
};

struct SensorArray {
    std::vector<std::size_t> positions;
    std::size_t count() const { return positions.size(); }
};

/// solver/medium.hpp:94-114 (sensor-major samples).
struct SensorData {
    std::vector<double> samples;
    int n_sensors = 0;
    int nt = 0;
    double dt = 0.0;
    double t0 = 0.0;

    std::span<double> trace(int s) { return {samples.data() + static_cast<std::size_t>(s) * nt, static_cast<std::size_t>(nt)}; }
    std::span<const double> trace(int s) const {
        return {samples.data() + static_cast<std::size_t>(s) * nt, static_cast<std::size_t>(nt)};
    }
    double& at(int s, int n) { return samples[static_cast<std::size_t>(s) * nt + n]; }
    double at(int s, int n) const { return samples[static_cast<std::size_t>(s) * nt + n]; }
    void check_finite() const {
        for (double v : samples)
            if (!std::isfinite(v)) throw NumericalError("sensor data contains non-finite values");
    }
};

/// solver/medium.hpp:118-133 (step-major).
struct BoundaryTrace {
    std::vector<std::size_t> layer_indices;
    std::vector<double> values;
    int nt = 0;
    bool empty() const { return layer_indices.empty(); }
    std::span<const double> at_step(int n) const {
        return {values.data() + static_cast<std::size_t>(n) * layer_indices.size(), layer_indices.size()};
    }
    std::size_t bytes() const { return values.size() * sizeof(double); }
};

inline std::vector<std::size_t> shell_indices(const Mask& mask, int thickness) {
    std::size_t n = 0;
    const Dims& d = mask.dims();
    detail::check(ustfwi_shell_indices(static_cast<int>(d.size()), d.data(), mask.bytes(), thickness, nullptr, &n));
    std::vector<std::size_t> out(n);
    detail::check(ustfwi_shell_indices(static_cast<int>(d.size()), d.data(), mask.bytes(), thickness, out.data(), &n));
    return out;
}

inline Mask ball_mask(const Dims& dims, const std::vector<double>& center, double radius_points) {
    std::vector<std::uint8_t> b(total_size(dims));
    detail::check(ustfwi_ball_mask(static_cast<int>(dims.size()), dims.data(), center.data(), radius_points, b.data()));
    Mask m(dims);
    for (std::size_t i = 0; i < b.size(); ++i) m.set(i, b[i] != 0);
    return m;
}

/// The device analogue of SpectralEngine (engine.hpp:17-151): owns one engine context on
/// one GPU (FFT plans, wavenumber/stagger tables, state of two steppers). One per worker.
class SpectralEngine {
public:
    explicit SpectralEngine(const Grid& grid, int device = 0) : grid_(grid) {
        const ustfwi_grid c = grid.to_c();
        ustfwi_gpu_ctx* h = nullptr;
        detail::check(ustfwi_gpu_create(device, &c, &h));
        ctx_.reset(h);
    }
    const Grid& grid() const { return grid_; }
    ustfwi_gpu_ctx* ctx() const { return ctx_.get(); }
    /// Follow the caller's simulation length (Grid::nt): an extended grid of a delayed encoding
    /// (nt + ceil(tau/dt)) reuses the same engine.
    void use_nt(int nt) {
        if (nt != grid_.nt) {
            detail::check(ustfwi_gpu_set_nt(ctx(), nt));
            grid_.nt = nt;
        }
    }

    /// engine.hpp:118-121
    void derivative(const Field& f, int axis, Stagger st, Field& out) {
        if (f.dims() != grid_.dims) throw std::invalid_argument("field dims do not match the grid");
        if (out.dims() != grid_.dims) out = Field(grid_.dims);
        detail::check(ustfwi_gpu_derivative(ctx(), f.data(), axis, static_cast<int>(st), out.data()));
    }

    // bind medium / sources / sensors (internal to the free functions below)
    void bind(const Medium& m) {
        if (m.c0.dims() != grid_.dims || m.rho0.dims() != grid_.dims ||
            (!m.alpha0.empty() && m.alpha0.dims() != grid_.dims))
            throw std::invalid_argument("medium fields must match the grid");
        if (!m.gamma.empty() && m.gamma.dims() != grid_.dims) throw std::invalid_argument("gamma mask must match the grid");
        detail::check(ustfwi_gpu_set_medium(ctx(), m.c0.data(), m.rho0.data(), m.alpha0.empty() ? nullptr : m.alpha0.data(),
                                            m.y, m.gamma.empty() ? nullptr : m.gamma.bytes(), m.c0_min, m.c0_max));
    }
    void bind(const SourceSet& s) {
        std::vector<std::size_t> off{0};
        std::vector<double> sig;
        for (const auto& x : s.signals) {
            sig.insert(sig.end(), x.begin(), x.end());
            off.push_back(sig.size());
        }
        if (sig.empty()) sig.push_back(0.0);
        std::vector<std::int32_t> d(s.delays.begin(), s.delays.end());
        detail::check(ustfwi_gpu_set_sources(ctx(), s.positions.size(), s.positions.data(), off.data(), sig.data(),
                                             s.weights.empty() ? nullptr : s.weights.data(), d.empty() ? nullptr : d.data()));
    }
    void bind(const SensorArray& s) { detail::check(ustfwi_gpu_set_sensors(ctx(), s.positions.size(), s.positions.data())); }

private:
    struct Del {
        void operator()(ustfwi_gpu_ctx* c) const { ustfwi_gpu_destroy(c); }
    };
    Grid grid_;
    std::unique_ptr<ustfwi_gpu_ctx, Del> ctx_;
};

/// solver/simulate.hpp:10-26
struct SimOptions {
    int boundary_thickness = 0;
    int snapshot_decimation = 0;  // not supported on the device path (must be 0)
    bool record_energy = false;   // not supported on the device path (must be false)
    bool pml_enabled = true;      // must be true on the device path
};

struct SimResult {
    SensorData data;
    BoundaryTrace trace;
    std::vector<Field> snapshots;
    std::vector<double> energy;
};

/// solver/simulate.hpp:30-105
inline SimResult simulate_forward(const Medium& medium, const SourceSet& sources, const SensorArray& sensors,
                                  const Grid& grid, const SimOptions& opt = {}, SpectralEngine* engine = nullptr) {
    grid.validate();
    if (opt.snapshot_decimation != 0 || opt.record_energy || !opt.pml_enabled)
        throw std::invalid_argument("snapshots / energy / PML-off are not supported by the device engine");
    std::optional<SpectralEngine> local;
    if (!engine) {
        local.emplace(grid);
        engine = &*local;
    }
    engine->use_nt(grid.nt);
    engine->bind(medium);
    engine->bind(sources);
    engine->bind(sensors);
    SimResult r;
    r.data.n_sensors = static_cast<int>(sensors.count());
    r.data.nt = grid.nt;
    r.data.dt = grid.dt;
    r.data.samples.assign(sensors.count() * static_cast<std::size_t>(grid.nt), 0.0);
    if (opt.boundary_thickness > 0) {
        if (medium.gamma.empty()) throw std::invalid_argument("boundary recording requires a gamma mask");
        r.trace.layer_indices = shell_indices(medium.gamma, opt.boundary_thickness);
        r.trace.nt = grid.nt;
        r.trace.values.assign(r.trace.layer_indices.size() * static_cast<std::size_t>(grid.nt), 0.0);
    }
    std::size_t n_shell = 0;
    detail::check(ustfwi_gpu_forward(engine->ctx(), opt.boundary_thickness, r.data.samples.data(),
                                     r.trace.values.empty() ? nullptr : r.trace.values.data(), &n_shell));
    return r;
}

/// solver/simulate.hpp:124-148
inline std::vector<double> synth_source_pulse(const Grid& grid, double center_freq_fraction, double c0_min) {
    const ustfwi_grid c = grid.to_c();
    int n = 0;
    detail::check(ustfwi_synth_source_pulse(&c, center_freq_fraction, c0_min, nullptr, &n));
    std::vector<double> out(static_cast<std::size_t>(n));
    detail::check(ustfwi_synth_source_pulse(&c, center_freq_fraction, c0_min, out.data(), &n));
    return out;
}

}  // namespace ustfwi
