// ustfwi drop-in (B200): medium / geometry types, the device SpectralEngine, the device
// WaveStepper and simulate_forward — the reference's solver/medium.hpp, solver/engine.hpp and
// solver/simulate.hpp API on top of libustfwi_b200.so.
#pragma once

#include <array>
#include <memory>
#include <optional>

#include "core.hpp"
#include "spectral.hpp"

namespace ustfwi {

/// solver/medium.hpp:15-21
inline double db2neper(double alpha_db, double y) {
    return 100.0 * alpha_db * (std::log(10.0) / 20.0) / std::pow(2.0 * M_PI * 1e6, y);
}
inline double neper2db(double alpha_np, double y) {
    return alpha_np / (100.0 * (std::log(10.0) / 20.0) / std::pow(2.0 * M_PI * 1e6, y));
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

    /// solver/medium.hpp:41-57 (the device upload repeats these checks with the same messages)
    void validate(const Grid& grid, bool dispersion_active = true) const {
        if (c0.dims() != grid.dims || rho0.dims() != grid.dims || (!alpha0.empty() && alpha0.dims() != grid.dims))
            throw std::invalid_argument("medium fields must match the grid");
        if (!gamma.empty() && gamma.dims() != grid.dims) throw std::invalid_argument("gamma mask must match the grid");
        for (std::size_t i = 0; i < c0.size(); ++i) {
            if (c0[i] < c0_min || c0[i] > c0_max) throw std::invalid_argument("c0 outside configured bounds");
            if (rho0[i] <= 0.0) throw std::invalid_argument("rho0 must be positive");
            if (!alpha0.empty() && alpha0[i] < 0.0) throw std::invalid_argument("alpha0 must be non-negative");
        }
        if (y <= 1.0 || y >= 3.0) throw std::invalid_argument("power-law exponent must be in (1,3)");
        if (dispersion_active && y == 2.0 && absorbing())
            throw std::invalid_argument("y = 2 requires the dispersion term to be disabled");
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
    std::span<double> at_step(int n) {
        return {values.data() + static_cast<std::size_t>(n) * layer_indices.size(), layer_indices.size()};
    }
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

/// solver/medium.hpp:137-165: one face-connected erosion step (the mask minus its 1-shell).
inline Mask erode(const Mask& mask) {
    Mask out = mask;
    if (mask.empty()) return out;
    for (std::size_t i : shell_indices(mask, 1)) out.set(i, false);
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

    /// engine.hpp:131-137 (device, fp32)
    void half_shift(const Field& f, int axis, int direction, Field& out) {
        if (f.dims() != grid_.dims) throw std::invalid_argument("field dims do not match the grid");
        if (out.dims() != grid_.dims) out = Field(grid_.dims);
        detail::check(ustfwi_gpu_half_shift(ctx(), f.data(), axis, direction, out.data()));
    }

    // ---- half-spectrum tables and multiplier helpers (engine.hpp:81-128), host fp64 ----
    std::size_t spectrum_size() const { return k2().size(); }
    const std::vector<double>& k2() const {
        if (k2_.empty()) {
            Dims sd = grid_.dims;
            sd.back() = grid_.dims.back() / 2 + 1;
            std::vector<std::vector<double>> k;
            for (std::size_t a = 0; a < grid_.dims.size(); ++a) k.push_back(fft_wavenumbers(grid_.dims[a], grid_.dx[a]));
            k2_.assign(total_size(sd), 0.0);
            kappa_.assign(k2_.size(), 0.0);
            detail::for_each_index(sd, [&](std::size_t idx, const Coord& c) {
                double s = 0.0;
                for (std::size_t a = 0; a < c.size(); ++a) s += k[a][static_cast<std::size_t>(c[a])] * k[a][static_cast<std::size_t>(c[a])];
                k2_[idx] = s;
                kappa_[idx] = sinc(0.5 * grid_.c_ref * grid_.dt * std::sqrt(s));
            });
        }
        return k2_;
    }
    const std::vector<double>& kappa() const {
        k2();
        return kappa_;
    }
    /// |k|^e, k = 0 bin 1 for e == 0 and 0 otherwise (engine.hpp:88-94)
    std::vector<double> power_multiplier(double exponent_of_k) const {
        const auto& q = k2();
        std::vector<double> m(q.size());
        for (std::size_t i = 0; i < m.size(); ++i)
            m[i] = q[i] == 0.0 ? (exponent_of_k == 0.0 ? 1.0 : 0.0) : std::pow(q[i], 0.5 * exponent_of_k);
        return m;
    }
    /// log|k|^2, 0 at k = 0 (engine.hpp:97-101)
    std::vector<double> log_k2_multiplier() const {
        const auto& q = k2();
        std::vector<double> m(q.size());
        for (std::size_t i = 0; i < m.size(); ++i) m[i] = q[i] == 0.0 ? 0.0 : std::log(q[i]);
        return m;
    }
    /// engine.hpp:103-128 load / multiplier_from_loaded / apply_multiplier: fp64 on the host
    /// (RealFft of spectral.hpp); diagnostics, never the device step.
    void load(const Field& f) {
        if (!rfft_) rfft_ = std::make_unique<RealFft>(grid_.dims);
        loaded_.resize(rfft_->spectrum_size());
        rfft_->forward(f.data(), loaded_.data());
    }
    void multiplier_from_loaded(const std::vector<double>& mult, Field& out) {
        if (loaded_.empty()) throw std::invalid_argument("no field loaded");
        std::vector<std::complex<double>> t(loaded_.size());
        for (std::size_t i = 0; i < t.size(); ++i) t[i] = loaded_[i] * mult[i];
        if (out.dims() != grid_.dims) out = Field(grid_.dims);
        rfft_->inverse(t.data(), out.data());
    }
    void apply_multiplier(const Field& f, const std::vector<double>& mult, Field& out) {
        load(f);
        multiplier_from_loaded(mult, out);
    }

    // device WaveStepper slots of this engine (the context hosts two steppers)
    int acquire_stepper() {
        for (int s = 0; s < 2; ++s)
            if (!stepper_used_[static_cast<std::size_t>(s)]) {
                stepper_used_[static_cast<std::size_t>(s)] = true;
                return s;
            }
        throw std::invalid_argument("a device SpectralEngine hosts at most two WaveSteppers");
    }
    void release_stepper(int s) {
        if (s >= 0 && s < 2) stepper_used_[static_cast<std::size_t>(s)] = false;
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
    mutable std::vector<double> k2_, kappa_;
    std::unique_ptr<RealFft> rfft_;
    std::vector<std::complex<double>> loaded_;
    std::array<bool, 2> stepper_used_{false, false};
};

/// solver/engine.hpp:170-177
struct StepperOptions {
    bool pml_enabled = true;
    double absorption_sign = 1.0;
    bool dispersion_enabled = true;
};

/// solver/engine.hpp:182-386 — the first-order k-space leapfrog stepper on the device. The
/// state (p, v, split rho, spectra) lives in HBM in one of the engine's two stepper slots;
/// each call below is one or a few device launches. pressure() / velocity() copy the fp32
/// device state into fp64 Fields. The engine's bound medium is the stepper's medium (a
/// second stepper on the same engine shares it).
class WaveStepper {
public:
    WaveStepper(const Grid& grid, const Medium& medium, SpectralEngine& engine, StepperOptions options = {})
        : grid_(grid), engine_(engine), opt_(options) {
        for (std::size_t a = 1; a < grid_.dx.size(); ++a)
            if (grid_.dx[a] != grid_.dx[0]) throw std::invalid_argument("wave stepper requires uniform grid spacing");
        dispersion_on_ = opt_.dispersion_enabled && medium.y != 2.0;
        medium.validate(grid_, dispersion_on_);
        engine_.use_nt(grid_.nt);
        engine_.bind(medium);  // CFL guard -> NumericalError (engine.hpp:196-197)
        slot_ = engine_.acquire_stepper();
        try {
            detail::check(ustfwi_gpu_stepper_init(engine_.ctx(), slot_, opt_.pml_enabled ? 1 : 0, opt_.absorption_sign,
                                                  opt_.dispersion_enabled ? 1 : 0));
        } catch (...) {
            engine_.release_stepper(slot_);
            throw;
        }
        absorbing_ = medium.absorbing();
        c0_sq_ = Field(grid_.dims);
        rho0_ = medium.rho0;
        for (std::size_t i = 0; i < c0_sq_.size(); ++i) c0_sq_[i] = medium.c0[i] * medium.c0[i];
    }
    ~WaveStepper() { engine_.release_stepper(slot_); }
    WaveStepper(const WaveStepper&) = delete;
    WaveStepper& operator=(const WaveStepper&) = delete;

    void reset() { detail::check(ustfwi_gpu_stepper_reset(engine_.ctx(), slot_)); }
    void update_velocity_density() { detail::check(ustfwi_gpu_stepper_update_velocity_density(engine_.ctx(), slot_)); }
    void inject_mass_source(std::size_t flat_index, double amplitude) {
        detail::check(ustfwi_gpu_stepper_inject(engine_.ctx(), slot_, 1, &flat_index, &amplitude));
    }
    /// extension: a whole step's sources in one call, applied in order
    void inject_mass_sources(const std::vector<std::size_t>& idx, const std::vector<double>& amp) {
        if (idx.size() != amp.size()) throw std::invalid_argument("index / amplitude size mismatch");
        detail::check(ustfwi_gpu_stepper_inject(engine_.ctx(), slot_, idx.size(), idx.data(), amp.data()));
    }
    void enforce_shell(const std::vector<std::size_t>& shell, std::span<const double> values) {
        if (values.size() < shell.size()) throw std::invalid_argument("shell values shorter than the shell");
        detail::check(ustfwi_gpu_stepper_enforce(engine_.ctx(), slot_, shell.size(), shell.data(), values.data()));
    }
    void refresh_pressure_from_density() { detail::check(ustfwi_gpu_stepper_refresh_pressure(engine_.ctx(), slot_)); }
    void update_pressure() { detail::check(ustfwi_gpu_stepper_update_pressure(engine_.ctx(), slot_)); }

    const Field& pressure() const {
        if (p_.dims() != grid_.dims) p_ = Field(grid_.dims);
        detail::check(ustfwi_gpu_stepper_read(engine_.ctx(), slot_, 0, p_.data()));
        return p_;
    }
    const std::vector<Field>& velocity() const {
        v_.resize(grid_.dims.size());
        for (std::size_t a = 0; a < v_.size(); ++a) {
            if (v_[a].dims() != grid_.dims) v_[a] = Field(grid_.dims);
            detail::check(ustfwi_gpu_stepper_read(engine_.ctx(), slot_, static_cast<int>(a) + 1, v_[a].data()));
        }
        return v_;
    }
    /// p at a few positions without copying the field (sensor sampling)
    std::vector<double> pressure_at(const std::vector<std::size_t>& idx) const {
        std::vector<double> out(idx.size());
        detail::check(ustfwi_gpu_stepper_gather(engine_.ctx(), slot_, idx.size(), idx.data(), out.data()));
        return out;
    }
    const Field& c0_squared() const { return c0_sq_; }
    int step_index() const {
        int k = 0;
        detail::check(ustfwi_gpu_stepper_step_index(engine_.ctx(), slot_, &k));
        return k;
    }
    bool absorbing() const { return absorbing_; }

    /// engine.hpp:350-366 energy diagnostics (host fp64 on the downloaded state)
    double kinetic_energy(const std::vector<Field>& v_prev) const {
        const auto& v = velocity();
        double e = 0.0;
        for (std::size_t a = 0; a < v.size(); ++a)
            for (std::size_t i = 0; i < rho0_.size(); ++i) e += 0.5 * rho0_[i] * v[a][i] * v_prev[a][i];
        return e;
    }
    double potential_energy(const Field& p) const {
        double e = 0.0;
        for (std::size_t i = 0; i < p.size(); ++i) e += 0.5 * p[i] * p[i] / (rho0_[i] * c0_sq_[i]);
        return e;
    }

private:
    Grid grid_;
    SpectralEngine& engine_;
    StepperOptions opt_;
    int slot_ = -1;
    bool absorbing_ = false;
    bool dispersion_on_ = true;
    Field c0_sq_, rho0_;
    mutable Field p_;
    mutable std::vector<Field> v_;
};

/// solver/engine.hpp:153-168
inline void apply_axis_profile(Field& f, const std::vector<double>& w, int axis) {
    const Dims& dims = f.dims();
    const auto ua = static_cast<std::size_t>(axis);
    std::size_t post = 1;
    for (std::size_t a = ua + 1; a < dims.size(); ++a) post *= static_cast<std::size_t>(dims[a]);
    const std::size_t n_axis = static_cast<std::size_t>(dims[ua]);
    const std::size_t pre = f.size() / (post * n_axis);
    for (std::size_t ip = 0; ip < pre; ++ip)
        for (std::size_t j = 0; j < n_axis; ++j)
            for (std::size_t q = 0; q < post; ++q) f[(ip * n_axis + j) * post + q] *= w[j];
}

/// solver/simulate.hpp:10-19
struct SimOptions {
    int boundary_thickness = 0;
    int snapshot_decimation = 0;
    bool record_energy = false;
    bool pml_enabled = true;
};

struct SimResult {
    SensorData data;
    BoundaryTrace trace;
    std::vector<Field> snapshots;
    std::vector<double> energy;
};

namespace detail {
/// simulate.hpp:49-103 step by step on the device WaveStepper: the path for the diagnostic
/// options (snapshots, energy, PML off); the fused forward below serves everything else.
inline SimResult simulate_with_stepper(const Medium& medium, const SourceSet& sources, const SensorArray& sensors,
                                       const Grid& grid, const SimOptions& opt, SpectralEngine& engine) {
    StepperOptions sopt;
    sopt.pml_enabled = opt.pml_enabled;
    WaveStepper stepper(grid, medium, engine, sopt);
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
    double dV = 1.0;
    for (double dx : grid.dx) dV *= dx;
    std::vector<Field> v_prev;
    Field p_prev;
    std::vector<std::size_t> idx;
    std::vector<double> amp;
    for (int n = 0; n < grid.nt; ++n) {
        if (opt.record_energy) {
            v_prev = stepper.velocity();
            p_prev = stepper.pressure();
        }
        stepper.update_velocity_density();
        idx.clear();
        amp.clear();
        for (std::size_t s = 0; s < sources.count(); ++s) {
            const double a = sources.sample(s, n);
            if (a != 0.0) {
                idx.push_back(sources.positions[s]);
                amp.push_back(a);
            }
        }
        if (!idx.empty()) stepper.inject_mass_sources(idx, amp);
        stepper.update_pressure();
        if (sensors.count()) {
            const auto v = stepper.pressure_at(sensors.positions);
            for (std::size_t s = 0; s < v.size(); ++s) r.data.at(static_cast<int>(s), n) = v[s];
        }
        if (!r.trace.empty()) {
            const auto v = stepper.pressure_at(r.trace.layer_indices);
            auto row = r.trace.at_step(n);
            std::copy(v.begin(), v.end(), row.begin());
        }
        if (opt.snapshot_decimation > 0 && n % opt.snapshot_decimation == 0) r.snapshots.push_back(stepper.pressure());
        if (opt.record_energy) r.energy.push_back((stepper.kinetic_energy(v_prev) + stepper.potential_energy(p_prev)) * dV);
    }
    r.data.check_finite();
    return r;
}
}  // namespace detail

/// solver/simulate.hpp:30-105
inline SimResult simulate_forward(const Medium& medium, const SourceSet& sources, const SensorArray& sensors,
                                  const Grid& grid, const SimOptions& opt = {}, SpectralEngine* engine = nullptr) {
    grid.validate();
    for (std::size_t s = 0; s < sources.count(); ++s)
        if (sources.positions[s] >= grid.points()) throw std::invalid_argument("source position outside grid");
    for (std::size_t s = 0; s < sensors.count(); ++s)
        if (sensors.positions[s] >= grid.points()) throw std::invalid_argument("sensor position outside grid");
    std::optional<SpectralEngine> local;
    if (!engine) {
        local.emplace(grid);
        engine = &*local;
    }
    if (opt.snapshot_decimation != 0 || opt.record_energy || !opt.pml_enabled)
        return detail::simulate_with_stepper(medium, sources, sensors, grid, opt, *engine);
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

/// solver/simulate.hpp:108-120: P(t_n) = dV sum over gamma of p^2 per snapshot
inline std::vector<double> field_power(const std::vector<Field>& snapshots, const Mask& gamma, double dV) {
    std::vector<double> power;
    power.reserve(snapshots.size());
    const auto idx = gamma.indices();
    for (const Field& p : snapshots) {
        double s = 0.0;
        for (std::size_t i : idx) s += p[i] * p[i];
        power.push_back(s * dV);
    }
    return power;
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
