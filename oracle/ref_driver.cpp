// C-ABI driver over the UNMODIFIED reference headers — TEST INFRASTRUCTURE ONLY.
//
// Built by oracle/Makefile into oracle/_ref/libustfwi_ref.so from the reference
// sources where they lie (/root/reference/proj/include, never copied) plus the
// in-repo FFTW-API shim. It exposes the reference's own hot-path entry points to the
// Python tests (golden generation) and to bench.py's CPU-baseline leg:
//   simulate_forward   simulate.hpp:30-105
//   gradient_time_reversal / compute_gradient (TR branch)   gradient.hpp:333-464,478-488
//   evaluate_loss      gradient.hpp:491-505
//   SpectralEngine::derivative  engine.hpp:118-121, spectral_derivative spectral.hpp:36-67
//   make_grid / choose_pml_size / make_pml  grid.hpp:70-103,153-178
//   shell_indices  medium.hpp:168-178, synth_source_pulse  simulate.hpp:124-148
// Status codes mirror the product C ABI: 0 ok, 1 invalid argument, 2 numerical, 9 other.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>

#include "ustfwi/adjoint/gradient.hpp"
#include "ustfwi/grid/filter.hpp"

extern "C" {

typedef struct {
    int ndim;
    int dims[3];
    double dx[3];
    double dt;
    int nt;
    int pml_size[3];
    double c_ref;
} RefGrid;

typedef struct {
    const double* c0;
    const double* rho0;
    const double* alpha0;  // may be null (lossless)
    double y;
    const uint8_t* gamma;  // may be null
    double c0_min;
    double c0_max;
} RefMedium;

typedef struct {
    size_t n;
    const size_t* pos;
    const size_t* sig_off;  // n + 1 offsets into sig
    const double* sig;
} RefSources;

}  // extern "C"

namespace {

thread_local std::string g_err;

ustfwi::Grid to_grid(const RefGrid* d) {
    ustfwi::Grid g;
    g.dims.assign(d->dims, d->dims + d->ndim);
    g.dx.assign(d->dx, d->dx + d->ndim);
    g.pml_size.assign(d->pml_size, d->pml_size + d->ndim);
    g.dt = d->dt;
    g.nt = d->nt;
    g.c_ref = d->c_ref;
    return g;
}

void from_grid(const ustfwi::Grid& g, RefGrid* d) {
    std::memset(d, 0, sizeof(*d));
    d->ndim = g.ndim();
    for (int a = 0; a < g.ndim(); ++a) {
        d->dims[a] = g.dims[static_cast<std::size_t>(a)];
        d->dx[a] = g.dx[static_cast<std::size_t>(a)];
        d->pml_size[a] = g.pml_size[static_cast<std::size_t>(a)];
    }
    d->dt = g.dt;
    d->nt = g.nt;
    d->c_ref = g.c_ref;
}

ustfwi::Medium to_medium(const ustfwi::Grid& g, const RefMedium* m) {
    ustfwi::Medium med;
    const std::size_t n = g.points();
    med.c0 = ustfwi::Field(g.dims);
    med.rho0 = ustfwi::Field(g.dims);
    med.alpha0 = ustfwi::Field(g.dims);
    std::memcpy(med.c0.data(), m->c0, n * sizeof(double));
    std::memcpy(med.rho0.data(), m->rho0, n * sizeof(double));
    if (m->alpha0) std::memcpy(med.alpha0.data(), m->alpha0, n * sizeof(double));
    med.y = m->y;
    med.c0_min = m->c0_min;
    med.c0_max = m->c0_max;
    if (m->gamma) {
        med.gamma = ustfwi::Mask(g.dims);
        for (std::size_t i = 0; i < n; ++i) med.gamma.set(i, m->gamma[i] != 0);
    }
    return med;
}

ustfwi::SourceSet to_sources(const RefSources* s) {
    ustfwi::SourceSet src;
    if (!s) return src;
    for (std::size_t i = 0; i < s->n; ++i) {
        src.positions.push_back(s->pos[i]);
        src.signals.emplace_back(s->sig + s->sig_off[i], s->sig + s->sig_off[i + 1]);
    }
    return src;
}

ustfwi::SensorArray to_sensors(size_t n, const size_t* pos) {
    ustfwi::SensorArray a;
    a.positions.assign(pos, pos + n);
    return a;
}

template <class Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const ustfwi::NumericalError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_make_grid(int ndim, const int* interior, double dx, double c_max, double duration,
                  double cfl, RefGrid* out) {
    return guarded([&] {
        ustfwi::Dims d(interior, interior + ndim);
        from_grid(ustfwi::make_grid(d, dx, c_max, duration, cfl), out);
    });
}

int ref_choose_pml_size(int ndim, const int* interior, int* out) {
    return guarded([&] {
        const auto t = ustfwi::choose_pml_size(ustfwi::Dims(interior, interior + ndim));
        for (int a = 0; a < ndim; ++a) out[a] = t[static_cast<std::size_t>(a)];
    });
}

int ref_make_pml(const RefGrid* grid, double alpha, double* regular, double* staggered) {
    return guarded([&] {
        const auto g = to_grid(grid);
        const auto pml = ustfwi::make_pml(g, alpha);
        std::size_t off = 0;
        for (int a = 0; a < g.ndim(); ++a) {
            const auto ua = static_cast<std::size_t>(a);
            std::memcpy(regular + off, pml.regular[ua].data(), pml.regular[ua].size() * sizeof(double));
            std::memcpy(staggered + off, pml.staggered[ua].data(),
                        pml.staggered[ua].size() * sizeof(double));
            off += pml.regular[ua].size();
        }
    });
}

int ref_engine_derivative(const RefGrid* grid, const double* f, int axis, int stagger, double* out) {
    return guarded([&] {
        const auto g = to_grid(grid);
        ustfwi::SpectralEngine eng(g);
        ustfwi::Field in(g.dims);
        std::memcpy(in.data(), f, g.points() * sizeof(double));
        ustfwi::Field o;
        eng.derivative(in, axis, static_cast<ustfwi::Stagger>(stagger), o);
        std::memcpy(out, o.data(), g.points() * sizeof(double));
    });
}

int ref_spectral_derivative(const RefGrid* grid, const double* f, int axis, int stagger, double* out) {
    return guarded([&] {
        const auto g = to_grid(grid);
        const auto kv = ustfwi::make_kvectors(g);
        ustfwi::Field in(g.dims);
        std::memcpy(in.data(), f, g.points() * sizeof(double));
        const auto o = ustfwi::spectral_derivative(in, axis, static_cast<ustfwi::Stagger>(stagger), kv);
        std::memcpy(out, o.data(), g.points() * sizeof(double));
    });
}

// fourier_interpolate (spectral.hpp:166-212)
int ref_fourier_interpolate(int ndim, const int* dims, const double* f, const int* new_dims, int blackman,
                            double* out) {
    return guarded([&] {
        ustfwi::Dims d(dims, dims + ndim), nd(new_dims, new_dims + ndim);
        ustfwi::Field in(d);
        std::memcpy(in.data(), f, in.size() * sizeof(double));
        const auto o = ustfwi::fourier_interpolate(in, nd, blackman ? ustfwi::SpectralWindow::blackman
                                                                    : ustfwi::SpectralWindow::none);
        std::memcpy(out, o.data(), o.size() * sizeof(double));
    });
}

// lowpass_filter_timeseries (filter.hpp:88-101)
int ref_lowpass_timeseries(const double* sig, size_t len, double dt, double cutoff_hz, double transition,
                           double atten_db, double* out) {
    return guarded([&] {
        std::vector<double> x(sig, sig + len);
        const auto o = ustfwi::lowpass_filter_timeseries(x, dt, cutoff_hz, transition, atten_db);
        std::memcpy(out, o.data(), o.size() * sizeof(double));
    });
}

int ref_fourier_shift(const RefGrid* grid, const double* f, int axis, double shift_cells, double* out) {
    return guarded([&] {
        const auto g = to_grid(grid);
        const auto kv = ustfwi::make_kvectors(g);
        ustfwi::Field in(g.dims);
        std::memcpy(in.data(), f, g.points() * sizeof(double));
        const auto o = ustfwi::fourier_shift(in, axis, shift_cells, kv);
        std::memcpy(out, o.data(), g.points() * sizeof(double));
    });
}

// Two-call protocol: pass out == nullptr to query the count.
int ref_shell_indices(int ndim, const int* dims, const uint8_t* mask, int thickness, size_t* out,
                      size_t* count) {
    return guarded([&] {
        ustfwi::Dims d(dims, dims + ndim);
        ustfwi::Mask m(d);
        for (std::size_t i = 0; i < m.size(); ++i) m.set(i, mask[i] != 0);
        const auto idx = ustfwi::shell_indices(m, thickness);
        if (out) std::memcpy(out, idx.data(), std::min(idx.size(), *count) * sizeof(size_t));
        *count = idx.size();
    });
}

int ref_synth_source_pulse(const RefGrid* grid, double frac, double c0_min, double* out, int* len) {
    return guarded([&] {
        const auto p = ustfwi::synth_source_pulse(to_grid(grid), frac, c0_min);
        if (out) std::memcpy(out, p.data(), std::min<std::size_t>(p.size(), static_cast<std::size_t>(*len)) * sizeof(double));
        *len = static_cast<int>(p.size());
    });
}

// Forward simulation. data_out: [n_sensors * nt] sensor-major. If boundary_thickness
// > 0 and trace_out != nullptr, trace_out receives [nt * n_shell] (step-major);
// n_shell_out gets the shell size. p_final_out (optional) receives the last pressure.
int ref_simulate_forward(const RefGrid* grid, const RefMedium* medium, const RefSources* sources,
                         size_t n_sensors, const size_t* sensor_pos, int boundary_thickness,
                         int pml_enabled, double* data_out, double* trace_out, size_t* n_shell_out) {
    return guarded([&] {
        const auto g = to_grid(grid);
        const auto med = to_medium(g, medium);
        ustfwi::SimOptions opt;
        opt.boundary_thickness = boundary_thickness;
        opt.pml_enabled = pml_enabled != 0;
        const auto res = ustfwi::simulate_forward(med, to_sources(sources),
                                                  to_sensors(n_sensors, sensor_pos), g, opt);
        std::memcpy(data_out, res.data.samples.data(), res.data.samples.size() * sizeof(double));
        if (n_shell_out) *n_shell_out = res.trace.layer_indices.size();
        if (trace_out)
            std::memcpy(trace_out, res.trace.values.data(), res.trace.values.size() * sizeof(double));
    });
}

// Time-reversal c0 gradient (the north-star hot path). observed: [n_sensors * nt].
int ref_gradient_tr(const RefGrid* grid, const RefMedium* medium, const RefSources* sources,
                    size_t n_sensors, const size_t* sensor_pos, const double* observed,
                    int boundary_thickness, double* grad_out, double* loss_out) {
    return guarded([&] {
        const auto g = to_grid(grid);
        const auto med = to_medium(g, medium);
        ustfwi::SensorData obs;
        obs.n_sensors = static_cast<int>(n_sensors);
        obs.nt = g.nt;
        obs.dt = g.dt;
        obs.samples.assign(observed, observed + n_sensors * static_cast<std::size_t>(g.nt));
        const auto res = ustfwi::gradient_time_reversal(med, to_sources(sources),
                                                        to_sensors(n_sensors, sensor_pos), obs, g,
                                                        boundary_thickness);
        std::memcpy(grad_out, res.grad.data(), g.points() * sizeof(double));
        *loss_out = res.loss;
    });
}

// compute_gradient (gradient.hpp:333-464), time-reversal method, GradientParam (0 c0, 1 rho0,
// 2 alpha0, 3 y), with the dispersion switch of GradientOptions (adjoint and replay steppers, gradient.hpp:22-32,381-384,424-431)
int ref_gradient_tr_opts(const RefGrid* grid, const RefMedium* medium, const RefSources* sources,
                         size_t n_sensors, const size_t* sensor_pos, const double* observed,
                         int boundary_thickness, int dispersion_enabled, int param, double* grad_out,
                         double* loss_out) {
    return guarded([&] {
        const auto g = to_grid(grid);
        const auto med = to_medium(g, medium);
        ustfwi::SensorData obs;
        obs.n_sensors = static_cast<int>(n_sensors);
        obs.nt = g.nt;
        obs.dt = g.dt;
        obs.samples.assign(observed, observed + n_sensors * static_cast<std::size_t>(g.nt));
        ustfwi::GradientOptions opt;
        opt.method = ustfwi::GradientMethod::time_reversal;
        opt.boundary_thickness = boundary_thickness;
        opt.dispersion_enabled = dispersion_enabled != 0;
        const auto res = ustfwi::compute_gradient(med, to_sources(sources), to_sensors(n_sensors, sensor_pos), obs,
                                                  g, static_cast<ustfwi::GradientParam>(param), opt);
        std::memcpy(grad_out, res.grad.data(), g.points() * sizeof(double));
        *loss_out = res.loss;
    });
}

int ref_evaluate_loss(const RefGrid* grid, const RefMedium* medium, const RefSources* sources,
                      size_t n_sensors, const size_t* sensor_pos, const double* observed,
                      double* loss_out) {
    return guarded([&] {
        const auto g = to_grid(grid);
        const auto med = to_medium(g, medium);
        ustfwi::SensorData obs;
        obs.n_sensors = static_cast<int>(n_sensors);
        obs.nt = g.nt;
        obs.dt = g.dt;
        obs.samples.assign(observed, observed + n_sensors * static_cast<std::size_t>(g.nt));
        *loss_out = ustfwi::evaluate_loss(med, to_sources(sources), to_sensors(n_sensors, sensor_pos),
                                          obs, g);
    });
}

// Steady-state step timing for the CPU baseline: builds one SpectralEngine and two
// WaveSteppers exactly as compute_gradient does and times `k_fwd` forward steps plus
// `k_pair` adjoint+replay pair-steps with the accumulator (gradient.hpp:443-454).
int ref_time_steps(const RefGrid* grid, const RefMedium* medium, int k_fwd, int k_pair,
                   double* sec_fwd_step, double* sec_pair_step) {
    return guarded([&] {
        const auto g = to_grid(grid);
        const auto med = to_medium(g, medium);
        ustfwi::SpectralEngine eng(g);
        ustfwi::WaveStepper fwd(g, med, eng);
        const std::size_t mid = g.points() / 2;
        auto t0 = std::chrono::steady_clock::now();
        for (int n = 0; n < k_fwd; ++n) {
            fwd.update_velocity_density();
            fwd.inject_mass_source(mid, n < 8 ? 1.0 : 0.0);
            fwd.update_pressure();
        }
        auto t1 = std::chrono::steady_clock::now();
        ustfwi::StepperOptions ropt;
        ropt.absorption_sign = -1.0;
        ustfwi::WaveStepper adj(g, med, eng);
        ustfwi::WaveStepper rep(g, med, eng, ropt);
        ustfwi::detail::GradientAccumulator acc(ustfwi::GradientParam::c0, med, g, eng, g.dt, true);
        acc.push(rep.pressure());
        acc.push(rep.pressure());
        auto t2 = std::chrono::steady_clock::now();
        for (int n = 0; n < k_pair; ++n) {
            adj.update_velocity_density();
            adj.inject_mass_source(mid, n < 8 ? 1.0 : 0.0);
            adj.update_pressure();
            rep.update_velocity_density();
            rep.update_pressure();
            acc.push(rep.pressure());
            acc.accumulate(adj.pressure());
        }
        auto t3 = std::chrono::steady_clock::now();
        *sec_fwd_step = k_fwd ? std::chrono::duration<double>(t1 - t0).count() / k_fwd : 0.0;
        *sec_pair_step = k_pair ? std::chrono::duration<double>(t3 - t2).count() / k_pair : 0.0;
    });
}

}  // extern "C"
