// Drop-in check: reference-style code (test_solver.cpp / gradient.hpp call shapes)
// compiled against include/ustfwi.hpp and run on the device engine.
// Build: g++ -std=c++20 -I include tests/cpp/dropin_test.cpp -L paper_2102_00755_b200 -lustfwi_b200
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "ustfwi.hpp"

using namespace ustfwi;

#define EXPECT(c)                                                              \
    do {                                                                       \
        if (!(c)) {                                                            \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
            std::exit(1);                                                      \
        }                                                                      \
    } while (0)

static std::size_t flat3(const Grid& g, int x, int y, int z) {
    return (static_cast<std::size_t>(x) * g.dims[1] + y) * g.dims[2] + z;
}

int main() {
    // grid setup (grid.hpp:91-103) and choose_pml_size known answers (test_grid.cpp:26-31)
    EXPECT(choose_pml_size({44}) == Dims{10});
    EXPECT(choose_pml_size({100}) == Dims{14});
    Grid g = make_grid({28, 28, 28}, 1e-3, 1800.0, 3e-5);
    EXPECT(g.dims == (Dims{64, 64, 64}));  // 28 + 2*18: the 2-smooth padding
    Medium m = make_homogeneous_medium(g);
    auto pulse = synth_source_pulse(g, 0.8, 1500.0);
    SpectralEngine eng(g);

    // zero sources -> zero data (test_solver.cpp:50-58)
    SensorArray sensors;
    sensors.positions = {flat3(g, 30, 30, 30), flat3(g, 20, 26, 22)};
    {
        auto r = simulate_forward(m, SourceSet{}, sensors, g, {}, &eng);
        for (double v : r.data.samples) EXPECT(v == 0.0);
    }
    // linearity (test_solver.cpp:82-119), fp32 tolerance
    SourceSet s1, s2, both;
    s1.positions = {flat3(g, 18, 20, 24)};
    s1.signals = {pulse};
    auto pulse2 = pulse;
    for (double& v : pulse2) v *= -0.7;
    s2.positions = {flat3(g, 24, 18, 20)};
    s2.signals = {pulse2};
    both.positions = {s1.positions[0], s2.positions[0]};
    both.signals = {pulse, pulse2};
    auto r1 = simulate_forward(m, s1, sensors, g, {}, &eng);
    auto r2 = simulate_forward(m, s2, sensors, g, {}, &eng);
    auto rb = simulate_forward(m, both, sensors, g, {}, &eng);
    double num = 0, den = 0;
    for (int n = 0; n < g.nt; ++n)
        for (int s = 0; s < 2; ++s) {
            const double sum = r1.data.at(s, n) + r2.data.at(s, n);
            num += (rb.data.at(s, n) - sum) * (rb.data.at(s, n) - sum);
            den += sum * sum;
        }
    EXPECT(den > 0 && std::sqrt(num / den) < 1e-5);

    // TR gradient (gradient.hpp:478-488): zero residual -> zero gradient; gradient zero outside gamma
    m.gamma = ball_mask(g.dims, {32, 32, 32}, 9.0);
    SensorData obs = r1.data;
    auto gr = gradient_time_reversal(m, s1, sensors, obs, g, 4, GradientParam::c0, &eng);
    EXPECT(gr.loss == 0.0 && max_abs(gr.grad) == 0.0);
    for (double& v : obs.samples) v = 0.0;
    gr = gradient_time_reversal(m, s1, sensors, obs, g, 4, GradientParam::c0, &eng);
    EXPECT(gr.loss > 0.0 && max_abs(gr.grad) > 0.0 && gr.n_simulations == 3);
    for (std::size_t i = 0; i < gr.grad.size(); ++i)
        if (!m.gamma[i]) EXPECT(gr.grad[i] == 0.0);
    // error convention: CFL violation -> NumericalError (engine.hpp:196-197)
    Grid bad = g;
    bad.dt = 1e-3 / 1500.0;
    bool threw = false;
    try {
        SpectralEngine e2(bad);
        simulate_forward(make_homogeneous_medium(bad), s1, sensors, bad, {}, &e2);
    } catch (const NumericalError&) {
        threw = true;
    }
    EXPECT(threw);
    // encoding: identity for n_s = 1, w = +1, tau = 0 is a plain SourceSet
    auto real = draw_realization(3, 0.0, g.dt, 20210201, 0, 7);
    auto real2 = draw_realization(3, 0.0, g.dt, 20210201, 0, 7);
    EXPECT(real.weights == real2.weights);
    // alpha0 gradient (GradientParam::alpha0) through the same call shape
    {
        SensorData zero = obs;
        auto ga = gradient_time_reversal(m, s1, sensors, zero, g, 4, GradientParam::alpha0, &eng);
        EXPECT(ga.loss > 0.0 && max_abs(ga.grad) > 0.0);
        // rho0 gradient (GradientParam::rho0, gradient.hpp:117-128,213-239)
        auto gr0 = gradient_time_reversal(m, s1, sensors, zero, g, 4, GradientParam::rho0, &eng);
        EXPECT(gr0.loss > 0.0 && max_abs(gr0.grad) > 0.0);
        // GradientOptions default method is full_storage (gradient.hpp:23): rejected, never
        // silently replaced; gradient_full_storage (gradient.hpp:466-476) throws the same way
        bool fs_threw = false;
        try {
            compute_gradient(m, s1, sensors, zero, g, GradientParam::c0, GradientOptions{}, &eng);
        } catch (const std::invalid_argument&) {
            fs_threw = true;
        }
        EXPECT(fs_threw);
        fs_threw = false;
        try {
            gradient_full_storage(m, s1, sensors, zero, g, GradientParam::c0, 1, &eng);
        } catch (const std::invalid_argument&) {
            fs_threw = true;
        }
        EXPECT(fs_threw);
    }
    // multigrid transfer (grid/spectral.hpp, grid/filter.hpp): up-down round trip, DC gain
    {
        Field f({8, 6, 10});
        for (std::size_t i = 0; i < f.size(); ++i) f[i] = std::sin(0.37 * static_cast<double>(i));
        Field up = fourier_interpolate(f, {16, 12, 20});
        Field back = fourier_interpolate(up, {8, 6, 10});
        double e = 0, n = 0;
        for (std::size_t i = 0; i < f.size(); ++i) {
            e += (back[i] - f[i]) * (back[i] - f[i]);
            n += f[i] * f[i];
        }
        EXPECT(std::sqrt(e / n) < 1e-5);
        std::vector<double> c(600, 0.5);
        auto lp = lowpass_filter_timeseries(c, 1e-7, 1e6);
        EXPECT(std::abs(lp[300] - 0.5) < 1e-5);
    }
    // SLBFGS curvature history: one secant pair of a 1-D quadratic gives H g = g / a
    {
        LbfgsState H(1);
        EXPECT(H.push({-1.5}, {-1.5 * 3.7}));
        EXPECT(std::abs(H.apply({1.3})[0] - 1.3 / 3.7) < 1e-15);
    }
    std::printf("dropin_test: all checks passed (nt=%d, loss=%.6e)\n", g.nt, gr.loss);
    return 0;
}
