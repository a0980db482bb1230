// Reference path adjoint/gradient.hpp (GradientParam, GradientMethod, GradientOptions,
// GradientResult, compute_gradient, gradient_full_storage, gradient_time_reversal, evaluate_loss;
// gradient.hpp:9-505) of the B200 drop-in, plus the SPEC source-encoding estimators.
#pragma once
#include "../grid.hpp"
#include "../gradient.hpp"
