// Reference path grid/spectral.hpp (Stagger, SpectralWindow, spectral_derivative, fourier_shift,
// fourier_interpolate; spectral.hpp:10-212) of the B200 drop-in. fourier_interpolate runs on the
// device (multigrid transfer, csrc/resample.cu); the others are fp64 host setup utilities.
#pragma once
#include "../spectral.hpp"
#include "../grid.hpp"
