// Reference path core/fft.hpp (RealFft, ComplexFft, fft_wavenumbers; fft.hpp:23-130) of the B200
// drop-in: fp64 host transforms for setup utilities (the device engine has its own kernels).
#pragma once
#include "../spectral.hpp"
