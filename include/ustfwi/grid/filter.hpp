// Reference path grid/filter.hpp (design_kaiser_lowpass, fft_convolve, lowpass_filter_timeseries;
// filter.hpp:38-101) of the B200 drop-in (the low-pass runs on the device, csrc/resample.cu).
#pragma once
#include "../spectral.hpp"
#include "../grid.hpp"
