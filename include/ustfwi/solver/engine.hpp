// Reference path solver/engine.hpp (SpectralEngine, StepperOptions, WaveStepper,
// apply_axis_profile; engine.hpp:17-386) of the B200 drop-in: the engine and its steppers live on
// the device (libustfwi_b200.so).
#pragma once
#include "../solver.hpp"
