// Reference path solver/simulate.hpp (SimOptions, SimResult, simulate_forward, field_power,
// synth_source_pulse; simulate.hpp:10-148) of the B200 drop-in.
#pragma once
#include "../grid.hpp"
#include "../solver.hpp"
