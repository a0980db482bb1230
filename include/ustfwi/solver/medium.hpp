// Reference path solver/medium.hpp (Medium, SourceSet, SensorArray, SensorData, BoundaryTrace,
// erode, shell_indices, ball_mask; medium.hpp:15-198) of the B200 drop-in.
#pragma once
#include "../solver.hpp"
