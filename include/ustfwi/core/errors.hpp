// Reference path core/errors.hpp (NumericalError, ToleranceError; errors.hpp:10-17) of the B200 drop-in.
#pragma once
#include "../core.hpp"
