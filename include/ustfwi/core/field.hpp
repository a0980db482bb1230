// Reference path core/field.hpp (Dims, Field, Mask, dot, norm2, max_abs, kahan_sum; field.hpp:14-153)
// of the B200 drop-in.
#pragma once
#include "../core.hpp"
