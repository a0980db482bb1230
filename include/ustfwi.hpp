// Umbrella header of the B200 drop-in for the reference's ustfwi hot path.
// Link: -L<repo>/paper_2102_00755_b200 -lustfwi_b200 (rpath to the same directory).
#pragma once
#include "ustfwi/core.hpp"
#include "ustfwi/solver.hpp"
#include "ustfwi/gradient.hpp"
#include "ustfwi/grid.hpp"
#include "ustfwi/io.hpp"
