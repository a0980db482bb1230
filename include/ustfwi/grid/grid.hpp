// Reference path grid/grid.hpp (Grid, choose_pml_size, make_grid, sinc, KVectors, make_kvectors,
// make_pml; grid.hpp:14-178) of the B200 drop-in.
#pragma once
#include "../core.hpp"
#include "../spectral.hpp"
