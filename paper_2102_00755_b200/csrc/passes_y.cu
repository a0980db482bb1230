// y pencil passes: the same kernels as passes.cu, compiled in their own translation unit with
// scalar complex add / subtract (USTFWI_FFT_SCALAR_ADD, see fft_smem.cuh): on B200 the packed
// FADD2 form makes the y pass slower while it speeds up the x pass and the z rows.
// Exports launch_pencil_fast_y(), called by launch_pencil_fast() for axis 1.
#define USTFWI_FFT_SCALAR_ADD 1
#define USTFWI_PASSES_Y_ONLY 1
#include "passes.cu"
