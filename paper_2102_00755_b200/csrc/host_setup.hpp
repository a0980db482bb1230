// Host-side setup shared by the C ABI and the device engine (C++17, fp64).
#pragma once

#include <cstdint>
#include <string>
#include <algorithm>
#include <thread>
#include <vector>

#include "../../include/ustfwi_capi.h"

namespace ustfwi_host {

// Thrown inside the library and mapped to USTFWI_ERR_* at the C boundary.
struct Error {
    int code;
    std::string msg;
};
[[noreturn]] void fail(int code, const std::string& msg);
void set_last_error(const std::string& msg);

std::string dims_str(const int* dims, int ndim);

void validate_grid(const ustfwi_grid& g);                       // grid.hpp:35-51
long largest_prime_factor(long n);                              // grid.hpp:55-64
std::vector<int> choose_pml_size(const std::vector<int>& interior);   // grid.hpp:70-86
ustfwi_grid make_grid(const std::vector<int>& interior, double dx, double c_max, double duration,
                      double cfl);                              // grid.hpp:91-103
// FFT-ordered angular wavenumbers, Nyquist negative (fft.hpp:121-130)
std::vector<double> wavenumbers(int n, double dx);
// exp(-sigma dt/2) profiles on the regular / staggered grid of one axis (grid.hpp:153-178)
void pml_profiles(const ustfwi_grid& g, int axis, double alpha, std::vector<double>& regular,
                  std::vector<double>& staggered);
double sinc(double x);                                          // grid.hpp:106-109

std::vector<uint8_t> erode(const std::vector<uint8_t>& mask, const std::vector<int>& dims);
std::vector<size_t> shell_indices(const std::vector<uint8_t>& mask, const std::vector<int>& dims,
                                  int thickness);               // medium.hpp:137-178
std::vector<double> synth_source_pulse(const ustfwi_grid& g, double frac, double c0_min);

// fn(begin, end) over [0, n) in contiguous chunks on up to hardware_concurrency threads
// (host-side field conversions at the API boundary; ~59M elements at config D)
template <class Fn>
void parallel_chunks(size_t n, Fn&& fn) {
    const size_t hw = std::max<size_t>(1, std::thread::hardware_concurrency());
    const size_t nt = std::min<size_t>(hw, std::max<size_t>(1, n / (1u << 20)));
    if (nt <= 1) {
        fn(size_t{0}, n);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(nt);
    const size_t step = (n + nt - 1) / nt;
    for (size_t t = 0; t < nt; ++t) {
        const size_t b = t * step, e = std::min(n, b + step);
        if (b < e) th.emplace_back([&fn, b, e] { fn(b, e); });
    }
    for (auto& x : th) x.join();
}

// counter-based realization stream (SPEC.md stochastic_estimators RNG contract)
uint64_t stream_word(uint64_t master_seed, uint64_t iteration, uint64_t index, uint64_t counter);

}  // namespace ustfwi_host
