// Multigrid transfer on the device:
//   fourier_interpolate   trigonometric resampling of a field with the optional separable
//                         Blackman taper (grid/spectral.hpp:117-212) — prolong_model
//   lowpass_timeseries    zero-phase Kaiser FIR low-pass of sampled series
//                         (grid/filter.hpp:13-101) — used by restrict_data
//   restrict_traces       restrict_data of SPEC.md:463-470 (spec only): Fourier resampling of
//                         each trace to ceil(nt/eta) samples, Kaiser low-pass, eta^(d-1) scale
//
// The N-D resampling is done one axis at a time: the reference resamples the full complex
// spectrum then inverts once; the operator is a tensor product of per-axis operators (the
// Nyquist split / fold rule of resample_spectrum_axis, the Blackman window and the size
// ratio all factor per axis), so the per-axis passes give the same result up to rounding.
// Each pass: TB lines per CTA in a line-fast shared-memory tile, Stockham FFT of length n,
// deterministic serial redistribution of the n bins into m per line, taper, inverse FFT of
// length m, real part out.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "fft_smem.cuh"
#include "host_setup.hpp"

namespace {

using ustfwi_dev::FftPlan;

constexpr int kTBMax = 16;     // lines per CTA (fewer for long lines: shared-memory bound)
constexpr int kThreads = 256;

struct Geom {
    long long nlines;  // pre * post
    long long post;    // stride of the axis (elements)
    int n, m;          // source / target length along the axis
};

__global__ void __launch_bounds__(kThreads) resample_axis_kernel(const float* __restrict__ in, float* __restrict__ out,
                                                                 Geom G, FftPlan pn, FftPlan pm,
                                                                 const float* __restrict__ win, float scale, int tb) {
    extern __shared__ float2 sm[];
    const int Lmax = max(G.n, G.m);
    float2* A = sm;
    float2* B = A + tb * Lmax;
    float2* Cb = B + tb * Lmax;
    const long long l0 = (long long)blockIdx.x * tb;
    const int nl = (int)min((long long)tb, G.nlines - l0);
    auto base = [&](long long l, int len) { return (l / G.post) * (long long)len * G.post + (l % G.post); };

    for (int t = threadIdx.x; t < tb * G.n; t += blockDim.x) {
        const int j = t / tb, i = t % tb;
        float v = 0.f;
        if (i < nl) v = in[base(l0 + i, G.n) + (long long)j * G.post];
        A[j * tb + i] = make_float2(v, 0.f);
    }
    __syncthreads();
    float2* spec = ustfwi_dev::smem_fft<false, true>(A, B, Cb, pn, tb, 1, tb);
    float2* T = (spec == B) ? Cb : B;
    for (int t = threadIdx.x; t < tb * G.m; t += blockDim.x) T[t] = make_float2(0.f, 0.f);
    __syncthreads();
    // resample_spectrum_axis (spectral.hpp:121-158): split the source Nyquist bin on
    // upsampling, fold +-m/2 into bin m/2 on downsampling; serial per line (fixed order)
    if (threadIdx.x < tb) {
        const int i = threadIdx.x;
        const int n = G.n, m = G.m;
        auto deposit = [&](int freq, float w, float2 v) {
            if (2 * abs(freq) > m) return;
            int bin = freq;
            if (2 * abs(freq) == m) bin = m / 2;
            if (bin < 0) bin += m;
            float2& d = T[bin * tb + i];
            d.x += w * v.x;
            d.y += w * v.y;
        };
        for (int j = 0; j < n; ++j) {
            const float2 v = spec[j * tb + i];
            if (n % 2 == 0 && j == n / 2) {
                deposit(n / 2, 0.5f, v);
                deposit(-n / 2, 0.5f, v);
            } else {
                deposit((2 * j < n) ? j : j - n, 1.f, v);
            }
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < tb * G.m; t += blockDim.x) {
        const int k = t / tb;
        const float w = scale * (win ? win[k] : 1.f);
        T[t].x *= w;
        T[t].y *= w;
    }
    __syncthreads();
    float2* res = ustfwi_dev::smem_fft<true, true>(T, A, spec, pm, tb, 1, tb);
    for (int t = threadIdx.x; t < tb * G.m; t += blockDim.x) {
        const int k = t / tb, i = t % tb;
        if (i < nl) out[base(l0 + i, G.m) + (long long)k * G.post] = res[t].x;
    }
}

// out[s][i] = sum_t h[t] * sig[s][i + delay - t]  (fft_convolve + delay shift, filter.hpp:71-101)
__global__ void fir_kernel(const float* __restrict__ sig, float* __restrict__ out, long long n_series, int len,
                           const float* __restrict__ h, int taps) {
    const int delay = (taps - 1) / 2;
    const long long total = n_series * len;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long s = e / len;
        const int i = (int)(e % len);
        const float* x = sig + s * len;
        float acc = 0.f;
        const int k = i + delay;  // full-convolution index
        const int t0 = max(0, k - (len - 1)), t1 = min(taps - 1, k);
        for (int t = t0; t <= t1; ++t) acc = fmaf(h[t], x[k - t], acc);
        out[e] = acc;
    }
}

struct Fail {
    int code;
    std::string msg;
};

#define RCK(x)                                                                                    \
    do {                                                                                          \
        cudaError_t e_ = (x);                                                                     \
        if (e_ != cudaSuccess) throw Fail{USTFWI_ERR_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)}; \
    } while (0)

// device allocations released at scope exit
struct Pool {
    std::vector<void*> p;
    template <class T>
    T* alloc(size_t n) {
        void* q = nullptr;
        cudaError_t e = cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T));
        if (e != cudaSuccess)
            throw Fail{e == cudaErrorMemoryAllocation ? USTFWI_ERR_OOM : USTFWI_ERR_CUDA,
                       std::string("allocation: ") + cudaGetErrorString(e)};
        p.push_back(q);
        return static_cast<T*>(q);
    }
    ~Pool() {
        for (void* q : p) cudaFree(q);
    }
};

FftPlan plan_for(Pool& pool, int L, cudaStream_t st) {
    FftPlan p{};
    p.L = L;
    int m = L;
    auto take = [&](int r) {
        while (m % r == 0 && p.nstages < ustfwi_dev::kMaxStages) {
            p.radix[p.nstages++] = r;
            m /= r;
        }
    };
    take(16);
    take(8);
    take(4);
    take(2);
    take(5);
    take(3);
    take(7);
    for (int f = 11; m > 1 && p.nstages < ustfwi_dev::kMaxStages; f += 2) take(f);
    if (m != 1) throw Fail{USTFWI_ERR_INVALID, "transform length " + std::to_string(L) + " has too many factors"};
    std::vector<float2> tw(static_cast<size_t>(L));
    for (int k = 0; k < L; ++k) {
        const double a = -2.0 * M_PI * static_cast<double>(k) / static_cast<double>(L);
        tw[static_cast<size_t>(k)] = make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
    }
    float2* d = pool.alloc<float2>(tw.size());
    RCK(cudaMemcpyAsync(d, tw.data(), tw.size() * sizeof(float2), cudaMemcpyHostToDevice, st));
    p.tw = d;
    return p;
}

// one axis of `in` (dims) -> `out` (dims with axis resized to m)
void resample_axis(Pool& pool, const float* in, float* out, const std::vector<long long>& dims, int axis, int m,
                   bool blackman, cudaStream_t st) {
    const int n = static_cast<int>(dims[static_cast<size_t>(axis)]);
    long long pre = 1, post = 1;
    for (int a = 0; a < axis; ++a) pre *= dims[static_cast<size_t>(a)];
    for (size_t a = static_cast<size_t>(axis) + 1; a < dims.size(); ++a) post *= dims[a];
    Geom G{pre * post, post, n, m};
    FftPlan pn = plan_for(pool, n, st), pm = plan_for(pool, m, st);
    float* win = nullptr;
    if (blackman) {  // spectral.hpp:196-205, per target axis
        std::vector<float> w(static_cast<size_t>(m));
        for (int k = 0; k < m; ++k) {
            int freq = k;
            if (2 * freq > m) freq -= m;
            const double x = M_PI * static_cast<double>(freq) / (m / 2);
            w[static_cast<size_t>(k)] = static_cast<float>(0.42 + 0.5 * std::cos(x) + 0.08 * std::cos(2.0 * x));
        }
        win = pool.alloc<float>(w.size());
        RCK(cudaMemcpyAsync(win, w.data(), w.size() * sizeof(float), cudaMemcpyHostToDevice, st));
    }
    const size_t per_line = 3 * static_cast<size_t>(std::max(n, m)) * sizeof(float2);
    const int tb = static_cast<int>(std::min<size_t>(kTBMax, (227 * 1024) / per_line));
    if (tb < 1) throw Fail{USTFWI_ERR_INVALID, "resampling length too large"};
    const size_t smem = per_line * static_cast<size_t>(tb);
    RCK(cudaFuncSetAttribute(resample_axis_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const long long blocks = (G.nlines + tb - 1) / tb;
    // scale m/n of the size ratio (spectral.hpp:207) and 1/m of the normalised inverse
    resample_axis_kernel<<<static_cast<unsigned>(blocks), kThreads, smem, st>>>(in, out, G, pn, pm, win,
                                                                              static_cast<float>(1.0 / n), tb);
    RCK(cudaGetLastError());
}

// design_kaiser_lowpass (filter.hpp:39-66), fp64 on the host
std::vector<double> kaiser_lowpass(double dt, double cutoff_hz, double transition, double atten_db) {
    const double nyquist = 0.5 / dt;
    if (!(cutoff_hz > 0.0) || cutoff_hz > nyquist) throw Fail{USTFWI_ERR_INVALID, "cutoff must lie in (0, Nyquist]"};
    auto i0 = [](double x) {
        double sum = 1.0, term = 1.0;
        const double x2 = x * x / 4.0;
        for (int k = 1; k < 64; ++k) {
            term *= x2 / (static_cast<double>(k) * k);
            sum += term;
            if (term < 1e-18 * sum) break;
        }
        return sum;
    };
    const double beta = atten_db > 50.0 ? 0.1102 * (atten_db - 8.7)
                        : atten_db >= 21.0 ? 0.5842 * std::pow(atten_db - 21.0, 0.4) + 0.07886 * (atten_db - 21.0)
                                           : 0.0;
    const double width_hz = transition * cutoff_hz;
    const double dw = 2.0 * M_PI * width_hz * dt;
    int half = static_cast<int>(std::ceil((atten_db - 7.95) / (2.285 * dw) / 2.0));
    half = std::max(half, 4);
    const int len = 2 * half + 1;
    const double i0b = i0(beta);
    const double wc = 2.0 * M_PI * (cutoff_hz + 0.5 * width_hz) * dt;
    std::vector<double> h(static_cast<size_t>(len));
    double sum = 0.0;
    for (int k = 0; k < len; ++k) {
        const double mm = k - half;
        const double ideal = (mm == 0.0) ? wc / M_PI : std::sin(wc * mm) / (M_PI * mm);
        const double r = mm / half;
        h[static_cast<size_t>(k)] = ideal * i0(beta * std::sqrt(std::max(0.0, 1.0 - r * r))) / i0b;
        sum += h[static_cast<size_t>(k)];
    }
    for (double& v : h) v /= sum;
    return h;
}

void lowpass_dev(Pool& pool, const float* in, float* out, long long n_series, int len, double dt, double cutoff,
                 double transition, double atten_db, cudaStream_t st) {
    const auto h = kaiser_lowpass(dt, cutoff, transition, atten_db);
    std::vector<float> hf(h.begin(), h.end());
    float* hd = pool.alloc<float>(hf.size());
    RCK(cudaMemcpyAsync(hd, hf.data(), hf.size() * sizeof(float), cudaMemcpyHostToDevice, st));
    const long long total = n_series * len;
    const unsigned blocks = static_cast<unsigned>(std::min<long long>((total + 255) / 256, 4 * 148 * 8));
    fir_kernel<<<std::max(blocks, 1u), 256, 0, st>>>(in, out, n_series, len, hd, static_cast<int>(hf.size()));
    RCK(cudaGetLastError());
}

template <class Fn>
int rguard(int device, Fn&& fn) {
    try {
        // argument checks run before the device is touched (std::invalid_argument semantics
        // hold without a GPU); the bodies select the device with use_device()
        (void)device;
        fn();
        return USTFWI_OK;
    } catch (const Fail& f) {
        ustfwi_host::set_last_error(f.msg);
        return f.code;
    } catch (const std::bad_alloc&) {
        ustfwi_host::set_last_error("host allocation failed");
        return USTFWI_ERR_OOM;
    }
}

struct Stream {
    cudaStream_t s = nullptr;
    Stream() { RCK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
    ~Stream() {
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    }
};

}  // namespace

extern "C" {

USTFWI_API int ustfwi_fourier_interpolate(int device, int ndim, const int* dims, const double* field,
                                          const int* new_dims, int blackman, double* out) {
    return rguard(device, [&] {
        if (ndim < 1 || ndim > 3 || !dims || !new_dims || !field || !out)
            throw Fail{USTFWI_ERR_INVALID, "target dimensionality mismatch"};
        for (int a = 0; a < ndim; ++a) {  // spectral.hpp:171-178
            if (new_dims[a] < 4 || new_dims[a] % 2 != 0)
                throw Fail{USTFWI_ERR_INVALID, "target dims must be even and >= 4"};
            if (dims[a] % 2 != 0) throw Fail{USTFWI_ERR_INVALID, "source dims must be even"};
        }
        RCK(cudaSetDevice(device));
        Stream st;
        Pool pool;
        std::vector<long long> cur(dims, dims + ndim);
        long long n_in = 1, n_max = 1;
        for (int a = 0; a < ndim; ++a) n_in *= dims[a];
        {
            std::vector<long long> d = cur;
            for (int a = ndim - 1; a >= 0; --a) {
                d[static_cast<size_t>(a)] = new_dims[a];
                long long t = 1;
                for (long long v : d) t *= v;
                n_max = std::max(n_max, t);
            }
        }
        n_max = std::max(n_max, n_in);
        std::vector<float> h(static_cast<size_t>(n_in));
        for (long long i = 0; i < n_in; ++i) h[static_cast<size_t>(i)] = static_cast<float>(field[i]);
        float* buf[2] = {pool.alloc<float>(static_cast<size_t>(n_max)), pool.alloc<float>(static_cast<size_t>(n_max))};
        RCK(cudaMemcpyAsync(buf[0], h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice, st.s));
        int src = 0;
        for (int a = ndim - 1; a >= 0; --a) {  // z first: contiguous lines
            if (cur[static_cast<size_t>(a)] == new_dims[a] && !blackman) continue;
            resample_axis(pool, buf[src], buf[1 - src], cur, a, new_dims[a], blackman != 0, st.s);
            cur[static_cast<size_t>(a)] = new_dims[a];
            src = 1 - src;
        }
        long long n_out = 1;
        for (long long v : cur) n_out *= v;
        std::vector<float> o(static_cast<size_t>(n_out));
        RCK(cudaMemcpyAsync(o.data(), buf[src], o.size() * sizeof(float), cudaMemcpyDeviceToHost, st.s));
        RCK(cudaStreamSynchronize(st.s));
        for (long long i = 0; i < n_out; ++i) out[i] = o[static_cast<size_t>(i)];
    });
}

USTFWI_API int ustfwi_lowpass_timeseries(int device, size_t n_series, size_t len, const double* sig, double dt,
                                         double cutoff_hz, double transition, double atten_db, double* out) {
    return rguard(device, [&] {
        if (!(cutoff_hz > 0.0) || cutoff_hz > 0.5 / dt)
            throw Fail{USTFWI_ERR_INVALID, "cutoff must lie in (0, Nyquist]"};
        if (len == 0 || n_series == 0) return;
        RCK(cudaSetDevice(device));
        Stream st;
        Pool pool;
        const size_t n = n_series * len;
        std::vector<float> h(n);
        for (size_t i = 0; i < n; ++i) h[i] = static_cast<float>(sig[i]);
        float* a = pool.alloc<float>(n);
        float* b = pool.alloc<float>(n);
        RCK(cudaMemcpyAsync(a, h.data(), n * sizeof(float), cudaMemcpyHostToDevice, st.s));
        lowpass_dev(pool, a, b, static_cast<long long>(n_series), static_cast<int>(len), dt, cutoff_hz, transition,
                    atten_db, st.s);
        RCK(cudaMemcpyAsync(h.data(), b, n * sizeof(float), cudaMemcpyDeviceToHost, st.s));
        RCK(cudaStreamSynchronize(st.s));
        for (size_t i = 0; i < n; ++i) out[i] = h[i];
    });
}

USTFWI_API int ustfwi_restrict_traces(int device, size_t n_series, size_t nt, const double* data, int eta, int ndim,
                                      double dt_fine, double cutoff_hz, double* out, size_t* nt_out) {
    return rguard(device, [&] {
        if (eta < 1) throw Fail{USTFWI_ERR_INVALID, "eta must be >= 1"};
        if (ndim < 1 || ndim > 3) throw Fail{USTFWI_ERR_INVALID, "ndim must be 1, 2 or 3"};
        const size_t ntc = (nt + static_cast<size_t>(eta) - 1) / static_cast<size_t>(eta);
        if (nt_out) *nt_out = ntc;
        if (!out) return;  // size query
        if (eta == 1) {  // identity
            std::copy(data, data + n_series * nt, out);
            return;
        }
        RCK(cudaSetDevice(device));
        Stream st;
        Pool pool;
        // zero-pad every trace to ntc * eta samples so that the Fourier resampling to ntc
        // points keeps the coarse spacing exactly eta * dt_fine (nt need not divide by eta)
        const size_t ntp = ntc * static_cast<size_t>(eta);
        const size_t n = n_series * ntp, nc = n_series * ntc;
        std::vector<float> h(std::max(n, nc), 0.f);
        for (size_t s = 0; s < n_series; ++s)
            for (size_t i = 0; i < nt; ++i) h[s * ntp + i] = static_cast<float>(data[s * nt + i]);
        float* a = pool.alloc<float>(n);
        float* b = pool.alloc<float>(nc);
        float* c = pool.alloc<float>(nc);
        RCK(cudaMemcpyAsync(a, h.data(), n * sizeof(float), cudaMemcpyHostToDevice, st.s));
        // Fourier resampling of each trace to the coarse sampling, then the Kaiser low-pass
        resample_axis(pool, a, b, {static_cast<long long>(n_series), static_cast<long long>(ntp)}, 1,
                      static_cast<int>(ntc), false, st.s);
        lowpass_dev(pool, b, c, static_cast<long long>(n_series), static_cast<int>(ntc), dt_fine * eta, cutoff_hz,
                    0.1, 60.0, st.s);
        RCK(cudaMemcpyAsync(h.data(), c, nc * sizeof(float), cudaMemcpyDeviceToHost, st.s));
        RCK(cudaStreamSynchronize(st.s));
        // amplitude scale eta^(d-1) (Appendix C)
        const double scale = std::pow(static_cast<double>(eta), ndim - 1);
        for (size_t i = 0; i < nc; ++i) out[i] = scale * h[i];
    });
}

}  // extern "C"
