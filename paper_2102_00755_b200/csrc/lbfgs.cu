// Device-resident limited-memory BFGS state for SLBFGS (Algorithm 2, Appendix D;
// SPEC.md optimizer module: two_loop_recursion, curvature-pair buffer with m_h = 64).
//
// The S / Y history lives in HBM as fp64 rings ([m_h][n], the reference precision), the
// two-loop recursion runs as a chain of kernels with every scalar (rho_i, alpha_i, beta) kept
// on the device, so one direction costs 2*m dot products + 2*m axpys and no host round
// trip. Dot products are deterministic: fixed grid, fixed per-thread order, fixed-order
// block and final reductions (bit-identical across runs).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "host_setup.hpp"

namespace {

constexpr int kDotBlocks = 296;  // 2 x 148 SMs
constexpr int kThreads = 256;

// partial[b] = sum over this block's grid-stride share of a[i]*b[i]
__global__ void __launch_bounds__(kThreads) dot_partial_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                               long long n, double* __restrict__ partial) {
    __shared__ double sh[kThreads];
    double s = 0.0;
    for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n; i += (long long)gridDim.x * kThreads)
        s = fma(a[i], b[i], s);
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = kThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

// fixed-order sum of the block partials, then
// mode 0: out = sum
// mode 1: out = rho * sum                     (alpha_i = rho_i s_i.q ; beta = rho_i y_i.r)
// mode 2: out = alpha - rho * sum             (coefficient of s_i in the second loop)
__global__ void dot_final_kernel(const double* __restrict__ partial, int nb, double* __restrict__ out, int mode,
                                 const double* __restrict__ rho, const double* __restrict__ alpha) {
    __shared__ double sh[kThreads];
    double s = 0.0;
    for (int i = threadIdx.x; i < nb; i += kThreads) s += partial[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = kThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double d = sh[0];
        if (mode == 0) *out = d;
        else if (mode == 1) *out = *rho * d;
        else *out = *alpha - *rho * d;
    }
}

// y[i] += sign * (*coef) * x[i]
__global__ void axpy_dev_kernel(double* __restrict__ y, const double* __restrict__ x, long long n,
                                const double* __restrict__ coef, double sign) {
    const double a = sign * *coef;
    for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n; i += (long long)gridDim.x * kThreads)
        y[i] = fma(a, x[i], y[i]);
}

// y[i] = s * x[i] with s a host scalar or a device scalar
__global__ void scale_copy_kernel(double* __restrict__ y, const double* __restrict__ x, long long n, double s,
                                  const double* __restrict__ s_dev) {
    const double a = s_dev ? s * *s_dev : s;
    for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n; i += (long long)gridDim.x * kThreads)
        y[i] = a * x[i];
}

struct Fail {
    int code;
    std::string msg;
};

#define LCK(x)                                                                                    \
    do {                                                                                          \
        cudaError_t e_ = (x);                                                                     \
        if (e_ != cudaSuccess) throw Fail{USTFWI_ERR_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)}; \
    } while (0)

}  // namespace

struct ustfwi_lbfgs {
    int device = 0;
    long long n = 0;
    int m = 0;
    cudaStream_t st = nullptr;
    double* S = nullptr;      // [m][n]
    double* Y = nullptr;      // [m][n]
    double* q = nullptr;      // work vector
    double* r = nullptr;      // work vector / result
    double* partial = nullptr;
    double* scal = nullptr;   // rho[m], alpha[m], tmp[4], gamma
    int count = 0;            // stored pairs
    int head = 0;             // slot of the next pair
    double gamma = 1.0;       // H0 = gamma * I (latest <s,y>/<y,y>)
    std::vector<double> rho_h;

    double* rho() { return scal; }
    double* alpha() { return scal + m; }
    double* tmp() { return scal + 2 * m; }
    double* gam() { return scal + 2 * m + 4; }

    void dot(const double* a, const double* b, double* out, int mode = 0, const double* rho_p = nullptr,
             const double* alpha_p = nullptr) {
        dot_partial_kernel<<<kDotBlocks, kThreads, 0, st>>>(a, b, n, partial);
        dot_final_kernel<<<1, kThreads, 0, st>>>(partial, kDotBlocks, out, mode, rho_p, alpha_p);
        LCK(cudaGetLastError());
    }
    double dot_host(const double* a, const double* b) {
        dot(a, b, tmp());
        double v = 0.0;
        LCK(cudaMemcpyAsync(&v, tmp(), sizeof(double), cudaMemcpyDeviceToHost, st));
        LCK(cudaStreamSynchronize(st));
        return v;
    }
    unsigned blocks() const { return static_cast<unsigned>(std::min<long long>((n + kThreads - 1) / kThreads, 4 * 148)); }
    int slot(int j) const { return (head - 1 - j + 2 * m) % m; }  // j = 0 newest

    // r = H_k g for the device vector g (standard two-loop recursion, SPEC two_loop_recursion)
    void two_loop(const double* g) {
        LCK(cudaMemcpyAsync(q, g, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
        for (int j = 0; j < count; ++j) {  // newest -> oldest
            const int k = slot(j);
            dot(S + (long long)k * n, q, alpha() + k, 1, rho() + k);
            axpy_dev_kernel<<<blocks(), kThreads, 0, st>>>(q, Y + (long long)k * n, n, alpha() + k, -1.0);
        }
        scale_copy_kernel<<<blocks(), kThreads, 0, st>>>(r, q, n, 1.0, gam());
        for (int j = count - 1; j >= 0; --j) {  // oldest -> newest
            const int k = slot(j);
            dot(Y + (long long)k * n, r, tmp() + 1, 2, rho() + k, alpha() + k);  // alpha_k - beta
            axpy_dev_kernel<<<blocks(), kThreads, 0, st>>>(r, S + (long long)k * n, n, tmp() + 1, 1.0);
        }
        LCK(cudaGetLastError());
    }
};

namespace {
template <class Fn>
int lguard(ustfwi_lbfgs* h, Fn&& fn) {
    try {
        if (h) LCK(cudaSetDevice(h->device));
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
}  // namespace

extern "C" {

USTFWI_API int ustfwi_lbfgs_create(int device, size_t n, int history, ustfwi_lbfgs** out) {
    return lguard(nullptr, [&] {
        if (!out) throw Fail{USTFWI_ERR_INVALID, "null output handle"};
        *out = nullptr;
        if (n == 0) throw Fail{USTFWI_ERR_INVALID, "vector length must be positive"};
        if (history < 1) throw Fail{USTFWI_ERR_INVALID, "history size must be >= 1"};
        LCK(cudaSetDevice(device));
        auto* h = new ustfwi_lbfgs;
        h->device = device;
        h->n = static_cast<long long>(n);
        h->m = history;
        auto al = [&](double** p, size_t cnt) {
            cudaError_t e = cudaMalloc(p, cnt * sizeof(double));
            if (e != cudaSuccess) {
                ustfwi_lbfgs_destroy(h);
                throw Fail{e == cudaErrorMemoryAllocation ? USTFWI_ERR_OOM : USTFWI_ERR_CUDA,
                           std::string("lbfgs allocation: ") + cudaGetErrorString(e)};
            }
        };
        if (cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking) != cudaSuccess) {
            delete h;
            throw Fail{USTFWI_ERR_CUDA, "stream creation failed"};
        }
        al(&h->S, n * static_cast<size_t>(history));
        al(&h->Y, n * static_cast<size_t>(history));
        al(&h->q, n);
        al(&h->r, n);
        al(&h->partial, kDotBlocks);
        al(&h->scal, 2 * static_cast<size_t>(history) + 5);
        h->rho_h.assign(static_cast<size_t>(history), 0.0);
        const double one = 1.0;
        LCK(cudaMemcpy(h->gam(), &one, sizeof(double), cudaMemcpyHostToDevice));
        *out = h;
    });
}

USTFWI_API int ustfwi_lbfgs_destroy(ustfwi_lbfgs* h) {
    if (!h) return USTFWI_OK;
    cudaSetDevice(h->device);
    if (h->st) cudaStreamSynchronize(h->st);
    for (double* p : {h->S, h->Y, h->q, h->r, h->partial, h->scal})
        if (p) cudaFree(p);
    if (h->st) cudaStreamDestroy(h->st);
    delete h;
    return USTFWI_OK;
}

USTFWI_API int ustfwi_lbfgs_reset(ustfwi_lbfgs* h) {
    return lguard(h, [&] {
        h->count = 0;
        h->head = 0;
        h->gamma = 1.0;
        const double one = 1.0;
        LCK(cudaMemcpyAsync(h->gam(), &one, sizeof(double), cudaMemcpyHostToDevice, h->st));
        LCK(cudaStreamSynchronize(h->st));
    });
}

USTFWI_API int ustfwi_lbfgs_push(ustfwi_lbfgs* h, const double* s, const double* y, double reject_tol, int* accepted) {
    return lguard(h, [&] {
        if (!h || !s || !y) throw Fail{USTFWI_ERR_INVALID, "null argument"};
        const int k = h->head;
        // stage in the work vectors: a rejected pair must not clobber the oldest stored one
        double* sk = h->q;
        double* yk = h->r;
        // s, y: host or device pointers (unified addressing)
        LCK(cudaMemcpyAsync(sk, s, h->n * sizeof(double), cudaMemcpyDefault, h->st));
        LCK(cudaMemcpyAsync(yk, y, h->n * sizeof(double), cudaMemcpyDefault, h->st));
        const double sy = h->dot_host(sk, yk);
        const double ss = h->dot_host(sk, sk);
        const double yy = h->dot_host(yk, yk);
        // curvature condition <s,y> > tol * |s| |y| (SPEC optimizer design decisions)
        const bool ok = std::isfinite(sy) && sy > reject_tol * std::sqrt(ss) * std::sqrt(yy) && yy > 0.0;
        if (accepted) *accepted = ok ? 1 : 0;
        if (!ok) return;
        LCK(cudaMemcpyAsync(h->S + (long long)k * h->n, sk, h->n * sizeof(double), cudaMemcpyDeviceToDevice, h->st));
        LCK(cudaMemcpyAsync(h->Y + (long long)k * h->n, yk, h->n * sizeof(double), cudaMemcpyDeviceToDevice, h->st));
        const double rho = 1.0 / sy;
        h->gamma = sy / yy;
        LCK(cudaMemcpyAsync(h->rho() + k, &rho, sizeof(double), cudaMemcpyHostToDevice, h->st));
        LCK(cudaMemcpyAsync(h->gam(), &h->gamma, sizeof(double), cudaMemcpyHostToDevice, h->st));
        LCK(cudaStreamSynchronize(h->st));
        h->rho_h[static_cast<size_t>(k)] = rho;
        h->head = (h->head + 1) % h->m;
        h->count = std::min(h->count + 1, h->m);
    });
}

// out = H_k g (two-loop recursion); empty history: H0 g with H0 = I
USTFWI_API int ustfwi_lbfgs_apply(ustfwi_lbfgs* h, const double* g, double* out) {
    return lguard(h, [&] {
        if (!h || !g || !out) throw Fail{USTFWI_ERR_INVALID, "null argument"};
        // g, out: host or device pointers (unified addressing): with device vectors the
        // recursion never leaves HBM
        LCK(cudaMemcpyAsync(h->r, g, h->n * sizeof(double), cudaMemcpyDefault, h->st));
        h->two_loop(h->r);
        LCK(cudaMemcpyAsync(out, h->r, h->n * sizeof(double), cudaMemcpyDefault, h->st));
        LCK(cudaStreamSynchronize(h->st));
    });
}

USTFWI_API int ustfwi_lbfgs_pairs(const ustfwi_lbfgs* h, int* count, double* gamma) {
    if (!h) return USTFWI_ERR_INVALID;
    if (count) *count = h->count;
    if (gamma) *gamma = h->gamma;
    return USTFWI_OK;
}

}  // extern "C"
