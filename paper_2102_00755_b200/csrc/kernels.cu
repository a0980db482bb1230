// Pass kernels of one k-space leapfrog step (sm_100a).
//
// The reference's WaveStepper step (engine.hpp:270-347) does 4 r2c + 6 c2r 3-D FFTs plus
// ~16 full-field elementwise sweeps. Here a step is 8 launches over 3 "pass" kinds:
//
//   Y pass  complex FFT along y of [ny][TB]-column tiles (kz chunk), optional ky multiplier
//   X pass  FFT_x -> multiply by kappa(|k|) * D_x(kx) -> IFFT_x, one input, 1..3 outputs
//   Z pass  row-local half-length complex FFT for r2c/c2r along the contiguous z axis,
//           FUSED with the elementwise velocity (Z-vel) or density/pressure (Z-rho)
//           updates, split-field PML, sparse source injection / shell enforcement,
//           sensor and shell gathers and the in-kernel c0 gradient correlation.
//
// kappa and the stagger phases are evaluated on the fly from per-axis tables, so no
// half-spectrum multiplier array (9 complex fields at fp64 in the reference,
// engine.hpp:46-78) is ever read from HBM.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "kernels.cuh"

namespace ustfwi_dev {

// ---------------------------------------------------------------------------------
// Pencil passes (Y and X)
// ---------------------------------------------------------------------------------

__device__ __forceinline__ float kappa_of(float k2, float half_cdt) {
    // sinc(0.5*c_ref*dt*|k|) with the series branch of grid.hpp:106-109
    const float x = half_cdt * sqrtf(k2);
    return (x < 1e-4f) ? 1.f - x * x * (1.f / 6.f) : sinf(x) / x;
}

// AXIS 1: y pencils (tile at fixed x = blockIdx.y), AXIS 0: x pencils (fixed y).
// INV selects the direction of the Y pass; the X pass is always forward-multiply-inverse.
template <int AXIS, int TB, bool INV>
__global__ void __launch_bounds__(256) pencil_pass_kernel(GridDev g, PencilJobs jobs) {
    extern __shared__ float2 smem[];
    const FftPlan& plan = AXIS == 0 ? g.px : g.py;
    const int L = plan.L;
    float2* buf[3] = {smem, smem + L * TB, smem + 2 * L * TB};
    float* kap = reinterpret_cast<float*>(smem + 3 * L * TB);

    const int c0 = blockIdx.x * TB;
    const int ncol = min(TB, g.nzh - c0);
    const long long pitch = (AXIS == 0) ? (long long)g.ny * g.nzp : (long long)g.nzp;
    const long long base = (AXIS == 0) ? (long long)blockIdx.y * g.nzp + c0
                                       : (long long)blockIdx.y * g.ny * g.nzp + c0;
    const int n_el = L * TB;

    if (AXIS == 0) {
        // kappa (or |k|^e) for the tile: k = (kx[j], ky[y], kz[c0 + c]); one multiplier kind
        // per launch
        const float ky = g.ky[blockIdx.y];
        const int kind = jobs.job[0].kappa;
        const bool power = kind >= 2;
        const float e = jobs.job[0].kexp;
        for (int t = threadIdx.x; t < n_el; t += blockDim.x) {
            const int j = t / TB, c = t % TB;
            const float kx = g.kx[j];
            const float kz = (c < ncol) ? g.kz[c0 + c] : 0.f;
            const float k2 = kx * kx + ky * ky + kz * kz;
            kap[t] = power ? kpow_mult(k2, e, kind) : kappa_of(k2, g.half_cdt);
        }
    }

    int loaded = -1;
    float2* spec = nullptr;  // X pass: forward spectrum of the loaded source
    for (int jb = 0; jb < jobs.n; ++jb) {
        const PencilJob jbk = jobs.job[jb];
        if (jbk.src != loaded) {
            const float2* s = jobs.buf[jbk.src] + base;
            for (int t = threadIdx.x; t < n_el; t += blockDim.x) {
                const int j = t / TB, c = t % TB;
                buf[0][t] = (c < ncol) ? s[j * pitch + c] : make_float2(0.f, 0.f);
            }
            __syncthreads();
            loaded = jbk.src;
            if (AXIS == 0) spec = smem_fft<false, true>(buf[0], buf[1], buf[2], plan, TB, 1, TB);
            else spec = buf[0];
        }
        // work buffers distinct from spec
        float2* w0 = (spec == buf[0]) ? buf[1] : buf[0];
        float2* w1 = (spec == buf[2]) ? buf[1] : buf[2];
        if (w1 == w0) w1 = buf[2];
        float2* in = spec;
        if (jbk.dmul != nullptr || (AXIS == 0 && jbk.kappa)) {
            for (int t = threadIdx.x; t < n_el; t += blockDim.x) {
                const int j = t / TB;
                float2 v = spec[t];
                if (jbk.dmul) v = cmul(v, __ldg(jbk.dmul + j));
                if (AXIS == 0 && jbk.kappa) v = cscale(v, kap[t]);
                w0[t] = v;
            }
            __syncthreads();
            in = w0;
        }
        float2* res;
        if (AXIS == 0) {
            res = (in == w0) ? smem_fft<true, true>(w0, w1, w0, plan, TB, 1, TB)
                             : smem_fft<true, true>(spec, w0, w1, plan, TB, 1, TB);
        } else {
            res = (in == w0) ? smem_fft<INV, true>(w0, w1, w0, plan, TB, 1, TB)
                             : smem_fft<INV, true>(spec, w0, w1, plan, TB, 1, TB);
        }
        float2* d = jobs.buf[jbk.dst] + base;
        for (int t = threadIdx.x; t < n_el; t += blockDim.x) {
            const int j = t / TB, c = t % TB;
            if (c < ncol) d[j * pitch + c] = res[t];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------
// Row (z) helpers: real FFT of length nz through a complex FFT of length M = nz/2.
// ---------------------------------------------------------------------------------

// Build Z[k] (k < M) from half-spectrum rows so that IFFT_M(Z) = interleaved real row
// times nz; premul optional (D_z table). Imaginary parts of the DC and Nyquist bins are
// dropped, as a c2r transform does.
__device__ __forceinline__ void c2r_prepare(const float2* __restrict__ src, long long pitch,
                                            int nrows, int M, const float2* __restrict__ premul,
                                            const float2* __restrict__ tw, float2* Z) {
    for (int t = threadIdx.x; t < nrows * M; t += blockDim.x) {
        const int r = t / M, k = t % M;
        const float2* row = src + r * pitch;
        float2 a = row[k], b = row[M - k];
        if (premul) {
            a = cmul(a, __ldg(premul + k));
            b = cmul(b, __ldg(premul + M - k));
        }
        if (k == 0) {
            a.y = 0.f;
            b.y = 0.f;
        }
        const float2 e = make_float2(a.x + b.x, a.y - b.y);      // a + conj(b)
        const float2 d0 = make_float2(a.x - b.x, a.y + b.y);     // a - conj(b)
        const float2 w = __ldg(tw + k);
        const float2 o = make_float2(d0.x * w.x + d0.y * w.y, d0.y * w.x - d0.x * w.y);  // * conj(w)
        Z[t] = make_float2(e.x - o.y, e.y + o.x);                 // e + i*o
    }
}

// From F = FFT_M(interleaved real row) write the nz/2+1 half-spectrum bins.
__device__ __forceinline__ void r2c_finish(const float2* __restrict__ F, int nrows, int M,
                                           const float2* __restrict__ tw, float2* __restrict__ dst,
                                           long long pitch) {
    const int H = M + 1;
    for (int t = threadIdx.x; t < nrows * H; t += blockDim.x) {
        const int r = t / H, k = t % H;
        const float2 a = F[r * M + (k == M ? 0 : k)];
        const float2 b = F[r * M + (k == 0 ? 0 : M - k)];
        const float2 e = make_float2(0.5f * (a.x + b.x), 0.5f * (a.y - b.y));  // (a+conj b)/2
        const float2 o = make_float2(0.5f * (a.y + b.y), -0.5f * (a.x - b.x)); // (a-conj b)/(2i)
        const float2 w = __ldg(tw + k);
        dst[r * pitch + k] = make_float2(e.x + (w.x * o.x - w.y * o.y), e.y + (w.x * o.y + w.y * o.x));
    }
}

__device__ __forceinline__ int lower_bound_dev(const int* __restrict__ a, int n, int key) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(a + mid) < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Inverse transforms of three spectral row blocks into real rows D[f] (scaled by 1/N).
__device__ __forceinline__ void rows_inverse3(const GridDev& g, float2* const U[3],
                                              const float2* premul2, long long row0, int nrows,
                                              float* D[3], float2* P1, float2* P2) {
    const int M = g.nz / 2;
    for (int f = 0; f < 3; ++f) {
        c2r_prepare(U[f] + row0 * g.nzp, g.nzp, nrows, M, f == 2 ? premul2 : nullptr, g.tw_rfft, P1);
        __syncthreads();
        const float2* res = smem_fft<true, false>(P1, P2, P1, g.pzh, nrows, M, 1);
        const float* rr = reinterpret_cast<const float*>(res);
        for (int t = threadIdx.x; t < nrows * g.nz; t += blockDim.x) D[f][t] = rr[t] * g.inv_n;
        __syncthreads();
    }
}

__device__ __forceinline__ void rows_forward(const GridDev& g, float* Dsrc, float2* dst,
                                             long long row0, int nrows, float2* P1, float2* P2) {
    const int M = g.nz / 2;
    const float2* res = smem_fft<false, false>(reinterpret_cast<float2*>(Dsrc), P1, P2, g.pzh, nrows, M, 1);
    r2c_finish(res, nrows, M, g.tw_rfft, dst + row0 * g.nzp, g.nzp);
    __syncthreads();
}

// ---------------------------------------------------------------------------------
// Z-vel: dp/dx_a (3 c2r) -> v_a = pml_a(pml_a v_a - dt/rho0~_a dp/dx_a) -> Fz v_a
// (update_velocity_density first half, engine.hpp:272-283)
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) zvel_kernel(GridDev g, float2* S0, float2* S1, float2* S2,
                                                   const float2* dz_plus, float* v0, float* v1,
                                                   float* v2, Pml pml, Coef r0, Coef r1, Coef r2,
                                                   int rows_per_cta) {
    extern __shared__ float smemf[];
    const int nz = g.nz;
    const int R = rows_per_cta;
    const long long row0 = (long long)blockIdx.x * R;
    const int nrows = (int)min((long long)R, g.rows - row0);
    float* D[3] = {smemf, smemf + R * nz, smemf + 2 * R * nz};
    float2* P1 = reinterpret_cast<float2*>(smemf + 3 * R * nz);
    float2* P2 = P1 + R * nz / 2;
    float2* U[3] = {S0, S1, S2};

    rows_inverse3(g, U, dz_plus, row0, nrows, D, P1, P2);

    float* v[3] = {v0, v1, v2};
    const Coef rr[3] = {r0, r1, r2};
    for (int t = threadIdx.x; t < nrows * nz; t += blockDim.x) {
        const long long row = row0 + t / nz;
        const int z = t % nz;
        const int x = (int)(row / g.ny), y = (int)(row % g.ny);
        const long long i = row * nz + z;
        const float pm[3] = {__ldg(pml.prof[0] + x), __ldg(pml.prof[1] + y), __ldg(pml.prof[2] + z)};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            float va = v[a][i];
            va = pm[a] * va;
            va = va - rr[a].at(i) * D[a][t];
            va = pm[a] * va;
            v[a][i] = va;
            D[a][t] = va;
        }
    }
    __syncthreads();
    for (int f = 0; f < 3; ++f) rows_forward(g, D[f], U[f], row0, nrows, P1, P2);
}

// ---------------------------------------------------------------------------------
// Z-rho: dv_a/dx_a (3 c2r) -> rho_a = pml_a(pml_a rho_a - dt rho0 dv_a) -> sources /
// shell -> p = c0^2 sum rho -> gathers, correlation, divergence check -> Fz p
// (update_velocity_density second half :284-291, inject :296-300 / enforce :304-307,
//  update_pressure :318-347, simulate.hpp:88-95, gradient.hpp:177-182)
// UPDATE=false: no derivative update, rho is read as is (refresh_pressure_from_density,
// engine.hpp:311-316, used to seed the time-reversal replay, gradient.hpp:435-436).
// ---------------------------------------------------------------------------------
template <bool UPDATE>
__global__ void __launch_bounds__(256) zrho_kernel(GridDev g, ZrhoArgs A) {
    extern __shared__ float smemf[];
    const int nz = g.nz;
    const int R = A.rows_per_cta;
    const long long row0 = (long long)blockIdx.x * R;
    const int nrows = (int)min((long long)R, g.rows - row0);
    float* D[3] = {smemf, smemf + R * nz, smemf + 2 * R * nz};
    float2* P1 = reinterpret_cast<float2*>(smemf + 3 * R * nz);
    float2* P2 = P1 + R * nz / 2;
    const int n_el = nrows * nz;
    const long long i0 = row0 * nz;

    if (UPDATE) {
        rows_inverse3(g, A.S, A.dz_minus, row0, nrows, D, P1, P2);
        for (int t = threadIdx.x; t < n_el; t += blockDim.x) {
            const long long row = row0 + t / nz;
            const int z = t % nz;
            const int x = (int)(row / g.ny), y = (int)(row % g.ny);
            const long long i = i0 + t;
            const float pm[3] = {__ldg(A.pml.prof[0] + x), __ldg(A.pml.prof[1] + y), __ldg(A.pml.prof[2] + z)};
            const float dr = A.dtrho0.at(i);
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                if (A.du_out[a]) A.du_out[a][i] = D[a][t];
                float ra = A.rho[a][i];
                ra = pm[a] * ra;
                ra = ra - dr * D[a][t];
                ra = pm[a] * ra;
                D[a][t] = ra;
            }
        }
    } else {
        for (int t = threadIdx.x; t < n_el; t += blockDim.x)
#pragma unroll
            for (int a = 0; a < 3; ++a) D[a][t] = A.rho[a][i0 + t];
    }
    __syncthreads();

    // sparse modifications of the split densities, after the update and before p
    const int lo_key = (int)i0, hi_key = (int)(i0 + n_el);
    if (A.inj.n_unique > 0) {
        const int lo = lower_bound_dev(A.inj.pos, A.inj.n_unique, lo_key);
        const int hi = lower_bound_dev(A.inj.pos, A.inj.n_unique, hi_key);
        for (int u = lo + threadIdx.x; u < hi; u += blockDim.x) {
            const int t = A.inj.pos[u] - lo_key;
            const float sc = A.inj.scale[u];
            for (int c = A.inj.csr[u]; c < A.inj.csr[u + 1]; ++c) {
                const int n = A.step_n - A.inj.delay[c];
                if (n < 0 || n >= A.inj.len[c]) continue;
                const float amp = A.inj.w[c] * A.inj.sig[A.inj.off[c] + (long long)n * A.inj.stride[c]];
                if (amp == 0.f) continue;
                for (int a = A.a_first; a < 3; ++a) D[a][t] += amp * sc;
            }
        }
    }
    if (A.enf.n > 0) {
        const int lo = lower_bound_dev(A.enf.pos, A.enf.n, lo_key);
        const int hi = lower_bound_dev(A.enf.pos, A.enf.n, hi_key);
        for (int j = lo + threadIdx.x; j < hi; j += blockDim.x) {
            const int pos = A.enf.pos[j];
            const float val = A.enf.vals[j] / (A.enf.ndim * __ldg(A.c0sq + pos));
            const int t = pos - lo_key;
            for (int a = A.a_first; a < 3; ++a) D[a][t] = val;
        }
    }
    __syncthreads();

    for (int t = threadIdx.x; t < n_el; t += blockDim.x) {
        const long long i = i0 + t;
        const float r0 = D[0][t], r1 = D[1][t], r2 = D[2][t];
        if (UPDATE || A.enf.n > 0) {
            A.rho[0][i] = r0;
            A.rho[1][i] = r1;
            A.rho[2][i] = r2;
        }
        const float p = __ldg(A.c0sq + i) * ((r0 + r1) + r2);
        if (A.p_out) A.p_out[i] = p;
        D[0][t] = p;
        if (A.corr.grad != nullptr) {
            const float c2 = __ldg(A.c0sq + i);
            const float w = 2.f / (c2 * sqrtf(c2));
            const bool adj = A.corr.p_new != nullptr;  // see Correlate::p_new
            const float pn = adj ? A.corr.p_new[i] : p, q = adj ? p : A.corr.q_adj[i];
            const float ddot = ((pn - 2.f * A.corr.p_mid[i]) + A.corr.p_old[i]) * A.corr.inv_dt;
            A.corr.grad[i] += w * ddot * q;
        }
        if (A.check_step > 0 && i == 0 && !isfinite(p)) atomicMin(A.diverged, A.check_step);
    }
    __syncthreads();

    if (A.sens.n > 0) {
        const int lo = lower_bound_dev(A.sens.pos, A.sens.n, lo_key);
        const int hi = lower_bound_dev(A.sens.pos, A.sens.n, hi_key);
        for (int s = lo + threadIdx.x; s < hi; s += blockDim.x)
            A.sens.out[A.sens.idx[s]] = D[0][A.sens.pos[s] - lo_key];
    }
    if (A.shell.n > 0) {
        const int lo = lower_bound_dev(A.shell.pos, A.shell.n, lo_key);
        const int hi = lower_bound_dev(A.shell.pos, A.shell.n, hi_key);
        for (int j = lo + threadIdx.x; j < hi; j += blockDim.x)
            A.shell.out[j] = D[0][A.shell.pos[j] - lo_key];
    }
    rows_forward(g, D[0], A.S[0], row0, nrows, P1, P2);
}

// ---------------------------------------------------------------------------------
// Plain transforms for SpectralEngine::derivative (engine.hpp:118-121)
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) zfwd_kernel(GridDev g, const float* src, float2* S, int rows_per_cta) {
    extern __shared__ float smemf[];
    const int nz = g.nz, R = rows_per_cta;
    const long long row0 = (long long)blockIdx.x * R;
    const int nrows = (int)min((long long)R, g.rows - row0);
    float* D = smemf;
    float2* P1 = reinterpret_cast<float2*>(smemf + R * nz);
    float2* P2 = P1 + R * nz / 2;
    for (int t = threadIdx.x; t < nrows * nz; t += blockDim.x) D[t] = src[row0 * nz + t];
    __syncthreads();
    rows_forward(g, D, S, row0, nrows, P1, P2);
}

__global__ void __launch_bounds__(256) zinv_kernel(GridDev g, const float2* S, const float2* premul,
                                                   float* out, int rows_per_cta) {
    extern __shared__ float smemf[];
    const int nz = g.nz, R = rows_per_cta, M = nz / 2;
    const long long row0 = (long long)blockIdx.x * R;
    const int nrows = (int)min((long long)R, g.rows - row0);
    float2* P1 = reinterpret_cast<float2*>(smemf);
    float2* P2 = P1 + R * M;
    c2r_prepare(S + row0 * g.nzp, g.nzp, nrows, M, premul, g.tw_rfft, P1);
    __syncthreads();
    const float2* res = smem_fft<true, false>(P1, P2, P1, g.pzh, nrows, M, 1);
    const float* rr = reinterpret_cast<const float*>(res);
    for (int t = threadIdx.x; t < nrows * nz; t += blockDim.x) out[row0 * nz + t] = rr[t] * g.inv_n;
}

// ---------------------------------------------------------------------------------
// Adjoint source (detail::adjoint_source, gradient.hpp:264-289), one thread per sensor:
// r[n] = f_sim(nt-1-n) - f_obs(nt-1-n) (fp64), loss partial = Kahan sum of r^2/2,
// q = inclusive cumsum over n (Algorithm 1 step 13). sim/obs/q are step-major [nt][ns].
// ---------------------------------------------------------------------------------
__global__ void adjoint_source_kernel(const float* __restrict__ sim, const double* __restrict__ obs,
                                      int nt, int ns, int integrate, float* __restrict__ q,
                                      double* __restrict__ loss_part) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= ns) return;
    double acc = 0.0, loss = 0.0, comp = 0.0;
    for (int n = 0; n < nt; ++n) {
        const long long src = (long long)(nt - 1 - n) * ns + s;
        const double r = (double)sim[src] - obs[src];
        const double term = 0.5 * r * r - comp;
        const double tt = loss + term;
        comp = (tt - loss) - term;
        loss = tt;
        acc = integrate ? acc + r : r;
        q[(long long)n * ns + s] = (float)acc;
    }
    loss_part[s] = loss;
}

// Deterministic fixed-order reduction of per-sensor losses (Kahan, single thread; ns is
// at most a few thousand), optionally added to an accumulator.
__global__ void loss_reduce_kernel(const double* __restrict__ part, int n, double* __restrict__ out,
                                   double* __restrict__ acc, int accumulate) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double sum = 0.0, comp = 0.0;
    for (int i = 0; i < n; ++i) {
        const double term = part[i] - comp;
        const double t = sum + term;
        comp = (t - sum) - term;
        sum = t;
    }
    *out = sum;
    if (acc) *acc = accumulate ? *acc + sum : sum;
}

// GradientAccumulator::take (gradient.hpp:206-210) + finite check (:460-462), then the
// mini-batch accumulator update.
__global__ void finalize_grad_kernel(const float* __restrict__ grad, const uint8_t* __restrict__ gamma,
                                     long long n, float* __restrict__ acc, int accumulate,
                                     int* __restrict__ nonfinite) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float gv = gamma[i] ? grad[i] : 0.f;
        if (!isfinite(gv)) atomicExch(nonfinite, 1);
        acc[i] = accumulate ? acc[i] + gv : gv;
    }
}

__global__ void check_finite_kernel(const float* __restrict__ a, long long n, int* __restrict__ flag) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        if (!isfinite(a[i])) atomicExch(flag, 1);
}

__global__ void scale_kernel(float* __restrict__ a, long long n, float s) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        a[i] *= s;
}

// ---------------------------------------------------------------------------------
// Absorbing media (engine.hpp:327-343) and the stand-alone correlation / gathers
// ---------------------------------------------------------------------------------
__global__ void abs_prep_kernel(long long n, AbsArgs A) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        A.sum[i] = (A.rho[0][i] + A.rho[1][i]) + A.rho[2][i];
        A.ain[i] = (A.dtrho0.at(i) * A.inv_dt) * ((A.du[0][i] + A.du[1][i]) + A.du[2][i]);
    }
}

__global__ void abs_pressure_kernel(long long n, AbsArgs A) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float c2 = A.c0sq[i];
        float p = c2 * (A.sum[i] + (A.sign * A.tau0[i]) * A.aout[i]);
        if (A.eta) p -= c2 * A.eta[i] * A.aout2[i];
        A.p_out[i] = p;
        if (A.check_step > 0 && i == 0 && !isfinite(p)) atomicMin(A.diverged, A.check_step);
    }
}

// GradientAccumulator::accumulate, c0 branch (gradient.hpp:177-203)
__global__ void correlate_kernel(long long n, const float* __restrict__ p_new, const float* __restrict__ c0sq,
                                 Correlate C) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float c2 = c0sq[i];
        const float q = C.q_adj[i];
        const float w = 2.f / (c2 * sqrtf(c2));
        float gv = C.grad[i];
        if (C.use_ddot) gv += w * (((p_new[i] - 2.f * C.p_mid[i]) + C.p_old[i]) * C.inv_dt) * q;
        if (C.a1_new) gv += C.wa1[i] * (0.5f * (C.a1_old[i] - C.a1_new[i])) * q;
        if (C.a1l_new) gv += C.wa1l[i] * (0.5f * (C.a1l_old[i] - C.a1l_new[i])) * q;
        if (C.a2_mid) gv += C.wa2[i] * C.a2_mid[i] * q * C.dt;
        if (C.a2l_mid) gv += C.wa2l[i] * C.a2l_mid[i] * q * C.dt;
        C.grad[i] = gv;
    }
}

__global__ void gather_kernel(const float* __restrict__ p, SparseGather G) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < G.n) G.out[G.idx ? G.idx[s] : s] = p[G.pos[s]];
}

// ---------------------------------------------------------------------------------
// Host-callable launchers
// ---------------------------------------------------------------------------------

template <int AXIS, int TB, bool INV>
static cudaError_t launch_pencil_t(const GridDev& g, const PencilJobs& jobs, cudaStream_t st) {
    const int L = AXIS == 0 ? g.px.L : g.py.L;
    const size_t smem = (size_t)3 * L * TB * sizeof(float2) + (AXIS == 0 ? (size_t)L * TB * sizeof(float) : 0);
    static std::atomic<unsigned long long> configured{0};
    once_per_device(configured, [&] {
        cudaFuncSetAttribute(pencil_pass_kernel<AXIS, TB, INV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024);
    });
    dim3 grid((g.nzh + TB - 1) / TB, AXIS == 0 ? g.ny : g.nx);
    pencil_pass_kernel<AXIS, TB, INV><<<grid, 256, smem, st>>>(g, jobs);
    return cudaGetLastError();
}

int pencil_tile_cols(int L) { return L <= 768 ? 8 : (L <= 1536 ? 4 : 2); }

bool use_generic_kernels() {
    static const bool generic = [] {
        const char* e = getenv("USTFWI_GENERIC");
        return e && e[0] == '1';
    }();
    return generic;
}

cudaError_t launch_pencil(int axis, bool inv, const GridDev& g, const PencilJobs& jobs, cudaStream_t st) {
    const int L = axis == 0 ? g.px.L : g.py.L;
    if (!use_generic_kernels() && fast_pencil_supported(L)) return launch_pencil_fast(axis, inv, g, jobs, st);
    const int tb = pencil_tile_cols(L);
    if (axis == 0) {
        if (tb == 8) return launch_pencil_t<0, 8, false>(g, jobs, st);
        if (tb == 4) return launch_pencil_t<0, 4, false>(g, jobs, st);
        return launch_pencil_t<0, 2, false>(g, jobs, st);
    }
    if (inv) {
        if (tb == 8) return launch_pencil_t<1, 8, true>(g, jobs, st);
        if (tb == 4) return launch_pencil_t<1, 4, true>(g, jobs, st);
        return launch_pencil_t<1, 2, true>(g, jobs, st);
    }
    if (tb == 8) return launch_pencil_t<1, 8, false>(g, jobs, st);
    if (tb == 4) return launch_pencil_t<1, 4, false>(g, jobs, st);
    return launch_pencil_t<1, 2, false>(g, jobs, st);
}

int zrows_per_cta(int nz) {
    int r = 2048 / nz;
    if (r < 1) r = 1;
    if (r > 16) r = 16;
    return r;
}

static size_t zsmem_bytes(int nz, int R) { return (size_t)5 * R * nz * sizeof(float); }

cudaError_t launch_zvel(const GridDev& g, float2* S[3], const float2* dz_plus, float* v[3], const Pml& pml,
                        const Coef r[3], cudaStream_t st) {
    if (!use_generic_kernels() && fast_rows_supported(g.nz)) return launch_zvel_fast(g, S, dz_plus, v, pml, r, st);
    const int R = zrows_per_cta(g.nz);
    static std::atomic<unsigned long long> configured{0};
    once_per_device(configured, [&] {
        cudaFuncSetAttribute(zvel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    });
    const unsigned blocks = (unsigned)((g.rows + R - 1) / R);
    zvel_kernel<<<blocks, 256, zsmem_bytes(g.nz, R), st>>>(g, S[0], S[1], S[2], dz_plus, v[0], v[1], v[2], pml,
                                                           r[0], r[1], r[2], R);
    return cudaGetLastError();
}

cudaError_t launch_zrho(const GridDev& g, ZrhoArgs a, bool update, cudaStream_t st) {
    if (update && !use_generic_kernels() && fast_rows_supported(g.nz)) return launch_zrho_fast(g, a, st);
    const int R = zrows_per_cta(g.nz);
    a.rows_per_cta = R;
    static std::atomic<unsigned long long> configured{0};
    once_per_device(configured, [&] {
        cudaFuncSetAttribute(zrho_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(zrho_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    });
    const unsigned blocks = (unsigned)((g.rows + R - 1) / R);
    if (update) zrho_kernel<true><<<blocks, 256, zsmem_bytes(g.nz, R), st>>>(g, a);
    else zrho_kernel<false><<<blocks, 256, zsmem_bytes(g.nz, R), st>>>(g, a);
    return cudaGetLastError();
}

cudaError_t launch_zfwd(const GridDev& g, const float* src, float2* S, cudaStream_t st) {
    const int R = zrows_per_cta(g.nz);
    const unsigned blocks = (unsigned)((g.rows + R - 1) / R);
    zfwd_kernel<<<blocks, 256, (size_t)3 * R * g.nz * sizeof(float), st>>>(g, src, S, R);
    return cudaGetLastError();
}

cudaError_t launch_zinv(const GridDev& g, const float2* S, const float2* premul, float* out, cudaStream_t st) {
    const int R = zrows_per_cta(g.nz);
    const unsigned blocks = (unsigned)((g.rows + R - 1) / R);
    zinv_kernel<<<blocks, 256, (size_t)2 * R * g.nz * sizeof(float), st>>>(g, S, premul, out, R);
    return cudaGetLastError();
}

cudaError_t launch_adjoint_source(const float* sim, const double* obs, int nt, int ns, int integrate, float* q,
                                  double* loss_part, double* loss_out, double* loss_acc, int accumulate,
                                  cudaStream_t st) {
    if (ns > 0) adjoint_source_kernel<<<(ns + 127) / 128, 128, 0, st>>>(sim, obs, nt, ns, integrate, q, loss_part);
    loss_reduce_kernel<<<1, 32, 0, st>>>(loss_part, ns, loss_out, loss_acc, accumulate);
    return cudaGetLastError();
}

static unsigned flat_blocks(long long n) {
    long long b = (n + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    if (b < 1) b = 1;
    return (unsigned)b;
}

cudaError_t launch_finalize_grad(const float* grad, const uint8_t* gamma, long long n, float* acc, int accumulate,
                                 int* nonfinite, cudaStream_t st) {
    finalize_grad_kernel<<<flat_blocks(n), 256, 0, st>>>(grad, gamma, n, acc, accumulate, nonfinite);
    return cudaGetLastError();
}

cudaError_t launch_check_finite(const float* a, long long n, int* flag, cudaStream_t st) {
    check_finite_kernel<<<flat_blocks(n), 256, 0, st>>>(a, n, flag);
    return cudaGetLastError();
}

cudaError_t launch_scale(float* a, long long n, float s, cudaStream_t st) {
    scale_kernel<<<flat_blocks(n), 256, 0, st>>>(a, n, s);
    return cudaGetLastError();
}

cudaError_t launch_abs_prep(long long n, const AbsArgs& a, cudaStream_t st) {
    abs_prep_kernel<<<flat_blocks(n), 256, 0, st>>>(n, a);
    return cudaGetLastError();
}

cudaError_t launch_abs_pressure(long long n, const AbsArgs& a, cudaStream_t st) {
    abs_pressure_kernel<<<flat_blocks(n), 256, 0, st>>>(n, a);
    return cudaGetLastError();
}

cudaError_t launch_correlate(long long n, const float* p_new, const float* c0sq, const Correlate& c, cudaStream_t st) {
    correlate_kernel<<<flat_blocks(n), 256, 0, st>>>(n, p_new, c0sq, c);
    return cudaGetLastError();
}

// Elementwise legs of GradientAccumulator::accumulate_rho0 (gradient.hpp:213-239, with the
// F3 compile fix): mode 0 tmp = rho0 q; 1 tmp = dp / rho~_a; 2 grad += dt out q;
// 3 tmp = dp drq / rho~_a^2; 4 grad += dt out. 1/rho~_a = (dt/rho~_a) / dt from the
// stepper's staggered coefficient (WaveStepper constructor, engine.hpp:219-231).
__global__ void rho0_elem_kernel(long long n, int mode, Rho0Args A) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        switch (mode) {
            case 0: A.tmp[i] = A.rho0.at(i) * A.q[i]; break;
            case 1: A.tmp[i] = A.dp[i] * (A.dtr.at(i) * A.inv_dt); break;
            case 2: A.grad[i] += A.dt * A.out[i] * A.q[i]; break;
            case 3: {
                const float ir = A.dtr.at(i) * A.inv_dt;
                A.tmp[i] = ir * ir * A.dp[i] * A.drq[i];
                break;
            }
            default: A.grad[i] += A.dt * A.out[i]; break;
        }
    }
}

cudaError_t launch_rho0_elem(long long n, int mode, const Rho0Args& a, cudaStream_t st) {
    rho0_elem_kernel<<<flat_blocks(n), 256, 0, st>>>(n, mode, a);
    return cudaGetLastError();
}

// Deterministic mini-batch mean (average_estimates; worker-count independence
// :328,337): gathered holds W ranks x slots gradients, realization r at rank r mod W, slot
// r / W; the sum runs in realization order in fp64 and is scaled by 1/B once, so the result
// is bit-identical for every W.
__global__ void ordered_mean_kernel(long long n, const float* __restrict__ gathered, int world, int slots,
                                    int batch, float* __restrict__ out) {
    const double inv_b = 1.0 / batch;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < batch; ++r) {
            const long long slot = (long long)(r % world) * slots + r / world;
            s += (double)gathered[slot * n + i];
        }
        out[i] = (float)(s * inv_b);
    }
}

cudaError_t launch_ordered_mean(long long n, const float* gathered, int world, int slots, int batch, float* out,
                                cudaStream_t st) {
    ordered_mean_kernel<<<flat_blocks(n), 256, 0, st>>>(n, gathered, world, slots, batch, out);
    return cudaGetLastError();
}

// WaveStepper::inject_mass_source / enforce_shell (engine.hpp:296-307) for the step-level C
// ABI: one thread applies the list in order (mode 0: rho_a[idx] += val, mode 1: rho_a[idx] =
// val for every active axis a), so repeated positions behave as the reference's loop.
__global__ void stepper_sparse_kernel(float* r0, float* r1, float* r2, int a_first, const int* __restrict__ idx,
                                      const float* __restrict__ val, int n, int mode) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    float* r[3] = {r0, r1, r2};
    for (int i = 0; i < n; ++i)
        for (int a = a_first; a < 3; ++a) {
            if (mode == 0) r[a][idx[i]] += val[i];
            else r[a][idx[i]] = val[i];
        }
}

__global__ void pick_kernel(const float* __restrict__ f, const int* __restrict__ idx, int n, float* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = f[idx[i]];
}

cudaError_t launch_stepper_sparse(float* const rho[3], int a_first, const int* idx, const float* val, int n, int mode,
                                  cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    stepper_sparse_kernel<<<1, 1, 0, st>>>(rho[0], rho[1], rho[2], a_first, idx, val, n, mode);
    return cudaGetLastError();
}

cudaError_t launch_pick(const float* f, const int* idx, int n, float* out, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    pick_kernel<<<(n + 255) / 256, 256, 0, st>>>(f, idx, n, out);
    return cudaGetLastError();
}

cudaError_t launch_gather(const float* p, const SparseGather& g, cudaStream_t st) {
    if (g.n <= 0) return cudaSuccess;
    gather_kernel<<<(g.n + 255) / 256, 256, 0, st>>>(p, g);
    return cudaGetLastError();
}

}  // namespace ustfwi_dev
