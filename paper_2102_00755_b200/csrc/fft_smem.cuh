// Batched mixed-radix Stockham FFT in shared memory (sm_100a).
//
// Replaces the FFTW transforms of the reference (core/fft.hpp:51-63, RealFft) inside
// the fused k-space derivative passes. A tile of `nlines` lines of length L lives in
// shared memory with element (line l, index j) at base + l*ls + j*es. Each Stockham
// stage reads the tile, applies the inter-stage twiddles, does a radix-R DFT in
// registers and writes the tile in autosorted order to the other buffer, so the result
// is in natural order after the last stage (no digit-reversal pass).
//
// Forward = exp(-2*pi*i*jk/L) (FFTW_FORWARD), inverse = exp(+...) and UNnormalised, as
// FFTW; the engine folds the 1/N of RealFft::inverse (fft.hpp:58-63) into one scale.
#pragma once

#include <cuda_runtime.h>

namespace ustfwi_dev {

constexpr int kMaxStages = 16;

struct FftPlan {
    int L;                       // transform length
    int nstages;                 // number of radix stages (0 when L == 1)
    int radix[kMaxStages];       // radices in execution order
    const float2* tw;            // tw[k] = exp(-2*pi*i*k/L), k in [0, L)
};

// Complex add / subtract. On the device these are the packed fp32 pair instructions of
// sm_100 (FADD2, per-lane IEEE round-to-nearest like FADD, bit-identical results): one issue
// instead of two. Measured on B200 (v79): faster x pass and z rows, slower y pass,
// so the y-pass translation unit (passes_y.cu) defines USTFWI_FFT_SCALAR_ADD. Packed complex
// multiplies (FMUL2 + FFMA2) were slower in the z rows and are not used.
__host__ __device__ __forceinline__ float2 cadd(float2 a, float2 b) {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000 && !defined(USTFWI_FFT_SCALAR_ADD)
    return __fadd2_rn(a, b);
#else
    return make_float2(a.x + b.x, a.y + b.y);
#endif
}
__host__ __device__ __forceinline__ float2 csub(float2 a, float2 b) {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000 && !defined(USTFWI_FFT_SCALAR_ADD)
    return __fadd2_rn(a, make_float2(-b.x, -b.y));
#else
    return make_float2(a.x - b.x, a.y - b.y);
#endif
}
// (fma(ax, bx, -ay*by), fma(ax, by, ay*bx))
__host__ __device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__host__ __device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
// multiply by sign*i  (sign = -1 forward, +1 inverse)
template <bool INV>
__host__ __device__ __forceinline__ float2 mul_si(float2 a) {
    return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

// ---- radix-R DFT kernels, in registers -------------------------------------------

template <int R, bool INV>
struct Dft;

template <bool INV>
struct Dft<2, INV> {
    __host__ __device__ __forceinline__ static void run(float2* v) {
        const float2 a = v[0], b = v[1];
        v[0] = cadd(a, b);
        v[1] = csub(a, b);
    }
};

template <bool INV>
struct Dft<3, INV> {
    __host__ __device__ __forceinline__ static void run(float2* v) {
        const float h = 0.86602540378443864676f;  // sqrt(3)/2
        const float2 s = cadd(v[1], v[2]);
        const float2 d = csub(v[1], v[2]);
        const float2 m = make_float2(v[0].x - 0.5f * s.x, v[0].y - 0.5f * s.y);
        const float2 r = cscale(mul_si<INV>(d), h);
        v[0] = cadd(v[0], s);
        v[1] = cadd(m, r);
        v[2] = csub(m, r);
    }
};

template <bool INV>
struct Dft<4, INV> {
    __host__ __device__ __forceinline__ static void run(float2* v) {
        const float2 a = cadd(v[0], v[2]), b = csub(v[0], v[2]);
        const float2 c = cadd(v[1], v[3]), d = mul_si<INV>(csub(v[1], v[3]));
        v[0] = cadd(a, c);
        v[2] = csub(a, c);
        v[1] = cadd(b, d);
        v[3] = csub(b, d);
    }
};

template <bool INV>
struct Dft<5, INV> {
    __host__ __device__ __forceinline__ static void run(float2* v) {
        const float c1 = 0.30901699437494742410f, c2 = -0.80901699437494742410f;
        const float s1 = 0.95105651629515357212f, s2 = 0.58778525229247312917f;
        const float2 p1 = cadd(v[1], v[4]), m1 = csub(v[1], v[4]);
        const float2 p2 = cadd(v[2], v[3]), m2 = csub(v[2], v[3]);
        const float2 x0 = v[0];
        const float2 a1 = make_float2(x0.x + c1 * p1.x + c2 * p2.x, x0.y + c1 * p1.y + c2 * p2.y);
        const float2 a2 = make_float2(x0.x + c2 * p1.x + c1 * p2.x, x0.y + c2 * p1.y + c1 * p2.y);
        const float2 b1 = mul_si<INV>(make_float2(s1 * m1.x + s2 * m2.x, s1 * m1.y + s2 * m2.y));
        const float2 b2 = mul_si<INV>(make_float2(s2 * m1.x - s1 * m2.x, s2 * m1.y - s1 * m2.y));
        v[0] = cadd(x0, cadd(p1, p2));
        v[1] = cadd(a1, b1);
        v[4] = csub(a1, b1);
        v[2] = cadd(a2, b2);
        v[3] = csub(a2, b2);
    }
};

template <bool INV>
struct Dft<7, INV> {
    __host__ __device__ __forceinline__ static void run(float2* v) {
        const float c[3] = {0.62348980185873353053f, -0.22252093395631440429f,
                            -0.90096886790241912624f};
        const float s[3] = {0.78183148246802980871f, 0.97492791218182360702f,
                            0.43388373911755812048f};
        float2 p[3], m[3];
#pragma unroll
        for (int n = 0; n < 3; ++n) {
            p[n] = cadd(v[n + 1], v[6 - n]);
            m[n] = csub(v[n + 1], v[6 - n]);
        }
        const float2 x0 = v[0];
        v[0] = cadd(x0, cadd(p[0], cadd(p[1], p[2])));
#pragma unroll
        for (int k = 1; k <= 3; ++k) {
            float2 a = x0, b = make_float2(0.f, 0.f);
#pragma unroll
            for (int n = 1; n <= 3; ++n) {
                const int q = (n * k) % 7;  // angle index 2*pi*q/7
                const float cq = q <= 3 ? c[q - 1] : c[7 - q - 1];
                const float sq = q <= 3 ? s[q - 1] : -s[7 - q - 1];
                a.x += cq * p[n - 1].x;
                a.y += cq * p[n - 1].y;
                b.x += sq * m[n - 1].x;
                b.y += sq * m[n - 1].y;
            }
            const float2 ib = mul_si<INV>(b);
            v[k] = cadd(a, ib);
            v[7 - k] = csub(a, ib);
        }
    }
};

template <bool INV>
struct Dft<8, INV> {
    __host__ __device__ __forceinline__ static void run(float2* v) {
        const float r = 0.70710678118654752440f;
        float2 a[4], b[4];
#pragma unroll
        for (int n = 0; n < 4; ++n) {
            a[n] = cadd(v[n], v[n + 4]);
            b[n] = csub(v[n], v[n + 4]);
        }
        // b[n] *= w8^n, w8 = exp(sign*2*pi*i/8)
        b[1] = INV ? make_float2(r * (b[1].x - b[1].y), r * (b[1].x + b[1].y))
                   : make_float2(r * (b[1].x + b[1].y), r * (b[1].y - b[1].x));
        b[2] = mul_si<INV>(b[2]);
        b[3] = INV ? make_float2(-r * (b[3].x + b[3].y), r * (b[3].x - b[3].y))
                   : make_float2(r * (b[3].y - b[3].x), -r * (b[3].x + b[3].y));
        Dft<4, INV>::run(a);
        Dft<4, INV>::run(b);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[2 * k] = a[k];
            v[2 * k + 1] = b[k];
        }
    }
};

template <bool INV>
struct Dft<16, INV> {
    __host__ __device__ __forceinline__ static void run(float2* v) {
        // 16 = 4 x 4: column DFTs, twiddle w16^(n1*k2), row DFTs
        float2 t[4][4];
#pragma unroll
        for (int n1 = 0; n1 < 4; ++n1) {
#pragma unroll
            for (int n2 = 0; n2 < 4; ++n2) t[n1][n2] = v[n1 + 4 * n2];
            Dft<4, INV>::run(t[n1]);
        }
        const float c1 = 0.92387953251128675613f, s1 = 0.38268343236508977173f;
        const float r = 0.70710678118654752440f;
        const float sg = INV ? 1.f : -1.f;
        // w16^q for q = n1*k2 in {0..9}
        const float2 w[10] = {make_float2(1.f, 0.f),      make_float2(c1, sg * s1),
                              make_float2(r, sg * r),      make_float2(s1, sg * c1),
                              make_float2(0.f, sg),        make_float2(-s1, sg * c1),
                              make_float2(-r, sg * r),     make_float2(-c1, sg * s1),
                              make_float2(-1.f, 0.f),      make_float2(-c1, -sg * s1)};
#pragma unroll
        for (int n1 = 1; n1 < 4; ++n1)
#pragma unroll
            for (int k2 = 1; k2 < 4; ++k2) t[n1][k2] = cmul(t[n1][k2], w[n1 * k2]);
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) {
            float2 u[4];
#pragma unroll
            for (int n1 = 0; n1 < 4; ++n1) u[n1] = t[n1][k2];
            Dft<4, INV>::run(u);
#pragma unroll
            for (int k1 = 0; k1 < 4; ++k1) v[k2 + 4 * k1] = u[k1];
        }
    }
};

// ---- one Stockham stage --------------------------------------------------------
// LINE_FAST: consecutive threads take consecutive lines (tile layout [L][lines],
// es = nlines, ls = 1); otherwise consecutive butterflies of one line (row layout).
template <int R, bool INV, bool LINE_FAST>
__device__ __forceinline__ void stockham_stage(const float2* __restrict__ src,
                                               float2* __restrict__ dst, int L, int Ns,
                                               int nlines, int ls, int es,
                                               const float2* __restrict__ tw) {
    const int m = L / R;
    const int span = L / (Ns * R);
    const int total = nlines * m;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
        int line, j;
        if (LINE_FAST) {
            line = t % nlines;
            j = t / nlines;
        } else {
            j = t % m;
            line = t / m;
        }
        const int k = j % Ns;
        const float2* s = src + line * ls;
        float2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = s[(j + r * m) * es];
        if (Ns > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) {
                float2 w = __ldg(tw + k * r * span);
                if (INV) w.y = -w.y;
                v[r] = cmul(v[r], w);
            }
        }
        Dft<R, INV>::run(v);
        float2* d = dst + line * ls;
        const int base = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) d[(base + r * Ns) * es] = v[r];
    }
}

// Generic odd radix (any prime not covered above); slow path, O(R^2) per butterfly.
template <bool INV, bool LINE_FAST>
__device__ void stockham_stage_generic(const float2* __restrict__ src, float2* __restrict__ dst,
                                       int R, int L, int Ns, int nlines, int ls, int es,
                                       const float2* __restrict__ tw) {
    const int m = L / R;
    const int span = L / (Ns * R);
    const int total = nlines * m;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
        int line, j;
        if (LINE_FAST) {
            line = t % nlines;
            j = t / nlines;
        } else {
            j = t % m;
            line = t / m;
        }
        const int k = j % Ns;
        const float2* s = src + line * ls;
        float2* d = dst + line * ls;
        const int base = (j - k) * R + k;
        for (int q = 0; q < R; ++q) {
            float2 acc = make_float2(0.f, 0.f);
            for (int r = 0; r < R; ++r) {
                float2 x = s[(j + r * m) * es];
                // combined twiddle exp(sign*2*pi*i*(k*r*span + q*r*L/R)/L)
                const int e = (k * r * span + ((q * r) % R) * m) % L;
                float2 w = __ldg(tw + e);
                if (INV) w.y = -w.y;
                acc = cadd(acc, cmul(x, w));
            }
            d[(base + q * Ns) * es] = acc;
        }
    }
}

// Run all stages. `in` is read by the first stage only and is never written unless it
// aliases `pong`; `ping` must not alias `in`. Returns the buffer holding the result.
// Ends with __syncthreads().
template <bool INV, bool LINE_FAST>
__device__ float2* smem_fft(float2* in, float2* ping, float2* pong, const FftPlan& p, int nlines,
                            int ls, int es) {
    const float2* src = in;
    float2* dst = ping;
    int Ns = 1;
    for (int s = 0; s < p.nstages; ++s) {
        const int R = p.radix[s];
        switch (R) {
            case 2: stockham_stage<2, INV, LINE_FAST>(src, dst, p.L, Ns, nlines, ls, es, p.tw); break;
            case 3: stockham_stage<3, INV, LINE_FAST>(src, dst, p.L, Ns, nlines, ls, es, p.tw); break;
            case 4: stockham_stage<4, INV, LINE_FAST>(src, dst, p.L, Ns, nlines, ls, es, p.tw); break;
            case 5: stockham_stage<5, INV, LINE_FAST>(src, dst, p.L, Ns, nlines, ls, es, p.tw); break;
            case 7: stockham_stage<7, INV, LINE_FAST>(src, dst, p.L, Ns, nlines, ls, es, p.tw); break;
            case 8: stockham_stage<8, INV, LINE_FAST>(src, dst, p.L, Ns, nlines, ls, es, p.tw); break;
            case 16: stockham_stage<16, INV, LINE_FAST>(src, dst, p.L, Ns, nlines, ls, es, p.tw); break;
            default:
                stockham_stage_generic<INV, LINE_FAST>(src, dst, R, p.L, Ns, nlines, ls, es, p.tw);
                break;
        }
        __syncthreads();
        Ns *= R;
        src = dst;
        dst = (dst == ping) ? pong : ping;
    }
    return const_cast<float2*>(src);
}

}  // namespace ustfwi_dev
