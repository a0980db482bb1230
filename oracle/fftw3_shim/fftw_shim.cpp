// FFTW3-API shim implementation (fp64) — TEST INFRASTRUCTURE ONLY (see fftw3.h).
//
// Mixed-radix Stockham autosort FFT. A 1-D transform of length n runs over a
// block laid out as [n][L] (L contiguous "lanes"), so the strided leading axes of
// a multi-dimensional array are transformed L lines at a time with unit-stride
// inner loops. Radices 4, 2, 3, 5 have closed-form butterflies; any other prime
// factor uses a direct O(p^2) DFT stage, so every length is supported.
#include "fftw3.h"

#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace {

using cd = std::complex<double>;

struct LinePlan {
    int n = 1;
    std::vector<int> radix;
    std::vector<cd> root;  // root[k] = exp(-2*pi*i*k/n)
};

LinePlan make_line_plan(int n) {
    LinePlan p;
    p.n = n;
    int m = n;
    while (m % 4 == 0) { p.radix.push_back(4); m /= 4; }
    while (m % 2 == 0) { p.radix.push_back(2); m /= 2; }
    for (int f = 3; m > 1; f += 2)
        while (m % f == 0) { p.radix.push_back(f); m /= f; }
    p.root.resize(static_cast<std::size_t>(n));
    for (int k = 0; k < n; ++k) {
        // reduce the angle to [0, pi/4]-friendly form via sin/cos of 2*pi*k/n
        const double a = -2.0 * M_PI * static_cast<double>(k) / static_cast<double>(n);
        p.root[static_cast<std::size_t>(k)] = cd(std::cos(a), std::sin(a));
    }
    return p;
}

// One Stockham stage: src/dst are [n][L]; Ns = product of the radices done so far.
void stage(const LinePlan& p, int R, int Ns, const cd* src, cd* dst, std::size_t L, int sign,
           std::vector<cd>& v, std::vector<cd>& w) {
    const int n = p.n;
    const int m = n / R;               // butterflies per line
    const int span = n / (Ns * R);     // twiddle index multiplier
    v.resize(static_cast<std::size_t>(R) * L);
    w.resize(static_cast<std::size_t>(R));
    for (int j = 0; j < m; ++j) {
        const int k = j % Ns;
        for (int r = 0; r < R; ++r) {
            cd t = p.root[static_cast<std::size_t>((static_cast<long>(k) * r * span) % n)];
            w[static_cast<std::size_t>(r)] = sign > 0 ? std::conj(t) : t;
        }
        for (int r = 0; r < R; ++r) {
            const cd* in = src + static_cast<std::size_t>(j + r * m) * L;
            cd* vr = v.data() + static_cast<std::size_t>(r) * L;
            const cd wr = w[static_cast<std::size_t>(r)];
            if (r == 0)
                for (std::size_t l = 0; l < L; ++l) vr[l] = in[l];
            else
                for (std::size_t l = 0; l < L; ++l) vr[l] = in[l] * wr;
        }
        const int base = (j / Ns) * Ns * R + k;
        cd* out[64];
        std::vector<cd*> out_big;
        cd** o = out;
        if (R > 64) {
            out_big.resize(static_cast<std::size_t>(R));
            o = out_big.data();
        }
        for (int r = 0; r < R; ++r) o[r] = dst + static_cast<std::size_t>(base + r * Ns) * L;
        const double s = sign > 0 ? 1.0 : -1.0;
        if (R == 2) {
            cd* a = v.data();
            cd* b = v.data() + L;
            for (std::size_t l = 0; l < L; ++l) {
                o[0][l] = a[l] + b[l];
                o[1][l] = a[l] - b[l];
            }
        } else if (R == 4) {
            cd* a0 = v.data();
            cd* a1 = v.data() + L;
            cd* a2 = v.data() + 2 * L;
            cd* a3 = v.data() + 3 * L;
            for (std::size_t l = 0; l < L; ++l) {
                const cd t0 = a0[l] + a2[l], t1 = a0[l] - a2[l];
                const cd t2 = a1[l] + a3[l];
                const cd d = a1[l] - a3[l];
                const cd t3 = cd(-s * d.imag(), s * d.real());  // s*i*d
                o[0][l] = t0 + t2;
                o[2][l] = t0 - t2;
                o[1][l] = t1 + t3;
                o[3][l] = t1 - t3;
            }
        } else if (R == 3) {
            const double c = -0.5, sn = s * std::sqrt(3.0) / 2.0;
            cd* a0 = v.data();
            cd* a1 = v.data() + L;
            cd* a2 = v.data() + 2 * L;
            for (std::size_t l = 0; l < L; ++l) {
                const cd sum = a1[l] + a2[l], dif = a1[l] - a2[l];
                const cd m1 = a0[l] + c * sum;
                const cd m2 = cd(-sn * dif.imag(), sn * dif.real());
                o[0][l] = a0[l] + sum;
                o[1][l] = m1 + m2;
                o[2][l] = m1 - m2;
            }
        } else {
            // direct DFT of length R across the lanes
            std::vector<cd> rr(static_cast<std::size_t>(R));
            for (int q = 0; q < R; ++q) {
                const double a = s * 2.0 * M_PI * q / R;
                rr[static_cast<std::size_t>(q)] = cd(std::cos(a), std::sin(a));
            }
            for (int q = 0; q < R; ++q) {
                cd* oq = o[q];
                for (std::size_t l = 0; l < L; ++l) oq[l] = v[l];
                for (int r = 1; r < R; ++r) {
                    const cd wqr = rr[static_cast<std::size_t>((q * r) % R)];
                    const cd* vr = v.data() + static_cast<std::size_t>(r) * L;
                    for (std::size_t l = 0; l < L; ++l) oq[l] += vr[l] * wqr;
                }
            }
        }
    }
}

// Transform data ([n][L]) in place; work must hold n*L values.
void line_fft(const LinePlan& p, cd* data, cd* work, std::size_t L, int sign) {
    if (p.n == 1) return;
    std::vector<cd> v, w;
    cd* src = data;
    cd* dst = work;
    int Ns = 1;
    for (int R : p.radix) {
        stage(p, R, Ns, src, dst, L, sign, v, w);
        Ns *= R;
        std::swap(src, dst);
    }
    if (src != data) std::memcpy(data, src, sizeof(cd) * static_cast<std::size_t>(p.n) * L);
}

enum class Kind { c2c, r2c, c2r };

}  // namespace

struct fftw_plan_s {
    Kind kind = Kind::c2c;
    int sign = FFTW_FORWARD;
    std::vector<int> dims;
    std::vector<LinePlan> axis;
    void* in = nullptr;
    void* out = nullptr;
};

namespace {

// Complex transform over axes [0, n_axes) of a row-major array whose shape is
// dims (the array may have further trailing dims folded into `tail`).
void transform_leading(fftw_plan_s& p, cd* data, const std::vector<int>& shape, int n_axes) {
    std::size_t total = 1;
    for (int d : shape) total *= static_cast<std::size_t>(d);
    std::vector<cd> work;
    for (int a = 0; a < n_axes; ++a) {
        const int n = shape[static_cast<std::size_t>(a)];
        if (n == 1) continue;
        std::size_t inner = 1;
        for (std::size_t b = static_cast<std::size_t>(a) + 1; b < shape.size(); ++b)
            inner *= static_cast<std::size_t>(shape[b]);
        const std::size_t block = static_cast<std::size_t>(n) * inner;
        const std::size_t outer = total / block;
        work.resize(block);
        for (std::size_t o = 0; o < outer; ++o)
            line_fft(p.axis[static_cast<std::size_t>(a)], data + o * block, work.data(), inner, p.sign);
    }
}

}  // namespace

extern "C" {

void* fftw_malloc(size_t n) {
    void* ptr = nullptr;
    if (posix_memalign(&ptr, 64, n ? n : 1) != 0) return nullptr;
    return ptr;
}

void fftw_free(void* p) { std::free(p); }

static fftw_plan make_plan(Kind kind, int rank, const int* n, void* in, void* out, int sign) {
    auto* p = new fftw_plan_s;
    p->kind = kind;
    p->sign = sign;
    p->dims.assign(n, n + rank);
    for (int a = 0; a < rank; ++a) p->axis.push_back(make_line_plan(n[a]));
    p->in = in;
    p->out = out;
    return p;
}

fftw_plan fftw_plan_dft_r2c(int rank, const int* n, double* in, fftw_complex* out, unsigned) {
    return make_plan(Kind::r2c, rank, n, in, out, FFTW_FORWARD);
}

fftw_plan fftw_plan_dft_c2r(int rank, const int* n, fftw_complex* in, double* out, unsigned) {
    return make_plan(Kind::c2r, rank, n, in, out, FFTW_BACKWARD);
}

fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out, int sign,
                        unsigned) {
    return make_plan(Kind::c2c, rank, n, in, out, sign);
}

void fftw_execute(const fftw_plan cp) {
    fftw_plan_s& p = *cp;
    const int rank = static_cast<int>(p.dims.size());
    std::size_t total = 1;
    for (int d : p.dims) total *= static_cast<std::size_t>(d);
    if (p.kind == Kind::c2c) {
        cd* out = reinterpret_cast<cd*>(p.out);
        if (p.out != p.in) std::memcpy(out, p.in, sizeof(cd) * total);
        transform_leading(p, out, p.dims, rank);
        return;
    }
    const int nl = p.dims.back();
    const int nh = nl / 2 + 1;
    const std::size_t lines = total / static_cast<std::size_t>(nl);
    std::vector<int> half = p.dims;
    half.back() = nh;
    const LinePlan& last = p.axis.back();
    std::vector<cd> buf(static_cast<std::size_t>(nl)), work(static_cast<std::size_t>(nl));
    if (p.kind == Kind::r2c) {
        const double* in = static_cast<const double*>(p.in);
        cd* out = reinterpret_cast<cd*>(p.out);
        for (std::size_t r = 0; r < lines; ++r) {
            for (int i = 0; i < nl; ++i) buf[static_cast<std::size_t>(i)] = in[r * nl + i];
            line_fft(last, buf.data(), work.data(), 1, FFTW_FORWARD);
            for (int k = 0; k < nh; ++k) out[r * nh + k] = buf[static_cast<std::size_t>(k)];
        }
        if (rank > 1) transform_leading(p, out, half, rank - 1);
        return;
    }
    // c2r: leading axes first (on a private copy), then Hermitian-extended lines.
    std::vector<cd> spec(reinterpret_cast<const cd*>(p.in),
                         reinterpret_cast<const cd*>(p.in) + lines * nh);
    if (rank > 1) transform_leading(p, spec.data(), half, rank - 1);
    double* out = static_cast<double*>(p.out);
    for (std::size_t r = 0; r < lines; ++r) {
        const cd* h = spec.data() + r * nh;
        for (int k = 0; k < nh; ++k) buf[static_cast<std::size_t>(k)] = h[k];
        for (int k = nh; k < nl; ++k) buf[static_cast<std::size_t>(k)] = std::conj(h[nl - k]);
        line_fft(last, buf.data(), work.data(), 1, FFTW_BACKWARD);
        for (int i = 0; i < nl; ++i) out[r * nl + i] = buf[static_cast<std::size_t>(i)].real();
    }
}

void fftw_destroy_plan(fftw_plan p) { delete p; }

}  // extern "C"
