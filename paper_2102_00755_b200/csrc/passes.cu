// Register/shared-memory pass kernels for the supported transform lengths (sm_100a).
//
// Each line transform of length L = N1 * N2 is a two-level Cooley-Tukey:
//   phase A  thread (col, n2) holds x[n2 + N2*n1] (N1 values), runs the N1-point codelet,
//            applies W_L^(n2*k1) and writes one transposed tile to shared memory;
//   phase B  thread (col, k1) reads its N2 values and runs the N2-point codelet, giving
//            X[k1 + N1*k2] in registers.
// Only one level lives in registers at a time (low register footprint -> several CTAs
// per SM), and the HBM tiles are staged asynchronously into shared memory:
//   pencil passes  cp.async 16-B granules of the strided [L][TB] tile (LDGSTS)
//   z passes       TMA bulk copies (cp.async.bulk + mbarrier) of the CTA's contiguous
//                  row blocks of every input field, all issued at CTA start
// so the loads of a CTA are all in flight before any compute, and the compute of one CTA
// overlaps the loads of the others. A forward-multiply-inverse sandwich (x pass) costs one
// HBM read and one HBM write per output; kappa and the stagger factors are applied between
// the halves. The z passes keep the elementwise velocity / density / pressure update,
// sparse sources and shell, gathers and the c0 correlation in the same kernel.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "async_copy.cuh"
#include "fft_reg.cuh"
#include "kernels.cuh"

namespace ustfwi_dev {

__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }

constexpr int cmax(int a, int b) { return a > b ? a : b; }

// kappa = sinc(h|k|) = sin(sqrt(u))/sqrt(u), u = (h|k|)^2, h = c_ref*dt/2 (engine.hpp:43).
// sinc(sqrt(u)) = sum_n (-u)^n / (2n+1)! is entire in u; with u <= 3 (the CFL bound
// c*dt/dx <= 2/pi gives h|k| <= sqrt(3)) eleven Horner terms are exact to < 1e-9, so no
// sin / sqrt / division is evaluated per spectral element.
__device__ __forceinline__ float kappa_of_u(float u) {
    float s = -1.f / 51090942171709440000.f;  // -1/21!
    s = fmaf(s, u, 1.f / 121645100408832000.f);
    s = fmaf(s, u, -1.f / 355687428096000.f);
    s = fmaf(s, u, 1.f / 1307674368000.f);
    s = fmaf(s, u, -1.f / 6227020800.f);
    s = fmaf(s, u, 1.f / 39916800.f);
    s = fmaf(s, u, -1.f / 362880.f);
    s = fmaf(s, u, 1.f / 5040.f);
    s = fmaf(s, u, -1.f / 120.f);
    s = fmaf(s, u, 1.f / 6.f);
    return fmaf(-s, u, 1.f);
}
__device__ __forceinline__ float kappa_fast(float k2, float half_cdt) { return kappa_of_u(half_cdt * half_cdt * k2); }

// |k|^e multipliers of the absorbing / alpha0 / y paths, kept out of line so the hot x-pass
// code (kappa) stays compact
static __device__ __noinline__ float kpow_mult_call(float k2, float e, int kind) { return kpow_mult(k2, e, kind); }

// ======================================================================================
// Pencil passes (x and y)
// ======================================================================================
template <int L, int N1, int TB, bool DB>
struct PencilCfg {
    static constexpr int N2 = L / N1;
    static constexpr int NT = TB * cmax(N1, N2);
    static constexpr int KP = N2 * TB + 8;  // float2 pitch of one k1 slab (+64 B against bank conflicts)
    // Good-Thomas split when gcd(N1, N2) == 1: no inter-level twiddles
    static constexpr bool PFA = cx_gcd(N1, N2) == 1;
    static constexpr int CR = PFA ? (N2 * cx_inv_mod(N2 % N1, N1)) % L : 0;  // = 1 mod N1, 0 mod N2
    static constexpr int CM = PFA ? (N1 * cx_inv_mod(N1 % N2, N2)) % L : 0;  // = 0 mod N1, 1 mod N2
    // tile buffer(s) (two with double-buffered prefetch) + transpose tile + twiddles
    static constexpr size_t SMEM = ((DB ? 2 : 1) * size_t(L) * TB + size_t(N1) * KP + L) * sizeof(float2);
    // x pass: + kappa of the current tile (shared by the source groups of the tile)
    static constexpr size_t SMEM_X = SMEM + size_t(L) * TB * sizeof(float);
    // row of input element (n1, n2) and of output element (k1, k2)
    __device__ __forceinline__ static int in_row(int n1, int n2) {
        if constexpr (PFA) {
            const int t = N2 * n1 + N1 * n2;
            return t >= L ? t - L : t;
        } else {
            return n2 + N2 * n1;
        }
    }
    __device__ __forceinline__ static int out_row(int kbase, int k2) {  // kbase = out_base(k1)
        if constexpr (PFA) {
            const int t = kbase + (k2 * CM) % L;
            return t >= L ? t - L : t;
        } else {
            return kbase + N1 * k2;
        }
    }
    __device__ __forceinline__ static int out_base(int k1) { return PFA ? (k1 * CR) % L : k1; }
};

// Persistent pencil pass. Work unit = (tile, source group): tile = TB consecutive spectral
// columns of one line set (x pencils at fixed y for AXIS 0, y pencils at fixed x for AXIS 1);
// a source group is a run of jobs reading the same scratch buffer. Each CTA walks its units
// with the next unit's tile prefetched by cp.async into the other buffer while the
// current one is transformed.
//   AXIS 0: forward x FFT, kappa (and D_x of the job), inverse x FFT, one store per job.
//   AXIS 1: y FFT in direction INV (inverse jobs may carry a D_y premultiplier).
template <int AXIS, bool INV, int L, int N1, int TB, int MINB, bool DB>
__global__ void __launch_bounds__(PencilCfg<L, N1, TB, DB>::NT, MINB)
    pencil_fast_kernel(const __grid_constant__ GridDev g, const __grid_constant__ PencilJobs jobs) {
    using C = PencilCfg<L, N1, TB, DB>;
    constexpr int N2 = C::N2, KP = C::KP, NT = C::NT;
    extern __shared__ float2 smem[];
    float2* xbuf0 = smem;                     // [L][TB] tiles, natural order
    float2* xbuf1 = DB ? smem + L * TB : smem;
    float2* ys = smem + (DB ? 2 : 1) * L * TB;  // transposed [N1][N2*TB (+pad)]
    float2* tw = ys + N1 * KP;                // W_L^k
    float* kap_s = reinterpret_cast<float*>(tw + L);  // x pass: kappa of the current tile
    const FftPlan& plan = AXIS == 0 ? g.px : g.py;
    for (int i = threadIdx.x; i < L; i += NT) tw[i] = plan.tw[i];

    // source groups of the job list
    int gstart[5];
    int ng = 0;
    for (int jb = 0; jb < jobs.n; ++jb)
        if (jb == 0 || jobs.job[jb].src != jobs.job[jb - 1].src) gstart[ng++] = jb;
    gstart[ng] = jobs.n;

    const int ntx = (g.nzh + TB - 1) / TB;
    const int ntiles = ntx * (AXIS == 0 ? g.ny : g.xn);
    const int line0 = AXIS == 0 ? 0 : g.x0;
    const int nunits = ((ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x) * ng;
    const int pitch = (AXIS == 0) ? g.ny * g.nzp : g.nzp;
    const int c = threadIdx.x % TB;
    const int ra = threadIdx.x / TB;  // n2 in phase A, k1 in phase B
    const bool inA = ra < N2, inB = ra < N1;

    struct Unit {
        int c0, ncol, line, grp;
        long long base;
    };
    auto unit_of = [&](int u) {
        Unit w;
        const int tile = (int)blockIdx.x + (u / ng) * (int)gridDim.x;
        w.grp = u % ng;
        w.line = line0 + tile / ntx;
        w.c0 = (tile % ntx) * TB;
        w.ncol = min(TB, g.nzh - w.c0);
        w.base = (AXIS == 0) ? (long long)w.line * g.nzp + w.c0 : (long long)w.line * g.ny * g.nzp + w.c0;
        return w;
    };
    // async tile load: 16-B granules (2 complex); columns past nzh are row padding
    auto prefetch = [&](int u, float2* xs) {
        if (u < nunits) {
            const Unit w = unit_of(u);
            const float2* s = jobs.buf[jobs.job[gstart[w.grp]].src] + w.base;
            constexpr int CH = TB / 2;
            for (int i = threadIdx.x; i < L * CH; i += NT) {
                const int row = i / CH, cc = 2 * (i % CH);
                if (cc < w.ncol) cp_async16(xs + row * TB + cc, s + row * pitch + cc);
            }
        }
        cp_async_commit();
    };

    if (DB) prefetch(0, xbuf0);
    for (int u = 0; u < nunits; ++u) {
        float2* xs = (u & 1) ? xbuf1 : xbuf0;
        if constexpr (DB) {
            prefetch(u + 1, (u & 1) ? xbuf0 : xbuf1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            prefetch(u, xs);
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        const Unit w = unit_of(u);
        const bool colok = c < w.ncol;
        const long long base = w.base;

        // forward transform of xs -> X[k1 + N1*k2] in phase-B registers
        auto forward = [&](float2 (&X)[N2]) {
            if (inA) {
                float2 a[N1];
#pragma unroll
                for (int n1 = 0; n1 < N1; ++n1) a[n1] = xs[C::in_row(n1, ra) * TB + c];
                RDft<N1, false>::run(a);
                if constexpr (!C::PFA) {
#pragma unroll
                    for (int k1 = 1; k1 < N1; ++k1) a[k1] = cmul(a[k1], tw[ra * k1]);
                }
#pragma unroll
                for (int k1 = 0; k1 < N1; ++k1) ys[k1 * KP + ra * TB + c] = a[k1];
            }
            __syncthreads();
            if (inB) {
#pragma unroll
                for (int n2 = 0; n2 < N2; ++n2) X[n2] = ys[ra * KP + n2 * TB + c];
                RDft<N2, false>::run(X);
            }
        };
        // inverse of b (phase-B registers, natural order) -> rows of dst
        auto inverse_store = [&](float2 (&b)[N2], float2* dst) {
            if (inB) {
                RDft<N2, true>::run(b);
                if constexpr (!C::PFA) {
#pragma unroll
                    for (int n2 = 1; n2 < N2; ++n2) b[n2] = cmul(b[n2], conjf2(tw[ra * n2]));
                }
            }
            __syncthreads();
            if (inB) {
#pragma unroll
                for (int n2 = 0; n2 < N2; ++n2) ys[ra * KP + n2 * TB + c] = b[n2];
            }
            __syncthreads();
            if (inA) {
                float2 a[N1];
#pragma unroll
                for (int k1 = 0; k1 < N1; ++k1) a[k1] = ys[k1 * KP + ra * TB + c];
                RDft<N1, true>::run(a);
                if (colok) {
                    float2* d = dst + base + c;
#pragma unroll
                    for (int n1 = 0; n1 < N1; ++n1) d[C::in_row(n1, ra) * pitch] = a[n1];
                }
            }
        };

        const int kb = C::out_base(ra);
        if (AXIS == 1 && !INV) {
            float2 X[N2];
            forward(X);
            if (inB && colok) {
                float2* d = jobs.buf[jobs.job[gstart[w.grp]].dst] + base + c;
#pragma unroll
                for (int k2 = 0; k2 < N2; ++k2) d[C::out_row(kb, k2) * pitch] = X[k2];
            }
        } else {
            if (AXIS == 0) {
                // forward, then keep kappa * X (natural order) in xs for the jobs of this group;
                // all jobs of one source share its kappa flag (kappa-free jobs are only the
                // staggered-density setup shift). Each phase-B thread later reads back only
                // the entries it wrote, so no barrier is needed.
                const bool kap = jobs.job[gstart[w.grp]].kappa != 0;
                float2 X[N2];
                forward(X);
                if (inB) {
                    if (kap && w.grp == 0) {
                        // kappa(|k|) (or |k|^e) of this tile, evaluated once for all its source groups
                        const float ky = g.ky[w.line];
                        const float kz = colok ? g.kz[w.c0 + c] : 0.f;
                        const int kind = jobs.job[gstart[w.grp]].kappa;
                        const bool power = kind >= 2;
                        const float e = jobs.job[gstart[w.grp]].kexp;
#pragma unroll
                        for (int k2 = 0; k2 < N2; ++k2) {
                            const int k = C::out_row(kb, k2);
                            const float kx = g.kx[k];
                            const float q2 = kx * kx + ky * ky + kz * kz;
                            kap_s[k * TB + c] = power ? kpow_mult_call(q2, e, kind) : kappa_fast(q2, g.half_cdt);
                        }
                    }
#pragma unroll
                    for (int k2 = 0; k2 < N2; ++k2) {
                        const int k = C::out_row(kb, k2);
                        xs[k * TB + c] = kap ? cscale(X[k2], kap_s[k * TB + c]) : X[k2];
                    }
                }
            }
            for (int jb = gstart[w.grp]; jb < gstart[w.grp + 1]; ++jb) {
                const PencilJob J = jobs.job[jb];
                float2 b[N2];
                if (inB) {
#pragma unroll
                    for (int k2 = 0; k2 < N2; ++k2) {
                        const int k = C::out_row(kb, k2);
                        float2 v = xs[k * TB + c];
                        if (J.dmul) v = cmul(v, __ldg(J.dmul + k));
                        b[k2] = v;
                    }
                }
                inverse_store(b, jobs.buf[J.dst]);
            }
        }
        __syncthreads();  // xs / ys free for the next prefetch into this buffer and the next unit
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// TMA variant of the pencil pass: the [L][TB] tile of a unit arrives by TMA tensor loads
// (one or two boxes, completion on an mbarrier per stage) and every output tile leaves by a
// TMA tensor store from shared memory, so no thread computes a global address. One thread
// of a warp that idles in phase A (the last thread) is the producer: it issues the loads /
// stores and waits for the store reads before a staging buffer is reused.
struct PencilMaps {
    CUtensorMap tm[3];  // per scratch buffer, the box shape of this pass
};

template <int AXIS, bool INV, int L, int N1, int TB, int MINB, bool DB>
__global__ void __launch_bounds__(PencilCfg<L, N1, TB, DB>::NT, MINB)
    pencil_tma_kernel(const __grid_constant__ GridDev g, const __grid_constant__ PencilJobs jobs,
                      const __grid_constant__ PencilMaps maps) {
    using C = PencilCfg<L, N1, TB, DB>;
    constexpr int N2 = C::N2, KP = C::KP, NT = C::NT;
    constexpr int NBUF = DB ? 2 : 1;
    constexpr int BOXR = L > 256 ? L / 2 : L;  // TMA box extent <= 256 rows
    constexpr int NBOX = L / BOXR;
    constexpr unsigned TILE_BYTES = unsigned(L) * TB * sizeof(float2);
    extern __shared__ __align__(128) unsigned char sm_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm_raw);          // one per stage
    float2* xbuf = reinterpret_cast<float2*>(sm_raw + 128);       // [NBUF][L][TB], 128-B aligned
    float2* ys = xbuf + NBUF * L * TB;                            // transposed [N1][KP]
    float2* tw = ys + N1 * KP;                                    // W_L^k
    float* kap_s = reinterpret_cast<float*>(tw + L);              // x pass: kappa of the tile
    float* hkx2_s = kap_s + L * TB;                               // x pass: (h kx)^2 per row
    const FftPlan& plan = AXIS == 0 ? g.px : g.py;
    const bool producer = threadIdx.x == NT - 1;
    if (threadIdx.x == 0) {
        for (int b = 0; b < NBUF; ++b) mbar_init(&bar[b], 1);
    }
    for (int i = threadIdx.x; i < L; i += NT) tw[i] = plan.tw[i];
    if constexpr (AXIS == 0) {
        for (int i = threadIdx.x; i < L; i += NT) {
            const float hk = g.half_cdt * g.kx[i];
            hkx2_s[i] = hk * hk;
        }
    }

    int gstart[5];
    int ng = 0;
    for (int jb = 0; jb < jobs.n; ++jb)
        if (jb == 0 || jobs.job[jb].src != jobs.job[jb - 1].src) gstart[ng++] = jb;
    gstart[ng] = jobs.n;

    const int ntx = (g.nzh + TB - 1) / TB;
    const int ntiles = ntx * (AXIS == 0 ? g.ny : g.xn);
    const int line0 = AXIS == 0 ? 0 : g.x0;
    const int nunits = ((ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x) * ng;
    const int c = threadIdx.x % TB;
    const int ra = threadIdx.x / TB;
    const bool inA = ra < N2, inB = ra < N1;
    const int kb = C::out_base(ra);
    __syncthreads();  // barriers initialised, twiddles staged

    // tile coordinates of unit u: (float column, line, first row) in the 3-D tensor view
    auto tile_of = [&](int u, int& line, int& col0, int& grp) {
        const int tile = (int)blockIdx.x + (u / ng) * (int)gridDim.x;
        grp = u % ng;
        line = line0 + tile / ntx;
        col0 = (tile % ntx) * TB;
    };
    auto box = [&](const CUtensorMap* tm, float2* s, int line, int col0, int q, bool load, uint64_t* b) {
        const int r0 = q * BOXR;
        const int e0 = 2 * col0;
        const int e1 = AXIS == 0 ? line : r0;
        const int e2 = AXIS == 0 ? r0 : line;
        if (load) tma_load_3d(s + r0 * TB, tm, e0, e1, e2, b);
        else tma_store_3d(tm, s + r0 * TB, e0, e1, e2);
    };
    auto prefetch = [&](int u) {
        if (producer && u < nunits) {
            int line, col0, grp;
            tile_of(u, line, col0, grp);
            const int b = u % NBUF;
            float2* xs = xbuf + b * L * TB;
            bulk_wait_read_all();  // the stage may still be the source of a store
            mbar_arrive_expect_tx(&bar[b], TILE_BYTES);
            const CUtensorMap* tm = &maps.tm[jobs.job[gstart[grp]].src];
#pragma unroll
            for (int q = 0; q < NBOX; ++q) box(tm, xs, line, col0, q, true, &bar[b]);
        }
    };
    auto store_tile = [&](float2* xs, int dst, int line, int col0) {
        fence_proxy_async_smem();
        __syncthreads();
        if (producer) {
#pragma unroll
            for (int q = 0; q < NBOX; ++q) box(&maps.tm[dst], xs, line, col0, q, false, nullptr);
            bulk_commit();
        }
    };

    if (DB) prefetch(0);
    for (int u = 0; u < nunits; ++u) {
        const int b = u % NBUF;
        float2* xs = xbuf + b * L * TB;
        if (DB) prefetch(u + 1);
        else prefetch(u);
        mbar_wait(&bar[b], (u / NBUF) & 1);
        int line, col0, grp;
        tile_of(u, line, col0, grp);
        const int gb = gstart[grp], ge = gstart[grp + 1];

        // forward transform of xs -> X (phase-B registers); xs is free afterwards
        auto forward = [&](float2 (&X)[N2]) {
            if (inA) {
                float2 a[N1];
#pragma unroll
                for (int n1 = 0; n1 < N1; ++n1) a[n1] = xs[C::in_row(n1, ra) * TB + c];
                RDft<N1, false>::run(a);
                if constexpr (!C::PFA) {
#pragma unroll
                    for (int k1 = 1; k1 < N1; ++k1) a[k1] = cmul(a[k1], tw[ra * k1]);
                }
#pragma unroll
                for (int k1 = 0; k1 < N1; ++k1) ys[k1 * KP + ra * TB + c] = a[k1];
            }
            __syncthreads();
            if (inB) {
#pragma unroll
                for (int n2 = 0; n2 < N2; ++n2) X[n2] = ys[ra * KP + n2 * TB + c];
                RDft<N2, false>::run(X);
            }
        };
        // inverse of b (phase-B registers, natural order), staged natural-order in xs, stored
        auto inverse_store = [&](float2 (&bb)[N2], int dst) {
            if (inB) {
                RDft<N2, true>::run(bb);
                if constexpr (!C::PFA) {
#pragma unroll
                    for (int n2 = 1; n2 < N2; ++n2) bb[n2] = cmul(bb[n2], conjf2(tw[ra * n2]));
                }
            }
            if (producer) bulk_wait_read_all();  // previous store out of xs
            __syncthreads();
            if (inB) {
#pragma unroll
                for (int n2 = 0; n2 < N2; ++n2) ys[ra * KP + n2 * TB + c] = bb[n2];
            }
            __syncthreads();
            if (inA) {
                float2 a[N1];
#pragma unroll
                for (int k1 = 0; k1 < N1; ++k1) a[k1] = ys[k1 * KP + ra * TB + c];
                RDft<N1, true>::run(a);
#pragma unroll
                for (int n1 = 0; n1 < N1; ++n1) xs[C::in_row(n1, ra) * TB + c] = a[n1];
            }
            store_tile(xs, dst, line, col0);
        };

        float2 X[N2];
        if (AXIS == 1 && !INV) {
            forward(X);
            if (inB) {
#pragma unroll
                for (int k2 = 0; k2 < N2; ++k2) xs[C::out_row(kb, k2) * TB + c] = X[k2];
            }
            store_tile(xs, jobs.job[gb].dst, line, col0);
        } else {
            if (AXIS == 0) {
                // forward x FFT then kappa (all jobs of a source share its kappa flag); kappa of
                // the tile is evaluated once (first source group) into thread-private slots
                forward(X);
                const int kind = jobs.job[gb].kappa;  // one multiplier kind per launch (CTA-uniform)
                if (kind && grp == 0) {
                    if (inB) {
                        const float ky = g.ky[line];
                        const float kz = col0 + c < g.nzh ? g.kz[col0 + c] : 0.f;
                        const bool power = kind >= 2;
                        const float e = jobs.job[gb].kexp;
                        if (power) {
                            for (int k2 = 0; k2 < N2; ++k2) {
                                const int k = C::out_row(kb, k2);
                                const float kx = g.kx[k];
                                kap_s[k * TB + c] = kpow_mult_call(kx * kx + ky * ky + kz * kz, e, kind);
                            }
                        } else {
                            // u = (h kx)^2 + (h ky)^2 + (h kz)^2, the x term from the shared table;
                            // kx^2 is even in k (kx[L-k] = -kx[k]), so kappa is evaluated for
                            // rows k <= L/2 only and mirrored through shared memory
                            const float hy = g.half_cdt * ky, hz = g.half_cdt * kz;
                            const float uyz = hy * hy + hz * hz;
#pragma unroll
                            for (int k2 = 0; k2 < N2; ++k2) {
                                const int k = C::out_row(kb, k2);
                                if (k <= L / 2) kap_s[k * TB + c] = kappa_of_u(hkx2_s[k] + uyz);
                            }
                        }
                    }
                    if (kind < 2) __syncthreads();  // mirrored entries written by other threads
                }
                if (inB && kind) {
#pragma unroll
                    for (int k2 = 0; k2 < N2; ++k2) {
                        const int k = C::out_row(kb, k2);
                        const int km = (kind < 2 && k > L / 2) ? L - k : k;
                        X[k2] = cscale(X[k2], kap_s[km * TB + c]);
                    }
                }
            } else if (inB) {
#pragma unroll
                for (int k2 = 0; k2 < N2; ++k2) X[k2] = xs[C::out_row(kb, k2) * TB + c];
            }
            for (int jb = gb; jb < ge; ++jb) {
                const PencilJob J = jobs.job[jb];
                float2 bb[N2];
                if (inB) {
#pragma unroll
                    for (int k2 = 0; k2 < N2; ++k2)
                        bb[k2] = J.dmul ? cmul(X[k2], __ldg(J.dmul + C::out_row(kb, k2))) : X[k2];
                }
                inverse_store(bb, J.dst);
            }
        }
        __syncthreads();  // ys / kappa slots free for the next unit
    }
    if (producer) bulk_wait_all();
}

#ifndef USTFWI_PASSES_Y_ONLY  // z rows: main translation unit only
// ======================================================================================
// Row (z) passes: real FFT of length nz = 2M through the M-point complex transform
// ======================================================================================
template <int M, int N1, int RW>
struct RowCfg {
    static constexpr int N2 = M / N1;
    static constexpr int TPR = cmax(N1, N2);  // threads per row
    static constexpr int NT = RW * TPR;
    static constexpr int NTG = (NT + 31) / 32 * 32;  // warp-aligned group size (named barriers)
    static constexpr int ZP = N2 + 1;         // transposed tile pitch (bank spread)
    static constexpr int ZT = N1 * ZP;        // float2 per row, transposed layout
    static constexpr int NZ = 2 * M;
    // fixed part of the shared memory: barrier, twiddles, transposed tile, natural tile
    static constexpr size_t FIXED = 16 + size_t(M) * 8 + size_t(RW) * ZT * 8 + size_t(RW) * M * 8;
};

// c2r phase B: half spectrum row (shared, nzh bins, optional premultiplier) -> twiddled
// inverse N2-point transforms, transposed into zt.
template <int M, int N1>
__device__ __forceinline__ void row_c2r_b(const float2* Xrow, const float2* __restrict__ premul,
                                          const float2* __restrict__ twr, const float2* twM, int k1, float2* zt_row) {
    constexpr int N2 = M / N1, ZP = N2 + 1;
    float2 z[N2];
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) {
        const int k = k1 + N1 * k2;
        float2 a = Xrow[k], b = Xrow[M - k];
        if (premul) {
            a = cmul(a, __ldg(premul + k));
            b = cmul(b, __ldg(premul + M - k));
        }
        if (k == 0) {
            a.y = 0.f;
            b.y = 0.f;
        }
        const float2 e = make_float2(a.x + b.x, a.y - b.y);
        const float2 d0 = make_float2(a.x - b.x, a.y + b.y);
        const float2 w = __ldg(twr + k);
        const float2 o = make_float2(d0.x * w.x + d0.y * w.y, d0.y * w.x - d0.x * w.y);
        z[k2] = make_float2(e.x - o.y, e.y + o.x);
    }
    RDft<N2, true>::run(z);
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) zt_row[k1 * ZP + n2] = n2 ? cmul(z[n2], conjf2(twM[k1 * n2])) : z[n2];
}

// c2r phase A: inverse N1-point codelet -> interleaved real pairs (scaled)
template <int M, int N1>
__device__ __forceinline__ void row_c2r_a(const float2* zt_row, int n2, float scale, float2 (&u)[N1]) {
    constexpr int ZP = M / N1 + 1;
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) u[k1] = zt_row[k1 * ZP + n2];
    RDft<N1, true>::run(u);
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) u[n1] = cscale(u[n1], scale);
}

// r2c phase A: pairs u[n1] (n = n2 + N2*n1) -> codelet + twiddle -> zt
template <int M, int N1>
__device__ __forceinline__ void row_r2c_a(float2 (&u)[N1], int n2, const float2* twM, float2* zt_row) {
    constexpr int ZP = M / N1 + 1;
    RDft<N1, false>::run(u);
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) zt_row[k1 * ZP + n2] = k1 ? cmul(u[k1], twM[n2 * k1]) : u[k1];
}
// r2c phase B: codelet -> natural order Z into zn
template <int M, int N1>
__device__ __forceinline__ void row_r2c_b(const float2* zt_row, int k1, float2* zn_row) {
    constexpr int N2 = M / N1, ZP = N2 + 1;
    float2 z[N2];
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) z[n2] = zt_row[k1 * ZP + n2];
    RDft<N2, false>::run(z);
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) zn_row[k1 + N1 * k2] = z[k2];
}
// split into the M+1 half-spectrum bins and store
template <int M, int TPR>
__device__ __forceinline__ void row_r2c_finish(const float2* zn_row, int lane, const float2* __restrict__ twr,
                                               float2* __restrict__ Xrow) {
    for (int k = lane; k <= M; k += TPR) {
        const float2 a = zn_row[k == M ? 0 : k];
        const float2 b = zn_row[k == 0 ? 0 : M - k];
        const float2 e = make_float2(0.5f * (a.x + b.x), 0.5f * (a.y - b.y));
        const float2 o = make_float2(0.5f * (a.y + b.y), -0.5f * (a.x - b.x));
        const float2 w = __ldg(twr + k);
        Xrow[k] = make_float2(e.x + (w.x * o.x - w.y * o.y), e.y + (w.x * o.y + w.y * o.x));
    }
}

struct ZvelFastArgs {
    GridDev g;
    float2* S[3];
    const float2* dz_plus;
    float* v[3];
    Pml pml;
    Coef r[3];
};

// staged bulk copy of `nrows` rows (row_elems elements of T each) of every field
struct Stager {
    uint64_t* bar;
    unsigned bytes = 0;
    template <class T>
    __device__ __forceinline__ void add(T* smem, const T* gmem, unsigned n_elems) {
        const unsigned nb = n_elems * sizeof(T);
        bulk_g2s(smem, gmem, nb, bar);
        bytes += nb;
    }
};

// One CTA per (row block, axis): the three velocity updates are independent
// (v_a needs only dp/dx_a, engine.hpp:275-283), so blockIdx.y selects the axis.
template <int M, int N1, int RW>
__global__ void __launch_bounds__(RowCfg<M, N1, RW>::NT) zvel_fast_kernel(const __grid_constant__ ZvelFastArgs A) {
    using C = RowCfg<M, N1, RW>;
    constexpr int N2 = C::N2, TPR = C::TPR, NZ = C::NZ, NT = C::NT;
    extern __shared__ __align__(128) unsigned char sm_raw[];
    const GridDev& g = A.g;
    const int a = blockIdx.y;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm_raw);
    float2* twM = reinterpret_cast<float2*>(sm_raw + 16);
    float2* zt = twM + M;
    float2* zn = zt + RW * C::ZT;
    float2* sS = zn + RW * M;                                   // [RW*nzp]
    float* sV = reinterpret_cast<float*>(sS + RW * g.nzp);      // [RW*NZ]
    float* sR = sV + RW * NZ;                                   // [RW*NZ] (non-uniform dt/rho0~ only)
    const bool coef_field = A.r[a].field != nullptr;
    float2* const Sa = A.S[a];
    float* const va = A.v[a];

    const long long row0 = (long long)g.x0 * g.ny + (long long)blockIdx.x * RW;
    const int nrows = (int)min((long long)RW, (long long)(g.x0 + g.xn) * g.ny - row0);
    if (threadIdx.x == 0) mbar_init(bar, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned total = nrows * g.nzp * 8u + nrows * NZ * 4u + (coef_field ? nrows * NZ * 4u : 0u);
        mbar_arrive_expect_tx(bar, total);
        Stager st{bar};
        st.add(sS, Sa + row0 * g.nzp, nrows * g.nzp);
        st.add(sV, va + row0 * NZ, nrows * NZ);
        if (coef_field) st.add(sR, A.r[a].field + row0 * NZ, nrows * NZ);
    }
    for (int i = threadIdx.x; i < M; i += NT) twM[i] = g.pzh.tw[i];
    const int r = threadIdx.x / TPR, lane = threadIdx.x % TPR;
    const bool rowok = r < nrows;
    const long long row = row0 + r;
    const int x = rowok ? (int)(row / g.ny) : 0, y = rowok ? (int)(row % g.ny) : 0;
    float2* zt_row = zt + r * C::ZT;
    float2* zn_row = zn + r * M;
    __syncthreads();
    mbar_wait(bar, 0);

    if (rowok && lane < N1) row_c2r_b<M, N1>(sS + r * g.nzp, a == 2 ? A.dz_plus : nullptr, g.tw_rfft, twM, lane, zt_row);
    __syncthreads();
    float2 u[N1];
    if (rowok && lane < N2) {
        row_c2r_a<M, N1>(zt_row, lane, g.inv_n, u);
        const float pa = a == 0 ? __ldg(A.pml.prof[0] + x) : (a == 1 ? __ldg(A.pml.prof[1] + y) : 0.f);
        const float* vs = sV + r * NZ;
        const float* rs = sR + r * NZ;
        float* vg = va + row * NZ;
        const float rsc = A.r[a].scalar;
#pragma unroll
        for (int n1 = 0; n1 < N1; ++n1) {
            const int n = lane + N2 * n1;
            float2 vv = *reinterpret_cast<const float2*>(vs + 2 * n);
            float2 pm = make_float2(pa, pa);
            if (a == 2) pm = *reinterpret_cast<const float2*>(A.pml.prof[2] + 2 * n);
            float2 rr = make_float2(rsc, rsc);
            if (coef_field) rr = *reinterpret_cast<const float2*>(rs + 2 * n);
            vv.x = pm.x * (pm.x * vv.x - rr.x * u[n1].x);
            vv.y = pm.y * (pm.y * vv.y - rr.y * u[n1].y);
            *reinterpret_cast<float2*>(vg + 2 * n) = vv;
            u[n1] = vv;
        }
    }
    __syncthreads();
    if (rowok && lane < N2) row_r2c_a<M, N1>(u, lane, twM, zt_row);
    __syncthreads();
    if (rowok && lane < N1) row_r2c_b<M, N1>(zt_row, lane, zn_row);
    __syncthreads();
    if (rowok) row_r2c_finish<M, TPR>(zn_row, lane, g.tw_rfft, Sa + row * g.nzp);
}

struct ZrhoFastArgs {
    GridDev g;
    ZrhoArgs a;
};

// Density update of one axis per CTA (engine.hpp:284-291): c2r of dv_a/dx_a (D_z- on z),
// rho_a = pml_a (pml_a rho_a - dt rho0 dv_a), written back. The three axes are independent.
template <int M, int N1, int RW>
__global__ void __launch_bounds__(RowCfg<M, N1, RW>::NT) zrho_axis_kernel(const __grid_constant__ ZrhoFastArgs P) {
    using C = RowCfg<M, N1, RW>;
    constexpr int N2 = C::N2, TPR = C::TPR, NZ = C::NZ, NT = C::NT;
    extern __shared__ __align__(128) unsigned char sm_raw[];
    const GridDev& g = P.g;
    const ZrhoArgs& A = P.a;
    const int a = blockIdx.y;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm_raw);
    float2* twM = reinterpret_cast<float2*>(sm_raw + 16);
    float2* zt = twM + M;
    float2* sS = zt + RW * C::ZT;                              // [RW*nzp]
    float* sR = reinterpret_cast<float*>(sS + RW * g.nzp);     // [RW*NZ] rho_a
    float* sD = sR + RW * NZ;                                  // dt*rho0 field (optional)
    const bool coef_field = A.dtrho0.field != nullptr;
    float* const ra = A.rho[a];

    const long long row0 = (long long)g.x0 * g.ny + (long long)blockIdx.x * RW;
    const int nrows = (int)min((long long)RW, (long long)(g.x0 + g.xn) * g.ny - row0);
    const long long i0 = row0 * NZ;
    if (threadIdx.x == 0) mbar_init(bar, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned total = nrows * g.nzp * 8u + nrows * NZ * 4u + (coef_field ? nrows * NZ * 4u : 0u);
        mbar_arrive_expect_tx(bar, total);
        Stager st{bar};
        st.add(sS, A.S[a] + row0 * g.nzp, nrows * g.nzp);
        st.add(sR, ra + i0, nrows * NZ);
        if (coef_field) st.add(sD, A.dtrho0.field + i0, nrows * NZ);
    }
    for (int i = threadIdx.x; i < M; i += NT) twM[i] = g.pzh.tw[i];
    const int r = threadIdx.x / TPR, lane = threadIdx.x % TPR;
    const bool rowok = r < nrows;
    const long long row = row0 + r;
    const int x = rowok ? (int)(row / g.ny) : 0, y = rowok ? (int)(row % g.ny) : 0;
    float2* zt_row = zt + r * C::ZT;
    __syncthreads();
    mbar_wait(bar, 0);

    if (rowok && lane < N1) row_c2r_b<M, N1>(sS + r * g.nzp, a == 2 ? A.dz_minus : nullptr, g.tw_rfft, twM, lane, zt_row);
    __syncthreads();
    if (rowok && lane < N2) {
        float2 u[N1];
        row_c2r_a<M, N1>(zt_row, lane, g.inv_n, u);
        const float pa = a == 0 ? __ldg(A.pml.prof[0] + x) : (a == 1 ? __ldg(A.pml.prof[1] + y) : 0.f);
        const float* rs = sR + r * NZ;
        const float* ds = sD + r * NZ;
        float* rg = ra + row * NZ;
        const float dsc = A.dtrho0.scalar;
#pragma unroll
        for (int n1 = 0; n1 < N1; ++n1) {
            const int n = lane + N2 * n1;
            float2 q = *reinterpret_cast<const float2*>(rs + 2 * n);
            float2 pm = make_float2(pa, pa);
            if (a == 2) pm = *reinterpret_cast<const float2*>(A.pml.prof[2] + 2 * n);
            float2 d = make_float2(dsc, dsc);
            if (coef_field) d = *reinterpret_cast<const float2*>(ds + 2 * n);
            if (A.du_out[a]) *reinterpret_cast<float2*>(A.du_out[a] + row * NZ + 2 * n) = u[n1];
            q.x = pm.x * (pm.x * q.x - d.x * u[n1].x);
            q.y = pm.y * (pm.y * q.y - d.y * u[n1].y);
            *reinterpret_cast<float2*>(rg + 2 * n) = q;
        }
    }
}

// Pressure step (update_pressure, engine.hpp:318-326) with the sparse work that sits between
// the density update and p (mass sources :296-300 / shell Dirichlet :304-307), the gathers
// (simulate.hpp:88-95), the TR correlation (gradient.hpp:177-182) and the r2c of p.
// Thread (row, n2) owns the pairs n = n2 + N2*n1 of its row in registers; sparse entries
// are applied by the owner thread.
template <int M, int N1, int RW>
__global__ void __launch_bounds__(RowCfg<M, N1, RW>::NT) zp_kernel(const __grid_constant__ ZrhoFastArgs P) {
    using C = RowCfg<M, N1, RW>;
    constexpr int N2 = C::N2, TPR = C::TPR, NZ = C::NZ, NT = C::NT;
    extern __shared__ __align__(128) unsigned char sm_raw[];
    const GridDev& g = P.g;
    const ZrhoArgs& A = P.a;
    float2* twM = reinterpret_cast<float2*>(sm_raw + 16);
    float2* zt = twM + M;
    float2* zn = zt + RW * C::ZT;
    __shared__ int sp[8];
    const long long row0 = (long long)g.x0 * g.ny + (long long)blockIdx.x * RW;
    const int nrows = (int)min((long long)RW, (long long)(g.x0 + g.xn) * g.ny - row0);
    const long long i0 = row0 * NZ;
    const int lo_key = (int)i0;
    if (threadIdx.x < 4) {  // one sparse set per thread
        const int k = threadIdx.x;
        if (k == 0) sparse_range(A.inj.pos, A.inj.n_unique, A.inj.blk8, row0, nrows, NZ, sp[0], sp[1]);
        if (k == 1) sparse_range(A.enf.pos, A.enf.n, A.enf.blk8, row0, nrows, NZ, sp[2], sp[3]);
        if (k == 2) sparse_range(A.sens.pos, A.sens.n, A.sens.blk8, row0, nrows, NZ, sp[4], sp[5]);
        if (k == 3) sparse_range(A.shell.pos, A.shell.n, A.shell.blk8, row0, nrows, NZ, sp[6], sp[7]);
    }
    for (int i = threadIdx.x; i < M; i += NT) twM[i] = g.pzh.tw[i];
    const int r = threadIdx.x / TPR, lane = threadIdx.x % TPR;
    const bool rowok = r < nrows;
    const bool act = rowok && lane < N2;
    const long long row = row0 + r;
    float2* zt_row = zt + r * C::ZT;
    float2* zn_row = zn + r * M;

    // all global loads of this thread's pairs first (memory-level parallelism)
    float2 q0[N1], q1[N1], q2[N1], c2[N1];
    if (act) {
#pragma unroll
        for (int n1 = 0; n1 < N1; ++n1) {
            const long long i = row * NZ + 2 * (lane + N2 * n1);
            q0[n1] = *reinterpret_cast<const float2*>(A.rho[0] + i);
            q1[n1] = *reinterpret_cast<const float2*>(A.rho[1] + i);
            q2[n1] = *reinterpret_cast<const float2*>(A.rho[2] + i);
            c2[n1] = *reinterpret_cast<const float2*>(A.c0sq + i);
        }
    }
    __syncthreads();  // sp[] ready

    // sparse sources / shell, applied by the owner of each position
    bool modified = false;
    auto owner_apply = [&](int pos, auto&& fn) {
        const int t = pos - lo_key;
        const int rr = t / NZ, z = t % NZ, n = z >> 1, comp = z & 1;
        if (!(act && rr == r && (n % N2) == lane)) return;
        const int n1 = n / N2;
#pragma unroll
        for (int k = 0; k < N1; ++k)
            if (k == n1) fn(k, comp);
    };
    auto set_rho = [&](int k, int comp, float v, bool add) {
        auto upd = [&](float2& q) {
            float& s = comp ? q.y : q.x;
            s = add ? s + v : v;
        };
        if (A.a_first <= 0) upd(q0[k]);
        if (A.a_first <= 1) upd(q1[k]);
        upd(q2[k]);
    };
    for (int u = sp[0]; u < sp[1]; ++u) {
        const int pos = A.inj.pos[u];
        const float sc = A.inj.scale[u];
        for (int cc = A.inj.csr[u]; cc < A.inj.csr[u + 1]; ++cc) {
            const int n = A.step_n - A.inj.delay[cc];
            if (n < 0 || n >= A.inj.len[cc]) continue;
            const float amp = A.inj.w[cc] * A.inj.sig[A.inj.off[cc] + (long long)n * A.inj.stride[cc]];
            if (amp == 0.f) continue;
            owner_apply(pos, [&](int k, int comp) {
                set_rho(k, comp, amp * sc, true);
                modified = true;
            });
        }
    }
    for (int j = sp[2]; j < sp[3]; ++j) {
        const int pos = A.enf.pos[j];
        owner_apply(pos, [&](int k, int comp) {
            const float c2v = comp ? c2[k].y : c2[k].x;
            set_rho(k, comp, A.enf.vals[j] / (A.enf.ndim * c2v), false);
            modified = true;
        });
    }

    float2 pv[N1];
    if (act) {
#pragma unroll
        for (int n1 = 0; n1 < N1; ++n1) {
            const long long i = row * NZ + 2 * (lane + N2 * n1);
            if (modified) {
                *reinterpret_cast<float2*>(A.rho[0] + i) = q0[n1];
                *reinterpret_cast<float2*>(A.rho[1] + i) = q1[n1];
                *reinterpret_cast<float2*>(A.rho[2] + i) = q2[n1];
            }
            float2 p;
            p.x = c2[n1].x * ((q0[n1].x + q1[n1].x) + q2[n1].x);
            p.y = c2[n1].y * ((q0[n1].y + q1[n1].y) + q2[n1].y);
            if (A.p_out) *reinterpret_cast<float2*>(A.p_out + i) = p;
            pv[n1] = p;
        }
        if (A.corr.grad != nullptr) {
#pragma unroll
            for (int n1 = 0; n1 < N1; ++n1) correlate_pair(A.corr, row * NZ + 2 * (lane + N2 * n1), pv[n1], c2[n1]);
        }
        if (A.check_step > 0 && row == 0 && lane == 0 && !isfinite(pv[0].x)) atomicMin(A.diverged, A.check_step);
    }
    for (int s = sp[4]; s < sp[5]; ++s)
        owner_apply(A.sens.pos[s], [&](int k, int comp) { A.sens.out[A.sens.idx[s]] = comp ? pv[k].y : pv[k].x; });
    for (int j = sp[6]; j < sp[7]; ++j)
        owner_apply(A.shell.pos[j], [&](int k, int comp) { A.shell.out[j] = comp ? pv[k].y : pv[k].x; });

    // forward r2c of p into S0
    if (act) row_r2c_a<M, N1>(pv, lane, twM, zt_row);
    __syncthreads();
    if (rowok && lane < N1) row_r2c_b<M, N1>(zt_row, lane, zn_row);
    __syncthreads();
    if (rowok) row_r2c_finish<M, TPR>(zn_row, lane, g.tw_rfft, A.S[0] + row * g.nzp);
}

// ======================================================================================
// Row (z) passes, paired-residue layout. M = N1*N2 complex points per real row of 2M.
// Thread t of a row owns the phase-B residues r0 = t and r1 = N1 - t (t = 0: 0 and N1/2), a
// set closed under k -> M - k, so the real-FFT split/merge pairs X[k], X[M-k] are both in its
// registers: every spectrum element is read from shared memory once. TPR = N1/2 threads per
// row, all busy in both phases (phase A: N2/TPR codelets each). Rows are staged by TMA bulk
// copies into padded, bank-conflict-free layouts and written back by TMA bulk stores.
// ======================================================================================
constexpr int pad_mod16(int x, int r) {
    while (x % 16 != r) ++x;
    return x;
}
constexpr int pad_mod8(int x, int r) {
    while (x % 8 != r) ++x;
    return x;
}

template <int M, int N1>
struct Z2 {
    static constexpr int N2 = M / N1;
    static constexpr int TPR = N1 / 2;
    static constexpr int NA = N2 / TPR;
    static constexpr int NZ = 2 * M;
    static constexpr int ZP = N2 + 1;                     // zt: [k1][n2] per row
    // complex per zt row. TPR = 8: the two rows of a half-warp are 2 apart (z2_thread), so
    // ZT = 4 mod 8 puts them 16 banks apart; otherwise consecutive rows on disjoint banks.
    static constexpr int ZT = TPR == 8 ? pad_mod8(N1 * ZP, 4) : pad_mod16(N1 * ZP, TPR % 16);
    static constexpr int VP = 2 * pad_mod16(M, 4);        // floats per staged real row
    static_assert(N1 % 2 == 0 && N2 % TPR == 0, "paired-residue split");
};

// Thread -> (row r, residue thread t). 64-bit shared accesses are served per half-warp; with
// TPR = 8 a half-warp holds two rows and the staged rows have pitches of 8 banks mod 32
// (nzp = 132 complex, VP = 264 floats), so the half-warp's rows are r and r + 2 (16 banks
// apart): warp w owns rows 4w + {0, 2, 1, 3}. Other TPR: consecutive rows.
template <int TPR>
__device__ __forceinline__ void z2_thread(int tid, int& r, int& t) {
    if constexpr (TPR == 8) {
        const int w = tid >> 5, l = tid & 31;
        r = 4 * w + 2 * ((l >> 3) & 1) + (l >> 4);
        t = l & 7;
    } else {
        r = tid / TPR;
        t = tid % TPR;
    }
}

// Twiddle tables W_M^(k1*n2) in the two layouts the phases read (conflict-free for
// consecutive t): twA[k1*N2 + n2] (r2c phase A, t -> n2), twB[n2*N1 + r] (c2r phase B, t -> r).
template <int M, int N1>
__device__ __forceinline__ void z2_fill_twiddles(const float2* tw, float2* twA, float2* twB, int tid, int nt) {
    constexpr int N2 = M / N1;
    for (int i = tid; i < M; i += nt) {
        twA[i] = tw[(i / N2) * (i % N2)];
        twB[i] = tw[(i / N1) * (i % N1)];
    }
}

// W_{2M}^k as (W_{2M}^r) * (W_{2M}^{N1*k2}), the second factor compile-time
template <int M, int N1, int K2>
__device__ __forceinline__ float2 twr_of(float2 wr) {
    return twmul<2 * M, N1 * K2, false>(wr);
}

// c2r phase B of one row: spectrum Xs (shared, >= M+1 bins) -> zt (shared), thread t. Called
// by every thread of the CTA: zt may alias the staged spectra of other rows, so the stores
// wait at a barrier until all rows have read theirs.
template <int M, int N1>
__device__ __forceinline__ void z2_c2r_b(const float2* Xs, const float2* pre, const float2* twB, float2 wr0,
                                         float2 wr1, int t, float2* zt, bool rowok) {
    using C = Z2<M, N1>;
    constexpr int N2 = C::N2, ZP = C::ZP;
    const int r0 = t, r1 = t == 0 ? N1 / 2 : N1 - t;
    float2 A[N2], B[N2];
    if (!rowok) Xs = pre = nullptr;
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) {
        A[k2] = Xs ? Xs[r0 + N1 * k2] : make_float2(0.f, 0.f);
        B[k2] = Xs ? Xs[r1 + N1 * k2] : make_float2(0.f, 0.f);
        if (pre) {
            A[k2] = cmul(A[k2], pre[r0 + N1 * k2]);
            B[k2] = cmul(B[k2], pre[r1 + N1 * k2]);
        }
    }
    float2 XM = Xs ? Xs[M] : make_float2(0.f, 0.f);
    if (pre) XM = cmul(XM, pre[M]);
    if (t == 0) {  // DC and Nyquist bins: real parts only (fft.hpp:58-63 keeps the real output)
        A[0].y = 0.f;
        XM.y = 0.f;
    }
    auto zval = [](float2 a, float2 b, float2 w) {
        const float2 e = make_float2(a.x + b.x, a.y - b.y);
        const float2 d0 = make_float2(a.x - b.x, a.y + b.y);
        const float2 o = make_float2(d0.x * w.x + d0.y * w.y, d0.y * w.x - d0.x * w.y);
        return make_float2(e.x - o.y, e.y + o.x);
    };
    float2 za[N2], zb[N2];
    static_for<0, N2>([&](auto K) {
        constexpr int k2 = decltype(K)::value;
        // partners of (r0, k2) and (r1, k2)
        const float2 pa = t == 0 ? (k2 == 0 ? XM : A[(N2 - k2) % N2]) : B[N2 - 1 - k2];
        const float2 pb = t == 0 ? B[N2 - 1 - k2] : A[N2 - 1 - k2];
        za[k2] = zval(A[k2], pa, twr_of<M, N1, k2>(wr0));
        zb[k2] = zval(B[k2], pb, twr_of<M, N1, k2>(wr1));
    });
    RDft<N2, true>::run(za);
    RDft<N2, true>::run(zb);
    __syncthreads();
    if (!rowok) return;
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) {
        zt[r0 * ZP + n2] = n2 ? cmul(za[n2], conjf2(twB[n2 * N1 + r0])) : za[n2];
        zt[r1 * ZP + n2] = n2 ? cmul(zb[n2], conjf2(twB[n2 * N1 + r1])) : zb[n2];
    }
}

// c2r phase A: codelet j of thread t (n2 = t + TPR*j) -> scaled real pairs u[n1] of n = n2 + N2*n1
template <int M, int N1>
__device__ __forceinline__ void z2_c2r_a(const float2* zt, int n2, float scale, float2 (&u)[N1]) {
    using C = Z2<M, N1>;
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) u[k1] = zt[k1 * C::ZP + n2];
    RDft<N1, true>::run(u);
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) u[n1] = cscale(u[n1], scale);
}

// r2c phase A: pairs u[n1] of codelet n2 -> forward N1 codelet + twiddle -> zt
template <int M, int N1>
__device__ __forceinline__ void z2_r2c_a(float2 (&u)[N1], int n2, const float2* twA, float2* zt) {
    using C = Z2<M, N1>;
    RDft<N1, false>::run(u);
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) zt[k1 * C::ZP + n2] = k1 ? cmul(u[k1], twA[k1 * C::N2 + n2]) : u[k1];
}

// r2c phase B + split: zt -> half spectrum X[0..M] written to Xs (thread t's bins)
template <int M, int N1>
__device__ __forceinline__ void z2_r2c_b(const float2* zt, float2 wr0, float2 wr1, int t, float2* Xs) {
    using C = Z2<M, N1>;
    constexpr int N2 = C::N2, ZP = C::ZP;
    const int r0 = t, r1 = t == 0 ? N1 / 2 : N1 - t;
    float2 A[N2], B[N2];
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) {
        A[n2] = zt[r0 * ZP + n2];
        B[n2] = zt[r1 * ZP + n2];
    }
    RDft<N2, false>::run(A);  // Z[r0 + N1*k2]
    RDft<N2, false>::run(B);  // Z[r1 + N1*k2]
    auto xval = [](float2 a, float2 b, float2 w) {
        const float2 e = make_float2(0.5f * (a.x + b.x), 0.5f * (a.y - b.y));
        const float2 o = make_float2(0.5f * (a.y + b.y), -0.5f * (a.x - b.x));
        return make_float2(e.x + (w.x * o.x - w.y * o.y), e.y + (w.x * o.y + w.y * o.x));
    };
    static_for<0, N2>([&](auto K) {
        constexpr int k2 = decltype(K)::value;
        const float2 pa = t == 0 ? A[(N2 - k2) % N2] : B[N2 - 1 - k2];
        const float2 pb = t == 0 ? B[N2 - 1 - k2] : A[N2 - 1 - k2];
        Xs[r0 + N1 * k2] = xval(A[k2], pa, twr_of<M, N1, k2>(wr0));
        Xs[r1 + N1 * k2] = xval(B[k2], pb, twr_of<M, N1, k2>(wr1));
    });
    if (t == 0) Xs[M] = xval(A[0], A[0], make_float2(-1.f, 0.f));
}

// per-row staging: S rows (nzp complex, contiguous in HBM), real rows into a padded pitch
template <int M, int N1, int RW>
struct Z2Smem {
    using C = Z2<M, N1>;
    static constexpr size_t head = 128;  // mbarrier
    static size_t bytes_rho(int nzp, int nreal) {  // zrho2_axis_kernel layout
        return 16 + size_t(M) * 8 + size_t(RW) * cmax(nzp, C::ZT) * 8 + size_t(nreal) * RW * C::VP * 4;
    }
    static size_t bytes(int nzp, int nreal) {
        // the staged spectra and zt share one region (z2_c2r_b)
        return head + size_t(2 * M) * 8 + size_t(M + 2) * 8 + size_t(RW) * cmax(nzp, C::ZT) * 8 +
               size_t(nreal) * RW * C::VP * 4;
    }
};

// Velocity update, one CTA per (row block, axis) (engine.hpp:275-283):
// c2r of kappa*D_a p (D_z+ on z), v_a = pml_a (pml_a v_a - dt/rho~_a * dp), r2c of v_a.
template <int M, int N1, int RW>
__global__ void __launch_bounds__(RW * Z2<M, N1>::TPR) zvel2_kernel(const __grid_constant__ ZvelFastArgs A) {
    using C = Z2<M, N1>;
    constexpr int N2 = C::N2, TPR = C::TPR, NA = C::NA, NZ = C::NZ, VP = C::VP, NT = RW * TPR;
    extern __shared__ __align__(128) unsigned char sm_raw[];
    const GridDev& g = A.g;
    const int a = blockIdx.y;
    const bool coef_field = A.r[a].field != nullptr;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm_raw);
    float2* twA = reinterpret_cast<float2*>(sm_raw + 128);
    float2* twB = twA + M;
    float2* pre = twB + M;                       // D_z+ table (axis 2)
    float2* sS = pre + (M + 2);  // [RW][nzp]; keep 16-B alignment for the bulk copies
    float2* zt = sS;             // [RW][ZT], aliases sS (z2_c2r_b)
    float* sV = reinterpret_cast<float*>(zt + RW * cmax(g.nzp, C::ZT));  // [RW][VP]
    float* sR = sV + RW * VP;                    // [RW][VP] (coefficient field)
    float2* const Sa = A.S[a];
    float* const va = A.v[a];
    const long long row0 = (long long)g.x0 * g.ny + (long long)blockIdx.x * RW;
    const int nrows = (int)min((long long)RW, (long long)(g.x0 + g.xn) * g.ny - row0);

    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_arrive_expect_tx(bar, nrows * g.nzp * 8u + (coef_field ? 2u : 1u) * nrows * NZ * 4u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const int l = threadIdx.x;
        if (l == 0) bulk_g2s(sS, Sa + row0 * g.nzp, nrows * g.nzp * 8u, bar);
        for (int i = l; i < nrows; i += 32) {
            bulk_g2s(sV + i * VP, va + (row0 + i) * NZ, NZ * 4u, bar);
            if (coef_field) bulk_g2s(sR + i * VP, A.r[a].field + (row0 + i) * NZ, NZ * 4u, bar);
        }
    }
    z2_fill_twiddles<M, N1>(g.pzh.tw, twA, twB, threadIdx.x, NT);
    if (a == 2)
        for (int i = threadIdx.x; i <= M; i += NT) pre[i] = A.dz_plus[i];
    int r, t;
    z2_thread<TPR>(threadIdx.x, r, t);
    const bool rowok = r < nrows;
    const long long row = row0 + r;
    const int x = rowok ? (int)(row / g.ny) : 0, y = rowok ? (int)(row % g.ny) : 0;
    const float2 wr0 = g.tw_rfft[t], wr1 = g.tw_rfft[t == 0 ? N1 / 2 : N1 - t];
    float2* ztr = zt + r * C::ZT;
    __syncthreads();
    mbar_wait(bar, 0);

    z2_c2r_b<M, N1>(sS + r * g.nzp, a == 2 ? pre : nullptr, twB, wr0, wr1, t, ztr, rowok);
    __syncthreads();
    if (rowok) {
        const float pa = a == 0 ? __ldg(A.pml.prof[0] + x) : (a == 1 ? __ldg(A.pml.prof[1] + y) : 0.f);
        const float rsc = A.r[a].scalar;
        float* vs = sV + r * VP;
        const float* rs = sR + r * VP;
#pragma unroll
        for (int j = 0; j < NA; ++j) {
            const int n2 = t + TPR * j;
            float2 u[N1];
            z2_c2r_a<M, N1>(ztr, n2, g.inv_n, u);
#pragma unroll
            for (int n1 = 0; n1 < N1; ++n1) {
                const int n = n2 + N2 * n1;
                float2 vv = *reinterpret_cast<const float2*>(vs + 2 * n);
                float2 pm = make_float2(pa, pa);
                if (a == 2) pm = __ldg(reinterpret_cast<const float2*>(A.pml.prof[2]) + n);
                float2 rr = make_float2(rsc, rsc);
                if (coef_field) rr = *reinterpret_cast<const float2*>(rs + 2 * n);
                vv.x = pm.x * (pm.x * vv.x - rr.x * u[n1].x);
                vv.y = pm.y * (pm.y * vv.y - rr.y * u[n1].y);
                *reinterpret_cast<float2*>(va + row * NZ + 2 * n) = vv;
                u[n1] = vv;
            }
            z2_r2c_a<M, N1>(u, n2, twA, ztr);  // the same zt entries this thread just read
        }
    }
    __syncthreads();
    if (rowok) z2_r2c_b<M, N1>(ztr, wr0, wr1, t, Sa + row * g.nzp);
}

// Density update of one axis per CTA (engine.hpp:284-291): c2r of dv_a/dx_a (D_z- on z),
// rho_a = pml_a (pml_a rho_a - dt rho0 dv_a).
template <int M, int N1, int RW>
__global__ void __launch_bounds__(RW * Z2<M, N1>::TPR) zrho2_axis_kernel(const __grid_constant__ ZrhoFastArgs P) {
    using C = Z2<M, N1>;
    constexpr int N2 = C::N2, TPR = C::TPR, NA = C::NA, NZ = C::NZ, VP = C::VP, NT = RW * TPR;
    extern __shared__ __align__(128) unsigned char sm_raw[];
    const GridDev& g = P.g;
    const ZrhoArgs& A = P.a;
    const int a = blockIdx.y;
    const bool coef_field = A.dtrho0.field != nullptr;
    // c2r only: one twiddle table, D_z- read through L1 (Z2SmemRho: 6 CTAs / SM at M = 128)
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm_raw);
    float2* twB = reinterpret_cast<float2*>(sm_raw + 16);
    float2* sS = twB + M;        // 16-B aligned for the bulk copies
    float2* zt = sS;             // aliases sS (z2_c2r_b)
    float* sR = reinterpret_cast<float*>(zt + RW * cmax(g.nzp, C::ZT));  // rho_a rows
    float* sD = sR + RW * VP;                               // dt*rho0 field rows (optional)
    float* const ra = A.rho[a];
    const long long row0 = (long long)g.x0 * g.ny + (long long)blockIdx.x * RW;
    const int nrows = (int)min((long long)RW, (long long)(g.x0 + g.xn) * g.ny - row0);

    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_arrive_expect_tx(bar, nrows * g.nzp * 8u + (coef_field ? 2u : 1u) * nrows * NZ * 4u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const int l = threadIdx.x;
        if (l == 0) bulk_g2s(sS, A.S[a] + row0 * g.nzp, nrows * g.nzp * 8u, bar);
        for (int i = l; i < nrows; i += 32) {
            bulk_g2s(sR + i * VP, ra + (row0 + i) * NZ, NZ * 4u, bar);
            if (coef_field) bulk_g2s(sD + i * VP, A.dtrho0.field + (row0 + i) * NZ, NZ * 4u, bar);
        }
    }
    for (int i = threadIdx.x; i < M; i += NT) twB[i] = g.pzh.tw[(i / N1) * (i % N1)];
    const float2* pre = a == 2 ? A.dz_minus : nullptr;
    int r, t;
    z2_thread<TPR>(threadIdx.x, r, t);
    const bool rowok = r < nrows;
    const long long row = row0 + r;
    const int x = rowok ? (int)(row / g.ny) : 0, y = rowok ? (int)(row % g.ny) : 0;
    const float2 wr0 = g.tw_rfft[t], wr1 = g.tw_rfft[t == 0 ? N1 / 2 : N1 - t];
    float2* ztr = zt + r * C::ZT;
    __syncthreads();
    mbar_wait(bar, 0);

    z2_c2r_b<M, N1>(sS + r * g.nzp, pre, twB, wr0, wr1, t, ztr, rowok);
    __syncthreads();
    if (rowok) {
        const float pa = a == 0 ? __ldg(A.pml.prof[0] + x) : (a == 1 ? __ldg(A.pml.prof[1] + y) : 0.f);
        const float dsc = A.dtrho0.scalar;
        float* rs = sR + r * VP;
        const float* ds = sD + r * VP;
#pragma unroll
        for (int j = 0; j < NA; ++j) {
            const int n2 = t + TPR * j;
            float2 u[N1];
            z2_c2r_a<M, N1>(ztr, n2, g.inv_n, u);
#pragma unroll
            for (int n1 = 0; n1 < N1; ++n1) {
                const int n = n2 + N2 * n1;
                float2 q = *reinterpret_cast<const float2*>(rs + 2 * n);
                float2 pm = make_float2(pa, pa);
                if (a == 2) pm = __ldg(reinterpret_cast<const float2*>(A.pml.prof[2]) + n);
                float2 d = make_float2(dsc, dsc);
                if (coef_field) d = *reinterpret_cast<const float2*>(ds + 2 * n);
                if (A.du_out[a]) *reinterpret_cast<float2*>(A.du_out[a] + row * NZ + 2 * n) = u[n1];
                q.x = pm.x * (pm.x * q.x - d.x * u[n1].x);
                q.y = pm.y * (pm.y * q.y - d.y * u[n1].y);
                *reinterpret_cast<float2*>(ra + row * NZ + 2 * n) = q;
            }
        }
    }
}

// Pressure step in the paired-residue layout (update_pressure, engine.hpp:318-326), with the
// sparse work between the density update and p (mass sources :296-300, shell Dirichlet
// :304-307), the gathers (simulate.hpp:88-95), the TR correlation (gradient.hpp:177-182)
// and the r2c of p. Sparse updates are applied by the owner thread of each position straight
// to the split densities in HBM, in reference order, before that thread reads them.
#ifndef USTFWI_ZP_CHUNK
#define USTFWI_ZP_CHUNK 2
#endif
#ifndef USTFWI_ZP_MINB
#define USTFWI_ZP_MINB 8
#endif
// the correlating variant: 4 elements per load batch at 4 CTAs / SM (110 registers) measured
// best on D200 (z-rho class 0.811 -> 0.803 ms; 2 at 6, 4 at 5 and 1 at 8 CTAs / SM measured)
#ifndef USTFWI_ZPC_MINB
#define USTFWI_ZPC_MINB 4
#endif
#ifndef USTFWI_ZPC_CHUNK
#define USTFWI_ZPC_CHUNK 4
#endif
template <int M, int N1, int RW, bool CORR, bool STORE_P>
__global__ void __launch_bounds__(RW * Z2<M, N1>::TPR, CORR ? USTFWI_ZPC_MINB : USTFWI_ZP_MINB)
    zp2_kernel(const __grid_constant__ ZrhoFastArgs P) {
    using C = Z2<M, N1>;
    constexpr int N2 = C::N2, TPR = C::TPR, NA = C::NA, NZ = C::NZ, NT = RW * TPR;
    extern __shared__ __align__(128) unsigned char sm_raw[];
    const GridDev& g = P.g;
    const ZrhoArgs& A = P.a;
    float2* twA = reinterpret_cast<float2*>(sm_raw);  // r2c only: one table
    float2* zt = twA + M;
    __shared__ int sp[8];
    const long long row0 = (long long)g.x0 * g.ny + (long long)blockIdx.x * RW;
    const int nrows = (int)min((long long)RW, (long long)(g.x0 + g.xn) * g.ny - row0);
    const long long i0 = row0 * NZ;
    const int lo_key = (int)i0;
    if (threadIdx.x < 4) {  // one sparse set per thread
        const int k = threadIdx.x;
        if (k == 0) sparse_range(A.inj.pos, A.inj.n_unique, A.inj.blk8, row0, nrows, NZ, sp[0], sp[1]);
        if (k == 1) sparse_range(A.enf.pos, A.enf.n, A.enf.blk8, row0, nrows, NZ, sp[2], sp[3]);
        if (k == 2) sparse_range(A.sens.pos, A.sens.n, A.sens.blk8, row0, nrows, NZ, sp[4], sp[5]);
        if (k == 3) sparse_range(A.shell.pos, A.shell.n, A.shell.blk8, row0, nrows, NZ, sp[6], sp[7]);
    }
    for (int i = threadIdx.x; i < M; i += NT) twA[i] = g.pzh.tw[(i / N2) * (i % N2)];
    int r, t;
    z2_thread<TPR>(threadIdx.x, r, t);
    const bool rowok = r < nrows;
    const long long row = row0 + r;
    float2* ztr = zt + r * C::ZT;
    __syncthreads();  // sp[] and twiddles ready

    // owner of flat position pos: row, pair n = z/2 with n % N2 in this thread's codelets
    auto owns = [&](int pos, int& j, int& n1, int& comp) {
        const int tt = pos - lo_key;
        const int rr = tt / NZ, z = tt % NZ, n = z >> 1;
        comp = z & 1;
        const int n2 = n % N2;
        if (!(rowok && rr == r && n2 % TPR == t)) return false;
        j = n2 / TPR;
        n1 = n / N2;
        return true;
    };
    // sparse density updates, in the reference order (sources, then the shell)
    if (rowok) {
        for (int u = sp[0]; u < sp[1]; ++u) {
            const int pos = A.inj.pos[u];
            int j, n1, comp;
            if (!owns(pos, j, n1, comp)) continue;
            const float sc = A.inj.scale[u];
            for (int cc = A.inj.csr[u]; cc < A.inj.csr[u + 1]; ++cc) {
                const int n = A.step_n - A.inj.delay[cc];
                if (n < 0 || n >= A.inj.len[cc]) continue;
                const float amp = A.inj.w[cc] * A.inj.sig[A.inj.off[cc] + (long long)n * A.inj.stride[cc]];
                if (amp == 0.f) continue;
                for (int aa = max(A.a_first, 0); aa < 3; ++aa) A.rho[aa][pos] += amp * sc;
            }
        }
        for (int q = sp[2]; q < sp[3]; ++q) {
            const int pos = A.enf.pos[q];
            int j, n1, comp;
            if (!owns(pos, j, n1, comp)) continue;
            const float v = A.enf.vals[q] / (A.enf.ndim * A.c0sq[pos]);
            for (int aa = max(A.a_first, 0); aa < 3; ++aa) A.rho[aa][pos] = v;
        }
    }

    float2 pv[NA][N1];
    if (rowok) {
        // ZPC elements per batch: every stream load of a batch is issued before its first
        // store (the stores to p_out / grad may alias the streams as far as the compiler
        // knows, so without batching each element waits out its own load latency). Pairs at
        // the 64-register cap (8 CTAs / SM, USTFWI_ZP_MINB) measured best: D200 1.705 ->
        // 1.695 s / gradient; 4 / 8 per batch or an uncapped 80-96 registers were slower
        constexpr int CH = CORR ? USTFWI_ZPC_CHUNK : USTFWI_ZP_CHUNK;
        constexpr int ZPC = N1 % CH == 0 ? CH : (N1 % 2 == 0 ? 2 : 1);
#pragma unroll
        for (int j = 0; j < NA; ++j) {
            const int n2 = t + TPR * j;
#pragma unroll
            for (int c0 = 0; c0 < N1; c0 += ZPC) {
                float2 q0[ZPC], q1[ZPC], q2[ZPC], c2[ZPC];
                float2 pm[CORR ? ZPC : 1], po[CORR ? ZPC : 1], pq[CORR ? ZPC : 1], gv[CORR ? ZPC : 1];
                // correlation: the replay's p_new (adjoint kernel) or q (replay kernel)
                const float* other = CORR ? (A.corr.p_new ? A.corr.p_new : A.corr.q_adj) : nullptr;
#pragma unroll
                for (int k = 0; k < ZPC; ++k) {
                    const long long i = row * NZ + 2 * (n2 + N2 * (c0 + k));
                    q0[k] = *reinterpret_cast<const float2*>(A.rho[0] + i);
                    q1[k] = *reinterpret_cast<const float2*>(A.rho[1] + i);
                    q2[k] = *reinterpret_cast<const float2*>(A.rho[2] + i);
                    c2[k] = __ldg(reinterpret_cast<const float2*>(A.c0sq + i));
                    if constexpr (CORR) {  // issued with the stream loads, before any store
                        pm[k] = *reinterpret_cast<const float2*>(A.corr.p_mid + i);
                        po[k] = *reinterpret_cast<const float2*>(A.corr.p_old + i);
                        pq[k] = *reinterpret_cast<const float2*>(other + i);
                        gv[k] = *reinterpret_cast<const float2*>(A.corr.grad + i);
                    }
                }
#pragma unroll
                for (int k = 0; k < ZPC; ++k) {
                    const int n1 = c0 + k;
                    const long long i = row * NZ + 2 * (n2 + N2 * n1);
                    float2 p;
                    p.x = c2[k].x * ((q0[k].x + q1[k].x) + q2[k].x);
                    p.y = c2[k].y * ((q0[k].y + q1[k].y) + q2[k].y);
                    if constexpr (STORE_P) *reinterpret_cast<float2*>(A.p_out + i) = p;
                    pv[j][n1] = p;
                    if constexpr (CORR) {
                        // correlate_pair with the loads hoisted: the same fp32 operations
                        const bool adj = A.corr.p_new != nullptr;
                        const float2 pn = adj ? pq[k] : p, qa = adj ? p : pq[k];
                        const float wx = 2.f / (c2[k].x * sqrtf(c2[k].x)), wy = 2.f / (c2[k].y * sqrtf(c2[k].y));
                        float2 g2 = gv[k];
                        g2.x += wx * (((pn.x - 2.f * pm[k].x) + po[k].x) * A.corr.inv_dt) * qa.x;
                        g2.y += wy * (((pn.y - 2.f * pm[k].y) + po[k].y) * A.corr.inv_dt) * qa.y;
                        *reinterpret_cast<float2*>(A.corr.grad + i) = g2;
                    }
                }
            }
        }
        if (A.check_step > 0 && row == 0 && t == 0 && !isfinite(pv[0][0].x)) atomicMin(A.diverged, A.check_step);
        // gathers of p by the owner thread
        auto gather = [&](int pos, float* out) {
            int j, n1, comp;
            if (!owns(pos, j, n1, comp)) return;
#pragma unroll
            for (int jj = 0; jj < NA; ++jj)
#pragma unroll
                for (int k = 0; k < N1; ++k)
                    if (jj == j && k == n1) *out = comp ? pv[jj][k].y : pv[jj][k].x;
        };
        for (int s = sp[4]; s < sp[5]; ++s) gather(A.sens.pos[s], A.sens.out + A.sens.idx[s]);
        for (int q = sp[6]; q < sp[7]; ++q) gather(A.shell.pos[q], A.shell.out + q);
        // forward r2c of p into S0
#pragma unroll
        for (int j = 0; j < NA; ++j) z2_r2c_a<M, N1>(pv[j], t + TPR * j, twA, ztr);
    }
    __syncthreads();
    if (rowok) {
        const float2 wr0 = g.tw_rfft[t], wr1 = g.tw_rfft[t == 0 ? N1 / 2 : N1 - t];
        z2_r2c_b<M, N1>(ztr, wr0, wr1, t, A.S[0] + row * g.nzp);
    }
}

#endif  // USTFWI_PASSES_Y_ONLY

// ======================================================================================
// dispatch
// ======================================================================================
namespace {

// Density update of all three axes and the pressure step in one CTA per row block
// (engine.hpp:284-291 + :296-347): per axis the staged spectrum rows are inverse transformed
// (D_z- on z), rho_a = pml_a (pml_a rho_a - dt rho0 dv_a) is formed in registers, the sparse
// work of the owner thread (sources += amp * scale, shell = value, reference order) is applied
// to the register value, rho_a is stored and summed; then p = c0^2 sum_a rho_a, the TR
// correlation, the gathers and the r2c of p follow as in zp2_kernel. Against the split
// zrho2_axis + zp2 pair it does not re-read the three split densities (48 instead of 60 B per
// voxel). Non-absorbing steps only (the absorbing path keeps the raw derivatives).
#ifndef USTFWI_PASSES_Y_ONLY
template <int M, int N1, int RW>
__global__ void __launch_bounds__(RW * Z2<M, N1>::TPR, 4) zrhop_kernel(const __grid_constant__ ZrhoFastArgs P) {
    using C = Z2<M, N1>;
    constexpr int N2 = C::N2, TPR = C::TPR, NA = C::NA, NZ = C::NZ, VP = C::VP, NT = RW * TPR;
    extern __shared__ __align__(128) unsigned char sm_raw[];
    const GridDev& g = P.g;
    const ZrhoArgs& A = P.a;
    const bool coef_field = A.dtrho0.field != nullptr;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm_raw);   // [0] spectra + rho rows, [1] coefficient rows
    __shared__ int sp[8];
    float2* twB = reinterpret_cast<float2*>(sm_raw + 32);  // c2r twiddles
    float2* twA = twB + M;                                   // r2c twiddles
    float2* sS = twA + M;                                    // [RW][nzp] staged spectrum rows
    float2* zt = sS;                                         // aliases sS (z2_c2r_b)
    float* sR = reinterpret_cast<float*>(zt + RW * cmax(g.nzp, C::ZT));  // rho_a rows
    float* sSum = sR + RW * VP;                              // running sum_a rho_a (owner-private slots)
    float* sD = sSum + RW * VP;                              // dt*rho0 rows (optional)
    const long long row0 = (long long)g.x0 * g.ny + (long long)blockIdx.x * RW;
    const int nrows = (int)min((long long)RW, (long long)(g.x0 + g.xn) * g.ny - row0);
    const long long i0 = row0 * NZ;
    const int lo_key = (int)i0;

    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
    }
    if (threadIdx.x < 4) {  // one sparse set per thread
        const int k = threadIdx.x;
        if (k == 0) sparse_range(A.inj.pos, A.inj.n_unique, A.inj.blk8, row0, nrows, NZ, sp[0], sp[1]);
        if (k == 1) sparse_range(A.enf.pos, A.enf.n, A.enf.blk8, row0, nrows, NZ, sp[2], sp[3]);
        if (k == 2) sparse_range(A.sens.pos, A.sens.n, A.sens.blk8, row0, nrows, NZ, sp[4], sp[5]);
        if (k == 3) sparse_range(A.shell.pos, A.shell.n, A.shell.blk8, row0, nrows, NZ, sp[6], sp[7]);
    }
    for (int i = threadIdx.x; i < M; i += NT) {
        twB[i] = g.pzh.tw[(i / N1) * (i % N1)];
        twA[i] = g.pzh.tw[(i / N2) * (i % N2)];
    }
    __syncthreads();  // barriers initialised
    auto stage = [&](int a) {  // thread 0 arms, warp 0 issues the axis's bulk copies
        if (threadIdx.x == 0)
            mbar_arrive_expect_tx(&bar[0], nrows * g.nzp * 8u + nrows * NZ * 4u);
        __syncwarp();
        if (threadIdx.x < 32) {
            const int l = threadIdx.x;
            if (l == 0) bulk_g2s(sS, A.S[a] + row0 * g.nzp, nrows * g.nzp * 8u, &bar[0]);
            for (int i = l; i < nrows; i += 32) bulk_g2s(sR + i * VP, A.rho[a] + (row0 + i) * NZ, NZ * 4u, &bar[0]);
        }
    };
    if (coef_field && threadIdx.x < 32) {
        if (threadIdx.x == 0) mbar_arrive_expect_tx(&bar[1], nrows * NZ * 4u);
        __syncwarp();
        for (int i = threadIdx.x; i < nrows; i += 32)
            bulk_g2s(sD + i * VP, A.dtrho0.field + (row0 + i) * NZ, NZ * 4u, &bar[1]);
    }
    const int a_first = max(A.a_first, 0);
    stage(a_first);
    int r, t;
    z2_thread<TPR>(threadIdx.x, r, t);
    const bool rowok = r < nrows;
    const long long row = row0 + r;
    const int x = rowok ? (int)(row / g.ny) : 0, y = rowok ? (int)(row % g.ny) : 0;
    const float2 wr0 = g.tw_rfft[t], wr1 = g.tw_rfft[t == 0 ? N1 / 2 : N1 - t];
    float2* ztr = zt + r * C::ZT;
    // owner of flat position pos: row, pair n = z/2 with n % N2 in this thread's codelets
    auto owns = [&](int pos, int& j, int& n1, int& comp) {
        const int tt = pos - lo_key;
        const int rr = tt / NZ, z = tt % NZ, n = z >> 1;
        comp = z & 1;
        const int n2 = n % N2;
        if (!(rowok && rr == r && n2 % TPR == t)) return false;
        j = n2 / TPR;
        n1 = n / N2;
        return true;
    };
    float* sumr = sSum + r * VP;
    if (coef_field) mbar_wait(&bar[1], 0);
    const float dsc = A.dtrho0.scalar;

    unsigned phase = 0;
    for (int a = a_first; a < 3; ++a) {
        mbar_wait(&bar[0], phase);
        phase ^= 1u;
        z2_c2r_b<M, N1>(sS + r * g.nzp, a == 2 ? A.dz_minus : nullptr, twB, wr0, wr1, t, ztr, rowok);
        __syncthreads();
        float2 q[NA][N1];
        if (rowok) {
            const float pa = a == 0 ? __ldg(A.pml.prof[0] + x) : (a == 1 ? __ldg(A.pml.prof[1] + y) : 0.f);
            const float* rs = sR + r * VP;
            const float* ds = sD + r * VP;
#pragma unroll
            for (int j = 0; j < NA; ++j) {
                const int n2 = t + TPR * j;
                float2 u[N1];
                z2_c2r_a<M, N1>(ztr, n2, g.inv_n, u);
#pragma unroll
                for (int n1 = 0; n1 < N1; ++n1) {
                    const int n = n2 + N2 * n1;
                    float2 v = *reinterpret_cast<const float2*>(rs + 2 * n);
                    float2 pm = make_float2(pa, pa);
                    if (a == 2) pm = __ldg(reinterpret_cast<const float2*>(A.pml.prof[2]) + n);
                    float2 d = make_float2(dsc, dsc);
                    if (coef_field) d = *reinterpret_cast<const float2*>(ds + 2 * n);
                    v.x = pm.x * (pm.x * v.x - d.x * u[n1].x);
                    v.y = pm.y * (pm.y * v.y - d.y * u[n1].y);
                    q[j][n1] = v;
                }
            }
            // sparse density updates of the owner thread, in the reference order (sources,
            // then the shell), on the register values
            auto modify = [&](int pos, bool set, float val) {
                int j, n1, comp;
                if (!owns(pos, j, n1, comp)) return;
#pragma unroll
                for (int jj = 0; jj < NA; ++jj)
#pragma unroll
                    for (int k = 0; k < N1; ++k)
                        if (jj == j && k == n1) {
                            float& e = comp ? q[jj][k].y : q[jj][k].x;
                            e = set ? val : e + val;
                        }
            };
            for (int uu = sp[0]; uu < sp[1]; ++uu) {
                const int pos = A.inj.pos[uu];
                const float sc = A.inj.scale[uu];
                for (int cc = A.inj.csr[uu]; cc < A.inj.csr[uu + 1]; ++cc) {
                    const int n = A.step_n - A.inj.delay[cc];
                    if (n < 0 || n >= A.inj.len[cc]) continue;
                    const float amp = A.inj.w[cc] * A.inj.sig[A.inj.off[cc] + (long long)n * A.inj.stride[cc]];
                    if (amp == 0.f) continue;
                    modify(pos, false, amp * sc);
                }
            }
            for (int qq = sp[2]; qq < sp[3]; ++qq) {
                const int pos = A.enf.pos[qq];
                modify(pos, true, A.enf.vals[qq] / (A.enf.ndim * A.c0sq[pos]));
            }
#pragma unroll
            for (int j = 0; j < NA; ++j) {
                const int n2 = t + TPR * j;
#pragma unroll
                for (int n1 = 0; n1 < N1; ++n1) {
                    const int n = n2 + N2 * n1;
                    *reinterpret_cast<float2*>(A.rho[a] + row * NZ + 2 * n) = q[j][n1];
                    float2* sm2 = reinterpret_cast<float2*>(sumr + 2 * n);
                    if (a == a_first) {
                        *sm2 = q[j][n1];
                    } else {
                        const float2 o = *sm2;
                        *sm2 = make_float2(o.x + q[j][n1].x, o.y + q[j][n1].y);
                    }
                }
            }
        }
        __syncthreads();  // sS / sR free for the next axis
        if (a + 1 < 3) stage(a + 1);
    }

    float2 pv[NA][N1];
    if (rowok) {
#pragma unroll
        for (int j = 0; j < NA; ++j) {
            const int n2 = t + TPR * j;
#pragma unroll
            for (int n1 = 0; n1 < N1; ++n1) {
                const long long i = row * NZ + 2 * (n2 + N2 * n1);
                const float2 c2 = __ldg(reinterpret_cast<const float2*>(A.c0sq + i));
                const float2 sm = *reinterpret_cast<const float2*>(sumr + 2 * (n2 + N2 * n1));
                float2 p;
                p.x = c2.x * sm.x;
                p.y = c2.y * sm.y;
                if (A.p_out) *reinterpret_cast<float2*>(A.p_out + i) = p;
                pv[j][n1] = p;
                if (A.corr.grad != nullptr) correlate_pair(A.corr, i, p, c2);
            }
        }
        if (A.check_step > 0 && row == 0 && t == 0 && !isfinite(pv[0][0].x)) atomicMin(A.diverged, A.check_step);
        auto gather = [&](int pos, float* out) {
            int j, n1, comp;
            if (!owns(pos, j, n1, comp)) return;
#pragma unroll
            for (int jj = 0; jj < NA; ++jj)
#pragma unroll
                for (int k = 0; k < N1; ++k)
                    if (jj == j && k == n1) *out = comp ? pv[jj][k].y : pv[jj][k].x;
        };
        for (int s2 = sp[4]; s2 < sp[5]; ++s2) gather(A.sens.pos[s2], A.sens.out + A.sens.idx[s2]);
        for (int q2 = sp[6]; q2 < sp[7]; ++q2) gather(A.shell.pos[q2], A.shell.out + q2);
#pragma unroll
        for (int j = 0; j < NA; ++j) z2_r2c_a<M, N1>(pv[j], t + TPR * j, twA, ztr);
    }
    __syncthreads();
    if (rowok) z2_r2c_b<M, N1>(ztr, wr0, wr1, t, A.S[0] + row * g.nzp);
}
#endif  // !USTFWI_PASSES_Y_ONLY

int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

template <int AXIS, bool INV, int L, int N1, int TB, int MINB, bool DB>
cudaError_t run_pencil(const GridDev& g, const PencilJobs& j, cudaStream_t st) {
    using C = PencilCfg<L, N1, TB, DB>;
    auto kern = pencil_fast_kernel<AXIS, INV, L, N1, TB, MINB, DB>;
    static std::atomic<unsigned long long> configured{0};
    constexpr size_t smem = AXIS == 0 ? C::SMEM_X : C::SMEM;
    once_per_device(configured, [&] { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); });
    const int ntiles = ((g.nzh + TB - 1) / TB) * (AXIS == 0 ? g.ny : g.xn);
    int grid = (!DB || ntiles < sm_count() * MINB) ? ntiles : sm_count() * MINB;
    if (DB && g.pgrid > 0 && g.pgrid < grid) grid = g.pgrid;
    kern<<<grid, C::NT, smem, st>>>(g, j);
    return cudaGetLastError();
}

// ---- TMA tensor maps of the scratch spectra, viewed as fp32 [nx][ny][2*nzp] ----
using EncodeTiledFn = PFN_cuTensorMapEncodeTiled_v12000;

EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<EncodeTiledFn>(nullptr);
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

bool use_pencil_tma() {
    static int on = -1;
    if (on < 0) {
        const char* e = std::getenv("USTFWI_PENCIL_TMA");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1 && encode_tiled() != nullptr;
}

// box = (2*TB floats, rows) along the pass axis; cached per thread (the map depends only on
// the buffer address, the grid and the box, so a reused address gives the same map)
bool pencil_map(CUtensorMap* out, const float2* buf, const GridDev& g, int axis, int TB, int boxr) {
    struct Entry {
        const float2* buf;
        int nx, ny, nzp, axis, tb, boxr;
        CUtensorMap map;
    };
    thread_local std::vector<Entry> cache;
    for (const Entry& e : cache)
        if (e.buf == buf && e.nx == g.nx && e.ny == g.ny && e.nzp == g.nzp && e.axis == axis && e.tb == TB &&
            e.boxr == boxr) {
            *out = e.map;
            return true;
        }
    cuuint64_t dims[3] = {2ull * g.nzp, static_cast<cuuint64_t>(g.ny), static_cast<cuuint64_t>(g.nx)};
    cuuint64_t strides[2] = {8ull * g.nzp, 8ull * g.nzp * g.ny};
    cuuint32_t box[3] = {2u * TB, axis == 0 ? 1u : static_cast<cuuint32_t>(boxr),
                         axis == 0 ? static_cast<cuuint32_t>(boxr) : 1u};
    cuuint32_t es[3] = {1, 1, 1};
    Entry e{buf, g.nx, g.ny, g.nzp, axis, TB, boxr, {}};
    if (encode_tiled()(&e.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float2*>(buf), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    if (cache.size() >= 64) cache.erase(cache.begin());
    cache.push_back(e);
    *out = e.map;
    return true;
}

template <int AXIS, bool INV, int L, int N1, int TB, int MINB, bool DB>
cudaError_t run_pencil_tma(const GridDev& g, const PencilJobs& j, cudaStream_t st) {
    using C = PencilCfg<L, N1, TB, DB>;
    constexpr int BOXR = L > 256 ? L / 2 : L;
    PencilMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    for (int f = 0; f < 3; ++f)
        if (j.buf[f] && !pencil_map(&maps.tm[f], j.buf[f], g, AXIS, TB, BOXR)) return cudaErrorInvalidValue;
    auto kern = pencil_tma_kernel<AXIS, INV, L, N1, TB, MINB, DB>;
    constexpr size_t smem = 128 + ((DB ? 2 : 1) * size_t(L) * TB + size_t(N1) * C::KP + L) * sizeof(float2) +
                            (AXIS == 0 ? size_t(L) * (TB + 1) * sizeof(float) : 0);
    static std::atomic<unsigned long long> configured{0};
    once_per_device(configured, [&] {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    const int ntiles = ((g.nzh + TB - 1) / TB) * (AXIS == 0 ? g.ny : g.xn);
    int grid = (!DB || ntiles < sm_count() * MINB) ? ntiles : sm_count() * MINB;
    if (DB && g.pgrid > 0 && g.pgrid < grid) grid = g.pgrid;
    static int occ = -1;
    if (occ < 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::NT, smem);
        if (std::getenv("USTFWI_CHAIN_STATS"))
            fprintf(stderr, "pencil_tma_kernel<%d,%d,%d>: %d CTAs per SM (smem %zu B)\n", AXIS, (int)INV, L, occ, smem);
    }
    kern<<<grid, C::NT, smem, st>>>(g, j, maps);
    return cudaGetLastError();
}

// x passes are instantiated in the main translation unit, y passes only in passes_y.cu
// (compiled with USTFWI_FFT_SCALAR_ADD, fft_smem.cuh)
template <int L, int N1, int TB, int MINB, bool DB>
cudaError_t pencil_sized(int axis, bool inv, const GridDev& g, const PencilJobs& j, cudaStream_t st) {
#ifdef USTFWI_PASSES_Y_ONLY
    if (axis != 1) return cudaErrorInvalidValue;
    if (use_pencil_tma())
        return inv ? run_pencil_tma<1, true, L, N1, TB, MINB, DB>(g, j, st)
                   : run_pencil_tma<1, false, L, N1, TB, MINB, DB>(g, j, st);
    return inv ? run_pencil<1, true, L, N1, TB, MINB, DB>(g, j, st)
               : run_pencil<1, false, L, N1, TB, MINB, DB>(g, j, st);
#else
    if (axis != 0) return cudaErrorInvalidValue;
    if (use_pencil_tma()) return run_pencil_tma<0, false, L, N1, TB, MINB, DB>(g, j, st);
    return run_pencil<0, false, L, N1, TB, MINB, DB>(g, j, st);
#endif
}

#ifndef USTFWI_PASSES_Y_ONLY
// ======================================================================================
// y-x-y chain: one persistent launch for Fy -> (Fx, multiply, Fx^-1) -> Fy^-1
// ======================================================================================
// The two pencil chains of a step (run_step) each read and write every spectrum three times
// when run as separate launches (18 S per voxel for the density chain). Here the grid is cut
// into kz-column slabs (TB columns, all x and y: 480 x 480 x 8 complex = 14.7 MB per field at
// config D) and the units of a slab run in order: phase A = y-forward tiles (one per x plane),
// phase B = x tiles (one per y line, kappa / D_x and the inverse x FFT), phase C = y-inverse
// tiles. A slab's spectra are written and re-read within tens of microseconds, so phases B
// and C hit L2 and each spectrum crosses HBM once each way (6 S instead of 18 S).
//
// Scheduling: units are claimed in global order (slab-major, phases in order) by an atomic
// counter; a unit's dependencies (all A units of its slab for B, all B units for C) are units
// claimed earlier. A CTA computes its units in claim order, prefetches the next unit's tile
// only when that unit's dependencies are already met, and before it blocks on a dependency
// it has signalled every unit it computed, so the smallest waiting unit always has all its
// producers running or done: no deadlock, and no CTA co-residency is assumed. Completion is
// signalled lazily (one unit later, `cp.async.bulk.wait_group N`) after the TMA stores have
// landed: async-proxy writes -> fence.proxy.async -> release atomic; consumers acquire the
// counter and fence before their TMA loads. Waits are bounded: after ~2^24 polls the kernel
// raises an error flag (checked on the host) instead of hanging.
struct ChainArgs {
    PencilJobs ph[3];   // phase A (y forward), B (x), C (y inverse)
    PencilMaps mx, my;  // tensor maps of the scratch buffers: x-pencil boxes, y-pencil boxes
    int* ctr;           // [0] claim counter, [1 + 3 s + p] completed units of slab s, phase p
    int* err;           // set on a dependency-wait timeout
    int nbatch;         // claim order: batch q = (phase, slab) of `lines` consecutive units
    unsigned char bphase[64], bslab[64];
    int eager;                      // signal every unit as soon as its stores landed
    unsigned long long* stats;      // per CTA: [units, deferred loads, wait cycles, mbar cycles]
};

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_n() { asm volatile("cp.async.bulk.wait_group %0;\n" ::"n"(N) : "memory"); }

// Units are tiles of one (phase, slab) batch; a CTA walks "tile steps" (unit, source group)
// through two TMA stages: while one tile is transformed the next one (the next source group of
// the same unit, or the first tile of the next claimed unit when its dependencies are met)
// is in flight. Batches are claimed in the order A0 A1 B0 B1 C0, then (A k, C k-1, B k) for
// k >= 2, then the last C: every batch's producers were claimed at least one batch earlier
// (no phase-boundary drain) while at most two slabs are live in L2.
template <int L, int N1, int TB, int MINB>
__global__ void __launch_bounds__(PencilCfg<L, N1, TB, true>::NT, MINB)
    chain_kernel(const __grid_constant__ GridDev g, const __grid_constant__ ChainArgs A) {
    using C = PencilCfg<L, N1, TB, true>;
    constexpr int N2 = C::N2, KP = C::KP, NT = C::NT;
    constexpr int BOXR = L > 256 ? L / 2 : L;  // TMA box extent <= 256 rows
    constexpr int NBOX = L / BOXR;
    constexpr unsigned TILE_BYTES = unsigned(L) * TB * sizeof(float2);
    extern __shared__ __align__(128) unsigned char sm_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm_raw);   // one per stage
    int* s_unit = reinterpret_cast<int*>(sm_raw + 64);     // [2] unit of each stage
    int* s_grp = s_unit + 2;                                // [2] source group of each stage
    int* s_loaded = s_unit + 4;                             // [2] tile load issued
    float2* xbuf = reinterpret_cast<float2*>(sm_raw + 128);  // [2][L][TB]
    float2* ys = xbuf + 2 * L * TB;
    float2* tw = ys + N1 * KP;
    float* kap_s = reinterpret_cast<float*>(tw + L);
    float* hkx2_s = kap_s + L * TB;
    const bool producer = threadIdx.x == NT - 1;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
    }
    for (int i = threadIdx.x; i < L; i += NT) {
        tw[i] = g.px.tw[i];
        const float hk = g.half_cdt * g.kx[i];
        hkx2_s[i] = hk * hk;
    }
    // source groups of the three phases' job lists
    int gs[3][5], ng[3];
#pragma unroll
    for (int p = 0; p < 3; ++p) {
        ng[p] = 0;
        for (int jb = 0; jb < A.ph[p].n; ++jb)
            if (jb == 0 || A.ph[p].job[jb].src != A.ph[p].job[jb - 1].src) gs[p][ng[p]++] = jb;
        gs[p][ng[p]] = A.ph[p].n;
    }
    const int lines = g.nx;  // == g.ny (chain_supported)
    const int total = lines * A.nbatch;
    const int c = threadIdx.x % TB;
    const int ra = threadIdx.x / TB;
    const bool inA = ra < N2, inB = ra < N1;
    const int kb = C::out_base(ra);

    auto decode = [&](int u, int& slab, int& phase, int& line) {
        const int q = u / lines;
        line = u - q * lines;
        phase = A.bphase[q];
        slab = A.bslab[q];
    };
    auto ready = [&](int u) {
        int slab, phase, line;
        decode(u, slab, phase, line);
        if (phase == 0) return true;
        return ld_acquire(A.ctr + 1 + 3 * slab + phase - 1) >= lines;
    };
    auto box = [&](int phase, int buf, float2* s, int line, int col0, int q, bool load, uint64_t* b) {
        const int r0 = q * BOXR;
        const int e0 = 2 * col0;
        const CUtensorMap* tm = phase == 1 ? &A.mx.tm[buf] : &A.my.tm[buf];
        const int e1 = phase == 1 ? line : r0;
        const int e2 = phase == 1 ? r0 : line;
        if (load) tma_load_3d(s + r0 * TB, tm, e0, e1, e2, b);
        else tma_store_3d(tm, s + r0 * TB, e0, e1, e2);
    };
    auto load_tile = [&](int u, int gi, int b) {  // producer only
        int slab, phase, line;
        decode(u, slab, phase, line);
        float2* xs = xbuf + b * L * TB;
        bulk_wait_read_all();  // the stage may still be the source of a store
        fence_proxy_async_global();
        mbar_arrive_expect_tx(&bar[b], TILE_BYTES);
        const int src = A.ph[phase].job[gs[phase][gi]].src;
#pragma unroll
        for (int q = 0; q < NBOX; ++q) box(phase, src, xs, line, slab * TB, q, true, &bar[b]);
    };
    // producer-side lazy completion: the last computed unit (counter slot) awaiting its stores
    int prev_slot = -1, unit_groups = 0;
    auto signal_prev_all = [&]() {  // producer only: every computed unit complete and counted
        if (prev_slot >= 0) {
            bulk_wait_all();
            fence_proxy_async_global();
            __threadfence();
            atomicAdd(A.ctr + prev_slot, 1);
            prev_slot = -1;
        }
    };
    unsigned long long st_units = 0, st_def = 0, st_wait = 0, st_mbar = 0;
    auto wait_ready = [&](int u) {  // producer only, blocking (bounded)
        const unsigned long long t0 = clock64();
        unsigned spins = 0;
        while (!ready(u)) {
            __nanosleep(64);
            if (++spins > (1u << 24)) {
                atomicExch(A.err, 1);
                break;
            }
        }
        st_wait += clock64() - t0;
    };

    if (producer) {
        const int u0 = atomicAdd(A.ctr, 1);
        s_unit[0] = u0;
        s_grp[0] = 0;
        s_loaded[0] = 0;
        if (u0 < total && ready(u0)) {
            load_tile(u0, 0, 0);
            s_loaded[0] = 1;
        }
    }
    unsigned uses[2] = {0u, 0u};
    int b = 0;
    for (;;) {
        __syncthreads();  // stage b's unit / group visible; the previous step's smem reads done
        const int u = s_unit[b];
        const int gi = s_grp[b];
        if (u >= total) break;
        int slab, phase, line;
        decode(u, slab, phase, line);
        if (producer) {
            if (!s_loaded[b]) {
                ++st_def;
                signal_prev_all();
                wait_ready(u);
                load_tile(u, gi, b);
            }
            int nu = u, ngi = gi + 1;
            bool rdy = true;
            if (ngi >= ng[phase]) {
                nu = atomicAdd(A.ctr, 1);
                ngi = 0;
                rdy = nu < total && ready(nu);
            }
            s_unit[b ^ 1] = nu;
            s_grp[b ^ 1] = ngi;
            s_loaded[b ^ 1] = 0;
            if (nu < total && rdy) {
                load_tile(nu, ngi, b ^ 1);
                s_loaded[b ^ 1] = 1;
            }
            if (gi == 0) unit_groups = 0;
        }
        {
            const unsigned long long t0 = A.stats ? clock64() : 0ull;
            mbar_wait(&bar[b], uses[b] & 1);
            if (A.stats && producer) st_mbar += clock64() - t0;
        }
        ++uses[b];
        const int col0 = slab * TB;
        const PencilJobs& jobs = A.ph[phase];
        float2* xs = xbuf + b * L * TB;

        auto store_tile = [&](int dst) {
            fence_proxy_async_smem();
            __syncthreads();
            if (producer) {
#pragma unroll
                for (int q = 0; q < NBOX; ++q) box(phase, dst, xs, line, col0, q, false, nullptr);
                bulk_commit();
                ++unit_groups;
            }
        };
        auto forward = [&](float2 (&X)[N2]) {
            if (inA) {
                float2 a[N1];
#pragma unroll
                for (int n1 = 0; n1 < N1; ++n1) a[n1] = xs[C::in_row(n1, ra) * TB + c];
                RDft<N1, false>::run(a);
                if constexpr (!C::PFA) {
#pragma unroll
                    for (int k1 = 1; k1 < N1; ++k1) a[k1] = cmul(a[k1], tw[ra * k1]);
                }
#pragma unroll
                for (int k1 = 0; k1 < N1; ++k1) ys[k1 * KP + ra * TB + c] = a[k1];
            }
            __syncthreads();
            if (inB) {
#pragma unroll
                for (int n2 = 0; n2 < N2; ++n2) X[n2] = ys[ra * KP + n2 * TB + c];
                RDft<N2, false>::run(X);
            }
        };
        auto inverse_store = [&](float2 (&bb)[N2], int dst) {
            if (inB) {
                RDft<N2, true>::run(bb);
                if constexpr (!C::PFA) {
#pragma unroll
                    for (int n2 = 1; n2 < N2; ++n2) bb[n2] = cmul(bb[n2], conjf2(tw[ra * n2]));
                }
            }
            if (producer) bulk_wait_read_all();  // previous store out of xs
            __syncthreads();
            if (inB) {
#pragma unroll
                for (int n2 = 0; n2 < N2; ++n2) ys[ra * KP + n2 * TB + c] = bb[n2];
            }
            __syncthreads();
            if (inA) {
                float2 a[N1];
#pragma unroll
                for (int k1 = 0; k1 < N1; ++k1) a[k1] = ys[k1 * KP + ra * TB + c];
                RDft<N1, true>::run(a);
#pragma unroll
                for (int n1 = 0; n1 < N1; ++n1) xs[C::in_row(n1, ra) * TB + c] = a[n1];
            }
            store_tile(dst);
        };

        const int gb = gs[phase][gi], ge = gs[phase][gi + 1];
        float2 X[N2];
        if (phase == 0) {
            forward(X);
            if (inB) {
#pragma unroll
                for (int k2 = 0; k2 < N2; ++k2) xs[C::out_row(kb, k2) * TB + c] = X[k2];
            }
            store_tile(jobs.job[gb].dst);
        } else {
            if (phase == 1) {
                forward(X);
                if (inB && jobs.job[gb].kappa) {
                    if (gi == 0) {  // kappa of the tile, reused by the unit's later source groups
                        const float ky = g.ky[line];
                        const float kz = col0 + c < g.nzh ? g.kz[col0 + c] : 0.f;
                        const float hy = g.half_cdt * ky, hz = g.half_cdt * kz;
                        const float uyz = hy * hy + hz * hz;
#pragma unroll
                        for (int k2 = 0; k2 < N2; ++k2) {
                            const int k = C::out_row(kb, k2);
                            kap_s[k * TB + c] = kappa_of_u(hkx2_s[k] + uyz);
                        }
                    }
#pragma unroll
                    for (int k2 = 0; k2 < N2; ++k2) X[k2] = cscale(X[k2], kap_s[C::out_row(kb, k2) * TB + c]);
                }
            } else if (inB) {
#pragma unroll
                for (int k2 = 0; k2 < N2; ++k2) X[k2] = xs[C::out_row(kb, k2) * TB + c];
            }
            for (int jb = gb; jb < ge; ++jb) {
                const PencilJob J = jobs.job[jb];
                float2 bb[N2];
                if (inB) {
#pragma unroll
                    for (int k2 = 0; k2 < N2; ++k2)
                        bb[k2] = J.dmul ? cmul(X[k2], __ldg(J.dmul + C::out_row(kb, k2))) : X[k2];
                }
                inverse_store(bb, J.dst);
            }
        }
        if (producer && gi + 1 == ng[phase]) {
            ++st_units;
            if (A.eager) {
                prev_slot = 1 + 3 * slab + phase;
                signal_prev_all();
            }
            // unit done: lazily count the previous unit, whose stores are older than this
            // unit's store groups
            else if (prev_slot >= 0) {
                if (unit_groups >= 3) bulk_wait_n<3>();
                else if (unit_groups == 2) bulk_wait_n<2>();
                else bulk_wait_n<1>();
                fence_proxy_async_global();
                __threadfence();
                atomicAdd(A.ctr + prev_slot, 1);
            }
            if (!A.eager) prev_slot = 1 + 3 * slab + phase;
        }
        b ^= 1;
    }
    if (producer) {
        signal_prev_all();
        if (A.stats) {
            unsigned long long* o = A.stats + 4 * blockIdx.x;
            o[0] += st_units;
            o[1] += st_def;
            o[2] += st_wait;
            o[3] += st_mbar;
        }
    }
}

// USTFWI_CHAIN_STATS=1: per-CTA wait statistics of the chain kernel (diagnostics)
unsigned long long* g_chain_stats = nullptr;
int g_chain_stats_n = 0;
unsigned long long* chain_stats_buffer(int nctas) {
    static const bool on = [] {
        const char* e = std::getenv("USTFWI_CHAIN_STATS");
        return e && e[0] == '1';
    }();
    if (!on) return nullptr;
    if (!g_chain_stats) {
        if (cudaMalloc(&g_chain_stats, sizeof(unsigned long long) * 4 * nctas) != cudaSuccess) return nullptr;
        cudaMemset(g_chain_stats, 0, sizeof(unsigned long long) * 4 * nctas);
        g_chain_stats_n = nctas;
    }
    return g_chain_stats;
}

template <int L, int N1, int TB, int MINB>
cudaError_t run_chain(const GridDev& g, const PencilJobs& ya, const PencilJobs& xb, const PencilJobs& yc, int* ctr,
                      int* err, cudaStream_t st) {
    using C = PencilCfg<L, N1, TB, true>;
    constexpr int BOXR = L > 256 ? L / 2 : L;
    ChainArgs a;
    std::memset(&a, 0, sizeof(a));
    a.ph[0] = ya;
    a.ph[1] = xb;
    a.ph[2] = yc;
    for (int f = 0; f < 3; ++f)
        if (ya.buf[f]) {
            if (!pencil_map(&a.mx.tm[f], ya.buf[f], g, 0, TB, BOXR)) return cudaErrorInvalidValue;
            if (!pencil_map(&a.my.tm[f], ya.buf[f], g, 1, TB, BOXR)) return cudaErrorInvalidValue;
        }
    a.ctr = ctr;
    a.err = err;
    static const int eager = [] {
        const char* e = std::getenv("USTFWI_CHAIN_EAGER");
        return e ? std::atoi(e) : 0;
    }();
    a.eager = eager;
    a.stats = chain_stats_buffer(sm_count() * MINB);
    const int ntx = (g.nzh + TB - 1) / TB;
    // claim order of the (phase, slab) batches: A0 A1 B0 B1 C0, then (A k, C k-1, B k), then the
    // last C (see chain_kernel)
    {
        std::vector<std::pair<int, int>> order;
        auto add = [&](int ph, int sl) {
            if (sl >= 0 && sl < ntx) order.push_back({ph, sl});
        };
        static const int mode = [] {
            const char* e = std::getenv("USTFWI_CHAIN_ORDER");
            return e ? std::atoi(e) : 0;
        }();
        if (mode == 1) {  // plain slab-major
            for (int k = 0; k < ntx; ++k) {
                add(0, k);
                add(1, k);
                add(2, k);
            }
        } else if (mode == 2) {  // wider gaps: A0 A1 A2 B0 B1 C0, then (A k, C k-2, B k-1), tail
            add(0, 0);
            add(0, 1);
            add(0, 2);
            add(1, 0);
            add(1, 1);
            add(2, 0);
            for (int k = 3; k < ntx; ++k) {
                add(0, k);
                add(2, k - 2);
                add(1, k - 1);
            }
            add(2, ntx - 2);
            add(1, ntx - 1);
            add(2, ntx - 1);
        } else {
            add(0, 0);
            add(0, 1);
            add(1, 0);
            add(1, 1);
            add(2, 0);
            for (int k = 2; k < ntx; ++k) {
                add(0, k);
                add(2, k - 1);
                add(1, k);
            }
            add(2, ntx - 1);
        }
        if (ntx < 4) {
            order.clear();
            for (int k = 0; k < ntx; ++k) {
                add(0, k);
                add(1, k);
                add(2, k);
            }
        }
        if (order.size() != static_cast<size_t>(3 * ntx) || order.size() > sizeof(a.bphase)) return cudaErrorInvalidValue;
        a.nbatch = static_cast<int>(order.size());
        for (size_t q = 0; q < order.size(); ++q) {
            a.bphase[q] = static_cast<unsigned char>(order[q].first);
            a.bslab[q] = static_cast<unsigned char>(order[q].second);
        }
    }
    cudaError_t e = cudaMemsetAsync(ctr, 0, sizeof(int) * (1 + 3 * ntx), st);
    if (e != cudaSuccess) return e;
    auto kern = chain_kernel<L, N1, TB, MINB>;
    constexpr size_t smem = 128 + (2 * size_t(L) * TB + size_t(N1) * C::KP + L) * sizeof(float2) +
                            size_t(L) * (TB + 1) * sizeof(float);
    static std::atomic<unsigned long long> configured{0};
    once_per_device(configured, [&] { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); });
    static int occ = -1;
    if (occ < 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::NT, smem);
        if (a.stats) fprintf(stderr, "chain_kernel: %d CTAs per SM (smem %zu B, %d threads)\n", occ, smem, C::NT);
    }
    kern<<<sm_count() * (occ > 0 ? std::min(occ, MINB) : MINB), C::NT, smem, st>>>(g, a);
    return cudaGetLastError();
}
#endif  // !USTFWI_PASSES_Y_ONLY

}  // namespace

#ifdef USTFWI_PASSES_Y_ONLY
cudaError_t launch_pencil_fast_y(bool inv, const GridDev& g, const PencilJobs& j, cudaStream_t st) {
    constexpr int axis = 1;
    switch (g.py.L) {
        case 32: return pencil_sized<32, 2, 16, 4, false>(axis, inv, g, j, st);
        case 64: return pencil_sized<64, 4, 16, 4, false>(axis, inv, g, j, st);
        case 96: return pencil_sized<96, 6, 16, 3, false>(axis, inv, g, j, st);
        case 128: return pencil_sized<128, 8, 16, 3, false>(axis, inv, g, j, st);
        case 144: return pencil_sized<144, 16, 16, 3, false>(axis, inv, g, j, st);
        case 256: return pencil_sized<256, 16, 16, 3, false>(axis, inv, g, j, st);
        case 480: return pencil_sized<480, 30, 8, 2, true>(axis, inv, g, j, st);  // TB 4 / 16: 0.298 / 0.232 ms
        default: return cudaErrorInvalidValue;
    }
}
#else
cudaError_t launch_pencil_fast_y(bool inv, const GridDev& g, const PencilJobs& j, cudaStream_t st);

bool fast_pencil_supported(int L) {
    switch (L) {
        case 32: case 64: case 96: case 128: case 144: case 256: case 480: return true;
        default: return false;
    }
}

cudaError_t launch_pencil_fast(int axis, bool inv, const GridDev& g, const PencilJobs& j, cudaStream_t st) {
    if (axis == 1) return launch_pencil_fast_y(inv, g, j, st);
    switch (g.px.L) {
        case 32: return pencil_sized<32, 2, 16, 4, false>(axis, inv, g, j, st);
        case 64: return pencil_sized<64, 4, 16, 4, false>(axis, inv, g, j, st);
        case 96: return pencil_sized<96, 6, 16, 3, false>(axis, inv, g, j, st);
        case 128: return pencil_sized<128, 8, 16, 3, false>(axis, inv, g, j, st);
        case 144: return pencil_sized<144, 16, 16, 3, false>(axis, inv, g, j, st);
        case 256: return pencil_sized<256, 16, 16, 3, false>(axis, inv, g, j, st);
        case 480:
            // measured on B200 (config D): Cooley-Tukey 30x16 for both passes (double-buffered
            // TMA tiles)
            if (axis == 0) {
                // USTFWI_X480=1: prime-factor 32x15 (spills at the 128-register cap with TMA
                // tiles; 0.352 vs 0.312 ms per launch at config D)
                static const int xv = [] {
                    const char* e = std::getenv("USTFWI_X480");
                    return e ? std::atoi(e) : 0;
                }();
                if (xv == 1) return pencil_sized<480, 32, 8, 2, true>(axis, inv, g, j, st);
                return pencil_sized<480, 30, 8, 2, true>(axis, inv, g, j, st);
            }
            return cudaErrorInvalidValue;
        default: return cudaErrorInvalidValue;
    }
}

// the fused y-x-y chain is compiled for the 480-point lines of config D / E level 2 (x and y
// share the plan) and 2 CTAs per SM
bool chain_supported(const GridDev& g) {
    return g.nx == 480 && g.ny == 480 && g.x0 == 0 && g.xn == g.nx && use_pencil_tma();
}

cudaError_t launch_chain(const GridDev& g, const PencilJobs& ya, const PencilJobs& xb, const PencilJobs& yc, int* ctr,
                         int* err, cudaStream_t st) {
    if (!chain_supported(g)) return cudaErrorInvalidValue;
    return run_chain<480, 30, 8, 2>(g, ya, xb, yc, ctr, err, st);
}

// totals of the chain-kernel wait statistics since the last call (USTFWI_CHAIN_STATS=1)
int chain_stats(unsigned long long out[4]) {
    for (int k = 0; k < 4; ++k) out[k] = 0;
    if (!g_chain_stats) return 0;
    std::vector<unsigned long long> h(4 * static_cast<size_t>(g_chain_stats_n));
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), g_chain_stats, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaMemset(g_chain_stats, 0, h.size() * sizeof(unsigned long long));
    for (size_t i = 0; i < h.size(); ++i) out[i % 4] += h[i];
    return g_chain_stats_n;
}

bool fast_rows_supported(int nz) {
    switch (nz) {
        case 64: case 96: case 128: case 144: case 256: return true;
        default: return false;
    }
}

namespace {
constexpr int kZRows = 8;

bool use_zrow2() {
    static int on = -1;
    if (on < 0) {
        const char* e = std::getenv("USTFWI_ZROW2");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

// smallest half length M = nz / 2 that takes the paired-residue rows: velocity (kind 0) and
// density / pressure (kind 1) passes; USTFWI_ZROW2_MIN="<vel>,<rho>" overrides (measurement)
int zrow2_min(int kind) {
    static int v[2] = {-1, -1};
    if (v[0] < 0) {
        v[0] = 64;
        v[1] = 128;
        if (const char* e = std::getenv("USTFWI_ZROW2_MIN")) std::sscanf(e, "%d,%d", &v[0], &v[1]);
    }
    return v[kind];
}

template <int M, int N1, int RW>
cudaError_t zvel2_run(const GridDev& g, const ZvelFastArgs& a, cudaStream_t st) {
    const size_t smem = Z2Smem<M, N1, RW>::bytes(g.nzp, a.r[0].field ? 2 : 1);
    auto kern = zvel2_kernel<M, N1, RW>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const dim3 blocks((unsigned)(((long long)g.xn * g.ny + RW - 1) / RW), 3);
    kern<<<blocks, RW * Z2<M, N1>::TPR, smem, st>>>(a);
    return cudaGetLastError();
}
// USTFWI_ZFUSE=1: the density update of the three axes and the pressure step in one kernel
// (zrhop_kernel) instead of zrho2_axis + zp2 (non-absorbing steps)
bool use_zfuse() {
    static int on = -1;
    if (on < 0) {
        const char* e = std::getenv("USTFWI_ZFUSE");
        on = (e && e[0] == '1') ? 1 : 0;
    }
    return on == 1;
}

template <int M, int N1, int RW>
cudaError_t zrho2_run(const GridDev& g, const ZrhoFastArgs& a, cudaStream_t st) {
    if (use_zfuse() && !a.a.du_out[0] && !a.a.du_out[1] && !a.a.du_out[2]) {
        using C = Z2<M, N1>;
        const size_t smem = 32 + size_t(2 * M) * 8 + size_t(RW) * cmax(g.nzp, C::ZT) * 8 +
                            size_t(a.a.dtrho0.field ? 3 : 2) * RW * C::VP * 4;
        auto kf = zrhop_kernel<M, N1, RW>;
        cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const unsigned blocks = (unsigned)(((long long)g.xn * g.ny + RW - 1) / RW);
        kf<<<blocks, RW * C::TPR, smem, st>>>(a);
        return cudaGetLastError();
    }
    const size_t smem = Z2Smem<M, N1, RW>::bytes_rho(g.nzp, a.a.dtrho0.field ? 2 : 1);
    auto kern = zrho2_axis_kernel<M, N1, RW>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const dim3 blocks((unsigned)(((long long)g.xn * g.ny + RW - 1) / RW), 3);
    kern<<<blocks, RW * Z2<M, N1>::TPR, smem, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // no pressure store (forward, adjoint): no store in the element loop, so the compiler may
    // issue later elements' loads early
    auto kp = a.a.corr.grad ? (a.a.p_out ? zp2_kernel<M, N1, RW, true, true> : zp2_kernel<M, N1, RW, true, false>)
                            : (a.a.p_out ? zp2_kernel<M, N1, RW, false, true> : zp2_kernel<M, N1, RW, false, false>);
    const size_t smem_p = (size_t(M) + size_t(RW) * Z2<M, N1>::ZT) * sizeof(float2);
    cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_p);
    kp<<<blocks.x, RW * Z2<M, N1>::TPR, smem_p, st>>>(a);
    return cudaGetLastError();
}
template <int M>
cudaError_t zvel2_sized(const GridDev& g, const ZvelFastArgs& a, cudaStream_t st) {
    if constexpr (M == 128) return zvel2_run<128, 16, 16>(g, a, st);
    else if constexpr (M == 64) return zvel2_run<64, 8, 16>(g, a, st);
    else if constexpr (M == 72) return zvel2_run<72, 6, 32>(g, a, st);
    else if constexpr (M == 48) return zvel2_run<48, 4, 32>(g, a, st);
    else return zvel2_run<32, 4, 32>(g, a, st);
}
template <int M>
cudaError_t zrho2_sized(const GridDev& g, const ZrhoFastArgs& a, cudaStream_t st) {
    if constexpr (M == 128) return zrho2_run<128, 16, 16>(g, a, st);
    else if constexpr (M == 64) return zrho2_run<64, 8, 16>(g, a, st);
    else if constexpr (M == 72) return zrho2_run<72, 6, 32>(g, a, st);
    else if constexpr (M == 48) return zrho2_run<48, 4, 32>(g, a, st);
    else return zrho2_run<32, 4, 32>(g, a, st);
}

template <int M, int N1>
cudaError_t zvel_sized(const GridDev& g, float2* S[3], const float2* dz_plus, float* v[3], const Pml& pml,
                       const Coef r[3], cudaStream_t st) {
    using C = RowCfg<M, N1, kZRows>;
    ZvelFastArgs a;
    a.g = g;
    for (int f = 0; f < 3; ++f) {
        a.S[f] = S[f];
        a.v[f] = v[f];
        a.r[f] = r[f];
    }
    a.dz_plus = dz_plus;
    a.pml = pml;
    // paired-residue rows where they win on B200: z-vel for M >= 64 (config B 0.036 -> 0.027 ms,
    // D 0.80 -> 0.54 ms), the density/pressure pair for M >= 128 only (config A/B: the
    // 8-row kernels are faster, 0.037 vs 0.062 ms at A)
    if (M >= zrow2_min(0) && use_zrow2()) return zvel2_sized<M>(g, a, st);
    const size_t smem = C::FIXED + size_t(kZRows) * g.nzp * 8 + size_t(r[0].field ? 2 : 1) * kZRows * C::NZ * 4;
    auto kern = zvel_fast_kernel<M, N1, kZRows>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const dim3 blocks((unsigned)(((long long)g.xn * g.ny + kZRows - 1) / kZRows), 3);
    kern<<<blocks, C::NT, smem, st>>>(a);
    return cudaGetLastError();
}
template <int M, int N1>
cudaError_t zrho_sized(const GridDev& g, const ZrhoArgs& za, cudaStream_t st) {
    using C = RowCfg<M, N1, kZRows>;
    ZrhoFastArgs a;
    a.g = g;
    a.a = za;
    const unsigned blocks = (unsigned)(((long long)g.xn * g.ny + kZRows - 1) / kZRows);
    // density update, one CTA per (row block, axis)
    if (M >= zrow2_min(1) && use_zrow2()) return zrho2_sized<M>(g, a, st);
    {
    const size_t smem1 = 16 + size_t(M) * 8 + size_t(kZRows) * C::ZT * 8 + size_t(kZRows) * g.nzp * 8 +
                         size_t(za.dtrho0.field ? 2 : 1) * kZRows * C::NZ * 4;
    auto k1 = zrho_axis_kernel<M, N1, kZRows>;
    cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
    k1<<<dim3(blocks, 3), C::NT, smem1, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    }
    // pressure, sparse work, gathers, correlation, r2c of p
    const size_t smem2 = C::FIXED;
    auto k2 = zp_kernel<M, N1, kZRows>;
    k2<<<blocks, C::NT, smem2, st>>>(a);
    return cudaGetLastError();
}
}  // namespace

cudaError_t launch_zvel_fast(const GridDev& g, float2* S[3], const float2* dz_plus, float* v[3], const Pml& pml,
                             const Coef r[3], cudaStream_t st) {
    switch (g.nz) {
        case 64: return zvel_sized<32, 8>(g, S, dz_plus, v, pml, r, st);
        case 96: return zvel_sized<48, 8>(g, S, dz_plus, v, pml, r, st);
        case 128: return zvel_sized<64, 8>(g, S, dz_plus, v, pml, r, st);
        case 144: return zvel_sized<72, 8>(g, S, dz_plus, v, pml, r, st);
        case 256: return zvel_sized<128, 8>(g, S, dz_plus, v, pml, r, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_zrho_fast(const GridDev& g, const ZrhoArgs& a, cudaStream_t st) {
    switch (g.nz) {
        case 64: return zrho_sized<32, 8>(g, a, st);
        case 96: return zrho_sized<48, 8>(g, a, st);
        case 128: return zrho_sized<64, 8>(g, a, st);
        case 144: return zrho_sized<72, 8>(g, a, st);
        case 256: return zrho_sized<128, 8>(g, a, st);
        default: return cudaErrorInvalidValue;
    }
}

#endif  // !USTFWI_PASSES_Y_ONLY

}  // namespace ustfwi_dev
