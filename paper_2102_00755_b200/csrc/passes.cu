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
#include <cuda_runtime.h>

#include "async_copy.cuh"
#include "fft_reg.cuh"
#include "kernels.cuh"

namespace ustfwi_dev {

__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }

constexpr int cmax(int a, int b) { return a > b ? a : b; }

__device__ __forceinline__ float kappa_fast(float k2, float half_cdt) {
    const float x = half_cdt * sqrtf(k2);
    return (x < 1e-4f) ? 1.f - x * x * (1.f / 6.f) : sinf(x) / x;
}

// ======================================================================================
// Pencil passes (x and y)
// ======================================================================================
template <int L, int N1, int TB>
struct PencilCfg {
    static constexpr int N2 = L / N1;
    static constexpr int NT = TB * cmax(N1, N2);
    static constexpr int KP = N2 * TB + 8;  // float2 pitch of one k1 slab (+64 B against bank conflicts)
    static constexpr size_t SMEM = (size_t(L) * TB + size_t(N1) * KP + L) * sizeof(float2);
};

// AXIS 0: x pencils at fixed y = blockIdx.y (forward * multiplier * inverse per job).
// AXIS 1: y pencils at fixed x = blockIdx.y, direction INV, optional premultiplier.
template <int AXIS, bool INV, int L, int N1, int TB, int MINB>
__global__ void __launch_bounds__(PencilCfg<L, N1, TB>::NT, MINB)
    pencil_fast_kernel(const __grid_constant__ GridDev g, const __grid_constant__ PencilJobs jobs) {
    using C = PencilCfg<L, N1, TB>;
    constexpr int N2 = C::N2, KP = C::KP, NT = C::NT;
    extern __shared__ float2 smem[];
    float2* xs = smem;             // [L][TB] tile, natural order
    float2* ys = xs + L * TB;      // transposed [N1][N2*TB (+pad)]
    float2* tw = ys + N1 * KP;     // W_L^k
    const FftPlan& plan = AXIS == 0 ? g.px : g.py;
    for (int i = threadIdx.x; i < L; i += NT) tw[i] = plan.tw[i];

    const int c0 = blockIdx.x * TB;
    const int ncol = min(TB, g.nzh - c0);
    const int pitch = (AXIS == 0) ? g.ny * g.nzp : g.nzp;
    const long long base = (AXIS == 0) ? (long long)blockIdx.y * g.nzp + c0 : (long long)blockIdx.y * g.ny * g.nzp + c0;
    const int c = threadIdx.x % TB;
    const int ra = threadIdx.x / TB;  // n2 in phase A, k1 in phase B
    const bool inA = ra < N2, inB = ra < N1;
    const bool colok = c < ncol;

    // async tile load: 16-B granules (2 complex); columns past nzh are padding of the row
    auto load_tile = [&](const float2* src) {
        constexpr int CH = TB / 2;
        const float2* s = src + base;
        for (int i = threadIdx.x; i < L * CH; i += NT) {
            const int row = i / CH, cc = 2 * (i % CH);
            if (cc < ncol) cp_async16(xs + row * TB + cc, s + row * pitch + cc);
        }
        cp_async_commit();
        cp_async_wait_all();
        __syncthreads();
    };
    // forward transform of the tile in xs -> X[k1 + N1*k2] in phase-B registers
    auto forward = [&](float2 (&X)[N2]) {
        if (inA) {
            float2 a[N1];
#pragma unroll
            for (int n1 = 0; n1 < N1; ++n1) a[n1] = xs[(ra + N2 * n1) * TB + c];
            RDft<N1, false>::run(a);
#pragma unroll
            for (int k1 = 1; k1 < N1; ++k1) a[k1] = cmul(a[k1], tw[ra * k1]);
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
#pragma unroll
            for (int n2 = 1; n2 < N2; ++n2) b[n2] = cmul(b[n2], conjf2(tw[ra * n2]));
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
                for (int n1 = 0; n1 < N1; ++n1) d[(ra + N2 * n1) * pitch] = a[n1];
            }
        }
    };

    int loaded = -1;
    for (int jb = 0; jb < jobs.n; ++jb) {
        const PencilJob J = jobs.job[jb];
        if (J.src != loaded) {
            load_tile(jobs.buf[J.src]);
            loaded = J.src;
            if (AXIS == 0) {
                // forward, then keep kappa * X (natural order) in xs for the jobs of this source
                float2 X[N2];
                forward(X);
                // (all jobs of one source share its kappa flag: true for every job list the
                // engine builds; kappa-free jobs are the staggered-density setup shift)
                if (inB) {
                    const float ky = g.ky[blockIdx.y];
                    const float kz = colok ? g.kz[c0 + c] : 0.f;
#pragma unroll
                    for (int k2 = 0; k2 < N2; ++k2) {
                        const int k = ra + N1 * k2;
                        const float kx = g.kx[k];
                        xs[k * TB + c] =
                            J.kappa ? cscale(X[k2], kappa_fast(kx * kx + ky * ky + kz * kz, g.half_cdt)) : X[k2];
                    }
                }
                // each phase-B thread reads back only the entries it wrote: no barrier needed
            }
        }
        if (AXIS == 1 && !INV) {
            float2 X[N2];
            forward(X);
            if (inB && colok) {
                float2* d = jobs.buf[J.dst] + base + c;
#pragma unroll
                for (int k2 = 0; k2 < N2; ++k2) d[(ra + N1 * k2) * pitch] = X[k2];
            }
            __syncthreads();  // phase-B reads of ys done before the next tile's phase A
            loaded = -1;
            continue;
        }
        float2 b[N2];
        if (inB) {
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2) {
                const int k = ra + N1 * k2;
                float2 v = xs[k * TB + c];
                if (J.dmul) v = cmul(v, __ldg(J.dmul + k));
                b[k2] = v;
            }
        }
        inverse_store(b, jobs.buf[J.dst]);
    }
}

// ======================================================================================
// Row (z) passes: real FFT of length nz = 2M through the M-point complex transform
// ======================================================================================
template <int M, int N1, int RW>
struct RowCfg {
    static constexpr int N2 = M / N1;
    static constexpr int TPR = cmax(N1, N2);  // threads per row
    static constexpr int NT = RW * TPR;
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

template <int M, int N1, int RW>
__global__ void __launch_bounds__(RowCfg<M, N1, RW>::NT) zvel_fast_kernel(const __grid_constant__ ZvelFastArgs A) {
    using C = RowCfg<M, N1, RW>;
    constexpr int N2 = C::N2, TPR = C::TPR, NZ = C::NZ, NT = C::NT;
    extern __shared__ __align__(128) unsigned char sm_raw[];
    const GridDev& g = A.g;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm_raw);
    float2* twM = reinterpret_cast<float2*>(sm_raw + 16);
    float2* zt = twM + M;
    float2* zn = zt + RW * C::ZT;
    float2* sS = zn + RW * M;                       // [3][RW*nzp]
    float* sV = reinterpret_cast<float*>(sS + 3 * RW * g.nzp);  // [3][RW*NZ]
    float* sR = sV + 3 * RW * NZ;                   // [3][RW*NZ] (non-uniform dt/rho0~ only)
    const bool coef_fields = A.r[0].field != nullptr;

    const long long row0 = (long long)blockIdx.x * RW;
    const int nrows = (int)min((long long)RW, g.rows - row0);
    if (threadIdx.x == 0) mbar_init(bar, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned total = 3u * nrows * g.nzp * 8u + 3u * nrows * NZ * 4u + (coef_fields ? 3u * nrows * NZ * 4u : 0u);
        mbar_arrive_expect_tx(bar, total);
        Stager st{bar};
        for (int f = 0; f < 3; ++f) st.add(sS + f * RW * g.nzp, A.S[f] + row0 * g.nzp, nrows * g.nzp);
        for (int f = 0; f < 3; ++f) st.add(sV + f * RW * NZ, A.v[f] + row0 * NZ, nrows * NZ);
        if (coef_fields)
            for (int f = 0; f < 3; ++f) st.add(sR + f * RW * NZ, A.r[f].field + row0 * NZ, nrows * NZ);
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

#pragma unroll 1
    for (int a = 0; a < 3; ++a) {
        if (rowok && lane < N1)
            row_c2r_b<M, N1>(sS + a * RW * g.nzp + r * g.nzp, a == 2 ? A.dz_plus : nullptr, g.tw_rfft, twM, lane, zt_row);
        __syncthreads();
        float2 u[N1];
        if (rowok && lane < N2) {
            row_c2r_a<M, N1>(zt_row, lane, g.inv_n, u);
            const float pa = a == 0 ? __ldg(A.pml.prof[0] + x) : (a == 1 ? __ldg(A.pml.prof[1] + y) : 0.f);
            const float* vs = sV + a * RW * NZ + r * NZ;
            const float* rs = sR + a * RW * NZ + r * NZ;
            float* vg = A.v[a] + row * NZ;
#pragma unroll
            for (int n1 = 0; n1 < N1; ++n1) {
                const int n = lane + N2 * n1;
                float2 vv = *reinterpret_cast<const float2*>(vs + 2 * n);
                float2 pm = make_float2(pa, pa);
                if (a == 2) pm = make_float2(__ldg(A.pml.prof[2] + 2 * n), __ldg(A.pml.prof[2] + 2 * n + 1));
                float2 rr = make_float2(A.r[a].scalar, A.r[a].scalar);
                if (coef_fields) rr = *reinterpret_cast<const float2*>(rs + 2 * n);
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
        if (rowok) row_r2c_finish<M, TPR>(zn_row, lane, g.tw_rfft, A.S[a] + row * g.nzp);
    }
}

struct ZrhoFastArgs {
    GridDev g;
    ZrhoArgs a;
};

template <int M, int N1, int RW>
__global__ void __launch_bounds__(RowCfg<M, N1, RW>::NT) zrho_fast_kernel(const __grid_constant__ ZrhoFastArgs P) {
    using C = RowCfg<M, N1, RW>;
    constexpr int N2 = C::N2, TPR = C::TPR, NZ = C::NZ, NT = C::NT;
    extern __shared__ __align__(128) unsigned char sm_raw[];
    const GridDev& g = P.g;
    const ZrhoArgs& A = P.a;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm_raw);
    float2* twM = reinterpret_cast<float2*>(sm_raw + 16);
    float2* zt = twM + M;
    float2* zn = zt + RW * C::ZT;
    float2* sS = zn + RW * M;                                   // [3][RW*nzp]
    float* sR = reinterpret_cast<float*>(sS + 3 * RW * g.nzp);  // [3][RW*NZ] rho
    float* sC = sR + 3 * RW * NZ;                               // c0^2
    const bool coef_field = A.dtrho0.field != nullptr;
    const bool corr = A.corr.grad != nullptr;
    float* sD = sC + RW * NZ;                                   // dt*rho0 field (optional)
    float* sK = sC + (coef_field ? 2 : 1) * RW * NZ;            // correlation: p_mid, p_old, q_adj, grad
    __shared__ int sp[8];

    const long long row0 = (long long)blockIdx.x * RW;
    const int nrows = (int)min((long long)RW, g.rows - row0);
    const long long i0 = row0 * NZ;
    if (threadIdx.x == 0) mbar_init(bar, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned fb = nrows * NZ * 4u;
        unsigned total = 3u * nrows * g.nzp * 8u + 4u * fb + (coef_field ? fb : 0u) + (corr ? 4u * fb : 0u);
        mbar_arrive_expect_tx(bar, total);
        Stager st{bar};
        for (int f = 0; f < 3; ++f) st.add(sS + f * RW * g.nzp, A.S[f] + row0 * g.nzp, nrows * g.nzp);
        for (int f = 0; f < 3; ++f) st.add(sR + f * RW * NZ, A.rho[f] + i0, nrows * NZ);
        st.add(sC, A.c0sq + i0, nrows * NZ);
        if (coef_field) st.add(sD, A.dtrho0.field + i0, nrows * NZ);
        if (corr) {
            st.add(sK, A.corr.p_mid + i0, nrows * NZ);
            st.add(sK + RW * NZ, A.corr.p_old + i0, nrows * NZ);
            st.add(sK + 2 * RW * NZ, A.corr.q_adj + i0, nrows * NZ);
            st.add(sK + 3 * RW * NZ, A.corr.grad + i0, nrows * NZ);
        }
    }
    if (threadIdx.x == 32 % NT) {
        const int lo_key = (int)i0, hi_key = (int)(i0 + (long long)nrows * NZ);
        auto lb = [](const int* a, int n, int key) {
            int lo = 0, hi = n;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (a[mid] < key) lo = mid + 1;
                else hi = mid;
            }
            return lo;
        };
        sp[0] = A.inj.n_unique ? lb(A.inj.pos, A.inj.n_unique, lo_key) : 0;
        sp[1] = A.inj.n_unique ? lb(A.inj.pos, A.inj.n_unique, hi_key) : 0;
        sp[2] = A.enf.n ? lb(A.enf.pos, A.enf.n, lo_key) : 0;
        sp[3] = A.enf.n ? lb(A.enf.pos, A.enf.n, hi_key) : 0;
        sp[4] = A.sens.n ? lb(A.sens.pos, A.sens.n, lo_key) : 0;
        sp[5] = A.sens.n ? lb(A.sens.pos, A.sens.n, hi_key) : 0;
        sp[6] = A.shell.n ? lb(A.shell.pos, A.shell.n, lo_key) : 0;
        sp[7] = A.shell.n ? lb(A.shell.pos, A.shell.n, hi_key) : 0;
    }
    for (int i = threadIdx.x; i < M; i += NT) twM[i] = g.pzh.tw[i];
    const int r = threadIdx.x / TPR, lane = threadIdx.x % TPR;
    const bool rowok = r < nrows;
    const long long row = row0 + r;
    const bool act = rowok && lane < N2;
    const int x = rowok ? (int)(row / g.ny) : 0, y = rowok ? (int)(row % g.ny) : 0;
    float2* zt_row = zt + r * C::ZT;
    float2* zn_row = zn + r * M;
    __syncthreads();
    mbar_wait(bar, 0);

    // density updates, written back in place into sR
#pragma unroll 1
    for (int a = 0; a < 3; ++a) {
        if (rowok && lane < N1)
            row_c2r_b<M, N1>(sS + a * RW * g.nzp + r * g.nzp, a == 2 ? A.dz_minus : nullptr, g.tw_rfft, twM, lane, zt_row);
        __syncthreads();
        if (act) {
            float2 u[N1];
            row_c2r_a<M, N1>(zt_row, lane, g.inv_n, u);
            const float pa = a == 0 ? __ldg(A.pml.prof[0] + x) : (a == 1 ? __ldg(A.pml.prof[1] + y) : 0.f);
            float* rs = sR + a * RW * NZ + r * NZ;
            const float* ds = sD + r * NZ;
#pragma unroll
            for (int n1 = 0; n1 < N1; ++n1) {
                const int n = lane + N2 * n1;
                float2 q = *reinterpret_cast<float2*>(rs + 2 * n);
                float2 pm = make_float2(pa, pa);
                if (a == 2) pm = make_float2(__ldg(A.pml.prof[2] + 2 * n), __ldg(A.pml.prof[2] + 2 * n + 1));
                float2 d = make_float2(A.dtrho0.scalar, A.dtrho0.scalar);
                if (coef_field) d = *reinterpret_cast<const float2*>(ds + 2 * n);
                q.x = pm.x * (pm.x * q.x - d.x * u[n1].x);
                q.y = pm.y * (pm.y * q.y - d.y * u[n1].y);
                *reinterpret_cast<float2*>(rs + 2 * n) = q;
            }
        }
        __syncthreads();
    }

    // sparse mass sources / Dirichlet shell on the split densities (after the update, before p)
    const int lo_key = (int)i0;
    for (int u = sp[0] + threadIdx.x; u < sp[1]; u += NT) {
        const int t = A.inj.pos[u] - lo_key;
        const float sc = A.inj.scale[u];
        for (int cc = A.inj.csr[u]; cc < A.inj.csr[u + 1]; ++cc) {
            const int n = A.step_n - A.inj.delay[cc];
            if (n < 0 || n >= A.inj.len[cc]) continue;
            const float amp = A.inj.w[cc] * A.inj.sig[A.inj.off[cc] + (long long)n * A.inj.stride[cc]];
            if (amp == 0.f) continue;
            for (int a = A.a_first; a < 3; ++a) sR[a * RW * NZ + t] += amp * sc;
        }
    }
    for (int j = sp[2] + threadIdx.x; j < sp[3]; j += NT) {
        const int t = A.enf.pos[j] - lo_key;
        const float val = A.enf.vals[j] / (A.enf.ndim * sC[t]);
        for (int a = A.a_first; a < 3; ++a) sR[a * RW * NZ + t] = val;
    }
    __syncthreads();

    // p = c0^2 ((rho_x + rho_y) + rho_z); stores; correlation; p kept in sR[0] for gathers + r2c
    float2 pv[N1];
    if (act) {
        float* gr = A.corr.grad;
#pragma unroll
        for (int n1 = 0; n1 < N1; ++n1) {
            const int n = lane + N2 * n1;
            const int t = r * NZ + 2 * n;
            const long long i = i0 + t;
            const float2 q0 = *reinterpret_cast<const float2*>(sR + t);
            const float2 q1 = *reinterpret_cast<const float2*>(sR + RW * NZ + t);
            const float2 q2 = *reinterpret_cast<const float2*>(sR + 2 * RW * NZ + t);
            *reinterpret_cast<float2*>(A.rho[0] + i) = q0;
            *reinterpret_cast<float2*>(A.rho[1] + i) = q1;
            *reinterpret_cast<float2*>(A.rho[2] + i) = q2;
            const float2 c2 = *reinterpret_cast<const float2*>(sC + t);
            float2 p;
            p.x = c2.x * ((q0.x + q1.x) + q2.x);
            p.y = c2.y * ((q0.y + q1.y) + q2.y);
            *reinterpret_cast<float2*>(A.p_out + i) = p;
            *reinterpret_cast<float2*>(sR + t) = p;
            if (corr) {
                const float2 pm = *reinterpret_cast<const float2*>(sK + t);
                const float2 po = *reinterpret_cast<const float2*>(sK + RW * NZ + t);
                const float2 qa = *reinterpret_cast<const float2*>(sK + 2 * RW * NZ + t);
                float2 gv = *reinterpret_cast<const float2*>(sK + 3 * RW * NZ + t);
                const float wx = 2.f / (c2.x * sqrtf(c2.x)), wy = 2.f / (c2.y * sqrtf(c2.y));
                gv.x += wx * (((p.x - 2.f * pm.x) + po.x) * A.corr.inv_dt) * qa.x;
                gv.y += wy * (((p.y - 2.f * pm.y) + po.y) * A.corr.inv_dt) * qa.y;
                *reinterpret_cast<float2*>(gr + i) = gv;
            }
            if (A.check_step > 0 && i == 0 && !isfinite(p.x)) atomicMin(A.diverged, A.check_step);
            pv[n1] = p;
        }
    }
    __syncthreads();
    for (int s = sp[4] + threadIdx.x; s < sp[5]; s += NT) A.sens.out[A.sens.idx[s]] = sR[A.sens.pos[s] - lo_key];
    for (int j = sp[6] + threadIdx.x; j < sp[7]; j += NT) A.shell.out[j] = sR[A.shell.pos[j] - lo_key];

    // forward r2c of p into S0
    if (act) row_r2c_a<M, N1>(pv, lane, twM, zt_row);
    __syncthreads();
    if (rowok && lane < N1) row_r2c_b<M, N1>(zt_row, lane, zn_row);
    __syncthreads();
    if (rowok) row_r2c_finish<M, TPR>(zn_row, lane, g.tw_rfft, A.S[0] + row * g.nzp);
}

// ======================================================================================
// dispatch
// ======================================================================================
namespace {

template <int AXIS, bool INV, int L, int N1, int TB, int MINB>
cudaError_t run_pencil(const GridDev& g, const PencilJobs& j, cudaStream_t st) {
    using C = PencilCfg<L, N1, TB>;
    auto kern = pencil_fast_kernel<AXIS, INV, L, N1, TB, MINB>;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
        configured = true;
    }
    dim3 grid((g.nzh + TB - 1) / TB, AXIS == 0 ? g.ny : g.nx);
    kern<<<grid, C::NT, C::SMEM, st>>>(g, j);
    return cudaGetLastError();
}

template <int L, int N1, int TB, int MINB>
cudaError_t pencil_sized(int axis, bool inv, const GridDev& g, const PencilJobs& j, cudaStream_t st) {
    if (axis == 0) return run_pencil<0, false, L, N1, TB, MINB>(g, j, st);
    return inv ? run_pencil<1, true, L, N1, TB, MINB>(g, j, st) : run_pencil<1, false, L, N1, TB, MINB>(g, j, st);
}

}  // namespace

bool fast_pencil_supported(int L) {
    switch (L) {
        case 32: case 64: case 96: case 128: case 144: case 256: case 480: return true;
        default: return false;
    }
}

cudaError_t launch_pencil_fast(int axis, bool inv, const GridDev& g, const PencilJobs& j, cudaStream_t st) {
    const int L = axis == 0 ? g.px.L : g.py.L;
    switch (L) {
        case 32: return pencil_sized<32, 2, 16, 4>(axis, inv, g, j, st);
        case 64: return pencil_sized<64, 4, 16, 4>(axis, inv, g, j, st);
        case 96: return pencil_sized<96, 6, 16, 4>(axis, inv, g, j, st);
        case 128: return pencil_sized<128, 8, 16, 4>(axis, inv, g, j, st);
        case 144: return pencil_sized<144, 9, 16, 3>(axis, inv, g, j, st);
        case 256: return pencil_sized<256, 16, 16, 3>(axis, inv, g, j, st);
        case 480: return pencil_sized<480, 30, 8, 3>(axis, inv, g, j, st);
        default: return cudaErrorInvalidValue;
    }
}

bool fast_rows_supported(int nz) {
    switch (nz) {
        case 64: case 96: case 128: case 144: case 256: return true;
        default: return false;
    }
}

namespace {
constexpr int kZRows = 8;

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
    const size_t smem = C::FIXED + size_t(3) * kZRows * g.nzp * 8 +
                        size_t(r[0].field ? 6 : 3) * kZRows * C::NZ * 4;
    auto kern = zvel_fast_kernel<M, N1, kZRows>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const unsigned blocks = (unsigned)((g.rows + kZRows - 1) / kZRows);
    kern<<<blocks, C::NT, smem, st>>>(a);
    return cudaGetLastError();
}
template <int M, int N1>
cudaError_t zrho_sized(const GridDev& g, const ZrhoArgs& za, cudaStream_t st) {
    using C = RowCfg<M, N1, kZRows>;
    ZrhoFastArgs a;
    a.g = g;
    a.a = za;
    const int nf = 4 + (za.dtrho0.field ? 1 : 0) + (za.corr.grad ? 4 : 0);
    const size_t smem = C::FIXED + size_t(3) * kZRows * g.nzp * 8 + size_t(nf) * kZRows * C::NZ * 4;
    auto kern = zrho_fast_kernel<M, N1, kZRows>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const unsigned blocks = (unsigned)((g.rows + kZRows - 1) / kZRows);
    kern<<<blocks, C::NT, smem, st>>>(a);
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

}  // namespace ustfwi_dev
