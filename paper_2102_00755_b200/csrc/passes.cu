// Register-resident pass kernels for the supported transform lengths (sm_100a).
//
// Each line transform of length L = N1 * N2 is a two-level Cooley-Tukey:
//   phase A  thread (col, n2) loads x[n2 + N2*n1] straight from HBM into registers,
//            does the N1-point codelet, applies W_L^(n2*k1) and writes one transposed tile
//            to shared memory;
//   phase B  thread (col, k1) reads its N2 values and does the N2-point codelet, giving
//            X[k1 + N1*k2] in registers.
// A forward-multiply-inverse sandwich (the x pass) therefore costs one HBM read, one HBM
// write per output and two shared-memory round trips; kappa and the stagger factors are
// applied in registers between the two halves. The z passes use the same scheme on the
// half-length complex transform of each real row (M = nz/2) and keep the elementwise
// velocity / density / pressure update, sparse sources and shell, gathers and the c0
// correlation in registers.
#include <cuda_runtime.h>

#include "fft_reg.cuh"
#include "kernels.cuh"

namespace ustfwi_dev {

__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }

constexpr int cmax(int a, int b) { return a > b ? a : b; }

// ======================================================================================
// Pencil passes (x and y)
// ======================================================================================
template <int L, int N1, int TB>
struct PencilCfg {
    static constexpr int N2 = L / N1;
    static constexpr int NT = TB * cmax(N1, N2);
    static constexpr int KP = N2 * TB + 8;  // float2 pitch of one k1 slab (+64 B against bank conflicts)
};

__device__ __forceinline__ float kappa_fast(float k2, float half_cdt) {
    const float x = half_cdt * sqrtf(k2);
    return (x < 1e-4f) ? 1.f - x * x * (1.f / 6.f) : sinf(x) / x;
}

// AXIS 0: x pencils at fixed y = blockIdx.y (always forward * multiplier * inverse).
// AXIS 1: y pencils at fixed x = blockIdx.y, direction INV, optional premultiplier.
template <int AXIS, bool INV, int L, int N1, int TB>
__global__ void __launch_bounds__(PencilCfg<L, N1, TB>::NT)
    pencil_fast_kernel(const __grid_constant__ GridDev g, const __grid_constant__ PencilJobs jobs) {
    using C = PencilCfg<L, N1, TB>;
    constexpr int N2 = C::N2, KP = C::KP;
    __shared__ float2 ys[N1 * KP];
    __shared__ float2 tw[L];
    const FftPlan& plan = AXIS == 0 ? g.px : g.py;
    for (int i = threadIdx.x; i < L; i += C::NT) tw[i] = plan.tw[i];

    const int c0 = blockIdx.x * TB;
    const int ncol = min(TB, g.nzh - c0);
    const long long pitch = (AXIS == 0) ? (long long)g.ny * g.nzp : (long long)g.nzp;
    const long long base = (AXIS == 0) ? (long long)blockIdx.y * g.nzp + c0 : (long long)blockIdx.y * g.ny * g.nzp + c0;
    const int c = threadIdx.x % TB;
    const int ra = threadIdx.x / TB;  // n2 in phase A, k1 in phase B
    const bool inA = ra < N2, inB = ra < N1;
    const bool colok = c < ncol;
    __syncthreads();

    float2 X[N2];
    float kap[N2];
    bool kap_ready = false;
    int loaded = -1;
    for (int jb = 0; jb < jobs.n; ++jb) {
        const PencilJob J = jobs.job[jb];
        const bool reload = J.src != loaded;
        if (AXIS == 0 || !INV) {
            if (reload) {
                // ---- forward transform of the source tile: phase A -> smem -> phase B
                if (loaded >= 0 || jb > 0) __syncthreads();
                if (inA) {
                    float2 a[N1];
                    const float2* s = jobs.buf[J.src] + base + c;
#pragma unroll
                    for (int n1 = 0; n1 < N1; ++n1)
                        a[n1] = colok ? s[(ra + N2 * n1) * pitch] : make_float2(0.f, 0.f);
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
                loaded = J.src;
            }
            if (AXIS == 1) {
                // forward y pass: store X[k1 + N1*k2]
                if (inB && colok) {
                    float2* d = jobs.buf[J.dst] + base + c;
#pragma unroll
                    for (int k2 = 0; k2 < N2; ++k2) d[(ra + N1 * k2) * pitch] = X[k2];
                }
                continue;
            }
            if (!kap_ready) {
                if (inB) {
                    const float ky = g.ky[blockIdx.y];
                    const float kz = colok ? g.kz[c0 + c] : 0.f;
#pragma unroll
                    for (int k2 = 0; k2 < N2; ++k2) {
                        const float kx = g.kx[ra + N1 * k2];
                        kap[k2] = kappa_fast(kx * kx + ky * ky + kz * kz, g.half_cdt);
                    }
                }
                kap_ready = true;
            }
        } else if (reload) {
            // inverse y pass: load the natural-order spectrum in phase B layout
            if (inB) {
                const float2* s = jobs.buf[J.src] + base + c;
#pragma unroll
                for (int k2 = 0; k2 < N2; ++k2) X[k2] = colok ? s[(ra + N1 * k2) * pitch] : make_float2(0.f, 0.f);
            }
            loaded = J.src;
        }
        // ---- inverse transform (x pass after the multiplier, or the inverse y pass)
        float2 b[N2];
        if (inB) {
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2) {
                float2 v = X[k2];
                if (J.dmul) v = cmul(v, __ldg(J.dmul + ra + N1 * k2));
                if (AXIS == 0 && J.kappa) v = cscale(v, kap[k2]);
                b[k2] = v;
            }
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
                float2* d = jobs.buf[J.dst] + base + c;
#pragma unroll
                for (int n1 = 0; n1 < N1; ++n1) d[(ra + N2 * n1) * pitch] = a[n1];
            }
        }
    }
}

// ======================================================================================
// Row (z) passes: real FFT of length nz = 2M through the M-point complex transform
// ======================================================================================
template <int M, int N1>
struct RowCfg {
    static constexpr int N2 = M / N1;
    static constexpr int TPR = cmax(N1, N2);           // threads per row
    static constexpr int RW = 256 / TPR;               // rows per CTA
    static constexpr int NT = RW * TPR;
    static constexpr int ZP = N2 + 1;                  // transposed tile pitch (bank spread)
    static constexpr int ZT = N1 * ZP;                 // float2 per row, transposed layout
};

// c2r of one row, phase B half: from the half spectrum (nzh bins, optional premultiplier)
// to the twiddled inverse N2-point transforms, written transposed into zt.
template <int M, int N1>
__device__ __forceinline__ void row_c2r_b(const float2* __restrict__ Xrow, const float2* __restrict__ premul,
                                          const float2* __restrict__ twr, const float2* twM, int k1,
                                          float2* zt_row) {
    using C = RowCfg<M, N1>;
    constexpr int N2 = C::N2;
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
    for (int n2 = 0; n2 < N2; ++n2) zt_row[k1 * C::ZP + n2] = n2 ? cmul(z[n2], conjf2(twM[k1 * n2])) : z[n2];
}

// phase A of the inverse: the N1-point inverse codelet -> interleaved real pairs (scaled)
template <int M, int N1>
__device__ __forceinline__ void row_c2r_a(const float2* zt_row, int n2, float scale, float2 (&u)[N1]) {
    using C = RowCfg<M, N1>;
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) u[k1] = zt_row[k1 * C::ZP + n2];
    RDft<N1, true>::run(u);
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) u[n1] = cscale(u[n1], scale);
}

// forward r2c of a row whose interleaved pairs u[n1] (n = n2 + N2*n1) are in registers:
// phase A codelet + twiddle -> zt (caller syncs) ...
template <int M, int N1>
__device__ __forceinline__ void row_r2c_a(float2 (&u)[N1], int n2, const float2* twM, float2* zt_row) {
    using C = RowCfg<M, N1>;
    RDft<N1, false>::run(u);
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) zt_row[k1 * C::ZP + n2] = k1 ? cmul(u[k1], twM[n2 * k1]) : u[k1];
}
// ... phase B codelet -> natural order Z into zn (caller syncs) ...
template <int M, int N1>
__device__ __forceinline__ void row_r2c_b(const float2* zt_row, int k1, float2* zn_row) {
    using C = RowCfg<M, N1>;
    constexpr int N2 = C::N2;
    float2 z[N2];
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) z[n2] = zt_row[k1 * C::ZP + n2];
    RDft<N2, false>::run(z);
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) zn_row[k1 + N1 * k2] = z[k2];
}
// ... split into the M+1 half-spectrum bins and store
template <int M, int N1>
__device__ __forceinline__ void row_r2c_finish(const float2* zn_row, int lane, const float2* __restrict__ twr,
                                               float2* __restrict__ Xrow) {
    using C = RowCfg<M, N1>;
    for (int k = lane; k <= M; k += C::TPR) {
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

template <int M, int N1>
__global__ void __launch_bounds__(RowCfg<M, N1>::NT) zvel_fast_kernel(const __grid_constant__ ZvelFastArgs A) {
    using C = RowCfg<M, N1>;
    constexpr int N2 = C::N2, RW = C::RW, TPR = C::TPR;
    constexpr int NZ = 2 * M;
    __shared__ float2 zt[RW * C::ZT];
    __shared__ float2 zn[RW * M];
    __shared__ float2 twM[M];
    const GridDev& g = A.g;
    for (int i = threadIdx.x; i < M; i += C::NT) twM[i] = g.pzh.tw[i];
    const int r = threadIdx.x / TPR, lane = threadIdx.x % TPR;
    const long long row = (long long)blockIdx.x * RW + r;
    const bool rowok = row < g.rows;
    const int x = rowok ? (int)(row / g.ny) : 0, y = rowok ? (int)(row % g.ny) : 0;
    float2* zt_row = zt + r * C::ZT;
    float2* zn_row = zn + r * M;
    __syncthreads();
#pragma unroll 1
    for (int a = 0; a < 3; ++a) {
        float2* S = A.S[a];
        if (rowok && lane < N1) row_c2r_b<M, N1>(S + row * g.nzp, a == 2 ? A.dz_plus : nullptr, g.tw_rfft, twM, lane, zt_row);
        __syncthreads();
        float2 u[N1];
        if (rowok && lane < N2) {
            row_c2r_a<M, N1>(zt_row, lane, g.inv_n, u);
            const float pa = a == 0 ? __ldg(A.pml.prof[0] + x) : (a == 1 ? __ldg(A.pml.prof[1] + y) : 0.f);
            float* v = A.v[a] + row * NZ;
#pragma unroll
            for (int n1 = 0; n1 < N1; ++n1) {
                const int n = lane + N2 * n1;
                float2 vv = *reinterpret_cast<const float2*>(v + 2 * n);
                float2 pm = make_float2(pa, pa);
                if (a == 2) pm = make_float2(__ldg(A.pml.prof[2] + 2 * n), __ldg(A.pml.prof[2] + 2 * n + 1));
                const long long i = row * NZ + 2 * n;
                const float r0 = A.r[a].at(i), r1 = A.r[a].at(i + 1);
                vv.x = pm.x * (pm.x * vv.x - r0 * u[n1].x);
                vv.y = pm.y * (pm.y * vv.y - r1 * u[n1].y);
                *reinterpret_cast<float2*>(v + 2 * n) = vv;
                u[n1] = vv;
            }
        }
        __syncthreads();
        if (rowok && lane < N2) row_r2c_a<M, N1>(u, lane, twM, zt_row);
        __syncthreads();
        if (rowok && lane < N1) row_r2c_b<M, N1>(zt_row, lane, zn_row);
        __syncthreads();
        if (rowok) row_r2c_finish<M, N1>(zn_row, lane, g.tw_rfft, S + row * g.nzp);
    }
}

struct ZrhoFastArgs {
    GridDev g;
    ZrhoArgs a;
};

template <int M, int N1>
__global__ void __launch_bounds__(RowCfg<M, N1>::NT) zrho_fast_kernel(const __grid_constant__ ZrhoFastArgs P) {
    using C = RowCfg<M, N1>;
    constexpr int N2 = C::N2, RW = C::RW, TPR = C::TPR;
    constexpr int NZ = 2 * M;
    __shared__ float2 zt[RW * C::ZT];
    __shared__ float2 zn[RW * M];
    __shared__ float2 twM[M];
    __shared__ int sp[8];
    const GridDev& g = P.g;
    const ZrhoArgs& A = P.a;
    for (int i = threadIdx.x; i < M; i += C::NT) twM[i] = g.pzh.tw[i];
    const int r = threadIdx.x / TPR, lane = threadIdx.x % TPR;
    const long long row0 = (long long)blockIdx.x * RW;
    const long long row = row0 + r;
    const bool rowok = row < g.rows;
    const bool act = rowok && lane < N2;  // phase A owner of pairs n = lane + N2*n1
    const int x = rowok ? (int)(row / g.ny) : 0, y = rowok ? (int)(row % g.ny) : 0;
    float2* zt_row = zt + r * C::ZT;
    float2* zn_row = zn + r * M;
    const long long i0 = row0 * NZ;
    const int lo_key = (int)i0;
    const int hi_key = (int)min((long long)(row0 + RW) * NZ, g.N);
    if (threadIdx.x == 0) {
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
    __syncthreads();

    // rho[a][n1] holds the pair (rho_a[2n], rho_a[2n+1]) for n = lane + N2*n1
    float2 rho[3][N1];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        float2 u[N1];
        if (rowok && lane < N1) row_c2r_b<M, N1>(A.S[a] + row * g.nzp, a == 2 ? A.dz_minus : nullptr, g.tw_rfft, twM, lane, zt_row);
        __syncthreads();
        if (act) {
            row_c2r_a<M, N1>(zt_row, lane, g.inv_n, u);
            const float pa = a == 0 ? __ldg(A.pml.prof[0] + x) : (a == 1 ? __ldg(A.pml.prof[1] + y) : 0.f);
            const float* rr = A.rho[a] + row * NZ;
#pragma unroll
            for (int n1 = 0; n1 < N1; ++n1) {
                const int n = lane + N2 * n1;
                float2 q = *reinterpret_cast<const float2*>(rr + 2 * n);
                float2 pm = make_float2(pa, pa);
                if (a == 2) pm = make_float2(__ldg(A.pml.prof[2] + 2 * n), __ldg(A.pml.prof[2] + 2 * n + 1));
                const long long i = row * NZ + 2 * n;
                const float d0 = A.dtrho0.at(i), d1 = A.dtrho0.at(i + 1);
                q.x = pm.x * (pm.x * q.x - d0 * u[n1].x);
                q.y = pm.y * (pm.y * q.y - d1 * u[n1].y);
                rho[a][n1] = q;
            }
        }
        __syncthreads();
    }

    // sparse mass sources / Dirichlet shell: applied by the owner thread, in registers
    auto owner_apply = [&](int pos, auto&& fn) {
        const int t = pos - lo_key;
        const int rr = t / NZ, z = t % NZ, n = z >> 1, comp = z & 1;
        if (!(act && rr == r && (n % N2) == lane)) return;
        const int n1 = n / N2;
#pragma unroll
        for (int k = 0; k < N1; ++k)
            if (k == n1) fn(k, comp);
    };
    for (int u = sp[0]; u < sp[1]; ++u) {
        const int pos = A.inj.pos[u];
        float add = 0.f;
        bool any = false;
        for (int cc = A.inj.csr[u]; cc < A.inj.csr[u + 1]; ++cc) {
            const int n = A.step_n - A.inj.delay[cc];
            if (n < 0 || n >= A.inj.len[cc]) continue;
            const float amp = A.inj.w[cc] * A.inj.sig[A.inj.off[cc] + (long long)n * A.inj.stride[cc]];
            if (amp == 0.f) continue;
            any = true;
            const float s = amp * A.inj.scale[u];
            owner_apply(pos, [&](int k, int comp) {
#pragma unroll
                for (int a = 0; a < 3; ++a)
                    if (a >= A.a_first) {
                        if (comp) rho[a][k].y += s;
                        else rho[a][k].x += s;
                    }
            });
        }
        (void)any;
        (void)add;
    }
    for (int j = sp[2]; j < sp[3]; ++j) {
        const int pos = A.enf.pos[j];
        owner_apply(pos, [&](int k, int comp) {
            const float val = A.enf.vals[j] / (A.enf.ndim * __ldg(A.c0sq + pos));
#pragma unroll
            for (int a = 0; a < 3; ++a)
                if (a >= A.a_first) {
                    if (comp) rho[a][k].y = val;
                    else rho[a][k].x = val;
                }
        });
    }

    // p = c0^2 ((rho_x + rho_y) + rho_z), stores, correlation
    float2 pv[N1];
    if (act) {
#pragma unroll
        for (int n1 = 0; n1 < N1; ++n1) {
            const int n = lane + N2 * n1;
            const long long i = row * NZ + 2 * n;
#pragma unroll
            for (int a = 0; a < 3; ++a) *reinterpret_cast<float2*>(A.rho[a] + i) = rho[a][n1];
            const float2 c2 = *reinterpret_cast<const float2*>(A.c0sq + i);
            float2 p;
            p.x = c2.x * ((rho[0][n1].x + rho[1][n1].x) + rho[2][n1].x);
            p.y = c2.y * ((rho[0][n1].y + rho[1][n1].y) + rho[2][n1].y);
            *reinterpret_cast<float2*>(A.p_out + i) = p;
            if (A.corr.grad != nullptr) {
                const float2 pm = *reinterpret_cast<const float2*>(A.corr.p_mid + i);
                const float2 po = *reinterpret_cast<const float2*>(A.corr.p_old + i);
                const float2 q = *reinterpret_cast<const float2*>(A.corr.q_adj + i);
                float2 gr = *reinterpret_cast<const float2*>(A.corr.grad + i);
                const float wx = 2.f / (c2.x * sqrtf(c2.x)), wy = 2.f / (c2.y * sqrtf(c2.y));
                gr.x += wx * (((p.x - 2.f * pm.x) + po.x) * A.corr.inv_dt) * q.x;
                gr.y += wy * (((p.y - 2.f * pm.y) + po.y) * A.corr.inv_dt) * q.y;
                *reinterpret_cast<float2*>(A.corr.grad + i) = gr;
            }
            if (A.check_step > 0 && i == 0 && !isfinite(p.x)) atomicMin(A.diverged, A.check_step);
            pv[n1] = p;
        }
    }
    // gathers of p (sensors, shell record) by the owner thread
    for (int s = sp[4]; s < sp[5]; ++s)
        owner_apply(A.sens.pos[s], [&](int k, int comp) { A.sens.out[A.sens.idx[s]] = comp ? pv[k].y : pv[k].x; });
    for (int j = sp[6]; j < sp[7]; ++j)
        owner_apply(A.shell.pos[j], [&](int k, int comp) { A.shell.out[j] = comp ? pv[k].y : pv[k].x; });

    // forward r2c of p into S0
    if (act) row_r2c_a<M, N1>(pv, lane, twM, zt_row);
    __syncthreads();
    if (rowok && lane < N1) row_r2c_b<M, N1>(zt_row, lane, zn_row);
    __syncthreads();
    if (rowok) row_r2c_finish<M, N1>(zn_row, lane, g.tw_rfft, A.S[0] + row * g.nzp);
}

// ======================================================================================
// dispatch
// ======================================================================================
namespace {

template <int AXIS, bool INV, int L, int N1, int TB>
cudaError_t run_pencil(const GridDev& g, const PencilJobs& j, cudaStream_t st) {
    dim3 grid((g.nzh + TB - 1) / TB, AXIS == 0 ? g.ny : g.nx);
    pencil_fast_kernel<AXIS, INV, L, N1, TB><<<grid, PencilCfg<L, N1, TB>::NT, 0, st>>>(g, j);
    return cudaGetLastError();
}

template <int L, int N1, int TB>
cudaError_t pencil_sized(int axis, bool inv, const GridDev& g, const PencilJobs& j, cudaStream_t st) {
    if (axis == 0) return run_pencil<0, false, L, N1, TB>(g, j, st);
    return inv ? run_pencil<1, true, L, N1, TB>(g, j, st) : run_pencil<1, false, L, N1, TB>(g, j, st);
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
        case 32: return pencil_sized<32, 2, 16>(axis, inv, g, j, st);
        case 64: return pencil_sized<64, 4, 16>(axis, inv, g, j, st);
        case 96: return pencil_sized<96, 6, 16>(axis, inv, g, j, st);
        case 128: return pencil_sized<128, 8, 16>(axis, inv, g, j, st);
        case 144: return pencil_sized<144, 9, 16>(axis, inv, g, j, st);
        case 256: return pencil_sized<256, 16, 16>(axis, inv, g, j, st);
        case 480: return pencil_sized<480, 30, 8>(axis, inv, g, j, st);
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
template <int M, int N1>
cudaError_t zvel_sized(const GridDev& g, float2* S[3], const float2* dz_plus, float* v[3], const Pml& pml,
                       const Coef r[3], cudaStream_t st) {
    using C = RowCfg<M, N1>;
    ZvelFastArgs a;
    a.g = g;
    for (int f = 0; f < 3; ++f) {
        a.S[f] = S[f];
        a.v[f] = v[f];
        a.r[f] = r[f];
    }
    a.dz_plus = dz_plus;
    a.pml = pml;
    const unsigned blocks = (unsigned)((g.rows + C::RW - 1) / C::RW);
    zvel_fast_kernel<M, N1><<<blocks, C::NT, 0, st>>>(a);
    return cudaGetLastError();
}
template <int M, int N1>
cudaError_t zrho_sized(const GridDev& g, const ZrhoArgs& za, cudaStream_t st) {
    using C = RowCfg<M, N1>;
    ZrhoFastArgs a;
    a.g = g;
    a.a = za;
    const unsigned blocks = (unsigned)((g.rows + C::RW - 1) / C::RW);
    zrho_fast_kernel<M, N1><<<blocks, C::NT, 0, st>>>(a);
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
