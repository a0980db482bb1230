// Device-side data structures shared by the pass kernels and the host orchestration.
#pragma once

#include <atomic>

#include <cstdint>

#include <cuda_runtime.h>

#include "fft_smem.cuh"

namespace ustfwi_dev {

// Geometry of one context. Real fields are [nx][ny][nz] (z fastest, field.hpp:14-17);
// spectral scratch is [nx][ny][nzp] float2 holding the nzh = nz/2+1 half-spectrum bins
// of the last axis (fft.hpp:27-29) with the row padded to nzp for aligned tiles.
struct GridDev {
    int nx, ny, nz, nzh, nzp;
    long long N;       // nx*ny*nz
    long long rows;    // nx*ny
    FftPlan px, py, pzh;        // complex plans along x, y and the half-length z plan
    const float2* tw_rfft;      // exp(-2*pi*i*k/nz), k in [0, nz/2]  (real-FFT split)
    const float* kx;            // wavenumbers per axis (fft.hpp:121-130), fp32
    const float* ky;
    const float* kz;
    float half_cdt;             // 0.5 * c_ref * dt   (kappa = sinc(half_cdt*|k|), engine.hpp:43)
    float inv_n;                // 1/N (RealFft::inverse normalisation, fft.hpp:58-63)
    int x0, xn;                 // x-plane window of the y and z passes (chunked steps): [x0, x0+xn)
    int pgrid;                  // persistent pencil grid override (0: MINB CTAs per SM)
};

// Sparse mass-source injection: unique sorted flat positions, CSR into contributions.
// amplitude(c, n) = w[c] * sig[off[c] + (n - delay[c]) * stride[c]]  for 0 <= n-delay < len[c]
// (SourceSet::sample, medium.hpp:80-84; encoded: SPEC.md:296-304). Each unique position
// adds amp * scale[u] to every split density (inject_mass_source, engine.hpp:296-300).
struct SparseInject {
    int n_unique;
    const int* pos;
    const int* csr;
    const int* off;
    const int* len;
    const int* stride;
    const int* delay;
    const float* w;
    const float* sig;
    const float* scale;
    const int* blk8 = nullptr;  // blk8[b] = first unique position >= b * 8 rows (row blocks of 8)
};

// Sparse gather of p (sensor gather simulate.hpp:88-90, shell record :91-95):
// out[idx[i]] = p[pos[i]], positions sorted ascending.
struct SparseGather {
    int n;
    const int* pos;
    const int* idx;
    float* out;
    const int* blk8 = nullptr;  // per 8-row block offsets into pos (see SparseInject)
};

// Dirichlet shell (enforce_shell, engine.hpp:304-307; scaling gradient.hpp:417-427):
// rho_a[pos[j]] = vals[j] / (ndim * c0^2(pos)), vals = raw recorded pressure.
struct SparseEnforce {
    int n;
    const int* pos;
    const float* vals;
    float ndim;
    const int* blk8 = nullptr;
};

// [lo, hi) of the sorted position list inside rows [row0, row0 + nrows): O(1) from the
// per-8-row-block offsets when the block is 8-row aligned, else a binary search
__device__ __forceinline__ void sparse_range(const int* pos, int n, const int* blk8, long long row0, int nrows,
                                             int nz, int& lo, int& hi) {
    if (n == 0) {
        lo = hi = 0;
        return;
    }
    if (blk8 && (row0 & 7) == 0) {
        lo = blk8[row0 >> 3];
        hi = blk8[(row0 + nrows + 7) >> 3];
        return;
    }
    auto lb = [&](long long key) {
        int a = 0, b = n;
        while (a < b) {
            const int mid = (a + b) >> 1;
            if (pos[mid] < key) a = mid + 1;
            else b = mid;
        }
        return a;
    };
    lo = lb(row0 * nz);
    hi = lb((row0 + nrows) * nz);
}

// In-kernel c0 correlation (GradientAccumulator, gradient.hpp:146-160,177-182):
// grad += (2/c0^3) * ((p_new - 2 p_mid) + p_old) / dt * q_adj
struct Correlate {
    const float* p_mid;
    const float* p_old;
    const float* q_adj;
    float* grad;
    float inv_dt;
    // GradientAccumulator::accumulate (gradient.hpp:177-203) beyond the c0 ddot term (used by
    // the stand-alone correlate kernel only): grad += wa1 (a1_old - a1_new)/2 q
    // + wa1l (a1l_old - a1l_new)/2 q + wa2 a2_mid q dt + wa2l a2l_mid q dt with a1 = |k|^y p,
    // a2 = |k|^(y+1) p, a1l / a2l the same times log|k|^2, of the replay pressures
    int use_ddot = 1;
    const float* a1_new = nullptr;
    const float* a1_old = nullptr;
    const float* a2_mid = nullptr;
    const float* a1l_new = nullptr;
    const float* a1l_old = nullptr;
    const float* a2l_mid = nullptr;
    const float* wa1 = nullptr;
    const float* wa2 = nullptr;
    const float* wa1l = nullptr;
    const float* wa2l = nullptr;
    float dt = 0.f;
    // set: the pressure kernel computing this correlation is the ADJOINT's (its own p is q) and
    // the replay's new pressure is read from p_new; null: the kernel is the replay's (its own
    // p is p_new) and q is read from q_adj
    const float* p_new = nullptr;
};

#ifdef __CUDACC__
// grad += (2/c0^3) ((p_new - 2 p_mid) + p_old) / dt * q for a pair of voxels at i (i even),
// with p the calling pressure kernel's own value (see Correlate::p_new); the same fp32
// operations in the same order whichever stepper's kernel runs it
__device__ __forceinline__ void correlate_pair(const Correlate& C, long long i, float2 p, float2 c2) {
    const float2 pm = *reinterpret_cast<const float2*>(C.p_mid + i);
    const float2 po = *reinterpret_cast<const float2*>(C.p_old + i);
    float2 pn, qa;
    if (C.p_new != nullptr) {
        pn = *reinterpret_cast<const float2*>(C.p_new + i);
        qa = p;
    } else {
        pn = p;
        qa = *reinterpret_cast<const float2*>(C.q_adj + i);
    }
    float2 gv = *reinterpret_cast<const float2*>(C.grad + i);
    const float wx = 2.f / (c2.x * sqrtf(c2.x)), wy = 2.f / (c2.y * sqrtf(c2.y));
    gv.x += wx * (((pn.x - 2.f * pm.x) + po.x) * C.inv_dt) * qa.x;
    gv.y += wy * (((pn.y - 2.f * pm.y) + po.y) * C.inv_dt) * qa.y;
    *reinterpret_cast<float2*>(C.grad + i) = gv;
}
#endif

// Per-axis PML profiles (make_pml, grid.hpp:153-178), fp32.
struct Pml {
    const float* prof[3];
};

// Medium coefficients: either a uniform scalar or a field (nullptr -> scalar).
struct Coef {
    const float* field;
    float scalar;
    __device__ __forceinline__ float at(long long i) const { return field ? __ldg(field + i) : scalar; }
};


// ---- pass arguments ---------------------------------------------------------------
struct PencilJob {
    int src;              // scratch buffer index read
    int dst;              // scratch buffer index written
    const float2* dmul;   // per-index factor along the pass axis (D_a table), nullable
    int kappa;            // X pass only: 1 multiply by kappa(|k|), 2 by |k|^kexp (power_multiplier),
                          // 3 by |k|^kexp log|k|^2
    float kexp;           // exponent of |k| for kappa == 2, 3 (engine.hpp:88-101)
};

// power_multiplier (engine.hpp:88-94): |k|^e over the half spectrum, the k = 0 bin 1 for
// e == 0 and 0 otherwise (fractional-Laplacian convention); kind 3: times log_k2_multiplier
// (engine.hpp:97-101, 0 at k = 0), as GradientAccumulator builds mult_a1l / mult_a2l
// (gradient.hpp:132-142)
__device__ __forceinline__ float kpow_mult(float k2, float e, int kind = 2) {
    if (k2 == 0.f) return (kind == 2 && e == 0.f) ? 1.f : 0.f;
    const float m = powf(k2, 0.5f * e);
    return kind == 3 ? m * logf(k2) : m;
}

struct PencilJobs {
    int n;
    PencilJob job[4];
    float2* buf[3];
};

struct ZrhoArgs {
    float2* S[3];
    const float2* dz_minus;
    float* rho[3];
    Pml pml;
    Coef dtrho0;
    const float* c0sq;
    float* p_out;
    int a_first;          // first active axis (3 - ndim): inactive split densities stay 0
    int step_n;           // source time index
    SparseInject inj;     // n_unique == 0 -> none
    SparseEnforce enf;    // n == 0 -> none
    SparseGather sens;    // n == 0 -> none
    SparseGather shell;   // n == 0 -> none
    Correlate corr;       // grad == nullptr -> none
    int check_step;       // >0: divergence check of p[0] at this stepper step index
    int* diverged;        // atomicMin of the failing step index
    int rows_per_cta;
    float* du_out[3];     // absorbing media: the raw derivative d_a^- v_a (engine.hpp:285), nullable
};

// Absorbing pressure (update_pressure, engine.hpp:327-343), after the sparse work:
//   sum = sum_a rho_a, ain = (dt rho0 / dt) sum_a du_a       (abs_prep)
//   p = c0^2 (sum + sign tau0 aout) - c0^2 eta aout2           (abs_pressure)
// with aout = |k|^(y-2) ain and aout2 = |k|^(y-1) sum applied spectrally in between.
struct AbsArgs {
    const float* rho[3];
    const float* du[3];
    Coef dtrho0;
    float inv_dt;
    float* sum;
    float* ain;
    const float* c0sq;
    const float* tau0;
    const float* eta;     // nullptr: no dispersion term
    const float* aout;
    const float* aout2;
    float sign;           // absorption_sign (+1 forward / adjoint, -1 replay, gradient.hpp:429-431)
    float* p_out;
    int check_step;
    int* diverged;
};


// rho0 gradient legs (GradientAccumulator::accumulate_rho0, gradient.hpp:213-239)
struct Rho0Args {
    Coef rho0;
    Coef dtr;             // dt / rho~_a of the axis (staggered density coefficient)
    float inv_dt, dt;
    const float* q;       // adjoint pressure
    const float* dp;
    const float* drq;
    const float* out;
    float* tmp;
    float* grad;
};

// cudaFuncSetAttribute is per device: run `set` once per device that launches the kernel
// (a process may drive several GPUs, one context each)
template <class F>
inline void once_per_device(std::atomic<unsigned long long>& mask, F&& set) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(mask.load() & bit)) {
        set();
        mask.fetch_or(bit);
    }
}

// ---- launchers (kernels.cu) ---------------------------------------------------------
int pencil_tile_cols(int L);
int zrows_per_cta(int nz);
cudaError_t launch_pencil(int axis, bool inv, const GridDev& g, const PencilJobs& jobs, cudaStream_t st);
cudaError_t launch_zvel(const GridDev& g, float2* S[3], const float2* dz_plus, float* v[3], const Pml& pml,
                        const Coef r[3], cudaStream_t st);
cudaError_t launch_zrho(const GridDev& g, ZrhoArgs a, bool update, cudaStream_t st);
cudaError_t launch_zfwd(const GridDev& g, const float* src, float2* S, cudaStream_t st);
cudaError_t launch_zinv(const GridDev& g, const float2* S, const float2* premul, float* out, cudaStream_t st);
cudaError_t launch_adjoint_source(const float* sim, const double* obs, int nt, int ns, int integrate, float* q,
                                  double* loss_part, double* loss_out, double* loss_acc, int accumulate,
                                  cudaStream_t st);
cudaError_t launch_finalize_grad(const float* grad, const uint8_t* gamma, long long n, float* acc, int accumulate,
                                 int* nonfinite, cudaStream_t st);
cudaError_t launch_check_finite(const float* a, long long n, int* flag, cudaStream_t st);
cudaError_t launch_scale(float* a, long long n, float s, cudaStream_t st);
cudaError_t launch_abs_prep(long long n, const AbsArgs& a, cudaStream_t st);
cudaError_t launch_abs_pressure(long long n, const AbsArgs& a, cudaStream_t st);
cudaError_t launch_correlate(long long n, const float* p_new, const float* c0sq, const Correlate& c, cudaStream_t st);
cudaError_t launch_gather(const float* p, const SparseGather& g, cudaStream_t st);
cudaError_t launch_rho0_elem(long long n, int mode, const Rho0Args& a, cudaStream_t st);
cudaError_t launch_stepper_sparse(float* const rho[3], int a_first, const int* idx, const float* val, int n, int mode,
                                  cudaStream_t st);
cudaError_t launch_pick(const float* f, const int* idx, int n, float* out, cudaStream_t st);
cudaError_t launch_ordered_mean(long long n, const float* gathered, int world, int slots, int batch, float* out,
                                cudaStream_t st);

// register-resident fast paths (passes.cu) for the compiled transform lengths
bool fast_pencil_supported(int L);
bool fast_rows_supported(int nz);
cudaError_t launch_pencil_fast(int axis, bool inv, const GridDev& g, const PencilJobs& jobs, cudaStream_t st);
cudaError_t launch_zvel_fast(const GridDev& g, float2* S[3], const float2* dz_plus, float* v[3], const Pml& pml,
                             const Coef r[3], cudaStream_t st);
cudaError_t launch_zrho_fast(const GridDev& g, const ZrhoArgs& a, cudaStream_t st);
bool use_generic_kernels();
bool chain_supported(const GridDev& g);
int chain_stats(unsigned long long out[4]);
cudaError_t launch_chain(const GridDev& g, const PencilJobs& ya, const PencilJobs& xb, const PencilJobs& yc, int* ctr,
                         int* err, cudaStream_t st);

}  // namespace ustfwi_dev
