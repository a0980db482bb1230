// Device engine: context (the device analogue of SpectralEngine + WaveSteppers,
// engine.hpp:17-386), the forward simulation (simulate.hpp:30-105) and the time-reversal
// c0 gradient (gradient.hpp:333-464) orchestrated as fused pass launches on one stream,
// and the device half of the C ABI (include/ustfwi_capi.h).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "host_setup.hpp"
#include "kernels.cuh"

using namespace ustfwi_dev;
using ustfwi_host::Error;
using ustfwi_host::fail;

namespace {

// NVTX ranges (SURVEY §5.1 tracing): header-only nvtx3, a no-op unless a tool attaches
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

#define CK(expr)                                                                               \
    do {                                                                                       \
        cudaError_t e_ = (expr);                                                               \
        if (e_ != cudaSuccess)                                                                 \
            fail(e_ == cudaErrorMemoryAllocation ? USTFWI_ERR_OOM : USTFWI_ERR_CUDA,           \
                 std::string(#expr) + ": " + cudaGetErrorString(e_));                          \
    } while (0)

enum { ST_NONE = 0, ST_PLUS = 1, ST_MINUS = 2, ST_SHIFT = 3, ST_SHIFTM = 4, ST_COUNT = 5 };
enum { KIND_Y = 0, KIND_X = 1, KIND_ZVEL = 2, KIND_ZRHO = 3, KIND_AUX = 4, KIND_CHAIN = 5 };

struct Sim {
    float* p = nullptr;
    float* v[3] = {};
    float* rho[3] = {};
    float2* S[3] = {};
    bool pml_off = false;   // StepperOptions::pml_enabled == false (engine.hpp:171,202-213)
    int* chain_ctr = nullptr;  // claim / completion counters of this simulation's chain kernel
    int pgrid = 0;             // persistent pencil grid of this simulation's passes (0: default)
};

// WaveStepper options and counters of the step-level C ABI (engine.hpp:170-177,344-346)
struct StepperState {
    bool init = false;
    float abs_sign = 1.f;
    bool dispersion = true;
    int step_index = 0;
};

// Device image of a SourceSet: unique positions (sorted) + CSR of contributions.
struct InjectSet {
    int n_unique = 0;
    std::vector<int> h_pos;            // unique positions
    std::vector<size_t> h_order;       // contribution order of the CSR arrays (stable sort by position)
    std::vector<size_t> h_src_pos;     // the positions / offsets / lengths the set was built from
    std::vector<int> h_off, h_len;
    size_t h_total = 0;
    int* pos = nullptr;
    int* csr = nullptr;
    int* off = nullptr;
    int* len = nullptr;
    int* stride = nullptr;
    int* delay = nullptr;
    float* w = nullptr;
    float* sig = nullptr;              // owned signal table (sources) or borrowed (adjoint q)
    float* scale = nullptr;
    int* blk8 = nullptr;               // per 8-row block offsets into pos
    SparseInject view(const float* sig_override = nullptr) const {
        SparseInject s;
        s.n_unique = n_unique;
        s.pos = pos;
        s.csr = csr;
        s.off = off;
        s.len = len;
        s.stride = stride;
        s.delay = delay;
        s.w = w;
        s.sig = sig_override ? sig_override : sig;
        s.scale = scale;
        s.blk8 = blk8;
        return s;
    }
};

// NCCL, resolved lazily with dlopen so the library has no link-time NCCL dependency
// (and shares whichever libnccl.so.2 the process already loaded, e.g. torch's).
struct NcclApi {
    void* h = nullptr;
    int (*get_unique_id)(void*) = nullptr;
    int (*comm_init_rank)(void**, int, const void*, int) = nullptr;  // ncclUniqueId passed by value (128 B)
    int (*all_gather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
    int (*comm_destroy)(void*) = nullptr;
    const char* (*error_string)(int) = nullptr;
};
struct NcclUniqueId {
    char internal[128];
};

NcclApi& nccl() {
    static NcclApi api;
    if (!api.h) {
        // the NCCL a process already uses (e.g. torch's, loaded first) wins through the soname;
        // otherwise USTFWI_NCCL_LIB (set by the Python layer to the pip NCCL that torch links,
        // so that a later `import torch` finds the NCCL version it was built against), else
        // the system libnccl.so.2
        api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        const char* path = std::getenv("USTFWI_NCCL_LIB");
        if (!api.h && path && *path) api.h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
        if (!api.h) api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!api.h) fail(USTFWI_ERR_NCCL, std::string("cannot load libnccl.so.2: ") + dlerror());
        api.get_unique_id = reinterpret_cast<int (*)(void*)>(dlsym(api.h, "ncclGetUniqueId"));
        api.all_gather = reinterpret_cast<int (*)(const void*, void*, size_t, int, void*, cudaStream_t)>(
            dlsym(api.h, "ncclAllGather"));
        api.comm_destroy = reinterpret_cast<int (*)(void*)>(dlsym(api.h, "ncclCommDestroy"));
        api.error_string = reinterpret_cast<const char* (*)(int)>(dlsym(api.h, "ncclGetErrorString"));
        if (!api.get_unique_id || !api.all_gather || !api.comm_destroy)
            fail(USTFWI_ERR_NCCL, "libnccl.so.2 lacks the expected symbols");
    }
    return api;
}

}  // namespace

struct ustfwi_gpu_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t stream2 = nullptr;   // time-reversal replay stream of the pair loop
    // SM-partitioned pair loop (USTFWI_GREEN): adjoint / replay streams of two
    // green contexts with disjoint SM sets
    cudaStream_t gstream[2] = {};
    CUgreenCtx gctx[2] = {};
    int gsm[2] = {};
    cudaEvent_t ev_gjoin = nullptr;
    cudaEvent_t ev_adj[2] = {}, ev_rep[2] = {}, ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_lag[8] = {};       // pair-loop phase shift (USTFWI_PAIR_LAG)
    float* adj_p2 = nullptr;          // second adjoint pressure buffer (pair loop)
    uint64_t launches = 0;
    ustfwi_grid grid{};
    int ndim = 3;
    int off_axis = 0;   // 3 - ndim: padded axis of reference axis 0
    GridDev g{};
    std::vector<void*> allocs;
    float* pinned = nullptr;          // N-float pinned host staging (medium upload, gradient download)
    float* pinned_stage() {
        if (!pinned) {
            void* p = nullptr;
            if (cudaMallocHost(&p, static_cast<size_t>(g.N) * sizeof(float)) != cudaSuccess)
                fail(USTFWI_ERR_CUDA, "pinned host staging allocation failed");
            pinned = static_cast<float*>(p);
        }
        return pinned;
    }

    float2* dmul[3][ST_COUNT] = {};  // per padded axis: none / plus / minus / shift +1/2 / shift -1/2 tables
    float* pml_reg[3] = {};
    float* pml_stag[3] = {};
    float* pml_one[3] = {};   // all-ones profiles (PML disabled)
    StepperState stp[2];
    float* stp_scratch = nullptr;   // pressure output of a density-only step
    int* stp_idx = nullptr;         // staging of the sparse step-level calls
    float* stp_val = nullptr;
    size_t stp_cap = 0;

    // medium
    bool has_medium = false;
    float* c0sq = nullptr;
    Coef dtrho0{};
    Coef dtr_stag[3]{};
    float* dtr_fields = nullptr;   // 4 fields when rho0 is not uniform
    uint8_t* gamma = nullptr;
    std::vector<uint8_t> gamma_host;
    std::vector<double> c0_host;

    Sim sim[2];
    // absorbing media (engine.hpp:233-246; gradient.hpp:63-74): coefficient fields and
    // per-stepper scratch, allocated only when alpha0 != 0
    bool absorbing = false;
    bool dispersion = false;       // y != 2 (engine.hpp:191)
    bool grad_dispersion = true;   // GradientOptions::dispersion_enabled (adjoint + replay)
    bool disp_active = false;      // dispersion term of the stepper currently running
    double y_pow = 1.5;
    float* abs_coef = nullptr;     // tau0, eta (2 fields)
    float* tau0 = nullptr;
    float* eta = nullptr;
    std::vector<double> alpha0_host;
    std::vector<double> rho0_host;  // GradientParam::rho0 (GradientAccumulator, gradient.hpp:117-128)
    Coef rho0c{};
    float* rho0_field = nullptr;
    // gradient parameter (GradientParam: 0 c0, 2 alpha0, 3 y) and the accumulator's extra
    // terms (gradient.hpp:56-142): weight fields wa1, wa2, wa1l, wa2l and the replay rings
    int grad_param = 0;
    struct AccPlan {
        bool ddot = true, a1 = false, a2 = false, a1l = false, a2l = false, rho0 = false;
        bool extra() const { return a1 || a2 || a1l || a2l || rho0 || !ddot; }
    } plan;
    float* acc_mem = nullptr;      // 4 weight fields + 12 ring fields
    float* wa[4] = {};
    float* a1lring[3] = {};
    float* a2lring[3] = {};
    struct AbsScratch {
        float* du[3] = {};
        float* ain = nullptr;
        float* aout = nullptr;
        float* aout2 = nullptr;
        float* sum = nullptr;
    } abs_s[2];
    float* abs_mem = nullptr;
    float* a1ring[3] = {};
    float* a2ring[3] = {};
    float* ring[3] = {};
    float* grad = nullptr;
    float* acc = nullptr;
    double* loss = nullptr;       // [0] last loss, [1] accumulated loss
    int* flags = nullptr;         // [0] diverged step (INT_MAX = ok), [1] nonfinite grad, [2] nonfinite data

    // sources / sensors / data
    InjectSet src, adj;
    std::vector<size_t> src_pos_host;
    int n_sens = 0;
    std::vector<size_t> sens_pos_host;
    int* sens_pos = nullptr;   // sorted
    int* sens_idx = nullptr;
    int* sens_blk8 = nullptr;
    float* data = nullptr;     // [nt][ns]
    double* obs = nullptr;     // [nt][ns]
    float* q = nullptr;        // [nt][ns]
    double* loss_part = nullptr;
    bool obs_ready = false;

    // shell
    int shell_thickness = 0;
    std::vector<size_t> shell_host;
    int* shell_pos = nullptr;
    int* shell_blk8 = nullptr;
    float* trace = nullptr;
    size_t trace_elems = 0;

    void* comm = nullptr;
    int nranks = 1, rank = 0;
    // CUDA graph of the gradient's device work, valid while nothing was re-bound (epoch)
    uint64_t epoch = 1;
    struct GraphKey {
        uint64_t epoch = 0;
        int thickness = 0;
        bool accumulate = false;
        bool operator==(const GraphKey& o) const {
            return epoch == o.epoch && thickness == o.thickness && accumulate == o.accumulate;
        }
    };
    GraphKey grad_key{}, seen_key{};
    cudaGraphExec_t grad_graph = nullptr;
    uint64_t grad_graph_launches = 0;
    void drop_graph() {
        if (grad_graph) cudaGraphExecDestroy(grad_graph);
        grad_graph = nullptr;
    }
    void touch() {
        ++epoch;
        drop_graph();
    }
    // mini-batch slots (ustfwi_gpu_run_gradient_slot / ustfwi_gpu_batch_mean): per-realization
    // masked gradients and losses of this rank, and the all-gathered copy of every rank's
    int n_slots = 0;
    float* slot_grad = nullptr;     // [n_slots][N]
    double* slot_loss = nullptr;    // [n_slots]
    float* gather_grad = nullptr;   // [nranks][n_slots][N]
    double* gather_loss = nullptr;  // [nranks][n_slots]

    // per-launch-class CUDA-event timing (ustfwi_gpu_set_profiling / ustfwi_gpu_kernel_stats)
    struct Pending {
        cudaEvent_t a, b;
        int kind;
        double bytes;
    };
    bool profiling = false;
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> event_pool;
    double prof_ms[USTFWI_KERNEL_KINDS] = {};
    double prof_bytes[USTFWI_KERNEL_KINDS] = {};
    uint64_t prof_n[USTFWI_KERNEL_KINDS] = {};

    cudaEvent_t get_event() {
        if (event_pool.empty()) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            return e;
        }
        cudaEvent_t e = event_pool.back();
        event_pool.pop_back();
        return e;
    }
    template <class F>
    void launch(int kind, double bytes, F&& f, cudaStream_t st) {
        if (!profiling) {
            count(f());
            return;
        }
        Pending pd{get_event(), get_event(), kind, bytes};
        CK(cudaEventRecord(pd.a, st));
        count(f());
        CK(cudaEventRecord(pd.b, st));
        pending.push_back(pd);
        if (pending.size() > 4096) resolve_profile();
    }
    void resolve_profile() {
        for (auto& pd : pending) {
            CK(cudaEventSynchronize(pd.b));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, pd.a, pd.b));
            prof_ms[pd.kind] += ms;
            prof_bytes[pd.kind] += pd.bytes;
            prof_n[pd.kind] += 1;
            event_pool.push_back(pd.a);
            event_pool.push_back(pd.b);
        }
        pending.clear();
    }

    template <class T>
    T* alloc(size_t count) {
        void* p = nullptr;
        CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
        allocs.push_back(p);
        return static_cast<T*>(p);
    }
    void release(void* p) {
        if (!p) return;
        auto it = std::find(allocs.begin(), allocs.end(), p);
        if (it != allocs.end()) {
            cudaFree(p);
            allocs.erase(it);
        }
    }
    template <class T>
    T* upload(const std::vector<T>& h) {
        T* d = alloc<T>(h.size());
        if (!h.empty()) CK(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, stream));
        return d;
    }
    void count(cudaError_t e) {
        if (e != cudaSuccess) fail(USTFWI_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
        ++launches;
    }
};

namespace {

using Ctx = ustfwi_gpu_ctx;

FftPlan make_plan(Ctx& c, int L) {
    FftPlan p{};
    p.L = L;
    int m = L;
    auto take = [&](int r) {
        while (m % r == 0 && p.nstages < kMaxStages) {
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
    for (int f = 11; m > 1 && p.nstages < kMaxStages; f += 2) take(f);
    if (m != 1) fail(USTFWI_ERR_INVALID, "transform length " + std::to_string(L) + " has too many factors");
    std::vector<float2> tw(static_cast<size_t>(L));
    for (int k = 0; k < L; ++k) {
        const double a = -2.0 * M_PI * static_cast<double>(k) / static_cast<double>(L);
        tw[static_cast<size_t>(k)] = make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
    }
    p.tw = c.upload(tw);
    return p;
}

long long rows_of(const Ctx& c) { return c.g.rows; }

std::vector<float> to_f32(const double* p, size_t n) {
    std::vector<float> out(n);
    for (size_t i = 0; i < n; ++i) out[i] = static_cast<float>(p[i]);
    return out;
}


void reset_sim(Ctx& c, Sim& s, bool with_p) {
    const size_t nb = static_cast<size_t>(c.g.N) * sizeof(float);
    const size_t sb = static_cast<size_t>(rows_of(c)) * c.g.nzp * sizeof(float2);
    for (int a = 0; a < 3; ++a) {
        CK(cudaMemsetAsync(s.v[a], 0, nb, c.stream));
        CK(cudaMemsetAsync(s.rho[a], 0, nb, c.stream));
    }
    CK(cudaMemsetAsync(s.S[0], 0, sb, c.stream));
    if (with_p && s.p) CK(cudaMemsetAsync(s.p, 0, nb, c.stream));
}

struct StepIO {
    SparseInject inj{};
    SparseEnforce enf{};
    SparseGather sens{};
    SparseGather shell{};
    Correlate corr{};
    int step_n = 0;
    int check_step = 0;
    float* p_out = nullptr;
    bool density_only = false;            // stop after the density update (WaveStepper API)
    // pair-loop phase shift (USTFWI_PAIR_LAG): the leader records lag_rec[k] after its k-th
    // pass of the step, the follower waits for lag_wait[k] before its k-th pass
    cudaEvent_t* lag_rec = nullptr;
    cudaEvent_t* lag_wait = nullptr;
    int lag_off = 0;                      // ... for the leader's (k + lag_off)-th pass
    cudaEvent_t wait_before_z = nullptr;  // cross-stream dependency of the pressure kernel
    // absorbing media
    float abs_sign = 1.f;                 // absorption_sign (-1 in the time-reversal replay)
};

// out = F^-1 { |k|^e F{in} } (SpectralEngine::apply_multiplier with power_multiplier(e),
// engine.hpp:88-94,123-126), through the sim's S1 scratch spectrum.
void apply_kpow(Ctx& c, Sim& s, const float* in, double e, float* out, cudaStream_t st, int kind = 2) {
    c.count(launch_zfwd(c.g, in, s.S[1], st));
    PencilJobs j{};
    j.buf[0] = s.S[1];
    j.n = 1;
    j.job[0] = {0, 0, nullptr, 0, 0.f};
    c.count(launch_pencil(1, false, c.g, j, st));
    j.job[0] = {0, 0, nullptr, kind, static_cast<float>(e)};
    c.count(launch_pencil(0, false, c.g, j, st));
    j.job[0] = {0, 0, nullptr, 0, 0.f};
    c.count(launch_pencil(1, true, c.g, j, st));
    c.count(launch_zinv(c.g, s.S[1], nullptr, out, st));
}

int sim_index(const Ctx& c, const Sim& s) { return &s == &c.sim[1] ? 1 : 0; }

// Absorbing update_pressure (engine.hpp:327-343) after the density update and the sparse
// work of the z pass (which left the lossless p in scratch): p = c0^2 (sum rho + s tau aout)
// - c0^2 eta aout2, then the gathers and the Fy Fz p of the next step.
void absorbing_tail(Ctx& c, Sim& s, const StepIO& io, cudaStream_t st) {
    auto& sc = c.abs_s[sim_index(c, s)];
    const long long N = c.g.N;
    AbsArgs A{};
    for (int a = 0; a < 3; ++a) {
        A.rho[a] = s.rho[a];
        A.du[a] = sc.du[a];
    }
    A.dtrho0 = c.dtrho0;
    A.inv_dt = static_cast<float>(1.0 / c.grid.dt);
    A.sum = sc.sum;
    A.ain = sc.ain;
    c.count(launch_abs_prep(N, A, st));
    apply_kpow(c, s, sc.ain, c.y_pow - 2.0, sc.aout, st);
    if (c.disp_active) apply_kpow(c, s, sc.sum, c.y_pow - 1.0, sc.aout2, st);
    A.c0sq = c.c0sq;
    A.tau0 = c.tau0;
    A.eta = c.disp_active ? c.eta : nullptr;
    A.aout = sc.aout;
    A.aout2 = sc.aout2;
    A.sign = io.abs_sign;
    A.p_out = io.p_out;
    A.check_step = io.check_step;
    A.diverged = c.flags;
    c.count(launch_abs_pressure(N, A, st));
    c.count(launch_gather(io.p_out, io.sens, st));
    c.count(launch_gather(io.p_out, io.shell, st));
    c.count(launch_zfwd(c.g, io.p_out, s.S[0], st));  // entry invariant of the next step: S0 = Fz p
}

// USTFWI_CHAIN=1 enables the fused y-x-y chain kernel (experimental, off by default): on a
// B200 at config D it measured 1.49 ms per chain launch against 0.50 + 0.89 ms for the three
// separate launches of the two chains (ncu: L2 hit rate 34 %, 2.9 GB of DRAM traffic for
// chain 1 against a 0.95 GB model: two live 44 MB slabs do not stay resident)
int chain_mode() {
    static int m = -1;
    if (m < 0) {
        const char* e = std::getenv("USTFWI_CHAIN");
        m = e ? std::atoi(e) : 0;
    }
    return m;
}
bool chain_enabled(const Ctx& c) {
    return chain_mode() > 0 && !use_generic_kernels() && chain_supported(c.g) && c.sim[0].chain_ctr;
}

// One leapfrog step of a stepper: update_velocity_density (engine.hpp:270-292), sparse
// injection / shell enforcement, update_pressure (:318-347), gathers. Entry invariant: S0 holds
// Fz p (the previous step's pressure kernel, or an initial state). The y / x / y passes on
// either side of the velocity and density z passes form two "y-x-y chains":
//   chain 1: Fy(S0); Fx -> kappa D_x+ / kappa -> Fx^-1; Fy^-1 (D_y+ on one output)
//   chain 2: Fy(v_a spectra); Fx -> kappa D_x- / kappa -> Fx^-1; Fy^-1 (D_y- on v_y)
// run either as three pencil launches each or as one persistent chain kernel that walks
// kz-column slabs through the three passes with the slab's spectra resident in L2
// (launch_chain, USTFWI_CHAIN).
void run_step(Ctx& c, Sim& s, const StepIO& io, cudaStream_t st) {
    GridDev g = c.g;
    g.pgrid = s.pgrid;
    int pass_k = 0;
    auto before = [&]() {
        if (io.lag_wait && pass_k + io.lag_off < 8) CK(cudaStreamWaitEvent(st, io.lag_wait[pass_k + io.lag_off], 0));
    };
    auto after = [&]() {
        if (io.lag_rec) CK(cudaEventRecord(io.lag_rec[pass_k], st));
        ++pass_k;
    };
    const double SB = static_cast<double>(g.rows) * g.nzh * sizeof(float2);  // one half spectrum
    const double FB = static_cast<double>(g.N) * sizeof(float);               // one real field
    auto pencil = [&](int axis, bool inv, const PencilJobs& j) {
        int loads = 0;
        for (int q = 0; q < j.n; ++q)
            if (q == 0 || j.job[q].src != j.job[q - 1].src) ++loads;
        before();
        c.launch(axis == 0 ? KIND_X : KIND_Y, (loads + j.n) * SB, [&] { return launch_pencil(axis, inv, g, j, st); }, st);
        after();
    };
    // one y-x-y chain: fused when supported, else three launches
    auto chain = [&](const PencilJobs& ya, const PencilJobs& xb, const PencilJobs& yc, bool fuse) {
        if (fuse && chain_enabled(c)) {
            // algorithmic bytes of the fused chain: the first reads and the last writes only
            int la = 0;
            for (int q = 0; q < ya.n; ++q)
                if (q == 0 || ya.job[q].src != ya.job[q - 1].src) ++la;
            c.launch(KIND_CHAIN, (la + yc.n) * SB, [&] { return launch_chain(g, ya, xb, yc, s.chain_ctr, c.flags + 3, st); },
                     st);
        } else {
            pencil(1, false, ya);
            pencil(0, false, xb);
            pencil(1, true, yc);
        }
    };
    float* const* stag = s.pml_off ? c.pml_one : c.pml_stag;
    float* const* regp = s.pml_off ? c.pml_one : c.pml_reg;
    PencilJobs ya{}, xb{}, yc{};
    for (int f = 0; f < 3; ++f) ya.buf[f] = xb.buf[f] = yc.buf[f] = s.S[f];
    // chain 1: S0 <- Fy S0; X: S0 <- kappa D_x+ , S1 <- kappa; Y^-1: S0, S2 <- T_kappa, S1 <- D_y+ T_kappa
    ya.n = 1;
    ya.job[0] = {0, 0, nullptr, 0};
    xb.n = 2;
    xb.job[0] = {0, 0, c.dmul[0][ST_PLUS], 1};
    xb.job[1] = {0, 1, nullptr, 1};
    yc.n = 3;
    yc.job[0] = {0, 0, nullptr, 0};
    yc.job[1] = {1, 2, nullptr, 0};
    yc.job[2] = {1, 1, c.dmul[1][ST_PLUS], 0};
    // chain 1 fused only in mode 1 (its slab holds up to three fields)
    chain(ya, xb, yc, chain_mode() == 1);
    // Z: c2r (D_z+ on S2), velocity update, r2c of v
    Pml ps{{stag[0], stag[1], stag[2]}};
    const double coef_b = c.dtr_stag[0].field ? 3 * FB : 0.0;
    before();
    c.launch(KIND_ZVEL, 6 * SB + 6 * FB + coef_b,
             [&] { return launch_zvel(g, s.S, c.dmul[2][ST_PLUS], s.v, ps, c.dtr_stag, st); }, st);
    after();
    // chain 2: Fy of Fz v_a; X: kappa D_x-, kappa, kappa; Y^-1 (D_y- on S1)
    ya.n = 3;
    for (int f = 0; f < 3; ++f) ya.job[f] = {f, f, nullptr, 0};
    xb.n = 3;
    xb.job[0] = {0, 0, c.dmul[0][ST_MINUS], 1};
    xb.job[1] = {1, 1, nullptr, 1};
    xb.job[2] = {2, 2, nullptr, 1};
    yc.n = 3;
    yc.job[0] = {0, 0, nullptr, 0};
    yc.job[1] = {1, 1, c.dmul[1][ST_MINUS], 0};
    yc.job[2] = {2, 2, nullptr, 0};
    if (chain_enabled(c) && chain_mode() == 2) {
        // the three fields of chain 2 are independent through all three passes: one fused
        // single-field chain each keeps one 14.7 MB slab per field live in L2
        for (int f = 0; f < 3; ++f) {
            PencilJobs a1 = ya, b1 = xb, c1 = yc;
            a1.n = b1.n = c1.n = 1;
            a1.job[0] = ya.job[f];
            b1.job[0] = xb.job[f];
            c1.job[0] = yc.job[f];
            chain(a1, b1, c1, true);
        }
    } else {
        chain(ya, xb, yc, true);
    }
    // Z: c2r (D_z- on S2), density update, sparse ops, pressure, gathers, Fz p -> S0
    ZrhoArgs a{};
    for (int f = 0; f < 3; ++f) {
        a.S[f] = s.S[f];
        a.rho[f] = s.rho[f];
    }
    a.dz_minus = c.dmul[2][ST_MINUS];
    a.pml = Pml{{regp[0], regp[1], regp[2]}};
    a.dtrho0 = c.dtrho0;
    a.c0sq = c.c0sq;
    a.p_out = io.p_out;
    a.a_first = c.off_axis;
    a.step_n = io.step_n;
    a.inj = io.inj;
    a.enf = io.enf;
    a.sens = io.sens;
    a.shell = io.shell;
    a.corr = io.corr;
    a.check_step = io.check_step;
    a.diverged = c.flags;
    if (c.absorbing) {
        // the z pass updates the densities, applies the sparse work and keeps the raw
        // derivatives; pressure, gathers and correlation follow in absorbing_tail
        auto& sc = c.abs_s[sim_index(c, s)];
        for (int f = 0; f < 3; ++f) a.du_out[f] = sc.du[f];
        a.p_out = sc.aout;
        a.sens = SparseGather{};
        a.shell = SparseGather{};
        a.corr = Correlate{};
        a.check_step = 0;
    }
    // the fast path splits the step into the per-axis density update and the pressure
    // kernel, which re-reads the three split densities (+3F)
    const bool split = !use_generic_kernels() && fast_rows_supported(g.nz);
    const double zb = 4 * SB + (split ? 11 : 8) * FB + (c.dtrho0.field ? FB : 0.0) + (io.corr.grad ? 5 * FB : 0.0) -
                      (io.p_out ? 0.0 : FB);
    if (io.wait_before_z) CK(cudaStreamWaitEvent(st, io.wait_before_z, 0));
    before();
    c.launch(KIND_ZRHO, zb, [&] { return launch_zrho(g, a, true, st); }, st);
    after();
    if (split) ++c.launches;
    if (c.absorbing && !io.density_only) absorbing_tail(c, s, io, st);
}

// blk8[b] = index of the first sorted position >= b * 8 rows (b = 0 .. ceil(rows/8)): the
// sparse work of an 8-row-aligned row block is found with two loads instead of a search
int* upload_blk8(Ctx& c, const std::vector<int>& sorted_pos) {
    const long long rows = c.g.rows, nz = c.g.nz;
    const long long nb = (rows + 7) / 8;
    std::vector<int> off(static_cast<size_t>(nb + 1));
    size_t k = 0;
    for (long long b = 0; b <= nb; ++b) {
        const long long key = b * 8 * nz;
        while (k < sorted_pos.size() && sorted_pos[k] < key) ++k;
        off[static_cast<size_t>(b)] = static_cast<int>(k);
    }
    return c.upload(off);
}

// Build the device InjectSet for `n` contributions at flat positions pos[i].
void build_inject(Ctx& c, InjectSet& set, const std::vector<size_t>& pos, const std::vector<int>& off,
                  const std::vector<int>& len, const std::vector<int>& stride, const std::vector<int>& delay,
                  const std::vector<float>& w) {
    for (void* p : {(void*)set.pos, (void*)set.csr, (void*)set.off, (void*)set.len, (void*)set.stride,
                    (void*)set.delay, (void*)set.w, (void*)set.scale, (void*)set.blk8})
        c.release(p);
    const size_t n = pos.size();
    std::vector<size_t> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return pos[a] < pos[b]; });
    set.h_order = order;
    std::vector<int> upos, csr{0}, o, l, st, d;
    std::vector<float> ww;
    for (size_t k = 0; k < n; ++k) {
        const size_t i = order[k];
        if (upos.empty() || static_cast<size_t>(upos.back()) != pos[i]) {
            if (!upos.empty()) csr.push_back(static_cast<int>(o.size()));
            upos.push_back(static_cast<int>(pos[i]));
        }
        o.push_back(off[i]);
        l.push_back(len[i]);
        st.push_back(stride[i]);
        d.push_back(delay[i]);
        ww.push_back(w[i]);
    }
    if (!upos.empty()) csr.push_back(static_cast<int>(o.size()));
    set.n_unique = static_cast<int>(upos.size());
    set.h_pos = upos;
    set.pos = c.upload(upos);
    set.csr = c.upload(csr);
    set.off = c.upload(o);
    set.len = c.upload(l);
    set.stride = c.upload(st);
    set.delay = c.upload(d);
    set.w = c.upload(ww);
    set.scale = c.alloc<float>(upos.size());
    set.blk8 = upload_blk8(c, upos);
}

// inject_mass_source scale 2*dt/(ndim*dx*c0(x)) (engine.hpp:296-300), from the current medium.
void refresh_scales(Ctx& c, InjectSet& set) {
    std::vector<float> sc(set.h_pos.size());
    for (size_t u = 0; u < sc.size(); ++u) {
        const double c0 = c.c0_host[static_cast<size_t>(set.h_pos[u])];
        sc[u] = static_cast<float>(2.0 * c.grid.dt / (c.ndim * c.grid.dx[0] * std::sqrt(c0 * c0)));
    }
    if (!sc.empty())
        CK(cudaMemcpyAsync(set.scale, sc.data(), sc.size() * sizeof(float), cudaMemcpyHostToDevice, c.stream));
}

void require_medium(const Ctx& c) {
    if (!c.has_medium) fail(USTFWI_ERR_INVALID, "medium not set (ustfwi_gpu_set_medium)");
}

void ensure_data_buffers(Ctx& c) {
    if (c.data) return;
    const size_t n = static_cast<size_t>(c.grid.nt) * std::max(c.n_sens, 1);
    c.data = c.alloc<float>(n);
    c.obs = c.alloc<double>(n);
    c.q = c.alloc<float>(n);
    c.loss_part = c.alloc<double>(std::max(c.n_sens, 1));
}

// Buffers whose length follows nt (sensor data, observed data, adjoint source) and the
// adjoint-source injection set at the sensors (contribution s reads q[n*ns + s]); called when
// the sensors or the simulation length change (ustfwi_gpu_set_nt: the encoded duration
// T + tau of a delayed realization).
void rebind_time_buffers(Ctx& c) {
    c.touch();
    for (void* q : {(void*)c.data, (void*)c.obs, (void*)c.q, (void*)c.loss_part}) c.release(q);
    c.data = nullptr;
    c.obs_ready = false;
    ensure_data_buffers(c);
    const size_t ns = c.sens_pos_host.size();
    std::vector<int> off(ns), len(ns, c.grid.nt), stride(ns, std::max<int>(1, c.n_sens)), delay(ns, 0);
    std::iota(off.begin(), off.end(), 0);
    std::vector<float> w(ns, 1.f);
    build_inject(c, c.adj, c.sens_pos_host, off, len, stride, delay, w);
}

void prepare_shell(Ctx& c, int thickness) {
    if (c.gamma_host.empty()) fail(USTFWI_ERR_INVALID, "boundary recording requires a gamma mask");
    if (thickness != c.shell_thickness || !c.shell_pos) {
        c.touch();
        c.release(c.shell_pos);
        c.shell_pos = nullptr;
        std::vector<int> dims(c.grid.dims, c.grid.dims + c.grid.ndim);
        c.shell_host = ustfwi_host::shell_indices(c.gamma_host, dims, thickness);
        std::vector<int> sp(c.shell_host.begin(), c.shell_host.end());
        c.shell_pos = c.upload(sp);
        c.release(c.shell_blk8);
        c.shell_blk8 = upload_blk8(c, sp);
        c.shell_thickness = thickness;
    }
    const size_t need = c.shell_host.size() * static_cast<size_t>(c.grid.nt);
    if (need > c.trace_elems) {
        c.touch();
        c.release(c.trace);
        c.trace = c.alloc<float>(need);
        c.trace_elems = need;
    }
}

void clear_flags(Ctx& c) {
    const int init[4] = {INT_MAX, 0, 0, 0};
    CK(cudaMemcpyAsync(c.flags, init, sizeof(init), cudaMemcpyHostToDevice, c.stream));
}

void check_flags(Ctx& c, bool grad_phase) {
    int f[4];
    CK(cudaMemcpyAsync(f, c.flags, sizeof(f), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    c.resolve_profile();
    if (f[3]) fail(USTFWI_ERR_CUDA, "y-x-y chain kernel: a dependency wait timed out");
    if (f[0] != INT_MAX) fail(USTFWI_ERR_NUMERICAL, "pressure field diverged at step " + std::to_string(f[0]));
    if (f[2]) fail(USTFWI_ERR_NUMERICAL, "sensor data contains non-finite values");
    if (grad_phase && f[1]) fail(USTFWI_ERR_NUMERICAL, "gradient contains non-finite values");
}

// simulate_forward (simulate.hpp:76-103): nt steps of stepper 0 with the source set,
// sensor gather into c.data ([nt][ns]) and optional shell record into c.trace.
void forward_prep(Ctx& c, int thickness) {
    require_medium(c);
    ensure_data_buffers(c);
    if (thickness > 0) prepare_shell(c, thickness);
    refresh_scales(c, c.src);
}

// the launches of the forward simulation only (no host transfers: capturable)
void forward_steps(Ctx& c, int thickness) {
    c.disp_active = c.dispersion;  // simulate_forward: default StepperOptions
    Sim& s = c.sim[0];
    s.pml_off = false;
    reset_sim(c, s, true);
    const int nt = c.grid.nt;
    const int n_shell = thickness > 0 ? static_cast<int>(c.shell_host.size()) : 0;
    StepIO io;
    io.inj = c.src.view();
    io.sens = SparseGather{c.n_sens, c.sens_pos, c.sens_idx, nullptr, c.sens_blk8};
    io.shell = SparseGather{n_shell, c.shell_pos, nullptr, nullptr, c.shell_blk8};
    // the forward pressure is only gathered (in-kernel, from registers) and transformed into
    // the next step's S0: not stored, except on the absorbing path, whose tail re-reads it
    io.p_out = c.absorbing ? s.p : nullptr;
    for (int n = 0; n < nt; ++n) {
        io.step_n = n;
        io.sens.out = c.data + static_cast<size_t>(n) * c.n_sens;
        if (n_shell) io.shell.out = c.trace + static_cast<size_t>(n) * n_shell;
        io.check_step = ((n + 1) & 63) == 0 ? n + 1 : 0;
        run_step(c, s, io, c.stream);
    }
    if (c.n_sens > 0) c.count(launch_check_finite(c.data, static_cast<long long>(nt) * c.n_sens, c.flags + 2, c.stream));
}

void forward_sim(Ctx& c, int thickness) {
    NvtxRange r("ustfwi forward");
    forward_prep(c, thickness);
    forward_steps(c, thickness);
}

// GradientAccumulator (gradient.hpp:50-142) for the selected parameter: which terms, their
// weight fields (fp32, from the fp64 formulas) and the rings of |k|^y-type replay fields.
void prepare_accumulator(Ctx& c) {
    const bool disp = c.grad_dispersion && c.y_pow != 2.0;  // dispersion_on_ (gradient.hpp:56)
    Ctx::AccPlan pl;
    if (c.grad_param == 0) {
        pl.a1 = c.absorbing;
        pl.a2 = c.absorbing && disp;
    } else if (c.grad_param == 2) {
        pl.ddot = false;
        pl.a1 = true;
        pl.a2 = disp;
    } else if (c.grad_param == 3) {
        pl.ddot = false;
        pl.a1 = pl.a1l = true;
        pl.a2 = pl.a2l = disp;
    } else if (c.grad_param == 1) {
        // rho0 (gradient.hpp:117-128): the correlation of accumulate_rho0 only; no absorption terms
        pl.ddot = false;
        pl.rho0 = true;
    } else {
        fail(USTFWI_ERR_INVALID, "unknown gradient parameter");
    }
    if (!(pl.ddot == c.plan.ddot && pl.a1 == c.plan.a1 && pl.a2 == c.plan.a2 && pl.a1l == c.plan.a1l &&
          pl.a2l == c.plan.a2l && pl.rho0 == c.plan.rho0))
        c.touch();
    c.plan = pl;
    if (!pl.extra()) return;
    const size_t N = static_cast<size_t>(c.g.N);
    if (pl.rho0) {
        // rho0 as a coefficient (scalar when uniform) and 5 scratch fields in acc_mem
        if (!c.acc_mem) {
            c.acc_mem = c.alloc<float>(16 * N);
            c.touch();
        }
        bool uniform = true;
        for (size_t i = 1; i < N && uniform; ++i) uniform = c.rho0_host[i] == c.rho0_host[0];
        if (uniform) {
            c.rho0c = Coef{nullptr, static_cast<float>(c.rho0_host[0])};
        } else {
            if (!c.rho0_field) {
                c.rho0_field = c.alloc<float>(N);
                c.touch();
            }
            const auto h = to_f32(c.rho0_host.data(), N);
            CK(cudaMemcpyAsync(c.rho0_field, h.data(), N * sizeof(float), cudaMemcpyHostToDevice, c.stream));
            CK(cudaStreamSynchronize(c.stream));
            c.rho0c = Coef{c.rho0_field, 0.f};
        }
        return;
    }
    if (!c.acc_mem) {
        c.touch();
        c.acc_mem = c.alloc<float>(16 * N);
        for (int k = 0; k < 4; ++k) c.wa[k] = c.acc_mem + k * N;
        for (int r = 0; r < 3; ++r) {
            c.a1ring[r] = c.acc_mem + (4 + r) * N;
            c.a2ring[r] = c.acc_mem + (7 + r) * N;
            c.a1lring[r] = c.acc_mem + (10 + r) * N;
            c.a2lring[r] = c.acc_mem + (13 + r) * N;
        }
    }
    const double y = c.y_pow;
    const double tan_term = disp ? std::tan(M_PI * y / 2.0) : 0.0;
    const double np_of_db = 100.0 * (std::log(10.0) / 20.0) / std::pow(2.0 * M_PI * 1e6, y);  // db2neper(1, y)
    const double log_conv = std::log(2.0 * M_PI * 1e6);
    std::vector<float> h(4 * N, 0.f);
    for (size_t i = 0; i < N; ++i) {
        const double cc = c.c0_host[i];
        const double a_np = c.alpha0_host.empty() ? 0.0 : np_of_db * c.alpha0_host[i];
        double w1 = 0, w2 = 0, w1l = 0, w2l = 0;
        if (c.grad_param == 0) {  // gradient.hpp:63-73
            w1 = -2.0 * a_np * (y - 1.0) * std::pow(cc, y - 2.0);
            w2 = 2.0 * a_np * y * std::pow(cc, y - 1.0) * tan_term;
        } else if (c.grad_param == 2) {  // :76-88
            w1 = -2.0 * np_of_db * std::pow(cc, y - 1.0);
            w2 = 2.0 * np_of_db * std::pow(cc, y) * tan_term;
        } else {  // :90-116
            const double tau = -2.0 * a_np * std::pow(cc, y - 1.0);
            const double lc = std::log(cc) - log_conv;
            w1 = tau * lc;
            w1l = 0.5 * tau;
            if (disp) {
                const double sec = 1.0 / std::cos(M_PI * y / 2.0);
                const double eta = 2.0 * a_np * std::pow(cc, y) * tan_term;
                w2 = eta * lc + M_PI * a_np * std::pow(cc, y) * sec * sec;
                w2l = 0.5 * eta;
            }
        }
        h[i] = static_cast<float>(w1);
        h[N + i] = static_cast<float>(w2);
        h[2 * N + i] = static_cast<float>(w1l);
        h[3 * N + i] = static_cast<float>(w2l);
    }
    CK(cudaMemcpyAsync(c.acc_mem, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice, c.stream));
    CK(cudaStreamSynchronize(c.stream));
}

// out = F^-1[ T(k_pa) * (kappa(|k|) if kappa) * F[in] ] through the scratch spectrum s.S[1]:
// SpectralEngine::derivative (T = D_pa^{+-}, kappa on; engine.hpp:118-121) and half_shift
// (T = e^{+-i k dx/2}, kappa off; engine.hpp:131-137) on the device passes.
void spectral_apply(Ctx& c, Sim& s, const float* in, int pa, const float2* tab, int kappa, float* out, cudaStream_t st) {
    c.count(launch_zfwd(c.g, in, s.S[1], st));
    PencilJobs j{};
    j.buf[0] = s.S[1];
    j.n = 1;
    j.job[0] = {0, 0, nullptr, 0, 0.f};
    c.count(launch_pencil(1, false, c.g, j, st));
    j.job[0] = {0, 0, pa == 0 ? tab : nullptr, kappa, 0.f};
    c.count(launch_pencil(0, false, c.g, j, st));
    j.job[0] = {0, 0, pa == 1 ? tab : nullptr, 0, 0.f};
    c.count(launch_pencil(1, true, c.g, j, st));
    c.count(launch_zinv(c.g, s.S[1], pa == 2 ? tab : nullptr, out, st));
}

// GradientAccumulator::accumulate_rho0 (gradient.hpp:213-239) for the replay pressure p (the
// window centre) and the adjoint pressure q: rq = rho0 q; per axis a: dp = D+_a p,
// drq = D+_a rq, grad += dt q D-_a(dp / rho~_a) + dt half_shift_{-1}(dp drq / rho~_a^2).
void rho0_correlate(Ctx& c, Sim& s, const float* p, const float* q, cudaStream_t st) {
    const long long N = c.g.N;
    const size_t n = static_cast<size_t>(N);
    float* rq = c.acc_mem;
    float* dp = c.acc_mem + n;
    float* drq = c.acc_mem + 2 * n;
    float* tmp = c.acc_mem + 3 * n;
    float* out = c.acc_mem + 4 * n;
    Rho0Args A{};
    A.rho0 = c.rho0c;
    A.dt = static_cast<float>(c.grid.dt);
    A.inv_dt = static_cast<float>(1.0 / c.grid.dt);
    A.q = q;
    A.grad = c.grad;
    A.dp = dp;
    A.drq = drq;
    A.out = out;
    A.tmp = rq;
    c.count(launch_rho0_elem(N, 0, A, st));
    A.tmp = tmp;
    for (int pa = c.off_axis; pa < 3; ++pa) {
        A.dtr = c.dtr_stag[pa];
        spectral_apply(c, s, p, pa, c.dmul[pa][ST_PLUS], 1, dp, st);
        spectral_apply(c, s, rq, pa, c.dmul[pa][ST_PLUS], 1, drq, st);
        c.count(launch_rho0_elem(N, 1, A, st));
        spectral_apply(c, s, tmp, pa, c.dmul[pa][ST_MINUS], 1, out, st);
        c.count(launch_rho0_elem(N, 2, A, st));
        c.count(launch_rho0_elem(N, 3, A, st));
        spectral_apply(c, s, tmp, pa, c.dmul[pa][ST_SHIFTM], 0, out, st);
        c.count(launch_rho0_elem(N, 4, A, st));
    }
}

// GradientAccumulator::push (gradient.hpp:147-160): the multiplier fields of the newest
// replay pressure ring[slot].
void acc_push(Ctx& c, Sim& s, int slot, cudaStream_t st) {
    if (!c.plan.extra()) return;
    const float* p = c.ring[slot];
    if (c.plan.a1) apply_kpow(c, s, p, c.y_pow, c.a1ring[slot], st);
    if (c.plan.a2) apply_kpow(c, s, p, c.y_pow + 1.0, c.a2ring[slot], st);
    if (c.plan.a1l) apply_kpow(c, s, p, c.y_pow, c.a1lring[slot], st, 3);
    if (c.plan.a2l) apply_kpow(c, s, p, c.y_pow + 1.0, c.a2lring[slot], st, 3);
}

// GradientAccumulator::accumulate (gradient.hpp:166-203) with newer = slot nw, mid, older.
void acc_correlate(Ctx& c, Correlate cr, int nw, int mid, int old, cudaStream_t st) {
    if (c.plan.rho0) {
        rho0_correlate(c, c.sim[1], c.ring[mid], cr.q_adj, st);
        return;
    }
    cr.use_ddot = c.plan.ddot ? 1 : 0;
    cr.dt = static_cast<float>(c.grid.dt);
    if (c.plan.a1) {
        cr.a1_new = c.a1ring[nw];
        cr.a1_old = c.a1ring[old];
        cr.wa1 = c.wa[0];
    }
    if (c.plan.a2) {
        cr.a2_mid = c.a2ring[mid];
        cr.wa2 = c.wa[1];
    }
    if (c.plan.a1l) {
        cr.a1l_new = c.a1lring[nw];
        cr.a1l_old = c.a1lring[old];
        cr.wa1l = c.wa[2];
    }
    if (c.plan.a2l) {
        cr.a2l_mid = c.a2lring[mid];
        cr.wa2l = c.wa[3];
    }
    c.count(launch_correlate(c.g.N, c.ring[nw], c.c0sq, cr, st));
}

// SM partition of the pair loop (USTFWI_GREEN=k, default 48 % of the SMs): the adjoint stream gets a green
// context of k SMs (rounded by the driver to its granularity of 8), the replay the rest, so
// the two streams' passes run side by side on disjoint SMs instead of both persistent grids
// filling the whole device in turn.
template <class F>
F driver_fn(const char* name, bool required = true) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || fn == nullptr) {
        if (required) fail(USTFWI_ERR_CUDA, std::string("driver entry point ") + name + " unavailable");
        return nullptr;
    }
    return reinterpret_cast<F>(fn);
}

void green_partition(Ctx& c, int want, int prio_a, int prio_b) {
    auto get_res = driver_fn<CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType)>("cuDeviceGetDevResource");
    auto split = driver_fn<CUresult (*)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned,
                                        unsigned)>("cuDevSmResourceSplitByCount");
    auto gen = driver_fn<CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned)>("cuDevResourceGenerateDesc");
    auto create = driver_fn<CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned)>("cuGreenCtxCreate");
    auto mkstream = driver_fn<CUresult (*)(CUstream*, CUgreenCtx, unsigned, int)>("cuGreenCtxStreamCreate");
    CUdevResource all{}, parts[1]{}, rest{};
    if (get_res(static_cast<CUdevice>(c.device), &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS)
        fail(USTFWI_ERR_CUDA, "cuDeviceGetDevResource failed");
    unsigned n = 1;
    if (split(parts, &n, &all, &rest, 0, static_cast<unsigned>(std::abs(want))) != CUDA_SUCCESS || n != 1)
        fail(USTFWI_ERR_CUDA, "cuDevSmResourceSplitByCount failed");
    // want > 0: the adjoint (which correlates) gets the k SMs, the replay the rest;
    // want < 0: the replay gets |k|, the adjoint the rest
    CUdevResource* res[2] = {&parts[0], &rest};
    if (want < 0) std::swap(res[0], res[1]);
    const int prio[2] = {prio_a, prio_b};
    for (int k = 0; k < 2; ++k) {
        CUdevResourceDesc d{};
        if (gen(&d, res[k], 1) != CUDA_SUCCESS) fail(USTFWI_ERR_CUDA, "cuDevResourceGenerateDesc failed");
        if (create(&c.gctx[k], d, static_cast<CUdevice>(c.device), CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS)
            fail(USTFWI_ERR_CUDA, "cuGreenCtxCreate failed");
        CUstream st{};
        if (mkstream(&st, c.gctx[k], CU_STREAM_NON_BLOCKING, prio[k]) != CUDA_SUCCESS)
            fail(USTFWI_ERR_CUDA, "cuGreenCtxStreamCreate failed");
        c.gstream[k] = reinterpret_cast<cudaStream_t>(st);
        c.gsm[k] = static_cast<int>(res[k]->sm.smCount);
    }
    CK(cudaEventCreateWithFlags(&c.ev_gjoin, cudaEventDisableTiming));
    if (std::getenv("USTFWI_VERBOSE"))
        std::fprintf(stderr, "[ustfwi] green partition: adjoint %d SMs, replay %d SMs\n", c.gsm[0], c.gsm[1]);
}

void drop_green(Ctx& c) {
    for (int k = 0; k < 2; ++k) {
        if (c.gstream[k]) {
            cudaStreamSynchronize(c.gstream[k]);
            cudaStreamDestroy(c.gstream[k]);
            c.gstream[k] = nullptr;
        }
    }
    if (c.ev_gjoin) cudaEventDestroy(c.ev_gjoin);
    c.ev_gjoin = nullptr;
    static auto destroy = driver_fn<CUresult (*)(CUgreenCtx)>("cuGreenCtxDestroy", false);
    for (int k = 0; k < 2; ++k) {
        if (c.gctx[k] && destroy) destroy(c.gctx[k]);
        c.gctx[k] = nullptr;
        c.gsm[k] = 0;
    }
}

// compute_gradient, TR branch (gradient.hpp:359-462), GradientParam c0 / alpha0 / y.
// The device work of one TR gradient after the host-side preparation: forward with shell
// record, adjoint source, interleaved adjoint + replay with the correlation into c.grad.
// Only stream operations (kernel launches, memsets, events): captured as one CUDA graph.
void gradient_core(Ctx& c, int thickness, bool accumulate) {
    const int nt = c.grid.nt, ns = c.n_sens, last = nt - 1;
    {
        NvtxRange r("ustfwi forward (shell record)");
        forward_steps(c, thickness);
    }
    NvtxRange r("ustfwi adjoint + time-reversal replay");
    c.disp_active = c.dispersion && c.grad_dispersion;  // adjoint + replay steppers (gradient.hpp:381,424-426)
    // adjoint source: reverse, Kahan loss, integrate (gradient.hpp:264-289,378-379)
    c.count(launch_adjoint_source(c.data, c.obs, nt, ns, 1, c.q, c.loss_part, c.loss, c.loss + 1,
                                  accumulate ? 1 : 0, c.stream));
    c.launches += 1;  // loss reduction kernel
    Sim& adj = c.sim[0];
    Sim& rep = c.sim[1];
    rep.pml_off = false;
    reset_sim(c, adj, true);
    reset_sim(c, rep, false);
    CK(cudaMemsetAsync(c.grad, 0, static_cast<size_t>(c.g.N) * sizeof(float), c.stream));
    const int n_shell = static_cast<int>(c.shell_host.size());
    auto shell_row = [&](int m) { return c.trace + static_cast<size_t>(m) * n_shell; };

    // The adjoint and the time-reversal replay run on two streams (two SM partitions when
    // green contexts are available), so their passes overlap; the only coupling is the
    // correlation. Plain c0 gradient: inside the adjoint's pressure kernel, from a 4-slot ring
    // of replay pressures (see the fused loop below). Otherwise: after each replay step, from
    // the adjoint pressure, double buffered (adjoint step n writes P[n&1] once replay step
    // n-2, its last reader, is done). Profiling serialises both on one stream so per-launch
    // event times stay meaningful.
    const bool dual = !c.profiling && c.stream2 != nullptr;
    const bool green = dual && c.gstream[0] != nullptr;
    cudaStream_t sa = c.stream, sb = dual ? c.stream2 : c.stream;
    float* P[2] = {adj.p, c.adj_p2};
    if (dual) {
        CK(cudaEventRecord(c.ev_fork, sa));
        if (green) {
            // the adjoint and the replay each on their own SM partition (persistent pencil
            // grids sized to the partition); the caller's stream joins both at the end
            sa = c.gstream[0];
            sb = c.gstream[1];
            CK(cudaStreamWaitEvent(sa, c.ev_fork, 0));
            adj.pgrid = 2 * c.gsm[0];
            rep.pgrid = 2 * c.gsm[1];
        }
        CK(cudaStreamWaitEvent(sb, c.ev_fork, 0));
    }

    // replay initial value: enforce g[last], refresh p (gradient.hpp:435-437)
    {
        ZrhoArgs a{};
        for (int f = 0; f < 3; ++f) {
            a.S[f] = rep.S[f];
            a.rho[f] = rep.rho[f];
        }
        a.pml = Pml{{c.pml_reg[0], c.pml_reg[1], c.pml_reg[2]}};
        a.dtrho0 = c.dtrho0;
        a.c0sq = c.c0sq;
        a.p_out = c.ring[0];
        a.a_first = c.off_axis;
        a.enf = SparseEnforce{n_shell, c.shell_pos, shell_row(last), static_cast<float>(c.ndim), c.shell_blk8};
        a.diverged = c.flags;
        c.count(launch_zrho(c.g, a, false, sb));
        acc_push(c, rep, 0, sb);  // GradientAccumulator::push of the initial value (gradient.hpp:147-160)
    }
    // look-ahead step (gradient.hpp:438-441)
    StepIO rio;
    rio.enf = SparseEnforce{n_shell, c.shell_pos, shell_row(last - 1), static_cast<float>(c.ndim), c.shell_blk8};
    rio.p_out = c.ring[1];
    rio.check_step = 0;
    rio.abs_sign = -1.f;  // replay stepper: absorption_sign = -1 (gradient.hpp:429-431)
    run_step(c, rep, rio, sb);
    acc_push(c, rep, 1, sb);

    // experiments (off by default): USTFWI_PAIR_GRID=k runs the pair loop's pencil passes on
    // persistent grids of k CTAs per SM; USTFWI_PAIR_LAG=1 makes the replay's k-th pass of a
    // step wait for the adjoint's k-th pass, so an x pass of one stream meets a y pass of the
    // other (complementary: issue bound vs HBM bound)
    static const int pair_grid = [] {
        const char* e = std::getenv("USTFWI_PAIR_GRID");
        return e ? std::atoi(e) : 0;
    }();
    static const int pair_lag = [] {
        const char* e = std::getenv("USTFWI_PAIR_LAG");
        return e ? std::atoi(e) : 0;
    }();
    if (dual && !green && pair_grid > 0) {
        int nsm = 0;
        CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c.device));
        adj.pgrid = rep.pgrid = pair_grid * nsm;
    }
    StepIO aio;
    aio.inj = c.adj.view(c.q);
    if (dual && pair_lag) {
        aio.lag_rec = c.ev_lag;
        rio.lag_wait = c.ev_lag;
        rio.lag_off = pair_lag - 1;  // USTFWI_PAIR_LAG=m: the replay trails by m-1 passes more
    }
    const float inv_dt = static_cast<float>(1.0 / c.grid.dt);
    const bool fused = !c.plan.extra() && !c.absorbing;
    if (fused) {
        // plain c0 gradient: the correlation of pair step n runs inside the ADJOINT's pressure
        // kernel, which holds q_n in registers and reads the replay's p_{n+1}, p_n, p_{n-1}
        // from a 4-slot ring, so the adjoint pressure is never stored or re-read (6 instead of
        // 7 fields of correlation traffic per pair step). The replay leads: adjoint step n waits
        // for replay step n; replay step n overwrites the ring slot last read by adjoint step
        // n-2 and waits for it.
        float* R4[4] = {c.ring[0], c.ring[1], c.ring[2], c.adj_p2};
        if (aio.lag_rec) {  // USTFWI_PAIR_LAG: here the replay leads
            std::swap(aio.lag_rec, rio.lag_rec);
            std::swap(aio.lag_wait, rio.lag_wait);
            std::swap(aio.lag_off, rio.lag_off);
        }
        for (int n = 1; n <= last - 1; ++n) {
            rio.enf.vals = shell_row(last - n - 1);
            rio.p_out = R4[(n + 1) & 3];
            rio.corr = Correlate{};
            rio.check_step = ((n + 1) & 63) == 0 ? n + 1 : 0;
            rio.wait_before_z = (dual && n >= 3) ? c.ev_adj[n & 1] : nullptr;  // adjoint n-2 done
            run_step(c, rep, rio, sb);
            if (dual) CK(cudaEventRecord(c.ev_rep[n & 1], sb));
            aio.step_n = n;
            aio.check_step = (n & 63) == 0 ? n : 0;
            aio.p_out = nullptr;
            Correlate corr{R4[n & 3], R4[(n - 1) & 3], nullptr, c.grad, inv_dt};
            corr.p_new = R4[(n + 1) & 3];
            aio.corr = corr;
            aio.wait_before_z = dual ? c.ev_rep[n & 1] : nullptr;  // replay step n done
            run_step(c, adj, aio, sa);
            if (dual) CK(cudaEventRecord(c.ev_adj[n & 1], sa));
        }
        if (dual) {
            CK(cudaEventRecord(c.ev_join, sb));
            CK(cudaStreamWaitEvent(sa, c.ev_join, 0));
            if (green) {
                CK(cudaEventRecord(c.ev_gjoin, sa));
                CK(cudaStreamWaitEvent(c.stream, c.ev_gjoin, 0));
            }
        }
        adj.pgrid = rep.pgrid = 0;
        return;
    }
    for (int n = 1; n <= last - 1; ++n) {
        aio.step_n = n;
        aio.check_step = (n & 63) == 0 ? n : 0;
        aio.p_out = P[n & 1];
        aio.wait_before_z = (dual && n >= 3) ? c.ev_rep[n & 1] : nullptr;  // replay n-2 done with P[n&1]
        run_step(c, adj, aio, sa);
        if (dual) CK(cudaEventRecord(c.ev_adj[n & 1], sa));
        rio.enf.vals = shell_row(last - n - 1);
        rio.p_out = c.ring[(n + 1) % 3];
        // absorption terms, alpha0 / y / rho0: the correlation after the replay step, from the rings
        const Correlate corr{c.ring[n % 3], c.ring[(n - 1) % 3], P[n & 1], c.grad, inv_dt};
        rio.corr = Correlate{};
        rio.check_step = ((n + 1) & 63) == 0 ? n + 1 : 0;
        rio.wait_before_z = dual ? c.ev_adj[n & 1] : nullptr;                 // adjoint step n done
        run_step(c, rep, rio, sb);
        acc_push(c, rep, (n + 1) % 3, sb);
        acc_correlate(c, corr, (n + 1) % 3, n % 3, (n - 1) % 3, sb);
        if (dual) CK(cudaEventRecord(c.ev_rep[n & 1], sb));
    }
    if (dual) {
        CK(cudaEventRecord(c.ev_join, sb));
        CK(cudaStreamWaitEvent(sa, c.ev_join, 0));
        if (green) {
            CK(cudaEventRecord(c.ev_gjoin, sa));
            CK(cudaStreamWaitEvent(c.stream, c.ev_gjoin, 0));
        }
    }
    adj.pgrid = rep.pgrid = 0;
}

bool use_graphs() {
    static int on = -1;
    if (on < 0) {
        const char* e = std::getenv("USTFWI_GRAPH");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

// compute_gradient, TR branch (gradient.hpp:359-462). The device part (gradient_core, ~9
// launches per simulation step = 105k launches at config D) is captured into a CUDA graph on
// the second call with the same configuration (the first call runs eagerly and warms every
// kernel's attributes) and replayed afterwards; any set_* call invalidates it (epoch).
void gradient_tr(Ctx& c, int thickness, bool accumulate, int slot = -1) {
    NvtxRange range("ustfwi gradient_tr");
    require_medium(c);
    if (c.gamma_host.empty()) fail(USTFWI_ERR_INVALID, "gradient computation requires a gamma mask");
    if (!c.obs_ready) fail(USTFWI_ERR_INVALID, "observed data not uploaded");
    if (thickness < 1) fail(USTFWI_ERR_INVALID, "shell thickness must be >= 1");
    forward_prep(c, thickness);
    prepare_accumulator(c);
    refresh_scales(c, c.adj);
    const Ctx::GraphKey key{c.epoch, thickness, accumulate};
    if (!use_graphs() || c.profiling) {
        gradient_core(c, thickness, accumulate);
    } else if (c.grad_graph && c.grad_key == key) {
        CK(cudaGraphLaunch(c.grad_graph, c.stream));
        c.launches += c.grad_graph_launches;
    } else if (c.seen_key == key) {
        c.drop_graph();
        const uint64_t l0 = c.launches;
        CK(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
        try {
            gradient_core(c, thickness, accumulate);
        } catch (...) {
            cudaGraph_t g = nullptr;
            cudaStreamEndCapture(c.stream, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        cudaGraph_t g = nullptr;
        CK(cudaStreamEndCapture(c.stream, &g));
        const cudaError_t e = cudaGraphInstantiate(&c.grad_graph, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) {
            c.grad_graph = nullptr;
            fail(USTFWI_ERR_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
        }
        c.grad_key = key;
        c.grad_graph_launches = c.launches - l0;
        CK(cudaGraphLaunch(c.grad_graph, c.stream));
    } else {
        gradient_core(c, thickness, accumulate);
        c.seen_key = key;
    }
    if (slot >= 0) {
        // mini-batch slot: the masked gradient and this realization's loss
        float* dst = c.slot_grad + static_cast<size_t>(slot) * static_cast<size_t>(c.g.N);
        c.count(launch_finalize_grad(c.grad, c.gamma, c.g.N, dst, 0, c.flags + 1, c.stream));
        CK(cudaMemcpyAsync(c.slot_loss + slot, c.loss, sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
        return;
    }
    c.count(launch_finalize_grad(c.grad, c.gamma, c.g.N, c.acc, accumulate ? 1 : 0, c.flags + 1, c.stream));
}

// Absorption coefficients (WaveStepper constructor engine.hpp:233-246 and the c0 branch
// of GradientAccumulator gradient.hpp:63-74), fp32 fields; dispersion on unless y == 2
// (engine.hpp:191). alpha0 == nullptr: lossless, scratch released.
void set_absorption(Ctx& c, const double* alpha0, double y, const double* c0) {
    c.release(c.abs_coef);
    c.release(c.abs_mem);
    c.abs_coef = c.abs_mem = nullptr;
    c.absorbing = alpha0 != nullptr;
    c.y_pow = y;
    c.dispersion = c.absorbing && y != 2.0;
    if (!c.absorbing) return;
    const size_t N = static_cast<size_t>(c.g.N);
    std::vector<float> h(2 * N);
    const double tan_term = c.dispersion ? std::tan(M_PI * y / 2.0) : 0.0;
    const double np_per_db = 100.0 * (std::log(10.0) / 20.0) / std::pow(2.0 * M_PI * 1e6, y);  // db2neper
    for (size_t i = 0; i < N; ++i) {
        const double a = np_per_db * alpha0[i];
        const double cc = c0[i];
        h[i] = static_cast<float>(-2.0 * a * std::pow(cc, y - 1.0));
        h[N + i] = static_cast<float>(2.0 * a * std::pow(cc, y) * tan_term);
    }
    c.abs_coef = c.alloc<float>(2 * N);
    CK(cudaMemcpyAsync(c.abs_coef, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice, c.stream));
    c.tau0 = c.abs_coef;
    c.eta = c.abs_coef + N;
    // per stepper: du x3, ain, aout, aout2, sum
    c.abs_mem = c.alloc<float>(14 * N);
    float* m = c.abs_mem;
    for (int k = 0; k < 2; ++k) {
        auto& sc = c.abs_s[k];
        for (int a = 0; a < 3; ++a) sc.du[a] = m + (k * 7 + a) * N;
        sc.ain = m + (k * 7 + 3) * N;
        sc.aout = m + (k * 7 + 4) * N;
        sc.aout2 = m + (k * 7 + 5) * N;
        sc.sum = m + (k * 7 + 6) * N;
    }
    CK(cudaMemsetAsync(c.abs_mem, 0, 14 * N * sizeof(float), c.stream));
}

template <class Fn>
int guarded(Ctx* c, Fn&& fn) {
    try {
        if (c) CK(cudaSetDevice(c->device));
        fn();
        return USTFWI_OK;
    } catch (const Error& e) {
        ustfwi_host::set_last_error(e.msg);
        return e.code;
    } catch (const std::bad_alloc&) {
        ustfwi_host::set_last_error("host allocation failed");
        return USTFWI_ERR_OOM;
    } catch (const std::exception& e) {
        ustfwi_host::set_last_error(e.what());
        return USTFWI_ERR_INVALID;
    }
}

// fourier_shift(rho0, axis, +1/2) (spectral.hpp:94-112) on the device: the multiplier
// depends on k_axis only, applied inside the pass of that axis.
void staggered_shift(Ctx& c, const float* src, int axis, float* out) {
    Sim& s = c.sim[1];
    c.count(launch_zfwd(c.g, src, s.S[0], c.stream));
    PencilJobs j{};
    for (int f = 0; f < 3; ++f) j.buf[f] = s.S[f];
    j.n = 1;
    j.job[0] = {0, 0, nullptr, 0};
    c.count(launch_pencil(1, false, c.g, j, c.stream));
    j.job[0] = {0, 0, axis == 0 ? c.dmul[0][ST_SHIFT] : nullptr, 0};
    // X pass always multiplies through a job; kappa off
    c.count(launch_pencil(0, false, c.g, j, c.stream));
    j.job[0] = {0, 0, axis == 1 ? c.dmul[1][ST_SHIFT] : nullptr, 0};
    c.count(launch_pencil(1, true, c.g, j, c.stream));
    c.count(launch_zinv(c.g, s.S[0], axis == 2 ? c.dmul[2][ST_SHIFT] : nullptr, out, c.stream));
}

}  // namespace

// =====================================================================================
// C ABI: device engine
// =====================================================================================
extern "C" {

int ustfwi_gpu_create(int device, const ustfwi_grid* grid, ustfwi_gpu_ctx** out) {
    *out = nullptr;
    auto* c = new (std::nothrow) Ctx;
    if (!c) return USTFWI_ERR_OOM;
    const int rc = guarded(nullptr, [&] {
        if (!grid) fail(USTFWI_ERR_INVALID, "null grid");
        ustfwi_host::validate_grid(*grid);
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            fail(USTFWI_ERR_CUDA, "no CUDA device available (the engine has no CPU fallback)");
        if (device < 0 || device >= ndev) fail(USTFWI_ERR_INVALID, "device index out of range");
        c->device = device;
        CK(cudaSetDevice(device));
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10)
            fail(USTFWI_ERR_CUDA, std::string("device ") + prop.name + " is not sm_100-class (built for sm_100a)");
        // The adjoint stream (the one the replay waits on before its pressure kernel) gets
        // the higher priority, so its CTAs are dispatched first whenever both streams have
        // a pass pending: D200 1.734 -> 1.711 s / gradient on one box (replay first: 1.716).
        // USTFWI_STREAM_PRIO=0 restores equal priorities, =2 favours the replay.
        int prio_a = 0, prio_b = 0;
        {
            const char* e = std::getenv("USTFWI_STREAM_PRIO");
            const char mode = e ? e[0] : '1';
            int lo = 0, hi = 0;
            CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            if (mode == '1') prio_a = hi;
            if (mode == '2') prio_b = hi;
        }
        CK(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_a));
        CK(cudaStreamCreateWithPriority(&c->stream2, cudaStreamNonBlocking, prio_b));
        {
            // SM-partitioned pair loop: the adjoint (which also correlates) on 48 % of the SMs,
            // rounded up to the driver's granularity of 8 (72 of 148), the replay (which leads,
            // and records) on the rest; measured on D200: adjoint 64 / 72 / 80 / 88 SMs ->
            // see DESIGN.md section 7. USTFWI_GREEN=0 disables it, =k asks for k adjoint SMs.
            const char* e = std::getenv("USTFWI_GREEN");
            const bool forced = e != nullptr;
            const int want = forced ? std::atoi(e) : (prop.multiProcessorCount * 48 + 99) / 100;
            if (want != 0 && std::abs(want) < prop.multiProcessorCount) {
                try {
                    green_partition(*c, want, prio_a, prio_b);
                } catch (const std::exception&) {
                    if (forced) throw;
                    drop_green(*c);  // e.g. no green-context support: shared-SM streams
                }
            }
        }
        for (int k = 0; k < 2; ++k) {
            CK(cudaEventCreateWithFlags(&c->ev_adj[k], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c->ev_rep[k], cudaEventDisableTiming));
        }
        CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
        for (auto& e : c->ev_lag) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
        c->grid = *grid;
        c->ndim = grid->ndim;
        c->off_axis = 3 - grid->ndim;
        int d3[3] = {1, 1, 1};
        double dx3[3] = {grid->dx[0], grid->dx[0], grid->dx[0]};
        for (int a = 0; a < grid->ndim; ++a) {
            d3[c->off_axis + a] = grid->dims[a];
            dx3[c->off_axis + a] = grid->dx[a];
        }
        GridDev& g = c->g;
        g.nx = d3[0];
        g.ny = d3[1];
        g.nz = d3[2];
        g.nzh = g.nz / 2 + 1;
        g.nzp = (g.nzh + 3) & ~3;
        g.rows = static_cast<long long>(g.nx) * g.ny;
        g.x0 = 0;
        g.xn = g.nx;
        g.N = g.rows * g.nz;
        if (g.N >= (1LL << 31)) fail(USTFWI_ERR_INVALID, "grid larger than 2^31 points is not supported");
        g.px = make_plan(*c, g.nx);
        g.py = make_plan(*c, g.ny);
        g.pzh = make_plan(*c, g.nz / 2);
        std::vector<float2> twr(static_cast<size_t>(g.nzh));
        for (int k = 0; k < g.nzh; ++k) {
            const double a = -2.0 * M_PI * k / g.nz;
            twr[static_cast<size_t>(k)] = make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
        }
        g.tw_rfft = c->upload(twr);
        g.half_cdt = static_cast<float>(0.5 * grid->c_ref * grid->dt);
        g.inv_n = static_cast<float>(1.0 / static_cast<double>(g.N));
        // per-axis wavenumbers, stagger/shift factors (engine.hpp:46-78) and PML (grid.hpp:153-178)
        float* kdev[3];
        ustfwi_grid g3{};
        g3.ndim = 3;
        for (int a = 0; a < 3; ++a) {
            g3.dims[a] = d3[a];
            g3.dx[a] = dx3[a];
            g3.pml_size[a] = 0;
        }
        for (int a = 0; a < grid->ndim; ++a) g3.pml_size[c->off_axis + a] = grid->pml_size[a];
        g3.dt = grid->dt;
        g3.nt = grid->nt;
        g3.c_ref = grid->c_ref;
        for (int a = 0; a < 3; ++a) {
            const int n = d3[a];
            const auto k = ustfwi_host::wavenumbers(n, dx3[a]);
            std::vector<float> kf(k.begin(), k.end());
            kdev[a] = c->upload(kf);
            std::vector<float2> tab[ST_COUNT];
            for (auto& t : tab) t.resize(static_cast<size_t>(n));
            for (int m = 0; m < n; ++m) {
                const double km = k[static_cast<size_t>(m)];
                const double h = 0.5 * km * dx3[a];
                const bool nyq = (m == n / 2);
                // i*k, i*k*e^{+ikdx/2}, i*k*e^{-ikdx/2}, e^{+ikdx/2}; real part only on the Nyquist bin
                tab[ST_NONE][m] = nyq ? make_float2(0.f, 0.f) : make_float2(0.f, static_cast<float>(km));
                tab[ST_PLUS][m] = make_float2(static_cast<float>(-km * std::sin(h)),
                                              nyq ? 0.f : static_cast<float>(km * std::cos(h)));
                tab[ST_MINUS][m] = make_float2(static_cast<float>(km * std::sin(h)),
                                               nyq ? 0.f : static_cast<float>(km * std::cos(h)));
                tab[ST_SHIFT][m] = make_float2(static_cast<float>(std::cos(h)), nyq ? 0.f : static_cast<float>(std::sin(h)));
                // half_shift direction -1: conj(e^{ikdx/2}), real part on the Nyquist bin (engine.hpp:66-73)
                tab[ST_SHIFTM][m] = make_float2(static_cast<float>(std::cos(h)), nyq ? 0.f : static_cast<float>(-std::sin(h)));
            }
            for (int s = 0; s < ST_COUNT; ++s) c->dmul[a][s] = c->upload(tab[s]);
            std::vector<double> r, st;
            if (g3.pml_size[a] > 0) {
                ustfwi_host::pml_profiles(g3, a, 2.0, r, st);
            } else {
                r.assign(static_cast<size_t>(n), 1.0);
                st.assign(static_cast<size_t>(n), 1.0);
            }
            c->pml_reg[a] = c->upload(std::vector<float>(r.begin(), r.end()));
            c->pml_stag[a] = c->upload(std::vector<float>(st.begin(), st.end()));
            c->pml_one[a] = c->upload(std::vector<float>(static_cast<size_t>(n), 1.f));
        }
        g.kx = kdev[0];
        g.ky = kdev[1];
        g.kz = kdev[2];
        // state of two steppers, the replay ring, gradient and accumulator
        const size_t N = static_cast<size_t>(g.N);
        const size_t NS = static_cast<size_t>(g.rows) * g.nzp;
        const int ntx8 = (g.nzh + 7) / 8;
        for (int s = 0; s < 2; ++s) {
            c->sim[s].chain_ctr = c->alloc<int>(static_cast<size_t>(1 + 3 * ntx8));
            for (int a = 0; a < 3; ++a) {
                c->sim[s].v[a] = c->alloc<float>(N);
                c->sim[s].rho[a] = c->alloc<float>(N);
                c->sim[s].S[a] = c->alloc<float2>(NS);
            }
        }
        c->sim[0].p = c->alloc<float>(N);
        c->adj_p2 = c->alloc<float>(N);
        for (int r = 0; r < 3; ++r) c->ring[r] = c->alloc<float>(N);
        c->grad = c->alloc<float>(N);
        c->acc = c->alloc<float>(N);
        c->c0sq = c->alloc<float>(N);
        c->gamma = c->alloc<uint8_t>(N);
        c->loss = c->alloc<double>(2);
        c->flags = c->alloc<int>(4);
        CK(cudaMemsetAsync(c->acc, 0, N * sizeof(float), c->stream));
        CK(cudaMemsetAsync(c->loss, 0, 2 * sizeof(double), c->stream));
        clear_flags(*c);
        CK(cudaStreamSynchronize(c->stream));
    });
    if (rc != USTFWI_OK) {
        ustfwi_gpu_destroy(c);
        return rc;
    }
    *out = c;
    return USTFWI_OK;
}

void ustfwi_gpu_destroy(ustfwi_gpu_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    c->drop_graph();
    if (c->comm) {
        try {
            nccl().comm_destroy(c->comm);
        } catch (...) {
        }
    }
    for (auto& pd : c->pending) {
        c->event_pool.push_back(pd.a);
        c->event_pool.push_back(pd.b);
    }
    for (cudaEvent_t e : c->event_pool) cudaEventDestroy(e);
    for (cudaEvent_t e : {c->ev_adj[0], c->ev_adj[1], c->ev_rep[0], c->ev_rep[1], c->ev_fork, c->ev_join})
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ev_lag)
        if (e) cudaEventDestroy(e);
    for (void* p : c->allocs) cudaFree(p);
    if (c->pinned) cudaFreeHost(c->pinned);
    drop_green(*c);
    if (c->stream2) {
        cudaStreamSynchronize(c->stream2);
        cudaStreamDestroy(c->stream2);
    }
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

int ustfwi_gpu_set_medium(ustfwi_gpu_ctx* c, const double* c0, const double* rho0, const double* alpha0, double y,
                          const uint8_t* gamma, double c0_min, double c0_max) {
    return guarded(c, [&] {
        // what a captured gradient graph bakes in from the medium: the density coefficients
        // (scalars when rho0 is uniform), the absorption plan, the exponent, the shell. A new
        // medium that leaves all of them unchanged (an optimizer iterate: new c0 values in
        // place) keeps the graph; anything else invalidates it
        const bool prev_plain = c->has_medium && !c->absorbing && c->dtr_fields == nullptr;
        const Coef prev_dtrho0 = c->dtrho0;
        const Coef prev_stag[3] = {c->dtr_stag[0], c->dtr_stag[1], c->dtr_stag[2]};
        const double prev_y = c->y_pow;
        struct Invalidate {  // on every exit (errors included) unless the graph is known valid
            Ctx* c;
            bool keep = false;
            ~Invalidate() {
                if (!keep) c->touch();
            }
        } inval{c};
        const size_t N = static_cast<size_t>(c->g.N);
        if (!c0 || !rho0) fail(USTFWI_ERR_INVALID, "medium fields must match the grid");
        // Medium::validate (medium.hpp:41-57); chunked over host threads, the first failing
        // check in index order decides the message
        struct Part {
            double cmax = 0.0;
            size_t bad_c0 = SIZE_MAX, bad_rho = SIZE_MAX, bad_a0 = SIZE_MAX;
            bool absorbing = false;
        };
        const size_t hw = std::max<size_t>(1, std::thread::hardware_concurrency());
        std::vector<Part> parts(hw);
        std::atomic<size_t> slot{0};
        ustfwi_host::parallel_chunks(N, [&](size_t b, size_t e) {
            Part p;
            for (size_t i = b; i < e; ++i) {
                if ((c0[i] < c0_min || c0[i] > c0_max) && p.bad_c0 == SIZE_MAX) p.bad_c0 = i;
                if (!(rho0[i] > 0.0) && p.bad_rho == SIZE_MAX) p.bad_rho = i;
                if (alpha0) {
                    if (alpha0[i] < 0.0 && p.bad_a0 == SIZE_MAX) p.bad_a0 = i;
                    if (alpha0[i] != 0.0) p.absorbing = true;
                }
                p.cmax = std::max(p.cmax, c0[i]);
            }
            parts[slot.fetch_add(1) % hw] = p;
        });
        bool absorbing = false;
        double cmax = 0.0;
        size_t bad_c0 = SIZE_MAX, bad_rho = SIZE_MAX, bad_a0 = SIZE_MAX;
        for (const Part& p : parts) {
            cmax = std::max(cmax, p.cmax);
            absorbing = absorbing || p.absorbing;
            bad_c0 = std::min(bad_c0, p.bad_c0);
            bad_rho = std::min(bad_rho, p.bad_rho);
            bad_a0 = std::min(bad_a0, p.bad_a0);
        }
        const size_t first = std::min({bad_c0, bad_rho, bad_a0});
        if (first != SIZE_MAX) {
            if (first == bad_c0) fail(USTFWI_ERR_INVALID, "c0 outside configured bounds");
            if (first == bad_rho) fail(USTFWI_ERR_INVALID, "rho0 must be positive");
            fail(USTFWI_ERR_INVALID, "alpha0 must be non-negative");
        }
        if (y <= 1.0 || y >= 3.0) fail(USTFWI_ERR_INVALID, "power-law exponent must be in (1,3)");
        // WaveStepper constructor checks (engine.hpp:188-197)
        for (int a = 1; a < c->grid.ndim; ++a)
            if (c->grid.dx[a] != c->grid.dx[0])
                fail(USTFWI_ERR_INVALID, "wave stepper requires uniform grid spacing");
        double min_dx = c->grid.dx[0];
        for (int a = 1; a < c->grid.ndim; ++a) min_dx = std::min(min_dx, c->grid.dx[a]);
        if (cmax * c->grid.dt / min_dx > 2.0 / M_PI * (1.0 + 1e-12))
            fail(USTFWI_ERR_NUMERICAL, "CFL violation: dt exceeds 2/pi * dx / c_max");
        const double dt = c->grid.dt;
        c->c0_host.resize(N);
        c->rho0_host.resize(N);
        CK(cudaStreamSynchronize(c->stream));  // the pinned staging buffer may be in flight
        float* c2 = c->pinned_stage();
        std::atomic<bool> uniform_ok{true};
        ustfwi_host::parallel_chunks(N, [&](size_t b, size_t e) {
            std::memcpy(c->c0_host.data() + b, c0 + b, (e - b) * sizeof(double));
            std::memcpy(c->rho0_host.data() + b, rho0 + b, (e - b) * sizeof(double));
            bool u = true;
            for (size_t i = b; i < e; ++i) {
                c2[i] = static_cast<float>(c0[i] * c0[i]);
                u = u && rho0[i] == rho0[0];
            }
            if (!u) uniform_ok = false;
        });
        CK(cudaMemcpyAsync(c->c0sq, c2, N * sizeof(float), cudaMemcpyHostToDevice, c->stream));
        const bool uniform_rho = uniform_ok;
        c->release(c->dtr_fields);
        c->dtr_fields = nullptr;
        if (uniform_rho) {
            // fourier_shift of a constant is the constant: scalar coefficients
            c->dtrho0 = Coef{nullptr, static_cast<float>(dt * rho0[0])};
            for (int a = 0; a < 3; ++a) c->dtr_stag[a] = Coef{nullptr, static_cast<float>(dt / rho0[0])};
        } else {
            c->dtr_fields = c->alloc<float>(4 * N);
            std::vector<float> f(N);
            for (size_t i = 0; i < N; ++i) f[i] = static_cast<float>(dt * rho0[i]);
            CK(cudaMemcpyAsync(c->dtr_fields, f.data(), N * sizeof(float), cudaMemcpyHostToDevice, c->stream));
            c->dtrho0 = Coef{c->dtr_fields, 0.f};
            std::vector<float> r(N);
            for (size_t i = 0; i < N; ++i) r[i] = static_cast<float>(rho0[i]);
            float* rdev = c->ring[0];  // scratch
            CK(cudaMemcpyAsync(rdev, r.data(), N * sizeof(float), cudaMemcpyHostToDevice, c->stream));
            std::vector<float> shifted(N);
            for (int a = 0; a < 3; ++a) {
                float* dst = c->dtr_fields + (a + 1) * N;
                if (a < c->off_axis) {
                    std::vector<float> cst(N);
                    for (size_t i = 0; i < N; ++i) cst[i] = static_cast<float>(dt / rho0[i]);
                    CK(cudaMemcpyAsync(dst, cst.data(), N * sizeof(float), cudaMemcpyHostToDevice, c->stream));
                    CK(cudaStreamSynchronize(c->stream));
                } else {
                    staggered_shift(*c, rdev, a, c->ring[1]);
                    CK(cudaMemcpyAsync(shifted.data(), c->ring[1], N * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
                    CK(cudaStreamSynchronize(c->stream));
                    for (size_t i = 0; i < N; ++i) {
                        if (!(shifted[i] > 0.f)) fail(USTFWI_ERR_INVALID, "staggered density must stay positive");
                        shifted[i] = static_cast<float>(dt / static_cast<double>(shifted[i]));
                    }
                    CK(cudaMemcpyAsync(dst, shifted.data(), N * sizeof(float), cudaMemcpyHostToDevice, c->stream));
                    CK(cudaStreamSynchronize(c->stream));
                }
                c->dtr_stag[a] = Coef{dst, 0.f};
            }
        }
        set_absorption(*c, absorbing ? alpha0 : nullptr, y, c0);
        if (alpha0) c->alpha0_host.assign(alpha0, alpha0 + N);
        else c->alpha0_host.clear();
        // the boundary shell (shell_indices, medium.hpp:168-178) depends on gamma only: keep
        // it when the new mask equals the bound one
        const bool same_gamma = gamma && c->gamma_host.size() == N && std::memcmp(c->gamma_host.data(), gamma, N) == 0;
        if (!same_gamma) {
            c->gamma_host.clear();
            if (gamma) {
                c->gamma_host.assign(gamma, gamma + N);
                CK(cudaMemcpyAsync(c->gamma, c->gamma_host.data(), N, cudaMemcpyHostToDevice, c->stream));
            }
            c->release(c->shell_pos);
            c->shell_pos = nullptr;
            c->shell_thickness = 0;
        }
        c->has_medium = true;
        CK(cudaStreamSynchronize(c->stream));
        const bool same_coef = uniform_rho && prev_dtrho0.scalar == c->dtrho0.scalar &&
                               prev_stag[0].scalar == c->dtr_stag[0].scalar &&
                               prev_stag[1].scalar == c->dtr_stag[1].scalar && prev_stag[2].scalar == c->dtr_stag[2].scalar;
        inval.keep = prev_plain && !absorbing && same_coef && prev_y == y && same_gamma &&
                     c->grad_param == USTFWI_PARAM_C0;
    });
}

int ustfwi_gpu_set_gradient_options(ustfwi_gpu_ctx* c, int dispersion_enabled) {
    return guarded(c, [&] {
        if (c->grad_dispersion != (dispersion_enabled != 0)) c->touch();
        c->grad_dispersion = dispersion_enabled != 0;
    });
}

int ustfwi_gpu_set_gradient_param(ustfwi_gpu_ctx* c, int param) {
    return guarded(c, [&] {
        if (param < 0 || param > 3) fail(USTFWI_ERR_INVALID, "unknown gradient parameter");
        if (param != c->grad_param) c->touch();
        c->grad_param = param;
    });
}

int ustfwi_gpu_set_sources(ustfwi_gpu_ctx* c, size_t n_src, const size_t* pos, const size_t* sig_off,
                           const double* sig, const double* weights, const int32_t* delay_steps) {
    return guarded(c, [&] {
        const size_t N = static_cast<size_t>(c->g.N);
        std::vector<size_t> p(pos, pos + n_src);
        for (size_t v : p)
            if (v >= N) fail(USTFWI_ERR_INVALID, "source position outside grid");
        const size_t total = n_src ? sig_off[n_src] : 0;
        if (total >= (1ull << 31)) fail(USTFWI_ERR_INVALID, "signal table too large");
        std::vector<int> off(n_src), len(n_src), stride(n_src, 1), delay(n_src, 0);
        std::vector<float> w(n_src, 1.f);
        for (size_t i = 0; i < n_src; ++i) {
            off[i] = static_cast<int>(sig_off[i]);
            len[i] = static_cast<int>(sig_off[i + 1] - sig_off[i]);
            if (weights) w[i] = static_cast<float>(weights[i]);
            if (delay_steps) delay[i] = delay_steps[i];
        }
        InjectSet& set = c->src;
        if (set.sig && n_src > 0 && p == set.h_src_pos && off == set.h_off && len == set.h_len && total == set.h_total) {
            // same emitters, new realization (weights / delays / signal values): update the
            // existing device tables in place, so a captured gradient graph stays valid
            std::vector<int> d(n_src);
            std::vector<float> ww(n_src);
            for (size_t k = 0; k < n_src; ++k) {
                d[k] = delay[set.h_order[k]];
                ww[k] = w[set.h_order[k]];
            }
            const auto sf = to_f32(sig, total);
            CK(cudaMemcpyAsync(set.delay, d.data(), n_src * sizeof(int), cudaMemcpyHostToDevice, c->stream));
            CK(cudaMemcpyAsync(set.w, ww.data(), n_src * sizeof(float), cudaMemcpyHostToDevice, c->stream));
            CK(cudaMemcpyAsync(set.sig, sf.data(), total * sizeof(float), cudaMemcpyHostToDevice, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            return;
        }
        c->touch();
        c->release(set.sig);
        set.sig = c->upload(to_f32(sig, total));
        build_inject(*c, set, p, off, len, stride, delay, w);
        set.h_src_pos = p;
        set.h_off = off;
        set.h_len = len;
        set.h_total = total;
        c->src_pos_host = p;
        CK(cudaStreamSynchronize(c->stream));
    });
}

int ustfwi_gpu_set_sensors(ustfwi_gpu_ctx* c, size_t n_sensors, const size_t* pos) {
    return guarded(c, [&] {
        const size_t N = static_cast<size_t>(c->g.N);
        std::vector<size_t> p(pos, pos + n_sensors);
        for (size_t v : p)
            if (v >= N) fail(USTFWI_ERR_INVALID, "sensor position outside grid");
        if (c->sens_pos && c->data && c->n_sens == static_cast<int>(n_sensors) && c->sens_pos_host == p)
            return;  // the bound sensor array: nothing to rebind (a captured graph stays valid)
        c->n_sens = static_cast<int>(n_sensors);
        c->sens_pos_host = p;
        std::vector<int> order(n_sensors);
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return p[static_cast<size_t>(a)] < p[static_cast<size_t>(b)]; });
        std::vector<int> sp(n_sensors), si(n_sensors);
        for (size_t k = 0; k < n_sensors; ++k) {
            sp[k] = static_cast<int>(p[static_cast<size_t>(order[k])]);
            si[k] = order[k];
        }
        for (void* q : {(void*)c->sens_pos, (void*)c->sens_idx}) c->release(q);
        c->sens_pos = c->upload(sp);
        c->sens_idx = c->upload(si);
        c->release(c->sens_blk8);
        c->sens_blk8 = upload_blk8(*c, sp);
        rebind_time_buffers(*c);
        CK(cudaStreamSynchronize(c->stream));
    });
}

int ustfwi_gpu_set_nt(ustfwi_gpu_ctx* c, int nt) {
    return guarded(c, [&] {
        if (nt < 3) fail(USTFWI_ERR_INVALID, "nt must be >= 3");
        if (nt == c->grid.nt) return;
        c->grid.nt = nt;
        rebind_time_buffers(*c);
        CK(cudaStreamSynchronize(c->stream));
    });
}

int ustfwi_gpu_forward(ustfwi_gpu_ctx* c, int boundary_thickness, double* data_out, double* trace_out,
                       size_t* n_shell_out) {
    return guarded(c, [&] {
        clear_flags(*c);
        forward_sim(*c, boundary_thickness);
        check_flags(*c, false);
        const int nt = c->grid.nt, ns = c->n_sens;
        if (data_out && ns > 0) {
            std::vector<float> h(static_cast<size_t>(nt) * ns);
            CK(cudaMemcpy(h.data(), c->data, h.size() * sizeof(float), cudaMemcpyDeviceToHost));
            for (int s = 0; s < ns; ++s)
                for (int n = 0; n < nt; ++n)
                    data_out[static_cast<size_t>(s) * nt + n] = h[static_cast<size_t>(n) * ns + s];
        }
        const size_t nsh = boundary_thickness > 0 ? c->shell_host.size() : 0;
        if (n_shell_out) *n_shell_out = nsh;
        if (trace_out && nsh > 0) {
            std::vector<float> h(nsh * static_cast<size_t>(nt));
            CK(cudaMemcpy(h.data(), c->trace, h.size() * sizeof(float), cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < h.size(); ++i) trace_out[i] = h[i];
        }
    });
}

int ustfwi_gpu_upload_observed(ustfwi_gpu_ctx* c, const double* observed) {
    return guarded(c, [&] {
        ensure_data_buffers(*c);
        const int nt = c->grid.nt, ns = c->n_sens;
        std::vector<double> h(static_cast<size_t>(nt) * ns);
        for (int s = 0; s < ns; ++s)
            for (int n = 0; n < nt; ++n) h[static_cast<size_t>(n) * ns + s] = observed[static_cast<size_t>(s) * nt + n];
        if (!h.empty()) CK(cudaMemcpyAsync(c->obs, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        c->obs_ready = true;
    });
}

int ustfwi_gpu_run_gradient(ustfwi_gpu_ctx* c, int boundary_thickness, int accumulate) {
    return guarded(c, [&] {
        clear_flags(*c);
        gradient_tr(*c, boundary_thickness, accumulate != 0);
        check_flags(*c, true);
    });
}

int ustfwi_gpu_download_gradient(ustfwi_gpu_ctx* c, double scale_div, double* grad_out, double* loss_out) {
    return guarded(c, [&] {
        const size_t N = static_cast<size_t>(c->g.N);
        if (!(scale_div >= 1.0)) fail(USTFWI_ERR_INVALID, "scale_div must be >= 1");
        if (grad_out) {
            const float* h = c->pinned_stage();
            CK(cudaMemcpyAsync(c->pinned, c->acc, N * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            ustfwi_host::parallel_chunks(N, [&](size_t b, size_t e) {
                for (size_t i = b; i < e; ++i) grad_out[i] = static_cast<double>(h[i]) / scale_div;
            });
        }
        if (loss_out) {
            double l[2];
            CK(cudaMemcpyAsync(l, c->loss, sizeof(l), cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            *loss_out = l[1] / scale_div;
        }
    });
}

int ustfwi_gpu_gradient_tr(ustfwi_gpu_ctx* c, const double* observed, int boundary_thickness, double* grad_out,
                           double* loss_out) {
    int rc = ustfwi_gpu_upload_observed(c, observed);
    if (rc == USTFWI_OK) rc = ustfwi_gpu_run_gradient(c, boundary_thickness, 0);
    if (rc == USTFWI_OK) rc = ustfwi_gpu_download_gradient(c, 1.0, grad_out, loss_out);
    return rc;
}

int ustfwi_gpu_evaluate_loss(ustfwi_gpu_ctx* c, const double* observed, double* loss_out) {
    return guarded(c, [&] {
        const int nt = c->grid.nt, ns = c->n_sens;
        clear_flags(*c);
        forward_sim(*c, 0);
        check_flags(*c, false);
        std::vector<float> h(static_cast<size_t>(nt) * ns);
        CK(cudaMemcpy(h.data(), c->data, h.size() * sizeof(float), cudaMemcpyDeviceToHost));
        // Kahan sum in (sensor, time) order as evaluate_loss (gradient.hpp:495-503)
        double loss = 0.0, comp = 0.0;
        for (int s = 0; s < ns; ++s)
            for (int n = 0; n < nt; ++n) {
                const double r = static_cast<double>(h[static_cast<size_t>(n) * ns + s]) - observed[static_cast<size_t>(s) * nt + n];
                const double term = 0.5 * r * r - comp;
                const double t = loss + term;
                comp = (t - loss) - term;
                loss = t;
            }
        *loss_out = loss;
    });
}

// ---- WaveStepper on the device (solver/engine.hpp:170-386), step by step ----------------

namespace {
Sim& stepper_sim(Ctx& c, int which) {
    if (which < 0 || which > 1) fail(USTFWI_ERR_INVALID, "stepper index must be 0 or 1");
    if (!c.stp[which].init) fail(USTFWI_ERR_INVALID, "stepper not initialised (ustfwi_gpu_stepper_init)");
    return c.sim[which];
}
void stage_sparse(Ctx& c, size_t n, const size_t* idx, const std::vector<float>& val) {
    if (n > c.stp_cap) {
        c.release(c.stp_idx);
        c.release(c.stp_val);
        c.stp_idx = c.alloc<int>(n);
        c.stp_val = c.alloc<float>(n);
        c.stp_cap = n;
    }
    std::vector<int> ii(n);
    for (size_t i = 0; i < n; ++i) {
        if (idx[i] >= static_cast<size_t>(c.g.N)) fail(USTFWI_ERR_INVALID, "position outside grid");
        ii[i] = static_cast<int>(idx[i]);
    }
    CK(cudaMemcpyAsync(c.stp_idx, ii.data(), n * sizeof(int), cudaMemcpyHostToDevice, c.stream));
    CK(cudaMemcpyAsync(c.stp_val, val.data(), n * sizeof(float), cudaMemcpyHostToDevice, c.stream));
}
// p = c0^2 sum_a rho_a and the entry invariant S0 = Fz p of the next step
void stepper_pressure(Ctx& c, Sim& s, int check_step) {
    ZrhoArgs a{};
    for (int f = 0; f < 3; ++f) {
        a.S[f] = s.S[f];
        a.rho[f] = s.rho[f];
    }
    a.pml = Pml{{c.pml_reg[0], c.pml_reg[1], c.pml_reg[2]}};
    a.dtrho0 = c.dtrho0;
    a.c0sq = c.c0sq;
    a.p_out = s.p;
    a.a_first = c.off_axis;
    a.check_step = check_step;
    a.diverged = c.flags;
    c.count(launch_zrho(c.g, a, false, c.stream));
}
}  // namespace

int ustfwi_gpu_stepper_init(ustfwi_gpu_ctx* c, int which, int pml_enabled, double absorption_sign,
                            int dispersion_enabled) {
    return guarded(c, [&] {
        if (which < 0 || which > 1) fail(USTFWI_ERR_INVALID, "stepper index must be 0 or 1");
        require_medium(*c);
        Sim& s = c->sim[which];
        if (!s.p) s.p = c->alloc<float>(static_cast<size_t>(c->g.N));
        if (!c->stp_scratch) c->stp_scratch = c->alloc<float>(static_cast<size_t>(c->g.N));
        s.pml_off = pml_enabled == 0;
        StepperState& t = c->stp[which];
        t.init = true;
        t.abs_sign = static_cast<float>(absorption_sign);
        t.dispersion = dispersion_enabled != 0;
        t.step_index = 0;
        reset_sim(*c, s, true);
        CK(cudaStreamSynchronize(c->stream));
    });
}

int ustfwi_gpu_stepper_reset(ustfwi_gpu_ctx* c, int which) {
    return guarded(c, [&] {
        Sim& s = stepper_sim(*c, which);
        reset_sim(*c, s, true);
        c->stp[which].step_index = 0;
        CK(cudaStreamSynchronize(c->stream));
    });
}

int ustfwi_gpu_stepper_update_velocity_density(ustfwi_gpu_ctx* c, int which) {
    return guarded(c, [&] {
        Sim& s = stepper_sim(*c, which);
        c->disp_active = c->dispersion && c->stp[which].dispersion;
        StepIO io;
        io.density_only = true;
        io.p_out = c->stp_scratch;
        run_step(*c, s, io, c->stream);
        CK(cudaStreamSynchronize(c->stream));
    });
}

int ustfwi_gpu_stepper_inject(ustfwi_gpu_ctx* c, int which, size_t n, const size_t* idx, const double* amp) {
    return guarded(c, [&] {
        Sim& s = stepper_sim(*c, which);
        std::vector<float> v(n);
        for (size_t i = 0; i < n; ++i) {
            if (idx[i] >= static_cast<size_t>(c->g.N)) fail(USTFWI_ERR_INVALID, "source position outside grid");
            const double c0 = c->c0_host[idx[i]];
            v[i] = static_cast<float>(amp[i] * (2.0 * c->grid.dt / (c->ndim * c->grid.dx[0] * std::sqrt(c0 * c0))));
        }
        stage_sparse(*c, n, idx, v);
        c->count(launch_stepper_sparse(s.rho, c->off_axis, c->stp_idx, c->stp_val, static_cast<int>(n), 0, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int ustfwi_gpu_stepper_enforce(ustfwi_gpu_ctx* c, int which, size_t n, const size_t* idx, const double* values) {
    return guarded(c, [&] {
        Sim& s = stepper_sim(*c, which);
        const auto v = to_f32(values, n);
        stage_sparse(*c, n, idx, v);
        c->count(launch_stepper_sparse(s.rho, c->off_axis, c->stp_idx, c->stp_val, static_cast<int>(n), 1, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int ustfwi_gpu_stepper_refresh_pressure(ustfwi_gpu_ctx* c, int which) {
    return guarded(c, [&] {
        Sim& s = stepper_sim(*c, which);
        stepper_pressure(*c, s, 0);
        CK(cudaStreamSynchronize(c->stream));
    });
}

int ustfwi_gpu_stepper_update_pressure(ustfwi_gpu_ctx* c, int which) {
    return guarded(c, [&] {
        Sim& s = stepper_sim(*c, which);
        StepperState& t = c->stp[which];
        const int k = ++t.step_index;
        const int check = (k & 63) == 0 ? k : 0;
        if (check) clear_flags(*c);
        if (c->absorbing) {
            c->disp_active = c->dispersion && t.dispersion;
            StepIO io;
            io.p_out = s.p;
            io.abs_sign = t.abs_sign;
            io.check_step = check;
            absorbing_tail(*c, s, io, c->stream);
        } else {
            stepper_pressure(*c, s, check);
        }
        if (check) check_flags(*c, false);
        CK(cudaStreamSynchronize(c->stream));
    });
}

int ustfwi_gpu_stepper_read(ustfwi_gpu_ctx* c, int which, int field, double* out) {
    return guarded(c, [&] {
        Sim& s = stepper_sim(*c, which);
        const float* src = nullptr;
        if (field == 0) src = s.p;
        else if (field >= 1 && field <= c->ndim) src = s.v[field - 1 + c->off_axis];
        else if (field >= 4 && field <= 3 + c->ndim) src = s.rho[field - 4 + c->off_axis];
        else fail(USTFWI_ERR_INVALID, "field must be 0 (p), 1..ndim (v_a) or 4..3+ndim (rho_a)");
        const size_t N = static_cast<size_t>(c->g.N);
        std::vector<float> h(N);
        CK(cudaMemcpyAsync(h.data(), src, N * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        for (size_t i = 0; i < N; ++i) out[i] = h[i];
    });
}

int ustfwi_gpu_stepper_gather(ustfwi_gpu_ctx* c, int which, size_t n, const size_t* idx, double* out) {
    return guarded(c, [&] {
        Sim& s = stepper_sim(*c, which);
        if (n == 0) return;
        stage_sparse(*c, n, idx, std::vector<float>(n, 0.f));
        c->count(launch_pick(s.p, c->stp_idx, static_cast<int>(n), c->stp_val, c->stream));
        std::vector<float> h(n);
        CK(cudaMemcpyAsync(h.data(), c->stp_val, n * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        for (size_t i = 0; i < n; ++i) out[i] = h[i];
    });
}

int ustfwi_gpu_stepper_step_index(ustfwi_gpu_ctx* c, int which, int* out) {
    return guarded(c, [&] {
        stepper_sim(*c, which);
        *out = c->stp[which].step_index;
    });
}

int ustfwi_gpu_half_shift(ustfwi_gpu_ctx* c, const double* f, int axis, int direction, double* out) {
    return guarded(c, [&] {
        if (axis < 0 || axis >= c->ndim) fail(USTFWI_ERR_INVALID, "axis out of range");
        const size_t N = static_cast<size_t>(c->g.N);
        const int pa = axis + c->off_axis;
        const auto h = to_f32(f, N);
        CK(cudaMemcpyAsync(c->ring[0], h.data(), N * sizeof(float), cudaMemcpyHostToDevice, c->stream));
        spectral_apply(*c, c->sim[1], c->ring[0], pa, c->dmul[pa][direction > 0 ? ST_SHIFT : ST_SHIFTM], 0, c->ring[1],
                       c->stream);
        std::vector<float> o(N);
        CK(cudaMemcpyAsync(o.data(), c->ring[1], N * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        for (size_t i = 0; i < N; ++i) out[i] = o[i];
    });
}

int ustfwi_gpu_derivative(ustfwi_gpu_ctx* c, const double* f, int axis, int stagger, double* out) {
    return guarded(c, [&] {
        if (axis < 0 || axis >= c->ndim) fail(USTFWI_ERR_INVALID, "axis out of range");
        if (stagger < 0 || stagger > 2) fail(USTFWI_ERR_INVALID, "bad stagger");
        const size_t N = static_cast<size_t>(c->g.N);
        const int pa = axis + c->off_axis;
        float* in = c->ring[0];
        float* res = c->ring[1];
        const auto h = to_f32(f, N);
        CK(cudaMemcpyAsync(in, h.data(), N * sizeof(float), cudaMemcpyHostToDevice, c->stream));
        Sim& s = c->sim[1];
        c->count(launch_zfwd(c->g, in, s.S[0], c->stream));
        PencilJobs j{};
        for (int q = 0; q < 3; ++q) j.buf[q] = s.S[q];
        j.n = 1;
        j.job[0] = {0, 0, nullptr, 0};
        c->count(launch_pencil(1, false, c->g, j, c->stream));
        j.job[0] = {0, 0, pa == 0 ? c->dmul[0][stagger] : nullptr, 1};
        c->count(launch_pencil(0, false, c->g, j, c->stream));
        j.job[0] = {0, 0, pa == 1 ? c->dmul[1][stagger] : nullptr, 0};
        c->count(launch_pencil(1, true, c->g, j, c->stream));
        c->count(launch_zinv(c->g, s.S[0], pa == 2 ? c->dmul[2][stagger] : nullptr, res, c->stream));
        std::vector<float> o(N);
        CK(cudaMemcpyAsync(o.data(), res, N * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        for (size_t i = 0; i < N; ++i) out[i] = o[i];
    });
}

int ustfwi_gpu_accumulator(ustfwi_gpu_ctx* c, float** grad_dev, double** loss_dev) {
    return guarded(c, [&] {
        if (grad_dev) *grad_dev = c->acc;
        if (loss_dev) *loss_dev = c->loss + 1;
    });
}

int ustfwi_gpu_synchronize(ustfwi_gpu_ctx* c) {
    return guarded(c, [&] { CK(cudaStreamSynchronize(c->stream)); });
}

void* ustfwi_gpu_stream(ustfwi_gpu_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }
uint64_t ustfwi_gpu_launch_count(const ustfwi_gpu_ctx* c) { return c ? c->launches : 0; }
size_t ustfwi_gpu_shell_size(const ustfwi_gpu_ctx* c) { return c ? c->shell_host.size() : 0; }

int ustfwi_gpu_set_profiling(ustfwi_gpu_ctx* c, int enable) {
    return guarded(c, [&] {
        c->touch();
        CK(cudaStreamSynchronize(c->stream));
        c->resolve_profile();
        c->profiling = enable != 0;
        for (int k = 0; k < USTFWI_KERNEL_KINDS; ++k) {
            c->prof_ms[k] = 0.0;
            c->prof_bytes[k] = 0.0;
            c->prof_n[k] = 0;
        }
    });
}

int ustfwi_gpu_kernel_stats(ustfwi_gpu_ctx* c, int kind, double* total_ms, uint64_t* launches, double* bytes) {
    return guarded(c, [&] {
        if (kind < 0 || kind >= USTFWI_KERNEL_KINDS) fail(USTFWI_ERR_INVALID, "bad kernel kind");
        CK(cudaStreamSynchronize(c->stream));
        c->resolve_profile();
        if (total_ms) *total_ms = c->prof_ms[kind];
        if (launches) *launches = c->prof_n[kind];
        if (bytes) *bytes = c->prof_bytes[kind];
    });
}

// diagnostics of the fused y-x-y chain kernel (USTFWI_CHAIN_STATS=1): CTAs, units, deferred
// (blocking) tile loads, cycles spent waiting for dependencies and for tiles, summed over CTAs
int ustfwi_gpu_chain_stats(uint64_t* out5) {
    return guarded(nullptr, [&] {
        unsigned long long t[4];
        const int n = chain_stats(t);
        out5[0] = static_cast<uint64_t>(n);
        for (int k = 0; k < 4; ++k) out5[k + 1] = t[k];
    });
}

int ustfwi_gpu_partition(ustfwi_gpu_ctx* c, int* adjoint_sms, int* replay_sms) {
    return guarded(c, [&] {
        if (adjoint_sms) *adjoint_sms = c->gstream[0] ? c->gsm[0] : 0;
        if (replay_sms) *replay_sms = c->gstream[1] ? c->gsm[1] : 0;
    });
}

int ustfwi_nccl_unique_id(char id_out[128]) {
    return guarded(nullptr, [&] {
        NcclUniqueId id;
        const int r = nccl().get_unique_id(&id);
        if (r != 0) fail(USTFWI_ERR_NCCL, "ncclGetUniqueId failed");
        std::memcpy(id_out, id.internal, 128);
    });
}

int ustfwi_gpu_comm_init(ustfwi_gpu_ctx* c, const char id[128], int nranks, int rank) {
    return guarded(c, [&] {
        if (nranks < 1 || rank < 0 || rank >= nranks) fail(USTFWI_ERR_INVALID, "bad rank / world size");
        auto& api = nccl();
        // ncclCommInitRank(ncclComm_t*, int nranks, ncclUniqueId commId, int rank): the id is
        // passed by value (128 bytes)
        using Fn = int (*)(void**, int, NcclUniqueId, int);
        auto fn = reinterpret_cast<Fn>(dlsym(api.h, "ncclCommInitRank"));
        if (!fn) fail(USTFWI_ERR_NCCL, "ncclCommInitRank missing");
        if (c->comm) {
            api.comm_destroy(c->comm);
            c->comm = nullptr;
        }
        NcclUniqueId uid;
        std::memcpy(uid.internal, id, 128);
        const int r = fn(&c->comm, nranks, uid, rank);
        if (r != 0) {
            c->comm = nullptr;
            fail(USTFWI_ERR_NCCL, std::string("ncclCommInitRank: ") + (api.error_string ? api.error_string(r) : "error"));
        }
        c->nranks = nranks;
        c->rank = rank;
    });
}

int ustfwi_gpu_batch_reserve(ustfwi_gpu_ctx* c, int slots) {
    return guarded(c, [&] {
        if (slots < 1) fail(USTFWI_ERR_INVALID, "slots must be >= 1");
        const size_t N = static_cast<size_t>(c->g.N);
        if (slots != c->n_slots) {
            for (void* p : {(void*)c->slot_grad, (void*)c->slot_loss, (void*)c->gather_grad, (void*)c->gather_loss})
                c->release(p);
            c->slot_grad = c->alloc<float>(static_cast<size_t>(slots) * N);
            c->slot_loss = c->alloc<double>(static_cast<size_t>(slots));
            c->gather_grad = nullptr;
            c->gather_loss = nullptr;
            c->n_slots = slots;
        }
        // empty slots (idle ranks, ragged batches) hold zeros and are never summed
        CK(cudaMemsetAsync(c->slot_grad, 0, static_cast<size_t>(slots) * N * sizeof(float), c->stream));
        CK(cudaMemsetAsync(c->slot_loss, 0, static_cast<size_t>(slots) * sizeof(double), c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int ustfwi_gpu_run_gradient_slot(ustfwi_gpu_ctx* c, int boundary_thickness, int slot) {
    return guarded(c, [&] {
        if (slot < 0 || slot >= c->n_slots) fail(USTFWI_ERR_INVALID, "slot out of range (ustfwi_gpu_batch_reserve)");
        clear_flags(*c);
        gradient_tr(*c, boundary_thickness, false, slot);
        check_flags(*c, true);
    });
}

int ustfwi_gpu_batch_mean(ustfwi_gpu_ctx* c, int batch) {
    return guarded(c, [&] {
        const int W = c->comm ? c->nranks : 1;
        const int slots = c->n_slots;
        if (slots < 1) fail(USTFWI_ERR_INVALID, "no mini-batch slots (ustfwi_gpu_batch_reserve)");
        if (batch < 1 || batch > W * slots) fail(USTFWI_ERR_INVALID, "batch must be in [1, world * slots]");
        const size_t N = static_cast<size_t>(c->g.N);
        const float* gathered = c->slot_grad;
        const double* gl = c->slot_loss;
        if (W > 1) {
            if (!c->gather_grad) {
                c->gather_grad = c->alloc<float>(static_cast<size_t>(W) * slots * N);
                c->gather_loss = c->alloc<double>(static_cast<size_t>(W) * slots);
            }
            auto& api = nccl();
            // ncclFloat32 = 7, ncclFloat64 = 8 (nccl.h); rank-major receive layout
            int r = api.all_gather(c->slot_grad, c->gather_grad, static_cast<size_t>(slots) * N, 7, c->comm, c->stream);
            if (r == 0) r = api.all_gather(c->slot_loss, c->gather_loss, static_cast<size_t>(slots), 8, c->comm, c->stream);
            if (r != 0) fail(USTFWI_ERR_NCCL, "ncclAllGather failed");
            gathered = c->gather_grad;
            gl = c->gather_loss;
        }
        c->count(launch_ordered_mean(c->g.N, gathered, W, slots, batch, c->acc, c->stream));
        std::vector<double> h(static_cast<size_t>(W) * slots);
        CK(cudaMemcpyAsync(h.data(), gl, h.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        double loss = 0.0;
        for (int q = 0; q < batch; ++q) loss += h[static_cast<size_t>((q % W) * slots + q / W)];
        loss *= 1.0 / batch;
        CK(cudaMemcpyAsync(c->loss + 1, &loss, sizeof(double), cudaMemcpyHostToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

}  // extern "C"
