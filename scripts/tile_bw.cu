// Bandwidth probe for the pencil-pass access pattern (no FFT): each CTA moves [L][TB]
// complex tiles with row pitch P (elements) from src to dst via cp.async 16-B granules into
// shared memory and plain 8-B stores, optionally double-buffered across tiles.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tile_bw scripts/tile_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void cp16(void* s, const void* g) {
    unsigned a = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(a), "l"(g) : "memory");
}

template <int L, int TB, int NT, bool DB>
__global__ void __launch_bounds__(NT) tiles(const float2* __restrict__ src, float2* __restrict__ dst, int pitch,
                                            int nlines, int ntx, int ntiles) {
    extern __shared__ float2 sm[];
    float2* buf[2] = {sm, DB ? sm + L * TB : sm};
    const int per = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    auto base_of = [&](int u) {
        const int tile = blockIdx.x + u * gridDim.x;
        const int line = tile / ntx, c0 = (tile % ntx) * TB;
        return (long long)line * (pitch == 132 ? 480 : 1) * 132 + c0;  // y: line = x plane; x: line = y row
    };
    auto load = [&](int u, float2* b) {
        if (u < per) {
            const float2* s = src + base_of(u);
            for (int i = threadIdx.x; i < L * TB / 2; i += NT) {
                const int row = i / (TB / 2), cc = 2 * (i % (TB / 2));
                cp16(b + row * TB + cc, s + (long long)row * pitch + cc);
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    if (DB) load(0, buf[0]);
    for (int u = 0; u < per; ++u) {
        float2* b = buf[u & 1];
        if (DB) {
            load(u + 1, buf[(u + 1) & 1]);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            load(u, b);
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        float2* d = dst + base_of(u);
        for (int i = threadIdx.x; i < L * TB; i += NT) {
            const int row = i / TB, c = i % TB;
            float2 v = b[i];
            v.x += 1.f;
            d[(long long)row * pitch + c] = v;
        }
        __syncthreads();
    }
}

template <int TB, int NT, bool DB>
void run(const char* name, float2* a, float2* b, int pitch, int ctas_per_sm) {
    constexpr int L = 480;
    const int ntx = 136 / TB, nlines = 480, ntiles = ntx * nlines;
    const size_t smem = (DB ? 2 : 1) * size_t(L) * TB * 8;
    auto k = tiles<L, TB, NT, DB>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = DB ? 148 * ctas_per_sm : ntiles;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) k<<<grid, NT, smem>>>(a, b, pitch, nlines, ntx, ntiles);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) k<<<grid, NT, smem>>>(a, b, pitch, nlines, ntx, ntiles);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = 2.0 * 480 * 480 * 136 * 8;  // read + write of the padded volume
    printf("%-34s TB=%2d DB=%d grid=%6d  %.3f ms  %.0f GB/s  (%s)\n", name, TB, DB, grid, ms / reps,
           bytes / (ms / reps * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    float2 *a, *b;
    const size_t n = 480ull * 480 * 132 + 64;
    cudaMalloc(&a, n * 8);
    cudaMalloc(&b, n * 8);
    cudaMemset(a, 0, n * 8);
    // y-pass pattern: pitch = nzp (132), lines = x planes
    run<8, 256, true>("y pitch, double-buffered 2/SM", a, b, 132, 2);
    run<8, 256, false>("y pitch, one tile per CTA", a, b, 132, 0);
    run<16, 256, true>("y pitch, double-buffered 2/SM", a, b, 132, 2);
    run<4, 128, true>("y pitch, double-buffered 4/SM", a, b, 132, 4);
    // x-pass pattern: pitch = ny*nzp (480*132), lines = y rows
    run<8, 256, true>("x pitch, double-buffered 2/SM", a, b, 480 * 132, 2);
    run<8, 256, false>("x pitch, one tile per CTA", a, b, 480 * 132, 0);
    run<16, 256, true>("x pitch, double-buffered 2/SM", a, b, 480 * 132, 2);
    run<4, 128, true>("x pitch, double-buffered 4/SM", a, b, 480 * 132, 4);
    return 0;
}
