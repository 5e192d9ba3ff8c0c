// tmem_probe.cu -- microbenchmark: tcgen05.ld / tcgen05.st (TMEM <-> registers) throughput and latency for the
// access pattern a TMEM-resident gradient tile would use (warp-uniform column, 32 lanes x 2 columns x 4 B), against
// the same read-modify-write on a shared-memory tile.  One CTA per SM, W warps; cycles per warp-RMW reported.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_probe tmem_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void tm_ld2(uint32_t taddr, float& a, float& b) {
    uint32_t r0, r1;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(taddr));
    a = __uint_as_float(r0);
    b = __uint_as_float(r1);
}
__device__ __forceinline__ void tm_st2(uint32_t taddr, float a, float b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(__float_as_uint(a)),
                 "r"(__float_as_uint(b)) : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// MODE 0: TMEM RMW of G literals per group (G loads, one wait, G stores, wait::st); MODE 1: same on smem (LDS.64/STS.64)
// MODE 2: TMEM loads only (G loads, one wait); MODE 3: TMEM RMW without the wait::st (stores ordered before the next
// group's loads by the per-thread order of tcgen05 operations on the same address -- to be checked by the result)
template <int MODE, int G>
__global__ void probe(int iters, float* out, long long* cyc) {
    __shared__ uint32_t taddr_s;
    extern __shared__ float2 tile[];   // [400][32 lanes] float2 per warp pair region
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (MODE != 1) {
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(&taddr_s)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (warp < 4)
            for (uint32_t c = 0; c < 256; c += 2) tm_st2(taddr_s + ((uint32_t)(32 * warp) << 16) + c, 0.f, 0.f);
        tm_wait_st();
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
    } else {
        for (int i = threadIdx.x; i < 128 * 32 * 4; i += blockDim.x) tile[i] = make_float2(0.f, 0.f);
        __syncthreads();
    }
    const uint32_t base = (MODE != 1 ? taddr_s : 0u) + ((uint32_t)(32 * (warp & 3)) << 16);
    float acc = 0.f;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t col[G];
#pragma unroll
        for (int g = 0; g < G; ++g) col[g] = ((uint32_t)(it * G + g) * 74u + (uint32_t)warp * 22u) & 254u;   // even columns < 256, cheap
        float2 v[G];
        if (MODE == 1) {
            float2* t = tile + (warp & 3) * 128 * 32 + lane;
#pragma unroll
            for (int g = 0; g < G; ++g) v[g] = t[((col[g] >> 1) & 127) * 32];
#pragma unroll
            for (int g = 0; g < G; ++g) t[((col[g] >> 1) & 127) * 32] = make_float2(v[g].x + 1.f, v[g].y + 1.f);
        } else {
#pragma unroll
            for (int g = 0; g < G; ++g) tm_ld2(base + col[g], v[g].x, v[g].y);
            tm_wait_ld();
            if (MODE == 0 || MODE == 3) {
#pragma unroll
                for (int g = 0; g < G; ++g) tm_st2(base + col[g], v[g].x + 1.f, v[g].y + 1.f);
                if (MODE == 0) tm_wait_st();
            } else {
#pragma unroll
                for (int g = 0; g < G; ++g) acc += v[g].x + v[g].y;
            }
        }
    }
    const long long t1 = clock64();
    if (lane == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
    if (MODE == 0 || MODE == 3) {   // total increments seen in this warp's quadrant (all warps of the quadrant)
        tm_wait_st();
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (warp < 4) {
            float tot = 0.f;
            for (uint32_t c = 0; c < 256; c += 2) {
                float a, b;
                tm_ld2(base + c, a, b);
                tm_wait_ld();
                tot += a + b;
            }
            acc = tot;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (MODE != 1) {
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
    }
}

template <int MODE, int G>
void run(const char* name, int warps) {
    const int iters = 4096, blocks = 148;
    float* out;
    long long* cyc;
    cudaMalloc(&out, blocks * 1024 * 4);
    cudaMalloc(&cyc, blocks * 32 * 8);
    const size_t smem = MODE == 1 ? 128 * 32 * 4 * sizeof(float2) : 0;
    if (smem) cudaFuncSetAttribute(probe<MODE, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe<MODE, G><<<blocks, 32 * warps, smem>>>(16, out, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<MODE, G><<<blocks, 32 * warps, smem>>>(iters, out, cyc);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[32];
    cudaMemcpy(h, cyc, warps * 8, cudaMemcpyDeviceToHost);
    const double ops = (double)iters * G * warps;   // warp-level column-pair accesses per SM
    const double clk = ms * 1e-3 * 1.965e9;
    float ho = 0;
    cudaMemcpy(&ho, out, 4, cudaMemcpyDeviceToHost);   // block 0 thread 0: quadrant 0 total (expect 2 x accesses of its warps)
    const double expect = warps == 4 ? 2.0 * (double)iters * G : -1.0;   // one warp per quadrant: no races
    printf("%-34s warps=%2d G=%d  %s  %.3f ms  %.2f SM-cycles per warp-access  (warp0 %.1f cyc/access)  %.0f B/clk/SM%s\n",
           name, warps, G, err == cudaSuccess ? "ok " : cudaGetErrorString(err), ms, clk / ops, (double)h[0] / (iters * G),
           ops * 256.0 * (MODE == 2 ? 1 : 2) / clk,
           (MODE == 0 || MODE == 3) && warps == 4 ? (ho == expect ? "  [sums exact]" : "  [SUMS WRONG]") : "");
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int w : {4, 8, 16}) {
        run<0, 7>("TMEM RMW (ld x2, wait, st x2)", w);
        run<0, 14>("TMEM RMW (ld x2, wait, st x2)", w);
        run<3, 14>("TMEM RMW, no wait::st", w);
        run<2, 7>("TMEM ld only", w);
        run<2, 14>("TMEM ld only", w);
        run<1, 7>("smem RMW (LDS.64 / STS.64)", w);
        run<1, 14>("smem RMW (LDS.64 / STS.64)", w);
    }
    return 0;
}
