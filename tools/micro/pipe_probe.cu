// Microbenchmark (design study): which SM pipes a warp-uniform 16 B fetch costs.
// Kernels run many resident warps, each issuing a long dependent-free stream of
//   0: LDG.128, all lanes the same address (L1 hit)
//   1: SHFL.IDX x4 (16 B per lane broadcast from lane 0)
//   2: LDS.128, all lanes the same address (shared-memory broadcast)
//   3: LDS.128, lanes at distinct 16 B words (conflict-free)
//   4: 0 and 1 interleaved (do they share a pipe?)
//   5: 0 and 2 interleaved
// and report warp-instructions per SM-clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_probe pipe_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) probe(const float4* __restrict__ g, int iters, float* sink) {
    __shared__ float4 s[256];
    const int lane = threadIdx.x & 31;
    s[threadIdx.x] = make_float4(threadIdx.x, 1, 2, 3);
    __syncthreads();
    float4 acc = make_float4(0, 0, 0, 0);
    float4 v = make_float4(lane, 1, 2, 3);
    int off = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll 8
        for (int u = 0; u < 8; ++u) {
            const int k = (off + u) & 63;
            if (MODE == 0 || MODE == 4 || MODE == 5) {
                float4 a;
                asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w) : "l"(g + k));
                acc.x += a.x; acc.y += a.y; acc.z += a.z; acc.w += a.w;
            }
            if (MODE == 1 || MODE == 4) {
                acc.x += __shfl_sync(0xffffffffu, v.x, k & 31);
                acc.y += __shfl_sync(0xffffffffu, v.y, k & 31);
                acc.z += __shfl_sync(0xffffffffu, v.z, k & 31);
                acc.w += __shfl_sync(0xffffffffu, v.w, k & 31);
            }
            if (MODE == 2 || MODE == 5) {
                float4 a;
                asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w)
                             : "r"(static_cast<unsigned>(__cvta_generic_to_shared(&s[k]))));
                acc.x += a.x; acc.y += a.y; acc.z += a.z; acc.w += a.w;
            }
            if (MODE == 3) {
                float4 a;
                asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w)
                             : "r"(static_cast<unsigned>(__cvta_generic_to_shared(&s[(lane + k) & 255]))));
                acc.x += a.x; acc.y += a.y; acc.z += a.z; acc.w += a.w;
            }
        }
        off += 8;
    }
    if (acc.x + acc.y + acc.z + acc.w == 1234.5f) sink[0] = 1.f;
}

int main() {
    float4* g;
    float* sink;
    cudaMalloc(&g, 64 * sizeof(float4));
    cudaMemset(g, 0, 64 * sizeof(float4));
    cudaMalloc(&sink, 64);
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);   // kHz
    const int blocks = sms * 8, iters = 2048;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[] = {"LDG.128 uniform", "SHFL x4", "LDS.128 uniform", "LDS.128 distinct",
                           "LDG.128 + SHFL x4", "LDG.128 + LDS.128 uniform"};
    for (int mode = 0; mode < 6; ++mode) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            switch (mode) {
                case 0: probe<0><<<blocks, 256>>>(g, iters, sink); break;
                case 1: probe<1><<<blocks, 256>>>(g, iters, sink); break;
                case 2: probe<2><<<blocks, 256>>>(g, iters, sink); break;
                case 3: probe<3><<<blocks, 256>>>(g, iters, sink); break;
                case 4: probe<4><<<blocks, 256>>>(g, iters, sink); break;
                case 5: probe<5><<<blocks, 256>>>(g, iters, sink); break;
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        const double warp_iters = double(blocks) * 8 * iters * 8;   // warps x inner iterations
        const double sm_clk = best * 1e-3 * 1965e6;                 // at the max clock
        printf("%-26s %.3f ms  %.3f inner-iterations / SM-clock\n", names[mode], best, warp_iters / sms / sm_clk);
    }
    printf("status %s (clock rate attr %d kHz)\n", cudaGetErrorString(cudaGetLastError()), clk);
    return 0;
}
