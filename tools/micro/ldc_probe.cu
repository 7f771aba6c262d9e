// Microbenchmark (design study): node-record fetch throughput through the L1
// data pipe (LDG) vs the constant cache (LDC, __constant__ bank) when lanes of a
// warp read the same record (top of a BVH) or K distinct records.
// Each thread walks a dependent chain of 56 B "node" reads (next index derived
// from the loaded data), many warps per SM, like the traversal's top levels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ldc_probe ldc_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

constexpr int kNodes = 1024;          // 64 KB of 64 B records
__constant__ float4 c_nodes[kNodes * 4];

__device__ __forceinline__ void ldg256(const float4* p, float4& a, float4& b) {
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w) : "l"(p));
}

template <int MODE>   // 0: global LDG (56 B), 1: constant LDC
__global__ void __launch_bounds__(128, 9) walk(const float4* __restrict__ g, int iters, int uniq, float* sink) {
    const int lane = threadIdx.x & 31;
    int idx = (lane % uniq) * 7 + 1;   // uniq distinct records per warp
    float acc = 0.f;
    for (int i = 0; i < iters; ++i) {
        float4 a, b, z;
        int2 r;
        const int k = idx & (kNodes - 1);
        if (MODE == 0) {
            ldg256(g + 4 * k, a, b);
            z = __ldg(g + 4 * k + 2);
            r = __ldg(reinterpret_cast<const int2*>(g + 4 * k + 3));
        } else {
            a = c_nodes[4 * k];
            b = c_nodes[4 * k + 1];
            z = c_nodes[4 * k + 2];
            const float4 rr = c_nodes[4 * k + 3];
            r = make_int2(__float_as_int(rr.x), __float_as_int(rr.y));
        }
        // ~slab-test-like arithmetic on the record, next index depends on it
        const float t0 = fminf(fmaxf(a.x * 1.1f, a.y), fmaxf(a.z, a.w));
        const float t1 = fminf(fmaxf(b.x * 0.9f, b.y), fmaxf(b.z, b.w));
        const float t2 = fmaxf(z.x, z.y) - fminf(z.z, z.w);
        acc += t0 + t1 + t2;
        idx = (t0 < t1 ? r.x : r.y) + (lane % uniq) * 7;
    }
    if (acc == 12345.f) sink[0] = acc;
    if (idx == -7) sink[1] = 1.f;
}

int main() {
    const int n = kNodes * 4;
    float4* h = new float4[n];
    for (int i = 0; i < kNodes; ++i) {
        h[4 * i] = make_float4(i, i + 1, i + 2, i + 3);
        h[4 * i + 1] = make_float4(i + 4, i + 5, i + 6, i + 7);
        h[4 * i + 2] = make_float4(1, 2, 3, 4);
        int r0 = (i * 2 + 1) % kNodes, r1 = (i * 2 + 2) % kNodes;
        float f0, f1;
        memcpy(&f0, &r0, 4);
        memcpy(&f1, &r1, 4);
        h[4 * i + 3] = make_float4(f0, f1, 0, 0);
    }
    float4* g;
    float* sink;
    cudaMalloc(&g, n * sizeof(float4));
    cudaMalloc(&sink, 64);
    cudaMemcpy(g, h, n * sizeof(float4), cudaMemcpyHostToDevice);
    cudaMemcpyToSymbol(c_nodes, h, n * sizeof(float4));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 9, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int uniq : {1, 2, 4, 8, 32}) {
        for (int mode = 0; mode < 2; ++mode) {
            float best = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(e0);
                if (mode == 0) walk<0><<<blocks, 128>>>(g, iters, uniq, sink);
                else walk<1><<<blocks, 128>>>(g, iters, uniq, sink);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
            }
            const double lane_fetches = double(blocks) * 128 * iters;
            printf("uniq %2d %s: %.3f ms, %.3g lane-node-fetches/s, %.3g warp-fetches/s\n", uniq,
                   mode ? "LDC" : "LDG", best, lane_fetches / (best * 1e-3), lane_fetches / 32 / (best * 1e-3));
        }
    }
    cudaError_t err = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(err));
    return 0;
}
