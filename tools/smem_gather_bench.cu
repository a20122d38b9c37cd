// Microbenchmark: random u16 gathers from a ~224 KB shared-memory table on
// B200, the access pattern of the DFA walk (row = state*4 + symbol).
//   chained:     s = tab[s*8 + c]  (dependent, like a DFA stream), U chains/thread
//   independent: x ^= tab[hash(i)] (no dependency)
// Reports lookups per SM-cycle. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kRows = 28000;  // ~224 KB of 8-byte rows

template <int U>
__global__ void chained(const uint16_t* gtab, int steps, unsigned long long* sink, long long* cycles) {
    extern __shared__ __align__(16) uint16_t tab[];
    for (int i = threadIdx.x; i < kRows * 4; i += blockDim.x) tab[i] = gtab[i];
    __syncthreads();
    uint32_t s[U], rng = threadIdx.x * 2654435761u + blockIdx.x * 40503u;
#pragma unroll
    for (int u = 0; u < U; ++u) s[u] = (threadIdx.x * 7 + u * 131) % kRows;
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(tab));
    long long t0 = clock64();
#pragma unroll 1
    for (int k = 0; k < steps; ++k) {
        rng = rng * 1664525u + 1013904223u;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t c2 = (rng >> (2 * u + 8)) & 6u;
            uint16_t v;
            asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(base + (s[u] << 3) + c2));
            s[u] = v;
        }
    }
    long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) acc += s[u];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) atomicMax(reinterpret_cast<unsigned long long*>(cycles), (unsigned long long)(t1 - t0));
}

extern __shared__ __align__(16) unsigned char acg_hot_smem[];
__device__ __forceinline__ uint32_t lds_hot(uint32_t off) {
    uint16_t v;
    asm volatile("{ .reg .u32 t; mov.u32 t, acg_hot_smem; add.u32 t, t, %1; ld.shared.u16 %0, [t]; }" : "=h"(v) : "r"(off));
    return v;
}
// the K1s step: a = (v*8 + c2) & 0x3FFFF ; v = LDS[a + base] ; acc |= v
template <int U>
__global__ void kstep(const uint16_t* gtab, int steps, unsigned long long* sink, long long* cycles) {
    for (int i = threadIdx.x; i < kRows * 4; i += blockDim.x) reinterpret_cast<uint16_t*>(acg_hot_smem)[i] = gtab[i];
    __syncthreads();
    uint32_t s[U], acc = 0, rng = threadIdx.x * 2654435761u + blockIdx.x * 40503u;
#pragma unroll
    for (int u = 0; u < U; ++u) s[u] = (threadIdx.x * 7 + u * 131) % kRows;
    long long t0 = clock64();
#pragma unroll 1
    for (int k = 0; k < steps; k += 4) {
        rng = rng * 1664525u + 1013904223u;
        const uint32_t w6 = rng & 0x06060606u;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t v = lds_hot((s[u] * 8u + __byte_perm(w6, 0u, 0x4440u + kk)) & 0x3FFFFu);
                acc |= v;
                s[u] = v;
            }
        }
    }
    long long t1 = clock64();
#pragma unroll
    for (int u = 0; u < U; ++u) acc += s[u];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) atomicMax(reinterpret_cast<unsigned long long*>(cycles), (unsigned long long)(t1 - t0));
}

__global__ void independent(const uint16_t* gtab, int steps, unsigned long long* sink, long long* cycles) {
    extern __shared__ __align__(16) uint16_t tab[];
    for (int i = threadIdx.x; i < kRows * 4; i += blockDim.x) tab[i] = gtab[i];
    __syncthreads();
    uint32_t rng = threadIdx.x * 2654435761u + blockIdx.x * 40503u, acc = 0;
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(tab));
    long long t0 = clock64();
#pragma unroll 1
    for (int k = 0; k < steps; ++k) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            rng = rng * 1664525u + 1013904223u;
            uint16_t v;
            asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(base + ((rng >> 8) % (kRows * 4)) * 2));
            acc ^= v;
        }
    }
    long long t1 = clock64();
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) atomicMax(reinterpret_cast<unsigned long long*>(cycles), (unsigned long long)(t1 - t0));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint16_t* h = new uint16_t[kRows * 4];
    uint32_t x = 12345;
    for (int i = 0; i < kRows * 4; ++i) {
        x = x * 1103515245u + 12345u;
        h[i] = (x >> 8) % kRows;
    }
    uint16_t* d;
    unsigned long long* sink;
    long long* cyc;
    cudaMalloc(&d, kRows * 8);
    cudaMalloc(&sink, 8ull * 148 * 1024);
    cudaMalloc(&cyc, 8);
    cudaMemcpy(d, h, kRows * 8, cudaMemcpyHostToDevice);
    const size_t smem = kRows * 8;
    cudaFuncSetAttribute(chained<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(chained<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(chained<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(chained<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(independent, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int steps = 4096;
    auto run = [&](const char* name, int U, int tpb, void (*k)(const uint16_t*, int, unsigned long long*, long long*)) {
        cudaMemset(cyc, 0, 8);
        k<<<sms, tpb, smem>>>(d, steps, sink, cyc);
        cudaMemset(cyc, 0, 8);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<<<sms, tpb, smem>>>(d, steps, sink, cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        long long c = 0;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        const double lookups = (double)tpb * U * steps;  // per SM
        printf("%-12s U=%d tpb=%4d  %.3f lookups/SM-cycle  (%.2f ms, %.0f G lookups/s chip)  err=%s\n", name, U,
               tpb, lookups / (double)c, ms, lookups * sms / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
    };
    cudaFuncSetAttribute(kstep<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kstep<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1) {
            // DFA-shaped table: rows point mostly at a few thousand "shallow" rows (skewed)
            FILE* f = fopen(getenv("TABLE") ? getenv("TABLE") : "", "rb");
            if (f) {
                size_t got = fread(h, 2, kRows * 4, f);
                fclose(f);
                printf("loaded %zu entries from the real table\n", got);
                for (int i = 0; i < kRows * 4; ++i) h[i] &= 0x7FFF;
                for (int i = 0; i < kRows * 4; ++i) if (h[i] >= kRows) h[i] = 0;
            } else {
                for (int i = 0; i < kRows * 4; ++i) {
                    x = x * 1103515245u + 12345u;
                    const uint32_t r = (x >> 8);
                    h[i] = (r & 3) ? (r >> 4) % 4000 : (r >> 4) % kRows;
                }
                printf("synthetic skewed table\n");
            }
            cudaMemcpy(d, h, kRows * 8, cudaMemcpyHostToDevice);
        }
        for (int tpb : {512, 1024}) {
            run("chained", 1, tpb, chained<1>);
            run("chained", 4, tpb, chained<4>);
            run("kstep", 1, tpb, kstep<1>);
            run("kstep", 4, tpb, kstep<4>);
        }
    }
    return 0;
}
