// Issue-rate probe for the DP-cell instruction mix on sm_100a: FFMA vs
// FFMA2 (packed f32x2), FMNMX vs FMNMX3, MUFU.SQRT, and the 6-dim cell mix.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o isa_rates isa_rates.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
#define NA 8
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ float min3(float a, float b, float c) { float r; asm volatile("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }
__device__ __forceinline__ float min2(float a, float b) { float r; asm volatile("min.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float sq(float a) { float r; asm volatile("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a)); return r; }
__device__ __forceinline__ float ffma(float a, float b, float c) { float r; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }

template <int OP>
__global__ void probe(int iters, float* sink, float s0) {
    float a[NA]; u64 p[NA];
    for (int k = 0; k < NA; ++k) { a[k] = s0 + threadIdx.x * 1e-3f + k; p[k] = __float_as_uint(a[k]) | ((u64)__float_as_uint(a[k] + 1) << 32); }
    const float b = 0.999f, c = 1e-4f;
    const u64 pb = __float_as_uint(b) | ((u64)__float_as_uint(b) << 32), pc = __float_as_uint(c) | ((u64)__float_as_uint(c) << 32);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < NA; ++k) {
            if (OP == 0) a[k] = ffma(a[k], b, c);
            if (OP == 1) p[k] = fma2(p[k], pb, pc);
            if (OP == 2) a[k] = min2(a[k], b + k);
            if (OP == 3) a[k] = min3(a[k], b + k, c + k);
            if (OP == 4) a[k] = sq(a[k]);
            if (OP == 5) { a[k] = ffma(a[k], b, c); if (k & 1) a[k - 1] = min2(a[k - 1], b + k); }      // 8 FFMA + 4 FMNMX
            if (OP == 6) { p[k] = fma2(p[k], pb, pc); if (k & 1) a[k] = min3(a[k], b + k, c + k); }    // 8 FFMA2 + 4 FMNMX3
            if (OP == 7) { a[k] = ffma(a[k], b, c); if (k == 0) a[1] = sq(a[1]); }                   // 8 FFMA + 1 MUFU
            if (OP == 9) { p[k] = fma2(p[k], pb, pc); if (k & 1) a[k - 1] = min2(a[k - 1], __uint_as_float((unsigned)p[k - 1])); }  // 8 FFMA2 + 4 FMNMX
            if (OP == 10) { a[k] = ffma(a[k], b, c); if (k & 1) a[k - 1] = min3(a[k - 1], b + k, c + k); }  // 8 FFMA + 4 FMNMX3
            if (OP == 11) { p[k] = fma2(p[k], pb, pc); if (k & 1) a[k] = sq(a[k]); }  // 8 FFMA2 + 4 MUFU
            if (OP == 8) { p[k] = fma2(p[k], pb, pc); a[k] = ffma(a[k], b, c); }                       // 8 FFMA2 + 8 FFMA
        }
    }
    float t = 0;
    for (int k = 0; k < NA; ++k) t += a[k] + __uint_as_float((unsigned)p[k]);
    if (t == 1234.5f) sink[threadIdx.x] = t;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* sink; cudaMalloc(&sink, 4096);
    const char* names[] = {"FFMA", "FFMA2", "FMNMX", "FMNMX3", "MUFU.SQRT", "8FFMA+4MNMX", "8FFMA2+4MNMX3", "8FFMA+1MUFU", "8FFMA2+8FFMA", "8FFMA2+4MNMX", "8FFMA+4MNMX3", "8FFMA2+4MUFU"};
    const double per[] = {1, 1, 1, 1, 1, 12.0 / 8, 12.0 / 8, 9.0 / 8, 2, 12.0 / 8, 12.0 / 8, 12.0 / 8};
    void (*ks[])(int, float*, float) = {probe<0>, probe<1>, probe<2>, probe<3>, probe<4>, probe<5>, probe<6>, probe<7>, probe<8>, probe<9>, probe<10>, probe<11>};
    const int iters = 20000, threads = 512, blocks = sms * 4;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int o = 0; o < 12; ++o) {
        ks[o]<<<blocks, threads>>>(100, sink, 1.f);
        cudaEventRecord(e0);
        ks[o]<<<blocks, threads>>>(iters, sink, 1.f);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double winst = (double)blocks * threads / 32 * iters * NA * per[o];
        double per_sm_clk = winst / sms / (ms * 1e-3 * clk * 1e3);
        printf("%-10s %.3f ms  warp-instr/clk/SM = %.3f (at max clock %d MHz)\n", names[o], ms, per_sm_clk, clk / 1000);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
