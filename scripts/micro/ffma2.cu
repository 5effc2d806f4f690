// FFMA2 (packed f32x2) vs FFMA vs DFMA issue throughput, 3-register-operand forms, and the
// planned FP32 filter cell pattern (2 FFMA2 recurrence + 1 FFMA2 test per 2 cells + sign OR).
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
    u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}
template <int ILP> __global__ void k_ffma2(u64* io, int iters) {
    u64 a[ILP]; const u64 b = io[threadIdx.x & 7], c = io[8 + (threadIdx.x & 7)];
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = io[16 + i];
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 32 / ILP; ++u)
#pragma unroll
            for (int i = 0; i < ILP; ++i) a[i] = fma2(a[i], b, c);
    u64 s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s ^= a[i];
    if (s == 12345) io[0] = s;
}
template <int ILP> __global__ void k_ffma(u64* io, int iters) {
    float a[ILP]; const float* f = (const float*)io; const float b = f[threadIdx.x & 7], c = f[8 + (threadIdx.x & 7)];
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = f[16 + i];
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 32 / ILP; ++u)
#pragma unroll
            for (int i = 0; i < ILP; ++i) a[i] = fmaf(a[i], b, c);
    float s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += a[i];
    if (s == 1.2345f) io[0] = 1;
}
template <int ILP> __global__ void k_dfma(u64* io, int iters) {
    double a[ILP]; const double* f = (const double*)io; const double b = f[threadIdx.x & 7], c = f[8 + (threadIdx.x & 7)];
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = f[16 + i];
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 32 / ILP; ++u)
#pragma unroll
            for (int i = 0; i < ILP; ++i) a[i] = fma(a[i], b, c);
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += a[i];
    if (s == 1.2345) io[0] = 1;
}
// cell pattern: P pairs of cells (2P cells) per row; per pair: cov = fma2(dfi, dg, cov);
// cov = fma2(df, dgi, cov); z = fma2(ca, bi, -cov) ; then OR of sign bits (LOP3 tree)
template <int P> __global__ void k_cell(u64* io, int iters) {
    u64 cov[P], dg[P], df[P], ca[P];
#pragma unroll
    for (int i = 0; i < P; ++i) { cov[i] = io[16 + i]; dg[i] = io[32 + i]; df[i] = io[48 + i]; ca[i] = io[64 + i]; }
    u64 dfi = io[threadIdx.x & 7], dgi = io[8 + (threadIdx.x & 7)], bi = io[80];
    unsigned acc = 0;
    for (int it = 0; it < iters; ++it) {
        unsigned orv = 0;
#pragma unroll
        for (int i = 0; i < P; ++i) {
            cov[i] = fma2(dfi, dg[i], cov[i]);
            cov[i] = fma2(df[i], dgi, cov[i]);
            u64 z = fma2(ca[i], bi, cov[i] ^ 0x8000000080000000ull);
            orv |= (unsigned)z | (unsigned)(z >> 32);
        }
        acc += orv >> 31;
        dfi += 0x10001; bi += 3;
    }
    u64 s = acc;
#pragma unroll
    for (int i = 0; i < P; ++i) s ^= cov[i];
    if (s == 12345) io[0] = s;
}
template <class F>
void run(const char* name, F kern, int ilp, double ops_per_iter, int warps_per_sm, int iters, u64* d) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int threads = 32 * warps_per_sm; if (threads > 1024) threads = 1024;
    int blocks = sms * (32 * warps_per_sm / threads);
    kern<<<blocks, threads>>>(d, 10);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); kern<<<blocks, threads>>>(d, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = (double)blocks * threads * iters * ops_per_iter;
    printf("%-6s ilp=%2d warps/SM=%2d  %.3e lane-ops/s  (%.2f per SM per clk @1.965GHz)\n", name, ilp, warps_per_sm,
           fl / (ms * 1e-3), fl / (ms * 1e-3) / sms / 1.965e9);
}
int main() {
    u64* d; cudaMalloc(&d, 4096); 
    u64 h[128]; for (int i = 0; i < 128; ++i) { float f[2] = {1.0f + i * 1e-3f, 0.5f - i * 1e-3f}; memcpy(&h[i], f, 8); }
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    int W[] = {8, 16, 24, 32};
    for (int w : W) {
        run("dfma", k_dfma<8>, 8, 32, w, 4000, d);
        run("ffma", k_ffma<8>, 8, 32, w, 4000, d);
        run("ffma2", k_ffma2<8>, 8, 32, w, 4000, d);   // instructions (each 2 lanes' worth of FMA)
        run("cell4", k_cell<4>, 4, 8, w, 20000, d);    // cells per iter per thread = 8
        run("cell8", k_cell<8>, 8, 16, w, 10000, d);
    }
    return 0;
}
