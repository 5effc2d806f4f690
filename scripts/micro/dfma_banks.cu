// DFMA dispatch rate vs operand sourcing: 3 distinct per-thread register pairs vs one reused.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k3(double* out, const double* in, int iters) {   // a = fma(b, c, a), all distinct
    const int t = threadIdx.x;
    double a[8], b[8], c[8];
    for (int i = 0; i < 8; ++i) { a[i] = in[(t + i) & 63]; b[i] = in[(t + 2 * i + 1) & 63]; c[i] = in[(t + 3 * i + 2) & 63]; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(b[i], c[i], a[i]);
#pragma unroll
        for (int i = 0; i < 8; ++i) b[i] = fma(c[i], a[i], b[i]);
    }
    double s = 0; for (int i = 0; i < 8; ++i) s += a[i] + b[i] + c[i];
    if (s == 1.5) out[0] = s;
}
__global__ void k2(double* out, const double* in, int iters) {   // a = fma(x, c, a): x shared (reuse)
    const int t = threadIdx.x;
    double a[8], c[8], x = in[t & 63], y = in[(t + 7) & 63];
    for (int i = 0; i < 8; ++i) { a[i] = in[(t + i) & 63]; c[i] = in[(t + 3 * i + 2) & 63]; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(x, c[i], a[i]);
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(c[i], y, a[i]);
    }
    double s = 0; for (int i = 0; i < 8; ++i) s += a[i] + c[i];
    if (s == 1.5) out[0] = s;
}
__global__ void kimm(double* out, const double* in, int iters) {  // a = fma(a, c, 1.0): 2 regs + imm
    const int t = threadIdx.x;
    double a[8], c[8];
    for (int i = 0; i < 8; ++i) { a[i] = in[(t + i) & 63]; c[i] = in[(t + 3 * i + 2) & 63]; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(-a[i], c[i], 1.0);
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(-a[i], c[i], 1.0);
    }
    double s = 0; for (int i = 0; i < 8; ++i) s += a[i] + c[i];
    if (s == 1.5) out[0] = s;
}
template <class K> void run(const char* name, K kern, int warps_per_sm, int iters) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *d, *in; cudaMalloc(&d, 8); cudaMalloc(&in, 64 * 8);
    double h[64]; for (int i = 0; i < 64; ++i) h[i] = 1.0 + 1e-3 * i; cudaMemcpy(in, h, 512, cudaMemcpyHostToDevice);
    int threads = 32 * warps_per_sm; if (threads > 1024) threads = 1024;
    int blocks = sms * (32 * warps_per_sm / threads);
    kern<<<blocks, threads>>>(d, in, 10);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); kern<<<blocks, threads>>>(d, in, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-5s warps/SM=%2d  %.3e DFMA/s  (%s)\n", name, warps_per_sm, (double)blocks * threads * iters * 16 / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
}
int main() {
    for (int w : {8, 16, 32}) { run("3reg", k3, w, 20000); run("reuse", k2, w, 20000); run("imm", kimm, w, 20000); }
}
