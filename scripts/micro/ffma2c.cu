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
    for (int i = 0; i < P; ++i) { const int t1 = threadIdx.x & 1; cov[i] = io[16 + i + t1]; dg[i] = io[32 + i + t1]; df[i] = io[48 + i + t1]; ca[i] = io[64 + i + t1]; }
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

// A: FFMA2 recurrence + FFMA2 test with pre-negated column factor, AND of sign words (LOP3)
template <int P> __global__ void k_cellA(u64* io, int iters) {
    u64 cov[P], dg[P], df[P], ca[P];
#pragma unroll
    for (int i = 0; i < P; ++i) { const int t1 = threadIdx.x & 1; cov[i] = io[16 + i + t1]; dg[i] = io[32 + i + t1]; df[i] = io[48 + i + t1]; ca[i] = io[64 + i + t1]; }
    u64 dfi = io[threadIdx.x & 7], dgi = io[8 + (threadIdx.x & 7)], bi = io[80];
    unsigned acc = 0;
    for (int it = 0; it < iters; ++it) {
        unsigned andv = 0xffffffffu;
#pragma unroll
        for (int i = 0; i < P; ++i) {
            cov[i] = fma2(dfi, dg[i], cov[i]);
            cov[i] = fma2(df[i], dgi, cov[i]);
            u64 z = fma2(ca[i], bi, cov[i]);
            andv &= (unsigned)z & (unsigned)(z >> 32);
        }
        acc += andv >> 31;
        dfi += 0x10001; bi += 3;
    }
    u64 s = acc;
#pragma unroll
    for (int i = 0; i < P; ++i) s ^= cov[i];
    if (s == 12345) io[0] = s;
}
// B: scalar FFMA version of A
template <int C> __global__ void k_cellB(u64* io, int iters) {
    const float* f = (const float*)io;
    float cov[C], dg[C], df[C], ca[C];
#pragma unroll
    for (int i = 0; i < C; ++i) { const int t1 = threadIdx.x & 1; cov[i] = f[32 + i + t1]; dg[i] = f[64 + i + t1]; df[i] = f[96 + i + t1]; ca[i] = f[128 + i + t1]; }
    float dfi = f[threadIdx.x & 7], dgi = f[8 + (threadIdx.x & 7)], bi = f[160];
    unsigned acc = 0;
    for (int it = 0; it < iters; ++it) {
        unsigned andv = 0xffffffffu;
#pragma unroll
        for (int i = 0; i < C; ++i) {
            cov[i] = fmaf(dfi, dg[i], cov[i]);
            cov[i] = fmaf(df[i], dgi, cov[i]);
            float z = fmaf(ca[i], bi, cov[i]);
            andv &= __float_as_uint(z);
        }
        acc += andv >> 31;
        dfi += 1e-7f; bi += 1e-7f;
    }
    float s = acc;
#pragma unroll
    for (int i = 0; i < C; ++i) s += cov[i];
    if (s == 1.2345f) io[0] = 1;
}
// R: FFMA2 recurrence only
template <int P> __global__ void k_cellR(u64* io, int iters) {
    u64 cov[P], dg[P], df[P];
#pragma unroll
    for (int i = 0; i < P; ++i) { const int t1 = threadIdx.x & 1; cov[i] = io[16 + i + t1]; dg[i] = io[32 + i + t1]; df[i] = io[48 + i + t1]; }
    u64 dfi = io[threadIdx.x & 7], dgi = io[8 + (threadIdx.x & 7)];
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < P; ++i) {
            cov[i] = fma2(dfi, dg[i], cov[i]);
            cov[i] = fma2(df[i], dgi, cov[i]);
        }
        dfi += 0x10001;
    }
    u64 s = 0;
#pragma unroll
    for (int i = 0; i < P; ++i) s ^= cov[i];
    if (s == 12345) io[0] = s;
}

// T: scalar FFMA recurrence + FFMA test, balanced AND tree
template <int C> __global__ void k_cellT(u64* io, int iters) {
    const float* f = (const float*)io;
    float cov[C], dg[C], df[C], ca[C];
#pragma unroll
    for (int i = 0; i < C; ++i) { const int t1 = threadIdx.x & 1; cov[i] = f[32 + i + t1]; dg[i] = f[64 + i + t1]; df[i] = f[96 + i + t1]; ca[i] = f[128 + i + t1]; }
    float dfi = f[threadIdx.x & 7], dgi = f[8 + (threadIdx.x & 7)], bi = f[160];
    unsigned acc = 0;
    for (int it = 0; it < iters; ++it) {
        unsigned z[C];
#pragma unroll
        for (int i = 0; i < C; ++i) {
            cov[i] = fmaf(dfi, dg[i], cov[i]);
            cov[i] = fmaf(df[i], dgi, cov[i]);
            z[i] = __float_as_uint(fmaf(ca[i], bi, cov[i]));
        }
#pragma unroll
        for (int w = 1; w < C; w *= 2)
#pragma unroll
            for (int i = 0; i + w < C; i += 2 * w) z[i] &= z[i + w];
        acc += z[0] >> 31;
        dfi += 1e-7f; bi += 1e-7f;
    }
    float s = acc;
#pragma unroll
    for (int i = 0; i < C; ++i) s += cov[i];
    if (s == 1.2345f) io[0] = 1;
}
// V: scalar FFMA recurrence + FMUL threshold + FSETP OR-accumulated predicate
template <int C> __global__ void k_cellV(u64* io, int iters) {
    const float* f = (const float*)io;
    float cov[C], dg[C], df[C], ca[C];
#pragma unroll
    for (int i = 0; i < C; ++i) { const int t1 = threadIdx.x & 1; cov[i] = f[32 + i + t1]; dg[i] = f[64 + i + t1]; df[i] = f[96 + i + t1]; ca[i] = f[128 + i + t1]; }
    float dfi = f[threadIdx.x & 7], dgi = f[8 + (threadIdx.x & 7)], bi = f[160];
    unsigned acc = 0;
    for (int it = 0; it < iters; ++it) {
        bool pa = false, pb = false;
#pragma unroll
        for (int i = 0; i < C; ++i) {
            cov[i] = fmaf(dfi, dg[i], cov[i]);
            cov[i] = fmaf(df[i], dgi, cov[i]);
            const bool h = cov[i] >= ca[i] * bi;
            if (i & 1) pb |= h; else pa |= h;
        }
        acc += (pa | pb);
        dfi += 1e-7f; bi += 1e-7f;
    }
    float s = acc;
#pragma unroll
    for (int i = 0; i < C; ++i) s += cov[i];
    if (s == 1.2345f) io[0] = 1;
}
// P: FFMA2 recurrence + FFMA2 test, balanced AND tree
template <int P> __global__ void k_cellP(u64* io, int iters) {
    u64 cov[P], dg[P], df[P], ca[P];
#pragma unroll
    for (int i = 0; i < P; ++i) { const int t1 = threadIdx.x & 1; cov[i] = io[16 + i + t1]; dg[i] = io[32 + i + t1]; df[i] = io[48 + i + t1]; ca[i] = io[64 + i + t1]; }
    u64 dfi = io[threadIdx.x & 7], dgi = io[8 + (threadIdx.x & 7)], bi = io[80];
    unsigned acc = 0;
    for (int it = 0; it < iters; ++it) {
        u64 z[P];
#pragma unroll
        for (int i = 0; i < P; ++i) {
            cov[i] = fma2(dfi, dg[i], cov[i]);
            cov[i] = fma2(df[i], dgi, cov[i]);
            z[i] = fma2(ca[i], bi, cov[i]);
        }
#pragma unroll
        for (int w = 1; w < P; w *= 2)
#pragma unroll
            for (int i = 0; i + w < P; i += 2 * w) z[i] &= z[i + w];
        acc += ((unsigned)z[0] & (unsigned)(z[0] >> 32)) >> 31;
        dfi += 0x10001; bi += 3;
    }
    u64 s = acc;
#pragma unroll
    for (int i = 0; i < P; ++i) s ^= cov[i];
    if (s == 12345) io[0] = s;
}
// Q: recurrence only, scalar FFMA
template <int C> __global__ void k_cellQ(u64* io, int iters) {
    const float* f = (const float*)io;
    float cov[C], dg[C], df[C];
#pragma unroll
    for (int i = 0; i < C; ++i) { const int t1 = threadIdx.x & 1; cov[i] = f[32 + i + t1]; dg[i] = f[64 + i + t1]; df[i] = f[96 + i + t1]; }
    float dfi = f[threadIdx.x & 7], dgi = f[8 + (threadIdx.x & 7)];
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < C; ++i) {
            cov[i] = fmaf(dfi, dg[i], cov[i]);
            cov[i] = fmaf(df[i], dgi, cov[i]);
        }
        dfi += 1e-7f;
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < C; ++i) s += cov[i];
    if (s == 1.2345f) io[0] = 1;
}
int main() {
    u64* d; cudaMalloc(&d, 4096);
    u64 h[256]; for (int i = 0; i < 256; ++i) { float f[2] = {1.0f + i * 1e-3f, 0.5f - i * 1e-3f}; memcpy(&h[i], f, 8); }
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    int W[] = {8, 16, 20};
    for (int w : W) {
        run("B8", k_cellB<8>, 8, 8, w, 20000, d);
        run("T8", k_cellT<8>, 8, 8, w, 20000, d);
        run("T16", k_cellT<16>, 16, 16, w, 10000, d);
        run("V8", k_cellV<8>, 8, 8, w, 20000, d);
        run("V16", k_cellV<16>, 16, 16, w, 10000, d);
        run("P4", k_cellP<4>, 4, 8, w, 20000, d);
        run("P8", k_cellP<8>, 8, 16, w, 10000, d);
        run("Q8", k_cellQ<8>, 8, 8, w, 20000, d);
        run("Q16", k_cellQ<16>, 16, 16, w, 10000, d);
    }
    return 0;
}
