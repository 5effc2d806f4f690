// The packed FP32 walk's row step (filter32.cu k_tile32) in isolation, features added one at a
// time, to see where its time goes: cells per SM per clock on one B200.
//   REC: the 16 FFMA2 of the recurrence      TEST: + 8 FFMA2 bound tests
//   TREE: + LOP3 sign tree                   BR: + per-row ISETP/BRA into a (never taken) slow path
//   SH: + the ring's 4 SHFL per row          LD: + row factors and column factors from shared memory
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o walkrow walkrow.cu && ./walkrow
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk2(float lo, float hi) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ u64 fma2(u64 x, u64 y, u64 z) { u64 d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x), "l"(y), "l"(z)); return d; }
__device__ __forceinline__ u64 bc2(float x) { return pk2(x, x); }
__device__ __forceinline__ unsigned and3(unsigned x, unsigned y, unsigned z) {
    unsigned d; asm("lop3.b32 %0, %1, %2, %3, 0x80;" : "=r"(d) : "r"(x), "r"(y), "r"(z)); return d;
}
constexpr int DP = 8, GRP = 8, CQS = 33;

template <int F_TEST, int F_TREE, int F_BR, int F_SH, int F_LD>
__global__ void __launch_bounds__(32, 12) k_walk(const float4* rows, const float4* cqs, u64* out, int iters) {
    __shared__ float4 srow[GRP];
    __shared__ float4 scq[GRP * CQS];
    __shared__ unsigned short msk[32 * GRP];
    const int lane = threadIdx.x;
    if (lane < GRP) srow[lane] = rows[lane];
    for (int k = lane; k < GRP * CQS; k += 32) scq[k] = cqs[k];
    __syncwarp();
    u64 cov[DP], F[DP], G[DP], NA[DP];
#pragma unroll
    for (int s = 0; s < DP; ++s) {
        cov[s] = pk2(1e-3f * s, 2e-3f * s); F[s] = pk2(1e-4f, 2e-4f); G[s] = pk2(3e-4f, 1e-4f);
        NA[s] = pk2(-1e30f, -1e30f);
    }
    float4 rr = rows[lane & 7];
    float4 prn = srow[0];
    unsigned acc = 0, nslow = 0, tacc = ~0u;
    for (int it = 0; it < iters; ++it) {
        u64 NAg[GRP];
        if (F_LD == 5) {   // the 8 entering columns' thresholds of this lane, once per group
#pragma unroll
            for (int kk = 0; kk < GRP; ++kk) {
                const float4 cq = scq[kk * CQS + lane];
                const float w = srow[kk].w;
                NAg[kk] = pk2(fmaxf(-cq.x, __fmul_ru(-w, cq.y)), fmaxf(-cq.z, __fmul_ru(-w, cq.w)));
            }
        }
#pragma unroll
        for (int kk = 0; kk < GRP; ++kk) {
            // F_LD: 1 row + column factors from smem, 2 column factors only, 3 row factors only,
            // 4 as 1 with the row factors prefetched one row ahead
            float4 pr;
            if (F_LD == 4) { pr = prn; prn = srow[(kk + 1) % GRP]; }
            else pr = (F_LD == 1 || F_LD == 3 || F_LD == 5) ? srow[kk] : rr;
            const int q = (kk + DP - 1) % DP;
            if (F_SH) {
                F[q] = __shfl_sync(0xffffffffu, F[q], (lane + 1) & 31);
                G[q] = __shfl_sync(0xffffffffu, G[q], (lane + 1) & 31);
            }
            if (F_LD == 5) NA[q] = NAg[kk];
            if (F_LD == 1 || F_LD == 2 || F_LD == 4) {
                const float4 cq = scq[kk * CQS + lane];
                NA[q] = pk2(fmaxf(-cq.x, __fmul_ru(-pr.w, cq.y)), fmaxf(-cq.z, __fmul_ru(-pr.w, cq.w)));
            }
            unsigned z[16];
#pragma unroll
            for (int s = 0; s < DP; ++s) {
                const int p = (s + kk) % DP;
                cov[s] = fma2(bc2(pr.x), G[p], cov[s]);
                cov[s] = fma2(F[p], bc2(pr.y), cov[s]);
                if (F_TEST) {
                    const u64 zz = fma2(NA[p], bc2(pr.z), cov[s]);
                    z[s] = (unsigned)zz; z[s + 8] = (unsigned)(zz >> 32);
                }
            }
            if (F_TEST && F_TREE) {
                const unsigned t0 = and3(z[0], z[8], z[1]), t1 = and3(z[9], z[2], z[10]);
                const unsigned t2 = and3(z[3], z[11], z[4]), t3 = and3(z[12], z[5], z[13]);
                const unsigned t4 = and3(z[6], z[14], z[7]);
                const unsigned t = and3(and3(t0, t1, t2), t3, and3(t4, z[15], ~0u));
                tacc &= t;
                // F_BR: 1 per-row divergent branch, 2 per-row uniform branch (vote), 3 divergent every
                // 2 rows, 4 uniform every 2 rows, 5 divergent every 4 rows, 6 divergent every 8 rows
                const int every = F_BR == 3 || F_BR == 4 ? 2 : F_BR == 5 ? 4 : F_BR == 6 ? 8 : 1;
                const bool uni = F_BR == 2 || F_BR == 4;
                const bool at = (kk % every) == every - 1;
                bool take = false;
                if (F_BR && at) take = uni ? __any_sync(0xffffffffu, (int)tacc >= 0) : (int)tacc >= 0;
                if (F_BR && at) tacc = ~0u;
                if (F_BR) {
                    if (__builtin_expect(take, 0)) {     // never taken with these data
                        unsigned m = 0;
#pragma unroll
                        for (int s = 0; s < DP; ++s) m |= ((unsigned)cov[s] >> 31) << s;
                        msk[lane * GRP + kk] = (unsigned short)m;
                        ++nslow;
                    }
                } else {
                    acc += t >> 31;
                }
            }
        }
        rr.x += 1e-7f;
    }
    u64 h = acc + nslow;
#pragma unroll
    for (int s = 0; s < DP; ++s) h ^= cov[s] ^ F[s] ^ G[s];
    if (h == 0x12345) out[0] = h + msk[lane];
}

// two lengths per walk: cov_{m+1} = cov_m + w dz_i dz_j (Welford), its own test; per row
// 16 rec + 8 test + 8 ext + 8 test FFMA2, a 32-value sign tree, one branch, 6 SHFL, 3 LDS
template <int F_BR>
__global__ void __launch_bounds__(32, 12) k_walk2(const float4* rows, const float4* cqs, u64* out, int iters) {
    __shared__ float4 srow[GRP], srow2[GRP];
    __shared__ float4 scq[GRP * CQS], scq2[GRP * CQS];
    __shared__ unsigned short msk[32 * GRP];
    const int lane = threadIdx.x;
    if (lane < GRP) { srow[lane] = rows[lane]; srow2[lane] = rows[lane]; }
    for (int k = lane; k < GRP * CQS; k += 32) { scq[k] = cqs[k]; scq2[k] = cqs[k]; }
    __syncwarp();
    u64 cov[DP], F[DP], G[DP], Z[DP], NA[DP], NB[DP];
#pragma unroll
    for (int s = 0; s < DP; ++s) {
        cov[s] = pk2(1e-3f * s, 2e-3f * s); F[s] = pk2(1e-4f, 2e-4f); G[s] = pk2(3e-4f, 1e-4f);
        Z[s] = pk2(2e-4f, 1e-4f); NA[s] = pk2(-1e30f, -1e30f); NB[s] = NA[s];
    }
    unsigned acc = 0, nslow = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < GRP; ++kk) {
            const float4 pr = srow[kk], pr2 = srow2[kk];
            const int q = (kk + DP - 1) % DP;
            F[q] = __shfl_sync(0xffffffffu, F[q], (lane + 1) & 31);
            G[q] = __shfl_sync(0xffffffffu, G[q], (lane + 1) & 31);
            Z[q] = __shfl_sync(0xffffffffu, Z[q], (lane + 1) & 31);
            const float4 cq = scq[kk * CQS + lane], cq2 = scq2[kk * CQS + lane];
            NA[q] = pk2(fmaxf(-cq.x, __fmul_ru(-pr.w, cq.y)), fmaxf(-cq.z, __fmul_ru(-pr.w, cq.w)));
            NB[q] = pk2(fmaxf(-cq2.x, __fmul_ru(-pr2.w, cq2.y)), fmaxf(-cq2.z, __fmul_ru(-pr2.w, cq2.w)));
            unsigned z[32];
#pragma unroll
            for (int s = 0; s < DP; ++s) {
                const int p = (s + kk) % DP;
                cov[s] = fma2(bc2(pr.x), G[p], cov[s]);
                cov[s] = fma2(F[p], bc2(pr.y), cov[s]);
                const u64 zz = fma2(NA[p], bc2(pr.z), cov[s]);
                const u64 c1 = fma2(bc2(pr2.x), Z[p], cov[s]);
                const u64 zz2 = fma2(NB[p], bc2(pr2.z), c1);
                z[s] = (unsigned)zz; z[s + 8] = (unsigned)(zz >> 32);
                z[s + 16] = (unsigned)zz2; z[s + 24] = (unsigned)(zz2 >> 32);
            }
            unsigned t[11];
#pragma unroll
            for (int u = 0; u < 10; ++u) t[u] = and3(z[3 * u], z[3 * u + 1], z[3 * u + 2]);
            t[10] = and3(z[30], z[31], ~0u);
            const unsigned t1 = and3(t[0], t[1], t[2]), t2 = and3(t[3], t[4], t[5]), t3 = and3(t[6], t[7], t[8]);
            const unsigned tt = and3(and3(t1, t2, t3), t[9], t[10]);
            if (F_BR) {
                if (__builtin_expect((int)tt >= 0, 0)) {
                    unsigned m = 0;
#pragma unroll
                    for (int s = 0; s < DP; ++s) m |= ((unsigned)cov[s] >> 31) << s;
                    msk[lane * GRP + kk] = (unsigned short)m;
                    ++nslow;
                }
            } else acc += tt >> 31;
        }
    }
    u64 h = acc + nslow;
#pragma unroll
    for (int s = 0; s < DP; ++s) h ^= cov[s] ^ F[s] ^ G[s] ^ Z[s];
    if (h == 0x12345) out[0] = h + msk[lane];
}

template <int BR>
void run2(const char* name, int warps_per_sm, float4* rows, float4* cqs, u64* out) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * warps_per_sm, iters = 4000;
    k_walk2<BR><<<blocks, 32>>>(rows, cqs, out, 10);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0); k_walk2<BR><<<blocks, 32>>>(rows, cqs, out, iters); cudaEventRecord(e1);
        cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const double upd = (double)blocks * 32 * 16 * GRP * iters * 2;   // cell-lengths
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-26s warps/SM=%2d  %.3e cell-lengths/s  %.2f per SM/clk\n", name, warps_per_sm,
           upd / (best * 1e-3), upd / (best * 1e-3) / sms / (clk * 1e3));
}

template <int A, int B, int C, int D, int E>
void run(const char* name, int warps_per_sm, float4* rows, float4* cqs, u64* out) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * warps_per_sm, iters = 4000;
    k_walk<A, B, C, D, E><<<blocks, 32>>>(rows, cqs, out, 10);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0); k_walk<A, B, C, D, E><<<blocks, 32>>>(rows, cqs, out, iters); cudaEventRecord(e1);
        cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const double cells = (double)blocks * 32 * 16 * GRP * iters;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-26s warps/SM=%2d  %.3e cells/s  %.2f cells/SM/clk (@%.3f GHz)  %.1f%% of 3-FMA roofline\n", name,
           warps_per_sm, cells / (best * 1e-3), cells / (best * 1e-3) / sms / (clk * 1e3), clk * 1e-6,
           100.0 * cells / (best * 1e-3) / sms / (clk * 1e3) / (128.0 / 3.0));
}

int main() {
    float4 *rows, *cqs; u64* out;
    cudaMalloc(&rows, 8 * sizeof(float4)); cudaMalloc(&cqs, 8 * 33 * sizeof(float4)); cudaMalloc(&out, 64);
    float4 hr[8], hc[8 * 33];
    for (int k = 0; k < 8; ++k) hr[k] = make_float4(1e-3f, 2e-3f, 1.0f, 0.5f);
    for (int k = 0; k < 8 * 33; ++k) hc[k] = make_float4(1e30f, 1.0f, 1e30f, 1.0f);
    cudaMemcpy(rows, hr, sizeof(hr), cudaMemcpyHostToDevice); cudaMemcpy(cqs, hc, sizeof(hc), cudaMemcpyHostToDevice);
    for (int w : {8, 10, 12}) {
        run2<1>("TWO LENGTHS full", w, rows, cqs, out);
        run2<0>("TWO LENGTHS no br", w, rows, cqs, out);
    }
    for (int w : {12, 16}) {
        run<0, 0, 0, 0, 0>("rec (16 FFMA2)", w, rows, cqs, out);
        run<1, 1, 0, 0, 0>("+tree", w, rows, cqs, out);
        run<1, 1, 1, 0, 0>("+tree+branch", w, rows, cqs, out);
        run<1, 1, 1, 1, 0>("+tree+branch+shfl", w, rows, cqs, out);
        run<1, 1, 1, 1, 1>("+tree+branch+shfl+lds", w, rows, cqs, out);
        run<1, 1, 0, 1, 1>("+tree+shfl+lds (no br)", w, rows, cqs, out);
        run<1, 1, 1, 1, 5>("full, NA precomputed/group", w, rows, cqs, out);
        run<1, 1, 1, 1, 2>("full, cq from smem only", w, rows, cqs, out);
        run<1, 1, 1, 1, 3>("full, rows from smem only", w, rows, cqs, out);
        run<1, 1, 1, 1, 4>("full, rows prefetched", w, rows, cqs, out);
        run<1, 1, 6, 1, 4>("full, rows pf, br/8 rows", w, rows, cqs, out);
        run<1, 1, 2, 1, 1>("full, uniform br/row", w, rows, cqs, out);
        run<1, 1, 3, 1, 1>("full, br per 2 rows", w, rows, cqs, out);
        run<1, 1, 4, 1, 1>("full, uniform br/2 rows", w, rows, cqs, out);
        run<1, 1, 5, 1, 1>("full, br per 4 rows", w, rows, cqs, out);
        run<1, 1, 6, 1, 1>("full, br per 8 rows", w, rows, cqs, out);
    }
    return 0;
}
