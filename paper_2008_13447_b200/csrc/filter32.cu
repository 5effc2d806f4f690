// filter32.cu -- the per-length tile walk with an FP32 bound filter, and the exact FP64
// evaluation of the cells it passes (1-best mode, lengths after a run's first).
//
// Same job as profile.cu's k_tile<false> + k_log_merge: every non-trivial cell (i, j) whose key
// r = 1 - cov(i,j) inv_i inv_j could beat the bound U of its row or its column must be folded
// into acc with its exact key. The walk needs only an approximate covariance to decide that,
// so it runs the diagonal recurrence (SCAMP form)
//     cov(i,j) = cov(i-1,j-1) + df_i dg_j + df_j dg_i
// in FP32 from each tile's FP64 seed, with a rigorous error slack eps folded into the seed:
//   |cov32 - cov| <= u [(2K + 1) Sr Sc + 3.02 K (DFr DGc + DFc DGr)] (1 + 1%),  u = 2^-24,
// K = S + 1 walked rows, Sr/Sc/DF/DG the maxima of the window norms s = ||x|| and of |df|, |dg|
// over the tile's rows / columns (per row: two FFMA roundings and the FP32-rounded inputs;
// |cov| <= s_i s_j by Cauchy-Schwarz). A cell passes when cov32 + eps >= cA_j b_i, where cA_j b_i <= q(max(U_i,U_j))
// s_i s_j (profile.cu's covariance-domain threshold, in FP32 rounded down): one FFMA per cell,
// its sign bit ANDed over the lane's cells. Passing cells are grouped into runs along their
// diagonals (the lane tracks which of its diagonals passed at its previous flagged row) and
// logged; k_runs evaluates each run exactly: a centred FP64 dot product at the run's first cell,
// the FP64 recurrence (as an ordered warp scan) along the run, the reference key formula, the
// exact hi(r) <= U tests and the 128-bit CAS fold. Nothing approximate reaches acc.
//
// Lane geometry: each lane owns D2 consecutive diagonals; a tile is 32 D2 diagonals x S rows
// (D2 = 16: two neighbouring FP64 tiles of the same row segment, whose FP64 seeds it reads and
// carries to the next length with the FP64 kernel's own Welford step -- bit-identical seeds).

#include "vlmp_internal.cuh"

namespace vlmp_impl {

#ifndef VLMP_D2
#define VLMP_D2 16
#endif
constexpr int D2 = VLMP_D2;                 // diagonals per lane (FP32 walk)
[[maybe_unused]] constexpr int BAND2 = 32 * D2;   // diagonals per FP32 tile (scalar walk)
[[maybe_unused]] constexpr int LPT = BAND / D2;     // lanes per FP64 tile (scalar walk)
constexpr int GR2 = D2;                     // rows per staging group (ring returns to phase)
constexpr int CQS = 33;                     // staged column-factor row stride (entries)
static_assert(D2 == 8 || D2 == 16, "D2: 8 or 16");
#ifndef VLMP_PACKED
#define VLMP_PACKED 1            // two-band packed walk (FFMA2 on band pairs); 0: scalar FFMA, 16 diagonals per lane
#endif
constexpr int WIN = VLMP_PACKED ? 8 : D2;   // rows a column meets in one lane (the w window)
#ifndef VLMP_PAIR_SEP
#define VLMP_PAIR_SEP 2          // packed walk: band B = band A + VLMP_PAIR_SEP bands (1: adjacent)
#endif
#ifndef VLMP_PRIO
#define VLMP_PRIO 1              // the short per-length kernels launch at the highest priority (two chains)
#endif
#ifndef VLMP_PF_RING
#define VLMP_PF_RING 1           // packed walk: entering columns' {df, dg} from a second sliding ring (0: lane-to-lane shuffles)
#endif
#ifndef VLMP_MASK_SHF
#define VLMP_MASK_SHF 1          // packed walk: a flagged row's mask from 8 FFMA2 + one funnel shift per cell
#endif
#ifndef VLMP_FILTER32_WARPS_PER_SM
#define VLMP_FILTER32_WARPS_PER_SM 16   // 128 registers: no spills (20 warps at 96 spill the staging plan)
#endif
#ifndef VLMP_RUN_MAXLEN
#define VLMP_RUN_MAXLEN 64       // packed walk: longer runs are logged in pieces of this many cells (k_runs: one warp per piece)
#endif
#ifndef VLMP_RUN_GAP
#define VLMP_RUN_GAP 28          // packed walk: runs of one diagonal at most this many rows apart are logged as one
#endif

// ---------------------------------------------------------------------------------
// per-length FP32 factors (after k_bound2 wrote U): p32 = {df, dg, b, w}, cq = {a, b}, where
// b = s 2^-k (rounded down), a = q(U) b, w = q(max U over rows o .. o+D2-1); +inf factors for
// invalid windows. Block maxima over 256 offsets for the walk's error slack, in
// magblk[3 * nb]: [0, nb) the window norm ||x_o|| 2^-k (from the prefix sums plus their
// rounding allowance), [nb, 2 nb) |df_o| 2^-k, [2 nb, 3 nb) |dg_o| 2^-k (all rounded up).
struct Prep32Args {
    const Prm* prm; const double* cum; const double* cum2;
    float4* p32; float2* cq; unsigned* magblk; long long nb;
    long long N, A; int m; double sscale; int* forced;
    float4* cq4;   // packed walk: {a_o, b_o, a_o', b_o'}, o' = o + PSEP (nullptr: not built)
    float4* pf4;   // packed walk, PSEP > 256: {df_o, df_o', dg_o, dg_o'} (lane 31's fresh pair)
};

// the column factors (cA, b) of offset o: +inf for windows past N or undefined; a forced offset
// (bound too weak for the covariance-domain test, or b out of range) passes every cell -- as a
// column cA = -inf (z = +inf), as a row b = NaN (z = NaN, sign bit clear); k_runs evaluates
// them exactly
__device__ __forceinline__ void col_factors(const Prm& p, long long o, long long N, double sscale,
                                            float& ca, float& b, bool& forced) {
    ca = INFINITY; b = INFINITY; forced = false;
    if (o < N && p.inv == p.inv) {
        b = qscale(p.inv, sscale);
        ca = __double2float_rd(qfac(p.U) * (double)b);
        if (q_forced(p, sscale)) { ca = -INFINITY; b = __int_as_float(0x7FC00000); forced = true; }
    }
}

constexpr int PSEP = VLMP_PAIR_SEP * BAND;   // diagonal offset of a packed tile's band B

__global__ void __launch_bounds__(256) k_prep32(Prep32Args a) {
    const long long o = blockIdx.x * 256LL + threadIdx.x;
    float msv = 0.f, mdf = 0.f, mdg = 0.f;
    if (o < a.A) {
        const Prm p = a.prm[o];
        const float df = (float)(p.df * a.sscale), dg = (float)(p.dg * a.sscale);
        float b, w = 3.0e38f, ca;
        bool forced;
        col_factors(p, o, a.N, a.sscale, ca, b, forced);
        if (forced && a.forced) atomicOr(a.forced, 1);
        if (a.cq4 && o + PSEP < a.A) {
            // packed walk: the band pair (o, o + PSEP) in one 16-byte entry, so the walk stages
            // each entering pair with one cp.async
            const Prm p2 = a.prm[o + PSEP];
            float ca2, b2; bool f2;
            col_factors(p2, o + PSEP, a.N, a.sscale, ca2, b2, f2);
            a.cq4[o] = make_float4(ca, b == b ? b : 1.0f, ca2, b2 == b2 ? b2 : 1.0f);
            if (a.pf4) a.pf4[o] = make_float4(df, (float)(p2.df * a.sscale), dg, (float)(p2.dg * a.sscale));
        }
        if (o < a.N) {
            float uw = -INFINITY;
#pragma unroll
            for (int k = 0; k < WIN; ++k)
                if (o + k < a.N) uw = fmaxf(uw, a.prm[o + k].U);
            if (uw != -INFINITY) w = __double2float_rd(qfac(uw));
            const double L = (double)a.m;
            const double s = a.cum[o + a.m] - a.cum[o], ss = a.cum2[o + a.m] - a.cum2[o];
            const double mu = s / L;
            const double vu = fmax(ss / L - mu * mu, 0.0) + 0x1p-44 * (fabs(ss) / L + mu * mu);
            msv = __double2float_ru(sqrt(vu * L) * a.sscale * (1.0 + 0x1p-20));
            mdf = __double2float_ru(fabs(p.df) * a.sscale * (1.0 + 0x1p-20));
            mdg = __double2float_ru(fabs(p.dg) * a.sscale * (1.0 + 0x1p-20));
        }
        a.p32[o] = make_float4(df, dg, b, w);
        a.cq[o] = make_float2(ca, b == b ? b : 1.0f);
    }
    // one 256-offset block per CTA: maxima over the block (non-negative floats order as integers)
    const unsigned v0 = __reduce_max_sync(FULLMASK, __float_as_uint(msv));
    const unsigned v1 = __reduce_max_sync(FULLMASK, __float_as_uint(mdf));
    const unsigned v2 = __reduce_max_sync(FULLMASK, __float_as_uint(mdg));
    __shared__ unsigned wm[3][8];
    if ((threadIdx.x & 31) == 0) { wm[0][threadIdx.x >> 5] = v0; wm[1][threadIdx.x >> 5] = v1; wm[2][threadIdx.x >> 5] = v2; }
    __syncthreads();
    if (threadIdx.x < 3) {
        unsigned r = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) r = max(r, wm[threadIdx.x][k]);
        a.magblk[threadIdx.x * a.nb + blockIdx.x] = r;
    }
}

// ---------------------------------------------------------------------------------
struct Tile32Args {
    const float4* p32; const float2* cq; const unsigned* magblk; long long nb;
    const double* __restrict__ tn; const double* __restrict__ mu; double* seeds;
    const int2* tiles;      // FP64 tile list (band, segment)
    const int4* tiles32;    // FP32 tiles: {FP64 tile of the lower band, of the upper band or -1,
                            //  band and segment of the lower one}
    Run* runs; unsigned long long* run_count; long long run_cap;
    unsigned long long* counters;   // [2] flagged lane-rows, [3] runs
    const int* forced;
    long long N, dlo; int n_tiles32, S, m, e, update_seeds;
    double sscale;
    unsigned long long* span;   // [2]: first CTA start, last CTA end (ns; nullptr: not timed)
    const float4* cq4;      // packed walk: band-pair column factors
    const float4* pf4;      // packed walk, PSEP > 256: band-pair {df, df', dg, dg'}
};

struct Smem32 {
    float4 row[2][GR2];          // {df, dg, b, w} of the group's rows
    float4 fresh[2][GR2];        // the column entering lane 31's ring at each row of the group
    float2 cq[2][GR2 * CQS];     // (a, b) of the column entering lane L at row kk: [kk * 33 + L]
    unsigned short rs[32 * D2];  // run start (row within the tile) per lane and diagonal
    unsigned short msk[32 * GR2];   // exact FP32 pass masks of a lane's flagged rows in a group
};

struct Plan32 {
    const char* src_rf; unsigned dst_rf;   // rows (lanes < GR2) / fresh columns (lanes 16..)
    const char* src_cq; unsigned dst_cq;   // entering column factors, D2 entries per lane
};
constexpr unsigned RF_BUF = sizeof(float4) * GR2;
constexpr unsigned CQ2_BUF = sizeof(float2) * GR2 * CQS;

template <int OFF_D, int OFF_S, int BYTES>
__device__ __forceinline__ void cpa(unsigned d, const char* s) {
    if (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0+%2], [%1+%3], 16;\n" :: "r"(d), "l"(s), "n"(OFF_D), "n"(OFF_S) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0+%2], [%1+%3], 8;\n" :: "r"(d), "l"(s), "n"(OFF_D), "n"(OFF_S) : "memory");
}
// 16 bytes through L1: column factors are re-read by the neighbouring tiles on the SM
template <int OFF_D, int OFF_S>
__device__ __forceinline__ void cpa_l1(unsigned d, const char* s) {
    asm volatile("cp.async.ca.shared.global [%0+%2], [%1+%3], 16;\n" :: "r"(d), "l"(s), "n"(OFF_D), "n"(OFF_S) : "memory");
}

template <int K>
__device__ __forceinline__ void stage_cq2(unsigned dc, const char* sc) {
    if constexpr (K < D2) {
        // entry f = lane + 32 K -> (kk, L) = (f % D2, f / D2) -> slot kk * 33 + L
        cpa<K * (32 / D2) * 8, K * 256, 8>(dc, sc);
        stage_cq2<K + 1>(dc, sc);
    }
}

__device__ __forceinline__ void stage32(const Plan32& p, int g, int b, int lane) {
    const long long gr = (long long)g * (GR2 * sizeof(float4));
    if ((lane & 15) < GR2) cpa<0, 0, 16>(p.dst_rf + (unsigned)b * RF_BUF, p.src_rf + gr);
    stage_cq2<0>(p.dst_cq + (unsigned)b * CQ2_BUF, p.src_cq + (long long)g * (GR2 * sizeof(float2)));
    cp_async_commit();
}

// the flagged-row mask is recomputed from cov / cA (live anyway) instead of keeping the row's
// z values alive across rows: volatile, so the compiler cannot merge it with the fast path's FMAs
__device__ __forceinline__ float fma_nocse(float a, float b, float c) {
    float d;
    asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

#if !VLMP_PACKED
__global__ void __launch_bounds__(32, VLMP_FILTER32_WARPS_PER_SM) k_tile32(Tile32Args a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem32& sm = *reinterpret_cast<Smem32*>(smem_raw);
    const int lane = threadIdx.x;
    const int wid = blockIdx.x;
    if (wid >= a.n_tiles32) return;
    const int4 t4 = a.tiles32[wid];
    const int2 pr2 = make_int2(t4.x, t4.y);
    const int2 tA = make_int2(t4.z, t4.w);
    const long long d0 = a.dlo + (long long)tA.x * BAND;
    const long long i0 = (long long)tA.y * a.S;
    const long long rows_valid = a.N - d0 - i0;
    // halves (FP64 tiles): empty or entirely trivial ones stay so at later lengths
    const bool liveA = rows_valid > 0 && d0 + BAND - 1 >= a.e;
    const bool liveB = pr2.y >= 0 && rows_valid - BAND > 0 && d0 + 2 * BAND - 1 >= a.e;
    if (!liveA && !liveB) return;
    const int half = lane / LPT;
    const bool live = half == 0 ? liveA : liveB;
    const int nrows = (int)(rows_valid < a.S ? rows_valid : a.S);
    const int ngroups = (nrows + GR2 - 1) / GR2;
    const long long cbase = i0 + d0 + (long long)D2 * lane;   // column of slot 0 at row i0

    // ---- FP32 error slack. Per walked row (two FFMA over FP32-rounded df, dg) the covariance
    // error grows by at most 2u|cov| + 3.02u(|df_i dg_j| + |df_j dg_i|), u = 2^-24, with
    // |cov| <= s_i s_j (Cauchy-Schwarz); S + 1 rows (with the seed pre-adjust) plus the seed's
    // conversion, over the maxima of s, |df|, |dg| on the tile's rows and columns.
    float eps;
    {
        const long long rb0 = i0 >> 8, rb1 = (i0 + nrows - 1) >> 8;
        const long long cb0 = (i0 + d0) >> 8, cb1 = (i0 + nrows - 1 + d0 + BAND2 - 1) >> 8;
        unsigned r[3] = {0, 0, 0}, c[3] = {0, 0, 0};
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            for (long long k = rb0 + lane; k <= rb1; k += 32) r[q] = max(r[q], a.magblk[q * a.nb + k]);
            for (long long k = cb0 + lane; k <= cb1; k += 32) c[q] = max(c[q], a.magblk[q * a.nb + k]);
            r[q] = __reduce_max_sync(FULLMASK, r[q]);
            c[q] = __reduce_max_sync(FULLMASK, c[q]);
        }
        const double Sr = __uint_as_float(r[0]), DFr = __uint_as_float(r[1]), DGr = __uint_as_float(r[2]);
        const double Sc = __uint_as_float(c[0]), DFc = __uint_as_float(c[1]), DGc = __uint_as_float(c[2]);
        const double K = (double)a.S + 1.0;
        const double bound = 0x1p-24 * 1.01 * ((2.0 * K + 1.0) * 1.001 * Sr * Sc + 3.02 * K * (DFr * DGc + DFc * DGr));
        eps = __double2float_ru(bound);
    }

    // ---- seeds: FP64 cov at row i0 (carried to length m+1 in place, as k_tile does). All
    // loads first (one batch), then the Welford step and the stores.
    float cov[D2];
    {
        const int w64 = half == 0 ? pr2.x : pr2.y;
        double* __restrict__ seedp = a.seeds + (long long)(live ? w64 : 0) * BAND + (lane % LPT) * D2;
        const double s2 = a.sscale * a.sscale;
        double c64[D2];
#pragma unroll
        for (int s = 0; s < D2; ++s) c64[s] = live ? seedp[s] : 0.0;
        if (live && a.update_seeds) {
            const double wgt = (double)a.m / (double)(a.m + 1);
            const double xi = (a.tn[i0 + a.m] - a.mu[i0]) * wgt;
            double xs[D2];
#pragma unroll
            for (int s = 0; s < D2; ++s) xs[s] = a.tn[cbase + s + a.m] - a.mu[cbase + s];
#pragma unroll
            for (int s = 0; s < D2; ++s) seedp[s] = fma(xi, xs[s], c64[s]);
        }
#pragma unroll
        for (int s = 0; s < D2; ++s)
            cov[s] = (live && d0 + D2 * lane + s >= a.e) ? __fadd_ru((float)(c64[s] * s2), eps) : -INFINITY;
    }

    // ---- column ring (profile.cu tile_body): phys p < D2-1 = slot p at row i0, phys D2-1 =
    // the column leaving slot 0 at row i0-1; cA = min(a_c, w_entry b_c) per resident column
    float cdf[D2], cdg[D2], cA[D2];
    {
        const float w0 = a.p32[i0].w;
#pragma unroll
        for (int s = 0; s < D2; ++s) {
            const long long c = s < D2 - 1 ? cbase + s : cbase - 1;
            const float4 pc = a.p32[c];
            cdf[s] = pc.x; cdg[s] = pc.y;
            const float2 q = a.cq[c];
            cA[s] = fminf(q.x, __fmul_rd(w0, q.y));
        }
        // pre-adjust so that the uniform recurrence at row i0 reproduces the seed
        const float4 pr = a.p32[i0];
        const float4 pl = a.p32[cbase + D2 - 1];
#pragma unroll
        for (int s = 0; s < D2; ++s) {
            const float df = s < D2 - 1 ? cdf[s] : pl.x, dg = s < D2 - 1 ? cdg[s] : pl.y;
            cov[s] = fmaf(-df, pr.y, cov[s]);
            cov[s] = fmaf(-pr.x, dg, cov[s]);
        }
    }

    // ---- staging plan
    Plan32 plan;
    {
        const int q = lane & 15;
        if (lane < 16) {
            plan.src_rf = reinterpret_cast<const char*>(a.p32 + i0 + q);
            plan.dst_rf = (unsigned)__cvta_generic_to_shared(&sm.row[0][q < GR2 ? q : 0]);
        } else {
            plan.src_rf = reinterpret_cast<const char*>(a.p32 + i0 + q + d0 + BAND2 - 1);
            plan.dst_rf = (unsigned)__cvta_generic_to_shared(&sm.fresh[0][q < GR2 ? q : 0]);
        }
        plan.src_cq = reinterpret_cast<const char*>(a.cq + i0 + d0 + D2 - 1 + lane);
        plan.dst_cq = (unsigned)__cvta_generic_to_shared(&sm.cq[0][(lane % D2) * CQS + lane / D2]);
    }

    // ---- runs. A flagged row's exact FP32 mask is recomputed at the next row (before the ring
    // moves on) and parked in shared memory; once per group the lane folds its flagged rows,
    // in row order, into runs: open = diagonals that passed at its last flagged row last_r.
    unsigned open = 0;
    int last_r = -2;
    unsigned nslow = 0;
    unsigned short* rs = sm.rs + lane * D2;
    unsigned short* msk = sm.msk + lane * GR2;
    auto emit = [&](int s, int r_start, int r_end) {
        const unsigned long long at = atomicAdd(a.run_count, 1ull);
        if ((long long)at < a.run_cap) {
            Run rr;
            rr.i = (int)(i0 + r_start); rr.j = rr.i + (int)(d0 + D2 * lane) + s; rr.len = r_end - r_start + 1;
            rr.pad = 0;
            a.runs[at] = rr;
        }
    };
    // rows gbase + t for the set bits t of flags (ascending), masks in msk[t]
    auto fold_rows = [&](unsigned flags, int gbase) {
        while (flags) {
            const int t = __ffs(flags) - 1; flags &= flags - 1;
            const int r = gbase + t;
            const unsigned mask = msk[t];
            unsigned ended, started;
            int endr;
            if (last_r == r - 1) { ended = open & ~mask; started = mask & ~open; endr = r - 1; }
            else { ended = open; started = mask; endr = last_r; }
            while (ended) { const int q = __ffs(ended) - 1; ended &= ended - 1; emit(q, rs[q], endr); }
            while (started) { const int q = __ffs(started) - 1; started &= started - 1; rs[q] = (unsigned short)r; }
            open = mask; last_r = r;
            ++nslow;
        }
    };

    stage32(plan, 0, 0, lane);
    cp_async_wait_all();
    __syncwarp();

    bool pass_prev = false;
    float bprev = 0.f;
    unsigned gflags = 0;      // flagged rows of the current group (bit kk)
    for (int g = 0; g < ngroups; ++g) {
        const int b = g & 1;
        if (g + 1 < ngroups) stage32(plan, g + 1, b ^ 1, lane);
#pragma unroll
        for (int kk = 0; kk < GR2; ++kk) {
            const float4 pr = sm.row[b][kk];
            // deferred: row kk-1 (previous group's last row at kk = 0) flagged -> its exact mask
            if (__builtin_expect(pass_prev, 0)) {
                const int kp = (kk + GR2 - 1) % D2;
                unsigned mask = 0;
#pragma unroll
                for (int s = 0; s < D2; ++s) {
                    const float z = fma_nocse(-cA[(s + kp) % D2], bprev, cov[s]);
                    mask |= (__float_as_uint(z) >> 31 ^ 1u) << s;
                }
                msk[(kk + GR2 - 1) % GR2] = (unsigned short)mask;
                gflags |= 1u << ((kk + GR2 - 1) % GR2);
            }
            if (kk == 0 && g > 0 && gflags) {   // the previous group's flagged rows -> runs
                fold_rows(gflags, (g - 1) * GR2);
                gflags = 0;
            }
            {   // rotation: phys (kk-1) mod D2 receives lane+1's outgoing column
                const int q = (kk + D2 - 1) % D2;
                if (lane == 0 && kk == 0) { const float4 f = sm.fresh[b][0]; cdf[q] = f.x; cdg[q] = f.y; }
                cdf[q] = __shfl_sync(FULLMASK, cdf[q], (lane + 1) & 31);
                cdg[q] = __shfl_sync(FULLMASK, cdg[q], (lane + 1) & 31);
                const float2 cq = sm.cq[b][kk * CQS + lane];
                cA[q] = fminf(cq.x, __fmul_rd(pr.w, cq.y));
            }
#pragma unroll
            for (int s = 0; s < D2; ++s) {
                const int p = (s + kk) % D2;
                cov[s] = fmaf(pr.x, cdg[p], cov[s]);
                cov[s] = fmaf(cdf[p], pr.y, cov[s]);
            }
            unsigned z[D2];
#pragma unroll
            for (int s = 0; s < D2; ++s) {
                const int p = (s + kk) % D2;
                z[s] = __float_as_uint(fmaf(-cA[p], pr.z, cov[s]));
            }
#pragma unroll
            for (int w = 1; w < D2; w *= 2)
#pragma unroll
                for (int s = 0; s + w < D2; s += 2 * w) z[s] &= z[s + w];
            pass_prev = (int)z[0] >= 0;            // some cell's z has its sign bit clear
            bprev = pr.z;
            if (kk + 1 < GR2 && lane == 0) {
                // slot 0's column (phys kk) is dead after this row: fetch the next fresh one now
                const float4 f = sm.fresh[b][kk + 1];
                cdf[kk % D2] = f.x; cdg[kk % D2] = f.y;
            }
        }
        cp_async_wait_all();
        __syncwarp();
    }
    if (pass_prev) {   // the last row
        constexpr int kp = (GR2 - 1) % D2;
        unsigned mask = 0;
#pragma unroll
        for (int s = 0; s < D2; ++s) {
            const float z = fmaf(-cA[(s + kp) % D2], bprev, cov[s]);
            mask |= (__float_as_uint(z) >> 31 ^ 1u) << s;
        }
        msk[GR2 - 1] = (unsigned short)mask;
        gflags |= 1u << (GR2 - 1);
    }
    if (gflags) fold_rows(gflags, (ngroups - 1) * GR2);
    while (open) { const int q = __ffs(open) - 1; open &= open - 1; emit(q, rs[q], last_r); }
    if (nslow) atomicAdd(a.counters + 2, (unsigned long long)nslow);
}

#else   // VLMP_PACKED: two-band packed walk
// Each lane owns 8 diagonals in band A (d0 + 8L + s) and the same 8 in band B (d0 + 256 + 8L
// + s): cells (s, A) and (s, B) form one FP32 register pair, and so do the ring slots of their
// columns (256 apart), which rotate together -- every update is a whole pair, every FFMA2
// operand is a natural pair or a broadcast (no half moves). Lane 31's new pair is (lane 0's
// outgoing B column, the fresh column d0 + 511 + i): lane 0 prepares it before the shuffle.
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk2(float lo, float hi) {
    u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r;
}
__device__ __forceinline__ float lo2(u64 v) { return __uint_as_float((unsigned)v); }
__device__ __forceinline__ float hi2(u64 v) { return __uint_as_float((unsigned)(v >> 32)); }
__device__ __forceinline__ u64 fma2(u64 x, u64 y, u64 z) {
    u64 d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x), "l"(y), "l"(z)); return d;
}
__device__ __forceinline__ u64 bc2(float x) { return pk2(x, x); }
// volatile: the flagged-row mask's FMAs must not be merged with the fast path's (see fma_nocse)
__device__ __forceinline__ u64 fma2_nocse(u64 x, u64 y, u64 z) {
    u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x), "l"(y), "l"(z)); return d;
}

// one 16-byte shared-memory read straight into two 64-bit register pairs (as a float4 read plus
// pk2 the compiler keeps the ring registers apart and copies the four words every row)
__device__ __forceinline__ void lds_pair(u64& x, u64& y, const float4* p) {
    asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"((unsigned)__cvta_generic_to_shared(p)));
}

__device__ __forceinline__ unsigned and3(unsigned x, unsigned y, unsigned z) {
    unsigned d; asm("lop3.b32 %0, %1, %2, %3, 0x80;" : "=r"(d) : "r"(x), "r"(y), "r"(z)); return d;
}

constexpr int DP = 8;        // diagonals per lane per band
constexpr int GRP = 8;       // rows per staging group (ring phase)
struct Smem32p {
    float4 row[2][GRP];          // {df, dg, b, w}
    // {aA, bA, aB, bB} of the column pairs in the tile's sliding 256-pair window, 8 pairs per
    // 9-entry chunk (the pad entry keeps lane L's read of entry 9 (L + g) + kk conflict free).
    // Lane L meets chunk (L + g) mod 33 in group g; each group only the chunk entering lane 31
    // is new -- 128 bytes staged per group, not the whole window.
    float4 cqr[33 * 9];
#if VLMP_PF_RING
    float4 pfr[33 * 9];          // the same window of {dfA, dfB, dgA, dgB}: the pair entering a lane's ring
#else
    float4 fresh[2][GRP];        // lane 31's entering column(s) at each row: PSEP = 256: the
                                 // B-band p32 entry; else the pf4 entry of the A-band column
#endif
    unsigned short rs[32 * 16];  // run starts per lane and cell (bits 0-7 band A, 8-15 band B)
    unsigned short msk[32 * GRP];
#if VLMP_RUN_GAP > 0
    unsigned short re[32 * 16];  // last row of a cell's closed, not yet logged run (gap bridging)
#endif
};

// lane 0's outgoing pair becomes lane 31's incoming one. Adjacent bands (PSEP = 256): (lane 0's
// band-B column, the fresh column) -- a half move; PSEP > 256: two fresh columns, loaded whole
// ({df, df'} and {dg, dg'} are the two 8-byte halves of the staged pf4 entry)
__device__ __forceinline__ void fresh_pair(u64& F, u64& G, const float4& f) {
    if (PSEP == BAND) { F = pk2(hi2(F), f.x); G = pk2(hi2(G), f.y); }
    else { F = reinterpret_cast<const u64*>(&f)[0]; G = reinterpret_cast<const u64*>(&f)[1]; }
}

__global__ void __launch_bounds__(32, VLMP_FILTER32_WARPS_PER_SM) k_tile32(Tile32Args a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem32p& sm = *reinterpret_cast<Smem32p*>(smem_raw);
    const int lane = threadIdx.x;
    const int wid = blockIdx.x;
    if (a.span && lane == 0) atomicMin(a.span, gtime());
    struct SpanEnd {   // the CTA's end on every return path
        unsigned long long* p; int lane;
        __device__ ~SpanEnd() { if (p && lane == 0) atomicMax(p + 1, gtime()); }
    } span_end{a.span, lane};
    if (wid >= a.n_tiles32) return;
    // one 16-byte descriptor per tile (the FP64 tile indices of both bands and the lower band's
    // (band, segment)): the prologue's loads below depend on it alone
    const int4 t4 = a.tiles32[wid];
    const int2 pr2 = make_int2(t4.x, t4.y);
    const long long d0 = a.dlo + (long long)t4.z * BAND;
    const long long i0 = (long long)t4.w * a.S;
    const long long rows_valid = a.N - d0 - i0;
    const bool liveA = rows_valid > 0 && d0 + BAND - 1 >= a.e;
    const bool liveB = pr2.y >= 0 && rows_valid - PSEP > 0 && d0 + PSEP + BAND - 1 >= a.e;
    if (!liveA && !liveB) return;
    const int nrows = (int)(rows_valid < a.S ? rows_valid : a.S);
    const int ngroups = (nrows + GRP - 1) / GRP;
    const long long cbA = i0 + d0 + (long long)DP * lane;   // band A column of slot 0 at row i0
    const long long cbB = cbA + PSEP;

    // ---- FP32 error slack. Per walked row (two FFMA over FP32-rounded df, dg) the covariance
    // error grows by at most 2u|cov| + 3.02u(|df_i dg_j| + |df_j dg_i|), u = 2^-24, with
    // |cov| <= s_i s_j (Cauchy-Schwarz); S + 1 rows (with the seed pre-adjust) plus the seed's
    // conversion, over the maxima of s, |df|, |dg| on the tile's rows and columns.
    // ---- staging: rows (lanes 0-7), fresh B columns (lanes 8-15), entering column factors.
    // Group 0's copies are issued first: they are in flight during the prologue's loads.
    // one 16-byte cp.async per lane and group: lanes 0-7 the group's rows, 8-15 the eight column
    // pairs' factors that enter lane 31 during the group, 16-23 their {df, dg} (PF_RING; else lane
    // 31's fresh columns). All sources advance by 128 bytes per group.
    const int q8 = lane & 7;
    const char* src_g; unsigned dst_g;
    if (lane < 8) {
        src_g = reinterpret_cast<const char*>(a.p32 + i0 + q8);
        dst_g = (unsigned)__cvta_generic_to_shared(&sm.row[0][q8]);
    } else if (lane < 16) {
        src_g = reinterpret_cast<const char*>(a.cq4 + i0 + d0 + DP - 1 + 248 + q8);
        dst_g = (unsigned)__cvta_generic_to_shared(&sm.cqr[q8]);
    } else {
#if VLMP_PF_RING
        src_g = reinterpret_cast<const char*>(a.pf4 + i0 + d0 + DP - 1 + 248 + q8);
        dst_g = (unsigned)__cvta_generic_to_shared(&sm.pfr[q8]);
#else
        src_g = PSEP == BAND ? reinterpret_cast<const char*>(a.p32 + i0 + q8 + d0 + 2 * BAND - 1)
                             : reinterpret_cast<const char*>(a.pf4 + i0 + q8 + d0 + BAND - 1);
        dst_g = (unsigned)__cvta_generic_to_shared(&sm.fresh[0][q8]);
#endif
    }
    constexpr unsigned RFP = sizeof(float4) * GRP, CHUNK = sizeof(float4) * 9;
    // running copy plan, the same instructions for every lane: the next group's source (+128 bytes
    // per group) and destination -- double-buffered rows (and fresh columns) alternate, a ring's
    // new chunk walks on by one (chunk (31 + g) mod 33 for group g)
    const bool dbuf = lane < 8 || (!VLMP_PF_RING && lane >= 16);
    const char* src_n = src_g + 128;
    const unsigned dst_step = dbuf ? RFP : CHUNK;
    const unsigned dst_span = dbuf ? 2 * RFP : 33 * CHUNK;
    const unsigned dst_lim = dst_g + dst_span;
    unsigned dst_n = dbuf ? dst_g + RFP : dst_g + 32 * CHUNK;
    auto stage = [&](int, int) {
        if (lane < 24) cpa<0, 0, 16>(dst_n, src_n);
        cp_async_commit();
        src_n += 128;
        dst_n += dst_step;
        if (dst_n >= dst_lim) dst_n -= dst_span;
    };
    {   // group 0: rows (fresh columns) and the whole window (entry f = lane + 32 k -> chunk f / 8)
        if (dbuf) cpa<0, 0, 16>(dst_g, src_g);
        const char* sc = reinterpret_cast<const char*>(a.cq4 + i0 + d0 + DP - 1 + lane);
        const unsigned dc = (unsigned)__cvta_generic_to_shared(&sm.cqr[9 * (lane / 8) + q8]);
#define STG(K) cpa_l1<(K) * 36 * 16, (K) * 512>(dc, sc);
        STG(0) STG(1) STG(2) STG(3) STG(4) STG(5) STG(6) STG(7)
#undef STG
#if VLMP_PF_RING
        const char* sf = reinterpret_cast<const char*>(a.pf4 + i0 + d0 + DP - 1 + lane);
        const unsigned df_ = (unsigned)__cvta_generic_to_shared(&sm.pfr[9 * (lane / 8) + q8]);
#define STG(K) cpa_l1<(K) * 36 * 16, (K) * 512>(df_, sf);
        STG(0) STG(1) STG(2) STG(3) STG(4) STG(5) STG(6) STG(7)
#undef STG
#endif
        cp_async_commit();
    }

    // ---- prologue loads in three independent batches (block maxima, ring, seeds): the warp
    // pays about one memory round trip for them, not one per dependent step
    // block maxima over the tile's rows and columns for the FP32 slack: <= 32 blocks each side
    // in practice, so one predicated load per lane and quantity
    unsigned r[3], c[3];
    const long long rb0 = i0 >> 8, rb1 = (i0 + nrows - 1) >> 8;
    const long long cb0 = (i0 + d0) >> 8, cb1 = (i0 + nrows - 1 + d0 + PSEP + BAND - 1) >> 8;
    {
        const bool rl = rb0 + lane <= rb1, cl = cb0 + lane <= cb1;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            r[q] = rl ? a.magblk[q * a.nb + rb0 + lane] : 0u;
            c[q] = cl ? a.magblk[q * a.nb + cb0 + lane] : 0u;
        }
    }

    // ---- ring of column pairs; N = -cA
    u64 F[DP], G[DP], NA[DP];
    {
        const float w0 = a.p32[i0].w;
#pragma unroll
        for (int s = 0; s < DP; ++s) {
            const long long ca = s < DP - 1 ? cbA + s : cbA - 1;
#if VLMP_PF_RING
            // the same 16-byte {dfA, dfB, dgA, dgB} / {aA, bA, aB, bB} entries the rings hold (the
            // ring registers then have one shape everywhere: no moves after the loop's reads)
            const float4 pf0 = a.pf4[ca];
            F[s] = pk2(pf0.x, pf0.y); G[s] = pk2(pf0.z, pf0.w);
            const float4 q0 = a.cq4[ca];
            NA[s] = pk2(fmaxf(-q0.x, __fmul_ru(-w0, q0.y)), fmaxf(-q0.z, __fmul_ru(-w0, q0.w)));
#else
            const float4 pa = a.p32[ca], pb = a.p32[ca + PSEP];
            F[s] = pk2(pa.x, pb.x); G[s] = pk2(pa.y, pb.y);
            const float2 qa = a.cq[ca], qb = a.cq[ca + PSEP];
            NA[s] = pk2(fmaxf(-qa.x, __fmul_ru(-w0, qa.y)), fmaxf(-qb.x, __fmul_ru(-w0, qb.y)));
#endif
        }
    }
    const float4 pr0 = a.p32[i0];
    const float4 plA = a.p32[cbA + DP - 1], plB = a.p32[cbB + DP - 1];

    float eps;
    {
        if (rb1 - rb0 >= 32 || cb1 - cb0 >= 32) {   // very long segments (S > 8192)
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                for (long long k = rb0 + 32 + lane; k <= rb1; k += 32) r[q] = max(r[q], a.magblk[q * a.nb + k]);
                for (long long k = cb0 + 32 + lane; k <= cb1; k += 32) c[q] = max(c[q], a.magblk[q * a.nb + k]);
            }
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            r[q] = __reduce_max_sync(FULLMASK, r[q]);
            c[q] = __reduce_max_sync(FULLMASK, c[q]);
        }
        const double Sr = __uint_as_float(r[0]), DFr = __uint_as_float(r[1]), DGr = __uint_as_float(r[2]);
        const double Sc = __uint_as_float(c[0]), DFc = __uint_as_float(c[1]), DGc = __uint_as_float(c[2]);
        const double K = (double)a.S + 1.0;
        const double bound = 0x1p-24 * 1.01 * ((2.0 * K + 1.0) * 1.001 * Sr * Sc + 3.02 * K * (DFr * DGc + DFc * DGr));
        eps = __double2float_ru(bound);
    }

    // ---- seeds of both bands (FP64, carried to m+1 in place as k_tile does)
    u64 cov[DP];
    {
        const double s2 = a.sscale * a.sscale;
        double* __restrict__ spA = a.seeds + (long long)pr2.x * BAND + DP * lane;
        double* __restrict__ spB = a.seeds + (long long)(liveB ? pr2.y : pr2.x) * BAND + DP * lane;
        double cA64[DP], cB64[DP];
#pragma unroll
        for (int s = 0; s < DP; ++s) { cA64[s] = liveA ? spA[s] : 0.0; cB64[s] = liveB ? spB[s] : 0.0; }
        if (a.update_seeds) {
            const double wgt = (double)a.m / (double)(a.m + 1);
            const double xi = (a.tn[i0 + a.m] - a.mu[i0]) * wgt;
            double xa[DP], xb[DP];
#pragma unroll
            for (int s = 0; s < DP; ++s) {
                xa[s] = a.tn[cbA + s + a.m] - a.mu[cbA + s];
                xb[s] = a.tn[cbB + s + a.m] - a.mu[cbB + s];
            }
#pragma unroll
            for (int s = 0; s < DP; ++s) {
                if (liveA) spA[s] = fma(xi, xa[s], cA64[s]);
                if (liveB) spB[s] = fma(xi, xb[s], cB64[s]);
            }
        }
#pragma unroll
        for (int s = 0; s < DP; ++s) {
            const float ca = (liveA && d0 + DP * lane + s >= a.e) ? __fadd_ru((float)(cA64[s] * s2), eps) : -INFINITY;
            const float cb = (liveB && d0 + PSEP + DP * lane + s >= a.e) ? __fadd_ru((float)(cB64[s] * s2), eps) : -INFINITY;
#if VLMP_DEV_NOPASS
            // dev ablation (wrong results, timing only): no cell ever passes, same instruction stream
            cov[s] = pk2(-1e30f, -1e30f); (void)ca; (void)cb;
#else
            cov[s] = pk2(ca, cb);
#endif
        }
    }
    // pre-adjust so that the uniform recurrence at row i0 reproduces the seed
#pragma unroll
    for (int s = 0; s < DP; ++s) {
        const u64 f = s < DP - 1 ? F[s] : pk2(plA.x, plB.x);
        const u64 g = s < DP - 1 ? G[s] : pk2(plA.y, plB.y);
        cov[s] = fma2(bc2(-pr0.y), f, cov[s]);
        cov[s] = fma2(bc2(-pr0.x), g, cov[s]);
    }

    // ---- runs (cells 0-7: band A diagonal d0 + 8L + s; 8-15: band B, + 256)
    unsigned open = 0;
    int last_r = -2;
    unsigned nslow = 0;
    unsigned short* rs = sm.rs + lane * 16;
    unsigned short* msk = sm.msk + lane * GRP;
    auto emit = [&](int c, int r_start, int r_end) {
        const int dcell = (int)(d0 + DP * lane) + (c & 7) + (c >> 3) * PSEP;
#if VLMP_RUN_MAXLEN > 0
        // a long run would keep one k_runs warp busy for its whole length (32 cells per scan step)
        // while the rest of the grid has drained: log it in pieces, each seeded by its own dot product
        for (; r_end - r_start + 1 > VLMP_RUN_MAXLEN; r_start += VLMP_RUN_MAXLEN) {
            const unsigned long long at = atomicAdd(a.run_count, 1ull);
            if ((long long)at < a.run_cap) {
                Run rp;
                rp.i = (int)(i0 + r_start); rp.j = rp.i + dcell; rp.len = VLMP_RUN_MAXLEN; rp.pad = 0;
                a.runs[at] = rp;
            }
        }
#endif
        Run rr;
        rr.i = (int)(i0 + r_start); rr.j = rr.i + dcell; rr.len = r_end - r_start + 1; rr.pad = 0;
        const unsigned long long at = atomicAdd(a.run_count, 1ull);
        if ((long long)at < a.run_cap) a.runs[at] = rr;
    };
#if VLMP_RUN_GAP > 0
    // a closed run waits (pend, re) for the next run of its diagonal: at most VLMP_RUN_GAP rows on,
    // the two are logged as one -- k_runs then pays one direct dot product instead of two, and the
    // gap's cells ride along in the same 32-cell scan chunk (every cell is tested exactly there)
    unsigned pend = 0;
    unsigned short* re = sm.re + lane * 16;
#endif
    auto fold_rows = [&](unsigned flags, int gbase) {
        while (flags) {
            const int t = __ffs(flags) - 1; flags &= flags - 1;
            const int r = gbase + t;
            const unsigned mask = msk[t];
            unsigned ended, started;
            int endr;
            if (last_r == r - 1) { ended = open & ~mask; started = mask & ~open; endr = r - 1; }
            else { ended = open; started = mask; endr = last_r; }
#if VLMP_RUN_GAP > 0
            pend |= ended;
            while (ended) { const int q = __ffs(ended) - 1; ended &= ended - 1; re[q] = (unsigned short)endr; }
            while (started) {
                const int q = __ffs(started) - 1; started &= started - 1;
                if (pend >> q & 1u) {
                    pend &= ~(1u << q);
                    if (r - (int)re[q] - 1 <= VLMP_RUN_GAP) continue;   // bridged: the run goes on from rs[q]
                    emit(q, rs[q], re[q]);
                }
                rs[q] = (unsigned short)r;
            }
#else
            while (ended) { const int q = __ffs(ended) - 1; ended &= ended - 1; emit(q, rs[q], endr); }
            while (started) { const int q = __ffs(started) - 1; started &= started - 1; rs[q] = (unsigned short)r; }
#endif
            open = mask; last_r = r;
            ++nslow;
        }
    };

    cp_async_wait_all();
    __syncwarp();

    bool pass_prev = false;
    float bprev = 0.f;
    unsigned gflags = 0;
    int chunk = lane;             // (lane + g) mod 33
    for (int g = 0; g < ngroups; ++g) {
        const int b = g & 1;
        if (g + 1 < ngroups) stage(g + 1, b ^ 1);
        const float4* cqp = sm.cqr + 9 * chunk;
#if VLMP_PF_RING
        const float4* pfp = sm.pfr + 9 * chunk;
#endif
        chunk = chunk == 32 ? 0 : chunk + 1;
#pragma unroll
        for (int kk = 0; kk < GRP; ++kk) {
            const float4 pr = sm.row[b][kk];
            if (__builtin_expect(pass_prev, 0)) {
                const int kp = (kk + GRP - 1) % DP;
#if VLMP_MASK_SHF
                u64 zz[DP];
#pragma unroll
                for (int s = 0; s < DP; ++s) zz[s] = fma2_nocse(NA[(s + kp) % DP], bc2(bprev), cov[s]);
                unsigned acc = 0;   // acc = (acc << 1) | sign, cell 15 (band B, s = 7) first
#pragma unroll
                for (int s = DP - 1; s >= 0; --s) acc = __funnelshift_l((unsigned)(zz[s] >> 32), acc, 1);
#pragma unroll
                for (int s = DP - 1; s >= 0; --s) acc = __funnelshift_l((unsigned)zz[s], acc, 1);
                const unsigned mask = ~acc;
#else
                unsigned mask = 0;
#pragma unroll
                for (int s = 0; s < DP; ++s) {
                    const u64 nq = NA[(s + kp) % DP];
                    const float za = fma_nocse(lo2(nq), bprev, lo2(cov[s]));
                    const float zb = fma_nocse(hi2(nq), bprev, hi2(cov[s]));
                    mask |= (__float_as_uint(za) >> 31 ^ 1u) << s;
                    mask |= (__float_as_uint(zb) >> 31 ^ 1u) << (s + 8);
                }
#endif
                msk[(kk + GRP - 1) % GRP] = (unsigned short)mask;
                gflags |= 1u << ((kk + GRP - 1) % GRP);
            }
            if (kk == 0 && g > 0 && gflags) { fold_rows(gflags, (g - 1) * GRP); gflags = 0; }
            {   // rotation: phys (kk-1) mod 8 receives lane+1's outgoing pair
                const int q = (kk + DP - 1) % DP;
#if VLMP_PF_RING
                // the entering pair's {df, dg} straight from the ring: one 16-byte read whose
                // halves are the two register pairs (no lane-to-lane shuffles, no fresh-column case)
                lds_pair(F[q], G[q], pfp + kk);
#else
                if (lane == 0 && kk == 0) fresh_pair(F[q], G[q], sm.fresh[b][0]);
                F[q] = __shfl_sync(FULLMASK, F[q], (lane + 1) & 31);
                G[q] = __shfl_sync(FULLMASK, G[q], (lane + 1) & 31);
#endif
                const float4 cq = cqp[kk];
                NA[q] = pk2(fmaxf(-cq.x, __fmul_ru(-pr.w, cq.y)), fmaxf(-cq.z, __fmul_ru(-pr.w, cq.w)));
            }
            unsigned z[16];
#pragma unroll
            for (int s = 0; s < DP; ++s) {
                const int p = (s + kk) % DP;
                cov[s] = fma2(bc2(pr.x), G[p], cov[s]);
                cov[s] = fma2(F[p], bc2(pr.y), cov[s]);
                const u64 zz = fma2(NA[p], bc2(pr.z), cov[s]);
                z[s] = (unsigned)zz; z[s + 8] = (unsigned)(zz >> 32);
            }
            {   // sign bits ANDed by a depth-3 tree of 3-input LOP3s (left to itself the compiler
                // chains 8 dependent LOP3s: ~32 cycles between the row's last FFMA2 and its branch)
                const unsigned t0 = and3(z[0], z[8], z[1]), t1 = and3(z[9], z[2], z[10]);
                const unsigned t2 = and3(z[3], z[11], z[4]), t3 = and3(z[12], z[5], z[13]);
                const unsigned t4 = and3(z[6], z[14], z[7]);
                z[0] = and3(and3(t0, t1, t2), t3, and3(t4, z[15], ~0u));
            }
            pass_prev = (int)z[0] >= 0;
            bprev = pr.z;
#if !VLMP_PF_RING
            if (kk + 1 < GRP && lane == 0) fresh_pair(F[kk % DP], G[kk % DP], sm.fresh[b][kk + 1]);
#endif
        }
        cp_async_wait_all();
        __syncwarp();
    }
    if (pass_prev) {
        constexpr int kp = (GRP - 1) % DP;
        unsigned mask = 0;
#pragma unroll
        for (int s = 0; s < DP; ++s) {
            const u64 nq = NA[(s + kp) % DP];
            const float za = fmaf(lo2(nq), bprev, lo2(cov[s]));
            const float zb = fmaf(hi2(nq), bprev, hi2(cov[s]));
            mask |= (__float_as_uint(za) >> 31 ^ 1u) << s;
            mask |= (__float_as_uint(zb) >> 31 ^ 1u) << (s + 8);
        }
        msk[GRP - 1] = (unsigned short)mask;
        gflags |= 1u << (GRP - 1);
    }
    if (gflags) fold_rows(gflags, (ngroups - 1) * GRP);
    while (open) { const int q = __ffs(open) - 1; open &= open - 1; emit(q, rs[q], last_r); }
#if VLMP_RUN_GAP > 0
    while (pend) { const int q = __ffs(pend) - 1; pend &= pend - 1; emit(q, rs[q], re[q]); }
#endif
    if (nslow) atomicAdd(a.counters + 2, (unsigned long long)nslow);
}
#endif  // VLMP_PACKED

// ---------------------------------------------------------------------------------
// Exact evaluation of the logged runs: one warp per run. Centred FP64 dot product at the first
// cell (lane-strided terms, fixed xor-tree reduction), then the diagonal recurrence along the
// run as an ordered inclusive warp scan of the per-step terms df_i dg_j + df_j dg_i; keys by
// the full-fold formula r = 1 - cov inv_i inv_j, exact tests hi(r) <= U (row and column side,
// as k_log_merge), 128-bit CAS folds. Deterministic (fixed reduction and scan orders).
// slots == nullptr: fold into the 1-best accumulators; else (m-best mode, m > 1 discords) append
// every cell that passes an exact test to its offset's candidate slots (SLOT_CAP per offset;
// k_select_m keeps the m smallest and recomputes offsets whose slots overflowed)
#ifndef VLMP_WDOT_ACC2
#define VLMP_WDOT_ACC2 0          // k_runs: two partial sums per lane in the direct dot product
#endif
#ifndef VLMP_RUNS_G
#define VLMP_RUNS_G 32            // lanes per run in k_runs (8 / 16: several runs per warp)
#endif
#ifdef VLMP_RUNS_MINB               // k_runs: minimum resident blocks per SM (register cap); default: none
#define VLMP_RUNS_BOUNDS __launch_bounds__(256, VLMP_RUNS_MINB)
#else
#define VLMP_RUNS_BOUNDS __launch_bounds__(256)
#endif
#ifndef VLMP_RUNS_GRID
#define VLMP_RUNS_GRID 8          // k_runs: blocks per SM in the grid
#endif

template <int G>
__global__ void VLMP_RUNS_BOUNDS k_runs(const Run* __restrict__ runs, const unsigned long long* run_count,
                                             long long cap, const Prm* __restrict__ prm,
                                             const double* __restrict__ tn, const double* __restrict__ mu,
                                             int m, int e, ulonglong2* acc, unsigned long long* counters,
                                             ulonglong2* slots, int* slot_cnt, unsigned long long* span) {
    if (span && threadIdx.x == 0) atomicMin(span, gtime());
    const unsigned long long cnt = *run_count;
    const long long nr = (long long)(cnt < (unsigned long long)cap ? cnt : (unsigned long long)cap);
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);                 // lane within the run's group
    const int gbase = lane & ~(G - 1);
    constexpr unsigned GM = G >= 32 ? 0xFFFFFFFFu : ((1u << (G & 31)) - 1u);
    const unsigned gmask = GM << gbase;
    const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / G;
    const long long nw = ((long long)gridDim.x * blockDim.x) / G;
    unsigned long long cells = 0, merged = 0;
    // group-cooperative centred dot product of windows (a, b): lane-strided terms, fixed xor tree
    auto wdot = [&](long long a_, long long b_) {
        const double ma = mu[a_], mb = mu[b_];
#if VLMP_WDOT_ACC2
        // two interleaved partial sums per lane (a shorter dependent FMA chain), fixed order
        double d = 0.0, d2 = 0.0;
        int k = gl;
        for (; k + G < m; k += 2 * G) {
            d = fma(tn[a_ + k] - ma, tn[b_ + k] - mb, d);
            d2 = fma(tn[a_ + k + G] - ma, tn[b_ + k + G] - mb, d2);
        }
        if (k < m) d = fma(tn[a_ + k] - ma, tn[b_ + k] - mb, d);
        d += d2;
#else
        double d = 0.0;
        for (int k = gl; k < m; k += G) d = fma(tn[a_ + k] - ma, tn[b_ + k] - mb, d);
#endif
#pragma unroll
        for (int off = G / 2; off >= 1; off >>= 1) d += __shfl_xor_sync(gmask, d, off, G);
        return d;
    };
    for (long long q = w0; q < nr; q += nw) {
        const Run R = runs[q];
        const long long i = R.i, j = R.j;
        const double dot = wdot(i, j);
        double carry = dot;
        // magnitude carried by the recurrence: |cov at the last exact point| + sum |steps| since.
        // Its rounding error is below 2^-47 of that (<= 160 roundings of 2^-53 each); a cell whose
        // own scale s_i s_j is below 1/8 of it (error above 2^-44 of the cell's scale, the key
        // resolution) is recomputed directly -- a run that walks out of a high-variance stretch.
        double mag = fabs(dot);
        const bool ok_diag = j - i >= e;
        for (int c0 = 0; c0 < R.len; c0 += G) {
            const int k = c0 + gl;
            const bool valid = k < R.len;
            double term = 0.0, ii = 0.0, ij = 0.0;
            float ui = -INFINITY, uj = -INFINITY;
            if (valid) {
                const Prm pi = prm[i + k], pj = prm[j + k];
                if (k > 0) term = fma(pi.df, pj.dg, pj.df * pi.dg);
                ii = pi.inv; ij = pj.inv; ui = pi.U; uj = pj.U;
            }
            float at = __double2float_ru(fabs(term));   // a bound: FP32, rounded up, is enough
            // inclusive scan over the chunk's nv cells only (runs are ~4 cells long on average):
            // the steps past nv would leave lanes < nv unchanged, so the sums are the same
            const int nv = R.len - c0 < G ? R.len - c0 : G;
#pragma unroll
            for (int off = 1; off < G; off <<= 1) {
                if (off >= nv) break;
                const double t = __shfl_up_sync(gmask, term, off, G);
                const float ta = __shfl_up_sync(gmask, at, off, G);
                if (gl >= off) { term += t; at = __fadd_ru(at, ta); }
            }
            double cv = carry + term;
            // |carried magnitude| <= 8 s_i s_j, i.e. (mag + at) inv_i inv_j <= 8 (NaN: invalid window)
            const bool inexact = valid && ok_diag && !((mag + (double)at) * (ii * ij) <= 8.0);
            unsigned redo = (__ballot_sync(gmask, inexact) >> gbase) & GM;
            if (redo) {   // rare: exact direct sums for the flagged cells of this chunk
                const unsigned tail = (__ballot_sync(gmask, valid) >> gbase) & GM;
                const int last = 31 - __clz(tail);
                redo |= 1u << last;              // the carry restarts from an exact value
                while (redo) {
                    const int l = __ffs(redo) - 1; redo &= redo - 1;
                    const double d = wdot(i + c0 + l, j + c0 + l);
                    if (gl == l) cv = d;
                }
                const double cl = __shfl_sync(gmask, cv, last, G);
                carry = cl; mag = fabs(cl);
            } else {
                carry = __shfl_sync(gmask, cv, nv - 1, G);
                mag += (double)__shfl_sync(gmask, at, nv - 1, G);
            }
            if (valid && ok_diag) {
                const double r = fma(-(cv * ii), ij, 1.0);
                const float h = __int_as_float(__double2hiint(r));
                const unsigned long long key = clamp_key(r) & ~PMASK;
                if (slots) {
                    if (h <= ui) {
                        const int at2 = atomicAdd(slot_cnt + i + k, 1);
                        if (at2 < SLOT_CAP) slots[(i + k) * SLOT_CAP + at2] = make_ulonglong2(key, (unsigned long long)(j + k));
                        ++merged;
                    }
                    if (h <= uj) {
                        const int at2 = atomicAdd(slot_cnt + j + k, 1);
                        if (at2 < SLOT_CAP) slots[(j + k) * SLOT_CAP + at2] = make_ulonglong2(key, (unsigned long long)(i + k));
                        ++merged;
                    }
                } else {
                    if (h <= ui) { acc_merge(acc + i + k, key, j + k); ++merged; }
                    if (h <= uj) { acc_merge(acc + j + k, key, i + k); ++merged; }
                }
            }
        }
        if (gl == 0) cells += (unsigned long long)R.len;
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        merged += __shfl_xor_sync(FULLMASK, merged, off);
        cells += __shfl_xor_sync(FULLMASK, cells, off);
    }
    // one pair of global atomics per block, not per warp
    __shared__ unsigned long long blk_cnt[2];
    if (threadIdx.x < 2) blk_cnt[threadIdx.x] = 0;
    __syncthreads();
    if (lane == 0 && (merged | cells)) { atomicAdd(&blk_cnt[0], merged); atomicAdd(&blk_cnt[1], cells); }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (blk_cnt[0]) atomicAdd(counters + 0, blk_cnt[0]);
        if (blk_cnt[1]) atomicAdd(counters + 4, blk_cnt[1]);
        if (span) atomicMax(span + 1, gtime());
    }
}

// ---------------------------------------------------------------------------------
// host side
int tile32_width() { return D2; }
const void* tile32_func() { return reinterpret_cast<const void*>(&k_tile32); }

#if VLMP_PACKED
using SmemT = Smem32p;
#else
using SmemT = Smem32;
#endif
size_t tile32_smem() { return sizeof(SmemT); }

// FP32 tiles from the FP64 tile list: D2 = 16 pairs (band b, band b+1) of one row segment,
// b - band_lo even; D2 = 8 keeps the FP64 tiles. Order follows the (longest-first) FP64 list.
void build_tiles32(const std::vector<int2>& tiles, long long band_lo, std::vector<int4>& out) {
    out.clear();
    if (D2 == 8) {
        for (size_t k = 0; k < tiles.size(); ++k) out.push_back(make_int4((int)k, -1, tiles[k].x, tiles[k].y));
        return;
    }
    std::vector<std::pair<long long, int>> keyed;   // (band, seg) -> index
    keyed.reserve(tiles.size());
    auto key = [](long long b, long long g) { return (b << 32) | g; };
    for (size_t k = 0; k < tiles.size(); ++k) keyed.push_back({key(tiles[k].x, tiles[k].y), (int)k});
    std::sort(keyed.begin(), keyed.end());
    auto find = [&](long long kk) {
        auto it = std::lower_bound(keyed.begin(), keyed.end(), std::make_pair(kk, -1));
        return (it != keyed.end() && it->first == kk) ? it->second : -1;
    };
    // packed walk: band b pairs with b + VLMP_PAIR_SEP (bands b mod 2 SEP < SEP lead); scalar: b, b + 1
    const long long sep = VLMP_PACKED ? VLMP_PAIR_SEP : 1;
    for (size_t k = 0; k < tiles.size(); ++k) {
        if (((long long)tiles[k].x - band_lo) % (2 * sep) >= sep) continue;
        out.push_back(make_int4((int)k, find(key((long long)tiles[k].x + sep, tiles[k].y)), tiles[k].x, tiles[k].y));
    }
}

int launch_filter32(vlmp_session* s, cudaStream_t st, const Prm* prm, const double* mu, long long N, int m, int e,
                    long long dl, int S, int update_seeds, long long n_t32, const int* forced,
                    ulonglong2* acc, Run* runs, unsigned long long* run_count, long long run_cap,
                    ulonglong2* slots, int* slot_cnt, unsigned long long* span) {
    const long long A = s->A;
    const long long nb = A / 256 + 1;
    Prep32Args pa{prm, s->d_cum, s->d_cum2, s->d_p32, s->d_cq32, s->d_magblk, nb, N, A, m, s->sscale,
                  const_cast<int*>(forced), (VLMP_PACKED && n_t32) ? s->d_cq4 : nullptr,
                  (VLMP_PACKED && n_t32 && (VLMP_PAIR_SEP > 1 || VLMP_PF_RING)) ? s->d_pf4 : nullptr};
#if VLMP_PRIO
    launch_hi(k_prep32, dim3((unsigned)blocks(A, 256)), dim3(256), 0, st, pa);
#else
    k_prep32<<<blocks(A, 256), 256, 0, st>>>(pa);
#endif
    if (n_t32) {
        Tile32Args ta{s->d_p32, s->d_cq32, s->d_magblk, nb, s->d_tn, mu, s->d_seeds, s->d_tiles, s->d_tiles32,
                      runs, run_count, run_cap, s->d_counters, forced, N, dl, (int)n_t32, S, m, e,
                      update_seeds, s->sscale, span, s->d_cq4, s->d_pf4};
        // span: [0, 1] k_tile32's and [2, 3] k_runs' first start / last end (bench.py's roofline)
        k_tile32<<<(unsigned)n_t32, 32, sizeof(SmemT), st>>>(ta);
#if VLMP_PRIO
        launch_hi(k_runs<VLMP_RUNS_G>, dim3(148 * VLMP_RUNS_GRID), dim3(256), 0, st, (const Run*)runs,
                  (const unsigned long long*)run_count, run_cap, prm, (const double*)s->d_tn, mu, m, e, acc, s->d_counters,
                  slots, slot_cnt, span ? span + 2 : (unsigned long long*)nullptr);
#else
        k_runs<VLMP_RUNS_G><<<148 * VLMP_RUNS_GRID, 256, 0, st>>>(runs, run_count, run_cap, prm, s->d_tn, mu, m, e, acc, s->d_counters,
                                        slots, slot_cnt, span ? span + 2 : nullptr);
#endif
    }
    return 0;
}

int filter32_setup() {
    cudaError_t e = cudaFuncSetAttribute(k_tile32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SmemT));
    if (e != cudaSuccess) return fail(VLMP_E_CUDA, std::string("k_tile32 smem: ") + cudaGetErrorString(e));
    return 0;
}

}  // namespace vlmp_impl
