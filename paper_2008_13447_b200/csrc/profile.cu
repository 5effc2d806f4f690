// profile.cu -- B200 (sm_100a) variable-length z-normalised matrix profile, phase 1.
//
// Hot path of arxiv 2008.13447 (MAD/VALMOD), rebuilt for the GPU: the exact
// matrix profile of one series at every window length in [lmin, lmax], from
// which VALMP, per-length motifs and discords are read off. Replaces the
// reference's per-length STOMP scan (profile.py:288-377) and its drivers
// (valmod.py:192-289, discords.py:144-247). See DESIGN.md for the derivations.
//
// Kernels (FP64 arithmetic on the CUDA cores; no tensor cores -- not a contraction):
//   k_params      per length: window mean/std from the host's prefix sums with the
//                 reference's exact op order (series.py:91-100) and the SCAMP-style
//                 recurrence factors df, dg, inv = 1/(sigma*sqrt(m)) (NaN = invalid),
//                 a 32-byte struct per offset (natural order; two buffers ping-pong
//                 so the bound can read the previous length's).
//   k_bound2      per length > first: an upper bound U[o] on offset o's key
//                 r = 1 - corr from the previous length's winners, O(1) per offset
//                 (stored keys -> covariances, one diagonal step, Welford to length m).
//   k_qprep       the filter's FP32 factors: b = sigma sqrt(m) 2^-k per offset and
//                 a = q(U) b, q(U) = 1 - R(U) - 2^-20, windowed over a lane's 8 rows.
//   k_tile<FULL>  one warp (one CTA) = one tile: 256 consecutive diagonals x S rows.
//                 Each lane owns D=8 diagonals and walks rows with the recurrence
//                 cov(i,j) = cov(i-1,j-1) + df_i dg_j + df_j dg_i   (2 DFMA per cell)
//                 over a register ring of column factors rotated lane to lane.
//                 FULL=false (filter): cell test hi(cov) >= hi(a_j b_i) (FMUL, LEA,
//                 ISETP); a passing lane logs its row's 8 covariances. FULL=true
//                 (first length, fallback, self-check): r = 1 - cov inv_i inv_j for
//                 every cell, exact folds with packed diagonal indices, warp-reduced
//                 rows, lane-travelling columns. Seeds (cov at each tile's first row)
//                 are carried to the next length with the Welford co-moment update.
//   k_log_merge   logged cells: bit-identical keys, exact row/column tests against U,
//                 lexicographic (key, index) minimum by 128-bit CAS.
//   k_finalize_walk  canonical pair distance of each winner (series.py:169-194).
//   k_valmp, k_smallest, k_discords, k_events, k_range_query: read-offs
//                 (valmod.py:57-73,170-177; discords.py:68-93; motifsets.py:105-165).
//   m-best mode (m-th discords): k_bound_m, k_log_slots, k_select_m, k_recompute_m,
//                 k_finalize_m, k_discords_m.

#include "vlmp_internal.cuh"

namespace vlmp_impl {

struct ParamArgs {
    const double* tn; const double* cum; const double* cum2;
    Prm* prm; double* mu;
    long long n, N, A; int m; double floor_;
};

__global__ void k_params(ParamArgs a) {
    long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (o >= a.A) return;
    const int m = a.m;
    double mu_o = 0.0, sd_o = 0.0, mu_p = 0.0, sd_p = 0.0;
    if (o < a.N) win_stats(a.cum, a.cum2, o, m, mu_o, sd_o);
    if (o >= 1 && o - 1 < a.N) win_stats(a.cum, a.cum2, o - 1, m, mu_p, sd_p);
    Prm p;
    p.inv = __longlong_as_double(0x7FF8000000000000ll);   // NaN: invalid window
    if (o < a.N && sd_o >= a.floor_) p.inv = 1.0 / (sd_o * sqrt((double)m));
    p.df = 0.0; p.dg = 0.0;
    if (o >= 1) {
        double tl = a.tn[o + m - 1], tp = a.tn[o - 1];
        p.df = (tl - tp) * 0.5;
        p.dg = (tl - mu_o) + (tp - mu_p);
    }
    p.U = INFINITY; p.pad = 0.f;
    a.prm[o] = p;
    a.mu[o] = mu_o;
}

void launch_params(vlmp_session* s, cudaStream_t st, Prm* prm, double* mu, int m) {
    ParamArgs pa{s->d_tn, s->d_cum, s->d_cum2, prm, mu, s->n, s->n - m + 1, s->A, m, s->floor_};
    k_params<<<blocks(s->A, 256), 256, 0, st>>>(pa);
}

// ---------------------------------------------------------------------------------
// O(1)-per-offset bound from the previous length's winners (1-best mode). Candidates:
// o's own winner c1 and its neighbours' winners shifted along their diagonals,
// (o, nn(o-1)+1) and (o, nn(o+1)-1). Their covariance at length m-1 comes from the stored
// key, cov = (1 - r) / (inv_o inv_c) (r kept to 2^-44), plus / minus one step of the
// diagonal recurrence; the Welford co-moment step carries it to length m. Any valid cell's
// key bounds the minimum; the reconstruction error (~1e-13) is far below the margin.
// exact centred co-moment of windows a, b at length m (direct sum, two accumulators): bounds
// must be keys of real cells, whatever the recurrence's accuracy on the series
__device__ inline double direct_cov(const double* __restrict__ tn, long long a, double ma, long long b, double mb, int m) {
    double c0 = 0.0, c1 = 0.0;
    int k = 0;
    for (; k + 1 < m; k += 2) {
        c0 = fma(tn[a + k] - ma, tn[b + k] - mb, c0);
        c1 = fma(tn[a + k + 1] - ma, tn[b + k + 1] - mb, c1);
    }
    if (k < m) c0 = fma(tn[a + k] - ma, tn[b + k] - mb, c0);
    return c0 + c1;
}

struct Bound2Args {
    const double* tn; const Prm* prm; const Prm* pprev; const double* mu_prev; const double* mu;
    const ulonglong2* acc_prev; Prm* out;
    long long N, Nprev; int m, e; double margin;
    unsigned long long* fix_cnt;   // offsets re-bounded by a direct dot product
    int exact;                     // bound = exact key of the chosen candidate (FP32 walk)
};

#ifndef VLMP_BOUND_ADJ
#define VLMP_BOUND_ADJ 0   // FP32 path: also bound by the own winner's neighbouring diagonals
#endif
__global__ void k_bound2(Bound2Args a) {
    const long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (o >= a.N) return;
    const double io = a.prm[o].inv;
    if (!(io == io)) { a.out[o].U = -INFINITY; return; }
    const int m = a.m;
    const double wgt = (double)(m - 1) / (double)m;
    const double xo = a.tn[o + m - 1] - a.mu_prev[o];
    double best = INFINITY, best_mag = 0.0;
    long long best_c = -1;
    // covp: the candidate's covariance at m-1 reconstructed from its stored key, plus at most
    // one recurrence step; mag bounds the magnitudes it was assembled from
    auto eval = [&](long long c, double covp, double mag) {
        const long long dd = c > o ? c - o : o - c;
        if (c < 0 || c >= a.N || dd < a.e) return;
        const double ic = a.prm[c].inv;
        if (!(ic == ic)) return;
        const double yc = a.tn[c + m - 1] - a.mu_prev[c];
        const double covm = fma(wgt * xo, yc, covp);
        const double r = fma(-(covm * io), ic, 1.0);
        if (r < best) { best = r; best_c = c; best_mag = mag + fabs(wgt * xo * yc) + fabs(covm); }
    };
    auto cov_of = [&](long long i, const ulonglong2& v) {   // winner's covariance at m-1
        const double r = __longlong_as_double((long long)v.x);
        return (1.0 - r) / (a.pprev[i].inv * a.pprev[(long long)v.y].inv);
    };
    if (o < a.Nprev) {
        const ulonglong2 v = a.acc_prev[o];
        if (v.x != KEY_NONE) { const double cv = cov_of(o, v); eval((long long)v.y, cv, fabs(cv)); }
    }
    if (o >= 1 && o - 1 < a.Nprev) {
        const ulonglong2 v = a.acc_prev[o - 1];
        if (v.x != KEY_NONE) {   // (o, c0+1) follows (o-1, c0) on its diagonal
            const long long c = (long long)v.y + 1;
            const Prm po = a.pprev[o], pc = a.pprev[c];
            const double cv = cov_of(o - 1, v), t1 = po.df * pc.dg, t2 = pc.df * po.dg;
            eval(c, cv + t1 + t2, fabs(cv) + fabs(t1) + fabs(t2));
        }
    }
    if (o + 1 < a.Nprev) {
        const ulonglong2 v = a.acc_prev[o + 1];
        if (v.x != KEY_NONE && v.y >= 1) {   // (o, c0-1) precedes (o+1, c0) on its diagonal
            const long long c0 = (long long)v.y;
            const Prm po = a.pprev[o + 1], pc = a.pprev[c0];
            const double cv = cov_of(o + 1, v), t1 = po.df * pc.dg, t2 = pc.df * po.dg;
            eval(c0 - 1, cv - t1 - t2, fabs(cv) + fabs(t1) + fabs(t2));
        }
    }
    if (!(best < INFINITY) && o < a.Nprev && a.acc_prev[o].x != KEY_NONE) {
        // the winner fell into the grown exclusion zone (|c1 - o| = e_{m-1} < e_m): the cell
        // one step further out, (o, c1 +- 1), by a direct centred dot product (rare)
        const long long c1 = (long long)a.acc_prev[o].y;
        const long long c = c1 > o ? c1 + 1 : c1 - 1;
        const long long dd = c > o ? c - o : o - c;
        if (c >= 0 && c < a.N && dd >= a.e) {
            const double ic = a.prm[c].inv;
            if (ic == ic) {
                const double mo = a.mu[o], mc = a.mu[c];
                double cv = 0.0;
                for (int k = 0; k < m; ++k) cv = fma(a.tn[o + k] - mo, a.tn[c + k] - mc, cv);
                best = fma(-(cv * io), ic, 1.0);
                best_c = -1;   // already exact
                atomicAdd(a.fix_cnt, 1ull);
            }
        }
    }
#if VLMP_BOUND_ADJ
    // the own winner's neighbouring diagonals (o, c1 -+ 1..ADJ) by direct centred sums (2m ADJ FMA
    // per offset): on smooth series a winner that moves between lengths mostly moves by one column,
    // and a tighter bound lets fewer cells through the walk into the exact runs
    if (a.exact && o < a.Nprev && a.acc_prev[o].x != KEY_NONE) {
        const long long c1 = (long long)a.acc_prev[o].y;
        for (int q = 0; q < 2 * VLMP_BOUND_ADJ; ++q) {
            const long long c = c1 + ((q & 1) ? -(q / 2 + 1) : (q / 2 + 1));
            const long long dd = c > o ? c - o : o - c;
            if (c < 0 || c >= a.N || dd < a.e) continue;
            const double ic = a.prm[c].inv;
            if (!(ic == ic)) continue;
            const double r = fma(-(direct_cov(a.tn, o, a.mu[o], c, a.mu[c], m) * io), ic, 1.0);
            if (r < best) { best = r; best_c = -1; }   // exact already
        }
    }
#endif
    if (a.exact && best_c >= 0 && !(best_mag * io * a.prm[best_c].inv <= 0x1p10)) {
        // the reconstruction's rounding (~2^-50 of the magnitudes it summed) could exceed the
        // 2^-26 margin relative to this cell's own scale s_o s_c: bound by its exact key instead
        const double cv = direct_cov(a.tn, o, a.mu[o], best_c, a.mu[best_c], m);
        best = fma(-(cv * io), a.prm[best_c].inv, 1.0);
        atomicAdd(a.fix_cnt, 1ull);
    }
    float out = INFINITY;   // no bound: every cell of this offset is a candidate
    if (best < INFINITY) out = __int_as_float(__double2hiint(fmax(best, 0.0) + a.margin));
    a.out[o].U = out;
}


// Bound of a shard's first length from its own partial minima (a full-fold pass over a
// sample of the bands): any folded cell is a valid cell of this length.
__global__ void k_bound_self(const ulonglong2* __restrict__ acc, Prm* prm, long long N, double margin,
                             const double* __restrict__ tn, const double* __restrict__ mu, int m, int exact) {
    const long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (o >= N) return;
    const double io = prm[o].inv;
    float u = -INFINITY;
    if (io == io) {
        const ulonglong2 v = acc[o];
        u = INFINITY;
        if (v.x != KEY_NONE) {
            double r = __longlong_as_double((long long)v.x);
            if (exact) {   // the folded winner's exact key (the fold's own key may be inaccurate)
                const long long c = (long long)v.y;
                r = fma(-(direct_cov(tn, o, mu[o], c, mu[c], m) * io), prm[c].inv, 1.0);
            }
            u = __int_as_float(__double2hiint(fmax(r, 0.0) + margin));
        }
    }
    prm[o].U = u;
}

// Filter thresholds in the covariance domain: qfac / qscale / q_forced (vlmp_internal.cuh).

// colq[o] = (a_o = q(U_o) b_o, b_o) for columns; rowq[o] = (b_o, q(Uwin_o)) for rows, where
// Uwin_o = max U[o .. o+D-1]: a column entering a lane at row o meets rows o .. o+D-1 there
__global__ void k_qprep(const Prm* __restrict__ prm, float2* colq, float2* rowq, long long N, long long A,
                        double sscale, int* forced) {
    const long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (o >= A) return;
    // invalid windows / past the end: factors +inf, so every threshold is +inf (never passes)
    if (o >= N) { colq[o] = make_float2(INFINITY, INFINITY); rowq[o] = make_float2(INFINITY, INFINITY); return; }
    const Prm p = prm[o];
    float uw = -INFINITY;
#pragma unroll
    for (int k = 0; k < D; ++k)
        if (o + k < N) uw = fmaxf(uw, prm[o + k].U);
    const float b = p.inv == p.inv ? qscale(p.inv, sscale) : INFINITY;
    const double qu = qfac(p.U);
    const float a = __double2float_rd(qu * (double)b);
    const float w = uw == -INFINITY ? 3.0e38f : __double2float_rd(qfac(uw));
    colq[o] = make_float2(a, b);
    rowq[o] = make_float2(b, w);
    if (forced && q_forced(p, sscale)) atomicOr(forced, 1);
}

// ---------------------------------------------------------------------------------


struct TileArgs {
    const Prm* prm; const double* mu; const double* tn;
    const int2* tiles;
    double* seeds;
    ulonglong2* acc;               // this length's accumulators, natural offsets
    unsigned long long* counters;  // [0] candidates logged, [1] unused, [2] flagged row steps
    RowRec* log;                   // this length's log of flagged lanes (filter kernel)
    unsigned long long* log_count; // this length's log fill counter
    long long log_cap;
    long long N, dlo;
    int n_tiles, S, m, e, update_seeds;
    const float2* colq;            // filter: column factors (a_j, b_j), natural offsets
    const float2* rowq;            // filter: row factors (b_i, q(Uwin_i))
    const int* forced;             // filter: nonzero => this length runs the full-fold body
    int hiC;                       // hi word of 2^(2k) * 2^-127 scaled float -> double bias
    const int* seed_map;           // tile list subset: seed slot of each listed tile (or nullptr)
};

__device__ inline double pack_low(double v, unsigned idx) {
    int lo = __double2loint(v), hi = __double2hiint(v);
    lo = (lo & ~(int)PMASK) | (int)idx;
    return __hiloint2double(hi, lo);
}



// Staging groups of GR rows. Over a group, lane L's ring receives columns
// c0 + D*L + kk (kk < GR, c0 = r0 + d0 + D - 1): NCOL = 31 D + GR distinct columns, staged
// once each (coalesced) into a linear buffer with one pad slot per 8 entries, so lane L's
// read of entry D*L + kk is bank-conflict free (D = 8: word 18 L + 2 kk' spans 32 banks).
#ifndef VLMP_GR
#define VLMP_GR 8
#endif
constexpr int GR = VLMP_GR;
static_assert(GR % D == 0 && GR <= 16, "a group must return the ring to its phase; 2 GR row halves <= 32 lanes");
constexpr int NCOL = 31 * D + GR;
__host__ __device__ constexpr int cpad(int f) { return f + (f >> 3); }
constexpr int CQN = cpad(NCOL - 1) + 1;
struct WarpSmem {
    Prm fresh[2][GR];        // the column entering lane 31's slot D-1 at each row of a group
    Prm row[2][GR];          // the group's row parameters
    float2 rq[2][GR];        // filter: the group's row factors
    float2 cq[2][CQN];       // filter: factors of the columns entering the lanes' rings (padded)
};

// Per-group staging by cp.async, planned once per tile: every lane's global source advances
// by a fixed stride per GR-row group and its shared destination alternates between two
// buffers, so a group costs a few LDGSTS with immediate offsets and a few adds.
//   row structs / fresh columns: GR rows, two 16-B halves each, plus the fresh column
//     r0 + q + d0 + BAND-1 that enters lane 31 at row r0 + q;
//   filter row factors of rows r0..r0+GR-1: 16-B chunks, lanes < GR/2;
//   filter column factors: the NCOL entering columns, entry f = lane + 32k (coalesced) to
//     cq[cpad(f)] = per-lane base + 36 k entries.
struct StagePlan {
    const char* src_pr; const char* src_fr; unsigned dst_pr, dst_fr;   // +GR*32 B per group
    const char* src_rq; unsigned dst_rq;      // rowq (+8 GR B per group), lanes < GR/2
    const char* src_cq; unsigned dst_cq;      // colq (+8 GR B per group)
};
constexpr unsigned PR_BUF = sizeof(Prm) * GR;            // fresh[b] / row[b] stride
constexpr unsigned RQ_BUF = sizeof(float2) * GR;
constexpr unsigned CQ_BUF = sizeof(float2) * CQN;

template <int OFF_D, int OFF_S, int BYTES>
__device__ __forceinline__ void cp_async_imm(unsigned d, const char* s) {
    if (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0+%2], [%1+%3], 16;\n" :: "r"(d), "l"(s), "n"(OFF_D), "n"(OFF_S) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0+%2], [%1+%3], 8;\n" :: "r"(d), "l"(s), "n"(OFF_D), "n"(OFF_S) : "memory");
}

template <bool FILTER>
__device__ __forceinline__ StagePlan make_plan(WarpSmem& w, const TileArgs& a, long long i0, long long d0,
                                               int lane) {
    StagePlan p;
    const int q = (lane >> 1) % GR, half = lane & 1;
    p.src_pr = reinterpret_cast<const char*>(a.prm + i0 + q) + 16 * half;
    p.src_fr = reinterpret_cast<const char*>(a.prm + i0 + q + d0 + BAND - 1) + 16 * half;
    p.dst_pr = (unsigned)__cvta_generic_to_shared(&w.row[0][q]) + 16 * half;
    p.dst_fr = (unsigned)__cvta_generic_to_shared(&w.fresh[0][q]) + 16 * half;
    if (4 * GR <= 32 && lane >= 16) { p.src_pr = p.src_fr; p.dst_pr = p.dst_fr; }   // one instruction
    if (FILTER) {
        const int r2 = lane % (GR / 2);
        p.src_rq = reinterpret_cast<const char*>(a.rowq + i0 + 2 * r2);
        p.dst_rq = (unsigned)__cvta_generic_to_shared(&w.rq[0][2 * r2]);
        p.src_cq = reinterpret_cast<const char*>(a.colq + i0 + d0 + D - 1 + lane);
        p.dst_cq = (unsigned)__cvta_generic_to_shared(&w.cq[0][cpad(lane)]);
    }
    return p;
}

template <int K>
__device__ __forceinline__ void stage_cq(unsigned dc, const char* sc, int lane) {
    if constexpr (32 * K < NCOL) {
        // entry f = lane + 32 K lands at cpad(f) = cpad(lane) + 36 K (lane + 32 K keeps lane's low bits)
        if (32 * (K + 1) <= NCOL || lane + 32 * K < NCOL) cp_async_imm<K * 36 * 8, K * 256, 8>(dc, sc);
        stage_cq<K + 1>(dc, sc, lane);
    }
}

// stage group g (rows i0 + GR*g ..) into buffer b
template <bool FILTER>
__device__ __forceinline__ void stage(const StagePlan& p, int g, int b, int lane) {
    const unsigned bsel = (unsigned)b;
    const long long gs = (long long)g * (GR * sizeof(Prm));
    if constexpr (4 * GR <= 32) {   // one instruction: lanes < 2GR rows, lanes >= 16 fresh columns
        if ((lane & 15) < 2 * GR) cp_async_imm<0, 0, 16>(p.dst_pr + bsel * PR_BUF, p.src_pr + gs);
    } else if (lane < 2 * GR) {
        cp_async_imm<0, 0, 16>(p.dst_pr + bsel * PR_BUF, p.src_pr + gs);
        cp_async_imm<0, 0, 16>(p.dst_fr + bsel * PR_BUF, p.src_fr + gs);
    }
    if (FILTER) {
        if (lane < GR / 2) cp_async_imm<0, 0, 16>(p.dst_rq + bsel * RQ_BUF, p.src_rq + (long long)g * (GR * 8));
        stage_cq<0>(p.dst_cq + bsel * CQ_BUF, p.src_cq + (long long)g * (GR * 8), lane);
    }
    cp_async_commit();
}

// high word of (double)(a*b rounded down): exponent rebiased, mantissa truncated (<= a*b)
__device__ __forceinline__ int q_hi(float a, float b, int hiC) {
    return (int)(__float_as_uint(__fmul_rd(a, b)) >> 3) + hiC;
}

// one flagged lane's record (per-lane atomic; the caller diverges)
__device__ __forceinline__ void log_one(const TileArgs& a, long long i, long long j0, const double (&cov)[D]) {
    const unsigned long long at = atomicAdd(a.log_count, 1ull);
    if ((long long)at < a.log_cap) {
        RowRec* r = a.log + at;
        r->i = (int)i; r->j0 = (int)j0; r->pad0 = 0; r->pad1 = 0;
#pragma unroll
        for (int s = 0; s < D; ++s) r->cov[s] = cov[s];
    }
}

template <bool FULL, bool MASKED>
__device__ __forceinline__ void tile_body(const TileArgs& a, WarpSmem& w, int wid, int lane,
                                          long long d0, long long i0, long long rows_valid) {
    const int dbase = lane * D;
    bool sval[D];
#pragma unroll
    for (int s = 0; s < D; ++s) sval[s] = !MASKED || (d0 + dbase + s >= a.e);

    double cov[D];
    double* seedp = a.seeds + (long long)wid * BAND + dbase;
#pragma unroll
    for (int s = 0; s < D; ++s) cov[s] = seedp[s];
    const long long cbase = i0 + d0 + dbase;   // column of slot 0 at row i0

    // Welford co-moment update of the seeds to length m+1:
    // C_{m+1} = C_m + m/(m+1) * (x_m - mean_m(x)) * (y_m - mean_m(y))
    if (a.update_seeds) {
        const double wgt = (double)a.m / (double)(a.m + 1);
        const double xi = (a.tn[i0 + a.m] - a.mu[i0]) * wgt;
#pragma unroll
        for (int s = 0; s < D; ++s)
            seedp[s] = fma(xi, a.tn[cbase + s + a.m] - a.mu[cbase + s], cov[s]);
    }

    // column ring: phys slot p holds the column of logical slot (p - kk) mod D at row step kk.
    // Each row, the column leaving lane L's slot 0 enters lane L-1's slot D-1 (shuffle);
    // lane 31 takes the fresh column i + d0 + 255 from shared memory.
    // The ring starts in its state "after row i0-1": phys p < D-1 holds the column of slot p
    // at row i0, phys D-1 holds the column leaving slot 0 at row i0-1 (cbase - 1), which the
    // first rotation hands to the left neighbour -- so every row, the first included, rotates.
    // Filter: cA[p] = q(max(U_col, Uwin[row the column entered this lane])) b_col, a lower
    // bound of q(max(U_i, U_col)) b_col for every row i the column meets in this lane.
    double cdf[D], cdg[D], cinv[D];
    float cA[D];
    {
        const float w0 = FULL ? 0.f : a.rowq[i0].y;
#pragma unroll
        for (int s = 0; s < D; ++s) {
            const long long c = s < D - 1 ? cbase + s : cbase - 1;
            const Prm pc = a.prm[c];
            cdf[s] = pc.df; cdg[s] = pc.dg; if (FULL) cinv[s] = pc.inv;
            if (!FULL) { const float2 q = a.colq[c]; cA[s] = fminf(q.x, __fmul_rd(w0, q.y)); }
        }
    }
    {   // pre-adjust so that the uniform recurrence at row i0 reproduces the seed
        const Prm pr = a.prm[i0];
        const Prm p7 = a.prm[cbase + D - 1];
#pragma unroll
        for (int s = 0; s < D; ++s) {
            const double df = s < D - 1 ? cdf[s] : p7.df, dg = s < D - 1 ? cdg[s] : p7.dg;
            cov[s] = fma(-df, pr.dg, cov[s]);
            cov[s] = fma(-pr.df, dg, cov[s]);
        }
    }
    double colacc[D];
    if (FULL) {
#pragma unroll
        for (int s = 0; s < D; ++s) colacc[s] = INFINITY;
    }
    double rowres = INFINITY, colres = INFINITY;   // FULL: stashed per-row results
    long long rowres_i = 0, colres_j = 0;
    unsigned long long nslow = 0;
    bool pass_prev = false;            // filter: row (i-1)'s pass predicate, acted on at row i

    const int S = a.S;
    const int nrows = (int)(rows_valid < S ? rows_valid : S);
    const int ngroups = (nrows + GR - 1) / GR;

    auto flush_full = [&]() {
        if (rowres < INFINITY) {
            const unsigned long long b = (unsigned long long)__double_as_longlong(rowres);
            acc_merge(a.acc + rowres_i, b & ~PMASK, rowres_i + d0 + (long long)(b & PMASK));
        }
        if (colres < INFINITY) {
            const unsigned long long b = (unsigned long long)__double_as_longlong(colres);
            const long long diag = BAND - 1 - (long long)(b & PMASK);
            acc_merge(a.acc + colres_j, b & ~PMASK, colres_j - d0 - diag);
        }
        rowres = INFINITY; colres = INFINITY;
    };

    const StagePlan plan = make_plan<!FULL>(w, a, i0, d0, lane);
    stage<!FULL>(plan, 0, 0, lane);
    cp_async_wait_all();
    __syncwarp();

    for (int g = 0; g < ngroups; ++g) {
        const int b = g & 1;
        if (g + 1 < ngroups) stage<!FULL>(plan, g + 1, b ^ 1, lane);
#pragma unroll
        for (int kk = 0; kk < GR; ++kk) {
            const long long i = i0 + (long long)g * GR + kk;
            const Prm pr = w.row[b][kk];
            {   // ring rotation: phys (kk-1) mod D receives lane+1's outgoing column
                const int q = (kk + D - 1) % D;
                // lane 0's outgoing column leaves the band: overwrite it with the fresh
                // column, then rotate by one lane so lane 31 receives it
                // (rows after a group's first: lane 0 loaded it at the end of the previous row)
                if (lane == 0 && kk == 0) {
                    const Prm f = w.fresh[b][kk];
                    cdf[q] = f.df; cdg[q] = f.dg; if (FULL) cinv[q] = f.inv;
                }
                const int src_lane = (lane + 1) & 31;
                cdf[q] = __shfl_sync(FULLMASK, cdf[q], src_lane);
                cdg[q] = __shfl_sync(FULLMASK, cdg[q], src_lane);
                if (FULL) cinv[q] = __shfl_sync(FULLMASK, cinv[q], src_lane);
                if (!FULL) {
                    const float2 cq = w.cq[b][cpad(dbase + kk)];
                    cA[q] = fminf(cq.x, __fmul_rd(w.rq[b][kk].y, cq.y));
                }
            }
            if (!FULL) {
                // Deferred test: row i-1's predicate is long resolved. cov[] still holds row
                // i-1's covariances (row i's recurrence has not run), so flagged lanes log them.
                // divergent per-lane slow path: no warp vote on the fast path
                if (pass_prev) {
                    log_one(a, i - 1, i - 1 + d0 + dbase, cov);
                    ++nslow;
                }
            }
#pragma unroll
            for (int s = 0; s < D; ++s) {
                const int p = (s + kk) % D;
                cov[s] = fma(pr.df, cdg[p], cov[s]);
                cov[s] = fma(cdf[p], pr.dg, cov[s]);
            }
            if (!FULL) {
                bool pa = false, pb = false;   // two independent predicate chains
                const float bi = w.rq[b][kk].x;
#pragma unroll
                for (int s = 0; s < D; ++s) {
                    const int p = (s + kk) % D;
                    // hi(cov) >= hi((double)t): t's exponent rebiased, mantissa truncated (<= t)
                    const int ht = q_hi(cA[p], bi, a.hiC);
                    const bool hit = sval[s] && (__double2hiint(cov[s]) >= ht);
                    if (s & 1) pb |= hit; else pa |= hit;
                }
                pass_prev = pa | pb;
            } else {
                // rows: lane-local packed min, then warp all-reduce (packed diag index => no exact ties)
                double rm = INFINITY;
#pragma unroll
                for (int s = 0; s < D; ++s) {
                    const int p = (s + kk) % D;
                    const double r = fma(-(cov[s] * pr.inv), cinv[p], 1.0);
                    double v = r < 0.0 ? 0.0 : r;     // clamp (NaN stays NaN)
                    if (!sval[s]) v = __longlong_as_double(0x7FF8000000000000ll);
                    const double pkr = pack_low(v, (unsigned)(dbase + s));
                    const double pkc = pack_low(v, (unsigned)(BAND - 1 - (dbase + s)));
                    rm = pkr < rm ? pkr : rm;
                    colacc[p] = pkc < colacc[p] ? pkc : colacc[p];
                }
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) {
                    const double o = __shfl_xor_sync(FULLMASK, rm, off);
                    rm = o < rm ? o : rm;
                }
                // the exiting column (logical slot 0, phys kk) travels to lane-1's slot D-1
                const double x = colacc[kk % D];
                double y = __shfl_down_sync(FULLMASK, x, 1);
                if (lane == 31) y = INFINITY;
                colacc[kk % D] = y;
                const double x0 = __shfl_sync(FULLMASK, x, 0);   // lane 0's exiting column
                const int slot = (int)((i - i0) & 31);
                if (lane == slot) { rowres = rm; rowres_i = i; colres = x0; colres_j = i + d0; }
                if (32 % GR != 0 && slot == 31) flush_full();   // every lane holds a stashed row
            }
            if (kk + 1 < GR && lane == 0) {
                // slot 0's column (phys kk) is dead after this row: lane 0 fetches the next row's
                // fresh column into it now, so the next rotation's shuffles need not wait
                const Prm f = w.fresh[b][kk + 1];
                cdf[kk % D] = f.df; cdg[kk % D] = f.dg; if (FULL) cinv[kk % D] = f.inv;
            }
        }
        if (FULL && 32 % GR == 0 && ((g + 1) * GR) % 32 == 0) flush_full();   // 32 rows stashed
        cp_async_wait_all();
        __syncwarp();
    }
    if (FULL) {
        flush_full();
        // after the last row (kk = D-1) and its rotate, phys p holds the column of logical
        // slot p at row i_end = i0 + GR*ngroups (GR is a multiple of D)
        const long long i_end = i0 + (long long)ngroups * GR;
#pragma unroll
        for (int p = 0; p < D; ++p) {
            const double v = colacc[p];
            if (v < INFINITY) {
                const long long j = i_end + d0 + dbase + p;
                const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
                const long long diag = BAND - 1 - (long long)(bits & PMASK);
                acc_merge(a.acc + j, bits & ~PMASK, j - d0 - diag);
            }
        }
    } else {
        if (pass_prev) {
            log_one(a, i0 + (long long)ngroups * GR - 1, i0 + (long long)ngroups * GR - 1 + d0 + dbase, cov);
            ++nslow;
        }
        if (nslow) atomicAdd(a.counters + 2, nslow);
    }
}

template <bool FULL>
__global__ void __launch_bounds__(WARPS_PER_CTA * 32, FULL ? FULL_MIN_BLOCKS : FILTER_MIN_BLOCKS)
k_tile(TileArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    WarpSmem* ws = reinterpret_cast<WarpSmem*>(smem_raw);
    const int lane = threadIdx.x & 31;
    const int wl = threadIdx.x >> 5;
    const int wid = blockIdx.x * WARPS_PER_CTA + wl;
    if (wid >= a.n_tiles) return;
    const int2 tl = a.tiles[wid];
    const int sw = a.seed_map ? a.seed_map[wid] : wid;   // seed slot of this tile
    const long long d0 = a.dlo + (long long)tl.x * BAND;
    const long long i0 = (long long)tl.y * a.S;
    const long long rows_valid = a.N - d0 - i0;
    if (rows_valid <= 0 || d0 + BAND - 1 < a.e) return;   // empty, or entirely trivial
    if (FULL || (a.forced && *a.forced)) {
        if (d0 < a.e) tile_body<true, true>(a, ws[wl], sw, lane, d0, i0, rows_valid);
        else tile_body<true, false>(a, ws[wl], sw, lane, d0, i0, rows_valid);
    } else {
        if (d0 < a.e) tile_body<false, true>(a, ws[wl], sw, lane, d0, i0, rows_valid);
        else tile_body<false, false>(a, ws[wl], sw, lane, d0, i0, rows_valid);
    }
}

// fold one length's log into its accumulators: recompute each logged cell's key with the
// tile kernel's FMA sequence (bit-identical), apply the exact row / column bound tests and
// the exclusion zone, and merge (key, index) with the 128-bit CAS
__global__ void k_log_merge(const RowRec* log, const unsigned long long* log_count, long long cap,
                            const Prm* prm, int e, ulonglong2* acc, unsigned long long* counters) {
    // MG consecutive lanes share one record (cells s < D, one each); every group takes R
    // records at once so the dependent loads (record -> window params -> accumulator) overlap
    constexpr int R = 4;
    const unsigned long long cnt = *log_count;
    const long long nrec = (long long)(cnt < (unsigned long long)cap ? cnt : (unsigned long long)cap);
    const int s = threadIdx.x & (MG - 1);
    unsigned long long merged = 0;
    const long long groups = ((long long)gridDim.x * blockDim.x) / MG;
    const long long stride = groups * R;
    const long long q_end = (nrec + stride - 1) / stride * stride;   // whole groups iterate together
    for (long long q0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / MG; q0 < q_end; q0 += stride) {
        long long iv[R], jv[R]; double cv[R];
        bool ok[R];
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const long long q = q0 + u * groups;
            ok[u] = q < nrec && s < D;
            iv[u] = 0; jv[u] = 0; cv[u] = 0.0;
            if (ok[u]) {
                const RowRec* rec = log + q;
                const int2 ij = *reinterpret_cast<const int2*>(rec);
                iv[u] = ij.x; jv[u] = (long long)ij.y + s; cv[u] = rec->cov[s];
                ok[u] = jv[u] - iv[u] >= e;
            }
        }
        double ii[R], ij_[R]; float ui[R], uj[R];
#pragma unroll
        for (int u = 0; u < R; ++u) {
            ii[u] = 0.0; ij_[u] = 0.0; ui[u] = -INFINITY; uj[u] = -INFINITY;
            if (ok[u]) {
                const Prm pr = prm[iv[u]], pc = prm[jv[u]];
                ii[u] = pr.inv; ij_[u] = pc.inv; ui[u] = pr.U; uj[u] = pc.U;
            }
        }
#pragma unroll
        for (int u = 0; u < R; ++u) {
            unsigned long long rk = KEY_NONE; long long rj = IDX_NONE;
            if (ok[u]) {
                const double r = fma(-(cv[u] * ii[u]), ij_[u], 1.0);
                const float h = __int_as_float(__double2hiint(r));
                const unsigned long long key = clamp_key(r) & ~PMASK;
                if (h <= ui[u]) { rk = key; rj = jv[u]; }
                if (h <= uj[u]) { acc_merge(acc + jv[u], key, iv[u]); ++merged; }
            }
            // the record's row-side candidates: one (key, index) minimum, one CAS
#pragma unroll
            for (int off = 1; off < MG; off <<= 1) {
                const unsigned long long ok2 = __shfl_xor_sync(FULLMASK, rk, off);
                const long long oj = __shfl_xor_sync(FULLMASK, rj, off);
                if (key_less(ok2, oj, rk, rj)) { rk = ok2; rj = oj; }
            }
            if (s == 0 && rj != IDX_NONE) { acc_merge(acc + iv[u], rk, rj); ++merged; }
        }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) merged += __shfl_xor_sync(FULLMASK, merged, off);
    if ((threadIdx.x & 31) == 0 && merged) atomicAdd(counters, merged);
}

// initial seeds: centred direct sums at the first length
struct SeedArgs {
    const double* tn; const double* mu; const int2* tiles; double* seeds;
    long long dlo; int n_tiles, S, m;
};

__global__ void k_seed_init(SeedArgs a) {
    const int lane = threadIdx.x & 31;
    const int wid = blockIdx.x * WARPS_PER_CTA + (threadIdx.x >> 5);
    if (wid >= a.n_tiles) return;
    const int2 tl = a.tiles[wid];
    const long long d0 = a.dlo + (long long)tl.x * BAND;
    const long long i0 = (long long)tl.y * a.S;
    const double mi = a.mu[i0];
    double acc[D], mc[D];
    const long long cb = i0 + d0 + lane * D;
#pragma unroll
    for (int s = 0; s < D; ++s) { acc[s] = 0.0; mc[s] = a.mu[cb + s]; }
    for (int k = 0; k < a.m; ++k) {
        const double x = a.tn[i0 + k] - mi;
#pragma unroll
        for (int s = 0; s < D; ++s) acc[s] = fma(x, a.tn[cb + s + k] - mc[s], acc[s]);
    }
    double* sp = a.seeds + (long long)wid * BAND + lane * D;
#pragma unroll
    for (int s = 0; s < D; ++s) sp[s] = acc[s];
}

// Carry every tile's seeds from length m_from to m_to without walking the tiles (a length
// shard's lengths before its first): the tile kernel's own Welford step per length, with
// the means recomputed in k_params' arithmetic (win_stats) -- bit-identical seeds.
__global__ void k_seed_forward(SeedArgs a, const double* __restrict__ cum, int m_to) {
    const int lane = threadIdx.x & 31;
    const int wid = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5);
    if (wid >= a.n_tiles) return;
    const int2 tl = a.tiles[wid];
    const long long d0 = a.dlo + (long long)tl.x * BAND;
    const long long i0 = (long long)tl.y * a.S;
    const long long cbase = i0 + d0 + lane * D;
    double* seedp = a.seeds + (long long)wid * BAND + lane * D;
    double sd[D];
#pragma unroll
    for (int s = 0; s < D; ++s) sd[s] = seedp[s];
    for (int m = a.m; m < m_to; ++m) {
        const double L = (double)m;
        const double wgt = (double)m / (double)(m + 1);
        const double mi = __ddiv_rn(__dsub_rn(cum[i0 + m], cum[i0]), L);
        const double xi = (a.tn[i0 + m] - mi) * wgt;
#pragma unroll
        for (int s = 0; s < D; ++s) {
            const double mc = __ddiv_rn(__dsub_rn(cum[cbase + s + m], cum[cbase + s]), L);
            sd[s] = fma(xi, a.tn[cbase + s + m] - mc, sd[s]);
        }
    }
#pragma unroll
    for (int s = 0; s < D; ++s) seedp[s] = sd[s];
}

__global__ void k_span_init(unsigned long long* span, int n_len) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n_len) { span[4 * t] = ~0ull; span[4 * t + 1] = 0; span[4 * t + 2] = ~0ull; span[4 * t + 3] = 0; }
}

__global__ void k_fill_acc(ulonglong2* acc, long long n) {
    long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (o < n) acc[o] = make_ulonglong2(KEY_NONE, (unsigned long long)IDX_NONE);
}

// previous-length winner indices (for the bound) straight from the accumulators
__global__ void k_acc_idx(const ulonglong2* acc, long long* idx, long long n) {
    long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (o < n) { ulonglong2 v = acc[o]; idx[o] = v.x == KEY_NONE ? -1 : (long long)v.y; }
}

// partial export / mask / import for the multi-GPU exact merge
__global__ void k_export(const ulonglong2* acc, unsigned long long* keys, long long* idx, long long total) {
    long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (q < total) { ulonglong2 v = acc[q]; keys[q] = v.x; idx[q] = (long long)v.y; }
}
__global__ void k_mask_idx(const unsigned long long* merged, const unsigned long long* keys, long long* idx, long long total) {
    long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (q < total && keys[q] != merged[q]) idx[q] = IDX_NONE;
}
__global__ void k_import(ulonglong2* acc, const unsigned long long* keys, const long long* idx, long long total) {
    long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (q < total) acc[q] = make_ulonglong2(keys[q], (unsigned long long)idx[q]);
}

// =================================================================================
// m-th discords (m > 1): per (length, offset) the m best neighbours, exact.
// The filter tile kernel runs with U = a bound on each offset's m-th best key; passing
// cells go to per-offset slots; k_select_m keeps the m smallest (key, index); offsets
// whose slots overflow are recomputed exactly from direct dot products.

struct BoundMArgs {
    const double* tn; const double* mu; Prm* prm;
    const long long* nn1;      // lmin: full-fold nearest neighbour per offset (or nullptr)
    const int* prevm;          // > lmin: previous length's m best per offset [A][mb] (or nullptr)
    long long N, Nprev, A; int m, e, mb; double margin;
};

// one warp per offset; candidates = previous m-best and their +-1 shifts (or the NN1
// neighbourhood at the first length); U = m-th smallest candidate key + margin
__global__ void k_bound_m(BoundMArgs a) {
    const int lane = threadIdx.x & 31;
    const long long o = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    if (o >= a.N) return;
    const double io = a.prm[o].inv;
    if (!(io == io)) { if (lane == 0) a.prm[o].U = -INFINITY; return; }
    long long cand[3 * MB_MAX + 8];
    int nc = 0;
    if (a.prevm) {
        for (int q = 0; q < a.mb; ++q) {
            const long long c = (o < a.Nprev) ? a.prevm[o * a.mb + q] : -1;
            if (c >= 0) { cand[nc++] = c; cand[nc++] = c - 1; cand[nc++] = c + 1; }
        }
    } else {
        const long long c1 = a.nn1[o];
        if (c1 >= 0)
            for (int t = -(a.mb + 1); t <= a.mb + 1; ++t) cand[nc++] = c1 + t;
        if (o >= 1) { const long long c = a.nn1[o - 1]; if (c >= 0) cand[nc++] = c + 1; }
        if (o + 1 < a.N) { const long long c = a.nn1[o + 1]; if (c >= 0) cand[nc++] = c - 1; }
    }
    double best[MB_MAX];
    for (int q = 0; q < MB_MAX; ++q) best[q] = INFINITY;
    const double mo = a.mu[o];
    for (int q0 = 0; q0 < nc; q0 += 4) {
        bool ok[4]; double mc[4], ic[4]; long long cc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            ok[u] = false; mc[u] = 0.0; ic[u] = 0.0; cc[u] = o;
            const int q = q0 + u;
            if (q < nc) {
                const long long c = cand[q];
                bool dup = false;
                for (int r = 0; r < q; ++r) dup |= (cand[r] == c);
                const long long dd = c > o ? c - o : o - c;
                if (!dup && c >= 0 && c < a.N && dd >= a.e) {
                    ic[u] = a.prm[c].inv; ok[u] = ic[u] == ic[u]; mc[u] = a.mu[c]; cc[u] = c;
                }
            }
        }
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int k = lane; k < a.m; k += 32) {
            const double x = a.tn[o + k] - mo;
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[u] = fma(x, a.tn[cc[u] + k] - mc[u], acc[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            double v = acc[u];
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(FULLMASK, v, off);
            if (ok[u]) {
                double key = fma(-(v * io), ic[u], 1.0);
                for (int q = 0; q < a.mb; ++q)            // insertion into the m smallest
                    if (key < best[q]) { const double t = best[q]; best[q] = key; key = t; }
            }
        }
    }
    if (lane == 0) {
        float out = INFINITY;
        const double bm = best[a.mb - 1];
        if (bm < INFINITY) out = __int_as_float(__double2hiint(fmax(bm, 0.0) + a.margin));
        a.prm[o].U = out;
    }
}

// filter-kernel log -> per-offset candidate slots (exact keys, exact tests)
__global__ void k_log_slots(const RowRec* log, const unsigned long long* log_count, long long cap,
                            const Prm* prm, int e, ulonglong2* slots, int* slot_cnt,
                            unsigned long long* counters) {
    const unsigned long long cnt = *log_count;
    const long long n = (long long)(cnt < (unsigned long long)cap ? cnt : (unsigned long long)cap);
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
         q += (long long)gridDim.x * blockDim.x) {
        const RowRec rec = log[q];
        const Prm pr = prm[rec.i];
        for (int s = 0; s < D; ++s) {
            const long long j = (long long)rec.j0 + s;
            if (j - rec.i < e) continue;
            const Prm pc = prm[j];
            const double r = fma(-(rec.cov[s] * pr.inv), pc.inv, 1.0);
            const float h = __int_as_float(__double2hiint(r));
            const unsigned long long key = clamp_key(r) & ~PMASK;
            if (h <= pr.U) {
                const int at = atomicAdd(slot_cnt + rec.i, 1);
                if (at < SLOT_CAP) slots[(long long)rec.i * SLOT_CAP + at] = make_ulonglong2(key, (unsigned long long)j);
            }
            if (h <= pc.U) {
                const int at = atomicAdd(slot_cnt + j, 1);
                if (at < SLOT_CAP) slots[j * SLOT_CAP + at] = make_ulonglong2(key, (unsigned long long)rec.i);
            }
        }
    }
}

// per offset: the m smallest (key, index) of its slots -> out[o][0..mb) (-1 = none);
// overflowing offsets are queued for an exact recompute; slot counters are reset
__global__ void k_select_m(ulonglong2* slots, int* slot_cnt, long long N, int mb, int* out,
                           long long* redo, unsigned long long* redo_cnt, const Prm* prm, double sscale) {
    const long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (o >= N) return;
    const int c = slot_cnt[o];
    slot_cnt[o] = 0;
    unsigned long long bk[MB_MAX]; long long bi[MB_MAX];
    for (int q = 0; q < MB_MAX; ++q) { bk[q] = KEY_NONE; bi[q] = IDX_NONE; }
    if (c > SLOT_CAP || q_forced(prm[o], sscale)) {
        const unsigned long long at = atomicAdd(redo_cnt, 1ull);
        redo[at] = o;
    } else {
        for (int t = 0; t < c; ++t) {
            const ulonglong2 v = slots[o * SLOT_CAP + t];
            unsigned long long k = v.x; long long i = (long long)v.y;
            for (int q = 0; q < mb; ++q)
                if (key_less(k, i, bk[q], bi[q])) {
                    const unsigned long long tk = bk[q]; const long long ti = bi[q];
                    bk[q] = k; bi[q] = i; k = tk; i = ti;
                }
        }
    }
    for (int q = 0; q < mb; ++q) out[o * mb + q] = bi[q] == IDX_NONE ? -1 : (int)bi[q];
}

// exact recompute of queued offsets: every valid neighbour's key from a direct centred
// dot product; block-wide m smallest
__global__ void k_recompute_m(const double* tn, const double* mu, const Prm* prm, const long long* redo,
                              const unsigned long long* redo_cnt, long long N, int m, int e, int mb,
                              int* out) {
    __shared__ unsigned long long sk[256 * MB_MAX];
    __shared__ long long si[256 * MB_MAX];
    const unsigned long long nred = *redo_cnt;
    for (unsigned long long r = blockIdx.x; r < nred; r += gridDim.x) {
        const long long o = redo[r];
        const double io = prm[o].inv, mo = mu[o];
        unsigned long long bk[MB_MAX]; long long bi[MB_MAX];
        for (int q = 0; q < MB_MAX; ++q) { bk[q] = KEY_NONE; bi[q] = IDX_NONE; }
        for (long long j = threadIdx.x; j < N; j += blockDim.x) {
            const long long dd = j > o ? j - o : o - j;
            if (dd < e) continue;
            const double ic = prm[j].inv;
            if (!(ic == ic) || !(io == io)) continue;
            const double mc = mu[j];
            double cv = 0.0;
            for (int k = 0; k < m; ++k) cv = fma(tn[o + k] - mo, tn[j + k] - mc, cv);
            unsigned long long key = clamp_key(fma(-(cv * io), ic, 1.0)) & ~PMASK;
            long long idx = j;
            for (int q = 0; q < mb; ++q)
                if (key_less(key, idx, bk[q], bi[q])) {
                    const unsigned long long tk = bk[q]; const long long ti = bi[q];
                    bk[q] = key; bi[q] = idx; key = tk; idx = ti;
                }
        }
        for (int q = 0; q < mb; ++q) { sk[threadIdx.x * MB_MAX + q] = bk[q]; si[threadIdx.x * MB_MAX + q] = bi[q]; }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long fk[MB_MAX]; long long fi[MB_MAX];
            for (int q = 0; q < MB_MAX; ++q) { fk[q] = KEY_NONE; fi[q] = IDX_NONE; }
            for (int t = 0; t < (int)blockDim.x; ++t)
                for (int q0 = 0; q0 < mb; ++q0) {
                    unsigned long long key = sk[t * MB_MAX + q0]; long long idx = si[t * MB_MAX + q0];
                    if (idx == IDX_NONE) break;
                    for (int q = 0; q < mb; ++q)
                        if (key_less(key, idx, fk[q], fi[q])) {
                            const unsigned long long tk = fk[q]; const long long ti = fi[q];
                            fk[q] = key; fi[q] = idx; key = tk; idx = ti;
                        }
                }
            for (int q = 0; q < mb; ++q) out[o * mb + q] = fi[q] == IDX_NONE ? -1 : (int)fi[q];
        }
        __syncthreads();
    }
}

// canonical distances of the m best, sorted ascending (discords.py:126-141)
__global__ void k_finalize_m(const double* tn, const double* cum, const double* cum2, const int* ipm,
                             double* mpm, long long n, long long A, int lmin, int mb, double floor_) {
    const long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int li = blockIdx.y;
    const int m = lmin + li;
    if (o >= n - m + 1) return;
    const long long base = ((long long)li * A + o) * mb;
    double v[MB_MAX];
    for (int q = 0; q < mb; ++q) {
        const int nb = ipm[base + q];
        v[q] = nb >= 0 ? pair_distance(tn, cum, cum2, o, nb, m, floor_) : INFINITY;
    }
    for (int q = 1; q < mb; ++q)
        for (int r = q; r > 0 && v[r] < v[r - 1]; --r) { const double t = v[r]; v[r] = v[r - 1]; v[r - 1] = t; }
    for (int q = 0; q < mb; ++q) mpm[base + q] = v[q];
}

// top-k m-th discords per length: ascending-offset greedy replay (discords.py:68-93,
// :48-50) of the canonical sorted distances, exact prefilter "some column beats row k-1";
// one warp per length, state in shared memory
__global__ void k_discords_m(const double* mpm, double* out_d, long long* out_o, long long n, long long A,
                             int lmin, int n_len, int k, int mb) {
    extern __shared__ unsigned char sm_raw[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int li = blockIdx.x * (blockDim.x >> 5) + wl;
    double* cd = reinterpret_cast<double*>(sm_raw) + (size_t)wl * 32 * MB_MAX * 2;
    long long* co = reinterpret_cast<long long*>(cd + 32 * MB_MAX);
    if (li >= n_len) return;
    const int m = lmin + li;
    const long long N = n - m + 1, e = (m + 1) / 2;
    for (int t = lane; t < k * mb; t += 32) { cd[t] = -INFINITY; co[t] = -1; }
    __syncwarp();
    for (long long base = 0; base < N; base += 32) {
        const long long o = base + lane;
        bool cand = false;
        if (o < N) {
            const double* b = mpm + ((long long)li * A + o) * mb;
            if (b[mb - 1] < INFINITY)
                for (int c = 0; c < mb; ++c) cand |= b[c] > cd[(k - 1) * mb + c];
        }
        unsigned bal = __ballot_sync(FULLMASK, cand);
        while (bal) {
            const int src = __ffs(bal) - 1;
            bal &= bal - 1;
            if (lane == 0) {
                const long long ov = base + src;
                const double* b = mpm + ((long long)li * A + ov) * mb;
                bool triv = false;
                for (int t = 0; t < k * mb; ++t) triv |= (co[t] >= 0 && llabs(ov - co[t]) < e);
                if (!triv) {
                    bool done = false;
                    for (int c = mb - 1; c >= 0 && !done; --c) {
                        const double d = b[c];
                        for (int r = 0; r < k; ++r) {
                            if (d > cd[r * mb + c]) {
                                for (int q = k - 1; q > r; --q) { cd[q * mb + c] = cd[(q - 1) * mb + c]; co[q * mb + c] = co[(q - 1) * mb + c]; }
                                cd[r * mb + c] = d; co[r * mb + c] = ov;
                                done = true;
                                break;
                            }
                        }
                    }
                }
            }
            __syncwarp();
        }
    }
    for (int t = lane; t < k * mb; t += 32) {
        out_d[(long long)li * k * mb + t] = cd[t];
        out_o[(long long)li * k * mb + t] = co[t];
    }
}



// filter log records per length: 16 per offset (quasi-periodic series flag many near-minimum
// cells), at most a quarter of the free device memory; an overflow re-runs exactly
size_t log_capacity(long long N0) {
    size_t want = std::max<size_t>((size_t)1 << 20, (size_t)(16 * N0));
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
        const size_t lim = free_b / 4 / sizeof(RowRec);
        if (want > lim) want = std::max<size_t>(lim, (size_t)1 << 18);
    }
    return want;
}

// launch order: longest tiles first (LPT), so the partial last segments of the bands fill
// the tail of each length's launch instead of leaving SMs idle behind full-size tiles
#ifndef VLMP_TILE_LPT
#define VLMP_TILE_LPT 1
#endif
void order_tiles(std::vector<int2>& tiles, long long N0, long long dl, int S) {
    if (!VLMP_TILE_LPT) return;
    auto rows = [&](const int2& t) {
        const long long r = N0 - (dl + (long long)t.x * BAND) - (long long)t.y * S;
        return r < S ? r : (long long)S;
    };
    std::stable_sort(tiles.begin(), tiles.end(), [&](const int2& a, const int2& b) { return rows(a) > rows(b); });
}

int seg_rows(long long n) {
    // S = G*D rows per tile (whole GR-row groups). Short segments keep the FP32 walk's error
    // slack small (it grows with the rows walked from the FP64 seed) and the launch tail fine;
    // the cost is the seed store, 8 B per (diagonal, segment) ~ 4 n^2 / S bytes. S = 1024
    // while that fits in a fifth of the device (config 4: 4.3 GB), doubling beyond.
#ifndef VLMP_SEG_G0
#define VLMP_SEG_G0 128
#endif
    long long G = VLMP_SEG_G0;
    size_t free_b = 0, total_b = 0;
    double budget = 8e9;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) budget = (double)total_b / 5.0;
    while (4.0 * (double)n * (double)n / (double)(G * D) > budget && G < 2048) G *= 2;
    return (int)(G * D);
}

long long dlo_for(int lmin) { return (lmin + 1) / 2; }

long long n_bands_for(long long n, int lmin) {
    long long N = n - lmin + 1;
    long long dl = dlo_for(lmin);
    return N - dl > 0 ? (N - dl + BAND - 1) / BAND : 0;
}

// work of band b summed over lengths: sum_l sum_{d in band, d >= e_l} (N_l - d)_+
double band_work(long long n, int lmin, int lmax, long long b) {
    double w = 0;
    long long d_lo = dlo_for(lmin) + b * BAND, d_hi = d_lo + BAND;
    for (int m = lmin; m <= lmax; ++m) {
        long long N = n - m + 1, e = (m + 1) / 2;
        long long lo = std::max(d_lo, e), hi = std::min(d_hi, N);
        if (hi <= lo) continue;
        // sum_{d=lo}^{hi-1} (N - d)
        w += (double)(hi - lo) * (double)N - ((double)(lo + hi - 1) * (double)(hi - lo)) / 2.0;
    }
    return w;
}


}  // namespace vlmp_impl

extern "C" {

int vlmp_band_count(vlmp_session* s, int32_t lmin, int64_t* n_bands) {
    if (!s || !n_bands) return fail(VLMP_E_INVALID_PARAMETERS, "null argument");
    *n_bands = n_bands_for(s->n, lmin);
    return 0;
}

int vlmp_band_split(vlmp_session* s, int32_t lmin, int32_t lmax, int32_t parts, int64_t* cuts) {
    if (!s || !cuts || parts < 1) return fail(VLMP_E_INVALID_PARAMETERS, "bad band split arguments");
    long long nb = n_bands_for(s->n, lmin);
    std::vector<double> w(nb);
    double tot = 0;
    for (long long b = 0; b < nb; ++b) { w[b] = band_work(s->n, lmin, lmax, b); tot += w[b]; }
    cuts[0] = 0;
    double acc = 0; long long b = 0;
    for (int p = 1; p < parts; ++p) {
        double target = tot * p / parts;
        while (b < nb && acc + w[b] <= target) acc += w[b++];
        cuts[p] = b;
    }
    cuts[parts] = nb;
    return 0;
}

// Lengths li_lo..li_hi (indices into [lmin, lmax]) of bands [band_lo, band_hi): a length
// shard starts with a full-fold pass at li_lo on seeds carried there from lmin (bit-identical
// to the single-run chain); accumulators of other lengths stay empty.
constexpr uint32_t F_NO_SAMPLED_START = 1u << 30;   // internal: first length by full folds

// dev aid (scripts/diag_bounds.py, run-log analysis): VLMP_DUMP_PRM / VLMP_DUMP_RUNS = file,
// VLMP_DUMP_LI = length index (default 64) -- one length's bounds or FP32-walk run log
static int debug_dump(cudaStream_t st, int li, const Prm* prm, long long N, const Run* runs,
                      const unsigned long long* run_count, long long run_cap) {
    const char* dp = getenv("VLMP_DUMP_PRM");
    const char* dr = getenv("VLMP_DUMP_RUNS");
    if (!dp && !dr) return 0;
    if (li != atoi(getenv("VLMP_DUMP_LI") ? getenv("VLMP_DUMP_LI") : "64")) return 0;
    CU(cudaStreamSynchronize(st));
    if (dp) {
        std::vector<Prm> h(N);
        CU(cudaMemcpy(h.data(), prm, N * sizeof(Prm), cudaMemcpyDeviceToHost));
        if (FILE* f = fopen(dp, "wb")) { fwrite(h.data(), sizeof(Prm), N, f); fclose(f); }
    }
    if (dr) {
        unsigned long long c = 0;
        CU(cudaMemcpy(&c, run_count, 8, cudaMemcpyDeviceToHost));
        c = std::min<unsigned long long>(c, (unsigned long long)run_cap);
        std::vector<Run> h(c);
        CU(cudaMemcpy(h.data(), runs, c * sizeof(Run), cudaMemcpyDeviceToHost));
        if (FILE* f = fopen(dr, "wb")) { fwrite(h.data(), sizeof(Run), c, f); fclose(f); }
    }
    return 0;
}

// Enqueues phase 1 (no host sync): the launch sequence, then async copies of the small
// counters the overflow check needs into pinned host memory. settle_profile() (called by
// every consumer of phase 1) waits for them, checks the logs and redoes the run if needed.
static int profile_impl(vlmp_session* s, int32_t lmin, int32_t lmax, int64_t band_lo,
                        int64_t band_hi, uint32_t flags, int li_lo = 0, int li_hi = -1) {
    CU(cudaSetDevice(s->device));
    cudaStream_t st = s->stream;
    const long long n = s->n, A = s->A;
    const int n_len = lmax - lmin + 1;
    const long long nb = n_bands_for(n, lmin);
    if (band_hi < 0 || band_hi > nb) band_hi = nb;
    if (band_lo < 0) band_lo = 0;
    if (s->tc_n != n) { s->tc_n = n; s->tc_S = seg_rows(n); s->tc_key[0] = -1; }
    const int S = s->tc_S;
    const long long N0 = n - lmin + 1, dl = dlo_for(lmin);
    // tile list using N at lmin (a superset of every later length's tiles), launched
    // longest-first (order_tiles); built and uploaded once per (series length, lmin, bands)
    const bool fp32_key = !(flags & (VLMP_F_FP64_FILTER | VLMP_F_FULL_EVERY_LENGTH)) && !getenv("VLMP_FP64_FILTER");
    const long long mode_key = (long long)flags | (fp32_key ? (1LL << 40) : 0);   // the sample list depends on both
    const bool tiles_cached = s->tc_key[0] == n && s->tc_key[1] == lmin && s->tc_key[2] == band_lo &&
                              s->tc_key[3] == band_hi && s->tc_key[4] == mode_key;
    std::vector<int2> tiles;
    if (!tiles_cached) {
        for (long long b = band_lo; b < band_hi; ++b) {
            long long rows = N0 - (dl + b * BAND);
            for (long long sg = 0; sg * S < rows; ++sg) tiles.push_back(make_int2((int)b, (int)sg));
        }
        order_tiles(tiles, N0, dl, S);
    }
    // a shard's first length: full folds over every SAMPLE-th band first (cheap), whose minima
    // bound the filtered pass over all bands -- instead of full folds everywhere
#ifndef VLMP_FIRST_SAMPLE
#define VLMP_FIRST_SAMPLE 8   // bands per folded band at a run's first length (4: 1.52 ms, 8: 1.32, 16: 1.49 at config 2)
#endif
    constexpr int SAMPLE = VLMP_FIRST_SAMPLE;
    // filtered lengths: FP32 walk + exact FP64 runs (filter32.cu) unless asked for the FP64 filter
    const bool fp32 = !(flags & (VLMP_F_FP64_FILTER | VLMP_F_FULL_EVERY_LENGTH)) && !getenv("VLMP_FP64_FILTER");
    const bool sampled_start = SAMPLE > 1 && (band_hi - band_lo) >= 8 * SAMPLE &&
                               !(flags & (VLMP_F_FULL_EVERY_LENGTH | F_NO_SAMPLED_START));
    // FP32 walk: the first length's folds only bound it (exact keys of their winners); its keys
    // come from the FP32 pass's exact runs like every other length's. Few bands: fold them all.
    const bool bound_start = sampled_start || fp32;
    const int sample = sampled_start ? SAMPLE : 1;
    std::vector<int2> tiles_s;
    std::vector<int> smap;
    for (size_t k = 0; k < tiles.size(); ++k)
        if ((tiles[k].x - band_lo) % sample == 0) { tiles_s.push_back(tiles[k]); smap.push_back((int)k); }
    const long long T = tiles_cached ? s->tc_T : (long long)tiles.size();
    int rc;
    if ((rc = ensure(s->d_tiles, s->tiles_cap, (size_t)std::max<long long>(T, 1)))) return rc;
    if ((rc = ensure(s->d_seeds, s->seeds_cap, (size_t)std::max<long long>(T, 1) * BAND))) return rc;
    if ((rc = ensure(s->d_acc, s->acc_cap, (size_t)n_len * A))) return rc;
    const size_t log_cap = log_capacity(N0);
    if ((rc = ensure(s->d_log, s->log_cap, log_cap))) return rc;
    if ((rc = ensure(s->d_logcnt, s->logcnt_cap, (size_t)n_len))) return rc;
    if ((rc = ensure(s->d_forced, s->forced_cap, (size_t)n_len))) return rc;
    if ((rc = ensure(s->d_fixcnt, s->fixcnt_cap, (size_t)n_len))) return rc;
    if (T && !tiles_cached) CU(cudaMemcpyAsync(s->d_tiles, tiles.data(), T * sizeof(int2), cudaMemcpyHostToDevice, st));
    const long long Ts = tiles_cached ? s->tc_Ts : (long long)tiles_s.size();
    if (bound_start && Ts && !tiles_cached) {
        if ((rc = ensure(s->d_tiles_s, s->tiles_s_cap, (size_t)Ts))) return rc;
        if ((rc = ensure(s->d_smap, s->smap_cap, (size_t)Ts))) return rc;
        CU(cudaMemcpyAsync(s->d_tiles_s, tiles_s.data(), Ts * sizeof(int2), cudaMemcpyHostToDevice, st));
        CU(cudaMemcpyAsync(s->d_smap, smap.data(), Ts * sizeof(int), cudaMemcpyHostToDevice, st));
    }
    std::vector<int4> tiles32;
    if (fp32) {
        if (!tiles_cached) build_tiles32(tiles, band_lo, tiles32);
        if ((rc = ensure(s->d_tiles32, s->tiles32_cap, std::max<size_t>(tiles32.size(), 1)))) return rc;
        if ((rc = ensure(s->d_p32, s->p32_cap, (size_t)A))) return rc;
        if ((rc = ensure(s->d_cq32, s->cq32_cap, (size_t)A))) return rc;
        if ((rc = ensure(s->d_cq4, s->cq4_cap, (size_t)A))) return rc;
        if ((rc = ensure(s->d_pf4, s->pf4_cap, (size_t)A))) return rc;
        if ((rc = ensure(s->d_magblk, s->magblk_cap, (size_t)(3 * (A / 256 + 1))))) return rc;
        if (!tiles32.empty())
            CU(cudaMemcpyAsync(s->d_tiles32, tiles32.data(), tiles32.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
    }
    const long long T32 = (fp32 && tiles_cached) ? s->tc_T32 : (long long)tiles32.size();
    if (!tiles_cached) {
        s->tc_key[0] = n; s->tc_key[1] = lmin; s->tc_key[2] = band_lo; s->tc_key[3] = band_hi;
        s->tc_key[4] = mode_key;
        s->tc_T = T; s->tc_Ts = Ts; s->tc_T32 = T32;
    }
    const long long run_cap_full = (long long)(s->log_cap * sizeof(RowRec) / sizeof(Run));
    const size_t smem = WARPS_PER_CTA * sizeof(WarpSmem);
    CU(cudaFuncSetAttribute(k_tile<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CU(cudaFuncSetAttribute(k_tile<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const double margin = 1.0 / (1 << 26);
    // VLMP_LOG_CAP (records) lowers the effective log capacity: a test hook that forces the
    // overflow -> exact full-fold re-run path
    long long eff_cap = (long long)s->log_cap;
    if (const char* env = getenv("VLMP_LOG_CAP")) eff_cap = std::max(1LL, std::min(eff_cap, atoll(env)));
    long long run_cap = run_cap_full;
    if (const char* env = getenv("VLMP_LOG_CAP")) run_cap = std::max(1LL, std::min(run_cap, atoll(env)));
    if (li_lo < 0) li_lo = 0;
    if (li_hi >= n_len || (li_hi < 0 && li_lo == 0)) li_hi = n_len - 1;   // default: every length
    if (li_hi < li_lo) li_hi = -1;                                        // empty shard: no work
    while (s->lev.size() < (size_t)2 * n_len) { cudaEvent_t ev; CU(cudaEventCreate(&ev)); s->lev.push_back(ev); }
    if ((rc = ensure(s->d_span, s->span_cap, (size_t)4 * n_len))) return rc;
    if ((size_t)4 * n_len > s->h_span_cap) {
        if (s->h_span) cudaFreeHost(s->h_span);
        s->h_span = nullptr; s->h_span_cap = 0;
        CU(cudaMallocHost((void**)&s->h_span, (size_t)4 * n_len * sizeof(unsigned long long)));
        s->h_span_cap = (size_t)4 * n_len;
    }
    if (fp32 && (rc = filter32_setup())) return rc;

    const bool dumping = getenv("VLMP_DUMP_PRM") || getenv("VLMP_DUMP_RUNS");
    // Two chains. A length of a small series is a short kernel sequence (config 2: ~4,000 tiles
    // for 2,368 resident warps, then k_runs, the bounds and the factors of the next length, each
    // waiting for the one before): the walk ramps up and drains every ~0.4 ms and the GPU idles
    // in between. So the range is cut into two contiguous halves of equal work that run
    // concurrently on two streams (forked and joined inside the graph): while one chain is
    // between walks, the other's tiles fill the SMs. The second chain starts like a length
    // shard (direct-sum seeds, sampled folds for its first bounds) with its own per-length
    // scratch; accumulators are per length and the counters atomic, so they are shared.
    int chains = 1, chain_cut = 0;
    {
        const char* ce = getenv("VLMP_CHAINS");
        const int want = ce ? atoi(ce) : 0;   // 0: automatic, 1: off, 2: on wherever it applies
        // >= 40 lengths: the second chain pays a first length (~4 lengths' time) and hides ~16 % of
        // the others' (a 32-length shard of config 2: 19.1 ms as one chain, 20.0 as two)
        const int lo0 = li_lo <= li_hi ? li_lo : 0;
        const bool ok = fp32 && flags == 0 && band_lo == 0 && band_hi == nb && li_hi - lo0 + 1 >= (want == 2 ? 16 : 40) && !dumping && T32 > 0;
        if (ok && (want == 2 || (want == 0 && T32 <= 16 * 2368))) {
            double tot = 0, acc_w = 0;
            auto work = [&](int li) { const double k = (double)(n - (lmin + li) + 1 - (lmin + li + 1) / 2); return k > 0 ? k * (k + 1) : 0.0; };
            for (int li = lo0; li <= li_hi; ++li) tot += work(li);
            int cut = lo0;
            for (; cut <= li_hi && acc_w + work(cut) <= 0.5 * tot; ++cut) acc_w += work(cut);
            cut = std::min(std::max(cut + 2, lo0 + 4), li_hi - 3);   // the second chain also pays a first length
            chains = 2; chain_cut = cut;
            if ((rc = ensure(s->x_prm, s->x_prm_cap, (size_t)A))) return rc;
            if ((rc = ensure(s->x_prm2, s->x_prm2_cap, (size_t)A))) return rc;
            if ((rc = ensure(s->x_mu, s->x_mu_cap, (size_t)A))) return rc;
            if ((rc = ensure(s->x_mu2, s->x_mu2_cap, (size_t)A))) return rc;
            if ((rc = ensure(s->x_p32, s->x_p32_cap, (size_t)A))) return rc;
            if ((rc = ensure(s->x_cq32, s->x_cq32_cap, (size_t)A))) return rc;
            if ((rc = ensure(s->x_cq4, s->x_cq4_cap, (size_t)A))) return rc;
            if ((rc = ensure(s->x_pf4, s->x_pf4_cap, (size_t)A))) return rc;
            if ((rc = ensure(s->x_magblk, s->x_magblk_cap, (size_t)(3 * (A / 256 + 1))))) return rc;
            if ((rc = ensure(s->x_seeds, s->x_seeds_cap, (size_t)std::max<long long>(T, 1) * BAND))) return rc;
            if ((rc = ensure(s->x_log, s->x_log_cap, s->log_cap))) return rc;
            if (!s->stream2) CU(cudaStreamCreateWithFlags(&s->stream2, cudaStreamNonBlocking));
            if (!s->ev_fork) CU(cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming));
            if (!s->ev_join) CU(cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming));
        }
    }
    auto swap_scratch = [&]() {
        std::swap(s->d_prm, s->x_prm); std::swap(s->d_prm2, s->x_prm2); std::swap(s->d_mu, s->x_mu);
        std::swap(s->d_mu2, s->x_mu2); std::swap(s->d_p32, s->x_p32); std::swap(s->d_cq32, s->x_cq32);
        std::swap(s->d_cq4, s->x_cq4); std::swap(s->d_pf4, s->x_pf4); std::swap(s->d_magblk, s->x_magblk);
        std::swap(s->d_seeds, s->x_seeds); std::swap(s->d_log, s->x_log);
    };
    // a CUDA graph of the whole sequence (VLMP_GRAPH=0 / dumping: plain stream launches). Inside
    // the graph, kernel times come from device-clock spans, not events (an event node between
    // kernels serialises the graph at every length: +12 ms per config-2 pass, measured)
    const bool use_graph = !dumping && !(getenv("VLMP_GRAPH") && atoi(getenv("VLMP_GRAPH")) == 0);
    // counters of the launch sequence (host bookkeeping only)
    double executed = 0, launches = 0, n_filtered = 0, n_full = 0, klaunch = 2, n_walk = 0;
    std::vector<int> timed;   // lengths whose tile pass ran (event pairs)
    std::vector<int> walked;  // lengths whose FP32 walk ran (k_tile32 / k_runs events)
    // The whole per-length sequence is pure stream work (no host decisions between lengths), so
    // it is captured once into a CUDA graph and re-launched while the key below is unchanged:
    // ~6 launches per length become one graph launch (no per-launch host cost in the step).
    // one chain: lengths li_lo..li_hi (the arguments shadow the call's range) on stream st,
    // with whatever per-length scratch the session's pointers name at the moment
    auto run_chain = [&](cudaStream_t st, int li_lo, int li_hi) -> int {
        int rc2;
        Run* runs = reinterpret_cast<Run*>(s->d_log);
        if (li_lo > 0 && li_lo <= li_hi && T) {
            if (fp32) {
                // a later length shard on the FP32 walk: the seeds only start the walk (its slack
                // covers their rounding; keys come from the exact runs), so they are direct sums at
                // the shard's first length -- no carry through the lengths before it
                const int m0 = lmin + li_lo;
                ParamArgs pa{s->d_tn, s->d_cum, s->d_cum2, s->d_prm, s->d_mu, n, n - m0 + 1, A, m0, s->floor_};
                k_params<<<blocks(A, 256), 256, 0, st>>>(pa);
                SeedArgs sa{s->d_tn, s->d_mu, s->d_tiles, s->d_seeds, dl, (int)T, S, m0};
                k_seed_init<<<blocks(T * 32, WARPS_PER_CTA * 32), WARPS_PER_CTA * 32, 0, st>>>(sa);
                klaunch += 2;
            } else {
                // FP64 walk: seeds at lmin (direct sums), carried to the shard's first length with
                // the tile kernel's own Welford step (bit-identical to the single-GPU chain)
                ParamArgs pa{s->d_tn, s->d_cum, s->d_cum2, s->d_prm, s->d_mu, n, n - lmin + 1, A, lmin, s->floor_};
                k_params<<<blocks(A, 256), 256, 0, st>>>(pa);
                SeedArgs sa{s->d_tn, s->d_mu, s->d_tiles, s->d_seeds, dl, (int)T, S, lmin};
                k_seed_init<<<blocks(T * 32, WARPS_PER_CTA * 32), WARPS_PER_CTA * 32, 0, st>>>(sa);
                k_seed_forward<<<blocks(T * 32, 128), 128, 0, st>>>(sa, s->d_cum, lmin + li_lo);
                klaunch += 3;
            }
        }
        for (int li = li_lo; li <= li_hi; ++li) {
            const int m = lmin + li;
            const long long N = n - m + 1;
            const int e = (m + 1) / 2;
            // window parameters ping-pong between two buffers: the bound reads length m-1's
            Prm* prm = (li & 1) ? s->d_prm2 : s->d_prm;
            double* mu = (li & 1) ? s->d_mu2 : s->d_mu;
            const Prm* prm_prev = (li & 1) ? s->d_prm : s->d_prm2;
            const double* mu_prev = (li & 1) ? s->d_mu : s->d_mu2;
            ParamArgs pa{s->d_tn, s->d_cum, s->d_cum2, prm, mu, n, N, A, m, s->floor_};
            launch_hi(k_params, dim3((unsigned)blocks(A, 256)), dim3(256), 0, st, pa);
            ++klaunch;
            const bool full = (li == li_lo) || (flags & VLMP_F_FULL_EVERY_LENGTH);
            if (li == 0 && T) {
                SeedArgs sa{s->d_tn, mu, s->d_tiles, s->d_seeds, dl, (int)T, S, m};
                k_seed_init<<<blocks(T * 32, WARPS_PER_CTA * 32), WARPS_PER_CTA * 32, 0, st>>>(sa);
                ++klaunch;
            }
            if (!full) {
                Bound2Args ba{s->d_tn, prm, prm_prev, mu_prev, mu, s->d_acc + (long long)(li - 1) * A, prm,
                              N, N + 1, m, e, margin, s->d_fixcnt + li, fp32 ? 1 : 0};
                launch_hi(k_bound2, dim3((unsigned)blocks(N, 256)), dim3(256), 0, st, ba);
                if (!fp32)
                    k_qprep<<<blocks(A, 256), 256, 0, st>>>(prm, s->d_colq, s->d_rowq, N, A, s->sscale,
                                                            s->d_forced + li);
                klaunch += 2;
            }
            timed.push_back(li);
            if (!use_graph) CU(cudaEventRecord(s->lev[2 * li], st));
            unsigned long long* span = s->d_span + 4 * li;
            if (T) {
                TileArgs ta{prm, mu, s->d_tn, s->d_tiles, s->d_seeds, s->d_acc + (long long)li * A,
                            s->d_counters, s->d_log, s->d_logcnt + li, eff_cap,
                            N, dl, (int)T, S, m, e, li + 1 <= li_hi,
                            s->d_colq, s->d_rowq, s->d_forced + li, s->hiC};
                if (full && li == li_lo && bound_start && Ts) {
                    // sampled full folds (seeds untouched) -> bounds -> filtered pass over all bands
                    TileArgs tsa = ta;
                    tsa.tiles = s->d_tiles_s; tsa.n_tiles = (int)Ts; tsa.seed_map = s->d_smap; tsa.update_seeds = 0;
                    k_tile<true><<<blocks(Ts, WARPS_PER_CTA), WARPS_PER_CTA * 32, smem, st>>>(tsa);
                    k_bound_self<<<blocks(N, 256), 256, 0, st>>>(s->d_acc + (long long)li * A, prm, N, margin,
                                                                 s->d_tn, mu, m, fp32 ? 1 : 0);
                    if (fp32) {
                        // the sampled folds only bound this length; its keys come from the exact runs
                        k_fill_acc<<<blocks(A, 256), 256, 0, st>>>(s->d_acc + (long long)li * A, A);
                        if ((rc2 = launch_filter32(s, st, prm, mu, N, m, e, dl, S, ta.update_seeds, T32,
                                                   s->d_forced + li, s->d_acc + (long long)li * A, runs,
                                                   s->d_logcnt + li, run_cap, nullptr, nullptr, span))) return rc2;
                        klaunch += 5; n_walk += 1; walked.push_back(li);
                    } else {
                        k_qprep<<<blocks(A, 256), 256, 0, st>>>(prm, s->d_colq, s->d_rowq, N, A, s->sscale,
                                                                s->d_forced + li);
                        k_tile<false><<<blocks(T, WARPS_PER_CTA), WARPS_PER_CTA * 32, smem, st>>>(ta);
                        k_log_merge<<<148 * 8, 256, 0, st>>>(s->d_log, s->d_logcnt + li, eff_cap,
                                                             prm, e, s->d_acc + (long long)li * A, s->d_counters);
                        klaunch += 4;
                    }
                } else if (full) k_tile<true><<<blocks(T, WARPS_PER_CTA), WARPS_PER_CTA * 32, smem, st>>>(ta);
                else if (fp32) {
                    if ((rc2 = launch_filter32(s, st, prm, mu, N, m, e, dl, S, ta.update_seeds, T32, s->d_forced + li,
                                               s->d_acc + (long long)li * A, runs, s->d_logcnt + li, run_cap,
                                               nullptr, nullptr, span)))
                        return rc2;
                    klaunch += 2; n_walk += 1; walked.push_back(li);
                    if (dumping && (rc2 = debug_dump(st, li, prm, N, runs, s->d_logcnt + li, run_cap))) return rc2;
                } else {
                    k_tile<false><<<blocks(T, WARPS_PER_CTA), WARPS_PER_CTA * 32, smem, st>>>(ta);
                    k_log_merge<<<148 * 8, 256, 0, st>>>(s->d_log, s->d_logcnt + li, eff_cap,
                                                         prm, e, s->d_acc + (long long)li * A, s->d_counters);
                    klaunch += 1;
                }
                launches += 1; klaunch += 1;
            }
            if (!use_graph) CU(cudaEventRecord(s->lev[2 * li + 1], st));
            CU(cudaGetLastError());
            for (long long b = band_lo; b < band_hi; ++b) {
                long long d0 = dl + b * BAND;
                long long rows = N - d0;
                if (rows <= 0 || d0 + BAND - 1 < e) continue;
                executed += (double)rows * BAND;
            }
            if (full) n_full += 1; else n_filtered += 1;
        }
        return 0;
    };
    auto enqueue = [&]() -> int {
        k_fill_acc<<<blocks((long long)n_len * A, 256), 256, 0, st>>>(s->d_acc, (long long)n_len * A);
        CU(cudaMemsetAsync(s->d_counters, 0, 8 * sizeof(unsigned long long), st));
        CU(cudaMemsetAsync(s->d_fixcnt, 0, n_len * sizeof(unsigned long long), st));
        CU(cudaMemsetAsync(s->d_logcnt, 0, n_len * sizeof(unsigned long long), st));
        CU(cudaMemsetAsync(s->d_forced, 0, n_len * sizeof(int), st));
        k_span_init<<<blocks(n_len, 128), 128, 0, st>>>(s->d_span, n_len);
        const int lo0 = li_lo <= li_hi ? li_lo : 0;
        if (chains == 1) return run_chain(st, lo0, li_hi);
        // fork: the second chain's stream joins the capture (or, without a graph, just waits)
        CU(cudaEventRecord(s->ev_fork, st));
        CU(cudaStreamWaitEvent(s->stream2, s->ev_fork, 0));
        int rc2 = run_chain(st, lo0, chain_cut - 1);
        swap_scratch();
        const int rc3 = rc2 ? 0 : run_chain(s->stream2, chain_cut, li_hi);
        swap_scratch();
        CU(cudaEventRecord(s->ev_join, s->stream2));
        CU(cudaStreamWaitEvent(st, s->ev_join, 0));
        return rc2 ? rc2 : rc3;
    };
    CU(cudaEventRecord(s->ev[0], st));
    if (use_graph) {
        // everything the captured launches bake in: shape, mode, buffers, series scalars
        std::vector<double> key = {(double)n, (double)A, (double)lmin, (double)lmax, (double)band_lo, (double)band_hi,
                                   (double)flags, (double)li_lo, (double)li_hi, (double)T, (double)Ts, (double)T32,
                                   (double)S, (double)eff_cap, (double)run_cap, s->sscale, s->floor_,
                                   (double)s->hiC, (double)bound_start, (double)fp32, (double)chains, (double)chain_cut,
                                   (double)(uintptr_t)s->x_prm, (double)(uintptr_t)s->x_prm2, (double)(uintptr_t)s->x_mu,
                                   (double)(uintptr_t)s->x_mu2, (double)(uintptr_t)s->x_p32, (double)(uintptr_t)s->x_cq32,
                                   (double)(uintptr_t)s->x_cq4, (double)(uintptr_t)s->x_pf4, (double)(uintptr_t)s->x_magblk,
                                   (double)(uintptr_t)s->x_seeds, (double)(uintptr_t)s->x_log};
        for (const void* ptr : {(const void*)s->d_acc, (const void*)s->d_tn, (const void*)s->d_cum, (const void*)s->d_cum2,
                                (const void*)s->d_prm, (const void*)s->d_prm2, (const void*)s->d_mu, (const void*)s->d_mu2,
                                (const void*)s->d_tiles, (const void*)s->d_tiles_s, (const void*)s->d_smap,
                                (const void*)s->d_seeds, (const void*)s->d_log, (const void*)s->d_logcnt,
                                (const void*)s->d_forced, (const void*)s->d_fixcnt, (const void*)s->d_tiles32,
                                (const void*)s->d_p32, (const void*)s->d_cq32, (const void*)s->d_cq4, (const void*)s->d_pf4,
                                (const void*)s->d_magblk, (const void*)s->d_colq, (const void*)s->d_rowq})
            key.push_back((double)(uintptr_t)ptr);
        if (!s->g_exec || key != s->g_key) {
            if (s->g_exec) { cudaGraphExecDestroy(s->g_exec); s->g_exec = nullptr; }
            s->g_key.clear();
            CU(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
            const int rc_cap = enqueue();
            cudaGraph_t g = nullptr;
            const cudaError_t ec = cudaStreamEndCapture(st, &g);
            if (rc_cap) { if (g) cudaGraphDestroy(g); return rc_cap; }
            if (ec != cudaSuccess) return fail(VLMP_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(ec));
            unsigned long long inst_flags = 0;
            if (chains > 1 && !getenv("VLMP_NO_NODE_PRIO")) {
                // With two chains the short kernels between a chain's walks must not queue behind the
                // other chain's pending walk blocks: every node but the walks gets the highest
                // priority, and the graph is instantiated to use node priorities (a launch
                // attribute set during capture does not reach the node; without the instantiate
                // flag the nodes run at the launch stream's priority).
                size_t nn = 0;
                int p_lo = 0, p_hi = 0;
                cudaDeviceGetStreamPriorityRange(&p_lo, &p_hi);
                if (cudaGraphGetNodes(g, nullptr, &nn) == cudaSuccess && nn) {
                    std::vector<cudaGraphNode_t> nodes(nn);
                    cudaGraphGetNodes(g, nodes.data(), &nn);
                    for (cudaGraphNode_t nd : nodes) {
                        cudaGraphNodeType ty;
                        if (cudaGraphNodeGetType(nd, &ty) != cudaSuccess || ty != cudaGraphNodeTypeKernel) continue;
                        cudaKernelNodeParams kp;
                        if (cudaGraphKernelNodeGetParams(nd, &kp) != cudaSuccess) continue;
                        cudaKernelNodeAttrValue v;
                        v.priority = kp.func == tile32_func() ? p_lo : p_hi;
                        cudaGraphKernelNodeSetAttribute(nd, cudaKernelNodeAttributePriority, &v);
                    }
                    inst_flags = cudaGraphInstantiateFlagUseNodePriority;
                }
                cudaGetLastError();
            }
            const cudaError_t ei = cudaGraphInstantiateWithFlags(&s->g_exec, g, inst_flags);
            cudaGraphDestroy(g);
            if (ei != cudaSuccess) { s->g_exec = nullptr; return fail(VLMP_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ei)); }
            s->g_key = key;
            s->g_cnt = {executed, launches, n_filtered, n_full, klaunch, n_walk};
            s->g_timed = timed; s->g_walked = walked;
        } else {
            // the cached sequence: its host-side counters are those of the capture
            executed = s->g_cnt[0]; launches = s->g_cnt[1]; n_filtered = s->g_cnt[2]; n_full = s->g_cnt[3];
            klaunch = s->g_cnt[4]; n_walk = s->g_cnt[5]; timed = s->g_timed; walked = s->g_walked;
        }
        CU(cudaGraphLaunch(s->g_exec, st));
    } else if ((rc = enqueue())) return rc;
    CU(cudaEventRecord(s->ev[1], st));
    CU(cudaMemcpyAsync(s->h_span, s->d_span, (size_t)4 * n_len * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    // the overflow check's inputs, copied behind the sequence (pinned: truly asynchronous)
    {
        const size_t need = 8 + 3 * (size_t)n_len;
        if (need > s->h_chk_cap) {
            if (s->h_chk) cudaFreeHost(s->h_chk);
            s->h_chk = nullptr; s->h_chk_cap = 0;
            CU(cudaMallocHost((void**)&s->h_chk, need * sizeof(unsigned long long)));
            s->h_chk_cap = need;
        }
        unsigned long long* h = s->h_chk;
        CU(cudaMemcpyAsync(h, s->d_counters, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(h + 8, s->d_logcnt, n_len * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(h + 8 + n_len, s->d_fixcnt, n_len * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(h + 8 + 2 * n_len, s->d_forced, n_len * sizeof(int), cudaMemcpyDeviceToHost, st));
    }
    CU(cudaGetLastError());
    PendingRun& pr = s->prun;
    pr = PendingRun{};
    pr.lmin = lmin; pr.lmax = lmax; pr.band_lo = band_lo; pr.band_hi = band_hi; pr.flags = flags;
    pr.li_lo = li_lo; pr.li_hi = li_hi; pr.fp32 = fp32; pr.sampled = sampled_start;
    pr.cap_used = fp32 ? run_cap : eff_cap; pr.S = S;
    pr.executed = executed; pr.launches = launches; pr.n_filtered = n_filtered; pr.n_full = n_full;
    pr.klaunch = klaunch; pr.graph = use_graph; pr.timed = timed; pr.walked = walked; pr.chains = chains;
    s->lmin = lmin; s->lmax = lmax; s->n_len = n_len;
    s->have_profile = true; s->have_final = false; s->have_finals = false;
    s->pending = true; s->stats_dirty = true;
    return 0;
}

}  // extern "C" (reopened below)

namespace vlmp_impl {

// Device-event timings of the last run (lazily: only vlmp_stats needs them).
// one exhaustive 1-best pass with the session lock held (pruned.cu's full lengths)
int profile_locked(vlmp_session* s, int lmin, int lmax) {
    return profile_impl(s, lmin, lmax, 0, -1, 0, 0, -1);
}

int fill_event_stats(vlmp_session* s) {
    if (!s->stats_dirty) return 0;
    const PendingRun& pr = s->prun;
    double first_ms = 0, tile_ms = 0, walk_ms = 0, runs_ms = 0;
    for (int li : pr.walked) {
        const unsigned long long* sp = s->h_span + 4 * li;
        if (sp[1] > sp[0]) walk_ms += (double)(sp[1] - sp[0]) * 1e-6;
        if (sp[3] > sp[2]) runs_ms += (double)(sp[3] - sp[2]) * 1e-6;
    }
    if (pr.chains > 1) {
        // two concurrent chains: their walk kernels share the SMs, so a launch's own span counts
        // time it spent beside the other chain's launch. The walk's time is the union of the
        // spans -- the time during which a walk kernel was running at all.
        std::vector<std::pair<unsigned long long, unsigned long long>> iv;
        for (int li : pr.walked) {
            const unsigned long long* sp = s->h_span + 4 * li;
            if (sp[1] > sp[0]) iv.push_back({sp[0], sp[1]});
        }
        std::sort(iv.begin(), iv.end());
        unsigned long long covered = 0, cur_lo = 0, cur_hi = 0;
        for (const auto& x : iv) {
            if (x.first > cur_hi) { covered += cur_hi - cur_lo; cur_lo = x.first; cur_hi = x.second; }
            else cur_hi = std::max(cur_hi, x.second);
        }
        covered += cur_hi - cur_lo;
        walk_ms = (double)covered * 1e-6;
    }
    if (const char* sp_path = getenv("VLMP_DUMP_SPANS")) {   // dev aid: per-length kernel spans (ns, device clock)
        if (FILE* f = fopen(sp_path, "w")) {
            for (int li : pr.walked) {
                const unsigned long long* sp = s->h_span + 4 * li;
                fprintf(f, "%d %llu %llu %llu %llu\n", li, sp[0], sp[1], sp[2], sp[3]);
            }
            fclose(f);
        }
    }
    if (!pr.graph) {
        for (int li : pr.timed) {
            float lm = 0; CU(cudaEventElapsedTime(&lm, s->lev[2 * li], s->lev[2 * li + 1]));
            tile_ms += lm;
            if (li == pr.li_lo) first_ms = lm;
        }
    } else {
        tile_ms = walk_ms + runs_ms;   // the graph carries no per-length events
    }
    float ms = 0; CU(cudaEventElapsedTime(&ms, s->ev[0], s->ev[1]));
    s->stats[0] = ms; s->stats[4] = tile_ms; s->stats[10] = first_ms;
    s->stats[20] = walk_ms; s->stats[21] = runs_ms;
    if (s->have_finals) { float fm = 0; if (cudaEventElapsedTime(&fm, s->ev[4], s->ev[5]) == cudaSuccess) s->stats[1] = fm; }
    s->stats_dirty = false;
    return 0;
}

// Wait for the pending phase 1, check its logs and, when one overflowed (it lost candidates),
// redo the run exactly: the FP32 walk's overflow on the FP64 filter path, then without the
// sampled first-length start (its bounds are the loosest), then with full folds everywhere.
// *redone tells a caller that already enqueued phase-2 work on the lost run to enqueue it again.
int settle_profile(vlmp_session* s, bool* redone) {
    int code = 0;
    while (s->pending) {
        CU(cudaStreamSynchronize(s->stream));
        s->pending = false;
        const PendingRun pr = s->prun;
        const int n_len = pr.lmax - pr.lmin + 1;
        const unsigned long long* h = s->h_chk;
        bool overflow = false;
        double max_log = 0, n_fix = 0;
        int n_forced = 0;
        for (int li = 0; li < n_len; ++li) {
            overflow |= (long long)h[8 + li] > pr.cap_used;
            max_log = std::max(max_log, (double)h[8 + li]);
            n_fix += (double)h[8 + n_len + li];
            n_forced += reinterpret_cast<const int*>(h + 8 + 2 * n_len)[li] != 0;
        }
        double W = 0;
        for (int m = pr.lmin; m <= pr.lmax; ++m) {
            long long k = (s->n - m + 1) - (m + 1) / 2;
            if (k > 0) W += (double)k * (double)(k + 1) / 2.0;
        }
        memset(s->stats, 0, sizeof(s->stats));
        s->stats[2] = pr.executed; s->stats[3] = W;
        s->stats[5] = pr.launches; s->stats[6] = pr.n_filtered; s->stats[7] = pr.n_full; s->stats[8] = (double)h[0];
        s->stats[9] = pr.klaunch; s->stats[11] = (double)h[2];
        s->stats[12] = n_fix; s->stats[14] = n_forced; s->stats[15] = max_log;
        s->stats[16] = pr.fp32 ? 1.0 : 0.0; s->stats[17] = pr.fp32 ? max_log : 0.0; s->stats[18] = (double)h[4];
        s->stats[19] = (double)pr.S; s->stats[22] = (double)pr.walked.size(); s->stats[23] = pr.graph ? 1.0 : 0.0;
        s->stats[24] = (double)pr.chains;
        s->stats_dirty = true;
        if (!overflow) break;
        if (redone) *redone = true;
        uint32_t f = pr.flags;
        if (pr.fp32) { f |= VLMP_F_FP64_FILTER; code = 3; }
        else if (pr.sampled) { f |= F_NO_SAMPLED_START; code = 1; }
        else if (!(f & VLMP_F_FULL_EVERY_LENGTH)) { f |= VLMP_F_FULL_EVERY_LENGTH; code = 2; }
        else return fail(VLMP_E_CUDA, "candidate log overflow with full folds");
        int rc = profile_impl(s, pr.lmin, pr.lmax, pr.band_lo, pr.band_hi, f, pr.li_lo, pr.li_hi);
        if (rc) return rc;
    }
    if (code) s->stats[13] = code;
    return 0;
}

}  // namespace vlmp_impl

extern "C" {

int vlmp_profile_range(vlmp_session* s, int32_t lmin, int32_t lmax, int64_t band_lo,
                       int64_t band_hi, uint32_t flags) {
    if (!s) return fail(VLMP_E_INVALID_PARAMETERS, "null session");
    if (s->n <= 0) return fail(VLMP_E_STATE, "no series uploaded");
    if (lmin > lmax) return fail(VLMP_E_INVALID_PARAMETERS, "lmin > lmax");
    if (lmin < 4) return fail(VLMP_E_INVALID_PARAMETERS, "minimum window length is 4");
    if (s->n < (long long)lmax + (lmax + 1) / 2)
        return fail(VLMP_E_SERIES_TOO_SHORT, "series cannot host a non-trivial pair at lmax");
    std::lock_guard<std::mutex> g(s->lock);
    return profile_impl(s, lmin, lmax, band_lo, band_hi, flags, 0, -1);
}

int vlmp_profile_lengths(vlmp_session* s, int32_t lmin, int32_t lmax, int32_t li_lo, int32_t li_hi,
                         uint32_t flags) {
    if (!s) return fail(VLMP_E_INVALID_PARAMETERS, "null session");
    if (s->n <= 0) return fail(VLMP_E_STATE, "no series uploaded");
    if (lmin > lmax) return fail(VLMP_E_INVALID_PARAMETERS, "lmin > lmax");
    if (lmin < 4) return fail(VLMP_E_INVALID_PARAMETERS, "minimum window length is 4");
    if (li_lo < 0 || li_hi < li_lo - 1 || li_hi > lmax - lmin)   // li_hi = li_lo - 1: empty shard
        return fail(VLMP_E_INVALID_PARAMETERS, "length shard outside [0, lmax - lmin]");
    if (s->n < (long long)lmax + (lmax + 1) / 2)
        return fail(VLMP_E_SERIES_TOO_SHORT, "series cannot host a non-trivial pair at lmax");
    std::lock_guard<std::mutex> g(s->lock);
    if (li_hi < li_lo) { li_lo = lmax - lmin + 1; li_hi = -1; }   // empty shard: setup only
    return profile_impl(s, lmin, lmax, 0, -1, flags, li_lo, li_hi);
}

int vlmp_partials_size(vlmp_session* s, int64_t* n_len, int64_t* stride) {
    if (!s || !s->have_profile) return fail(VLMP_E_STATE, "no profile run");
    *n_len = s->n_len; *stride = s->A;
    return 0;
}

int vlmp_partials_export(vlmp_session* s, void* keys, void* idx) {
    if (!s || !s->have_profile) return fail(VLMP_E_STATE, "no profile run");
    std::lock_guard<std::mutex> g(s->lock);
    { const int rc = settle_profile(s, nullptr); if (rc) return rc; }
    CU(cudaSetDevice(s->device));
    const long long total = (long long)s->n_len * s->A;
    k_export<<<blocks(total, 256), 256, 0, s->stream>>>(s->d_acc, (unsigned long long*)keys, (long long*)idx, total);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(s->stream));
    return 0;
}

int vlmp_partials_mask_idx(vlmp_session* s, const void* merged_keys, const void* keys, void* idx) {
    if (!s || !s->have_profile) return fail(VLMP_E_STATE, "no profile run");
    std::lock_guard<std::mutex> g(s->lock);
    { const int rc = settle_profile(s, nullptr); if (rc) return rc; }
    CU(cudaSetDevice(s->device));
    const long long total = (long long)s->n_len * s->A;
    k_mask_idx<<<blocks(total, 256), 256, 0, s->stream>>>((const unsigned long long*)merged_keys,
                                                            (const unsigned long long*)keys, (long long*)idx, total);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(s->stream));
    return 0;
}

int vlmp_partials_import(vlmp_session* s, const void* keys, const void* idx) {
    if (!s || !s->have_profile) return fail(VLMP_E_STATE, "no profile run");
    std::lock_guard<std::mutex> g(s->lock);
    { const int rc = settle_profile(s, nullptr); if (rc) return rc; }
    CU(cudaSetDevice(s->device));
    const long long total = (long long)s->n_len * s->A;
    k_import<<<blocks(total, 256), 256, 0, s->stream>>>(s->d_acc, (const unsigned long long*)keys, (const long long*)idx, total);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(s->stream));
    return 0;
}

int vlmp_profile_mbest(vlmp_session* s, int32_t lmin, int32_t lmax, int32_t mb) {
    if (!s) return fail(VLMP_E_INVALID_PARAMETERS, "null session");
    if (s->n <= 0) return fail(VLMP_E_STATE, "no series uploaded");
    if (lmin > lmax) return fail(VLMP_E_INVALID_PARAMETERS, "lmin > lmax");
    if (lmin < 4) return fail(VLMP_E_INVALID_PARAMETERS, "minimum window length is 4");
    if (mb < 1 || mb > MB_MAX) return fail(VLMP_E_INVALID_PARAMETERS, "m must be in [1, 8]");
    if (s->n < (long long)lmax + (lmax + 1) / 2)
        return fail(VLMP_E_SERIES_TOO_SHORT, "series cannot host a non-trivial pair at lmax");
    std::lock_guard<std::mutex> g(s->lock);
    return mbest_impl(s, lmin, lmax, mb);
}

}  // extern "C" (reopened below)

namespace vlmp_impl {
// the m-best profile run (caller holds the session lock): d_ipm / d_mpm of [lmin, lmax]
int mbest_impl(vlmp_session* s, int32_t lmin, int32_t lmax, int32_t mb) {
    { const int rc0 = settle_profile(s, nullptr); if (rc0) return rc0; }
    CU(cudaSetDevice(s->device));
    cudaStream_t st = s->stream;
    const long long n = s->n, A = s->A;
    const int n_len = lmax - lmin + 1;
    const long long nb = n_bands_for(n, lmin);
    const int S = seg_rows(n);
    const long long N0 = n - lmin + 1, dl = dlo_for(lmin);
    std::vector<int2> tiles;
    for (long long b = 0; b < nb; ++b) {
        long long rows = N0 - (dl + b * BAND);
        for (long long sg = 0; sg * S < rows; ++sg) tiles.push_back(make_int2((int)b, (int)sg));
    }
    order_tiles(tiles, N0, dl, S);
    const long long T = (long long)tiles.size();
    // the tile buffers below are overwritten with this run's all-band list: the cached 1-best
    // tile lists (profile_impl's tc_key) and any earlier m-best result are void from here on
    s->tc_key[0] = -1;
    s->mbest = 0; s->mb_lmin = s->mb_n_len = 0; s->mb_A = 0;
    int rc;
    if ((rc = ensure(s->d_tiles, s->tiles_cap, (size_t)std::max<long long>(T, 1)))) return rc;
    if ((rc = ensure(s->d_seeds, s->seeds_cap, (size_t)std::max<long long>(T, 1) * BAND))) return rc;
    if ((rc = ensure(s->d_acc, s->acc_cap, (size_t)A))) return rc;
    const size_t log_cap = log_capacity(N0);
    if ((rc = ensure(s->d_log, s->log_cap, log_cap))) return rc;
    if ((rc = ensure(s->d_logcnt, s->logcnt_cap, (size_t)n_len))) return rc;
    if ((rc = ensure(s->d_slots, s->slots_cap, (size_t)A * SLOT_CAP))) return rc;
    if ((rc = ensure(s->d_slotcnt, s->slotcnt_cap, (size_t)A))) return rc;
    if ((rc = ensure(s->d_ipm, s->ipm_cap, (size_t)n_len * A * mb))) return rc;
    if ((rc = ensure(s->d_redo, s->redo_cap, (size_t)A))) return rc;
    if (!s->d_ro_cnt) CU(cudaMalloc((void**)&s->d_ro_cnt, 8));
    CU(cudaMemsetAsync(s->d_logcnt, 0, n_len * sizeof(unsigned long long), st));
    CU(cudaMemsetAsync(s->d_slotcnt, 0, A * sizeof(int), st));
    CU(cudaMemsetAsync(s->d_counters, 0, 8 * sizeof(unsigned long long), st));
    if (T) CU(cudaMemcpyAsync(s->d_tiles, tiles.data(), T * sizeof(int2), cudaMemcpyHostToDevice, st));
    const size_t smem = WARPS_PER_CTA * sizeof(WarpSmem);
    CU(cudaFuncSetAttribute(k_tile<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CU(cudaFuncSetAttribute(k_tile<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // the filtered pass: FP32 walk + exact runs into the candidate slots (filter32.cu) unless the
    // FP64 walk + covariance log is asked for (VLMP_FP64_FILTER, A/B checks)
    const bool fp32 = !getenv("VLMP_FP64_FILTER");
    std::vector<int4> tiles32;
    Run* runs = reinterpret_cast<Run*>(s->d_log);
    const long long run_cap = (long long)(s->log_cap * sizeof(RowRec) / sizeof(Run));
    if (fp32) {
        build_tiles32(tiles, 0, tiles32);
        if ((rc = ensure(s->d_tiles32, s->tiles32_cap, std::max<size_t>(tiles32.size(), 1)))) return rc;
        if ((rc = ensure(s->d_p32, s->p32_cap, (size_t)A))) return rc;
        if ((rc = ensure(s->d_cq32, s->cq32_cap, (size_t)A))) return rc;
        if ((rc = ensure(s->d_cq4, s->cq4_cap, (size_t)A))) return rc;
        if ((rc = ensure(s->d_pf4, s->pf4_cap, (size_t)A))) return rc;
        if ((rc = ensure(s->d_magblk, s->magblk_cap, (size_t)(3 * (A / 256 + 1))))) return rc;
        if ((rc = ensure(s->d_forced, s->forced_cap, (size_t)n_len))) return rc;
        CU(cudaMemsetAsync(s->d_forced, 0, n_len * sizeof(int), st));
        if (!tiles32.empty())
            CU(cudaMemcpyAsync(s->d_tiles32, tiles32.data(), tiles32.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
        if ((rc = filter32_setup())) return rc;
    }
    const long long T32 = (long long)tiles32.size();
    CU(cudaEventRecord(s->ev[0], st));
    const double margin = 1.0 / (1 << 26);
    long long redo_total = 0;
    for (int li = 0; li < n_len; ++li) {
        const int m = lmin + li;
        const long long N = n - m + 1;
        const int e = (m + 1) / 2;
        ParamArgs pa{s->d_tn, s->d_cum, s->d_cum2, s->d_prm, s->d_mu, n, N, A, m, s->floor_};
        k_params<<<blocks(A, 256), 256, 0, st>>>(pa);
        TileArgs ta{s->d_prm, s->d_mu, s->d_tn, s->d_tiles, s->d_seeds, s->d_acc,
                    s->d_counters, s->d_log, s->d_logcnt + li, (long long)s->log_cap,
                    N, dl, (int)T, S, m, e, 0, s->d_colq, s->d_rowq, nullptr, s->hiC};
        BoundMArgs bm{s->d_tn, s->d_mu, s->d_prm, nullptr, nullptr, N, N + 1, A, m, e, mb, margin};
        if (li == 0) {
            if (T) {
                SeedArgs sa{s->d_tn, s->d_mu, s->d_tiles, s->d_seeds, dl, (int)T, S, m};
                k_seed_init<<<blocks(T * 32, WARPS_PER_CTA * 32), WARPS_PER_CTA * 32, 0, st>>>(sa);
                // nearest neighbours of the first length (seeds untouched) -> bound candidates
                k_fill_acc<<<blocks(A, 256), 256, 0, st>>>(s->d_acc, A);
                k_tile<true><<<blocks(T, WARPS_PER_CTA), WARPS_PER_CTA * 32, smem, st>>>(ta);
            }
            k_acc_idx<<<blocks(N, 256), 256, 0, st>>>(s->d_acc, s->d_previdx, N);
            bm.nn1 = s->d_previdx;
        } else {
            bm.prevm = s->d_ipm + (long long)(li - 1) * A * mb;
        }
        k_bound_m<<<blocks(N * 32, 256), 256, 0, st>>>(bm);
        if (fp32) {
            // forced offsets (weak bounds) pass every cell of the walk: their slots overflow and
            // k_recompute_m takes them exactly
            if ((rc = launch_filter32(s, st, s->d_prm, s->d_mu, N, m, e, dl, S, li + 1 < n_len, T32,
                                      s->d_forced + li, s->d_acc, runs, s->d_logcnt + li, run_cap,
                                      s->d_slots, s->d_slotcnt))) return rc;
        } else {
            // no full-fold fallback here (it folds the 1-best only): forced offsets are recomputed
            k_qprep<<<blocks(A, 256), 256, 0, st>>>(s->d_prm, s->d_colq, s->d_rowq, N, A, s->sscale, nullptr);
            if (T) {
                ta.update_seeds = li + 1 < n_len;
                k_tile<false><<<blocks(T, WARPS_PER_CTA), WARPS_PER_CTA * 32, smem, st>>>(ta);
                k_log_slots<<<296, 128, 0, st>>>(s->d_log, s->d_logcnt + li, (long long)s->log_cap, s->d_prm, e,
                                                 s->d_slots, s->d_slotcnt, s->d_counters);
            }
        }
        CU(cudaMemsetAsync(s->d_ro_cnt, 0, 8, st));
        int* out = s->d_ipm + (long long)li * A * mb;
        k_select_m<<<blocks(N, 256), 256, 0, st>>>(s->d_slots, s->d_slotcnt, N, mb, out, s->d_redo, s->d_ro_cnt,
                                                  s->d_prm, s->sscale);
        k_recompute_m<<<148, 256, 0, st>>>(s->d_tn, s->d_mu, s->d_prm, s->d_redo, s->d_ro_cnt, N, m, e, mb, out);
        unsigned long long nred = 0;
        CU(cudaMemcpyAsync(&nred, s->d_ro_cnt, 8, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        redo_total += (long long)nred;
        CU(cudaGetLastError());
    }
    CU(cudaEventRecord(s->ev[1], st));
    CU(cudaEventSynchronize(s->ev[1]));
    float ms = 0; CU(cudaEventElapsedTime(&ms, s->ev[0], s->ev[1]));
    std::vector<unsigned long long> lc(n_len);
    CU(cudaMemcpy(lc.data(), s->d_logcnt, n_len * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    for (auto c : lc)
        if ((long long)c > (fp32 ? run_cap : (long long)s->log_cap))
            return fail(VLMP_E_CUDA, "m-best candidate log overflow (bounds too weak for this series)");
    // finalize: canonical sorted distances of the m best; MP/IP (first neighbour) for VALMP
    if ((rc = ensure(s->d_mpm, s->mpm_cap, (size_t)n_len * A * mb))) return rc;
    dim3 grid(blocks(N0, 128), n_len);
    k_finalize_m<<<grid, 128, 0, st>>>(s->d_tn, s->d_cum, s->d_cum2, s->d_ipm, s->d_mpm, n, A, lmin, mb, s->floor_);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(st));
    s->lmin = lmin; s->lmax = lmax; s->n_len = n_len; s->mbest = mb;
    s->mb_lmin = lmin; s->mb_n_len = n_len; s->mb_A = A; s->mb_n = n;
    s->have_profile = false; s->have_final = false; s->have_finals = false;
    memset(s->stats, 0, sizeof(s->stats));
    s->stats[0] = ms; s->stats[13] = (double)redo_total;
    return 0;
}
}  // namespace vlmp_impl

extern "C" {

int vlmp_get_profile_m(vlmp_session* s, int32_t length, double* dist, int64_t* nbr) {
    if (!s || s->mbest < 1 || !s->d_mpm || s->mb_A != s->A || s->mb_n != s->n)
        return fail(VLMP_E_STATE, "no m-best run for the current series");
    if (length < s->mb_lmin || length >= s->mb_lmin + s->mb_n_len)
        return fail(VLMP_E_INVALID_PARAMETERS, "length outside the run");
    std::lock_guard<std::mutex> g(s->lock);
    CU(cudaSetDevice(s->device));
    const int mb = s->mbest;
    const long long N = s->n - length + 1;
    const long long off = (long long)(length - s->mb_lmin) * s->A * mb;
    std::vector<int> tmp(N * mb);
    CU(cudaMemcpyAsync(dist, s->d_mpm + off, N * mb * 8, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaMemcpyAsync(tmp.data(), s->d_ipm + off, N * mb * 4, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    for (long long q = 0; q < N * mb; ++q) nbr[q] = tmp[q];
    return 0;
}

int vlmp_discords_m(vlmp_session* s, int32_t k, double* out_dist, int64_t* out_off) {
    if (!s || s->mbest < 1 || !s->d_mpm || s->mb_A != s->A || s->mb_n != s->n)
        return fail(VLMP_E_STATE, "no m-best run for the current series");
    if (k < 1 || k > 32) return fail(VLMP_E_INVALID_PARAMETERS, "k must be in [1, 32]");
    const int mb = s->mbest;
    if (k * mb > 32 * MB_MAX) return fail(VLMP_E_INVALID_PARAMETERS, "k*m too large");
    std::lock_guard<std::mutex> g(s->lock);
    CU(cudaSetDevice(s->device));
    const long long cnt = (long long)s->mb_n_len * k * mb;
    int rc;
    if ((rc = ensure(s->d_ro_i64, s->ro_i64_cap, (size_t)cnt))) return rc;
    if ((rc = ensure(s->d_ro_f64, s->ro_f64_cap, (size_t)cnt))) return rc;
    const int wpb = 4;
    const size_t sm = (size_t)wpb * 32 * MB_MAX * 16;
    k_discords_m<<<blocks((long long)s->mb_n_len * 32, wpb * 32), wpb * 32, sm, s->stream>>>(
        s->d_mpm, s->d_ro_f64, s->d_ro_i64, s->n, s->A, s->mb_lmin, s->mb_n_len, k, mb);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(out_dist, s->d_ro_f64, cnt * 8, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaMemcpyAsync(out_off, s->d_ro_i64, cnt * 8, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    return 0;
}

}  // extern "C"
