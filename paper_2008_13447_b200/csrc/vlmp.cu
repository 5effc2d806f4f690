// vlmp.cu -- B200 (sm_100a) variable-length z-normalised matrix profile.
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

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/vlmp.h"

namespace {

#ifndef VLMP_D
#define VLMP_D 8
#endif
constexpr int D = VLMP_D;         // diagonals per lane (even, <= 16)
constexpr int BAND = 32 * D;      // diagonals per warp tile
constexpr int ceil_log2(int v) { int b = 0; while ((1 << b) < v) ++b; return b; }
constexpr int PBITS = ceil_log2(BAND);   // packed local index bits (full-fold keys)
constexpr int MG = 1 << ceil_log2(D);    // lanes per log record in k_log_merge
static_assert(D % 2 == 0 && D <= 16, "D: even, at most 16");
constexpr unsigned long long PMASK = (1ull << PBITS) - 1;
#ifndef VLMP_WARPS_PER_CTA
#define VLMP_WARPS_PER_CTA 1
#endif
#ifndef VLMP_FILTER_WARPS_PER_SM
#define VLMP_FILTER_WARPS_PER_SM 20   // 96 registers
#endif
constexpr int WARPS_PER_CTA = VLMP_WARPS_PER_CTA;
constexpr int FILTER_MIN_BLOCKS = VLMP_FILTER_WARPS_PER_SM / WARPS_PER_CTA;
constexpr int FULL_MIN_BLOCKS = 16 / WARPS_PER_CTA;               // 128 registers
constexpr unsigned FULLMASK = 0xffffffffu;
constexpr unsigned long long KEY_NONE = 0x7FF0000000000000ull;   // bits of +inf
constexpr long long IDX_NONE = 0x7FFFFFFFFFFFFFFFll;

thread_local std::string g_err;

int fail(int code, const std::string& msg) { g_err = msg; return code; }

#define CU(call)                                                                   \
    do {                                                                           \
        cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess)                                                     \
            return fail(VLMP_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)


// ---------------------------------------------------------------------------------
// exact window statistics (series.py:91-100): no contraction, numpy op order
__device__ inline void win_stats(const double* __restrict__ cum, const double* __restrict__ cum2,
                                 long long o, int m, double& mu, double& sd) {
    double s = __dsub_rn(cum[o + m], cum[o]);
    double ss = __dsub_rn(cum2[o + m], cum2[o]);
    double L = (double)m;
    double u = __ddiv_rn(s, L);
    double var = __dsub_rn(__ddiv_rn(ss, L), __dmul_rn(u, u));
    if (!(var >= 0.0)) var = 0.0;
    mu = u;
    sd = __dsqrt_rn(var);
}

// series.py:81-89 (stats: sigma = sqrt(var) if var > 0 else 0) -- used by pair_distance
__device__ inline void win_stats_pd(const double* __restrict__ cum, const double* __restrict__ cum2,
                                    long long o, int m, double& mu, double& sd) {
    double s = __dsub_rn(cum[o + m], cum[o]);
    double ss = __dsub_rn(cum2[o + m], cum2[o]);
    double L = (double)m;
    double u = __ddiv_rn(s, L);
    double var = __dsub_rn(__ddiv_rn(ss, L), __dmul_rn(u, u));
    mu = u;
    sd = var > 0.0 ? __dsqrt_rn(var) : 0.0;
}

// canonical pair distance (series.py:169-194): dot in (min,max) order, sequential sum
__device__ double pair_distance(const double* __restrict__ t, const double* __restrict__ cum,
                                const double* __restrict__ cum2, long long i, long long j, int m,
                                double floor_) {
    long long a = i <= j ? i : j, b = i <= j ? j : i;
    double mua, sda, mub, sdb;
    win_stats_pd(cum, cum2, a, m, mua, sda);
    win_stats_pd(cum, cum2, b, m, mub, sdb);
    if (sda < floor_ || sdb < floor_) return INFINITY;
    double qt = 0.0;
    for (int k = 0; k < m; ++k) qt = __dadd_rn(qt, __dmul_rn(t[a + k], t[b + k]));
    double L = (double)m;
    double num = __dsub_rn(qt, __dmul_rn(__dmul_rn(L, mua), mub));
    double den = __dmul_rn(__dmul_rn(L, sda), sdb);
    double rad = __dmul_rn(__dmul_rn(2.0, L), __dsub_rn(1.0, __ddiv_rn(num, den)));
    return rad > 0.0 ? __dsqrt_rn(rad) : 0.0;
}

// ---------------------------------------------------------------------------------
// Per-length window parameters, natural layout, 32-byte AoS so one warp-contiguous
// run of offsets is a coalesced 1 KB read (and two 16-byte cp.async per entry).
struct __align__(32) Prm {
    double df;    // (t[o+m-1] - t[o-1]) / 2                       (0 at o = 0)
    double dg;    // (t[o+m-1] - mu_o) + (t[o-1] - mu_{o-1})        (0 at o = 0)
    double inv;   // 1 / (sigma_o sqrt(m)); NaN = invalid window (constant / past the end)
    float U;      // bound on the offset's best key, high word as float (filter kernel)
    float pad;
};

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

// ---------------------------------------------------------------------------------
// O(1)-per-offset bound from the previous length's winners (1-best mode). Candidates:
// o's own winner c1 and its neighbours' winners shifted along their diagonals,
// (o, nn(o-1)+1) and (o, nn(o+1)-1). Their covariance at length m-1 comes from the stored
// key, cov = (1 - r) / (inv_o inv_c) (r kept to 2^-44), plus / minus one step of the
// diagonal recurrence; the Welford co-moment step carries it to length m. Any valid cell's
// key bounds the minimum; the reconstruction error (~1e-13) is far below the margin.
struct Bound2Args {
    const double* tn; const Prm* prm; const Prm* pprev; const double* mu_prev; const double* mu;
    const ulonglong2* acc_prev; Prm* out;
    long long N, Nprev; int m, e; double margin;
    unsigned long long* fix_cnt;   // offsets re-bounded by a direct dot product
};

__global__ void k_bound2(Bound2Args a) {
    const long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (o >= a.N) return;
    const double io = a.prm[o].inv;
    if (!(io == io)) { a.out[o].U = -INFINITY; return; }
    const int m = a.m;
    const double wgt = (double)(m - 1) / (double)m;
    const double xo = a.tn[o + m - 1] - a.mu_prev[o];
    double best = INFINITY;
    auto eval = [&](long long c, double covp) {
        const long long dd = c > o ? c - o : o - c;
        if (c < 0 || c >= a.N || dd < a.e) return;
        const double ic = a.prm[c].inv;
        if (!(ic == ic)) return;
        const double covm = fma(wgt * xo, a.tn[c + m - 1] - a.mu_prev[c], covp);
        best = fmin(best, fma(-(covm * io), ic, 1.0));
    };
    auto cov_of = [&](long long i, const ulonglong2& v) {   // winner's covariance at m-1
        const double r = __longlong_as_double((long long)v.x);
        return (1.0 - r) / (a.pprev[i].inv * a.pprev[(long long)v.y].inv);
    };
    if (o < a.Nprev) {
        const ulonglong2 v = a.acc_prev[o];
        if (v.x != KEY_NONE) eval((long long)v.y, cov_of(o, v));
    }
    if (o >= 1 && o - 1 < a.Nprev) {
        const ulonglong2 v = a.acc_prev[o - 1];
        if (v.x != KEY_NONE) {   // (o, c0+1) follows (o-1, c0) on its diagonal
            const long long c = (long long)v.y + 1;
            const Prm po = a.pprev[o], pc = a.pprev[c];
            eval(c, cov_of(o - 1, v) + po.df * pc.dg + pc.df * po.dg);
        }
    }
    if (o + 1 < a.Nprev) {
        const ulonglong2 v = a.acc_prev[o + 1];
        if (v.x != KEY_NONE && v.y >= 1) {   // (o, c0-1) precedes (o+1, c0) on its diagonal
            const long long c0 = (long long)v.y;
            const Prm po = a.pprev[o + 1], pc = a.pprev[c0];
            eval(c0 - 1, cov_of(o + 1, v) - po.df * pc.dg - pc.df * po.dg);
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
                atomicAdd(a.fix_cnt, 1ull);
            }
        }
    }
    float out = INFINITY;   // no bound: every cell of this offset is a candidate
    if (best < INFINITY) out = __int_as_float(__double2hiint(fmax(best, 0.0) + a.margin));
    a.out[o].U = out;
}


// ---------------------------------------------------------------------------------
// Filter thresholds in the covariance domain. A cell (i, j) must reach the exact tests when
// its key r = 1 - cov inv_i inv_j satisfies hi(r) <= max(U_i, U_j), i.e. r <= R(U) with
// R(U) the largest double of that high word. With q(U) = 1 - R(U) - 2^-20 and s = 1/inv:
//   r <= R(U)  =>  cov >= q(U) s_i s_j            (2^-20 >> the FP64 rounding of r)
// so the tile kernel tests  hi(cov) >= hi(t),  t = a_j * b_i  (FP32, rounded down), with
// b = s 2^-k (per-session power-of-two scale) and a_j = q(max(U_j, Uwin_i)) b_j -- no
// per-cell FP64 work beyond the recurrence. q < 2^-20 (a bound at corr ~ 0) is clamped to
// 0, which still passes every cell of positive covariance; only offsets whose OWN bound is
// that weak may need non-positive-covariance cells: they are "forced" (1-best: the length
// falls back to the exact full-fold kernel; m-best: the offset is recomputed exactly).
constexpr double QSLACK = 1.0 / (1 << 20);

__device__ inline double qfac(float u) {
    const double R = __hiloint2double(__float_as_int(u), (int)0xFFFFFFFF);
    const double q = 1.0 - R - QSLACK;
    return q >= QSLACK ? q : 0.0;      // also 0 for u = +inf / NaN
}

__device__ inline float qscale(double inv, double sscale) {
    return __double2float_rd((1.0 / inv) * sscale);   // NaN for an invalid window
}

// the offset's own bound is too weak for the covariance-domain filter (see above)
__device__ inline bool q_forced(const Prm& p, double sscale) {
    if (!(p.inv == p.inv)) return false;
    const float b = qscale(p.inv, sscale);
    return qfac(p.U) == 0.0 || !(b >= 0x1p-40f && b <= 0x1p40f);
}

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
struct Cand { int o; int idx; unsigned long long key; };   // candidate (offset, neighbour, key)

// A filter-kernel log record: a lane whose cells passed the bound at row i; its 8 cells are
// (i, j0 + s) and cov[s] is their covariance, so the merge kernel can recompute the exact
// keys with the kernel's own FMA sequence (bit-identical) and apply the exact tests.
struct __align__(16) RowRec { int i; int j0; int pad0, pad1; double cov[D]; };

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
};

__device__ inline bool key_less(unsigned long long k1, long long i1, unsigned long long k2, long long i2) {
    return k1 < k2 || (k1 == k2 && i1 < i2);
}

// exact lexicographic (key, idx) min into a 16-byte accumulator (128-bit CAS)
__device__ void acc_merge(ulonglong2* slot, unsigned long long key, long long idx) {
    unsigned __int128* p = reinterpret_cast<unsigned __int128*>(slot);
    const volatile unsigned long long* vp = reinterpret_cast<volatile unsigned long long*>(slot);
    unsigned __int128 cur = ((unsigned __int128)vp[1] << 64) | vp[0];
    const unsigned __int128 want = ((unsigned __int128)(unsigned long long)idx << 64) | key;
    while (key_less(key, idx, (unsigned long long)cur, (long long)(cur >> 64))) {
        unsigned __int128 prev = atomicCAS(p, cur, want);
        if (prev == cur) return;
        cur = prev;
    }
}

__device__ inline unsigned long long clamp_key(double r) {
    return r < 0.0 ? 0ull : (unsigned long long)__double_as_longlong(r);
}

__device__ inline double pack_low(double v, unsigned idx) {
    int lo = __double2loint(v), hi = __double2hiint(v);
    lo = (lo & ~(int)PMASK) | (int)idx;
    return __hiloint2double(hi, lo);
}

__device__ inline void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ inline void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }


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
    const long long d0 = a.dlo + (long long)tl.x * BAND;
    const long long i0 = (long long)tl.y * a.S;
    const long long rows_valid = a.N - d0 - i0;
    if (rows_valid <= 0 || d0 + BAND - 1 < a.e) return;   // empty, or entirely trivial
    if (FULL || (a.forced && *a.forced)) {
        if (d0 < a.e) tile_body<true, true>(a, ws[wl], wid, lane, d0, i0, rows_valid);
        else tile_body<true, false>(a, ws[wl], wid, lane, d0, i0, rows_valid);
    } else {
        if (d0 < a.e) tile_body<false, true>(a, ws[wl], wid, lane, d0, i0, rows_valid);
        else tile_body<false, false>(a, ws[wl], wid, lane, d0, i0, rows_valid);
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

__global__ void k_fill_acc(ulonglong2* acc, long long n) {
    long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (o < n) acc[o] = make_ulonglong2(KEY_NONE, (unsigned long long)IDX_NONE);
}

// previous-length winner indices (for the bound) straight from the accumulators
__global__ void k_acc_idx(const ulonglong2* acc, long long* idx, long long n) {
    long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (o < n) { ulonglong2 v = acc[o]; idx[o] = v.x == KEY_NONE ? -1 : (long long)v.y; }
}

// ---------------------------------------------------------------------------------
struct FinArgs {
    const double* tn; const double* cum; const double* cum2;
    const ulonglong2* acc;      // [n_len][A]
    double* mp; int* ip;        // [n_len][A]
    long long n, A; int lmin, n_len; double floor_;
    int li_lo, li_hi;           // lengths finalized here; others get (+inf, -1) (length shards)
};


// Same values, one thread per offset walking the lengths upward: pair_distance's dot
// product is a sequential left-to-right sum over k < m, so when an offset keeps the same
// canonical pair (a, b) from length m-1 to m its sum at m is the sum at m-1 plus one term
// -- bit-identical to recomputing it. Only neighbour changes pay the O(m) sum.
__global__ void k_finalize_walk(FinArgs a) {
    const long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (o >= a.n - a.lmin + 1) return;
    long long pa = -1, pb = -1; int pm = -1;
    double qt = 0.0;
    for (int li = 0; li < a.n_len; ++li) {
        const int m = a.lmin + li;
        if (o > a.n - m) break;
        if (li < a.li_lo || li > a.li_hi) {   // another shard's length: neutral for MIN / MAX
            a.mp[(long long)li * a.A + o] = INFINITY;
            a.ip[(long long)li * a.A + o] = -1;
            continue;
        }
        const ulonglong2 v = a.acc[(long long)li * a.A + o];
        double d = INFINITY; int j = -1;
        if (v.x != KEY_NONE) {
            j = (int)v.y;
            const long long lo = o <= j ? o : j, hi = o <= j ? j : o;
            double mua, sda, mub, sdb;
            win_stats_pd(a.cum, a.cum2, lo, m, mua, sda);
            win_stats_pd(a.cum, a.cum2, hi, m, mub, sdb);
            if (lo == pa && hi == pb && m == pm + 1) {
                qt = __dadd_rn(qt, __dmul_rn(a.tn[lo + m - 1], a.tn[hi + m - 1]));
            } else {
                qt = 0.0;
#pragma unroll 8
                for (int k = 0; k < m; ++k) qt = __dadd_rn(qt, __dmul_rn(a.tn[lo + k], a.tn[hi + k]));
            }
            pa = lo; pb = hi; pm = m;
            if (sda >= a.floor_ && sdb >= a.floor_) {
                const double L = (double)m;
                const double num = __dsub_rn(qt, __dmul_rn(__dmul_rn(L, mua), mub));
                const double den = __dmul_rn(__dmul_rn(L, sda), sdb);
                const double rad = __dmul_rn(__dmul_rn(2.0, L), __dsub_rn(1.0, __ddiv_rn(num, den)));
                d = rad > 0.0 ? __dsqrt_rn(rad) : 0.0;
            }
        }
        a.mp[(long long)li * a.A + o] = d;
        a.ip[(long long)li * a.A + o] = j;
    }
}

struct ValmpArgs {
    const double* mp; const int* ip;
    double* dist; double* norm; long long* len; long long* idx; unsigned char* pop;
    long long n, A; int lmin, n_len;
};

// valmod.py:57-73: lnorm = mp * sqrt(1/length); strict improvement, ascending lengths
__global__ void k_valmp(ValmpArgs a) {
    const long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long n0 = a.n - a.lmin + 1;
    if (o >= n0) return;
    double bd = INFINITY, bn = INFINITY; long long bl = 0, bi = -1; bool pop = false;
    for (int li = 0; li < a.n_len; ++li) {
        const int m = a.lmin + li;
        if (o > a.n - m) break;
        const double mpv = a.mp[(long long)li * a.A + o];
        const double ln = __dmul_rn(mpv, __dsqrt_rn(__ddiv_rn(1.0, (double)m)));
        if (ln < INFINITY && (!pop || bn > ln)) {
            bd = mpv; bn = ln; bl = m; bi = a.ip[(long long)li * a.A + o]; pop = true;
        }
    }
    a.dist[o] = bd; a.norm[o] = bn; a.len[o] = bl; a.idx[o] = bi; a.pop[o] = pop ? 1 : 0;
}

// per length: the K smallest (mp, offset) rows (K <= 64), block-wide selection
struct SmallArgs {
    const double* mp; const int* ip; long long* off; long long* nbr; double* d;
    long long n, A; int lmin, K;
};

__device__ inline bool row_less(double d1, long long o1, double d2, long long o2) {
    return d1 < d2 || (d1 == d2 && o1 < o2);
}

__global__ void k_smallest(SmallArgs a) {
    constexpr int T = 256, KMAX = 64;
    const int li = blockIdx.x;
    const int m = a.lmin + li;
    const long long N = a.n - m + 1;
    const double* mp = a.mp + (long long)li * a.A;
    // each thread: local sorted list of K
    double ld[KMAX]; long long lo[KMAX];
    const int K = a.K;
    for (int q = 0; q < K; ++q) { ld[q] = INFINITY; lo[q] = -1; }
    for (long long o = threadIdx.x; o < N; o += T) {
        const double v = mp[o];
        if (!(v < INFINITY)) continue;
        if (!row_less(v, o, ld[K - 1], lo[K - 1] < 0 ? (1ll << 62) : lo[K - 1])) continue;
        int q = K - 1;
        while (q > 0 && row_less(v, o, ld[q - 1], lo[q - 1] < 0 ? (1ll << 62) : lo[q - 1])) {
            ld[q] = ld[q - 1]; lo[q] = lo[q - 1]; --q;
        }
        ld[q] = v; lo[q] = o;
    }
    __shared__ double sd[T];
    __shared__ long long so[T];
    // merge: repeated K rounds of block argmin over heads (K small)
    __shared__ int head[T];
    head[threadIdx.x] = 0;
    __syncthreads();
    for (int q = 0; q < K; ++q) {
        const int h = head[threadIdx.x];
        double v = h < K ? ld[h] : INFINITY;
        long long ov = h < K ? lo[h] : -1;
        if (ov < 0) v = INFINITY;
        sd[threadIdx.x] = v; so[threadIdx.x] = ov < 0 ? (1ll << 62) : ov;
        __syncthreads();
        for (int w = T / 2; w >= 1; w >>= 1) {
            if (threadIdx.x < w) {
                if (row_less(sd[threadIdx.x + w], so[threadIdx.x + w], sd[threadIdx.x], so[threadIdx.x])) {
                    sd[threadIdx.x] = sd[threadIdx.x + w]; so[threadIdx.x] = so[threadIdx.x + w];
                }
            }
            __syncthreads();
        }
        const double bv = sd[0]; const long long bo = so[0];
        __syncthreads();
        if (bv < INFINITY && ov == bo) head[threadIdx.x] = h + 1;
        if (threadIdx.x == 0) {
            const long long dst = (long long)li * K + q;
            if (bv < INFINITY) { a.off[dst] = bo; a.nbr[dst] = a.ip[(long long)li * a.A + bo]; a.d[dst] = bv; }
            else { a.off[dst] = -1; a.nbr[dst] = -1; a.d[dst] = INFINITY; }
        }
        __syncthreads();
    }
}

// per length: top-k 1st discords, ascending-offset greedy replay (discords.py:68-93,
// :48-50, oracle.py:137-145) with the exact prefilter d > dist[k-1]; one warp per length
struct DiscArgs {
    const double* mp; double* out_d; long long* out_o;
    long long n, A; int lmin, n_len, k;
};

__global__ void k_discords(DiscArgs a) {
    // one warp per length replays the reference's ascending-offset greedy insertion; lane r
    // holds list entry r (sorted descending), 8 chunks of the profile are loaded ahead
    const int lane = threadIdx.x & 31;
    const int li = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (li >= a.n_len) return;
    const int m = a.lmin + li;
    const long long N = a.n - m + 1;
    const long long e = (m + 1) / 2;
    const double* mp = a.mp + (long long)li * a.A;
    constexpr int AHEAD = 8;
    const int k = a.k;                       // <= 32
    double cd = -INFINITY; long long co = -1;
    for (long long base = 0; base < N; base += 32 * AHEAD) {
        double dv8[AHEAD];
#pragma unroll
        for (int u = 0; u < AHEAD; ++u) {
            const long long o = base + 32 * u + lane;
            dv8[u] = o < N ? mp[o] : INFINITY;
        }
#pragma unroll
        for (int u = 0; u < AHEAD; ++u) {
            const double thr = __shfl_sync(FULLMASK, cd, k - 1);
            const double d = dv8[u];
            unsigned bal = __ballot_sync(FULLMASK, (d < INFINITY) && (d > thr));
            while (bal) {
                const int src = __ffs(bal) - 1;
                bal &= bal - 1;
                const double dv = __shfl_sync(FULLMASK, d, src);
                const long long ov = base + 32 * u + src;
                const bool mine = lane < k;
                if (__any_sync(FULLMASK, mine && co >= 0 && llabs(ov - co) < e)) continue;   // trivial match
                // before the first strictly smaller entry
                const int at = __popc(__ballot_sync(FULLMASK, mine && !(dv > cd)));
                if (at >= k) continue;
                const double ud = __shfl_up_sync(FULLMASK, cd, 1);
                const long long uo = __shfl_up_sync(FULLMASK, co, 1);
                if (mine && lane > at) { cd = ud; co = uo; }
                if (lane == at) { cd = dv; co = ov; }
            }
        }
    }
    if (lane < k) { a.out_d[(long long)li * k + lane] = cd; a.out_o[(long long)li * k + lane] = co; }
}

// Motif-set range queries (motifsets.py:158-165 row_profile path, profile.py:235-260):
// offsets j with dist(owner, j) < radius at the query's length, the owner's full row with
// the reference's formula and evaluation order; trivial zone and constant windows excluded.
struct RangeArgs {
    const double* tn; const double* cum; const double* cum2;
    const long long* owner; const int* len; const double* radius;
    long long* members; unsigned long long* counts; long long cap;
    long long n; double floor_;
};

__global__ void k_range_query(RangeArgs a) {
    const int q = blockIdx.y;
    const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int m = a.len[q];
    const long long N = a.n - m + 1;
    if (j >= N) return;
    const long long i = a.owner[q];
    const long long e = (m + 1) / 2;
    const long long lo = i - e + 1 > 0 ? i - e + 1 : 0, hi = i + e < N ? i + e : N;
    if (j >= lo && j < hi) return;
    double mui, sdi, muj, sdj;
    win_stats_pd(a.cum, a.cum2, i, m, mui, sdi);
    win_stats_pd(a.cum, a.cum2, j, m, muj, sdj);
    if (!(sdj >= a.floor_)) return;
    double qt = 0.0;
    for (int k = 0; k < m; ++k) qt = fma(a.tn[i + k], a.tn[j + k], qt);
    const double L = (double)m;
    const double qraw = __ddiv_rn(__dsub_rn(qt, __dmul_rn(__dmul_rn(L, mui), muj)),
                                  __dmul_rn(__dmul_rn(L, sdi), sdj));
    double rad = __dmul_rn(__dmul_rn(2.0, L), __dsub_rn(1.0, qraw));
    if (rad < 0.0) rad = 0.0;                    // np.maximum(rad, 0): NaN stays NaN
    const double d = __dsqrt_rn(rad);
    if (d < a.radius[q]) {
        const unsigned long long at = atomicAdd(a.counts + q, 1ull);
        if ((long long)at < a.cap) a.members[(long long)q * a.cap + (long long)at] = j;
    }
}

// VALMP improvement events with norm <= tau (motifsets.py:105-117 stream)
struct EvArgs {
    const double* mp; const int* ip; double tau;
    long long* ev_off; long long* ev_nbr; long long* ev_len; double* ev_d; double* ev_n;
    unsigned long long* count; long long cap;
    long long n, A; int lmin, n_len;
};

__global__ void k_events(EvArgs a) {
    const long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long n0 = a.n - a.lmin + 1;
    if (o >= n0) return;
    double bn = INFINITY; bool pop = false;
    for (int li = 0; li < a.n_len; ++li) {
        const int m = a.lmin + li;
        if (o > a.n - m) break;
        const double mpv = a.mp[(long long)li * a.A + o];
        const double ln = __dmul_rn(mpv, __dsqrt_rn(__ddiv_rn(1.0, (double)m)));
        if (ln < INFINITY && (!pop || bn > ln)) {
            bn = ln; pop = true;
            if (ln <= a.tau) {
                const unsigned long long q = atomicAdd(a.count, 1ull);
                if ((long long)q < a.cap) {
                    a.ev_off[q] = o; a.ev_nbr[q] = a.ip[(long long)li * a.A + o]; a.ev_len[q] = m;
                    a.ev_d[q] = mpv; a.ev_n[q] = ln;
                }
            }
        }
    }
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

// FP64 FMA peak: 8 independent chains per thread
__global__ void k_dfma_peak(double* out, int iters, double x) {
    double a0 = x, a1 = x + 1, a2 = x + 2, a3 = x + 3, a4 = x + 4, a5 = x + 5, a6 = x + 6, a7 = x + 7;
    const double b = 0.999999, c = 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 12345.678) out[0] = s;
}


// =================================================================================
// m-th discords (m > 1): per (length, offset) the m best neighbours, exact.
// The filter tile kernel runs with U = a bound on each offset's m-th best key; passing
// cells go to per-offset slots; k_select_m keeps the m smallest (key, index); offsets
// whose slots overflow are recomputed exactly from direct dot products.
constexpr int MB_MAX = 8;                 // largest supported m
constexpr int SLOT_CAP = 24;              // candidate slots per offset per length

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

}  // namespace

// =================================================================================
struct vlmp_session {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;       // near-diagonal (masked) bands, overlapped with the main launch
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    cudaEvent_t ev[8] = {};
    std::mutex lock;
    // series
    long long n = 0, A = 0;
    double floor_ = 0.0;
    double* d_tn = nullptr; double* d_cum = nullptr; double* d_cum2 = nullptr;
    // per-length scratch
    Prm* d_prm = nullptr; double* d_mu = nullptr;
    Prm* d_prm2 = nullptr; double* d_mu2 = nullptr;     // previous length's (1-best bound)
    long long* d_previdx = nullptr;
    float2* d_colq = nullptr; float2* d_rowq = nullptr;   // filter factors (k_qprep)
    int* d_forced = nullptr; size_t forced_cap = 0;      // per-length: full-fold fallback
    unsigned long long* d_fixcnt = nullptr; size_t fixcnt_cap = 0;   // per-length re-bounded offsets
    double sscale = 1.0; int hiC = 896 << 20;            // filter: 2^-k scale, hi-word bias
    // tiles / seeds
    int2* d_tiles = nullptr; size_t tiles_cap = 0;
    double* d_seeds = nullptr; size_t seeds_cap = 0;
    // accumulators [n_len][A]
    ulonglong2* d_acc = nullptr; size_t acc_cap = 0;
    double* d_mp = nullptr; int* d_ip = nullptr; size_t mp_cap = 0;
    unsigned long long* d_counters = nullptr;
    RowRec* d_log = nullptr; size_t log_cap = 0;        // filter-kernel log of flagged lanes
    unsigned long long* d_logcnt = nullptr; size_t logcnt_cap = 0;   // per-length fill counters
    // valmp
    double* d_vdist = nullptr; double* d_vnorm = nullptr; long long* d_vlen = nullptr;
    long long* d_vidx = nullptr; unsigned char* d_vpop = nullptr; size_t v_cap = 0;
    // read-off scratch (persistent: per-call cudaMallocAsync re-maps pool memory every sync)
    long long* d_ro_i64 = nullptr; size_t ro_i64_cap = 0;
    double* d_ro_f64 = nullptr; size_t ro_f64_cap = 0;
    unsigned long long* d_ro_cnt = nullptr;
    // m-best mode (m > 1 discords)
    int mbest = 1;
    ulonglong2* d_slots = nullptr; size_t slots_cap = 0;
    int* d_slotcnt = nullptr; size_t slotcnt_cap = 0;
    int* d_ipm = nullptr; size_t ipm_cap = 0;
    double* d_mpm = nullptr; size_t mpm_cap = 0;
    long long* d_redo = nullptr; size_t redo_cap = 0;
    // run state
    int lmin = 0, lmax = 0, n_len = 0; bool have_profile = false, have_final = false, have_finals = false;
    double stats[16] = {};
    std::vector<cudaEvent_t> lev;   // 2 per length: tile-kernel start/stop
};

namespace {

template <class T>
int ensure(T*& p, size_t& cap, size_t count) {
    if (count <= cap && p) return 0;
    if (p) cudaFree(p);
    p = nullptr; cap = 0;
    cudaError_t e = cudaMalloc((void**)&p, std::max<size_t>(count, 1) * sizeof(T));
    if (e != cudaSuccess) return fail(VLMP_E_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    cap = count;
    return 0;
}

template <class T>
int ensure1(T*& p, size_t count) { size_t cap = 0; if (p) { cudaFree(p); p = nullptr; } return ensure(p, cap, count); }

inline unsigned blocks(long long n, int t) { return (unsigned)((n + t - 1) / t); }

// filter log records per length: 8 per offset (quasi-periodic series flag many near-minimum
// cells), at most a quarter of the free device memory; an overflow re-runs exactly
size_t log_capacity(long long N0) {
    size_t want = std::max<size_t>((size_t)1 << 20, (size_t)(8 * N0));
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
    // S = G*D rows per tile (whole GR-row groups); larger for longer series to bound the
    // number of tiles and the seed store (config 5: S = 16384, ~1.1M tiles, 2.2 GB of seeds)
#ifndef VLMP_SEG_G0
#define VLMP_SEG_G0 128
#endif
    long long G = VLMP_SEG_G0;
    while (G * D * 256 < n && G < 2048) G *= 2;
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

}  // namespace

extern "C" {

const char* vlmp_last_error(void) { return g_err.c_str(); }

int vlmp_create(vlmp_session** out, int device) {
    if (!out) return fail(VLMP_E_INVALID_PARAMETERS, "null out");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(VLMP_E_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return fail(VLMP_E_INVALID_PARAMETERS, "bad device id");
    CU(cudaSetDevice(device));
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return fail(VLMP_E_CUDA, "libvlmp is built for sm_100a (B200) only");
    vlmp_session* s = new vlmp_session();
    s->device = device;
    CU(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    int prio_lo = 0, prio_hi = 0;
    CU(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    CU(cudaStreamCreateWithPriority(&s->side, cudaStreamNonBlocking, prio_hi));   // dispatch first
    CU(cudaEventCreateWithFlags(&s->fork_ev, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&s->join_ev, cudaEventDisableTiming));
    for (auto& ev : s->ev) CU(cudaEventCreate(&ev));
    CU(cudaMalloc((void**)&s->d_counters, 8 * sizeof(unsigned long long)));
    *out = s;
    return 0;
}

void vlmp_destroy(vlmp_session* s) {
    if (!s) return;
    cudaSetDevice(s->device);
    cudaStreamSynchronize(s->stream);
    void* ptrs[] = {s->d_tn, s->d_cum, s->d_cum2, s->d_prm, s->d_mu, s->d_prm2, s->d_mu2,
                    s->d_previdx, s->d_colq, s->d_rowq, s->d_forced, s->d_fixcnt, s->d_tiles, s->d_seeds, s->d_acc, s->d_mp, s->d_ip, s->d_counters,
                    s->d_log, s->d_logcnt, s->d_ro_i64, s->d_ro_f64, s->d_ro_cnt,
                    s->d_slots, s->d_slotcnt, s->d_ipm, s->d_mpm, s->d_redo, s->d_vdist, s->d_vnorm, s->d_vlen, s->d_vidx, s->d_vpop};
    for (void* p : ptrs) if (p) cudaFree(p);
    for (auto& ev : s->ev) if (ev) cudaEventDestroy(ev);
    for (auto& ev : s->lev) cudaEventDestroy(ev);
    if (s->stream) cudaStreamDestroy(s->stream);
    if (s->side) cudaStreamDestroy(s->side);
    if (s->fork_ev) cudaEventDestroy(s->fork_ev);
    if (s->join_ev) cudaEventDestroy(s->join_ev);
    delete s;
}

int vlmp_set_series(vlmp_session* s, const double* t, const double* cum, const double* cum2,
                    int64_t n, double sigma_floor) {
    if (!s || !t || !cum || !cum2) return fail(VLMP_E_INVALID_PARAMETERS, "null argument");
    if (n <= 0) return fail(VLMP_E_EMPTY_SERIES, "series holds no points");
    std::lock_guard<std::mutex> g(s->lock);
    CU(cudaSetDevice(s->device));
    long long A = ((n + 1024 + 255) / 256) * 256 + 256;
    s->n = n; s->A = A; s->floor_ = sigma_floor;
    int rc;
    if ((rc = ensure1(s->d_tn, 2 * A + 4096))) return rc;
    if ((rc = ensure1(s->d_cum, n + 1))) return rc;
    if ((rc = ensure1(s->d_cum2, n + 1))) return rc;
    if ((rc = ensure1(s->d_prm, A))) return rc;
    if ((rc = ensure1(s->d_mu, A))) return rc;
    if ((rc = ensure1(s->d_prm2, A))) return rc;
    if ((rc = ensure1(s->d_mu2, A))) return rc;
    if ((rc = ensure1(s->d_previdx, A))) return rc;
    if ((rc = ensure1(s->d_colq, A))) return rc;
    if ((rc = ensure1(s->d_rowq, A))) return rc;
    {   // filter scale: b = sigma sqrt(m) 2^-k stays O(1) whatever the series' units
        double ss = 0.0;
        for (long long i = 0; i < n; ++i) ss += t[i] * t[i];
        const double rms = std::sqrt(ss / (double)n);
        int k = (rms > 0.0 && std::isfinite(rms)) ? std::ilogb(rms) + 4 : 0;
        k = std::max(-400, std::min(400, k));
        s->sscale = std::ldexp(1.0, -k);
        s->hiC = (896 + 2 * k) << 20;
    }
    CU(cudaMemsetAsync(s->d_tn, 0, (2 * A + 4096) * sizeof(double), s->stream));
    CU(cudaMemcpyAsync(s->d_tn, t, n * sizeof(double), cudaMemcpyHostToDevice, s->stream));
    CU(cudaMemcpyAsync(s->d_cum, cum, (n + 1) * sizeof(double), cudaMemcpyHostToDevice, s->stream));
    CU(cudaMemcpyAsync(s->d_cum2, cum2, (n + 1) * sizeof(double), cudaMemcpyHostToDevice, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    s->have_profile = s->have_final = s->have_finals = false;
    return 0;
}

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
static int profile_impl(vlmp_session* s, int32_t lmin, int32_t lmax, int64_t band_lo,
                        int64_t band_hi, uint32_t flags, bool* overflow_out, int li_lo = 0,
                        int li_hi = -1) {
    CU(cudaSetDevice(s->device));
    cudaStream_t st = s->stream;
    const long long n = s->n, A = s->A;
    const int n_len = lmax - lmin + 1;
    const long long nb = n_bands_for(n, lmin);
    if (band_hi < 0 || band_hi > nb) band_hi = nb;
    if (band_lo < 0) band_lo = 0;
    const int S = seg_rows(n);
    const long long N0 = n - lmin + 1, dl = dlo_for(lmin);
    // tile list using N at lmin (a superset of every later length's tiles), launched
    // longest-first (order_tiles)
    std::vector<int2> tiles;
    for (long long b = band_lo; b < band_hi; ++b) {
        long long rows = N0 - (dl + b * BAND);
        for (long long sg = 0; sg * S < rows; ++sg) tiles.push_back(make_int2((int)b, (int)sg));
    }
    order_tiles(tiles, N0, dl, S);
    const long long T = (long long)tiles.size();
    int rc;
    if ((rc = ensure(s->d_tiles, s->tiles_cap, (size_t)std::max<long long>(T, 1)))) return rc;
    if ((rc = ensure(s->d_seeds, s->seeds_cap, (size_t)std::max<long long>(T, 1) * BAND))) return rc;
    if ((rc = ensure(s->d_acc, s->acc_cap, (size_t)n_len * A))) return rc;
    const size_t log_cap = log_capacity(N0);
    if ((rc = ensure(s->d_log, s->log_cap, log_cap))) return rc;
    if ((rc = ensure(s->d_logcnt, s->logcnt_cap, (size_t)n_len))) return rc;
    if ((rc = ensure(s->d_forced, s->forced_cap, (size_t)n_len))) return rc;
    if ((rc = ensure(s->d_fixcnt, s->fixcnt_cap, (size_t)n_len))) return rc;
    CU(cudaMemsetAsync(s->d_fixcnt, 0, n_len * sizeof(unsigned long long), st));
    CU(cudaMemsetAsync(s->d_logcnt, 0, n_len * sizeof(unsigned long long), st));
    CU(cudaMemsetAsync(s->d_forced, 0, n_len * sizeof(int), st));
    if (T) CU(cudaMemcpyAsync(s->d_tiles, tiles.data(), T * sizeof(int2), cudaMemcpyHostToDevice, st));
    const size_t smem = WARPS_PER_CTA * sizeof(WarpSmem);
    CU(cudaFuncSetAttribute(k_tile<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CU(cudaFuncSetAttribute(k_tile<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_fill_acc<<<blocks((long long)n_len * A, 256), 256, 0, st>>>(s->d_acc, (long long)n_len * A);
    CU(cudaMemsetAsync(s->d_counters, 0, 8 * sizeof(unsigned long long), st));
    CU(cudaEventRecord(s->ev[0], st));

    double executed = 0, launches = 0, n_filtered = 0, n_full = 0, tile_ms = 0, klaunch = 2;
    const double margin = 1.0 / (1 << 26);
    // VLMP_LOG_CAP (records) lowers the effective log capacity: a test hook that forces the
    // overflow -> exact full-fold re-run path
    long long eff_cap = (long long)s->log_cap;
    if (const char* env = getenv("VLMP_LOG_CAP")) eff_cap = std::max(1LL, std::min(eff_cap, atoll(env)));
    if (li_lo < 0) li_lo = 0;
    if (li_hi >= n_len || (li_hi < 0 && li_lo == 0)) li_hi = n_len - 1;   // default: every length
    if (li_hi < li_lo) li_hi = -1;                                        // empty shard: no work
    std::vector<int> timed;   // lengths whose tile pass ran (event pairs)
    if (li_lo > 0 && li_lo <= li_hi && T) {
        // a later length shard: seeds at lmin (direct sums), carried to its first length
        ParamArgs pa{s->d_tn, s->d_cum, s->d_cum2, s->d_prm, s->d_mu, n, n - lmin + 1, A, lmin, s->floor_};
        k_params<<<blocks(A, 256), 256, 0, st>>>(pa);
        SeedArgs sa{s->d_tn, s->d_mu, s->d_tiles, s->d_seeds, dl, (int)T, S, lmin};
        k_seed_init<<<blocks(T * 32, WARPS_PER_CTA * 32), WARPS_PER_CTA * 32, 0, st>>>(sa);
        k_seed_forward<<<blocks(T * 32, 128), 128, 0, st>>>(sa, s->d_cum, lmin + li_lo);
        klaunch += 3;
    }
    for (int li = (li_lo <= li_hi ? li_lo : 0); li <= li_hi; ++li) {
        const int m = lmin + li;
        const long long N = n - m + 1;
        const int e = (m + 1) / 2;
        // window parameters ping-pong between two buffers: the bound reads length m-1's
        Prm* prm = (li & 1) ? s->d_prm2 : s->d_prm;
        double* mu = (li & 1) ? s->d_mu2 : s->d_mu;
        const Prm* prm_prev = (li & 1) ? s->d_prm : s->d_prm2;
        const double* mu_prev = (li & 1) ? s->d_mu : s->d_mu2;
        ParamArgs pa{s->d_tn, s->d_cum, s->d_cum2, prm, mu, n, N, A, m, s->floor_};
        k_params<<<blocks(A, 256), 256, 0, st>>>(pa);
        ++klaunch;
        const bool full = (li == li_lo) || (flags & VLMP_F_FULL_EVERY_LENGTH);
        if (li == 0 && T) {
            SeedArgs sa{s->d_tn, mu, s->d_tiles, s->d_seeds, dl, (int)T, S, m};
            k_seed_init<<<blocks(T * 32, WARPS_PER_CTA * 32), WARPS_PER_CTA * 32, 0, st>>>(sa);
            ++klaunch;
        }
        if (!full) {
            Bound2Args ba{s->d_tn, prm, prm_prev, mu_prev, mu, s->d_acc + (long long)(li - 1) * A, prm,
                          N, N + 1, m, e, margin, s->d_fixcnt + li};
            k_bound2<<<blocks(N, 256), 256, 0, st>>>(ba);
            k_qprep<<<blocks(A, 256), 256, 0, st>>>(prm, s->d_colq, s->d_rowq, N, A, s->sscale,
                                                    s->d_forced + li);
            klaunch += 2;
        }
        while (s->lev.size() < (size_t)2 * (li + 1)) {
            cudaEvent_t ev; CU(cudaEventCreate(&ev)); s->lev.push_back(ev);
        }
        timed.push_back(li);
        CU(cudaEventRecord(s->lev[2 * li], st));
        if (T) {
            TileArgs ta{prm, mu, s->d_tn, s->d_tiles, s->d_seeds, s->d_acc + (long long)li * A,
                        s->d_counters, s->d_log, s->d_logcnt + li, eff_cap,
                        N, dl, (int)T, S, m, e, li + 1 <= li_hi,
                        s->d_colq, s->d_rowq, s->d_forced + li, s->hiC};
            if (full) k_tile<true><<<blocks(T, WARPS_PER_CTA), WARPS_PER_CTA * 32, smem, st>>>(ta);
            else {
                k_tile<false><<<blocks(T, WARPS_PER_CTA), WARPS_PER_CTA * 32, smem, st>>>(ta);
                k_log_merge<<<148 * 8, 256, 0, st>>>(s->d_log, s->d_logcnt + li, eff_cap,
                                                     prm, e, s->d_acc + (long long)li * A, s->d_counters);
                klaunch += 1;
            }
            launches += 1; klaunch += 1;
        }
        CU(cudaEventRecord(s->lev[2 * li + 1], st));
        CU(cudaGetLastError());
        for (long long b = band_lo; b < band_hi; ++b) {
            long long d0 = dl + b * BAND;
            long long rows = N - d0;
            if (rows <= 0 || d0 + BAND - 1 < e) continue;
            executed += (double)rows * BAND;
        }
        if (full) n_full += 1; else n_filtered += 1;
    }
    CU(cudaEventRecord(s->ev[1], st));
    CU(cudaEventSynchronize(s->ev[1]));
    double first_ms = 0;
    for (int li : timed) {
        float lm = 0; CU(cudaEventElapsedTime(&lm, s->lev[2 * li], s->lev[2 * li + 1]));
        tile_ms += lm;
        if (li == li_lo) first_ms = lm;
    }
    float ms = 0; CU(cudaEventElapsedTime(&ms, s->ev[0], s->ev[1]));
    unsigned long long cnt[8];
    CU(cudaMemcpy(cnt, s->d_counters, sizeof(cnt), cudaMemcpyDeviceToHost));
    bool overflow = false;
    double max_log = 0;
    {   // a candidate log that overflowed lost candidates: the caller redoes the run exactly
        std::vector<unsigned long long> lc(n_len);
        CU(cudaMemcpy(lc.data(), s->d_logcnt, n_len * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        for (auto c : lc) { overflow |= (long long)c > eff_cap; max_log = std::max(max_log, (double)c); }
    }
    int n_forced = 0;
    double n_fix = 0;
    {
        std::vector<int> fl(n_len);
        CU(cudaMemcpy(fl.data(), s->d_forced, n_len * sizeof(int), cudaMemcpyDeviceToHost));
        for (int f : fl) n_forced += f != 0;
        std::vector<unsigned long long> fx(n_len);
        CU(cudaMemcpy(fx.data(), s->d_fixcnt, n_len * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        for (auto f : fx) n_fix += (double)f;
    }
    double W = 0;
    for (int m = lmin; m <= lmax; ++m) {
        long long k = (n - m + 1) - (m + 1) / 2;
        if (k > 0) W += (double)k * (double)(k + 1) / 2.0;
    }
    s->lmin = lmin; s->lmax = lmax; s->n_len = n_len;
    s->have_profile = true; s->have_final = false; s->have_finals = false;
    memset(s->stats, 0, sizeof(s->stats));
    s->stats[0] = ms; s->stats[2] = executed; s->stats[3] = W; s->stats[4] = tile_ms;
    s->stats[5] = launches; s->stats[6] = n_filtered; s->stats[7] = n_full; s->stats[8] = (double)cnt[0];
    s->stats[9] = klaunch; s->stats[10] = first_ms; s->stats[11] = (double)cnt[2];
    s->stats[12] = n_fix; s->stats[14] = n_forced; s->stats[15] = max_log;
    *overflow_out = overflow;
    return 0;
}

int vlmp_profile_range(vlmp_session* s, int32_t lmin, int32_t lmax, int64_t band_lo,
                       int64_t band_hi, uint32_t flags) {
    if (!s) return fail(VLMP_E_INVALID_PARAMETERS, "null session");
    if (s->n <= 0) return fail(VLMP_E_STATE, "no series uploaded");
    if (lmin > lmax) return fail(VLMP_E_INVALID_PARAMETERS, "lmin > lmax");
    if (lmin < 4) return fail(VLMP_E_INVALID_PARAMETERS, "minimum window length is 4");
    if (s->n < (long long)lmax + (lmax + 1) / 2)
        return fail(VLMP_E_SERIES_TOO_SHORT, "series cannot host a non-trivial pair at lmax");
    std::lock_guard<std::mutex> g(s->lock);
    bool overflow = false;
    int rc = profile_impl(s, lmin, lmax, band_lo, band_hi, flags, &overflow);
    if (rc == 0 && overflow) {
        // candidates were dropped (pathological bounds): exact full folds at every length
        rc = profile_impl(s, lmin, lmax, band_lo, band_hi, flags | VLMP_F_FULL_EVERY_LENGTH, &overflow);
        s->stats[13] = 1;
    }
    return rc;
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
    bool overflow = false;
    if (li_hi < li_lo) { li_lo = lmax - lmin + 1; li_hi = -1; }   // empty shard: setup only
    int rc = profile_impl(s, lmin, lmax, 0, -1, flags, &overflow, li_lo, li_hi);
    if (rc == 0 && overflow) {
        rc = profile_impl(s, lmin, lmax, 0, -1, flags | VLMP_F_FULL_EVERY_LENGTH, &overflow, li_lo, li_hi);
        s->stats[13] = 1;
    }
    return rc;
}

int vlmp_partials_size(vlmp_session* s, int64_t* n_len, int64_t* stride) {
    if (!s || !s->have_profile) return fail(VLMP_E_STATE, "no profile run");
    *n_len = s->n_len; *stride = s->A;
    return 0;
}

int vlmp_partials_export(vlmp_session* s, void* keys, void* idx) {
    if (!s || !s->have_profile) return fail(VLMP_E_STATE, "no profile run");
    std::lock_guard<std::mutex> g(s->lock);
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
    CU(cudaSetDevice(s->device));
    const long long total = (long long)s->n_len * s->A;
    k_import<<<blocks(total, 256), 256, 0, s->stream>>>(s->d_acc, (const unsigned long long*)keys, (const long long*)idx, total);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(s->stream));
    return 0;
}

static int finalize_impl(vlmp_session* s, int li_lo, int li_hi, bool readoffs) {
    CU(cudaSetDevice(s->device));
    cudaStream_t st = s->stream;
    const long long A = s->A, n = s->n;
    int rc;
    if ((size_t)s->n_len * A > s->mp_cap || !s->d_mp || !s->d_ip) {
        if ((rc = ensure1(s->d_mp, (size_t)s->n_len * A))) return rc;
        if ((rc = ensure1(s->d_ip, (size_t)s->n_len * A))) return rc;
        s->mp_cap = (size_t)s->n_len * A;
    }
    const long long n0 = n - s->lmin + 1;
    size_t vc = s->v_cap;
    if (vc < (size_t)n0 || !s->d_vdist) {
        if ((rc = ensure1(s->d_vdist, n0))) return rc;
        if ((rc = ensure1(s->d_vnorm, n0))) return rc;
        if ((rc = ensure1(s->d_vlen, n0))) return rc;
        if ((rc = ensure1(s->d_vidx, n0))) return rc;
        if ((rc = ensure1(s->d_vpop, n0))) return rc;
        s->v_cap = n0;
    }
    CU(cudaEventRecord(s->ev[4], st));
    if (li_lo <= li_hi) {
        FinArgs fa{s->d_tn, s->d_cum, s->d_cum2, s->d_acc, s->d_mp, s->d_ip, n, A, s->lmin, s->n_len, s->floor_,
                   li_lo, li_hi};
        k_finalize_walk<<<blocks(n0, 64), 64, 0, st>>>(fa);
        s->stats[9] += 1;
    }
    if (readoffs) {
        ValmpArgs va{s->d_mp, s->d_ip, s->d_vdist, s->d_vnorm, s->d_vlen, s->d_vidx, s->d_vpop, n, A, s->lmin, s->n_len};
        k_valmp<<<blocks(n0, 256), 256, 0, st>>>(va);
        s->stats[9] += 1;
    }
    CU(cudaEventRecord(s->ev[5], st));
    CU(cudaGetLastError());
    CU(cudaEventSynchronize(s->ev[5]));
    float ms = 0; CU(cudaEventElapsedTime(&ms, s->ev[4], s->ev[5]));
    s->stats[1] = ms;
    s->have_final = readoffs;
    s->have_finals = true;
    return 0;
}

int vlmp_finalize(vlmp_session* s) {
    if (!s || !s->have_profile) return fail(VLMP_E_STATE, "no profile run");
    std::lock_guard<std::mutex> g(s->lock);
    return finalize_impl(s, 0, s->n_len - 1, true);
}

int vlmp_finalize_lengths(vlmp_session* s, int32_t li_lo, int32_t li_hi) {
    if (!s || !s->have_profile) return fail(VLMP_E_STATE, "no profile run");
    if (li_lo < 0 || li_hi < li_lo - 1 || li_hi >= s->n_len)
        return fail(VLMP_E_INVALID_PARAMETERS, "length range outside the profiled range");
    std::lock_guard<std::mutex> g(s->lock);
    return finalize_impl(s, li_lo, li_hi, false);
}

int vlmp_final_buffers(vlmp_session* s, void** mp, void** ip, int64_t* n_len, int64_t* stride) {
    if (!s || !s->have_finals) return fail(VLMP_E_STATE, "no finalized values");
    if (!mp || !ip || !n_len || !stride) return fail(VLMP_E_INVALID_PARAMETERS, "null argument");
    *mp = s->d_mp; *ip = s->d_ip; *n_len = s->n_len; *stride = s->A;
    return 0;
}

int vlmp_finalize_readoffs(vlmp_session* s) {
    if (!s || !s->have_finals) return fail(VLMP_E_STATE, "no finalized values");
    std::lock_guard<std::mutex> g(s->lock);
    return finalize_impl(s, 0, -1, true);
}

int vlmp_get_valmp(vlmp_session* s, double* dist, double* norm, int64_t* lengths, int64_t* indices,
                   uint8_t* populated) {
    if (!s || !s->have_final) return fail(VLMP_E_STATE, "not finalized");
    std::lock_guard<std::mutex> g(s->lock);
    CU(cudaSetDevice(s->device));
    const long long n0 = s->n - s->lmin + 1;
    CU(cudaMemcpyAsync(dist, s->d_vdist, n0 * 8, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaMemcpyAsync(norm, s->d_vnorm, n0 * 8, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaMemcpyAsync(lengths, s->d_vlen, n0 * 8, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaMemcpyAsync(indices, s->d_vidx, n0 * 8, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaMemcpyAsync(populated, s->d_vpop, n0, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    return 0;
}

int vlmp_get_profile(vlmp_session* s, int32_t length, double* mp, int64_t* ip) {
    if (!s || !s->have_final) return fail(VLMP_E_STATE, "not finalized");
    if (length < s->lmin || length > s->lmax) return fail(VLMP_E_INVALID_PARAMETERS, "length outside the run");
    std::lock_guard<std::mutex> g(s->lock);
    CU(cudaSetDevice(s->device));
    const long long N = s->n - length + 1;
    const long long off = (long long)(length - s->lmin) * s->A;
    std::vector<int> tmp(N);
    CU(cudaMemcpyAsync(mp, s->d_mp + off, N * 8, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaMemcpyAsync(tmp.data(), s->d_ip + off, N * 4, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    for (long long o = 0; o < N; ++o) ip[o] = tmp[o];
    return 0;
}

int vlmp_smallest_rows(vlmp_session* s, int32_t k2, int64_t* out_off, int64_t* out_nbr, double* out_d) {
    if (!s || !s->have_final) return fail(VLMP_E_STATE, "not finalized");
    if (k2 < 1 || k2 > 64) return fail(VLMP_E_INVALID_PARAMETERS, "k2 must be in [1, 64]");
    std::lock_guard<std::mutex> g(s->lock);
    CU(cudaSetDevice(s->device));
    const long long cnt = (long long)s->n_len * k2;
    int rc;
    if ((rc = ensure(s->d_ro_i64, s->ro_i64_cap, (size_t)(2 * cnt)))) return rc;
    if ((rc = ensure(s->d_ro_f64, s->ro_f64_cap, (size_t)cnt))) return rc;
    long long* d_off = s->d_ro_i64; long long* d_nbr = s->d_ro_i64 + cnt; double* d_d = s->d_ro_f64;
    SmallArgs sa{s->d_mp, s->d_ip, d_off, d_nbr, d_d, s->n, s->A, s->lmin, k2};
    k_smallest<<<s->n_len, 256, 0, s->stream>>>(sa);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(out_off, d_off, cnt * 8, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaMemcpyAsync(out_nbr, d_nbr, cnt * 8, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaMemcpyAsync(out_d, d_d, cnt * 8, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    s->stats[9] += 1;
    return 0;
}

int vlmp_discords(vlmp_session* s, int32_t k, double* out_dist, int64_t* out_off) {
    if (!s || !s->have_final) return fail(VLMP_E_STATE, "not finalized");
    if (k < 1 || k > 32) return fail(VLMP_E_INVALID_PARAMETERS, "k must be in [1, 32]");
    std::lock_guard<std::mutex> g(s->lock);
    CU(cudaSetDevice(s->device));
    const long long cnt = (long long)s->n_len * k;
    int rc;
    if ((rc = ensure(s->d_ro_i64, s->ro_i64_cap, (size_t)cnt))) return rc;
    if ((rc = ensure(s->d_ro_f64, s->ro_f64_cap, (size_t)cnt))) return rc;
    double* d_d = s->d_ro_f64; long long* d_o = s->d_ro_i64;
    DiscArgs da{s->d_mp, d_d, d_o, s->n, s->A, s->lmin, s->n_len, k};
    k_discords<<<s->n_len, 32, 0, s->stream>>>(da);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(out_dist, d_d, cnt * 8, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaMemcpyAsync(out_off, d_o, cnt * 8, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    s->stats[9] += 1;
    return 0;
}

int vlmp_ranking_events(vlmp_session* s, double tau, int64_t cap, int64_t* ev_off, int64_t* ev_nbr,
                        int64_t* ev_len, double* ev_dist, double* ev_norm, int64_t* count) {
    if (!s || !s->have_final) return fail(VLMP_E_STATE, "not finalized");
    std::lock_guard<std::mutex> g(s->lock);
    CU(cudaSetDevice(s->device));
    cudaStream_t st = s->stream;
    long long c = std::max<long long>(cap, 1);
    int rc;
    if ((rc = ensure(s->d_ro_i64, s->ro_i64_cap, (size_t)(3 * c)))) return rc;
    if ((rc = ensure(s->d_ro_f64, s->ro_f64_cap, (size_t)(2 * c)))) return rc;
    if (!s->d_ro_cnt) CU(cudaMalloc((void**)&s->d_ro_cnt, 8));
    long long *d_o = s->d_ro_i64, *d_nb = s->d_ro_i64 + c, *d_l = s->d_ro_i64 + 2 * c;
    double *d_d = s->d_ro_f64, *d_n = s->d_ro_f64 + c;
    unsigned long long* d_c = s->d_ro_cnt;
    CU(cudaMemsetAsync(d_c, 0, 8, st));
    const long long n0 = s->n - s->lmin + 1;
    EvArgs ea{s->d_mp, s->d_ip, tau, d_o, d_nb, d_l, d_d, d_n, d_c, cap, s->n, s->A, s->lmin, s->n_len};
    k_events<<<blocks(n0, 256), 256, 0, st>>>(ea);
    CU(cudaGetLastError());
    unsigned long long hc = 0;
    CU(cudaMemcpyAsync(&hc, d_c, 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    long long take = std::min<long long>((long long)hc, cap);
    if (take > 0) {
        CU(cudaMemcpyAsync(ev_off, d_o, take * 8, cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(ev_nbr, d_nb, take * 8, cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(ev_len, d_l, take * 8, cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(ev_dist, d_d, take * 8, cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(ev_norm, d_n, take * 8, cudaMemcpyDeviceToHost, st));
    }
    CU(cudaStreamSynchronize(st));
    *count = (int64_t)hc;
    return 0;
}

int vlmp_range_query(vlmp_session* s, int64_t n_q, const int64_t* owners, const int32_t* lengths,
                     const double* radii, int64_t cap, int64_t* members, int64_t* counts) {
    if (!s || (n_q > 0 && (!owners || !lengths || !radii || !members || !counts)) || n_q < 0 || cap < 0)
        return fail(VLMP_E_INVALID_PARAMETERS, "bad range query arguments");
    if (s->n <= 0) return fail(VLMP_E_STATE, "no series uploaded");
    if (n_q == 0) return 0;
    long long max_n = 0;
    for (long long q = 0; q < n_q; ++q) {
        if (lengths[q] < 4 || lengths[q] > s->n || owners[q] < 0 || owners[q] > s->n - lengths[q])
            return fail(VLMP_E_INVALID_PARAMETERS, "range query owner/length outside the series");
        max_n = std::max<long long>(max_n, s->n - lengths[q] + 1);
    }
    std::lock_guard<std::mutex> g(s->lock);
    CU(cudaSetDevice(s->device));
    cudaStream_t st = s->stream;
    const long long c = std::max<long long>(cap, 1);
    long long* d_own = nullptr; int* d_len = nullptr; double* d_rad = nullptr;
    long long* d_mem = nullptr; unsigned long long* d_cnt = nullptr;
    CU(cudaMallocAsync((void**)&d_own, n_q * 8, st));
    CU(cudaMallocAsync((void**)&d_len, n_q * 4, st));
    CU(cudaMallocAsync((void**)&d_rad, n_q * 8, st));
    CU(cudaMallocAsync((void**)&d_mem, n_q * c * 8, st));
    CU(cudaMallocAsync((void**)&d_cnt, n_q * 8, st));
    CU(cudaMemcpyAsync(d_own, owners, n_q * 8, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(d_len, lengths, n_q * 4, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(d_rad, radii, n_q * 8, cudaMemcpyHostToDevice, st));
    CU(cudaMemsetAsync(d_cnt, 0, n_q * 8, st));
    RangeArgs ra{s->d_tn, s->d_cum, s->d_cum2, d_own, d_len, d_rad, d_mem, d_cnt, c, s->n, s->floor_};
    dim3 grid((unsigned)((max_n + 255) / 256), (unsigned)n_q);
    k_range_query<<<grid, 256, 0, st>>>(ra);
    CU(cudaGetLastError());
    std::vector<unsigned long long> hc(n_q);
    CU(cudaMemcpyAsync(hc.data(), d_cnt, n_q * 8, cudaMemcpyDeviceToHost, st));
    if (cap > 0) CU(cudaMemcpyAsync(members, d_mem, n_q * cap * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    for (long long q = 0; q < n_q; ++q) counts[q] = (int64_t)hc[q];
    cudaFreeAsync(d_own, st); cudaFreeAsync(d_len, st); cudaFreeAsync(d_rad, st);
    cudaFreeAsync(d_mem, st); cudaFreeAsync(d_cnt, st);
    CU(cudaStreamSynchronize(st));
    s->stats[9] += 1;
    return 0;
}

int vlmp_stats(vlmp_session* s, double* out, int32_t n_out) {
    if (!s || !out) return fail(VLMP_E_INVALID_PARAMETERS, "null argument");
    for (int q = 0; q < n_out && q < 16; ++q) out[q] = s->stats[q];
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
        // no full-fold fallback here (it folds the 1-best only): forced offsets are recomputed
        k_qprep<<<blocks(A, 256), 256, 0, st>>>(s->d_prm, s->d_colq, s->d_rowq, N, A, s->sscale, nullptr);
        if (T) {
            ta.update_seeds = li + 1 < n_len;
            k_tile<false><<<blocks(T, WARPS_PER_CTA), WARPS_PER_CTA * 32, smem, st>>>(ta);
            k_log_slots<<<296, 128, 0, st>>>(s->d_log, s->d_logcnt + li, (long long)s->log_cap, s->d_prm, e,
                                             s->d_slots, s->d_slotcnt, s->d_counters);
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
        if (c > s->log_cap) return fail(VLMP_E_CUDA, "m-best candidate log overflow (bounds too weak for this series)");
    // finalize: canonical sorted distances of the m best; MP/IP (first neighbour) for VALMP
    if ((rc = ensure(s->d_mpm, s->mpm_cap, (size_t)n_len * A * mb))) return rc;
    dim3 grid(blocks(N0, 128), n_len);
    k_finalize_m<<<grid, 128, 0, st>>>(s->d_tn, s->d_cum, s->d_cum2, s->d_ipm, s->d_mpm, n, A, lmin, mb, s->floor_);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(st));
    s->lmin = lmin; s->lmax = lmax; s->n_len = n_len; s->mbest = mb;
    s->have_profile = false; s->have_final = false; s->have_finals = false;
    memset(s->stats, 0, sizeof(s->stats));
    s->stats[0] = ms; s->stats[13] = (double)redo_total;
    return 0;
}

int vlmp_get_profile_m(vlmp_session* s, int32_t length, double* dist, int64_t* nbr) {
    if (!s || s->mbest < 1 || !s->d_mpm) return fail(VLMP_E_STATE, "no m-best run");
    if (length < s->lmin || length > s->lmax) return fail(VLMP_E_INVALID_PARAMETERS, "length outside the run");
    std::lock_guard<std::mutex> g(s->lock);
    CU(cudaSetDevice(s->device));
    const int mb = s->mbest;
    const long long N = s->n - length + 1;
    const long long off = (long long)(length - s->lmin) * s->A * mb;
    std::vector<int> tmp(N * mb);
    CU(cudaMemcpyAsync(dist, s->d_mpm + off, N * mb * 8, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaMemcpyAsync(tmp.data(), s->d_ipm + off, N * mb * 4, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    for (long long q = 0; q < N * mb; ++q) nbr[q] = tmp[q];
    return 0;
}

int vlmp_discords_m(vlmp_session* s, int32_t k, double* out_dist, int64_t* out_off) {
    if (!s || !s->d_mpm) return fail(VLMP_E_STATE, "no m-best run");
    if (k < 1 || k > 32) return fail(VLMP_E_INVALID_PARAMETERS, "k must be in [1, 32]");
    const int mb = s->mbest;
    if (k * mb > 32 * MB_MAX) return fail(VLMP_E_INVALID_PARAMETERS, "k*m too large");
    std::lock_guard<std::mutex> g(s->lock);
    CU(cudaSetDevice(s->device));
    const long long cnt = (long long)s->n_len * k * mb;
    int rc;
    if ((rc = ensure(s->d_ro_i64, s->ro_i64_cap, (size_t)cnt))) return rc;
    if ((rc = ensure(s->d_ro_f64, s->ro_f64_cap, (size_t)cnt))) return rc;
    const int wpb = 4;
    const size_t sm = (size_t)wpb * 32 * MB_MAX * 16;
    k_discords_m<<<blocks((long long)s->n_len * 32, wpb * 32), wpb * 32, sm, s->stream>>>(
        s->d_mpm, s->d_ro_f64, s->d_ro_i64, s->n, s->A, s->lmin, s->n_len, k, mb);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(out_dist, s->d_ro_f64, cnt * 8, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaMemcpyAsync(out_off, s->d_ro_i64, cnt * 8, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    return 0;
}

int vlmp_event_record(vlmp_session* s, int32_t slot) {
    if (!s || slot < 0 || slot > 1) return fail(VLMP_E_INVALID_PARAMETERS, "slot must be 0 or 1");
    CU(cudaSetDevice(s->device));
    CU(cudaEventRecord(s->ev[6 + slot], s->stream));
    return 0;
}

int vlmp_event_elapsed(vlmp_session* s, float* ms) {
    if (!s || !ms) return fail(VLMP_E_INVALID_PARAMETERS, "null argument");
    CU(cudaSetDevice(s->device));
    CU(cudaEventSynchronize(s->ev[7]));
    CU(cudaEventElapsedTime(ms, s->ev[6], s->ev[7]));
    return 0;
}

int vlmp_measure_fp64_peak(vlmp_session* s, double* fma_per_s) {
    if (!s || !fma_per_s) return fail(VLMP_E_INVALID_PARAMETERS, "null argument");
    std::lock_guard<std::mutex> g(s->lock);
    CU(cudaSetDevice(s->device));
    int sms = 0;
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device));
    double* d_out = nullptr;
    CU(cudaMalloc((void**)&d_out, 8));
    const int threads = 512, per_sm = 4, iters = 2048;
    const unsigned grid = sms * per_sm;
    k_dfma_peak<<<grid, threads, 0, s->stream>>>(d_out, 16, 1.0);   // warm-up
    CU(cudaEventRecord(s->ev[6], s->stream));
    k_dfma_peak<<<grid, threads, 0, s->stream>>>(d_out, iters, 1.0);
    CU(cudaEventRecord(s->ev[7], s->stream));
    CU(cudaEventSynchronize(s->ev[7]));
    float ms = 0; CU(cudaEventElapsedTime(&ms, s->ev[6], s->ev[7]));
    CU(cudaFree(d_out));
    const double fmas = (double)grid * threads * iters * 16.0 * 8.0;
    *fma_per_s = fmas / (ms * 1e-3);
    return 0;
}

}  // extern "C"
