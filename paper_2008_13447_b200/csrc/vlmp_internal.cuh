// vlmp_internal.cuh -- shared declarations of the libvlmp translation units
// (profile.cu: phase 1 kernels + host; readout.cu: phase 2 / read-offs; session.cu:
// sessions, series upload, timing). See profile.cu for the kernel map.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <algorithm>
#include <cstddef>
#include <mutex>
#include <string>
#include <vector>
#include "../../include/vlmp.h"

namespace vlmp_impl {

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

extern thread_local std::string g_err;   // session.cu

inline int fail(int code, const std::string& msg) { g_err = msg; return code; }

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
__device__ inline double pair_distance(const double* __restrict__ t, const double* __restrict__ cum,
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

// A filter-kernel log record: a lane whose cells passed the bound at row i; its 8 cells are
// (i, j0 + s) and cov[s] is their covariance, so the merge kernel can recompute the exact
// keys with the kernel's own FMA sequence (bit-identical) and apply the exact tests.
struct __align__(16) RowRec { int i; int j0; int pad0, pad1; double cov[D]; };


// ---------------------------------------------------------------------------------
// shared device helpers (profile.cu, filter32.cu)
__device__ inline bool key_less(unsigned long long k1, long long i1, unsigned long long k2, long long i2) {
    return k1 < k2 || (k1 == k2 && i1 < i2);
}

// exact lexicographic (key, idx) min into a 16-byte accumulator (128-bit CAS)
__device__ inline void acc_merge(ulonglong2* slot, unsigned long long key, long long idx) {
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

// device clock (ns) for kernel spans: one atomicMin at a CTA's start and one atomicMax at its end
// give a launch's first-start-to-last-end time without events (which would split a CUDA graph)
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}

// timing event on a stream that may be capturing a CUDA graph (profile_impl): inside a capture
// the record must become an external event node, outside it is a plain record
inline cudaError_t rec_event(cudaEvent_t ev, cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal)
                                               : cudaEventRecord(ev, st);
}

// Launch at the device's highest priority. With two chains sharing the GPU the short kernels
// between a chain's walks (k_runs, parameters, bounds, factors) otherwise queue behind every
// pending block of the other chain's walk (~200 us each time; ~2 us at high priority). This
// attribute reaches plain stream launches (VLMP_GRAPH=0); a captured node does not keep it, so
// profile_impl sets cudaKernelNodeAttributePriority on the graph's nodes and instantiates it
// with cudaGraphInstantiateFlagUseNodePriority.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_hi(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                             Args&&... args) {
    static int hi = [] { int lo_ = 0, hi_ = 0; cudaDeviceGetStreamPriorityRange(&lo_, &hi_); return hi_; }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid; cfg.blockDim = block; cfg.dynamicSmemBytes = smem; cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributePriority; at[0].val.priority = hi;
    cfg.attrs = at; cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

__device__ inline void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ inline void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Filter thresholds in the covariance domain (profile.cu k_qprep, filter32.cu k_prep32). A cell
// (i, j) must reach the exact tests when its key r = 1 - cov inv_i inv_j satisfies
// hi(r) <= max(U_i, U_j), i.e. r <= R(U) with R(U) the largest double of that high word. With
// q(U) = 1 - R(U) - 2^-20 and s = 1/inv:  r <= R(U)  =>  cov >= q(U) s_i s_j  (2^-20 >> the
// FP64 rounding of r). q < 2^-20 (a bound at corr ~ 0) is clamped to 0, which still passes every
// cell of positive covariance; only offsets whose OWN bound is that weak may need
// non-positive-covariance cells: they are "forced" (the length falls back to exact full folds).
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

constexpr int MB_MAX = 8;                 // m-best mode: largest supported m
constexpr int SLOT_CAP = 24;              // m-best mode: candidate slots per offset per length

// FP32 filter (filter32.cu): a run of consecutive passing cells along one diagonal of a tile,
// (i, j), (i+1, j+1), ..., len cells; evaluated exactly in FP64 by k_runs
struct __align__(16) Run { int i; int j; int len; int pad; };

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

// profile.cu: wait for / check / redo a pending phase 1; device-event timings of the last run
int settle_profile(vlmp_session* s, bool* redone);
int mbest_impl(vlmp_session* s, int32_t lmin, int32_t lmax, int32_t mb);   // lock held by the caller
void launch_params(vlmp_session* s, cudaStream_t st, Prm* prm, double* mu, int m);
// pruned.cu
struct PrunedState;
void pruned_free(vlmp_session* s);
int fill_event_stats(vlmp_session* s);
// lock held by the caller: one exhaustive 1-best pass (profile.cu) and its phase 2 (readout.cu)
int profile_locked(vlmp_session* s, int lmin, int lmax);
int finalize_lengths_locked(vlmp_session* s, int li_lo, int li_hi);
}  // namespace vlmp_impl

using namespace vlmp_impl;

// =================================================================================
// a phase-1 run that was enqueued but not yet checked (profile.cu settle_profile)
struct PendingRun {
    int lmin = 0, lmax = 0; long long band_lo = 0, band_hi = -1; uint32_t flags = 0;
    int li_lo = 0, li_hi = -1; bool fp32 = false, sampled = false, graph = false;
    long long cap_used = 0; int S = 0;
    double executed = 0, launches = 0, n_filtered = 0, n_full = 0, klaunch = 0;
    std::vector<int> timed, walked;
    int chains = 1;   // 2: the length range ran as two concurrent chains (kernel spans overlap)
};

struct vlmp_session {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[8] = {};
    std::mutex lock;
    // series
    long long n = 0, A = 0;
    double floor_ = 0.0;
    double* d_tn = nullptr; double* d_cum = nullptr; double* d_cum2 = nullptr;
    size_t tn_cap = 0, cum_cap = 0, cum2_cap = 0, prm_cap = 0, mu_cap = 0, prm2_cap = 0, mu2_cap = 0,
           previdx_cap = 0, colq_cap = 0, rowq_cap = 0;
    // per-length scratch
    Prm* d_prm = nullptr; double* d_mu = nullptr;
    Prm* d_prm2 = nullptr; double* d_mu2 = nullptr;     // previous length's (1-best bound)
    long long* d_previdx = nullptr;
    float2* d_colq = nullptr; float2* d_rowq = nullptr;   // filter factors (k_qprep)
    int* d_forced = nullptr; size_t forced_cap = 0;      // per-length: full-fold fallback
    float4* d_p32 = nullptr; size_t p32_cap = 0;         // FP32 filter: {df, dg, b, w}
    float2* d_cq32 = nullptr; size_t cq32_cap = 0;       // FP32 filter: {a, b}
    float4* d_cq4 = nullptr; size_t cq4_cap = 0;         // packed walk: band-pair {a, b, a', b'}
    float4* d_pf4 = nullptr; size_t pf4_cap = 0;         // packed walk: band-pair {df, df', dg, dg'}
    unsigned* d_magblk = nullptr; size_t magblk_cap = 0; // FP32 filter: per-256-offset magnitude bound
    int4* d_tiles32 = nullptr; size_t tiles32_cap = 0;   // FP32 filter tiles (pairs of FP64 tiles)
    unsigned long long* d_fixcnt = nullptr; size_t fixcnt_cap = 0;   // per-length re-bounded offsets
    double sscale = 1.0; int hiC = 896 << 20;            // filter: 2^-k scale, hi-word bias
    // tiles / seeds (host tile lists cached per (n, lmin, bands, flags): tc_*)
    long long tc_n = -1, tc_key[5] = {-1, -1, -1, -1, -1}, tc_T = 0, tc_Ts = 0, tc_T32 = 0;
    int tc_S = 0;
    int2* d_tiles = nullptr; size_t tiles_cap = 0;
    int2* d_tiles_s = nullptr; size_t tiles_s_cap = 0;   // sampled bands of a shard's first length
    int* d_smap = nullptr; size_t smap_cap = 0;          // their seed slots
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
    int mbest = 0;                        // m of the last m-best run (0: none valid)
    int mb_lmin = 0, mb_n_len = 0; long long mb_A = 0, mb_n = 0;   // the run it describes
    ulonglong2* d_slots = nullptr; size_t slots_cap = 0;
    int* d_slotcnt = nullptr; size_t slotcnt_cap = 0;
    int* d_ipm = nullptr; size_t ipm_cap = 0;
    double* d_mpm = nullptr; size_t mpm_cap = 0;
    long long* d_redo = nullptr; size_t redo_cap = 0;
    // run state
    int lmin = 0, lmax = 0, n_len = 0; bool have_profile = false, have_final = false, have_finals = false;
    double stats[25] = {};
    bool pending = false, stats_dirty = false;          // phase 1 enqueued, not yet settled
    PendingRun prun;
    unsigned long long* h_chk = nullptr; size_t h_chk_cap = 0;   // pinned: its overflow counters
    unsigned char* h_col = nullptr; size_t h_col_cap = 0;        // pinned staging of vlmp_finalize_collect
    std::vector<cudaEvent_t> lev;   // 2 per length: tile-kernel start/stop
    unsigned long long* d_span = nullptr; size_t span_cap = 0;   // [n_len][4] k_tile32 / k_runs spans (ns)
    unsigned long long* h_span = nullptr; size_t h_span_cap = 0;
    // the per-length launch sequence of profile_impl as one CUDA graph, re-launched while its
    // key (shape, buffers, series scalars) is unchanged
    cudaGraphExec_t g_exec = nullptr;
    std::vector<double> g_key;
    std::vector<double> g_cnt; std::vector<int> g_timed, g_walked;   // its host-side counters
    // second chain: on small series the two halves of the length range are walked concurrently
    // (profile_impl), each with its own per-length scratch; accumulators and counters are shared
    Prm* x_prm = nullptr; Prm* x_prm2 = nullptr; double* x_mu = nullptr; double* x_mu2 = nullptr;
    float4* x_p32 = nullptr; float2* x_cq32 = nullptr; float4* x_cq4 = nullptr; float4* x_pf4 = nullptr;
    unsigned* x_magblk = nullptr; double* x_seeds = nullptr; RowRec* x_log = nullptr;
    size_t x_prm_cap = 0, x_prm2_cap = 0, x_mu_cap = 0, x_mu2_cap = 0, x_p32_cap = 0, x_cq32_cap = 0,
           x_cq4_cap = 0, x_pf4_cap = 0, x_magblk_cap = 0, x_seeds_cap = 0, x_log_cap = 0;
    cudaStream_t stream2 = nullptr; cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    vlmp_impl::PrunedState* pp = nullptr;                  // pruned discord scan (pruned.cu)
};

namespace vlmp_impl {
// filter32.cu
int tile32_width();
const void* tile32_func();   // the FP32 walk kernel (profile.cu: graph node priorities)
size_t tile32_smem();
int filter32_setup();
void build_tiles32(const std::vector<int2>& tiles, long long band_lo, std::vector<int4>& out);
int launch_filter32(vlmp_session* s, cudaStream_t st, const Prm* prm, const double* mu, long long N, int m, int e,
                    long long dl, int S, int update_seeds, long long n_t32, const int* forced,
                    ulonglong2* acc, Run* runs, unsigned long long* run_count, long long run_cap,
                    ulonglong2* slots = nullptr, int* slot_cnt = nullptr, unsigned long long* span = nullptr);
// profile.cu: wait for / check / redo a pending phase 1; device-event timings of the last run
int settle_profile(vlmp_session* s, bool* redone);
int mbest_impl(vlmp_session* s, int32_t lmin, int32_t lmax, int32_t mb);   // lock held by the caller
void launch_params(vlmp_session* s, cudaStream_t st, Prm* prm, double* mu, int m);
// pruned.cu
struct PrunedState;
void pruned_free(vlmp_session* s);
int fill_event_stats(vlmp_session* s);
}  // namespace vlmp_impl
