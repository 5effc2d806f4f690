// pruned.cu -- MAD's pruned top-k m-th discord scan on the GPU (the reference's
// topkm_discord_discovery / topkm_next_length, discords.py:144-247, over its partial profiles,
// profile.py:66-232): exact like the exhaustive path, but most rows never get a full profile.
//
// Per row the scan keeps P stored neighbours (the reference keeps p; `PartialProfiles`): m = 1
// keeps the nearest one (from the exhaustive 1-best pass: the FP32 walk + exact runs), m > 1 keeps
// P = min(8, max(p, m)) (from the exhaustive m-best pass); at the first length (and after any full
// fallback length) the stored set comes from that pass (`_harvest_select` over the row), with the
// centred co-moments C (direct sums), m_f = max bound factor over them and sigma_base.
//   * each later length advances every stored co-moment by the Welford step
//     C_{l+1} = C_l + l/(l+1) (x_l - mu_x)(y_l - mu_y)  (O(1), `PartialProfiles.advance`), drops
//     entries whose neighbour left the series, turned constant or became trivial, and certifies
//     the row when its m-th stored distance is below m_f sigma_base / sigma_l (VALMOD's Eq. 2:
//     no unstored pair can be closer -- `thresholds`, `certify_step`).
// The replay (one warp, `update_fixed_length_discords` in ascending offsets) takes certified rows'
// stored m best (canonical values, discords.py:126-141), skips a non-certified row whose stored
// distances (upper bounds of its true m best) beat no cell of the matrix's last row (discords.py:
// 176-181), and stops at the first non-certified row it cannot skip. The rows of the window
// [stop, stop + max(2048, stop)) that could matter at the current last row (a superset of the
// window's stops: the last row only grows) are then recomputed exactly -- m = 1: blocks of <= 128
// consecutive rows (k_pp_block), m > 1: full rows (k_pp_rows) -- their stored entries refreshed
// at this length (`set_row`), and the replay resumes. A length whose modelled recompute cost
// exceeds an exhaustive pass runs that pass instead and re-harvests every row (VALMOD's full
// recompute). DESIGN.md §2c has the measured A/B against the exhaustive path.
#include "vlmp_internal.cuh"
#include <time.h>

namespace vlmp_impl {

constexpr int PP_MAX = MB_MAX;        // stored entries per row
constexpr int RBATCH = 64;            // full rows recomputed per replay stop (at most)
constexpr int RC_T = 256;             // threads of a full-row CTA
constexpr int RC_R = 8;               // columns per thread
constexpr int RC_COLS = RC_T * RC_R;  // columns per CTA
constexpr int KMAX_CELLS = 32 * MB_MAX;
constexpr double PP_MARGIN = 1e-9;    // approximate values vs exact decisions

struct PPCand { unsigned long long key; long long j; double cov; };
struct PBlock { long long a; int len; int pad; };   // a block of rows [a, a + len) (m = 1 recomputes)

struct ReplayState {
    long long pos;            // next owner to process
    int status;               // 0 running / 1 need rows / 2 done
    int nlist;                // rows listed for recompute
    double d[KMAX_CELLS];     // the k x m matrix (row-major)
    long long o[KMAX_CELLS];
};

struct PrunedState {
    int P = 0, mb = 1, k = 1;
    long long rows = 0;
    int* nbr = nullptr; double* cov = nullptr; size_t ent_cap = 0;          // [rows][P]
    double* mf = nullptr; double* sb = nullptr; unsigned char* ok = nullptr; size_t row_cap = 0;
    double* ub = nullptr; int* ubn = nullptr; double* ex = nullptr; size_t mrow_cap = 0;   // [rows][mb]
    unsigned char* cert = nullptr; unsigned char* done = nullptr;
    ReplayState* rs = nullptr; ReplayState* h_rs = nullptr;
    long long* list = nullptr;
    PPCand* cand = nullptr; size_t cand_cap = 0;
    unsigned long long* cnt = nullptr; unsigned long long* h_cnt = nullptr;   // [4] per length
    long long* h_list = nullptr;                                              // m = 1 row blocks
    PBlock* blk = nullptr; PBlock* h_blk = nullptr;
    int* row_blk = nullptr; int* h_row_blk = nullptr; size_t row_blk_cap = 0;
    ulonglong2* racc = nullptr;
    long long dbg_blocks = 0;                                                 // VLMP_PRUNED_DEBUG
};

__device__ __forceinline__ bool cand_less(unsigned long long k1, long long j1, unsigned long long k2, long long j2) {
    return k1 < k2 || (k1 == k2 && j1 < j2);
}

// ---------------------------------------------------------------------------------
// stored entries from an exhaustive m-best run (ipm: [row][P] neighbours in key order), one warp
// per row; also the exact canonical m best (sorted) so the replay can take every row as "done"
struct HarvestArgs {
    const double* tn; const double* cum; const double* cum2; const Prm* prm; const double* mu;
    const int* ipm; long long N; int m, P, mb; double floor_;
    int* nbr; double* cov; double* mf; double* sb; unsigned char* ok;
    double* ex; unsigned char* done; unsigned char* cert;
};

__global__ void k_pp_harvest(HarvestArgs a) {
    const int lane = threadIdx.x & 31;
    const long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    if (i >= a.N) return;
    const double io = a.prm[i].inv, mi = a.mu[i];
    const bool row_ok = io == io;
    double fmax_ = 0.0;
    int nvalid = 0;
    for (int q = 0; q < a.P; ++q) {
        const int j = a.ipm[i * a.P + q];
        double acc = 0.0;
        if (row_ok && j >= 0) {
            const double mj = a.mu[j];
            for (int k = lane; k < a.m; k += 32) acc = fma(a.tn[i + k] - mi, a.tn[j + k] - mj, acc);
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(FULLMASK, acc, off);
        if (lane == 0) {
            a.nbr[i * a.P + q] = (row_ok && j >= 0) ? j : -1;
            a.cov[i * a.P + q] = acc;
            if (row_ok && j >= 0) {
                const double qq = acc * io * a.prm[j].inv;
                const double qp = qq > 0.0 ? qq : 0.0;
                fmax_ = fmax(fmax_, sqrt((double)a.m * fmax(0.0, 1.0 - qp * qp)));
                ++nvalid;
            }
        }
    }
    // exact canonical values of the m best (discords.py:126-141), lanes c < mb in parallel
    double v = INFINITY;
    if (lane < a.mb && row_ok) {
        const int j = a.ipm[i * a.P + lane];
        if (j >= 0) v = pair_distance(a.tn, a.cum, a.cum2, i, j, a.m, a.floor_);
    }
    double vals[MB_MAX];
#pragma unroll
    for (int c = 0; c < MB_MAX; ++c) vals[c] = __shfl_sync(FULLMASK, v, c);
    if (lane == 0) {
        for (int q = 1; q < a.mb; ++q)
            for (int r = q; r > 0 && vals[r] < vals[r - 1]; --r) { const double t = vals[r]; vals[r] = vals[r - 1]; vals[r - 1] = t; }
        for (int c = 0; c < a.mb; ++c) a.ex[i * a.mb + c] = vals[c];
        // fewer live cells than P: the stored set is the whole row, but cells that are constant now
        // may turn valid later -- never certify such a row (recompute when it matters)
        a.mf[i] = nvalid == a.P ? fmax_ : 0.0;
        a.sb[i] = row_ok ? 1.0 / (io * sqrt((double)a.m)) : 0.0;
        a.ok[i] = row_ok ? 1 : 0;
        a.done[i] = 1; a.cert[i] = 0;
    }
}

// ---------------------------------------------------------------------------------
// one length step of every stored entry (PartialProfiles.advance + thresholds + certify)
struct AdvanceArgs {
    const double* tn; const Prm* prm; const double* mu_prev;
    long long rows, N, n; int m, e, P, mb;      // m = the new length
    int* nbr; double* cov; const double* mf; const double* sb; unsigned char* ok;
    double* ub; int* ubn; unsigned char* cert; unsigned char* done;
    unsigned long long* cnt;                     // [0] certified rows, [1] non-certified live rows
};

__global__ void k_pp_advance(AdvanceArgs a) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    unsigned nc = 0, nn = 0;
    if (i < a.rows) {
        const int m0 = a.m - 1;
        const double w = (double)m0 / (double)a.m;
        bool rok = a.ok[i] && i < a.N;
        const double io = rok ? a.prm[i].inv : 0.0;
        rok = rok && io == io;
        unsigned long long bk[MB_MAX]; long long bj[MB_MAX];
        for (int c = 0; c < MB_MAX; ++c) { bk[c] = KEY_NONE; bj[c] = IDX_NONE; }
        if (rok) {
            const double xi = (a.tn[i + m0] - a.mu_prev[i]) * w;
            for (int q = 0; q < a.P; ++q) {
                const long long j = a.nbr[i * a.P + q];
                if (j < 0) continue;
                const long long dd = j > i ? j - i : i - j;
                bool alive = j < a.N && dd >= a.e;
                double ij = 0.0;
                if (alive) { ij = a.prm[j].inv; alive = ij == ij; }
                if (!alive) { a.nbr[i * a.P + q] = -1; continue; }
                const double c = fma(xi, a.tn[j + m0] - a.mu_prev[j], a.cov[i * a.P + q]);
                a.cov[i * a.P + q] = c;
                unsigned long long key = clamp_key(fma(-(c * io), ij, 1.0)) & ~PMASK;
                long long jj = j;
                for (int t = 0; t < a.mb; ++t)
                    if (cand_less(key, jj, bk[t], bj[t])) {
                        const unsigned long long tk = bk[t]; const long long tj = bj[t];
                        bk[t] = key; bj[t] = jj; key = tk; jj = tj;
                    }
            }
        } else if (a.ok[i]) a.ok[i] = 0;   // the owner left the series or turned constant: sticky
        double last = INFINITY;
        for (int c = 0; c < a.mb; ++c) {
            double d = INFINITY;
            if (bk[c] != KEY_NONE) d = sqrt(2.0 * (double)a.m * __longlong_as_double((long long)bk[c]));
            a.ub[i * a.mb + c] = d;
            a.ubn[i * a.mb + c] = bj[c] == IDX_NONE ? -1 : (int)bj[c];
            last = d;
        }
        bool ct = false;
        if (rok && last < INFINITY) {
            const double thr = a.mf[i] * a.sb[i] * io * sqrt((double)a.m);   // m_f sigma_base / sigma_l
            ct = last * (1.0 + PP_MARGIN) < thr * (1.0 - PP_MARGIN);
        }
        a.cert[i] = ct ? 1 : 0;
        a.done[i] = 0;
        if (i < a.N && io == io) { if (ct) nc = 1; else nn = 1; }
    }
    nc = __reduce_add_sync(FULLMASK, nc); nn = __reduce_add_sync(FULLMASK, nn);
    if ((threadIdx.x & 31) == 0 && (nc | nn)) { atomicAdd(a.cnt + 0, (unsigned long long)nc); atomicAdd(a.cnt + 1, (unsigned long long)nn); }
}

// ---------------------------------------------------------------------------------
// the replay (update_fixed_length_discords over ascending owners), one warp
struct ReplayArgs {
    const double* tn; const double* cum; const double* cum2; const Prm* prm;
    const double* ub; const int* ubn; const double* ex; const unsigned char* cert; const unsigned char* done;
    long long N; int m, e, k, mb; double floor_;
    ReplayState* rs; long long* list;
    double* out_d; long long* out_o;         // this length's k x m result
    int list_cap;                            // rows listed per stop
    long long win_min;                       // shortest listing window
};

__global__ void __launch_bounds__(32) k_pp_replay(ReplayArgs a) {
    __shared__ double cd[KMAX_CELLS];
    __shared__ long long co[KMAX_CELLS];
    const int lane = threadIdx.x;
    const int KM = a.k * a.mb;
    for (int t = lane; t < KM; t += 32) { cd[t] = a.rs->d[t]; co[t] = a.rs->o[t]; }
    __syncwarp();
    const double* last = cd + (a.k - 1) * a.mb;
    // the values an owner would offer, and whether they could change the matrix now
    auto values = [&](long long o, double* v, int& kind) {   // kind 0 skip, 1 exact, 2 certified, 3 stored
        kind = 0;
        if (!(a.prm[o].inv == a.prm[o].inv)) return;
        if (a.done[o]) { kind = 1; for (int c = 0; c < a.mb; ++c) v[c] = a.ex[o * a.mb + c]; if (!(v[a.mb - 1] < INFINITY)) kind = 0; }
        else { kind = a.cert[o] ? 2 : 3; for (int c = 0; c < a.mb; ++c) v[c] = a.ub[o * a.mb + c]; }
    };
    auto maybe = [&](const double* v, int kind) {
        if (kind == 0) return false;
        for (int c = 0; c < a.mb; ++c)
            if (kind == 1 ? v[c] > last[c] : v[c] * (1.0 + PP_MARGIN) > last[c]) return true;
        return false;
    };
    long long pos = a.rs->pos;
    int status = 2;
    while (pos < a.N) {
        const long long o = pos + lane;
        double v[MB_MAX]; int kind = 0;
        if (o < a.N) values(o, v, kind);
        unsigned bal = __ballot_sync(FULLMASK, maybe(v, kind));
        long long next = pos + 32;
        bool stop = false;
        while (bal) {
            const int src = __ffs(bal) - 1;
            bal &= bal - 1;
            const long long ov = pos + src;
            double w[MB_MAX]; int kw;
            values(ov, w, kw);                                      // warp-uniform
            if (!maybe(w, kw)) continue;                            // the last row moved past it
            bool triv = false;
            for (int t = lane; t < KM; t += 32) triv |= (co[t] >= 0 && llabs(ov - co[t]) < a.e);
            if (__any_sync(FULLMASK, triv)) continue;
            if (kw == 3) {                                          // needs its full row: stop here
                stop = true; next = ov;
                break;
            }
            if (kw == 2) {                                          // certified: canonical values
                double cv = INFINITY;
                if (lane < a.mb) {
                    const int j = a.ubn[ov * a.mb + lane];
                    if (j >= 0) cv = pair_distance(a.tn, a.cum, a.cum2, ov, j, a.m, a.floor_);
                }
                for (int c = 0; c < a.mb; ++c) w[c] = __shfl_sync(FULLMASK, cv, c);
                for (int q = 1; q < a.mb; ++q)
                    for (int r = q; r > 0 && w[r] < w[r - 1]; --r) { const double t = w[r]; w[r] = w[r - 1]; w[r - 1] = t; }
            }
            if (lane == 0) {                                        // columns m..1, rows top-down
                bool placed = false;
                for (int c = a.mb - 1; c >= 0 && !placed; --c) {
                    const double d = w[c];
                    for (int r = 0; r < a.k; ++r)
                        if (d > cd[r * a.mb + c]) {
                            for (int q = a.k - 1; q > r; --q) { cd[q * a.mb + c] = cd[(q - 1) * a.mb + c]; co[q * a.mb + c] = co[(q - 1) * a.mb + c]; }
                            cd[r * a.mb + c] = d; co[r * a.mb + c] = ov;
                            placed = true;
                            break;
                        }
                }
            }
            __syncwarp();
        }
        pos = next;
        if (stop) { status = 1; break; }
    }
    // list the rows to recompute: non-certified, not done, and able to matter now (a superset of
    // those the replay will stop at: the last row never decreases)
    int nl = 0;
    if (status == 1) {
        // every row of the window [pos, pos + max(win_min, pos)) that could matter at the current
        // last row: the last row only grows, so this is a superset of the window's stops, and the
        // windows double -- a length takes O(log N) stops (the running last row is low only near
        // the start of the series, where the windows are short)
        const long long wend = pos + (pos > a.win_min ? pos : a.win_min);
        for (long long b = pos; b < a.N && b < wend && nl < a.list_cap; b += 32) {
            const long long o = b + lane;
            double v[MB_MAX]; int kind = 0;
            if (o < a.N && o < wend) values(o, v, kind);
            const bool want = kind == 3 && maybe(v, kind);
            const unsigned bw = __ballot_sync(FULLMASK, want);
            const int at = nl + __popc(bw & ((1u << lane) - 1));
            if (want && at < a.list_cap) a.list[at] = o;
            nl += __popc(bw);
        }
        if (nl > a.list_cap) nl = a.list_cap;
    }
    for (int t = lane; t < KM; t += 32) {
        a.rs->d[t] = cd[t]; a.rs->o[t] = co[t];
        if (status == 2) { a.out_d[t] = cd[t]; a.out_o[t] = co[t]; }
    }
    if (lane == 0) { a.rs->pos = pos; a.rs->status = status; a.rs->nlist = nl; }
}

__global__ void k_pp_replay_init(ReplayState* rs, int km) {
    const int t = threadIdx.x;
    if (t < km) { rs->d[t] = -INFINITY; rs->o[t] = -1; }
    if (t == 0) { rs->pos = 0; rs->status = 0; rs->nlist = 0; }
}

// ---------------------------------------------------------------------------------
// full rows of the listed owners: every valid non-trivial cell's key from a centred direct dot
// product (owner window centred in shared memory; columns centred by mu_j S, S = sum of the
// centred owner window), the CTA's P smallest (key, j) with their co-moments
struct RowsArgs {
    const double* tn; const Prm* prm; const double* mu;
    const long long* list; long long N; int m, e, P, chunks;
    PPCand* cand;                                   // [slot][chunk][P]
};

__global__ void __launch_bounds__(RC_T) k_pp_rows(RowsArgs a) {
    extern __shared__ __align__(16) double smr[];
    const int slot = blockIdx.y, chunk = blockIdx.x, tid = threadIdx.x;
    const long long i = a.list[slot];
    const double io = a.prm[i].inv, mi = a.mu[i];
    double* xo = smr;                               // [m] centred owner window
    double* tw = smr + ((a.m + 1) & ~1);            // [RC_COLS + m] series segment
    __shared__ double red[RC_T / 32];
    __shared__ PPCand wc[RC_T / 32][PP_MAX];
    const long long c0 = (long long)chunk * RC_COLS;
    double ps = 0.0;
    for (int k = tid; k < a.m; k += RC_T) { const double x = a.tn[i + k] - mi; xo[k] = x; ps += x; }
    for (int k = tid; k < RC_COLS + a.m; k += RC_T) tw[k] = c0 + k < a.N + a.m - 1 ? a.tn[c0 + k] : 0.0;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) ps += __shfl_xor_sync(FULLMASK, ps, off);
    if ((tid & 31) == 0) red[tid >> 5] = ps;
    __syncthreads();
    double S = 0.0;
#pragma unroll
    for (int w = 0; w < RC_T / 32; ++w) S += red[w];
    // RC_R consecutive columns per thread: acc[r] = sum_k xo[k] t[j + r + k]
    const int jl = tid * RC_R;
    double acc[RC_R];
#pragma unroll
    for (int r = 0; r < RC_R; ++r) acc[r] = 0.0;
    int k = 0;
    for (; k + 8 <= a.m; k += 8) {
        double tv[RC_R + 8], xv[8];
#pragma unroll
        for (int u = 0; u < RC_R + 8; u += 2) { const double2 p = *reinterpret_cast<const double2*>(tw + jl + k + u); tv[u] = p.x; tv[u + 1] = p.y; }
#pragma unroll
        for (int u = 0; u < 8; u += 2) { const double2 p = *reinterpret_cast<const double2*>(xo + k + u); xv[u] = p.x; xv[u + 1] = p.y; }
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int r = 0; r < RC_R; ++r) acc[r] = fma(xv[u], tv[r + u], acc[r]);
    }
    for (; k < a.m; ++k)
#pragma unroll
        for (int r = 0; r < RC_R; ++r) acc[r] = fma(xo[k], tw[jl + r + k], acc[r]);
    // the thread's P smallest
    unsigned long long bk[PP_MAX]; long long bj[PP_MAX]; double bc[PP_MAX];
    for (int q = 0; q < PP_MAX; ++q) { bk[q] = KEY_NONE; bj[q] = IDX_NONE; bc[q] = 0.0; }
#pragma unroll
    for (int r = 0; r < RC_R; ++r) {
        const long long j = c0 + jl + r;
        if (j >= a.N) continue;
        const long long dd = j > i ? j - i : i - j;
        if (dd < a.e) continue;
        const double ij = a.prm[j].inv;
        if (!(ij == ij) || !(io == io)) continue;
        const double cv = acc[r] - a.mu[j] * S;
        unsigned long long key = clamp_key(fma(-(cv * io), ij, 1.0)) & ~PMASK;
        long long jj = j; double cc = cv;
        for (int q = 0; q < a.P; ++q)
            if (cand_less(key, jj, bk[q], bj[q])) {
                const unsigned long long tk = bk[q]; const long long tj = bj[q]; const double tc = bc[q];
                bk[q] = key; bj[q] = jj; bc[q] = cc; key = tk; jj = tj; cc = tc;
            }
    }
    // warp: P rounds of extract-min over the lanes' sorted lists
    const int lane = tid & 31, wid = tid >> 5;
    int head = 0;
    for (int q = 0; q < a.P; ++q) {
        unsigned long long hk = head < a.P ? bk[head] : KEY_NONE; long long hj = head < a.P ? bj[head] : IDX_NONE;
        unsigned long long mk = hk; long long mj = hj; int ml = lane;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            const unsigned long long ok2 = __shfl_xor_sync(FULLMASK, mk, off);
            const long long oj = __shfl_xor_sync(FULLMASK, mj, off);
            const int ol = __shfl_xor_sync(FULLMASK, ml, off);
            if (cand_less(ok2, oj, mk, mj) || (ok2 == mk && oj == mj && ol < ml)) { mk = ok2; mj = oj; ml = ol; }
        }
        const double mc = __shfl_sync(FULLMASK, head < a.P ? bc[head] : 0.0, ml);
        if (lane == ml) ++head;
        if (lane == 0) wc[wid][q] = PPCand{mk, mj, mc};
    }
    __syncthreads();
    if (wid == 0) {   // merge the warps' lists: lane w < 8 holds warp w's sorted list
        int h = 0;
        for (int q = 0; q < a.P; ++q) {
            unsigned long long mk = KEY_NONE; long long mj = IDX_NONE; int ml = lane;
            if (lane < RC_T / 32 && h < a.P) { mk = wc[lane][h].key; mj = wc[lane][h].j; }
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) {
                const unsigned long long ok2 = __shfl_xor_sync(FULLMASK, mk, off);
                const long long oj = __shfl_xor_sync(FULLMASK, mj, off);
                const int ol = __shfl_xor_sync(FULLMASK, ml, off);
                if (cand_less(ok2, oj, mk, mj) || (ok2 == mk && oj == mj && ol < ml)) { mk = ok2; mj = oj; ml = ol; }
            }
            double mc = 0.0;
            if (lane == ml && lane < RC_T / 32 && h < a.P) mc = wc[lane][h].cov;
            mc = __shfl_sync(FULLMASK, mc, ml);
            if (lane == ml) ++h;
            if (lane == 0) a.cand[((long long)slot * a.chunks + chunk) * a.P + q] = PPCand{mk, mj, mc};
        }
    }
}

// per listed row: the P best over its chunks -> refreshed stored entries (set_row at this length:
// neighbours, co-moments, m_f, sigma_base) and the exact canonical m best; one warp per row
struct MergeArgs {
    const double* tn; const double* cum; const double* cum2; const Prm* prm;
    const long long* list; const PPCand* cand; int chunks, P, mb, m; double floor_;
    int* nbr; double* cov; double* mf; double* sb; unsigned char* ok; double* ex; unsigned char* done;
};

__global__ void k_pp_rows_merge(MergeArgs a) {
    const int lane = threadIdx.x & 31;
    const int slot = blockIdx.x;
    const long long i = a.list[slot];
    const PPCand* c = a.cand + (long long)slot * a.chunks * a.P;
    // each lane: the P best of its chunks (sorted insertion), then P extract-min rounds
    unsigned long long bk[PP_MAX]; long long bj[PP_MAX]; double bc[PP_MAX];
    for (int q = 0; q < PP_MAX; ++q) { bk[q] = KEY_NONE; bj[q] = IDX_NONE; bc[q] = 0.0; }
    for (int ch = lane; ch < a.chunks; ch += 32)
        for (int q0 = 0; q0 < a.P; ++q0) {
            const PPCand v = c[(long long)ch * a.P + q0];
            if (v.j == IDX_NONE) break;
            unsigned long long key = v.key; long long jj = v.j; double cc = v.cov;
            for (int q = 0; q < a.P; ++q)
                if (cand_less(key, jj, bk[q], bj[q])) {
                    const unsigned long long tk = bk[q]; const long long tj = bj[q]; const double tc = bc[q];
                    bk[q] = key; bj[q] = jj; bc[q] = cc; key = tk; jj = tj; cc = tc;
                }
        }
    const double io = a.prm[i].inv;
    int head = 0, nvalid = 0;
    double fmax_ = 0.0;
    long long best[PP_MAX];
    for (int q = 0; q < a.P; ++q) {
        unsigned long long mk = head < a.P ? bk[head] : KEY_NONE; long long mj = head < a.P ? bj[head] : IDX_NONE;
        int ml = lane;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            const unsigned long long ok2 = __shfl_xor_sync(FULLMASK, mk, off);
            const long long oj = __shfl_xor_sync(FULLMASK, mj, off);
            const int ol = __shfl_xor_sync(FULLMASK, ml, off);
            if (cand_less(ok2, oj, mk, mj) || (ok2 == mk && oj == mj && ol < ml)) { mk = ok2; mj = oj; ml = ol; }
        }
        const double mc = __shfl_sync(FULLMASK, head < a.P ? bc[head] : 0.0, ml);
        if (lane == ml) ++head;
        best[q] = mj == IDX_NONE ? -1 : mj;
        if (lane == 0) {
            a.nbr[i * a.P + q] = (int)best[q];
            a.cov[i * a.P + q] = mc;
        }
        if (mj != IDX_NONE) {
            const double qq = mc * io * a.prm[mj].inv;
            const double qp = qq > 0.0 ? qq : 0.0;
            fmax_ = fmax(fmax_, sqrt((double)a.m * fmax(0.0, 1.0 - qp * qp)));
            ++nvalid;
        }
    }
    double v = INFINITY;
    if (lane < a.mb && best[lane < PP_MAX ? lane : 0] >= 0 && lane < a.P)
        v = pair_distance(a.tn, a.cum, a.cum2, i, best[lane], a.m, a.floor_);
    double vals[MB_MAX];
#pragma unroll
    for (int q = 0; q < MB_MAX; ++q) vals[q] = __shfl_sync(FULLMASK, v, q);
    if (lane == 0) {
        for (int q = 1; q < a.mb; ++q)
            for (int r = q; r > 0 && vals[r] < vals[r - 1]; --r) { const double t = vals[r]; vals[r] = vals[r - 1]; vals[r - 1] = t; }
        for (int q = 0; q < a.mb; ++q) a.ex[i * a.mb + q] = vals[q];
        a.mf[i] = nvalid == a.P ? fmax_ : 0.0;
        a.sb[i] = 1.0 / (io * sqrt((double)a.m));
        a.ok[i] = 1;
        a.done[i] = 1;
    }
}

// ---------------------------------------------------------------------------------
// Row blocks (m = 1): the replay's wanted rows come in clusters (the running k-th value is low
// at the start of the series; discord candidates sit around anomalies), so they are recomputed
// as blocks of consecutive rows [a, a + len), len <= PB_B: one centred FP64 direct sum per
// signed diagonal delta = j - i at the block's first row (the seed), then the FP64 diagonal
// recurrence (SCAMP form, as k_runs) down the block -- 2 N m + ~10 N len flops for len rows
// instead of len N m. One warp per CTA walks PB_W consecutive diagonals (8 per lane, a register
// ring of column parameters rotated by shuffles as in the tile walks); per row the warp's
// minimum packed key (key at 2^-44, low 8 bits = the diagonal within the chunk, so ties go to
// the smaller column) is folded into a shared per-row best, then one 128-bit CAS per row and
// CTA into racc. A cell whose recurrence magnitude (|seed| + sum |steps|, FP32 bound) exceeds
// 4 s_i s_j is recomputed directly and the carry restarts there (k_runs' rule, for <= 128 steps).
constexpr int PB_DL = 8;                    // diagonals per lane
constexpr int PB_W = 32 * PB_DL;            // diagonals per chunk (8-bit local index = PBITS)
constexpr int PB_B = 128;                   // rows per block
constexpr double PB_MAG = 4.0;              // recurrence magnitude limit (x s_i s_j): <= 2^-43 error
constexpr int LIST_CAP = 8192;              // rows listed per replay stop (m = 1)
constexpr int WIN_MIN = 2048;               // shortest listing window after a stop (rows)
static_assert(PB_W == BAND, "the packed local diagonal index uses PBITS bits");

struct BlockArgs {
    const double* tn; const Prm* prm; const double* mu;
    const PBlock* blk; long long N; int m, e, nchunks_max;
    ulonglong2* racc;                         // [block][PB_B]
};

struct PBSmem {
    double rdf[PB_B], rdg[PB_B], rinv[PB_B]; // the block's rows
    unsigned long long rk[PB_B]; long long rj[PB_B];   // per-row best of this CTA
};

__device__ __forceinline__ double pb_direct(const double* __restrict__ tn, const double* __restrict__ mu,
                                            long long i, long long j, int m) {
    const double mi = mu[i], mj = mu[j];
    double d = 0.0;
    for (int k = 0; k < m; ++k) d = fma(tn[i + k] - mi, tn[j + k] - mj, d);
    return d;
}

__global__ void __launch_bounds__(32) k_pp_block(BlockArgs a) {
    extern __shared__ __align__(16) double pbx[];    // [m] centred owner window, [PB_W + m + 16] segment
    __shared__ PBSmem sm;
    const int lane = threadIdx.x;
    const PBlock B = a.blk[blockIdx.y];
    const long long a0 = B.a;
    const int L = B.len;
    const int m = a.m;
    const long long dlo = -(a0 + L - 1);                     // lowest signed diagonal with a cell
    const long long dhi = a.N - 1 - a0;                      // highest
    const long long nch = (dhi - dlo + PB_W) / PB_W;
    double* xo = pbx;
    double* seg = pbx + ((m + 1) & ~1);
    const double mu_a = a.mu[a0];
    for (int r = lane; r < L; r += 32) {
        const Prm p = a.prm[a0 + r];
        sm.rdf[r] = p.df; sm.rdg[r] = p.dg; sm.rinv[r] = p.inv;
        sm.rk[r] = ~0ull; sm.rj[r] = IDX_NONE;
    }
    double ps = 0.0;
    for (int k = lane; k < m; k += 32) { const double x = a.tn[a0 + k] - mu_a; xo[k] = x; ps += x; }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) ps += __shfl_xor_sync(FULLMASK, ps, off);
    const double S = ps;                                     // sum of the centred owner window
    __syncwarp();
    for (long long ch = blockIdx.x; ch < nch; ch += gridDim.x) {
        const long long d0 = dlo + ch * PB_W;
        // chunk entirely inside the trivial zone (-e, e): nothing to do
        if (d0 > -(long long)a.e && d0 + PB_W - 1 < (long long)a.e) continue;
        const long long jb = a0 + d0;                         // column of diagonal d0 at row a0
        // segment t[jb .. jb + PB_W + m), shifted by c0 (local DC removal), 0 outside the series
        const long long lo = jb > 0 ? jb : 0;
        const double c0 = a.tn[lo];
        for (int k = lane; k < PB_W + m + 8; k += 32) {
            const long long g = jb + k;
            seg[k] = (g >= 0 && g < a.N + m - 1) ? a.tn[g] - c0 : 0.0;
        }
        __syncwarp();
        // seeds at row a0 for the lane's diagonals d0 + 8 lane + s (register-tiled direct sums)
        double acc[PB_DL];
#pragma unroll
        for (int s = 0; s < PB_DL; ++s) acc[s] = 0.0;
        const int jl = PB_DL * lane;
        int k = 0;
        for (; k + 8 <= m; k += 8) {
            double tv[PB_DL + 8], xv[8];
#pragma unroll
            for (int u = 0; u < PB_DL + 8; u += 2) { const double2 p = *reinterpret_cast<const double2*>(seg + jl + k + u); tv[u] = p.x; tv[u + 1] = p.y; }
#pragma unroll
            for (int u = 0; u < 8; u += 2) { const double2 p = *reinterpret_cast<const double2*>(xo + k + u); xv[u] = p.x; xv[u + 1] = p.y; }
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
                for (int s = 0; s < PB_DL; ++s) acc[s] = fma(xv[u], tv[s + u], acc[s]);
        }
        for (; k < m; ++k)
#pragma unroll
            for (int s = 0; s < PB_DL; ++s) acc[s] = fma(xo[k], seg[jl + s + k], acc[s]);
        // cov = sum x (t - c0) - (mu_j - c0) S; NaN for diagonals without a seed at row a0
        // (trivial, or entering the series later: seeded directly when they do)
        double cov[PB_DL], mag[PB_DL];
#pragma unroll
        for (int s = 0; s < PB_DL; ++s) {
            const long long dd = d0 + jl + s;
            const long long j = a0 + dd;
            const bool triv = dd > -(long long)a.e && dd < (long long)a.e;
            cov[s] = (!triv && j >= 0 && j < a.N) ? acc[s] - (a.mu[j] - c0) * S : __longlong_as_double(0x7FF8000000000000ll);
            mag[s] = fabs(cov[s]);
        }
        // column ring: slot s holds column j = i + d0 + 8 lane + s at row i (rotated by index)
        double cdf[PB_DL], cdg[PB_DL], cin[PB_DL];
#pragma unroll
        for (int s = 0; s < PB_DL; ++s) {
            const long long j = jb + jl + s;
            if (j >= 0 && j < a.N) { const Prm p = a.prm[j]; cdf[s] = p.df; cdg[s] = p.dg; cin[s] = p.inv; }
            else { cdf[s] = 0.0; cdg[s] = 0.0; cin[s] = __longlong_as_double(0x7FF8000000000000ll); }
        }
        for (int r0 = 0; r0 < L; r0 += PB_DL) {
#pragma unroll
            for (int q = 0; q < PB_DL; ++q) {
                const int r = r0 + q;
                if (r >= L) break;
                const long long i = a0 + r;
                const double fi = sm.rdf[r], gi = sm.rdg[r], ii = sm.rinv[r];
                if (r > 0) {
                    // rotate: the column leaving slot (q-1) mod 8 moves to lane-1; lane 31 loads
                    // the entering column i + d0 + 8*32 + 7 (the slot's new column)
                    const int ph = (q + PB_DL - 1) % PB_DL;
                    double nf = __shfl_down_sync(FULLMASK, cdf[ph], 1), ng = __shfl_down_sync(FULLMASK, cdg[ph], 1),
                           ni = __shfl_down_sync(FULLMASK, cin[ph], 1);
                    if (lane == 31) {
                        const long long j = i + d0 + PB_W - 1;
                        if (j >= 0 && j < a.N) { const Prm p = a.prm[j]; nf = p.df; ng = p.dg; ni = p.inv; }
                        else { nf = 0.0; ng = 0.0; ni = __longlong_as_double(0x7FF8000000000000ll); }
                    }
                    cdf[ph] = nf; cdg[ph] = ng; cin[ph] = ni;
                }
                unsigned long long best = ~0ull;
#pragma unroll
                for (int s = 0; s < PB_DL; ++s) {
                    const int p = (s + q) % PB_DL;           // slot of diagonal s at this row
                    const long long dd = d0 + jl + s;
                    const long long j = i + dd;
                    if (r > 0) {
                        const double term = fma(fi, cdg[p], cdf[p] * gi);
                        cov[s] += term;
                        mag[s] += fabs(term);
                        if (dd < 0 && j == 0) {                // the diagonal enters the series here
                            cov[s] = dd > -(long long)a.e ? __longlong_as_double(0x7FF8000000000000ll)
                                                          : pb_direct(a.tn, a.mu, i, j, m);
                            mag[s] = fabs(cov[s]);
                        }
                    }
                    const double g = ii * cin[p];             // 1 / (s_i s_j); NaN: invalid cell
                    if (mag[s] * g > PB_MAG && j >= 0 && j < a.N) {   // false for NaN
                        cov[s] = pb_direct(a.tn, a.mu, i, j, m);      // recurrence error could exceed 2^-44
                        mag[s] = fabs(cov[s]);
                    }
                    const double rr = fma(-cov[s], g, 1.0);
                    const unsigned long long key = (rr == rr) ? ((clamp_key(rr) & ~PMASK) | (unsigned long long)(jl + s)) : ~0ull;
                    best = key < best ? key : best;
                }
                // warp minimum of the packed keys: high words, then low words among the ties
                const unsigned hi = (unsigned)(best >> 32);
                const unsigned mh = __reduce_min_sync(FULLMASK, hi);
                const unsigned eq = __ballot_sync(FULLMASK, hi == mh);
                unsigned ml = 0xFFFFFFFFu;
                if (hi == mh) ml = __reduce_min_sync(eq, (unsigned)best);
                ml = __shfl_sync(FULLMASK, ml, __ffs(eq) - 1);
                if (lane == 0 && mh != 0xFFFFFFFFu) {
                    const unsigned long long pk = ((unsigned long long)mh << 32) | ml;
                    const unsigned long long kk = pk & ~PMASK;
                    const long long jj = i + d0 + (long long)(pk & PMASK);
                    if (kk < KEY_NONE && key_less(kk, jj, sm.rk[r], sm.rj[r])) { sm.rk[r] = kk; sm.rj[r] = jj; }
                }
            }
        }
        __syncwarp();
    }
    __syncwarp();
    for (int r = lane; r < L; r += 32)
        if (sm.rj[r] != IDX_NONE) acc_merge(a.racc + (long long)blockIdx.y * PB_B + r, sm.rk[r], sm.rj[r]);
}

// per block row: its exact nearest neighbour from racc -> refreshed stored entry (P = 1 of it:
// the co-moment by a direct sum, m_f = 0 so the row is not certified from it), the canonical
// distance (discords.py:126-141), done. One warp per row.
struct BFinArgs {
    const double* tn; const double* cum; const double* cum2; const Prm* prm; const double* mu;
    const PBlock* blk; const int* row_blk; int m, P; double floor_;
    const ulonglong2* racc; long long nrows;
    int* nbr; double* cov; double* mf; double* sb; unsigned char* ok; double* ex; unsigned char* done;
};

__global__ void k_pp_block_finish(BFinArgs a) {
    const int lane = threadIdx.x & 31;
    const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    if (w >= a.nrows) return;
    const int b = a.row_blk[w];
    const PBlock B = a.blk[b];
    const int r = (int)(w - a.row_blk[a.nrows + b]);          // row within the block
    const long long i = B.a + r;
    const ulonglong2 v = a.racc[(long long)b * PB_B + r];
    const double io = a.prm[i].inv;
    const bool have = io == io && v.y != (unsigned long long)IDX_NONE && v.x < KEY_NONE;
    const long long j = have ? (long long)v.y : -1;
    double c = 0.0;
    if (have) {
        const double mi = a.mu[i], mj = a.mu[j];
        for (int k = lane; k < a.m; k += 32) c = fma(a.tn[i + k] - mi, a.tn[j + k] - mj, c);
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) c += __shfl_xor_sync(FULLMASK, c, off);
    }
    for (int q = lane; q < a.P; q += 32) { a.nbr[i * a.P + q] = q == 0 ? (int)j : -1; if (q == 0) a.cov[i * a.P] = c; }
    if (lane == 0) {
        a.ex[i] = have ? pair_distance(a.tn, a.cum, a.cum2, i, j, a.m, a.floor_) : INFINITY;
        a.mf[i] = 0.0;
        a.sb[i] = io == io ? 1.0 / (io * sqrt((double)a.m)) : 0.0;
        a.ok[i] = io == io ? 1 : 0;
        a.done[i] = 1;
    }
}

__global__ void k_fill_racc(ulonglong2* p, long long n) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t < n) p[t] = make_ulonglong2(KEY_NONE, (unsigned long long)IDX_NONE);
}

// ---------------------------------------------------------------------------------
void pruned_free(vlmp_session* s) {
    PrunedState* p = s->pp;
    if (!p) return;
    void* ptrs[] = {p->nbr, p->cov, p->mf, p->sb, p->ok, p->ub, p->ubn, p->ex, p->cert, p->done, p->rs, p->list,
                    p->cand, p->cnt, p->blk, p->row_blk, p->racc};
    for (void* q : ptrs) if (q) cudaFree(q);
    if (p->h_rs) cudaFreeHost(p->h_rs);
    if (p->h_cnt) cudaFreeHost(p->h_cnt);
    if (p->h_list) cudaFreeHost(p->h_list);
    if (p->h_blk) cudaFreeHost(p->h_blk);
    if (p->h_row_blk) cudaFreeHost(p->h_row_blk);
    delete p;
    s->pp = nullptr;
}

static int pp_alloc(vlmp_session* s, long long rows, int P, int mb, int k) {
    if (!s->pp) s->pp = new PrunedState();
    PrunedState* p = s->pp;
    int rc;
    if ((size_t)rows * P > p->ent_cap) {
        if ((rc = ensure1(p->nbr, (size_t)rows * P))) return rc;
        if ((rc = ensure1(p->cov, (size_t)rows * P))) return rc;
        p->ent_cap = (size_t)rows * P;
    }
    if ((size_t)rows > p->row_cap) {
        if ((rc = ensure1(p->mf, rows))) return rc;
        if ((rc = ensure1(p->sb, rows))) return rc;
        if ((rc = ensure1(p->ok, rows))) return rc;
        if ((rc = ensure1(p->cert, rows))) return rc;
        if ((rc = ensure1(p->done, rows))) return rc;
        p->row_cap = rows;
    }
    if ((size_t)rows * mb > p->mrow_cap) {
        if ((rc = ensure1(p->ub, (size_t)rows * mb))) return rc;
        if ((rc = ensure1(p->ubn, (size_t)rows * mb))) return rc;
        if ((rc = ensure1(p->ex, (size_t)rows * mb))) return rc;
        p->mrow_cap = (size_t)rows * mb;
    }
    if (!p->rs) {
        CU(cudaMalloc((void**)&p->rs, sizeof(ReplayState)));
        CU(cudaMallocHost((void**)&p->h_rs, sizeof(ReplayState)));
        CU(cudaMalloc((void**)&p->list, LIST_CAP * sizeof(long long)));
        CU(cudaMallocHost((void**)&p->h_list, LIST_CAP * sizeof(long long)));
        CU(cudaMalloc((void**)&p->cnt, 4 * sizeof(unsigned long long)));
        CU(cudaMallocHost((void**)&p->h_cnt, 4 * sizeof(unsigned long long)));
        CU(cudaMalloc((void**)&p->blk, LIST_CAP * sizeof(PBlock)));
        CU(cudaMallocHost((void**)&p->h_blk, LIST_CAP * sizeof(PBlock)));
        CU(cudaMalloc((void**)&p->racc, (size_t)LIST_CAP * PB_B * sizeof(ulonglong2)));
    }
    const size_t rb = (size_t)std::min<long long>((long long)LIST_CAP * PB_B, rows) + LIST_CAP;
    if (rb > p->row_blk_cap) {
        if (p->h_row_blk) { cudaFreeHost(p->h_row_blk); p->h_row_blk = nullptr; }
        if ((rc = ensure1(p->row_blk, rb))) return rc;
        CU(cudaMallocHost((void**)&p->h_row_blk, rb * sizeof(int)));
        p->row_blk_cap = rb;
    }
    const long long chunks = (rows + RC_COLS - 1) / RC_COLS + 1;
    if ((size_t)(RBATCH * chunks * PP_MAX) > p->cand_cap) {
        if ((rc = ensure1(p->cand, (size_t)RBATCH * chunks * PP_MAX))) return rc;
        p->cand_cap = (size_t)RBATCH * chunks * PP_MAX;
    }
    p->rows = rows; p->P = P; p->mb = mb; p->k = k;
    return 0;
}

// exhaustive m-best pass at length m (all rows exact), stored entries harvested from it
static int pp_full_length(vlmp_session* s, int m, int P, int mb) {
    int rc;
    PrunedState* p = s->pp;
    cudaStream_t st = s->stream;
    const long long N = s->n - m + 1;
    const int* ipm;
    if (P == 1) {
        // m = 1 keeps one stored neighbour per row: the exhaustive 1-best pass (FP32 walk + exact
        // runs) gives it; its phase 2 leaves the neighbours in d_ip
        if ((rc = profile_locked(s, m, m))) return rc;
        if ((rc = finalize_lengths_locked(s, 0, 0))) return rc;
        launch_params(s, st, s->d_prm, s->d_mu, m);
        ipm = s->d_ip;
    } else {
        // mbest_impl leaves this length's window parameters in d_prm / d_mu
        if ((rc = mbest_impl(s, m, m, P))) return rc;
        ipm = s->d_ipm;
    }
    HarvestArgs ha{s->d_tn, s->d_cum, s->d_cum2, s->d_prm, s->d_mu, ipm, N, m, P, mb, s->floor_,
                   p->nbr, p->cov, p->mf, p->sb, p->ok, p->ex, p->done, p->cert};
    k_pp_harvest<<<blocks(N * 32, 256), 256, 0, st>>>(ha);
    CU(cudaGetLastError());
    return 0;
}

static double host_seconds() {
    timespec ts; clock_gettime(CLOCK_MONOTONIC, &ts); return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

// modelled cost (seconds on one B200) of an exhaustive pass at one length and of one row block:
// the budget that decides when a length falls back to the full pass
static double full_cost(long long N) { return 0.5 * (double)N * (double)N / 5.5e12 + 2e-3; }
static double block_cost(long long N, int m, int len) {
    return 2.0 * (double)N * (double)m / 5e12 + 2.0 * (double)N * len / 2.0e12 + 20e-6;
}

// m = 1: group the listed rows (ascending) into blocks [a, a + len), len <= PB_B, a block taking
// every listed row inside its window (unlisted rows in between are recomputed too: a row costs
// a walk step, a new block a seed per diagonal); returns the number of blocks and rows
static void make_blocks(const long long* list, int nl, long long N, PBlock* blk, int* row_blk, int& nblk,
                        long long& nrows) {
    nblk = 0; nrows = 0;
    int q = 0;
    while (q < nl) {
        const long long a0 = list[q];
        long long last = a0;
        while (q < nl && list[q] < a0 + PB_B && list[q] < N) { last = list[q]; ++q; }
        if (a0 >= N) break;
        blk[nblk] = PBlock{a0, (int)(last - a0 + 1), 0};
        nrows += last - a0 + 1;
        ++nblk;
    }
    // row -> block map: [0, nrows) block of each row, [nrows, nrows + nblk) first row index of each block
    long long w = 0;
    for (int b = 0; b < nblk; ++b) {
        row_blk[nrows + b] = (int)w;
        for (int r = 0; r < blk[b].len; ++r) row_blk[w++] = b;
    }
}

// replay one length to completion, recomputing full rows on demand; *rows_out = rows recomputed,
// *gave_up = the modelled cost of the recomputes passed the budget (the caller falls back to a
// full pass), *stops = replay stops
static int pp_replay_length(vlmp_session* s, int m, const Prm* prm, const double* mu, double budget_s,
                            double* out_d, long long* out_o, long long* rows_out, bool* gave_up, int* stops) {
    PrunedState* p = s->pp;
    cudaStream_t st = s->stream;
    const long long N = s->n - m + 1;
    const int e = (m + 1) / 2;
    const bool blocks_path = p->mb == 1;
    k_pp_replay_init<<<1, KMAX_CELLS, 0, st>>>(p->rs, p->k * p->mb);
    ReplayArgs ra{s->d_tn, s->d_cum, s->d_cum2, prm, p->ub, p->ubn, p->ex, p->cert, p->done, N, m, e, p->k, p->mb,
                  s->floor_, p->rs, p->list, out_d, out_o, blocks_path ? LIST_CAP : RBATCH, (long long)WIN_MIN};
    const int chunks = (int)((N + RC_COLS - 1) / RC_COLS);
    const size_t smem = ((size_t)((m + 1) & ~1) + RC_COLS + m + 8) * sizeof(double);
    const size_t bsmem = ((size_t)((m + 1) & ~1) + PB_W + m + 16) * sizeof(double);
    if (blocks_path && bsmem + sizeof(PBSmem) > 227 * 1024)
        return fail(VLMP_E_INVALID_PARAMETERS, "pruned scan: window length too large for a row block's shared memory");
    if (blocks_path) CU(cudaFuncSetAttribute(k_pp_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem));
    else CU(cudaFuncSetAttribute(k_pp_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    *rows_out = 0; *gave_up = false; *stops = 0;
    double spent = 0.0;
    for (;;) {
        k_pp_replay<<<1, 32, 0, st>>>(ra);
        CU(cudaMemcpyAsync(p->h_rs, p->rs, offsetof(ReplayState, d), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if (p->h_rs->status == 2) return 0;
        const int nl = p->h_rs->nlist;
        if (nl <= 0) return fail(VLMP_E_CUDA, "pruned replay stopped without rows to recompute");
        ++*stops;
        if (!blocks_path) {
            if (spent + nl * block_cost(N, m, 1) * (double)m / 8.0 > budget_s) { *gave_up = true; return 0; }
            spent += nl * block_cost(N, m, 1) * (double)m / 8.0;
            *rows_out += nl;
            RowsArgs wa{s->d_tn, prm, mu, p->list, N, m, e, p->P, chunks, p->cand};
            k_pp_rows<<<dim3(chunks, nl), RC_T, smem, st>>>(wa);
            MergeArgs ma{s->d_tn, s->d_cum, s->d_cum2, prm, p->list, p->cand, chunks, p->P, p->mb, m, s->floor_,
                         p->nbr, p->cov, p->mf, p->sb, p->ok, p->ex, p->done};
            k_pp_rows_merge<<<nl, 32, 0, st>>>(ma);
            CU(cudaGetLastError());
            continue;
        }
        CU(cudaMemcpyAsync(p->h_list, p->list, nl * sizeof(long long), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        int nblk = 0; long long nrows = 0;
        make_blocks(p->h_list, nl, N, p->h_blk, p->h_row_blk, nblk, nrows);
        p->dbg_blocks += nblk;
        double cost = 0.0;
        for (int b = 0; b < nblk; ++b) cost += block_cost(N, m, p->h_blk[b].len);
        if (spent + cost > budget_s) { *gave_up = true; return 0; }
        spent += cost;
        *rows_out += nrows;
        CU(cudaMemcpyAsync(p->blk, p->h_blk, nblk * sizeof(PBlock), cudaMemcpyHostToDevice, st));
        CU(cudaMemcpyAsync(p->row_blk, p->h_row_blk, (nrows + nblk) * sizeof(int), cudaMemcpyHostToDevice, st));
        k_fill_racc<<<blocks((long long)nblk * PB_B, 256), 256, 0, st>>>(p->racc, (long long)nblk * PB_B);
        const long long nch = (N + PB_B + PB_W) / PB_W;
        const long long want_ctas = 148LL * 16;
        const unsigned G = (unsigned)std::max<long long>(1, std::min<long long>(nch, (want_ctas + nblk - 1) / nblk));
        BlockArgs ba{s->d_tn, prm, mu, p->blk, N, m, e, (int)nch, p->racc};
        k_pp_block<<<dim3(G, nblk), 32, bsmem, st>>>(ba);
        BFinArgs fa{s->d_tn, s->d_cum, s->d_cum2, prm, mu, p->blk, p->row_blk, m, p->P, s->floor_, p->racc, nrows,
                    p->nbr, p->cov, p->mf, p->sb, p->ok, p->ex, p->done};
        k_pp_block_finish<<<blocks(nrows * 32, 256), 256, 0, st>>>(fa);
        CU(cudaGetLastError());
    }
}

// mbest_impl's finalize leaves the canonical values in d_mpm: the first length's result is the
// exhaustive replay on them (k_discords_m needs P == mb there; our replay reads ex instead)
int pruned_impl(vlmp_session* s, int lmin, int lmax, int k, int mb, int P, double* out_d, long long* out_o,
                double* counters) {
    const int n_len = lmax - lmin + 1;
    const long long rows = s->n - lmin + 1, A = s->A;
    int rc;
    if ((rc = pp_alloc(s, rows, P, mb, k))) return rc;
    PrunedState* p = s->pp;
    cudaStream_t st = s->stream;
    double* d_out = nullptr; long long* o_out = nullptr;
    const size_t cells = (size_t)n_len * k * mb;
    CU(cudaMalloc((void**)&d_out, cells * sizeof(double)));
    CU(cudaMalloc((void**)&o_out, cells * sizeof(long long)));
    auto cleanup = [&]() { cudaFree(d_out); cudaFree(o_out); };
    cudaEvent_t e0 = s->ev[2], e1 = s->ev[3];
    CU(cudaEventRecord(e0, st));
    long long full_lengths = 0;
    // VLMP_PRUNED_BUDGET: scale of the recompute budget (diagnostics: a large value never falls back)
    const char* bs_env = getenv("VLMP_PRUNED_BUDGET");
    const double budget_scale = bs_env ? atof(bs_env) : 1.0;
    const bool dbg = getenv("VLMP_PRUNED_DEBUG") != nullptr;
    for (int li = 0; li < n_len; ++li) {
        const int m = lmin + li;
        const long long N = s->n - m + 1;
        long long nrec = 0;
        int stops = 0;
        bool full = li == 0, gave_up = false;
        p->dbg_blocks = 0;
        const double t_len0 = dbg ? host_seconds() : 0.0;
        CU(cudaMemsetAsync(p->cnt, 0, 4 * sizeof(unsigned long long), st));
        if (!full) {
            // this length's window parameters (ping-pong with the previous length's means)
            Prm* prm = (li & 1) ? s->d_prm2 : s->d_prm;
            double* mu = (li & 1) ? s->d_mu2 : s->d_mu;
            const double* mu_prev = (li & 1) ? s->d_mu : s->d_mu2;
            launch_params(s, st, prm, mu, m);
            AdvanceArgs aa{s->d_tn, prm, mu_prev, rows, N, s->n, m, (m + 1) / 2, P, mb, p->nbr, p->cov, p->mf,
                           p->sb, p->ok, p->ub, p->ubn, p->cert, p->done, p->cnt};
            k_pp_advance<<<blocks(rows, 256), 256, 0, st>>>(aa);
            if ((rc = pp_replay_length(s, m, prm, mu, budget_scale * full_cost(N), d_out + (size_t)li * k * mb,
                                       o_out + (size_t)li * k * mb, &nrec, &gave_up, &stops))) { cleanup(); return rc; }
            if (gave_up) full = true;
        }
        if (full) {
            if ((rc = pp_full_length(s, m, P, mb))) { cleanup(); return rc; }
            bool dummy = false; long long r0 = 0; int st0 = 0;
            if ((rc = pp_replay_length(s, m, s->d_prm, s->d_mu, 0.0, d_out + (size_t)li * k * mb,
                                       o_out + (size_t)li * k * mb, &r0, &dummy, &st0))) { cleanup(); return rc; }
            ++full_lengths;
            // the next length reads these means as the previous length's: keep the ping-pong parity
            if (li & 1) {
                CU(cudaMemcpyAsync(s->d_prm2, s->d_prm, A * sizeof(Prm), cudaMemcpyDeviceToDevice, st));
                CU(cudaMemcpyAsync(s->d_mu2, s->d_mu, A * sizeof(double), cudaMemcpyDeviceToDevice, st));
            }
        }
        CU(cudaMemcpyAsync(p->h_cnt, p->cnt, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if (dbg)
            fprintf(stderr, "pruned length %d: %s stops %d blocks %lld rows %lld  %.2f ms\n", m, full ? "FULL" : "pruned",
                    stops, p->dbg_blocks, nrec, 1e3 * (host_seconds() - t_len0));
        if (counters) {
            double* c = counters + (size_t)li * 4;
            c[0] = full ? (double)N : (double)p->h_cnt[0];     // certified (or exact) rows
            c[1] = full ? 0.0 : (double)p->h_cnt[1];           // non-certified live rows
            c[2] = (double)nrec;                               // full rows recomputed
            c[3] = full ? 1.0 : 0.0;                           // exhaustive pass at this length
        }
    }
    CU(cudaEventRecord(e1, st));
    CU(cudaMemcpyAsync(out_d, d_out, cells * sizeof(double), cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(out_o, o_out, cells * sizeof(long long), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    cleanup();
    memset(s->stats, 0, sizeof(s->stats));
    s->stats[0] = ms; s->stats[7] = (double)full_lengths;
    s->stats_dirty = false;
    s->mbest = 0;                    // d_ipm / d_mpm now hold the last full length only
    // the 1-best buffers describe one fallback length, not a profile of [lmin, lmax]: read-offs
    // of the session's profile state must not pick them up
    s->have_profile = false; s->have_final = false; s->have_finals = false;
    return 0;
}

}  // namespace vlmp_impl

extern "C" {

int vlmp_discords_pruned(vlmp_session* s, int32_t lmin, int32_t lmax, int32_t k, int32_t m, int32_t p,
                         double* out_dist, int64_t* out_off, double* counters) {
    if (!s || !out_dist || !out_off) return fail(VLMP_E_INVALID_PARAMETERS, "null argument");
    if (s->n <= 0) return fail(VLMP_E_STATE, "no series uploaded");
    if (lmin > lmax || lmin < 4) return fail(VLMP_E_INVALID_PARAMETERS, "bad length range");
    if (k < 1 || k > 32 || m < 1 || m > MB_MAX) return fail(VLMP_E_INVALID_PARAMETERS, "k in [1, 32], m in [1, 8]");
    if (p < m) return fail(VLMP_E_INVALID_PARAMETERS, "p must be at least m");
    if (s->n < (long long)lmax + (lmax + 1) / 2)
        return fail(VLMP_E_SERIES_TOO_SHORT, "series cannot host a non-trivial pair at lmax");
    // m = 1: one stored neighbour per row (its exact distance carried from length to length is the
    // row's upper bound; rows whose bound can matter are recomputed in blocks); m > 1: P <= 8
    const int P = m == 1 ? 1 : std::min(PP_MAX, std::max(p, m));
    std::lock_guard<std::mutex> g(s->lock);
    CU(cudaSetDevice(s->device));
    { const int rc = settle_profile(s, nullptr); if (rc) return rc; }
    return pruned_impl(s, lmin, lmax, k, m, P, out_dist, reinterpret_cast<long long*>(out_off), counters);
}

}  // extern "C"
