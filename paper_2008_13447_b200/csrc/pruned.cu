// pruned.cu -- MAD's pruned top-k m-th discord scan on the GPU (the reference's
// topkm_discord_discovery / topkm_next_length, discords.py:144-247, over its partial profiles,
// profile.py:66-232): exact like the exhaustive path, but most rows never get a full profile.
//
// Per row the scan keeps P <= 8 stored neighbours (the reference keeps p; `PartialProfiles`):
//   * at lmin (and after any full fallback length) the stored set is the row's P best cells of the
//     exhaustive m-best profile (the P smallest bound factors f = sqrt(l (1 - max(q,0)^2)) are the
//     P largest correlations, `_harvest_select`), their centred co-moments C (direct sums),
//     m_f = max f over them and sigma_base = the row's sigma at that length;
//   * each later length advances every stored co-moment by the Welford step
//     C_{l+1} = C_l + l/(l+1) (x_l - mu_x)(y_l - mu_y)  (O(1), `PartialProfiles.advance`), drops
//     entries whose neighbour left the series, turned constant or became trivial, and certifies
//     the row when its m-th stored distance is below m_f sigma_base / sigma_l (VALMOD's Eq. 2:
//     no unstored pair can be closer -- `thresholds`, `certify_step`).
// The replay (one warp, `update_fixed_length_discords` in ascending offsets) takes certified rows'
// stored m best (canonical values, discords.py:126-141), skips a non-certified row whose stored
// distances (upper bounds of its true m best) beat no cell of the matrix's last row (discords.py:
// 176-181), and stops at the first non-certified row it cannot skip: the host then recomputes a
// batch of full rows -- that row and the following non-certified rows that could still matter
// (the last row of the matrix never decreases, so that set is a superset) -- refreshes their
// stored entries at this length (`set_row`) and resumes the replay. A length whose recomputes
// would cost more than an exhaustive pass runs the exhaustive m-best profile instead and
// re-harvests every row (VALMOD's full recompute).
#include "vlmp_internal.cuh"

namespace vlmp_impl {

constexpr int PP_MAX = MB_MAX;        // stored entries per row
constexpr int RBATCH = 64;            // full rows recomputed per replay stop (at most)
constexpr int RC_T = 256;             // threads of a full-row CTA
constexpr int RC_R = 8;               // columns per thread
constexpr int RC_COLS = RC_T * RC_R;  // columns per CTA
constexpr int KMAX_CELLS = 32 * MB_MAX;
constexpr double PP_MARGIN = 1e-9;    // approximate values vs exact decisions

struct PPCand { unsigned long long key; long long j; double cov; };

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
        for (long long b = pos; b < a.N && nl < RBATCH; b += 32) {
            const long long o = b + lane;
            double v[MB_MAX]; int kind = 0;
            if (o < a.N) values(o, v, kind);
            const bool want = kind == 3 && maybe(v, kind);
            const unsigned bw = __ballot_sync(FULLMASK, want);
            const int at = nl + __popc(bw & ((1u << lane) - 1));
            if (want && at < RBATCH) a.list[at] = o;
            nl += __popc(bw);
        }
        if (nl > RBATCH) nl = RBATCH;
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
void pruned_free(vlmp_session* s) {
    PrunedState* p = s->pp;
    if (!p) return;
    void* ptrs[] = {p->nbr, p->cov, p->mf, p->sb, p->ok, p->ub, p->ubn, p->ex, p->cert, p->done, p->rs, p->list,
                    p->cand, p->cnt};
    for (void* q : ptrs) if (q) cudaFree(q);
    if (p->h_rs) cudaFreeHost(p->h_rs);
    if (p->h_cnt) cudaFreeHost(p->h_cnt);
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
        CU(cudaMalloc((void**)&p->list, RBATCH * sizeof(long long)));
        CU(cudaMalloc((void**)&p->cnt, 4 * sizeof(unsigned long long)));
        CU(cudaMallocHost((void**)&p->h_cnt, 4 * sizeof(unsigned long long)));
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
    if ((rc = mbest_impl(s, m, m, P))) return rc;
    PrunedState* p = s->pp;
    cudaStream_t st = s->stream;
    const long long N = s->n - m + 1;
    // mbest_impl left this length's window parameters in d_prm / d_mu
    HarvestArgs ha{s->d_tn, s->d_cum, s->d_cum2, s->d_prm, s->d_mu, s->d_ipm, N, m, P, mb, s->floor_,
                   p->nbr, p->cov, p->mf, p->sb, p->ok, p->ex, p->done, p->cert};
    k_pp_harvest<<<blocks(N * 32, 256), 256, 0, st>>>(ha);
    CU(cudaGetLastError());
    return 0;
}

// replay one length to completion, recomputing full rows on demand; *rows_out = rows recomputed,
// *gave_up = the budget of recomputed rows ran out (the caller falls back to a full pass)
static int pp_replay_length(vlmp_session* s, int m, const Prm* prm, const double* mu, long long row_budget,
                            double* out_d, long long* out_o, long long* rows_out, bool* gave_up) {
    PrunedState* p = s->pp;
    cudaStream_t st = s->stream;
    const long long N = s->n - m + 1;
    const int e = (m + 1) / 2;
    k_pp_replay_init<<<1, KMAX_CELLS, 0, st>>>(p->rs, p->k * p->mb);
    ReplayArgs ra{s->d_tn, s->d_cum, s->d_cum2, prm, p->ub, p->ubn, p->ex, p->cert, p->done, N, m, e, p->k, p->mb,
                  s->floor_, p->rs, p->list, out_d, out_o};
    const int chunks = (int)((N + RC_COLS - 1) / RC_COLS);
    const size_t smem = ((size_t)((m + 1) & ~1) + RC_COLS + m + 8) * sizeof(double);
    CU(cudaFuncSetAttribute(k_pp_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    *rows_out = 0; *gave_up = false;
    for (;;) {
        k_pp_replay<<<1, 32, 0, st>>>(ra);
        CU(cudaMemcpyAsync(p->h_rs, p->rs, offsetof(ReplayState, d), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if (p->h_rs->status == 2) return 0;
        const int nl = p->h_rs->nlist;
        if (nl <= 0) return fail(VLMP_E_CUDA, "pruned replay stopped without rows to recompute");
        if (*rows_out + nl > row_budget) { *gave_up = true; return 0; }
        *rows_out += nl;
        RowsArgs wa{s->d_tn, prm, mu, p->list, N, m, e, p->P, chunks, p->cand};
        k_pp_rows<<<dim3(chunks, nl), RC_T, smem, st>>>(wa);
        MergeArgs ma{s->d_tn, s->d_cum, s->d_cum2, prm, p->list, p->cand, chunks, p->P, p->mb, m, s->floor_,
                     p->nbr, p->cov, p->mf, p->sb, p->ok, p->ex, p->done};
        k_pp_rows_merge<<<nl, 32, 0, st>>>(ma);
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
    for (int li = 0; li < n_len; ++li) {
        const int m = lmin + li;
        const long long N = s->n - m + 1;
        // a full row costs ~N m FP64 FMA, an exhaustive m-best length ~N^2/2 cells at a few FP32
        // FMA each: past ~N / (4 m) recomputed rows the exhaustive pass is cheaper
        const long long budget = std::max<long long>(RBATCH, N / (4LL * m));
        long long nrec = 0;
        bool full = li == 0, gave_up = false;
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
            if ((rc = pp_replay_length(s, m, prm, mu, budget, d_out + (size_t)li * k * mb, o_out + (size_t)li * k * mb,
                                       &nrec, &gave_up))) { cleanup(); return rc; }
            if (gave_up) full = true;
        }
        if (full) {
            if ((rc = pp_full_length(s, m, P, mb))) { cleanup(); return rc; }
            bool dummy = false; long long r0 = 0;
            if ((rc = pp_replay_length(s, m, s->d_prm, s->d_mu, 0, d_out + (size_t)li * k * mb,
                                       o_out + (size_t)li * k * mb, &r0, &dummy))) { cleanup(); return rc; }
            ++full_lengths;
            // the next length reads these means as the previous length's: keep the ping-pong parity
            if (li & 1) {
                CU(cudaMemcpyAsync(s->d_prm2, s->d_prm, A * sizeof(Prm), cudaMemcpyDeviceToDevice, st));
                CU(cudaMemcpyAsync(s->d_mu2, s->d_mu, A * sizeof(double), cudaMemcpyDeviceToDevice, st));
            }
        }
        CU(cudaMemcpyAsync(p->h_cnt, p->cnt, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
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
    const int P = std::min(PP_MAX, std::max(p, m));
    std::lock_guard<std::mutex> g(s->lock);
    CU(cudaSetDevice(s->device));
    { const int rc = settle_profile(s, nullptr); if (rc) return rc; }
    return pruned_impl(s, lmin, lmax, k, m, P, out_dist, reinterpret_cast<long long*>(out_off), counters);
}

}  // extern "C"
