// readout.cu -- phase 2 of libvlmp: exact profile values of the per-length winners and the
// read-offs built on them (VALMP, smallest rows, discords, ranking events, motif-set range
// queries). Kernels: k_finalize_walk, k_valmp, k_smallest, k_discords, k_range_query, k_events.
#include "vlmp_internal.cuh"

namespace vlmp_impl {

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
// gridDim.y chunks of lengths per offset (more threads in flight); a chunk's first pair sums
// from scratch, which is the same sequential sum the incremental path extends
__global__ void k_finalize_walk(FinArgs a) {
    const long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (o >= a.n - a.lmin + 1) return;
    long long pa = -1, pb = -1; int pm = -1;
    double qt = 0.0;
    const int l0 = (int)((long long)a.n_len * blockIdx.y / gridDim.y);
    const int l1 = (int)((long long)a.n_len * (blockIdx.y + 1) / gridDim.y);
    for (int li = l0; li < l1; ++li) {
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
    // holds list entry r (sorted descending), 32 chunks of the profile are loaded ahead
    const int lane = threadIdx.x & 31;
    const int li = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (li >= a.n_len) return;
    const int m = a.lmin + li;
    const long long N = a.n - m + 1;
    const long long e = (m + 1) / 2;
    const double* mp = a.mp + (long long)li * a.A;
    constexpr int AHEAD = 32;
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
            double thr = __shfl_sync(FULLMASK, cd, k - 1);
            const double d = dv8[u];
            const long long ol = base + 32 * u + lane;
            unsigned bal = __ballot_sync(FULLMASK, (d < INFINITY) && (d > thr));
            while (bal) {
                // every pending candidate against the current list at once: those below the
                // first non-trivial one are trivial matches of an unchanged list (rejected as
                // in the sequential replay); the rest are re-checked after each insertion
                bool triv = false;
                for (int r = 0; r < k; ++r) {
                    const long long cr = __shfl_sync(FULLMASK, co, r);
                    triv |= cr >= 0 && llabs(ol - cr) < e;
                }
                const unsigned live = bal & __ballot_sync(FULLMASK, !triv);
                if (!live) break;
                const int src = __ffs(live) - 1;
                bal &= ~((2u << src) - 1u);          // src and every (trivial) candidate before it
                const double dv = __shfl_sync(FULLMASK, d, src);
                const long long ov = base + 32 * u + src;
                const bool mine = lane < k;
                // before the first strictly smaller entry
                const int at = __popc(__ballot_sync(FULLMASK, mine && !(dv > cd)));
                if (at < k) {
                    const double ud = __shfl_up_sync(FULLMASK, cd, 1);
                    const long long uo = __shfl_up_sync(FULLMASK, co, 1);
                    if (mine && lane > at) { cd = ud; co = uo; }
                    if (lane == at) { cd = dv; co = ov; }
                    thr = __shfl_sync(FULLMASK, cd, k - 1);
                    bal &= __ballot_sync(FULLMASK, d > thr);
                }
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

// One full row from scratch (profile.py:263-269 row_profile -> _row_arrays :235-260): dot
// products qt_j = sum_k t[i+k] t[j+k] (direct FP64; the reference uses FFT correlation, within
// ~1e-11), window statistics as moving_stats, then the owner-first distance and bound factor in
// numpy's operation order; trivial cells and constant neighbours are +inf. One thread per column,
// the owner window staged in shared memory.
struct RowArgs {
    const double* tn; const double* cum; const double* cum2;
    long long n, i; int m; double floor_;
    double* dist; double* f; double* qt;
};

__global__ void k_row_profile(RowArgs a) {
    extern __shared__ double xo[];
    for (int k = threadIdx.x; k < a.m; k += blockDim.x) xo[k] = a.tn[a.i + k];
    __syncthreads();
    const long long N = a.n - a.m + 1;
    const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (j >= N) return;
    double qt = 0.0;
    for (int k = 0; k < a.m; ++k) qt = fma(xo[k], a.tn[j + k], qt);
    double mui, sdi, muj, sdj;
    win_stats(a.cum, a.cum2, a.i, a.m, mui, sdi);
    win_stats(a.cum, a.cum2, j, a.m, muj, sdj);
    const long long e = (a.m + 1) / 2;
    const long long lo = a.i - e + 1 > 0 ? a.i - e + 1 : 0, hi = a.i + e < N ? a.i + e : N;
    const bool bad = !(sdj >= a.floor_) || (j >= lo && j < hi);
    const double L = (double)a.m;
    const double q = __ddiv_rn(__dsub_rn(qt, __dmul_rn(__dmul_rn(L, mui), muj)), __dmul_rn(__dmul_rn(L, sdi), sdj));
    double rad = __dmul_rn(__dmul_rn(2.0, L), __dsub_rn(1.0, q));
    if (rad < 0.0) rad = 0.0;                    // np.maximum(rad, 0): NaN stays NaN
    a.dist[j] = bad ? INFINITY : __dsqrt_rn(rad);
    if (a.f) {
        double qc = q < -1.0 ? -1.0 : (q > 1.0 ? 1.0 : q);   // np.clip (NaN stays NaN)
        if (qc < 0.0) qc = 0.0;
        a.f[j] = bad ? INFINITY : __dsqrt_rn(__dmul_rn(L, __dsub_rn(1.0, __dmul_rn(qc, qc))));
    }
    if (a.qt) a.qt[j] = qt;
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


}  // namespace vlmp_impl

extern "C" {

static int finalize_enqueue(vlmp_session* s, int li_lo, int li_hi, bool readoffs);

static int finalize_impl(vlmp_session* s, int li_lo, int li_hi, bool readoffs) {
    CU(cudaSetDevice(s->device));
    // phase 2 is enqueued behind a still-unchecked phase 1 (no host sync between them); if the
    // check then redoes phase 1, phase 2 is enqueued again behind the redo
    for (int attempt = 0; attempt < 2; ++attempt) {
        int rc = finalize_enqueue(s, li_lo, li_hi, readoffs);
        if (rc) return rc;
        bool redone = false;
        if ((rc = settle_profile(s, &redone))) return rc;
        if (!redone) break;
    }
    CU(cudaEventSynchronize(s->ev[5]));
    s->stats[9] += (li_lo <= li_hi ? 1 : 0) + (readoffs ? 1 : 0);
    s->have_final = readoffs;
    s->have_finals = true;
    s->stats_dirty = true;
    return 0;
}

static int finalize_enqueue(vlmp_session* s, int li_lo, int li_hi, bool readoffs) {
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
        const unsigned chunks = (unsigned)std::min(8, std::max(1, s->n_len / 8));
        k_finalize_walk<<<dim3(blocks(n0, 64), chunks), 64, 0, st>>>(fa);
    }
    if (readoffs) {
        ValmpArgs va{s->d_mp, s->d_ip, s->d_vdist, s->d_vnorm, s->d_vlen, s->d_vidx, s->d_vpop, n, A, s->lmin, s->n_len};
        k_valmp<<<blocks(n0, 256), 256, 0, st>>>(va);
    }
    CU(cudaEventRecord(s->ev[5], st));
    CU(cudaGetLastError());
    return 0;
}

}  // extern "C"

namespace vlmp_impl {
// phase 2 of lengths li_lo..li_hi with the session lock held (pruned.cu's full lengths)
int finalize_lengths_locked(vlmp_session* s, int li_lo, int li_hi) { return finalize_impl(s, li_lo, li_hi, false); }
}  // namespace vlmp_impl

extern "C" {

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

// vlmp_finalize_collect: phase 2 and the standard read-offs enqueued behind phase 1 in one go,
// copied into pinned staging, one host wait. Staging layout (8-byte words, then the VALMP
// populated bytes): rows off / nbr / d [cr each], discords d / off [cd each], valmp dist /
// norm / len / idx [n0 each], pop [n0 bytes].
static int collect_enqueue(vlmp_session* s, int k2, int k, bool want_v, int end_event, long long cr, long long cd,
                           long long n0) {
    int rc = finalize_enqueue(s, 0, s->n_len - 1, true);
    if (rc) return rc;
    cudaStream_t st = s->stream;
    long long* i64 = s->d_ro_i64; double* f64 = s->d_ro_f64;
    unsigned char* h = s->h_col;
    long long* h8 = reinterpret_cast<long long*>(h);
    if (k2) {
        SmallArgs sa{s->d_mp, s->d_ip, i64, i64 + cr, f64, s->n, s->A, s->lmin, k2};
        k_smallest<<<s->n_len, 256, 0, st>>>(sa);
        CU(cudaMemcpyAsync(h8, i64, 2 * cr * 8, cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(h8 + 2 * cr, f64, cr * 8, cudaMemcpyDeviceToHost, st));
    }
    if (k) {
        DiscArgs da{s->d_mp, f64 + cr, i64 + 2 * cr, s->n, s->A, s->lmin, s->n_len, k};
        k_discords<<<s->n_len, 32, 0, st>>>(da);
        CU(cudaMemcpyAsync(h8 + 3 * cr, f64 + cr, cd * 8, cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(h8 + 3 * cr + cd, i64 + 2 * cr, cd * 8, cudaMemcpyDeviceToHost, st));
    }
    if (want_v) {
        long long* hv = h8 + 3 * cr + 2 * cd;
        CU(cudaMemcpyAsync(hv, s->d_vdist, n0 * 8, cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(hv + n0, s->d_vnorm, n0 * 8, cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(hv + 2 * n0, s->d_vlen, n0 * 8, cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(hv + 3 * n0, s->d_vidx, n0 * 8, cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(hv + 4 * n0, s->d_vpop, n0, cudaMemcpyDeviceToHost, st));
    }
    if (end_event >= 0) CU(cudaEventRecord(s->ev[6 + end_event], st));
    CU(cudaGetLastError());
    return 0;
}

int vlmp_finalize_collect(vlmp_session* s, int32_t k2, int64_t* rows_off, int64_t* rows_nbr, double* rows_d,
                          int32_t k, double* disc_dist, int64_t* disc_off,
                          double* v_dist, double* v_norm, int64_t* v_len, int64_t* v_idx, uint8_t* v_pop,
                          int32_t end_event) {
    if (!s || !s->have_profile) return fail(VLMP_E_STATE, "no profile run");
    if (k2 < 0 || k2 > 64) return fail(VLMP_E_INVALID_PARAMETERS, "k2 must be in [0, 64]");
    if (k < 0 || k > 32) return fail(VLMP_E_INVALID_PARAMETERS, "k must be in [0, 32]");
    if (end_event < -1 || end_event > 1) return fail(VLMP_E_INVALID_PARAMETERS, "end_event must be -1, 0 or 1");
    if ((k2 && (!rows_off || !rows_nbr || !rows_d)) || (k && (!disc_dist || !disc_off)))
        return fail(VLMP_E_INVALID_PARAMETERS, "null output buffer");
    const bool want_v = v_dist != nullptr;
    if (want_v && (!v_norm || !v_len || !v_idx || !v_pop)) return fail(VLMP_E_INVALID_PARAMETERS, "null VALMP buffer");
    std::lock_guard<std::mutex> g(s->lock);
    CU(cudaSetDevice(s->device));
    const long long cr = (long long)s->n_len * k2, cd = (long long)s->n_len * k;
    const long long n0 = s->n - s->lmin + 1;
    int rc;
    if ((rc = ensure(s->d_ro_i64, s->ro_i64_cap, (size_t)std::max(1LL, 2 * cr + cd)))) return rc;
    if ((rc = ensure(s->d_ro_f64, s->ro_f64_cap, (size_t)std::max(1LL, cr + cd)))) return rc;
    const size_t need = (size_t)(3 * cr + 2 * cd + (want_v ? 4 * n0 : 0)) * 8 + (want_v ? (size_t)n0 : 0) + 8;
    if (s->h_col_cap < need) {
        if (s->h_col) cudaFreeHost(s->h_col);
        s->h_col = nullptr; s->h_col_cap = 0;
        CU(cudaMallocHost((void**)&s->h_col, need));
        s->h_col_cap = need;
    }
    // as finalize_impl: everything is enqueued behind the unchecked phase 1; a redo of phase 1
    // (lost run log) enqueues it all again behind the redo
    for (int attempt = 0; attempt < 2; ++attempt) {
        if ((rc = collect_enqueue(s, k2, k, want_v, end_event, cr, cd, n0))) return rc;
        bool redone = false;
        if ((rc = settle_profile(s, &redone))) return rc;
        if (!redone) break;
    }
    CU(cudaStreamSynchronize(s->stream));
    s->stats[9] += 1 + (k2 ? 1 : 0) + (k ? 1 : 0);
    s->have_final = true;
    s->have_finals = true;
    s->stats_dirty = true;
    const long long* h8 = reinterpret_cast<const long long*>(s->h_col);
    if (k2) {
        memcpy(rows_off, h8, cr * 8);
        memcpy(rows_nbr, h8 + cr, cr * 8);
        memcpy(rows_d, h8 + 2 * cr, cr * 8);
    }
    if (k) {
        memcpy(disc_dist, h8 + 3 * cr, cd * 8);
        memcpy(disc_off, h8 + 3 * cr + cd, cd * 8);
    }
    if (want_v) {
        const long long* hv = h8 + 3 * cr + 2 * cd;
        memcpy(v_dist, hv, n0 * 8);
        memcpy(v_norm, hv + n0, n0 * 8);
        memcpy(v_len, hv + 2 * n0, n0 * 8);
        memcpy(v_idx, hv + 3 * n0, n0 * 8);
        memcpy(v_pop, hv + 4 * n0, n0);
    }
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

int vlmp_row_profile(vlmp_session* s, int64_t owner, int32_t length, double* dist, double* f, double* qt) {
    if (!s || !dist) return fail(VLMP_E_INVALID_PARAMETERS, "null argument");
    if (s->n <= 0) return fail(VLMP_E_STATE, "no series uploaded");
    if (length < 4 || 2LL * length > s->n || owner < 0 || owner > s->n - length)
        return fail(VLMP_E_INVALID_PARAMETERS, "row owner/length outside the series");
    std::lock_guard<std::mutex> g(s->lock);
    CU(cudaSetDevice(s->device));
    cudaStream_t st = s->stream;
    const long long N = s->n - length + 1;
    double* d = nullptr;
    CU(cudaMallocAsync((void**)&d, 3 * N * sizeof(double), st));
    RowArgs ra{s->d_tn, s->d_cum, s->d_cum2, s->n, (long long)owner, length, s->floor_, d, f ? d + N : nullptr,
               qt ? d + 2 * N : nullptr};
    k_row_profile<<<blocks(N, 256), 256, (size_t)length * sizeof(double), st>>>(ra);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(dist, d, N * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (f) CU(cudaMemcpyAsync(f, d + N, N * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (qt) CU(cudaMemcpyAsync(qt, d + 2 * N, N * sizeof(double), cudaMemcpyDeviceToHost, st));
    CU(cudaFreeAsync(d, st));
    CU(cudaStreamSynchronize(st));
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

}  // extern "C"
