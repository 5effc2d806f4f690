/*
 * vlmp_oracle.c -- CPU restatement of the reference's exhaustive matrix-profile path.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the parity checker (and the bench's
 * cpu_baseline / --impl reference arm). Only tests/, __graft_entry__.smoke() and
 * bench.py may load it. The product path (paper_2008_13447_b200) never does.
 *
 * Restates, in plain C with IEEE double arithmetic and no FMA contraction
 * (compiled with -ffp-contract=off):
 *   - DataSeries.moving_stats        /root/reference/pkg/src/seriesmine/series.py:91-100
 *   - policy.exclusion_zone          /root/reference/pkg/src/seriesmine/policy.py:17-19
 *   - _scan_chunk + _row_arrays      /root/reference/pkg/src/seriesmine/profile.py:235-260, 288-326
 *     (row-major STOMP over CHUNK_ROWS=2048 chunks, first-argmin tie rule,
 *      constant rows -> +inf / -1). Deviation: the chunk's seed row is a direct
 *      sequential dot product instead of scipy.fft (series.py:124-138); both are
 *      the same dot products, FFT rounding differs by ~1e-11 relative.
 *   - pair_distance / znorm_distance /root/reference/pkg/src/seriesmine/series.py:169-194
 *   - update_fixed_length_discords   /root/reference/pkg/src/seriesmine/discords.py:68-93
 *     + has_trivial (:48-50), replayed in ascending offset order as the
 *     brute-force reference does (oracle.py:137-145), m = 1.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define CHUNK_ROWS 2048

static int64_t excl_zone(int64_t m) { return (m + 1) / 2; }   /* ceil(m/2) */

/* series.py:91-100 (s, ss, mu = s/L, var = ss/L - mu*mu, clamp, sqrt) */
void vlmpo_stats(const double* cum, const double* cum2, int64_t n, int64_t m,
                 double* mu, double* sd) {
    int64_t n_dp = n - m + 1;
    for (int64_t i = 0; i < n_dp; ++i) {
        double s = cum[i + m] - cum[i];
        double ss = cum2[i + m] - cum2[i];
        double u = s / (double)m;
        double var = ss / (double)m - u * u;
        if (!(var >= 0.0)) var = 0.0;   /* np.maximum(var, 0.0) */
        mu[i] = u;
        sd[i] = sqrt(var);
    }
}

typedef struct {
    const double* t; const double* mu; const double* sd;
    int64_t n, m, n_dp; double floor_;
    double* mp; int64_t* ip;
    int64_t mbest; double* bm; int64_t* bmi;   /* optional m best per row (profile.py:319-326) */
    int64_t next_chunk, row_lo, row_hi;
    pthread_mutex_t lock;
} job_t;

static void scan_chunk(job_t* J, int64_t start, int64_t stop, double* qt, double* prev) {
    const double* t = J->t; const double* mu = J->mu; const double* sd = J->sd;
    const int64_t n_dp = J->n_dp, m = J->m;
    const double L = (double)m;
    const int64_t e = excl_zone(m);
    /* seed row: qt[j] = dot(t[start:start+m], t[j:j+m]) */
    for (int64_t j = 0; j < n_dp; ++j) {
        double acc = 0.0;
        for (int64_t k = 0; k < m; ++k) acc += t[start + k] * t[j + k];
        qt[j] = acc;
    }
    for (int64_t i = start; i < stop; ++i) {
        if (i > start) {
            double* tmp = prev; prev = qt; qt = tmp;
            double ti0 = t[i - 1], ti1 = t[i + m - 1];
            for (int64_t j = n_dp - 1; j >= 1; --j)
                qt[j] = (prev[j - 1] - t[j - 1] * ti0) + t[j + m - 1] * ti1;
            double acc = 0.0;
            for (int64_t k = 0; k < m; ++k) acc += t[i + k] * t[k];
            qt[0] = acc;
        }
        if (i < J->row_lo || i >= J->row_hi) continue;
        if (sd[i] < J->floor_) {
            J->mp[i] = INFINITY; J->ip[i] = -1;
            for (int64_t q = 0; q < J->mbest; ++q) { J->bm[i * J->mbest + q] = INFINITY; J->bmi[i * J->mbest + q] = -1; }
            continue;
        }
        int64_t lo = i - e + 1 > 0 ? i - e + 1 : 0;
        int64_t hi = i + e < n_dp ? i + e : n_dp;
        double a_mu = L * mu[i];
        double a_sd = L * sd[i];
        double best = INFINITY; int64_t bj = -1;
        double mbd[16]; int64_t mbj[16];
        for (int64_t q = 0; q < J->mbest; ++q) { mbd[q] = INFINITY; mbj[q] = -1; }
        for (int64_t j = 0; j < n_dp; ++j) {
            if (j >= lo && j < hi) continue;
            if (!(sd[j] >= J->floor_)) continue;
            double denom = a_sd * sd[j];
            double q_raw = (qt[j] - a_mu * mu[j]) / denom;
            double rad = (2.0 * L) * (1.0 - q_raw);
            if (!(rad >= 0.0)) rad = 0.0;     /* np.maximum(rad, 0.0) (NaN stays NaN in numpy; denom>0 here) */
            double d = sqrt(rad);
            if (d < best) { best = d; bj = j; }   /* first argmin */
            if (J->mbest > 0 && d < mbd[J->mbest - 1]) {   /* m best by (dist, index) */
                int64_t q = J->mbest - 1;
                while (q > 0 && d < mbd[q - 1]) { mbd[q] = mbd[q - 1]; mbj[q] = mbj[q - 1]; --q; }
                mbd[q] = d; mbj[q] = j;
            }
        }
        for (int64_t q = 0; q < J->mbest; ++q) { J->bm[i * J->mbest + q] = mbd[q]; J->bmi[i * J->mbest + q] = mbj[q]; }
        J->mp[i] = best; J->ip[i] = (best < INFINITY) ? bj : -1;
        if (!(best < INFINITY)) J->mp[i] = INFINITY;
    }
}

static void* worker(void* arg) {
    job_t* J = (job_t*)arg;
    double* qt = (double*)malloc(sizeof(double) * (size_t)J->n_dp);
    double* prev = (double*)malloc(sizeof(double) * (size_t)J->n_dp);
    for (;;) {
        pthread_mutex_lock(&J->lock);
        int64_t c = J->next_chunk++;
        pthread_mutex_unlock(&J->lock);
        int64_t start = c * CHUNK_ROWS;
        if (start >= J->n_dp) break;
        int64_t stop = start + CHUNK_ROWS < J->n_dp ? start + CHUNK_ROWS : J->n_dp;
        if (stop <= J->row_lo || start >= J->row_hi) continue;
        scan_chunk(J, start, stop, qt, prev);
    }
    free(qt); free(prev);
    return NULL;
}

/*
 * Exact matrix profile at length m for rows [row_lo, row_hi) (profile.py:329-377).
 * mp/ip have n-m+1 entries; rows outside the range are left untouched.
 * Returns 0, or -1 on bad arguments.
 */
int vlmpo_profile_m(const double* t, const double* cum, const double* cum2, int64_t n,
                    int64_t m, double sigma_floor, int64_t row_lo, int64_t row_hi,
                    double* mp, int64_t* ip, int64_t mbest, double* bm, int64_t* bmi, int nthreads);

int vlmpo_profile(const double* t, const double* cum, const double* cum2, int64_t n,
                  int64_t m, double sigma_floor, int64_t row_lo, int64_t row_hi,
                  double* mp, int64_t* ip, int nthreads) {
    return vlmpo_profile_m(t, cum, cum2, n, m, sigma_floor, row_lo, row_hi, mp, ip, 0, NULL, NULL, nthreads);
}

/* as vlmpo_profile, plus the mbest (<= 16) smallest (distance, index) per row into
   bm/bmi [n_dp][mbest] (profile.py:319-326 m_track) */
int vlmpo_profile_m(const double* t, const double* cum, const double* cum2, int64_t n,
                    int64_t m, double sigma_floor, int64_t row_lo, int64_t row_hi,
                    double* mp, int64_t* ip, int64_t mbest, double* bm, int64_t* bmi, int nthreads) {
    if (mbest < 0 || mbest > 16) return -1;
    if (m < 1 || m > n) return -1;
    int64_t n_dp = n - m + 1;
    if (row_lo < 0) row_lo = 0;
    if (row_hi > n_dp) row_hi = n_dp;
    double* mu = (double*)malloc(sizeof(double) * (size_t)n_dp);
    double* sd = (double*)malloc(sizeof(double) * (size_t)n_dp);
    vlmpo_stats(cum, cum2, n, m, mu, sd);
    job_t J;
    J.t = t; J.mu = mu; J.sd = sd; J.n = n; J.m = m; J.n_dp = n_dp; J.floor_ = sigma_floor;
    J.mp = mp; J.ip = ip; J.next_chunk = 0; J.row_lo = row_lo; J.row_hi = row_hi;
    J.mbest = mbest; J.bm = bm; J.bmi = bmi;
    pthread_mutex_init(&J.lock, NULL);
    if (nthreads < 1) nthreads = 1;
    pthread_t th[256];
    if (nthreads > 256) nthreads = 256;
    for (int k = 0; k < nthreads; ++k) pthread_create(&th[k], NULL, worker, &J);
    for (int k = 0; k < nthreads; ++k) pthread_join(th[k], NULL);
    pthread_mutex_destroy(&J.lock);
    free(mu); free(sd);
    return 0;
}

/* series.py:81-89 stats() of one window */
static void win_stats(const double* cum, const double* cum2, int64_t i, int64_t m,
                      double* mu, double* sigma) {
    double s = cum[i + m] - cum[i];
    double ss = cum2[i + m] - cum2[i];
    double u = s / (double)m;
    double var = ss / (double)m - u * u;
    *mu = u;
    *sigma = var > 0.0 ? sqrt(var) : 0.0;
}

/* series.py:169-194: canonical (min,max) order, +inf when either window is constant */
double vlmpo_pair_distance(const double* t, const double* cum, const double* cum2,
                           int64_t i, int64_t j, int64_t m, double sigma_floor) {
    int64_t a = i <= j ? i : j, b = i <= j ? j : i;
    double mua, sda, mub, sdb;
    win_stats(cum, cum2, a, m, &mua, &sda);
    win_stats(cum, cum2, b, m, &mub, &sdb);
    if (sda < sigma_floor || sdb < sigma_floor) return INFINITY;
    double qt = 0.0;
    for (int64_t k = 0; k < m; ++k) qt += t[a + k] * t[b + k];
    double L = (double)m;
    double rad = (2.0 * L) * (1.0 - (qt - (L * mua) * mub) / ((L * sda) * sdb));
    return rad > 0.0 ? sqrt(rad) : 0.0;
}

/*
 * Top-k 1st discords at one length (discords.py:68-93, :48-50; oracle.py:137-145).
 * vals[o] is the owner's canonical NN distance (+inf / NaN = no valid neighbour:
 * skipped). Offsets are replayed in ascending order. out_dist/out_off have k
 * cells, initialised here to -inf / -1.
 */
void vlmpo_discords_m1(const double* vals, int64_t n_dp, int64_t m, int64_t k,
                       double* out_dist, int64_t* out_off) {
    int64_t e = excl_zone(m);
    for (int64_t r = 0; r < k; ++r) { out_dist[r] = -INFINITY; out_off[r] = -1; }
    for (int64_t o = 0; o < n_dp; ++o) {
        double d = vals[o];
        if (!(d < INFINITY)) continue;               /* constant owner / no neighbour */
        int trivial = 0;
        for (int64_t r = 0; r < k; ++r) {
            int64_t occ = out_off[r];
            if (occ >= 0 && llabs(o - occ) < e) { trivial = 1; break; }
        }
        if (trivial) continue;
        for (int64_t r = 0; r < k; ++r) {
            if (d > out_dist[r]) {
                for (int64_t q = k - 1; q > r; --q) { out_dist[q] = out_dist[q - 1]; out_off[q] = out_off[q - 1]; }
                out_dist[r] = d; out_off[r] = o;
                break;
            }
        }
    }
}

/*
 * Top-k m-th discords at one length (discords.py:68-93, :48-50): vals[o][mb] are the
 * owner's canonical match distances ascending; owners whose mb-th value is not finite
 * are skipped. out_* are [k][mb].
 */
void vlmpo_discords_km(const double* vals, int64_t n_dp, int64_t m, int64_t k, int64_t mb,
                       double* out_dist, int64_t* out_off) {
    int64_t e = excl_zone(m);
    for (int64_t r = 0; r < k * mb; ++r) { out_dist[r] = -INFINITY; out_off[r] = -1; }
    for (int64_t o = 0; o < n_dp; ++o) {
        const double* b = vals + o * mb;
        if (!(b[mb - 1] < INFINITY)) continue;
        int trivial = 0;
        for (int64_t r = 0; r < k * mb; ++r)
            if (out_off[r] >= 0 && llabs(o - out_off[r]) < e) { trivial = 1; break; }
        if (trivial) continue;
        int done = 0;
        for (int64_t c = mb - 1; c >= 0 && !done; --c) {
            double d = b[c];
            for (int64_t r = 0; r < k; ++r) {
                if (d > out_dist[r * mb + c]) {
                    for (int64_t q = k - 1; q > r; --q) {
                        out_dist[q * mb + c] = out_dist[(q - 1) * mb + c];
                        out_off[q * mb + c] = out_off[(q - 1) * mb + c];
                    }
                    out_dist[r * mb + c] = d; out_off[r * mb + c] = o;
                    done = 1;
                    break;
                }
            }
        }
    }
}
