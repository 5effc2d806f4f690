/*
 * vlmp.h -- C ABI of the B200-native variable-length matrix profile (libvlmp.so).
 *
 * The reference (seriesmine, pure Python/NumPy) has no native FFI; its drop-in
 * boundary is the pair of Python entry points
 *   valmod(series, lmin, lmax, p, *, ranking, trace, threads)
 *       /root/reference/pkg/src/seriesmine/valmod.py:192-258
 *   topkm_discord_discovery(series, lmin, lmax, k, m, p, *, trace, threads)
 *       /root/reference/pkg/src/seriesmine/discords.py:206-247
 * plus compute_matrix_profile (profile.py:329-377) which the CLI calls.
 * paper_2008_13447_b200 re-exposes those names in Python and reaches the GPU
 * only through the functions below (ctypes; plain pointers and sizes, no torch
 * types). Host pointers are caller-owned numpy buffers, never retained past the
 * call. The library owns all device memory.
 *
 * Every function returns 0 on success or a VLMP_E_* code; the message is in
 * vlmp_last_error() (thread-local). Codes map 1:1 onto the reference's
 * SeriesMineError subclasses (exceptions.py:4-56).
 */
#ifndef VLMP_H
#define VLMP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    VLMP_OK = 0,
    VLMP_E_INVALID_PARAMETERS = 1,   /* InvalidParametersError   exceptions.py:47 */
    VLMP_E_SERIES_TOO_SHORT = 2,     /* SeriesTooShortError      exceptions.py:35 */
    VLMP_E_ALL_CONSTANT = 3,         /* AllConstantError         exceptions.py:39 */
    VLMP_E_EMPTY_SERIES = 4,         /* EmptySeriesError         exceptions.py:8  */
    VLMP_E_CUDA = 10,                /* device / driver failure (no CPU fallback) */
    VLMP_E_STATE = 11,               /* call order violated (e.g. no run yet)     */
    VLMP_E_NOMEM = 12
};

typedef struct vlmp_session vlmp_session;

/* Create a session on a CUDA device (one session = one device, one in-flight call). */
int vlmp_create(vlmp_session** out, int device);
void vlmp_destroy(vlmp_session* s);
const char* vlmp_last_error(void);

/*
 * Upload one series. t, cum, cum2 are the reference DataSeries' values, _cum and
 * _cum2 (series.py:57-67: cum has n+1 entries with a leading 0, sequential
 * np.cumsum) and sigma_floor (policy.py:27-39). Window statistics are derived
 * on the device from cum/cum2 with the reference's exact operation order, so
 * mean/std are bit-identical to DataSeries.moving_stats (series.py:91-100).
 */
int vlmp_set_series(vlmp_session* s, const double* t, const double* cum,
                    const double* cum2, int64_t n, double sigma_floor);

/*
 * Phase 1: the exhaustive per-length matrix profile for lengths [lmin, lmax]
 * restricted to diagonal bands [band_lo, band_hi) (band_hi < 0 = all bands).
 * Single-GPU callers pass the whole range; multi-GPU callers shard bands
 * (vlmp_band_split) and merge the partial per-length minima with
 * vlmp_partials_* + an NCCL min all-reduce before phase 2.
 * flags: VLMP_F_FULL_EVERY_LENGTH forces the exact full-fold kernel at every
 * length (no bound filter) -- a self-check mode, slower. VLMP_F_FP64_FILTER walks the
 * filtered lengths with the FP64 recurrence and covariance log (profile.cu k_tile<false> +
 * k_log_merge) instead of the default FP32 walk + exact FP64 run evaluation (filter32.cu);
 * both are exact, the flag exists for A/B checks and is the fallback the library takes
 * itself when the FP32 run log overflows or a bound is too weak for it.
 * With flags 0, all bands, >= 40 lengths and at most 16 waves of tiles per length (small
 * series) the two halves of the length range run as two concurrent chains on two streams
 * inside the call's CUDA graph (same results; environment VLMP_CHAINS=1 turns it off).
 */
#define VLMP_F_FULL_EVERY_LENGTH 1u
#define VLMP_F_FP64_FILTER 2u
int vlmp_profile_range(vlmp_session* s, int32_t lmin, int32_t lmax,
                       int64_t band_lo, int64_t band_hi, uint32_t flags);

/*
 * Length shard for multi-GPU runs: phase 1 for length indices li_lo..li_hi of
 * [lmin, lmax] (all bands). On the default FP32 walk the tile seeds are centred direct
 * sums at the shard's first length (they only start the filter walk; every key comes from
 * the exact FP64 runs), that length takes its bounds from full folds over a sample of the
 * bands, and every length of the shard runs the FP32 walk + exact runs. (With
 * VLMP_F_FP64_FILTER the seeds are carried from lmin by the tile kernel's Welford step.)
 * Accumulators of other lengths stay empty: each (length, offset) has exactly one owner
 * rank, so the per-length minima equal a single run's (keys may differ in their last
 * bits where a run starts elsewhere; neighbours agree except at ties within ~1e-15).
 */
int vlmp_profile_lengths(vlmp_session* s, int32_t lmin, int32_t lmax, int32_t li_lo, int32_t li_hi,
                         uint32_t flags);

/* Number of 256-diagonal bands and a work-balanced contiguous split of them. */
int vlmp_band_count(vlmp_session* s, int32_t lmin, int64_t* n_bands);
int vlmp_band_split(vlmp_session* s, int32_t lmin, int32_t lmax, int32_t parts,
                    int64_t* cuts /* parts+1 entries */);

/*
 * Exact cross-GPU merge of the partial per-(length, offset) minima. The caller
 * allocates device buffers keys[n_len * stride] (uint64: order-preserving bits of
 * the clamped key; +inf bits = none) and idx[n_len * stride] (int64 neighbour;
 * INT64_MAX = none) on this session's device (e.g. torch tensors):
 *   export  -> all-reduce(MIN) keys into merged -> mask_idx (idx := INT64_MAX where
 *   the local key != merged key) -> all-reduce(MIN) idx -> import(merged, idx).
 * This is the lexicographic (value, smallest index) rule of profile.py:308.
 */
int vlmp_partials_size(vlmp_session* s, int64_t* n_len, int64_t* stride);
int vlmp_partials_export(vlmp_session* s, void* keys, void* idx);
int vlmp_partials_mask_idx(vlmp_session* s, const void* merged_keys, const void* keys, void* idx);
int vlmp_partials_import(vlmp_session* s, const void* keys, const void* idx);

/*
 * Phase 2: from the (merged) per-length minima compute the exact per-offset
 * profile values (canonical pair distance, series.py:169-194), the VALMP fold
 * (valmod.py:57-73), and keep MP/IP of every length device-resident.
 */
int vlmp_finalize(vlmp_session* s);

/*
 * Phase 2 split for length shards: profile values of length indices li_lo..li_hi only
 * ((+inf, -1) for the others, neutral for a MIN / MAX all-reduce), the device buffers
 * MP [n_len][stride] (double) and IP [n_len][stride] (int32) for the collective, then
 * the read-off state (VALMP fold) from whatever the buffers hold.
 */
int vlmp_finalize_lengths(vlmp_session* s, int32_t li_lo, int32_t li_hi);
int vlmp_final_buffers(vlmp_session* s, void** mp, void** ip, int64_t* n_len, int64_t* stride);
int vlmp_finalize_readoffs(vlmp_session* s);

/* Read-offs (all after vlmp_finalize). */
int vlmp_get_valmp(vlmp_session* s, double* dist, double* norm, int64_t* lengths,
                   int64_t* indices, uint8_t* populated /* n - lmin + 1 each */);
int vlmp_get_profile(vlmp_session* s, int32_t length, double* mp, int64_t* ip
                     /* n - length + 1 each */);
/*
 * Per length, the 2k smallest (mp, offset) rows, ascending (first = the
 * length's top-1 motif owner, valmod.py:170-177). out_off/out_nbr/out_d are
 * [n_len][2k]; unused slots have offset -1.
 */
int vlmp_smallest_rows(vlmp_session* s, int32_t k2, int64_t* out_off,
                       int64_t* out_nbr, double* out_d);
/* Top-k 1st discords per length (discords.py:68-93 replay): [n_len][k]. */
int vlmp_discords(vlmp_session* s, int32_t k, double* out_dist, int64_t* out_off);
/*
 * Phase 2 and the standard read-offs in one call with a single host wait: vlmp_finalize, then
 * (k2 > 0) vlmp_smallest_rows(k2), (k > 0) vlmp_discords(k) and (v_dist != NULL)
 * vlmp_get_valmp, all enqueued behind phase 1 and copied through pinned staging -- the same
 * outputs as those four calls (the read-off set valmod.py:192-258 + discords.py:206-247 +
 * the per-length rankings need), without the device idling between them while the host
 * wakes up. end_event (0 / 1, or -1 for none) records vlmp_event_record's slot on the stream
 * after the last copy and before the host waits.
 */
int vlmp_finalize_collect(vlmp_session* s, int32_t k2, int64_t* rows_off, int64_t* rows_nbr,
                          double* rows_d, int32_t k, double* disc_dist, int64_t* disc_off,
                          double* v_dist, double* v_norm, int64_t* v_len, int64_t* v_idx,
                          uint8_t* v_pop, int32_t end_event);
/*
 * VALMP improvement events with norm <= tau, in (length, offset) order
 * (the stream valmod feeds to a PairRanking, motifsets.py:105-117).
 * Returns the total count in *count (may exceed cap; then call again).
 */
int vlmp_ranking_events(vlmp_session* s, double tau, int64_t cap, int64_t* ev_off,
                        int64_t* ev_nbr, int64_t* ev_len, double* ev_dist,
                        double* ev_norm, int64_t* count);

/*
 * m-th discords (discords.py:206-247 with m > 1): for every length and offset the m best
 * neighbours (exact, smallest-index ties), their canonical distances sorted ascending.
 * Independent of vlmp_profile_range's state. m in [1, 8].
 */
int vlmp_profile_mbest(vlmp_session* s, int32_t lmin, int32_t lmax, int32_t m);
/* dist[N][m] (ascending canonical values), nbr[N][m] (key order; -1 = none). */
int vlmp_get_profile_m(vlmp_session* s, int32_t length, double* dist, int64_t* nbr);
/* Top-k m-th discords per length (k x m matrices, discords.py:68-93): [n_len][k][m]. */
int vlmp_discords_m(vlmp_session* s, int32_t k, double* out_dist, int64_t* out_off);

/*
 * Pruned top-k m-th discord scan (MAD, discords.py:144-247 over profile.py:66-232's partial
 * profiles): the first length runs an exhaustive pass and stores each row's best neighbours
 * (m = 1: the nearest one, from the 1-best profile; m > 1: P = min(8, max(p, m)) from the m-best
 * profile); every later length advances them in O(1) (Welford co-moment step), certifies rows by
 * VALMOD's lower bound (Eq. 2), replays the insertion policy and recomputes exact rows only for
 * owners whose stored bound could still enter the matrix -- m = 1 in blocks of consecutive rows
 * (one direct seed per diagonal, then the FP64 diagonal recurrence), in doubling windows so a
 * length takes O(log N) replay stops -- or falls back to an exhaustive pass when the modelled
 * recompute cost exceeds it. Same matrices as the exhaustive path (tests/test_gpu_pruned.py).
 * out_dist / out_off: [n_len][k][m]; counters (optional): [n_len][4] = certified rows,
 * non-certified live rows, full rows recomputed, 1 if the length ran exhaustively.
 */
int vlmp_discords_pruned(vlmp_session* s, int32_t lmin, int32_t lmax, int32_t k, int32_t m, int32_t p,
                         double* out_dist, int64_t* out_off, double* counters);

/*
 * One full row from scratch (profile.py:263-269 row_profile, the formulas of _row_arrays
 * :235-260): for every window j of this length, dist[j] (owner-first, numpy's operation order;
 * +inf for trivial matches and constant neighbours), f[j] the bound factor
 * sqrt(l (1 - max(q, 0)^2)) (optional), qt[j] the dot product of the two raw windows
 * (optional; direct FP64 sums where the reference uses FFT correlation). Arrays of
 * n - length + 1 doubles. Needs only vlmp_set_series.
 */
int vlmp_row_profile(vlmp_session* s, int64_t owner, int32_t length, double* dist, double* f, double* qt);

/*
 * Motif-set range queries (motifsets.py:158-165, the row_profile path of _range_members):
 * for query q, every offset j with dist(owners[q], j) < radii[q] at length lengths[q],
 * from the owner's full row with the reference formula (profile.py:235-260); trivial
 * matches and constant windows excluded. Needs only vlmp_set_series. members is
 * [n_q][cap] (unordered); counts[q] may exceed cap (then only cap were stored).
 */
int vlmp_range_query(vlmp_session* s, int64_t n_q, const int64_t* owners, const int32_t* lengths,
                     const double* radii, int64_t cap, int64_t* members, int64_t* counts);

/*
 * Timings and counters of the last phase-1/phase-2 run:
 * out[0] profile ms (device), out[1] finalize ms, out[2] executed pair updates,
 * out[3] W (non-trivial pair updates), out[4] tile-kernel ms, out[5] tile-kernel
 * launches, out[6] filtered lengths, out[7] full lengths, out[8] slow-path
 * candidate merges, out[9] total kernel launches, out[10] first-length tile ms,
 * out[11] flagged filter lane-rows (log records), out[12] offsets whose bound needed a direct dot product, out[13] exact redo count (1-best:
 * 1 = redone without the sampled first-length start after a log overflow, 2 = redone
 * with full folds at every length; m-best: offsets recomputed), out[14] lengths that fell back to full folds (an offset's own bound
 * too weak for the covariance-domain filter), out[15] largest per-length log fill,
 * out[16] 1 if the filtered lengths ran the FP32 walk (filter32.cu), out[17] largest
 * per-length run count of that walk, out[18] cells evaluated exactly in its runs, out[19] the
 * row-segment length S of the tile walks, out[20] k_tile32 ms (sum over its launches, CUDA
 * events on the session stream; with two chains the union of their spans), out[21] k_runs ms,
 * out[22] k_tile32 launches, out[23] 1 if the per-length sequence ran as a CUDA graph, out[24]
 * the number of concurrent chains the length range ran as (2 on small series: the two halves
 * of the range on two streams; VLMP_CHAINS=1 turns it off) (n_out <= 25).
 */
int vlmp_stats(vlmp_session* s, double* out, int32_t n_out);

/*
 * Device-timeline timing on the session's stream: record slot 0 (start) and
 * slot 1 (stop); elapsed waits for slot 1 and returns milliseconds.
 */
int vlmp_event_record(vlmp_session* s, int32_t slot);
int vlmp_event_elapsed(vlmp_session* s, float* ms);

/*
 * Window mean / std of every offset at one length, computed on the device by the routine the
 * kernels use (series.py:91-100 operation order) from the uploaded prefix sums -- equal bit for
 * bit to DataSeries.moving_stats (test_gpu_scale.py). mu, sd: n - length + 1 each.
 */
int vlmp_window_stats(vlmp_session* s, int32_t length, double* mu, double* sd);

/* FP64 FMA peak microbenchmark (DFMA instr/s on this device, all SMs). */
int vlmp_measure_fp64_peak(vlmp_session* s, double* fma_per_s);
/* FP32 FMA peak microbenchmark (FFMA lane-ops/s, register operands, all SMs, best of 3):
 * the roofline denominator of the FP32 walk (k_tile32). */
int vlmp_measure_fp32_peak(vlmp_session* s, double* fma_per_s);

#ifdef __cplusplus
}
#endif
#endif /* VLMP_H */
