// session.cu -- libvlmp sessions: device/stream setup, series upload, counters, device
// timing and the FP64 peak microbenchmark used as the roofline denominator.
#include "vlmp_internal.cuh"

namespace vlmp_impl {

thread_local std::string g_err;

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

// FP32 FMA peak: 8 independent FFMA chains per thread (register operands, as the walk's FFMA2)
__global__ void k_ffma_peak(float* out, int iters, float x) {
    float a0 = x, a1 = x + 1, a2 = x + 2, a3 = x + 3, a4 = x + 4, a5 = x + 5, a6 = x + 6, a7 = x + 7;
    const float b = 0.999999f + 1e-7f * threadIdx.x, c = 1e-9f * blockIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
            a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
        }
    }
    float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 12345.678f) out[0] = s;
}

// window statistics of every offset at one length, with the device routine k_params and the
// finalize use (win_stats: series.py:91-100 op order, no contraction) -- exported for the
// bit-exactness test against DataSeries.moving_stats
__global__ void k_win_stats(const double* cum, const double* cum2, long long N, int m, double* mu, double* sd) {
    const long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (o >= N) return;
    double a, b;
    win_stats(cum, cum2, o, m, a, b);
    mu[o] = a; sd[o] = b;
}

}  // namespace vlmp_impl

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
                    s->d_previdx, s->d_colq, s->d_rowq, s->d_forced, s->d_fixcnt, s->d_tiles, s->d_tiles_s, s->d_smap, s->d_seeds, s->d_acc, s->d_mp, s->d_ip, s->d_counters,
                    s->d_log, s->d_logcnt, s->d_p32, s->d_cq32, s->d_cq4, s->d_pf4, s->d_magblk, s->d_tiles32, s->d_ro_i64, s->d_ro_f64, s->d_ro_cnt,
                    s->d_slots, s->d_slotcnt, s->d_ipm, s->d_mpm, s->d_redo, s->d_vdist, s->d_vnorm, s->d_vlen, s->d_vidx, s->d_vpop};
    for (void* p : ptrs) if (p) cudaFree(p);
    void* xptrs[] = {s->x_prm, s->x_prm2, s->x_mu, s->x_mu2, s->x_p32, s->x_cq32, s->x_cq4, s->x_pf4,
                     s->x_magblk, s->x_seeds, s->x_log};
    for (void* p : xptrs) if (p) cudaFree(p);
    if (s->ev_fork) cudaEventDestroy(s->ev_fork);
    if (s->ev_join) cudaEventDestroy(s->ev_join);
    if (s->stream2) cudaStreamDestroy(s->stream2);
    for (auto& ev : s->ev) if (ev) cudaEventDestroy(ev);
    for (auto& ev : s->lev) cudaEventDestroy(ev);
    if (s->d_span) cudaFree(s->d_span);
    if (s->h_span) cudaFreeHost(s->h_span);
    if (s->g_exec) cudaGraphExecDestroy(s->g_exec);
    if (s->h_chk) cudaFreeHost(s->h_chk);
    if (s->h_col) cudaFreeHost(s->h_col);
    pruned_free(s);
    if (s->stream) cudaStreamDestroy(s->stream);
    delete s;
}

int vlmp_set_series(vlmp_session* s, const double* t, const double* cum, const double* cum2,
                    int64_t n, double sigma_floor) {
    if (!s || !t || !cum || !cum2) return fail(VLMP_E_INVALID_PARAMETERS, "null argument");
    if (n <= 0) return fail(VLMP_E_EMPTY_SERIES, "series holds no points");
    std::lock_guard<std::mutex> g(s->lock);
    CU(cudaSetDevice(s->device));
    long long A = ((n + 1024 + 255) / 256) * 256 + 256;
    // nothing of the previous series survives: the session reads as empty until every buffer
    // below is allocated and filled (a failed allocation leaves n = 0, so later calls refuse)
    if (s->pending) { cudaStreamSynchronize(s->stream); s->pending = false; }
    s->n = 0; s->A = 0;
    s->have_profile = s->have_final = s->have_finals = false;
    s->mbest = 0; s->mb_n_len = 0;
    if (s->tc_n != n) { s->tc_n = -1; s->tc_key[0] = -1; }   // tile lists depend on n only
    int rc;
    // grow-only: cudaFree / cudaMalloc synchronise the device and cost up to ~1 s on a
    // loaded allocator -- a repeat call with the same (or a shorter) series allocates nothing
    if ((rc = ensure(s->d_tn, s->tn_cap, (size_t)(2 * A + 4096)))) return rc;
    if ((rc = ensure(s->d_cum, s->cum_cap, (size_t)(n + 1)))) return rc;
    if ((rc = ensure(s->d_cum2, s->cum2_cap, (size_t)(n + 1)))) return rc;
    if ((rc = ensure(s->d_prm, s->prm_cap, (size_t)A))) return rc;
    if ((rc = ensure(s->d_mu, s->mu_cap, (size_t)A))) return rc;
    if ((rc = ensure(s->d_prm2, s->prm2_cap, (size_t)A))) return rc;
    if ((rc = ensure(s->d_mu2, s->mu2_cap, (size_t)A))) return rc;
    if ((rc = ensure(s->d_previdx, s->previdx_cap, (size_t)A))) return rc;
    if ((rc = ensure(s->d_colq, s->colq_cap, (size_t)A))) return rc;
    if ((rc = ensure(s->d_rowq, s->rowq_cap, (size_t)A))) return rc;
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
    s->n = n; s->A = A; s->floor_ = sigma_floor;
    return 0;
}

int vlmp_stats(vlmp_session* s, double* out, int32_t n_out) {
    if (!s || !out) return fail(VLMP_E_INVALID_PARAMETERS, "null argument");
    {
        std::lock_guard<std::mutex> g(s->lock);
        int rc = settle_profile(s, nullptr);
        if (!rc) rc = fill_event_stats(s);
        if (rc) return rc;
    }
    for (int q = 0; q < n_out && q < 25; ++q) out[q] = s->stats[q];
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

int vlmp_window_stats(vlmp_session* s, int32_t length, double* mu, double* sd) {
    if (!s || !mu || !sd) return fail(VLMP_E_INVALID_PARAMETERS, "null argument");
    if (s->n <= 0) return fail(VLMP_E_STATE, "no series uploaded");
    if (length < 1 || length > s->n) return fail(VLMP_E_INVALID_PARAMETERS, "length outside [1, n]");
    std::lock_guard<std::mutex> g(s->lock);
    CU(cudaSetDevice(s->device));
    const long long N = s->n - length + 1;
    double* d = nullptr;
    CU(cudaMalloc((void**)&d, 2 * N * sizeof(double)));
    k_win_stats<<<blocks(N, 256), 256, 0, s->stream>>>(s->d_cum, s->d_cum2, N, length, d, d + N);
    cudaError_t e1 = cudaMemcpyAsync(mu, d, N * sizeof(double), cudaMemcpyDeviceToHost, s->stream);
    cudaError_t e2 = cudaMemcpyAsync(sd, d + N, N * sizeof(double), cudaMemcpyDeviceToHost, s->stream);
    cudaError_t e3 = cudaStreamSynchronize(s->stream);
    cudaFree(d);
    CU(e1); CU(e2); CU(e3);
    return 0;
}

int vlmp_measure_fp32_peak(vlmp_session* s, double* fma_per_s) {
    if (!s || !fma_per_s) return fail(VLMP_E_INVALID_PARAMETERS, "null argument");
    std::lock_guard<std::mutex> g(s->lock);
    CU(cudaSetDevice(s->device));
    int sms = 0;
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device));
    float* d_out = nullptr;
    CU(cudaMalloc((void**)&d_out, 8));
    const int threads = 512, per_sm = 4, iters = 4096;
    const unsigned grid = sms * per_sm;
    k_ffma_peak<<<grid, threads, 0, s->stream>>>(d_out, 16, 1.0f);   // warm-up
    double best = 0;
    for (int rep = 0; rep < 3; ++rep) {
        CU(cudaEventRecord(s->ev[6], s->stream));
        k_ffma_peak<<<grid, threads, 0, s->stream>>>(d_out, iters, 1.0f);
        CU(cudaEventRecord(s->ev[7], s->stream));
        CU(cudaEventSynchronize(s->ev[7]));
        float ms = 0; CU(cudaEventElapsedTime(&ms, s->ev[6], s->ev[7]));
        best = std::max(best, (double)grid * threads * iters * 16.0 * 8.0 / (ms * 1e-3));
    }
    CU(cudaFree(d_out));
    *fma_per_s = best;
    return 0;
}

}  // extern "C"
