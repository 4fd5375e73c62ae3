/*
 * ks_oracle.c -- CPU restatement of the kernelscope operator (TEST
 * INFRASTRUCTURE ONLY; see ks_oracle.h).  Compile with -ffp-contract=off.
 *
 * Reference: /root/reference/proj/src/conv_core.cpp.  Each routine names the
 * lines it restates.  The loops are written over an h-range so the timed CPU
 * baseline can fan channel slices out over threads without changing any
 * rounding (channels are independent).
 */
#include "ks_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>

/* ---- splitmix64 (include/kernelscope/rng.hpp:12-28) ---------------------- */
static const uint64_t KSO_GAMMA = 0x9E3779B97F4A7C15ull;

static uint64_t kso_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* The state after n calls is seed + n*gamma (mod 2^64); next() returns the
 * mix of the post-increment state, so draw n (1-based) is mix(seed+n*gamma). */
uint64_t kso_splitmix64_at(uint64_t seed, uint64_t n) { return kso_mix(seed + n * KSO_GAMMA); }

void kso_fill_pm1(uint64_t seed, uint64_t first, float* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t u = kso_splitmix64_at(seed, first + (uint64_t)i + 1u);
        /* next_unit(): top 53 bits * 2^-53; next_pm1(): float(2u - 1) in double. */
        const double unit = (double)(u >> 11) * 0x1.0p-53;
        out[i] = (float)(2.0 * unit - 1.0);
    }
}

/* ---- mul_add (src/conv_core.cpp:14-19) ----------------------------------- */
static inline float mul_add_f32(float acc, float a, float b, int mode) {
    return mode == KSO_FUSED ? fmaf(a, b, acc) : acc + a * b;
}
static inline double mul_add_f64(double acc, double a, double b, int mode) {
    return mode == KSO_FUSED ? fma(a, b, acc) : acc + a * b;
}

static inline int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }
static inline int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }

/* The three paths are generated once per element type T with MULADD. */
#define KSO_DEFINE_PATHS(T, SUF, MULADD)                                                      \
    /* forward_impl (src/conv_core.cpp:21-46): per (b,h,t), taps j in [j_lo,j_hi)          \
     * ascending from acc = +0; out-of-row taps are skipped (:35-36). */                     \
    static void fwd_rows_##SUF(const T* x, const T* k, T* y, int64_t B, int64_t H,          \
                               int64_t L, int64_t K, int mode, int64_t h0, int64_t h1) {    \
        const int64_t p = K / 2; /* pad_width (include/kernelscope/shape.hpp:16) */           \
        for (int64_t b = 0; b < B; ++b)                                                      \
            for (int64_t h = h0; h < h1; ++h) {                                              \
                const T* xr = x + (b * H + h) * L;                                           \
                const T* kr = k + h * K;                                                     \
                T* yr = y + (b * H + h) * L;                                                 \
                for (int64_t t = 0; t < L; ++t) {                                            \
                    const int64_t j_lo = imax(0, p - t);                                     \
                    const int64_t j_hi = imin(K, L + p - t);                                 \
                    T acc = 0;                                                               \
                    for (int64_t j = j_lo; j < j_hi; ++j)                                    \
                        acc = MULADD(acc, xr[t + j - p], kr[j], mode);                       \
                    yr[t] = acc;                                                             \
                }                                                                            \
            }                                                                                \
    }                                                                                        \
    /* backward_input_impl (src/conv_core.cpp:48-75): offset q = K-1-p (:56), reversed    \
     * kernel k[K-1-j] (:68). */                                                             \
    static void dx_rows_##SUF(const T* gy, const T* k, T* dx, int64_t B, int64_t H,         \
                              int64_t L, int64_t K, int mode, int64_t h0, int64_t h1) {     \
        const int64_t q = K - 1 - K / 2;                                                     \
        for (int64_t b = 0; b < B; ++b)                                                      \
            for (int64_t h = h0; h < h1; ++h) {                                              \
                const T* gr = gy + (b * H + h) * L;                                          \
                const T* kr = k + h * K;                                                     \
                T* dr = dx + (b * H + h) * L;                                                \
                for (int64_t t = 0; t < L; ++t) {                                            \
                    const int64_t j_lo = imax(0, q - t);                                     \
                    const int64_t j_hi = imin(K, L + q - t);                                 \
                    T acc = 0;                                                               \
                    for (int64_t j = j_lo; j < j_hi; ++j)                                    \
                        acc = MULADD(acc, gr[t + j - q], kr[K - 1 - j], mode);               \
                    dr[t] = acc;                                                             \
                }                                                                            \
            }                                                                                \
    }                                                                                        \
    /* WeightTerm::operator() (src/conv_core.cpp:88-95): a plain product, +0 when the x  \
     * tap leaves the row; mode is ignored. */                                               \
    static inline T term_##SUF(const T* gy, const T* x, int64_t H, int64_t h, int64_t d,   \
                               int64_t L, int64_t flat) {                                    \
        const int64_t b = flat / L;                                                          \
        const int64_t t = flat - b * L;                                                      \
        const int64_t xi = t + d;                                                            \
        if (xi < 0 || xi >= L) return (T)0;                                                  \
        return gy[(b * H + h) * L + t] * x[(b * H + h) * L + xi];                            \
    }                                                                                        \
    /* reduce_pairwise (src/conv_core.cpp:113-118): midpoint split lo+(hi-lo)/2. */          \
    static T pairwise_##SUF(const T* gy, const T* x, int64_t H, int64_t h, int64_t d,      \
                            int64_t L, int64_t lo, int64_t hi) {                             \
        if (hi - lo == 1) return term_##SUF(gy, x, H, h, d, L, lo);                          \
        const int64_t mid = lo + (hi - lo) / 2;                                              \
        const T a = pairwise_##SUF(gy, x, H, h, d, L, lo, mid);                              \
        const T c = pairwise_##SUF(gy, x, H, h, d, L, mid, hi);                              \
        return a + c;                                                                        \
    }                                                                                        \
    /* reduce_sequential (src/conv_core.cpp:98-111). */                                      \
    static T sequential_##SUF(const T* gy, const T* x, int64_t B, int64_t H, int64_t h,    \
                              int64_t d, int64_t L, int mode) {                              \
        T acc = 0;                                                                           \
        const int64_t t_lo = imax(0, -d), t_hi = imin(L, L - d);                             \
        for (int64_t b = 0; b < B; ++b) {                                                    \
            const T* gr = gy + (b * H + h) * L;                                              \
            const T* xr = x + (b * H + h) * L;                                               \
            for (int64_t t = t_lo; t < t_hi; ++t) acc = MULADD(acc, gr[t], xr[t + d], mode); \
        }                                                                                    \
        return acc;                                                                          \
    }                                                                                        \
    /* reduce_chunked (src/conv_core.cpp:122-146): sequential partial per flat chunk,     \
     * `total += partial` whenever the chunk id changes, then once at the end. */            \
    static T chunked_##SUF(const T* gy, const T* x, int64_t B, int64_t H, int64_t h,       \
                           int64_t d, int64_t L, int64_t chunk, int mode) {                  \
        const int64_t t_lo = imax(0, -d), t_hi = imin(L, L - d);                             \
        T total = 0, partial = 0;                                                            \
        int64_t current = 0;                                                                 \
        for (int64_t b = 0; b < B; ++b) {                                                    \
            const T* gr = gy + (b * H + h) * L;                                              \
            const T* xr = x + (b * H + h) * L;                                               \
            for (int64_t t = t_lo; t < t_hi; ++t) {                                          \
                const int64_t c = (b * L + t) / chunk;                                       \
                if (c != current) {                                                          \
                    total += partial;                                                        \
                    partial = 0;                                                             \
                    current = c;                                                             \
                }                                                                            \
                partial = MULADD(partial, gr[t], xr[t + d], mode);                           \
            }                                                                                \
        }                                                                                    \
        total += partial;                                                                    \
        return total;                                                                        \
    }                                                                                        \
    /* backward_weight_impl (src/conv_core.cpp:148-181). */                                  \
    static void dw_rows_##SUF(const T* gy, const T* x, T* dk, int64_t B, int64_t H,         \
                              int64_t L, int64_t K, int scheme, int64_t chunk, int mode,    \
                              int64_t h0, int64_t h1) {                                      \
        const int64_t p = K / 2, flat_n = B * L;                                             \
        for (int64_t h = h0; h < h1; ++h)                                                    \
            for (int64_t j = 0; j < K; ++j) {                                                \
                const int64_t d = j - p;                                                     \
                T acc = 0;                                                                   \
                if (scheme == KSO_PAIRWISE)                                                  \
                    acc = pairwise_##SUF(gy, x, H, h, d, L, 0, flat_n);                      \
                else if (scheme == KSO_CHUNKED && chunk < flat_n)                            \
                    acc = chunked_##SUF(gy, x, B, H, h, d, L, chunk, mode);                  \
                else /* sequential, or chunk >= B*L (:172-174) */                            \
                    acc = sequential_##SUF(gy, x, B, H, h, d, L, mode);                      \
                dk[h * K + j] = acc;                                                         \
            }                                                                                \
    }

KSO_DEFINE_PATHS(float, f32, mul_add_f32)
KSO_DEFINE_PATHS(double, f64, mul_add_f64)

void kso_forward_f32(const float* x, const float* k, float* y, int64_t B, int64_t H,
                     int64_t L, int64_t K, int mode) {
    fwd_rows_f32(x, k, y, B, H, L, K, mode, 0, H);
}
void kso_forward_f64(const double* x, const double* k, double* y, int64_t B, int64_t H,
                     int64_t L, int64_t K, int mode) {
    fwd_rows_f64(x, k, y, B, H, L, K, mode, 0, H);
}
void kso_backward_input_f32(const float* gy, const float* k, float* dx, int64_t B,
                            int64_t H, int64_t L, int64_t K, int mode) {
    dx_rows_f32(gy, k, dx, B, H, L, K, mode, 0, H);
}
void kso_backward_input_f64(const double* gy, const double* k, double* dx, int64_t B,
                            int64_t H, int64_t L, int64_t K, int mode) {
    dx_rows_f64(gy, k, dx, B, H, L, K, mode, 0, H);
}
int kso_backward_weight_f32(const float* gy, const float* x, float* dk, int64_t B,
                            int64_t H, int64_t L, int64_t K, int scheme, int64_t chunk,
                            int mode) {
    if (scheme == KSO_CHUNKED && chunk < 1) return -1;
    dw_rows_f32(gy, x, dk, B, H, L, K, scheme, chunk, mode, 0, H);
    return 0;
}
int kso_backward_weight_f64(const double* gy, const double* x, double* dk, int64_t B,
                            int64_t H, int64_t L, int64_t K, int scheme, int64_t chunk,
                            int mode) {
    if (scheme == KSO_CHUNKED && chunk < 1) return -1;
    dw_rows_f64(gy, x, dk, B, H, L, K, scheme, chunk, mode, 0, H);
    return 0;
}

/* tests/support/oracle.hpp:73-90: exact integer dW. */
void kso_backward_weight_i64(const float* gy, const float* x, int64_t* dk, int64_t B,
                             int64_t H, int64_t L, int64_t K) {
    const int64_t p = K / 2;
    for (int64_t h = 0; h < H; ++h)
        for (int64_t j = 0; j < K; ++j) {
            int64_t acc = 0;
            for (int64_t b = 0; b < B; ++b)
                for (int64_t t = 0; t < L; ++t) {
                    const int64_t xi = t + j - p;
                    if (xi >= 0 && xi < L)
                        acc += (int64_t)gy[(b * H + h) * L + t] * (int64_t)x[(b * H + h) * L + xi];
                }
            dk[h * K + j] = acc;
        }
}

/* ---- channel-slice fan-out (timed CPU baseline only) --------------------- */
typedef struct {
    int path; /* 0 fwd, 1 dx, 2 dw, 3 dw in fp64 (a, b, out are double*) */
    const float *a, *b;
    float* out;
    int64_t B, H, L, K, chunk, h0, h1;
    int mode, scheme;
} kso_job;

static void* kso_run_job(void* arg) {
    const kso_job* j = (const kso_job*)arg;
    if (j->path == 0)
        fwd_rows_f32(j->a, j->b, j->out, j->B, j->H, j->L, j->K, j->mode, j->h0, j->h1);
    else if (j->path == 1)
        dx_rows_f32(j->a, j->b, j->out, j->B, j->H, j->L, j->K, j->mode, j->h0, j->h1);
    else if (j->path == 2)
        dw_rows_f32(j->a, j->b, j->out, j->B, j->H, j->L, j->K, j->scheme, j->chunk, j->mode,
                    j->h0, j->h1);
    else
        dw_rows_f64((const double*)(const void*)j->a, (const double*)(const void*)j->b,
                    (double*)(void*)j->out, j->B, j->H, j->L, j->K, j->scheme, j->chunk, j->mode,
                    j->h0, j->h1);
    return NULL;
}

static void kso_fan_out(kso_job proto, int threads) {
    if (threads < 1) threads = 1;
    if (threads > proto.H) threads = (int)proto.H;
    pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    kso_job* jobs = (kso_job*)calloc((size_t)threads, sizeof(kso_job));
    for (int i = 0; i < threads; ++i) {
        jobs[i] = proto;
        jobs[i].h0 = proto.H * i / threads;
        jobs[i].h1 = proto.H * (i + 1) / threads;
        pthread_create(&tid[i], NULL, kso_run_job, &jobs[i]);
    }
    for (int i = 0; i < threads; ++i) pthread_join(tid[i], NULL);
    free(tid);
    free(jobs);
}

void kso_forward_f32_mt(const float* x, const float* k, float* y, int64_t B, int64_t H,
                        int64_t L, int64_t K, int mode, int threads) {
    kso_job j = {0, x, k, y, B, H, L, K, 0, 0, H, mode, 0};
    kso_fan_out(j, threads);
}
void kso_backward_input_f32_mt(const float* gy, const float* k, float* dx, int64_t B,
                               int64_t H, int64_t L, int64_t K, int mode, int threads) {
    kso_job j = {1, gy, k, dx, B, H, L, K, 0, 0, H, mode, 0};
    kso_fan_out(j, threads);
}
int kso_backward_weight_f32_mt(const float* gy, const float* x, float* dk, int64_t B,
                               int64_t H, int64_t L, int64_t K, int scheme, int64_t chunk,
                               int mode, int threads) {
    if (scheme == KSO_CHUNKED && chunk < 1) return -1;
    kso_job j = {2, gy, x, dk, B, H, L, K, chunk, 0, H, mode, scheme};
    kso_fan_out(j, threads);
    return 0;
}

/* fp64 dW fanned out over channels (the parity tests' truth at full size). */
int kso_backward_weight_f64_mt(const double* gy, const double* x, double* dk, int64_t B,
                               int64_t H, int64_t L, int64_t K, int scheme, int64_t chunk,
                               int mode, int threads) {
    if (scheme == KSO_CHUNKED && chunk < 1) return -1;
    kso_job j = {3, (const float*)(const void*)gy, (const float*)(const void*)x, (float*)(void*)dk,
                 B, H, L, K, chunk, 0, H, mode, scheme};
    kso_fan_out(j, threads);
    return 0;
}
