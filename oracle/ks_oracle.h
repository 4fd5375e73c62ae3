/*
 * ks_oracle.h -- CPU restatement of the kernelscope depthwise-conv1d operator.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA path in
 * paper_2604_25422_b200/.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it; the product library never
 * links or calls it.
 *
 * Every function restates the reference algorithm in plain C and cites the
 * reference line it follows (paths relative to /root/reference/proj).  It is
 * pinned two ways (see tests/test_oracle.py):
 *   - against the known-answer tests of tests/test_conv_core.cpp, and
 *   - bit-for-bit against oracle/_ref/libksref.so, the reference's own
 *     src/conv_core.cpp compiled from its sources by oracle/Makefile, through
 *     the golden fixtures committed under tests/golden/.
 *
 * Build with -ffp-contract=off (src/CMakeLists.txt:14-17): MulAddMode::Separate
 * must round the multiply and the add separately.
 */
#ifndef KS_ORACLE_H
#define KS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* MulAddMode (include/kernelscope/conv_core.hpp:45). */
enum { KSO_SEPARATE = 0, KSO_FUSED = 1 };
/* SumScheme (include/kernelscope/conv_core.hpp:14-18). */
enum { KSO_SEQUENTIAL = 0, KSO_PAIRWISE = 1, KSO_CHUNKED = 2 };

/* splitmix64 stream (include/kernelscope/rng.hpp:12-28) with O(1) skip-ahead:
 * writes draws first+1 .. first+n of the stream seeded with `seed` as
 * float(2*unit-1).  fill order of validate(): x, then k, then gy
 * (src/conv_core.cpp:241-247). */
void kso_fill_pm1(uint64_t seed, uint64_t first, float* out, int64_t n);
uint64_t kso_splitmix64_at(uint64_t seed, uint64_t n); /* n-th draw, 1-based */

/* conv::forward (src/conv_core.cpp:21-46). */
void kso_forward_f32(const float* x, const float* k, float* y, int64_t B, int64_t H,
                     int64_t L, int64_t K, int mode);
void kso_forward_f64(const double* x, const double* k, double* y, int64_t B, int64_t H,
                     int64_t L, int64_t K, int mode);
/* conv::backward_input (src/conv_core.cpp:48-75), q = K-1-p. */
void kso_backward_input_f32(const float* gy, const float* k, float* dx, int64_t B,
                            int64_t H, int64_t L, int64_t K, int mode);
void kso_backward_input_f64(const double* gy, const double* k, double* dx, int64_t B,
                            int64_t H, int64_t L, int64_t K, int mode);
/* conv::backward_weight (src/conv_core.cpp:148-181).  Returns 0, or -1 for
 * chunked with chunk < 1 (src/conv_core.cpp:154-156). */
int kso_backward_weight_f32(const float* gy, const float* x, float* dk, int64_t B,
                            int64_t H, int64_t L, int64_t K, int scheme, int64_t chunk,
                            int mode);
int kso_backward_weight_f64(const double* gy, const double* x, double* dk, int64_t B,
                            int64_t H, int64_t L, int64_t K, int scheme, int64_t chunk,
                            int mode);
/* Exact int64 weight gradient for integer-valued inputs
 * (tests/support/oracle.hpp:73-90). */
void kso_backward_weight_i64(const float* gy, const float* x, int64_t* dk, int64_t B,
                             int64_t H, int64_t L, int64_t K);

/* Row-sliced multi-thread fan-out of the three fp32 paths: channel h is
 * independent, so slicing over h is bitwise identical to the single call
 * (SPEC.md:121).  Used only for the timed CPU baseline. */
void kso_forward_f32_mt(const float* x, const float* k, float* y, int64_t B, int64_t H,
                        int64_t L, int64_t K, int mode, int threads);
void kso_backward_input_f32_mt(const float* gy, const float* k, float* dx, int64_t B,
                               int64_t H, int64_t L, int64_t K, int mode, int threads);
int kso_backward_weight_f32_mt(const float* gy, const float* x, float* dk, int64_t B,
                               int64_t H, int64_t L, int64_t K, int scheme, int64_t chunk,
                               int mode, int threads);
int kso_backward_weight_f64_mt(const double* gy, const double* x, double* dk, int64_t B,
                               int64_t H, int64_t L, int64_t K, int scheme, int64_t chunk,
                               int mode, int threads);

#ifdef __cplusplus
}
#endif
#endif
