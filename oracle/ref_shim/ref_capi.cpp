// ref_capi.cpp -- extern "C" shim over the UNMODIFIED reference operator
// (/root/reference/proj/src/conv_core.cpp), compiled from the reference's own
// sources by oracle/Makefile into oracle/_ref/libksref.so.
//
// TEST INFRASTRUCTURE ONLY: used to pin the C restatement (oracle/ks_oracle.c),
// to generate tests/golden/ fixtures, and as the timed CPU reference arm of
// bench.py.  The namespace is renamed at compile time
// (-Dkernelscope=kernelscope_ref) so it can never be confused with, or link
// against, the product's kernelscope:: drop-in.
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "kernelscope/conv_core.hpp"
#include "kernelscope/rng.hpp"

using namespace kernelscope;
using conv::AccumulationScheme;
using conv::MulAddMode;

namespace {

template <typename T>
Tensor3T<T> wrap3(const T* p, std::int64_t B, std::int64_t H, std::int64_t L) {
    Tensor3T<T> t(B, H, L);
    std::memcpy(t.data.data(), p, sizeof(T) * t.data.size());
    return t;
}

template <typename T>
Kernel2T<T> wrap2(const T* p, std::int64_t H, std::int64_t K) {
    Kernel2T<T> k(H, K);
    std::memcpy(k.data.data(), p, sizeof(T) * k.data.size());
    return k;
}

AccumulationScheme scheme_of(int scheme, std::int64_t chunk) {
    switch (scheme) {
        case 1: return AccumulationScheme::pairwise();
        case 2: return AccumulationScheme::chunked(chunk);
        default: return AccumulationScheme::sequential();
    }
}

MulAddMode mode_of(int mode) { return mode == 1 ? MulAddMode::Fused : MulAddMode::Separate; }

template <typename T>
int run_path(int path, const T* a, const T* b, T* out, std::int64_t B, std::int64_t H,
             std::int64_t L, std::int64_t K, int scheme, std::int64_t chunk, int mode) {
    try {
        const ConvShape s(B, H, L, K);
        if (path == 0) {
            auto y = conv::forward(wrap3(a, B, H, L), wrap2(b, H, K), s, mode_of(mode));
            std::memcpy(out, y.data.data(), sizeof(T) * y.data.size());
        } else if (path == 1) {
            auto dx = conv::backward_input(wrap3(a, B, H, L), wrap2(b, H, K), s, mode_of(mode));
            std::memcpy(out, dx.data.data(), sizeof(T) * dx.data.size());
        } else {
            auto dk = conv::backward_weight(wrap3(a, B, H, L), wrap3(b, B, H, L), s,
                                            scheme_of(scheme, chunk), mode_of(mode));
            std::memcpy(out, dk.data.data(), sizeof(T) * dk.data.size());
        }
        return 0;
    } catch (const DimensionError&) {
        return -1;
    }
}

// Channel-sliced fan-out: every thread gathers channel h into a ConvShape(B,1,L,K)
// problem, runs the reference on it and scatters the result back.  Channels are
// independent, so this is bitwise identical to the single call.
int run_path_mt(int path, const float* a, const float* b, float* out, std::int64_t B,
                std::int64_t H, std::int64_t L, std::int64_t K, int scheme, std::int64_t chunk,
                int mode, int threads) {
    if (threads < 1) threads = 1;
    if (threads > H) threads = static_cast<int>(H);
    std::vector<std::thread> pool;
    std::vector<int> rc(static_cast<std::size_t>(threads), 0);
    for (int i = 0; i < threads; ++i) {
        pool.emplace_back([=, &rc] {
            const std::int64_t h0 = H * i / threads, h1 = H * (i + 1) / threads;
            std::vector<float> sa(static_cast<std::size_t>(B * L));
            std::vector<float> sb(path == 2 ? static_cast<std::size_t>(B * L)
                                            : static_cast<std::size_t>(K));
            std::vector<float> so(path == 2 ? static_cast<std::size_t>(K)
                                            : static_cast<std::size_t>(B * L));
            for (std::int64_t h = h0; h < h1; ++h) {
                for (std::int64_t bb = 0; bb < B; ++bb)
                    std::memcpy(&sa[bb * L], a + (bb * H + h) * L, sizeof(float) * L);
                if (path == 2) {
                    for (std::int64_t bb = 0; bb < B; ++bb)
                        std::memcpy(&sb[bb * L], b + (bb * H + h) * L, sizeof(float) * L);
                } else {
                    std::memcpy(sb.data(), b + h * K, sizeof(float) * K);
                }
                rc[i] |= run_path<float>(path, sa.data(), sb.data(), so.data(), B, 1, L, K,
                                         scheme, chunk, mode);
                if (path == 2) {
                    std::memcpy(out + h * K, so.data(), sizeof(float) * K);
                } else {
                    for (std::int64_t bb = 0; bb < B; ++bb)
                        std::memcpy(out + (bb * H + h) * L, &so[bb * L], sizeof(float) * L);
                }
            }
        });
    }
    for (auto& t : pool) t.join();
    for (int r : rc)
        if (r) return r;
    return 0;
}

} // namespace

extern "C" {

int ksref_forward_f32(const float* x, const float* k, float* y, std::int64_t B, std::int64_t H,
                      std::int64_t L, std::int64_t K, int mode) {
    return run_path<float>(0, x, k, y, B, H, L, K, 0, 0, mode);
}
int ksref_forward_f64(const double* x, const double* k, double* y, std::int64_t B,
                      std::int64_t H, std::int64_t L, std::int64_t K, int mode) {
    return run_path<double>(0, x, k, y, B, H, L, K, 0, 0, mode);
}
int ksref_backward_input_f32(const float* gy, const float* k, float* dx, std::int64_t B,
                             std::int64_t H, std::int64_t L, std::int64_t K, int mode) {
    return run_path<float>(1, gy, k, dx, B, H, L, K, 0, 0, mode);
}
int ksref_backward_input_f64(const double* gy, const double* k, double* dx, std::int64_t B,
                             std::int64_t H, std::int64_t L, std::int64_t K, int mode) {
    return run_path<double>(1, gy, k, dx, B, H, L, K, 0, 0, mode);
}
int ksref_backward_weight_f32(const float* gy, const float* x, float* dk, std::int64_t B,
                              std::int64_t H, std::int64_t L, std::int64_t K, int scheme,
                              std::int64_t chunk, int mode) {
    return run_path<float>(2, gy, x, dk, B, H, L, K, scheme, chunk, mode);
}
int ksref_backward_weight_f64(const double* gy, const double* x, double* dk, std::int64_t B,
                              std::int64_t H, std::int64_t L, std::int64_t K, int scheme,
                              std::int64_t chunk, int mode) {
    return run_path<double>(2, gy, x, dk, B, H, L, K, scheme, chunk, mode);
}
int ksref_forward_f32_mt(const float* x, const float* k, float* y, std::int64_t B,
                         std::int64_t H, std::int64_t L, std::int64_t K, int mode, int threads) {
    return run_path_mt(0, x, k, y, B, H, L, K, 0, 0, mode, threads);
}
int ksref_backward_input_f32_mt(const float* gy, const float* k, float* dx, std::int64_t B,
                                std::int64_t H, std::int64_t L, std::int64_t K, int mode,
                                int threads) {
    return run_path_mt(1, gy, k, dx, B, H, L, K, 0, 0, mode, threads);
}
int ksref_backward_weight_f32_mt(const float* gy, const float* x, float* dk, std::int64_t B,
                                 std::int64_t H, std::int64_t L, std::int64_t K, int scheme,
                                 std::int64_t chunk, int mode, int threads) {
    return run_path_mt(2, gy, x, dk, B, H, L, K, scheme, chunk, mode, threads);
}

// validate()'s input stream: x (B*H*L draws), then k (H*K), then gy (B*H*L)
// from SplitMix64(seed) (src/conv_core.cpp:241-247).
void ksref_fill_inputs(std::uint64_t seed, float* x, float* k, float* gy, std::int64_t B,
                       std::int64_t H, std::int64_t L, std::int64_t K) {
    SplitMix64 rng(seed);
    Tensor3 tx(B, H, L), tg(B, H, L);
    Kernel2 tk(H, K);
    fill_pm1(rng, tx);
    fill_pm1(rng, tk);
    fill_pm1(rng, tg);
    std::memcpy(x, tx.data.data(), sizeof(float) * tx.data.size());
    std::memcpy(k, tk.data.data(), sizeof(float) * tk.data.size());
    std::memcpy(gy, tg.data.data(), sizeof(float) * tg.data.size());
}

// conv::validate (src/conv_core.cpp:236-280) with the given schemes; writes
// fwd/bwd_in max_abs,max_rel, per-scheme dk max_abs,max_rel and the spread.
int ksref_validate(std::int64_t B, std::int64_t H, std::int64_t L, std::int64_t K,
                   std::uint64_t seed, const int* schemes, const std::int64_t* chunks,
                   int n_schemes, double* out /* 4 + 2*n + 2 */) {
    try {
        std::vector<AccumulationScheme> v;
        for (int i = 0; i < n_schemes; ++i) v.push_back(scheme_of(schemes[i], chunks[i]));
        const auto rep = conv::validate(ConvShape(B, H, L, K), seed, v);
        out[0] = rep.fwd.max_abs;
        out[1] = rep.fwd.max_rel;
        out[2] = rep.bwd_in.max_abs;
        out[3] = rep.bwd_in.max_rel;
        for (int i = 0; i < n_schemes; ++i) {
            out[4 + 2 * i] = rep.dk[i].err.max_abs;
            out[5 + 2 * i] = rep.dk[i].err.max_rel;
        }
        out[4 + 2 * n_schemes] = rep.dk_spread_abs;
        out[5 + 2 * n_schemes] = rep.dk_spread_rel;
        return 0;
    } catch (const DimensionError&) {
        return -1;
    }
}

} // extern "C"
