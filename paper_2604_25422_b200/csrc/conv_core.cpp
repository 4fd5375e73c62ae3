// conv_core.cpp -- the kernelscope::conv C++ API (drop-in for
// /root/reference/proj/src/conv_core.cpp) implemented over the C ABI.
//
// Shape checks happen here first, with the reference's exact DimensionError
// texts (tensor.hpp:79-105, src/conv_core.cpp:154-156); the arithmetic runs in
// the sm_100a kernels behind ks_dwconv1d_*_host.  A CUDA/NCCL failure or a
// missing device throws std::runtime_error -- there is no CPU fallback.
#include "kernelscope/conv_core.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>

#include "kernelscope/rng.hpp"
#include "ks_dwconv1d.h"

namespace kernelscope::conv {

namespace {

int mode_of(MulAddMode m) { return m == MulAddMode::Fused ? KS_MULADD_FUSED : KS_MULADD_SEPARATE; }

int scheme_of(const AccumulationScheme& s) {
    switch (s.kind) {
        case SumScheme::Sequential: return KS_DW_SEQUENTIAL;
        case SumScheme::PairwiseTree: return KS_DW_PAIRWISE;
        case SumScheme::ChunkedTwoStage: return KS_DW_CHUNKED;
        case SumScheme::Hierarchical: return KS_DW_HIERARCHICAL;
    }
    return -1;
}

void throw_on(ks_status s, const char* what) {
    if (s == KS_OK) return;
    std::string msg = std::string(what) + ": " + ks_status_string(s);
    const std::string detail = ks_last_error_string();
    if (!detail.empty()) msg += " (" + detail + ")";
    switch (s) {
        case KS_ERR_DIM_B:
        case KS_ERR_DIM_H:
        case KS_ERR_DIM_L:
        case KS_ERR_DIM_K:
        case KS_ERR_BAD_CHUNK: throw DimensionError(msg);
        default: throw std::runtime_error("kernelscope-b200 " + msg);
    }
}

template <typename T>
Tensor3T<T> forward_t(const Tensor3T<T>& x, const Kernel2T<T>& k, const ConvShape& s, MulAddMode mode) {
    check_tensor3(x, s, "forward: x");
    check_kernel2(k, s, "forward: k");
    Tensor3T<T> y(s.B, s.H, s.L);
    ks_status st;
    if constexpr (sizeof(T) == 4)
        st = ks_dwconv1d_fwd_f32_host(x.data.data(), k.data.data(), y.data.data(), s.B, s.H, s.L, s.K,
                                      mode_of(mode));
    else
        st = ks_dwconv1d_fwd_f64_host(x.data.data(), k.data.data(), y.data.data(), s.B, s.H, s.L, s.K,
                                      mode_of(mode));
    throw_on(st, "forward");
    return y;
}

template <typename T>
Tensor3T<T> backward_input_t(const Tensor3T<T>& gy, const Kernel2T<T>& k, const ConvShape& s,
                             MulAddMode mode) {
    check_tensor3(gy, s, "backward_input: gy");
    check_kernel2(k, s, "backward_input: k");
    Tensor3T<T> dx(s.B, s.H, s.L);
    ks_status st;
    if constexpr (sizeof(T) == 4)
        st = ks_dwconv1d_dx_f32_host(gy.data.data(), k.data.data(), dx.data.data(), s.B, s.H, s.L, s.K,
                                     mode_of(mode));
    else
        st = ks_dwconv1d_dx_f64_host(gy.data.data(), k.data.data(), dx.data.data(), s.B, s.H, s.L, s.K,
                                     mode_of(mode));
    throw_on(st, "backward_input");
    return dx;
}

template <typename T>
Kernel2T<T> backward_weight_t(const Tensor3T<T>& gy, const Tensor3T<T>& x, const ConvShape& s,
                              const AccumulationScheme& scheme, MulAddMode mode) {
    check_tensor3(gy, s, "backward_weight: gy");
    check_tensor3(x, s, "backward_weight: x");
    if (scheme.kind == SumScheme::ChunkedTwoStage && scheme.chunk_size < 1)
        throw DimensionError("backward_weight: chunk_size must be >= 1, got " +
                             std::to_string(scheme.chunk_size));
    Kernel2T<T> dk(s.H, s.K);
    ks_status st;
    if constexpr (sizeof(T) == 4)
        st = ks_dwconv1d_dw_f32_host(gy.data.data(), x.data.data(), dk.data.data(), s.B, s.H, s.L, s.K,
                                     scheme_of(scheme), scheme.chunk_size, mode_of(mode));
    else
        st = ks_dwconv1d_dw_f64_host(gy.data.data(), x.data.data(), dk.data.data(), s.B, s.H, s.L, s.K,
                                     scheme_of(scheme), scheme.chunk_size, mode_of(mode));
    throw_on(st, "backward_weight");
    return dk;
}

template <typename C>
auto widen(const C& c) {
    if constexpr (std::is_same_v<C, Tensor3>) {
        Tensor3d out(c.B, c.H, c.L);
        std::copy(c.data.begin(), c.data.end(), out.data.begin());
        return out;
    } else {
        Kernel2d out(c.H, c.K);
        std::copy(c.data.begin(), c.data.end(), out.data.begin());
        return out;
    }
}

// Per-element error against the fp64 result rounded to fp32 (the reference's
// score(), src/conv_core.cpp:197-207).
template <typename CF, typename CD>
ErrorStat score(const CF& got, const CD& oracle) {
    ErrorStat e;
    for (std::size_t i = 0; i < got.data.size(); ++i) {
        const double ref = static_cast<double>(static_cast<float>(oracle.data[i]));
        const double diff = std::abs(static_cast<double>(got.data[i]) - ref);
        e.max_abs = std::max(e.max_abs, diff);
        e.max_rel = std::max(e.max_rel, diff / std::max(std::abs(ref), kRelErrFloor));
    }
    return e;
}

}  // namespace

Tensor3 forward(const Tensor3& x, const Kernel2& k, const ConvShape& s, MulAddMode m) {
    return forward_t(x, k, s, m);
}
Tensor3d forward(const Tensor3d& x, const Kernel2d& k, const ConvShape& s, MulAddMode m) {
    return forward_t(x, k, s, m);
}
Tensor3 backward_input(const Tensor3& gy, const Kernel2& k, const ConvShape& s, MulAddMode m) {
    return backward_input_t(gy, k, s, m);
}
Tensor3d backward_input(const Tensor3d& gy, const Kernel2d& k, const ConvShape& s, MulAddMode m) {
    return backward_input_t(gy, k, s, m);
}
Kernel2 backward_weight(const Tensor3& gy, const Tensor3& x, const ConvShape& s,
                        const AccumulationScheme& scheme, MulAddMode m) {
    return backward_weight_t(gy, x, s, scheme, m);
}
Kernel2d backward_weight(const Tensor3d& gy, const Tensor3d& x, const ConvShape& s,
                         const AccumulationScheme& scheme, MulAddMode m) {
    return backward_weight_t(gy, x, s, scheme, m);
}

// conv::validate (reference src/conv_core.cpp:236-280), on the GPU.
ValidationReport validate(const ConvShape& shape, std::uint64_t seed,
                          std::span<const AccumulationScheme> schemes) {
    if (schemes.empty()) throw DimensionError("validate: at least one accumulation scheme required");
    SplitMix64 rng(seed);
    Tensor3 x(shape.B, shape.H, shape.L);
    Kernel2 k(shape.H, shape.K);
    Tensor3 gy(shape.B, shape.H, shape.L);
    fill_pm1(rng, x);
    fill_pm1(rng, k);
    fill_pm1(rng, gy);
    const Tensor3d xd = widen(x);
    const Kernel2d kd = widen(k);
    const Tensor3d gyd = widen(gy);

    ValidationReport rep{shape, seed, {}, {}, {}, 0.0, 0.0};
    rep.fwd = score(forward(x, k, shape), forward(xd, kd, shape));
    rep.bwd_in = score(backward_input(gy, k, shape), backward_input(gyd, kd, shape));

    const Kernel2d dk_oracle = backward_weight(gyd, xd, shape, AccumulationScheme::sequential());
    double peak = 0.0;
    for (double v : dk_oracle.data) peak = std::max(peak, std::abs(v));

    std::vector<Kernel2> dks;
    dks.reserve(schemes.size());
    for (const auto& sc : schemes) {
        dks.push_back(backward_weight(gy, x, shape, sc));
        rep.dk.push_back({sc, score(dks.back(), dk_oracle)});
    }
    for (std::size_t a = 0; a < dks.size(); ++a)
        for (std::size_t b = a + 1; b < dks.size(); ++b)
            for (std::size_t i = 0; i < dks[a].data.size(); ++i)
                rep.dk_spread_abs = std::max(
                    rep.dk_spread_abs,
                    std::abs(static_cast<double>(dks[a].data[i]) - static_cast<double>(dks[b].data[i])));
    rep.dk_spread_rel = rep.dk_spread_abs / std::max(peak, kRelErrFloor);
    return rep;
}

std::vector<SweepStep> validate_sweep(const ConvShape& base, std::uint64_t seed, int steps,
                                      std::span<const AccumulationScheme> schemes) {
    std::vector<SweepStep> out;
    std::int64_t B = base.B;
    for (int i = 0; i < steps; ++i, B *= 4) {
        const ConvShape s(B, base.H, base.L, base.K);
        const ValidationReport rep = validate(s, seed + static_cast<std::uint64_t>(i), schemes);
        double dk_max = 0.0;
        for (const auto& e : rep.dk) dk_max = std::max(dk_max, e.err.max_abs);
        out.push_back({s, s.flat_reduction(), rep.fwd, rep.bwd_in, dk_max, rep.dk_spread_abs, rep.dk_spread_rel});
    }
    return out;
}

int sweep_nondecreasing_steps(std::span<const SweepStep> sweep) {
    int n = 0;
    for (std::size_t i = 1; i < sweep.size(); ++i)
        if (sweep[i].dk_max_abs >= sweep[i - 1].dk_max_abs) ++n;
    return n;
}

}  // namespace kernelscope::conv
