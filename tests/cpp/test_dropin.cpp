// test_dropin.cpp -- C++ tests of the kernelscope::conv drop-in (GPU).
//
// Complements the reference's own tests/test_conv_core.cpp (built against this
// library as oracle/_ref/ref_test_conv_core): here every path is compared
// bit-for-bit with the plain-C restatement in oracle/ks_oracle.c (TEST
// INFRASTRUCTURE, linked only into this test), across both MulAddModes, every
// reference scheme, odd/even K, K > L, ragged L and the DimensionError contract.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "kernelscope/conv_core.hpp"
#include "kernelscope/rng.hpp"
#include "ks_oracle.h"

using namespace kernelscope;
using conv::AccumulationScheme;
using conv::MulAddMode;

namespace {

struct Case {
    Tensor3 x, gy;
    Kernel2 k;
};

Case make_case(const ConvShape& s, std::uint64_t seed) {
    SplitMix64 rng(seed);
    Case c{Tensor3(s.B, s.H, s.L), Tensor3(s.B, s.H, s.L), Kernel2(s.H, s.K)};
    fill_pm1(rng, c.x);
    fill_pm1(rng, c.k);
    fill_pm1(rng, c.gy);
    return c;
}

template <typename V>
bool same_bits(const V& a, const V& b) {
    return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(a[0])) == 0;
}

const ConvShape kShapes[] = {
    {1, 1, 3, 3},   {2, 3, 17, 5},  {2, 2, 5, 4},    {3, 2, 33, 8},   {2, 2, 10, 16},
    {4, 3, 64, 1},  {2, 2, 7, 12},  {1, 2, 300, 7},  {2, 1, 1030, 64}, {3, 2, 4099, 9},
    {2, 2, 257, 200}, {16, 4, 1024, 64}, {2, 1, 8192, 7}, {1, 1, 5000, 33},
};

}  // namespace

TEST_CASE("forward and backward_input are bitwise equal to the restated reference") {
    for (const auto& s : kShapes) {
        const auto c = make_case(s, 7 + static_cast<std::uint64_t>(s.L));
        for (int m = 0; m < 2; ++m) {
            const auto mode = m ? MulAddMode::Fused : MulAddMode::Separate;
            const auto y = conv::forward(c.x, c.k, s, mode);
            std::vector<float> yo(static_cast<std::size_t>(s.tensor_elems()));
            kso_forward_f32(c.x.data.data(), c.k.data.data(), yo.data(), s.B, s.H, s.L, s.K, m);
            CHECK(same_bits(y.data, yo));
            const auto dx = conv::backward_input(c.gy, c.k, s, mode);
            std::vector<float> dxo(static_cast<std::size_t>(s.tensor_elems()));
            kso_backward_input_f32(c.gy.data.data(), c.k.data.data(), dxo.data(), s.B, s.H, s.L, s.K, m);
            CHECK(same_bits(dx.data, dxo));
        }
    }
}

TEST_CASE("backward_weight reference schemes are bitwise equal") {
    for (const auto& s : kShapes) {
        if (s.tensor_elems() > 200000) continue;  // sequential chains are slow at depth
        const auto c = make_case(s, 3 + static_cast<std::uint64_t>(s.K));
        const AccumulationScheme schemes[] = {AccumulationScheme::sequential(), AccumulationScheme::pairwise(),
                                              AccumulationScheme::chunked(7), AccumulationScheme::chunked(1024),
                                              AccumulationScheme::chunked(1 << 30)};
        for (const auto& sc : schemes) {
            for (int m = 0; m < 2; ++m) {
                const auto dk = conv::backward_weight(c.gy, c.x, s, sc, m ? MulAddMode::Fused : MulAddMode::Separate);
                std::vector<float> dko(static_cast<std::size_t>(s.kernel_elems()));
                const int ks = sc.kind == conv::SumScheme::PairwiseTree ? KSO_PAIRWISE
                               : sc.kind == conv::SumScheme::ChunkedTwoStage ? KSO_CHUNKED
                                                                             : KSO_SEQUENTIAL;
                kso_backward_weight_f32(c.gy.data.data(), c.x.data.data(), dko.data(), s.B, s.H, s.L, s.K, ks,
                                        sc.chunk_size, m);
                CHECK(same_bits(dk.data, dko));
            }
        }
    }
}

TEST_CASE("double overloads are bitwise equal to the restated reference") {
    for (const auto& s : {ConvShape(2, 3, 17, 5), ConvShape(3, 2, 33, 8), ConvShape(2, 2, 100, 31)}) {
        const auto c = make_case(s, 11);
        Tensor3d xd(s.B, s.H, s.L), gyd(s.B, s.H, s.L);
        Kernel2d kd(s.H, s.K);
        std::copy(c.x.data.begin(), c.x.data.end(), xd.data.begin());
        std::copy(c.gy.data.begin(), c.gy.data.end(), gyd.data.begin());
        std::copy(c.k.data.begin(), c.k.data.end(), kd.data.begin());
        std::vector<double> o(static_cast<std::size_t>(s.tensor_elems()));
        kso_forward_f64(xd.data.data(), kd.data.data(), o.data(), s.B, s.H, s.L, s.K, 0);
        CHECK(same_bits(conv::forward(xd, kd, s).data, o));
        kso_backward_input_f64(gyd.data.data(), kd.data.data(), o.data(), s.B, s.H, s.L, s.K, 1);
        CHECK(same_bits(conv::backward_input(gyd, kd, s, MulAddMode::Fused).data, o));
        std::vector<double> ok(static_cast<std::size_t>(s.kernel_elems()));
        kso_backward_weight_f64(gyd.data.data(), xd.data.data(), ok.data(), s.B, s.H, s.L, s.K, KSO_SEQUENTIAL, 0, 0);
        CHECK(same_bits(conv::backward_weight(gyd, xd, s, AccumulationScheme::sequential()).data, ok));
        kso_backward_weight_f64(gyd.data.data(), xd.data.data(), ok.data(), s.B, s.H, s.L, s.K, KSO_PAIRWISE, 0, 0);
        CHECK(same_bits(conv::backward_weight(gyd, xd, s, AccumulationScheme::pairwise()).data, ok));
    }
}

TEST_CASE("hierarchical dW is deterministic and within 1e-4 normwise of the fp64 truth") {
    for (const auto& s : kShapes) {
        const auto c = make_case(s, 5);
        const auto a = conv::backward_weight(c.gy, c.x, s, AccumulationScheme::hierarchical(), MulAddMode::Fused);
        const auto b = conv::backward_weight(c.gy, c.x, s, AccumulationScheme::hierarchical(), MulAddMode::Fused);
        CHECK(same_bits(a.data, b.data));
        std::vector<double> gyd(c.gy.data.begin(), c.gy.data.end()), xd(c.x.data.begin(), c.x.data.end());
        std::vector<double> truth(static_cast<std::size_t>(s.kernel_elems()));
        kso_backward_weight_f64(gyd.data(), xd.data(), truth.data(), s.B, s.H, s.L, s.K, KSO_PAIRWISE, 0, 0);
        double peak = 0, diff = 0;
        for (std::size_t i = 0; i < truth.size(); ++i) {
            peak = std::max(peak, std::abs(truth[i]));
            diff = std::max(diff, std::abs(truth[i] - static_cast<double>(a.data[i])));
        }
        CHECK(diff <= 1e-4 * std::max(peak, 1e-12));
    }
}

TEST_CASE("dimension errors keep the reference's axis text") {
    const ConvShape s(2, 2, 5, 4);
    const auto c = make_case(s, 3);
    CHECK_THROWS_WITH_AS(conv::forward(Tensor3(2, 2, 6), c.k, s), doctest::Contains("axis L"), DimensionError);
    CHECK_THROWS_WITH_AS(conv::forward(c.x, Kernel2(2, 3), s), doctest::Contains("axis K"), DimensionError);
    CHECK_THROWS_WITH_AS(conv::backward_input(Tensor3(3, 2, 5), c.k, s), doctest::Contains("axis B"), DimensionError);
    CHECK_THROWS_WITH_AS(conv::backward_weight(c.gy, Tensor3(2, 3, 5), s, AccumulationScheme::sequential()),
                         doctest::Contains("axis H"), DimensionError);
    AccumulationScheme bad{conv::SumScheme::ChunkedTwoStage, 0};
    CHECK_THROWS_AS(conv::backward_weight(c.gy, c.x, s, bad), DimensionError);
    CHECK_THROWS_AS(AccumulationScheme::chunked(0), DimensionError);
}

TEST_CASE("validate on the GPU keeps the reference's bounds") {
    const AccumulationScheme schemes[] = {AccumulationScheme::sequential(), AccumulationScheme::chunked(1024)};
    const auto rep = conv::validate(ConvShape(64, 8, 48, 48), 1, schemes);
    CHECK(rep.fwd.max_abs <= 4e-6);
    CHECK(rep.fwd.max_abs > 0.0);
    CHECK(rep.bwd_in.max_abs <= 4e-6);
    CHECK(rep.dk_spread_abs > 0.0);
}

TEST_CASE("concurrent callers: the drop-in is safe for concurrent use (SPEC.md:120-121)") {
    // 8 host threads call forward / backward_input / backward_weight at once,
    // each on its own shape and data (every call takes its own streams and the
    // library's scratch pool, first created under a lock); every result must
    // equal the same call made alone.
    constexpr int kThreads = 8;
    std::vector<ConvShape> shapes;
    std::vector<Case> cases;
    for (int i = 0; i < kThreads; ++i) {
        shapes.push_back(ConvShape(2 + i % 3, 3 + i % 2, 2048 + 32 * i, 3 + 2 * i));
        cases.push_back(make_case(shapes.back(), 100 + static_cast<std::uint64_t>(i)));
    }
    struct Out {
        Tensor3 y{1, 1, 1}, dx{1, 1, 1};
        Kernel2 dk{1, 1}, dkh{1, 1};
    };
    auto run = [&](int i, Out& o) {
        const auto& s = shapes[static_cast<std::size_t>(i)];
        const auto& c = cases[static_cast<std::size_t>(i)];
        const auto mode = i % 2 ? MulAddMode::Fused : MulAddMode::Separate;
        o.y = conv::forward(c.x, c.k, s, mode);
        o.dx = conv::backward_input(c.gy, c.k, s, mode);
        o.dk = conv::backward_weight(c.gy, c.x, s, AccumulationScheme::chunked(512), mode);
        o.dkh = conv::backward_weight(c.gy, c.x, s, AccumulationScheme::hierarchical(), mode);
    };
    std::vector<Out> alone(kThreads), together(kThreads);
    for (int i = 0; i < kThreads; ++i) run(i, alone[static_cast<std::size_t>(i)]);
    for (int rep = 0; rep < 3; ++rep) {
        std::vector<std::thread> ts;
        for (int i = 0; i < kThreads; ++i) ts.emplace_back(run, i, std::ref(together[static_cast<std::size_t>(i)]));
        for (auto& t : ts) t.join();
        for (int i = 0; i < kThreads; ++i) {
            const auto& a = alone[static_cast<std::size_t>(i)];
            const auto& b = together[static_cast<std::size_t>(i)];
            CHECK(same_bits(a.y.data, b.y.data));
            CHECK(same_bits(a.dx.data, b.dx.data));
            CHECK(same_bits(a.dk.data, b.dk.data));
            CHECK(same_bits(a.dkh.data, b.dkh.data));
        }
    }
}
