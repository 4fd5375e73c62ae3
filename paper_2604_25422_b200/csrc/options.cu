// options.cu -- the library's tuning options (tier switches and pipeline
// depths), set explicitly through ks_set_option() and read once per call from
// an atomic table.
//
// Every default is the measured choice (DESIGN.md §5 lists the A/B behind
// each).  Options exist so tests can pin two tiers against each other bit for
// bit and so experiments can sweep a depth without a rebuild; the product
// never reads the environment.  A tuning build (-DKS_TUNING_ENV, see
// tools/build_variant.sh) additionally seeds the table once, at the first
// option read, from environment variables named KS_<NAME>.
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "ks_common.cuh"

namespace ks {

namespace {

struct OptDef {
    const char* name;
    int64_t dflt, lo, hi;
};

// order = enum Opt (ks_common.cuh)
constexpr OptDef kDefs[kOptCount] = {
    {"disable_tma", 0, 0, 1},    // 1: generic (non-TMA) kernels only
    {"ldg", 1, 0, 2},            // stencil_ldg for fwd/dX (L >= 256): 0 never, 1 auto (K <= 10; L < 2048: K <= 12, Fused K <= 16 from L = 1024; L < 1024: K <= 32), 2 K <= 32
    {"sts", 1, 0, 2},            // fwd/dX through bwd_short: 0 never (stencil_tma), 1 auto (K <= 16; Separate K <= 28, Fused K <= 32 from L = 4096), 2 K <= 32
    {"bwds", 1, 0, 1},           // dW (K <= 32) / fused backward (K <= 16) through bwd_short (0: dw_tma)
    {"dst", 0, 0, 1},            // bwd_short stencil outputs by 256-bit stores instead of TMA stores
    {"dwtma_j16", 1, 0, 1},      // dw_tma: one 16-tap group for 8 < K <= 16 (0: two 8-tap groups)
    {"dwtma_ns", 0, 0, 6},       // dw_tma stages (0: auto)
    {"pad_skip", 1, 0, 1},       // stencil_pad / dw_pad: skip all-halo tap blocks
    {"pad_ns", 0, 0, 4},         // stencil_pad stages (0: auto)
    {"pad_prod", -1, -1, 1},     // stencil_pad producer lane (1) or CTA-barrier refill (0); -1 auto
    {"dwpad_ns", 0, 0, 4},       // dw_pad stages (0: auto)
    {"stencil_pad", 1, 0, 2},    // K > 32 fwd/dX through stencil_pad: 0 never (stencil_tma), 1 auto (not Separate K < 1024), 2 always
    {"stencil_r", 0, 0, 32},     // stencil_tma register tile (0: auto, 32: R = 32 at short K)
    {"stencil_nt", 0, 0, 1024},  // stencil_tma threads (0: auto)
    {"stencil_ns", 0, 0, 8},     // stencil_tma stages (0: auto)
    {"host_block_mb", 64, 1, 4096},  // host-buffer entry points: bytes per streamed block
    {"stencil_bl", -1, -1, 1},   // stencil_pad's batch-lane kernel: 1 always, 0 never, -1 auto (K >= L / 4)
    {"dw_ctas", 8192, 64, 1 << 20},
    {"dw_mrow", 1, 0, 1},
    {"dwpad_min_k", 48, 17, 8192},   // smallest K whose dW takes dw_pad (below: dw_tma)        // K <= 16 dW with L < 2048: items of whole rows (0: one 2048-wide tile per row)
    {"sts_rows", -1, -1, 1},     // bwd_short stencils: one CTA per row (1), persistent grid (0), -1 auto (rows in Fused mode)  // HIERARCHICAL stage 1 (dw_tma / bwd_short / dw_rows / generic): target CTAs (sets G)
    {"pdl", -1, -1, 1},          // programmatic dependent launch of the kernels after prep_taps / stage 1: 1 on, 0 off, -1 small grids
};

std::atomic<int64_t> g_opts[kOptCount];
std::once_flag g_once;

void init_opts() {
    for (int i = 0; i < kOptCount; ++i) g_opts[i].store(kDefs[i].dflt, std::memory_order_relaxed);
#ifdef KS_TUNING_ENV
    for (int i = 0; i < kOptCount; ++i) {
        char env[64] = "KS_";
        for (int c = 0; kDefs[i].name[c] && c < 56; ++c) {
            const char ch = kDefs[i].name[c];
            env[3 + c] = (ch >= 'a' && ch <= 'z') ? static_cast<char>(ch - 32) : ch;
            env[4 + c] = '\0';
        }
        if (const char* v = getenv(env)) {
            const long long x = atoll(v);
            if (x >= kDefs[i].lo && x <= kDefs[i].hi) g_opts[i].store(x, std::memory_order_relaxed);
        }
    }
#endif
}

int find(const char* name) {
    if (!name) return -1;
    for (int i = 0; i < kOptCount; ++i)
        if (strcmp(kDefs[i].name, name) == 0) return i;
    return -1;
}

}  // namespace

int64_t opt_pdl() { return opt(kOptPdl); }

int64_t opt(Opt o) {
    std::call_once(g_once, init_opts);
    return g_opts[o].load(std::memory_order_relaxed);
}

}  // namespace ks

using namespace ks;

extern "C" {

ks_status ks_set_option(const char* name, int64_t value) {
    const int i = find(name);
    if (i < 0) return KS_ERR_BAD_OPTION;
    std::call_once(g_once, init_opts);
    if (value == KS_OPTION_DEFAULT) value = kDefs[i].dflt;
    if (value < kDefs[i].lo || value > kDefs[i].hi) return KS_ERR_BAD_OPTION;
    g_opts[i].store(value, std::memory_order_relaxed);
    return KS_OK;
}

ks_status ks_get_option(const char* name, int64_t* value) {
    if (!value) return KS_ERR_NULL;
    const int i = find(name);
    if (i < 0) return KS_ERR_BAD_OPTION;
    *value = opt(static_cast<Opt>(i));
    return KS_OK;
}

}  // extern "C"
