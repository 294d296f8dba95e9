// options.cpp — option table (options.h): defaults, valid values, the
// environment at first use, and the per-process overrides of oz2g_set_option.
#include "options.h"

#include <atomic>
#include <cctype>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

namespace oz2g {

namespace {

struct Spec {
    const char* name;
    long long def;
    long long lo, hi;          // valid range
    const long long* allowed;  // or an explicit list (terminated by INT64 min)
};

constexpr long long kEnd = LLONG_MIN;
const long long kCv[] = {4, 8, kEnd};
const long long kEpi[] = {0, 4, 8, kEnd};
const long long kStages[] = {4, 5, 6, kEnd};
const long long kRowscan[] = {0, 256, 512, 1024, kEnd};

const Spec kSpecs[OPT_COUNT] = {
    {"gemm", 0, 0, 2, nullptr},
    {"fused", 0, 0, 2, nullptr},
    {"fused_mc", 0, 0, 1, nullptr},
    {"fused_fence", 1, 0, 1, nullptr},
    {"spec", -1, -1, 2, nullptr},
    {"graph", 1, 0, 1, nullptr},
    {"pdl", 1, 0, 2, nullptr},
    {"group_m", 0, 0, 1 << 20, nullptr},
    {"group_n", 0, 0, 1 << 20, nullptr},
    {"l2hint", 0, 0, 3, nullptr},
    {"crt_overlap", 0, 0, 64, nullptr},
    {"crt_cv", 8, 0, 0, kCv},
    {"wblock_min_mb", 2048, 0, 1ll << 40, nullptr},
    {"gemm_fence", 0, 0, 1, nullptr},
    {"epi_warps", 0, 0, 0, kEpi},
    {"pair_stages", 4, 0, 0, kStages},
    {"rowscan_threads", 0, 0, 0, kRowscan},
    {"resid_stream", 0, 0, 1, nullptr},
    {"spec_tail", 1, 1, 3, nullptr},
    {"dist_pipeline", 1, 0, 1, nullptr},
    {"debug_sync", 0, 0, 1, nullptr},
    {"resid_fast", 1, 0, 1, nullptr},
};

bool valid(const Spec& s, long long v) {
    if (s.allowed) {
        for (const long long* a = s.allowed; *a != kEnd; ++a)
            if (*a == v) return true;
        return false;
    }
    return v >= s.lo && v <= s.hi;
}

std::atomic<long long> g_vals[OPT_COUNT];
std::once_flag g_once;

// OZ2G_<NAME>: an integer in range, or for "gemm" the variant's name; an
// unparsable or out-of-range value keeps the default (as before the table).
void init_from_env() {
    for (int i = 0; i < OPT_COUNT; ++i) {
        const Spec& s = kSpecs[i];
        long long v = s.def;
        std::string env = "OZ2G_";
        for (const char* c = s.name; *c; ++c) env += (char)std::toupper((unsigned char)*c);
        if (const char* e = std::getenv(env.c_str())) {
            if (i == OPT_GEMM && std::strcmp(e, "pair") == 0) v = 1;
            else if (i == OPT_GEMM && std::strcmp(e, "mcast") == 0) v = 2;
            else if (i != OPT_GEMM || std::isdigit((unsigned char)e[0])) {
                char* end = nullptr;
                const long long x = std::strtoll(e, &end, 10);
                if (end != e && valid(s, x)) v = x;
            }
        }
        g_vals[i].store(v, std::memory_order_relaxed);
    }
}

}  // namespace

long long opt(Opt o) {
    std::call_once(g_once, init_from_env);
    return g_vals[o].load(std::memory_order_relaxed);
}

int opt_index(const char* name) {
    if (!name) return -1;
    for (int i = 0; i < OPT_COUNT; ++i)
        if (std::strcmp(name, kSpecs[i].name) == 0) return i;
    return -1;
}

const char* opt_name(int index) { return index >= 0 && index < OPT_COUNT ? kSpecs[index].name : nullptr; }

bool opt_set(int index, long long value) {
    if (index < 0 || index >= OPT_COUNT || !valid(kSpecs[index], value)) return false;
    std::call_once(g_once, init_from_env);
    g_vals[index].store(value, std::memory_order_relaxed);
    return true;
}

}  // namespace oz2g
