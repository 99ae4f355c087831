// Kernel-choice switches: see options.h and sewald_gpu_set_option.
#include "options.h"

#include <atomic>
#include <cstdlib>
#include <cstring>

namespace sewald_b200 {
namespace {

int env_default(int which) {
    auto env = [](const char* n) { return getenv(n); };
    const char* e = nullptr;
    switch (which) {
        case SEWALD_OPT_RS_SYM:  // 0 never, 1 auto, 2 force (targets == sources)
            e = env("SEWALD_RS_SYM");
            if (!e) return 1;
            if (e[0] == '0') return 0;
            return strcmp(e, "force") == 0 ? 2 : 1;
        case SEWALD_OPT_GATHER:  // -1 auto, 0 warp, 1 z-sweep, 2 tiles
            e = env("SEWALD_GATHER");
            if (!e) return -1;
            if (!strcmp(e, "warp")) return 0;
            if (!strcmp(e, "sweep")) return 1;
            if (!strcmp(e, "tile")) return 2;
            return -1;
        case SEWALD_OPT_GATHER_MMA:
            e = env("SEWALD_GATHER_MMA");
            return (e && e[0] == '0') ? 0 : 1;
        case SEWALD_OPT_GATHER_L:
            e = env("SEWALD_GATHER_L");
            return e ? atoi(e) : 0;
        case SEWALD_OPT_SPREAD_SWEEP:
            e = env("SEWALD_SPREAD_SWEEP");
            return e && e[0] ? (e[0] == '0' ? 0 : 1) : -1;
        case SEWALD_OPT_SPREAD_MMA:
            e = env("SEWALD_SPREAD_MMA");
            return (e && e[0] == '0') ? 0 : 1;
        case SEWALD_OPT_SPREAD_MMA_L:
            e = env("SEWALD_SPREAD_MMA_L");
            return e ? atoi(e) : 23;
        case SEWALD_OPT_SPREAD_CACHED:
            e = env("SEWALD_SPREAD_CACHED");
            return (e && e[0] == '0') ? 0 : 1;
        case SEWALD_OPT_SPREAD_ROWSWEEP:
            e = env("SEWALD_SPREAD_ROWSWEEP");
            return (e && e[0] == '1') ? 1 : 0;
        case SEWALD_OPT_SPREAD_FUSED:
            e = env("SEWALD_SPREAD_FUSED");
            return (e && e[0] == '0') ? 0 : 1;
        case SEWALD_OPT_GATHER_WIDE:
            e = env("SEWALD_GATHER_WIDE");
            return e ? atoi(e) : 2;
        case SEWALD_OPT_GATHER_FUSED:
            e = env("SEWALD_GATHER_FUSED");
            return (e && e[0] == '1') ? 1 : 0;
        case SEWALD_OPT_SPREAD_SORT:
            e = env("SEWALD_SPREAD_SORT");
            return (e && e[0] == '0') ? 0 : 1;
        case SEWALD_OPT_GATHER_SORT:
            e = env("SEWALD_GATHER_SORT");
            return (e && e[0] == '0') ? 0 : 1;
        case SEWALD_OPT_D0_YFUSED:
            e = env("SEWALD_D0_YFUSED");
            return (e && e[0] == '0') ? 0 : 1;
    }
    return 0;
}

bool valid(int which, int v) {
    switch (which) {
        case SEWALD_OPT_RS_SYM: return v >= 0 && v <= 2;
        case SEWALD_OPT_GATHER: return v >= -1 && v <= 2;
        case SEWALD_OPT_GATHER_MMA: return v == 0 || v == 1;
        case SEWALD_OPT_GATHER_L: return v == 0 || v == 15 || v == 19 || v == 23 || v == 31;
        case SEWALD_OPT_SPREAD_SWEEP: return v >= -1 && v <= 1;
        case SEWALD_OPT_SPREAD_MMA: return v == 0 || v == 1;
        case SEWALD_OPT_SPREAD_MMA_L: return v == 19 || v == 23;
        case SEWALD_OPT_SPREAD_CACHED: return v == 0 || v == 1;
        case SEWALD_OPT_SPREAD_ROWSWEEP: return v == 0 || v == 1;
        case SEWALD_OPT_SPREAD_FUSED: return v == 0 || v == 1 || v == 2;
        case SEWALD_OPT_GATHER_WIDE: return v >= 0 && v <= 2;
        case SEWALD_OPT_GATHER_FUSED: return v == 0 || v == 1;
        case SEWALD_OPT_SPREAD_SORT: return v == 0 || v == 1;
        case SEWALD_OPT_GATHER_SORT: return v == 0 || v == 1;
        case SEWALD_OPT_D0_YFUSED: return v == 0 || v == 1;
    }
    return false;
}

struct Table {
    std::atomic<int> v[SEWALD_OPT_COUNT];
    std::atomic<int> epoch{0};
    Table() {
        for (int i = 0; i < SEWALD_OPT_COUNT; ++i) v[i].store(env_default(i));
    }
};

Table& table() {
    static Table t;
    return t;
}

}  // namespace

int option(int which) { return (which >= 0 && which < SEWALD_OPT_COUNT) ? table().v[which].load() : 0; }

int options_epoch() { return table().epoch.load(); }

bool set_option(int which, int value) {
    if (which < 0 || which >= SEWALD_OPT_COUNT || !valid(which, value)) return false;
    table().v[which].store(value);
    table().epoch.fetch_add(1);
    return true;
}

}  // namespace sewald_b200

extern "C" {

int sewald_gpu_set_option(int which, int value) {
    return sewald_b200::set_option(which, value) ? SEWALD_OK : SEWALD_EINVAL;
}

int sewald_gpu_get_option(int which, int* value) {
    if (!value || which < 0 || which >= SEWALD_OPT_COUNT) return SEWALD_EINVAL;
    *value = sewald_b200::option(which);
    return SEWALD_OK;
}

}  // extern "C"
