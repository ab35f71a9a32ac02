// Library-level entry points of the C ABI (include/spamm_b200.h).
#include <stdlib.h>

#include <atomic>

#include "common.cuh"

static std::atomic<int64_t> g_launches{0};

void spamm_note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

bool spamm_pdl_enabled()
{
    static const bool on = [] {
        const char *e = getenv("SPAMM_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

int spamm_num_sms()
{
    static const int sms = [] {
        int dev = 0, n = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1)
            n = 148;      // B200
        return n;
    }();
    return sms;
}

extern "C" int64_t spamm_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

extern "C" int spamm_abi_version(void) { return SPAMM_ABI_VERSION; }

extern "C" int64_t spamm_level_offset_of(int t) { return spamm_level_offset(t); }

extern "C" const char *spamm_error_string(int code)
{
    switch (code) {
        case SPAMM_OK: return "ok";
        case SPAMM_EINVAL: return "invalid argument";
        case SPAMM_ECUDA: return "CUDA runtime error";
        case SPAMM_EWORKSPACE: return "workspace too small";
        default: return "unknown error";
    }
}
