// Multi-GPU helper of the C ABI: the one exchange step of the row-block split, for hosts that hold an
// ncclComm_t.  The library does not link NCCL: the few entry points it needs are
// looked up in the running process (dlsym), so it uses whichever NCCL the host has loaded -- PyTorch's
// bundled one, or the system's -- and the library stays loadable where there is none.
// The reference is single process; this has no counterpart there.
#include <dlfcn.h>

#include "common.cuh"

namespace {
typedef int (*nccl_all_gather_t)(const void *, void *, size_t, int, void *, cudaStream_t);
typedef int (*nccl_group_t)(void);
struct NcclApi {
    nccl_all_gather_t all_gather = nullptr;
    nccl_group_t group_start = nullptr, group_end = nullptr;
    bool ok = false;
};
const NcclApi &nccl_api()
{
    static const NcclApi api = [] {
        NcclApi a;
        void *h = RTLD_DEFAULT;
        a.all_gather = reinterpret_cast<nccl_all_gather_t>(dlsym(h, "ncclAllGather"));
        if (!a.all_gather) {          // not loaded yet by the host: try the usual names
            for (const char *name : {"libnccl.so.2", "libnccl.so"}) {
                if (void *lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL)) {
                    h = lib;
                    a.all_gather = reinterpret_cast<nccl_all_gather_t>(dlsym(h, "ncclAllGather"));
                    if (a.all_gather) break;
                }
            }
        }
        a.group_start = reinterpret_cast<nccl_group_t>(dlsym(h, "ncclGroupStart"));
        a.group_end = reinterpret_cast<nccl_group_t>(dlsym(h, "ncclGroupEnd"));
        a.ok = a.all_gather && a.group_start && a.group_end;
        return a;
    }();
    return api;
}
constexpr int kNcclInt8 = 0;      // ncclInt8 / ncclChar: the payload travels as bytes
}  // namespace

// All-gather of the ranks' packed leaves (parallel.allgather_shards): every rank contributes `cap` slots
// (its stored leaves first, the rest marked by the key 0xFFFFFFFF, which spamm_index_leaves skips) of
// keys [cap] int32, records [cap][272] float32 and leaf square sums [cap] float64; rank r's part lands at
// slot r * cap of the outputs, which are the buffers the tree of B is then indexed on.  One NCCL group
// of three collectives on `stream`; comm is the caller's ncclComm_t.
extern "C" int spamm_exchange_allgather(void *nccl_comm, const uint32_t *keys, const float *records,
                                        const double *leaf_sq, int64_t cap, uint32_t *out_keys, float *out_records,
                                        double *out_leaf_sq, void *stream)
{
    if (!nccl_comm || cap < 0 || (cap > 0 && (!keys || !records || !leaf_sq || !out_keys || !out_records || !out_leaf_sq)))
        return SPAMM_EINVAL;
    if (cap == 0) return SPAMM_OK;
    const NcclApi &api = nccl_api();
    if (!api.ok) return SPAMM_ECUDA;        // no NCCL in this process
    cudaStream_t st = (cudaStream_t)stream;
    int rc = api.group_start();
    rc |= api.all_gather(keys, out_keys, (size_t)cap * 4, kNcclInt8, nccl_comm, st);
    rc |= api.all_gather(records, out_records, (size_t)cap * SPAMM_REC_BYTES, kNcclInt8, nccl_comm, st);
    rc |= api.all_gather(leaf_sq, out_leaf_sq, (size_t)cap * 8, kNcclInt8, nccl_comm, st);
    rc |= api.group_end();
    return rc == 0 ? SPAMM_OK : SPAMM_ECUDA;
}
