// qx_dist.cu -- multi-GPU reduction of peak summaries over NCCL (one process
// per GPU).  The data path never moves samples between GPUs: each rank
// computes the (value, smallest lag, ties) summary of its own lag range
// (a stream shard with its (template-1)-sample halo, or a pair shard), and
// the only collective is this summary reduction: 8 int64 per rank.
//
// Protocol (exact for any int64 value and lag, no agreed lag base needed):
//   round 1  ncclAllReduce MAX over {value (INT64_MIN when the rank holds no
//            lags), NaN seen, x all-zero, a block failed, its status,
//            1 - (y all-zero in every block)}
//   round 2  one NCCL group: MAX over {-lag of the ranks holding the global
//            max} and SUM over {their tie counts}
// which is argmax_set's summary of the unsharded correlogram
// (/root/reference/pkg/src/qxcorr/estimator.py:50-57): the max value, the
// smallest lag attaining it, and how many lags attain it.  The reference has
// no distributed code (its only parallelism is the thread pool of
// harness.py:301-305); this is new.
//
// NCCL is resolved at run time (dlsym in the process, else dlopen of
// libnccl.so.2), so the library has no link-time NCCL dependency and uses the
// same NCCL as the caller's communicator (e.g. torch's ProcessGroupNCCL).
#include <dlfcn.h>
#include <climits>
#include <mutex>

#include "nccl.h"
#include "qx_internal.h"

namespace qx {

struct NcclFns {
    decltype(&ncclAllReduce) allreduce = nullptr;
    decltype(&ncclAllGather) allgather = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclCommCount) count = nullptr;
    decltype(&ncclCommUserRank) user_rank = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};

static const NcclFns* nccl_fns(const char** why)
{
    static NcclFns f;
    static const char* err = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = RTLD_DEFAULT;
        if (!dlsym(h, "ncclAllReduce")) {
            h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!h) {
                err = "libnccl.so.2 not found (load NCCL before calling the *_nccl entry points)";
                return;
            }
        }
        f.allreduce = (decltype(f.allreduce))dlsym(h, "ncclAllReduce");
        f.allgather = (decltype(f.allgather))dlsym(h, "ncclAllGather");
        f.group_start = (decltype(f.group_start))dlsym(h, "ncclGroupStart");
        f.group_end = (decltype(f.group_end))dlsym(h, "ncclGroupEnd");
        f.count = (decltype(f.count))dlsym(h, "ncclCommCount");
        f.user_rank = (decltype(f.user_rank))dlsym(h, "ncclCommUserRank");
        f.error_string = (decltype(f.error_string))dlsym(h, "ncclGetErrorString");
        if (!f.allreduce || !f.allgather || !f.group_start || !f.group_end || !f.count || !f.user_rank)
            err = "NCCL symbols missing";
    });
    *why = err;
    return err ? nullptr : &f;
}

// summary = {value, lag, ties, nan, degx, degy_all, bad, badst}
__global__ void k_red_prep1(const long long* __restrict__ sum, long long* __restrict__ r1)
{
    if (threadIdx.x) return;
    r1[0] = sum[2] ? sum[0] : LLONG_MIN;
    r1[1] = sum[3];
    r1[2] = sum[4];
    r1[3] = sum[6];
    r1[4] = sum[7];
    r1[5] = 1 - sum[5];
}

__global__ void k_red_prep2(const long long* __restrict__ sum, const long long* __restrict__ r1,
                            long long* __restrict__ r2)
{
    if (threadIdx.x) return;
    const bool holder = sum[2] && sum[0] == r1[0];
    r2[0] = holder ? -sum[1] : LLONG_MIN;  // MAX -> the smallest lag among holders
    r2[1] = holder ? sum[2] : 0;           // SUM -> their tie count
}

__global__ void k_red_final(const long long* __restrict__ r1, const long long* __restrict__ r2,
                            long long* __restrict__ out)
{
    if (threadIdx.x) return;
    const bool any = r2[1] != 0;
    out[0] = any ? r1[0] : 0;
    out[1] = any ? -r2[0] : 0;
    out[2] = r2[1];
    out[3] = r1[1];
    out[4] = r1[2];
    out[5] = 1 - r1[5];
    out[6] = r1[3];
    out[7] = r1[4];
}

// reduce the device int64[8] summary over `comm` in place, on `s`;
// scratch: >= 16 device int64
const char* summary_allreduce(void* comm, long long* summary, long long* scratch, cudaStream_t s)
{
    const char* why = nullptr;
    const NcclFns* f = nccl_fns(&why);
    if (!f) return why;
    ncclComm_t c = (ncclComm_t)comm;
    long long *r1 = scratch, *r2 = scratch + 8;
    k_red_prep1<<<1, 32, 0, s>>>(summary, r1);
    if (cudaGetLastError() != cudaSuccess) return "prep launch";
    if (f->allreduce(r1, r1, 6, ncclInt64, ncclMax, c, s) != ncclSuccess) return "ncclAllReduce (round 1)";
    k_red_prep2<<<1, 32, 0, s>>>(summary, r1, r2);
    if (cudaGetLastError() != cudaSuccess) return "prep launch";
    if (f->group_start() != ncclSuccess) return "ncclGroupStart";
    const bool ok = f->allreduce(r2, r2, 1, ncclInt64, ncclMax, c, s) == ncclSuccess &&
                    f->allreduce(r2 + 1, r2 + 1, 1, ncclInt64, ncclSum, c, s) == ncclSuccess;
    if (f->group_end() != ncclSuccess || !ok) return "ncclAllReduce (round 2)";
    k_red_final<<<1, 32, 0, s>>>(r1, r2, summary);
    if (cudaGetLastError() != cudaSuccess) return "final launch";
    return nullptr;
}

// all ranks' `n` records of `bytes` each -> out[rank * n ...] (ncclAllGather)
const char* records_allgather(void* comm, const void* mine, size_t bytes, void* out, cudaStream_t s)
{
    const char* why = nullptr;
    const NcclFns* f = nccl_fns(&why);
    if (!f) return why;
    if (f->allgather(mine, out, bytes, ncclUint8, (ncclComm_t)comm, s) != ncclSuccess) return "ncclAllGather";
    return nullptr;
}

const char* comm_rank_size(void* comm, int* rank, int* size)
{
    const char* why = nullptr;
    const NcclFns* f = nccl_fns(&why);
    if (!f) return why;
    if (f->user_rank((ncclComm_t)comm, rank) != ncclSuccess || f->count((ncclComm_t)comm, size) != ncclSuccess)
        return "ncclCommUserRank/ncclCommCount";
    return nullptr;
}

}  // namespace qx
