// qx_abi.cu -- the C ABI (include/qxcorr_b200.h): argument validation with the
// reference's error semantics, quantiser tables, transform-plan cache,
// per-context scratch, and dispatch to the kernels.
#include <climits>
#include <cmath>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/qxcorr_b200.h"
#include "qx_internal.h"

namespace qx {
int thresholds(int kind, long long k, double step, const double* thr, int dtype, double* out);
cudaError_t quantize_launch(const void* x, int64_t ld, int64_t n, int64_t batch, int dtype, const QTable& q,
                            int64_t* codes, unsigned long long* sums, unsigned* flags, cudaStream_t s);
int64_t packed_words(int64_t n, int bits);
cudaError_t quantize_packed_launch(const void* x, int64_t ld, int64_t n, int64_t batch, int dtype, const QTable& q,
                                   int bits, uint32_t* codes, unsigned long long* sums, unsigned* flags, int sms,
                                   cudaStream_t s);
cudaError_t stats_to_results(const unsigned long long* stats, void* results, int64_t batch, cudaStream_t s);
cudaError_t pcm16_launch(const void* in, int64_t n, float* out, int sms, cudaStream_t s);
bool tc_window_eligible(const NttCall& c, int64_t nx, int64_t ny);
cudaError_t tc_window_run(const NttCall& c, int64_t nx, cudaStream_t s);
bool popc_eligible(const NttCall& c, int64_t nx, int64_t ny, bool auto_path);
cudaError_t popc_run(const NttCall& c, int64_t nx, cudaStream_t s);
size_t popc_planes_words(int64_t batch, int64_t nx, int64_t ny);
void popc_schedule(const NttCall& c, int64_t nx, int* G_out, std::vector<int>& out);
cudaError_t merge_blocks_launch(const MergeSegs& segs, long long lag_shift, void* partials, int* counter,
                                long long* out, int sms, cudaStream_t s);
const char* summary_allreduce(void* comm, long long* summary, long long* scratch, cudaStream_t s);
const char* records_allgather(void* comm, const void* mine, size_t bytes, void* out, cudaStream_t s);
const char* comm_rank_size(void* comm, int* rank, int* size);
}  // namespace qx

using namespace qx;

// NTT primes p < 2^30 (lazy [0,4p) arithmetic) with their 2-adicity and a
// primitive root, largest first.
struct PrimeInfo {
    uint32_t p, g;
    int adicity;
};
static const PrimeInfo kPrimes[] = {
    {1012924417u, 5, 21}, {1004535809u, 3, 21}, {998244353u, 3, 23},
    {985661441u, 3, 22},  {469762049u, 3, 26},  {167772161u, 3, 25},
};

struct Arena {
    void* ptr = nullptr;
    size_t size = 0;
    uint64_t gen = 0;  // bumped on every reallocation (plans re-derive their pointers)
};

namespace qx {
cudaError_t set_max_smem(const void* fn, size_t bytes)
{
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({fn, dev})) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done.insert({fn, dev});
    return e;
}

int device_sms()
{
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cache[dev]) {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = sms;
    }
    return cache[dev];
}
}  // namespace qx

// Every entry point runs on the context's device and restores the caller's
// current device on return (a context for GPU 1 never switches torch's
// current device).
struct DevGuard {
    int prev = -1;
    explicit DevGuard(int dev)
    {
        int cur = 0;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
    }
    ~DevGuard()
    {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

static Knobs knobs_from_env()
{
    Knobs k;
    auto num = [](const char* name, int64_t dflt) -> int64_t {
        const char* v = getenv(name);
        return (v && *v) ? atoll(v) : dflt;
    };
    k.chunk_pairs = num("QX_CHUNK_PAIRS", 0);
    k.sweep_lanes = (int)num("QX_SWEEP_LANES", 0);
    k.sweep_chunks = (int)num("QX_SWEEP_CHUNKS", 0);
    k.sweep_taper = (int)std::max<int64_t>(1, num("QX_SWEEP_TAPER", 2));
    k.sweep_even = getenv("QX_SWEEP_EVEN") != nullptr;
    k.sweep_restage = num("QX_SWEEP_RESTAGE", 1) != 0;
    k.sweep_compute = num("QX_SWEEP_COMPUTE", 1) != 0;
    k.popc = num("QX_POPC", 1) != 0;
    k.popc_timing = num("QX_POPC_TIMING", 0) != 0;
    k.tc_f4 = num("QX_TC_F4", 1) != 0;
    k.zero_copy = num("QX_ZERO_COPY", 1) != 0;
    if (const char* ev = getenv("QX_SWEEP_PLAN")) {
        for (const char* p = ev; *p && k.sweep_plan_n < 16;) {
            const int64_t v = atoll(p);
            if (v > 0) k.sweep_plan[k.sweep_plan_n++] = v;
            while (*p && *p != ',') ++p;
            if (*p == ',') ++p;
        }
    }
    return k;
}

// A compute lane of the sweep entry point: its own stream and scratch, so
// the quantiser pairs of one staged chunk run concurrently (their launches
// fill each other's tail waves).
struct Lane {
    Arena scratch, counters;
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
};
constexpr int kMaxLanes = 8;
constexpr size_t kZeroCopyBytes = 1 << 20;  // qx_plan_run_host reads pinned rows in place up to this size

struct qx_context {
    int device = 0;
    std::recursive_mutex mu;
    std::map<std::pair<uint32_t, int>, std::pair<NttTables, void*>> tables;
    std::map<std::pair<uint32_t, int>, std::pair<OuterTables, void*>> otables;
    std::map<std::string, std::vector<double>> thr_cache;
    // popc path: per-shape CTA schedules (device int[G + 1]) and their G
    std::map<std::tuple<int64_t, int64_t, int64_t, int64_t, int64_t>, std::pair<void*, int>> popc_sched;
    Arena scratch;     // Y/R/stats/partials
    Arena counters;    // zero-initialised ints, reset by the kernels
    Arena stage;       // host-API staging (x, y, results)
    Arena records;     // template search: per-block results, merge partials
    Arena mcounter;    // template search: merge counter (zeroed once, reset by the kernel)
    Arena dist;        // multi-GPU summary reduction scratch (16 int64)
    cudaStream_t host_stream = nullptr;
    cudaStream_t copy_stream = nullptr;   // H2D of the sweep entry point
    std::vector<cudaEvent_t> chunk_ev;    // per staged chunk (lazily created)
    Lane lanes[kMaxLanes];                // sweep compute lanes (lazily created)
    cudaEvent_t fork = nullptr;           // device sweep: caller stream -> lanes
    Profiler prof;
    Knobs knobs;
    std::string last_error;
    // stream ordering of the shared arenas: the last stream that enqueued
    // work on this context, and an event recorded after that work.  A call
    // on another stream first waits for it (ctx_begin), so scratch, counters,
    // staging and records are never used by two streams at once.
    cudaStream_t last_stream = nullptr;
    bool used = false;
    cudaEvent_t last_ev = nullptr;
};

// The ordering event is recorded lazily, on the previous stream, only when a
// call arrives on a different one: it then covers everything enqueued there
// so far (a superset of the previous call's work), and same-stream calls --
// the common case -- pay no event record.
static cudaError_t ctx_begin(qx_context* ctx, cudaStream_t s)
{
    if (!ctx->used || ctx->last_stream == s) return cudaSuccess;
    if (!ctx->last_ev) {
        cudaError_t e = cudaEventCreateWithFlags(&ctx->last_ev, cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaEventRecord(ctx->last_ev, ctx->last_stream);
    if (e != cudaSuccess) {
        // the previous stream is gone (destroyed by its owner): order by a
        // full device synchronisation instead
        cudaGetLastError();
        return cudaDeviceSynchronize();
    }
    return cudaStreamWaitEvent(s, ctx->last_ev, 0);
}

static cudaError_t ctx_end(qx_context* ctx, cudaStream_t s);

// RAII: order `s` after the context's previous stream on entry, record the
// context event on `s` on exit
struct StreamOrder {
    qx_context* c;
    cudaStream_t s;
    StreamOrder(qx_context* c_, cudaStream_t s_) : c(c_), s(s_) { ctx_begin(c, s); }
    ~StreamOrder() { ctx_end(c, s); }
};

static cudaError_t ctx_end(qx_context* ctx, cudaStream_t s)
{
    ctx->last_stream = s;
    ctx->used = true;
    return cudaSuccess;
}

static qx_status fail(qx_context* ctx, qx_status s, const std::string& msg)
{
    if (ctx) ctx->last_error = msg;
    return s;
}

static qx_status cuda_fail(qx_context* ctx, cudaError_t e, const char* where)
{
    return fail(ctx, QX_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

static cudaError_t arena_reserve(Arena& a, size_t bytes, bool zero)
{
    if (a.size >= bytes) return cudaSuccess;
    if (a.ptr) {
        cudaError_t e = cudaFree(a.ptr);  // synchronising: prior users are done
        if (e != cudaSuccess) return e;
        a.ptr = nullptr;
        a.size = 0;
    }
    size_t want = bytes + bytes / 4;
    cudaError_t e = cudaMalloc(&a.ptr, want);
    if (e != cudaSuccess) return e;
    a.size = want;
    ++a.gen;
    if (zero) {
        // the consumers run on non-blocking streams, which do not order
        // after the legacy stream: finish the zeroing before returning
        e = cudaMemset(a.ptr, 0, want);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        return e;
    }
    return cudaSuccess;
}

extern "C" {

int qx_abi_version(void) { return QX_ABI_VERSION; }

const char* qx_status_string(qx_status s)
{
    switch (s) {
    case QX_OK: return "ok";
    case QX_ERR_INVALID: return "invalid argument";
    case QX_DEGENERATE_QUANTIZATION: return "quantizes to all zeros";
    case QX_DEGENERATE_INPUT: return "all-zero input";
    case QX_BOUND_EXCEEDED: return "coefficient bound N_min*K_u*K_v exceeds the supported int64 range";
    case QX_INTERNAL_OVERFLOW: return "internal overflow";
    case QX_ERR_CUDA: return "CUDA error";
    case QX_ERR_UNSUPPORTED: return "unsupported shape or parameter";
    case QX_ERR_NOMEM: return "out of memory";
    case QX_ERR_NONFINITE: return "NaN input";
    }
    return "unknown status";
}

qx_status qx_context_create(int device, qx_context** out)
{
    if (!out) return QX_ERR_INVALID;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return QX_ERR_CUDA;
    DevGuard g(device);
    qx_context* c = new qx_context();
    c->device = device;
    c->knobs = knobs_from_env();
    cudaError_t e = cudaStreamCreateWithFlags(&c->host_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return QX_ERR_CUDA;
    }
    *out = c;
    return QX_OK;
}

void qx_context_destroy(qx_context* c)
{
    if (!c) return;
    DevGuard g(c->device);
    cudaDeviceSynchronize();
    if (c->last_ev) cudaEventDestroy(c->last_ev);
    for (auto& kv : c->tables) cudaFree(kv.second.second);
    for (auto& kv : c->otables) cudaFree(kv.second.second);
    for (auto& kv : c->popc_sched) cudaFree(kv.second.first);
    for (Arena* a : {&c->scratch, &c->counters, &c->stage, &c->records, &c->mcounter, &c->dist})
        if (a->ptr) cudaFree(a->ptr);
    if (c->host_stream) cudaStreamDestroy(c->host_stream);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    for (cudaEvent_t ev : c->chunk_ev) cudaEventDestroy(ev);
    if (c->fork) cudaEventDestroy(c->fork);
    for (Lane& l : c->lanes) {
        for (Arena* a : {&l.scratch, &l.counters})
            if (a->ptr) cudaFree(a->ptr);
        if (l.stream) cudaStreamDestroy(l.stream);
        if (l.done) cudaEventDestroy(l.done);
    }
    delete c;
}

const char* qx_context_last_error(const qx_context* c) { return c ? c->last_error.c_str() : ""; }

qx_status qx_context_set_option(qx_context* c, const char* name, int64_t value)
{
    if (!c || !name) return QX_ERR_INVALID;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    Knobs& k = c->knobs;
    const std::string n(name);
    if (n == "chunk_pairs") k.chunk_pairs = value < 0 ? 0 : value;
    else if (n == "sweep_lanes") k.sweep_lanes = (int)std::max<int64_t>(0, value);
    else if (n == "sweep_chunks") k.sweep_chunks = (int)std::max<int64_t>(0, value);
    else if (n == "sweep_taper") k.sweep_taper = (int)std::max<int64_t>(1, value);
    else if (n == "sweep_even") k.sweep_even = value != 0;
    else if (n == "sweep_restage") k.sweep_restage = value != 0;
    else if (n == "sweep_compute") k.sweep_compute = value != 0;
    else if (n == "popc") k.popc = value != 0;
    else if (n == "popc_timing") k.popc_timing = value != 0;
    else if (n == "tc_f4") k.tc_f4 = value != 0;
    else if (n == "zero_copy") k.zero_copy = value != 0;
    else return fail(c, QX_ERR_INVALID, "unknown option " + n);
    return QX_OK;
}

}  // extern "C"

// ------------------------------------------------------------ validation

// Quantizer.__post_init__ (quantize.py:37-51) semantics
static qx_status check_quantizer(qx_context* ctx, const qx_quantizer* q, int dtype)
{
    if (!q) return fail(ctx, QX_ERR_INVALID, "quantizer is NULL");
    if (q->kind == QX_Q_CODES) {
        if (dtype != QX_I64) return fail(ctx, QX_ERR_INVALID, "integer codes require dtype int64");
        if (q->k < 0) return fail(ctx, QX_ERR_INVALID, "bound must be >= 0");
        return QX_OK;
    }
    if (dtype != QX_F32 && dtype != QX_F64)
        return fail(ctx, QX_ERR_INVALID, "quantised inputs must be float32 or float64");
    if (q->k < 1) return fail(ctx, QX_ERR_INVALID, "level bound k must be >= 1");
    if (q->kind == QX_Q_SIGN) {
        if (q->k != 1) return fail(ctx, QX_ERR_INVALID, "sign quantizer has k == 1");
    } else if (q->kind == QX_Q_UNIFORM) {
        if (!(q->step > 0)) return fail(ctx, QX_ERR_INVALID, "uniform step must be > 0");
    } else if (q->kind == QX_Q_CUSTOM) {
        if (!q->thresholds) return fail(ctx, QX_ERR_INVALID, "custom quantizer needs thresholds");
        for (int64_t i = 1; i < 2 * q->k; ++i)
            if (!(q->thresholds[i] > q->thresholds[i - 1]))
                return fail(ctx, QX_ERR_INVALID, "thresholds must be strictly increasing");
        if (!(q->thresholds[q->k - 1] <= 0.0 && 0.0 < q->thresholds[q->k]))
            return fail(ctx, QX_ERR_INVALID, "level 0 must contain the input 0");
    } else {
        return fail(ctx, QX_ERR_INVALID, "unknown quantizer kind");
    }
    if (q->k > kMaxThr / 2) return fail(ctx, QX_ERR_UNSUPPORTED, "quantizer level bound k > 128");
    return QX_OK;
}

static qx_status make_qtable(qx_context* ctx, const qx_quantizer* q, int dtype, QTable* t)
{
    memset(t, 0, sizeof(*t));
    t->k = (int)(q->kind == QX_Q_CODES ? q->k : q->k);
    if (q->kind == QX_Q_CODES) {
        t->mode = QM_CODES;
        t->tsize = 0;
        return QX_OK;
    }
    t->mode = q->k == 1 ? QM_K1 : (q->kind == QX_Q_UNIFORM ? QM_UNIFORM : QM_BSEARCH);
    int ts = 1, tb = 0;
    while (ts < 2 * q->k) {
        ts <<= 1;
        ++tb;
    }
    t->tsize = ts;
    t->tbits = tb;
    t->inv_step = q->kind == QX_Q_UNIFORM ? 1.0 / q->step : 1.0;
    // cache key: every parameter byte
    std::string key((const char*)&q->kind, 4);
    key.append((const char*)&q->k, 8);
    key.append((const char*)&q->step, 8);
    key.append((const char*)&dtype, 4);
    if (q->kind == QX_Q_CUSTOM) key.append((const char*)q->thresholds, (size_t)(16 * q->k));
    auto it = ctx->thr_cache.find(key);
    if (it == ctx->thr_cache.end()) {
        std::vector<double> v((size_t)(2 * q->k));
        thresholds(q->kind, q->k, q->step, q->thresholds, dtype == QX_F32 ? DT_F32 : DT_F64, v.data());
        it = ctx->thr_cache.emplace(key, std::move(v)).first;
    }
    for (int i = 0; i < ts; ++i) t->thr[i] = i < 2 * q->k ? it->second[i] : NAN;
    return QX_OK;
}

static qx_status check_signals(qx_context* ctx, const qx_signals* s, const char* name)
{
    if (!s || !s->data) return fail(ctx, QX_ERR_INVALID, std::string(name) + " is NULL");
    if (s->n < 1) return fail(ctx, QX_ERR_INVALID, "samples must be a non-empty 1-D sequence");
    // inputs are read-only, so rows may overlap (0 <= ld < n: sliding windows
    // of one stream) or repeat (ld == 0: one template against many blocks)
    if (s->ld < 0) return fail(ctx, QX_ERR_INVALID, std::string(name) + ": ld < 0");
    if (s->dtype < QX_F32 || s->dtype > QX_I64) return fail(ctx, QX_ERR_INVALID, "bad dtype");
    return QX_OK;
}

static int ceil_log2(int64_t v)
{
    int l = 0;
    while ((1ll << l) < v) ++l;
    return l;
}

static qx_status get_tables(qx_context* ctx, const PrimeInfo& pi, int lp, NttTables* out)
{
    auto key = std::make_pair(pi.p, lp);
    auto it = ctx->tables.find(key);
    if (it == ctx->tables.end()) {
        NttTables t;
        void* blk = nullptr;
        cudaError_t e = ntt_make_tables(pi.p, pi.g, lp, &t, &blk);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "twiddle tables");
        it = ctx->tables.emplace(key, std::make_pair(t, blk)).first;
    }
    *out = it->second.first;
    return QX_OK;
}

static qx_status get_outer_tables(qx_context* ctx, const PrimeInfo& pi, int lp, int logm, OuterTables* out)
{
    auto key = std::make_pair(pi.p, lp);
    auto it = ctx->otables.find(key);
    if (it == ctx->otables.end()) {
        OuterTables t;
        void* blk = nullptr;
        cudaError_t e = ntt_make_outer_tables(pi.p, pi.g, lp, logm, &t, &blk);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "outer twiddle tables");
        it = ctx->otables.emplace(key, std::make_pair(t, blk)).first;
    }
    *out = it->second.first;
    return QX_OK;
}

static uint64_t powmod64(uint64_t a, uint64_t e, uint64_t p)
{
    uint64_t r = 1;
    a %= p;
    while (e) {
        if (e & 1) r = (unsigned __int128)r * a % p;
        a = (unsigned __int128)a * a % p;
        e >>= 1;
    }
    return r;
}

// Common front half: validate, build the call, reserve scratch.
struct Prepared {
    NttCall call;
    int64_t nx, ny;
    int path;
};

static qx_status prepare(qx_context* ctx, const qx_signals* x, const qx_signals* y, int64_t batch,
                         const qx_quantizer* qx_, const qx_quantizer* qy_, int64_t lag_lo, int64_t lag_hi,
                         bool argmax, qx_path path, Prepared* out, Arena* scratch = nullptr,
                         Arena* counters = nullptr, bool split2 = false)
{
    Arena& scr = scratch ? *scratch : ctx->scratch;
    Arena& cnt = counters ? *counters : ctx->counters;
    qx_status st;
    if (batch < 1) return fail(ctx, QX_ERR_INVALID, "batch must be >= 1");
    if ((st = check_signals(ctx, x, "x")) != QX_OK) return st;
    if ((st = check_signals(ctx, y, "y")) != QX_OK) return st;
    if ((st = check_quantizer(ctx, qx_, x->dtype)) != QX_OK) return st;
    if ((st = check_quantizer(ctx, qy_, y->dtype)) != QX_OK) return st;
    const int64_t nx = x->n, ny = y->n;
    const int64_t ku = qx_->k > 1 ? qx_->k : 1, kv = qy_->k > 1 ? qy_->k : 1;
    const int64_t nmin = nx < ny ? nx : ny;
    // _check_coeff_bound (intxcorr.py:89-93)
    const unsigned __int128 bound = (unsigned __int128)nmin * (uint64_t)ku * (uint64_t)kv;
    if (bound > ((unsigned __int128)1 << 59))
        return fail(ctx, QX_BOUND_EXCEEDED, "coefficient bound N_min*K_u*K_v exceeds the supported int64 range");
    const int64_t nout = nx + ny - 1;
    const int64_t first_lag = y->start - (x->start + nx - 1);
    int64_t t_lo = 0, t_hi = nout - 1;
    if (argmax) {
        // window in t, computed without overflow
        if (lag_lo != INT64_MIN) {
            __int128 v = (__int128)lag_lo - first_lag;
            if (v > t_lo) t_lo = v > (__int128)t_hi ? t_hi + 1 : (int64_t)v;
        }
        if (lag_hi != INT64_MAX) {
            __int128 v = (__int128)lag_hi - first_lag;
            if (v < t_hi) t_hi = v < 0 ? -1 : (int64_t)v;
        }
        if (t_lo > t_hi) return fail(ctx, QX_ERR_INVALID, "lag window does not intersect the overlap range");
    }
    NttCall& c = out->call;
    memset(&c, 0, sizeof(c));
    c.knobs = &ctx->knobs;
    c.split2 = split2;
    c.op[0].data = x->data;
    c.op[0].ld = x->ld;
    c.op[0].n = nx;
    c.op[0].reverse = 1;
    c.op[0].dtype = x->dtype == QX_F32 ? DT_F32 : (x->dtype == QX_F64 ? DT_F64 : DT_I64);
    c.op[1].data = y->data;
    c.op[1].ld = y->ld;
    c.op[1].n = ny;
    c.op[1].reverse = 0;
    c.op[1].dtype = y->dtype == QX_F32 ? DT_F32 : (y->dtype == QX_F64 ? DT_F64 : DT_I64);
    if ((st = make_qtable(ctx, qx_, x->dtype, &c.op[0].q)) != QX_OK) return st;
    if ((st = make_qtable(ctx, qy_, y->dtype, &c.op[1].q)) != QX_OK) return st;
    c.batch = batch;
    c.nout = nout;
    c.am.first_lag = first_lag;
    c.am.t_lo = t_lo;
    c.am.t_hi = t_hi;
    out->nx = nx;
    out->ny = ny;
    // bounded lag windows go to the tcgen05 int8 Toeplitz kernel (qx_tc.cu)
    const bool tc_ok = argmax && tc_window_eligible(c, nx, ny);
    if (path == QX_PATH_DIRECT && !tc_ok)
        return fail(ctx, QX_ERR_UNSUPPORTED, "tensor-core window path: window > 4112 lags, nx > 4593 or k > 127");
    // word-parallel 1-level codes (qx_popc.cu): small single pairs
    const bool popc_ok = argmax && !(path == QX_PATH_AUTO && tc_ok) && popc_eligible(c, nx, ny, path == QX_PATH_AUTO);
    if (path == QX_PATH_POPC && !popc_ok)
        return fail(ctx, QX_ERR_UNSUPPORTED, "popc path: needs k = 1 quantisers on float rows, nx <= 65536 and "
                                             "a lag window whose planes fit shared memory");
    out->path = (path == QX_PATH_DIRECT || (path == QX_PATH_AUTO && tc_ok)) ? QX_PATH_DIRECT
                : (path == QX_PATH_POPC || (path == QX_PATH_AUTO && popc_ok)) ? QX_PATH_POPC : QX_PATH_NTT;
    if (out->path == QX_PATH_POPC) {
        c.am.pstride = kMaxPartialsLarge;
        const size_t sb = (size_t)batch * 8 * 8, pb = (size_t)batch * c.am.pstride * 3 * 8;
        const size_t spb = (size_t)batch * kMaxPartialsLarge * 16;
        const size_t plb = popc_planes_words(batch, nx, ny) * 4;
        cudaError_t e = arena_reserve(scr, sb + pb + spb + plb + 256, false);
        if (e == cudaSuccess) e = arena_reserve(cnt, (size_t)batch * 8, true);  // ticket + barrier per pair
        if (e != cudaSuccess) return cuda_fail(ctx, e, "scratch");
        c.stats = (unsigned long long*)scr.ptr;
        c.am.partials = (long long*)((char*)scr.ptr + sb);
        c.popc_spart = (unsigned*)((char*)scr.ptr + sb + pb);
        c.popc_planes = (uint32_t*)((char*)scr.ptr + sb + pb + spb);
        // the CTA schedule of this shape (host partition, uploaded once)
        const auto key = std::make_tuple(nx, ny, c.am.t_lo, c.am.t_hi, batch);
        auto it = ctx->popc_sched.find(key);
        if (it == ctx->popc_sched.end()) {
            std::vector<int> sched;
            int G = 1;
            popc_schedule(c, nx, &G, sched);
            void* d = nullptr;
            e = cudaMalloc(&d, sched.size() * sizeof(int));
            if (e == cudaSuccess) e = cudaMemcpy(d, sched.data(), sched.size() * sizeof(int), cudaMemcpyHostToDevice);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "popc schedule");
            it = ctx->popc_sched.emplace(key, std::make_pair(d, G)).first;
        }
        c.popc_sched = (const int*)it->second.first;
        c.popc_G = it->second.second;
        c.am.counters = (int*)cnt.ptr;
        c.prof = &ctx->prof;
        return QX_OK;
    }
    if (out->path == QX_PATH_DIRECT) {
        const size_t sb = (size_t)batch * 8 * 8;
        cudaError_t e = arena_reserve(scr, sb + 256, false);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "scratch");
        c.stats = (unsigned long long*)scr.ptr;
        c.prof = &ctx->prof;
        return QX_OK;
    }

    const int lp = ceil_log2(nout) < 10 ? 10 : ceil_log2(nout);
    if (lp > 26) return fail(ctx, QX_ERR_UNSUPPORTED, "full-lag correlation longer than 2^26 points");
    // P > 2^19: outer radix-2^logm pass around 2^lq four-step sub-transforms
    const int large = lp > 19;
    const int logm = large ? (lp - 19 > 3 ? lp - 19 : 3) : 0;
    const int lq = lp - logm;
    // primes: product must exceed 2*bound + 1 (centred lift)
    std::vector<const PrimeInfo*> ps;
    for (const PrimeInfo& pi : kPrimes)
        if (pi.adicity >= lp) ps.push_back(&pi);
    int np = 0;
    unsigned __int128 M = 1;
    while (np < (int)ps.size() && np < 3) {
        M *= ps[np]->p;
        ++np;
        if ((M - 1) / 2 >= bound) break;
    }
    if ((M - 1) / 2 < bound) return fail(ctx, QX_ERR_UNSUPPORTED, "no prime set covers this coefficient bound");
    c.np = np;
    c.large = large;
    c.logm = logm;
    c.lq = lq;
    for (int i = 0; i < np; ++i) {
        if ((st = get_tables(ctx, *ps[i], lq, &c.tab[i])) != QX_OK) return st;
        if (large && (st = get_outer_tables(ctx, *ps[i], lp, logm, &c.otab[i])) != QX_OK) return st;
        uint64_t mprev = 1;
        for (int j = 0; j < i; ++j) mprev = (unsigned __int128)mprev * ps[j]->p % ps[i]->p;
        c.garner_inv[i] = i ? powmod64(mprev, ps[i]->p - 2, ps[i]->p) : 1;
    }
    const int64_t P = 1ll << lp;
    c.zero_upper = (nx <= P / 2 && ny <= P / 2);
    // words of scratch per pair: Y (2 operands) | Z | [large: OUT (2) | RI (np)] | R (np > 1)
    const int64_t per_pair = (3 + (large ? 2 + np : 0) + (np > 1 ? np : 0)) * P;
    // pairs per launch group: as many as fit ~1.5 GiB of scratch.  Large
    // grids beat L2 residency here (measured on C2: 16 -> 64 pairs per launch
    // = 2.91 -> 2.41 ms/step; tail waves of 1-CTA/SM kernels dominate).
    int64_t chunk = (1536ll << 20) / (per_pair * 4);
    if (ctx->knobs.chunk_pairs > 0) chunk = ctx->knobs.chunk_pairs;
    if (chunk < 1) chunk = 1;
    if (chunk > batch) chunk = batch;
    c.chunk = chunk;
    const size_t wb = (size_t)chunk * per_pair * 4;
    const size_t sb = (size_t)batch * 8 * 8;
    c.am.pstride = large ? kMaxPartialsLarge : kMaxPartials;
    const size_t pb = argmax ? (size_t)batch * c.am.pstride * 3 * 8 : 0;
    cudaError_t e = arena_reserve(scr, wb + sb + pb + 256, false);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "scratch");
    e = arena_reserve(cnt, (size_t)batch * 4, true);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "counters");
    char* base = (char*)scr.ptr;
    uint32_t* w = (uint32_t*)base;
    c.Y = w;
    w += (size_t)chunk * 2 * P;
    c.Z = w;
    w += (size_t)chunk * P;
    if (large) {
        c.OUT = w;
        w += (size_t)chunk * 2 * P;
        c.RI = w;
        w += (size_t)chunk * np * P;
    }
    c.R = np > 1 ? w : nullptr;
    c.stats = (unsigned long long*)(base + wb);
    c.am.partials = argmax ? (long long*)(base + wb + sb) : nullptr;
    c.am.counters = (int*)cnt.ptr;
    c.prof = &ctx->prof;
    return QX_OK;
}

extern "C" {

qx_status qx_quantizer_thresholds(const qx_quantizer* q, qx_dtype dtype, double* out)
{
    if (!out) return QX_ERR_INVALID;
    qx_status st = check_quantizer(nullptr, q, dtype);
    if (st != QX_OK) return st;
    if (q->kind == QX_Q_CODES) return QX_ERR_INVALID;
    thresholds(q->kind, q->k, q->step, q->thresholds, dtype == QX_F32 ? DT_F32 : DT_F64, out);
    return QX_OK;
}

qx_status qx_quantize(qx_context* ctx, const qx_quantizer* q, const qx_signals* x, int64_t batch, int64_t* codes,
                      int64_t* sumsq, int64_t* nnz, void* stream)
{
    if (!ctx) return QX_ERR_INVALID;
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    DevGuard dg(ctx->device);
    StreamOrder order(ctx, (cudaStream_t)stream);
    qx_status st;
    if (batch < 1 || !codes) return fail(ctx, QX_ERR_INVALID, "bad batch or output");
    if ((st = check_signals(ctx, x, "x")) != QX_OK) return st;
    if ((st = check_quantizer(ctx, q, x->dtype)) != QX_OK) return st;
    if (q->kind == QX_Q_CODES) return fail(ctx, QX_ERR_INVALID, "input already quantised");
    QTable t;
    if ((st = make_qtable(ctx, q, x->dtype, &t)) != QX_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = arena_reserve(ctx->scratch, (size_t)batch * 16 + 64, false);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "scratch");
    unsigned long long* sums = (unsigned long long*)ctx->scratch.ptr;
    unsigned* flags = (unsigned*)((char*)ctx->scratch.ptr + batch * 16);
    e = cudaMemsetAsync(ctx->scratch.ptr, 0, (size_t)batch * 16 + 64, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "memset");
    ctx->prof.pre(KK_QUANT, s);
    e = quantize_launch(x->data, x->ld, x->n, batch, x->dtype == QX_F32 ? DT_F32 : DT_F64, t, codes, sums, flags, s);
    ctx->prof.post(KK_QUANT, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "quantize");
    if (sumsq) {
        e = cudaMemcpy2DAsync(sumsq, 8, sums, 16, 8, (size_t)batch, cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "copy sums");
    }
    if (nnz) {
        e = cudaMemcpy2DAsync(nnz, 8, sums + 1, 16, 8, (size_t)batch, cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "copy nnz");
    }
    return QX_OK;
}

}  // extern "C"

// qx_estimate_batch on explicit scratch arenas (the sweep's compute lanes)
// split2: `results` holds two records per pair and the 2-SM template-search
// mode may write them (qx_template_search)
extern "C" {

qx_status qx_quantize_packed(qx_context* ctx, const qx_quantizer* q, const qx_signals* x, int64_t batch, int bits,
                             uint32_t* codes, int64_t* sumsq, int64_t* nnz, int32_t* flags, void* stream)
{
    if (!ctx) return QX_ERR_INVALID;
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    DevGuard dg(ctx->device);
    StreamOrder order(ctx, (cudaStream_t)stream);
    qx_status st;
    if (batch < 1 || !codes) return fail(ctx, QX_ERR_INVALID, "bad batch or output");
    if ((st = check_signals(ctx, x, "x")) != QX_OK) return st;
    if ((st = check_quantizer(ctx, q, x->dtype)) != QX_OK) return st;
    if (q->kind == QX_Q_CODES) return fail(ctx, QX_ERR_INVALID, "input already quantised");
    if (bits != 1 && bits != 2 && bits != 4 && bits != 8) return fail(ctx, QX_ERR_INVALID, "bits must be 1, 2, 4 or 8");
    if (bits == 1 && q->k != 1) return fail(ctx, QX_ERR_INVALID, "1-bit planes need a 1-level quantizer (k == 1)");
    if (bits > 1 && q->k > (1 << (bits - 1)) - 1)
        return fail(ctx, QX_ERR_INVALID, "level bound k does not fit the packed field (k <= 2^(bits-1) - 1)");
    QTable t;
    if ((st = make_qtable(ctx, q, x->dtype, &t)) != QX_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = arena_reserve(ctx->scratch, (size_t)batch * 16 + 64, false);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "scratch");
    unsigned long long* sums = (unsigned long long*)ctx->scratch.ptr;
    unsigned* fl = (unsigned*)((char*)ctx->scratch.ptr + batch * 16);
    e = cudaMemsetAsync(ctx->scratch.ptr, 0, (size_t)batch * 16 + 64, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "memset");
    ctx->prof.pre(KK_QUANT, s);
    e = quantize_packed_launch(x->data, x->ld, x->n, batch, x->dtype == QX_F32 ? DT_F32 : DT_F64, t, bits, codes, sums,
                               fl, device_sms(), s);
    ctx->prof.post(KK_QUANT, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "quantize");
    if (sumsq && (e = cudaMemcpy2DAsync(sumsq, 8, sums, 16, 8, (size_t)batch, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
        return cuda_fail(ctx, e, "copy sums");
    if (nnz && (e = cudaMemcpy2DAsync(nnz, 8, sums + 1, 16, 8, (size_t)batch, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
        return cuda_fail(ctx, e, "copy nnz");
    if (flags && (e = cudaMemcpyAsync(flags, fl, 4, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
        return cuda_fail(ctx, e, "copy flags");
    return QX_OK;
}

int64_t qx_packed_words(int64_t n, int bits) { return packed_words(n, bits); }

}  // extern "C"

static qx_status estimate_batch_on(qx_context* ctx, const qx_signals* x, const qx_signals* y, int64_t batch,
                                   const qx_quantizer* qx_, const qx_quantizer* qy_, int64_t lag_lo, int64_t lag_hi,
                                   qx_path path, qx_result* results, void* stream, Arena* scratch, Arena* counters,
                                   bool split2 = false)
{
    Prepared pr;
    qx_status st = prepare(ctx, x, y, batch, qx_, qy_, lag_lo, lag_hi, true, path, &pr, scratch, counters, split2);
    if (st != QX_OK) return st;
    // two records per pair came only from the retired 2-SM kernel
    if (split2) return QX_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    pr.call.am.results = results;
    cudaError_t e = cudaSuccess;
    if (pr.path != QX_PATH_POPC)  // the popc path writes (or zeroes) its statistics itself
        e = cudaMemsetAsync(pr.call.stats, 0, (size_t)batch * 64, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "memset stats");
    e = pr.path == QX_PATH_DIRECT ? tc_window_run(pr.call, pr.nx, s)
        : pr.path == QX_PATH_POPC ? popc_run(pr.call, pr.nx, s) : ntt_run(pr.call, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "kernel launch");
    return QX_OK;
}

// Compute lanes of the sweep entry points: up to 4 streams (QX_SWEEP_LANES),
// one per quantiser pair in turn, each with its own scratch, so the sweep's
// independent correlations overlap instead of each draining the machine.
static cudaError_t open_lanes(qx_context* ctx, int64_t nq, int* nl_out, int64_t most = 0)
{
    int nl = (int)std::min<int64_t>(nq, 4);
    if (ctx->knobs.sweep_lanes > 0)
        nl = (int)std::max<int64_t>(1, std::min<int64_t>(most > 0 ? most : nq, ctx->knobs.sweep_lanes));
    nl = std::min(nl, kMaxLanes);
    cudaError_t e = cudaSuccess;
    for (int l = 0; l < nl && e == cudaSuccess; ++l) {
        Lane& L = ctx->lanes[l];
        if (!L.stream) e = cudaStreamCreateWithFlags(&L.stream, cudaStreamNonBlocking);
        if (e == cudaSuccess && !L.done) e = cudaEventCreateWithFlags(&L.done, cudaEventDisableTiming);
    }
    if (e == cudaSuccess && !ctx->fork) e = cudaEventCreateWithFlags(&ctx->fork, cudaEventDisableTiming);
    *nl_out = nl;
    return e;
}

extern "C" {

qx_status qx_estimate_batch(qx_context* ctx, const qx_signals* x, const qx_signals* y, int64_t batch,
                            const qx_quantizer* qx_, const qx_quantizer* qy_, int64_t lag_lo, int64_t lag_hi,
                            qx_path path, qx_result* results, void* stream)
{
    if (!ctx) return QX_ERR_INVALID;
    if (!results) return fail(ctx, QX_ERR_INVALID, "results is NULL");
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    DevGuard dg(ctx->device);
    StreamOrder order(ctx, (cudaStream_t)stream);
    Prepared pr;
    qx_status st = prepare(ctx, x, y, batch, qx_, qy_, lag_lo, lag_hi, true, path, &pr);
    if (st != QX_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    pr.call.am.results = results;
    cudaError_t e = cudaSuccess;
    if (pr.path != QX_PATH_POPC)  // the popc path writes (or zeroes) its statistics itself
        e = cudaMemsetAsync(pr.call.stats, 0, (size_t)batch * 64, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "memset stats");
    e = pr.path == QX_PATH_DIRECT ? tc_window_run(pr.call, pr.nx, s)
        : pr.path == QX_PATH_POPC ? popc_run(pr.call, pr.nx, s) : ntt_run(pr.call, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "kernel launch");
    return QX_OK;
}

}  // extern "C"

// A prepared qx_estimate_batch call (fixed shapes, quantisers, window and
// path): validation, threshold tables, path choice and scratch layout are
// done once; qx_plan_run only swaps in the data pointers and launches.
struct qx_plan {
    qx_context* ctx = nullptr;
    qx_signals x{}, y{};
    int64_t batch = 0;
    qx_quantizer qx{}, qy{};
    std::vector<double> tx, ty;  // custom thresholds (the caller's array may go away)
    int64_t lag_lo = 0, lag_hi = 0;
    qx_path path = QX_PATH_AUTO;
    Prepared pr;
    uint64_t gen_s = 0, gen_c = 0;  // arena generations the pointers in pr were derived from
    void* dstage = nullptr;         // qx_plan_run_host: device copies of the rows + results
    size_t dstage_bytes = 0;
    qx_result* hres = nullptr;      // qx_plan_run_host, zero-copy mode: mapped pinned result records
    size_t hres_bytes = 0;
    ~qx_plan()
    {
        if (dstage || hres) {
            DevGuard dg(ctx->device);
            if (dstage) cudaFree(dstage);
            if (hres) cudaFreeHost(hres);
        }
    }
};

// device alias of a pinned (page-locked, mapped) host pointer, or null
static const void* pinned_device_alias(const void* h)
{
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

static qx_status plan_prepare(qx_plan* p)
{
    qx_status st = prepare(p->ctx, &p->x, &p->y, p->batch, &p->qx, &p->qy, p->lag_lo, p->lag_hi, true, p->path, &p->pr);
    if (st != QX_OK) return st;
    p->gen_s = p->ctx->scratch.gen;
    p->gen_c = p->ctx->counters.gen;
    return QX_OK;
}

extern "C" {

qx_status qx_plan_create(qx_context* ctx, const qx_signals* x, const qx_signals* y, int64_t batch,
                         const qx_quantizer* qx_, const qx_quantizer* qy_, int64_t lag_lo, int64_t lag_hi,
                         qx_path path, qx_plan** out)
{
    if (!ctx || !out) return QX_ERR_INVALID;
    *out = nullptr;
    if (!x || !y || !qx_ || !qy_) return fail(ctx, QX_ERR_INVALID, "x, y and both quantizers are required");
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    DevGuard dg(ctx->device);
    qx_plan* p = new qx_plan();
    p->ctx = ctx;
    p->x = *x;
    p->y = *y;
    // shapes only: the data pointers come with every qx_plan_run
    static const char kDummy = 0;
    if (!p->x.data) p->x.data = &kDummy;
    if (!p->y.data) p->y.data = &kDummy;
    p->batch = batch;
    p->qx = *qx_;
    p->qy = *qy_;
    if (qx_->kind == QX_Q_CUSTOM && qx_->thresholds && qx_->k > 0) {
        p->tx.assign(qx_->thresholds, qx_->thresholds + 2 * qx_->k);
        p->qx.thresholds = p->tx.data();
    }
    if (qy_->kind == QX_Q_CUSTOM && qy_->thresholds && qy_->k > 0) {
        p->ty.assign(qy_->thresholds, qy_->thresholds + 2 * qy_->k);
        p->qy.thresholds = p->ty.data();
    }
    p->lag_lo = lag_lo;
    p->lag_hi = lag_hi;
    p->path = path;
    qx_status st = plan_prepare(p);
    if (st != QX_OK) {
        delete p;
        return st;
    }
    *out = p;
    return QX_OK;
}

qx_status qx_plan_run(qx_plan* p, const void* x, const void* y, qx_result* results, void* stream)
{
    if (!p) return QX_ERR_INVALID;
    qx_context* ctx = p->ctx;
    if (!x || !y || !results) return fail(ctx, QX_ERR_INVALID, "x, y and results are required");
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    DevGuard dg(ctx->device);
    StreamOrder order(ctx, (cudaStream_t)stream);
    if (p->gen_s != ctx->scratch.gen || p->gen_c != ctx->counters.gen) {
        // another call regrew the context's scratch: re-derive the pointers
        qx_status st = plan_prepare(p);
        if (st != QX_OK) return st;
    }
    NttCall& c = p->pr.call;
    c.op[0].data = x;
    c.op[1].data = y;
    c.am.results = results;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    if (p->pr.path != QX_PATH_POPC) e = cudaMemsetAsync(c.stats, 0, (size_t)p->batch * 64, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "memset stats");
    e = p->pr.path == QX_PATH_DIRECT ? tc_window_run(c, p->pr.nx, s)
        : p->pr.path == QX_PATH_POPC ? popc_run(c, p->pr.nx, s) : ntt_run(c, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "kernel launch");
    return QX_OK;
}

// qx_plan_run from HOST rows: the plan's own device staging (allocated on
// first use), H2D of the rows' extent, the same launches as qx_plan_run on
// the context's host stream, D2H of the results, one synchronisation.  With
// page-locked rows the copies are asynchronous DMA; pageable rows go
// through the driver's staging (correct, slower).
qx_status qx_plan_run_host(qx_plan* p, const void* x, const void* y, qx_result* results)
{
    if (!p) return QX_ERR_INVALID;
    qx_context* ctx = p->ctx;
    if (!x || !y || !results) return fail(ctx, QX_ERR_INVALID, "x, y and results are required");
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    DevGuard dg(ctx->device);
    static const size_t esz[] = {4, 8, 8};
    const int64_t batch = p->batch;
    const size_t xb = (size_t)((batch - 1) * p->x.ld + p->x.n) * esz[p->x.dtype];
    const size_t yb = (size_t)((batch - 1) * p->y.ld + p->y.n) * esz[p->y.dtype];
    const size_t xa = (xb + 255) & ~(size_t)255, ya = (yb + 255) & ~(size_t)255;
    const size_t rb = (size_t)batch * sizeof(qx_result);
    cudaError_t e = cudaSuccess;
    // Small inputs in pinned host memory (latency-bound single pairs, BASELINE
    // config 1): no staging copies at all.  The kernels read the rows once,
    // straight over PCIe through the buffers' device aliases, and write the
    // records into a mapped pinned buffer of the plan: two H2D copies and one
    // D2H copy (each a driver call and a DMA start) leave the call's latency.
    if (xb + yb <= kZeroCopyBytes && ctx->knobs.zero_copy) {
        const void* xd = pinned_device_alias(x);
        const void* yd = xd ? pinned_device_alias(y) : nullptr;
        if (xd && yd) {
            if (p->hres_bytes < rb) {
                if (p->hres) cudaFreeHost(p->hres);
                p->hres = nullptr;
                p->hres_bytes = 0;
                e = cudaHostAlloc((void**)&p->hres, rb, cudaHostAllocMapped);
                if (e != cudaSuccess) return cuda_fail(ctx, e, "plan result buffer");
                p->hres_bytes = rb;
            }
            qx_result* hd = nullptr;
            e = cudaHostGetDevicePointer((void**)&hd, p->hres, 0);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "plan result buffer");
            cudaStream_t s = ctx->host_stream;
            qx_status st = qx_plan_run(p, xd, yd, hd, s);
            if (st != QX_OK) return st;
            e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "sync");
            memcpy(results, p->hres, rb);
            for (int64_t b = 0; b < batch; ++b)
                if (results[b].status) return (qx_status)results[b].status;
            return QX_OK;
        }
    }
    if (p->dstage_bytes < xa + ya + rb) {
        if (p->dstage) cudaFree(p->dstage);
        p->dstage = nullptr;
        p->dstage_bytes = 0;
        e = cudaMalloc(&p->dstage, xa + ya + rb);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "plan staging");
        p->dstage_bytes = xa + ya + rb;
    }
    char* d = (char*)p->dstage;
    cudaStream_t s = ctx->host_stream;
    e = cudaMemcpyAsync(d, x, xb, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d + xa, y, yb, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "H2D");
    qx_result* rd = (qx_result*)(d + xa + ya);
    qx_status st = qx_plan_run(p, d, d + xa, rd, s);
    if (st != QX_OK) return st;
    e = cudaMemcpyAsync(results, rd, rb, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "D2H");
    for (int64_t b = 0; b < batch; ++b)
        if (results[b].status) return (qx_status)results[b].status;
    return QX_OK;
}

int qx_plan_path(const qx_plan* p) { return p ? p->pr.path : -1; }

void qx_plan_destroy(qx_plan* p) { delete p; }

qx_status qx_xcorr_full(qx_context* ctx, const qx_signals* x, const qx_signals* y, int64_t batch,
                        const qx_quantizer* qx_, const qx_quantizer* qy_, int64_t* values, qx_result* stats,
                        qx_path path, void* stream)
{
    if (!ctx) return QX_ERR_INVALID;
    if (!values) return fail(ctx, QX_ERR_INVALID, "values is NULL");
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    DevGuard dg(ctx->device);
    StreamOrder order(ctx, (cudaStream_t)stream);
    Prepared pr;
    qx_status st = prepare(ctx, x, y, batch, qx_, qy_, INT64_MIN, INT64_MAX, false, path, &pr);
    if (st != QX_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    pr.call.values = values;
    cudaError_t e = cudaMemsetAsync(pr.call.stats, 0, (size_t)batch * 64, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "memset stats");
    e = ntt_run(pr.call, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "ntt launch");
    if (stats) {
        e = stats_to_results(pr.call.stats, stats, batch, s);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "stats");
    }
    return QX_OK;
}

static const char* kKindNames[QX_PROFILE_KINDS] = {"ntt_pass1", "ntt_pass2", "ntt_pass3", "crt_combine",
                                                    "quantize", "direct", "other", "direct_f4", "popc", ""};

const char* qx_profile_kind_name(int kind)
{
    return (kind >= 0 && kind < QX_PROFILE_KINDS) ? kKindNames[kind] : "";
}

qx_status qx_profile_begin(qx_context* ctx, int timed)
{
    if (!ctx) return QX_ERR_INVALID;
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    DevGuard dg(ctx->device);
    Profiler& p = ctx->prof;
    p.on = true;
    p.timed = timed != 0;
    p.launches = 0;
    for (long long& c : p.count) c = 0;
    p.nrec = 0;
    return QX_OK;
}

qx_status qx_profile_end(qx_context* ctx, qx_profile* out)
{
    if (!ctx || !out) return QX_ERR_INVALID;
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    DevGuard dg(ctx->device);
    Profiler& p = ctx->prof;
    memset(out, 0, sizeof(*out));
    out->launches = p.launches;
    for (int i = 0; i < QX_PROFILE_KINDS; ++i) out->count[i] = p.count[i];
    for (int i = 0; i < p.nrec; ++i) {
        cudaError_t e = cudaEventSynchronize(p.recs[i].b);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "profile sync");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, p.recs[i].a, p.recs[i].b);
        out->ms[p.recs[i].kind] += ms;
    }
    p.on = false;
    p.nrec = 0;
    return QX_OK;
}

qx_status qx_estimate_batch_host(qx_context* ctx, const qx_signals* x, const qx_signals* y, int64_t batch,
                                 const qx_quantizer* qx_, const qx_quantizer* qy_, int64_t lag_lo,
                                 int64_t lag_hi, qx_path path, qx_result* results)
{
    if (!ctx) return QX_ERR_INVALID;
    if (!results) return fail(ctx, QX_ERR_INVALID, "results is NULL");
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    DevGuard dg(ctx->device);
    StreamOrder order(ctx, ctx->host_stream);
    qx_status st;
    if ((st = check_signals(ctx, x, "x")) != QX_OK) return st;
    if ((st = check_signals(ctx, y, "y")) != QX_OK) return st;
    static const size_t esz[] = {4, 8, 8};
    // extent of the rows (they may overlap or repeat)
    const size_t xb = (size_t)((batch - 1) * x->ld + x->n) * esz[x->dtype];
    const size_t yb = (size_t)((batch - 1) * y->ld + y->n) * esz[y->dtype];
    const size_t xa = (xb + 255) & ~(size_t)255, ya = (yb + 255) & ~(size_t)255;
    const size_t rb = (size_t)batch * sizeof(qx_result);
    cudaError_t e = arena_reserve(ctx->stage, xa + ya + rb, false);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "staging");
    char* d = (char*)ctx->stage.ptr;
    cudaStream_t s = ctx->host_stream;
    e = cudaMemcpyAsync(d, x->data, xb, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d + xa, y->data, yb, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "H2D");
    qx_signals xd = *x, yd = *y;
    xd.data = d;
    yd.data = d + xa;
    qx_result* rd = (qx_result*)(d + xa + ya);
    st = qx_estimate_batch(ctx, &xd, &yd, batch, qx_, qy_, lag_lo, lag_hi, path, rd, s);
    if (st != QX_OK) return st;
    e = cudaMemcpyAsync(results, rd, rb, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "D2H");
    for (int64_t b = 0; b < batch; ++b)
        if (results[b].status) return (qx_status)results[b].status;
    return QX_OK;
}

// template search blocks (lags): the tensor-core window path's tile when
// the template fits it -- 32768 on the 2-SM fp4 mode (two records per
// block), 8192 on the 1-SM fp4 mode, 4096 on the int8 one -- else the
// largest block whose full correlogram fits one 2^19 transform
static int64_t tsearch_block(const qx_context* ctx, const qx_signals* t, const qx_signals* s,
                             const qx_quantizer* qa, const qx_quantizer* qb, qx_path path, bool* f2)
{
    *f2 = false;
    const int64_t nt = t->n;
    const bool tc = path != QX_PATH_NTT && path != QX_PATH_POPC && nt + 15 <= 4608 && nt % 4 == 0 &&
                    t->dtype == QX_F32 && s->dtype == QX_F32;
    if (!tc) return (1ll << 19) - 2 * nt + 2;
    const int64_t ka = qa->k, kb = qb->k;
    auto mode = [](const qx_quantizer* q) { return q->k == 1 ? 0 : (q->kind == QX_Q_UNIFORM ? 1 : 2); };
    const bool f4 = ctx->knobs.tc_f4 && ka <= 4 && kb <= 4 && mode(qa) == mode(qb) &&
                    (double)nt * ka * kb < 16777216.0;
    // (the 2-SM fp4 mode with 32768-lag blocks is retired: slower)
    *f2 = false;
    return f4 ? 8192 : 4096;
}

qx_status qx_template_search(qx_context* ctx, const qx_signals* tpl, const qx_signals* sig, const qx_quantizer* qx_,
                             const qx_quantizer* qy_, int64_t block, qx_path path, int64_t* summary, void* stream)
{
    if (!ctx) return QX_ERR_INVALID;
    if (!summary) return fail(ctx, QX_ERR_INVALID, "summary is NULL");
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    DevGuard dg(ctx->device);
    StreamOrder order(ctx, (cudaStream_t)stream);
    qx_status st;
    if ((st = check_signals(ctx, tpl, "template")) != QX_OK) return st;
    if ((st = check_signals(ctx, sig, "stream")) != QX_OK) return st;
    if ((st = check_quantizer(ctx, qx_, tpl->dtype)) != QX_OK) return st;
    if ((st = check_quantizer(ctx, qy_, sig->dtype)) != QX_OK) return st;
    const int64_t nt = tpl->n, ns = sig->n, nvalid = ns - nt + 1;
    if (nvalid < 1) return fail(ctx, QX_ERR_INVALID, "template longer than the stream");
    bool f2 = false;
    if (block <= 0) block = tsearch_block(ctx, tpl, sig, qx_, qy_, path, &f2);
    if (block < 1) return fail(ctx, QX_ERR_INVALID, "template too long for the block transform");
    // runs of blocks: [2-SM 32768-lag blocks (2 records each)], `block`-lag
    // blocks, one shorter remainder block
    const int64_t big = 32768;
    int64_t n2 = f2 ? nvalid / big : 0;
    if (n2 < 2) n2 = 0;  // the 2-SM mode runs clusters over >= 2 blocks
    // records: 2 per 32768-lag block (<= 1 per `block` lags, block <= 16384)
    // or 1 per `block`-lag block, + the remainder
    const int64_t nrec = nvalid / block + 2;
    const int sms = device_sms();
    const size_t rb = (size_t)nrec * sizeof(qx_result), pb = (size_t)sms * 64;
    cudaError_t e = arena_reserve(ctx->records, rb + pb + 256, false);
    if (e == cudaSuccess) e = arena_reserve(ctx->mcounter, 256, true);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "template search scratch");
    qx_result* recs = (qx_result*)ctx->records.ptr;
    void* partials = (char*)ctx->records.ptr + ((rb + 255) & ~(size_t)255);
    static const size_t esz[] = {4, 8, 8};
    const size_t es = esz[sig->dtype];
    MergeSegs segs = {};
    // block b of a run starting at stream sample s0: the template (stride-0
    // row) against samples [s0 + b*B, s0 + b*B + B + nt - 1): overlapping
    // strided rows, no copies
    qx_signals x = *tpl, y = *sig;
    x.ld = 0;
    x.start = 0;
    y.start = 0;
    qx_result* r = recs;
    int64_t s0 = 0;
    int ns_ = 0;
    if (n2) {
        y.n = big + nt - 1;
        y.ld = big;
        st = estimate_batch_on(ctx, &x, &y, n2, qx_, qy_, 0, big - 1, path, r, stream, nullptr, nullptr, true);
        if (st == QX_ERR_UNSUPPORTED) {
            n2 = 0;  // not on the 2-SM mode: every block on `block`
        } else {
            if (st != QX_OK) return st;
            segs.seg[ns_++] = MergeSeg{(const long long*)r, 2 * n2, 2, big, 0};
            r += 2 * n2;
            s0 = n2 * big;
        }
    }
    const int64_t nfull = (nvalid - s0) / block, rem = (nvalid - s0) % block;
    if (nfull) {
        y.data = (const char*)sig->data + (size_t)s0 * es;
        y.n = block + nt - 1;
        y.ld = block;
        st = estimate_batch_on(ctx, &x, &y, nfull, qx_, qy_, 0, block - 1, path, r, stream, nullptr, nullptr);
        if (st != QX_OK) return st;
        segs.seg[ns_++] = MergeSeg{(const long long*)r, nfull, 1, block, s0};
        r += nfull;
        s0 += nfull * block;
    }
    if (rem) {
        x.ld = 0;  // still the stride-0 template row: the shared-template modes take it
        y.data = (const char*)sig->data + (size_t)s0 * es;
        y.n = rem + nt - 1;
        y.ld = y.n;
        st = estimate_batch_on(ctx, &x, &y, 1, qx_, qy_, 0, rem - 1, path, r, stream, nullptr, nullptr);
        if (st != QX_OK) return st;
        segs.seg[ns_++] = MergeSeg{(const long long*)r, 1, 1, rem, s0};
    }
    ctx->prof.pre(KK_OTHER, (cudaStream_t)stream);
    e = merge_blocks_launch(segs, (long long)(sig->start - tpl->start), partials, (int*)ctx->mcounter.ptr,
                            (long long*)summary, sms, (cudaStream_t)stream);
    ctx->prof.post(KK_OTHER, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "merge launch");
    return QX_OK;
}

qx_status qx_decode_pcm16(qx_context* ctx, const void* pcm, int64_t n, float* out, void* stream)
{
    if (!ctx) return QX_ERR_INVALID;
    if (!pcm || !out || n < 1) return fail(ctx, QX_ERR_INVALID, "pcm/out must be non-NULL and n >= 1");
    if ((uintptr_t)pcm % 16 || (uintptr_t)out % 16) return fail(ctx, QX_ERR_INVALID, "pcm/out must be 16-byte aligned");
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    DevGuard dg(ctx->device);
    StreamOrder order(ctx, (cudaStream_t)stream);
    const int sms = device_sms();
    cudaStream_t s = (cudaStream_t)stream;
    ctx->prof.pre(KK_QUANT, s);
    cudaError_t e = pcm16_launch(pcm, n, out, sms, s);
    ctx->prof.post(KK_QUANT, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "decode_pcm16");
    return QX_OK;
}

qx_status qx_estimate_sweep(qx_context* ctx, const qx_signals* x, const qx_signals* y, int64_t batch, int64_t nq,
                            const qx_quantizer* qxs, const qx_quantizer* qys, int64_t lag_lo, int64_t lag_hi,
                            qx_path path, qx_result* results, void* stream)
{
    if (!ctx) return QX_ERR_INVALID;
    if (!results || !qxs || !qys) return fail(ctx, QX_ERR_INVALID, "results/quantizers is NULL");
    if (nq < 1) return fail(ctx, QX_ERR_INVALID, "nq must be >= 1");
    if (batch < 1) return fail(ctx, QX_ERR_INVALID, "batch must be >= 1");
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    DevGuard dg(ctx->device);
    StreamOrder order(ctx, (cudaStream_t)stream);
    qx_status st;
    if ((st = check_signals(ctx, x, "x")) != QX_OK) return st;
    if ((st = check_signals(ctx, y, "y")) != QX_OK) return st;
    int nl = 0;
    cudaError_t e = open_lanes(ctx, nq, &nl);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "lanes");
    // fork: the lanes start after the caller's stream has produced x and y
    cudaStream_t s = (cudaStream_t)stream;
    if ((e = cudaEventRecord(ctx->fork, s)) != cudaSuccess) return cuda_fail(ctx, e, "fork");
    for (int l = 0; l < nl && e == cudaSuccess; ++l) e = cudaStreamWaitEvent(ctx->lanes[l].stream, ctx->fork, 0);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "fork");
    for (int64_t q = 0; q < nq; ++q) {
        Lane& L = ctx->lanes[q % nl];
        st = estimate_batch_on(ctx, x, y, batch, &qxs[q], &qys[q], lag_lo, lag_hi, path, results + q * batch,
                               L.stream, &L.scratch, &L.counters);
        if (st != QX_OK) return st;
    }
    // join: the caller's stream continues after every lane
    for (int l = 0; l < nl && e == cudaSuccess; ++l) {
        e = cudaEventRecord(ctx->lanes[l].done, ctx->lanes[l].stream);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ctx->lanes[l].done, 0);
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "lane join");
    return QX_OK;
}

qx_status qx_estimate_sweep_host(qx_context* ctx, const qx_signals* x, const qx_signals* y, int64_t batch,
                                 int64_t nq, const qx_quantizer* qxs, const qx_quantizer* qys, int64_t lag_lo,
                                 int64_t lag_hi, qx_path path, qx_result* results)
{
    if (!ctx) return QX_ERR_INVALID;
    if (!results || !qxs || !qys) return fail(ctx, QX_ERR_INVALID, "results/quantizers is NULL");
    if (nq < 1) return fail(ctx, QX_ERR_INVALID, "nq must be >= 1");
    if (batch < 1) return fail(ctx, QX_ERR_INVALID, "batch must be >= 1");
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    DevGuard dg(ctx->device);
    StreamOrder order(ctx, ctx->host_stream);
    qx_status st;
    if ((st = check_signals(ctx, x, "x")) != QX_OK) return st;
    if ((st = check_signals(ctx, y, "y")) != QX_OK) return st;
    static const size_t esz[] = {4, 8, 8};
    const size_t ex = esz[x->dtype], ey = esz[y->dtype];
    const size_t xb = (size_t)((batch - 1) * x->ld + x->n) * ex;
    const size_t yb = (size_t)((batch - 1) * y->ld + y->n) * ey;
    const size_t xa = (xb + 255) & ~(size_t)255, ya = (yb + 255) & ~(size_t)255;
    const size_t rb = (size_t)(nq * batch) * sizeof(qx_result);
    cudaError_t e = arena_reserve(ctx->stage, xa + ya + rb, false);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "staging");
    if (!ctx->copy_stream && (e = cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking)) != cudaSuccess)
        return cuda_fail(ctx, e, "copy stream");
    char* d = (char*)ctx->stage.ptr;
    qx_result* rd = (qx_result*)(d + xa + ya);
    cudaStream_t s = ctx->host_stream, cs = ctx->copy_stream;
    // chunks of disjoint rows are staged on the copy stream while the compute
    // stream works on the previous chunk; overlapping / repeated rows are
    // staged whole (one chunk)
    const bool disjoint = x->ld >= x->n && y->ld >= y->n;
    // quantiser pairs run on up to 4 compute lanes (streams with their own
    // scratch), so a chunk's launches overlap and small chunks stay efficient
    int nl = 0;
    // (QX_SWEEP_LANES may exceed nq here: consecutive chunks then run on different lanes)
    if ((e = open_lanes(ctx, nq, &nl, 2 * nq)) != cudaSuccess) return cuda_fail(ctx, e, "lanes");
    // chunks of >= 8 pairs (>= 16 on one lane: smaller launches lose their
    // tail waves), at most 8
    int64_t nchunk = disjoint ? std::max<int64_t>(1, std::min<int64_t>(batch / (nl > 1 ? 8 : 16), nl > 1 ? 8 : 4)) : 1;
    // (a chunk count only applies to disjoint rows: overlapping / repeated
    // rows are always staged whole)
    if (disjoint && ctx->knobs.sweep_chunks > 0) nchunk = std::min<int64_t>(batch, ctx->knobs.sweep_chunks);
    const int64_t per = (batch + nchunk - 1) / nchunk;
    // chunk bounds: with lanes and >= 4 chunks the first and last chunks are
    // half size (less exposed copy before the first launch, shorter compute
    // tail after the last copy)
    std::vector<std::pair<int64_t, int64_t>> chunks;  // (first pair, pairs)
    {
        // tapered ends (first and last chunk per/T pairs, T = QX_SWEEP_TAPER, default 2):
        // less copy exposed before the first launch, a shorter compute tail
        const bool taper = nl > 1 && nchunk >= 4 && per >= 2 && !ctx->knobs.sweep_even;
        const int64_t T = ctx->knobs.sweep_taper;
        const int64_t q = std::max<int64_t>(1, per / T);
        int64_t b0 = 0;
        while (b0 < batch) {
            int64_t nb = (taper && b0 == 0) ? q : per;
            // taper: end on a q-pair chunk (the one before takes the remainder)
            if (taper && b0 > 0 && batch - b0 > q && batch - b0 - nb < q) nb = batch - b0 - q;
            nb = std::min(nb, batch - b0);
            chunks.emplace_back(b0, nb);
            b0 += nb;
        }
        // QX_SWEEP_PLAN="a,b,c,...": explicit chunk sizes (used when they sum to batch)
        if (ctx->knobs.sweep_plan_n && disjoint) {
            std::vector<std::pair<int64_t, int64_t>> plan;
            int64_t at = 0;
            for (int i = 0; i < ctx->knobs.sweep_plan_n; ++i) plan.emplace_back(at, ctx->knobs.sweep_plan[i]), at += ctx->knobs.sweep_plan[i];
            if (at == batch) chunks.swap(plan);
        }
        nchunk = (int64_t)chunks.size();
    }
    while ((int64_t)ctx->chunk_ev.size() < nchunk) {
        cudaEvent_t ev;
        if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return cuda_fail(ctx, e, "event");
        ctx->chunk_ev.push_back(ev);
    }
    // the previous call's compute must be done with the staging buffer
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(ctx, e, "sync");
    // measurement knob: QX_SWEEP_RESTAGE=0 skips the H2D copies (the staging
    // buffer still holds the previous call's identical inputs) to time the
    // same schedule compute-only
    const bool copy = ctx->knobs.sweep_restage;
    // and QX_SWEEP_COMPUTE=0 times the copies alone (results: the previous call's)
    const bool compute = ctx->knobs.sweep_compute;
    for (int64_t c = 0; c < nchunk; ++c) {
        const int64_t b0 = chunks[c].first, nb = chunks[c].second;
        const size_t xo = (size_t)(b0 * x->ld) * ex, yo = (size_t)(b0 * y->ld) * ey;
        const size_t xn = disjoint ? (size_t)((nb - 1) * x->ld + x->n) * ex : xb;
        const size_t yn = disjoint ? (size_t)((nb - 1) * y->ld + y->n) * ey : yb;
        e = copy ? cudaMemcpyAsync(d + xo, (const char*)x->data + xo, xn, cudaMemcpyHostToDevice, cs) : cudaSuccess;
        if (e == cudaSuccess && copy)
            e = cudaMemcpyAsync(d + xa + yo, (const char*)y->data + yo, yn, cudaMemcpyHostToDevice, cs);
        if (e == cudaSuccess) e = cudaEventRecord(ctx->chunk_ev[c], cs);
        for (int l = 0; l < nl && e == cudaSuccess; ++l) e = cudaStreamWaitEvent(ctx->lanes[l].stream, ctx->chunk_ev[c], 0);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "H2D");
        qx_signals xd = *x, yd = *y;
        xd.data = d + xo;
        yd.data = d + xa + yo;
        for (int64_t q = 0; q < nq && compute; ++q) {
            Lane& L = ctx->lanes[(c * nq + q) % nl];
            st = estimate_batch_on(ctx, &xd, &yd, nb, &qxs[q], &qys[q], lag_lo, lag_hi, path, rd + q * batch + b0,
                                   L.stream, &L.scratch, &L.counters);
            if (st != QX_OK) return st;
        }
    }
    for (int l = 0; l < nl && e == cudaSuccess; ++l) {
        e = cudaEventRecord(ctx->lanes[l].done, ctx->lanes[l].stream);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ctx->lanes[l].done, 0);
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "lane join");
    e = cudaMemcpyAsync(results, rd, rb, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "D2H");
    for (int64_t i = 0; i < nq * batch; ++i)
        if (results[i].status) return (qx_status)results[i].status;
    return QX_OK;
}

// ---------------------------------------------------------------- multi-GPU

qx_status qx_summary_reduce_nccl(qx_context* ctx, int64_t* summary, void* comm, void* stream)
{
    if (!ctx) return QX_ERR_INVALID;
    if (!summary || !comm) return fail(ctx, QX_ERR_INVALID, "summary/comm is NULL");
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    DevGuard dg(ctx->device);
    StreamOrder order(ctx, (cudaStream_t)stream);
    cudaError_t e = arena_reserve(ctx->dist, 16 * 8, false);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "dist scratch");
    if (const char* why = summary_allreduce(comm, (long long*)summary, (long long*)ctx->dist.ptr, (cudaStream_t)stream))
        return fail(ctx, QX_ERR_CUDA, std::string("summary reduction: ") + why);
    return QX_OK;
}

qx_status qx_template_search_nccl(qx_context* ctx, const qx_signals* tpl, const qx_signals* sig, const qx_quantizer* qx_,
                                  const qx_quantizer* qy_, int64_t block, qx_path path, void* comm, int64_t* summary,
                                  void* stream)
{
    if (!ctx) return QX_ERR_INVALID;
    if (!summary || !comm) return fail(ctx, QX_ERR_INVALID, "summary/comm is NULL");
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    DevGuard dg(ctx->device);
    StreamOrder order(ctx, (cudaStream_t)stream);
    qx_status st;
    if ((st = check_signals(ctx, tpl, "template")) != QX_OK) return st;
    if (!sig || sig->n < 0) return fail(ctx, QX_ERR_INVALID, "stream is NULL");
    if (sig->n >= tpl->n) {
        st = qx_template_search(ctx, tpl, sig, qx_, qy_, block, path, summary, stream);
        if (st != QX_OK) return st;
    } else {
        // this rank's slice holds no valid lag: an empty summary (ties = 0,
        // y all-zero so the AND over ranks ignores it) joins the reduction
        static const int64_t empty[8] = {0, 0, 0, 0, 0, 1, 0, 0};
        cudaError_t e = cudaMemcpyAsync(summary, empty, sizeof(empty), cudaMemcpyHostToDevice, (cudaStream_t)stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);  // `empty` is pageable
        if (e != cudaSuccess) return cuda_fail(ctx, e, "empty summary");
    }
    return qx_summary_reduce_nccl(ctx, summary, comm, stream);
}

qx_status qx_estimate_batch_nccl(qx_context* ctx, const qx_signals* x, const qx_signals* y, int64_t batch,
                                 const qx_quantizer* qx_, const qx_quantizer* qy_, int64_t lag_lo, int64_t lag_hi,
                                 qx_path path, qx_result* results, void* comm, qx_result* all, void* stream)
{
    if (!ctx) return QX_ERR_INVALID;
    if (!results || !comm) return fail(ctx, QX_ERR_INVALID, "results/comm is NULL");
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    DevGuard dg(ctx->device);
    StreamOrder order(ctx, (cudaStream_t)stream);
    qx_status st = qx_estimate_batch(ctx, x, y, batch, qx_, qy_, lag_lo, lag_hi, path, results, stream);
    if (st != QX_OK || !all) return st;
    if (const char* why = records_allgather(comm, results, (size_t)batch * sizeof(qx_result), all, (cudaStream_t)stream))
        return fail(ctx, QX_ERR_CUDA, std::string("result gather: ") + why);
    return QX_OK;
}

qx_status qx_comm_rank_size(void* comm, int* rank, int* size)
{
    if (!comm || !rank || !size) return QX_ERR_INVALID;
    return comm_rank_size(comm, rank, size) ? QX_ERR_CUDA : QX_OK;
}

}  // extern "C"
