// qx_internal.h -- host/device argument blocks shared by the kernels and
// the C-ABI implementation (not part of the public ABI; see
// include/qxcorr_b200.h for that).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "qx_common.cuh"

namespace qx {

constexpr int kMaxThr = 256;  // threshold table capacity (k <= 128)

// Quantiser as the kernels see it: mode + table, passed by value (kernel
// parameter space) and staged into shared memory by each CTA.
struct QTable {
    int mode;       // QMode
    int k;          // level bound K
    int tsize;      // padded table size (power of two >= 2k)
    int tbits;
    double inv_step;
    double thr[kMaxThr];  // T[i], +inf padded; float32 tables hold exact floats
};

enum DType : int { DT_F32 = 0, DT_F64 = 1, DT_I64 = 2, DT_U32 = 3 /* internal: residues */ };

struct OperandDesc {
    const void* data;  // batch rows, row b at data + b*ld elements
    int64_t ld;
    int64_t n;         // samples per row
    int reverse;       // 1: operand is time-reversed (the x side)
    int dtype;         // DType
    QTable q;
};

// Per-pair statistics filled by pass 1: [pair][op][4] =
//   {sum of code^2, nonzero count, flag bits, unused}
enum StatFlag : unsigned { SF_NONFINITE = 1u, SF_CODE_RANGE = 2u };

struct ArgmaxOut {
    // device result records (public layout qx_result, see qxcorr_b200.h)
    void* results;
    int64_t first_lag;   // lag of correlogram index t = 0
    int64_t t_lo, t_hi;  // inclusive window on t
    long long* partials; // [batch][pstride][3]
    int* counters;       // [batch]
    int pstride;         // partial records per pair (>= CTAs per pair of any argmax launch)
};
constexpr int kMaxPartials = 64;        // four-step passes / combine
constexpr int kMaxPartialsLarge = 512;  // outer inverse of the large-P path

// Tables for one (prime, log2 P) transform plan, device pointers.
struct NttTables {
    ModP m;
    uint32_t p;
    int lp, l1, l2;
    const uint2* g1f;  // DIF group twiddles for N1 = 2^l1 (Shoup pairs, Sched layout)
    const uint2* g1i;  // DIT (inverse) group twiddles for N1
    const uint2* g2f;  // same for N2
    const uint2* g2i;
    const uint2* twf;  // forward four-step twiddles [P] (Shoup pairs)
    const uint2* twi;  // inverse four-step twiddles [P] incl. R/P (Shoup pairs; the R cancels the
                       // pointwise Montgomery product's R^-1)
    const uint2* twab; // twf factored per n2: 32 per-lane A then N1/32 per-row B (null if N1 < 32)
    const uint2* twib; // twi factored per k1pos: 32 per-lane A then N2/32 per-row B (null if N2 < 32)
};

// Optional per-launch accounting (qx_profile_begin/end): counts every kernel
// launch and, when timed, brackets it with CUDA events on its stream.
enum KernelKind : int { KK_PASS1 = 0, KK_PASS2, KK_PASS3, KK_COMBINE, KK_QUANT, KK_DIRECT, KK_OTHER, KK_DIRECT_F4, KK_POPC, KK_N };
struct Profiler {
    bool on = false, timed = false;
    long long launches = 0;
    long long count[KK_N + 1] = {0};
    struct Rec { int kind; cudaEvent_t a, b; };
    Rec* recs = nullptr;
    int nrec = 0, cap = 0;
    cudaEvent_t pending = nullptr;
    void pre(int kind, cudaStream_t s);
    void post(int kind, cudaStream_t s);
};

// Outer-pass tables of the large-P path (P = M * Q, M = 2^logm).
struct OuterTables {
    const uint2* gf;      // DIF group twiddles for M
    const uint2* gi;      // DIT group twiddles for M (directly after gf)
    const uint32_t* tl;   // omega_P^a * R,                 a < 8192
    const uint32_t* th;   // omega_P^(8192 b) * R,          b < P / 8192
    const uint32_t* tli;  // omega_P^-a * M^-1 * R
    const uint32_t* thi;  // omega_P^-(8192 b) * R
    const uint2* rf;      // omega_M^t  (Shoup pairs), t < M/2: register-resident outer DIF
    const uint2* ri;      // omega_M^-t (Shoup pairs), t < M/2: register-resident outer DIT
    const uint2* tcf;     // omega_P^(+tid * bitrev(r)) [r][tid], tid < 256 (Shoup pairs): per-thread factor
    const uint2* tci;     // omega_P^(-tid * bitrev(r)) [r][tid]   of the outer four-step twiddles
    const uint2* ucf;     // per-tile factor omega_P^(+256 tile * bitrev(r)) [tile][r] (Shoup pairs)
    const uint2* uci;     // per-tile factor M^-1 omega_P^(-256 tile * bitrev(r)) [tile][r]
};

// Tuning / measurement knobs of a context: the QX_* environment variables
// are read ONCE when the context is created (qx_context_create) and can be
// changed afterwards only through qx_context_set_option; no entry point reads
// the environment per call.
struct Knobs {
    int64_t chunk_pairs = 0;   // QX_CHUNK_PAIRS: NTT pairs per launch group (0: ~1.5 GiB of scratch)
    int sweep_lanes = 0;       // QX_SWEEP_LANES: sweep compute lanes (0: min(nq, 4))
    int sweep_chunks = 0;      // QX_SWEEP_CHUNKS: host-sweep staging chunks (0: plan; disjoint rows only)
    int sweep_taper = 2;       // QX_SWEEP_TAPER: first/last chunk = per/T pairs
    int sweep_even = 0;        // QX_SWEEP_EVEN=1: no tapered ends
    int sweep_restage = 1;     // QX_SWEEP_RESTAGE=0: skip the H2D copies (compute-only timing)
    int sweep_compute = 1;     // QX_SWEEP_COMPUTE=0: skip the kernels (copy-only timing)
    int popc = 1;              // QX_POPC=0: never pick the popc path on AUTO
    int popc_timing = 0;       // QX_POPC_TIMING=1: popc correlation kernel prints its phase times
    int tc_f4 = 1;             // QX_TC_F4=0: no fp4 tensor-core template search
    int zero_copy = 1;         // QX_ZERO_COPY=0: qx_plan_run_host always stages small pinned rows on the device
    int64_t sweep_plan[16] = {0};  // QX_SWEEP_PLAN="a,b,...": explicit host-sweep chunk sizes
    int sweep_plan_n = 0;
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device)
cudaError_t set_max_smem(const void* fn, size_t bytes);
// SM count of the current device (cached per device)
int device_sms();

struct NttCall {
    const Knobs* knobs;     // the context's knobs (never null)
    OperandDesc op[2];
    int64_t batch;
    int64_t nout;           // n_u + n_v - 1
    int np;                 // number of primes (1..3)
    NttTables tab[3];
    uint64_t garner_inv[3]; // inv(p0*..*p_{i-1}) mod p_i
    int zero_upper;         // both operands fit the lower half of P
    // scratch (device)
    uint32_t* Y;              // [chunk][2][P] forward transforms, Y^T layout
    uint32_t* Z;              // [chunk][P] pass-2 output (natural layout)
    uint32_t* R;              // [chunk][np][P] residues (np > 1)
    unsigned long long* stats;  // [batch][2][4]
    // outputs: exactly one of
    ArgmaxOut am;             // argmax mode (am.results != nullptr)
    int64_t* values;          // full correlogram mode [batch][nout]
    int64_t chunk;            // pairs per launch group
    Profiler* prof;           // may be null
    // large-P path (lp > 19): tab[] are the inner (2^lq) tables
    int large, logm, lq;
    OuterTables otab[3];
    uint32_t* OUT;            // [2][chunk][P] outer forward output
    uint32_t* RI;             // [chunk*M][np][Q] inner inverse residues
    unsigned* popc_spart;     // popc path: [batch][G][4] per-CTA nonzero counts and flags
    uint32_t* popc_planes;    // popc path: [batch][2 (nxw + nyw)] code bit planes
    const int* popc_sched;    // popc path: [G + 1] first block of each CTA (per-shape cache)
    int popc_G;               // popc path: CTAs per pair
    int split2;               // the caller takes 2 records per pair (2-SM template-search blocks)
};

// Template-search merge input: up to three runs of per-block records
// (qx_result layout); record i of a run covers lags base + (i / rpb) * block + ...
struct MergeSeg {
    const long long* recs;
    int64_t n;      // records
    int rpb;        // records per block (2: the 2-SM mode's per-CTA halves)
    int64_t block;  // lags per block
    int64_t base;   // stream lag of the run's first block
};
struct MergeSegs {
    MergeSeg seg[3];
};

// launches every pass of the NTT correlation for all pairs on `stream`
cudaError_t ntt_run(const NttCall& c, cudaStream_t stream);
// builds host-side twiddle tables for (p, lp) and uploads them
cudaError_t ntt_make_tables(uint32_t p, uint32_t g, int lp, NttTables* out, void** dev_block);
cudaError_t ntt_make_outer_tables(uint32_t p, uint32_t g, int lp, int logm, OuterTables* out, void** dev_block);

}  // namespace qx
