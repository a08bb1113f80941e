/*
 * qxcorr_b200.h -- C ABI of the B200-native quantise -> integer
 * cross-correlation -> argmax engine (libqxcorr_b200.so).
 *
 * Plain C types only (no torch, no C++): a ctypes / cffi / cgo / JNI binding
 * can bind every symbol directly.  The entry points replace the reference
 * `qxcorr` hot path (/root/reference/pkg/src/qxcorr):
 *
 *   qx_quantize              <- quantize.apply / Quantizer.__call__
 *                               (quantize.py:53-65, 105-107)
 *   qx_quantize_packed       <- the same map as bit-packed b-bit codes
 *                               (b = 1, 2, 4, 8; apply() transfers these)
 *   qx_quantizer_thresholds  <- the same map, as an exact threshold table
 *                               (quantize.py:53-65)
 *   qx_xcorr_full            <- xcorr_int_bf / xcorr_int_ks
 *                               (intxcorr.py:96-100, 259-265): the full
 *                               correlogram, bit-identical int64 values
 *   qx_estimate_batch        <- estimate() lines 1-5 + argmax_set summary
 *                               (estimator.py:60-94, 50-57), batched, with an
 *                               optional lag window (new; parity = the full
 *                               reference correlogram sliced to the window)
 *   qx_estimate_batch_host   <- the same from host buffers (H2D/D2H inside)
 *   qx_estimate_sweep[_host] <- estimate() once per quantiser pair of a
 *                               bit-depth sweep (harness.py:141-147), device
 *                               rows / host buffers
 *   qx_template_search       <- estimate(template, stream) over the valid lags
 *
 * Conventions
 *   - Device pointers are caller-owned; `stream` is a cudaStream_t (NULL =
 *     legacy default stream).  Calls only enqueue work, except the *_host
 *     variants which synchronise.
 *   - Correlation index t in [0, n_x + n_y - 1) holds lag
 *     first_lag + t with first_lag = y.start - (x.start + n_x - 1)
 *     (signals.py:100-105, intxcorr.py:85-86); value(t) =
 *     sum_m u[m] * v[m + lag] on the quantised codes u = q_x(x), v = q_y(y).
 *   - Errors map 1:1 onto the reference's exceptions (see qx_status).
 */
#ifndef QXCORR_B200_H
#define QXCORR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QX_ABI_VERSION 4

typedef enum qx_status {
    QX_OK = 0,
    QX_ERR_INVALID = 1,              /* ValueError: bad argument */
    QX_DEGENERATE_QUANTIZATION = 2,  /* errors.DegenerateQuantization (estimator.py:83-86) */
    QX_DEGENERATE_INPUT = 3,         /* errors.DegenerateInput (intxcorr.py:109-110) */
    QX_BOUND_EXCEEDED = 4,           /* ValueError, N_min*K_u*K_v > 2^59 (intxcorr.py:89-93) */
    QX_INTERNAL_OVERFLOW = 5,        /* errors.InternalOverflow (intxcorr.py:140-141, 254-255) */
    QX_ERR_CUDA = 6,                 /* RuntimeError: CUDA failure */
    QX_ERR_UNSUPPORTED = 7,          /* shape/parameter outside this build's kernels */
    QX_ERR_NOMEM = 8,
    QX_ERR_NONFINITE = 9             /* NaN input (reference behaviour undefined) */
} qx_status;

typedef enum qx_dtype { QX_F32 = 0, QX_F64 = 1, QX_I64 = 2 } qx_dtype;

typedef enum qx_qkind {
    QX_Q_SIGN = 0,     /* quantize.sign()            (quantize.py:76-78) */
    QX_Q_UNIFORM = 1,  /* quantize.uniform(k, step)  (quantize.py:81-82) */
    QX_Q_CUSTOM = 2,   /* quantize.custom(thresholds)(quantize.py:85-89) */
    QX_Q_CODES = 3     /* input is already integer codes, |c| <= k (IntSignal) */
} qx_qkind;

typedef struct qx_quantizer {
    int32_t kind;              /* qx_qkind */
    int32_t reserved;
    int64_t k;                 /* level bound K (>= 1) */
    double step;               /* uniform step (> 0) */
    const double *thresholds;  /* custom: 2k strictly increasing, host memory */
} qx_quantizer;

typedef struct qx_signals {
    const void *data;  /* batch rows; row b starts at element b*ld */
    int32_t dtype;     /* qx_dtype */
    int32_t reserved;
    int64_t n;         /* samples per row (>= 1) */
    int64_t ld;        /* row stride in elements (>= 0; rows may overlap or repeat) */
    int64_t start;     /* Signal.start of every row */
} qx_signals;

/* Path selection for the argmax entry points.  AUTO picks DIRECT (tcgen05
 * tensor-core Toeplitz tiles) for lag windows of at most 4112 lags with
 * n_x <= 4593 and k <= 127 on float rows; else POPC (word-parallel XOR/AND +
 * popc on 1-level codes) for k = 1 quantisers on small single pairs (batch *
 * n_x * window <= 2^31, n_x <= 65536); else NTT (exact full-lag
 * number-theoretic transforms).  NTT / DIRECT / POPC force one path
 * (QX_ERR_UNSUPPORTED if its shape limits are not met).  qx_xcorr_full
 * always runs the NTT. */
typedef enum qx_path { QX_PATH_AUTO = 0, QX_PATH_NTT = 1, QX_PATH_DIRECT = 2, QX_PATH_POPC = 3 } qx_path;

/* per-pair flags in qx_result.flags */
#define QX_RF_DEGENERATE_X 1 /* x quantizes to all zeros */
#define QX_RF_DEGENERATE_Y 2
#define QX_RF_NONFINITE 4    /* NaN seen in x or y */
#define QX_RF_CODE_RANGE 8   /* integer codes outside [-k, k] */

typedef struct qx_result {
    int64_t value;   /* peak integer correlation (EstimationResult.peak_value_int) */
    int64_t lag;     /* smallest lag attaining it (argmax_set()[0]) */
    int64_t ties;    /* number of lags attaining it (len(argmax_set)) */
    int64_t sumsq_x; /* sum of squared codes of x: l2_norm(u)**2 */
    int64_t sumsq_y;
    int64_t nnz_x;   /* nonzero codes in x */
    int64_t nnz_y;
    int32_t flags;   /* QX_RF_* */
    int32_t status;  /* qx_status for this pair */
} qx_result;

typedef struct qx_context qx_context;

qx_status qx_context_create(int device, qx_context **out);
void qx_context_destroy(qx_context *ctx);
const char *qx_status_string(qx_status s);
const char *qx_context_last_error(const qx_context *ctx);

/* Tuning / measurement options of a context.  Their defaults come from the
 * QX_* environment variables, read once by qx_context_create (never per
 * call); this call changes them afterwards.  Names: "chunk_pairs",
 * "sweep_lanes", "sweep_chunks", "sweep_taper", "sweep_even",
 * "sweep_restage" (0: the host sweep skips its H2D copies -- compute-only
 * timing), "sweep_compute" (0: it skips its kernels -- copy-only timing),
 * "popc", "popc_timing" (1: the popc correlation kernel prints its phase
 * times), "tc_f4", "zero_copy" (0: qx_plan_run_host always stages the rows
 * on the device; by default rows of at most 1 MiB in pinned host memory are
 * read in place over PCIe and the records written to a mapped pinned buffer).
 * QX_ERR_INVALID for an unknown name.
 *
 * Threading and streams: every entry point locks the context, runs on the
 * context's device and restores the caller's current device.  Work enqueued
 * on a stream other than the previous call's waits for that call's work, so
 * the context's scratch is never used by two streams at once (use one
 * context per stream for concurrency). */
qx_status qx_context_set_option(qx_context *ctx, const char *name, int64_t value);
int qx_abi_version(void);

/* Exact threshold table of a quantiser for inputs of `dtype` (F32/F64):
 * out[i], i < 2k, is the smallest value of that type whose level is
 * >= i - k + 1, so level(v) = -k + #{i : v >= out[i]}.  out is 2k doubles
 * (float32 tables hold exactly representable floats). Host only. */
qx_status qx_quantizer_thresholds(const qx_quantizer *q, qx_dtype dtype, double *out);

/* codes[b*n + i] = q(x[b*ld + i]) as int64 (quantize.apply), plus per-row
 * sum of squares and nonzero counts (sumsq/nnz may be NULL). Device pointers. */
qx_status qx_quantize(qx_context *ctx, const qx_quantizer *q, const qx_signals *x, int64_t batch,
                      int64_t *codes, int64_t *sumsq, int64_t *nnz, void *stream);

/* Bit-packed codes (the fused quantiser of the north star, subsystem 1):
 * q(x[b*ld + i]) for every sample, packed little-endian into 32-bit words,
 * row b at codes + b * qx_packed_words(n, bits):
 *   bits = 2, 4, 8: two's-complement code of sample i in bits
 *                   [bits*(i % (32/bits)), +bits) of word i / (32/bits);
 *                   needs k <= 2^(bits-1) - 1 (QX_ERR_INVALID otherwise);
 *   bits = 1:       1-level quantisers (k == 1): two planes of ceil(n/32)
 *                   words, sign (code < 0) then nonzero (code != 0), sample i
 *                   at bit i % 32 of word i / 32.
 * Float rows are read with 16-byte vector loads when row starts are 16-byte
 * aligned.  sumsq / nnz (device int64[batch], optional) receive the per-row
 * sum of squared codes and nonzero count; flags (device int32, optional)
 * receives QX_RF_NONFINITE if any sample is NaN.  Enqueued on `stream`. */
qx_status qx_quantize_packed(qx_context *ctx, const qx_quantizer *q, const qx_signals *x, int64_t batch, int bits,
                             uint32_t *codes, int64_t *sumsq, int64_t *nnz, int32_t *flags, void *stream);
/* words per packed row (both planes for bits = 1) */
int64_t qx_packed_words(int64_t n, int bits);

/* Full correlograms values[b*(nx+ny-1) + t] of q_x(x_b) against q_y(y_b).
 * stats (optional, device) receives sumsq/nnz/flags per pair. */
qx_status qx_xcorr_full(qx_context *ctx, const qx_signals *x, const qx_signals *y, int64_t batch,
                        const qx_quantizer *qx, const qx_quantizer *qy, int64_t *values,
                        qx_result *stats, qx_path path, void *stream);

/* Peak summary per pair over lags [lag_lo, lag_hi] (clipped to the full
 * range; INT64_MIN/INT64_MAX = all lags).  results: device, batch entries. */
qx_status qx_estimate_batch(qx_context *ctx, const qx_signals *x, const qx_signals *y,
                            int64_t batch, const qx_quantizer *qx, const qx_quantizer *qy,
                            int64_t lag_lo, int64_t lag_hi, qx_path path, qx_result *results,
                            void *stream);

/* Prepared estimate_batch call (the low-latency form of qx_estimate_batch
 * for repeated calls of one shape, e.g. BASELINE config 1 served pair after
 * pair): qx_plan_create validates the shapes (x/y data may be NULL), builds
 * the quantiser tables, picks the path and lays out the scratch once;
 * qx_plan_run then takes only the row pointers (same shapes, dtypes, ld and
 * start as at creation) and enqueues exactly what qx_estimate_batch would,
 * with identical results.  A plan belongs to its context (destroy it first)
 * and, like the context, is used by one thread at a time. */
typedef struct qx_plan qx_plan;
qx_status qx_plan_create(qx_context *ctx, const qx_signals *x, const qx_signals *y, int64_t batch,
                         const qx_quantizer *qx, const qx_quantizer *qy, int64_t lag_lo, int64_t lag_hi,
                         qx_path path, qx_plan **out);
qx_status qx_plan_run(qx_plan *plan, const void *x, const void *y, qx_result *results, void *stream);
/* qx_plan_run from HOST rows and a HOST results array (batch entries): the
 * plan stages the rows' extent into its own device buffer, runs, copies the
 * results back and synchronises (page-locked rows: asynchronous DMA).  Rows of
 * at most 1 MiB in page-locked memory are not staged at all: the kernels read
 * them in place through their device alias and write the records to a mapped
 * page-locked buffer of the plan (option "zero_copy").
 * Returns the first per-pair error status, as qx_estimate_batch_host. */
qx_status qx_plan_run_host(qx_plan *plan, const void *x, const void *y, qx_result *results);
/* the qx_path the plan runs (never QX_PATH_AUTO) */
int qx_plan_path(const qx_plan *plan);
void qx_plan_destroy(qx_plan *plan);

/* As qx_estimate_batch, but x/y data and results are HOST pointers; the
 * library stages the inputs to the device, runs, copies results back and
 * synchronises.  Returns the first per-pair error status if any. */
qx_status qx_estimate_batch_host(qx_context *ctx, const qx_signals *x, const qx_signals *y,
                                 int64_t batch, const qx_quantizer *qx, const qx_quantizer *qy,
                                 int64_t lag_lo, int64_t lag_hi, qx_path path, qx_result *results);

/* Sweep of nq quantiser pairs over one batch of DEVICE rows (the bit-depth
 * sweep of BASELINE config 2 with its inputs resident in HBM): estimate() of
 * estimator.py:60-94 once per (qx[q], qy[q]), the quantiser pairs on up to
 * four concurrent compute lanes (streams with their own scratch) forked from
 * and joined back to `stream`; results (device) [q*batch + b] as
 * qx_estimate_batch.  Enqueued; does not synchronise. */
qx_status qx_estimate_sweep(qx_context *ctx, const qx_signals *x, const qx_signals *y,
                            int64_t batch, int64_t nq, const qx_quantizer *qx,
                            const qx_quantizer *qy, int64_t lag_lo, int64_t lag_hi,
                            qx_path path, qx_result *results, void *stream);

/* Sweep of nq quantiser pairs over one batch from HOST buffers (the
 * bit-depth sweep of BASELINE config 2, i.e. estimate() of estimator.py:60-94
 * once per (qx[q], qy[q])): the inputs are staged to the device once, in
 * pair chunks on a copy stream that overlaps the correlation of the previous
 * chunk; results[q*batch + b] is pair b under quantiser pair q.  Synchronises;
 * returns the first per-pair error status if any. */
qx_status qx_estimate_sweep_host(qx_context *ctx, const qx_signals *x, const qx_signals *y,
                                 int64_t batch, int64_t nq, const qx_quantizer *qx,
                                 const qx_quantizer *qy, int64_t lag_lo, int64_t lag_hi,
                                 qx_path path, qx_result *results);

/* Template search (BASELINE config 5): estimate(x=template, y=stream) of
 * estimator.py:60-94 restricted to the VALID lags (template fully inside the
 * stream), as its argmax_set summary (estimator.py:50-57).  tpl and sig are
 * single device rows (tpl->n <= sig->n).  The valid lags are cut into blocks
 * of `block` lags (<= 0: the path's tile -- 8192 on the fp4 tensor-core mode,
 * 4096 on the int8 one, else the largest block one 2^19 transform holds);
 * block b correlates the template with the overlapping strided stream row
 * [b*block, b*block + block + tpl->n - 1) and the per-block summaries are
 * merged on the device.  Enqueued on `stream`; writes the device int64[8]
 *   summary = {peak value, smallest lag at it (stream coordinates:
 *              + sig->start - tpl->start), ties, NaN seen, x all-zero,
 *              y all-zero in every block, a block failed, its status}
 * (the last four carry DegenerateQuantization / ValueError of
 * estimator.py:83-86 to the caller).  Replaces the caller-side loop of
 * estimate() calls over stream windows; no reference symbol has this name. */
qx_status qx_template_search(qx_context *ctx, const qx_signals *tpl, const qx_signals *sig,
                             const qx_quantizer *qx, const qx_quantizer *qy, int64_t block,
                             qx_path path, int64_t *summary, void *stream);

/* ---- Multi-GPU (one process per GPU; `comm` is an ncclComm_t, e.g. the
 * communicator of torch's ProcessGroupNCCL).  NCCL is resolved at run time
 * from the calling process (else libnccl.so.2), so this library has no
 * link-time NCCL dependency.  The samples never cross GPUs: each rank
 * searches its own lag range and the ranks exchange only 8-word summaries
 * (the reference has no distributed code; its only parallelism is the
 * thread pool of harness.py:301-305).
 *
 * qx_summary_reduce_nccl: the device int64[8] template-search summary (see
 * qx_template_search) of every rank -> the summary of the union of their
 * lag ranges, on every rank: max value, smallest lag attaining it, summed
 * ties (argmax_set, estimator.py:50-57), NaN / x-degenerate / failure flags
 * OR-ed, y-degenerate AND-ed.  Two collectives: MAX over the values and
 * flags, then one NCCL group of MAX (smallest holder lag) and SUM (holder
 * ties).  Exact for every int64 value and lag.  Enqueued on `stream`. */
qx_status qx_summary_reduce_nccl(qx_context *ctx, int64_t *summary, void *comm, void *stream);

/* Sharded template search (BASELINE config 5 over G GPUs): `sig` is THIS
 * rank's stream slice -- its share of the valid lags plus the
 * (template - 1)-sample halo, with sig->start = the slice's first sample in
 * stream coordinates -- and `summary` receives the reduced summary of the
 * whole stream on every rank (a rank whose slice is shorter than the
 * template contributes an empty summary).  = qx_template_search on the slice
 * + qx_summary_reduce_nccl. */
qx_status qx_template_search_nccl(qx_context *ctx, const qx_signals *tpl, const qx_signals *sig,
                                  const qx_quantizer *qx, const qx_quantizer *qy, int64_t block,
                                  qx_path path, void *comm, int64_t *summary, void *stream);

/* Pair-sharded batch (BASELINE configs 2/3 over G GPUs): qx_estimate_batch on
 * this rank's `batch` pairs into `results` (device), then, if `all` is not
 * NULL, ncclAllGather of every rank's records into all[rank * batch + b]
 * (equal `batch` on every rank).  No other collective: pairs are
 * independent. */
qx_status qx_estimate_batch_nccl(qx_context *ctx, const qx_signals *x, const qx_signals *y, int64_t batch,
                                 const qx_quantizer *qx, const qx_quantizer *qy, int64_t lag_lo,
                                 int64_t lag_hi, qx_path path, qx_result *results, void *comm,
                                 qx_result *all, void *stream);

/* rank and size of an NCCL communicator (ncclCommUserRank / ncclCommCount) */
qx_status qx_comm_rank_size(void *comm, int *rank, int *size);

/* Device decode of a mono PCM16 payload (little-endian int16, e.g. the data
 * chunk of a WAV file) to float32 samples pcm / 32768: the sample decode of
 * signalgen.load_wav_bytes (signalgen.py:150-172).  Exact, so the float32
 * entry points quantise these samples exactly as the reference quantises its
 * float64 ones.  pcm and out are 16-byte aligned device pointers. */
qx_status qx_decode_pcm16(qx_context *ctx, const void *pcm, int64_t n, float *out, void *stream);

/* Launch accounting for measurement (bench.py): between begin and end every
 * kernel the library launches is counted per kind and, when `timed`, bracketed
 * by CUDA events on its own stream.  qx_profile_end synchronises and returns
 * summed device milliseconds per kind (names via qx_profile_kind_name). */
#define QX_PROFILE_KINDS 10
typedef struct qx_profile {
    int64_t launches;
    int64_t count[QX_PROFILE_KINDS];
    double ms[QX_PROFILE_KINDS];
} qx_profile;
qx_status qx_profile_begin(qx_context *ctx, int timed);
qx_status qx_profile_end(qx_context *ctx, qx_profile *out);
const char *qx_profile_kind_name(int kind);

#ifdef __cplusplus
}
#endif
#endif /* QXCORR_B200_H */
