/*
 * tuner.h — C ABI of libdroplet_b200.so, the B200-native hot path of
 * "Explore as a Storm, Exploit as a Raindrop" (arXiv 2406.20037): measuring
 * candidate kernel schedules for Ansor-style sampling and Droplet Search.
 *
 * Citations: P:N = PAPER.md line N; R-xx = the readings table in DESIGN.md §3.
 *
 * Conventions (all calls):
 *  - Every call returns tuner_status; nothing throws or aborts across the ABI.
 *    On a non-OK status, tuner_last_error() returns a thread-local message.
 *  - Input arrays/structs are borrowed for the duration of the call and copied
 *    if retained.  Output arrays are caller-allocated with the stated capacity.
 *  - Device buffers (x, w, y, y_ref, y_absref) are caller-owned device memory
 *    (e.g. torch tensors' data_ptr()); the library never frees them.  The
 *    library owns only its internal scratch (freed by tuner_destroy).
 *  - A handle is not thread-safe: use one host thread per handle.
 *  - SPMD: when world > 1 every rank makes the same sequence of calls with the
 *    same arguments (except rank, device pointers and stream); every output is
 *    then identical on all ranks.
 *  - A bad candidate is not an error: it is a sample status.  Errors are API
 *    misuse and device/communication failure.  After TUNER_ECUDA the handle is
 *    dead and every later call on it returns TUNER_ESTATE.
 *
 * Layouts (R-C1..R-C3):
 *  - dense        : Y[m,n]     = sum_k X[m,k] W[n,k]        row-major, W is [N,K]
 *  - batch_matmul : Y[b,m,n]   = sum_k X[b,m,k] W[b,n,k]
 *  - conv2d       : Y[n,p,q,k] = sum_{r,s,c} X[n, p*sh-ph+r*dh, q*sw-pw+s*dw, c] W[k,r,s,c]
 *                   X NHWC, W KRSC, Y NPQK, zero padding, groups = 1,
 *                   P = (H + 2ph - dh(R-1) - 1)/sh + 1 (Q alike).
 *  - depthwise_conv2d : Y[n,p,q,c] = sum_{r,s} X[n, p*sh-ph+r*dh, q*sw-pw+s*dw, c] W[c,r,s]
 *                   groups = C = K (R-C5; the MobileNet / MnasNet / ShuffleNet /
 *                   EfficientNet layers): X NHWC, W [C][R][S], Y NPQC.
 *  - TUNER_F32 : x, w, y are float32.  TUNER_BF16 : x, w are bfloat16 (inputs
 *    already rounded), y is float32 (fp32 accumulation, R-C4).
 */
#ifndef DROPLET_B200_TUNER_H
#define DROPLET_B200_TUNER_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TUNER_MAX_KNOBS 16
#define TUNER_MAX_VALUES 64 /* per knob */

typedef struct tuner tuner_t; /* opaque, library-owned */

typedef enum {
    TUNER_OK = 0,
    TUNER_EINVAL = 1,    /* bad argument (NULL, budget < 1, NaN in cost table, ...) */
    TUNER_EDIM = 2,      /* index-vector length != the sketch's number of knobs */
    TUNER_ERANGE = 3,    /* index >= cardinality, unknown sketch, or a statically
                            invalid point passed where a valid one is required */
    TUNER_EOVERFLOW = 4, /* a sketch space larger than 2^62 points */
    TUNER_ESTATE = 5,    /* e.g. tuner_best before any measurement; dead handle */
    TUNER_ECUDA = 6,     /* CUDA error (sticky errors kill the handle) */
    TUNER_ENCCL = 7,     /* NCCL / collective failure */
    TUNER_ENOMEM = 8
} tuner_status;

typedef enum {
    TUNER_OP_DENSE = 0,
    TUNER_OP_BATCH_MATMUL = 1,
    TUNER_OP_CONV2D = 2,
    TUNER_OP_DEPTHWISE_CONV2D = 3
} tuner_op;
typedef enum { TUNER_F32 = 0, TUNER_BF16 = 1 } tuner_dtype;

/* Problem shape.  dense uses m, n, k (b ignored, taken as 1); batch_matmul uses
 * b, m, n, k; conv2d uses N, C, H, W, K, R, S and the stride/pad/dilation;
 * depthwise_conv2d the same with K == C (else TUNER_EINVAL).  */
typedef struct {
    int32_t dtype; /* tuner_dtype */
    int64_t b, m, n, k;
    int64_t N, C, H, W, K, R, S;
    int32_t stride_h, stride_w, pad_h, pad_w, dil_h, dil_w;
} tuner_shape;

/* The search space of one sketch (Def. 2.1: "one dimension for
 * each parameter that is allowed to vary").  values is the concatenation of
 * each knob's strictly increasing value list: knob d's values are
 * values[sum_{e<d} card[e] .. + card[d]).  In measured mode every value must be
 * one the sketch supports (see tuner_sketch_space), else TUNER_EINVAL.  In
 * cost-table mode sketch ids are free labels. */
typedef struct {
    int32_t sketch;        /* kernel template id (tuner_sketch_id) */
    int32_t nknobs;        /* <= TUNER_MAX_KNOBS */
    const int32_t* card;   /* [nknobs], each 1..TUNER_MAX_VALUES */
    const int32_t* values; /* [sum card] */
} tuner_knob_space;

/* A coordinate: the sketch plus an index vector into each knob's
 * value list.  n must equal the sketch's nknobs (else TUNER_EDIM). */
typedef struct {
    int32_t sketch;
    int32_t n;
    int32_t idx[TUNER_MAX_KNOBS];
} tuner_point;

typedef enum {
    TUNER_S_OK = 0,
    TUNER_S_INVALID = 1,    /* statically invalid: never launched, never a trial */
    TUNER_S_TIMEOUT = 2,    /* verify run exceeded opts.timeout_ms */
    TUNER_S_WRONG = 3,      /* max_err above tolerance (1e-4 f32, 2e-2 bf16) */
    TUNER_S_LAUNCH_FAIL = 4 /* launch error (non-sticky) */
} tuner_sample_status;

/* One measured candidate (a "sample" in the paper's sense).  cost_ns =
 * trimmed-mean per-launch time of the repeats (R-M2), +inf unless status ==
 * TUNER_S_OK.  rank = the rank that measured it. */
typedef struct {
    tuner_point pt;
    double cost_ns;
    double max_err;
    int32_t status;
    int32_t rank;
} tuner_result;

/* Droplet policies (tuner_droplet): PLAIN = the paper's prose, P:297-304 (best improving
 * neighbour of the +-1 ring, stop when none); GROW = after each ring move along u, probe the
 * doubling ray x_prev + 2^j u as one batch (R-D9, north_star "grows its step"); RADIUS = when
 * the +-1 ring holds no improving point, measure the axis-aligned ring at index distance
 * r = 2, 3, ... until one does (move there, r back to 1) or no ring point is in range -- then
 * converged, and the result is optimal along every axis line (R-D16: the original Droplet's
 * speculation, which P:276-277 says the paper removed). */
typedef enum { TUNER_DS_PLAIN = 0, TUNER_DS_GROW = 1, TUNER_DS_RADIUS = 2 } tuner_ds_policy;

/* Host-side all-gather used when set (e.g. a gloo process group through the
 * Python binding): every rank contributes `bytes` bytes from `send`; `recv`
 * (world * bytes) receives the rank-ordered concatenation.  Return 0 on success. */
typedef int (*tuner_allgather_fn)(void* ctx, const void* send, void* recv, int64_t bytes);

typedef struct {
    int32_t warmup;    /* untimed launches before timing (default 2) */
    int32_t repeats;   /* timed repeats; cost = their trimmed mean (default 10) */
    int32_t number;    /* launches per timed repeat, 0 = auto (>= 20 us per repeat) */
    double timeout_ms; /* verify-run time limit (default 1000) */
    uint64_t seed;     /* sampler seed (R-S1) */
    int32_t policy;    /* tuner_ds_policy (default GROW) */
    double alpha;      /* 0: strict cost compare; in (0,1): Droplet moves only when the
                          neighbour is also significantly faster (two-sided exact
                          Wilcoxon rank-sum on the repeat timings, p < alpha; P:410,
                          P:615, R-W1) */
    int32_t max_batch; /* candidates per measured batch / collective (default 512) */
    int32_t verify;    /* 1: verify every candidate (default), 0: skip */
    double early_cut;  /* > 0: a candidate whose verify run is slower than early_cut x
                          the best cost known so far is ranked by that run alone
                          (no timed repeats; SURVEY d.5).  0 = off (default). */
    /* cost-table mode (R-T1): dense costs per sketch in linear-id order,
     * concatenated in the order of `spaces`; +inf = invalid; NaN -> EINVAL.
     * Copied at create; no device is touched in this mode. */
    const double* cost_table;
    int64_t cost_table_len;
    /* optional, with cost_table: cost_nsamp (1..16) repeat timings per point,
     * [point][cost_nsamp] in the table's order, used by the alpha > 0 test */
    const double* cost_samples;
    int32_t cost_nsamp;
    /* multi-GPU candidate sharding (R-M1): batch item j is measured by rank
     * j mod world; results are all-gathered.  With world > 1 either
     * `allgather` is set or `nccl_unique_id` (128 bytes from
     * tuner_nccl_unique_id on rank 0) is given and NCCL is used (else
     * TUNER_EINVAL).  An exchange given at world 1 is used as well. */
    int32_t rank, world;
    const void* nccl_unique_id;
    tuner_allgather_fn allgather;
    void* allgather_ctx;
    /* measured mode: caller-owned device buffers (see layouts above) */
    const void* x;
    const void* w;
    void* y;
    /* optional verification reference (device, fp32, same shape as y); when
     * NULL the library computes it with its naive fp64 kernel (Def. 2.1). */
    const float* y_ref;
    const float* y_absref; /* sum |x||w| per output, device fp32 */
    void* stream;          /* cudaStream_t (e.g. a torch stream); NULL = default */
    /* optional append-only JSONL trial log: every measured
     * candidate is appended as one line keyed by the problem (op, shape, dtype); at create,
     * the lines of an existing log with this tuner's key and sketches are replayed into the
     * history (no re-measurement: a killed tuning job resumes where it stopped).  NULL = off.
     * Rank 0 writes; every rank replays.  A malformed line -> TUNER_EINVAL at create. */
    const char* trial_log;
} tuner_opts;

typedef struct {
    tuner_point best;
    double best_cost;
    int32_t trials_used; /* new measurements in this call (R-D14) */
    int32_t rounds;      /* ring steps + ray steps (R-D15) */
    int32_t converged;   /* 1: every valid neighbour of best measured, none better */
    int32_t traj_len;    /* accepted points incl. the start */
} tuner_droplet_report;

typedef struct {
    const void* x;
    const void* w;
    void* y;
} tuner_buffers;

/* Fill *o with the defaults listed above. */
void tuner_opts_default(tuner_opts* o);

/* Sketch catalogue.  tuner_sketches lists the sketch ids that implement (op,
 * dtype); tuner_sketch_space returns a sketch's full supported knob space
 * (card[TUNER_MAX_KNOBS], values[TUNER_MAX_KNOBS*TUNER_MAX_VALUES]);
 * tuner_knob_name returns a static string ("BM", "SPLIT_K", ...) or NULL.
 * Sketch ids (a sketch = one fixed sequence of transformations of the loop nest,
 * Def. 2.1; its knobs are the annotations):
 *   0 simt_gemm_f32 / 1 simt_igemm_conv_f32     register-staged SIMT tiles (fp32)
 *   7 simt_pipe_gemm_f32 / 8 simt_pipe_conv_f32 cp.async multistage SIMT tiles (fp32)
 *   9 simt_direct_conv_f32 / 10 ..._bf16        direct conv, C <= 16 stems
 *   2 tc_gemm_bf16 / 3 tc_igemm_conv_bf16       tcgen05 / TMEM / TMA (bf16 in, fp32 out)
 *   4 simt_igemm_conv_bf16                      SIMT implicit GEMM on bf16 inputs
 *   5 simt_dwconv_f32 / 6 simt_dwconv_bf16      depthwise conv
 *   11 tc_halo_conv_bf16                        tcgen05 conv, halo row tiles (stride 1, C % 64 == 0) */
tuner_status tuner_sketches(int32_t op, int32_t dtype, int32_t* ids, int32_t cap, int32_t* n_out);
tuner_status tuner_sketch_space(int32_t sketch, int32_t* nknobs, int32_t* card, int32_t* values);
/* The static validity rule of a sketch ("sketch rules are hardware-dependent"; P:596-599
 * schedules exceeding the hardware's limits are invalid) for one point given by its knob VALUES
 * (not indices; nvalues = the sketch's knob count) on a problem shape, without a tuner handle
 * and without a device: the rule tuner_point_valid applies in measured mode.  *valid = 0/1.
 * EINVAL on a NULL pointer or a bad shape, ERANGE on an unknown sketch, EDIM on a wrong count. */
tuner_status tuner_sketch_valid(int32_t op, const tuner_shape* shape, int32_t sketch, const int32_t* values,
                                int32_t nvalues, int32_t* valid);
const char* tuner_sketch_name(int32_t sketch);
const char* tuner_knob_name(int32_t sketch, int32_t knob);

/* Create a tuner for one layer (one kernel, "a graph of kernels").
 * spaces: the sketches to search (nspaces >= 1).  In measured mode opts->x/w/y
 * must be set and the device current on the calling thread is used. */
tuner_status tuner_create(int32_t op, const tuner_shape* shape, const tuner_knob_space* spaces,
                          int32_t nspaces, const tuner_opts* opts, tuner_t** out);

/* Static validity of a point for this tuner's shape (Ansor's hardware-
 * dependent rules; thread / shared-memory / TMEM limits).  *valid = 0/1. */
tuner_status tuner_point_valid(const tuner_t* t, const tuner_point* pt, int32_t* valid);

/* Ansor-style proposal (R-S1): draw n distinct, statically valid,
 * not-yet-measured points with the SplitMix64 sampler, measure them (sharded,
 * in batches of max_batch), append them to history.  out: caller array of n;
 * *n_out = number actually drawn (< n only if 64*n draws were exhausted). */
tuner_status tuner_sample(tuner_t* t, int32_t n, tuner_result* out, int32_t* n_out);

/* Grid search, an exploitation alternative of RQ4 (AutoTVM's grid
 * tuner): measure the next n statically valid, not-yet-measured points in
 * enumeration order (sketch order, then row-major linear id, last knob fastest),
 * continuing from where the previous tuner_grid call stopped.  out: caller array
 * of n; *n_out < n only when the space is exhausted. */
tuner_status tuner_grid(tuner_t* t, int32_t n, tuner_result* out, int32_t* n_out);

/* Ansor-style evolutionary exploration (reading R-E1; the learned cost
 * model is out of scope, so every child is measured): generation 0 is
 * tuner_sample's draw of min(pop, n) points; each later generation breeds up to
 * min(pop, n - used) new valid, unmeasured children from the `elite` best
 * measured points by uniform crossover (same sketch) and one resampled knob.
 * out: caller array of n; *n_out = points measured (< n if the space runs dry).
 * EINVAL if pop < 1 or elite < 1. */
tuner_status tuner_evolve(tuner_t* t, int32_t n, int32_t pop, int32_t elite, tuner_result* out,
                          int32_t* n_out);

/* Multi-layer trial budget (Ansor's task scheduler; reading
 * R-F3): every layer first explores min(floor(budget/L), 64) trials (at least 1),
 * then the remaining trials go in `increment`-sized grants to the layer with the
 * largest weight x best cost, after dropping layers whose weight x best cost is
 * below drop_frac of the model total.  Exploration is tuner_evolve(pop, elite).
 * layers: L tuner handles (one per distinct kernel); weights[L] > 0 (occurrences
 * in the model); trials[L] receives the trials spent per layer.  SPMD-safe. */
tuner_status tuner_schedule(tuner_t* const* layers, int32_t nlayers, const double* weights, int64_t budget,
                            int32_t increment, double drop_frac, int32_t pop, int32_t elite, int64_t* trials);

/* Measure an explicit list of points (e.g. exhaustive grid).
 * Already-measured points are returned from the memo and not re-measured. */
tuner_status tuner_measure(tuner_t* t, const tuner_point* pts, int32_t n, tuner_result* out);

/* Droplet Search (R-D2..R-D15) from `start` with at most `budget`
 * new measurements (100).  traj: optional caller array of traj_cap
 * accepted points.  EINVAL if budget < 1; EDIM / ERANGE for a bad start. */
tuner_status tuner_droplet(tuner_t* t, const tuner_point* start, int32_t budget, tuner_point* traj,
                           int32_t traj_cap, tuner_droplet_report* report);

/* The repeat timings (ns per launch, <= 16) behind a measured point's cost:
 * out[cap], *n_out = count.  ERANGE if the point was never measured. */
tuner_status tuner_timings(const tuner_t* t, const tuner_point* pt, float* out, int32_t cap, int32_t* n_out);

/* Best-of-N: first argmin of cost over history (R-B1).  ESTATE if empty. */
tuner_status tuner_best(const tuner_t* t, tuner_result* out);

/* The same restricted to one sketch's points: the start of a per-sketch Droplet Search
 * (R-D17: Droplet moves inside one sketch's space, so DPAnsor over several sketches
 * hands each sketch's best configuration to its own Droplet run).  ERANGE if the sketch is not
 * in this tuner's spaces; ESTATE if none of its points has a finite cost. */
tuner_status tuner_best_of_sketch(const tuner_t* t, int32_t sketch, tuner_result* out);

/* All measured samples in measurement order. */
tuner_status tuner_history(const tuner_t* t, tuner_result* out, int64_t cap, int64_t* n_out);

/* Run candidate `cfg` once on caller buffers, asynchronously on `stream`
 * (NULL = the tuner's stream).  Split-K schedules zero y first (part of the
 * schedule).  ERANGE if cfg is statically invalid; ESTATE in cost-table mode.
 * Stream-K schedules (tcgen05 SCHED >= 1) use a workspace owned by the handle,
 * allocated at the first such launch: that launch must not be inside a stream
 * capture (ESTATE), and such launches of one handle must be ordered (one stream). */
tuner_status kernel_run(const tuner_t* t, const tuner_point* cfg, const tuner_buffers* buf,
                        void* stream);

/* The naive schedule of Def. 2.1 on the device in fp64: y_ref (fp32)
 * and y_absref = sum |x||w| (fp32), used as the verification reference. */
tuner_status tuner_reference(const tuner_t* t, const tuner_buffers* buf, float* y_ref,
                             float* y_absref, void* stream);

/* Counters since create: candidate kernel launches (incl. graph nodes),
 * measured candidates, collectives issued, host wall ns inside measurement; and the
 * measurement tiers (measured mode, this rank): early_cut = candidates ranked by their
 * verify run alone (R-M3), light = candidates timed with 3 repeats instead of R,
 * precise = candidates re-timed over the long windows of R-M4, calibrations = cross-rank
 * batch winners re-timed on rank 0 (world > 1). */
typedef struct {
    int64_t kernel_launches;
    int64_t candidates;
    int64_t collectives;
    int64_t batches;
    double measure_wall_ns;
    int64_t early_cut;
    int64_t light;
    int64_t precise;
    int64_t calibrations;
    int64_t replayed; /* history entries restored from opts.trial_log at create */
} tuner_stats;
tuner_status tuner_get_stats(const tuner_t* t, tuner_stats* out);

/* 128-byte NCCL unique id (call on rank 0, broadcast to the others). */
tuner_status tuner_nccl_unique_id(void* out128);

void tuner_destroy(tuner_t* t);
const char* tuner_last_error(void);

/* Total candidate-kernel launches by this process (all handles). */
int64_t tuner_global_launch_count(void);

/* The significance test of the paper's methodology ("the p-value (produced via the
 * non-parametric Wilcoxon rank-sum test)"; reading R-W1): two-sided exact rank-sum
 * test on midranks of the samples a[n1] and b[n2] (e.g. two candidates' repeat timings from
 * tuner_timings) -> *p in (0, 1]; 1 when either side is empty.  EINVAL for NULL pointers or
 * more than 16 samples per side.  The same routine gates Droplet's moves when alpha > 0. */
tuner_status tuner_rank_sum_p(const float* a, int32_t n1, const float* b, int32_t n2, double* p);

/* FP32 pipe peak microbenchmark (BASELINE.md §2 "the build must measure it
 * with an FFMA microbenchmark"): the roofline denominator of the SIMT sketches.  Runs on the
 * current device on a private stream and synchronises; best of 5 timed launches of
 * (SMs x 8) CTAs x 256 threads, each thread 16 independent FMA recurrences.
 * mode 0: 3-register FFMA; 1: FFMA2 (fma.rn.f32x2, the form the SIMT sketches issue);
 * 2: FFMA with immediate operands.  *tflops = 2 x FMAs / time; *ms (may be NULL) = the
 * launch time.  TUNER_EINVAL for a bad mode or NULL tflops, TUNER_ECUDA without a device. */
tuner_status tuner_probe_fp32_peak(int32_t mode, double* tflops, double* ms);

#ifdef __cplusplus
}
#endif
#endif /* DROPLET_B200_TUNER_H */
