/*
 * tfft.h — C ABI of the B200-native fault-tolerant batched FFT
 * (libtfft.so, built from paper_2405_02520_b200/csrc/).
 *
 * Plain pointers, sizes and status codes only: no torch / Python types.
 * Device pointers are CUDA global-memory addresses on the plan's device;
 * `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 * Every call is stream-ordered. A plan handle must not be used concurrently
 * from two host threads. Status: TFFT_OK (0) or an error code; the message of
 * the last error on the calling thread is returned by tfft_last_error().
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/pkg/src/fftshield/...).
 */
#ifndef TFFT_H
#define TFFT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum tfft_status {
    TFFT_OK = 0,
    TFFT_EINVAL = 1,        /* bad argument      -> Python ValueError   */
    TFFT_ECUDA = 3,         /* CUDA failure      -> Python RuntimeError */
    TFFT_ENOMEM = 4,        /* allocation failed -> Python MemoryError  */
    TFFT_EUNSUPPORTED = 5,  /* size/precision not built                 */
    TFFT_EIO = 6            /* file I/O failure  -> Python OSError      */
};

enum tfft_precision { TFFT_FP32 = 0, TFFT_FP64 = 1 };

/* abft/protected.py:28-32 (Scheme) */
enum tfft_scheme {
    TFFT_SCHEME_NONE = 0,
    TFFT_SCHEME_ONE_SIDED = 1,
    TFFT_SCHEME_TWO_SIDED_THREAD = 2,
    TFFT_SCHEME_TWO_SIDED_GROUP = 3
};

/* Injection point of a fault (fault_lab/bits.py:30-45 FaultSpec.stage):
 * "input" | "stage:<k>" | "output". */
enum tfft_where { TFFT_AT_NONE = 0, TFFT_AT_INPUT = 1, TFFT_AT_STAGE = 2, TFFT_AT_OUTPUT = 3 };

/* One transient single-bit fault (fault_lab/bits.py:30-53 FaultSpec +
 * apply_fault). `element` indexes the (batch, n) view the reference hook
 * sees at `where` (for stage:<k> that is the reference's intermediate
 * layout). component: 0 = re, 1 = im. */
typedef struct tfft_fault {
    int64_t signal;
    int64_t element;
    int32_t where;
    int32_t stage;
    int32_t component;
    int32_t bit;
} tfft_fault;

/* One flagged signal (abft/pipeline.py:45-49 FlaggedSignal). */
typedef struct tfft_flag {
    int64_t group;
    int64_t signal;       /* global index in the batch */
    double discrepancy;   /* relative discrepancy (inf when non-finite) */
} tfft_flag;

/* abft/protected.py:35-60 RunReport. Arrays are caller-owned; counts may
 * exceed the capacities (entries beyond capacity are dropped). */
typedef struct tfft_report {
    int64_t groups;
    int64_t recompute_count;
    int64_t pass_count;
    double max_rel_discrepancy;
    int64_t n_flagged;
    int64_t n_corrected;
    int64_t n_unrecoverable;
    tfft_flag *flagged;        int64_t flagged_cap;
    int64_t *corrected_group;  int64_t *corrected_signal; int64_t corrected_cap;
    int64_t *unrecoverable;    int64_t unrecoverable_cap;
    int32_t fault_fired;
} tfft_report;

typedef struct tfft_plan tfft_plan;

/* fft_core/plan.py:64-101 make_plan + fit_group_size, twiddle.py:77-105
 * build_twiddles. `dims` (nstages entries, product n) is the API-visible
 * stage split; bs the checksum group size. Device twiddle tables and the
 * workspace are owned by the plan. */
int tfft_plan_create(tfft_plan **out, int64_t n, int precision, int nstages,
                     const int64_t *dims, int64_t bs, int device);
int tfft_plan_destroy(tfft_plan *plan);

/* fft_core/execute.py:56-79 fft_execute: out-of-place, natural order, inverse
 * conjugates the factors and scales by 1/n. `in` is never written. */
int tfft_execute(tfft_plan *plan, const void *in, void *out, int64_t batch,
                 int inverse, void *stream);

/* abft/protected.py:63-166 run_protected. etw: input-side row (e^T W, or
 * e^T W^-1 when inverse) and values: encoding weights, both device arrays of
 * n elements in the plan's complex dtype; values == NULL selects the Wang
 * weights w3^(k mod 3) computed in-kernel. fault may be NULL. Blocks until the
 * report is filled (one small device->host copy). */
int tfft_run_protected(tfft_plan *plan, const void *in, void *out, int64_t batch,
                       int scheme, double delta, double abs_floor,
                       const void *etw, const void *values,
                       const tfft_fault *fault, int inverse,
                       tfft_report *report, void *stream);

/* Host-buffer variant of tfft_run_protected (the numpy path of
 * abft/protected.py:63-166 and cli.py:62-64): `in`/`out` are HOST arrays of
 * batch*n complex elements (pinned memory streams at full PCIe rate; pageable
 * memory works through the driver's staging). The batch streams through a
 * ring of device chunks (whole checksum groups) with H2D, the fused
 * protected transform and D2H overlapped on three streams; the report is that
 * of one call over the whole batch. etw/values are device arrays as above.
 * Blocks until `out` and the report are complete. */
int tfft_run_protected_host(tfft_plan *plan, const void *in, void *out, int64_t batch,
                            int scheme, double delta, double abs_floor,
                            const void *etw, const void *values,
                            const tfft_fault *fault, int inverse,
                            tfft_report *report, void *stream);

/* signal_io.py:11-24 read_signals size check: number of n-sample signals of
 * the precision in a raw interleaved (re, im) little-endian file, or
 * TFFT_EINVAL ("input length mismatch ...") when the size is not a positive
 * whole number of signals. */
int tfft_signal_file_batch(const char *path, int64_t n, int precision, int64_t *batch);

/* cli.py:54-67 cmd_transform over files (signal_io.py:11-33 formats): reads
 * the raw input file, runs the protected transform and writes the raw output
 * file (created/truncated), streaming chunks of whole groups through pinned
 * staging with file reads, H2D, the fused transform, D2H and file writes of
 * different chunks overlapped (a writer thread retires chunks in order).
 * *batch receives the signal count. The output is written even when groups
 * are unrecoverable (the report says so); I/O errors return TFFT_EIO. */
int tfft_run_protected_file(tfft_plan *plan, const char *in_path, const char *out_path,
                            int scheme, double delta, double abs_floor,
                            const void *etw, const void *values, const tfft_fault *fault,
                            int inverse, int64_t *batch, tfft_report *report, void *stream);

/* Batched fault-injection campaign (fault_lab/campaign.py:95-195, the run
 * loop of run_campaign): `runs` independent run_protected calls of
 * `run_batch` signals each (in/out: device arrays of runs*run_batch*n
 * elements, run r at rows r*run_batch...), fused into ONE protected launch.
 * faults[r] is run r's single fault with a run-relative signal index
 * (where == TFFT_AT_NONE for a clean run); faults may be NULL. Outputs:
 * run_max_rel[r] (host, runs doubles) = run r's report.max_rel_discrepancy;
 * run_fired[r] (host, may be NULL) = whether run r's fault fired; the report
 * aggregates flags / corrections / unrecoverable groups with global indices
 * (groups never span runs). Blocks until done. */
int tfft_run_campaign(tfft_plan *plan, const void *in, void *out, int64_t runs,
                      int64_t run_batch, int scheme, double delta, double abs_floor,
                      const void *etw, const void *values, const tfft_fault *faults,
                      int inverse, double *run_max_rel, int32_t *run_fired,
                      tfft_report *report, void *stream);

/* HBM passes one unfaulted transform of this plan launches (1 for n <= 2^13;
 * large 2-stage plans execute as 3 short-L passes). The
 * reference's pass accounting (RunReport.pass_count) is unaffected. */
int tfft_plan_exec_passes(const tfft_plan *plan);

/* Checksum granularity of the protected calls on this plan, for the paper's
 * scheme comparison (TurboFFT one-sided vs thread-level vs threadblock-level;
 * not a reference interface): 0 = threadblock-level two-sided checksums per
 * signal (default, the reference's decisions), 1 = thread-level: every radix
 * tile verified by the thread computing it (Wang encoding per tile; flags
 * are then per-tile discrepancies, not the reference's). Level 1 is built for
 * n <= 2^13 with the Wang encoding (values == NULL). */
int tfft_set_check_level(tfft_plan *plan, int level);

/* Online correction of the single-kernel sizes (n <= 2^13) runs on the
 * device, queued right behind the fused transform (enable = 1, default): a
 * flagged call costs no extra host round trip. enable = 0 makes the host
 * decide first and launch the same correction kernel with its job list
 * (identical results; used to test one against the other). */
int tfft_set_device_correction(tfft_plan *plan, int enable);

/* The two halves of tfft_run_protected, for callers that queue several
 * protected transforms before reading their reports (one in-flight protected
 * call per plan): _launch enqueues the fused transform and the tiny
 * detection-summary copy without blocking; _finish waits for that summary,
 * takes the per-group decisions and runs any correction / recompute. The
 * arguments of _finish must repeat those given to _launch. */
int tfft_protect_launch(tfft_plan *plan, const void *in, void *out, int64_t batch,
                        int scheme, double delta, double abs_floor,
                        const void *etw, const void *values,
                        const tfft_fault *fault, int inverse,
                        tfft_report *report, void *stream);
int tfft_protect_finish(tfft_plan *plan, const void *in, void *out, int64_t batch,
                        int scheme, double delta, double abs_floor,
                        const void *etw, const void *values, int inverse,
                        tfft_report *report, void *stream);

/* kernels/_stockham.pyx:46-65 tile_fft (the reference's backend plugin
 * point, kernels/__init__.py:28-39): unscaled DFT of every row of a (t, l)
 * matrix, natural order, inverse conjugates. host != 0: in/out are host
 * arrays (copied through pinned staging). dtype_bytes: 8 complex64,
 * 16 complex128. */
int tfft_tile_fft(const void *in, void *out, int64_t t, int64_t l, int dtype_bytes,
                  int inverse, int host, void *stream);

/* abft/pipeline.py:72-85 encode_group over one group xg (bs, n): s0 = sum_b
 * x_b, s1 = sum_b (b+1) x_b, c_in[b] = x_b . row, x_l1[b] = sum |x_b|.
 * Outputs are device arrays (s0, s1: n complex; c_in: bs complex; x_l1: bs
 * real), any of them may be NULL. */
int tfft_encode_group(tfft_plan *plan, const void *xg, int64_t bs, const void *row,
                      void *s0, void *s1, void *c_in, void *x_l1, void *stream);

/* abft/pipeline.py:104-135 detect: rel[b] for each of the bs outputs (device
 * real array), NaN/Inf -> +inf. floor_coef is FLOOR_COEF[precision]
 * (pipeline.py:16,100-101: the caller's `precision` argument, not the data
 * dtype). */
int tfft_detect(tfft_plan *plan, const void *yg, int64_t bs, const void *values,
                const void *c_in, const void *x_l1, double abs_floor, double floor_coef,
                void *rel, void *raw, void *stream);

/* abft/pipeline.py:164-192 correct_group core: out[f] = FFT(s0) - sum_{b!=f} y_b
 * computed into `fixed` (n elements). */
int tfft_correct_signal(tfft_plan *plan, const void *s0, const void *yg, int64_t bs,
                        int64_t f, void *fixed, int inverse, void *stream);

/* abft/element.py:33-92 two_sided_element on one r x B tile (1 <= r <= 32),
 * complex128 device arrays, row-major (r, B). _encode: y[:, j] = DFT_r of
 * column j, row_in[j] = etw_row . x[:, j] (row side), xe = x @ vals_col
 * (column side). _verify (after any injection into y): rel[j] per column,
 * result (host int[3]) = {0 clean | 1 corrected | 2 several columns flagged |
 * 3 row/column disagreements inconsistent, row, col}; a corrected y is
 * fixed in place. Blocks until result is filled. */
int tfft_element_encode(int r, int64_t B, const void *x, void *y, const void *etw_row,
                        const void *vals_col, void *row_in, void *xe, void *stream);
int tfft_element_verify(int r, int64_t B, void *y, const void *row_in, const void *xe,
                        const void *vals_row, const void *vals_col, double delta, double abs_floor,
                        void *rel, int32_t *result, void *stream);

/* fault_lab/bits.py:11-27,48-53 flip_bit/apply_fault on device memory:
 * XOR bit `bit` of real word `word` (2*element + component) of buf. */
int tfft_flip_bit(void *buf, int64_t word, int bit, int dtype_bytes, void *stream);

/* One reference stage on its own (fft_core/execute.py:28-53 stage_pass plus
 * the _run_stages reshuffle), used when a caller hooks every stage
 * (execute.py:56-79 `on_stage`). Stage k reads `in` and writes `out` in the
 * library's pass layout; no 1/n scaling. Single-stage plans: k == 0 is the
 * whole unscaled transform. */
int tfft_execute_stage(tfft_plan *plan, int k, const void *in, void *out, int64_t batch,
                       int inverse, void *stream);

/* buf[i] *= s for count complex elements (the inverse 1/n, execute.py:77-78). */
int tfft_scale(void *buf, int64_t count, int dtype_bytes, double s, void *stream);

/* Tuning hooks of the plan generator (paper_2405_02520_b200/codegen.py):
 * number of compiled launch variants of the single-kernel size 2^logn, and a
 * process-wide override of which one launches (variant < 0 restores the
 * tuned default). Used by tools/tune.py; not needed by callers. */
int tfft_tune_variants(int precision, int logn);
int tfft_tune_select(int precision, int logn, int variant);
/* Same for the multi-pass stage kernels of dim 2^logl; kind 0 = first stage,
 * 1 = middle (3-stage), 2 = last. */
int tfft_tune_pass_variants(int precision, int logl);
int tfft_tune_pass_select(int precision, int logl, int kind, int variant);

/* The complete flagged / corrected / unrecoverable lists of the plan's last
 * protected call (abft/protected.py:35-60 RunReport), for callers whose
 * report buffers were smaller than the counts that call returned: fills the
 * lists up to the caps of `report` and sets the three counts. */
int tfft_report_fetch(const tfft_plan *plan, tfft_report *report);

/* fft_core/reference.py:12-39 dft_reference: direct O(n^2) DFT of `batch`
 * complex128 device rows of ANY length 1 <= n <= 2^14 (ORACLE_MAX_N),
 * y_j = sum_k x_k w^(jk), inverse conjugates and scales by 1/n. A kernel of
 * its own, sharing nothing with the FFT path (the independent check). */
int tfft_dft(const void *in, void *out, int64_t batch, int64_t n, int inverse, void *stream);

/* Kernels this library has launched in the process so far (every launch
 * site increments it): bench.py's `gpu_launches` is the difference across
 * the timed region. */
int tfft_launch_count(int64_t *count);

const char *tfft_last_error(void);
int tfft_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TFFT_H */
