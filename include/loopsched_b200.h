/*
 * loopsched_b200.h -- C ABI of the B200 measurement & scoring hot path.
 *
 * The reference (`loopsched`, pure Python) has no native boundary; these entry
 * points are what its Python seams bind through ctypes:
 *
 *   reference seam (file:line)                         replaced by
 *   -------------------------------------------------  --------------------------------
 *   search._measure_batch(cands, spec, jobs)           ls_runner_measure
 *     src/search.py:249-256, called at :345
 *   search.simulate_latency(e0, spec) (baseline)       ls_runner_baseline  (hardware mode)
 *     src/search.py:326; src/machine.py:228-254        ls_sim_latency_batch (parity mode)
 *   costmodel.featurize(p, spec)                       ls_featurize_batch
 *     src/costmodel.py:21-79; looked up at src/search.py:141
 *   CostModel.predict_features(f) / _Validator._predict ls_score_batch
 *     src/costmodel.py:98-102; src/search.py:109-111
 *   trace.validate_trace(e0, t) / replay(.., "follow") ls_replay_batch
 *     src/trace.py:163-265 (+ ScheduleState, src/schedule.py:123-974);
 *     called from _Validator.candidate, src/search.py:113-121
 *   ir.structural_hash(p)                              ls_program_hash
 *     src/ir.py:625-629
 *
 * Programs cross the boundary in the reference's own interchange format: the
 * text of `ir.serialize(program)` (`src/ir.py:708-715`).  The caller owns every
 * array passed in or out; the library owns device memory, streams and caches.
 * No call throws or exits: each returns an ls_status and, on failure, leaves a
 * thread-local message in ls_last_error().  There is no CPU fallback: every
 * compute entry point fails with LS_ERR_CUDA when no B200 is present.
 */
#ifndef LOOPSCHED_B200_H_
#define LOOPSCHED_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LS_OK = 0,
  LS_ERR_ARG = 1,      /* bad argument / unsupported request                  */
  LS_ERR_PARSE = 2,    /* a program text failed to parse                      */
  LS_ERR_CUDA = 3,     /* CUDA error or no usable device                      */
  LS_ERR_STATE = 4     /* call order violated (e.g. measure before workload)  */
} ls_status;

/* MachineSpec (src/machine.py:22-55); unroll_discount as the exact fraction
 * Fraction(str(unroll_discount)) = unroll_num / unroll_den. */
typedef struct {
  int64_t cores, vector_lanes, cache_capacity, hit_cost, miss_cost, flop_cost, tensor_unit_cost;
  int64_t unroll_num, unroll_den;
} ls_machine_spec;

/* CostModel parameters (src/costmodel.py:82-102). */
typedef struct {
  double w[9], mean[9], scale[9], intercept;
  int64_t n_records;
  int32_t is_fit;
} ls_linear_model;

/* per-program analysis status */
enum { LS_PROG_OK = 0, LS_PROG_PARSE = 1, LS_PROG_ANALYSIS = 2, LS_PROG_OVERFLOW = 3 };

/* ---- batched cost model / exact simulator (K7, K8) -------------------- */

/* Exact simulate_latency of each program as num/den (K8). */
ls_status ls_sim_latency_batch(int device, const char* const* programs, const size_t* lens, int n,
                               const ls_machine_spec* spec, int64_t* num, int64_t* den, int32_t* status);
/* featurize of each program, row-major n x 9 (K7a). */
ls_status ls_featurize_batch(int device, const char* const* programs, const size_t* lens, int n,
                             const ls_machine_spec* spec, double* feats, int32_t* status);
/* predict_features over rows of an n x 9 feature matrix (K7b). */
ls_status ls_score_batch(int device, const double* feats, int n, const ls_linear_model* model, double* out);
/* K7 + K8 fused in one launch; any output pointer may be NULL. */
ls_status ls_analyze_batch(int device, const char* const* programs, const size_t* lens, int n,
                           const ls_machine_spec* spec, const ls_linear_model* model, int64_t* num,
                           int64_t* den, double* feats, double* pred, int32_t* status);

/* Device-resident batches: parse + encode + upload once, analyze many times
 * (the kernel-only timing path; `value` in bench.py). */
typedef struct ls_batch ls_batch;
ls_status ls_batch_create(int device, const char* const* programs, const size_t* lens, int n, ls_batch** out);
ls_status ls_batch_analyze(ls_batch* b, const ls_machine_spec* spec, const ls_linear_model* model, int flags);
ls_status ls_batch_results(ls_batch* b, int64_t* num, int64_t* den, double* feats, double* pred, int32_t* status);
ls_status ls_batch_elapsed_ms(ls_batch* b, float* ms); /* device time of the last analyze */
void ls_batch_destroy(ls_batch* b);

/* ---- hardware Runner ---------------------------------------------------- */

typedef enum { LS_DTYPE_F32 = 0, LS_DTYPE_BF16 = 1 } ls_dtype;

typedef struct {
  int32_t dtype;           /* ls_dtype of the device copies of the inputs; with    */
                           /* LS_DTYPE_F32 a tcgen05 tile runs as 3xTF32           */
  int32_t min_repeats;     /* timed launches per candidate (lower bound)          */
  int32_t max_repeats;     /* upper bound                                          */
  double target_ms;        /* repeats sized so one candidate runs ~target_ms       */
  double timeout_ms;       /* device-side deadline cap for the checked launch      */
  double rtol, atol;       /* parity tolerance against the e0 reference output     */
  int32_t flush_l2;        /* nonzero: cold-L2 timing -- every timed repeat runs   */
                           /* after a 256 MB scrub and is timed alone (no graphs) */
  int32_t carry_best;      /* nonzero: the device best-so-far behind timeout_factor */
                           /* deadlines persists across ls_runner_measure calls of */
                           /* one workload (small tuning batches); reset by        */
                           /* ls_runner_set_workload                                */
  double timeout_factor;   /* >0: deadline = clamp(factor x best-so-far, floor,   */
  double timeout_floor_ms; /*      timeout_ms), tracked on the device              */
  double single_shot_factor; /* >0: a candidate whose checked launch is slower than */
                           /* factor x the batch's fastest checked launch skips the */
                           /* timed repeats; its latency is the checked launch      */
                           /* (repeats = 0)                                         */
} ls_runner_opts;

/* per-candidate status */
enum {
  LS_RUN_OK = 0,
  LS_RUN_ILLEGAL = 1,      /* instantiator: config beyond hardware limits        */
  LS_RUN_UNSUPPORTED = 2,  /* program structure outside the mapping convention   */
  LS_RUN_PARSE = 3,
  LS_RUN_LAUNCH = 4,
  LS_RUN_PARITY = 5,       /* output differs from the reference output           */
  LS_RUN_TIMEOUT = 6       /* checked launch passed its deadline; latency_ns is  */
                           /* the abort time, a lower bound                      */
};

/* kernel families */
enum { LS_FAM_NONE = 0, LS_FAM_NAIVE = 1, LS_FAM_SIMT = 2, LS_FAM_TCGEN05 = 3, LS_FAM_LOOPNEST = 4,
       LS_FAM_GENERIC = 5, LS_FAM_NESTGEN = 6, LS_FAM_SIMT_AFFINE = 7, LS_FAM_TCGEN05_CONV = 8 };

typedef struct {
  int32_t status;
  int32_t family;
  int32_t repeats;
  int32_t cfg[13];         /* family-specific instantiation      */
  double latency_ns;       /* mean device time of one launch (incl. memsets)    */
  double max_abs_err;
  int64_t mismatches;
  double checked_ns;       /* the checked launch alone (one isolated launch     */
                           /* between events, L2-warm, no back-to-back overlap) */
} ls_result;

typedef struct ls_runner ls_runner;

ls_status ls_runner_create(int device, const ls_runner_opts* opts, ls_runner** out);
/* e0 program text plus its input tensors as float32 host arrays, in the
 * order the program declares its input buffers (random_inputs order).
 * Returns once the host arrays have been consumed (they may be freed); the
 * fp64 reference run of e0 stays queued on the runner's stream, and a
 * failure there is reported by the next call that waits on it. */
ls_status ls_runner_set_workload(ls_runner* r, const char* e0, size_t len, const float* const* host_inputs,
                                 int n_inputs);
ls_status ls_runner_measure(ls_runner* r, const char* const* programs, const size_t* lens, int n,
                            ls_result* out);
/* The unscheduled e0 through the same instantiator (the baseline latency). */
ls_status ls_runner_baseline(ls_runner* r, ls_result* out);
/* Instantiation only (no launch): family + config + status per program. */
ls_status ls_runner_plan(ls_runner* r, const char* const* programs, const size_t* lens, int n, ls_result* out);
/* Host-only instantiation (no device needed): the plan (family, config,
 * status) of each program against workload e0 for the given runner dtype. */
ls_status ls_plan_programs(const char* e0, size_t e0_len, const char* const* programs, const size_t* lens, int n,
                           int32_t dtype, ls_result* out);
/* Copy the output buffer of the last launched candidate (float32). */
ls_status ls_runner_last_output(ls_runner* r, float* host, size_t count);
/* Copy the reference output computed by the e0 reference kernel (float64). */
ls_status ls_runner_reference_output(ls_runner* r, double* host, size_t count);
/* Device time spent in the last ls_runner_measure call (ms, all candidates). */
ls_status ls_runner_elapsed_ms(ls_runner* r, float* ms);
/* Kernel launches (candidates + parity/deadline/spin helpers) of the last measure call. */
ls_status ls_runner_launch_count(ls_runner* r, int64_t* count);
/* Host-side timing of the last measure call: [0] phase-A enqueue ms, [1]
 * phase-B enqueue ms, [2] device spin us.  Passing n > 7 with out[7] > 0 sets
 * the per-call host cost (us) used to size the spin. */
ls_status ls_runner_debug_stats(ls_runner* r, double* out, int n);
/* Change the checked-launch deadline cap (timeout_ms of the options) of later
 * measure calls, e.g. to a multiple of the measured e0 baseline. */
ls_status ls_runner_set_timeout(ls_runner* r, double timeout_ms);
/* Diagnostics: launch one tcgen05 candidate `launches` times back to back
 * (one CUDA graph, PDL-chained like the timed repeats) with
 * per-CTA %globaltimer stamps (8 u64 per CTA: start, setup done, first stage
 * landed, accumulator done, partial tile staged, zeroing flag acquired,
 * stored, smid). */
ls_status ls_runner_trace_tc(ls_runner* r, const char* program, size_t len, int launches, uint64_t* out,
                             int max_ctas, int* n_ctas);
void ls_runner_destroy(ls_runner* r);

/* ---- native trace replay / validation (host side, src/trace.py:163-265) ---
 * A replayer holds one workload e0 (`ir.serialize` text).  ls_replay_batch
 * replays each trace -- the text of the reference's `serialize_trace(t)`
 * (src/trace.py:80-86), which _Validator already uses as its cache key -- with
 * the recorded decisions, exactly as validate_trace does, and returns per trace:
 *   ACCEPTED: program = ir.serialize(final program), hash = ir.structural_hash,
 *             trace = serialize_trace(normalized trace)      (src/trace.py:196-198)
 *   REJECTED: (reason, index) of the reference's Rejected verdict
 *   DEFER:    the reference would raise something other than ReplayError on
 *             this input (a malformed trace); the caller replays it with the
 *             reference to get the reference's behaviour.
 * Strings are malloc'd; release them with ls_replay_free. */
enum { LS_REPLAY_ACCEPTED = 0, LS_REPLAY_REJECTED = 1, LS_REPLAY_DEFER = 2 };
typedef struct {
  int32_t status;
  int32_t index;    /* REJECTED: instruction index (-1: workload hash mismatch) */
  uint64_t hash;    /* ACCEPTED: structural hash of the final program */
  char* program;
  char* trace;
  char* reason;
} ls_replay_result;
typedef struct ls_replayer ls_replayer;
ls_status ls_replayer_create(const char* e0, size_t len, ls_replayer** out);
ls_status ls_replayer_hash(ls_replayer* r, uint64_t* out); /* ir.structural_hash(e0) */
ls_status ls_replay_batch(ls_replayer* r, const char* const* traces, const size_t* lens, int n,
                          ls_replay_result* out);
void ls_replay_free(ls_replay_result* res, int n);
/* replay(e0, t, mode="resample", seed) (src/trace.py:163-188): the samplers
 * draw fresh decisions from CPython's random.Random(seed), bit-exact (the
 * fresh candidates of evolve, src/search.py:149-159); same result form. */
ls_status ls_replay_resample(ls_replayer* r, const char* trace, size_t len, uint64_t seed, ls_replay_result* out);
void ls_replayer_destroy(ls_replayer* r);
/* Look-ahead: every single-decision neighbour of each
 * member trace -- exactly the traces `mutate` (src/trace.py:287-309) can
 * propose -- is replayed on the host pool (a member is replayed once, each
 * neighbour from a snapshot before its changed decision).  The result holds
 * the programs of the structural hashes this replayer has not handed out
 * before (to be featurized in one batch); neighbours expanded earlier are
 * skipped.  Strings live until ls_neighbours_destroy.  stats: replayed,
 * accepted, rejected, deferred. */
typedef struct ls_neighbours ls_neighbours;
ls_status ls_replay_neighbours(ls_replayer* r, const char* const* traces, const size_t* lens, int n,
                               ls_neighbours** out);
ls_status ls_neighbours_count(ls_neighbours* nb, int* count);
ls_status ls_neighbours_get(ls_neighbours* nb, int i, uint64_t* hash, const char** program);
ls_status ls_neighbours_stats(ls_neighbours* nb, int64_t* out4);
void ls_neighbours_destroy(ls_neighbours* nb);
/* ir.structural_hash of a serialized program */
ls_status ls_program_hash(const char* program, size_t len, uint64_t* out);

const char* ls_last_error(void);
const char* ls_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LOOPSCHED_B200_H_ */
