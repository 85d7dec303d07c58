/*
 * mltune_b200.h — C ABI of libmltune_b200.so, the sm_100a implementation of
 * the mltune auto-tuner hot path (Falch & Elster, arXiv 1506.00842).
 *
 * The reference package `mltune` is pure Python; its "plugin seams" for this
 * path are Python functions and duck types. Each entry point below replaces
 * one of them (reference paths relative to /root/reference/pkg/src/mltune):
 *
 *   mlt_decode            ParamSpace.decode_indices        paramspace.py:184-193
 *   mlt_valid_mask        ParamSpace.static_valid_mask     paramspace.py:201-213 (+ ValidityRule.satisfied_mask :92-107)
 *   mlt_encode            Encoder.encode_indices           model.py:88-97
 *   mlt_predict_indices   Ensemble.predict_indices         model.py:300-301 (forward_batch :146-154, predict_log_batch :162-164)
 *   mlt_predict_features  Ensemble.predict_features        model.py:290-294
 *   mlt_top_m             tuner.top_m_predicted            tuner.py:95-131 (one contiguous slice or an index list)
 *   mlt_merge_top_m       the final lexsort of tuner.py:128-131, applied to per-GPU lists
 *   mlt_train_member(s)   model._fit / train_ensemble      model.py:194-249, :308-341
 *   mlt_surrogate_times   SurrogateRunner.true_times / measured_times  measurement.py:212-238
 *   mlt_surrogate_best    exhaustive_search over a surrogate tuner.py:191-224
 *   mlt_{conv,stereo,ray}bench_*  the paper's benchmark kernels behind runner.measure (measurement.py:250-258)
 *   mlt_host_permutations the per-epoch rng.permutation draws of _fit     model.py:218 (host helper, no GPU)
 *   mlt_format_predictions the `mltune predict` CSV rows                   cli.py:346-351 (host helper, no GPU)
 *
 * Conventions
 *   - Plain C types only; every pointer argument is HOST memory owned by the
 *     caller unless the name says `dev_`.
 *   - Return value: MLT_OK (0) or a negative status; mlt_last_error() gives a
 *     thread-local message. Status -> Python exception mapping:
 *       MLT_EINVAL -> ValueError, MLT_EMISMATCH -> ConfigMismatchError,
 *       MLT_EDATA -> InsufficientDataError, MLT_EDIVERGED -> DivergenceError,
 *       MLT_ECUDA / MLT_EINTERNAL -> RuntimeError.
 *   - Every call is synchronous on the context's stream (library-owned, or the
 *     caller's via mlt_ctx_set_stream). Calls on one context are serialised
 *     by a per-context mutex (safe to share across threads; concurrent work on
 *     one device runs in parallel only through several contexts).
 *   - There is no CPU fallback: without a usable sm_100 device every compute
 *     entry point fails with MLT_ECUDA (mlt_host_permutations is host-only:
 *     it reproduces the reference's RNG stream, it computes nothing of the path).
 */
#ifndef MLTUNE_B200_H
#define MLTUNE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define MLT_API __attribute__((visibility("default")))
#else
#define MLT_API
#endif

#define MLT_ABI_VERSION 1

#define MLT_OK 0
#define MLT_EINVAL -1
#define MLT_EMISMATCH -2
#define MLT_EDATA -3
#define MLT_EDIVERGED -4
#define MLT_ECUDA -5
#define MLT_EINTERNAL -6

#define MLT_MAX_PARAMS 32

/* Validity-rule kinds (paramspace.py:28-31). */
#define MLT_RULE_MAX_PRODUCT 0
#define MLT_RULE_MAX_WEIGHTED_SUM 1
#define MLT_RULE_FORBIDDEN 2

/* A finite parameter space: mixed radix, last parameter fastest
 * (paramspace.py:110-193), plus static validity rules evaluated on VALUES
 * with numpy int64 (wrap-around) semantics (paramspace.py:92-107). */
typedef struct mlt_space {
  int32_t n_params;            /* P, 1..MLT_MAX_PARAMS */
  const int32_t* radix;        /* [P] value count per parameter */
  const int64_t* values;       /* [sum(radix)] value lists, parameter-major */
  int32_t n_rules;             /* R >= 0 */
  const int32_t* rule_kind;    /* [R] MLT_RULE_* */
  const int32_t* rule_nops;    /* [R] operand count per rule */
  const int32_t* rule_pos;     /* [sum(nops)] operand parameter positions */
  const int64_t* rule_coeff;   /* [sum(nops)] coefficients (banned values for FORBIDDEN) */
  const int64_t* rule_bound;   /* [R] bound (unused for FORBIDDEN) */
} mlt_space;

/* A bagged ensemble of k one-hidden-layer sigmoid networks (model.py:114-170,
 * :272-301) plus its encoder (value counts; feature = rank / max(count-1, 1)). */
typedef struct mlt_ensemble {
  int32_t k;                   /* members */
  int32_t d;                   /* inputs (= encoder parameters) */
  int32_t h;                   /* hidden units per member (30 in mltune) */
  const int32_t* counts;       /* [d] encoder value counts */
  const double* w1;            /* [k][h][d] weights_hidden */
  const double* b1;            /* [k][h]    biases_hidden */
  const double* w2;            /* [k][h]    weights_out */
  const double* b2;            /* [k]       bias_out */
  const double* mean;          /* [k]       target_mean */
  const double* std;           /* [k]       target_std */
} mlt_ensemble;

/* Diagnostics of one mlt_top_m call. */
typedef struct mlt_sweep_stats {
  int64_t configs;             /* configurations swept */
  int64_t candidates;          /* guard-band candidates rescored in fp64 */
  int32_t path;                /* 0 = fp32 sweep + fp64 guard band, 1 = fp64 materialise + sort,
                                  2 = constant ensemble (every configuration ties): first valid indices */
  int32_t group;               /* hidden units per reciprocal in the fp32 sweep (1..4) */
  double delta;                /* a-priori bound on |fp32 - fp64| mean log time */
  float sweep_ms;              /* device time of the sweep kernel (profiling on) */
  float total_ms;              /* device time of the whole call   (profiling on) */
  int32_t launches;            /* kernels launched by this call */
  int32_t split;               /* parameters in the inner (per-thread) factor */
  int64_t raw_candidates;      /* configurations the streaming band kept before the exact filter */
  double evaluated_frac;       /* (configuration, unit) pairs evaluated / all: 1 without pruning */
} mlt_sweep_stats;

typedef struct mlt_ctx mlt_ctx;

MLT_API int mlt_abi_version(void);
MLT_API const char* mlt_last_error(void);

MLT_API int mlt_ctx_create(int device, mlt_ctx** out);
MLT_API int mlt_ctx_destroy(mlt_ctx* ctx);
/* Use `stream` (a cudaStream_t; cudaStreamLegacy = (void*)1 for the legacy
 * default stream) for all work; NULL restores the library's own stream. Work
 * already queued on the previous stream is ordered before the new stream's. */
MLT_API int mlt_ctx_set_stream(mlt_ctx* ctx, void* stream);
/* When on, mlt_top_m records CUDA events around its kernels (mlt_sweep_stats). */
MLT_API int mlt_ctx_set_profiling(mlt_ctx* ctx, int on);
/* Kernels launched by this context so far. */
MLT_API int64_t mlt_ctx_launches(mlt_ctx* ctx);
/* Tuning / test knobs (value -1 restores the default):
 *   MLT_OPT_PATH      0 = force the fp32 sweep + fp64 guard band, 1 = force fp64 materialise + sort
 *   MLT_OPT_GROUP     hidden units per reciprocal in the fp32 sweep (1, 2 or 3)
 *   MLT_OPT_CAND_CAP  capacity of the guard-band candidate buffer (entries)         */
#define MLT_OPT_PATH 1
#define MLT_OPT_GROUP 2
#define MLT_OPT_CAND_CAP 3
/*   MLT_OPT_PRUNE     1 = exact bound-based pruning in the fp32 sweep: a work item whose
 *                     partial sums plus a rigorous lower bound of the remaining hidden
 *                     units exceed the threshold stops early (same top-m; fewer
 *                     configurations fully evaluated). 0 (default) = evaluate all.   */
#define MLT_OPT_PRUNE 4
/*   MLT_OPT_CHUNK     configurations per sweep chunk (default 2^27): longer slices are swept
 *                     chunk by chunk and the per-chunk top-m merged (bounded memory).   */
#define MLT_OPT_CHUNK 5
/*   MLT_OPT_TABLE_CACHE 1 (default) = a plan keeps its factored sweep tables between calls
 *                     with the same slice shape; 0 = rebuild them on every call (what a
 *                     fresh ensemble costs; bench.py times the headline step this way).  */
#define MLT_OPT_TABLE_CACHE 6
/*   MLT_OPT_HALF_ITEMS  1 = sweep with two CTAs per SM, each owning half a work item
 *                     (no tail launch); 0 (default) = one CTA per SM on whole items.
 *   MLT_OPT_TAIL_SPLIT  1 (default) = the items of the last, partial wave of the sweep
 *                     run in a second launch split into quarter items; 0 = off.        */
#define MLT_OPT_HALF_ITEMS 7
#define MLT_OPT_TAIL_SPLIT 8
MLT_API int mlt_ctx_set_option(mlt_ctx* ctx, int key, int64_t value);

/* A1: values[n][P] = decode(idx[n]).                 paramspace.py:184-193 */
MLT_API int mlt_decode(mlt_ctx* ctx, const mlt_space* space, const int64_t* idx, int64_t n,
               int64_t* values_out);
/* A2: mask[n] = every rule satisfied.               paramspace.py:201-213 */
MLT_API int mlt_valid_mask(mlt_ctx* ctx, const mlt_space* space, const int64_t* idx, int64_t n,
                   uint8_t* mask_out);
/* A3: feat[n][d] = digit / max(count-1, 1).         model.py:88-97 */
MLT_API int mlt_encode(mlt_ctx* ctx, const int32_t* counts, int32_t d, const int64_t* idx, int64_t n,
               double* feat_out);
/* A4-A6: fp64 predicted seconds for configuration indices. model.py:300-301 */
MLT_API int mlt_predict_indices(mlt_ctx* ctx, const mlt_ensemble* ens, const int64_t* idx, int64_t n,
                        double* pred_out);
/* A6: fp64 predicted seconds for a feature matrix X[n][d]. model.py:290-294 */
MLT_API int mlt_predict_features(mlt_ctx* ctx, const mlt_ensemble* ens, const double* x, int64_t n,
                         double* pred_out);

/* A4: raw member outputs out[k][n] = w2 . sigmoid(W1 x + b1) + b2 for a
 * feature matrix X[n][d] (Network.forward_batch, model.py:146-154). */
MLT_API int mlt_member_outputs(mlt_ctx* ctx, const mlt_ensemble* ens, const double* x, int64_t n,
                       double* out);

/* A7: the m statically-valid configurations with the lowest predicted time
 * (ascending; ties by ascending index) among
 *   - the contiguous slice [begin, end) of the space, when idx_list == NULL, or
 *   - the n_list indices of idx_list (sweep_cap subset, tuner.py:104-105).
 * Writes *out_n <= m results. tuner.py:95-131. */
MLT_API int mlt_top_m(mlt_ctx* ctx, const mlt_space* space, const mlt_ensemble* ens, int64_t m,
              int64_t begin, int64_t end, const int64_t* idx_list, int64_t n_list,
              int64_t* out_idx, double* out_pred, int64_t* out_n, mlt_sweep_stats* stats);

/* Single-process multi-GPU mlt_top_m (SURVEY §8(b) mlt_sweep_topn_multi,
 * replacing tuner.py:95-131 on a node): the slice [begin, end) -- or the
 * n_list indices of idx_list -- is cut into n_ctx contiguous shards, context
 * i sweeps shard i on its own device (one host thread each, concurrently) and
 * the per-shard lists are merged by (prediction, index). Contexts must be
 * distinct (a context is not re-entrant); several may share a device.
 * stats: counts summed, times the max over contexts. */
MLT_API int mlt_top_m_multi(mlt_ctx* const* ctxs, int32_t n_ctx, const mlt_space* space, const mlt_ensemble* ens,
                    int64_t m, int64_t begin, int64_t end, const int64_t* idx_list, int64_t n_list,
                    int64_t* out_idx, double* out_pred, int64_t* out_n, mlt_sweep_stats* stats);

/* Resident variant for repeated sweeps of one (space, ensemble): uploads the
 * descriptors once; mlt_plan_top_m then does the whole step on the device. */
typedef struct mlt_plan mlt_plan;
MLT_API int mlt_plan_create(mlt_ctx* ctx, const mlt_space* space, const mlt_ensemble* ens, mlt_plan** out);
MLT_API int mlt_plan_top_m(mlt_plan* plan, int64_t m, int64_t begin, int64_t end,
                   int64_t* out_idx, double* out_pred, int64_t* out_n, mlt_sweep_stats* stats);
MLT_API int mlt_plan_destroy(mlt_plan* plan);

/* Device-resident step for the multi-GPU path: the whole
 * top-m of [begin, end) is enqueued on the context's stream and written to
 * the DEVICE record rec[2m+1] (int64): rec[0..m) indices (-1 = padding),
 * rec[m..2m) the fp64 bit patterns of the predictions (+inf = padding),
 * rec[2m] a status word (0 = exact result; 1 = the guard band overflowed,
 * 2 = too many survivors for the one-CTA sort: redo this shard with
 * mlt_plan_top_m). No host wait on the fast path, so an NCCL all-gather of
 * the records can be enqueued right behind it; where only the exact fp64
 * path applies (m > 1024, tiny slices) the call runs it synchronously and
 * uploads the record. tuner.py:95-131 over one shard. */
MLT_API int mlt_plan_top_m_record(mlt_plan* plan, int64_t m, int64_t begin, int64_t end, int64_t* dev_rec);

/* Merge n_rec gathered records (n_rec x (2m+1) int64, DEVICE memory, layout
 * of mlt_plan_top_m_record) into the global top-m by (prediction, index):
 * the final lexsort of tuner.py:128-131. *out_status = OR of the records'
 * status words (nonzero: some shard must be redone). One host wait. */
MLT_API int mlt_merge_records(mlt_ctx* ctx, const int64_t* dev_recs, int64_t n_rec, int64_t m,
                      int64_t* out_idx, double* out_pred, int64_t* out_n, int64_t* out_status);

/* Merge per-shard top-m lists (e.g. after an all-gather across GPUs) into the
 * global top-m by (prediction, index). Entries with idx < 0 are padding.
 * dev_idx / dev_pred are DEVICE pointers on the context's device. */
MLT_API int mlt_merge_top_m(mlt_ctx* ctx, const int64_t* dev_idx, const double* dev_pred, int64_t n,
                    int64_t m, int64_t* out_idx, double* out_pred, int64_t* out_n);

/* A9-A10: train k members with mini-batch momentum SGD in fp64 (model.py:194-249).
 * All random draws are made by the caller with the reference RNG stream:
 *   x[n_rows][d]            training features (all valid rows)
 *   t[sum(n_m)]             standardized targets, member-major, member m uses rows rows[off_m + r]
 *   rows[sum(n_m)]          row index into x for member m's r-th example
 *   n_m[k]                  examples per member
 *   init_w1[k][h][d], init_w2[k][h]   initial weights (b1 = 0, b2 = 0)
 *   perms[sum(epochs*n_m)]  per-epoch permutations, member-major then epoch-major
 * Outputs (per member): w1[k][h][d], b1[k][h], w2[k][h], b2[k], loss_first[k],
 * loss_final[k], diverged_epoch[k] (0 = finite throughout). */
typedef struct mlt_train_desc {
  int32_t k, d, h;
  int32_t epochs, batch_size;
  double learning_rate, momentum;
  int64_t n_rows;
  const double* x;
  const double* t;
  const int32_t* rows;
  const int32_t* n_m;
  const double* init_w1;
  const double* init_w2;
  const int32_t* perms;
} mlt_train_desc;

MLT_API int mlt_train_members(mlt_ctx* ctx, const mlt_train_desc* desc, double* w1, double* b1,
                      double* w2, double* b2, double* loss_first, double* loss_final,
                      int32_t* diverged_epoch);

/* Host helper for A10's draws (model.py:218): `count` successive
 * `rng.permutation(n[g])` results of each of n_gen numpy Generators, written
 * generator-major to out (count * n[g] int32 each). bitgens[g] is numpy's
 * bitgen_t* (`Generator.bit_generator.ctypes.bit_generator`): the bits come
 * from numpy's own PCG64 and advance its state exactly as numpy would. Runs
 * on `threads` host threads (0 = all); no GPU involved. */
MLT_API int mlt_host_permutations(void* const* bitgens, int32_t n_gen, const int32_t* n, int32_t count,
                                  int32_t* out, int32_t threads);

/* Host helper for the `mltune predict` CSV (cli.py:346-351): writes n lines
 * "<idx>,<pred %.17g>\n" into out (capacity cap bytes), *used = bytes written;
 * MLT_EINVAL if they do not fit. Runs on `threads` host threads (0 = all). */
MLT_API int mlt_format_predictions(const int64_t* idx, const double* pred, int64_t n, char* out, int64_t cap,
                                   int64_t* used, int32_t threads);

/* ---------------------------------------------------------------------------
 * A12: the analytic surrogate device (SurrogateSpec / SurrogateRunner,
 * measurement.py:146-238): base time x matching term factors (in spec order),
 * launch rules -> invalid, frozen log-normal noise from splitmix64 + ndtri.
 * ------------------------------------------------------------------------- */
typedef struct mlt_surrogate {
  double base_time;
  int32_t n_terms;             /* T */
  const int32_t* term_nparams; /* [T] 1 or 2 */
  const int32_t* term_pos;     /* [T][2] parameter positions (second ignored for 1-param terms) */
  const int64_t* term_match;   /* [T][2] matched VALUES */
  const double* term_factor;   /* [T] */
  double log_sigma;            /* sqrt(log1p(noise_cv^2)) as the caller computes it; 0 = no noise */
  uint64_t seed;
  int32_t n_rules;             /* launch-failure rules, same encoding as mlt_space */
  const int32_t* rule_kind;
  const int32_t* rule_nops;
  const int32_t* rule_pos;
  const int64_t* rule_coeff;
  const int64_t* rule_bound;
} mlt_surrogate;

/* times[n], ok[n] for configuration indices: reps = 0 -> true_times
 * (measurement.py:212-226), reps >= 1 -> measured_times(indices, reps)
 * (:228-238). Times are NaN where a launch rule fires. Static space rules are
 * NOT applied (as in the reference runner). */
MLT_API int mlt_surrogate_times(mlt_ctx* ctx, const mlt_space* space, const mlt_surrogate* spec, const int64_t* idx,
                                int64_t n, int32_t reps, double* times, uint8_t* ok);
/* Exhaustive search over [begin, end) (tuner.py:191-224): among statically
 * valid, launchable configurations, the minimum (time, index) with times
 * measured with `reps` repetitions (0 = noise-free); *n_valid = how many were
 * measured, *n_below = how many were strictly faster than `threshold` (the
 * rank of a tuned result). *best_idx = -1 when none is valid. */
MLT_API int mlt_surrogate_best(mlt_ctx* ctx, const mlt_space* space, const mlt_surrogate* spec, int64_t begin,
                               int64_t end, int32_t reps, double threshold, int64_t* best_idx, double* best_time,
                               int64_t* n_valid, int64_t* n_below);

/* ---------------------------------------------------------------------------
 * Benchmark kernels behind the runner protocol (the
 * reference has only the seam: ExternalRunner / runner.measure,
 * measurement.py:274-348, tuner.py:80-92). The paper's three benchmarks
 * (Tables 1-2) with their knobs realised on sm_100a.
 * ------------------------------------------------------------------------- */
typedef struct mlt_convbench mlt_convbench;

/* Device-resident W x H fp32 image: `image` (host, W*H floats) or, when NULL,
 * uniform [0,1) from a splitmix64 hash of (seed, pixel index). */
MLT_API int mlt_convbench_create(int device, int32_t width, int32_t height, const float* image, uint64_t seed,
                                 mlt_convbench** out);
MLT_API int mlt_convbench_destroy(mlt_convbench* bench);
/* knobs[9] = {wg_x, wg_y, ppt_x, ppt_y, use_image, use_local, padding, interleaved, unroll}.
 * *status: 0 valid, 1 invalid-launch (Outcome "invalid-launch"). *seconds: min over reps. */
MLT_API int mlt_convbench_run(mlt_convbench* bench, const int32_t* knobs, int32_t reps, double* seconds,
                              int32_t* status);
/* Output of the last run / the input image, W*H floats (host). */
MLT_API int mlt_convbench_output(mlt_convbench* bench, float* host_out);
MLT_API int mlt_convbench_input(mlt_convbench* bench, float* host_in);
MLT_API const char* mlt_convbench_last_error(void);

/* Stereo matching (Tables 1-2; bench_stereo.cu): winner-take-all SAD
 * disparity over D disparities and a (2R+1)^2 window, 8-bit W x H images.
 * `left`/`right` (host, W*H bytes each) or, when both NULL, a synthetic pair
 * (random right image; left = right shifted by a piecewise-constant disparity
 * field + noise) from `seed`. */
typedef struct mlt_stereobench mlt_stereobench;
MLT_API int mlt_stereobench_create(int device, int32_t width, int32_t height, int32_t disparities, int32_t radius,
                                   const uint8_t* left, const uint8_t* right, uint64_t seed, mlt_stereobench** out);
MLT_API int mlt_stereobench_destroy(mlt_stereobench* bench);
/* knobs[11] = {wg_x, wg_y, ppt_x, ppt_y, img_left, img_right, local_left, local_right,
 *              unroll_disparity, unroll_diff_x, unroll_diff_y}; status/seconds as for conv. */
MLT_API int mlt_stereobench_run(mlt_stereobench* bench, const int32_t* knobs, int32_t reps, double* seconds,
                                int32_t* status);
MLT_API int mlt_stereobench_output(mlt_stereobench* bench, uint8_t* host_disparity);
/* Budgeted screening for exhaustive sweeps (see mlt_raybench_set_budget). */
MLT_API int mlt_stereobench_set_budget(mlt_stereobench* bench, uint64_t budget_ns);
MLT_API int mlt_stereobench_input(mlt_stereobench* bench, uint8_t* host_left, uint8_t* host_right);
MLT_API const char* mlt_stereobench_last_error(void);

/* Volume raycasting (Tables 1-2; bench_raycast.cu): an image_w x
 * image_h RGBA fp32 image from a vx x vy x vz 8-bit volume (x fastest) with a
 * 256-entry RGBA transfer function, orthographic rays, front-to-back
 * compositing. `volume` / `transfer` (host) or NULL for the synthetic
 * volume (from `seed`) / the default transfer function. */
typedef struct mlt_raybench mlt_raybench;
MLT_API int mlt_raybench_create(int device, int32_t image_w, int32_t image_h, int32_t vx, int32_t vy, int32_t vz,
                                const uint8_t* volume, const float* transfer, uint64_t seed, mlt_raybench** out);
MLT_API int mlt_raybench_destroy(mlt_raybench* bench);
/* knobs[10] = {wg_x, wg_y, ppt_x, ppt_y, img_data, img_transfer, local_transfer, const_transfer,
 *              interleaved, unroll_ray}; status/seconds as for conv. */
MLT_API int mlt_raybench_run(mlt_raybench* bench, const int32_t* knobs, int32_t reps, double* seconds, int32_t* status);
MLT_API int mlt_raybench_output(mlt_raybench* bench, float* host_rgba);
/* Budgeted screening for exhaustive sweeps: each launch stops starting new
 * pixels budget_ns after it began (a slower configuration then times as
 * >= budget_ns); 0 = normal measurement (the default). */
MLT_API int mlt_raybench_set_budget(mlt_raybench* bench, uint64_t budget_ns);
MLT_API int mlt_raybench_volume(mlt_raybench* bench, uint8_t* host_volume);
MLT_API int mlt_raybench_transfer(mlt_raybench* bench, float* host_rgba256);
/* 19 floats: centre[3], u[3], v[3], dir[3], 1/dir[3], scale, width/2, height/2, opacity threshold */
MLT_API int mlt_raybench_camera(mlt_raybench* bench, float* host_cam19);
MLT_API const char* mlt_raybench_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* MLTUNE_B200_H */
