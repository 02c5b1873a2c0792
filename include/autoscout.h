/*
 * autoscout.h -- C ABI of the B200-native AutoScout candidate-scoring library (libautoscout.so).
 *
 * What it computes.  AutoScout (arXiv 2603.11603) searches a hierarchical configuration space
 * of sparse structural knobs and dense execution knobs "valid only under specific upstream
 * decisions" (masking function M(s), :171).  The data-parallel hot path
 * built here scores MANY candidate configurations at once (BASELINE.json north_star): for each
 * candidate index it decodes the configuration, applies conditional validity, runs the
 * analytical iteration-time/memory simulator, evaluates a GP posterior and an acquisition
 * against the profiled set, and keeps a top-k ("the top-K configurations ... are prioritized
 * for re-evaluation").  All readings of ambiguous passages are listed in
 * DESIGN.md §3; formulas in SURVEY.md Appendix A.
 *
 * Conventions.
 *  - Every call returns as_status; nothing throws across the ABI.  On error the thread-local
 *    message is available from autoscout_last_error().
 *  - "host" pointers are caller-owned CPU memory read/written during the call only.
 *    "device" pointers are caller-owned CUDA memory on the handle's device (typically PyTorch
 *    tensors) that must stay alive until the enqueued work on `cuda_stream` completes.
 *  - cuda_stream is a cudaStream_t passed as void* (NULL = legacy default stream).
 *  - A handle is bound to one CUDA device (or to none: cuda_device = -1 gives a host-only
 *    handle that supports parsing and the host introspection calls, never scoring).  Handles
 *    are not thread-safe; use one per thread/rank.
 *  - Index spaces (R2-R4): the RAW index is the mixed-radix number of the digit
 *    tuple, first-declared feature most significant.  A CVI position p in [0, n_cvi) is the
 *    p-th raw index, ascending, that satisfies the canonical-inactive rule and every structural
 *    (non-resource) constraint of the space.  n_cvi must be < 2^32.
 *  - Scores: higher is better.  EI is reported as log EI; LCB as kappa*sigma - mu; SIM as
 *    -ln(cost_sim).  Ties are broken by the smaller raw index.
 */
#ifndef AUTOSCOUT_H
#define AUTOSCOUT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct as_space as_space; /* opaque */

typedef enum {
  AS_OK = 0,
  AS_ERR_INVALID_ARG = 1,    /* null pointer, bad enum, k out of range, non-finite/<=0 cost */
  AS_ERR_SPACE_SCHEMA = 2,   /* malformed JSON, unknown key/type, default not in domain */
  AS_ERR_SPACE_CYCLE = 3,    /* cyclic activation dependency */
  AS_ERR_SPACE_ORDER = 4,    /* forward gate reference, or a tail gating group not contiguous (R4) */
  AS_ERR_SPACE_EMPTY = 5,    /* empty domain or no valid configuration */
  AS_ERR_INDEX_RANGE = 6,    /* raw >= n_raw, cvi >= n_cvi, batch outside [0, n_cvi) */
  AS_ERR_INVALID_CONFIG = 7, /* observed configuration not valid (structure or resource check) */
  AS_ERR_NO_OBSERVATIONS = 8,/* EI requested with no observed configuration */
  AS_ERR_NUMERIC = 9,        /* Cholesky of the GP covariance failed */
  AS_ERR_CAPACITY = 10,      /* a compile-time limit (features, domain size, M, k', n_cvi) exceeded */
  AS_ERR_STATE = 11,         /* call not valid in the handle's state (e.g. topk before score, host-only handle) */
  AS_ERR_UNCERTIFIED = 12,   /* top-k returned but the FP32 screen could not be certified */
  AS_ERR_CUDA = 13,          /* CUDA runtime error */
  AS_ERR_OOM = 14            /* device allocation failed */
} as_status;

typedef enum { AS_MODE_RANGE = 0, AS_MODE_SAMPLE = 1, AS_MODE_LIST = 2 } as_mode;
typedef enum { AS_ACQ_EI = 0, AS_ACQ_LCB = 1, AS_ACQ_SIM = 2 } as_acq;

typedef struct {
  uint64_t n_raw;        /* product of the domain sizes */
  uint64_t n_cvi;        /* number of structurally valid configurations */
  int32_t n_features;    /* d */
  int32_t n_structures;  /* distinct assignments of the structural prefix */
  int32_t n_prefix;      /* structural prefix length (R4) */
  int32_t n_components;  /* tail gating groups */
  int32_t n_observed;    /* M of the current fit */
  int32_t max_observed;  /* capacity for M */
  uint64_t n_launches;   /* kernels this handle has launched so far (generate, score, merge, refine, mask) */
  uint64_t fit_upload_bytes; /* host->device bytes of the last observe()/observe_clear() GP upload */
} as_space_info;

typedef struct {
  int32_t mode;          /* as_mode.  RANGE: candidate j is CVI position begin+j.
                            SAMPLE: candidate j is pi_seed(begin+j), a Feistel permutation of [0,n_cvi).
                            LIST: candidate j is CVI position d_positions[begin+j] (an optimizer-
                            driven batch, e.g. autoscout_neighbors) */
  int32_t acq;           /* as_acq */
  uint64_t begin;        /* first position (RANGE), first sample ordinal (SAMPLE), first list entry (LIST) */
  uint64_t count;        /* number of candidates; RANGE/SAMPLE: begin+count <= n_cvi */
  uint64_t seed;         /* SAMPLE permutation seed */
  double kappa;          /* LCB exploration weight (default 2) */
  double xi;             /* EI margin (default 0) */
  int32_t k;             /* the top-k that autoscout_topk will request (1..1024); sizes the pool */
  int32_t accumulate;    /* 0: reset the running pool before merging this batch; 1: merge into it */
  float* d_scores;       /* device, nullable, [count] in batch order: FP32 score, -INF if masked */
  uint64_t* d_raw;       /* device, nullable, [count] raw index of each candidate */
  uint64_t* d_valid_count; /* device, nullable: atomically incremented by #valid candidates */
  const uint64_t* d_positions; /* LIST only (else ignored): device array of CVI positions, caller-owned;
                            it must stay valid until the autoscout_topk / autoscout_topk_pool call
                            of this pool returns (certification may re-score recorded batches).
                            An entry >= n_cvi is scored as masked (-INF, raw UINT64_MAX). */
  float* d_screen;       /* device, nullable, [4*count] in batch order, parity/debug output of the
                            FP32 screen that admits candidates: mu, sigma^2, the
                            screen score acq(mu, sigma^2) and its certified upper bound
                            acq(mu - d_mu, sigma^2 + d_s2) + margin, exactly as the kernel uses them
                            (independent of d_scores, which switches the kernel to an FP64
                            acquisition).  Written by the one-hot tensor-core kernel (the path
                            taken for M >= 64 or batches >= 2^20 candidates); untouched (NaN
                            prefill is the caller's) for other paths and masked candidates. */
} as_score_args;

/* Parse and validate a space JSON document (schema: DESIGN.md §2), build the
 * per-structure tables of the compact valid index, and upload them to `cuda_device` (-1: host only).
 * Source: SPEC.md:54-62 load_space; Table 1. */
as_status autoscout_space_create(const char* space_json, int32_t cuda_device, as_space** out);
void autoscout_space_destroy(as_space* s);
/* Sizes of the parsed space (host; out is caller-owned).  n_cvi counts the configurations that
 * satisfy the canonical-inactive rule and the structural constraints ("each edge
 * represents a valid refinement"; SPEC.md:90-98 enumerate, :109 world-size rule; reading R4). */
as_status autoscout_space_info(const as_space* s, as_space_info* out);

/* Append n profiled configurations (raw index, cost > 0 in objective units) and refit the GP on
 * the host in FP64 (Cholesky; alpha = K^-1 r; W = L^-1; f* = min ln c), then upload the fit on
 * `cuda_stream`.  n may be 0 (refit only).  Errors: INDEX_RANGE, INVALID_CONFIG, INVALID_ARG,
 * CAPACITY (M > max_observed), NUMERIC.  Source: PAPER.md:263-265 (profiled vs simulated
 * evaluations); GP reading DESIGN.md R9. */
as_status autoscout_observe(as_space* s, const uint64_t* raw_idx, const double* cost, int64_t n,
                            void* cuda_stream);
as_status autoscout_observe_clear(as_space* s);
/* Host introspection of the current fit: M, b (prior offset), f* (incumbent ln cost). */
as_status autoscout_observe_info(const as_space* s, int32_t* m_out, double* b_out, double* fstar_out);

/* Enqueue the scoring of a batch (generate + score + pool-merge launches, asynchronous): for every
 * candidate index decode the configuration of the hierarchical space ("subsequent
 * decisions are valid only under specific upstream decisions", :137, :171 masking function M(s)),
 * apply validity (Table 1 gates PAPER.md:507, :510; SPEC.md:81-89 is_feasible; the resource check
 * of the simulator), run the analytical simulator (reading R6: SPEC.md:486-497 and
 * the paper's own simulators are regressions), score
 * it against the profiled set (GP posterior + acquisition, readings R1, R9, R10; north_star), and
 * keep the CTA top-k' for "the top-K configurations ... prioritized for re-evaluation"
 * (PAPER.md:265).  Candidates are generated from indices in registers; per-candidate outputs are
 * optional and caller-owned.  accumulate = 1 merges into the running pool and requires the same
 * acq / kappa / xi as the pool's first batch.  A refit (observe, observe_clear, set_gp_hyper)
 * empties the pool.
 * Errors: INDEX_RANGE, NO_OBSERVATIONS, INVALID_ARG (also kappa < 0 or non-finite kappa / xi,
 * mixed acquisition with accumulate), STATE (host-only handle), CUDA. */
as_status autoscout_score_batch(as_space* s, const as_score_args* a, void* cuda_stream);

/* Finalize ("re-evaluation" of the top-K; ties by the lower index, SPEC.md:197,
 * :506, reading R11): FP64 re-score of the running pool, order (score desc, raw asc), one entry
 * per configuration (a configuration scored twice is returned once), certification
 * (doubles the pool and re-scores the recorded batches on failure).  Writes
 * n_out = min(k, #valid finite scores) entries to the host arrays raw_out/score_out (length >= k).
 * Synchronizes `cuda_stream`.  Errors: STATE (nothing scored), UNCERTIFIED, CUDA. */
as_status autoscout_topk(as_space* s, int32_t k, uint64_t* raw_out, double* score_out, int32_t* n_out,
                         void* cuda_stream);

/* Sharding.  Pool entries are {double score; uint64_t raw} (16 bytes), ordered
 * (score desc, raw asc).  topk_pool: refine the local pool and copy up to `cap` entries to host
 * memory; n_out = entries written; *cut_out = an entry that every locally scored candidate NOT in
 * the exported pool ranks after or equals in the total order (cut score = upper bound on its
 * score; score -INF when nothing was dropped).  topk_merge: merge `n_pools` gathered pools laid out
 * as [n_pools][cap] entries with per-pool counts and cuts ([n_pools] entries); certify globally:
 * certified iff the k-th merged entry ranks strictly before every cut.  Host-only work: valid on
 * a host-only handle (s may be NULL).  *certified_out = 1 if the merged top-k is certified. */
as_status autoscout_topk_pool(as_space* s, int32_t k, void* pool_out, int32_t cap, int32_t* n_out,
                              void* cut_out, void* cuda_stream);
as_status autoscout_topk_merge(const as_space* s, const void* pools, const int32_t* counts,
                               const void* cuts, int32_t n_pools, int32_t cap, int32_t k,
                               uint64_t* raw_out, double* score_out, int32_t* n_out,
                               int32_t* certified_out);

/* Device-resident sharding: the pools stay in device memory and
 * are exchanged with ONE all_gather_into_tensor (NCCL over NVLink); only the final top-k is read
 * back.  Packed pool = cap + 2 entries of {double score; uint64_t raw} (16 B):
 *   [0] header: score = n (number of exported entries, as a double), raw = 1 if locally certified;
 *   [1] cut: every candidate scored on this handle but not exported ranks after or equals it in
 *       the total order (score desc, raw asc); score -INF if nothing was dropped;
 *   [2, 2 + n) entries in the total order, one per configuration; the rest {-INF, UINT64_MAX}.
 * topk_pool_device: FP64 refine of the running pool, device sort + de-duplication + pack into
 *   d_pool_out (device, caller-owned, (cap + 2) * 16 bytes); grows k' and re-scores the recorded
 *   batches while the local top-k is not certified (reads back 4 bytes per attempt).  Syncs the
 *   stream.  Errors: STATE (nothing scored / host-only handle), INVALID_ARG, CUDA.
 * topk_merge_device: merge n_pools packed pools laid out contiguously in d_pools (device,
 *   n_pools * (cap + 2) entries: the all-gather output) into d_out (device, k + 2 entries, same
 *   layout: header {n, certified}, the best cut of all pools, the global top-k).  Certified iff the
 *   k-th merged entry ranks strictly before every pool's cut (PAPER.md:265 top-K re-evaluation;
 *   ties SPEC.md:197).  Asynchronous on cuda_stream. */
as_status autoscout_topk_pool_device(as_space* s, int32_t k, void* d_pool_out, int32_t cap, void* cuda_stream);
as_status autoscout_topk_merge_device(as_space* s, const void* d_pools, int32_t n_pools, int32_t cap, int32_t k,
                                      void* d_out, void* cuda_stream);

/* Exact host introspection (parity and tests).
 * decode: digits of a raw index by mixed radix, first-declared feature most significant (reading
 *   R2, "deterministic order"); digits_out host [n_features]; valid_out = 1 iff the
 *   configuration is canonical (inactive features at their default), meets
 *   every constraint and passes the resource check.  AS_ERR_INDEX_RANGE if raw >= n_raw.
 * cvi_to_raw: raw index of CVI position cvi (the cvi-th valid-structure configuration in raw
 *   order, reading R4; SPEC.md:90-98 enumerate).  AS_ERR_INDEX_RANGE if cvi >= n_cvi.
 * sample_to_cvi: the SAMPLE-mode position pi_seed(ordinal) (reading R3, a Feistel bijection of
 *   [0, n_cvi)).  AS_ERR_INDEX_RANGE if ordinal >= n_cvi. */
as_status autoscout_decode(const as_space* s, uint64_t raw, int32_t* digits_out, int32_t* valid_out);
/* Activity of every feature of a raw index (host): bit j of *active_mask_out = feature j is active
 * (its activation predicate holds over earlier features; PAPER.md:171 masking function
 * M(s)).  AS_ERR_INDEX_RANGE if raw >= n_raw. */
as_status autoscout_activity(const as_space* s, uint64_t raw, uint32_t* active_mask_out);
as_status autoscout_cvi_to_raw(const as_space* s, uint64_t cvi, uint64_t* raw_out);
as_status autoscout_sample_to_cvi(const as_space* s, uint64_t seed, uint64_t ordinal, uint64_t* cvi_out);
/* ML-II evidence of GP hyper-parameter settings, batched on the device (
 * the paper fixes no surrogate and no hyper-parameters, R1, R21).  hyp: host,
 * n_set x (d + 2) doubles per setting [lengthscale_0 .. lengthscale_{d-1}, sf2, sn2], all > 0.
 * lml_out: host, n_set log marginal likelihoods of the current observed residuals
 * r = y - m0 - b under N(0, k(x_i, x_j) + sn2 I) (the kernel of the space), -INF where the matrix is
 * not positive definite.  Synchronous on cuda_stream.  AS_ERR_NO_OBSERVATIONS with M = 0,
 * AS_ERR_STATE on a host-only handle, AS_ERR_INVALID_ARG for a non-positive entry. */
as_status autoscout_gp_lml(as_space* s, const double* hyp, int32_t n_set, double* lml_out, void* cuda_stream);
/* Replace the GP hyper-parameters (lengthscale: d host doubles; sf2, sn2 > 0) and refit the
 * current observed set under them (as observe_clear + observe of the same observations). */
as_status autoscout_set_gp_hyper(as_space* s, const double* lengthscale, double sf2, double sn2);
/* ML-II by batched evidence (R21): setting 0 = the current hyper-parameters, settings
 * 1..n_set-1 drawn log-uniformly (lengthscales in [0.1, 10], sf2 in [1e-3, 10], sn2/sf2 in
 * [1e-6, 1e-1]) from counter-based splitmix64(seed ^ 0x3111 ^ (64 h + k)) uniforms; all evaluated
 * by autoscout_gp_lml in one launch; the best (lowest index on ties) is returned through
 * best_hyp_out (host, d + 2, nullable), best_lml_out, best_index_out and, if apply != 0, set with
 * autoscout_set_gp_hyper. */
as_status autoscout_ml2(as_space* s, int32_t n_set, uint64_t seed, int32_t apply, double* best_hyp_out,
                        double* best_lml_out, int32_t* best_index_out, void* cuda_stream);
/* GP prior mean m0 of a configuration under the current fit (host, FP64; R9, R20):
 * source_out = 1 if it is the regression-simulator ensemble (space JSON gp.prior = "ensemble"
 * and at least one simulator with holdout R^2 > 0 after the last observe; SURVEY.md §8(f) NEXT-1,
 * PAPER.md:518-548), else 0 and m0 = ln cost_sim of the analytical simulator.  The same m0 is
 * used on the device for every candidate.  AS_ERR_INDEX_RANGE if raw >= n_raw. */
as_status autoscout_prior(const as_space* s, uint64_t raw, double* m0_out, int32_t* source_out);
/* The four Table 2 simulators of the last fit (PAPER.md:524-531 order: 3D-Parallelism,
 * 5D-Parallelism, DDP-Aware, Communication-Aware): holdout R^2 (-INF = not fitted: fewer than
 * |subset|+2 training observations) and weights max(0,R^2)/sum;
 * available_out = 0 when every R^2 <= 0 ("Unavailable") or gp.prior = "sim".
 * Arrays are host, 4 entries each, nullable. */
as_status autoscout_ensemble_info(const as_space* s, double* r2_out, double* w_out, int32_t* available_out);
/* Exact CVI position of a raw index (host).  member_out = 1 iff raw is in the compact valid index
 * (G1 canonical + every non-resource constraint, R4), and then cvi_out is its position;
 * otherwise cvi_out = number of members with a smaller raw index.  AS_ERR_INDEX_RANGE if
 * raw >= n_raw.  Inverse of autoscout_cvi_to_raw on members. */
as_status autoscout_raw_to_cvi(const as_space* s, uint64_t raw, uint64_t* cvi_out, int32_t* member_out);
/* MCTS subtree as a batch ("each node corresponds to a
 * partial configuration ... each edge represents a valid refinement"): the configurations whose
 * first n_assigned features (declaration order) carry digits[0..n_assigned) form one contiguous
 * CVI range [begin, begin+count) -- the structural digits are the most significant (R2, R4) --
 * so AS_MODE_RANGE over it scores every completion of the partial assignment in one launch.
 * n_assigned = 0: the whole CVI.  count = 0 if no member has that prefix.  AS_ERR_INVALID_ARG
 * for n_assigned outside [0, d] or a digit outside its domain. */
as_status autoscout_subtree_range(const as_space* s, const int32_t* digits, int32_t n_assigned,
                                  uint64_t* begin_out, uint64_t* count_out);
/* Coordinate-neighbour batch of a configuration (PAPER.md:173
 * "perturbs the active parameter along its current search direction", SPEC.md:230-247 propose /
 * update with step doubling): for every ACTIVE feature of kind "dense" of `raw` in declaration
 * order, every step 2^e (e = 0, 1, ... while 2^e < n_f) and direction +1 then -1, the
 * configuration with that digit moved by the step, if it stays in the domain and is a CVI member
 * (moving a gate can make the neighbour non-canonical: it is then skipped).  Writes the CVI
 * positions in that order to cvi_out (host, cap entries); n_out = the number of neighbours.
 * AS_ERR_CAPACITY (n_out still set) if n_out > cap; AS_ERR_INDEX_RANGE if raw >= n_raw.
 * The base configuration itself need not be valid.  Score the result with AS_MODE_LIST. */
as_status autoscout_neighbors(const as_space* s, uint64_t raw, uint64_t* cvi_out, int32_t cap, int32_t* n_out);
/* FP64 simulator + resource check of one configuration (host; reading R6: SPEC.md:486-497, SURVEY.md
 * A.3/A.4).  ok_out = G4 passes (memory <= capacity).  AS_ERR_INDEX_RANGE if raw >= n_raw. */
as_status autoscout_simulate(const as_space* s, uint64_t raw, double* cost_out, double* mem_out,
                             int32_t* ok_out);
/* Mask kernel (the masking function M(s) of PAPER.md:171 over raw index ranges, for exhaustive
 * parity with enumeration): validity bit of every raw index in
 * [raw_begin, raw_begin+count) -> d_bits (device, (count+31)/32 words, bit i of word w =
 * raw_begin+32w+i); d_valid_count (device, nullable) += number of valid.  Valid = canonical-
 * inactive + structural constraints (reading R5) + resource check
 * (reading R7).  AS_ERR_INDEX_RANGE if the range exceeds n_raw. */
as_status autoscout_mask_range(as_space* s, uint64_t raw_begin, uint64_t count, uint32_t* d_bits,
                               uint64_t* d_valid_count, void* cuda_stream);

/* Posterior path of the score kernel: 0 = auto (the one-hot tensor-core kernel if its shared memory
 * fits and M >= 64 or the batch has >= 2^20 candidates; else, for M >= 64, the SIMT-r^2 tensor-core
 * kernel; else the fused SIMT FP32 kernel),
 * 1 = force SIMT, 2 = force tensor cores with r^2 on the SIMT pipes (3xTF32 L^-1 k),
 * 3 = force tensor cores for both r^2 (one-hot FP16 contraction) and L^-1 k.  All compute the
 * same quantities; the override exists for A/B parity tests and
 * profiling.  Errors: AS_ERR_INVALID_ARG for other values; a forced path whose shared memory
 * does not fit fails at score time with AS_ERR_CAPACITY. */
as_status autoscout_set_path(as_space* s, int32_t path);

/* Candidates per generate + score slice on the one-hot tensor-core path: each slice's
 * compact list of valid candidates needs up to 40 B per candidate of device memory (default 2^27
 * candidates = 5.4 GB worst case, one slice for the 10^8 bench batch).  Results do not depend on it.
 * AS_ERR_INVALID_ARG outside [128, 2^31]. */
as_status autoscout_set_slice(as_space* s, uint64_t max_candidates);

/* Asynchronous observe (enable != 0; spaces with the simulator prior, gp.prior = "sim"): observe()
 * validates and decodes the new observations synchronously (its argument errors are reported as
 * before), then returns while a host thread computes the GP fit and the device-layout operand
 * tables (P:263-265's "profiled set" update).  Every later call that reads the
 * fit waits for it first; score_batch launches the fit-independent candidate generation of its
 * first slice (decode, mask, simulator) before waiting, so the host fit overlaps GPU work.  An
 * error of the deferred fit (AS_ERR_NUMERIC: covariance not positive definite) is returned by that
 * next call, once; the handle then keeps the previous observed set.  Results are identical to the
 * synchronous mode.  Only observed sets of >= 128 points are fitted asynchronously (smaller fits
 * take tens of microseconds and stay inline).  Off by default; with enable = 0 any pending fit is
 * completed first. */
as_status autoscout_set_async_observe(as_space* s, int32_t enable);

/* Device-time of the last score kernel launch in ms (CUDA events on the launching stream,
 * recorded when `timing` was enabled), for the roofline report in bench.py. */
as_status autoscout_set_timing(as_space* s, int32_t enable);
as_status autoscout_last_kernel_ms(as_space* s, double* score_ms, double* merge_ms);
/* Split of the last timed launch on the one-hot tensor-core path (set_path 3 / auto): device time
 * of the candidate-generation kernels (decode + mask + simulator -> compact list) and of the
 * tensor-core score kernels, summed over the batch's slices.  Both are 0 for
 * the other paths.  AS_ERR_STATE if timing was off. */
as_status autoscout_last_phase_ms(as_space* s, double* gen_ms, double* score_ms);

const char* autoscout_last_error(void); /* thread-local */

#ifdef __cplusplus
}
#endif
#endif /* AUTOSCOUT_H */
