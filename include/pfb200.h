/*
 * pfb200.h -- C ABI of the B200-native NLL engine (library: libpfb200.so).
 *
 * This is the drop-in boundary for the reference's hot path: the per-event
 * PDF evaluation + negative-log-likelihood reduction that the minimiser calls
 * at every step (GooFit 2.0, re-derived as the Python package "parafit").
 * The reference has no native FFI of its own; its plug points are Python
 * protocols, and every entry point below replaces exactly one of them:
 *
 *   pfb_nll / pfb_nll_block_sums   <- engine.nll_block_sums + math.fsum
 *                                     (/root/reference/pkg/src/parafit/engine.py:190-243)
 *   pfb_nll_partial_async          <- sharding.partial_nll (sharding.py:94-114)
 *   pfb_acc_round / pfb_finalize   <- sharding.reduce_partials / reduction.round_exact
 *                                     (sharding.py:117-131, reduction.py:127-137)
 *   pfb_terms_block_sums           <- reduction.block_sums + math.fsum (reduction.py:59-75)
 *   pfb_exact_sum_host             <- reduction.ExactAccumulator.round (reduction.py:78-118)
 *   pfb_shard_bounds               <- sharding.shard (sharding.py:68-91), bounds only
 *   pfb_grid_*                     <- dalitz.integration_grid / compute_integrals
 *                                     (dalitz.py:246-329)
 *   pfb_plan_*                     <- the PdfNode tree + KIND_OPS dispatch (pdf.py:58-105,234-269)
 *
 * Conventions
 *   - Every function returns a status code (0 = PFB_OK); codes map 1:1 onto the
 *     reference exception classes (errors.py), see enum pfb_status.
 *   - Host pointers are borrowed for the duration of the call. Device buffers are
 *     owned by the handle that allocated them and freed by its *_destroy.
 *   - One driver thread per context; calls on a context are not re-entrant.
 *   - All arithmetic is IEEE binary64 on CUDA cores (never tensor cores, never FP32).
 */
#ifndef PFB200_H
#define PFB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PFB_ABI_VERSION 1

/* Fixed reduction block: reference DEFAULT_BLOCK (reduction.py:25). */
#define PFB_BLOCK 4096

/* Exact second-stage accumulator: 68 signed 32-bit-digit limbs covering
 * 2^-1074 .. 2^1102, then 4 special counters.  Summed (int64) across shards and
 * GPUs with one allreduce; rounded once (round-half-even) = math.fsum. */
#define PFB_NLIMBS 68
#define PFB_ACC_POSINF 68
#define PFB_ACC_NEGINF 69
#define PFB_ACC_NAN 70
#define PFB_ACC_FAILS 71 /* number of events that failed a density check */
#define PFB_ACC_WORDS 72

/* Status codes <-> reference exceptions (/root/reference/pkg/src/parafit/errors.py). */
enum pfb_status {
    PFB_OK = 0,
    PFB_E_NONPOSITIVE_DENSITY = 1, /* NonPositiveDensity(index, value)   errors.py:89 */
    PFB_E_NONFINITE_DENSITY = 2,   /* NonFiniteDensity(index)            errors.py:54 */
    PFB_E_NEGATIVE_DENSITY = 3,    /* NegativeDensity(index, value)      errors.py:62 */
    PFB_E_FRACTION_OUT_OF_RANGE = 4, /* FractionOutOfRange               errors.py:79 */
    PFB_E_EMPTY_DATASET = 5,       /* EmptyDataSet                       errors.py:98 */
    PFB_E_NONPOSITIVE_NORM = 6,    /* NonPositiveNorm                    errors.py:71 */
    PFB_E_DEGENERATE_GRID = 7,     /* DegenerateGrid                     errors.py:111 */
    PFB_E_INVALID_SUM = 8,         /* math.fsum ValueError (inf + -inf)  */
    PFB_E_NONPOSITIVE_EXPECTATION = 9, /* NonPositiveExpectation(bin, value) errors.py:102 */
    PFB_E_ENVELOPE_HIT = 10,       /* toy generation: a density above the envelope
                                      (mcgen.py _EnvelopeHit; caller rescans) */
    PFB_E_ATTEMPTS_EXHAUSTED = 11, /* AttemptsExhausted                  errors.py */
    PFB_E_PEER_TIMEOUT = 12,       /* a peer rank never posted its accumulator */
    PFB_E_UNBOUNDED_OBSERVABLE = 13, /* UnboundedObservable               errors.py:75 */
    PFB_E_OUT_OF_BOUNDS = 14,      /* OutOfBounds (set_value, core.py:126-142) */
    PFB_E_INVALID_ARGUMENT = 20,
    PFB_E_UNSUPPORTED_PLAN = 21,
    PFB_E_CUDA = 30,
    PFB_E_NO_DEVICE = 31,
    PFB_E_OUT_OF_MEMORY = 32
};

/* Node kinds: reference KIND_OPS keys (pdf.py:234-240, dalitz.py:413). */
enum pfb_kind {
    PFB_GAUSSIAN = 1,    /* exp(-0.5((x-mu)/sigma)^2)        pdf.py:122-127 */
    PFB_EXPONENTIAL = 2, /* exp(alpha x)                     pdf.py:141-144 */
    PFB_POLYNOMIAL = 3,  /* sum_k c_k x^k (Horner)           pdf.py:164-178 */
    PFB_ADD = 4,         /* sum_k w_k child_k/norm_k          pdf.py:205-219 */
    PFB_PROD = 5,        /* prod_k child_k/norm_k             pdf.py:222-227 */
    PFB_DALITZ = 6       /* |sum_k c_k BW_k Z_k|^2            dalitz.py:181-230,380-384 */
};

/* One PDF-tree node, listed in post-order (PdfNode.walk, pdf.py:86-90): the
 * children of a node are the `nchild` subtrees immediately preceding it. */
typedef struct pfb_node {
    int32_t kind;   /* enum pfb_kind */
    int32_t nchild; /* add/prod: >= 2; primitives: 0 */
    int32_t col0;   /* store column of the first observable (-1 if none) */
    int32_t col1;   /* store column of the second observable (dalitz s13), else -1 */
    int32_t nparam; /* raw parameter values this node consumes from `values` */
    int32_t aux;    /* dalitz: index into the pfb_dalitz_desc array; else 0 */
} pfb_node;

/* Raw per-call parameter values, concatenated in node (post-)order:
 *   gaussian [mu, sigma]; exponential [alpha]; polynomial [c0..c_{n-1}];
 *   add [f0..f_{k-2}] (last weight implied, pdf.py:205-210); prod [];
 *   dalitz, per term [mass, width, magnitude, phase] (dalitz.py:369-371).
 * Norms: one value per node, same order (engine.resolve_norms, engine.py:162). */

#define PFB_MAX_DALITZ_TERMS 16

/* A DecayChannel (dalitz.py:47-77) plus the structural part of its terms
 * (ResonanceTerm.pair / .spin, dalitz.py:86-106). */
typedef struct pfb_dalitz_desc {
    double mother_mass, m1, m2, m3;
    int32_t nterms;
    int32_t pair[PFB_MAX_DALITZ_TERMS]; /* 12, 13 or 23 */
    int32_t spin[PFB_MAX_DALITZ_TERMS]; /* 0 or 1 */
} pfb_dalitz_desc;

/* Error record: the first failing check in the reference's evaluation order. */
typedef struct pfb_err {
    int32_t code;  /* enum pfb_status */
    int32_t node;  /* post-order node index of the failing check (-1: root p>0 check) */
    int64_t index; /* NonPositiveDensity: global (index_offset + local);
                      NonFinite/Negative: chunk-local, as the reference reports */
    double value;  /* offending value (NaN when the reference carries none) */
} pfb_err;

typedef struct pfb_ctx pfb_ctx;
typedef struct pfb_store pfb_store;
typedef struct pfb_plan pfb_plan;
typedef struct pfb_grid pfb_grid;
typedef struct pfb_objective pfb_objective;

/* Normalisation programs of a pfb_objective node (see pfb_objective_create). */
enum pfb_norm_kind {
    PFB_NORM_CONST = 0,       /* `value` (add / prod: 1, pdf.py:238-239; or a norm fixed for the fit) */
    PFB_NORM_GAUSSIAN = 1,    /* _gaussian_norm over [lo, hi] (pdf.py:130-138) */
    PFB_NORM_EXPONENTIAL = 2, /* _exponential_norm over [lo, hi] (pdf.py:147-161) */
    PFB_NORM_DALITZ = 3,      /* dalitz_norm with a fixed overlap matrix (dalitz.py:332-349) */
    PFB_NORM_QUADRATURE = 4   /* pfb_quadrature of the node's own plan over a rule store
                                 (_polynomial_norm, pdf.py:192-199) */
};
typedef struct pfb_obj_node {
    int32_t norm_kind;  /* enum pfb_norm_kind */
    int32_t weight_col; /* PFB_NORM_QUADRATURE: the rule store's weight column */
    double lo, hi;      /* observable bounds (gaussian / exponential) */
    double value;       /* PFB_NORM_CONST */
    pfb_plan* quad_plan;        /* PFB_NORM_QUADRATURE: plan of the node alone (root norm 1) */
    const pfb_store* quad_rule; /* PFB_NORM_QUADRATURE: abscissas + weights */
} pfb_obj_node;


/* ---- library / context ---------------------------------------------------- */
int pfb_version(void);
const char* pfb_strerror(int code);
int pfb_device_count(int* out);
int pfb_ctx_create(int device, pfb_ctx** out);
int pfb_ctx_destroy(pfb_ctx* ctx);
/* Run all work of this context on an existing cudaStream_t (e.g. torch's current
 * stream, so NCCL collectives order naturally); NULL restores the private stream. */
int pfb_ctx_set_stream(pfb_ctx* ctx, void* cuda_stream);
void* pfb_ctx_stream(pfb_ctx* ctx);
/* Block until all work enqueued on the context's stream has finished. */
int pfb_ctx_synchronize(pfb_ctx* ctx);
/* Tuning: warps cooperating on one 4096-event block (0 = automatic; 1,2,4,8). */
int pfb_ctx_set_warps_per_block(pfb_ctx* ctx, int warps);
/* Kernel structure (all modes give the NLL within rounding of the reference;
 * within a mode totals are bitwise invariant under launch shape and ranges):
 *  1 (default) TMA-fed kernels -- the unit-sum kernel for log-domain plans
 *    (C2; the register-window SIMT form of the same blocks up to 8 blocks
 *    per SM), the TMA product kernel for two-column product evaluators
 *    (Dalitz), per-warp bulk prefetch for one-column ones (C1; the TMA
 *    product kernel from 24 blocks per SM);
 *  2 the reference-tree TMA kernel for log-domain plans, per-warp bulk
 *    prefetch for every product evaluator;
 *  3 the TMA product kernel for every product evaluator;
 *  4 as 1, with the one-column SumPdf (C1 / C5) on the warp-task kernel;
 *  0 the SIMT log-domain streaming kernel (reference tree) everywhere. */
int pfb_ctx_set_pipeline(pfb_ctx* ctx, int mode);
/* Number of engine kernels launched on this context since creation. */
int pfb_ctx_launch_count(pfb_ctx* ctx, int64_t* out);
/* Device time (ms) of the most recent NLL kernel, measured with CUDA events on
 * the launching stream (only when timing is enabled). */
int pfb_ctx_enable_timing(pfb_ctx* ctx, int on);
int pfb_ctx_last_kernel_ms(pfb_ctx* ctx, float* out);

/* ---- event store: device-resident SoA columns (core.UnbinnedDataSet, core.py:215-309) */
int pfb_store_create(pfb_ctx* ctx, int32_t ncols, int64_t n_events, pfb_store** out);
int pfb_store_upload(pfb_store* st, int32_t col, const double* host, int64_t offset, int64_t count);
/* Borrow caller-owned device columns (must stay alive while the store is used). */
int pfb_store_wrap(pfb_ctx* ctx, int32_t ncols, int64_t n_events, const double* const* dev_cols,
                   pfb_store** out);
int pfb_store_device_ptr(pfb_store* st, int32_t col, void** out);
int pfb_store_destroy(pfb_store* st);

/* ---- plan: flattened PDF tree ---------------------------------------------- */
int pfb_plan_compile(pfb_ctx* ctx, const pfb_node* nodes, int32_t nnodes,
                     const pfb_dalitz_desc* dalitz, int32_t ndalitz, pfb_plan** out);
int pfb_plan_destroy(pfb_plan* plan);
/* Which evaluator the plan uses: 0 literal interpreter, 1 sum-of-products
 * log-domain, 2 Dalitz (recompute), 3 Dalitz (lineshape cache). */
int pfb_plan_evaluator(const pfb_plan* plan, int32_t* out);
/* Lineshape cache for Dalitz plans: 0 off (recompute per event), 1 on, 2 auto. */
int pfb_plan_set_lineshape_cache(pfb_plan* plan, int32_t mode);
/* Number of per-event amplitude rows recomputed by the lineshape cache so far. */
int pfb_plan_cache_recomputes(const pfb_plan* plan, int64_t* out);

/* ---- NLL ---------------------------------------------------------------------
 * -sum_{i in [begin,end)} ln(eval(x_i)/norm_root), block sums by the reference
 * half-folding tree per 4096-event block (relative to `begin`), combined exactly
 * and rounded once.  Bitwise equal to engine.nll for any begin/end grouping that
 * the reference would use.  `index_offset` is added to NonPositiveDensity
 * indices (engine._nll_terms `offset`, engine.py:177-186). */
int pfb_nll(pfb_ctx* ctx, const pfb_plan* plan, const pfb_store* st, int64_t begin, int64_t end,
            int64_t index_offset, const double* values, int32_t nvalues, const double* norms,
            int32_t nnorms, double* out_nll, pfb_err* out_err);
/* Same evaluation, returning the per-block sums (engine.nll_block_sums). */
int pfb_nll_block_sums(pfb_ctx* ctx, const pfb_plan* plan, const pfb_store* st, int64_t begin,
                       int64_t end, int64_t index_offset, const double* values, int32_t nvalues,
                       const double* norms, int32_t nnorms, double* out_block_sums,
                       int64_t n_out, pfb_err* out_err);
/* Batched objective: the NLL at `npts` <= 16 parameter
 * points -- e.g. the 2P finite-difference points of fitting.fd_gradient
 * (fitting.py:140-151) or the Hesse stencil (fitting.py:180-213) -- each
 * bitwise equal to its own pfb_nll.  HBM-bound plans evaluate all points in
 * ONE pass over the events (the stage stays in shared memory while every point
 * is folded); others run one fused launch per point.  values: npts rows of
 * nvalues; norms: npts rows of nnorms; out_nll / out_err: npts entries.
 * Returns the first failing point's status (in point order) or PFB_OK. */
int pfb_nll_batch(pfb_ctx* ctx, const pfb_plan* plan, const pfb_store* st, int64_t begin, int64_t end,
                  int64_t index_offset, const double* values, int32_t npts, int32_t nvalues,
                  const double* norms, int32_t nnorms, double* out_nll, pfb_err* out_err);
/* Enqueue (no host sync) the exact partial of [begin,end) into `dev_acc`
 * (PFB_ACC_WORDS int64 on the device, overwritten).  Sum these across ranks with
 * one allreduce, then pfb_finalize.  The local error record is kept in the
 * context (pfb_last_error). */
int pfb_nll_partial_async(pfb_ctx* ctx, const pfb_plan* plan, const pfb_store* st, int64_t begin,
                          int64_t end, int64_t index_offset, const double* values,
                          int32_t nvalues, const double* norms, int32_t nnorms, int64_t* dev_acc);
/* Enqueue one fused NLL launch (no host synchronisation, no fix-up launch):
 * the finishing CTA writes the exact accumulator to dev_acc (PFB_ACC_WORDS
 * int64, device memory) and [deferred-block count, error key] to
 * dev_status[0..1].  For back-to-back throughput measurement (bench.py): a
 * step is valid when its deferred count is 0 and its key ~0; its NLL is
 * pfb_acc_round(dev_acc), bitwise pfb_nll's.  Fractions out of range return
 * PFB_E_FRACTION_OUT_OF_RANGE without a launch. */
int pfb_nll_enqueue(pfb_ctx* ctx, const pfb_plan* plan, const pfb_store* st, int64_t begin, int64_t end,
                    const double* values, int32_t nvalues, const double* norms, int32_t nnorms, int64_t* dev_acc,
                    int64_t* dev_status);
/* Round a (reduced) device accumulator; synchronises the context stream.
 * out_fails = failed events/blocks summed over the ranks, + 1 when this
 * context's last partial had fractions out of range (pdf._fractions,
 * pdf.py:205-210: checked on the host, never in the accumulator). */
int pfb_finalize(pfb_ctx* ctx, const int64_t* dev_acc, double* out_nll, int64_t* out_fails);
/* The first error of the context's last partial in reference evaluation order
 * (FractionOutOfRange included). */
int pfb_last_error(pfb_ctx* ctx, pfb_err* out_err);
/* *out = 1 when the last partial's fractions were out of range
 * (FractionOutOfRange pending; pfb_last_error reports it). */
int pfb_ctx_last_fraction_failure(pfb_ctx* ctx, int32_t* out);
/* End-to-end: host columns (pinned or pageable) streamed to the device in
 * chunks on two copy/compute streams, evaluated, reduced.  Same result bits as
 * pfb_nll over the uploaded store. */
int pfb_nll_host(pfb_ctx* ctx, const pfb_plan* plan, const double* const* host_cols,
                 int32_t ncols, int64_t n_events, const double* values, int32_t nvalues,
                 const double* norms, int32_t nnorms, double* out_nll, pfb_err* out_err);

/* ---- reduction kernels on given terms (known-answer tests) -------------------- */
int pfb_terms_block_sums(pfb_ctx* ctx, const double* host_terms, int64_t n, double* out_block_sums,
                         double* out_total);
/* Host-side exact sum through the same limb code the device uses. */
int pfb_exact_sum_host(const double* values, int64_t n, double* out);
/* Round an accumulator held in host memory. */
int pfb_acc_round(const int64_t* acc, double* out);
/* Add values to a host accumulator (same digit split as the device). */
int pfb_acc_add_host(int64_t* acc, const double* values, int64_t n);

/* ---- binned data -------------------------------------------- */
/* BinnedDataSet.fill (core.py:370-379): histogram events [begin, end) of the
 * store columns cols[0..naxes) into contents[prod(nbins)] (host, row-major,
 * last axis fastest), adding each bin's count.  Per event and axis the bin is
 * clip(int64(floor((x - lower) / width)), 0, nbins - 1) with numpy's cast
 * semantics (NaN / inf -> INT64_MIN -> bin 0): bit-exact. */
int pfb_bin_fill(pfb_ctx* ctx, const pfb_store* store, int64_t begin, int64_t end, int32_t naxes,
                 const int32_t* cols, const double* lower, const double* width, const int64_t* nbins,
                 double* inout_contents);
/* ---- the minimiser's objective in C (replaces FitManager.fcn's objective,
 * fitting.py:436-447, + nll's host part, engine.py:214-243) ------------------
 * Binds plan + store + [begin, end) once.  value_src[r] (plan raw value r) is
 * an index into the free-parameter vector x or -1 (then value_const[r]);
 * nodes[i] gives node i's normalisation program.  pfb_objective_eval maps x to
 * the raw values, recomputes only the norms whose inputs changed (bitwise),
 * and runs the fused NLL (== pfb_nll on the same values / norms).  A norm
 * failure returns PFB_E_NONPOSITIVE_NORM / PFB_E_UNBOUNDED_OBSERVABLE with
 * err->node (callers re-evaluate that point through the reference path for
 * the reference's exception).  eval_batch: npts <= 16 points (rows of x),
 * one pass over the events where the plan allows (pfb_nll_batch); the
 * points' quadrature norms are launched back to back into separate result
 * slots and waited for once; points after a host norm failure (in
 * sequential order) are not evaluated. */
int pfb_objective_create(pfb_ctx* ctx, pfb_plan* plan, const pfb_store* store, int64_t begin, int64_t end,
                         int32_t nfree, const int32_t* value_src, const double* value_const,
                         const pfb_obj_node* nodes, const double* dalitz_matrix, pfb_objective** out);
/* Bounds of the free parameters (set_value's check, core.py:126-142): an x
 * outside them (or NaN) returns PFB_E_OUT_OF_BOUNDS without evaluating. */
int pfb_objective_set_bounds(pfb_objective* obj, const double* lower, const double* upper);
int pfb_objective_eval(pfb_objective* obj, const double* x, int32_t nfree, double* out_nll, pfb_err* out_err);
int pfb_objective_eval_batch(pfb_objective* obj, const double* xs, int32_t npts, int32_t nfree, double* out_nll,
                             pfb_err* out_err);
/* Persistent evaluation (on != 0): calls go through a kernel that stays
 * resident between calls -- the call's arguments are written into a mapped
 * pinned mailbox and a doorbell word, the kernel (one CTA per SM, polling)
 * runs the pass and posts the result into mapped memory: no launch and no
 * stream synchronisation per call.  Same canonical blocks, so the same bits
 * as the one-shot kernels.  Shapes without a persistent kernel, deferred
 * blocks (the exact fix-up) and any other device work on the context fall
 * back to / stop it (it restarts on the next call); it also leaves by itself
 * after 20 ms without a call.  off: stop it now. */
int pfb_objective_set_persistent(pfb_objective* obj, int32_t on);
/* Stop the context's resident kernel, if any. */
int pfb_ctx_persist_stop(pfb_ctx* ctx);
/* Diagnostics (PFB_PERSIST_TRACE set when the kernel starts): %globaltimer ns
 * of the last call -- doorbell seen, CTAs released, last CTA starts / ends its
 * pass, result posted. */
int pfb_ctx_persist_trace(pfb_ctx* ctx, uint64_t* out5);
/* New overlap matrix (2 K^2 doubles, re/im) after a shape change. */
int pfb_objective_set_matrix(pfb_objective* obj, const double* dalitz_matrix);
int pfb_objective_destroy(pfb_objective* obj);

/* Normalisation integral by quadrature (north_star item 4; pdf._polynomial_norm +
 * gauss_legendre_points, pdf.py:181-199): sum_j w_j * f(x_j) with f the plan's
 * unnormalised density (pass the root norm as 1) at the abscissas held in the
 * store's observable columns and the weights in column `weight_col`; each
 * product rounded once, the sum exact (correctly rounded dot product).
 * Density errors (NegativeDensity, NonFiniteDensity, ...) carry the abscissa
 * index, as the reference kernel on the abscissa array reports them. */
int pfb_quadrature(pfb_ctx* ctx, const pfb_plan* plan, const pfb_store* nodes, int32_t weight_col,
                   const double* values, int32_t nvalues, const double* norms, int32_t nnorms, double* out,
                   pfb_err* out_err);
/* binned_nll (engine.py:246-276): sum_b [nu_b - n_b ln nu_b] (observed bins;
 * nu_b otherwise), nu_b = (total * p(centre_b)) * volume, with p from the
 * literal interpreter on `centers` (one row per bin, the plan's column order)
 * and the sum exact (math.fsum).  Errors: the node kernels' (as pfb_nll, index
 * = bin), FractionOutOfRange, then PFB_E_NONPOSITIVE_EXPECTATION (index = first
 * observed bin with nu <= 0, value = nu). */
int pfb_binned_nll(pfb_ctx* ctx, const pfb_plan* plan, const pfb_store* centers, const double* contents,
                   int64_t nbins, double total, double volume, const double* values, int32_t nvalues,
                   const double* norms, int32_t nnorms, double* out_nll, pfb_err* out_err);

/* ---- toy generation, stream-exact ----------------------------- */
/* One numpy PCG64 stream: the 128-bit state and increment of
 * np.random.PCG64(SeedSequence(seed).spawn(streams)[i]).state. */
typedef struct {
    uint64_t state_hi, state_lo, inc_hi, inc_lo;
} pfb_pcg64;

typedef struct {
    int64_t attempts;     /* candidates drawn (stats["attempts"] / ["box_draws"]) */
    int64_t accepted;     /* stats["accepted"] contribution of this stream */
    int64_t in_boundary;  /* stats["in_boundary_draws"] (Dalitz) */
    int64_t produced;     /* events written */
    double observed;      /* PFB_E_ENVELOPE_HIT: the chunk's maximum density */
    int64_t ambiguous;    /* candidates of the consumed chunks whose accept decision (or the chunk's
                             envelope check) lies within 2^-47 relative of the density: 0 means the
                             sample is the reference's bit for bit (device densities follow the
                             reference's operation order; libm may differ from numpy by ulps) */
} pfb_gen_stats;

/* mcgen._scan_max (mcgen.py:52-54): max of the plan's unnormalised root
 * density (norms[root] = 1, children's norms as the reference passes them)
 * over points midpoints of [lo, hi]. */
int pfb_pcg_scan_1d(pfb_ctx* ctx, const pfb_plan* plan, const double* values, int32_t nvalues,
                    const double* norms, int32_t nnorms, double lo, double hi, int64_t points, double* out_max);
/* _dalitz_scan_grid + _masked_intensity_max (mcgen.py:209-222) on an n x n grid. */
int pfb_pcg_scan_dalitz(pfb_ctx* ctx, const pfb_dalitz_desc* channel, const double* term_values, int32_t n,
                        double* out_max);
/* _accept_reject_1d for one stream (mcgen.py:66-97): writes the accepted
 * samples (in the reference's order, the first n_wanted) to out column 0 at
 * out_offset.  PFB_E_ENVELOPE_HIT (stats->observed) asks the caller to rescan
 * and restart, PFB_E_ATTEMPTS_EXHAUSTED when the budget runs out. */
int pfb_pcg_generate_1d(pfb_ctx* ctx, const pfb_plan* plan, const double* values, int32_t nvalues,
                        const double* norms, int32_t nnorms, double lo, double hi, double envelope,
                        const pfb_pcg64* stream, int64_t n_wanted, int64_t budget, pfb_store* out,
                        int64_t out_offset, pfb_gen_stats* stats);
/* One stream of _dalitz_streams (mcgen.py:232-257): columns 0/1 = s12/s13. */
int pfb_pcg_generate_dalitz(pfb_ctx* ctx, const pfb_dalitz_desc* channel, const double* term_values,
                            double envelope, const pfb_pcg64* stream, int64_t n_wanted, int64_t budget,
                            pfb_store* out, int64_t out_offset, pfb_gen_stats* stats);

/* ---- binary SoA ingest ---------------------------------------- */
/* Rows of a 1-D little-endian float64 .npy column file (replaces the CSV path
 * dataio.py:20-83 for large runs). */
int pfb_npy_length(const char* path, int64_t* n_out);
/* Rows [src_offset, src_offset + count) of a .npy column straight into device
 * column `col` at dst_offset (pinned double-buffered, overlapped reads and
 * copies; no host copy of the column). */
int pfb_store_load_npy(pfb_store* store, int32_t col, const char* path, int64_t src_offset, int64_t dst_offset,
                       int64_t count);
/* The dataset range check (core.py:262-272) on the device: first row of
 * [begin, end) with x < lower, x > upper or non-finite (-1 if none). */
int pfb_store_check_range(pfb_store* store, int32_t col, int64_t begin, int64_t end, double lower, double upper,
                          int64_t* first_bad, double* bad_value);

/* ---- cross-GPU accumulator exchange over peer memory ------------------ */
/* Replaces the NCCL all-reduce of the 72-limb accumulator between the
 * one-process-per-GPU ranks with one single-CTA kernel over NVLink peer
 * memory.  Setup: pfb_peer_create (mailbox in this GPU's HBM; out_handle
 * receives its 64-byte cudaIpcMemHandle), exchange the handles between ranks
 * (e.g. torch.distributed.all_gather_object), pfb_peer_open.  Each call:
 * pfb_peer_allreduce sums dev_acc[0..72) over the ranks in place (rank order,
 * integer limbs: bitwise the single-GPU accumulator); PFB_E_PEER_TIMEOUT if a
 * peer does not post within timeout_s.  pfb_peer_attach / pfb_peer_mailbox
 * wire peers living in the same process (raw device pointers). */
int pfb_peer_create(pfb_ctx* ctx, int32_t rank, int32_t world, uint8_t* out_handle);
int pfb_peer_open(pfb_ctx* ctx, const uint8_t* handles);
int pfb_peer_attach(pfb_ctx* ctx, const void* const* mailboxes);
int pfb_peer_mailbox(pfb_ctx* ctx, void** out);
int pfb_peer_allreduce(pfb_ctx* ctx, int64_t* dev_acc, double timeout_s);
/* One NLL call over this rank's shard [begin, end) with the exchange fused
 * into the kernel: the CTA that finishes the launch trades the 72-limb
 * accumulator with every rank's mailbox over NVLink peer memory and exports
 * the global sum -- one launch per call, no separate collective (replaces
 * pfb_nll_partial_async + pfb_peer_allreduce / NCCL + pfb_finalize on the
 * common path).  Collective: every rank calls it with the same parameters.
 * *out_slow = 1 (and PFB_OK) when some rank deferred blocks to the exact
 * fix-up or hit an error: every rank then sees 1 and must redo the call on
 * the unfused path, which runs the fix-up and reports errors with their
 * global indices.  Fractions out of range (the same on every rank) also give
 * *out_slow = 1, without a launch.  PFB_E_PEER_TIMEOUT if a peer does not
 * post in timeout_s. */
int pfb_nll_peer(pfb_ctx* ctx, const pfb_plan* plan, const pfb_store* store, int64_t begin, int64_t end,
                 int64_t index_offset, const double* values, int32_t nvalues, const double* norms,
                 int32_t nnorms, double timeout_s, double* out_nll, int32_t* out_slow);

/* ---- sharding ------------------------------------------------------------------ */
/* Reference shard() bounds: bounds[0..workers] (sharding.py:80-85). */
int pfb_shard_bounds(int64_t n, int32_t workers, int64_t block, int64_t* bounds);

/* ---- Dalitz normalisation grid (dalitz.py:246-349) ----------------------------- */
int pfb_grid_create(pfb_ctx* ctx, const pfb_dalitz_desc* channel, int32_t nx, int32_t ny,
                    pfb_grid** out);
int pfb_grid_info(const pfb_grid* g, int64_t* n_inside, double* cell_area);
/* Row-major (s12 outer) in-boundary mask, nx*ny bytes. Bit-exact with the reference. */
int pfb_grid_mask(const pfb_grid* g, uint8_t* host_mask);
/* Overlap integrals I[i][j] = sum A_i conj(A_j) dA over the in-boundary nodes.
 * The grid keeps one device amplitude row per term: rows flagged in `rows` are
 * recomputed; matrix entries touching a term flagged in `stale` are recomputed,
 * all other entries are left as found in `inout_matrix` (complex, row-major,
 * interleaved re/im, K*K*2) -- the reference's prior reuse (dalitz.py:296-328).
 * `mass_width` holds [mass_i, width_i] per term. */
int pfb_grid_integrals(pfb_ctx* ctx, pfb_grid* g, int32_t nterms, const int32_t* pair,
                       const int32_t* spin, const double* mass_width, const uint8_t* rows,
                       const uint8_t* stale, double* inout_matrix);
int pfb_grid_destroy(pfb_grid* g);

/* ---- synthetic events (toy MC; mcgen.generate_1d / generate_dalitz, mcgen.py:105-257) */
/* Dalitz accept-reject into store columns 0 (s12) and 1 (s13): candidates
 * uniform in the (s12, s13) box (Philox4x32-10, counter = candidate index),
 * kept inside the kinematic boundary when u*envelope < |sum c_k A_k|^2, written in
 * candidate order (deterministic per seed).  term_values: [mass, width,
 * magnitude, phase] per term. */
int pfb_gen_dalitz(pfb_ctx* ctx, const pfb_dalitz_desc* channel, const double* term_values,
                   double envelope, uint64_t seed, int64_t n_events, pfb_store* out,
                   int64_t* out_candidates);
/* kind 0: f*Gauss(mu,sigma) + (1-f)*Exp(alpha) on [lo,hi] into column 0;
 * kind 1: Gauss(mu,sigma) on [lo,hi] into column 0 x Exp(alpha) into column 1. */
int pfb_gen_1d(pfb_ctx* ctx, int32_t kind, double mu, double sigma, double alpha, double f,
               double lo, double hi, uint64_t seed, int64_t n_events, pfb_store* out);
int pfb_store_download(pfb_store* st, int32_t col, double* host, int64_t offset, int64_t count);

/* ---- microbenchmarks used for the roofline denominators ------------------------ */
int pfb_fp64_peak(pfb_ctx* ctx, double* out_tflops);
/* Timing support (not on the NLL path): on the context stream, read
 * flush_bytes of flush_buf (a device buffer; L2 eviction) and keep every SM
 * busy for `cycles` clocks, so that a launch queued behind it is timed
 * without host-launch latency.  Uses the NLL kernels' shared-memory carveout. */
int pfb_ctx_spin(pfb_ctx* ctx, int64_t cycles, const double* flush_buf, int64_t flush_bytes);
/* Read-bandwidth microbenchmark of `bytes` of a device buffer: mode 0 SIMT
 * 16-byte loads, 1 bulk-copy ring (1 CTA/SM), 2 bulk-copy ring (2 CTAs/SM)
 * with chunk_kb-KB stages; median GB/s over reps launches. */
int pfb_read_bw(pfb_ctx* ctx, const double* buf, int64_t bytes, int32_t mode, int32_t chunk_kb, int32_t reps,
                double* out_gbps);
/* Launch fixed-cost microbenchmark: mode 0 empty kernel, 1 + NllArgs
 * parameter block, 2 + constant-bank reads, 3 + accumulator epilogue. */
int pfb_overhead_probe(pfb_ctx* ctx, int32_t mode, int32_t reps, double* out_us);

#ifdef __cplusplus
}
#endif
#endif /* PFB200_H */
