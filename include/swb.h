/*
 * swb.h — C ABI of the B200 SW# hot path (libswb.so).
 *
 * This is the drop-in boundary for the reference package `wavealign`
 * (/root/reference/pkg/src/wavealign).  The reference's operator API for the
 * hot path is the wavefront engine plus two numba kernels; every entry point
 * below replaces one of them and is bound from Python with ctypes
 * (paper_1304_5966_b200/_lib.py).  No torch types cross this boundary: plain
 * pointers, sizes and POD structs only.
 *
 *   swb_pass        replaces WavefrontEngine.run_wavefront(PassSpec) -> PassResult
 *                   (engine.py:188-282) and, below it, kernels.affine_block
 *                   (kernels.py:21-88).  The PassSpec callables become enums:
 *                   left_border/top_h/top_f -> swb_border (engine.py:340-401),
 *                   prune -> swb_pass_desc.prune (phase1.py:55-59),
 *                   band -> has_band/band_lo/band_hi (engine.py:225-231).
 *   swb_crossings   replaces phase3.find_crossing (phase3.py:136-190), batched
 *                   over one Myers-Miller level: both half passes, the
 *                   middle-row combination and _pick_crossing (phase3.py:123-133)
 *                   run on the device.
 *   swb_leaves      replaces kernels.leaf_solve (kernels.py:91-185) as called by
 *                   phase3._solve_leaf (phase3.py:200-247), batched.
 *
 * Conventions (mirroring the reference):
 *   rows = seq1 ("target"), columns = seq2 ("query"); cell (i, j) is DP
 *   (i+1, j+1); a gap of length k costs gap_open + k*gap_extend (model.py:6);
 *   Op codes 0 '=', 1 'X', 2 'I' (consumes seq2), 3 'D' (consumes seq1)
 *   (model.py:32-36).  All arithmetic is exact integer arithmetic.
 *
 * Return codes: 0 = ok; negative = error class, message in swb_last_error()
 * (thread-local).  No exception crosses the ABI.  The Python layer maps
 * SWB_EINVAL/SWB_ERANGE/SWB_EUNSUPPORTED -> ValueError, SWB_ECUDA -> WorkerPanic
 * (errors.py:35-36), SWB_EMISMATCH -> ScoreMismatch (errors.py:41-45).
 *
 * Threading: one swb_ctx per (process, device); calls on one context are
 * serialised by the context's mutex, different contexts may be used from
 * different threads concurrently (split mode runs two engines at once,
 * split.py:111-122).  ctypes releases the GIL for the duration of a call.
 */
#ifndef SWB_H
#define SWB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SWB_OK 0
#define SWB_EINVAL (-1)
#define SWB_ECUDA (-2)
#define SWB_ERANGE (-3)
#define SWB_EUNSUPPORTED (-4)
#define SWB_EMISMATCH (-5)

/* Border families, engine.py:340-401 (local_borders, restricted_borders,
 * global_borders(lead="free"|"continue"|"charge")). */
#define SWB_BORDER_LOCAL 0
#define SWB_BORDER_RESTRICTED 1
#define SWB_BORDER_GLOBAL_FREE 2
#define SWB_BORDER_GLOBAL_CONTINUE 3
#define SWB_BORDER_GLOBAL_CHARGE 4

/* Best-cell tracking, kernels.py:16-18. */
#define SWB_TRACK_NONE 0
#define SWB_TRACK_MIN 1 /* best positive cell, ties to smallest (i, j) */
#define SWB_TRACK_MAX 2 /* best cell of any sign, ties to largest (i, j) */

typedef struct swb_ctx swb_ctx;

/* ScoringScheme (model.py:129-191) restricted to what the kernels need.
 * sub is k x k row-major, sub[a*k + b] = score of seq1 code a vs seq2 code b,
 * k <= 32.  Alphabets of <= 7 symbols whose sub + gap_open + gap_extend fit a
 * signed byte use register profiles (PRMT); larger ones (protein, BLOSUM62)
 * a shared-memory table. */
typedef struct {
  int32_t k;
  int32_t sub[1024];
  int32_t gap_open;
  int32_t gap_extend;
  int32_t max_sub;
} swb_scheme;

/* One wavefront pass (PassSpec, engine.py:93-117).  Rows are seq1 codes
 * [off1, off1+len1) of the uploaded sequence seq1, reversed when rev1 != 0
 * (row r then reads code[off1 + len1 - 1 - r]); columns likewise. */
typedef struct {
  int32_t seq1;
  int32_t seq2;
  int64_t off1;
  int64_t len1;
  int64_t off2;
  int64_t len2;
  int32_t rev1;
  int32_t rev2;
  int32_t border;     /* SWB_BORDER_* */
  int32_t clamp_zero; /* local recurrence: H = max(..., 0) */
  int32_t track;      /* SWB_TRACK_* */
  int32_t has_band;   /* admissible (row - col) interval [band_lo, band_hi] */
  int64_t band_lo;
  int64_t band_hi;
  int32_t prune;            /* 0 off; 1 phase-1 running-best bound (phase1.py:55-59, local);
                               2 fixed target (restricted search: no path through a skipped
                                 block reaches prune_target); 3 target at corner (no path
                                 through a skipped block reaches DP (corner_i, corner_j)
                                 with score prune_target) */
  int32_t want_final_rows;  /* fill final_row_h/f (PassResult, engine.py:120-131) */
  int64_t* final_row_h;     /* caller-owned int64[len2 + 1] or NULL */
  int64_t* final_row_f;     /* sentinel-derived values are reported <= SWB_NEG_REPORT */
  /* Row slab of a pass split across GPUs; all zero for a whole pass.
   * row_offset: DP row of this slab's first row (left border, reported best_i).
   * ext_in_*:  device pointers (local memory, written by the GPU above through
   *            peer mapping) holding the bottom DP row (H-go-ge, F) of the slab
   *            above and its column progress counter; replaces the top border.
   * ext_out_*: device pointers (peer memory of the GPU below) receiving this
   *            slab's bottom row and progress.  Slab rows must be a multiple of
   *            32 x rows_per_lane except for the last slab; no band. */
  int64_t row_offset;
  int64_t prune_target;
  int64_t corner_i;
  int64_t corner_j;
  uint64_t ext_in_buf;
  uint64_t ext_in_progress;
  uint64_t ext_out_buf;
  uint64_t ext_out_progress;
  /* rows of the whole pass below this slab (0 for a whole pass): the prune
   * bounds count the rows a path can still take on the GPUs below. */
  int64_t rows_after;
  /* Tile bound maps of the (seq1, seq2) pair (swb_bounds_reset, DESIGN.md
   * §3.6).  bound_write: 0 none, 1 record an upper bound of this pass's H per
   * 1024 x 1024 forward tile into the forward map, 2 into the reverse map.
   * bound_read: 0 none, 1 / 2 skip a block (prune kinds 2 and 3 only) when
   * max(block inputs) + W max_sub + (map max over the block's tiles) +
   * bound_offset < prune_target. */
  int32_t bound_write;
  int32_t bound_read;
  int64_t bound_offset;
  /* Running best shared between the row slabs of one pass (prune kind 1):
   * device pointer to an int32 word, zero before the pass, that every slab
   * reads (system scope) and raises with atomicMax — local memory on one GPU
   * or a CUDA-IPC peer mapping across GPUs.  0: the pass keeps its own
   * running best.  Any slab's best is a real cell score, so a shared best is
   * as sound as the reference's barrier-refreshed one (engine.py:260-261). */
  uint64_t shared_best;
} swb_pass_desc;

/* PassResult (engine.py:120-131) minus the final rows (written in place). */
typedef struct {
  int64_t best_score; /* track NONE: 0 */
  int64_t best_i;     /* cell coordinates; -1 when nothing tracked */
  int64_t best_j;
  int64_t cells_executed;
  int64_t tiles_total;    /* warp-strip x 32-column tiles */
  int64_t tiles_executed;
  int64_t tiles_pruned;
  int64_t tiles_banded_out;
  double kernel_ms; /* CUDA-event time of the launch that carried this pass */
  int32_t kernel;        /* 0: 32-bit lane kernel, 1: packed 16x2 kernel, 2: int64 kernel */
  int32_t rows_per_lane; /* R of that launch (packed: R row pairs per lane) */
} swb_pass_out;

/* Myers-Miller subproblem (phase3.Subproblem, phase3.py:46-67). */
typedef struct {
  int64_t si, sj; /* start (inclusive) */
  int64_t ei, ej; /* end (exclusive) */
  int64_t expected;
  int32_t start_vgap;
  int32_t end_vgap;
  /* optional tile-bound pruning: when use_bounds != 0 and
   * the pair's maps were filled by phases 1 and 2, prefix / suffix are the
   * scores of the optimal path before (si, sj) and after (ei, ej). */
  int32_t use_bounds;
  int32_t pad;
  int64_t prefix;
  int64_t suffix;
} swb_subproblem;

/* find_crossing result (phase3.py:136-190). status 0 = ok, 1 = ScoreMismatch
 * (best != expected; best reported in `upper`). */
typedef struct {
  int64_t mid_i, mid_j;
  int64_t upper, lower;
  int32_t gap_join;
  int32_t status;
} swb_crossing;

/* Reported value for sentinel-derived (minus-infinity) DP entries: the
 * reference uses NEG_INF = -(2**61) (kernels.py:14); values below
 * SWB_NEG_REPORT are sentinel-derived and are mapped onto NEG_INF + drift. */
#define SWB_NEG_INF_REF (-(int64_t)2305843009213693952LL)
#define SWB_NEG_REPORT (-(int64_t)536870912LL)

/* --- lifecycle ------------------------------------------------------------ */
swb_ctx* swb_ctx_create(int32_t device);
void swb_ctx_destroy(swb_ctx* ctx);
const char* swb_last_error(void);
int32_t swb_version(void);

/* --- sequences --------------------------------------------------------------
 * Upload host codes (uint8, one code per residue, values < k) to the device;
 * the context keeps the forward copy and a reversed copy so reversed slices
 * (phase2.py:153-154, phase3.py:159-162, split.py:105-107) need no host copy. */
int32_t swb_seq_upload(swb_ctx* ctx, const uint8_t* codes, int64_t n, int32_t* seq_id);
int32_t swb_seq_release(swb_ctx* ctx, int32_t seq_id);

/* --- passes ------------------------------------------------------------------
 * Run n independent passes in one persistent launch (run_wavefront x n). */
int32_t swb_pass(swb_ctx* ctx, const swb_scheme* scheme, const swb_pass_desc* descs,
                 int32_t n, swb_pass_out* outs);

/* --- tile bound maps ------------------------------------------------------------
 * (Re)allocate and clear the forward and reverse tile maps of the pair
 * (seq1, seq2): ceil(n1/1024) x ceil(n2/1024) int32 each.  One pair at a time
 * per context; a later call for another pair replaces them. */
int32_t swb_bounds_reset(swb_ctx* ctx, int32_t seq1, int32_t seq2);
/* Diagnostics: copy the forward (which = 1) or reverse (2) map, row-major
 * nr x nc, raw encoding (value + 2^30, -1 = never written) into out[0..cap);
 * returns nr * nc (the size when out is NULL). */
int64_t swb_bounds_read(swb_ctx* ctx, int32_t which, int32_t* out, int64_t cap);
/* Device address and element count (nr * nc) of the forward (1) or reverse
 * (2) map, for collectives that assemble one map from the row slabs of several
 * GPUs (multigpu.align_distributed).  Row tile t occupies [t * nc, (t+1) * nc). */
int32_t swb_bounds_device(swb_ctx* ctx, int32_t which, uint64_t* ptr, int64_t* n, int64_t* nc);

/* --- Myers-Miller level --------------------------------------------------------
 * For each subproblem (rows >= 2 required): run the upper forward and the
 * lower reverse global passes (lead modes as phase3.py:165-176, band as
 * phase3.py:83-98 when band != 0), combine the middle rows and pick the
 * crossing with _pick_crossing's tie rules.  cells_out (optional) receives the
 * number of DP cells executed. */
int32_t swb_crossings(swb_ctx* ctx, const swb_scheme* scheme, int32_t seq1, int32_t seq2,
                      const swb_subproblem* subs, int32_t n, int32_t band,
                      swb_crossing* out, int64_t* cells_out);

/* --- leaves --------------------------------------------------------------------
 * Batched leaf_solve.  Leaf t writes its ops (forward order) to
 * ops_out[ops_offsets[t] ...], capacity rows+cols; counts[t] = op count or -1
 * on a traceback dead end; scores[t] = achieved score (F or H at (rows, cols)
 * per end_vgap), SWB_NEG_INF_REF on a dead end.  Band per phase3.py:230-233
 * when band == 1, the explicit (row - col) interval [prefix, suffix] of each
 * subproblem when band == 2 (leaf_solve's lo / hi arguments, kernels.py:91),
 * else the full rectangle. */
int32_t swb_leaves(swb_ctx* ctx, const swb_scheme* scheme, int32_t seq1, int32_t seq2,
                   const swb_subproblem* leaves, int32_t n, int32_t band,
                   uint8_t* ops_out, const int64_t* ops_offsets, int64_t* counts,
                   int64_t* scores);

/* --- measurement ----------------------------------------------------------------
 * Integer/DPX issue-rate microbenchmark (warp-lane ops per second, whole chip);
 * the roofline denominator for the cell-update kernels. */
typedef struct {
  double viaddmnmx;
  double vimnmx3;
  double viaddmnmx_relu;
  double iadd;
  double prmt;
  double imad;
  double ms_last;
  int32_t sms;
} swb_int_peak;
int32_t swb_measure_int_peak(swb_ctx* ctx, swb_int_peak* out);

/* Tuning knobs: "max_ctas_per_sm" (0 = occupancy limit), "rows_per_lane"
 * (0 = automatic, else an instantiated rows-per-lane), "x2" (1 = allow the
 * packed 16x2 score-pass kernel), "x2_R" (its rows per lane, 0 = automatic),
 * "mm_prune" (corner-target pruning in Myers-Miller halves), "claim_mode"
 * (0 auto, 1 CTA claiming, 2 warp claiming), "proto", "reset_debug",
 * "job_major", "bound_maps", "live_ranges", "p2_R", "mm_R", "mm_static",
 * "mm_dyn", "chain_wait" (acquire polling in chain-shaped passes),
 * "chain_cta" (chain-shaped passes in CTA chunks),
 * "chain_chunk" (4 or 8 strips per chunk), "x2_blk" (packed kernel steps per
 * block: 0 = by rounds of items, 32, 64), "map_tile_log2",
 * "wide_log2" (int64-kernel threshold, §3.11), "watchdog_ms", "claim_log",
 * "min_R", "live_big". */
int32_t swb_set_option(swb_ctx* ctx, const char* name, int64_t value);
/* Current value of a tuning option (-1 for an unknown name). */
int64_t swb_get_option(swb_ctx* ctx, const char* name);

/* Diagnostics: out[0] = cycles warps spent waiting on the strip above,
 * out[1] = total strip cycles, summed over all passes since "reset_debug". */
int32_t swb_debug_stats(swb_ctx* ctx, int64_t* out, int32_t n);
/* Per-strip (start ns, end ns, wait ns) of the most recent pass launch; returns
 * the number of values available. */
int32_t swb_debug_times(swb_ctx* ctx, int64_t* out, int32_t n);
/* Per-strip record of the most recent pass launch, 12 values per strip:
 * (cb_static << 32 | cb_start), (ce << 32 | early-exit column or -1),
 * (blocks executed << 32 | blocks skipped), (live lo << 32 | live hi of the
 * producer), times the strip was run, (smid << 32 | cta << 8 | warp), start
 * ns, 0, then the strip result (score key, i, j, has).  Returns the number of
 * values available (out may be null). */
int32_t swb_debug_strips(swb_ctx* ctx, int64_t* out, int32_t n);
/* Claim log (option "claim_log" or env SWB_CLAIM_LOG): out[0] = entries ever
 * written, out[8 + 4k ...] = ring entry k (launch id, kind << 56 | smid << 40 |
 * cta << 8 | warp, value, globaltimer ns); kind 1 = claimed item, 2 = claim
 * counter at CTA start, 3 = progress of strip 0 at CTA start. */
int32_t swb_debug_claims(swb_ctx* ctx, int64_t* out, int32_t n);

/* CUDA events on the context's stream around a caller-defined region
 * (bench timing of K steps on the launching stream). */
int32_t swb_timer_start(swb_ctx* ctx);
int32_t swb_timer_stop(swb_ctx* ctx, double* ms);
/* Overwrite `bytes` (0: 512 MiB, > the 126 MB L2) of scratch on the stream to
 * evict earlier working sets from L2 between timed steps. */
int32_t swb_flush_l2(swb_ctx* ctx, int64_t bytes);

/* --- multi-GPU boundary rows ------------------------------------
 * A boundary is int2[n2] + one int32 progress counter in device memory of the
 * consuming GPU.  Export/import turn it into a peer pointer for the producing
 * GPU's process (CUDA IPC over NVLink). */
int32_t swb_boundary_alloc(swb_ctx* ctx, int64_t n2, uint64_t* buf, uint64_t* progress);
int32_t swb_boundary_reset(swb_ctx* ctx, uint64_t progress);
int32_t swb_boundary_free(swb_ctx* ctx, uint64_t buf, uint64_t progress);
int32_t swb_ipc_export(swb_ctx* ctx, uint64_t ptr, uint8_t* handle64);
int32_t swb_ipc_import(swb_ctx* ctx, const uint8_t* handle64, uint64_t* ptr);
int32_t swb_ipc_close(swb_ctx* ctx, uint64_t ptr);

/* Device-side timing of the most recent swb_pass launch (ms, CUDA events). */
double swb_last_kernel_ms(swb_ctx* ctx);
/* Number of kernels this context launched since creation (for gpu_launches). */
int64_t swb_launch_count(swb_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* SWB_H */
