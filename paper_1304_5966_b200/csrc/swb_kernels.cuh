// Device code of the SW# wavefront pass (B200, sm_100a).
//
// One persistent kernel replaces WavefrontEngine.run_wavefront (engine.py:188-282)
// together with kernels.affine_block (kernels.py:21-88).
//
// Decomposition:
//   * A *warp-strip* is 32 lanes x R rows of seq1.  Lane l owns rows
//     [R0 + l*R, R0 + (l+1)*R) and keeps their H and E in registers; it sweeps the
//     strip's column range one column per step.  Lane l processes column s - l at
//     step s, so the vertical dependency (H, F of the row above) arrives from lane
//     l-1 by one __shfl_up per value per step, and the diagonal is the value that
//     arrived one step earlier.
//   * Warp-strips are chained through global memory: the strip's bottom row
//     (H, F) is flushed every 32 steps to a row buffer, followed by a release
//     store of the strip's progress counter; the strip below acquires it.  Two
//     row buffers per pass suffice (ordering argument in DESIGN.md §3.3).
//   * Work items are (pass, strip) pairs claimed in order by an atomic counter,
//     so any number of independent passes (Myers-Miller levels, the two halves
//     of split mode) share one launch; a strip only waits on an item claimed
//     before it, so the persistent launch cannot deadlock.
//
// Cell update (all int32, DPX; H kept as hm = H - (go+ge), E plain, F plain):
//   h2 = max(diag_m + (s + go + ge), E [, 0])        VIADDMNMX(.RELU)
//   F  = max(F - ge, h2_above - go - ge)              VIADDMNMX  (1-op F chain)
//   hm = max(F - (go+ge), h2 - (go+ge)) = H - (go+ge) IADD + VIADDMNMX
//   E' = max(E - ge, hm)                              VIADDMNMX
// F may use the pre-F value h2 of the row above instead of H because
// F - (go+ge) <= F - ge (go >= 0): max(F - ge, max(h2, F) - go - ge) ==
// max(F - ge, h2 - go - ge).  The substitution score s + go + ge is one PRMT
// (sign-replicating byte select) from a per-column profile word.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <climits>

#include <type_traits>

#include "swb_internal.h"

// Debug build (make CHECKED=1 -> libswb_checked.so): every global and shared
// index of the pass kernels goes through SWB_IX(i, n), which reports an index
// outside [0, n) with its source line and substitutes 0, so the run continues
// and every bad access of a launch is listed.  Compiled out otherwise.
#ifdef SWB_CHECKED
#include <cstdio>
// [0] violations, [1] line, [2] index, [3] bound of the first one (read by the host)
static __device__ long long g_swb_chk[4];
static __device__ __noinline__ long long swb_chk_fail(long long i, long long n, int line) {
  if (atomicAdd((unsigned long long*)&g_swb_chk[0], 1ULL) == 0) {
    g_swb_chk[1] = line;
    g_swb_chk[2] = i;
    g_swb_chk[3] = n;
  }
  printf("SWB_CHECK line %d: index %lld outside [0, %lld) block %d thread %d\n", line, i, n,
         (int)blockIdx.x, (int)threadIdx.x);
  return 0;
}
#define SWB_IX(i, n)                                                              \
  ((((long long)(i)) >= 0 && ((long long)(i)) < (long long)(n)) ? (long long)(i)  \
                                                              : swb_chk_fail((i), (n), __LINE__))
#else
#define SWB_IX(i, n) (i)
#endif

namespace swb {

constexpr int kTrackNone = 0;
constexpr int kTrackMin = 1;
constexpr int kTrackMax = 2;
constexpr int kPadCode = 7;  // row code for padding rows (profile byte -128)
// Progress counters of consecutive strips sit one 128-byte line apart: every
// counter is polled by its consumer and released by its producer each block,
// and 32 counters to a line made each line a shared hot spot in L2.
constexpr int kProgStride = 32;

struct JobDev {
  const uint8_t* rows;  // code of row i = rows[i * rstep]
  const uint8_t* cols;  // code of column j = cols[j * cstep]
  int32_t rstep, cstep;
  int32_t n1, n2;
  int32_t border;
  int32_t fill_h;  // H written into skipped cells: 0 (local) or NEG
  int32_t has_band, band_lo, band_hi;
  int32_t prune;         // 0 off, 1 running best (local), 2 fixed target, 3 target at corner
  int32_t prune_target;
  int32_t corner_i, corner_j;  // DP corner the path must reach (prune kind 3)
  int32_t nstrips;
  int32_t want_final;
  int64_t item_base;
  int2* buf[2];          // row buffers (hm, F), n2 entries each
  int32_t* progress;     // per strip (stride kProgStride): columns < progress of strip s are published
  int32_t* fin_h;        // final row H (DP columns 1..n2) or null
  int32_t* fin_f;
  int4* strip_res;       // per strip (score_m, i, j, has)
  unsigned long long* strip_times;  // per strip (start ns, end ns, wait ns) diagnostics
  unsigned long long* counters;  // [0] cells, [1] blocks executed, [2] blocks pruned,
                                 // [3] cycles spent waiting on the strip above, [4] strip cycles
  int32_t* prune_best;   // running best score (plain) for pruning
  int32_t row_offset;    // DP row of row 0 (row slab of a multi-GPU pass)
  int32_t rows_after;    // rows of the pass below this slab (prune bounds)
  int2* ext_in;          // strip 0 top input from the GPU above (null: top border)
  int32_t* ext_in_prog;
  int2* ext_out;         // last strip bottom row to the GPU below (null: local buffer)
  int32_t* ext_out_prog;
  // tile bound maps: 1024 x 1024 tiles of the forward
  // (seq1 x seq2) plane, int32 max(bound) + 2^30, -1 = never written (+inf)
  int32_t* bmap_out;       // this pass writes an upper bound of its H per tile
  const int32_t* bmap_in;  // this pass skips blocks the map proves useless
  int32_t map_nr, map_nc;  // tiles
  int32_t map_r0, map_rdir, map_c0, map_cdir;  // forward index of pass row/col 0, direction
  int32_t bound_offset;    // skip iff in + W max_sub + map max + bound_offset < prune_target
  int32_t range_offset;    // static ranges: tile useful iff fwd + rev + range_offset >= target
  const int32_t* rmap_fwd; // static strip ranges from both maps (null: band only)
  const int32_t* rmap_rev;
  int2* alive;             // per strip (live lo + 1, live hi + 1), 0 = unset (restricted passes)
  int32_t live_mode;       // bit 0: late start, bit 1: early exit
  int32_t best_sys;        // prune_best is shared across slabs / GPUs (informational)
  int4* bmap_live;         // writer: per row tile (-(lo+1), hi, covered) of the columns it swept
  const int4* rmap_live;   // reader: unwritten reverse-map tiles outside that interval are fill
  int32_t bin_rev;         // bmap_in is the reverse map (rmap_live applies to it)
  int32_t map_shift;       // log2 of the tile edge (10: 1024 x 1024 tiles)
};

static_assert(sizeof(JobDev) % 16 == 0, "JobDev arrays are staged next to int4 data");

struct PassParams {
  const JobDev* jobs;
  int32_t njobs;
  int32_t pad0;
  int64_t total_items;
  unsigned long long* claim;
  int32_t goe, ge, max_sub;
  int32_t proto;            // publication protocol variant (diagnostics)
  int32_t key_mul;          // == 32; opaque to ptxas so the key stays an IMAD
  int32_t group;            // > 0: CTA-level claiming of `group` strips (see pass_kernel)
  int32_t mirror;           // CTA mode, single round, 2 warps/sub-partition: mirror pairs
  uint32_t tlo[8], thi[8];  // profile word per column code
  const int2* item_map;     // claim order -> (job, strip); null: job-major by item_base
  int32_t warp_claim;       // 1: per-warp claiming even for few jobs (range-limited passes)
  int32_t chain_wait;       // chain-shaped passes: poll with ld.acquire, short back-off
  int32_t wild_const;       // packed kernel, WILD: sub + go + ge of code-4 rows (any column)
  int32_t chunk;            // > 0: CTA claims `chunk` consecutive strips (item_map: job, first)
  int32_t big;              // substitution table mode (tab) instead of tlo/thi
  const int32_t* tab;       // 32 x 33 table, device (big schemes)
  int32_t pad_pp[2];
  unsigned long long launch_id;   // diagnostics: context launch counter at this launch
  unsigned long long* claim_log;  // diagnostics ring (claim_log in swb_kernels.cuh) or null
  unsigned long long* strip_dbg;  // per strip (item_base + s) 8 words: ranges, exit,
                                  // block counts, live input (swb_debug_strips)
};

// Diagnostics log (swb_debug_claims): a monotonic ring over all launches of a
// context; entries (launch id, kind | sm | cta | warp, value, globaltimer).
__device__ __forceinline__ void claim_log(const PassParams& P, int kind, unsigned long long v) {
  if (!P.claim_log) return;
  const unsigned long long k = atomicAdd(P.claim_log, 1ULL) & 4095ULL;
  unsigned smid;
  asm("mov.u32 %0, %%smid;" : "=r"(smid));
  unsigned long long g;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
  unsigned long long* e = P.claim_log + 8 + 4 * k;
  e[0] = P.launch_id;
  e[1] = ((unsigned long long)kind << 56) | ((unsigned long long)smid << 40) |
         ((unsigned long long)blockIdx.x << 8) | (threadIdx.x >> 5);
  e[2] = v;
  e[3] = g;
}

// Work item -> (job, strip).  Multi-job launches claim strips strip-major
// across jobs (item_map) so that every pass of a level advances together and
// a warp never holds a strip whose producer is far behind; a strip's producer
// (strip s-1 of the same job) is always claimed earlier, so the persistent
// launch stays deadlock-free.
__device__ __forceinline__ int item_job(const PassParams& P, long long item, int* strip) {
  if (P.item_map) {
    const int2 m = P.item_map[item];
    *strip = m.y;
    return m.x;
  }
  int lo = 0, hi = P.njobs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (P.jobs[mid].item_base <= item) lo = mid;
    else hi = mid - 1;
  }
  *strip = (int)(item - P.jobs[lo].item_base);
  return lo;
}

__device__ __forceinline__ int vmaxadd(int a, int b, int c) { return __viaddmax_s32(a, b, c); }

__device__ __forceinline__ int imad(int a, int b, int c) {
  int d;
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

__device__ __forceinline__ uint32_t prmt(uint32_t lo, uint32_t hi, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(lo), "r"(hi), "r"(sel));
  return d;
}

__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(int32_t* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int ld_acquire_sys(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(int32_t* p, int v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int ld_relaxed_sys(const int32_t* p) {
  int v;
  asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void fence_acq_rel() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

__device__ __forceinline__ int ld_relaxed(const int32_t* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Running best for pruning: a pass's own word, or one word shared by the row
// slabs of a pass (swb_pass_desc.shared_best), possibly in a peer GPU's memory.
// GPU-scope accesses serve both: the value is a stale-only hint (any value once
// written is a real cell score), the reduction is atomic at the word's home L2
// whichever GPU issues it, and a branch on the scope here measured 1-2 % of a
// C2 pass (the hot kernels issue these every 32-column block).
__device__ __forceinline__ int load_best(const JobDev& J) { return ld_relaxed(J.prune_best); }
__device__ __forceinline__ void raise_best(const JobDev& J, int v) { atomicMax(J.prune_best, v); }

// Spin until *p >= need with exponential back-off: a waiting warp shares its
// SM sub-partition with a computing one, so it must not steal issue slots;
// the cap keeps the overshoot small against a producer that publishes every
// 32 steps (~2 us), which is what a chain along the diagonal waits on.
#ifndef SWB_WAIT_CAP_NS
#define SWB_WAIT_CAP_NS 256
#endif
constexpr unsigned kWaitCapNs = SWB_WAIT_CAP_NS;
constexpr unsigned kFarWaitCapNs = 2048;  // producer not started: it is strips away

// Chain-shaped passes (phase 2, Myers-Miller halves: a few strips in flight,
// each waiting on its producer at every block): poll with ld.acquire so the
// successful poll is the acquire (one L2 round trip instead of two), and keep
// the back-off short (the poller is alone on its sub-partition).
__device__ __forceinline__ int wait_acquire(const int32_t* p, int need) {
  int v = ld_acquire(p);
  unsigned ns = 0;
  while (v < need) {
    if (ns) __nanosleep(ns);
    ns = ns ? (ns < 64 ? ns * 2 : 64) : 16;
    v = ld_acquire(p);
  }
  return v;
}
__device__ __forceinline__ void wait_progress(const int32_t* p, int need, bool sys = false) {
  unsigned ns = 32;
  while ((sys ? ld_relaxed_sys(p) : ld_relaxed(p)) < need) {
    __nanosleep(ns);
    ns = ns < kWaitCapNs ? ns * 2 : kWaitCapNs;
  }
}

// ---- Tile bound maps ------------------------------------
// A pass may record, per 1024 x 1024 tile of the forward plane, an upper
// bound of its H values (every block contributes max(inputs) + W max_sub, an
// upper bound of every cell it covers), and a later pass may skip a block
// when even the best continuation the map allows cannot reach its target.
constexpr long long kBoundEnc = 1LL << 30;

__device__ __forceinline__ int bound_enc(long long v) {
  v += kBoundEnc;
  return v < 0 ? 0 : (v > 0x7fffffffLL ? 0x7fffffff : (int)v);
}

// forward tile range [lo, hi] of pass rows (or columns) [a, b], a <= b
__device__ __forceinline__ void tile_range(int base, int dir, int a, int b, int ntiles, int shift,
                                           int& lo, int& hi) {
  int fa = base + dir * a, fb = base + dir * b;
  if (fa > fb) {
    const int t = fa;
    fa = fb;
    fb = t;
  }
  lo = fa < 0 ? 0 : (fa >> shift);
  hi = fb < 0 ? 0 : (fb >> shift);
  if (lo > ntiles - 1) lo = ntiles - 1;
  if (hi > ntiles - 1) hi = ntiles - 1;
}

// Per-warp writer: holds the (at most two) column tiles the current block
// touches and flushes a tile with atomicMax once the blocks have moved past
// it, so a strip issues ~2 atomics per 1024 columns.  State is warp-uniform.
struct BoundWriter {
  int t0 = -1, t1 = -1;
  long long v0 = 0, v1 = 0;
  int rt_lo = 0, rt_hi = -1;
};

__device__ __forceinline__ void bw_flush(const JobDev& J, const BoundWriter& w, int t,
                                         long long v, int lane) {
  if (t < 0) return;
  const int rt = w.rt_lo + lane;
  if (rt <= w.rt_hi) atomicMax(J.bmap_out + SWB_IX((long long)rt * J.map_nc + SWB_IX(t, J.map_nc), (long long)J.map_nr * J.map_nc), bound_enc(v));
}

__device__ __forceinline__ void bw_add(const JobDev& J, BoundWriter& w, int ta, int tb,
                                       long long v, int lane) {
  if (w.t0 >= 0 && w.t0 != ta && w.t0 != tb) {
    bw_flush(J, w, w.t0, w.v0, lane);
    w.t0 = -1;
  }
  if (w.t1 >= 0 && w.t1 != ta && w.t1 != tb) {
    bw_flush(J, w, w.t1, w.v1, lane);
    w.t1 = -1;
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int t = k ? tb : ta;
    if (k && tb == ta) break;
    if (t == w.t0) w.v0 = w.v0 > v ? w.v0 : v;
    else if (t == w.t1) w.v1 = w.v1 > v ? w.v1 : v;
    else if (w.t0 < 0) { w.t0 = t; w.v0 = v; }
    else { w.t1 = t; w.v1 = v; }
  }
}

// A strip with a live column range sweeps only [c_lo, c_hi] (pass columns);
// record, per row tile, the hull of the forward columns its strips swept so a
// reader can tell "never written because fill" from "never visited".
__device__ __forceinline__ void live_record(const JobDev& J, int rt_lo, int rt_hi, int c_lo,
                                            int c_hi) {
  for (int rt = rt_lo; rt <= rt_hi; ++rt) {
    int4* e = J.bmap_live + SWB_IX(rt, J.map_nr);
    atomicMax(&e->z, 1);
    if (c_lo <= c_hi) {
      int fa = J.map_c0 + J.map_cdir * c_lo, fb = J.map_c0 + J.map_cdir * c_hi;
      if (fa > fb) {
        const int t = fa;
        fa = fb;
        fb = t;
      }
      atomicMax(&e->x, -(fa + 1));
      atomicMax(&e->y, fb);
    }
  }
}

// Decode one reverse-map tile for a reader: raw -1 is +inf unless the tile
// lies outside the swept interval of its row tile (then fill).
__device__ __forceinline__ bool map_unknown(const JobDev& J, int raw, int rt, int ct) {
  if (raw >= 0) return false;
  if (!J.rmap_live) return true;
  const int4 e = J.rmap_live[SWB_IX(rt, J.map_nr)];
  if (!e.z) return true;
  const int lo = -e.x - 1, hi = e.y;
  const int t0 = ct << J.map_shift, t1 = t0 + (1 << J.map_shift) - 1;
  return !(t1 < lo || t0 > hi);
}

__device__ __forceinline__ void bw_finish(const JobDev& J, BoundWriter& w, int lane) {
  bw_flush(J, w, w.t0, w.v0, lane);
  bw_flush(J, w, w.t1, w.v1, lane);
  w.t0 = w.t1 = -1;
}

// Per-warp reader with a one-entry cache (the tile set changes every ~32 blocks).
// Returns the decoded maximum over rows tiles [rt_lo, rt_hi] x columns tiles
// [ta, tb], or LLONG_MAX when any of them was never written.
struct BoundReader {
  int ta = -2, tb = -2;
  long long val = 0;
  int rt_lo = 0, rt_hi = -1;
};

__device__ __forceinline__ long long br_get(const JobDev& J, BoundReader& r, int ta, int tb,
                                            int lane) {
  if (ta == r.ta && tb == r.tb) return r.val;
  const int nct = tb - ta + 1;
  const int n = (r.rt_hi - r.rt_lo + 1) * nct;
  int m = -1;
  bool unknown = false;
  if (lane < n) {
    const int rt = r.rt_lo + lane / nct, ct = ta + lane % nct;
    m = __ldcg(J.bmap_in + SWB_IX((long long)SWB_IX(rt, J.map_nr) * J.map_nc + SWB_IX(ct, J.map_nc), (long long)J.map_nr * J.map_nc));
    if (m < 0) {
      unknown = !J.bin_rev || map_unknown(J, m, rt, ct);
      if (!unknown) m = 0;  // swept fill
    }
  }
  unknown = __any_sync(0xffffffffu, unknown);
  m = __reduce_max_sync(0xffffffffu, m);
  r.ta = ta;
  r.tb = tb;
  r.val = unknown ? LLONG_MAX : (long long)m - kBoundEnc;
  return r.val;
}

// Border values, engine.py:340-401.  I is a DP row, J a DP column.
__device__ __forceinline__ int left_h(int border, int I, int go, int ge) {
  switch (border) {
    case SWB_BORDER_LOCAL: return 0;
    case SWB_BORDER_RESTRICTED: return I == 0 ? 0 : SWB_NEG32;
    case SWB_BORDER_GLOBAL_FREE: return I == 0 ? 0 : -go - I * ge;
    case SWB_BORDER_GLOBAL_CONTINUE: return I == 0 ? SWB_NEG32 : -I * ge;
    default: return I == 0 ? SWB_NEG32 : -go - I * ge;  // charge
  }
}

__device__ __forceinline__ int top_h(int border, int J, int go, int ge) {
  switch (border) {
    case SWB_BORDER_LOCAL: return 0;
    case SWB_BORDER_RESTRICTED: return J == 0 ? 0 : SWB_NEG32;
    case SWB_BORDER_GLOBAL_FREE: return J == 0 ? 0 : -go - J * ge;
    default: return SWB_NEG32;  // continue / charge: origin blocked, no top row
  }
}

// Column range of strip s: all columns, or the band's admissible columns for
// the strip's rows (cells outside are skipped with the fill values, as the
// reference does for banded-out blocks, engine.py:225-231, :286-293).
template <int R>
__device__ __forceinline__ void strip_range(const JobDev& J, int s, int& cb, int& ce) {
  if (!J.has_band) {
    cb = 0;
    ce = J.n2;
    return;
  }
  const int r0 = s * 32 * R;
  int r1 = r0 + 32 * R - 1;
  if (r1 > J.n1 - 1) r1 = J.n1 - 1;
  long long lo = (long long)r0 - J.band_hi;
  long long hi = (long long)r1 - J.band_lo + 1;
  if (lo < 0) lo = 0;
  if (hi > J.n2) hi = J.n2;
  if (hi < lo) hi = lo;
  cb = (int)lo;
  ce = (int)hi;
}

// Static strip range from the tile maps (Myers-Miller halves):
// a cell can be on an optimal path of the subproblem only if its tile passes
// fwd + rev + range_offset >= target (phase-1 H bound + phase-2 reverse bound);
// the strip sweeps the hull of its useful tiles, everything else is fill.
// Deterministic in the maps, so producer and consumer agree on each range.
template <int R>
__device__ __forceinline__ void static_range(const JobDev& J, int s, int& cb, int& ce) {
  if (cb >= ce) return;
  const int lane = threadIdx.x & 31;
  const int r0 = s * 32 * R;
  const int r1 = (r0 + 32 * R < J.n1 ? r0 + 32 * R : J.n1) - 1;
  int rt_lo, rt_hi, ct_lo, ct_hi;
  tile_range(J.map_r0, J.map_rdir, r0, r1, J.map_nr, J.map_shift, rt_lo, rt_hi);
  tile_range(J.map_c0, J.map_cdir, cb, ce - 1, J.map_nc, J.map_shift, ct_lo, ct_hi);
  int fmin = 0x7fffffff, fmax = -1;
  for (int base = ct_lo; base <= ct_hi; base += 32) {
    const int ct = base + lane;
    bool useful = false;
    if (ct <= ct_hi) {
      for (int rt = rt_lo; rt <= rt_hi; ++rt) {
        const long long k = (long long)rt * J.map_nc + ct;
        const int a = __ldcg(J.rmap_fwd + SWB_IX(k, (long long)J.map_nr * J.map_nc));
        int b = __ldcg(J.rmap_rev + SWB_IX(k, (long long)J.map_nr * J.map_nc));
        if (b < 0 && !map_unknown(J, b, rt, ct)) b = 0;  // swept fill
        if (a < 0 || b < 0 ||
            (long long)a + b - 2 * kBoundEnc + J.range_offset >= (long long)J.prune_target)
          useful = true;
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, useful);
    if (m) {
      if (fmin == 0x7fffffff) fmin = base + __ffs(m) - 1;
      fmax = base + 31 - __clz(m);
    }
  }
  if (fmax < 0) {
    ce = cb;
    return;
  }
  const long long flo = (long long)fmin << J.map_shift, fhi = (((long long)fmax + 1) << J.map_shift) - 1;
  long long lo, hi;  // pass columns
  if (J.map_cdir > 0) {
    lo = flo - J.map_c0;
    hi = fhi - J.map_c0;
  } else {
    lo = J.map_c0 - fhi;
    hi = J.map_c0 - flo;
  }
  if (lo > cb) cb = (int)(lo < ce ? lo : ce);
  if (hi + 1 < ce) ce = (int)(hi + 1 > cb ? hi + 1 : cb);
}

struct WarpSmem {
  int4 ring[64];  // per column c: (top hm, top F, profile lo, profile hi) at [c & 63]
  int2 out[32];   // lane-31 outputs of the current 32-step block
};

// Chain chunks: a CTA runs 4 consecutive strips of one
// chain, and each producer strip also hands its bottom row to the consumer
// warp of the same CTA through shared memory: a 128-column ring plus the
// published column, read as a seqlock (a column older than prog - 96 may be
// overwritten by the block in flight and is read from the global row buffer,
// which keeps the full protocol of §3.2).  prog = INT_MAX: producer done.
struct ChainChan {
  int2 buf[128];
  volatile int prog;
  volatile int ahi;  // mirror of alive[s].y (0 = unknown)
};

// Best-cell tracking without a slow path: every cell's H is folded with its
// row into a 32-bit key (H - go - ge) * 32 + rank, rank = 31 - r (TRACK_MIN,
// smaller row wins ties) or r (TRACK_MAX, larger row wins), so one max over
// the keys of a column yields the best value and the tie-winning row, and a
// strict (MIN) / non-strict (MAX) comparison against the running key keeps
// the smallest (MIN) / largest (MAX) column of that row (kernels.py:73-84).
constexpr int kKeyClamp = -(1 << 25);

// BIG: substitutions from a shared-memory table (alphabets up to 32 codes or
// scores outside the int8 profile): the ring carries the
// column code's table row offset and every cell does one LDS instead of PRMT.
template <int R, bool LOCAL, int TRACK, bool FINAL, bool BIG>
__device__ __noinline__ void run_strip(const PassParams& P, const JobDev& Jg, int s,
                                       WarpSmem* sm, const uint32_t* __restrict__ tlo_s,
                                       const uint32_t* __restrict__ thi_s,
                                       ChainChan* cin = nullptr, ChainChan* cout = nullptr) {
  const int* __restrict__ tab_s = reinterpret_cast<const int*>(tlo_s);  // BIG: the table
  const JobDev J = Jg;
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    // diagnostics: who ran the strip, how often, when
    unsigned long long* d = P.strip_dbg + 8 * (J.item_base + s);
    d[4] = P.launch_id;  // which launch ran it
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    d[5] = ((unsigned long long)smid << 32) | ((unsigned long long)blockIdx.x << 8) | (threadIdx.x >> 5);
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    d[6] = g;
  }
  const int goe = P.goe, ge = P.ge;
  const int go = goe - ge;
  const int n1 = J.n1, n2 = J.n2;
  const int R0 = s * 32 * R;
  const int lrow0 = R0 + lane * R;
  int nvalid = n1 - lrow0;
  nvalid = nvalid < 0 ? 0 : (nvalid > R ? R : nvalid);
  const int fillm = J.fill_h - goe;

  int cb, ce;
  strip_range<R>(J, s, cb, ce);
  int cbp = 0, cep = 0;
  if (s > 0) strip_range<R>(J, s - 1, cbp, cep);
  if (J.rmap_fwd) {
    static_range<R>(J, s, cb, ce);
    if (s > 0) static_range<R>(J, s - 1, cbp, cep);
  }
  const int cb0 = cb;
  const int2* __restrict__ inbuf = J.buf[(s + 1) & 1];  // written by strip s-1
  int2* __restrict__ outbuf = J.buf[s & 1];
  int32_t* my_progress = J.progress + (long long)SWB_IX(s, J.nstrips) * kProgStride;
  const int32_t* up_progress = s > 0 ? J.progress + (long long)(s - 1) * kProgStride : nullptr;
  // multi-GPU row slab: strip 0 consumes the slab above (another GPU), the
  // last strip produces into the slab below (peer memory); sys-scope ordering
  const bool ext_in = (s == 0) && (J.ext_in != nullptr);
  const bool ext_out = (s == J.nstrips - 1) && (J.ext_out != nullptr);
  const bool first = (s == 0) && !ext_in;  // top border of the whole pass
  if (ext_in) {
    inbuf = J.ext_in;
    up_progress = J.ext_in_prog;
    cbp = 0;
    cep = n2;
  }
  if (ext_out) {
    outbuf = J.ext_out;
    my_progress = J.ext_out_prog;
  }

  // Live column range of a restricted pass.  Its left border
  // is -inf below row 0, so a strip's cells stay fill until the first live
  // output of its producer: the strip starts there instead of walking the
  // fill, and leaves as soon as it is back in fill state with no live input
  // ahead.  The producer's outputs outside [alo_p, ahi_p) are fill.
  const bool dyn = J.alive != nullptr && !ext_in && !ext_out;
  int alo_p = 0, ahi_p = 0x7fffffff;
  bool lo_set = false;
  if (dyn && first) ahi_p = 0;  // the restricted top border is -inf
  if (dyn && (J.live_mode & 1) && s > 0 && cb < ce) {
    // The producer stores its live lo before the progress release that covers
    // it and its live hi before its final release, so "no live output" is only
    // concluded after acquiring the final progress.
    // Most warps of a chain-shaped pass sit here, strips ahead of the front:
    // they poll relaxed (an acquire per poll invalidates L1 and, summed over
    // a thousand warps, loads L2 under the strips that do compute) and back
    // off further while their producer has not even started.
    unsigned ns = 32;
    for (;;) {
      const int p0 = ld_relaxed(up_progress);
      if (p0 >= cep || ld_relaxed(&J.alive[SWB_IX(s - 1, J.nstrips)].x) > 0) {
        const int p = ld_acquire(up_progress);
        const int ax = ld_relaxed(&J.alive[SWB_IX(s - 1, J.nstrips)].x);
        if (ax > 0) {
          alo_p = ax - 1;
          break;
        }
        if (p >= cep) {
          const int ay = ld_relaxed(&J.alive[SWB_IX(s - 1, J.nstrips)].y);
          alo_p = 0x7fffffff;
          if (ay > 0) ahi_p = ay - 1;
          break;
        }
      }
      __nanosleep(ns);
      const unsigned cap = (P.chain_wait && p0 == 0) ? kFarWaitCapNs : kWaitCapNs;
      ns = ns < cap ? ns * 2 : cap;
    }
    // each lane polled on its own: agree on one start (the values are final
    // once read, so the lanes agree anyway; the broadcast makes it explicit)
    alo_p = __shfl_sync(0xffffffffu, alo_p, 0);
    ahi_p = __reduce_min_sync(0xffffffffu, ahi_p);
    if (alo_p >= ahi_p || alo_p >= ce) cb = ce;
    else if (alo_p > cb) cb = alo_p;
  }

  if (cb >= ce) {
    if (dyn && J.bmap_live && J.bmap_out && lane == 0) {
      int rl, rh;
      tile_range(J.map_r0, J.map_rdir, R0, (R0 + 32 * R < n1 ? R0 + 32 * R : n1) - 1, J.map_nr, J.map_shift, rl, rh);
      live_record(J, rl, rh, 1, 0);  // covered, nothing swept
    }
    if (lane == 0) {
      if (dyn) J.alive[SWB_IX(s, J.nstrips)].y = cb + 1;  // no live output
      if (ext_out) st_release_sys(my_progress, 0x7fffffff);
      else st_release(my_progress, 0x7fffffff);
      J.strip_res[s] = make_int4(0, -1, -1, 0);
      P.strip_dbg[8 * (J.item_base + s) + 0] = ((unsigned long long)(unsigned)cb0 << 32) | (unsigned)cb;
      P.strip_dbg[8 * (J.item_base + s) + 1] = ((unsigned long long)(unsigned)ce << 32) | 0xffffffffu;
      P.strip_dbg[8 * (J.item_base + s) + 2] = 0;
      P.strip_dbg[8 * (J.item_base + s) + 3] = ((unsigned long long)(unsigned)alo_p << 32) | (unsigned)ahi_p;
      {
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        P.strip_dbg[8 * (J.item_base + s) + 7] = g;
      }
      if (cout) {
        cout->ahi = cb + 1;
        __threadfence_block();
        cout->prog = 0x7fffffff;
      }
    }
    return;
  }

  BoundWriter bw;
  BoundReader brd;
  if (J.bmap_out) {
    const int r_hi = (R0 + 32 * R < n1 ? R0 + 32 * R : n1) - 1;
    tile_range(J.map_r0, J.map_rdir, R0, r_hi, J.map_nr, J.map_shift, bw.rt_lo, bw.rt_hi);
  }
  if (J.bmap_in) tile_range(J.map_r0, J.map_rdir, R0 - 1, R0 + 32 * R, J.map_nr, J.map_shift, brd.rt_lo, brd.rt_hi);

  // Row codes -> PRMT selectors (byte a, sign replicated into bytes 1..3).
  uint32_t sel[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = lrow0 + r;
    if (BIG) {
      sel[r] = (i < n1) ? (uint32_t)J.rows[SWB_IX((long long)i * J.rstep, (long long)n1 * J.rstep)] : 32u;  // 32: pad, entry 0
      continue;
    }
    uint32_t a = (i < n1) ? (uint32_t)J.rows[SWB_IX((long long)i * J.rstep, (long long)n1 * J.rstep)] : (uint32_t)kPadCode;
    sel[r] = a | ((a | 8u) << 4) | ((a | 8u) << 8) | ((a | 8u) << 12);
  }

  // Left state at column cb (E holds the value for the column about to run).
  int H[R], H2[R], E[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    H2[r] = 0;
    const int hl = (cb == 0) ? left_h(J.border, J.row_offset + lrow0 + r + 1, go, ge) - goe : fillm;
    H[r] = hl;
    E[r] = vmaxadd(SWB_NEG32, -ge, hl);
  }
  // Diagonal for row 0 at column cb: H(lrow0 - 1, cb - 1).
  int diag;
  if (cb == 0) {
    diag = left_h(J.border, J.row_offset + lrow0, go, ge) - goe;
  } else if (lane != 0) {
    diag = fillm;
  } else if (first) {
    diag = top_h(J.border, cb, go, ge) - goe;
  } else if (cb - 1 >= cbp && cb - 1 < cep && cb - 1 >= alo_p && cb - 1 < ahi_p) {
    wait_progress(up_progress, cb, ext_in);
    if (ext_in) (void)ld_acquire_sys(up_progress);
    else fence_acq_rel();
    diag = __ldcg(inbuf + SWB_IX(cb - 1, n2)).x;
  } else {
    diag = fillm;
  }

  int bkey = (TRACK == kTrackMin) ? (-goe) * 32 + 31 : INT32_MIN;
  // 32 read from the launch parameters so the key multiply-add stays an IMAD
  // on the FMA pipe instead of a LEA on the (saturated) integer ALU pipe.
  const int k32 = P.key_mul;
  int bj = -1;

  int rstar = -1, lstar = -1;
  if (FINAL) {
    const int off = n1 - 1 - R0;
    lstar = off / R;
    rstar = off % R;
  }

  int out_hm = fillm, out_f = SWB_NEG32;
  int known_prog = 0, prune_seen = 0, published = 0;
  int code_next = (cb + lane < ce) ? (int)J.cols[SWB_IX((long long)(cb + lane) * J.cstep, (long long)n2 * J.cstep)] : 0;
  long long pruned_blocks = 0, exec_blocks = 0;
  long long wait_cycles = 0;
  const long long t_strip0 = clock64();
  unsigned long long g0, gw = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  const int s_end = ce + 31;

  // One column of this lane's R rows.  GUARD: ramp blocks where some lanes
  // are outside [cb, ce).
  auto step = [&](const int k, const int step_no, const bool guard, int (&Hin)[R], int (&Hout)[R],
                  auto trk_tag) {
    constexpr bool TRK = decltype(trk_tag)::value && (TRACK != kTrackNone);
    const int col = step_no - lane;
    const int4 rv = sm->ring[col & 63];
    int up_h = __shfl_up_sync(0xffffffffu, out_hm, 1);
    int up_f = __shfl_up_sync(0xffffffffu, out_f, 1);
    if (lane == 0) {
      up_h = rv.x;
      up_f = rv.y;
    }
    if (!guard || (col >= cb && col < ce)) {
      const uint32_t tl = (uint32_t)rv.z, th = (uint32_t)rv.w;
      int d = diag;
      diag = up_h;
      int fv = up_f;
      int hab = up_h;
      int cm = INT32_MIN, kprev = INT32_MIN;
      int fh = 0, ff = 0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int sv = BIG ? tab_s[SWB_IX(rv.z + (int)sel[r], 32 * 33)] : (int)prmt(tl, th, sel[r]);
        const int h2 = LOCAL ? __viaddmax_s32_relu(d, sv, E[r]) : __viaddmax_s32(d, sv, E[r]);
        fv = vmaxadd(fv, -ge, hab);
        const int h2m = h2 - goe;
        const int hm = vmaxadd(fv, -goe, h2m);
        E[r] = vmaxadd(E[r], -ge, hm);
        d = Hin[r];
        Hout[r] = hm;
        hab = h2m;
        if (TRK) {
          const int rank = (TRACK == kTrackMin) ? 31 - r : r;
          // padding rows (i >= n1, last strip only) need no guard: their
          // values are strictly below a real cell already seen (DESIGN.md
          // §3.5); a lane whose best decodes to a padding row is dropped.
          const int key = imad((LOCAL ? hm : (hm > kKeyClamp ? hm : kKeyClamp)), k32, rank);
          if (r & 1) cm = __vimax3_s32(cm, kprev, key);
          else if (r == R - 1) cm = cm > key ? cm : key;
          kprev = key;
        }
        if (FINAL && r == rstar) {
          fh = hm;
          ff = fv;
        }
      }
      out_hm = Hout[R - 1];
      out_f = fv;
      if (TRK && TRACK == kTrackMin) {
        if (cm > bkey) {
          bkey = cm;
          bj = col;
        }
      } else if (TRK && TRACK == kTrackMax) {
        if (cm >= bkey) {
          bkey = cm;
          bj = col;
        }
      }
      if (FINAL && lane == lstar) {
        J.fin_h[SWB_IX(col, n2)] = fh + goe;
        J.fin_f[SWB_IX(col, n2)] = ff;
      }
      if (lane == 31) sm->out[k] = make_int2(out_hm, out_f);
    } else {
      // lane outside [cb, ce) in a ramp block: carry the state across
#pragma unroll
      for (int r = 0; r < R; ++r) Hout[r] = Hin[r];
    }
  };

  bool prev_skipped = false, exited = false;
  int lazy_pub = 0;
  int exit_col = 0;
  int known_prog2 = 0;  // progress of strip s-2 (previous writer of our buffer)
  for (int s0 = cb; s0 < s_end; s0 += 32) {
    // early exit (restricted passes): fill state and no live input at or
    // after column s0 - 1 (lane 0's next diagonal): every later cell is fill
    if (dyn && (J.live_mode & 2) && prev_skipped && ahi_p < s0) {
      exited = true;
      exit_col = s0;
      if (lane == 0) {
        J.alive[SWB_IX(s, J.nstrips)].y = (s0 - 31 > cb ? s0 - 31 : cb) + 1;
        if (cout) cout->ahi = (s0 - 31 > cb ? s0 - 31 : cb) + 1;
      }
      break;
    }
    // (1) stage lane-0 inputs and profile words for columns [s0, s0 + 32).
    // The column codes were prefetched one block ahead; the producer's
    // progress is polled only when the last observed value does not cover
    // this block, and acquired with one ld.acquire.
    // running best: every lane loads it (stale-only, any lane's value is
    // sound); the skip / tracking decisions below are made warp-uniform by votes
    if (LOCAL && J.prune == 1) prune_seen = load_best(J);
    {
      const int c = s0 + lane;
      const int code = code_next;
      {
        const int cn = c + 32;
        code_next = (cn < ce) ? (int)J.cols[SWB_IX((long long)cn * J.cstep, (long long)n2 * J.cstep)] : 0;
      }
      if (!first && s0 < cep && s0 + 32 > cbp) {
        const int need = (s0 + 32 < cep) ? s0 + 32 : cep;
        if (known_prog < need && cin) {
          unsigned long long a0, a1;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a0));
          int v = cin->prog;
          while (v < need) {
            __nanosleep(20);
            v = cin->prog;
          }
          __threadfence_block();
          known_prog = v;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a1));
          gw += a1 - a0;
          if (dyn && ahi_p == 0x7fffffff) {
            const int ay = cin->ahi;
            if (ay > 0) ahi_p = ay - 1;
          }
        } else if (known_prog < need && P.chain_wait && !ext_in) {
          unsigned long long a0, a1;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a0));
          known_prog = wait_acquire(up_progress, need);
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a1));
          gw += a1 - a0;
          if (dyn && ahi_p == 0x7fffffff) {
            const int ay = ld_relaxed(&J.alive[SWB_IX(s - 1, J.nstrips)].y);
            if (ay > 0) ahi_p = ay - 1;
          }
        } else if (known_prog < need) {
          // one acquiring load when the producer is already ahead; poll
          // relaxed only when it is not
          known_prog = ext_in ? ld_acquire_sys(up_progress) : ld_acquire(up_progress);
          if (known_prog < need) {
            const long long tw = clock64();
            unsigned long long a0, a1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a0));
            wait_progress(up_progress, need, ext_in);
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a1));
            gw += a1 - a0;
            wait_cycles += clock64() - tw;
            known_prog = ext_in ? ld_acquire_sys(up_progress) : ld_acquire(up_progress);
          }
          if (dyn && ahi_p == 0x7fffffff) {
            const int ay = ld_relaxed(&J.alive[SWB_IX(s - 1, J.nstrips)].y);
            if (ay > 0) ahi_p = ay - 1;
          }
        }
      }
      if (c < ce) {
        int th, tf;
        if (first) {
          th = top_h(J.border, c + 1, go, ge) - goe;
          tf = SWB_NEG32;
        } else if (c >= cbp && c < cep && c >= alo_p && c < ahi_p) {
          int2 v;
          if (cin) {
            v = cin->buf[c & 127];
            __threadfence_block();
            if (c < cin->prog - 96) {  // slot may have been reused: global row buffer
              if (ld_acquire(up_progress) <= c) wait_acquire(up_progress, c + 1);
              v = __ldcg(inbuf + SWB_IX(c, n2));
            }
          } else {
            v = __ldcg(inbuf + SWB_IX(c, n2));
          }
          th = v.x;
          tf = v.y;
        } else {
          th = fillm;
          tf = SWB_NEG32;
        }
        if (BIG) sm->ring[c & 63] = make_int4(th, tf, (int)SWB_IX(code, 32) * 33, 0);
        else sm->ring[c & 63] = make_int4(th, tf, (int)tlo_s[SWB_IX(code, 8)], (int)thi_s[SWB_IX(code, 8)]);
      }
      // Everything that steers control flow around the warp-synchronous steps
      // must be warp-uniform: every lane loaded the running best and the
      // producer's live end on its own, at slightly different times, and a
      // lane that skipped or left early while the others ran the block would
      // pair its shuffles with theirs (shfl.sync matches any shfl.sync of the
      // same mask).  Lane 0's running best is as stale-safe as any; a known
      // live end is final, so the minimum over lanes adopts it.
      if (dyn) ahi_p = __reduce_min_sync(0xffffffffu, ahi_p);
      __syncwarp();  // ring stores visible to the steps
    }
    const bool steady = (s0 - 31 >= cb) && (s0 + 32 <= ce);
    // A restricted pass may also skip its ramp blocks: lanes that have not
    // reached cb yet hold -inf state (left border below row 0), so resetting
    // them to fill changes nothing; other border families keep finite left
    // states there and prune steady blocks only.
    const bool prunable = steady || J.border == SWB_BORDER_RESTRICTED;

    // (2) pruning: skip the whole 32-step block when no path through it can
    // matter.  kind 1 (phase 1): cannot reach the running best
    // (phase1.py:24-41, :55-59; strict); kind 2 (restricted search): cannot
    // reach the known target anywhere; kind 3 (Myers-Miller halves): cannot be
    // on a path that reaches the subproblem's end corner with the expected
    // score.  Skipped cells get the fill of engine.py:286-293.
    bool skip = false;
    // Tracking is needed only where a cell could still reach the running best
    // (a cell below it can never be the final answer): most blocks of a
    // homologous pair run the untracked loop (no keys, no column max).
    bool track_block = true;
    // input maximum of the block (state, values in flight, staged top row):
    // with the band's and pruning's fills it bounds every cell of the block
    // from above once max_sub per column is added
    long long inm = 0;
    if ((J.prune && prunable) || J.bmap_out || (J.bmap_in && prunable)) {
      int m = out_hm > diag ? out_hm : diag;
#pragma unroll
      for (int r = 0; r < R; ++r) m = m > H[r] ? m : H[r];
      if (s0 + lane < ce) {
        const int tv = sm->ring[(s0 + lane) & 63].x;
        m = m > tv ? m : tv;
      }
      m = __reduce_max_sync(0xffffffffu, m);
      inm = (long long)m + goe;
    }
    if (J.prune && prunable) {
      const int rem_r = n1 - R0 + J.rows_after;
      const int rem_c = n2 - (s0 - 31);
      const long long ms = P.max_sub;
      if (J.prune == 1) {
        const long long bound = (inm > 0 ? inm : 0) + ms * (long long)(rem_r < rem_c ? rem_r : rem_c);
        // votes keep both decisions warp-uniform (each lane's best is sound)
        skip = __any_sync(0xffffffffu, bound < (long long)prune_seen);
        // a path inside the 63-column-wide skewed block gains <= 63 * max_sub
        track_block = __any_sync(0xffffffffu,
                                 (inm > 0 ? inm : 0) + 63LL * ms >= (long long)prune_seen);
      } else if (J.prune == 2) {
        const long long bound = inm + ms * (long long)(rem_r < rem_c ? rem_r : rem_c);
        skip = bound < (long long)J.prune_target;
        // the pass maximum equals the target (phase 2): a block none of whose
        // cells can reach it cannot hold the answer, so it runs untracked
        track_block = inm + 63LL * ms >= (long long)J.prune_target;
      } else {
        int i_hi = R0 + 32 * R;
        if (i_hi > n1) i_hi = n1;
        const long long di_max = (long long)J.corner_i - (R0 + 1);
        const long long dj_max = (long long)J.corner_j - (s0 - 31 + 1);
        const long long off = (long long)J.corner_i - J.corner_j;
        const long long dlo = off - ((long long)(i_hi - 1) - (s0 - 31));
        const long long dhi = off - ((long long)R0 - (s0 + 31));
        long long k = 0;
        if (dlo > 0) k = dlo;
        else if (dhi < 0) k = -dhi;
        const long long ub = ms * (di_max < dj_max ? di_max : dj_max) - (k > 0 ? go + (long long)ge * k : 0);
        // + 2 go + ge: a completion may continue an open gap, and the two
        // halves of a gap join each charge one opening fee
        skip = inm + ub + 2LL * go + ge < (long long)J.prune_target;
      }
    }
    // tile bound maps: skip when even the best continuation
    // the map allows cannot reach the target; record this block's bound
    if (J.bmap_in && prunable && !skip) {
      int ta, tb;
      tile_range(J.map_c0, J.map_cdir, s0 - 32, s0 + 32, J.map_nc, J.map_shift, ta, tb);
      const long long mx = br_get(J, brd, ta, tb, lane);
      if (mx != LLONG_MAX &&
          inm + 63LL * P.max_sub + mx + J.bound_offset < (long long)J.prune_target)
        skip = true;
    }
    if (J.bmap_out) {
      const int lo = s0 - 31 > cb ? s0 - 31 : cb;
      const int hi = s0 + 31 < ce - 1 ? s0 + 31 : ce - 1;
      if (lo <= hi) {
        int ta, tb;
        tile_range(J.map_c0, J.map_cdir, lo, hi, J.map_nc, J.map_shift, ta, tb);
        bw_add(J, bw, ta, tb, (LOCAL && inm < 0 ? 0 : inm) + 63LL * P.max_sub, lane);
      }
    }

    if (skip) {
      ++pruned_blocks;
      const int negE = vmaxadd(SWB_NEG32, -ge, fillm);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        H[r] = fillm;
        E[r] = negE;
      }
      diag = (lane == 0) ? sm->ring[(s0 + 31) & 63].x : fillm;
      out_hm = fillm;
      out_f = SWB_NEG32;
      sm->out[lane] = make_int2(fillm, SWB_NEG32);
      __syncwarp();
    } else {
      ++exec_blocks;
      // (3) 32 steps.
      // two columns per iteration with ping-pong H registers: the old H of
      // a row (the next row's diagonal) survives without register moves
      using T1 = std::integral_constant<bool, true>;
      using T0 = std::integral_constant<bool, false>;
      if (steady && !track_block) {
#pragma unroll 1
        for (int k = 0; k < 32; k += 2) {
          step(k, s0 + k, false, H, H2, T0{});
          step(k + 1, s0 + k + 1, false, H2, H, T0{});
        }
      } else if (steady) {
#pragma unroll 1
        for (int k = 0; k < 32; k += 2) {
          step(k, s0 + k, false, H, H2, T1{});
          step(k + 1, s0 + k + 1, false, H2, H, T1{});
        }
      } else if (!track_block) {
#pragma unroll 1
        for (int k = 0; k < 32; k += 2) {
          step(k, s0 + k, true, H, H2, T0{});
          step(k + 1, s0 + k + 1, true, H2, H, T0{});
        }
      } else {
#pragma unroll 1
        for (int k = 0; k < 32; k += 2) {
          step(k, s0 + k, true, H, H2, T1{});
          step(k + 1, s0 + k + 1, true, H2, H, T1{});
        }
      }
      __syncwarp();
    }

    prev_skipped = skip;

    // (4) flush lane-31 outputs for columns [s0 - 31, s0 + 1) and publish.
    {
      const int c = s0 - 31 + lane;
      // Buffer s & 1 was written by strip s-2.  Strip s-1 normally consumed
      // those columns before we could compute them, but a strip that skips
      // columns (empty or narrowed range, late start, early exit) does not,
      // so make sure strip s-2 is done with them before overwriting.
      if (s >= 2 && !ext_out) {
        const int hi = s0 + 1 < ce ? s0 + 1 : ce;
        if (hi > cb && known_prog2 < hi) {
          if (P.chain_wait) {
            known_prog2 = wait_acquire(J.progress + (long long)SWB_IX(s - 2, J.nstrips) * kProgStride, hi);
          } else {
            const int32_t* p2 = J.progress + (long long)(s - 2) * kProgStride;
            if (ld_relaxed(p2) < hi) wait_progress(p2, hi);
            known_prog2 = ld_acquire(p2);
          }
        }
      }
      if (c >= cb && c < ce) __stcg(outbuf + SWB_IX(c, n2), sm->out[lane]);
      if (dyn && !lo_set) {
        // first live output: consumers start there (ordered by the release below)
        const unsigned m = __ballot_sync(0xffffffffu, c >= cb && c < ce &&
                                                          sm->out[lane].x > -(1 << 29));
        if (m) {
          lo_set = true;
          if (lane == 0) J.alive[SWB_IX(s, J.nstrips)].x = s0 - 31 + __ffs(m);  // (lo + 1)
        }
      }
      if (ext_out) __threadfence_system();
      else if (P.proto == 0) __threadfence();
      else if (P.proto == 1) fence_acq_rel();
      __syncwarp();
      if (lane == 0) {
        int pub = s0 + 1;
        if (pub > ce) pub = ce;
        // a producer whose consumer reads the shared-memory ring releases the
        // global progress every 4th block only (its readers: the consumer's
        // start and ring fallback, strip s+2's buffer check)
        if (pub >= cb && (!cout || pub >= ce || (++lazy_pub & 3) == 0)) {
          if (ext_out) st_release_sys(my_progress, pub);
          else st_release(my_progress, pub);
        }
      }
      if (cout) {
        if (c >= cb && c < ce) cout->buf[c & 127] = sm->out[lane];
        __syncwarp();
        __threadfence_block();
        int pub = s0 + 1;
        if (pub > ce) pub = ce;
        if (lane == 0 && pub >= cb) cout->prog = pub;
      }
    }

    // (5) running best for pruning (monotone, never ahead of the truth).
    if (LOCAL && J.prune == 1 && TRACK == kTrackMin) {
      // publish only improvements and only above what is already known:
      // one contended atomic per warp and block would cost every warp a
      // global round trip on the critical path
      const int bm = __reduce_max_sync(0xffffffffu, bkey >> 5);
      if (bm > -goe && bm + goe > published && bm + goe > prune_seen) {
        published = bm + goe;
        if (lane == 0) raise_best(J, published);
      }
    }
  }
  if (J.bmap_out) bw_finish(J, bw, lane);
  if (dyn && J.bmap_live && J.bmap_out && lane == 0)
    live_record(J, bw.rt_lo, bw.rt_hi, cb, exited ? exit_col - 1 : ce - 1);
  // done: consumers need columns < their own end, strip s+2 needs "finished"
  if (lane == 0) {
    if (dyn && !exited) J.alive[SWB_IX(s, J.nstrips)].y = ce + 1;
    if (ext_out) st_release_sys(my_progress, 0x7fffffff);
    else st_release(my_progress, 0x7fffffff);
    if (cout) {
      if (dyn && !exited) cout->ahi = ce + 1;
      __threadfence_block();
      cout->prog = 0x7fffffff;
    }
  }

  // Strip result: decode the key, then warp reduction with the mode's tie
  // rule (engine.py:247-259).
  if (TRACK != kTrackNone) {
    int b = bkey >> 5;
    const int rk = bkey & 31;
    int ii = (bj >= 0) ? lrow0 + ((TRACK == kTrackMin) ? 31 - rk : rk) : -1;
    int jj = bj;
    if (ii >= n1) ii = jj = -1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int ob = __shfl_down_sync(0xffffffffu, b, o);
      const int oi = __shfl_down_sync(0xffffffffu, ii, o);
      const int oj = __shfl_down_sync(0xffffffffu, jj, o);
      bool take;
      if (oi < 0) take = false;
      else if (ii < 0) take = true;
      else if (TRACK == kTrackMin)
        take = ob > b || (ob == b && (oi < ii || (oi == ii && oj < jj)));
      else
        take = ob > b || (ob == b && (oi > ii || (oi == ii && oj > jj)));
      if (take) {
        b = ob;
        ii = oi;
        jj = oj;
      }
    }
    if (lane == 0) J.strip_res[SWB_IX(s, J.nstrips)] = make_int4(b, ii, jj, ii >= 0 ? 1 : 0);
  } else if (lane == 0) {
    J.strip_res[s] = make_int4(0, -1, -1, 0);
  }
  if (lane == 0) {
    int rows_here = n1 - R0;
    if (rows_here > 32 * R) rows_here = 32 * R;
    const long long cells =
        (long long)(ce - cb) * rows_here - pruned_blocks * 32LL * rows_here;
    atomicAdd(&J.counters[0], (unsigned long long)(cells > 0 ? cells : 0));
    atomicAdd(&J.counters[1], (unsigned long long)exec_blocks);
    atomicAdd(&J.counters[2], (unsigned long long)pruned_blocks);
    atomicAdd(&J.counters[3], (unsigned long long)wait_cycles);
    atomicAdd(&J.counters[4], (unsigned long long)(clock64() - t_strip0));
    unsigned long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    J.strip_times[3 * s + 0] = g0;
    J.strip_times[3 * s + 1] = g1;
    P.strip_dbg[8 * (J.item_base + s) + 0] = ((unsigned long long)(unsigned)cb0 << 32) | (unsigned)cb;
    P.strip_dbg[8 * (J.item_base + s) + 1] = ((unsigned long long)(unsigned)ce << 32) | (unsigned)(exited ? exit_col : -1);
    P.strip_dbg[8 * (J.item_base + s) + 2] = ((unsigned long long)exec_blocks << 32) | (unsigned long long)pruned_blocks;
    P.strip_dbg[8 * (J.item_base + s) + 3] = ((unsigned long long)(unsigned)alo_p << 32) | (unsigned)ahi_p;
    P.strip_dbg[8 * (J.item_base + s) + 7] = g1;
    // proto 9 (diagnostics): the strip's final column range instead of the wait time
    J.strip_times[3 * s + 2] =
        P.proto == 9 ? (((unsigned long long)(unsigned)cb << 32) | (unsigned)ce) : gw;
  }
}

template <int R, bool LOCAL, int TRACK, bool BIG>
__device__ __forceinline__ void run_item(const PassParams& P, long long item, WarpSmem* sm,
                                         const uint32_t* tlo_s, const uint32_t* thi_s) {
  int s = 0;
  const JobDev& J = P.jobs[item_job(P, item, &s)];
  if (J.want_final && s == J.nstrips - 1)
    run_strip<R, LOCAL, TRACK, true, BIG>(P, J, s, sm, tlo_s, thi_s);
  else
    run_strip<R, LOCAL, TRACK, false, BIG>(P, J, s, sm, tlo_s, thi_s);
}

template <int R, bool LOCAL, int TRACK, bool BIG>
__device__ __forceinline__ void run_chunk_strip(const PassParams& P, const JobDev& J, int s,
                                                WarpSmem* sm, const uint32_t* tlo_s,
                                                const uint32_t* thi_s, ChainChan* cin,
                                                ChainChan* cout) {
  if (J.want_final && s == J.nstrips - 1)
    run_strip<R, LOCAL, TRACK, true, BIG>(P, J, s, sm, tlo_s, thi_s, cin, cout);
  else
    run_strip<R, LOCAL, TRACK, false, BIG>(P, J, s, sm, tlo_s, thi_s, cin, cout);
}

// Persistent launch.  Two claiming modes:
//  * P.group == 0: every warp claims one strip at a time (many small passes,
//    e.g. a Myers-Miller level).
//  * P.group  > 0: one CTA per SM with 4*w warps (w per SM sub-partition)
//    claims 4*w consecutive strips at once; warp i runs on sub-partition i % 4
//    and takes strip base + (i % 4) * w + i / 4, so the w warps sharing a
//    sub-partition hold ADJACENT strips of the chain: when one waits for its
//    producer the other (its producer or consumer) gets the issue slots, and
//    every sub-partition carries the same load.
template <int R, bool LOCAL, int TRACK, bool BIG = false>
__global__ void __launch_bounds__(256) pass_kernel(const PassParams P) {
  __shared__ WarpSmem wsm[8];
  __shared__ uint32_t tlo_s[BIG ? 32 * 33 : 8], thi_s[8];
  __shared__ long long base_s;
  if (BIG) {
    for (int x = threadIdx.x; x < 32 * 33; x += blockDim.x) tlo_s[x] = (uint32_t)P.tab[x];
  } else if (threadIdx.x < 8) {
    tlo_s[threadIdx.x] = P.tlo[threadIdx.x];
    thi_s[threadIdx.x] = P.thi[threadIdx.x];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  WarpSmem* sm = &wsm[warp];
  if (P.chunk > 0) {
    // chain chunks: 32 x P.chunk threads (4 or 8 warps), warp w runs strip
    // first + w of the claimed chunk
    __shared__ ChainChan chan[8];
    for (;;) {
      if (threadIdx.x == 0) base_s = (long long)atomicAdd(P.claim, 1ULL);
      if (lane == 0) {
        chan[warp].prog = 0;
        chan[warp].ahi = 0;
      }
      __syncthreads();
      const long long c = base_s;
      if (c >= P.total_items) break;
      const int2 m = P.item_map[c];
      const JobDev& J = P.jobs[m.x];
      const int s = m.y + warp;
      if (s < J.nstrips) {
        ChainChan* cin = (warp > 0) ? &chan[warp - 1] : nullptr;
        ChainChan* cout = (warp < P.chunk - 1 && s + 1 < J.nstrips) ? &chan[warp] : nullptr;
        run_chunk_strip<R, LOCAL, TRACK, BIG>(P, J, s, sm, tlo_s, thi_s, cin, cout);
      }
      __syncthreads();
    }
    return;
  }
  if (P.group > 0) {
    const int w = (int)(blockDim.x >> 7);
    for (;;) {
      if (threadIdx.x == 0) base_s = (long long)atomicAdd(P.claim, (unsigned long long)P.group);
      __syncthreads();
      const long long base = base_s;
      __syncthreads();
      if (base >= P.total_items) break;
      long long item = base + (warp & 3) * w + (warp >> 2);
      if (P.mirror) {
        // single round, two warps per sub-partition: sub-partition p holds
        // strips p and total-1-p.  The top strips (never pruned, on the
        // critical path) share issue slots with bottom strips, which are idle
        // during the pipeline ramp and mostly pruned.
        const long long p = base / 2 + (warp & 3);
        const long long q = P.total_items - 1 - p;
        item = (warp >> 2) == 0 ? (p <= q ? p : P.total_items) : (p < q ? q : P.total_items);
      }
      if (item < P.total_items) run_item<R, LOCAL, TRACK, BIG>(P, item, sm, tlo_s, thi_s);
    }
    return;
  }
  if (P.claim_log && lane == 0) {
    claim_log(P, 2, (unsigned long long)ld_relaxed((const int32_t*)P.claim));
    claim_log(P, 3, (unsigned long long)(unsigned)ld_relaxed(P.jobs[0].progress));
  }
  for (;;) {
    long long item = 0;
    if (lane == 0) item = (long long)atomicAdd(P.claim, 1ULL);
    if (lane == 0) claim_log(P, 1, (unsigned long long)item);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= P.total_items) break;
    run_item<R, LOCAL, TRACK, BIG>(P, item, sm, tlo_s, thi_s);
  }
}

}  // namespace swb
