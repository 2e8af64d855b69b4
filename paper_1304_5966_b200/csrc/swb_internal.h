// Internal declarations shared by the libswb.so translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/swb.h"

// int32 sentinel for minus infinity on the device (the reference uses
// -(2**61) in int64, kernels.py:14).  Drift from the sentinel is bounded by
// swb_check_range(): sentinel-derived values stay below SWB_NEG_REPORT and
// real values stay above it.
#define SWB_NEG32 (-(1 << 30))

struct swb_seq {
  uint8_t* fwd = nullptr;  // device, n codes
  uint8_t* rev = nullptr;  // device, reversed copy
  int64_t n = 0;
  int64_t cap = 0;  // allocated bytes of fwd / rev
  bool live = false;
  bool has_code4 = false;  // holds code 4 (the DNA wildcard 'N' of the default alphabet)
};

// A grow-only device scratch buffer.
struct swb_buf {
  void* p = nullptr;
  size_t cap = 0;
};

struct swb_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::mutex mu;
  std::vector<swb_seq> seqs;
  int sms = 0;
  double last_kernel_ms = 0.0;
  int64_t launches = 0;
  int max_ctas_per_sm = 0;  // 0 = occupancy limit
  int force_R = 0;          // 0 = pick rows-per-lane from the pass height
  long long dbg_wait_cycles = 0, dbg_strip_cycles = 0;
  int proto = 2;
  int claim_mode = 0;
  bool trace = false;
  int mm_prune = 1;
  int job_major = 0;   // 1: claim strips job by job (no strip-major item map)
  int x2_enabled = 1;  // packed 16x2 kernel for eligible phase-1 passes
  int x2_R = 0;  // force the packed kernel's rows per lane (diagnostics)
  std::vector<unsigned long long> dbg_times;
  std::vector<long long> dbg_strips;  // last launch: 8 words per strip (swb_debug_strips)
  // tile bound maps of one sequence pair
  int bmap_seq1 = -1, bmap_seq2 = -1;
  int bmap_nr = 0, bmap_nc = 0;
  int bmap_shift = 10;          // tile edge 2^bmap_shift of the current maps
  int map_shift = 10;           // option map_tile_log2: edge of the next maps
  int bmaps_on = 1;             // option "bound_maps": 0 disables reads and writes
  int live_ranges = 3;  // restricted passes: bit 0 late start, bit 1 early exit
  int claim_log_on = 0; // option claim_log: record claims in a device ring (swb_debug_claims)
  int chain_chunk = 8;  // strips per CTA of chain-shaped passes (4 or 8)
  int min_R = 0;        // smallest rows-per-lane the shape model may pick (diagnostics)
  int wide_log2 = 28;   // passes with dynamic range >= 2^wide_log2 run on the int64 kernel
  int watchdog_ms = 0;  // > 0: report a pass launch still running after this long
  int live_big = 3;     // live_ranges bits kept for shared-table (large alphabet) passes
  int x2_blk = 0;       // packed kernel steps per block: 0 auto (rounds), 32, 64
  int last_x2_blk = 0;  // block length of the last packed launch (diagnostics)
  int p2_R = 8;         // rows per lane of bound-pruned restricted passes (phase 2)
  int mm_R = 8;         // rows per lane of range-limited Myers-Miller passes
  int mm_static = 1;    // static strip ranges for Myers-Miller halves
  int mm_dyn = 1;       // per-block tile-bound skipping in Myers-Miller halves
  int chain_wait = 1;
  int chain_cta = 1;    // chain-shaped passes in chunks of 4 strips per CTA (shared-memory handoff)   // acquire polling with short back-off in chain-shaped passes
  swb_buf bmap_fwd, bmap_rev, bmap_live;
  // scratch
  swb_buf dbg_buf, claim_log, wide_buf;      // per-strip diagnostics of the last launch
  swb_buf pass_finals;  // final rows of swb_pass calls (whole call, all launch groups)
  swb_buf jobs, rowbuf, progress, results, finals, misc, host_pinned, flush;
  cudaEvent_t tev0 = nullptr, tev1 = nullptr;
};

void swb_set_error(const char* fmt, ...);
int swb_fail(int code, const char* fmt, ...);
void* swb_scratch(swb_buf& b, size_t bytes);  // device; nullptr on failure
void* swb_scratch_host(swb_buf& b, size_t bytes);

#define SWB_CUDA(call)                                                           \
  do {                                                                           \
    cudaError_t _e = (call);                                                     \
    if (_e != cudaSuccess)                                                       \
      return swb_fail(SWB_ECUDA, "%s failed: %s (%s:%d)", #call,                 \
                      cudaGetErrorString(_e), __FILE__, __LINE__);               \
  } while (0)

#define SWB_API_BEGIN(ctx)                                                       \
  if ((ctx) == nullptr) return swb_fail(SWB_EINVAL, "null context");             \
  std::lock_guard<std::mutex> _swb_lock((ctx)->mu);                              \
  {                                                                              \
    cudaError_t _se = cudaSetDevice((ctx)->device);                              \
    if (_se != cudaSuccess)                                                      \
      return swb_fail(SWB_ECUDA, "cudaSetDevice: %s", cudaGetErrorString(_se));  \
  }

#define SWB_API_END() return SWB_OK
