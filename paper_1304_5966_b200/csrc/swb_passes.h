// Internal pass-request interface shared by swb_pass.cu and swb_mm.cu.
#pragma once

#include <vector>

#include "swb_internal.h"

constexpr int kTabStride = 33;  // table row per column code: 32 row codes + the pad code

struct SchemeInt {
  int goe, ge, go, max_sub, k;
  uint32_t tlo[8], thi[8];
  int big = 0;                     // 1: shared-memory table (k > 7 or wide scores)
  int32_t tab[32 * kTabStride];    // tab[c * 33 + a] = sub(a, c) + go + ge; a = 32: pad (0)
};

struct PassReq {
  const uint8_t* rows = nullptr;
  const uint8_t* cols = nullptr;
  int rstep = 1, cstep = 1;
  int n1 = 0, n2 = 0;
  int border = 0;
  bool local = false;
  int track = 0;
  bool has_band = false;
  long long band_lo = 0, band_hi = 0;
  int prune = 0;  // 0 off, 1 running best, 2 fixed target, 3 target at corner
  long long prune_target = 0;
  long long corner_i = 0, corner_j = 0;
  bool want_final = false;
  int32_t* fin_h_dev = nullptr;  // device int32[n2] (cell columns); allocated if null
  int32_t* fin_f_dev = nullptr;
  int force_R = 0;
  long long row_offset = 0;
  int2* ext_in = nullptr;
  int32_t* ext_in_prog = nullptr;
  int2* ext_out = nullptr;
  int32_t* ext_out_prog = nullptr;
  long long rows_after = 0;  // pass rows below this slab (prune bounds)
  int32_t* shared_best = nullptr;  // running best shared between slabs (system scope)
  // tile bound maps
  int32_t* bmap_out = nullptr;
  const int32_t* bmap_in = nullptr;
  int map_nr = 0, map_nc = 0, map_r0 = 0, map_rdir = 1, map_c0 = 0, map_cdir = 1;
  int map_shift = 10;  // log2 of the tile edge
  long long bound_offset = 0;
  int4* bmap_live = nullptr;          // live-range sweep hulls per row tile (writer)
  const int4* rmap_live = nullptr;    // reader side of the same
  int bin_rev = 0;                    // bmap_in is the reverse map
  const int32_t* rmap_fwd = nullptr;  // static strip ranges (swb_kernels.cuh static_range)
  const int32_t* rmap_rev = nullptr;
  long long range_offset = 0;
  // filled by swb_run_passes
  int R = 0;
  bool x2 = false;  // packed 16x2 phase-1 kernel
  bool rows_code4 = false;  // the row sequence holds code 4
  bool x2_wild = false;     // packed kernel with the constant-row wildcard (code 4)
  bool wide = false;        // int64 kernel (swb_wide.cu): range beyond the int32 kernels
  int64_t* fin64_h_dev = nullptr;  // wide passes: int64 final rows (device)
  int64_t* fin64_f_dev = nullptr;
  int nstrips = 0;
  long long res_offset = 0;
  long long best_score = 0, best_i = -1, best_j = -1;
  long long cells = 0, blocks_exec = 0, blocks_pruned = 0, blocks_total = 0;
  double kernel_ms = 0.0;
};

int swb_prepare_scheme(const swb_scheme* s, SchemeInt* out);
int swb_check_range(const SchemeInt& sc, long long n1, long long n2);
int swb_resolve_seq(swb_ctx* ctx, int32_t id, int64_t off, int64_t len, int32_t rev,
                    const uint8_t** base, int* step);
void swb_bind_maps(swb_ctx* ctx, PassReq* r, long long off1, long long len1, bool rev1,
                   long long off2, long long len2, bool rev2, int write, int read,
                   long long offset);
int swb_run_passes(swb_ctx* ctx, const SchemeInt& sc, std::vector<PassReq>& reqs,
                   double* kernel_ms_total);
namespace swb {
int swb_run_wide(swb_ctx* ctx, const SchemeInt& sc, const std::vector<PassReq*>& reqs,
                 double* kernel_ms);
}
