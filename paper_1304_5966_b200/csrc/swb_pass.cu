// Host side of the wavefront pass: PassSpec -> device jobs -> one persistent
// launch per (recurrence, tracking, rows-per-lane) class -> PassResult.
// Replaces WavefrontEngine.run_wavefront (engine.py:188-282).
#include <algorithm>
#include <chrono>
#include <thread>
#include <cstdio>
#include <cstring>
#include <vector>

#include "swb_launch.cuh"

using namespace swb;

// Pre-fill the final rows of every job of one launch (cells the pass skips
// keep the fill values): one launch for all jobs; blockIdx.x strides the
// jobs, blockIdx.y splits long rows.
__global__ void fill_finals_kernel(const swb::JobDev* __restrict__ jobs, int nj) {
  for (int t = blockIdx.x; t < nj; t += gridDim.x) {
    const swb::JobDev& J = jobs[t];
    if (!J.want_final) continue;
    for (int x = blockIdx.y * blockDim.x + threadIdx.x; x < J.n2; x += gridDim.y * blockDim.x) {
      J.fin_h[x] = J.fill_h;
      J.fin_f[x] = SWB_NEG32;
    }
  }
}

int swb_prepare_scheme(const swb_scheme* s, SchemeInt* out) {
  if (!s) return swb_fail(SWB_EINVAL, "null scheme");
  if (s->k < 1 || s->k > 32)
    return swb_fail(SWB_EUNSUPPORTED, "alphabet size %d not supported (1..32)", s->k);
  if (s->gap_open < 0 || s->gap_extend < 1)
    return swb_fail(SWB_EINVAL, "gap_open must be >= 0 and gap_extend >= 1");
  const int goe = s->gap_open + s->gap_extend;
  int mx = INT32_MIN;
  for (int a = 0; a < s->k; ++a)
    for (int b = 0; b < s->k; ++b) mx = std::max(mx, s->sub[a * s->k + b]);
  out->goe = goe;
  out->ge = s->gap_extend;
  out->go = s->gap_open;
  out->k = s->k;
  out->max_sub = mx;
  if (mx != s->max_sub)
    return swb_fail(SWB_EINVAL, "max_sub %d does not match the matrix maximum %d", s->max_sub, mx);
  // register profiles (PRMT bytes) when they fit, else the shared table
  out->big = s->k > 7;
  for (int a = 0; a < s->k && !out->big; ++a)
    for (int b = 0; b < s->k; ++b) {
      const int v = s->sub[a * s->k + b] + goe;
      if (v < -127 || v > 127) out->big = 1;
    }
  memset(out->tab, 0, sizeof(out->tab));
  for (int c = 0; c < s->k; ++c)
    for (int a = 0; a < s->k; ++a) out->tab[c * kTabStride + a] = s->sub[a * s->k + c] + goe;
  if (out->big) return SWB_OK;
  for (int b = 0; b < 8; ++b) {
    uint8_t bytes[8];
    for (int a = 0; a < 8; ++a) {
      int v = -128;
      if (a < s->k && b < s->k) v = s->sub[a * s->k + b] + goe;
      bytes[a] = (uint8_t)(int8_t)v;
    }
    memcpy(&out->tlo[b], bytes, 4);
    memcpy(&out->thi[b], bytes + 4, 4);
  }
  return SWB_OK;
}

// Dynamic range of a pass: real DP values lie in [-D, D]; sentinel-derived
// ones in NEG32 +- D.
static long long pass_range(const SchemeInt& sc, long long n1, long long n2) {
  return (long long)sc.ge * (n1 + n2) + 2LL * sc.goe +
         (long long)std::max(sc.max_sub, 0) * std::min(n1, n2) + 1024;
}

int swb_check_range(const SchemeInt& sc, long long n1, long long n2) {
  // Keep both inside their half of the int32 range (see SWB_NEG_REPORT).
  const long long D = pass_range(sc, n1, n2);
  if (D >= (1LL << 28))
    return swb_fail(SWB_ERANGE,
                    "pass %lld x %lld with gap_extend %d / max_sub %d exceeds the int32 "
                    "dynamic range of the device kernels",
                    n1, n2, sc.ge, sc.max_sub);
  return SWB_OK;
}

int swb_resolve_seq(swb_ctx* ctx, int32_t id, int64_t off, int64_t len, int32_t rev,
                    const uint8_t** base, int* step) {
  if (id < 0 || id >= (int32_t)ctx->seqs.size() || !ctx->seqs[id].live)
    return swb_fail(SWB_EINVAL, "bad sequence id %d", id);
  const swb_seq& s = ctx->seqs[id];
  if (off < 0 || len < 0 || off + len > s.n)
    return swb_fail(SWB_EINVAL, "slice [%lld, %lld) outside sequence of length %lld",
                    (long long)off, (long long)(off + len), (long long)s.n);
  if (!rev) {
    *base = s.fwd + off;
    *step = 1;
  } else {
    // row r reads code[off + len - 1 - r] == rev[n - off - len + r]
    *base = s.rev + (s.n - off - len);
    *step = 1;
  }
  return SWB_OK;
}

namespace {

// Lane-kernel dispatch (swb_launch_local.cu / _none.cu / _track.cu).
int dispatch(swb_ctx* ctx, int R, const PassParams* P, long long items, bool local, int track,
             int ctas_per_sm, int* occ_out) {
  if (local) return dispatch_local(ctx, R, P, items, track, ctas_per_sm, occ_out);
  if (track == kTrackNone) return dispatch_other_none(ctx, R, P, items, ctas_per_sm, occ_out);
  return dispatch_other_track(ctx, R, P, items, track, ctas_per_sm, occ_out);
}

// Launch-shape model.  A warp-step costs ~5.7 integer-ALU
// instructions per row at 2 cycles each; a lone warp per SM sub-partition
// reaches ~60% of that rate, two or more saturate it.  Strips of one pass
// form a chain, so the pass runs at the pace of the most loaded sub-partition.
struct Shape {
  int R = 32;
  int ctas_per_sm = 0;
};

Shape choose_shape(swb_ctx* ctx, const std::vector<PassReq*>& jobs, bool local, int track,
                   bool x2, bool big) {
  bool x2f = false;  // packed kernel with final rows: its own instantiations
  for (const PassReq* r : jobs) x2f |= x2 && r->want_final;
  const int* cand = x2f ? kX2FinalR : x2 ? kX2R : big ? (local ? kBigLocalR : kBigOtherR) : (local ? kLocalR : kOtherR);
  const int ncand = x2f   ? (int)(sizeof(kX2FinalR) / sizeof(int))
                    : x2  ? (int)(sizeof(kX2R) / sizeof(int))
                    : big ? (local ? (int)(sizeof(kBigLocalR) / sizeof(int))
                                   : (int)(sizeof(kBigOtherR) / sizeof(int)))
                          : (local ? (int)(sizeof(kLocalR) / sizeof(int))
                                   : (int)(sizeof(kOtherR) / sizeof(int)));
  const int rows_mul = x2 ? 64 : 32;
  const int smsp = ctx->sms * 4;
  Shape best;
  double best_t = 1e300;
  for (int q = 0; q < ncand; ++q) {
    const int R = cand[q];
    if (R < ctx->min_R) continue;
    int occ = 0;
    const int rc = x2    ? dispatch_x2(ctx, R, nullptr, 0, 0, &occ, false, x2f)
                   : big ? dispatch_big(ctx, R, nullptr, 0, local, track, 0, &occ)
                         : dispatch(ctx, R, nullptr, 0, local, track, 0, &occ);
    if (rc != cudaSuccess || occ < 1) continue;
    const long long rows_item = (long long)rows_mul * R;
    long long strips = 0, chain = 0;
    for (const PassReq* r : jobs) {
      const long long sj = (r->n1 + rows_item - 1) / rows_item;
      strips += sj;
      chain = std::max(chain, (long long)r->n2 + (x2 ? 128LL : 64LL) * sj);
    }
    // integer-ALU cycles per warp-step: 5.7 per row (x2: 5.5 per packed row pair)
    const double alu = x2 ? 2.0 * (5.5 * R + 6.0) : 2.0 * (5.7 * R + 10.0);
    const double lat = 1.7 * alu;
    const long long w_need = (strips + smsp - 1) / smsp;
    const int w = (int)std::min<long long>(w_need, occ);
    const long long rounds = (w_need + occ - 1) / occ;
    const double step = std::max(w * alu, lat);
    // total work bound vs chain bound
    double work = 0.0;
    for (const PassReq* r : jobs)
      work += (double)((r->n1 + rows_item - 1) / rows_item) * (double)(r->n2 + 64) * alu;
    const double t = std::max((double)rounds * (double)chain * step, work / smsp);
    if (t < best_t * 0.999) {
      best_t = t;
      best.R = R;
      best.ctas_per_sm = w;
    }
  }
  return best;
}

struct Arena {
  char* base = nullptr;
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) & ~(size_t)255;
    T* p = reinterpret_cast<T*>(base + off);
    off += sizeof(T) * std::max<size_t>(count, 1);
    return p;
  }
};

}  // namespace

// Watchdog dump: claim counter, per-strip progress / live range / diagnostics
// record of a launch that is still running, read on a second stream.
static void swb_watchdog_dump(swb_ctx* ctx, const unsigned long long* d_claim, const int32_t* d_prog,
                              const int2* d_alive, const unsigned long long* d_sdbg,
                              long long strips, long long items) {
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return;
  const long long n = std::min<long long>(strips, 4096);
  unsigned long long* h = nullptr;
  if (cudaMallocHost(&h, 8 * (1 + n + n + 8 * n)) != cudaSuccess) return;
  unsigned long long* hc = h;
  int32_t* hp = reinterpret_cast<int32_t*>(h + 1);
  int2* ha = reinterpret_cast<int2*>(h + 1 + n);
  unsigned long long* hd = h + 1 + 2 * n;
  cudaMemcpyAsync(hc, d_claim, 8, cudaMemcpyDeviceToHost, st);
  cudaMemcpy2DAsync(hp, 4, d_prog, 4 * kProgStride, 4, n, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(ha, d_alive, 8 * n, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(hd, d_sdbg, 64 * n, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  fprintf(stderr, "[swb watchdog] launch %lld: claim %llu of %lld items, %lld strips\n",
          (long long)ctx->launches, hc[0], items, strips);
  for (long long q = 0; q < n; ++q)
    fprintf(stderr,
            "[swb watchdog] strip %lld: progress %d alive (%d,%d) cb %d/%d ce %d exit %d "
            "exec %llu skip %llu live (%d,%d) launch %llu sm %llu cta %llu warp %llu t0 %llu\n",
            q, hp[q], ha[q].x, ha[q].y, (int)(hd[8 * q] >> 32), (int)(unsigned)hd[8 * q],
            (int)(hd[8 * q + 1] >> 32), (int)(unsigned)hd[8 * q + 1], hd[8 * q + 2] >> 32,
            hd[8 * q + 2] & 0xffffffffu, (int)(hd[8 * q + 3] >> 32), (int)(unsigned)hd[8 * q + 3],
            hd[8 * q + 4], hd[8 * q + 5] >> 32, (hd[8 * q + 5] >> 8) & 0xffffff, hd[8 * q + 5] & 0xff, hd[8 * q + 6]);
  fflush(stderr);
}

int swb_run_passes(swb_ctx* ctx, const SchemeInt& sc, std::vector<PassReq>& reqs,
                   double* kernel_ms_total) {
  if (kernel_ms_total) *kernel_ms_total = 0.0;
  // group: (local, track, R)
  std::vector<int> order(reqs.size());
  for (size_t q = 0; q < reqs.size(); ++q) {
    order[q] = (int)q;
    PassReq& r = reqs[q];
    if (r.n1 < 1 || r.n2 < 1) return swb_fail(SWB_EINVAL, "cannot tile an empty matrix");
    // Passes whose values do not fit the int32 kernels run on the int64 kernel
    // (swb_wide.cu), as the reference computes in int64: the border ramps and
    // scores (pass_range < 2^28) and, for tracked passes, the int32 key H * 32 +
    // rank (max_sub * min(n1, n2) < 2^26).  Option "wide_log2" lowers both
    // limits (tests drive every pass through the wide kernel with it).
    const long long lim = 1LL << ctx->wide_log2;
    r.wide = pass_range(sc, r.row_offset + r.n1, r.n2) >= lim ||
             (r.track != kTrackNone &&
              (long long)std::max(sc.max_sub, 0) * std::min<long long>(r.row_offset + r.n1, r.n2) +
                      sc.goe >= (lim >> 2) - 64);
  }
  // packed 16x2 fast path eligibility (swb_x2.cuh header)
  // W max_sub <= 1021 (W = BLK + 63 columns of a block's window): 16-bit
  // endpoint keys (swb_x2.cuh).  Window bound: neighbouring cells differ by at
  // most go + ge + max_sub, so every value of a warp's window (<= 1024 rows + W
  // columns, plus BLK columns of growth) lies within kX2Span of the window
  // maximum and the relative frame never clamps one (x2_frame_ok).
  const long long ms = std::max(sc.max_sub, 0);
  // Five codes are allowed when code 4 scores the same against every column
  // (the default DNA alphabet's 'N' wildcard): its rows take a constant added
  // in the cell update instead of a profile byte (swb_x2.cuh, WILD).
  int wild_const = -1;
  if (sc.k == 5 && !sc.big) {
    wild_const = (int)(sc.thi[0] & 0xff);
    for (int b = 0; b < 5; ++b)
      if ((int)(sc.thi[b] & 0xff) != wild_const) wild_const = -1;
    if (wild_const > 127) wild_const = -1;
  }
  bool x2_scheme = (sc.k <= 4 || wild_const >= 0) && !sc.big && ctx->x2_enabled &&
                   x2_frame_ok(32, sc.goe, ms);
  // 64-step blocks need the wider window's key room and frame (swb_x2.cuh)
  const bool x2_blk64_ok = x2_frame_ok(64, sc.goe, ms);
  for (int b = 0; b < sc.k && x2_scheme; ++b)
    for (int a = 0; a < 4 && a < sc.k; ++a) {
      const int v = (int)(int8_t)((sc.tlo[b] >> (8 * a)) & 0xff);
      if (v < 0 || v > 127) x2_scheme = false;
    }
  for (PassReq& r : reqs)
    r.x2 = x2_scheme && r.local && r.track == kTrackMin && !r.has_band &&
           r.prune <= 1 && (!r.bmap_out || r.map_shift == kX2MapShift) &&
           // relative 16-bit frames: only the absolute H (boundary rows, running
           // best) must fit int32, which the wide limit already guarantees when
           // it is at its default
           (!r.wide || (ctx->wide_log2 >= 28 &&
                        ms * std::min<long long>(r.row_offset + r.n1, r.n2) < (1LL << 29))) &&
           // rows_per_lane forces the 32-bit kernel, except on row slabs where
           // it only fixes the strip granularity (64 x kX2SlabR rows here)
           (r.force_R == 0 || r.ext_in || r.ext_out) &&
           (!r.ext_out || r.n1 % (64 * kX2SlabR) == 0);  // slab bottom row = item bottom row
  for (PassReq& r : reqs) {
    r.x2_wild = r.x2 && sc.k == 5 && r.rows_code4;
    if (r.x2) r.wide = false;
  }
  // the wide passes leave the grouped launches and run on the int64 kernel
  std::vector<PassReq*> wide;
  {
    std::vector<int> keep;
    for (int q : order) {
      if (reqs[q].wide) wide.push_back(&reqs[q]);
      else keep.push_back(q);
    }
    order.swap(keep);
  }
  // one launch per (recurrence, tracking, kernel) class; rows-per-lane per class
  auto cls = [&](int q) {
    return (reqs[q].x2_wild ? 200 : reqs[q].x2 ? 100 : 0) + (reqs[q].local ? 10 : 0) + reqs[q].track;
  };
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cls(a) < cls(b); });
  std::vector<int> cls_ctas(reqs.size(), 0);
  for (size_t a = 0; a < order.size();) {
    size_t b = a;
    std::vector<PassReq*> js;
    while (b < order.size() && cls(order[b]) == cls(order[a])) js.push_back(&reqs[order[b++]]);
    Shape sh = choose_shape(ctx, js, js[0]->local, js[0]->track, js[0]->x2, sc.big != 0);
    if (js[0]->x2 && ctx->x2_R) sh.R = ctx->x2_R;
    if (js[0]->x2)
      for (PassReq* r : js)
        if (r->ext_out) sh.R = kX2SlabR;  // slabs are cut in multiples of 64 x kX2SlabR rows
    for (PassReq* r : js) {
      int fr = r->force_R;
      // shared-table kernels have fewer heights: a forced height (row slabs
      // use 32) maps to the largest instantiated one, which divides it
      if (fr && sc.big && (fr > 16 || (!r->local && fr > 8))) fr = r->local ? 16 : 8;
      r->R = (fr && !r->x2) ? fr : sh.R;
      cls_ctas[r - &reqs[0]] = sh.ctas_per_sm;
    }
    a = b;
  }
  for (const PassReq& r : reqs)
    if (r.ext_out && r.n1 % (32 * r.R) != 0)
      return swb_fail(SWB_EINVAL,
                      "row slab of %d rows feeding another slab must be a multiple of 32 x %d "
                      "(set rows_per_lane)", r.n1, r.R);
  // Final rows the caller did not place get their own buffer for the whole
  // call: the per-group arena below is reused by the next launch group, and
  // the rows are copied to the host only after every group has run.
  {
    long long fcols = 0;
    for (const PassReq& r : reqs)
      if (r.want_final && r.fin_h_dev == nullptr) fcols += 2LL * r.n2 + 64;
    if (fcols > 0) {
      int32_t* f = (int32_t*)swb_scratch(ctx->pass_finals, sizeof(int32_t) * (size_t)fcols);
      if (!f) return swb_fail(SWB_ECUDA, "out of device memory for final rows");
      long long o = 0;
      for (PassReq& r : reqs)
        if (r.want_final && r.fin_h_dev == nullptr) {
          r.fin_h_dev = f + o;
          r.fin_f_dev = f + o + r.n2;
          o += ((2LL * r.n2 + 63) / 64) * 64;
        }
    }
  }
  auto key = [&](int q) { return cls(q) * 1000 + reqs[q].R; };
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return key(a) < key(b); });

  size_t g0 = 0;
  while (g0 < order.size()) {
    size_t g1 = g0;
    while (g1 < order.size() && key(order[g1]) == key(order[g0])) ++g1;
    const PassReq& head = reqs[order[g0]];
    const int R = head.R;
    const int nj = (int)(g1 - g0);

    // layout
    long long total_strips = 0, total_cols = 0;
    for (size_t t = g0; t < g1; ++t) {
      PassReq& r = reqs[order[t]];
      const long long rows_item = (r.x2 ? 64LL : 32LL) * R;
      r.nstrips = (int)((r.n1 + rows_item - 1) / rows_item);
      total_strips += r.nstrips;
      total_cols += r.n2;
    }
    size_t bytes = 256 * 8 + sizeof(JobDev) * nj + sizeof(int32_t) * kProgStride * total_strips +
                   sizeof(int2) * total_strips + 256 + sizeof(int32_t) * 32 * kTabStride + 256 +
                   sizeof(unsigned long long) * 5 * nj + sizeof(int32_t) * nj + 64 +
                   sizeof(int4) * total_strips + 24 * total_strips + sizeof(int2) * 2 * total_cols +
                   4096 + 256 * 8 * (size_t)nj +
                   sizeof(int2) * total_strips + 256;
    Arena A;
    A.base = (char*)swb_scratch(ctx->rowbuf, bytes);
    if (!A.base) return swb_fail(SWB_ECUDA, "out of device memory (%zu bytes of pass scratch)", bytes);
    JobDev* d_jobs = A.take<JobDev>(nj);
    // zeroed region
    size_t zero_begin = (A.off + 255) & ~(size_t)255;
    int32_t* d_prog = A.take<int32_t>(kProgStride * total_strips);
    unsigned long long* d_cnt = A.take<unsigned long long>(5 * nj);
    int32_t* d_pbest = A.take<int32_t>(nj);
    unsigned long long* d_claim = A.take<unsigned long long>(1);
    int2* d_alive = A.take<int2>(total_strips);  // live ranges (restricted passes)
    size_t zero_end = A.off;
    int32_t* d_tab = sc.big ? A.take<int32_t>(32 * kTabStride) : nullptr;
    int4* d_res = A.take<int4>(total_strips);
    unsigned long long* d_times = A.take<unsigned long long>(3 * total_strips);
    // host staging (pinned)
    // (every section 256-byte aligned: int4 needs 16-byte alignment on the host too)
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t h_off_res = al(sizeof(JobDev) * nj);
    const size_t h_off_cnt = h_off_res + al(sizeof(int4) * total_strips);
    const size_t h_off_map = h_off_cnt + al(sizeof(unsigned long long) * 5 * nj);
    const size_t hbytes = h_off_map + al(sizeof(int2) * total_strips) + 256;
    char* hbase = (char*)swb_scratch_host(ctx->host_pinned, hbytes);
    if (!hbase) return swb_fail(SWB_ECUDA, "pinned host allocation failed");
    JobDev* h_jobs = reinterpret_cast<JobDev*>(hbase);
    int4* h_res = reinterpret_cast<int4*>(hbase + h_off_res);
    unsigned long long* h_cnt = reinterpret_cast<unsigned long long*>(hbase + h_off_cnt);
    int2* h_map = reinterpret_cast<int2*>(hbase + h_off_map);

    long long item = 0, strip_off = 0;
    for (int t = 0; t < nj; ++t) {
      PassReq& r = reqs[order[g0 + t]];
      JobDev& J = h_jobs[t];
      memset(&J, 0, sizeof(J));
      J.rows = r.rows;
      J.rstep = r.rstep;
      J.cols = r.cols;
      J.cstep = r.cstep;
      J.n1 = r.n1;
      J.n2 = r.n2;
      J.border = r.border;
      J.fill_h = r.local ? 0 : SWB_NEG32;
      J.has_band = r.has_band ? 1 : 0;
      if (r.has_band) {
        long long lo = std::max<long long>(r.band_lo, -(1LL << 30));
        long long hi = std::min<long long>(r.band_hi, (1LL << 30));
        J.band_lo = (int32_t)lo;
        J.band_hi = (int32_t)hi;
      }
      J.prune = r.prune;
      J.prune_target = (int32_t)std::max<long long>(std::min<long long>(r.prune_target, 1LL << 29),
                                                    -(1LL << 29));
      J.corner_i = (int32_t)r.corner_i;
      J.corner_j = (int32_t)r.corner_j;
      J.row_offset = (int32_t)r.row_offset;
      J.ext_in = r.ext_in;
      J.ext_in_prog = r.ext_in_prog;
      J.ext_out = r.ext_out;
      J.ext_out_prog = r.ext_out_prog;
      J.rows_after = (int32_t)r.rows_after;
      J.bmap_out = r.bmap_out;
      J.bmap_in = r.bmap_in;
      J.map_nr = r.map_nr;
      J.map_nc = r.map_nc;
      J.map_shift = r.map_shift;
      J.map_r0 = r.map_r0;
      J.map_rdir = r.map_rdir;
      J.map_c0 = r.map_c0;
      J.map_cdir = r.map_cdir;
      J.bound_offset = (int32_t)std::max<long long>(std::min<long long>(r.bound_offset, 1LL << 29),
                                                    -(1LL << 29));
      J.alive = (r.border == SWB_BORDER_RESTRICTED && !r.ext_in && !r.ext_out && ctx->live_ranges)
                    ? d_alive + strip_off : nullptr;
      // (option live_big masks the live-range features of shared-table passes;
      // diagnostics only since the warp-divergent early exit was fixed)
      J.live_mode = sc.big ? (ctx->live_ranges & ctx->live_big) : ctx->live_ranges;
      J.bmap_live = (J.alive && r.bmap_live) ? r.bmap_live : nullptr;
      J.rmap_live = r.rmap_live;
      J.bin_rev = r.bin_rev;
      J.rmap_fwd = r.rmap_fwd;
      J.rmap_rev = r.rmap_rev;
      J.range_offset = (int32_t)std::max<long long>(std::min<long long>(r.range_offset, 1LL << 29),
                                                    -(1LL << 29));
      J.nstrips = r.nstrips;
      J.want_final = r.want_final ? 1 : 0;
      J.item_base = item;
      J.buf[0] = A.take<int2>(r.n2);
      J.buf[1] = A.take<int2>(r.n2);
      J.progress = d_prog + strip_off * kProgStride;
      J.strip_res = d_res + strip_off;
      J.strip_times = d_times + 3 * strip_off;
      J.counters = d_cnt + 5 * t;
      J.prune_best = r.shared_best ? r.shared_best : d_pbest + t;
      J.best_sys = r.shared_best ? 1 : 0;
      if (r.want_final) {
        J.fin_h = r.fin_h_dev;
        J.fin_f = r.fin_f_dev;
      }
      r.res_offset = strip_off;
      item += r.nstrips;
      strip_off += r.nstrips;
    }
    // Chain-shaped passes (a corridor from the tile maps: phase 2, Myers-Miller
    // halves) with long chains run in chunks of 4 consecutive strips per CTA
    // (swb_kernels.cuh ChainChan); the claim map then lists (job, first strip)
    bool chain_chunks = false;
    if (ctx->chain_cta && !head.x2) {
      bool chainy = false, ext = false;
      for (size_t t = g0; t < g1; ++t) {
        chainy |= reqs[order[t]].rmap_fwd != nullptr || reqs[order[t]].bmap_in != nullptr;
        ext |= reqs[order[t]].ext_in != nullptr || reqs[order[t]].ext_out != nullptr;
      }
      chain_chunks = chainy && !ext && total_strips >= 8LL * nj;
    }
    long long chunk_items = 0;
    // strip-major claim order across jobs (item_job in swb_kernels.cuh)
    int2* d_map = nullptr;
    if (chain_chunks) {
      d_map = A.take<int2>(total_strips);
      int max_strips = 0;
      for (int t = 0; t < nj; ++t) max_strips = std::max(max_strips, h_jobs[t].nstrips);
      for (int st = 0; st < max_strips; st += ctx->chain_chunk)
        for (int t = 0; t < nj; ++t)
          if (st < h_jobs[t].nstrips) h_map[chunk_items++] = make_int2(t, st);
    } else if (nj > 1 && !ctx->job_major) {  // (group-mode launches drop it, see launch_any)
      d_map = A.take<int2>(total_strips);
      long long q = 0;
      int max_strips = 0;
      for (int t = 0; t < nj; ++t) max_strips = std::max(max_strips, h_jobs[t].nstrips);
      for (int st = 0; st < max_strips; ++st)
        for (int t = 0; t < nj; ++t)
          if (st < h_jobs[t].nstrips) h_map[q++] = make_int2(t, st);
    }
    if (A.off > bytes) return swb_fail(SWB_ECUDA, "internal: pass arena overflow");

    SWB_CUDA(cudaMemcpyAsync(d_jobs, h_jobs, sizeof(JobDev) * nj, cudaMemcpyHostToDevice, ctx->stream));
    if (d_tab)
      SWB_CUDA(cudaMemcpyAsync(d_tab, sc.tab, sizeof(int32_t) * 32 * kTabStride,
                               cudaMemcpyHostToDevice, ctx->stream));
    if (d_map)
      SWB_CUDA(cudaMemcpyAsync(d_map, h_map,
                               sizeof(int2) * (chain_chunks ? chunk_items : total_strips),
                               cudaMemcpyHostToDevice, ctx->stream));
    SWB_CUDA(cudaMemsetAsync(A.base + zero_begin, 0, zero_end - zero_begin, ctx->stream));
    bool any_final = false;
    for (int t = 0; t < nj && !any_final; ++t) any_final = reqs[order[g0 + t]].want_final;
    if (any_final) {
      const int gx = std::min(nj, 8 * ctx->sms);
      const int gy = std::max(1, std::min(64, 8 * ctx->sms / gx));
      fill_finals_kernel<<<dim3(gx, gy), 256, 0, ctx->stream>>>(d_jobs, nj);
      ctx->launches++;
    }
    SWB_CUDA(cudaGetLastError());

    PassParams P;
    memset(&P, 0, sizeof(P));
    P.jobs = d_jobs;
    P.njobs = nj;
    P.total_items = item;
    P.claim = d_claim;
    P.goe = sc.goe;
    P.ge = sc.ge;
    P.max_sub = sc.max_sub;
    P.proto = ctx->proto;
    P.key_mul = 32;
    P.item_map = d_map;
    P.big = sc.big;
    P.tab = d_tab;
    // diagnostics record outside the pass arena (the arena layout stays as is)
    unsigned long long* d_sdbg =
        (unsigned long long*)swb_scratch(ctx->dbg_buf, sizeof(unsigned long long) * 8 * total_strips);
    if (!d_sdbg) return swb_fail(SWB_ECUDA, "out of device memory (strip diagnostics)");
    P.strip_dbg = d_sdbg;
    P.launch_id = (unsigned long long)ctx->launches;
    if (ctx->claim_log_on) {
      if (!ctx->claim_log.p) {
        if (!swb_scratch(ctx->claim_log, 8 * (8 + 4 * 4096))) return swb_fail(SWB_ECUDA, "claim log");
        SWB_CUDA(cudaMemsetAsync(ctx->claim_log.p, 0, 8 * (8 + 4 * 4096), ctx->stream));
        SWB_CUDA(cudaStreamSynchronize(ctx->stream));
      }
      P.claim_log = (unsigned long long*)ctx->claim_log.p;
    }
    // passes restricted to a narrow corridor are chains along the diagonal:
    // spread their strips over warps and interleave the jobs (no pairing)
    for (size_t t = g0; t < g1; ++t)
      if (reqs[order[t]].rmap_fwd) P.warp_claim = 1;
    P.chain_wait = P.warp_claim && ctx->chain_wait;
    if (chain_chunks) {
      P.chunk = ctx->chain_chunk;
      P.total_items = chunk_items;
    }
    memcpy(P.tlo, sc.tlo, sizeof(P.tlo));
    memcpy(P.thi, sc.thi, sizeof(P.thi));

    SWB_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
    int rc;
    int ctas = ctx->max_ctas_per_sm ? ctx->max_ctas_per_sm : cls_ctas[order[g0]];
    P.wild_const = wild_const;
    bool any_final_x2 = false;
    for (size_t t = g0; t < g1; ++t) any_final_x2 |= head.x2 && reqs[order[t]].want_final;
    // packed kernel block length: 64 steps (half the handoffs, releases and
    // re-bases per column) for a single pass of more than one round of items;
    // 32 for single-round passes, where the longer handoff lag and the longer
    // optimistic re-runs cost more than they save, and for launches of several
    // passes (split=2's halves, row slabs), whose pruning the coarser blocks
    // weaken
    const bool auto64 = item > (long long)ctx->sms * 8 && g1 - g0 == 1;
    const int x2_blk = (ctx->x2_blk == 64 || (ctx->x2_blk == 0 && auto64)) && x2_blk64_ok ? 64 : 32;
    if (head.x2) ctx->last_x2_blk = x2_blk;
    rc = head.x2  ? dispatch_x2(ctx, R, &P, item, ctas, nullptr, head.x2_wild, any_final_x2, x2_blk)
         : sc.big ? dispatch_big(ctx, R, &P, item, head.local, head.track, ctas, nullptr)
                  : dispatch(ctx, R, &P, item, head.local, head.track, ctas, nullptr);
    if (rc) return rc;
    SWB_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
    SWB_CUDA(cudaMemcpyAsync(h_res, d_res, sizeof(int4) * total_strips, cudaMemcpyDeviceToHost,
                             ctx->stream));
    SWB_CUDA(cudaMemcpyAsync(h_cnt, d_cnt, sizeof(unsigned long long) * 5 * nj,
                             cudaMemcpyDeviceToHost, ctx->stream));
    if (ctx->watchdog_ms > 0) {
      // Watchdog (diagnostics): a launch that has not finished in time is
      // described from a second stream while it still runs, then reported.
      const auto t_start = std::chrono::steady_clock::now();
      for (;;) {
        const cudaError_t q = cudaStreamQuery(ctx->stream);
        if (q == cudaSuccess) break;
        if (q != cudaErrorNotReady) SWB_CUDA(q);
        const double el = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                                    t_start).count();
        if (el > ctx->watchdog_ms) {
          swb_watchdog_dump(ctx, d_claim, d_prog, d_alive, d_sdbg, total_strips, P.total_items);
          return swb_fail(SWB_ECUDA, "watchdog: pass launch (%d jobs, %lld strips) still running after %d ms",
                          nj, total_strips, ctx->watchdog_ms);
        }
        std::this_thread::sleep_for(std::chrono::microseconds(200));
      }
    }
    SWB_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->dbg_times.resize(3 * total_strips);
    SWB_CUDA(cudaMemcpy(ctx->dbg_times.data(), d_times, 24 * total_strips, cudaMemcpyDeviceToHost));
    ctx->dbg_strips.resize(12 * total_strips);
    {
      std::vector<unsigned long long> t(8 * total_strips);
      SWB_CUDA(cudaMemcpy(t.data(), d_sdbg, 64 * total_strips, cudaMemcpyDeviceToHost));
      for (long long q = 0; q < total_strips; ++q) {
        for (int w = 0; w < 8; ++w) ctx->dbg_strips[12 * q + w] = (long long)t[8 * q + w];
        ctx->dbg_strips[12 * q + 8] = h_res[q].x;
        ctx->dbg_strips[12 * q + 9] = h_res[q].y;
        ctx->dbg_strips[12 * q + 10] = h_res[q].z;
        ctx->dbg_strips[12 * q + 11] = h_res[q].w;
      }
    }
#ifdef SWB_CHECKED
    {
      long long chk[4];
      int (*takes[])(long long*) = {chk_take_local, chk_take_other, chk_take_track, chk_take_big,
                                    chk_take_x2, chk_take_x2w};
      for (auto take : takes) {
        if (take(chk) == 0 && chk[0])
          return swb_fail(SWB_ECUDA,
                          "device bounds check: %lld bad indices, first at swb_kernels.cuh:%lld "
                          "(index %lld outside [0, %lld))", chk[0], chk[1], chk[2], chk[3]);
      }
    }
#endif
    float ms = 0.f;
    SWB_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    ctx->last_kernel_ms = ms;
    if (kernel_ms_total) *kernel_ms_total += ms;
    if (ctx->trace) {
      long long cells = 0, maxn1 = 0, maxn2 = 0;
      for (int t = 0; t < nj; ++t) {
        const PassReq& r = reqs[order[g0 + t]];
        maxn1 = std::max<long long>(maxn1, r.n1);
        maxn2 = std::max<long long>(maxn2, r.n2);
      }
      for (int t = 0; t < nj; ++t) cells += (long long)h_cnt[5 * t + 0];
      fprintf(stderr,
              "[swb] launch local=%d track=%d R=%d jobs=%d strips=%lld max_n1=%lld max_n2=%lld "
              "cells=%lld ms=%.3f gcups=%.1f\n",
              (int)head.local, head.track, R, nj, total_strips, maxn1, maxn2, cells, ms,
              cells / (ms * 1e6));
    }

    for (int t = 0; t < nj; ++t) {
      PassReq& r = reqs[order[g0 + t]];
      r.kernel_ms = ms;
      long long bs = 0, bi = -1, bj = -1;
      bool have = false;
      for (int q = 0; q < r.nstrips; ++q) {
        const int4 v = h_res[r.res_offset + q];
        if (!v.w) continue;
        const long long s = (long long)v.x + sc.goe, i = v.y, j = v.z;
        bool take;
        if (!have) take = true;
        else if (r.track == kTrackMin)
          take = s > bs || (s == bs && (i < bi || (i == bi && j < bj)));
        else
          take = s > bs || (s == bs && (i > bi || (i == bi && j > bj)));
        if (take) {
          bs = s;
          bi = i;
          bj = j;
          have = true;
        }
      }
      if (r.track == kTrackMin) {
        if (!have || bs <= 0) {
          bs = 0;
          bi = bj = -1;
        }
      } else if (r.track == kTrackNone || !have) {
        bs = SWB_NEG_INF_REF;
        bi = bj = -1;
      } else if (bs < SWB_NEG_REPORT) {
        bs = SWB_NEG_INF_REF + (bs - (long long)SWB_NEG32);
      }
      r.best_score = bs;
      r.best_i = bi >= 0 ? bi + r.row_offset : bi;
      r.best_j = bj;
      r.cells = (long long)h_cnt[5 * t + 0];
      r.blocks_exec = (long long)h_cnt[5 * t + 1];
      r.blocks_pruned = (long long)h_cnt[5 * t + 2];
      ctx->dbg_wait_cycles += (long long)h_cnt[5 * t + 3];
      ctx->dbg_strip_cycles += (long long)h_cnt[5 * t + 4];
      // packed kernel: every block of every item is executed or pruned
      r.blocks_total = r.x2 ? r.blocks_exec + r.blocks_pruned
                            : (long long)r.nstrips * ((r.n2 + 31) / 32);
    }
    g0 = g1;
  }
  if (!wide.empty()) {
    double wms = 0.0;
    const int rc = swb_run_wide(ctx, sc, wide, &wms);
    if (rc) return rc;
    if (kernel_ms_total) *kernel_ms_total += wms;
  }
  return SWB_OK;
}

static inline long long left_h_host(int border, long long I, int go, int ge) {
  switch (border) {
    case SWB_BORDER_LOCAL: return 0;
    case SWB_BORDER_RESTRICTED: return I == 0 ? 0 : SWB_NEG_INF_REF;
    case SWB_BORDER_GLOBAL_FREE: return I == 0 ? 0 : -go - I * ge;
    case SWB_BORDER_GLOBAL_CONTINUE: return I == 0 ? SWB_NEG_INF_REF : -I * ge;
    default: return I == 0 ? SWB_NEG_INF_REF : -go - I * ge;
  }
}

static inline long long left_f_host(int border, long long I, int go, int ge) {
  switch (border) {
    case SWB_BORDER_LOCAL:
    case SWB_BORDER_RESTRICTED: return SWB_NEG_INF_REF;
    case SWB_BORDER_GLOBAL_FREE: return I == 0 ? SWB_NEG_INF_REF : -go - I * ge;
    case SWB_BORDER_GLOBAL_CONTINUE: return I == 0 ? 0 : -I * ge;
    default: return I == 0 ? -(long long)go : -go - I * ge;
  }
}

static inline long long widen(int32_t v) {
  if ((long long)v < SWB_NEG_REPORT) return SWB_NEG_INF_REF + ((long long)v - (long long)SWB_NEG32);
  return v;
}

void swb_bind_maps(swb_ctx* ctx, PassReq* r, long long off1, long long len1, bool rev1,
                   long long off2, long long len2, bool rev2, int write, int read,
                   long long offset) {
  int32_t* fwd = reinterpret_cast<int32_t*>(ctx->bmap_fwd.p);
  int32_t* rev = reinterpret_cast<int32_t*>(ctx->bmap_rev.p);
  r->map_nr = ctx->bmap_nr;
  r->map_nc = ctx->bmap_nc;
  r->map_shift = ctx->bmap_shift;
  r->map_r0 = (int)(rev1 ? off1 + len1 - 1 : off1);
  r->map_rdir = rev1 ? -1 : 1;
  r->map_c0 = (int)(rev2 ? off2 + len2 - 1 : off2);
  r->map_cdir = rev2 ? -1 : 1;
  r->bmap_out = write == 1 ? fwd : (write == 2 ? rev : nullptr);
  r->bmap_in = read == 1 ? fwd : (read == 2 ? rev : nullptr);
  int4* live = reinterpret_cast<int4*>(ctx->bmap_live.p);
  if (write == 2) r->bmap_live = live;  // reverse map writers record their swept hull
  r->rmap_live = live;
  r->bin_rev = read == 2 ? 1 : 0;
  r->bound_offset = offset;
}

extern "C" int32_t swb_bounds_reset(swb_ctx* ctx, int32_t seq1, int32_t seq2) {
  SWB_API_BEGIN(ctx);
  if (seq1 < 0 || seq1 >= (int)ctx->seqs.size() || !ctx->seqs[seq1].live || seq2 < 0 ||
      seq2 >= (int)ctx->seqs.size() || !ctx->seqs[seq2].live)
    return swb_fail(SWB_EINVAL, "bad sequence id");
  const int sh = ctx->map_shift;  // tile edge 2^sh (option map_tile_log2)
  const long long nr = std::max<long long>(1, (ctx->seqs[seq1].n + (1LL << sh) - 1) >> sh);
  const long long nc = std::max<long long>(1, (ctx->seqs[seq2].n + (1LL << sh) - 1) >> sh);
  const size_t bytes = sizeof(int32_t) * (size_t)nr * (size_t)nc;
  void* f = swb_scratch(ctx->bmap_fwd, bytes);
  void* r = f ? swb_scratch(ctx->bmap_rev, bytes) : nullptr;
  if (!f || !r) return swb_fail(SWB_ECUDA, "out of device memory for bound maps (%zu bytes)", 2 * bytes);
  SWB_CUDA(cudaMemsetAsync(f, 0xff, bytes, ctx->stream));  // -1: never written (+inf)
  SWB_CUDA(cudaMemsetAsync(r, 0xff, bytes, ctx->stream));
  // per row tile sweep hull of the reverse pass: (-(lo+1), hi, covered) = empty
  int4* lv = (int4*)swb_scratch(ctx->bmap_live, sizeof(int4) * (size_t)nr);
  if (!lv) return swb_fail(SWB_ECUDA, "out of device memory for bound maps");
  {
    std::vector<int4> init((size_t)nr, make_int4(INT32_MIN, -1, 0, 0));
    SWB_CUDA(cudaMemcpyAsync(lv, init.data(), sizeof(int4) * (size_t)nr, cudaMemcpyHostToDevice,
                             ctx->stream));
    SWB_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  ctx->bmap_seq1 = seq1;
  ctx->bmap_seq2 = seq2;
  ctx->bmap_nr = (int)nr;
  ctx->bmap_nc = (int)nc;
  ctx->bmap_shift = sh;
  SWB_API_END();
}

extern "C" int64_t swb_bounds_read(swb_ctx* ctx, int32_t which, int32_t* out, int64_t cap) {
  if (!ctx) return -1;
  const long long n = (long long)ctx->bmap_nr * ctx->bmap_nc;
  if (!out || cap <= 0) return n;
  const swb_buf& b = which == 2 ? ctx->bmap_rev : ctx->bmap_fwd;
  if (!b.p) return 0;
  cudaStreamSynchronize(ctx->stream);
  if (cudaMemcpy(out, b.p, sizeof(int32_t) * (size_t)std::min<long long>(n, cap),
                 cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  return n;
}

extern "C" int32_t swb_bounds_device(swb_ctx* ctx, int32_t which, uint64_t* ptr, int64_t* n,
                                     int64_t* nc) {
  SWB_API_BEGIN(ctx);
  if (!ptr || !n || !nc || (which != 1 && which != 2))
    return swb_fail(SWB_EINVAL, "swb_bounds_device: bad arguments");
  const swb_buf& b = which == 2 ? ctx->bmap_rev : ctx->bmap_fwd;
  if (!b.p || ctx->bmap_seq1 < 0) return swb_fail(SWB_EINVAL, "no tile maps (swb_bounds_reset first)");
  SWB_CUDA(cudaStreamSynchronize(ctx->stream));
  *ptr = (uint64_t)(uintptr_t)b.p;
  *n = (int64_t)ctx->bmap_nr * ctx->bmap_nc;
  *nc = ctx->bmap_nc;
  SWB_API_END();
}

extern "C" int64_t swb_get_option(swb_ctx* ctx, const char* name) {
  if (!ctx || !name) return -1;
  if (!strcmp(name, "max_ctas_per_sm")) return ctx->max_ctas_per_sm;
  if (!strcmp(name, "x2_R")) return ctx->x2_R;
  if (!strcmp(name, "x2_blk")) return ctx->x2_blk;
  if (!strcmp(name, "last_x2_blk")) return ctx->last_x2_blk;
  if (!strcmp(name, "x2")) return ctx->x2_enabled;
  if (!strcmp(name, "job_major")) return ctx->job_major;
  if (!strcmp(name, "bound_maps")) return ctx->bmaps_on;
  if (!strcmp(name, "mm_R")) return ctx->mm_R;
  if (!strcmp(name, "mm_static")) return ctx->mm_static;
  if (!strcmp(name, "mm_dyn")) return ctx->mm_dyn;
  if (!strcmp(name, "chain_wait")) return ctx->chain_wait;
  if (!strcmp(name, "chain_cta")) return ctx->chain_cta;
  if (!strcmp(name, "live_ranges")) return ctx->live_ranges;
  if (!strcmp(name, "live_big")) return ctx->live_big;
  if (!strcmp(name, "watchdog_ms")) return ctx->watchdog_ms;
  if (!strcmp(name, "wide_log2")) return ctx->wide_log2;
  if (!strcmp(name, "chain_chunk")) return ctx->chain_chunk;
  if (!strcmp(name, "map_tile_log2")) return ctx->bmap_seq1 >= 0 ? ctx->bmap_shift : ctx->map_shift;
  if (!strcmp(name, "p2_R")) return ctx->p2_R;
  if (!strcmp(name, "mm_prune")) return ctx->mm_prune;
  if (!strcmp(name, "claim_mode")) return ctx->claim_mode;
  if (!strcmp(name, "proto")) return ctx->proto;
  if (!strcmp(name, "rows_per_lane")) return ctx->force_R;
  return -1;
}

extern "C" int32_t swb_set_option(swb_ctx* ctx, const char* name, int64_t value) {
  if (!ctx || !name) return swb_fail(SWB_EINVAL, "bad arguments");
  if (!strcmp(name, "max_ctas_per_sm")) {
    ctx->max_ctas_per_sm = (int)value;
    return SWB_OK;
  }
  if (!strcmp(name, "x2_blk")) {
    if (value != 0 && value != 32 && value != 64) return swb_fail(SWB_EINVAL, "x2_blk must be 0, 32 or 64");
    ctx->x2_blk = (int)value;  // 0: by rounds of items
    return SWB_OK;
  }
  if (!strcmp(name, "x2_R")) {
    ctx->x2_R = (int)value;
    return SWB_OK;
  }
  if (!strcmp(name, "x2")) {
    ctx->x2_enabled = (int)value;
    return SWB_OK;
  }
  if (!strcmp(name, "job_major")) {
    ctx->job_major = (int)value;
    return SWB_OK;
  }
  if (!strcmp(name, "bound_maps")) {
    ctx->bmaps_on = (int)value;
    return SWB_OK;
  }
  if (!strcmp(name, "mm_dyn")) {
    ctx->mm_dyn = (int)value;
    return SWB_OK;
  }
  if (!strcmp(name, "chain_wait")) {
    ctx->chain_wait = (int)value;
    return SWB_OK;
  }
  if (!strcmp(name, "chain_cta")) {
    ctx->chain_cta = (int)value;
    return SWB_OK;
  }
  if (!strcmp(name, "mm_static")) {
    ctx->mm_static = (int)value;
    return SWB_OK;
  }
  if (!strcmp(name, "p2_R")) {
    ctx->p2_R = (int)value;
    return SWB_OK;
  }
  if (!strcmp(name, "map_tile_log2")) {
    if (value < 8 || value > 12) return swb_fail(SWB_EINVAL, "map_tile_log2 must be in [8, 12]");
    ctx->map_shift = (int)value;  // takes effect at the next swb_bounds_reset
    return SWB_OK;
  }
  if (!strcmp(name, "chain_chunk")) {
    if (value != 4 && value != 8) return swb_fail(SWB_EINVAL, "chain_chunk must be 4 or 8");
    ctx->chain_chunk = (int)value;
    return SWB_OK;
  }
  if (!strcmp(name, "min_R")) {
    ctx->min_R = (int)value;
    return SWB_OK;
  }
  if (!strcmp(name, "wide_log2")) {
    if (value < 4 || value > 28) return swb_fail(SWB_EINVAL, "wide_log2 must be in [4, 28]");
    ctx->wide_log2 = (int)value;
    return SWB_OK;
  }
  if (!strcmp(name, "claim_log")) {
    ctx->claim_log_on = (int)value;
    return SWB_OK;
  }
  if (!strcmp(name, "watchdog_ms")) {
    ctx->watchdog_ms = (int)value;
    return SWB_OK;
  }
  if (!strcmp(name, "live_big")) {
    ctx->live_big = (int)value;
    return SWB_OK;
  }
  if (!strcmp(name, "live_ranges")) {
    ctx->live_ranges = (int)value;
    return SWB_OK;
  }
  if (!strcmp(name, "mm_R")) {
    ctx->mm_R = (int)value;  // rows per lane of range-limited Myers-Miller passes (0: auto)
    return SWB_OK;
  }
  if (!strcmp(name, "mm_prune")) {
    ctx->mm_prune = (int)value;
    return SWB_OK;
  }
  if (!strcmp(name, "claim_mode")) {
    ctx->claim_mode = (int)value;  // 0 auto, 1 force CTA claiming, 2 force warp claiming
    return SWB_OK;
  }
  if (!strcmp(name, "proto")) {
    ctx->proto = (int)value;
    return SWB_OK;
  }
  if (!strcmp(name, "reset_debug")) {
    ctx->dbg_wait_cycles = ctx->dbg_strip_cycles = 0;
    return SWB_OK;
  }
  if (!strcmp(name, "rows_per_lane")) {
    if (value < 0 || value > 32)
      return swb_fail(SWB_EINVAL, "rows_per_lane must be 0 (auto) or an instantiated value <= 32");
    ctx->force_R = (int)value;
    return SWB_OK;
  }
  return swb_fail(SWB_EINVAL, "unknown option %s", name);
}

extern "C" int32_t swb_pass(swb_ctx* ctx, const swb_scheme* scheme, const swb_pass_desc* descs,
                            int32_t n, swb_pass_out* outs) {
  SWB_API_BEGIN(ctx);
  if (n < 0 || (n > 0 && (!descs || !outs))) return swb_fail(SWB_EINVAL, "bad arguments");
  SchemeInt sc;
  int rc = swb_prepare_scheme(scheme, &sc);
  if (rc) return rc;
  std::vector<PassReq> reqs(n);
  for (int q = 0; q < n; ++q) {
    const swb_pass_desc& d = descs[q];
    PassReq& r = reqs[q];
    rc = swb_resolve_seq(ctx, d.seq1, d.off1, d.len1, d.rev1, &r.rows, &r.rstep);
    if (rc == SWB_OK) r.rows_code4 = ctx->seqs[d.seq1].has_code4;
    if (rc) return rc;
    rc = swb_resolve_seq(ctx, d.seq2, d.off2, d.len2, d.rev2, &r.cols, &r.cstep);
    if (rc) return rc;
    r.n1 = (int)d.len1;
    r.n2 = (int)d.len2;
    if (d.border < SWB_BORDER_LOCAL || d.border > SWB_BORDER_GLOBAL_CHARGE)
      return swb_fail(SWB_EINVAL, "bad border %d", d.border);
    if (d.track < 0 || d.track > 2) return swb_fail(SWB_EINVAL, "bad track mode %d", d.track);
    r.border = d.border;
    r.local = d.clamp_zero != 0;
    r.track = d.track;
    if (r.local && (d.border != SWB_BORDER_LOCAL || d.track != SWB_TRACK_MIN || d.has_band))
      return swb_fail(SWB_EUNSUPPORTED, "clamped passes must use local borders, TRACK_MIN, no band");
    if (d.prune < 0 || d.prune > 3) return swb_fail(SWB_EINVAL, "bad prune kind %d", d.prune);
    if (r.local && d.prune > 1) return swb_fail(SWB_EUNSUPPORTED, "local passes prune on the running best");
    if (!r.local && d.prune == 1) return swb_fail(SWB_EUNSUPPORTED, "running-best pruning needs a local pass");
    r.has_band = d.has_band != 0;
    r.band_lo = d.band_lo;
    r.band_hi = d.band_hi;
    r.prune = d.prune;
    r.prune_target = d.prune_target;
    r.corner_i = d.corner_i;
    r.corner_j = d.corner_j;
    r.want_final = d.want_final_rows != 0;
    if (r.want_final && (!d.final_row_h || !d.final_row_f))
      return swb_fail(SWB_EINVAL, "want_final_rows needs final_row_h/final_row_f");
    r.force_R = ctx->force_R;
    r.row_offset = d.row_offset;
    r.ext_in = reinterpret_cast<int2*>(d.ext_in_buf);
    r.ext_in_prog = reinterpret_cast<int32_t*>(d.ext_in_progress);
    r.ext_out = reinterpret_cast<int2*>(d.ext_out_buf);
    r.ext_out_prog = reinterpret_cast<int32_t*>(d.ext_out_progress);
    if (d.rows_after < 0 || d.rows_after >= (1LL << 31))
      return swb_fail(SWB_ERANGE, "rows_after out of range");
    r.rows_after = d.rows_after;
    r.shared_best = reinterpret_cast<int32_t*>(d.shared_best);
    if (r.shared_best && (!r.local || d.prune != 1))
      return swb_fail(SWB_EINVAL, "shared_best applies to local passes with running-best pruning");
    if ((r.ext_in || r.ext_out || r.row_offset) && r.has_band)
      return swb_fail(SWB_EUNSUPPORTED, "row slabs (multi-GPU) do not support a band");
    if ((r.ext_in == nullptr) != (r.ext_in_prog == nullptr) ||
        (r.ext_out == nullptr) != (r.ext_out_prog == nullptr))
      return swb_fail(SWB_EINVAL, "ext boundary needs both a buffer and a progress counter");
    if (r.row_offset < 0 || r.row_offset + r.n1 >= (1LL << 31))
      return swb_fail(SWB_ERANGE, "row_offset out of range");
    if (d.bound_write < 0 || d.bound_write > 2 || d.bound_read < 0 || d.bound_read > 2)
      return swb_fail(SWB_EINVAL, "bad bound map mode");
    if ((d.bound_write || d.bound_read) && ctx->bmaps_on) {
      if (d.seq1 != ctx->bmap_seq1 || d.seq2 != ctx->bmap_seq2)
        return swb_fail(SWB_EINVAL, "bound maps were not reset for sequences (%d, %d)", d.seq1,
                        d.seq2);
      if (d.bound_read && d.prune != 2 && d.prune != 3)
        return swb_fail(SWB_EINVAL, "bound_read needs a target (prune kind 2 or 3)");
      swb_bind_maps(ctx, &r, d.off1, d.len1, d.rev1 != 0, d.off2, d.len2, d.rev2 != 0,
                    d.bound_write, d.bound_read, d.bound_offset);
      // a bound-pruned restricted pass is a chain along the path: short strips
      if (d.bound_read && !r.local && !r.force_R && ctx->p2_R) r.force_R = ctx->p2_R;
    }
  }
  double ms = 0.0;
  rc = swb_run_passes(ctx, sc, reqs, &ms);
  if (rc) return rc;
  for (int q = 0; q < n; ++q) {
    const swb_pass_desc& d = descs[q];
    PassReq& r = reqs[q];
    swb_pass_out& o = outs[q];
    o.best_score = r.best_score;
    o.best_i = r.best_i;
    o.best_j = r.best_j;
    o.cells_executed = r.cells;
    o.tiles_total = r.blocks_total;
    o.tiles_executed = r.blocks_exec;
    o.tiles_pruned = r.blocks_pruned;
    o.tiles_banded_out = std::max<long long>(0, r.blocks_total - r.blocks_exec - r.blocks_pruned);
    o.kernel_ms = r.kernel_ms;
    o.kernel = r.wide ? 2 : (r.x2 ? 1 : 0);
    o.rows_per_lane = r.R;
    if (r.want_final && r.wide) {  // int64 kernel: the reference's values as they are
      SWB_CUDA(cudaMemcpyAsync(d.final_row_h + 1, r.fin64_h_dev, sizeof(int64_t) * r.n2,
                               cudaMemcpyDeviceToHost, ctx->stream));
      SWB_CUDA(cudaMemcpyAsync(d.final_row_f + 1, r.fin64_f_dev, sizeof(int64_t) * r.n2,
                               cudaMemcpyDeviceToHost, ctx->stream));
      SWB_CUDA(cudaStreamSynchronize(ctx->stream));
      d.final_row_h[0] = left_h_host(r.border, r.n1, sc.go, sc.ge);
      d.final_row_f[0] = left_f_host(r.border, r.n1, sc.go, sc.ge);
    } else if (r.want_final) {
      std::vector<int32_t> th(r.n2), tf(r.n2);
      SWB_CUDA(cudaMemcpyAsync(th.data(), r.fin_h_dev, sizeof(int32_t) * r.n2,
                               cudaMemcpyDeviceToHost, ctx->stream));
      SWB_CUDA(cudaMemcpyAsync(tf.data(), r.fin_f_dev, sizeof(int32_t) * r.n2,
                               cudaMemcpyDeviceToHost, ctx->stream));
      SWB_CUDA(cudaStreamSynchronize(ctx->stream));
      d.final_row_h[0] = left_h_host(r.border, r.n1, sc.go, sc.ge);
      d.final_row_f[0] = left_f_host(r.border, r.n1, sc.go, sc.ge);
      for (int c = 0; c < r.n2; ++c) {
        d.final_row_h[c + 1] = widen(th[c]);
        d.final_row_f[c + 1] = widen(tf[c]);
      }
    }
  }
  SWB_API_END();
}

extern "C" int32_t swb_boundary_alloc(swb_ctx* ctx, int64_t n2, uint64_t* buf, uint64_t* progress) {
  SWB_API_BEGIN(ctx);
  if (n2 < 1 || !buf || !progress) return swb_fail(SWB_EINVAL, "bad arguments");
  void* b = nullptr;
  void* p = nullptr;
  SWB_CUDA(cudaMalloc(&b, sizeof(int2) * (size_t)n2));
  SWB_CUDA(cudaMalloc(&p, 256));
  SWB_CUDA(cudaMemset(p, 0, 256));
  *buf = reinterpret_cast<uint64_t>(b);
  *progress = reinterpret_cast<uint64_t>(p);
  SWB_API_END();
}

extern "C" int32_t swb_boundary_reset(swb_ctx* ctx, uint64_t progress) {
  SWB_API_BEGIN(ctx);
  SWB_CUDA(cudaMemsetAsync(reinterpret_cast<void*>(progress), 0, sizeof(int32_t), ctx->stream));
  SWB_CUDA(cudaStreamSynchronize(ctx->stream));
  SWB_API_END();
}

extern "C" int32_t swb_boundary_free(swb_ctx* ctx, uint64_t buf, uint64_t progress) {
  SWB_API_BEGIN(ctx);
  SWB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (buf) SWB_CUDA(cudaFree(reinterpret_cast<void*>(buf)));
  if (progress) SWB_CUDA(cudaFree(reinterpret_cast<void*>(progress)));
  SWB_API_END();
}

extern "C" int32_t swb_ipc_export(swb_ctx* ctx, uint64_t ptr, uint8_t* handle64) {
  SWB_API_BEGIN(ctx);
  if (!ptr || !handle64) return swb_fail(SWB_EINVAL, "bad arguments");
  cudaIpcMemHandle_t h;
  SWB_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(ptr)));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle64, &h, 64);
  SWB_API_END();
}

extern "C" int32_t swb_ipc_import(swb_ctx* ctx, const uint8_t* handle64, uint64_t* ptr) {
  SWB_API_BEGIN(ctx);
  if (!ptr || !handle64) return swb_fail(SWB_EINVAL, "bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  void* p = nullptr;
  SWB_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  *ptr = reinterpret_cast<uint64_t>(p);
  SWB_API_END();
}

extern "C" int32_t swb_ipc_close(swb_ctx* ctx, uint64_t ptr) {
  SWB_API_BEGIN(ctx);
  if (ptr) SWB_CUDA(cudaIpcCloseMemHandle(reinterpret_cast<void*>(ptr)));
  SWB_API_END();
}

extern "C" int32_t swb_debug_times(swb_ctx* ctx, int64_t* out, int32_t n) {
  if (!ctx || !out) return swb_fail(SWB_EINVAL, "bad arguments");
  int32_t m = (int32_t)ctx->dbg_times.size();
  for (int32_t q = 0; q < n && q < m; ++q) out[q] = (int64_t)ctx->dbg_times[q];
  return m;
}

extern "C" int32_t swb_debug_strips(swb_ctx* ctx, int64_t* out, int32_t n) {
  if (!ctx) return swb_fail(SWB_EINVAL, "bad arguments");
  const int32_t m = (int32_t)ctx->dbg_strips.size();
  for (int32_t q = 0; out && q < n && q < m; ++q) out[q] = ctx->dbg_strips[q];
  return m;
}

extern "C" int32_t swb_debug_claims(swb_ctx* ctx, int64_t* out, int32_t n) {
  if (!ctx) return swb_fail(SWB_EINVAL, "bad arguments");
  const int32_t m = 8 + 4 * 4096;
  if (!ctx->claim_log.p || !out) return ctx->claim_log.p ? m : 0;
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return swb_fail(SWB_ECUDA, "sync");
  if (cudaMemcpy(out, ctx->claim_log.p, 8 * (size_t)std::min(n, m), cudaMemcpyDeviceToHost) != cudaSuccess)
    return swb_fail(SWB_ECUDA, "copy");
  return m;
}

extern "C" int32_t swb_debug_stats(swb_ctx* ctx, int64_t* out, int32_t n) {
  if (!ctx || !out) return swb_fail(SWB_EINVAL, "bad arguments");
  const int64_t v[2] = {ctx->dbg_wait_cycles, ctx->dbg_strip_cycles};
  for (int q = 0; q < n && q < 2; ++q) out[q] = v[q];
  return SWB_OK;
}
