// Wide (int64) wavefront pass: the device path for passes whose dynamic range
// does not fit the int32 kernels (scores, lengths or gap costs so large that
// max_sub * min(n1, n2) reaches 2^26 or the border ramps 2^28).  The reference
// computes in int64 with NEG_INF = -(2**61) (kernels.py:14); so does this
// kernel, so it accepts every pass the reference accepts.
//
// Same decomposition as run_strip (swb_kernels.cuh), without its
// optimisations: one warp per strip of 32 lanes x kWideR rows, lane l at
// column step - l, the row above arriving by __shfl_up_sync; strips chain
// through (H, F) row buffers in HBM and a release/acquire progress counter per
// strip, published every 32 columns.  Cell update and tracking follow
// kernels.affine_block (kernels.py:44-87) literally: E, F, H = max(diag + sub,
// E, F [, 0]); TRACK_MIN keeps h > 0 with ties to the smallest (i, j),
// TRACK_MAX ties to the largest.  Bands are strip-granular (results do not
// depend on band granularity, SURVEY.md §0 finding 1); no pruning, no tile
// maps (a later pass that reads the maps sees "unknown" tiles, which is sound).
#include <algorithm>
#include <cstring>
#include <vector>

#include "swb_kernels.cuh"
#include "swb_passes.h"

namespace swb {
namespace {

constexpr int kWideR = 4;  // rows per lane
constexpr long long kNeg64 = -(1LL << 61);

struct WideJob {
  const uint8_t* rows;
  const uint8_t* cols;
  int32_t n1, n2;
  int32_t border, clamp, track, has_band;
  long long band_lo, band_hi;
  long long fill_h;
  int32_t nstrips, want_final;
  long long item_base;
  longlong2* buf[2];     // (H, F) of a strip's bottom row, per column
  int32_t* progress;     // per strip: columns < progress published
  long long* fin_h;      // final row (DP columns 1..n2) or null
  long long* fin_f;
  longlong4* strip_res;  // per strip (score, i, j, has)
  unsigned long long* cells;
};

struct WideParams {
  const WideJob* jobs;
  int32_t njobs;
  int32_t k;
  long long total_items;
  unsigned long long* claim;
  long long go, ge;
  const int32_t* sub;  // k x k, sub[a * k + b]
};

__device__ __forceinline__ long long left_h64(int border, long long I, long long go, long long ge) {
  switch (border) {
    case SWB_BORDER_LOCAL: return 0;
    case SWB_BORDER_RESTRICTED: return I == 0 ? 0 : kNeg64;
    case SWB_BORDER_GLOBAL_FREE: return I == 0 ? 0 : -go - I * ge;
    case SWB_BORDER_GLOBAL_CONTINUE: return I == 0 ? kNeg64 : -I * ge;
    default: return I == 0 ? kNeg64 : -go - I * ge;  // charge
  }
}

__device__ __forceinline__ long long top_h64(int border, long long J, long long go, long long ge) {
  switch (border) {
    case SWB_BORDER_LOCAL: return 0;
    case SWB_BORDER_RESTRICTED: return J == 0 ? 0 : kNeg64;
    case SWB_BORDER_GLOBAL_FREE: return J == 0 ? 0 : -go - J * ge;
    default: return kNeg64;  // continue / charge: origin blocked, no top row
  }
}

__device__ __forceinline__ void wide_range(const WideJob& J, int s, int& cb, int& ce) {
  cb = 0;
  ce = J.n2;
  if (!J.has_band) return;
  const long long r0 = (long long)s * 32 * kWideR;
  long long r1 = r0 + 32 * kWideR - 1;
  if (r1 > J.n1 - 1) r1 = J.n1 - 1;
  long long lo = r0 - J.band_hi, hi = r1 - J.band_lo + 1;
  if (lo < 0) lo = 0;
  if (hi > J.n2) hi = J.n2;
  if (hi < lo) hi = lo;
  cb = (int)lo;
  ce = (int)hi;
}

__device__ __forceinline__ bool better(int track, long long h, long long i, long long j,
                                       long long bs, long long bi, long long bj) {
  if (track == kTrackMin)
    return h > 0 && (h > bs || (h == bs && (i < bi || (i == bi && j < bj))));
  return h > bs || (h == bs && (i > bi || (i == bi && j > bj)));
}

__device__ void wide_strip(const WideParams& P, const WideJob& J, int s) {
  const int lane = threadIdx.x & 31;
  const long long go = P.go, ge = P.ge, goe = go + ge;
  const int n1 = J.n1;
  const int R0 = s * 32 * kWideR;
  const int lrow0 = R0 + lane * kWideR;
  int cb, ce, cbp = 0, cep = 0;
  wide_range(J, s, cb, ce);
  if (s > 0) wide_range(J, s - 1, cbp, cep);
  const longlong2* inbuf = J.buf[(s + 1) & 1];
  longlong2* outbuf = J.buf[s & 1];
  const bool first = s == 0;

  int code[kWideR];
#pragma unroll
  for (int r = 0; r < kWideR; ++r) {
    const int i = lrow0 + r;
    code[r] = i < n1 ? (int)J.rows[i] : -1;
  }
  long long H[kWideR], E[kWideR];
#pragma unroll
  for (int r = 0; r < kWideR; ++r) {
    H[r] = cb == 0 ? left_h64(J.border, lrow0 + r + 1, go, ge) : J.fill_h;
    E[r] = kNeg64;
  }
  // diagonal of row 0 at column cb: H(lrow0 - 1, cb - 1)
  long long diag;
  if (cb == 0) diag = left_h64(J.border, lrow0, go, ge);
  else diag = J.fill_h;  // lane 0: set below from the producer's row
  long long out_h = J.fill_h, out_f = kNeg64;
  long long bs = J.track == kTrackMin ? 0 : kNeg64, bi = -1, bj = -1;
  int known = 0, known2 = 0;
  const int fin_lane = (n1 - 1 - R0) / kWideR, fin_r = (n1 - 1 - R0) % kWideR;
  const bool final_strip = J.want_final && s == J.nstrips - 1;
  unsigned long long cells = 0;

  // lane 0's top input at a column: border row, producer row, or fill
  auto top_at = [&](int c, long long& th, long long& tf) {
    if (first) {
      th = top_h64(J.border, c + 1, go, ge);
      tf = kNeg64;
    } else if (c >= cbp && c < cep) {
      if (known <= c) {
        const int need = c + 32 < cep ? c + 32 : cep;
        int v = ld_acquire(J.progress + (s - 1));
        while (v < need) {
          __nanosleep(64);
          v = ld_acquire(J.progress + (s - 1));
        }
        known = v;
      }
      const longlong2 t = __ldcg(inbuf + c);
      th = t.x;
      tf = t.y;
    } else {
      th = J.fill_h;
      tf = kNeg64;
    }
  };
  if (lane == 0 && cb > 0) {
    long long th, tf;
    top_at(cb - 1, th, tf);
    diag = th;
  }

  for (int st = cb; st < ce + 31; ++st) {
    const int c = st - lane;
    long long up_h = __shfl_up_sync(0xffffffffu, out_h, 1);
    long long up_f = __shfl_up_sync(0xffffffffu, out_f, 1);
    const bool act = c >= cb && c < ce;
    if (lane == 0 && act) top_at(c, up_h, up_f);
    if (act) {
      const int sc = (int)J.cols[c];
      long long d = diag;
      diag = up_h;  // next column's diagonal for row 0
      long long f = up_f, hab = up_h, fh = 0, ff = 0;
#pragma unroll
      for (int r = 0; r < kWideR; ++r) {
        long long e = H[r] - goe;
        if (E[r] - ge > e) e = E[r] - ge;
        long long t = hab - goe;
        f = f - ge;
        if (t > f) f = t;
        long long h = code[r] >= 0 ? d + P.sub[code[r] * P.k + sc] : kNeg64;
        if (e > h) h = e;
        if (f > h) h = f;
        if (J.clamp && h < 0) h = 0;
        d = H[r];
        H[r] = h;
        E[r] = e;
        hab = h;
        const int i = lrow0 + r;
        if (i < n1 && J.track != kTrackNone && better(J.track, h, i, c, bs, bi, bj)) {
          bs = h;
          bi = i;
          bj = c;
        }
        if (r == fin_r) {
          fh = h;
          ff = f;
        }
      }
      out_h = hab;
      out_f = f;
      if (final_strip && lane == fin_lane) {
        J.fin_h[c] = fh;
        J.fin_f[c] = ff;
      }
    }
    // the bottom row of the strip, lane 31; every 32 columns publish
    const int c31 = st - 31;
    if (lane == 31 && c31 >= cb && c31 < ce) {
      if (s >= 2 && known2 <= c31) {  // strip s-2 must be done with this column
        int v = ld_acquire(J.progress + (s - 2));
        while (v <= c31) {
          __nanosleep(64);
          v = ld_acquire(J.progress + (s - 2));
        }
        known2 = v;
      }
      outbuf[c31] = make_longlong2(out_h, out_f);
      if (((c31 - cb) & 31) == 31 || c31 == ce - 1) {
        __threadfence();
        st_release(J.progress + s, c31 + 1);
      }
    }
  }
  if (lane == 31) {
    __threadfence();
    st_release(J.progress + s, 0x7fffffff);
  }
  int rows_here = n1 - R0;
  if (rows_here > 32 * kWideR) rows_here = 32 * kWideR;
  if (lane == 0) cells = (unsigned long long)(ce - cb) * (unsigned long long)rows_here;
  // strip result with the mode's tie rule (engine.py:247-259)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long os = __shfl_down_sync(0xffffffffu, bs, o);
    const long long oi = __shfl_down_sync(0xffffffffu, bi, o);
    const long long oj = __shfl_down_sync(0xffffffffu, bj, o);
    if (oi >= 0 && (bi < 0 || better(J.track == kTrackNone ? kTrackMax : J.track, os, oi, oj, bs, bi,
                                     bj))) {
      bs = os;
      bi = oi;
      bj = oj;
    }
  }
  if (lane == 0) {
    J.strip_res[s] = make_longlong4(bs, bi, bj, bi >= 0 ? 1 : 0);
    atomicAdd(J.cells, cells);
  }
}

__global__ void __launch_bounds__(128) wide_kernel(const WideParams P) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    long long item = 0;
    if (lane == 0) item = (long long)atomicAdd(P.claim, 1ULL);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= P.total_items) break;
    int lo = 0, hi = P.njobs - 1;
    while (lo < hi) {
      const int m = (lo + hi + 1) >> 1;
      if (P.jobs[m].item_base <= item) lo = m;
      else hi = m - 1;
    }
    wide_strip(P, P.jobs[lo], (int)(item - P.jobs[lo].item_base));
    __syncwarp();
  }
}

__global__ void wide_fill_kernel(const WideJob* jobs, int nj) {
  for (int t = blockIdx.x; t < nj; t += gridDim.x) {
    const WideJob& J = jobs[t];
    if (!J.want_final) continue;
    for (int x = threadIdx.x; x < J.n2; x += blockDim.x) {
      J.fin_h[x] = J.fill_h;
      J.fin_f[x] = kNeg64;
    }
  }
}

}  // namespace

// Run the wide passes of one swb_pass / swb_crossings call in one launch; fills
// each request's results, and its int64 final rows into fin64_*_dev
// (allocated here when null).
int swb_run_wide(swb_ctx* ctx, const SchemeInt& sc, const std::vector<PassReq*>& reqs,
                 double* kernel_ms) {
  if (kernel_ms) *kernel_ms = 0.0;
  if (reqs.empty()) return SWB_OK;
  const int nj = (int)reqs.size();
  long long strips = 0, cols = 0, fcols = 0;
  for (PassReq* r : reqs) {
    if (r->ext_in || r->ext_out || r->row_offset)
      return swb_fail(SWB_EUNSUPPORTED, "row slabs need the int32 dynamic range");
    r->nstrips = (r->n1 + 32 * kWideR - 1) / (32 * kWideR);
    strips += r->nstrips;
    cols += r->n2;
    if (r->want_final && !r->fin64_h_dev) fcols += r->n2;
  }
  const size_t bytes = sizeof(WideJob) * nj + 4 * strips + sizeof(longlong4) * strips +
                       sizeof(longlong2) * 2 * cols + 16 * fcols + 8 * nj + 4 * 1024 +
                       8 * 256 + 16 * 256 * (size_t)nj;
  char* base = (char*)swb_scratch(ctx->wide_buf, bytes);
  if (!base) return swb_fail(SWB_ECUDA, "out of device memory (%zu bytes, wide pass)", bytes);
  size_t off = 0;
  auto take = [&](size_t n) {
    off = (off + 255) & ~(size_t)255;
    char* p = base + off;
    off += std::max<size_t>(n, 1);
    return p;
  };
  WideJob* d_jobs = (WideJob*)take(sizeof(WideJob) * nj);
  const size_t z0 = (off + 255) & ~(size_t)255;
  int32_t* d_prog = (int32_t*)take(4 * strips);
  unsigned long long* d_cells = (unsigned long long*)take(8 * nj);
  unsigned long long* d_claim = (unsigned long long*)take(8);
  const size_t z1 = off;
  longlong4* d_res = (longlong4*)take(sizeof(longlong4) * strips);
  int32_t* d_sub = (int32_t*)take(4 * 1024);
  std::vector<WideJob> h(nj);
  long long item = 0, soff = 0;
  for (int t = 0; t < nj; ++t) {
    PassReq& r = *reqs[t];
    WideJob& J = h[t];
    memset(&J, 0, sizeof(J));
    J.rows = r.rows;
    J.cols = r.cols;
    J.n1 = r.n1;
    J.n2 = r.n2;
    J.border = r.border;
    J.clamp = r.local ? 1 : 0;
    J.track = r.track;
    J.has_band = r.has_band ? 1 : 0;
    J.band_lo = r.band_lo;
    J.band_hi = r.band_hi;
    J.fill_h = r.local ? 0 : kNeg64;
    J.nstrips = r.nstrips;
    J.want_final = r.want_final ? 1 : 0;
    J.item_base = item;
    J.buf[0] = (longlong2*)take(sizeof(longlong2) * r.n2);
    J.buf[1] = (longlong2*)take(sizeof(longlong2) * r.n2);
    J.progress = d_prog + soff;
    J.strip_res = d_res + soff;
    J.cells = d_cells + t;
    if (r.want_final) {
      if (!r.fin64_h_dev) {
        r.fin64_h_dev = (int64_t*)take(8 * r.n2);
        r.fin64_f_dev = (int64_t*)take(8 * r.n2);
      }
      J.fin_h = (long long*)r.fin64_h_dev;
      J.fin_f = (long long*)r.fin64_f_dev;
    }
    r.res_offset = soff;
    item += r.nstrips;
    soff += r.nstrips;
  }
  if (off > bytes) return swb_fail(SWB_ECUDA, "internal: wide pass arena overflow");
  int32_t subv[1024] = {0};
  for (int a = 0; a < sc.k; ++a)
    for (int b = 0; b < sc.k; ++b) subv[a * sc.k + b] = sc.tab[b * kTabStride + a] - sc.goe;
  SWB_CUDA(cudaMemcpyAsync(d_jobs, h.data(), sizeof(WideJob) * nj, cudaMemcpyHostToDevice,
                           ctx->stream));
  SWB_CUDA(cudaMemcpyAsync(d_sub, subv, 4 * sc.k * sc.k, cudaMemcpyHostToDevice, ctx->stream));
  SWB_CUDA(cudaMemsetAsync(base + z0, 0, z1 - z0, ctx->stream));
  bool any_final = false;
  for (PassReq* r : reqs) any_final |= r->want_final;
  if (any_final) {
    wide_fill_kernel<<<std::min(nj, 1024), 256, 0, ctx->stream>>>(d_jobs, nj);
    ctx->launches++;
  }
  WideParams P;
  P.jobs = d_jobs;
  P.njobs = nj;
  P.k = sc.k;
  P.total_items = item;
  P.claim = d_claim;
  P.go = sc.go;
  P.ge = sc.ge;
  P.sub = d_sub;
  int per_sm = 0;
  SWB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, wide_kernel, 128, 0));
  const long long grid = std::min<long long>((long long)std::max(per_sm, 1) * ctx->sms,
                                             std::max(1LL, (item + 3) / 4));
  SWB_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
  wide_kernel<<<(int)grid, 128, 0, ctx->stream>>>(P);
  ctx->launches++;
  SWB_CUDA(cudaGetLastError());
  SWB_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
  std::vector<longlong4> res(strips);
  std::vector<unsigned long long> cells(nj);
  SWB_CUDA(cudaMemcpyAsync(res.data(), d_res, sizeof(longlong4) * strips, cudaMemcpyDeviceToHost,
                           ctx->stream));
  SWB_CUDA(cudaMemcpyAsync(cells.data(), d_cells, 8 * nj, cudaMemcpyDeviceToHost, ctx->stream));
  SWB_CUDA(cudaStreamSynchronize(ctx->stream));
  float ms = 0.f;
  SWB_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  ctx->last_kernel_ms = ms;
  if (kernel_ms) *kernel_ms = ms;
  for (int t = 0; t < nj; ++t) {
    PassReq& r = *reqs[t];
    long long bs = 0, bi = -1, bj = -1;
    bool have = false;
    for (int q = 0; q < r.nstrips; ++q) {
      const longlong4 v = res[r.res_offset + q];
      if (!v.w) continue;
      bool take_it;
      if (!have) take_it = true;
      else if (r.track == kTrackMin)
        take_it = v.x > bs || (v.x == bs && (v.y < bi || (v.y == bi && v.z < bj)));
      else
        take_it = v.x > bs || (v.x == bs && (v.y > bi || (v.y == bi && v.z > bj)));
      if (take_it) {
        bs = v.x;
        bi = v.y;
        bj = v.z;
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
    }
    r.best_score = bs;
    r.best_i = bi;
    r.best_j = bj;
    r.cells = (long long)cells[t];
    r.blocks_total = (long long)r.nstrips * ((r.n2 + 31) / 32);
    r.blocks_exec = r.blocks_total;
    r.blocks_pruned = 0;
    r.kernel_ms = ms;
    r.R = kWideR;
  }
  return SWB_OK;
}

}  // namespace swb
