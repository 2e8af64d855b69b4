// Myers-Miller reconstruction on the device: one launch per recursion level.
//
//   swb_crossings  replaces phase3.find_crossing (phase3.py:136-190): the upper
//                  forward and lower reverse global passes of every subproblem of
//                  the level run as jobs of one persistent pass launch; a combine
//                  kernel forms hh = Hup + Hdn[::-1], ff = Fup + Fdn[::-1] + go in
//                  int64 and applies _pick_crossing's tie rule (phase3.py:123-133).
//   swb_leaves     replaces kernels.leaf_solve (kernels.py:91-185): one warp per
//                  leaf fills the banded Gotoh matrices (row-parallel: F and the
//                  diagonal term per lane, E by a warp max-scan, exact because
//                  go >= 0) and lane 0 replays leaf_solve's traceback verbatim.
#include <algorithm>
#include <cstring>
#include <vector>

#include "swb_kernels.cuh"
#include "swb_passes.h"

using namespace swb;

namespace {

__host__ __device__ inline long long widen64(int v) {
  return (long long)v < SWB_NEG_REPORT ? SWB_NEG_INF_REF + ((long long)v - (long long)SWB_NEG32)
                                       : (long long)v;
}

__host__ __device__ inline long long left_h64(int border, long long I, int go, int ge) {
  switch (border) {
    case SWB_BORDER_LOCAL: return 0;
    case SWB_BORDER_RESTRICTED: return I == 0 ? 0 : SWB_NEG_INF_REF;
    case SWB_BORDER_GLOBAL_FREE: return I == 0 ? 0 : -go - I * ge;
    case SWB_BORDER_GLOBAL_CONTINUE: return I == 0 ? SWB_NEG_INF_REF : -I * ge;
    default: return I == 0 ? SWB_NEG_INF_REF : -go - I * ge;
  }
}

__host__ __device__ inline long long left_f64(int border, long long I, int go, int ge) {
  switch (border) {
    case SWB_BORDER_LOCAL:
    case SWB_BORDER_RESTRICTED: return SWB_NEG_INF_REF;
    case SWB_BORDER_GLOBAL_FREE: return I == 0 ? SWB_NEG_INF_REF : -go - I * ge;
    case SWB_BORDER_GLOBAL_CONTINUE: return I == 0 ? 0 : -I * ge;
    default: return I == 0 ? -(long long)go : -go - I * ge;
  }
}

struct CombineDev {
  const int32_t *uh, *uf, *dh, *df;  // final rows (cell columns 0..cols-1 -> DP 1..cols)
  // int64 final rows of passes that ran on the wide kernel (swb_wide.cu), else null
  const long long *uh64, *uf64, *dh64, *df64;
  int32_t cols;
  int32_t rows_up, rows_dn;
  int32_t border_up, border_dn;
  int64_t expected;
};

struct CombineOut {
  long long best;
  long long j;
  long long upper, lower;
  int gap;
  int status;
};

__device__ inline long long up_h(const CombineDev& c, int j, int go, int ge) {
  return j == 0 ? left_h64(c.border_up, c.rows_up, go, ge)
                : (c.uh64 ? c.uh64[j - 1] : widen64(c.uh[j - 1]));
}
__device__ inline long long up_f(const CombineDev& c, int j, int go, int ge) {
  return j == 0 ? left_f64(c.border_up, c.rows_up, go, ge)
                : (c.uf64 ? c.uf64[j - 1] : widen64(c.uf[j - 1]));
}
__device__ inline long long dn_h(const CombineDev& c, int q, int go, int ge) {
  return q == 0 ? left_h64(c.border_dn, c.rows_dn, go, ge)
                : (c.dh64 ? c.dh64[q - 1] : widen64(c.dh[q - 1]));
}
__device__ inline long long dn_f(const CombineDev& c, int q, int go, int ge) {
  return q == 0 ? left_f64(c.border_dn, c.rows_dn, go, ge)
                : (c.df64 ? c.df64[q - 1] : widen64(c.df[q - 1]));
}

// One CTA per subproblem: max over hh/ff, then the first column attaining it.
__global__ void __launch_bounds__(256) combine_kernel(const CombineDev* subs, CombineOut* out,
                                                      int go, int ge) {
  const CombineDev c = subs[blockIdx.x];
  __shared__ long long red[256];
  __shared__ long long rj[2][256];
  const int cols = c.cols;
  long long m = LLONG_MIN;
  for (int j = threadIdx.x; j <= cols; j += blockDim.x) {
    const long long hh = up_h(c, j, go, ge) + dn_h(c, cols - j, go, ge);
    const long long ff = up_f(c, j, go, ge) + dn_f(c, cols - j, go, ge) + go;
    m = max(m, max(hh, ff));
  }
  red[threadIdx.x] = m;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = max(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  const long long best = red[0];
  long long jh = LLONG_MAX, jf = LLONG_MAX;
  for (int j = threadIdx.x; j <= cols; j += blockDim.x) {
    const long long hh = up_h(c, j, go, ge) + dn_h(c, cols - j, go, ge);
    const long long ff = up_f(c, j, go, ge) + dn_f(c, cols - j, go, ge) + go;
    if (hh == best && j < jh) jh = j;
    if (ff == best && j < jf) jf = j;
  }
  rj[0][threadIdx.x] = jh;
  rj[1][threadIdx.x] = jf;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      rj[0][threadIdx.x] = min(rj[0][threadIdx.x], rj[0][threadIdx.x + s]);
      rj[1][threadIdx.x] = min(rj[1][threadIdx.x], rj[1][threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    CombineOut o;
    const long long h = rj[0][0], f = rj[1][0];
    o.best = best;
    o.gap = !(h <= f);  // plain join wins ties at equal column
    o.j = o.gap ? f : h;
    const int j = (int)o.j;
    if (o.gap) {
      o.upper = up_f(c, j, go, ge);
      o.lower = dn_f(c, cols - j, go, ge);
    } else {
      o.upper = up_h(c, j, go, ge);
      o.lower = dn_h(c, cols - j, go, ge);
    }
    o.status = best == c.expected ? 0 : 1;
    out[blockIdx.x] = o;
  }
}

// Chunked combine: the top Myers-Miller levels have few subproblems of
// millions of columns, which one CTA each scanned at a single SM's bandwidth
// (C3: 130 ms over the levels).  Each CTA now reduces kCombChunk columns of one
// subproblem to (max hh, first j) and (max ff, first j); one warp per
// subproblem merges its chunks and applies combine_kernel's rule.
constexpr int kCombChunk = 16384;

struct CombArena {  // 256-byte aligned carving of one scratch allocation
  char* base = nullptr;
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) & ~(size_t)255;
    T* p = reinterpret_cast<T*>(base + off);
    off += sizeof(T) * (count > 0 ? count : 1);
    return p;
  }
};

struct CombinePart {
  long long mh, mf;
  int jh, jf;
};

// (m, j) pairs: larger m wins, equal m -> smaller j
__device__ inline void take_first_max(long long& m, int& j, long long om, int oj) {
  if (om > m || (om == m && oj < j)) {
    m = om;
    j = oj;
  }
}

__global__ void __launch_bounds__(256) combine_part_kernel(const CombineDev* subs,
                                                           const int* chunk_sub,
                                                           const int* chunk_lo,
                                                           CombinePart* parts, int go, int ge) {
  const CombineDev c = subs[chunk_sub[blockIdx.x]];
  const int lo = chunk_lo[blockIdx.x];
  const int hi = min(lo + kCombChunk, c.cols + 1);
  const int cols = c.cols;
  long long mh = LLONG_MIN, mf = LLONG_MIN;
  int jh = INT_MAX, jf = INT_MAX;
  for (int j = lo + threadIdx.x; j < hi; j += blockDim.x) {  // increasing j: strict > keeps the first
    const long long hh = up_h(c, j, go, ge) + dn_h(c, cols - j, go, ge);
    const long long ff = up_f(c, j, go, ge) + dn_f(c, cols - j, go, ge) + go;
    if (hh > mh) { mh = hh; jh = j; }
    if (ff > mf) { mf = ff; jf = j; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    take_first_max(mh, jh, __shfl_down_sync(0xffffffffu, mh, o), __shfl_down_sync(0xffffffffu, jh, o));
    take_first_max(mf, jf, __shfl_down_sync(0xffffffffu, mf, o), __shfl_down_sync(0xffffffffu, jf, o));
  }
  __shared__ CombinePart w[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) w[warp] = CombinePart{mh, mf, jh, jf};
  __syncthreads();
  if (threadIdx.x == 0) {
    CombinePart r = w[0];
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      take_first_max(r.mh, r.jh, w[k].mh, w[k].jh);
      take_first_max(r.mf, r.jf, w[k].mf, w[k].jf);
    }
    parts[blockIdx.x] = r;
  }
}

__global__ void __launch_bounds__(256) combine_final_kernel(const CombineDev* subs, int n,
                                                            const int* part_off,
                                                            const CombinePart* parts,
                                                            CombineOut* out, int go, int ge) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= n) return;
  long long mh = LLONG_MIN, mf = LLONG_MIN;
  int jh = INT_MAX, jf = INT_MAX;
  for (int q = part_off[t] + lane; q < part_off[t + 1]; q += 32) {
    take_first_max(mh, jh, parts[q].mh, parts[q].jh);
    take_first_max(mf, jf, parts[q].mf, parts[q].jf);
  }
  for (int o = 16; o > 0; o >>= 1) {
    take_first_max(mh, jh, __shfl_down_sync(0xffffffffu, mh, o), __shfl_down_sync(0xffffffffu, jh, o));
    take_first_max(mf, jf, __shfl_down_sync(0xffffffffu, mf, o), __shfl_down_sync(0xffffffffu, jf, o));
  }
  if (lane == 0) {
    const CombineDev c = subs[t];
    const long long best = max(mh, mf);
    const long long h = mh == best ? jh : LLONG_MAX, f = mf == best ? jf : LLONG_MAX;
    CombineOut o;
    o.best = best;
    o.gap = !(h <= f);  // plain join wins ties at equal column
    o.j = o.gap ? f : h;
    const int j = (int)o.j;
    if (o.gap) {
      o.upper = up_f(c, j, go, ge);
      o.lower = dn_f(c, c.cols - j, go, ge);
    } else {
      o.upper = up_h(c, j, go, ge);
      o.lower = dn_h(c, c.cols - j, go, ge);
    }
    o.status = best == c.expected ? 0 : 1;
    out[t] = o;
  }
}

// ---- leaves -------------------------------------------------------------------

struct LeafDev {
  const uint8_t* c1;
  const uint8_t* c2;
  int32_t n, m;
  int32_t svg, evg;
  int32_t lo, hi;
  int64_t mat_off;  // offset (elements) of this leaf's H/E/F matrices
  int64_t ops_off;
};

__global__ void __launch_bounds__(32) leaf_kernel(const LeafDev* leaves, int32_t* mats,
                                                  uint8_t* ops, long long* counts,
                                                  long long* scores, const int32_t* sub_g,
                                                  int k, int go, int ge) {
  __shared__ int32_t sub[1024];
  const int lane = threadIdx.x;
  for (int x = lane; x < k * k; x += 32) sub[x] = sub_g[x];
  __syncwarp();
  const LeafDev L = leaves[blockIdx.x];
  const int n = L.n, m = L.m, W = m + 1;
  const int goe = go + ge;
  const long long area = (long long)(n + 1) * W;
  int32_t* H = mats + L.mat_off;
  int32_t* E = H + area;
  int32_t* F = E + area;
  const int NEG = SWB_NEG32;

  // row 0 and column 0 (kernels.py:106-118)
  for (int j = lane; j <= m; j += 32) {
    int h = NEG, e = NEG, f = NEG;
    if (L.svg) {
      if (j == 0) f = 0;
    } else {
      if (j == 0) h = 0;
      else h = e = -go - j * ge;
    }
    H[j] = h;
    E[j] = e;
    F[j] = f;
  }
  __syncwarp();
  for (int i = 1; i <= n; ++i) {
    int32_t* Hr = H + (long long)i * W;
    int32_t* Er = E + (long long)i * W;
    int32_t* Fr = F + (long long)i * W;
    const int32_t* Hp = Hr - W;
    const int32_t* Fp = Fr - W;
    const int a = L.c1[i - 1];
    int jlo = i - L.hi, jhi = i - L.lo;
    if (jlo < 1) jlo = 1;
    if (jhi > m) jhi = m;
    // column 0 of this row
    if (lane == 0) {
      const int v = L.svg ? -i * ge : -go - i * ge;
      Hr[0] = v;
      Fr[0] = v;
      Er[0] = NEG;
    }
    // carry for E: value at column jlo from its left neighbour (border or NEG)
    int carry = INT32_MIN;  // X = E + ge*j, prefix max
    if (jlo <= jhi) {
      const int hl = (jlo - 1 == 0) ? (L.svg ? -i * ge : -go - i * ge) : NEG;
      const int el = NEG;
      int e0 = hl - goe;
      if (el - ge > e0) e0 = el - ge;
      carry = e0 + ge * jlo;
    }
    for (int base = 1; base <= m; base += 32) {
      const int j = base + lane;
      const bool in = (j <= m);
      const bool band = in && j >= jlo && j <= jhi;
      int hprime = NEG, f = NEG, t = INT32_MIN;
      if (band) {
        int fv = Hp[j] - goe;
        const int ft = Fp[j] - ge;
        if (ft > fv) fv = ft;
        f = fv;
        int hv = Hp[j - 1] + sub[a * k + L.c2[j - 1]];
        if (f > hv) hv = f;
        hprime = hv;
        // contribution to E at column j+1
        if (j + 1 <= jhi) t = hv - goe + ge * (j + 1);
      }
      // E at column j: X[j] = max(carry, T[jlo+1..j]) where T[j'] is from lane j'-1
      int tprev = __shfl_up_sync(0xffffffffu, t, 1);
      if (lane == 0) tprev = INT32_MIN;
      // inclusive max-scan of tprev across lanes
      int x = tprev;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o && y > x) x = y;
      }
      if (carry > x) x = carry;
      if (band) {
        const int e = (j == jlo) ? carry - ge * j : x - ge * j;
        int hv = hprime;
        if (e > hv) hv = e;
        Hr[j] = hv;
        Er[j] = e;
        Fr[j] = f;
      } else if (in) {
        Hr[j] = NEG;
        Er[j] = NEG;
        Fr[j] = NEG;
      }
      // carry into the next chunk: X at the chunk's last column, plus the
      // last lane's own contribution to the following column
      const int xl = __shfl_sync(0xffffffffu, x, 31);
      const int tl = __shfl_sync(0xffffffffu, t, 31);
      carry = xl > tl ? xl : tl;
    }
    __syncwarp();
  }
  __syncwarp();

  // traceback, kernels.py:143-185 (ops written back to front, then compacted)
  if (lane == 0) {
    long long score;
    int state;
    if (L.evg) {
      score = widen64(F[(long long)n * W + m]);
      state = 2;
    } else {
      score = widen64(H[(long long)n * W + m]);
      state = 0;
    }
    int i = n, j = m;
    const long long cap = (long long)n + m;
    long long q = cap;
    uint8_t* o = ops + L.ops_off;
    bool dead = false;
    // numpy negative-index wrap of the reference (H[i, -1] == H[i, m]) is kept
    auto at = [&](const int32_t* M, int ii, int jj) -> int {
      if (ii < 0) ii += n + 1;
      if (jj < 0) jj += W;
      return M[(long long)ii * W + jj];
    };
    while ((i > 0 || j > 0) && !dead) {
      if (state == 0) {
        const int h = at(H, i, j);
        if (i > 0 && j > 0 && h == at(H, i - 1, j - 1) + sub[L.c1[i - 1] * k + L.c2[j - 1]]) {
          o[--q] = (L.c1[i - 1] == L.c2[j - 1]) ? 0 : 1;
          --i;
          --j;
        } else if (j > 0 && h == at(E, i, j)) {
          state = 1;
        } else if (i > 0 && h == at(F, i, j)) {
          state = 2;
        } else {
          dead = true;
        }
      } else if (state == 1) {
        o[--q] = 2;
        const int e = at(E, i, j);
        if (e == at(H, i, j - 1) - goe) state = 0;
        else if (e != at(E, i, j - 1) - ge) dead = true;
        --j;
      } else {
        o[--q] = 3;
        const int f = at(F, i, j);
        if (f == at(H, i - 1, j) - goe) state = 0;
        else if (f != at(F, i - 1, j) - ge) dead = true;
        --i;
      }
    }
    if (dead) {
      counts[blockIdx.x] = -1;
      scores[blockIdx.x] = SWB_NEG_INF_REF;
    } else {
      counts[blockIdx.x] = cap - q;
      scores[blockIdx.x] = score;
    }
  }
  __syncwarp();
  const long long cnt = counts[blockIdx.x];
  if (cnt > 0) {
    const long long cap = (long long)n + m;
    uint8_t* o = ops + L.ops_off;
    for (long long b = 0; b < cnt; b += 32) {
      uint8_t v = 0;
      if (b + lane < cnt) v = o[cap - cnt + b + lane];
      __syncwarp();
      if (b + lane < cnt) o[b + lane] = v;
      __syncwarp();
    }
  }
}

long long mm_band_lo(long long rows, long long cols, long long score, const SchemeInt& sc,
                     long long* hi) {
  // phase3.band_interval (phase3.py:83-98); floor division as in Python
  const long long d = rows - cols;
  const long long denom = sc.max_sub + 2LL * sc.ge;
  long long num = (long long)sc.max_sub * (rows + cols) - 2 * score;
  long long g = num >= 0 ? num / denom : -((-num + denom - 1) / denom);
  const long long ad = d < 0 ? -d : d;
  if (g < ad) g = ad;
  if (g > rows + cols) g = rows + cols;
  const long long pad = (g - ad) / 2;
  *hi = std::max(0LL, d) + pad;
  return std::min(0LL, d) - pad;
}

}  // namespace

extern "C" int32_t swb_crossings(swb_ctx* ctx, const swb_scheme* scheme, int32_t seq1,
                                 int32_t seq2, const swb_subproblem* subs, int32_t n, int32_t band,
                                 swb_crossing* out, int64_t* cells_out) {
  SWB_API_BEGIN(ctx);
  if (n < 0 || (n > 0 && (!subs || !out))) return swb_fail(SWB_EINVAL, "bad arguments");
  if (n == 0) return SWB_OK;
  SchemeInt sc;
  int rc = swb_prepare_scheme(scheme, &sc);
  if (rc) return rc;
  if (seq1 < 0 || seq1 >= (int)ctx->seqs.size() || !ctx->seqs[seq1].live || seq2 < 0 ||
      seq2 >= (int)ctx->seqs.size() || !ctx->seqs[seq2].live)
    return swb_fail(SWB_EINVAL, "bad sequence id");
  const swb_seq& S1 = ctx->seqs[seq1];
  const swb_seq& S2 = ctx->seqs[seq2];

  // final-row storage: 4 int32 arrays of `cols` per subproblem
  long long total = 0;
  for (int t = 0; t < n; ++t) {
    const swb_subproblem& s = subs[t];
    const long long rows = s.ei - s.si, cols = s.ej - s.sj;
    if (rows < 2 || cols < 1 || s.si < 0 || s.sj < 0 || s.ei > S1.n || s.ej > S2.n)
      return swb_fail(SWB_EINVAL, "subproblem %d (%lld x %lld) is not splittable", t, rows, cols);
    total += 4 * cols;
  }
  int32_t* fin = (int32_t*)swb_scratch(ctx->finals, sizeof(int32_t) * (size_t)total + 256);
  if (!fin) return swb_fail(SWB_ECUDA, "out of device memory for final rows");

  std::vector<PassReq> reqs(2 * (size_t)n);
  std::vector<CombineDev> comb(n);
  long long off = 0;
  // tile-bound pruning: slack for the junction gaps and the
  // cell counted by both halves
  const bool maps = ctx->bmaps_on && seq1 == ctx->bmap_seq1 && seq2 == ctx->bmap_seq2;
  int min_sub = 0;
  for (int a = 0; a < scheme->k; ++a)
    for (int b = 0; b < scheme->k; ++b) min_sub = std::min(min_sub, scheme->sub[a * scheme->k + b]);
  const long long slack = 4LL * sc.goe + 2LL * (std::max(sc.max_sub, 0) - min_sub);
  for (int t = 0; t < n; ++t) {
    const swb_subproblem& s = subs[t];
    const int rows = (int)(s.ei - s.si), cols = (int)(s.ej - s.sj);
    const int midr = rows / 2;
    long long lo = 0, hi = 0;
    if (band) lo = mm_band_lo(rows, cols, s.expected, sc, &hi);
    PassReq& up = reqs[2 * t];
    PassReq& dn = reqs[2 * t + 1];
    // upper: seq1[si, si+midr) forward x seq2[sj, ej) forward (phase3.py:159-168)
    up.rows = S1.fwd + s.si;
    up.cols = S2.fwd + s.sj;
    up.n1 = midr;
    up.n2 = cols;
    up.border = s.start_vgap ? SWB_BORDER_GLOBAL_CONTINUE : SWB_BORDER_GLOBAL_FREE;
    up.local = false;
    up.track = kTrackNone;
    up.has_band = band != 0;
    up.band_lo = lo;
    up.band_hi = hi;
    up.want_final = true;
    up.fin_h_dev = fin + off;
    up.fin_f_dev = fin + off + cols;
    // lower: reversed seq1[si+midr, ei) x reversed seq2[sj, ej) (phase3.py:160-176)
    dn.rows = S1.rev + (S1.n - s.ei);
    dn.cols = S2.rev + (S2.n - s.ej);
    dn.n1 = rows - midr;
    dn.n2 = cols;
    dn.border = s.end_vgap ? SWB_BORDER_GLOBAL_CHARGE : SWB_BORDER_GLOBAL_FREE;
    dn.local = false;
    dn.track = kTrackNone;
    dn.has_band = band != 0;
    dn.band_lo = (long long)rows - cols - hi;
    dn.band_hi = (long long)rows - cols - lo;
    dn.want_final = true;
    dn.fin_h_dev = fin + off + 2 * cols;
    dn.fin_f_dev = fin + off + 3 * cols;
    up.force_R = dn.force_R = ctx->force_R;
    if (ctx->mm_prune) {
      // only cells that can still lie on a path of the expected score to the
      // far corner matter for the crossing (prune kind 3)
      up.prune = dn.prune = 3;
      up.prune_target = dn.prune_target = s.expected;
      up.corner_i = dn.corner_i = rows;
      up.corner_j = dn.corner_j = cols;
    }
    up.prune_target = dn.prune_target = s.expected;
    if (maps && s.use_bounds) {
      // upper half: a cell c can be on an optimal S->T path only if
      //   U(c) + R'(c) - suffix(T) + slack >= expected   (R' = phase-2 map)
      swb_bind_maps(ctx, &up, s.si, midr, false, s.sj, cols, false, 0, ctx->mm_dyn ? 2 : 0,
                    slack - s.suffix);
      // lower half: L(c) + H_fwd(c) - prefix(S) + slack >= expected (phase-1 map)
      swb_bind_maps(ctx, &dn, s.si + midr, rows - midr, true, s.sj, cols, true, 0,
                    ctx->mm_dyn ? 1 : 0, slack - s.prefix);
      // static strip ranges: a tile can hold an optimal S->T cell only if
      //   Hf(tile) + R'(tile) + slack - prefix(S) - suffix(T) >= expected
      if (ctx->mm_static)
      for (PassReq* q : {&up, &dn}) {
        q->rmap_fwd = reinterpret_cast<const int32_t*>(ctx->bmap_fwd.p);
        q->rmap_rev = reinterpret_cast<const int32_t*>(ctx->bmap_rev.p);
        q->range_offset = slack - s.prefix - s.suffix;
        // the pass is a chain along the path: its length grows with strip
        // height (rows + lag per strip at R-row step cost), so short strips
        if (!ctx->force_R && ctx->mm_R) q->force_R = ctx->mm_R;
      }
    }
    CombineDev& c = comb[t];
    c.uh = up.fin_h_dev;
    c.uf = up.fin_f_dev;
    c.dh = dn.fin_h_dev;
    c.df = dn.fin_f_dev;
    c.cols = cols;
    c.rows_up = midr;
    c.rows_dn = rows - midr;
    c.border_up = up.border;
    c.border_dn = dn.border;
    c.expected = s.expected;
    off += 4LL * cols;
  }
  double ms = 0.0;
  rc = swb_run_passes(ctx, sc, reqs, &ms);
  if (rc) return rc;
  for (int t = 0; t < n; ++t) {  // halves that ran on the int64 kernel
    CombineDev& c = comb[t];
    c.uh64 = c.uf64 = c.dh64 = c.df64 = nullptr;
    if (reqs[2 * t].wide) {
      c.uh64 = (const long long*)reqs[2 * t].fin64_h_dev;
      c.uf64 = (const long long*)reqs[2 * t].fin64_f_dev;
    }
    if (reqs[2 * t + 1].wide) {
      c.dh64 = (const long long*)reqs[2 * t + 1].fin64_h_dev;
      c.df64 = (const long long*)reqs[2 * t + 1].fin64_f_dev;
    }
  }
  long long cells = 0;
  for (auto& r : reqs) cells += r.cells;
  if (cells_out) *cells_out = cells;

  // chunks of kCombChunk columns: (subproblem, first column) per chunk, and
  // each subproblem's first chunk
  std::vector<int> chunk_sub, chunk_lo, part_off(n + 1, 0);
  for (int t = 0; t < n; ++t) {
    part_off[t] = (int)chunk_sub.size();
    for (long long lo = 0; lo <= comb[t].cols; lo += kCombChunk) {
      chunk_sub.push_back(t);
      chunk_lo.push_back((int)lo);
    }
  }
  part_off[n] = (int)chunk_sub.size();
  const size_t nch = chunk_sub.size();
  CombArena CA;
  CA.base = (char*)swb_scratch(ctx->misc, sizeof(CombineDev) * n + sizeof(CombineOut) * n +
                                              sizeof(int) * (2 * nch + n + 1) +
                                              sizeof(CombinePart) * nch + 6 * 256);
  if (!CA.base) return swb_fail(SWB_ECUDA, "out of device memory");
  CombineDev* d_comb = CA.take<CombineDev>(n);
  CombineOut* d_out = CA.take<CombineOut>(n);
  int* d_csub = CA.take<int>(nch);
  int* d_clo = CA.take<int>(nch);
  int* d_poff = CA.take<int>(n + 1);
  CombinePart* d_parts = CA.take<CombinePart>(nch);
  SWB_CUDA(cudaMemcpyAsync(d_comb, comb.data(), sizeof(CombineDev) * n, cudaMemcpyHostToDevice,
                           ctx->stream));
  SWB_CUDA(cudaMemcpyAsync(d_csub, chunk_sub.data(), sizeof(int) * nch, cudaMemcpyHostToDevice,
                           ctx->stream));
  SWB_CUDA(cudaMemcpyAsync(d_clo, chunk_lo.data(), sizeof(int) * nch, cudaMemcpyHostToDevice,
                           ctx->stream));
  SWB_CUDA(cudaMemcpyAsync(d_poff, part_off.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice,
                           ctx->stream));
  if (ctx->proto == 15) {  // the one-CTA-per-subproblem combine (A/B)
    combine_kernel<<<n, 256, 0, ctx->stream>>>(d_comb, d_out, sc.go, sc.ge);
    ctx->launches++;
  } else {
    combine_part_kernel<<<(unsigned)nch, 256, 0, ctx->stream>>>(d_comb, d_csub, d_clo, d_parts,
                                                                sc.go, sc.ge);
    combine_final_kernel<<<(n + 7) / 8, 256, 0, ctx->stream>>>(d_comb, n, d_poff, d_parts, d_out,
                                                               sc.go, sc.ge);
    ctx->launches += 2;
  }
  SWB_CUDA(cudaGetLastError());
  std::vector<CombineOut> h(n);
  SWB_CUDA(cudaMemcpyAsync(h.data(), d_out, sizeof(CombineOut) * n, cudaMemcpyDeviceToHost,
                           ctx->stream));
  SWB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int t = 0; t < n; ++t) {
    const swb_subproblem& s = subs[t];
    const int rows = (int)(s.ei - s.si);
    out[t].mid_i = s.si + rows / 2;
    out[t].mid_j = s.sj + h[t].j;
    out[t].upper = h[t].status ? h[t].best : h[t].upper;
    out[t].lower = h[t].lower;
    out[t].gap_join = h[t].gap;
    out[t].status = h[t].status;
  }
  SWB_API_END();
}

extern "C" int32_t swb_leaves(swb_ctx* ctx, const swb_scheme* scheme, int32_t seq1, int32_t seq2,
                              const swb_subproblem* leaves, int32_t n, int32_t band,
                              uint8_t* ops_out, const int64_t* ops_offsets, int64_t* counts,
                              int64_t* scores) {
  SWB_API_BEGIN(ctx);
  if (n < 0 || (n > 0 && (!leaves || !ops_out || !ops_offsets || !counts || !scores)))
    return swb_fail(SWB_EINVAL, "bad arguments");
  if (n == 0) return SWB_OK;
  SchemeInt sc;
  int rc = swb_prepare_scheme(scheme, &sc);
  if (rc) return rc;
  if (seq1 < 0 || seq1 >= (int)ctx->seqs.size() || !ctx->seqs[seq1].live || seq2 < 0 ||
      seq2 >= (int)ctx->seqs.size() || !ctx->seqs[seq2].live)
    return swb_fail(SWB_EINVAL, "bad sequence id");
  const swb_seq& S1 = ctx->seqs[seq1];
  const swb_seq& S2 = ctx->seqs[seq2];
  int32_t subv[1024];
  for (int x = 0; x < sc.k * sc.k; ++x) subv[x] = scheme->sub[x];

  long long ops_total = 0;
  for (int t = 0; t < n; ++t) {
    const swb_subproblem& s = leaves[t];
    const long long rows = s.ei - s.si, cols = s.ej - s.sj;
    if (rows < 1 || cols < 1 || s.si < 0 || s.sj < 0 || s.ei > S1.n || s.ej > S2.n)
      return swb_fail(SWB_EINVAL, "leaf %d (%lld x %lld) is empty or out of range", t, rows, cols);
    int rc2 = swb_check_range(sc, rows, cols);
    if (rc2) return rc2;
    ops_total = std::max<long long>(ops_total, ops_offsets[t] + rows + cols);
  }
  // batches bounded by matrix scratch (3 int32 matrices per leaf)
  const long long kMatCap = 1LL << 30;  // elements (4 GiB)
  uint8_t* d_ops = nullptr;
  {
    void* p = swb_scratch(ctx->results, (size_t)ops_total + 256);
    if (!p) return swb_fail(SWB_ECUDA, "out of device memory for leaf ops");
    d_ops = (uint8_t*)p;
  }
  int32_t* d_sub = nullptr;
  int t0 = 0;
  std::vector<LeafDev> L;
  while (t0 < n) {
    long long mat = 0;
    int t1 = t0;
    L.clear();
    while (t1 < n) {
      const swb_subproblem& s = leaves[t1];
      const long long rows = s.ei - s.si, cols = s.ej - s.sj;
      const long long need = 3 * (rows + 1) * (cols + 1);
      if (t1 > t0 && mat + need > kMatCap) break;
      LeafDev d;
      d.c1 = S1.fwd + s.si;
      d.c2 = S2.fwd + s.sj;
      d.n = (int)rows;
      d.m = (int)cols;
      d.svg = s.start_vgap;
      d.evg = s.end_vgap;
      long long lo, hi;
      if (band == 2) {  // explicit interval (kernels.leaf_solve's lo / hi arguments)
        lo = s.prefix;
        hi = s.suffix;
      } else if (band) {
        lo = mm_band_lo(rows, cols, s.expected, sc, &hi);
      } else {
        lo = -(rows + cols);
        hi = rows + cols;
      }
      d.lo = (int)std::max<long long>(lo, -(1LL << 30));
      d.hi = (int)std::min<long long>(hi, 1LL << 30);
      d.mat_off = mat;
      d.ops_off = ops_offsets[t1];
      L.push_back(d);
      mat += need;
      ++t1;
    }
    const int nb = t1 - t0;
    const size_t meta = sizeof(LeafDev) * nb + 2 * sizeof(long long) * nb + 1024 * 4 + 1024;
    char* base = (char*)swb_scratch(ctx->jobs, meta);
    int32_t* mats = (int32_t*)swb_scratch(ctx->progress, sizeof(int32_t) * (size_t)mat + 256);
    if (!base || !mats) return swb_fail(SWB_ECUDA, "out of device memory for leaf matrices");
    LeafDev* d_l = (LeafDev*)base;
    long long* d_cnt = (long long*)(base + ((sizeof(LeafDev) * nb + 255) & ~(size_t)255));
    long long* d_sc = d_cnt + nb;
    d_sub = (int32_t*)(d_sc + nb);
    SWB_CUDA(cudaMemcpyAsync(d_l, L.data(), sizeof(LeafDev) * nb, cudaMemcpyHostToDevice, ctx->stream));
    SWB_CUDA(cudaMemcpyAsync(d_sub, subv, sizeof(int32_t) * sc.k * sc.k, cudaMemcpyHostToDevice,
                             ctx->stream));
    leaf_kernel<<<nb, 32, 0, ctx->stream>>>(d_l, mats, d_ops, d_cnt, d_sc, d_sub, sc.k, sc.go, sc.ge);
    ctx->launches++;
    SWB_CUDA(cudaGetLastError());
    SWB_CUDA(cudaMemcpyAsync(counts + t0, d_cnt, sizeof(long long) * nb, cudaMemcpyDeviceToHost, ctx->stream));
    SWB_CUDA(cudaMemcpyAsync(scores + t0, d_sc, sizeof(long long) * nb, cudaMemcpyDeviceToHost, ctx->stream));
    SWB_CUDA(cudaStreamSynchronize(ctx->stream));
    t0 = t1;
  }
  SWB_CUDA(cudaMemcpyAsync(ops_out, d_ops, (size_t)ops_total, cudaMemcpyDeviceToHost, ctx->stream));
  SWB_CUDA(cudaStreamSynchronize(ctx->stream));
  SWB_API_END();
}
