/*
 * swb_oracle.c — TEST INFRASTRUCTURE ONLY (parity checker and CPU baseline).
 *
 * A plain-C restatement of the reference `wavealign` hot path
 * (/root/reference/pkg/src/wavealign).  Only tests/, __graft_entry__.smoke()
 * and bench.py's CPU-baseline / reference arm may load this library; the
 * product path (paper_1304_5966_b200) never does.
 *
 * Restated functions (reference file:line):
 *   orc_fill_full       oracle._fill + _matrices          oracle.py:38-109
 *   orc_local_end       oracle_local score/end            oracle.py:146-164
 *   orc_global_score    oracle_global score (+vgap)       oracle.py:167-201
 *   orc_affine_block    kernels.affine_block              kernels.py:21-88
 *   orc_run_wavefront   WavefrontEngine.run_wavefront     engine.py:188-282
 *                       borders                           engine.py:340-401
 *                       phase-1 prune hook                phase1.py:55-59
 *   orc_leaf_solve      kernels.leaf_solve                kernels.py:91-185
 *
 * All arithmetic is int64 with the reference sentinel NEG_INF = -(2**61).
 * The anti-diagonal schedule runs the blocks of one anti-diagonal on OpenMP
 * threads with a barrier between anti-diagonals; per-block bests are merged
 * in block order after the barrier and the prune best is refreshed only at
 * barriers, exactly as engine.py:216-262, so results are independent of the
 * thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define NEG_INF (-(int64_t)2305843009213693952LL)

enum { BORDER_LOCAL = 0, BORDER_RESTRICTED = 1, BORDER_FREE = 2, BORDER_CONTINUE = 3, BORDER_CHARGE = 4 };
enum { TRACK_NONE = 0, TRACK_MIN = 1, TRACK_MAX = 2 };

typedef struct {
  int64_t s, i, j;
} orc_best;

/* ---- borders, engine.py:340-401 ------------------------------------------- */

static void border_left(int border, int64_t I, int64_t go, int64_t ge, int64_t* h, int64_t* e,
                        int64_t* f) {
  *e = NEG_INF;
  switch (border) {
    case BORDER_LOCAL:
      *h = 0;
      *f = NEG_INF;
      break;
    case BORDER_RESTRICTED:
      *h = I == 0 ? 0 : NEG_INF;
      *f = NEG_INF;
      break;
    case BORDER_FREE:
      *h = I == 0 ? 0 : -go - I * ge;
      *f = I == 0 ? NEG_INF : *h;
      break;
    case BORDER_CONTINUE:
      *h = I == 0 ? NEG_INF : -I * ge;
      *f = I == 0 ? 0 : -I * ge;
      break;
    default: /* charge */
      *h = I == 0 ? NEG_INF : -go - I * ge;
      *f = I == 0 ? -go : -go - I * ge;
      break;
  }
}

void orc_top_border(int border, int64_t n2, int64_t go, int64_t ge, int64_t* top_h, int64_t* top_f) {
  for (int64_t J = 0; J <= n2; ++J) {
    top_f[J] = NEG_INF;
    switch (border) {
      case BORDER_LOCAL: top_h[J] = 0; break;
      case BORDER_RESTRICTED: top_h[J] = J == 0 ? 0 : NEG_INF; break;
      case BORDER_FREE: top_h[J] = J == 0 ? 0 : -go - J * ge; break;
      default: top_h[J] = NEG_INF; break;
    }
  }
}

/* ---- kernels.affine_block, kernels.py:21-88 ---------------------------------- */

orc_best orc_affine_block(const uint8_t* c1, const uint8_t* c2, const int64_t* sub, int k,
                          int64_t go, int64_t ge, int64_t r0, int64_t r1, int64_t cs, int64_t ce,
                          int64_t* row_h, int64_t* row_f, int64_t* col_h, int64_t* col_e,
                          int64_t corner, int clamp0, int track) {
  orc_best b;
  b.s = track == TRACK_MIN ? 0 : NEG_INF;
  b.i = b.j = -1;
  const int64_t height = r1 - r0;
  int64_t diag_top = corner;
  for (int64_t c = cs; c < ce; ++c) {
    const int64_t top = row_h[c + 1];
    int64_t f = row_f[c + 1];
    int64_t diag = diag_top, up = top;
    const int64_t* srow = sub + c2[c];
    for (int64_t q = 0; q < height; ++q) {
      const int64_t r = r0 + q;
      const int64_t lh = col_h[q], le = col_e[q];
      int64_t e = lh - go - ge, t = le - ge;
      if (t > e) e = t;
      t = up - go - ge;
      f -= ge;
      if (t > f) f = t;
      int64_t h = diag + srow[(int64_t)c1[r] * k];
      if (e > h) h = e;
      if (f > h) h = f;
      if (clamp0 && h < 0) h = 0;
      diag = lh;
      col_h[q] = h;
      col_e[q] = e;
      up = h;
      if (track == TRACK_MIN) {
        if (h > 0 && (h > b.s || (h == b.s && (r < b.i || (r == b.i && c < b.j))))) {
          b.s = h; b.i = r; b.j = c;
        }
      } else if (track == TRACK_MAX) {
        if (h > b.s || (h == b.s && (r > b.i || (r == b.i && c > b.j)))) {
          b.s = h; b.i = r; b.j = c;
        }
      }
    }
    row_h[c + 1] = up;
    row_f[c + 1] = f;
    diag_top = top;
  }
  return b;
}

/* ---- WavefrontEngine.run_wavefront, engine.py:188-282 ---------------------------- */

typedef struct {
  const uint8_t* c1;
  int64_t n1;
  const uint8_t* c2;
  int64_t n2;
  const int64_t* sub; /* k x k */
  int32_t k;
  int32_t border;
  int64_t go, ge;
  int32_t clamp0, track;
  int32_t has_band;
  int64_t band_lo, band_hi;
  int32_t prune;
  int64_t max_sub;
  int64_t fill_h;
  int64_t block_rows, block_cols;
  int32_t threads;
  int64_t* top_h; /* n2+1, in/out (becomes the final row) */
  int64_t* top_f;
  int64_t row_offset; /* DP row of this pass's row 0 within a larger pass (row slabs) */
} orc_pass;

typedef struct {
  int64_t best, bi, bj;
  int64_t total_blocks, executed, pruned, banded, cells;
} orc_result;

int orc_run_wavefront(const orc_pass* P, orc_result* out) {
  const int64_t rows = P->n1, cols = P->n2;
  if (rows < 1 || cols < 1) return -1;
  int64_t br = P->block_rows < rows ? P->block_rows : rows;
  int64_t bc = P->block_cols < cols ? P->block_cols : cols;
  if (br < 1) br = 1;
  if (bc < 1) bc = 1;
  const int64_t gr = (rows + br - 1) / br, gc = (cols + bc - 1) / bc;
  int64_t* row_h = P->top_h;
  int64_t* row_f = P->top_f;
  int64_t* col_h = (int64_t*)malloc(sizeof(int64_t) * rows);
  int64_t* col_e = (int64_t*)malloc(sizeof(int64_t) * rows);
  int64_t* corner = (int64_t*)malloc(sizeof(int64_t) * gr);
  int64_t* next_corner = (int64_t*)malloc(sizeof(int64_t) * gr);
  orc_best* res = (orc_best*)malloc(sizeof(orc_best) * gr);
  unsigned char* run = (unsigned char*)malloc(gr);
  if (!col_h || !col_e || !corner || !next_corner || !res || !run) return -2;
  for (int64_t bi = 0; bi < gr; ++bi) {
    const int64_t r0 = bi * br;
    const int64_t r1 = r0 + br < rows ? r0 + br : rows;
    int64_t h, e, f;
    border_left(P->border, P->row_offset + r0, P->go, P->ge, &h, &e, &f);
    corner[bi] = h;
    for (int64_t r = r0; r < r1; ++r) {
      border_left(P->border, P->row_offset + r + 1, P->go, P->ge, &h, &e, &f);
      col_h[r] = h;
      col_e[r] = e;
    }
  }
  orc_best best;
  best.s = P->track == TRACK_MIN ? 0 : NEG_INF;
  best.i = best.j = -1;
  int64_t barrier_best = 0, n_exec = 0, n_pruned = 0, n_banded = 0, cells = 0;
  const int64_t n_diag = gr + gc - 1;
  for (int64_t d = 0; d < n_diag; ++d) {
    const int64_t bi_lo = d - gc + 1 > 0 ? d - gc + 1 : 0;
    const int64_t bi_hi = d < gr - 1 ? d : gr - 1;
    /* skip decisions are taken before any block of the wave runs (engine.py:220-245) */
    for (int64_t bi = bi_lo; bi <= bi_hi; ++bi) {
      const int64_t bj = d - bi;
      const int64_t r0 = bi * br, r1 = r0 + br < rows ? r0 + br : rows;
      const int64_t c0 = bj * bc, c1 = c0 + bc < cols ? c0 + bc : cols;
      run[bi] = 1;
      if (P->has_band && (r0 - c1 + 1 > P->band_hi || r1 - 1 - c0 < P->band_lo)) {
        run[bi] = 2;
      } else if (P->prune) {
        int64_t m = corner[bi];
        for (int64_t c = c0 + 1; c <= c1; ++c) m = row_h[c] > m ? row_h[c] : m;
        for (int64_t r = r0; r < r1; ++r) m = col_h[r] > m ? col_h[r] : m;
        const int64_t remaining = (rows - r0) < (cols - c0) ? (rows - r0) : (cols - c0);
        const int64_t inm = m > 0 ? m : 0;
        if (inm + P->max_sub * remaining < barrier_best) run[bi] = 3;
      }
      next_corner[bi] = row_h[c1]; /* pkg.corner = row_h[c1] (engine.py:288, :299) */
    }
#pragma omp parallel for schedule(dynamic, 1) num_threads(P->threads > 0 ? P->threads : 1)
    for (int64_t bi = bi_lo; bi <= bi_hi; ++bi) {
      const int64_t bj = d - bi;
      const int64_t r0 = bi * br, r1 = r0 + br < rows ? r0 + br : rows;
      const int64_t c0 = bj * bc, c1 = c0 + bc < cols ? c0 + bc : cols;
      if (run[bi] == 1) {
        res[bi] = orc_affine_block(P->c1, P->c2, P->sub, P->k, P->go, P->ge, r0, r1, c0, c1, row_h,
                                   row_f, col_h + r0, col_e + r0, corner[bi], P->clamp0, P->track);
      } else {
        /* _skip, engine.py:286-293 */
        for (int64_t c = c0 + 1; c <= c1; ++c) {
          row_h[c] = P->fill_h;
          row_f[c] = NEG_INF;
        }
        for (int64_t r = r0; r < r1; ++r) {
          col_h[r] = P->fill_h;
          col_e[r] = NEG_INF;
        }
      }
    }
    for (int64_t bi = bi_lo; bi <= bi_hi; ++bi) {
      const int64_t bj = d - bi;
      const int64_t r0 = bi * br, r1 = r0 + br < rows ? r0 + br : rows;
      const int64_t c0 = bj * bc, c1 = c0 + bc < cols ? c0 + bc : cols;
      corner[bi] = next_corner[bi];
      if (run[bi] == 2) { ++n_banded; continue; }
      if (run[bi] == 3) { ++n_pruned; continue; }
      ++n_exec;
      cells += (r1 - r0) * (c1 - c0);
      const orc_best b = res[bi];
      if (P->track == TRACK_MIN) {
        if (b.s > 0 && (b.s > best.s || (b.s == best.s && (b.i < best.i || (b.i == best.i && b.j < best.j)))))
          best = b;
      } else if (P->track == TRACK_MAX) {
        if (b.i >= 0 && (b.s > best.s || (b.s == best.s && (b.i > best.i || (b.i == best.i && b.j > best.j)))))
          best = b;
      }
    }
    if (P->prune && best.s > barrier_best) barrier_best = best.s;
  }
  {
    int64_t h, e, f;
    border_left(P->border, P->row_offset + rows, P->go, P->ge, &h, &e, &f);
    row_h[0] = h;
    row_f[0] = f;
  }
  out->best = best.s;
  out->bi = best.i;
  out->bj = best.j;
  out->total_blocks = gr * gc;
  out->executed = n_exec;
  out->pruned = n_pruned;
  out->banded = n_banded;
  out->cells = cells;
  free(col_h);
  free(col_e);
  free(corner);
  free(next_corner);
  free(res);
  free(run);
  return 0;
}

/* ---- full-matrix oracle, oracle.py:38-109, :146-201 --------------------------------- */

/* mode: 0 local, 1 affine (global), 2 pinned; start_vgap per oracle.py:93-105.
 * H/E/F are caller-owned (n1+1)*(n2+1) int64 arrays. */
int orc_fill_full(const uint8_t* c1, int64_t n1, const uint8_t* c2, int64_t n2, const int64_t* sub,
                  int32_t k, int64_t go, int64_t ge, int32_t mode, int32_t start_vgap, int64_t* H,
                  int64_t* E, int64_t* F) {
  const int64_t W = n2 + 1;
  for (int64_t x = 0; x < (n1 + 1) * W; ++x) H[x] = E[x] = F[x] = NEG_INF;
  if (mode == 0) {
    for (int64_t j = 0; j <= n2; ++j) H[j] = 0;
    for (int64_t i = 0; i <= n1; ++i) H[i * W] = 0;
  } else if (mode == 1) {
    H[0] = 0;
    for (int64_t j = 1; j <= n2; ++j) H[j] = E[j] = -go - j * ge;
    for (int64_t i = 1; i <= n1; ++i) H[i * W] = F[i * W] = -go - i * ge;
  } else {
    H[0] = 0;
  }
  if (start_vgap) {
    for (int64_t j = 0; j <= n2; ++j) H[j] = E[j] = F[j] = NEG_INF;
    F[0] = 0;
    for (int64_t i = 1; i <= n1; ++i) {
      F[i * W] = H[i * W] = -i * ge;
      E[i * W] = NEG_INF;
    }
  }
  for (int64_t i = 1; i <= n1; ++i) {
    for (int64_t j = 1; j <= n2; ++j) {
      int64_t e = H[i * W + j - 1] - go - ge, t = E[i * W + j - 1] - ge;
      if (t > e) e = t;
      int64_t f = H[(i - 1) * W + j] - go - ge;
      t = F[(i - 1) * W + j] - ge;
      if (t > f) f = t;
      int64_t h = H[(i - 1) * W + j - 1] + sub[(int64_t)c1[i - 1] * k + c2[j - 1]];
      if (e > h) h = e;
      if (f > h) h = f;
      if (mode == 0 && h < 0) h = 0;
      E[i * W + j] = e;
      F[i * W + j] = f;
      H[i * W + j] = h;
    }
  }
  return 0;
}

/* Linear-memory local score and lexicographically smallest end (oracle.py:146-164:
 * row-major argmax of H).  Returns score; end written as (ei, ej) in DP indices. */
int64_t orc_local_end(const uint8_t* c1, int64_t n1, const uint8_t* c2, int64_t n2, const int64_t* sub,
                      int32_t k, int64_t go, int64_t ge, int64_t* ei, int64_t* ej) {
  int64_t* Hr = (int64_t*)malloc(sizeof(int64_t) * (n2 + 1));
  int64_t* Fr = (int64_t*)malloc(sizeof(int64_t) * (n2 + 1));
  for (int64_t j = 0; j <= n2; ++j) {
    Hr[j] = 0;
    Fr[j] = NEG_INF;
  }
  int64_t best = 0, bi = 0, bj = 0;
  for (int64_t i = 1; i <= n1; ++i) {
    int64_t diag = 0, hleft = 0, e = NEG_INF;
    const int64_t* srow = sub + (int64_t)c1[i - 1] * k;
    for (int64_t j = 1; j <= n2; ++j) {
      int64_t t = e - ge, en = hleft - go - ge;
      e = t > en ? t : en;
      int64_t f = Fr[j] - ge, fn = Hr[j] - go - ge;
      f = f > fn ? f : fn;
      int64_t h = diag + srow[c2[j - 1]];
      if (e > h) h = e;
      if (f > h) h = f;
      if (h < 0) h = 0;
      diag = Hr[j];
      Hr[j] = h;
      Fr[j] = f;
      hleft = h;
      if (h > best) {
        best = h;
        bi = i;
        bj = j;
      }
    }
  }
  free(Hr);
  free(Fr);
  *ei = bi;
  *ej = bj;
  return best;
}

/* ---- kernels.leaf_solve, kernels.py:91-185 ----------------------------------------------- */

int64_t orc_leaf_solve(const uint8_t* c1, int64_t n, const uint8_t* c2, int64_t m, const int64_t* sub,
                       int32_t k, int64_t go, int64_t ge, int32_t start_vgap, int32_t end_vgap,
                       int64_t lo, int64_t hi, uint8_t* ops_out, int64_t cap, int64_t* count) {
  const int64_t W = m + 1;
  int64_t* H = (int64_t*)malloc(sizeof(int64_t) * (n + 1) * W);
  int64_t* E = (int64_t*)malloc(sizeof(int64_t) * (n + 1) * W);
  int64_t* F = (int64_t*)malloc(sizeof(int64_t) * (n + 1) * W);
  for (int64_t x = 0; x < (n + 1) * W; ++x) H[x] = E[x] = F[x] = NEG_INF;
  if (start_vgap) {
    F[0] = 0;
    for (int64_t i = 1; i <= n; ++i) F[i * W] = H[i * W] = -i * ge;
  } else {
    H[0] = 0;
    for (int64_t j = 1; j <= m; ++j) E[j] = H[j] = -go - j * ge;
    for (int64_t i = 1; i <= n; ++i) F[i * W] = H[i * W] = -go - i * ge;
  }
  for (int64_t i = 1; i <= n; ++i) {
    int64_t jlo = i - hi, jhi = i - lo;
    if (jlo < 1) jlo = 1;
    if (jhi > m) jhi = m;
    for (int64_t j = jlo; j <= jhi; ++j) {
      int64_t e = H[i * W + j - 1] - go - ge, t = E[i * W + j - 1] - ge;
      if (t > e) e = t;
      int64_t f = H[(i - 1) * W + j] - go - ge;
      t = F[(i - 1) * W + j] - ge;
      if (t > f) f = t;
      int64_t h = H[(i - 1) * W + j - 1] + sub[(int64_t)c1[i - 1] * k + c2[j - 1]];
      if (e > h) h = e;
      if (f > h) h = f;
      E[i * W + j] = e;
      F[i * W + j] = f;
      H[i * W + j] = h;
    }
  }
  int64_t score;
  int state;
  if (end_vgap) {
    score = F[n * W + m];
    state = 2;
  } else {
    score = H[n * W + m];
    state = 0;
  }
  int64_t i = n, j = m, q = cap;
  int dead = 0;
  while ((i > 0 || j > 0) && !dead) {
    if (state == 0) {
      if (i > 0 && j > 0 && H[i * W + j] == H[(i - 1) * W + j - 1] + sub[(int64_t)c1[i - 1] * k + c2[j - 1]]) {
        ops_out[--q] = c1[i - 1] == c2[j - 1] ? 0 : 1;
        --i;
        --j;
      } else if (j > 0 && H[i * W + j] == E[i * W + j]) {
        state = 1;
      } else if (i > 0 && H[i * W + j] == F[i * W + j]) {
        state = 2;
      } else {
        dead = 1;
      }
    } else if (state == 1) {
      ops_out[--q] = 2;
      if (E[i * W + j] == H[i * W + j - 1] - go - ge) state = 0;
      else if (E[i * W + j] != E[i * W + j - 1] - ge) dead = 1;
      --j;
    } else {
      ops_out[--q] = 3;
      if (F[i * W + j] == H[(i - 1) * W + j] - go - ge) state = 0;
      else if (F[i * W + j] != F[(i - 1) * W + j] - ge) dead = 1;
      --i;
    }
  }
  free(H);
  free(E);
  free(F);
  if (dead) {
    *count = -1;
    return NEG_INF;
  }
  const int64_t cnt = cap - q;
  memmove(ops_out, ops_out + q, (size_t)cnt);
  *count = cnt;
  return score;
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
