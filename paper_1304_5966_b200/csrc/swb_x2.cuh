// Packed 16x2 score pass (phase 1 fast path).
//
// One warp runs a 64-lane virtual pipeline: the low 16 bits of every register
// hold strip A (rows [R0, R0 + 32R)), the high 16 bits strip B (the next 32R
// rows).  Lane l processes column s - l of A and column s - l - 32 of B at step
// s, so B's lane 0 consumes A's lane 31 output of the previous step and B's
// bottom row is the item's output to the next warp.  Every DP instruction is a
// DPX S16x2 op or a carry-free 32-bit IMAD on two 16-bit fields, i.e. two
// cells per instruction (5 ALU-pipe + 2 FMA-pipe instructions per cell pair):
//
//   s   = PRMT(T[colA], T[colB], sel_r)           two zero-extended bytes (sub + go + ge)
//   ds  = IMAD(hm_diag, 1, s)                     packed add, no carry (fields in [0, 32767])
//   h2  = VIMNMX3.S16x2(ds, E, FLOOR)             max(diag + sub, E, floor)
//   F   = VIADDMNMX.S16x2(F, -ge, h2m_above)
//   h2m = IMAD(h2, 1, -(go+ge) packed)            packed subtract, no borrow (h2 >= FLOOR)
//   hm  = VIADDMNMX.S16x2(F, -(go+ge), h2m)
//   E'  = VIADDMNMX.S16x2(E, -ge, hm)
//
// Values are stored relative to a warp-wide base: rel = abs - base + 1024.
// FLOOR (rel 1024) is abs max(0, base): with base = 0 it is the local-alignment
// clamp at 0 exactly; with base > 0 it only raises values that lie more than
// 26000 below the warp's maximum, which no true value in the warp's window can:
// by induction over rows and columns, neighbouring cells of H (and E, F against
// their H) differ by at most max_sub + go + ge, the window spans at most 1024
// rows + W columns (W = BLK + 63, BLK = 64 steps per block), and the host only
// selects this kernel when (1025 + W)(go + ge + max_sub) + BLK max_sub + go + ge
// <= 25000.  So no value is ever clamped by the frame and every value is exact
// (DESIGN.md §3.5).  The base is re-chosen every block from the warp maximum
// and the incoming top row.
//
// Endpoint tracking (reference TRACK_MIN: largest score, then smallest row,
// then smallest column) uses packed 16-bit keys relative to a per-block
// reference V_ref = max(V, M + W max_sub - 1022) of each lane half, V its
// running best and M the warp maximum at the block start:
//   key = 32 * max(hm - V_ref + 1, 0) + (31 - r).
// No cell of the W-column block exceeds M + W max_sub, so keys stay below
// 32768 and are exact; cells below V_ref are below M, hence strictly below the
// final best, and cannot be the endpoint.  Each step folds its keys into a
// running maximum that is also stored to shared memory; at the end of each
// 32-step half of a block a lane half whose maximum beats its best's key
// (32 + rank, or 31 when V_ref > V) binary-searches the stored maxima for the
// first step that reached it, and the keys are re-framed on the new best.
// Requires W max_sub <= 1021.
//
// The producer's row enters through lane 0 as IMAD(shfl(x), 65536, top): the
// shuffle from lane 31 moves A's bottom into B's half while the top value
// fills A's half; the other lanes compute IMAD(shfl(x), 1, 0).
//
// Scope: local passes, TRACK_MIN, no band, no final rows, alphabets of <= 4
// codes with 0 <= sub + go + ge <= 127 (plus a fifth code that scores the same
// against every column: the default DNA alphabet's 'N', WILD instantiation),
// whole passes or row slabs whose rows are a multiple of 64R.  Everything else
// uses run_strip.
#pragma once

#include "swb_kernels.cuh"

namespace swb {

constexpr int kX2Off = 1024;     // rel value of the floor
constexpr int kX2Span = 26000;   // max - base kept below this
constexpr int kX2KeyRoom = 1022; // key t field stays <= 1023
// Tile edge of the bound maps this kernel writes: a compile-time 1024 (the
// runtime edge of swb_kernels.cuh cost 5 % of an unrelated pass here through
// register allocation, even unexecuted); the host keeps other edges off it.
constexpr int kX2MapShift = 10;
// Steps per block BLK (one producer handoff, one release, one re-base per
// block): 32, or 64 for passes of several rounds of items (the host's choice,
// swb_pass.cu); a 64-step block tracks in two 32-step halves (keys resolved
// per half).  A block's skewed window spans BLK + 63 columns.
template <int BLK>
struct WarpSmemX2 {
  static_assert(BLK == 32 || BLK == 64, "packed block length");
  uint32_t prof[BLK + 64];  // profile word of column s0 - 64 + w (0 outside [0, n2))
  int2 tz[2 * BLK];         // [0, BLK): rel (h, f) of the producer's row at s0 + k; then 0
  uint2 out[BLK];           // raw packed (hm, F) of lane 31 at step k (B's bottom row)
  uint32_t trk[32][32];     // [k][lane]: running packed key maximum after step k (per half)
};
// per CTA of `warps` warps: the warps' areas, then the 8 profile words
template <int BLK>
__host__ __device__ constexpr size_t x2_smem_bytes(int warps) {
  return (size_t)warps * sizeof(WarpSmemX2<BLK>) + 64;
}
// host eligibility of a scheme for block length blk (header: keys and frame)
__host__ __device__ constexpr bool x2_frame_ok(int blk, long long goe, long long ms) {
  return (blk + 63) * ms <= 1021 && (1025LL + blk + 63) * (goe + ms) + blk * ms + goe <= 25000;
}

__device__ __forceinline__ uint32_t vimax3_2(uint32_t a, uint32_t b, uint32_t c) {
  return (uint32_t)__vimax3_s16x2((int)a, (int)b, (int)c);
}
__device__ __forceinline__ uint32_t viaddmax_2(uint32_t a, uint32_t b, uint32_t c) {
  return (uint32_t)__viaddmax_s16x2((int)a, (int)b, (int)c);
}
__device__ __forceinline__ uint32_t viaddmax_relu_2(uint32_t a, uint32_t b, uint32_t c) {
  return (uint32_t)__viaddmax_s16x2_relu((int)a, (int)b, (int)c);
}
__device__ __forceinline__ uint32_t pack2(int lo, int hi) {
  return ((uint32_t)lo & 0xffffu) | ((uint32_t)hi << 16);
}
__device__ __forceinline__ int lo16(uint32_t x) { return (int)(short)(x & 0xffffu); }
__device__ __forceinline__ int hi16(uint32_t x) { return (int)x >> 16; }
__device__ __forceinline__ int clamp_rel(long long v) {
  return v < 0 ? 0 : (v > 32767 ? 32767 : (int)v);
}

template <int R, bool WILD, bool FINAL, int BLK>
__device__ __forceinline__ void run_strip_x2(const PassParams& P, const JobDev& Jg, int s,
                                          WarpSmemX2<BLK>* sm, const uint32_t* __restrict__ tw_s) {
  constexpr int kX2Blk = BLK;
  constexpr int kX2Win = BLK + 63;  // columns a block's skewed window spans
  static_assert(R <= 32, "rank field is 5 bits");
  // by-value copy of the job descriptor: its fields live in registers in the
  // hot loop (a reference instead: 192 registers, but C2 246 -> 263 ms); the
  // 304-byte stack frame is written once per strip
  const JobDev J = Jg;
  const int lane = threadIdx.x & 31;
  const int goe = P.goe, ge = P.ge;
  const int n1 = J.n1, n2 = J.n2;
  const int R0 = s * 64 * R;
  const int rowA = R0 + lane * R;
  const int rowB = R0 + 32 * R + lane * R;
  const int2* __restrict__ inbuf = J.buf[(s + 1) & 1];
  int2* __restrict__ outbuf = J.buf[s & 1];
  int32_t* my_progress = J.progress + (long long)s * kProgStride;
  const int32_t* up_progress = s > 0 ? J.progress + (long long)(s - 1) * kProgStride : nullptr;
  // multi-GPU row slab: item 0 consumes the slab above, the
  // last item produces into the slab below through peer memory (sys scope)
  const bool ext_in = (s == 0) && (J.ext_in != nullptr);
  const bool ext_out = (s == J.nstrips - 1) && (J.ext_out != nullptr);
  const bool has_top = s > 0 || ext_in;
  if (ext_in) {
    inbuf = J.ext_in;
    up_progress = J.ext_in_prog;
  }
  if (ext_out) {
    outbuf = J.ext_out;
    my_progress = J.ext_out_prog;
  }

  // selectors: byte0 <- T[colA] byte a, byte2 <- T[colB] byte b, bytes 1 and 3
  // replicate the (zero) sign of a profile byte; padding rows select zeros.
  // WILD: code-4 rows select zeros like padding rows and take the scheme's
  // constant through wadj (added with the diagonal), so a profile word still
  // holds 4 codes.
  uint32_t sel[R];
  uint32_t wadj[WILD ? R : 1];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int ia = rowA + r, ib = rowB + r;
    uint32_t a = (ia < n1) ? (uint32_t)J.rows[(long long)ia * J.rstep] : 8u;
    uint32_t b = (ib < n1) ? 4u + (uint32_t)J.rows[(long long)ib * J.rstep] : 8u;
    if (WILD) {
      wadj[r] = (a == 4u ? (uint32_t)P.wild_const : 0u) | (b == 8u && ib < n1 ? (uint32_t)P.wild_const << 16 : 0u);
      if (a == 4u) a = 8u;
    }
    sel[r] = a | ((a | 8u) << 4) | (b << 8) | ((b | 8u) << 12);
  }
  // Every profile word an inactive half may read must be a valid one: a byte
  // >= 128 would be sign-replicated by PRMT and its carry in the packed IMAD
  // add would reach the other half.
  for (int q = lane; q < kX2Blk + 64; q += 32) sm->prof[q] = 0u;
  for (int q = lane; q < kX2Blk; q += 32) sm->tz[kX2Blk + q] = make_int2(0, 0);
  __syncwarp();

  const uint32_t FLOOR2 = pack2(kX2Off, kX2Off);
  const uint32_t ZERO2 = 0u;
  const uint32_t NGE2 = pack2(-ge, -ge);
  const uint32_t NGOE2 = pack2(-goe, -goe);
  const int NGOE32 = -(goe * 65536 + goe);  // carry-free packed subtract of goe
  const int k32 = P.key_mul;
  const int up_mul = lane == 0 ? 65536 : 1;
  const int src_lane = (lane + 31) & 31;
  const int tz_off = lane == 0 ? 0 : kX2Blk;
  uint32_t rk[R];
#pragma unroll
  for (int r = 0; r < R; ++r) rk[r] = (uint32_t)(31 - r) * 0x10001u;

  int base = 0;
  // local left border: H = 0 -> hm = -goe; E = max(NEG - ge, hm) = hm
  const uint32_t hm0 = pack2(kX2Off - goe, kX2Off - goe);
  uint32_t H[R], H2[R], E[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    H[r] = hm0;
    H2[r] = hm0;
    E[r] = hm0;
  }
  uint32_t diag = hm0;
  uint32_t out_hm = hm0, out_f = 0u;

  // running best per half: hm value (absolute), rank 31 - r, column
  int vA = -goe, vB = -goe, rkA = 31, rkB = 31;
  int bjA = -1, bjB = -1;
  // per-block key frame: V_ref per half, 1 - V_ref(rel) and the best's key
  long long vrA = 0, vrB = 0;
  uint32_t nv2 = 0u, kb2 = 0u, bk2 = 0u;
  uint32_t bmax2 = 0u;   // optimistic blocks: packed maximum of E every 4th step
  int opt_cool = 0;      // candidate blocks to track directly after a hit
  auto set_frame = [&](long long mabs_w) {
    const long long lowv = mabs_w + (long long)kX2Win * P.max_sub - kX2KeyRoom;
    vrA = vA > lowv ? vA : lowv;
    vrB = vB > lowv ? vB : lowv;
    long long ra = vrA - base + kX2Off, rb = vrB - base + kX2Off;
    ra = ra < 0 ? 0 : (ra > 32767 ? 32767 : ra);
    rb = rb < 0 ? 0 : (rb > 32767 ? 32767 : rb);
    nv2 = pack2(1 - (int)ra, 1 - (int)rb);
    kb2 = pack2(vrA == vA ? 32 + rkA : 31, vrB == vB ? 32 + rkB : 31);
    bk2 = kb2;
  };

  BoundWriter bw;  // tile bound map of this pass's H
  if (J.bmap_out) {
    const int r_hi = (R0 + 64 * R < n1 ? R0 + 64 * R : n1) - 1;
    tile_range(J.map_r0, J.map_rdir, R0, r_hi, J.map_nr, kX2MapShift, bw.rt_lo, bw.rt_hi);
  }

  // FINAL (last item of a pass that wants its final rows, split mode): the lane,
  // packed row and half holding DP row n1 write (H, F) of every column they
  // compute; skipped cells keep the fill values written before the launch
  int lstar = -1, rstar = 0, hstar = 0;
  if (FINAL) {
    const int off = n1 - 1 - R0;
    hstar = off >= 32 * R ? 1 : 0;
    const int o2 = off - hstar * 32 * R;
    lstar = o2 / R;
    rstar = o2 % R;
  }

  int known_prog = 0, prune_seen = 0, published = 0;
  constexpr int NH = kX2Blk / 32;  // 32-column slices per block
  int code_next[NH];
#pragma unroll
  for (int h = 0; h < NH; ++h)
    code_next[h] = (32 * h + lane < n2) ? (int)J.cols[(long long)(32 * h + lane) * J.cstep] : 0;
  long long pruned_blocks = 0, exec_blocks = 0, wait_cycles = 0;
  const long long t_strip0 = clock64();
  unsigned long long g0, gw = 0, g_diag = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  const int s_end = n2 + 63;

  auto step = [&](const int k, const int st, const bool guard, uint32_t (&Hin)[R],
                  uint32_t (&Hout)[R], auto trk_tag) {
    constexpr int MODE = decltype(trk_tag)::value;  // 0 untracked, 1 keys, 2 optimistic (= 0 here)
    constexpr bool TRK = MODE == 1;
    const int colA = st - lane, colB = colA - 32;
    const int2 tp = sm->tz[SWB_IX(tz_off + k, 2 * BLK)];
    const uint32_t tl = sm->prof[SWB_IX(64 - lane + k, BLK + 64)],
                   th = sm->prof[SWB_IX(32 - lane + k, BLK + 64)];
    const uint32_t up_h =
        (uint32_t)imad((int)__shfl_sync(0xffffffffu, out_hm, src_lane), up_mul, tp.x);
    const uint32_t up_f =
        (uint32_t)imad((int)__shfl_sync(0xffffffffu, out_f, src_lane), up_mul, tp.y);
    const bool actA = !guard || (colA >= 0 && colA < n2);
    const bool actB = !guard || (colB >= 0 && colB < n2);
    if (guard && !actA && !actB) {
#pragma unroll
      for (int r = 0; r < R; ++r) Hout[r] = Hin[r];
      if (TRK) sm->trk[SWB_IX(k & 31, 32)][lane] = bk2;
      return;
    }
    const uint32_t keep = guard ? ((actA ? 0u : 0xffffu) | (actB ? 0u : 0xffff0000u)) : 0u;
    uint32_t d = diag;
    diag = guard ? ((up_h & ~keep) | (diag & keep)) : up_h;
    uint32_t fv = up_f;
    uint32_t hab = up_h;
    uint32_t cm = guard ? 0u : bk2, kp = 0u;
    uint32_t fh = 0u, ff = 0u;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t sv = prmt(tl, th, sel[r]);
      const uint32_t ds = WILD ? d + sv + wadj[r] : (uint32_t)imad((int)d, 1, (int)sv);
      const uint32_t h2 = vimax3_2(ds, E[r], FLOOR2);
      fv = viaddmax_2(fv, NGE2, hab);
      const uint32_t h2m = (uint32_t)imad((int)h2, 1, NGOE32);
      const uint32_t hm = viaddmax_2(fv, NGOE2, h2m);
      const uint32_t en = viaddmax_2(E[r], NGE2, hm);
      E[r] = guard ? ((en & ~keep) | (E[r] & keep)) : en;
      d = Hin[r];
      Hout[r] = guard ? ((hm & ~keep) | (Hin[r] & keep)) : hm;
      hab = h2m;
      if (FINAL && r == rstar) {
        fh = hm;
        ff = fv;
      }
      if (TRK) {
        const uint32_t t = viaddmax_relu_2(hm, nv2, NGE2);  // any c <= 0: max(hm + nv, 0)
        const uint32_t key = (uint32_t)imad((int)t, k32, (int)rk[r]);
        if (r & 1) cm = vimax3_2(cm, kp, key);
        else if (r == R - 1) cm = vimax3_2(cm, key, key);
        kp = key;
      }
    }
    out_hm = Hout[R - 1];
    out_f = fv;
    if (TRK) {
      bk2 = guard ? vimax3_2(bk2, cm & ~keep, 0u) : cm;
      sm->trk[SWB_IX(k & 31, 32)][lane] = bk2;
    }
    if (lane == 31 && actB) sm->out[SWB_IX(k, BLK)] = make_uint2(out_hm, out_f);
    if (FINAL && lane == lstar) {
      const int col = hstar ? colB : colA;
      if (col >= 0 && col < n2) {
        const int off = base - kX2Off;
        J.fin_h[SWB_IX(col, n2)] = (hstar ? hi16(fh) : lo16(fh)) + off + goe;
        J.fin_f[SWB_IX(col, n2)] = (hstar ? hi16(ff) : lo16(ff)) + off;
      }
    }
  };

  // Diagnostics (proto 16 / 17): start the item only once its producer leads
  // by 96 / 160 columns, i.e. with more slack in the chain (C2 -0.7 %,
  // unrelated +2 / +6 %: off by default)
  if ((P.proto == 16 || P.proto == 17) && has_top) {
    const int lead = P.proto == 16 ? 96 : 160;
    wait_progress(up_progress, lead < n2 ? lead : n2, ext_in);
  }
  for (int s0 = 0; s0 < s_end; s0 += kX2Blk) {
    // (1) wait for and read the producer's bottom row for [s0, s0 + BLK); shift
    //     the profile window and stage the new columns' words
    int top_h[NH], top_f[NH];
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      top_h[h] = -goe;  // local top border: H = 0, F = -inf
      top_f[h] = SWB_NEG32;
    }
    // The running best also decides tracking, so it is kept with pruning off.
    // It steers skip / tracking around the shuffling steps, so it must be the
    // same in every lane (a lane that skipped while the others ran would pair
    // its shuffles with theirs): the warp reconverges and loads it with ONE
    // warp-wide load of one address, which returns one value to all lanes.
    // (A broadcast or vote here measured 3-4 % slower on C2.)
    __syncwarp();
    prune_seen = load_best(J);
    {
      int code[NH];
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        code[h] = code_next[h];
        const int cn = s0 + kX2Blk + 32 * h + lane;
        code_next[h] = (cn < n2) ? (int)J.cols[SWB_IX((long long)cn * J.cstep, (long long)n2 * J.cstep)] : 0;
      }
      if (has_top && s0 < n2) {
        const int need = (s0 + kX2Blk < n2) ? s0 + kX2Blk : n2;
        if (known_prog < need) {
          // one acquiring load when the producer is already ahead (the common
          // case off the chain); poll relaxed only when it is not
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
        }
      }
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const int c = s0 + 32 * h + lane;
        if (has_top && c < n2) {
          const int2 v = __ldcg(inbuf + SWB_IX(c, n2));
          top_h[h] = v.x;
          top_f[h] = v.y;
        }
      }
      // keep the window's last 64 columns, then the block's new ones
      const uint32_t p1 = sm->prof[SWB_IX(kX2Blk + lane, BLK + 64)],
                     p2 = sm->prof[SWB_IX(kX2Blk + 32 + lane, BLK + 64)];
      __syncwarp();
      sm->prof[lane] = p1;
      sm->prof[32 + lane] = p2;
#pragma unroll
      for (int h = 0; h < NH; ++h)
        sm->prof[SWB_IX(64 + 32 * h + lane, BLK + 64)] = s0 + 32 * h + lane < n2 ? tw_s[SWB_IX(code[h], 8)] : 0u;
    }

    // (1b) re-base: warp maximum over the state and the incoming top row
    int mrel = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      mrel = __vimax3_s32(mrel, lo16(H[r]), hi16(H[r]));
    }
    mrel = __vimax3_s32(mrel, lo16(out_hm), hi16(out_hm));
    long long mabs = (long long)mrel + base - kX2Off;  // hm (H - go - ge), absolute
#pragma unroll
    for (int h = 0; h < NH; ++h)
      if (s0 + 32 * h + lane < n2 && (long long)top_h[h] > mabs) mabs = top_h[h];
    const int mabs_w = __reduce_max_sync(0xffffffffu, (int)(mabs > INT32_MAX ? INT32_MAX : mabs));
    {
      long long nb = (long long)mabs_w + goe - kX2Span;
      if (nb < 0) nb = 0;
      if (nb != base) {
        // shift by -(nb - base) per field, clamping at rel 0 (a lower bound, see header)
        long long rem = nb - base;
        while (rem != 0) {
          const int d2 = rem > 32767 ? 32767 : (rem < -32767 ? -32767 : (int)rem);
          const uint32_t sh = pack2(-d2, -d2);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            H[r] = viaddmax_2(H[r], sh, ZERO2);
            E[r] = viaddmax_2(E[r], sh, ZERO2);
          }
          diag = viaddmax_2(diag, sh, ZERO2);
          out_hm = viaddmax_2(out_hm, sh, ZERO2);
          out_f = viaddmax_2(out_f, sh, ZERO2);
          rem -= d2;
        }
        base = (int)nb;
      }
    }
    // the producer's row in this block's frame (lane 0 injects it at step k)
#pragma unroll
    for (int h = 0; h < NH; ++h)
      sm->tz[SWB_IX(32 * h + lane, 2 * BLK)] = make_int2(clamp_rel((long long)top_h[h] - base + kX2Off),
                                        clamp_rel((long long)top_f[h] - base + kX2Off));
    __syncwarp();
    const bool steady = (s0 >= 63) && (s0 + kX2Blk <= n2);
    if (P.proto == 10 && g_diag == 0 && s0 + kX2Blk > R0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_diag));

    // (2) pruning / tracking decision on the block's skewed window
    bool skip = false, track_block = true;
    if (steady) {
      const long long inm = (long long)mabs_w + goe;
      const long long ms = P.max_sub;
      track_block = (inm > 0 ? inm : 0) + (long long)kX2Win * ms >= (long long)prune_seen;
      if (J.prune == 1) {
        const int rem_r = n1 - R0 + J.rows_after;
        const int rem_c = n2 - (s0 - 63);
        const long long bound = (inm > 0 ? inm : 0) + ms * (long long)(rem_r < rem_c ? rem_r : rem_c);
        skip = bound < (long long)prune_seen;
      }
    }

    if (J.bmap_out) {
      const int lo = s0 - 63 > 0 ? s0 - 63 : 0;
      const int hi = s0 + kX2Blk - 1 < n2 - 1 ? s0 + kX2Blk - 1 : n2 - 1;
      if (lo <= hi) {
        int ta, tb;
        tile_range(J.map_c0, J.map_cdir, lo, hi, J.map_nc, kX2MapShift, ta, tb);
        const long long inm = (long long)mabs_w + goe;
        bw_add(J, bw, ta, tb, (inm > 0 ? inm : 0) + (long long)kX2Win * P.max_sub, lane);
      }
    }

    if (skip) {
      ++pruned_blocks;
      // fill: H = 0 (hm = -goe), E/F = -inf (clamped at the floor)
      const int hf = clamp_rel((long long)-goe - base + kX2Off);
      const uint32_t fill = pack2(hf, hf);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        H[r] = fill;
        E[r] = fill;
      }
      // lane 0's next diagonal is the real top input of the block's last column
      diag = fill;
      if (lane == 0) diag = pack2(sm->tz[kX2Blk - 1].x, hf);
      out_hm = fill;
      out_f = 0u;
    } else {
      ++exec_blocks;
      const bool trk_on = !steady || track_block;
      if (trk_on) set_frame(mabs_w);
      using T1 = std::integral_constant<int, 1>;
      using T0 = std::integral_constant<int, 0>;
      using T2 = std::integral_constant<int, 2>;
      bool tracked_run = true;
      if (steady && track_block && opt_cool == 0) {
        // Optimistic: the block can only matter if one of its cells reaches
        // the running best (a smaller cell is never the endpoint).  Run it
        // untracked with an upper bound of its maximum and re-run it tracked
        // from the saved state if the bound reaches the best.
        uint32_t Hs[R], Es[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          Hs[r] = H[r];
          Es[r] = E[r];
        }
        const uint32_t diag_s = diag, ohm_s = out_hm, of_s = out_f;
        // E' = max(E - ge, hm) >= hm, so E after step k + 3 bounds hm of steps
        // k .. k + 3 from above within 3 ge: one packed maximum of E every
        // four steps bounds the block's maximum (0.125 instead of 0.5 ALU per pair)
        bmax2 = 0u;
#pragma unroll 1
        for (int k = 0; k < kX2Blk; k += 4) {
          step(k, s0 + k, false, H, H2, T2{});
          step(k + 1, s0 + k + 1, false, H2, H, T2{});
          step(k + 2, s0 + k + 2, false, H, H2, T2{});
          step(k + 3, s0 + k + 3, false, H2, H, T2{});
#pragma unroll
          for (int r = 0; r + 1 < R; r += 2) bmax2 = vimax3_2(bmax2, E[r], E[r + 1]);
          if (R & 1) bmax2 = vimax3_2(bmax2, E[R - 1], E[R - 1]);
        }
        const int mrel2 = __reduce_max_sync(0xffffffffu, lo16(bmax2) > hi16(bmax2) ? lo16(bmax2)
                                                                                    : hi16(bmax2));
        if ((long long)mrel2 + 3LL * ge + base - kX2Off + goe >= (long long)prune_seen) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            H[r] = Hs[r];
            E[r] = Es[r];
          }
          diag = diag_s;
          out_hm = ohm_s;
          out_f = of_s;
          __syncwarp();
          opt_cool = 4;
        } else {
          tracked_run = false;
        }
      }
      // a strictly better cell in at least one lane half: first step of the
      // 32-step half [h0, h0 + 32) reaching it
      bool found = false;
      auto resolve_half = [&](int h0) {
        __syncwarp();
        found |= !__all_sync(0xffffffffu, bk2 == kb2);
        if (bk2 != kb2) {
          auto resolve = [&](bool hiHalf, int key, int colbase, int& v, int& rk_, int& bj,
                             long long vref) {
            int lo = 0;
#pragma unroll
            for (int stp = 16; stp > 0; stp >>= 1) {
              const uint32_t w = sm->trk[SWB_IX(lo + stp - 1, 32)][lane];
              if ((hiHalf ? hi16(w) : lo16(w)) < key) lo += stp;
            }
            v = (int)(vref + (key >> 5) - 1);
            rk_ = key & 31;
            bj = colbase + lo;
          };
          const int ka = lo16(bk2), kbh = hi16(bk2);
          if (ka > lo16(kb2)) resolve(false, ka, s0 + h0 - lane, vA, rkA, bjA, vrA);
          if (kbh > hi16(kb2)) resolve(true, kbh, s0 + h0 - lane - 32, vB, rkB, bjB, vrB);
        }
        __syncwarp();
        if (h0 + 32 < kX2Blk) set_frame(mabs_w);  // keys of the next half against the new best
      };
      if (!tracked_run) {
      } else if (steady && !track_block) {
#pragma unroll 1
        for (int k = 0; k < kX2Blk; k += 2) {
          step(k, s0 + k, false, H, H2, T0{});
          step(k + 1, s0 + k + 1, false, H2, H, T0{});
        }
      } else if (steady) {
#pragma unroll 1
        for (int h0 = 0; h0 < kX2Blk; h0 += 32) {
#pragma unroll 1
          for (int k = h0; k < h0 + 32; k += 2) {
            step(k, s0 + k, false, H, H2, T1{});
            step(k + 1, s0 + k + 1, false, H2, H, T1{});
          }
          resolve_half(h0);
        }
      } else {
#pragma unroll 1
        for (int h0 = 0; h0 < kX2Blk; h0 += 32) {
#pragma unroll 1
          for (int k = h0; k < h0 + 32; k += 2) {
            step(k, s0 + k, true, H, H2, T1{});
            step(k + 1, s0 + k + 1, true, H2, H, T1{});
          }
          resolve_half(h0);
        }
      }
      __syncwarp();
      // a tracked block that found nothing new lets the next candidate try
      // the optimistic run again
      if (steady && track_block && tracked_run) {
        if (found) opt_cool = 4;
        else if (opt_cool > 0) --opt_cool;
      }
    }
    __syncwarp();

    // (4) flush B's bottom row for columns [s0 - 63, s0 - 63 + BLK) and publish
    {
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const int cf = s0 - 63 + 32 * h + lane;
        if (cf >= 0 && cf < n2) {
          int2 o = make_int2(-goe, SWB_NEG32);  // pruned block: the fill values
          if (!skip) {
            const uint2 raw = sm->out[SWB_IX(32 * h + lane, BLK)];
            const int off = base - kX2Off;
            o = make_int2(hi16(raw.x) + off, hi16(raw.y) + off);
          }
          __stcg(outbuf + SWB_IX(cf, n2), o);
        }
      }
      if (ext_out) __threadfence_system();
      __syncwarp();
      if (lane == 0) {
        int pub = s0 - 63 + kX2Blk;
        if (pub > n2) pub = n2;
        if (pub > 0) {
          if (ext_out) st_release_sys(my_progress, pub);
          else st_release(my_progress, pub);
        }
      }
    }

    // (5) running best (pruning and the tracking decision)
    {
      // publish only improvements and only above what is already known:
      // one contended atomic per warp and block would cost every warp a
      // global round trip on the critical path
      const int bm = __reduce_max_sync(0xffffffffu, vA > vB ? vA : vB);
      if (bm > -goe && bm + goe > published && bm + goe > prune_seen) {
        published = bm + goe;
        if (lane == 0) raise_best(J, published);
      }
    }
  }
  if (J.bmap_out) bw_finish(J, bw, lane);
  if (lane == 0) {
    if (ext_out) st_release_sys(my_progress, 0x7fffffff);
    else st_release(my_progress, 0x7fffffff);
  }

  // item result: best of both halves, then warp reduction (smallest (i, j) on ties)
  int b = vA, ii = -1, jj = -1;
  if (bjA >= 0) {
    ii = rowA + (31 - rkA);
    jj = bjA;
  }
  if (bjB >= 0) {
    const int ib = rowB + (31 - rkB);
    if (ii < 0 || vB > b || (vB == b && (ib < ii || (ib == ii && bjB < jj)))) {
      b = vB;
      ii = ib;
      jj = bjB;
    }
  }
  if (ii >= n1) ii = jj = -1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int ob = __shfl_down_sync(0xffffffffu, b, o);
    const int oi = __shfl_down_sync(0xffffffffu, ii, o);
    const int oj = __shfl_down_sync(0xffffffffu, jj, o);
    bool take;
    if (oi < 0) take = false;
    else if (ii < 0) take = true;
    else take = ob > b || (ob == b && (oi < ii || (oi == ii && oj < jj)));
    if (take) {
      b = ob;
      ii = oi;
      jj = oj;
    }
  }
  if (lane == 0) {
    J.strip_res[s] = make_int4(b, ii, jj, ii >= 0 ? 1 : 0);
    int rows_here = n1 - R0;
    if (rows_here > 64 * R) rows_here = 64 * R;
    const long long cells = (long long)n2 * rows_here - pruned_blocks * (long long)kX2Blk * rows_here;
    atomicAdd(&J.counters[0], (unsigned long long)(cells > 0 ? cells : 0));
    atomicAdd(&J.counters[1], (unsigned long long)exec_blocks);
    atomicAdd(&J.counters[2], (unsigned long long)pruned_blocks);
    atomicAdd(&J.counters[3], (unsigned long long)wait_cycles);
    atomicAdd(&J.counters[4], (unsigned long long)(clock64() - t_strip0));
    unsigned long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    J.strip_times[3 * s + 0] = g0;
    J.strip_times[3 * s + 1] = g1;
    J.strip_times[3 * s + 2] = P.proto == 10 ? g_diag : gw;  // proto 10: diagonal entry time
  }
}

// FINAL kernels also serve passes that want their final rows (split mode): the
// last item of such a pass runs the FINAL strip code.  (A lambda here is not
// always inlined; an outlined strip body addresses shared memory generically.)
template <int R, bool WILD, bool FINAL, int BLK>
__device__ __forceinline__ void run_item_x2(const PassParams& P, long long item,
                                            WarpSmemX2<BLK>* sm, const uint32_t* tw_s) {
  int s = 0;
  const int j = item_job(P, item, &s);
  if (FINAL && P.jobs[j].want_final && s == P.jobs[j].nstrips - 1)
    run_strip_x2<R, WILD, FINAL, BLK>(P, P.jobs[j], s, sm, tw_s);
  else
    run_strip_x2<R, WILD, false, BLK>(P, P.jobs[j], s, sm, tw_s);
}

template <int R, bool WILD, bool FINAL, int BLK>
__global__ void __launch_bounds__(256, 1) pass_kernel_x2(const PassParams P) {
  // dynamic shared memory, x2_smem_bytes<BLK>(blockDim.x / 32) (launch_any)
  extern __shared__ __align__(16) unsigned char x2_dyn[];
  WarpSmemX2<BLK>* wsm = reinterpret_cast<WarpSmemX2<BLK>*>(x2_dyn);
  uint32_t* tw_s = reinterpret_cast<uint32_t*>(wsm + (blockDim.x >> 5));
  long long* base_s = reinterpret_cast<long long*>(tw_s + 8);
  if (threadIdx.x < 8) tw_s[threadIdx.x] = P.tlo[threadIdx.x];
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  WarpSmemX2<BLK>* sm = &wsm[warp];
  if (P.group > 0) {
    const int w = (int)(blockDim.x >> 7);
    for (;;) {
      if (threadIdx.x == 0) *base_s = (long long)atomicAdd(P.claim, (unsigned long long)P.group);
      __syncthreads();
      const long long base = *base_s;
      __syncthreads();
      if (base >= P.total_items) break;
      long long item = base + (warp & 3) * w + (warp >> 2);
      // single round, two warps per sub-partition: items p and p + half share
      // one, so the two reach their diagonals (tracked blocks on the pass's
      // critical chain) half a pass apart (C2: 242 -> 232 ms against the
      // mirrored pairs (p, last - p), kept as proto 12; unrelated +1.5 %)
      if (P.mirror == 1) {
        const long long half = (P.total_items + 1) / 2;
        const long long p = base / 2 + (warp & 3);
        const long long q = p + half;
        item = (warp >> 2) == 0 ? (p < half ? p : P.total_items) : (q < P.total_items ? q : P.total_items);
      } else if (P.mirror) {
        const long long p = base / 2 + (warp & 3);
        const long long q = P.total_items - 1 - p;
        item = (warp >> 2) == 0 ? (p <= q ? p : P.total_items) : (p < q ? q : P.total_items);
      }
      if (item < P.total_items) run_item_x2<R, WILD, FINAL, BLK>(P, item, sm, tw_s);
    }
    return;
  }
  for (;;) {
    long long item = 0;
    if (lane == 0) item = (long long)atomicAdd(P.claim, 1ULL);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= P.total_items) break;
    run_item_x2<R, WILD, FINAL, BLK>(P, item, sm, tw_s);
  }
}

}  // namespace swb
