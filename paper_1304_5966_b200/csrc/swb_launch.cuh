// Kernel instantiation and launch (shared by the swb_launch_*.cu translation
// units, which compile the pass kernels in parallel; swb_pass.cu holds the
// host logic).  Each dispatch function launches (P != null) or reports the
// occupancy (occ_out != null) of one kernel family for rows-per-lane R.
#pragma once

#include <algorithm>

#include "swb_kernels.cuh"
#include "swb_passes.h"
#include "swb_x2.cuh"

namespace swb {

// Rows-per-lane instantiations.  Local TRACK_MIN passes (phase 1, split) get a
// dense set so a single large pass can be cut into exactly as many warp-strips
// as the SM sub-partitions hold; the other modes get a coarse set.
constexpr int kLocalR[] = {8, 16, 20, 24, 28, 32};
constexpr int kOtherR[] = {8, 16, 24, 32};  // (2 measured no faster, and spilled)
// Shared-table kernels (large alphabets): few strip heights.
constexpr int kBigLocalR[] = {8, 16};
constexpr int kBigOtherR[] = {8};
// packed 16x2 phase-1 kernel (swb_x2.cuh): R packed rows per lane, 64R rows per item
constexpr int kX2R[] = {8, 10, 12, 14, 16};
constexpr int kX2SlabR = 16;  // multigpu.SLAB_ROWS_PER_LANE x 32 rows = 64 x 16
// final rows (split mode) are instantiated for the two largest heights only
constexpr int kX2FinalR[] = {14, 16};

int dispatch_local(swb_ctx* ctx, int R, const PassParams* P, long long items, int track,
                   int ctas_per_sm, int* occ_out);
int dispatch_other_none(swb_ctx* ctx, int R, const PassParams* P, long long items,
                        int ctas_per_sm, int* occ_out);
int dispatch_other_track(swb_ctx* ctx, int R, const PassParams* P, long long items, int track,
                         int ctas_per_sm, int* occ_out);
int dispatch_big(swb_ctx* ctx, int R, const PassParams* P, long long items, bool local, int track,
                 int ctas_per_sm, int* occ_out);
// blk: steps per block of the packed kernel, 32 or 64 (swb_x2.cuh)
int dispatch_x2(swb_ctx* ctx, int R, const PassParams* P, long long items, int ctas_per_sm,
                int* occ_out, bool wild = false, bool final_rows = false, int blk = 32);
int dispatch_x2_b32(swb_ctx* ctx, int R, const PassParams* P, long long items, int ctas_per_sm,
                    int* occ_out, bool wild, bool final_rows);
int dispatch_x2_b64(swb_ctx* ctx, int R, const PassParams* P, long long items, int ctas_per_sm,
                    int* occ_out, bool wild, bool final_rows);

// checked builds: each translation unit reports (and clears) its own record
int chk_take_local(long long* out);
int chk_take_other(long long* out);
int chk_take_track(long long* out);
int chk_take_big(long long* out);
int chk_take_x2(long long* out);
int chk_take_x2w(long long* out);

#ifdef SWB_CHECKED
#define SWB_CHK_TAKE(name)                                                          \
  int name(long long* out) {                                                        \
    if (cudaMemcpyFromSymbol(out, g_swb_chk, 4 * sizeof(long long)) != cudaSuccess) \
      return -1;                                                                    \
    const long long zero[4] = {0, 0, 0, 0};                                         \
    cudaMemcpyToSymbol(g_swb_chk, zero, sizeof(zero));                              \
    return 0;                                                                       \
  }
#else
#define SWB_CHK_TAKE(name)  \
  int name(long long* out) { \
    out[0] = 0;             \
    return 0;               \
  }
#endif

template <int R, bool LOCAL, int TRACK, bool BIG = false>
int kernel_occupancy(int* per_sm) {
  return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      per_sm, pass_kernel<R, LOCAL, TRACK, BIG>, 128, 0);
}

// warp_smem > 0: the kernel takes warp_smem bytes of dynamic shared memory per
// warp plus 64 (the packed kernel, x2_smem_bytes); 0: static shared memory only
template <typename K>
int launch_any(swb_ctx* ctx, K kern, const PassParams& Pin, long long items, int ctas_per_sm,
               size_t warp_smem = 0) {
  PassParams P = Pin;
  auto dyn = [&](int threads) -> size_t { return warp_smem ? (threads / 32) * warp_smem + 64 : 0; };
  int per_sm = 0;
  SWB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, dyn(128)));
  if (per_sm < 1) return swb_fail(SWB_ECUDA, "pass kernel does not fit on an SM");
  if (ctas_per_sm > 0 && per_sm > ctas_per_sm) per_sm = ctas_per_sm;
  if (P.chunk > 0) {
    const long long cap = (long long)per_sm * ctx->sms;
    const int grid = (int)std::min(cap, std::max((long long)P.total_items, 1LL));
    int per = per_sm;
    if (P.chunk > 4) {  // 8-warp chunks: occupancy of the wider CTA
      SWB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 32 * P.chunk, dyn(32 * P.chunk)));
      if (per < 1) return swb_fail(SWB_ECUDA, "chunk CTA does not fit on an SM");
    }
    const int grid2 = (int)std::min((long long)per * ctx->sms, std::max((long long)P.total_items, 1LL));
    kern<<<P.chunk > 4 ? grid2 : grid, 32 * P.chunk, dyn(32 * P.chunk), ctx->stream>>>(P);
    ctx->launches++;
    SWB_CUDA(cudaGetLastError());
    return SWB_OK;
  }
  if (ctx->claim_mode != 2 && (ctx->claim_mode == 1 || (P.njobs <= 4 && !P.warp_claim)) &&
      per_sm <= 2 && items > (long long)ctx->sms * 4) {
    // one CTA per SM, per_sm warps per sub-partition, adjacent strips paired
    const int threads = 128 * per_sm;
    int fit = 0;
    SWB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, kern, threads, dyn(threads)));
    if (fit >= 1) {
      // adjacent strips of one chain share a sub-partition: job-major order
      P.item_map = nullptr;
      P.group = 4 * per_sm;
      // pairs of items per sub-partition (swb_x2.cuh; the lane kernel mirrors)
      P.mirror = (per_sm == 2 && items <= 8LL * ctx->sms && ctx->proto != 8) ? (ctx->proto == 12 ? 2 : 1) : 0;
      // dynamic shared memory pins the layout to exactly one CTA per SM
      const int pin = (int)std::max<size_t>(120 * 1024, dyn(threads));
      SWB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pin));
      kern<<<ctx->sms, threads, pin, ctx->stream>>>(P);
      ctx->launches++;
      SWB_CUDA(cudaGetLastError());
      return SWB_OK;
    }
  }
  P.group = 0;
  P.mirror = 0;
  long long cap = (long long)per_sm * ctx->sms;
  long long need = (items + 3) / 4;
  int grid = (int)std::min(cap, std::max(need, 1LL));
  kern<<<grid, 128, dyn(128), ctx->stream>>>(P);
  ctx->launches++;
  SWB_CUDA(cudaGetLastError());
  return SWB_OK;
}

template <int R, bool LOCAL, int TRACK, bool BIG = false>
int launch_kernel(swb_ctx* ctx, const PassParams& Pin, long long items, int ctas_per_sm) {
  return launch_any(ctx, pass_kernel<R, LOCAL, TRACK, BIG>, Pin, items, ctas_per_sm);
}

}  // namespace swb
