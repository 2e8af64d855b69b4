// Packed 16x2 phase-1 pass kernels (swb_x2.cuh).  This translation unit
// instantiates the 32-step-block kernels; swb_launch_x2w.cu includes it with
// SWB_X2_TU_BLK = 64 for the 64-step-block ones (compiled in parallel).
#include "swb_launch.cuh"

#ifndef SWB_X2_TU_BLK
#define SWB_X2_TU_BLK 32
#endif

namespace swb {
namespace {

constexpr int kTuBlk = SWB_X2_TU_BLK;

template <int R, bool FINAL>
int dispatch_x2_R(swb_ctx* ctx, const PassParams* P, long long items, int ctas_per_sm,
                  int* occ_out, bool wild) {
  constexpr size_t ws = sizeof(WarpSmemX2<kTuBlk>);
  if (occ_out)
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        occ_out, pass_kernel_x2<R, false, FINAL, kTuBlk>, 128, x2_smem_bytes<kTuBlk>(4));
  return wild ? launch_any(ctx, pass_kernel_x2<R, true, FINAL, kTuBlk>, *P, items, ctas_per_sm, ws)
              : launch_any(ctx, pass_kernel_x2<R, false, FINAL, kTuBlk>, *P, items, ctas_per_sm, ws);
}

}  // namespace

#if SWB_X2_TU_BLK == 32
int dispatch_x2_b32(swb_ctx* ctx, int R, const PassParams* P, long long items, int ctas_per_sm,
                    int* occ_out, bool wild, bool final_rows) {
#else
int dispatch_x2_b64(swb_ctx* ctx, int R, const PassParams* P, long long items, int ctas_per_sm,
                    int* occ_out, bool wild, bool final_rows) {
#endif
  if (final_rows) {
    switch (R) {
      case 14: return dispatch_x2_R<14, true>(ctx, P, items, ctas_per_sm, occ_out, wild);
      case 16: return dispatch_x2_R<16, true>(ctx, P, items, ctas_per_sm, occ_out, wild);
      default: break;
    }
    return swb_fail(SWB_EINVAL, "packed rows_per_lane %d has no final-row instantiation", R);
  }
  switch (R) {
    case 8: return dispatch_x2_R<8, false>(ctx, P, items, ctas_per_sm, occ_out, wild);
    case 10: return dispatch_x2_R<10, false>(ctx, P, items, ctas_per_sm, occ_out, wild);
    case 12: return dispatch_x2_R<12, false>(ctx, P, items, ctas_per_sm, occ_out, wild);
    case 14: return dispatch_x2_R<14, false>(ctx, P, items, ctas_per_sm, occ_out, wild);
    case 16: return dispatch_x2_R<16, false>(ctx, P, items, ctas_per_sm, occ_out, wild);
    default: break;
  }
  return swb_fail(SWB_EINVAL, "packed rows_per_lane %d not instantiated", R);
}

#if SWB_X2_TU_BLK == 32
int dispatch_x2(swb_ctx* ctx, int R, const PassParams* P, long long items, int ctas_per_sm,
                int* occ_out, bool wild, bool final_rows, int blk) {
  return blk == 64 ? dispatch_x2_b64(ctx, R, P, items, ctas_per_sm, occ_out, wild, final_rows)
                   : dispatch_x2_b32(ctx, R, P, items, ctas_per_sm, occ_out, wild, final_rows);
}

SWB_CHK_TAKE(chk_take_x2)
#else
SWB_CHK_TAKE(chk_take_x2w)
#endif

}  // namespace swb
