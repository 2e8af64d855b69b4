// Packed 16x2 phase-1 pass kernels (swb_x2.cuh).
#include "swb_launch.cuh"

namespace swb {
namespace {

template <int R, bool FINAL>
int dispatch_x2_R(swb_ctx* ctx, const PassParams* P, long long items, int ctas_per_sm,
                  int* occ_out, bool wild) {
  if (occ_out)
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        occ_out, pass_kernel_x2<R, false, FINAL>, 128, 0);
  return wild ? launch_any(ctx, pass_kernel_x2<R, true, FINAL>, *P, items, ctas_per_sm)
              : launch_any(ctx, pass_kernel_x2<R, false, FINAL>, *P, items, ctas_per_sm);
}

}  // namespace

int dispatch_x2(swb_ctx* ctx, int R, const PassParams* P, long long items, int ctas_per_sm,
                int* occ_out, bool wild, bool final_rows) {
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


SWB_CHK_TAKE(chk_take_x2)

}  // namespace swb
