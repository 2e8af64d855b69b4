// Shared-table pass kernels (large alphabets).
#include "swb_launch.cuh"

namespace swb {
namespace {

template <int R>
int dispatch_big_R(swb_ctx* ctx, const PassParams* P, long long items, bool local, int track,
                   int ctas_per_sm, int* occ_out) {
  if (local) {
    if (track != kTrackMin) return swb_fail(SWB_EUNSUPPORTED, "local passes support TRACK_MIN only");
    if (occ_out) return kernel_occupancy<R, true, kTrackMin, true>(occ_out);
    return launch_kernel<R, true, kTrackMin, true>(ctx, *P, items, ctas_per_sm);
  }
  if (track == kTrackNone) {
    if (occ_out) return kernel_occupancy<R, false, kTrackNone, true>(occ_out);
    return launch_kernel<R, false, kTrackNone, true>(ctx, *P, items, ctas_per_sm);
  }
  if (track == kTrackMin) {
    if (occ_out) return kernel_occupancy<R, false, kTrackMin, true>(occ_out);
    return launch_kernel<R, false, kTrackMin, true>(ctx, *P, items, ctas_per_sm);
  }
  if (occ_out) return kernel_occupancy<R, false, kTrackMax, true>(occ_out);
  return launch_kernel<R, false, kTrackMax, true>(ctx, *P, items, ctas_per_sm);
}

}  // namespace

int dispatch_big(swb_ctx* ctx, int R, const PassParams* P, long long items, bool local, int track,
                 int ctas_per_sm, int* occ_out) {
  if (R == 8) return dispatch_big_R<8>(ctx, P, items, local, track, ctas_per_sm, occ_out);
  if (R == 16 && local) return dispatch_big_R<16>(ctx, P, items, local, track, ctas_per_sm, occ_out);
  return swb_fail(SWB_EINVAL, "rows_per_lane %d not instantiated for large alphabets", R);
}


SWB_CHK_TAKE(chk_take_big)

}  // namespace swb
