// Local (phase-1 / split) lane-kernel pass instantiations, TRACK_MIN.
#include "swb_launch.cuh"

namespace swb {

int dispatch_local(swb_ctx* ctx, int R, const PassParams* P, long long items, int track,
                   int ctas_per_sm, int* occ_out) {
  if (track != kTrackMin) return swb_fail(SWB_EUNSUPPORTED, "local passes support TRACK_MIN only");
  switch (R) {
#define SWB_CASE(RR)                                                               \
  case RR:                                                                         \
    if (occ_out) return kernel_occupancy<RR, true, kTrackMin>(occ_out);            \
    return launch_kernel<RR, true, kTrackMin>(ctx, *P, items, ctas_per_sm);
    SWB_CASE(8)
    SWB_CASE(16)
    SWB_CASE(20)
    SWB_CASE(24)
    SWB_CASE(28)
    SWB_CASE(32)
#undef SWB_CASE
    default: break;
  }
  return swb_fail(SWB_EINVAL, "rows_per_lane %d not instantiated for local passes", R);
}

SWB_CHK_TAKE(chk_take_local)

}  // namespace swb
