// Restricted / global lane-kernel pass instantiations (phase 2, split
// finishing, Myers-Miller halves): every tracking mode.  SWB_OTHER_TRACK
// selects the tracking modes this translation unit instantiates so the
// Makefile can compile them in parallel (swb_launch_none.cu / _track.cu).
#include "swb_launch.cuh"

namespace swb {

template <int R, int TRACK>
int dispatch_other_R(swb_ctx* ctx, const PassParams* P, long long items, int ctas_per_sm,
                     int* occ_out) {
  if (occ_out) return kernel_occupancy<R, false, TRACK>(occ_out);
  return launch_kernel<R, false, TRACK>(ctx, *P, items, ctas_per_sm);
}

template <int TRACK>
int dispatch_other_T(swb_ctx* ctx, int R, const PassParams* P, long long items, int ctas_per_sm,
                     int* occ_out) {
  switch (R) {
    case 8: return dispatch_other_R<8, TRACK>(ctx, P, items, ctas_per_sm, occ_out);
    case 16: return dispatch_other_R<16, TRACK>(ctx, P, items, ctas_per_sm, occ_out);
    case 24: return dispatch_other_R<24, TRACK>(ctx, P, items, ctas_per_sm, occ_out);
    case 32: return dispatch_other_R<32, TRACK>(ctx, P, items, ctas_per_sm, occ_out);
    default: break;
  }
  return swb_fail(SWB_EINVAL, "rows_per_lane %d not instantiated for this pass mode", R);
}

#if SWB_OTHER_TRACK == 0
int dispatch_other_none(swb_ctx* ctx, int R, const PassParams* P, long long items,
                        int ctas_per_sm, int* occ_out) {
  return dispatch_other_T<kTrackNone>(ctx, R, P, items, ctas_per_sm, occ_out);
}
SWB_CHK_TAKE(chk_take_other)
#else
int dispatch_other_track(swb_ctx* ctx, int R, const PassParams* P, long long items, int track,
                         int ctas_per_sm, int* occ_out) {
  if (track == kTrackMin) return dispatch_other_T<kTrackMin>(ctx, R, P, items, ctas_per_sm, occ_out);
  return dispatch_other_T<kTrackMax>(ctx, R, P, items, ctas_per_sm, occ_out);
}
SWB_CHK_TAKE(chk_take_track)
#endif

}  // namespace swb
