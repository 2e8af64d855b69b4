#define SWB_OTHER_TRACK 0
#include "swb_launch_other.cu"
