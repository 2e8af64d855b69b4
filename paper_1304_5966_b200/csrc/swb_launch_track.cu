#define SWB_OTHER_TRACK 1
#include "swb_launch_other.cu"
