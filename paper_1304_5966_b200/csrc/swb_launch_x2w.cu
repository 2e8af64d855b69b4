// Packed 16x2 kernels with 64-step blocks (swb_launch_x2.cu, swb_x2.cuh).
#define SWB_X2_TU_BLK 64
#include "swb_launch_x2.cu"
