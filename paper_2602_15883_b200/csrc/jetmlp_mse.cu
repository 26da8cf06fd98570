// Instantiations of the fused jet-MLP kernel for MODE_MSE.
#include "jetmlp_dispatch.cuh"
FR_DEFINE_MODE_ENTRY(MSE)
