// Fused jet-MLP kernel instantiations: MODE_MSE, float.
#include "jetmlp_dispatch.cuh"
FR_DEFINE_MODE_ENTRY(MSE, float, f32)
