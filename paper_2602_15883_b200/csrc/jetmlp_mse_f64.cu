// Fused jet-MLP kernel instantiations: MODE_MSE, double.
#include "jetmlp_dispatch.cuh"
FR_DEFINE_MODE_ENTRY(MSE, double, f64)
