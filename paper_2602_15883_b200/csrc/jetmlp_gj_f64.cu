// Fused jet-MLP kernel instantiations: MODE_GJ (ghost-derivative extension), double.
#include "jetmlp_dispatch.cuh"
FR_DEFINE_MODE_ENTRY(GJ, double, f64)
