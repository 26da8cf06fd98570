// Fused jet-MLP kernel instantiations: MODE_VALUE, double.
#include "jetmlp_dispatch.cuh"
FR_DEFINE_MODE_ENTRY(VALUE, double, f64)
