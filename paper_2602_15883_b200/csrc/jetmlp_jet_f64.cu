// Fused jet-MLP kernel instantiations: MODE_JET, double.
#include "jetmlp_dispatch.cuh"
FR_DEFINE_MODE_ENTRY(JET, double, f64)
