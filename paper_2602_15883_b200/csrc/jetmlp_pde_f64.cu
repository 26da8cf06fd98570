// Fused jet-MLP kernel instantiations: MODE_PDE, double.
#include "jetmlp_dispatch.cuh"
FR_DEFINE_MODE_ENTRY(PDE, double, f64)
