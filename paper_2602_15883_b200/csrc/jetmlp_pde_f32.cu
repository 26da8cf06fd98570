// Fused jet-MLP kernel instantiations: MODE_PDE, float.
#include "jetmlp_dispatch.cuh"
FR_DEFINE_MODE_ENTRY(PDE, float, f32)
