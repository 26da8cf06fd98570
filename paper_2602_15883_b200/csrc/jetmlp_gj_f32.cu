// Fused jet-MLP kernel instantiations: MODE_GJ (ghost-derivative extension), float.
#include "jetmlp_dispatch.cuh"
FR_DEFINE_MODE_ENTRY(GJ, float, f32)
