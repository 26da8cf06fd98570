// Fused jet-MLP kernel instantiations: MODE_VALUE, float.
#include "jetmlp_dispatch.cuh"
FR_DEFINE_MODE_ENTRY(VALUE, float, f32)
