// Fused jet-MLP kernel instantiations: MODE_JET, float.
#include "jetmlp_dispatch.cuh"
FR_DEFINE_MODE_ENTRY(JET, float, f32)
