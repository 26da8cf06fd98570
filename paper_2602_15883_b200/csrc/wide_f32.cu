// Layer-wise wide jet-MLP kernel instantiations, float.
#include "wide_dispatch.cuh"
FR_DEFINE_WIDE_ENTRY(float, f32)
