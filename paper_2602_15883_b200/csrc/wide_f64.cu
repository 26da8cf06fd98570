// Layer-wise wide jet-MLP kernel instantiations, double.
#include "wide_dispatch.cuh"
FR_DEFINE_WIDE_ENTRY(double, f64)
