// Whole-epoch kernel instantiations (PDE + MSE heads in one launch), float.
#include "jetmlp_dispatch.cuh"
FR_DEFINE_EPOCH_ENTRY(float, f32)
