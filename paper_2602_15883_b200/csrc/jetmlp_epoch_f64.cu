// Whole-epoch kernel instantiations (PDE + MSE heads in one launch), double.
#include "jetmlp_dispatch.cuh"
FR_DEFINE_EPOCH_ENTRY(double, f64)
