// Compile-time instantiation table for the jet-MLP kernel: one translation
// unit per mode, dispatching (dtype, activation, regime, padded width).
#pragma once
#include "jetmlp_kernel.cuh"

namespace fr {

struct KInfo {
  int nt;            // threads per CTA
  int ppt;           // points per tile
  int stash_elems;   // per-CTA stash elements (of T)
  size_t smem;       // dynamic shared memory bytes
};

template <typename T, int ACT, int MODE, int REG, int W>
int run_mode(const KArgs* a, int grid, cudaStream_t st, KInfo* info, int L) {
  using C = JetCfg<T, ACT, MODE, REG, W>;
  const size_t smem = C::smem_bytes(L);
  if (info) {
    info->nt = C::NT;
    info->ppt = C::PPT;
    info->stash_elems = C::NT * C::stash_per_thread(L);
    info->smem = smem;
  }
  if (!a) return 0;
  auto k = jetmlp_kernel<T, ACT, MODE, REG, W>;
  // raise the opt-in shared-memory limit once (not a stream operation, but kept
  // out of the steady state so that captured epochs only contain launches)
  static size_t smem_set = 0;
  if (smem > smem_set) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return int(e);
    smem_set = smem;
  }
  k<<<grid, C::NT, smem, st>>>(*a);
  return int(cudaGetLastError());
}

// returns -1 when the combination is not compiled in
template <int MODE>
int dispatch_mode(int dtype, int act, int reg, int w, const KArgs* a, int grid, cudaStream_t st,
                  KInfo* info, int L) {
#define FR_CASE_W(T, ACT, REG)                                                        \
  if (w == 16) return run_mode<T, ACT, MODE, REG, 16>(a, grid, st, info, L);          \
  if (w == 32) return run_mode<T, ACT, MODE, REG, 32>(a, grid, st, info, L);          \
  if (w == 64) return run_mode<T, ACT, MODE, REG, 64>(a, grid, st, info, L);          \
  return -1;
#define FR_CASE_REG(T, ACT)                                   \
  switch (reg) {                                              \
    case REG_STEADY2D: { FR_CASE_W(T, ACT, REG_STEADY2D) }     \
    case REG_UNSTEADY2D: { FR_CASE_W(T, ACT, REG_UNSTEADY2D) } \
    case REG_UNSTEADY3D: { FR_CASE_W(T, ACT, REG_UNSTEADY3D) } \
    default: return -1;                                       \
  }
#define FR_CASE_ACT(T)                             \
  if (act == ACT_TANH) { FR_CASE_REG(T, ACT_TANH) } \
  if (act == ACT_SIN) { FR_CASE_REG(T, ACT_SIN) }   \
  return -1;
  if (dtype == 0) { FR_CASE_ACT(float) }
  if (dtype == 1) { FR_CASE_ACT(double) }
  return -1;
#undef FR_CASE_ACT
#undef FR_CASE_REG
#undef FR_CASE_W
}

}  // namespace fr

#define FR_DEFINE_MODE_ENTRY(M)                                                                  \
  namespace fr {                                                                                 \
  int mode_entry_##M(int dtype, int act, int reg, int w, const KArgs* a, int grid, cudaStream_t st, \
                     KInfo* info, int L) {                                                       \
    return dispatch_mode<MODE_##M>(dtype, act, reg, w, a, grid, st, info, L);                    \
  }                                                                                              \
  }
