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
  int ppt_mse;       // epoch kernel: points per MSE tile
  int cps = 1;       // epoch kernel: resident CTAs per SM (persistent grid = SMs x cps)
};

// Load a kernel and set its shared-memory attributes once per device, at plan /
// workspace time.  With lazy module loading (the CUDA 12 default) a kernel's
// first launch waits for the device to go idle; a gated epoch kernel whose
// first launch sits behind a still-running transport would then wait for the
// transport to finish instead of overlapping it (and its exchange timeout would
// never fire).  `loaded` is a per-kernel-instance bitmask of device ordinals.
template <typename K>
int ensure_loaded(K k, size_t smem, bool carveout, unsigned long long& loaded) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return int(e);
  const unsigned long long bit = 1ull << (dev & 63);
  if (__atomic_load_n(&loaded, __ATOMIC_ACQUIRE) & bit) return 0;
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, k);  // forces the module load
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  // all of the unified L1/shared array as shared memory, so the resident CTAs fit
  if (e == cudaSuccess && carveout) e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return int(e);
  __atomic_fetch_or(&loaded, bit, __ATOMIC_RELEASE);
  return 0;
}

template <int V>
struct IntC {
  static constexpr int value = V;
};

template <class F>
int dispatch_act_reg(int act, int reg, F&& go) {
  if (act == ACT_TANH) {
    if (reg == REG_STEADY2D) return go(IntC<ACT_TANH>{}, IntC<REG_STEADY2D>{});
    if (reg == REG_UNSTEADY2D) return go(IntC<ACT_TANH>{}, IntC<REG_UNSTEADY2D>{});
    if (reg == REG_UNSTEADY3D) return go(IntC<ACT_TANH>{}, IntC<REG_UNSTEADY3D>{});
  }
  if (act == ACT_SIN) {
    if (reg == REG_STEADY2D) return go(IntC<ACT_SIN>{}, IntC<REG_STEADY2D>{});
    if (reg == REG_UNSTEADY2D) return go(IntC<ACT_SIN>{}, IntC<REG_UNSTEADY2D>{});
    if (reg == REG_UNSTEADY3D) return go(IntC<ACT_SIN>{}, IntC<REG_UNSTEADY3D>{});
  }
  return -1;
}

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
  auto k = jetmlp_kernel<T, ACT, MODE, REG, W>;
  // load + raise the opt-in shared-memory limit once per device (not a stream
  // operation: kept out of the steady state so captured epochs only contain
  // launches); every workspace query does it, before any launch
  static unsigned long long loaded = 0;
  static size_t smem_set = 0;
  if (smem > smem_set) {
    loaded = 0;  // a larger L needs the attribute raised again
    smem_set = smem;
  }
  if (int r = ensure_loaded(k, smem_set, false, loaded)) return r;
  if (!a) return 0;
  k<<<grid, C::NT, smem, st>>>(*a);
  ++g_kernel_launches;
  return int(cudaGetLastError());
}

template <typename T, int ACT, int REG, int W, bool TC>
int run_epoch_v(const EpochArgs* e, int grid, cudaStream_t st, KInfo* info, int L);

// tc: split-TF32 tensor-core contractions (FR_MATH_TF32X3; FP32, W = 64 only)
template <typename T, int ACT, int REG, int W>
int run_epoch(const EpochArgs* e, int grid, cudaStream_t st, KInfo* info, int L, int tc) {
  if constexpr (sizeof(T) == 4 && W == 64 && EpochCfg<T, ACT, REG, W>::CPS == 1) {
    if (tc) return run_epoch_v<T, ACT, REG, W, true>(e, grid, st, info, L);
  } else {
    if (tc) return -1;
  }
  return run_epoch_v<T, ACT, REG, W, false>(e, grid, st, info, L);
}

template <typename T, int ACT, int REG, int W, bool TC>
int run_epoch_v(const EpochArgs* e, int grid, cudaStream_t st, KInfo* info, int L) {
  using E = EpochCfg<T, ACT, REG, W>;
  using CP = JetCfg<T, ACT, MODE_PDE, REG, W, E::NT>;
  using CM = JetCfg<T, ACT, MODE_MSE, REG, W, E::NT>;
  const size_t smem = CP::smem_bytes(L, TC) > CM::smem_bytes(L, TC) ? CP::smem_bytes(L, TC) : CM::smem_bytes(L, TC);
  const int sp = CP::stash_per_thread(L) > CM::stash_per_thread(L) ? CP::stash_per_thread(L) : CM::stash_per_thread(L);
  if (info) {
    info->nt = CP::NT;
    info->ppt = CP::PPT;
    info->ppt_mse = CM::PPT;
    info->stash_elems = CP::NT * sp;
    info->smem = smem;
    info->cps = E::CPS;
  }
  auto k = jetmlp_epoch_kernel<T, ACT, REG, W, TC>;
  static unsigned long long loaded = 0;
  static size_t smem_set = 0;
  if (smem > smem_set) {
    loaded = 0;
    smem_set = smem;
  }
  if (int r = ensure_loaded(k, smem_set, true, loaded)) return r;
  if (!e) return 0;
  k<<<grid, CP::NT, smem, st>>>(*e);
  ++g_kernel_launches;
  return int(cudaGetLastError());
}

// returns -1 when the combination is not compiled in
template <int MODE, typename T>
int dispatch_mode_t(int act, int reg, int w, const KArgs* a, int grid, cudaStream_t st, KInfo* info, int L) {
  auto go = [&](auto act_c, auto reg_c) -> int {
    constexpr int ACT = decltype(act_c)::value, REG = decltype(reg_c)::value;
    if (w == 16) return run_mode<T, ACT, MODE, REG, 16>(a, grid, st, info, L);
    if (w == 64) return run_mode<T, ACT, MODE, REG, 64>(a, grid, st, info, L);
    return -1;
  };
  return dispatch_act_reg(act, reg, go);
}

template <typename T>
int dispatch_epoch_t(int act, int reg, int w, const EpochArgs* e, int grid, cudaStream_t st, KInfo* info, int L,
                     int tc) {
  auto go = [&](auto act_c, auto reg_c) -> int {
    constexpr int ACT = decltype(act_c)::value, REG = decltype(reg_c)::value;
    if (w == 16) return tc ? -1 : run_epoch<T, ACT, REG, 16>(e, grid, st, info, L, 0);
    if (w == 64) return run_epoch<T, ACT, REG, 64>(e, grid, st, info, L, tc);
    return -1;
  };
  return dispatch_act_reg(act, reg, go);
}

}  // namespace fr

// one translation unit per (mode, dtype) keeps the parallel build short
#define FR_DEFINE_MODE_ENTRY(M, T, TAG)                                                                \
  namespace fr {                                                                                      \
  int mode_entry_##M##_##TAG(int act, int reg, int w, const KArgs* a, int grid, cudaStream_t st,       \
                             KInfo* info, int L) {                                                    \
    return dispatch_mode_t<MODE_##M, T>(act, reg, w, a, grid, st, info, L);                           \
  }                                                                                                   \
  }
#ifdef FR_PHASE_TIMERS
#define FR_PHASE_READER(TAG)                                                          \
  extern "C" int fr_debug_phase_cycles_##TAG(unsigned long long* out, int reset) {    \
    cudaMemcpyFromSymbol(out, fr::g_phase_cycles, sizeof(unsigned long long) * 16);   \
    cudaMemcpyFromSymbol(out + 16, fr::g_tc_cycles, sizeof(unsigned long long) * 16); \
    if (reset) {                                                                      \
      unsigned long long z[16] = {0};                                                 \
      cudaMemcpyToSymbol(fr::g_phase_cycles, z, sizeof(z));                           \
      cudaMemcpyToSymbol(fr::g_tc_cycles, z, sizeof(z));                              \
    }                                                                                 \
    return 0;                                                                         \
  }
#else
#define FR_PHASE_READER(TAG)
#endif
#define FR_DEFINE_EPOCH_ENTRY(T, TAG)                                                                  \
  namespace fr {                                                                                      \
  int epoch_entry_##TAG(int act, int reg, int w, const EpochArgs* e, int grid, cudaStream_t st,        \
                        KInfo* info, int L, int tc) {                                                 \
    return dispatch_epoch_t<T>(act, reg, w, e, grid, st, info, L, tc);                                \
  }                                                                                                   \
  }                                                                                                   \
  FR_PHASE_READER(TAG)
