// Launch sequence and instantiation table of the layer-wise wide kernels.
#pragma once
#include "jetmlp_dispatch.cuh"
#include "wide_kernel.cuh"

namespace fr {

template <typename T, int ACT, int MODE, int REG>
int run_wide(const WArgs* ap, int ks, cudaStream_t st, WInfo* info) {
  using C = WideCfg<T, ACT, MODE, REG>;
  if (info) {
    info->ppt = C::PPT;
    info->rows = C::ROWS;
    info->nt = C::NT;
    info->stq = C::STQ;
  }
  if (!ap) return 0;
  const WArgs& a = *ap;
  static bool attrs = false;
  if (!attrs) {
    cudaFuncSetAttribute(wide_fwd_kernel<T, ACT, MODE, REG>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::gemm_smem()));
    cudaFuncSetAttribute(wide_dx_kernel<T, ACT, MODE, REG>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::gemm_smem()));
    cudaFuncSetAttribute(wide_dw_kernel<T, ACT, MODE, REG>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::dw_smem()));
    cudaFuncSetAttribute(wide_head_kernel<T, ACT, MODE, REG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(C::head_smem(512)));
    attrs = true;
  }
  const dim3 gt(a.ntiles, a.WP / C::UB);
  wide_l0_kernel<T, ACT, MODE, REG><<<gt, C::NT, 0, st>>>(a);
  for (int l = 1; l < a.L; ++l) wide_fwd_kernel<T, ACT, MODE, REG><<<gt, C::NT, C::gemm_smem(), st>>>(a, l);
  wide_head_kernel<T, ACT, MODE, REG><<<a.ntiles, C::NT, C::head_smem(a.WP), st>>>(a);
  if constexpr (C::BWD) {
    for (int l = a.L - 1; l >= 1; --l) wide_dx_kernel<T, ACT, MODE, REG><<<gt, C::NT, C::gemm_smem(), st>>>(a, l);
    const dim3 gw(a.WP / 64, a.WP / 64, ks);
    for (int l = a.L - 1; l >= 1; --l) wide_dw_kernel<T, ACT, MODE, REG><<<gw, C::DW_NT, C::dw_smem(), st>>>(a, l);
    wide_dwL_kernel<T, ACT, MODE, REG><<<ks, 256, 0, st>>>(a);
    wide_dw0_kernel<T, ACT, MODE, REG><<<dim3(ks, (a.WP + 255) / 256), 256, 0, st>>>(a);
    g_kernel_launches += 2 * (a.L - 1) + 2;
  }
  g_kernel_launches += a.L + 1;
  return int(cudaGetLastError());
}

template <typename T>
int dispatch_wide_t(int mode, int act, int reg, const WArgs* a, int ks, cudaStream_t st, WInfo* info) {
  auto go = [&](auto act_c, auto reg_c) -> int {
    constexpr int ACT = decltype(act_c)::value, REG = decltype(reg_c)::value;
    switch (mode) {
      case MODE_PDE: return run_wide<T, ACT, MODE_PDE, REG>(a, ks, st, info);
      case MODE_MSE: return run_wide<T, ACT, MODE_MSE, REG>(a, ks, st, info);
      case MODE_VALUE: return run_wide<T, ACT, MODE_VALUE, REG>(a, ks, st, info);
      case MODE_JET: return run_wide<T, ACT, MODE_JET, REG>(a, ks, st, info);
    }
    return -1;
  };
  return dispatch_act_reg(act, reg, go);
}

}  // namespace fr

#define FR_DEFINE_WIDE_ENTRY(T, TAG)                                                                      \
  namespace fr {                                                                                         \
  int wide_entry_##TAG(int mode, int act, int reg, const WArgs* a, int ks, cudaStream_t st, WInfo* info) { \
    return dispatch_wide_t<T>(mode, act, reg, a, ks, st, info);                                           \
  }                                                                                                      \
  }
