// TF32 tensor-core wide-expert training kernels (PDE and MSE heads), FP32 I/O.
#include "jetmlp_dispatch.cuh"
#include "tcwide_kernel.cuh"

namespace fr {

template <int ACT, int MODE, int REG>
int run_tcwide(const WArgs* ap, int ks, cudaStream_t st, WInfo* info) {
  using C = TcCfg<ACT, MODE, REG>;
  if (info) {
    info->ppt = C::PPT;
    info->rows = 128;
    info->nt = C::NT;
    info->stq = 0;
  }
  if (!ap) return 0;
  const WArgs& a = *ap;
  const int NB = a.WP <= 256 ? a.WP : a.WP / 2;
  static bool attrs = false;
  if (!attrs) {
    cudaFuncSetAttribute(tcw_fwd_kernel<ACT, MODE, REG>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::gemm_smem(256)));
    cudaFuncSetAttribute(tcw_dx_kernel<ACT, MODE, REG>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::gemm_smem(256)));
    cudaFuncSetAttribute(tcw_dw_kernel<ACT, MODE, REG>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::dw_smem(256)));
    cudaFuncSetAttribute(tcw_head_kernel<ACT, MODE, REG>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::head_smem(512)));
    attrs = true;
  }
  const dim3 gt(a.ntiles, a.WP / NB);
  for (int l = 1; l < a.L; ++l) tcw_fwd_kernel<ACT, MODE, REG><<<gt, C::NT, C::gemm_smem(NB), st>>>(a, l, NB);
  tcw_head_kernel<ACT, MODE, REG><<<a.ntiles, C::NT, C::head_smem(a.WP), st>>>(a);
  for (int l = a.L - 1; l >= 1; --l) tcw_dx_kernel<ACT, MODE, REG><<<gt, C::NT, C::gemm_smem(NB), st>>>(a, l, NB);
  const dim3 gw((a.WP + 127) / 128, a.WP / NB, ks);
  for (int l = a.L - 1; l >= 1; --l) tcw_dw_kernel<ACT, MODE, REG><<<gw, C::DW_NT, C::dw_smem(NB), st>>>(a, l, NB);
  tcw_dwL_kernel<ACT, MODE, REG><<<ks, 128, 0, st>>>(a);
  tcw_dw0_kernel<ACT, MODE, REG><<<dim3(ks, (a.WP + 127) / 128), 128, 0, st>>>(a);
  g_kernel_launches += 3 * (a.L - 1) + 3;
  return int(cudaGetLastError());
}

int tcwide_entry_f32(int mode, int act, int reg, const WArgs* a, int ks, cudaStream_t st, WInfo* info) {
  auto go = [&](auto act_c, auto reg_c) -> int {
    constexpr int ACT = decltype(act_c)::value, REG = decltype(reg_c)::value;
    switch (mode) {
      case MODE_PDE: return run_tcwide<ACT, MODE_PDE, REG>(a, ks, st, info);
      case MODE_MSE: return run_tcwide<ACT, MODE_MSE, REG>(a, ks, st, info);
    }
    return -1;
  };
  return dispatch_act_reg(act, reg, go);
}

}  // namespace fr
