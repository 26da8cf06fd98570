// TF32 tensor-core wide-expert training kernels (PDE and MSE heads), FP32 I/O.
#include "jetmlp_dispatch.cuh"
#include <algorithm>
#include <cstdlib>
#include <string>

#include "tcwide_kernel.cuh"

namespace fr {

// FR_TC_FWD=tile / FR_TC_DX=tile select the one-tile-per-CTA forward / adjoint
// kernels (A/B measurements)
static bool tc_persistent_fwd() {
  static const bool v = [] {
    const char* e = getenv("FR_TC_FWD");
    return !(e && std::string(e) == "tile");
  }();
  return v;
}
static bool tc_persistent_dx() {
  static const bool v = [] {
    const char* e = getenv("FR_TC_DX");
    return !(e && std::string(e) == "tile");
  }();
  return v;
}
// FR_TC_DWQ=0 selects the weight gradient from row-quad-major Zbar^T copies
// written by the adjoint / head kernels (A/B measurements); default:
// tcw_dwq_kernel reads Zbar straight from the k-quad adjoint slabs
static bool tc_dwq() {
  static const bool v = [] {
    const char* e = getenv("FR_TC_DWQ");
    return !(e && std::string(e) == "0");
  }();
  return v;
}
static int tc_dx_cq() {
  static const int v = [] {
    const char* e = getenv("FR_TC_DX_CQ");
    return (e && std::string(e) == "4") ? 4 : 8;
  }();
  return v;
}
static int tc_num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

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
  const bool dwq = tc_dwq() && ap->WP <= 256;  // tcw_dwq_kernel covers WP <= 256
  WArgs av = *ap;
  if (dwq) av.zt = nullptr;  // no Zbar^T copies
  const WArgs& a = av;
  const int NB = a.nb;
  static bool attrs = false;
  if (!attrs) {
    cudaFuncSetAttribute(tcw_fwd_kernel<ACT, MODE, REG>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::gemm_smem(256)));
    cudaFuncSetAttribute(tcw_fwdp_kernel<ACT, MODE, REG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(sizeof(float) * TCP_NS * C::fwdp_stage_floats(256)));
    cudaFuncSetAttribute(tcw_dx_kernel<ACT, MODE, REG>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::gemm_smem(256)));
    cudaFuncSetAttribute(tcw_dxp_kernel<ACT, MODE, REG, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(tcp_dx_smem<C, 4>(256)));
    cudaFuncSetAttribute(tcw_dxp_kernel<ACT, MODE, REG, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         226 * 1024);
    cudaFuncSetAttribute(tcw_dw_kernel<ACT, MODE, REG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(tcw_head_kernel<ACT, MODE, REG>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::head_smem(512)));
    cudaFuncSetAttribute(tcw_dwq_kernel<ACT, MODE, REG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
    attrs = true;
  }
  const dim3 gt(a.ntiles, a.WP / NB);
  if (tc_persistent_fwd()) {
    const long long items = (long long)a.ntiles * (a.WP / NB);
    const int grid = int(std::min<long long>(items, tc_num_sms()));
    const size_t smem = sizeof(float) * TCP_NS * C::fwdp_stage_floats(NB);
    for (int l = 1; l < a.L; ++l) tcw_fwdp_kernel<ACT, MODE, REG><<<grid, TCP_FWD_NT, smem, st>>>(a, l);
  } else {
    for (int l = 1; l < a.L; ++l) tcw_fwd_kernel<ACT, MODE, REG><<<gt, TC_FWD_NT, C::gemm_smem(NB), st>>>(a, l);
  }
  tcw_head_kernel<ACT, MODE, REG><<<a.ntiles, C::NT, C::head_smem(a.WP), st>>>(a);
  if (tc_persistent_dx()) {
    const long long items = (long long)a.ntiles * (a.WP / NB);
    const int grid = int(std::min<long long>(items, tc_num_sms()));
    // 32-unit epilogue steps where the buffers fit (D150 dx 1.36 -> 1.20 ms;
    // an N block of 208 ends with a 16-unit step); FR_TC_DX_CQ=4 forces 16
    if (tc_dx_cq() == 8 && tcp_dx_smem<C, 8>(NB) <= 226 * 1024) {
      for (int l = a.L - 1; l >= 1; --l)
        tcw_dxp_kernel<ACT, MODE, REG, 8><<<grid, TCP_DX_NT, tcp_dx_smem<C, 8>(NB), st>>>(a, l);
    } else {
      for (int l = a.L - 1; l >= 1; --l)
        tcw_dxp_kernel<ACT, MODE, REG, 4><<<grid, TCP_DX_NT, tcp_dx_smem<C, 4>(NB), st>>>(a, l);
    }
  } else {
    for (int l = a.L - 1; l >= 1; --l) tcw_dx_kernel<ACT, MODE, REG><<<gt, TC_DX_NT, C::gemm_smem(NB), st>>>(a, l);
  }
  // dW: all ceil(WP/128) k-blocks of an N block accumulate in TMEM (<= 512
  // columns); N block = the largest multiple of 16 dividing WP that fits
  const int nkb = (a.WP + 127) / 128;
  int nbw = std::min(256, 512 / nkb) / 16 * 16;
  while (a.WP % nbw) nbw -= 16;
  const int splits = std::max(1, std::min(ks, 148 / (a.WP / nbw)));
  const dim3 gw(a.WP / nbw, splits);
  if (dwq) {
    // converters hold <= 8 quads of each operand per warp; TMEM: nkb x NB (rounded to 32)
    if (a.WP > 256 || nkb * ((nbw + 31) / 32 * 32) > 512)
      return int(cudaErrorInvalidValue);
    const size_t stage = dwq_stage_bytes(a.WP, nbw);
    // as many stages as fit (+ 1 KB for the alignment of the ring)
    int ns = int(std::min<size_t>(DWQ_MAXNS, (225 * 1024) / stage));
    if (const char* e = getenv("FR_DWQ_NS")) ns = std::max(1, std::min(ns, atoi(e)));  // debugging
    // tensor map over the k-quad adjoint slabs ([L * tiles][WP/4][128][4])
    CUtensorMap tmB;
    if (kquad_map(&tmB, a.adj, a.WP, (long long)a.L * a.ntiles, 32, nbw / 4)) return int(cudaErrorNotSupported);
    for (int l = a.L - 1; l >= 1; --l)
      tcw_dwq_kernel<ACT, MODE, REG><<<gw, 320, stage * ns + 1024, st>>>(a, l, nbw, ns, tmB);
  } else {
    const size_t stage = C::dw_stage_bytes(a.WP, nbw);
    const int ns = int(std::min<size_t>(TC_DW_MAXNS, (200 * 1024) / stage));
    for (int l = a.L - 1; l >= 1; --l)
      tcw_dw_kernel<ACT, MODE, REG><<<gw, C::DW_NT, stage * ns, st>>>(a, l, nbw, ns);
  }
  // per-tile partials are laid out on the tensor width WP; gpart on the
  // parameter layout (width WK): dW_0 | db_0 rows of WP -> rows of WK, and
  // dW_L (WP x NOUT) | db_L -> W_L rows then b_L at off_w(L) + WK * NOUT
  const ParamLayout pl{C::DIN, a.WK, C::NOUT, a.L};
  const int len0 = (C::DIN + 1) * a.WP, lenL = a.WP * C::NOUT + C::NOUT;
  tcw_partials_kernel<<<dim3((len0 + 255) / 256, ks), 256, 0, st>>>(a.p0, len0, a.ntiles, a.gpart, a.np_pad, pl.off_w(0),
                                                                      a.WP, a.WK);
  tcw_partials_kernel<<<dim3((lenL + 255) / 256, ks), 256, 0, st>>>(a.pL, lenL, a.ntiles, a.gpart, a.np_pad,
                                                                      pl.off_w(a.L), a.WP * C::NOUT, a.WK * C::NOUT);
  g_kernel_launches += 3 * (a.L - 1) + 3;
  return int(cudaGetLastError());
}

// row-quad-major Zbar^T copies are only written (and allocated) for the
// transposed-copy weight gradient
bool tcwide_needs_zt(int WP) { return !(tc_dwq() && WP <= 256); }

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
