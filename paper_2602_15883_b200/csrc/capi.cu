// C ABI: plan, parameter preparation, reductions, Adam, ghost packing, and the
// reference's activation-jet seam.  See include/flowrec_b200.h.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/flowrec_b200.h"
#include "jetmlp_dispatch.cuh"
#include "wide_kernel.cuh"

namespace fr {
#define FR_DECL(NAME) \
  int NAME##_f32(int, int, int, const KArgs*, int, cudaStream_t, KInfo*, int); \
  int NAME##_f64(int, int, int, const KArgs*, int, cudaStream_t, KInfo*, int);
FR_DECL(mode_entry_PDE)
FR_DECL(mode_entry_MSE)
FR_DECL(mode_entry_VALUE)
FR_DECL(mode_entry_JET)
FR_DECL(mode_entry_GJ)
#undef FR_DECL
int epoch_entry_f32(int, int, int, const EpochArgs*, int, cudaStream_t, KInfo*, int, int);
int wide_entry_f32(int, int, int, const WArgs*, int, cudaStream_t, WInfo*);
int wide_entry_f64(int, int, int, const WArgs*, int, cudaStream_t, WInfo*);
int tcwide_entry_f32(int, int, int, const WArgs*, int, cudaStream_t, WInfo*);
bool tcwide_needs_zt(int WP);
int epoch_entry_f64(int, int, int, const EpochArgs*, int, cudaStream_t, KInfo*, int, int);
}  // namespace fr

namespace fr {
long long g_kernel_launches = 0;
}
using namespace fr;

extern "C" long long fr_kernel_launches(void) { return g_kernel_launches; }

static thread_local std::string g_err;

static int fail(const char* fmt, ...) __attribute__((format(printf, 1, 2)));
static int fail(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return 1;
}
// error entry for the other translation units (nccl_transport.cu)
namespace fr {
int fail_msg(const char* msg) {
  g_err = msg;
  return 1;
}
}  // namespace fr
static int cuda_fail(cudaError_t e, const char* where) {
  return fail("%s: CUDA error %d (%s)", where, int(e), cudaGetErrorString(e));
}
#define FR_CUDA(call, where)                        \
  do {                                              \
    cudaError_t e_ = (call);                        \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

struct fr_plan {
  fr_plan_info info;
  ParamLayout pl;
  int* d_map = nullptr;      // real flat index -> padded index      [n_params]
  int* d_mapT = nullptr;     // real flat index -> {W^T copy, fwd slab, dx slab, fwd lo slab, dx lo slab} or -1
                             // [MAPT * n_params]; the lo entries hold f - tf32_trunc(f) (split TF32)
  long long tcw_f = 0, tcw_d = 0;  // kp offsets of the tensor-core operand slabs (0: none)
  long long tc3 = 0;               // kp offset of the W=64 split-TF32 weight slabs (0: none)
  int tc_nb = 0;                   // N of the tensor-core MMAs (output units per CTA)
  int tc_w = 0;                    // tensor width of the TF32 kernels (hidden width rounded to 16 / 32)
  int* d_inv = nullptr;      // kernel-param element -> real index or -1 [kp_elems]
};

extern "C" const char* fr_last_error(void) { return g_err.c_str(); }
extern "C" const char* fr_version(void) { return "flowrec_b200 0.1.0 sm_100a"; }

static int preload_capi_kernels();  // defined at the end of this file
constexpr int MAPT = 5;              // kernel-param copies per flat parameter (fr_plan::d_mapT)
constexpr int FR_INV_LO = 1 << 30;   // inv[] flag: this element holds the split-TF32 low part
constexpr int FR_INV_HI = 1 << 29;   // inv[] flag: ... the split-TF32 high part

// split-TF32 weight pair (fr::tf32_rna, jetmlp_kernel.cuh): hi = round-to-nearest
// TF32 of f (exactly representable, so the tensor core's truncating read is
// exact), lo = the TF32 rounding of f - hi; both errors are unbiased
// (|lo| <= 2^-11 |f|)
template <typename T>
__device__ __forceinline__ T tf32_hi(T v) {
  if constexpr (sizeof(T) == 4) return tf32_rna(v);
  else return v;
}
template <typename T>
__device__ __forceinline__ T tf32_lo(T v) {
  if constexpr (sizeof(T) == 4) return tf32_rna(v - tf32_rna(v));
  else return T(0);
}
extern "C" int fr_plan_destroy(fr_plan* p);

static int regime_dims(int regime, int* din, int* nout, int* nvel) {
  switch (regime) {
    case FR_STEADY2D: *din = 2; *nout = 3; *nvel = 2; return 0;
    case FR_UNSTEADY2D: *din = 3; *nout = 3; *nvel = 2; return 0;
    case FR_UNSTEADY3D: *din = 4; *nout = 4; *nvel = 3; return 0;
    default: return 1;
  }
}

extern "C" int fr_plan_create(const int* arch, int n_arch, int act, int regime, double inv_re, int dtype,
                              fr_plan** out) {
  if (!out) return fail("fr_plan_create: out is NULL");
  *out = nullptr;
  if (!arch || n_arch < 3) return fail("architecture needs at least one hidden layer (got %d entries)", n_arch);
  for (int i = 0; i < n_arch; ++i)
    if (arch[i] < 1) return fail("zero-width layer in architecture (entry %d = %d)", i, arch[i]);
  if (act != FR_ACT_TANH && act != FR_ACT_SIN) return fail("unsupported activation kind %d", act);
  if (dtype != FR_F32 && dtype != FR_F64) return fail("unsupported dtype %d", dtype);
  int din, nout, nvel;
  if (regime_dims(regime, &din, &nout, &nvel)) return fail("unknown regime kind %d", regime);
  if (arch[0] != din) return fail("regime expects %d inputs, architecture has %d", din, arch[0]);
  if (arch[n_arch - 1] != nout)
    return fail("regime expects %d outputs, architecture has %d", nout, arch[n_arch - 1]);
  const int width = arch[1];
  for (int i = 1; i < n_arch - 1; ++i)
    if (arch[i] != width) return fail("hidden layers must share one width (ExpertConfig); got %d and %d", width, arch[i]);
  // widths <= 64 run the fused per-tile kernels; wider experts the layer-wise
  // kernels, padded to whole 64-unit blocks (zero weights: exact)
  int wpad;
  if (width <= 16) wpad = 16;
  else if (width <= 64) wpad = 64;
  else if (width <= 1024) wpad = (width + 63) / 64 * 64;
  else return fail("hidden width %d > 1024 is not supported", width);
  if (!(inv_re > 0.0) || !std::isfinite(inv_re)) return fail("inv_re must be positive and finite");

  fr_plan* p = new fr_plan();
  fr_plan_info& I = p->info;
  I.n_in = din; I.n_out = nout; I.n_vel = nvel;
  I.hidden_layers = n_arch - 2; I.width = width; I.width_pad = wpad;
  I.dtype = dtype; I.act = act; I.regime = regime; I.inv_re = inv_re;
  const int L = I.hidden_layers;
  p->pl = ParamLayout{din, wpad, nout, L};
  I.np_pad = p->pl.np_pad();
  I.kp_elems = p->pl.total();
  // tensor-core operand slabs of the hidden weights (FP32 wide experts): per
  // layer, per N block of NB units, per 16-deep K chunk, a contiguous K-major
  // [4 quads][NB][4] slab -- one for the forward (N = out units, K = in units)
  // and one for the adjoint (N = in units, K = out units)
  // The TF32 kernels run on their own tensor width WT: the hidden width rounded
  // up to the 16-deep K chunk (to 32 above 256 units, so that N = WT/2 is a
  // multiple of 16), not to the 64-unit blocks of the SIMT layout -- padded
  // units carry zero weights either way, so skipping them is exact (D150:
  // 192 -> 160, E: 256 -> 208 units).  Parameters keep the 64-padded layout.
  const bool tc_ok = dtype == FR_F32 && wpad > 64 && wpad <= 512 && I.hidden_layers >= 2;
  const int tc_w = width <= 256 ? (width + 15) / 16 * 16 : (width + 31) / 32 * 32;
  const int tc_nb = tc_w <= 256 ? tc_w : tc_w / 2;
  I.tc_width = tc_ok ? tc_w : 0;
  if (tc_ok) {
    p->tc_nb = tc_nb;
    p->tc_w = tc_w;
    p->tcw_f = (I.kp_elems + 3) & ~3;
    p->tcw_d = p->tcw_f + (long long)(I.hidden_layers - 1) * tc_w * tc_w;
    I.kp_elems = int(p->tcw_d + (long long)(I.hidden_layers - 1) * tc_w * tc_w);
  }
  // W = 64 FP32 fused epoch kernel on the tensor cores (FR_MATH_TF32X3): per
  // hidden layer a forward [k/4][out][4] and an adjoint [k/4][in][4] K-major
  // UMMA slab, each as {hi = f, lo = f - trunc_tf32(f)} (8192 floats), so a
  // contraction is Ah*Bh + Ah*Bl + Al*Bh on tcgen05 (3xTF32, ~FP32 accuracy)
  const bool tc3_ok = dtype == FR_F32 && wpad == 64 && I.hidden_layers >= 2;
  if (tc3_ok) {
    p->tc3 = (I.kp_elems + 3) & ~3;
    I.kp_elems = int(p->tc3 + (long long)(I.hidden_layers - 1) * 2 * 8192);
  }
  // [k/4][128][4]: n < 64 the hi part of B[k][n], n >= 64 the lo part of B[k][n - 64]
  auto tc3_idx = [&](int l, int dir, int lo, int n_unit, int k_unit) -> int {
    return int(p->tc3 + ((long long)(l - 1) * 2 + dir) * 8192 + (k_unit / 4) * 512 + (lo * 64 + n_unit) * 4 +
               (k_unit % 4));
  };
  // wide FP32 experts train on the tcgen05 TF32 path by default (hidden
  // contractions of >= 128 units are real dense GEMMs); fr_plan_set_math
  // switches back to FP32 SIMT
  // FP32 W = 64 plans: split-TF32 tcgen05 contractions in the fused epoch
  // kernel (1.23x the FP32 SIMT epoch at config C, parity ~6e-7)
  I.math = tc_ok ? FR_MATH_TF32 : tc3_ok ? FR_MATH_TF32X3 : FR_MATH_SIMT;
  auto tc_slab = [&](long long base, int l, int n_unit, int k_unit) -> int {
    const int nnb = tc_w / tc_nb, nch = tc_w / 16;
    const int nb = n_unit / tc_nb, n = n_unit % tc_nb, c = k_unit / 16, kq = (k_unit % 16) / 4, j = k_unit % 4;
    return int(base + ((long long)((l - 1) * nnb + nb) * nch + c) * tc_nb * 16 + kq * tc_nb * 4 + n * 4 + j);
  };
  // real flat layout W0,b0,W1,b1,... (network.py:112-115)
  std::vector<int> map, mapT;
  std::vector<int> inv(I.kp_elems, -1);
  for (int l = 0; l <= L; ++l) {
    const int fi = (l == 0) ? din : width;
    const int fo = (l == L) ? nout : width;
    const int fo_pad = (l == L) ? nout : wpad;
    for (int i = 0; i < fi; ++i)
      for (int o = 0; o < fo; ++o) {
        const int pidx = p->pl.off_w(l) + i * fo_pad + o;
        inv[pidx] = int(map.size());
        int tidx = -1, fidx = -1, didx = -1, flo = -1, dlo = -1;
        if (l >= 1 && l < L) {
          tidx = p->pl.off_wt(l) + o * wpad + i;
          inv[tidx] = int(map.size());
          if (tc_ok) {
            fidx = tc_slab(p->tcw_f, l, o, i);
            didx = tc_slab(p->tcw_d, l, i, o);
            inv[fidx] = int(map.size());
            inv[didx] = int(map.size());
          }
          if (tc3_ok) {
            // forward B[n = out][k = in], adjoint B[n = in][k = out]
            fidx = tc3_idx(l, 0, 0, o, i);
            didx = tc3_idx(l, 1, 0, i, o);
            flo = tc3_idx(l, 0, 1, o, i);
            dlo = tc3_idx(l, 1, 1, i, o);
            inv[fidx] = inv[didx] = int(map.size()) | FR_INV_HI;
            inv[flo] = inv[dlo] = int(map.size()) | FR_INV_LO;
          }
        }
        map.push_back(pidx);
        mapT.push_back(tidx);
        mapT.push_back(fidx);
        mapT.push_back(didx);
        mapT.push_back(flo);
        mapT.push_back(dlo);
      }
    for (int o = 0; o < fo; ++o) {
      const int pidx = p->pl.off_b(l) + o;
      inv[pidx] = int(map.size());
      map.push_back(pidx);
      for (int r = 0; r < MAPT; ++r) mapT.push_back(-1);
    }
  }
  I.n_params = int(map.size());
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&I.num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_map, sizeof(int) * map.size());
  if (e == cudaSuccess) e = cudaMalloc(&p->d_inv, sizeof(int) * inv.size());
  if (e == cudaSuccess) e = cudaMalloc(&p->d_mapT, sizeof(int) * mapT.size());
  if (e == cudaSuccess) e = cudaMemcpy(p->d_mapT, mapT.data(), sizeof(int) * mapT.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(p->d_map, map.data(), sizeof(int) * map.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(p->d_inv, inv.data(), sizeof(int) * inv.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(p->d_map);
    cudaFree(p->d_inv);
    cudaFree(p->d_mapT);
    delete p;
    return cuda_fail(e, "fr_plan_create");
  }
  // the transport's signal kernel (and the epoch's reductions / optimiser)
  // must be resident before a gated epoch kernel spins on them: with lazy
  // module loading (CUDA_MODULE_LOADING=LAZY, the default) a first launch
  // would otherwise wait for the device to idle.  Once per plan (plans are
  // per device), not per launch.
  if (int rc = preload_capi_kernels()) {
    fr_plan_destroy(p);
    return rc;
  }
  *out = p;
  return 0;
}

extern "C" int fr_plan_destroy(fr_plan* p) {
  if (!p) return 0;
  cudaFree(p->d_map);
  cudaFree(p->d_inv);
  cudaFree(p->d_mapT);
  delete p;
  return 0;
}

extern "C" int fr_plan_set_math(fr_plan* p, int math) {
  if (!p) return fail("fr_plan_set_math: NULL plan");
  if (math == FR_MATH_SIMT) {
    p->info.math = math;
    return 0;
  }
  if (math == FR_MATH_TF32X3) {
    if (p->tc3 == 0)
      return fail("split-TF32 tensor-core math covers FP32 plans of hidden width <= 64 with >= 2 hidden layers");
    p->info.math = math;
    return 0;
  }
  if (math != FR_MATH_TF32) return fail("unknown math mode %d", math);
  const fr_plan_info& I = p->info;
  if (I.dtype != FR_F32) return fail("TF32 tensor-core math needs an FP32 plan");
  if (p->tc_nb == 0)
    return fail("TF32 tensor-core math covers hidden widths 65..512 with >= 2 hidden layers (got %d x %d)", I.width,
                I.hidden_layers);
  p->info.math = math;
  return 0;
}

extern "C" int fr_plan_get_info(const fr_plan* p, fr_plan_info* out) {
  if (!p || !out) return fail("fr_plan_get_info: NULL argument");
  *out = p->info;
  return 0;
}

static int mode_call(const fr_plan* p, int mode, const KArgs* a, int grid, cudaStream_t st, KInfo* info) {
  const fr_plan_info& I = p->info;
  const bool f32 = I.dtype == FR_F32;
  const int act = I.act, reg = I.regime, w = I.width_pad, L = I.hidden_layers;
  int r;
  switch (mode) {
    case FR_MODE_PDE:
      r = f32 ? mode_entry_PDE_f32(act, reg, w, a, grid, st, info, L) : mode_entry_PDE_f64(act, reg, w, a, grid, st, info, L);
      break;
    case FR_MODE_MSE:
      r = f32 ? mode_entry_MSE_f32(act, reg, w, a, grid, st, info, L) : mode_entry_MSE_f64(act, reg, w, a, grid, st, info, L);
      break;
    case FR_MODE_VALUE:
      r = f32 ? mode_entry_VALUE_f32(act, reg, w, a, grid, st, info, L)
              : mode_entry_VALUE_f64(act, reg, w, a, grid, st, info, L);
      break;
    case FR_MODE_JET:
      r = f32 ? mode_entry_JET_f32(act, reg, w, a, grid, st, info, L) : mode_entry_JET_f64(act, reg, w, a, grid, st, info, L);
      break;
    case FR_MODE_GJ:
      r = f32 ? mode_entry_GJ_f32(act, reg, w, a, grid, st, info, L) : mode_entry_GJ_f64(act, reg, w, a, grid, st, info, L);
      break;
    default: return fail("unknown mode %d", mode);
  }
  if (r == -1) return fail("kernel variant not compiled (mode %d dtype %d act %d regime %d width %d)", mode, I.dtype, I.act, I.regime, I.width_pad);
  if (r != 0) return cuda_fail(cudaError_t(r), "jet-MLP kernel launch");
  return 0;
}

static int epoch_call(const fr_plan* p, const EpochArgs* e, int grid, cudaStream_t st, KInfo* info) {
  const fr_plan_info& I = p->info;
  const int tc = I.math == FR_MATH_TF32X3;
  const int r = I.dtype == FR_F32
                    ? epoch_entry_f32(I.act, I.regime, I.width_pad, e, grid, st, info, I.hidden_layers, tc)
                    : epoch_entry_f64(I.act, I.regime, I.width_pad, e, grid, st, info, I.hidden_layers, tc);
  if (r == -1) return fail("epoch kernel variant not compiled (math %d)", I.math);
  if (r != 0) return cuda_fail(cudaError_t(r), "epoch kernel launch");
  return 0;
}

constexpr int WIDE_KS = 32;  // gradient-partial rows (row splits) of the SIMT wide kernels
constexpr int TC_KS = 128;   // ... of the tensor-core wide kernels

static bool is_wide(const fr_plan* p) { return p->info.width_pad > 64; }
// training heads of TF32 plans run on the tcgen05 kernels (prediction stays SIMT)
static bool is_tc(const fr_plan* p, int mode) {
  return is_wide(p) && p->tc_nb > 0 && p->info.math == FR_MATH_TF32 && (mode == FR_MODE_PDE || mode == FR_MODE_MSE);
}
static int wide_ks(const fr_plan* p, int mode) { return is_tc(p, mode) ? TC_KS : WIDE_KS; }

static int wide_call(const fr_plan* p, int mode, const WArgs* a, cudaStream_t st, WInfo* wi) {
  const fr_plan_info& I = p->info;
  const int r = is_tc(p, mode) ? tcwide_entry_f32(mode, I.act, I.regime, a, TC_KS, st, wi)
                : I.dtype == FR_F32 ? wide_entry_f32(mode, I.act, I.regime, a, WIDE_KS, st, wi)
                                    : wide_entry_f64(mode, I.act, I.regime, a, WIDE_KS, st, wi);
  if (r == -1) return fail("wide kernel variant not compiled");
  if (r != 0) return cuda_fail(cudaError_t(r), "wide kernel launch");
  return 0;
}

struct WideSizes {
  long long ntiles, act, stash, ybar, total;  // elements of T
};
static int wide_sizes(const fr_plan* p, int mode, long long n, WideSizes* z, WInfo* wi) {
  if (wide_call(p, mode, nullptr, nullptr, wi)) return 1;
  const fr_plan_info& I = p->info;
  const long long L = I.hidden_layers, WP = is_tc(p, mode) ? p->tc_w : I.width_pad;
  z->ntiles = (n + wi->ppt - 1) / wi->ppt;
  z->act = L * z->ntiles * WP * wi->rows;
  const bool bwd = (mode == FR_MODE_PDE || mode == FR_MODE_MSE || mode == FR_MODE_GJ);
  // SIMT: activation stash; tensor cores: row-quad-major S_l and Zbar_l copies
  z->stash = !bwd ? 0
             : is_tc(p, mode) ? (tcwide_needs_zt(int(WP)) ? 2 : 1) * L * z->ntiles * WP * 128
                              : L * z->ntiles * (WP / 64) * (long long)wi->stq * wi->nt;
  // SIMT: Ybar rows; tensor cores: per-tile dW_0|db_0 and dW_L|db_L partials
  z->ybar = !bwd ? 0
            : is_tc(p, mode) ? z->ntiles * ((I.n_in + 1) * WP + WP * I.n_out + I.n_out)
                             : z->ntiles * wi->rows * I.n_out;
  auto al = [](long long e) { return (e + 63) / 64 * 64; };
  z->total = al(z->act) + (bwd ? al(z->act) : 0) + al(z->stash) + al(z->ybar);
  return 0;
}

extern "C" int fr_plan_workspace(const fr_plan* p, int mode, long long n, fr_workspace* out) {
  if (!p || !out) return fail("fr_plan_workspace: NULL argument");
  if (n < 0) return fail("negative point count");
  if (is_wide(p)) {
    WideSizes z;
    WInfo wi{};
    if (wide_sizes(p, mode, n, &z, &wi)) return 1;
    const bool bwd = (mode == FR_MODE_PDE || mode == FR_MODE_MSE || mode == FR_MODE_GJ);
    const size_t esz = p->info.dtype == FR_F32 ? 4 : 8;
    const int ks = wide_ks(p, mode);
    out->grid = ks;
    out->threads = wi.nt;
    out->points_per_tile = wi.ppt;
    out->jet_streams = 1 + 2 * p->info.n_in;
    out->gpart_elems = bwd ? (long long)ks * p->info.np_pad : 0;
    out->lpart_elems = bwd ? z.ntiles * 2 : 0;
    out->loss_rows = bwd ? int(z.ntiles) : 0;
    out->scratch_bytes = z.total * (long long)esz;
    out->smem_bytes = 0;
    out->wide = is_tc(p, mode) ? 2 : 1;
    out->tiles = z.ntiles;
    return 0;
  }
  KInfo ki{};
  if (mode_call(p, mode, nullptr, 0, nullptr, &ki)) return 1;
  const fr_plan_info& I = p->info;
  const long long ntiles = (n + ki.ppt - 1) / ki.ppt;
  const int sms = I.num_sms > 0 ? I.num_sms : 148;
  out->grid = int(ntiles < sms ? ntiles : sms);
  out->tiles = ntiles;
  out->threads = ki.nt;
  out->points_per_tile = ki.ppt;
  out->jet_streams = 1 + 2 * I.n_in;
  const bool bwd = (mode == FR_MODE_PDE || mode == FR_MODE_MSE || mode == FR_MODE_GJ);
  out->gpart_elems = bwd ? (long long)out->grid * I.np_pad : 0;
  out->lpart_elems = bwd ? (long long)out->grid * 2 : 0;
  const size_t esz = I.dtype == FR_F32 ? 4 : 8;
  out->scratch_bytes = bwd ? (long long)out->grid * ki.stash_elems * (long long)esz : 0;
  out->smem_bytes = ki.smem;
  out->loss_rows = bwd ? out->grid : 0;
  out->wide = 0;
  return 0;
}

// Layer-wise path: fill WArgs over a caller scratch buffer (or a stream-ordered
// allocation for the forward-only entry points, which take no workspace) and
// launch the sequence.
static int launch_wide(const fr_plan* p, int mode, WArgs& a, long long n, void* scratch, cudaStream_t st) {
  const fr_plan_info& I = p->info;
  WideSizes z;
  WInfo wi{};
  if (wide_sizes(p, mode, n, &z, &wi)) return 1;
  if (n == 0) return 0;
  const size_t esz = I.dtype == FR_F32 ? 4 : 8;
  void* owned = nullptr;
  if (!scratch) {
    FR_CUDA(cudaMallocAsync(&owned, size_t(z.total) * esz, st), "wide workspace allocation");
    scratch = owned;
  }
  auto al = [](long long e) { return (e + 63) / 64 * 64; };
  char* base = static_cast<char*>(scratch);
  const bool bwd = (mode == FR_MODE_PDE || mode == FR_MODE_MSE || mode == FR_MODE_GJ);
  a.act = base;
  base += al(z.act) * esz;
  if (bwd) {
    a.adj = base;
    base += al(z.act) * esz;
  }
  a.stash = base;
  base += al(z.stash) * esz;
  a.ybar = base;
  a.n = n;
  a.ntiles = int(z.ntiles);
  a.L = I.hidden_layers;
  a.WP = is_tc(p, mode) ? p->tc_w : I.width_pad;
  a.WK = I.width_pad;
  a.np_pad = I.np_pad;
  a.ks_rows = wide_ks(p, mode);
  if (is_tc(p, mode)) {
    a.tcw_f = p->tcw_f;
    a.tcw_d = p->tcw_d;
    a.nb = p->tc_nb;
    a.p0 = static_cast<float*>(a.ybar);
    a.pL = a.p0 + size_t(z.ntiles) * (I.n_in + 1) * a.WP;
    a.st = static_cast<float*>(a.stash);
    a.zt = tcwide_needs_zt(a.WP) ? a.st + size_t(a.L) * z.ntiles * a.WP * 128 : nullptr;
  }
  a.inv_re = I.inv_re;
  if (bwd) FR_CUDA(cudaMemsetAsync(a.gpart, 0, sizeof(double) * size_t(a.ks_rows) * I.np_pad, st), "gpart zero");
  const int r = wide_call(p, mode, &a, st, nullptr);
  if (owned) cudaFreeAsync(owned, st);
  return r;
}

// ---------------------------------------------------------------------------
template <typename T>
__global__ void prepare_kernel(const double* __restrict__ flat, const int* __restrict__ inv, T* kp, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int r = inv[i];
    if (r < 0) {
      kp[i] = T(0);
    } else if (r & FR_INV_LO) {
      kp[i] = tf32_lo(T(flat[r & ~FR_INV_LO]));
    } else if (r & FR_INV_HI) {
      kp[i] = tf32_hi(T(flat[r & ~FR_INV_HI]));
    } else {
      kp[i] = T(flat[r]);
    }
  }
}

extern "C" int fr_prepare_params(const fr_plan* p, const double* flat, void* kparams, fr_stream_t stream) {
  if (!p || !flat || !kparams) return fail("fr_prepare_params: NULL argument");
  const int n = p->info.kp_elems;
  const int blocks = (n + 255) / 256;
  if (p->info.dtype == FR_F32)
    prepare_kernel<float><<<blocks, 256, 0, stream>>>(flat, p->d_inv, static_cast<float*>(kparams), n);
  else
    prepare_kernel<double><<<blocks, 256, 0, stream>>>(flat, p->d_inv, static_cast<double*>(kparams), n);
  ++g_kernel_launches;
  FR_CUDA(cudaGetLastError(), "fr_prepare_params");
  return 0;
}

static int launch_train(const fr_plan* p, int mode, KArgs& a, long long n, cudaStream_t st) {
  if (is_wide(p)) {
    WArgs w{};
    w.kp = a.kp; w.pts = a.pts; w.tu = a.tu; w.tp = a.tp; w.out = a.out;
    w.gpart = a.gpart; w.lpart = a.lpart;
    w.coef = a.coef; w.pcoef = a.pcoef; w.has_p = a.has_p;
    for (int c = 0; c < 4; ++c) w.velw[c] = a.velw[c];
    return launch_wide(p, mode, w, n, a.scratch, st);
  }
  fr_workspace ws;
  if (fr_plan_workspace(p, mode, n, &ws)) return 1;
  a.n = n;
  a.L = p->info.hidden_layers;
  a.np_pad = p->info.np_pad;
  KInfo ki{};
  if (mode_call(p, mode, nullptr, 0, nullptr, &ki)) return 1;
  a.stash_elems = ki.stash_elems;
  a.inv_re = p->info.inv_re;
  if (ws.grid == 0) return 0;
  return mode_call(p, mode, &a, ws.grid, st, nullptr);
}

extern "C" int fr_pde_fwd_bwd(const fr_plan* p, const void* kparams, const void* pts, long long n, double coef,
                              double* gpart, double* lpart, void* scratch, fr_stream_t stream) {
  if (!p || !kparams || (n > 0 && (!pts || !gpart || !lpart || !scratch)))
    return fail("fr_pde_fwd_bwd: NULL argument");
  if (n < 0) return fail("fr_pde_fwd_bwd: negative point count");
  KArgs a{};
  a.kp = kparams; a.pts = pts; a.gpart = gpart; a.lpart = lpart; a.scratch = scratch;
  a.coef = coef;
  return launch_train(p, FR_MODE_PDE, a, n, stream);
}

extern "C" int fr_mse_fwd_bwd(const fr_plan* p, const void* kparams, const void* pts, const void* target_u,
                              const void* target_p, long long n, const double* vel_w, double vel_coef,
                              double p_coef, double* gpart, double* lpart, void* scratch, fr_stream_t stream) {
  if (!p || !kparams || (n > 0 && (!pts || !target_u || !gpart || !lpart || !scratch)))
    return fail("fr_mse_fwd_bwd: NULL argument");
  if (n < 0) return fail("fr_mse_fwd_bwd: negative point count");
  KArgs a{};
  a.kp = kparams; a.pts = pts; a.tu = target_u; a.tp = target_p;
  a.gpart = gpart; a.lpart = lpart; a.scratch = scratch;
  a.coef = vel_coef; a.pcoef = p_coef; a.has_p = target_p != nullptr;
  for (int c = 0; c < 4; ++c) a.velw[c] = 1.0;
  if (vel_w)
    for (int c = 0; c < p->info.n_vel; ++c) a.velw[c] = vel_w[c];
  return launch_train(p, FR_MODE_MSE, a, n, stream);
}

static int epoch_info(const fr_plan* p, KInfo* ki) {
  if (is_wide(p)) return fail("the fused epoch kernel needs hidden width <= 64 (use the per-dataset entry points)");
  return epoch_call(p, nullptr, 0, nullptr, ki);
}

extern "C" int fr_epoch_workspace(const fr_plan* p, long long n_colloc, const long long* n_sets, int n_set_count,
                                  fr_workspace* out) {
  return fr_epoch_workspace_capped(p, n_colloc, n_sets, n_set_count, 0, out);
}

extern "C" int fr_epoch_workspace_capped(const fr_plan* p, long long n_colloc, const long long* n_sets,
                                         int n_set_count, int max_ctas, fr_workspace* out) {
  if (!p || !out || n_set_count < 0 || n_set_count > 3 || (n_set_count && !n_sets) || max_ctas < 0)
    return fail("fr_epoch_workspace: bad arguments");
  KInfo ki{};
  if (epoch_info(p, &ki)) return 1;
  int sms = p->info.num_sms > 0 ? p->info.num_sms : 148;
  if (max_ctas > 0 && max_ctas < sms) sms = max_ctas;  // an SM budget: the grid is sms x CTAs per SM
  sms *= ki.cps;
  long long tiles = (n_colloc + ki.ppt - 1) / ki.ppt;
  for (int i = 0; i < n_set_count; ++i) tiles += (n_sets[i] + ki.ppt_mse - 1) / ki.ppt_mse;
  out->grid = int(tiles < sms ? (tiles > 0 ? tiles : 1) : sms);
  out->tiles = tiles;
  out->threads = ki.nt;
  out->points_per_tile = ki.ppt;
  out->jet_streams = 0;
  out->gpart_elems = (long long)out->grid * p->info.np_pad;
  out->lpart_elems = (long long)out->grid * 2 * (1 + n_set_count);
  out->scratch_bytes = (long long)out->grid * ki.stash_elems * (p->info.dtype == FR_F32 ? 4 : 8);
  out->smem_bytes = ki.smem;
  return 0;
}

__global__ void signal_kernel(unsigned* word, unsigned value, unsigned delay_ns) {
  if (delay_ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
      __nanosleep(1000);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < delay_ns);
  }
  __threadfence_system();
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(word), "r"(value) : "memory");
}

extern "C" int fr_epoch_fwd_bwd(const fr_plan* p, const void* kparams, const void* colloc, long long n_colloc,
                                double pde_coef, const fr_mse_set* sets, int n_set_count, const double* vel_w,
                                double* gpart, double* const* lpart_blocks, void* scratch, fr_stream_t stream) {
  return fr_epoch_fwd_bwd_gated(p, kparams, colloc, n_colloc, pde_coef, sets, n_set_count, vel_w, gpart,
                                lpart_blocks, scratch, nullptr, stream);
}

extern "C" int fr_epoch_fwd_bwd_gated(const fr_plan* p, const void* kparams, const void* colloc, long long n_colloc,
                                      double pde_coef, const fr_mse_set* sets, int n_set_count, const double* vel_w,
                                      double* gpart, double* const* lpart_blocks, void* scratch,
                                      const fr_epoch_gate* gate, fr_stream_t stream) {
  if (!p || !kparams || !colloc || n_colloc < 1 || !gpart || !lpart_blocks || !scratch || n_set_count < 0 ||
      n_set_count > 3 || (n_set_count && !sets))
    return fail("fr_epoch_fwd_bwd: bad arguments");
  // a gate with a NULL word only caps the grid (ungated epochs of a trainer whose
  // workspace was sized with fr_epoch_workspace_capped must launch the same grid)
  if (gate && (gate->first_gated_set < 0 || gate->max_ctas < 0)) return fail("fr_epoch_fwd_bwd_gated: bad gate");
  if (gate && p->info.width_pad > 64) return fail("fr_epoch_fwd_bwd_gated: fused epoch path only (width <= 64)");
  long long ns[3] = {0, 0, 0};
  for (int i = 0; i < n_set_count; ++i) {
    if (sets[i].n < 0 || (sets[i].n > 0 && (!sets[i].pts || !sets[i].target_u)))
      return fail("fr_epoch_fwd_bwd: bad MSE set %d", i);
    ns[i] = sets[i].n;
  }
  for (int i = 0; i < 1 + n_set_count; ++i)
    if (!lpart_blocks[i]) return fail("fr_epoch_fwd_bwd: NULL loss-partial block %d", i);
  fr_workspace ws;
  if (fr_epoch_workspace_capped(p, n_colloc, ns, n_set_count, gate ? gate->max_ctas : 0, &ws)) return 1;
  KInfo ki{};
  if (epoch_info(p, &ki)) return 1;
  const fr_plan_info& I = p->info;
  EpochArgs e{};
  auto fill = [&](KArgs& a, long long n) {
    a.kp = kparams;
    a.gpart = gpart;
    a.scratch = scratch;
    a.n = n;
    a.L = I.hidden_layers;
    a.np_pad = I.np_pad;
    a.stash_elems = ki.stash_elems;
    a.inv_re = I.inv_re;
    for (int c = 0; c < 4; ++c) a.velw[c] = 1.0;
    if (vel_w)
      for (int c = 0; c < I.n_vel; ++c) a.velw[c] = vel_w[c];
  };
  fill(e.pde, n_colloc);
  const long long tc3 = I.math == FR_MATH_TF32X3 ? p->tc3 : 0;
  e.pde.tc3 = tc3;
  e.pde.pts = colloc;
  e.pde.coef = pde_coef;
  e.pde.lpart = lpart_blocks[0];
  e.n_mse = n_set_count;
  for (int i = 0; i < n_set_count; ++i) {
    fill(e.mse[i], sets[i].n);
    e.mse[i].tc3 = tc3;
    e.mse[i].pts = sets[i].pts;
    e.mse[i].tu = sets[i].target_u;
    e.mse[i].tp = sets[i].target_p;
    e.mse[i].has_p = sets[i].target_p != nullptr;
    e.mse[i].coef = sets[i].vel_coef;
    e.mse[i].pcoef = sets[i].p_coef;
    e.mse[i].lpart = lpart_blocks[1 + i];
    if (gate && gate->gate && i >= gate->first_gated_set) {
      e.mse[i].gate = gate->gate;
      e.mse[i].gate_round = gate->gate_round;
      e.mse[i].gate_mult = gate->gate_mult;
      e.mse[i].flags = gate->flags;
      e.mse[i].gate_timeout_ns = (unsigned long long)(gate->timeout_ms ? gate->timeout_ms : 60000u) * 1000000ull;
    }
  }
  return epoch_call(p, &e, ws.grid, stream, nullptr);
}

extern "C" int fr_signal(unsigned* word, unsigned value, unsigned delay_ns, fr_stream_t stream) {
  if (!word) return fail("fr_signal: NULL word");
  signal_kernel<<<1, 1, 0, stream>>>(word, value, delay_ns);
  ++g_kernel_launches;
  FR_CUDA(cudaGetLastError(), "fr_signal");
  return 0;
}

extern "C" int fr_ghost_jet_fwd_bwd(const fr_plan* p, const void* kparams, const void* pts, const void* target_du,
                                    long long n, const double* vel_w, double coef, double* gpart, double* lpart,
                                    void* scratch, fr_stream_t stream) {
  if (!p || !kparams || (n > 0 && (!pts || !target_du || !gpart || !lpart || !scratch)))
    return fail("fr_ghost_jet_fwd_bwd: NULL argument");
  if (n < 0) return fail("fr_ghost_jet_fwd_bwd: negative point count");
  if (is_wide(p)) return fail("fr_ghost_jet_fwd_bwd: hidden width > 64 is not supported by the extension");
  KArgs a{};
  a.kp = kparams; a.pts = pts; a.tu = target_du; a.gpart = gpart; a.lpart = lpart; a.scratch = scratch;
  a.coef = coef;
  for (int c = 0; c < 4; ++c) a.velw[c] = 1.0;
  if (vel_w)
    for (int c = 0; c < p->info.n_vel; ++c) a.velw[c] = vel_w[c];
  return launch_train(p, FR_MODE_GJ, a, n, stream);
}

extern "C" int fr_value_fwd(const fr_plan* p, const void* kparams, const void* pts, long long n, void* out,
                            fr_stream_t stream) {
  if (!p || !kparams || (n > 0 && (!pts || !out))) return fail("fr_value_fwd: NULL argument");
  KArgs a{};
  a.kp = kparams; a.pts = pts; a.out = out;
  return launch_train(p, FR_MODE_VALUE, a, n, stream);
}

extern "C" int fr_jet_fwd(const fr_plan* p, const void* kparams, const void* pts, long long n, void* out,
                          fr_stream_t stream) {
  if (!p || !kparams || (n > 0 && (!pts || !out))) return fail("fr_jet_fwd: NULL argument");
  KArgs a{};
  a.kp = kparams; a.pts = pts; a.out = out;
  return launch_train(p, FR_MODE_JET, a, n, stream);
}

// ---------------------------------------------------------------------------
// 32 parameters x 16 row groups per block: coalesced 256-byte row reads, the 16
// partial sums combined in a fixed order, then a fixed-order block sum of g^2
// for the optimiser's global norm.
constexpr int RG_P = 32, RG_R = 16;  // 16 row groups: short dependent chains over the ~148 partial rows
__global__ void __launch_bounds__(RG_P * RG_R) reduce_grad_kernel(const double* __restrict__ gpart, int rows, int np_pad,
                                                                  const int* __restrict__ map, int n, double* grad,
                                                                  int accumulate, double* norm_parts) {
  __shared__ double part[RG_R][RG_P];
  const int tx = threadIdx.x % RG_P, ty = threadIdx.x / RG_P;
  const int i = blockIdx.x * RG_P + tx;
  double s = 0.0;
  if (i < n) {
    const double* col = gpart + map[i];
    int r = ty;
#pragma unroll 4
    for (; r < rows; r += RG_R) s += col[size_t(r) * np_pad];
  }
  part[ty][tx] = s;
  __syncthreads();
  if (ty == 0) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < RG_R; ++q) t += part[q][tx];
    double g = 0.0;
    if (i < n) {
      g = accumulate ? grad[i] + t : t;
      grad[i] = g;
    }
    if (norm_parts) {
      double sq = g * g;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sq += __shfl_down_sync(0xffffffffu, sq, o);
      if (tx == 0) norm_parts[blockIdx.x] = sq;
    }
  }
}

extern "C" int fr_reduce_grad_parts(const fr_plan* p) { return p ? (p->info.n_params + RG_P - 1) / RG_P : 0; }

extern "C" int fr_reduce_grad(const fr_plan* p, const double* gpart, int rows, double* grad, int accumulate,
                              double* norm_parts, fr_stream_t stream) {
  if (!p || !grad || (rows > 0 && !gpart)) return fail("fr_reduce_grad: NULL argument");
  const int n = p->info.n_params;
  if (rows <= 0 && accumulate && !norm_parts) return 0;
  reduce_grad_kernel<<<(n + RG_P - 1) / RG_P, RG_P * RG_R, 0, stream>>>(gpart, rows > 0 ? rows : 0, p->info.np_pad,
                                                                        p->d_map, n, grad, accumulate, norm_parts);
  ++g_kernel_launches;
  FR_CUDA(cudaGetLastError(), "fr_reduce_grad");
  return 0;
}

struct SegRows {
  int n;
  int rows[8];
};
// ---------------------------------------------------------------------------
// Adam (optim.py:20-49) with the epoch bookkeeping of objective.py:183-198 and
// worker.py:231-244.  Multi-CTA: every block redundantly forms the global norm
// and the loss parts from the partials in the same fixed order, updates its
// slice of parameters and refreshes the kernel copy; the last block to finish
// advances the step counter.  f64 arithmetic uses explicit round-to-nearest
// intrinsics so no FMA contraction changes the reference's rounding sequence.
// ---------------------------------------------------------------------------
constexpr int ADAM_NT = 256;

__device__ double block_sum_fixed(double v, double* red) {
  // fixed-shape tree: identical order in every block and on every run
  red[threadIdx.x] = v;
  __syncthreads();
  for (int w = ADAM_NT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}

// N independent values through the same fixed-shape tree at once (one barrier
// per level for all of them): bit-identical to N block_sum_fixed calls
template <int N>
__device__ void block_sum_fixed_n(double (&v)[N], double* red /* N * ADAM_NT */) {
#pragma unroll
  for (int k = 0; k < N; ++k) red[k * ADAM_NT + threadIdx.x] = v[k];
  __syncthreads();
  for (int w = ADAM_NT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
#pragma unroll
      for (int k = 0; k < N; ++k)
        red[k * ADAM_NT + threadIdx.x] = __dadd_rn(red[k * ADAM_NT + threadIdx.x], red[k * ADAM_NT + threadIdx.x + w]);
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = red[k * ADAM_NT];
  __syncthreads();
}

// One block per segment, the same strided partial sums + fixed tree as the
// optimiser kernel's loss reduction below, so `sums` equals the history row's
// parts bit for bit (and the wide path's tens of thousands of tile rows reduce
// in parallel).
__global__ void __launch_bounds__(ADAM_NT) reduce_loss_kernel(const double* __restrict__ lpart, SegRows seg,
                                                              double* sums) {
  __shared__ double red[ADAM_NT];
  const int s = blockIdx.x;
  int r0 = 0;
  for (int i = 0; i < s; ++i) r0 += seg.rows[i];
  double x = 0.0, y = 0.0;
  for (int r = r0 + threadIdx.x; r < r0 + seg.rows[s]; r += ADAM_NT) {
    x += lpart[2 * r];
    y += lpart[2 * r + 1];
  }
  x = block_sum_fixed(x, red);
  y = block_sum_fixed(y, red);
  if (threadIdx.x == 0) {
    sums[2 * s] = x;
    sums[2 * s + 1] = y;
  }
}

extern "C" int fr_reduce_loss(const double* lpart, const int* seg_rows_host, int n_seg, double* sums,
                              fr_stream_t stream) {
  if (!sums || !seg_rows_host || n_seg < 1 || n_seg > 8) return fail("fr_reduce_loss: bad arguments");
  SegRows seg{};
  seg.n = n_seg;
  int total = 0;
  for (int i = 0; i < n_seg; ++i) {
    seg.rows[i] = seg_rows_host[i];
    total += seg_rows_host[i];
  }
  if (total > 0 && !lpart) return fail("fr_reduce_loss: NULL lpart");
  reduce_loss_kernel<<<n_seg, ADAM_NT, 0, stream>>>(lpart, seg, sums);
  ++g_kernel_launches;
  FR_CUDA(cudaGetLastError(), "fr_reduce_loss");
  return 0;
}

template <typename T>
__global__ void __launch_bounds__(ADAM_NT) adam_kernel(fr_adam_args a, int n, const int* __restrict__ map,
                                                       const int* __restrict__ mapT) {
  __shared__ double red9[9 * ADAM_NT];
  const int tid = threadIdx.x;
  const long long step0 = *a.step;  // steps taken so far
  const long long row = step0 - a.row_base;

  // ---- global gradient norm (optim.py:20-28) ----
  double acc = 0.0;
  if (a.norm_parts) {
    for (int i = tid; i < a.n_norm_parts; i += ADAM_NT) acc = __dadd_rn(acc, a.norm_parts[i]);
  } else {
    for (int i = tid; i < n; i += ADAM_NT) acc = __dadd_rn(acc, __dmul_rn(a.grad[i], a.grad[i]));
  }
  // the norm and the 8 loss sums share one pass of the fixed tree (identical
  // per-value order to separate trees: the history row still equals
  // fr_reduce_loss's sums bit for bit)
  double vals[9];
  vals[0] = acc;
  if (a.lpart) {
    int r0 = 0;
    for (int sgi = 0; sgi < 4; ++sgi) {
      double x = 0.0, y = 0.0;
      for (int r = r0 + tid; r < r0 + a.seg_rows[sgi]; r += ADAM_NT) {
        x += a.lpart[2 * r];
        y += a.lpart[2 * r + 1];
      }
      vals[1 + 2 * sgi] = x;
      vals[2 + 2 * sgi] = y;
      r0 += a.seg_rows[sgi];
    }
  } else {
#pragma unroll
    for (int k = 1; k < 9; ++k) vals[k] = 0.0;
  }
  block_sum_fixed_n<9>(vals, red9);
  const double norm = sqrt(vals[0]);

  // ---- loss parts, history row, finiteness (objective.py:183-198) ----
  bool skip = false;
  if (a.lpart) {
    double sums[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) sums[k] = vals[1 + k];
    const double obs = a.n_obs > 0 ? sums[0] / a.n_obs : 0.0;
    const double pde = sums[2] / a.n_colloc;
    const double gu = a.n_ghost_total > 0 ? (sums[4] + sums[6]) / a.n_ghost_total : 0.0;
    const double gps = a.n_ghost_space > 0 ? sums[5] / a.n_ghost_space : 0.0;
    const double gpt = a.n_ghost_time > 0 ? sums[7] / a.n_ghost_time : 0.0;
    // compose_loss (physics.py:214-224), left to right
    double total = __dmul_rn(a.w_obs, obs);
    total = __dadd_rn(total, __dmul_rn(a.w_pde, pde));
    total = __dadd_rn(total, __dmul_rn(a.w_ghost_u, gu));
    total = __dadd_rn(total, __dmul_rn(a.w_ghost_p_space, gps));
    total = __dadd_rn(total, __dmul_rn(a.w_ghost_p_time, gpt));
    skip = !isfinite(total);
    if (blockIdx.x == 0 && tid == 0) {
      if (a.history) {
        double* h = a.history + 7 * row;
        h[0] = double(step0);
        h[1] = obs; h[2] = pde; h[3] = gu; h[4] = gps; h[5] = gpt;
        h[6] = a.sched[3 * row];
      }
      if (skip) atomicOr(a.flags, FR_FLAG_NONFINITE_LOSS);
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    if (a.grad_norm) a.grad_norm[row] = norm;
    if (!isfinite(norm)) atomicOr(a.flags, FR_FLAG_NONFINITE_GRAD);
  }
  skip = skip || !isfinite(norm);

  // ---- update (optim.py:31-49) ----
  const int i = blockIdx.x * ADAM_NT + tid;
  if (!skip && i < n) {
    // clip_by_global_norm: `clip_norm is not None and norm > clip_norm`; None is
    // NaN here, so the comparison is false (optim.py:26-27)
    const double scale = (norm > a.clip_norm) ? a.clip_norm / norm : 1.0;
    const double lr = a.sched[3 * row];
    const double bc1 = a.sched[3 * row + 1];
    const double bc2 = a.sched[3 * row + 2];
    const double omb1 = 1.0 - a.beta1, omb2 = 1.0 - a.beta2;
    double g = a.grad[i];
    if (scale != 1.0) {
      g = __dmul_rn(g, scale);
      a.grad[i] = g;
    }
    const double m = __dadd_rn(__dmul_rn(a.m[i], a.beta1), __dmul_rn(omb1, g));
    const double v = __dadd_rn(__dmul_rn(a.v[i], a.beta2), __dmul_rn(__dmul_rn(omb2, g), g));
    a.m[i] = m;
    a.v[i] = v;
    const double mh = __ddiv_rn(m, bc1);
    const double vh = __ddiv_rn(v, bc2);
    const double upd = __ddiv_rn(__dmul_rn(lr, mh), __dadd_rn(__dsqrt_rn(vh), a.eps));
    const double p = __dsub_rn(a.params[i], upd);
    a.params[i] = p;
    if (a.kparams) {
      T* kp = static_cast<T*>(a.kparams);
      kp[map[i]] = T(p);
      if (mapT[MAPT * i] >= 0) kp[mapT[MAPT * i]] = T(p);
      // entries 1, 2: the wide path's TF32 slabs (plain copies) or the W=64
      // split-TF32 hi slabs (entries 3, 4 -- their lo parts -- are set then)
      const bool split = mapT[MAPT * i + 3] >= 0;
#pragma unroll
      for (int r = 1; r < 3; ++r)
        if (mapT[MAPT * i + r] >= 0) kp[mapT[MAPT * i + r]] = split ? tf32_hi(T(p)) : T(p);
#pragma unroll
      for (int r = 3; r < MAPT; ++r)
        if (mapT[MAPT * i + r] >= 0) kp[mapT[MAPT * i + r]] = tf32_lo(T(p));
    }
  }
  // ---- the last block advances the step counter ----
  if (!skip) {
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      const int done = atomicAdd(a.sync_counter, 1);
      if (done == int(gridDim.x) - 1) {
        *a.step = step0 + 1;
        *a.sync_counter = 0;
        __threadfence();
      }
    }
  }
}

extern "C" int fr_adam_step(const fr_plan* p, const fr_adam_args* args, fr_stream_t stream) {
  if (!args || !args->params || !args->grad || !args->m || !args->v || !args->step || !args->sched ||
      !args->flags || !args->sync_counter)
    return fail("fr_adam_step: NULL argument");
  if (args->n < 1 || args->n > (1LL << 30)) return fail("fr_adam_step: bad parameter count %lld", args->n);
  if (args->kparams && !p) return fail("fr_adam_step: refreshing kernel params needs the plan");
  if (p && args->n != p->info.n_params)
    return fail("fr_adam_step: n=%lld does not match the plan's %d parameters", args->n, p->info.n_params);
  if (args->lpart && !(args->n_colloc > 0)) return fail("fr_adam_step: n_colloc must be positive");
  const int n = int(args->n);
  const int blocks = (n + ADAM_NT - 1) / ADAM_NT;
  const int* map = p ? p->d_map : nullptr;
  const int* mapT = p ? p->d_mapT : nullptr;
  if (!p || p->info.dtype == FR_F32)
    adam_kernel<float><<<blocks, ADAM_NT, 0, stream>>>(*args, n, map, mapT);
  else
    adam_kernel<double><<<blocks, ADAM_NT, 0, stream>>>(*args, n, map, mapT);
  ++g_kernel_launches;
  FR_CUDA(cudaGetLastError(), "fr_adam_step");
  return 0;
}

// ---------------------------------------------------------------------------
template <typename T>
__global__ void pack_ghost_kernel(const T* __restrict__ y, const T* __restrict__ ya, long long n, int nout,
                                  int nvel, T* out_u, T* out_p) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    for (int c = 0; c < nvel; ++c) out_u[i * nvel + c] = y[i * nout + c];
    const T pv = y[i * nout + nvel];
    out_p[i] = ya ? pv - ya[i * nout + nvel] : pv;
  }
}

extern "C" int fr_pack_ghost(const fr_plan* p, const void* y, const void* y_anchor, long long n, void* out_u,
                             void* out_p, fr_stream_t stream) {
  if (!p || (n > 0 && (!y || !out_u || !out_p))) return fail("fr_pack_ghost: NULL argument");
  if (n <= 0) return 0;
  const int blocks = int((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024);
  if (p->info.dtype == FR_F32)
    pack_ghost_kernel<float><<<blocks, 256, 0, stream>>>(static_cast<const float*>(y), static_cast<const float*>(y_anchor), n,
                                                         p->info.n_out, p->info.n_vel, static_cast<float*>(out_u),
                                                         static_cast<float*>(out_p));
  else
    pack_ghost_kernel<double><<<blocks, 256, 0, stream>>>(static_cast<const double*>(y), static_cast<const double*>(y_anchor),
                                                          n, p->info.n_out, p->info.n_vel, static_cast<double*>(out_u),
                                                          static_cast<double*>(out_p));
  ++g_kernel_launches;
  FR_CUDA(cudaGetLastError(), "fr_pack_ghost");
  return 0;
}

// ---------------------------------------------------------------------------
// Peer-memory ghost transport (see flowrec_b200.h).  One CTA per edge: thread 0
// waits until the destination has finished the epoch that last read these
// target rows, the block stores the rows straight into the destination's
// memory (NVLink peer stores when it is another GPU), then thread 0 publishes
// them with a system-scope release add on the destination's ready counter.
// ---------------------------------------------------------------------------
struct GhostEdges {
  fr_ghost_edge e[FR_MAX_GHOST_EDGES];
};

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <typename T>
__global__ void __launch_bounds__(256) ghost_put_kernel(const T* __restrict__ y, const T* __restrict__ yj,
                                                        GhostEdges E, int nout, int nvel, int nin,
                                                        const unsigned* my_epochs, unsigned long long timeout_ns,
                                                        int* flags) {
  const fr_ghost_edge& e = E.e[blockIdx.x];
  __shared__ int ok;
  if (threadIdx.x == 0) {
    const unsigned need = *my_epochs;
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    int good = 1;
    while (int(ld_acquire_sys(e.epochs) - need) < 0) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        if (flags) atomicOr(flags, FR_FLAG_EXCHANGE_TIMEOUT);
        good = 0;
        break;
      }
      __nanosleep(500);
    }
    ok = good;
  }
  __syncthreads();
  if (!ok) return;  // the destination never freed its rows: leave them, the host raises DeadlockError
  T* u = static_cast<T*>(e.u);
  T* p = static_cast<T*>(e.p);
  T* du = static_cast<T*>(e.du);
  const T* yr = y + e.y_row * nout;
  const T* ya = e.anchor_row >= 0 ? y + e.anchor_row * nout : nullptr;
  for (long long i = threadIdx.x; i < e.n; i += blockDim.x) {
    for (int c = 0; c < nvel; ++c) u[i * nvel + c] = yr[i * nout + c];
    const T pv = yr[i * nout + nvel];
    p[i] = ya ? pv - ya[i * nout + nvel] : pv;
  }
  if (du && yj) {
    // jet rows (1 + 2 nin) x nout per point: first-derivative blocks 1..nin
    const int S = 1 + 2 * nin;
    const T* jr = yj + e.y_row * S * nout;
    const long long tot = e.n * nin * nvel;
    for (long long q = threadIdx.x; q < tot; q += blockDim.x) {
      const long long i = q / (nin * nvel);
      const int j = int(q / nvel % nin), c = int(q % nvel);
      du[q] = jr[(i * S + 1 + j) * nout + c];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(e.ready) : "memory");
  }
}

__global__ void counter_add_kernel(unsigned* word, unsigned v) {
  __threadfence_system();
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(word), "r"(v) : "memory");
}

extern "C" int fr_ipc_alloc(size_t bytes, void** ptr, void* handle_out) {
  if (!ptr || !handle_out || bytes == 0) return fail("fr_ipc_alloc: bad arguments");
  *ptr = nullptr;
  void* d = nullptr;
  FR_CUDA(cudaMalloc(&d, bytes), "fr_ipc_alloc");
  cudaError_t e = cudaMemset(d, 0, bytes);
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, d);
  if (e != cudaSuccess) {
    cudaFree(d);
    return cuda_fail(e, "fr_ipc_alloc");
  }
  static_assert(sizeof(h) == 64, "IPC handle size");
  std::memcpy(handle_out, &h, sizeof(h));
  *ptr = d;
  return 0;
}

extern "C" int fr_ipc_open(const void* handle, void** ptr) {
  if (!handle || !ptr) return fail("fr_ipc_open: NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  FR_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "fr_ipc_open");
  return 0;
}

extern "C" int fr_ipc_close(void* ptr) {
  if (!ptr) return 0;
  FR_CUDA(cudaIpcCloseMemHandle(ptr), "fr_ipc_close");
  return 0;
}

extern "C" int fr_ipc_free(void* ptr) {
  if (!ptr) return 0;
  FR_CUDA(cudaFree(ptr), "fr_ipc_free");
  return 0;
}

extern "C" int fr_ghost_put(const fr_plan* p, const void* y, const void* y_jet, int n_edges, const fr_ghost_edge* edges,
                            const unsigned* my_epochs, unsigned timeout_ms, int* flags, fr_stream_t stream) {
  if (!p || !edges || !my_epochs || n_edges < 0 || n_edges > FR_MAX_GHOST_EDGES)
    return fail("fr_ghost_put: bad arguments");
  if (n_edges == 0) return 0;
  if (!y) return fail("fr_ghost_put: NULL producer output");
  GhostEdges E{};
  for (int i = 0; i < n_edges; ++i) {
    const fr_ghost_edge& e = edges[i];
    if (e.n < 0 || (e.n > 0 && (!e.u || !e.p)) || !e.ready || !e.epochs || e.y_row < 0)
      return fail("fr_ghost_put: bad edge %d", i);
    if (e.du && !y_jet) return fail("fr_ghost_put: edge %d carries derivatives but y_jet is NULL", i);
    E.e[i] = e;
  }
  const fr_plan_info& I = p->info;
  const unsigned long long tns = (unsigned long long)(timeout_ms ? timeout_ms : 600000u) * 1000000ull;
  if (I.dtype == FR_F32)
    ghost_put_kernel<float><<<n_edges, 256, 0, stream>>>(static_cast<const float*>(y), static_cast<const float*>(y_jet),
                                                          E, I.n_out, I.n_vel, I.n_in, my_epochs, tns, flags);
  else
    ghost_put_kernel<double><<<n_edges, 256, 0, stream>>>(static_cast<const double*>(y),
                                                           static_cast<const double*>(y_jet), E, I.n_out, I.n_vel,
                                                           I.n_in, my_epochs, tns, flags);
  ++g_kernel_launches;
  FR_CUDA(cudaGetLastError(), "fr_ghost_put");
  return 0;
}

extern "C" int fr_counter_add(unsigned* word, unsigned value, fr_stream_t stream) {
  if (!word) return fail("fr_counter_add: NULL word");
  counter_add_kernel<<<1, 1, 0, stream>>>(word, value);
  ++g_kernel_launches;
  FR_CUDA(cudaGetLastError(), "fr_counter_add");
  return 0;
}

// ---------------------------------------------------------------------------
// GPU-side dataset sampling, bit-exact with NumPy's Generator(PCG64).uniform
// (decomposition.py:64-70: one rng.uniform(lo, hi, size=n) per column, columns
// in layout order).  PCG64 = 128-bit LCG, XSL-RR 128/64 output of the stepped
// state; next_double = (x >> 11) * 2^-53; uniform = lo + (hi - lo) * u with
// round-to-nearest f64 ops (no contraction), as NumPy's random_uniform.  Draw d
// of the stream (d = skip + column * n + row) is reached by LCG jump-ahead, so
// every thread produces its own contiguous run of draws.
// ---------------------------------------------------------------------------
typedef unsigned __int128 u128;
struct UniformCols {
  double lo[8], range[8];
};

__device__ __forceinline__ u128 pcg_mult() {
  return (u128(0x2360ED051FC65DA4ull) << 64) | u128(0x4385DF649FCCF645ull);
}

__device__ __forceinline__ u128 pcg_advance(u128 state, u128 inc, unsigned long long delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta > 0) {
    if (delta & 1ull) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__device__ __forceinline__ unsigned long long pcg_output(u128 s) {
  const unsigned long long x = (unsigned long long)(s >> 64) ^ (unsigned long long)s;
  const unsigned rot = unsigned(s >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

__global__ void __launch_bounds__(256) pcg64_uniform_kernel(unsigned long long s_hi, unsigned long long s_lo,
                                                            unsigned long long i_hi, unsigned long long i_lo,
                                                            unsigned long long skip, long long n, int ncols,
                                                            UniformCols cols, long long per_thread, double* out64,
                                                            float* out32) {
  const long long total = n * ncols;
  const long long d0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * per_thread;
  if (d0 >= total) return;
  const u128 inc = (u128(i_hi) << 64) | u128(i_lo);
  // state before draw d0: advanced skip + d0 steps; each draw steps first
  u128 st = pcg_advance((u128(s_hi) << 64) | u128(s_lo), inc, skip + (unsigned long long)d0);
  const u128 mult = pcg_mult();
  const long long d1 = d0 + per_thread < total ? d0 + per_thread : total;
  for (long long d = d0; d < d1; ++d) {
    st = st * mult + inc;
    const double u = double(pcg_output(st) >> 11) * (1.0 / 9007199254740992.0);
    const int j = int(d / n);
    const long long i = d - (long long)j * n;
    const double v = __dadd_rn(cols.lo[j], __dmul_rn(cols.range[j], u));
    if (out64) out64[i * ncols + j] = v;
    if (out32) out32[i * ncols + j] = float(v);
  }
}

extern "C" int fr_pcg64_uniform(const unsigned long long* state4, unsigned long long skip, long long n, int n_cols,
                                const double* lo, const double* hi, double* out64, float* out32,
                                fr_stream_t stream) {
  if (!state4 || !lo || !hi || n < 0 || n_cols < 1 || n_cols > 8 || (!out64 && !out32))
    return fail("fr_pcg64_uniform: bad arguments");
  if (n == 0) return 0;
  UniformCols c{};
  for (int j = 0; j < n_cols; ++j) {
    c.lo[j] = lo[j];
    c.range[j] = hi[j] - lo[j];  // NumPy: _range = high - low (a Python float subtraction)
    if (!std::isfinite(c.range[j])) return fail("fr_pcg64_uniform: non-finite range in column %d", j);
  }
  const long long total = n * n_cols;
  const long long per_thread = 64;  // sequential steps per thread after one jump-ahead
  const long long threads = (total + per_thread - 1) / per_thread;
  const int blocks = int((threads + 255) / 256);
  pcg64_uniform_kernel<<<blocks, 256, 0, stream>>>(state4[0], state4[1], state4[2], state4[3], skip, n, n_cols, c,
                                                   per_thread, out64, out32);
  ++g_kernel_launches;
  FR_CUDA(cudaGetLastError(), "fr_pcg64_uniform");
  return 0;
}

// ---------------------------------------------------------------------------
// Reference seam (_kernels): elementwise jet propagation on stacked f64 arrays
// ((1 + 2d) * batch, width).  Semantics of numpy_backend.py:43-89, including
// "written" (accumulate=0) versus "added" adjoints.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void factors(int kind, double s, double c, double* d1, double* d2, double* d3) {
  if (kind == FR_ACT_TANH) {
    *d1 = __dsub_rn(1.0, __dmul_rn(s, s));
    *d2 = __dmul_rn(__dmul_rn(s, *d1), -2.0);
    if (d3) *d3 = __dmul_rn(__dadd_rn(__dmul_rn(*d1, *d1), __dmul_rn(s, *d2)), -2.0);
  } else {
    *d1 = c;
    *d2 = -s;
    if (d3) *d3 = -c;
  }
}

__global__ void act_fwd_kernel(int kind, const double* z, double* s, const double* aux, double* d1o, double* d2o,
                               long long batch, int d, int width) {
  const long long total = batch * width;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const double sv = s[e];
    double d1, d2;
    factors(kind, sv, kind == FR_ACT_TANH ? 0.0 : aux[e], &d1, &d2, nullptr);
    d1o[e] = d1;
    d2o[e] = d2;
    for (int j = 0; j < d; ++j) {
      const long long gi = (1 + j) * total + e;
      const long long li = (1 + d + j) * total + e;
      const double zg = z[gi];
      s[gi] = __dmul_rn(d1, zg);
      s[li] = __dadd_rn(__dmul_rn(__dmul_rn(d2, zg), zg), __dmul_rn(d1, z[li]));
    }
  }
}

__global__ void act_bwd_kernel(int kind, const double* z, const double* s, const double* aux, const double* sbar,
                               double* zbar, long long batch, int d, int width, int accumulate) {
  const long long total = batch * width;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    double d1, d2, d3;
    factors(kind, s[e], kind == FR_ACT_TANH ? 0.0 : aux[e], &d1, &d2, &d3);
    double acc = __dmul_rn(sbar[e], d1);
    for (int j = 0; j < d; ++j) {
      const long long gi = (1 + j) * total + e;
      const long long li = (1 + d + j) * total + e;
      const double zg = z[gi], sg = sbar[gi], sl = sbar[li];
      const double t1 = __dmul_rn(sg, __dmul_rn(d2, zg));
      const double t2 = __dmul_rn(sl, __dadd_rn(__dmul_rn(__dmul_rn(d3, zg), zg), __dmul_rn(d2, z[li])));
      acc = __dadd_rn(acc, __dadd_rn(t1, t2));
      const double tg = __dadd_rn(__dmul_rn(sg, d1), __dmul_rn(__dmul_rn(__dmul_rn(2.0, d2), zg), sl));
      const double tl = __dmul_rn(sl, d1);
      zbar[gi] = accumulate ? __dadd_rn(zbar[gi], tg) : tg;
      zbar[li] = accumulate ? __dadd_rn(zbar[li], tl) : tl;
    }
    zbar[e] = accumulate ? __dadd_rn(zbar[e], acc) : acc;
  }
}

extern "C" int fr_jet_act_forward(int kind, const double* z, double* s, const double* aux, double* d1, double* d2,
                                  long long batch, int n_inputs, int width, fr_stream_t stream) {
  if (kind != FR_ACT_TANH && kind != FR_ACT_SIN) return fail("unknown activation kind %d", kind);
  if (!z || !s || !d1 || !d2 || (kind == FR_ACT_SIN && !aux)) return fail("fr_jet_act_forward: NULL argument");
  if (batch < 0 || n_inputs < 0 || width < 1) return fail("fr_jet_act_forward: bad shape");
  const long long total = batch * width;
  if (total == 0) return 0;
  const int blocks = int((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
  act_fwd_kernel<<<blocks, 256, 0, stream>>>(kind, z, s, aux, d1, d2, batch, n_inputs, width);
  ++g_kernel_launches;
  FR_CUDA(cudaGetLastError(), "fr_jet_act_forward");
  return 0;
}

extern "C" int fr_jet_act_backward(int kind, const double* z, const double* s, const double* aux, const double* sbar,
                                   double* zbar, long long batch, int n_inputs, int width, int accumulate,
                                   fr_stream_t stream) {
  if (kind != FR_ACT_TANH && kind != FR_ACT_SIN) return fail("unknown activation kind %d", kind);
  if (!z || !s || !sbar || !zbar || (kind == FR_ACT_SIN && !aux)) return fail("fr_jet_act_backward: NULL argument");
  if (batch < 0 || n_inputs < 0 || width < 1) return fail("fr_jet_act_backward: bad shape");
  const long long total = batch * width;
  if (total == 0) return 0;
  const int blocks = int((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
  act_bwd_kernel<<<blocks, 256, 0, stream>>>(kind, z, s, aux, sbar, zbar, batch, n_inputs, width, accumulate);
  ++g_kernel_launches;
  FR_CUDA(cudaGetLastError(), "fr_jet_act_backward");
  return 0;
}

// ---------------------------------------------------------------------------
// FP32 FFMA probe: 16 independent accumulators per thread, 4 FMAs per operand
// load-free inner step; measures the SIMT FP32 roofline on this part.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) ffma_kernel(int iters, float* out) {
  float a[16];
  const float x = 1.0f + 1e-7f * threadIdx.x, y = 0.999999f;
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = float(i) * 1e-3f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 32; ++r)
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], y, x);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

extern "C" int fr_bench_ffma(int grid, int iters, int, float* out, fr_stream_t stream) {
  if (grid < 1 || iters < 1 || !out) return fail("fr_bench_ffma: bad arguments");
  ffma_kernel<<<grid, 256, 0, stream>>>(iters, out);
  ++g_kernel_launches;
  FR_CUDA(cudaGetLastError(), "fr_bench_ffma");
  return 0;
}

// ---------------------------------------------------------------------------
static int preload_capi_kernels() {
  cudaFuncAttributes fa;
  FR_CUDA(cudaFuncGetAttributes(&fa, signal_kernel), "preload fr_signal");
  FR_CUDA(cudaFuncGetAttributes(&fa, reduce_grad_kernel), "preload fr_reduce_grad");
  FR_CUDA(cudaFuncGetAttributes(&fa, reduce_loss_kernel), "preload fr_reduce_loss");
  FR_CUDA(cudaFuncGetAttributes(&fa, adam_kernel<float>), "preload fr_adam_step");
  FR_CUDA(cudaFuncGetAttributes(&fa, adam_kernel<double>), "preload fr_adam_step");
  FR_CUDA(cudaFuncGetAttributes(&fa, pack_ghost_kernel<float>), "preload fr_pack_ghost");
  FR_CUDA(cudaFuncGetAttributes(&fa, pack_ghost_kernel<double>), "preload fr_pack_ghost");
  FR_CUDA(cudaFuncGetAttributes(&fa, prepare_kernel<float>), "preload fr_prepare_params");
  FR_CUDA(cudaFuncGetAttributes(&fa, prepare_kernel<double>), "preload fr_prepare_params");
  FR_CUDA(cudaFuncGetAttributes(&fa, ghost_put_kernel<float>), "preload fr_ghost_put");
  FR_CUDA(cudaFuncGetAttributes(&fa, ghost_put_kernel<double>), "preload fr_ghost_put");
  FR_CUDA(cudaFuncGetAttributes(&fa, counter_add_kernel), "preload fr_counter_add");
  return 0;
}
