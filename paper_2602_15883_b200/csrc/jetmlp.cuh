// Fused jet-MLP kernels for sm_100a (FP32 SIMT product path, FP64 parity build).
//
// One persistent CTA per SM walks tiles of collocation / observation / ghost
// points.  For each tile it runs the whole per-point chain of the reference's
// PDE / MSE tapes (pkg/src/flowrec/autodiff/builders.py:24-141) without any
// HBM round trip of the activations:
//
//   forward   L x [stacked-jet affine -> jet activation]   (tape.py:22-124)
//             output affine                                (builders.py:35)
//   head      Navier-Stokes residual + square-sum          (physics.py:70-93,
//             or MSE against targets                        builders.py:51-141)
//   backward  reverse sweep of the same chain              (tape.py:335-371)
//
// The S jet streams of a point (value, d/dx_j, d2/dx_j^2) share every weight
// matrix, so one shared-memory weight fragment feeds S x 8 FMAs per thread.
// Activation jets never leave the SM except for a per-CTA L2-resident stash of
// the pre-activation derivative streams that the backward sweep re-reads.
//
// Layouts (all in shared memory):
//   activations / adjoints: k-quad layout A[(k>>2)*RS4 + row*4 + (k&3)] with
//       RS4 padded to 4 banks mod 32, row = point*S + stream (jet modes) or
//       row = point (value modes) -- every LDS.128 / STS.128 conflict-free;
//   weight slots: row-major [W][W] copies of W_l (forward) or W_l^T (dX),
//       double-buffered with cp.async.
// Gradient partials are accumulated per CTA in FP64 with red.add, each address
// of a CTA's row written by exactly one thread, and reduced across CTAs in a
// fixed order by fr_reduce_grad, so a rerun is bit-identical (the reference's
// determinism contract, tape.py:1-6).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fr {

// running count of kernels this library has enqueued (host side; the bench's
// gpu_launches claim is a difference of this counter around one epoch)
extern long long g_kernel_launches;

enum { ACT_TANH = 0, ACT_SIN = 1 };
enum { REG_STEADY2D = 0, REG_UNSTEADY2D = 1, REG_UNSTEADY3D = 2 };
enum { MODE_PDE = 0, MODE_MSE = 1, MODE_VALUE = 2, MODE_JET = 3, MODE_GJ = 4 };

// Input layout (t,)x,y[,z]; outputs velocity + p (physics.py:17-67).
template <int REG> struct Regime;
template <> struct Regime<REG_STEADY2D> {
  static constexpr int DIN = 2, NSP = 2, NVEL = 2, NOUT = 3, HAS_T = 0;
};
template <> struct Regime<REG_UNSTEADY2D> {
  static constexpr int DIN = 3, NSP = 2, NVEL = 2, NOUT = 3, HAS_T = 1;
};
template <> struct Regime<REG_UNSTEADY3D> {
  static constexpr int DIN = 4, NSP = 3, NVEL = 3, NOUT = 4, HAS_T = 1;
};

// Jet streams carried per point.  PDE mode drops the reference's d2/dt2 block
// (computed at builders.py:95 but never read by the residual, physics.py:89;
// its adjoint is identically zero).  JET mode (predict_jet) keeps every block.
// GJ mode (ghost-derivative matching, the opt-in C^1 interface extension)
// carries value + first derivatives only.
template <int MODE, int REG> struct Streams {
  using R = Regime<REG>;
  static constexpr bool JET = (MODE == MODE_PDE || MODE == MODE_JET || MODE == MODE_GJ);
  static constexpr int NG = JET ? R::DIN : 0;
  static constexpr int LAP0 = (MODE == MODE_PDE) ? R::HAS_T : 0;
  static constexpr int NL = (JET && MODE != MODE_GJ) ? (R::DIN - LAP0) : 0;
  static constexpr int S = 1 + NG + NL;
  // rows owned by one thread: all streams of one point (jet modes) so the
  // activation jet is register-local, or 6 independent points (value modes).
  static constexpr int RPT = JET ? S : 6;
};

constexpr int FLAG_EXCHANGE_TIMEOUT = 4;  // == FR_FLAG_EXCHANGE_TIMEOUT (flowrec_b200.h)

struct KArgs {
  const void* kp;       // kernel params (T), padded layout, see ParamLayout
  const void* pts;      // (n, DIN) T
  const void* tu;       // MSE: (n, NVEL) T ; GJ: (n, DIN, NVEL) T derivative targets
  const void* tp;       // MSE: (n,) T or null
  void* out;            // VALUE: (n, NOUT) T ; JET: (n, S, NOUT) T
  double* gpart;        // [gridDim.x][np_pad] gradient partials
  double* lpart;        // [gridDim.x][2] loss partials (sq, sq_p)
  void* scratch;        // [gridDim.x][stash_elems] T
  long long n;
  int L;                // hidden layers
  int np_pad;           // padded parameter count (gradient partial row length)
  int stash_elems;      // per-CTA stash size in elements of T
  double coef;          // PDE: lambda_pde/N ; MSE: velocity coefficient
  double pcoef;         // MSE: pressure coefficient (used iff has_p)
  double inv_re;        // PDE: 1/Re (physics.py:80)
  double velw[4];       // MSE: velocity component weights
  int has_p;            // MSE: pressure head present
  const unsigned* gate; // MSE: wait before the first tile (ghost overlap) until *gate != 0, or,
  const unsigned* gate_round;  // when non-null, until *gate >= *gate_round * gate_mult
  unsigned gate_mult;          //   (monotonic arrival counter of the peer-memory transport)
  int* flags;           // FLAG_EXCHANGE_TIMEOUT on a timed-out gate wait
  unsigned long long gate_timeout_ns;
  long long tc3;        // kp offset of the split-TF32 weight slabs (epoch kernel, FR_MATH_TF32X3), else 0
};

// Padded flat parameter layout used by the kernels (T precision):
//   W0 [DIN][W], b0 [W], {W_l [W][W], b_l [W]} l=1..L-1, W_L [W][NOUT], b_L [NOUT]
//   (same order as the reference's flat vector, network.py:72-115, with hidden
//   width padded to W), then 16-byte aligned transposes W_l^T, l=1..L-1.
struct ParamLayout {
  int din, w, nout, L;
  __host__ __device__ int off_w(int l) const {
    if (l == 0) return 0;
    return din * w + w + (l - 1) * (w * w + w);
  }
  __host__ __device__ int off_b(int l) const {
    if (l == 0) return din * w;
    if (l < L) return off_w(l) + w * w;
    return off_w(L) + w * nout;
  }
  __host__ __device__ int np_pad() const { return off_w(L) + w * nout + nout; }
  __host__ __device__ int off_wt(int l) const {  // l in 1..L-1
    int base = (np_pad() + 3) & ~3;
    return base + (l - 1) * w * w;
  }
  __host__ __device__ int total() const { return off_wt(L); }
};

}  // namespace fr
