// Kernel template bodies (included by the per-mode translation units).
#pragma once
#include "jetmlp.cuh"
#include "tcgen05.cuh"

namespace fr {

// optional per-phase cycle counters (instrumented builds only: -DFR_PHASE_TIMERS)
#ifdef FR_PHASE_TIMERS
__device__ unsigned long long g_phase_cycles[16];
#define FR_MARK(id)                         \
  do {                                      \
    if (threadIdx.x == 0) {                 \
      const long long t_ = clock64();       \
      ph_acc[id] += t_ - ph_last;           \
      ph_last = t_;                         \
    }                                       \
  } while (0)
#else
#define FR_MARK(id) \
  do {              \
  } while (0)
#endif

// ---------------------------------------------------------------------------
// scalar math (accurate libm versions: first-layer arguments reach |z|~17 on
// the cylinder box, so tanh.approx / __sinf are not acceptable)
// ---------------------------------------------------------------------------
__device__ __forceinline__ float tanh_t(float x) { return tanhf(x); }
__device__ __forceinline__ double tanh_t(double x) { return tanh(x); }
__device__ __forceinline__ void sincos_t(float x, float* s, float* c) { sincosf(x, s, c); }
__device__ __forceinline__ void sincos_t(double x, double* s, double* c) { sincos(x, s, c); }

// sigma and its derivative factors (numpy_backend.py:23-40)
template <int ACT, typename T>
__device__ __forceinline__ void act_eval(T z, T& s, T& c) {
  if constexpr (ACT == ACT_TANH) {
    s = tanh_t(z);
    c = T(0);
  } else {
    sincos_t(z, &s, &c);
  }
}
template <int ACT, typename T>
__device__ __forceinline__ void act_d12(T s, T c, T& d1, T& d2) {
  if constexpr (ACT == ACT_TANH) {
    d1 = T(1) - s * s;
    d2 = (s * d1) * T(-2);
  } else {
    d1 = c;
    d2 = -s;
  }
}
template <int ACT, typename T>
__device__ __forceinline__ T act_d3(T s, T c, T d1, T d2) {
  if constexpr (ACT == ACT_TANH) {
    return (d1 * d1 + s * d2) * T(-2);
  } else {
    return -c;
  }
}

// ---------------------------------------------------------------------------
// vectorised shared-memory block copies
// ---------------------------------------------------------------------------
template <typename T, int N>
struct VecW {
  static constexpr int V =
      sizeof(T) == 4 ? ((N % 4 == 0) ? 4 : ((N % 2 == 0) ? 2 : 1)) : ((N % 2 == 0) ? 2 : 1);
};

template <typename T, int N>
__device__ __forceinline__ void vload(T (&dst)[N], const T* src) {
  constexpr int V = VecW<T, N>::V;
#pragma unroll
  for (int i = 0; i < N; i += V) {
    if constexpr (sizeof(T) == 4 && V == 4) {
      float4 v = *reinterpret_cast<const float4*>(src + i);
      dst[i] = v.x; dst[i + 1] = v.y; dst[i + 2] = v.z; dst[i + 3] = v.w;
    } else if constexpr (sizeof(T) == 4 && V == 2) {
      float2 v = *reinterpret_cast<const float2*>(src + i);
      dst[i] = v.x; dst[i + 1] = v.y;
    } else if constexpr (sizeof(T) == 8 && V == 2) {
      double2 v = *reinterpret_cast<const double2*>(src + i);
      dst[i] = v.x; dst[i + 1] = v.y;
    } else {
      dst[i] = src[i];
    }
  }
}

template <typename T, int N>
__device__ __forceinline__ void vstore(T* dst, const T (&src)[N]) {
  constexpr int V = VecW<T, N>::V;
#pragma unroll
  for (int i = 0; i < N; i += V) {
    if constexpr (sizeof(T) == 4 && V == 4) {
      *reinterpret_cast<float4*>(dst + i) = make_float4(src[i], src[i + 1], src[i + 2], src[i + 3]);
    } else if constexpr (sizeof(T) == 4 && V == 2) {
      *reinterpret_cast<float2*>(dst + i) = make_float2(src[i], src[i + 1]);
    } else if constexpr (sizeof(T) == 8 && V == 2) {
      *reinterpret_cast<double2*>(dst + i) = make_double2(src[i], src[i + 1]);
    } else {
      dst[i] = src[i];
    }
  }
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// ---------------------------------------------------------------------------
// compile-time configuration
// ---------------------------------------------------------------------------
#ifndef FR_VALUE_RPT
#define FR_VALUE_RPT 2  // ghost producer at P = 8 (~6k points): 33 -> 20 us (1: 18 us; 6: the MSE heads)
#endif
template <typename T, int ACT, int MODE, int REG, int W, int NT_ = 0>
struct JetCfg {
  using R = Regime<REG>;
  using St = Streams<MODE, REG>;
  static constexpr int DIN = R::DIN, NOUT = R::NOUT, NVEL = R::NVEL, HAS_T = R::HAS_T;
  static constexpr int S = St::S, NG = St::NG, NL = St::NL, LAP0 = St::LAP0;
  // value-only rows per thread: 6 for the MSE heads; VALUE (the per-epoch ghost
  // producer on a few thousand points) FR_VALUE_RPT, smaller tiles over more SMs
  static constexpr int RPT = MODE == MODE_VALUE ? FR_VALUE_RPT : St::RPT;
  static constexpr bool JET = St::JET;
  static constexpr bool BWD = (MODE == MODE_PDE || MODE == MODE_MSE || MODE == MODE_GJ);
  // 12 warps per SM where the FP32 tile buffers still fit (W = 64, <= 6 streams);
  // otherwise 8 (FP32) or 4 (FP64 parity build)
  static constexpr int NT_DEFAULT = sizeof(T) == 4 ? ((W == 64 && St::RPT <= 6) ? 384 : 256) : 128;
  static constexpr int NT = NT_ ? NT_ : NT_DEFAULT;
  static constexpr int G = W / 8;          // unit groups of 8 per row group
  static constexpr int NRG = NT / G;       // row groups
  static constexpr int ROWS = NRG * RPT;   // rows per tile
  static constexpr int PPT = JET ? NRG : ROWS;  // points per tile
  static constexpr int PP = JET ? 1 : RPT;      // points per thread
  static constexpr int SIN = (ACT == ACT_SIN) ? 1 : 0;
  static constexpr int NST0 = 1 + SIN;                       // layer-0 stash / (point,unit)
  // hidden-layer stash per (point, unit), jet modes: sigma(z_v) [cos z_v for
  // sin] and the pre-activation derivative streams z_g[NG], z_l[NL] -- enough
  // to rebuild both the layer's S output streams (the next layer's dW input)
  // and its adjoint factors {d1, d2 z_g, d3 z_g^2 + d2 z_l} with the forward's
  // own expressions, at half the footprint of storing both (the stash then
  // stays L2-resident)
  static constexpr int NSTH = JET ? S + SIN : NST0;
  // k-quad layout: element (row, k) at (k>>2)*RS4 + row*4 + (k&3).  RS4 is
  // padded so that consecutive quads start 4 banks apart: the 8 lanes of a
  // quarter-warp touching 8 consecutive quads then cover all 32 banks.
  static constexpr int RS4_BASE = 4 * ROWS;
  static constexpr int RS4 = sizeof(T) == 4 ? RS4_BASE + ((4 - RS4_BASE % 32) + 32) % 32
                                            : RS4_BASE + ((2 - RS4_BASE % 16) + 16) % 16;
  static constexpr int XELEMS = (W / 4) * RS4;
  // dW phase: (W/8)^2 thread tiles of 8k x 8u, RSPLIT row ranges combined in
  // the (then free) activation buffer
  static constexpr int KT = W / 8;
  // largest split with one thread per (tile, range), rows divisible, and the
  // R-1 partials of the flat combine fitting in the activation buffer
  static constexpr int rsplit_fit(int r) {
    return (r > 1 && (r * KT * KT > NT || r * W * W > XELEMS || ROWS % r != 0)) ? rsplit_fit(r - 1) : r;
  }
  static constexpr int RSPLIT = rsplit_fit(NT / (KT * KT) > 0 ? NT / (KT * KT) : 1);
  static_assert(W % 8 == 0, "width must be a multiple of 8");
  static_assert(NT % G == 0, "thread count must be divisible by unit groups");
  static_assert(ROWS % 2 == 0, "tile rows must be even");

  __host__ __device__ static int stash_per_thread(int L) { return 8 * PP * (NST0 + (L - 1) * NSTH); }
  __host__ __device__ static int stash_layer_base(int l) {
    return l == 0 ? 0 : 8 * PP * (NST0 + (l - 1) * NSTH);
  }
  // shared memory carve (elements of T), all blocks 16-byte aligned
  __host__ __device__ static constexpr int al(int n) { return (n + 3) & ~3; }
  // tc: the split-TF32 tensor-core epoch path (weight slots hold {hi, lo} slabs)
  __host__ __device__ static int smem_elems(int L, bool tc = false) {
    int e = 0;
    e += al(XELEMS);                       // Xs
    if (BWD) e += al(XELEMS);              // Gs
    e += (tc ? 4 : 2) * W * W;             // weight slots
    e += al(DIN * W);                      // W0s
    e += al(L * W);                        // hidden biases
    e += al(W * NOUT);                     // WLs
    e += 4;                                // bLs
    e += al(ROWS * NOUT);                  // Ys
    if (BWD) e += al(ROWS * NOUT);         // Ybs
    e += al(PPT * DIN);                    // Ps
    if (tc) e += 256;                      // 1 KB: the base is aligned up for the MN-major dW atoms
    // (MSE targets are read from global in the head; the db partials alias Ys,
    // which is dead once the head has run)
    return e;
  }
  static_assert(!BWD || ROWS * NOUT >= NT, "db partials alias Ys");
  // the per-thread loss partials of the final reduction alias Xs (free by then)
  static_assert(XELEMS * sizeof(T) >= 2 * NT * sizeof(double), "loss-reduction scratch must fit in Xs");
  __host__ __device__ static size_t smem_bytes(int L, bool tc = false) { return size_t(smem_elems(L, tc)) * sizeof(T); }
};

// Ghost-overlap gate (fr_epoch_gate): spin with back-off until the transport
// stream has published this rank's ghost targets; bounded, so a lost peer
// becomes a flagged error instead of a hung GPU.
// With `round` the gate is a monotonic arrival counter written by peers over
// NVLink (fr_ghost_put): wait until it reaches *round * mult (system scope).
static __device__ __noinline__ void gate_wait(const unsigned* gate, const unsigned* round, unsigned mult, int* flags,
                                              unsigned long long timeout_ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  const unsigned target = round ? *round * mult : 1u;
  for (;;) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(gate) : "memory");
    if (int(v - target) >= 0) return;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      if (flags) atomicOr(flags, FLAG_EXCHANGE_TIMEOUT);
      return;
    }
    __nanosleep(1000);
  }
}

// element (row, k) of a k-quad buffer
template <int RS4>
__device__ __forceinline__ int kqi(int row, int k) {
  return (k >> 2) * RS4 + row * 4 + (k & 3);
}

// Units owned by unit-group g: {4g..4g+3} and {W/2+4g..W/2+4g+3}.  A
// quarter-warp (8 consecutive g) then reads one contiguous 128-byte row
// segment of a weight matrix per LDS.128 -- conflict-free.
template <int W>
__device__ __forceinline__ int unit_of(int g, int j) {
  return (j < 4) ? 4 * g + j : W / 2 + 4 * g + (j - 4);
}

// fire-and-forget f64 add into a gradient partial.  Every address of a CTA's
// partial row has exactly one writer thread per phase, and same-thread
// operations to one location stay in program order, so the result is the
// same fixed-order sum on every run.
__device__ __forceinline__ void red_add(double* p, double v) { atomicAdd(p, v); }

// FP32 inner-loop unroll factors (tuned on B200; overridable for sweeps)
#ifndef FR_EPOCH_2CTA
#define FR_EPOCH_2CTA 0  // two 192-thread CTAs per SM: measured slower (5.89 vs 5.40 ms), kept as a tuning switch
#endif
#ifndef FR_TC_DW
// tensor-core weight gradient (tc3_dw): MN-major BASE32B operands staged from
// the k-quad buffers through the idle 32 KB weight slot.  Correct (grad ~1e-6),
// but with one 32-row chunk buffer the staging copies, the per-chunk MMA
// round trip and the TMEM drain cost as much as the SIMT FFMA2 dW they replace
// (phase timers: 5.7k + 5.1k + 3.4k vs 13.7k cycles per tile-layer; 16-row
// double-buffered chunks are slower still), so off.  DESIGN.md 4.
#define FR_TC_DW 0
#endif
#ifndef FR_DW_SPLIT6
#define FR_DW_SPLIT6 0  // TC epoch: SIMT dW over 6 row ranges (all 12 warps): measured 1.5% slower, off
#endif
#ifndef FR_TC_DX_EARLY
#define FR_TC_DX_EARLY 1  // issue the dX hi passes before the SIMT dW (they then share shared-memory bandwidth)
#endif
#ifndef FR_GEMM_UNROLL
#define FR_GEMM_UNROLL 8
#endif
#ifndef FR_DW_UNROLL
#define FR_DW_UNROLL 4
#endif

#ifndef FR_DW_UNROLL_TC
#define FR_DW_UNROLL_TC 2  // split-TF32 kernel: 4.28 -> 4.16 ms at config C (unroll 1: 4.34, 3: 4.31, 4: 4.28, 8: 4.20)
#endif
constexpr int kGemmUnroll = FR_GEMM_UNROLL;
constexpr int kDwUnroll = FR_DW_UNROLL;
constexpr int kDwUnrollTC = FR_DW_UNROLL_TC;

// ---------------------------------------------------------------------------
// packed FP32 pairs (sm_100a FFMA2: fma.rn.f32x2, one issue slot for two FMAs).
// Each lane is an ordinary fma.rn.f32, so results are bit-identical to FFMA;
// the point is halving the issue slots the FP32 contractions take, which frees
// the dispatcher for the LDS / address / epilogue instructions in between.
// ---------------------------------------------------------------------------
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 f2_pack(float a, float b) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_unpack(f32x2 v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
// d.{x,y} = fma(a, b.{x,y}, d.{x,y})  (scalar a broadcast: FFMA2 R, Ra.F32, Rb.F32x2, Rd.F32x2)
__device__ __forceinline__ void f2_fma(f32x2& d, float a, f32x2 b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(f2_pack(a, a)), "l"(b));
}
// two pairs from 16 aligned bytes of shared memory
__device__ __forceinline__ void f2_lds(f32x2& p0, f32x2& p1, const float* src) {
  const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(src);
  p0 = v.x;
  p1 = v.y;
}

// FP32 core of gemm_rows: unit pairs (0,1) (2,3) (4,5) (6,7) accumulate as
// FFMA2 with the row activation broadcast; the per-element fma chain (k
// ascending) is the same as the scalar path's.  acc2[r][q] = units
// unit_of(g, 2q), unit_of(g, 2q + 1) of row rg*RPT + r.
template <int W, int RPT, int RS4>
__device__ __forceinline__ void gemm_rows_f2(const float* __restrict__ A, const float* __restrict__ B, int rg, int g,
                                             f32x2 (&acc2)[RPT][4]) {
#pragma unroll
  for (int r = 0; r < RPT; ++r)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc2[r][q] = 0ull;
  const float* ap = A + rg * (4 * RPT);
  const float* bp = B + 4 * g;
#pragma unroll kGemmUnroll
  for (int kq = 0; kq < W / 4; ++kq) {
    float av[4 * RPT];
    vload(av, ap + kq * RS4);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      f32x2 b[4];
      f2_lds(b[0], b[1], bp + (4 * kq + kk) * W);
      f2_lds(b[2], b[3], bp + (4 * kq + kk) * W + W / 2);
#pragma unroll
      for (int r = 0; r < RPT; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) f2_fma(acc2[r][q], av[4 * r + kk], b[q]);
    }
  }
}

// store_block for packed pairs: row r's units {4g..4g+3} are (acc2[r][0], acc2[r][1])
// and {W/2+4g..} are (acc2[r][2], acc2[r][3]) -- 16 contiguous bytes each, so
// the pairs go to shared memory as they are (no unpacking moves)
template <int W, int RPT, int RS4>
__device__ __forceinline__ void store_block_f2(float* __restrict__ buf, int rg, int g, const f32x2 (&acc2)[RPT][4]) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float* dst = buf + (g + h * (W / 8)) * RS4 + rg * (4 * RPT);
#pragma unroll
    for (int r = 0; r < RPT; ++r)
      *reinterpret_cast<ulonglong2*>(dst + 4 * r) = make_ulonglong2(acc2[r][2 * h], acc2[r][2 * h + 1]);
  }
}

template <typename T, int W, int RPT, int RS4>
__device__ __forceinline__ void gemm_rows_scalar(const T* __restrict__ A, const T* __restrict__ B, int rg, int g,
                                                 T (&acc)[RPT][8]);

// acc[r][j] = sum_k A(rg*RPT + r, k) * B[k][unit_of(g, j)]
template <typename T, int W, int RPT, int RS4>
__device__ __forceinline__ void gemm_rows(const T* __restrict__ A, const T* __restrict__ B, int rg, int g,
                                          T (&acc)[RPT][8]) {
  if constexpr (sizeof(T) == 4) {
    f32x2 acc2[RPT][4];
    gemm_rows_f2<W, RPT, RS4>(reinterpret_cast<const float*>(A), reinterpret_cast<const float*>(B), rg, g, acc2);
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float x, y;
        f2_unpack(acc2[r][q], x, y);
        acc[r][2 * q] = T(x);
        acc[r][2 * q + 1] = T(y);
      }
  } else {
    gemm_rows_scalar<T, W, RPT, RS4>(A, B, rg, g, acc);
  }
}

// FP64 (parity build): plain FMA chain, k ascending
template <typename T, int W, int RPT, int RS4>
__device__ __forceinline__ void gemm_rows_scalar(const T* __restrict__ A, const T* __restrict__ B, int rg, int g,
                                                 T (&acc)[RPT][8]) {
#pragma unroll
  for (int r = 0; r < RPT; ++r)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[r][j] = T(0);
  const T* ap = A + rg * (4 * RPT);
  const T* bp = B + 4 * g;
#pragma unroll 8
  for (int kq = 0; kq < W / 4; ++kq) {
    T av[4 * RPT];
    vload(av, ap + kq * RS4);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      T b0[4], b1[4];
      vload(b0, bp + (4 * kq + kk) * W);
      vload(b1, bp + (4 * kq + kk) * W + W / 2);
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[r][j] = fma(av[4 * r + kk], b0[j], acc[r][j]);
          acc[r][4 + j] = fma(av[4 * r + kk], b1[j], acc[r][4 + j]);
        }
      }
    }
  }
}

// store a thread's [RPT][8] block (rows rg*RPT.., units unit_of(g, .)) into a k-quad buffer
template <typename T, int W, int RPT, int RS4>
__device__ __forceinline__ void store_block(T* __restrict__ buf, int rg, int g, const T (&v)[RPT][8]) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    T tmp[4 * RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) tmp[4 * r + c] = v[r][4 * h + c];
    vstore(buf + (g + h * (W / 8)) * RS4 + rg * (4 * RPT), tmp);
  }
}

template <typename T, int W, int RPT, int RS4>
__device__ __forceinline__ void load_block(T (&v)[RPT][8], const T* __restrict__ buf, int rg, int g) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    T tmp[4 * RPT];
    vload(tmp, buf + (g + h * (W / 8)) * RS4 + rg * (4 * RPT));
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) v[r][4 * h + c] = tmp[4 * r + c];
  }
}

// ---------------------------------------------------------------------------
// per-CTA activation stash (L2-resident).  Element q of thread t of a layer
// region lives at quad (q >> 2): [(q >> 2) * 4 * NT + 4 * t + (q & 3)], so a
// thread's consecutive elements share 16-byte quads and runs of them move as
// STG.128 / STG.64 (LDG likewise) while each warp access stays coalesced.
// `lb` below is the layer base already offset by 4 * t.
// ---------------------------------------------------------------------------
template <int NT, typename T>
__device__ __forceinline__ T& sq(T* lb, int q) {
  return lb[(q >> 2) * (4 * NT) + (q & 3)];
}
template <typename T>
__device__ __forceinline__ void vst2(T* p, T a, T b) {
  if constexpr (sizeof(T) == 4) *reinterpret_cast<float2*>(p) = make_float2(a, b);
  else *reinterpret_cast<double2*>(p) = make_double2(a, b);
}
template <typename T>
__device__ __forceinline__ void vld2(const T* p, T& a, T& b) {
  if constexpr (sizeof(T) == 4) { const float2 v = *reinterpret_cast<const float2*>(p); a = v.x; b = v.y; }
  else { const double2 v = *reinterpret_cast<const double2*>(p); a = v.x; b = v.y; }
}
// v[0..N) -> elements q0..q0+N-1 (q0 is a compile-time constant after unrolling,
// so every branch below folds)
template <int NT, int N, typename T>
__device__ __forceinline__ void st_run(T* lb, int q0, const T (&v)[N]) {
#pragma unroll
  for (int i = 0; i + 1 < N; i += 2) {
    const int q = q0 + i;
    T* p = &sq<NT>(lb, q);
    if ((q & 3) == 0 && i + 4 <= N) {
      if constexpr (sizeof(T) == 4) *reinterpret_cast<float4*>(p) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      else { vst2(p, v[i], v[i + 1]); vst2(p + 2, v[i + 2], v[i + 3]); }
    } else if ((q & 3) == 2 && i >= 2 && i + 2 <= N) {
      // second half of the quad stored at i - 2
    } else if ((q & 1) == 0) {
      vst2(p, v[i], v[i + 1]);
    } else {
      *p = v[i];
      sq<NT>(lb, q + 1) = v[i + 1];
    }
  }
  if constexpr (N & 1) sq<NT>(lb, q0 + N - 1) = v[N - 1];
}
template <int NT, int N, typename T>
__device__ __forceinline__ void ld_run(T (&v)[N], const T* lb, int q0) {
#pragma unroll
  for (int i = 0; i + 1 < N; i += 2) {
    const int q = q0 + i;
    const T* p = &sq<NT>(const_cast<T*>(lb), q);
    if ((q & 3) == 0 && i + 4 <= N) {
      if constexpr (sizeof(T) == 4) {
        const float4 x = *reinterpret_cast<const float4*>(p);
        v[i] = x.x; v[i + 1] = x.y; v[i + 2] = x.z; v[i + 3] = x.w;
      } else {
        vld2(p, v[i], v[i + 1]);
        vld2(p + 2, v[i + 2], v[i + 3]);
      }
    } else if ((q & 3) == 2 && i >= 2 && i + 2 <= N) {
    } else if ((q & 1) == 0) {
      vld2(p, v[i], v[i + 1]);
    } else {
      v[i] = *p;
      v[i + 1] = sq<NT>(const_cast<T*>(lb), q + 1);
    }
  }
  if constexpr (N & 1) v[N - 1] = sq<NT>(const_cast<T*>(lb), q0 + N - 1);
}

// ---------------------------------------------------------------------------
// Split-TF32 hidden-layer contractions on the 5th-generation tensor core
// (FR_MATH_TF32X3, FP32 W = 64 epoch kernel).  out[row][n] = sum_k A[row][k] B[k][n]
// over the tile's ROWS rows.  A lives in the k-quad shared layout, which IS
// the K-major SWIZZLE_NONE UMMA layout (SBO = 128 B, LBO = RS4 * 4 B); B is a
// pre-tiled [k/4][128][4] slab whose n < 64 half holds hi = rna_tf32(W) and
// whose n >= 64 half holds lo = rna_tf32(W - hi) (LBO = 2 KB).  The tensor
// core reads FP32 operands as TF32 (truncated), so with
// A_lo = rna_tf32(A - trunc(A)) held in a second buffer
//     A B ~= trunc(A) [B_hi | B_lo]  (one N = 128 MMA: both terms at once)
//           + A_lo B_hi               (N = 64, into the B_lo half),
// FP32-level accuracy (the dropped A_lo B_lo and the roundings of the lo
// parts are <= ~2^-21 relative and unbiased).  M = 128-row blocks
// (ceil(ROWS / 128); the last reads past the tile, those D rows are never
// read), K = 8 per instruction, accumulators in TMEM columns
// [128 b, 128 b + 128): the big term in the first 64, the corrections in the
// other 64, summed in FP32 when D is drained.  One thread issues; one commit
// tracks every MMA it issued; one warp per (block, TMEM lane quadrant) drains.
// ---------------------------------------------------------------------------
struct TcState {
  uint32_t tmem;      // TMEM base (512 columns)
  uint64_t* mbar;     // MMA-completion barrier
  uint32_t phase;     // parity of the next completion
  uint64_t* mbar_dw;  // weight-gradient chunk barriers [2] (one per staging buffer)
  uint32_t dw_phase;  // their next-completion parities (bit b = buffer b)
};

// bounded mbarrier wait: a lost completion traps (kernel error) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* mbar, uint32_t parity) {
  const uint32_t a = tc::smem_u32(mbar);
  uint32_t done = 0;
  unsigned long long t0 = 0;
  for (int spin = 0; !done; ++spin) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (!done && (spin & 1023) == 1023) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (t0 == 0) t0 = now;
      else if (now - t0 > 2000000000ull) __trap();
    }
  }
}

__device__ __forceinline__ void tc_wait(TcState& t) {
  const uint32_t a = tc::smem_u32(t.mbar);
  uint32_t done = 0;
  unsigned long long t0 = 0;
  for (int spin = 0; !done; ++spin) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(done)
        : "r"(a), "r"(t.phase)
        : "memory");
    if (!done && (spin & 1023) == 1023) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (t0 == 0) t0 = now;
      else if (now - t0 > 2000000000ull) __trap();
    }
  }
  t.phase ^= 1u;
}

#ifdef FR_PHASE_TIMERS
// tc3 sub-phase cycles (thread 0): [10] A_lo transform, [11] MMA wait, [12] drain
__device__ unsigned long long g_tc_cycles[16];
#define FR_TC_MARK(id)                                               \
  do {                                                               \
    if (threadIdx.x == 0) {                                          \
      const long long t_ = clock64();                                \
      atomicAdd(&g_tc_cycles[id], (unsigned long long)(t_ - tc_last)); \
      tc_last = t_;                                                  \
    }                                                                \
  } while (0)
#define FR_TC_START long long tc_last = clock64()
#else
#define FR_TC_MARK(id) \
  do {                 \
  } while (0)
#define FR_TC_START \
  do {              \
  } while (0)
#endif

__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
__device__ __forceinline__ float tf32_rna(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
// the A-side low part: what the tensor core's truncating read of A misses, rounded to TF32
__device__ __forceinline__ float tf32_alo(float x) { return tf32_rna(x - tf32_trunc(x)); }

// The issue loops are the critical path of a 64-wide contraction (48 MMAs of
// 32..64 tensor cycles each), so descriptors are built once and advanced by
// adding the byte offset >> 4 to the start-address field (addresses stay
// below 256 KB: no carry out of the 14-bit field), and the accumulate flag is
// a literal.
__device__ __forceinline__ void mma_tf32_lit(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             bool accumulate) {
  if (accumulate)
    asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n" ::"r"(tmem_d), "l"(adesc), "l"(bdesc),
                 "r"(idesc));
  else
    asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 0;\n" ::"r"(tmem_d), "l"(adesc), "l"(bdesc),
                 "r"(idesc));
}

// trunc(A) [B_hi | B_lo] for every M block (no commit), issued by thread `issuer`
template <int ROWS, int RS4>
__device__ __forceinline__ void tc3_issue_hi(const float* A, const float* Bslab, const TcState& t, int issuer = 0) {
  constexpr int NB = (ROWS + 127) / 128;
  static_assert(NB * 128 <= 512, "accumulators fit the 512 TMEM columns");
  if (threadIdx.x == issuer) {
    const uint32_t id = tc::idesc_tf32(128, 128);
    const uint64_t a0 = tc::desc(A, RS4 * 4, 128), b0 = tc::desc(Bslab, 2048, 128);
    tc::fence_after();
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
        mma_tf32_lit(t.tmem + 128 * b, a0 + uint64_t(((512 * b + 2 * RS4 * ks) * 4) >> 4),
                     b0 + uint64_t((1024 * ks * 4) >> 4), id, ks != 0);
  }
}

// A_lo B_hi into the correction half, then one commit for everything the
// issuer issued (it must be the thread that issued the hi passes)
template <int ROWS, int RS4>
__device__ __forceinline__ void tc3_issue_lo(const float* Alo, const float* Bslab, const TcState& t, int issuer = 0) {
  constexpr int NB = (ROWS + 127) / 128;
  if (threadIdx.x == issuer) {
    const uint32_t id = tc::idesc_tf32(128, 64);
    const uint64_t a0 = tc::desc(Alo, RS4 * 4, 128), b0 = tc::desc(Bslab, 2048, 128);
    tc::fence_after();
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
        mma_tf32_lit(t.tmem + 128 * b + 64, a0 + uint64_t(((512 * b + 2 * RS4 * ks) * 4) >> 4),
                     b0 + uint64_t((1024 * ks * 4) >> 4), id, true);
    tc::mma_commit(t.mbar);
  }
}

// wait for the commit, then out[row][n] = D[row][n] + D[row][64 + n] (k-quad layout)
template <int ROWS, int RS4, int NT>
__device__ __forceinline__ void tc3_drain(float* out, TcState& t) {
  constexpr int NB = (ROWS + 127) / 128;
  FR_TC_START;
  tc_wait(t);
  tc::fence_after();
  FR_TC_MARK(11);
  // warp w takes (M block, lane quadrant) pairs wq = w, w + NT/32, ...; a warp
  // may only read TMEM lane quadrant w % 4, so wq % 4 == w % 4 always
  static_assert((NT / 32) % 4 == 0, "drain warps come in TMEM lane-quadrant groups of four");
  for (int wq = threadIdx.x >> 5; wq < 4 * NB; wq += NT / 32) {
    const int q = wq & 3, b = wq >> 2;
    const int row = 128 * b + 32 * q + (threadIdx.x & 31);
    const uint32_t ta = t.tmem + (uint32_t(32 * q) << 16) + uint32_t(128 * b);
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 32) {
      // both halves' loads in flight before one wait
      uint32_t v[32], w[32];
      tc::tmem_ld32_nowait(ta + c0, v);
      tc::tmem_ld32_nowait(ta + 64 + c0, w);
      tc::tmem_wait();
      if (row < ROWS) {
#pragma unroll
        for (int cc = 0; cc < 8; ++cc)
          *reinterpret_cast<float4*>(out + ((c0 >> 2) + cc) * RS4 + 4 * row) =
              make_float4(__uint_as_float(v[4 * cc]) + __uint_as_float(w[4 * cc]),
                          __uint_as_float(v[4 * cc + 1]) + __uint_as_float(w[4 * cc + 1]),
                          __uint_as_float(v[4 * cc + 2]) + __uint_as_float(w[4 * cc + 2]),
                          __uint_as_float(v[4 * cc + 3]) + __uint_as_float(w[4 * cc + 3]));
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  FR_TC_MARK(12);
}

// Weight gradient of one hidden layer on the tensor core:
//     dW[i][o] = sum_rows H[row][i] Zbar[row][o]
// with K = rows, both operands MN-major (units contiguous).  sm_100a reads
// MN-major TF32 only in the SWIZZLE_128B_BASE32B canonical layout (512-byte
// atoms of 4 K rows x 32 MN elements, 32-byte chunks XOR-swizzled by the row;
// LBO = MN-group stride, SBO = K-group stride -- tools/tc_mn_probe.py), and a
// k-quad 16-byte piece (one row, 4 units) stays contiguous in it, so staging a
// chunk of RC rows is one LDS.128 + two STS.128 (hi, lo) per piece:
//     A = [H ; H_lo]   (M = 128: in-units hi, then lo)
//     B = [Zb ; Zb_lo] (N = 128: out-units hi, then lo)
// and ONE M = N = 128 MMA per 8 rows yields every split product at once:
// D[i][o] = H_hi Z_hi, D[i][64 + o] = H_hi Z_lo, D[64 + i][o] = H_lo Z_hi (the
// fourth quadrant, H_lo Z_lo, is dropped).  The accumulator lives in TMEM
// columns [384, 512) for the whole tile; the three quadrants are summed in
// FP32 and red.add-ed into the CTA's f64 gradient row once per tile.  (hi is
// the raw FP32 value, which the tensor core reads truncated; lo =
// rna_tf32(x - trunc(x)).)  `stg` is the idle weight slot (32 KB, 512-byte
// aligned): NBUF chunk buffers of RC rows; `scratch` 4160 floats (free once
// the chunks are staged).
#ifndef FR_TC_DW_RC
#define FR_TC_DW_RC 32
#endif
__device__ __forceinline__ int b32_at(int m, int k, int RC) {
  return (((m >> 5) * (RC >> 2) + (k >> 2)) << 7) + ((k & 3) << 5) + (((((m & 31) >> 3) ^ k) & 3) << 3) + (m & 7);
}
// The dX hi passes of the same layer (A = dx_a, B = dx_b) are issued right
// after the last chunk, so the weight-gradient MMAs never queue behind them.
template <int ROWS, int RS4, int NT, int W>
__device__ __forceinline__ void tc3_dw(const float* H, const float* Zb, float* stg, float* scratch, double* gp_w,
                                       TcState& t, int issuer, const float* dx_a, const float* dx_b) {
  constexpr int RC = (FR_TC_DW_RC == 32 && ROWS % 32 == 0) ? 32 : 16, NBUF = 32 / RC;  // 32 rows x {A, B} = 32 KB
  static_assert(W == 64 && ROWS % RC == 0, "tensor-core weight gradient: W = 64, 16-row chunks");
  constexpr int NCH = ROWS / RC, OPF = 128 * RC;  // floats per operand ([4 MN groups][RC / 4 K groups][128])
  constexpr uint32_t DCOL = 384;
  const int tid = threadIdx.x;
  const uint32_t id = tc::idesc_tf32(128, 128, 1, 1);
  FR_TC_START;
#pragma unroll 1
  for (int c = 0; c < NCH; ++c) {
    const int b = c % NBUF;
    float* buf = stg + 2 * OPF * b;
    if (c >= NBUF) {  // the chunk-(c - NBUF) MMAs must be done with this buffer
      mbar_wait_bounded(t.mbar_dw + b, (t.dw_phase >> b) & 1u);
      t.dw_phase ^= 1u << b;
    }
    FR_TC_MARK(13);
    const int r0 = RC * c;
    for (int it = tid; it < 2 * RC * 16; it += NT) {
      const int which = it / (RC * 16), r = (it >> 4) % RC, q = it & 15;
      const float4 v = *reinterpret_cast<const float4*>((which ? Zb : H) + q * RS4 + (r0 + r) * 4);
      float* dst = buf + which * OPF;
      *reinterpret_cast<float4*>(dst + b32_at(4 * q, r, RC)) = v;
      *reinterpret_cast<float4*>(dst + b32_at(64 + 4 * q, r, RC)) =
          make_float4(tf32_alo(v.x), tf32_alo(v.y), tf32_alo(v.z), tf32_alo(v.w));
    }
    FR_TC_MARK(14);
    tc::fence_proxy_async();
    __syncthreads();
    FR_TC_MARK(15);
    if (tid == issuer) {
      tc::fence_after();
      const uint64_t a0 = tc::desc(buf, RC / 4 * 512, 512) | (uint64_t(1) << 61);
      const uint64_t b0 = tc::desc(buf + OPF, RC / 4 * 512, 512) | (uint64_t(1) << 61);
#pragma unroll
      for (int ks = 0; ks < RC / 8; ++ks)
        mma_tf32_lit(t.tmem + DCOL, a0 + uint64_t((1024 * ks) >> 4), b0 + uint64_t((1024 * ks) >> 4), id,
                     c != 0 || ks != 0);
      tc::mma_commit(t.mbar_dw + b);
    }
  }
  tc3_issue_hi<ROWS, RS4>(dx_a, dx_b, t, issuer);
  // the last NBUF chunks' completions (the last covers every MMA before it)
#pragma unroll
  for (int k = NCH >= NBUF ? NCH - NBUF : 0; k < NCH; ++k) {
    const int b = k % NBUF;
    mbar_wait_bounded(t.mbar_dw + b, (t.dw_phase >> b) & 1u);
    t.dw_phase ^= 1u << b;
  }
  tc::fence_after();
  FR_TC_MARK(13);
  // drain: lanes 64..127 (H_lo Z_hi) into shared memory [o][i] (stride 65:
  // conflict-free both ways), lanes 0..63 add H_hi Z_hi + H_hi Z_lo to it, then
  // every thread red.adds a coalesced run of the 64 x 64 block once
  const int w = tid >> 5, q = w & 3;
  if (w < 4 && q >= 2) {
    const int i = 32 * (q - 2) + (tid & 31);
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 16) {
      float v[16];
      tc::tmem_ld16(t.tmem + (uint32_t(32 * q) << 16) + DCOL + c0, v);
#pragma unroll
      for (int k = 0; k < 16; ++k) scratch[(c0 + k) * 65 + i] = v[k];
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (w < 4 && q < 2) {
    const int i = 32 * q + (tid & 31);
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 16) {
      float v[16], z[16];
      tc::tmem_ld16(t.tmem + (uint32_t(32 * q) << 16) + DCOL + c0, v);
      tc::tmem_ld16(t.tmem + (uint32_t(32 * q) << 16) + DCOL + 64 + c0, z);
#pragma unroll
      for (int k = 0; k < 16; ++k) scratch[(c0 + k) * 65 + i] += v[k] + z[k];
    }
  }
  tc::fence_before();
  __syncthreads();
  for (int e = tid; e < W * W; e += NT) {
    const int i = e / W, o = e % W;
    red_add(gp_w + e, double(scratch[o * 65 + i]));
  }
  __syncthreads();
  FR_TC_MARK(9);
}

// A_lo of a whole k-quad buffer, out of place (dst may not alias src)
template <int RS4, int NT>
__device__ __forceinline__ void tc3_make_lo(float* dst, const float* src) {
  FR_TC_START;
  __syncthreads();  // dst may still be read by the caller's previous phase (the dW combine reads Xs)
  for (int i = 4 * threadIdx.x; i < 16 * RS4; i += 4 * NT) {
    const float4 v = *reinterpret_cast<const float4*>(src + i);
    *reinterpret_cast<float4*>(dst + i) = make_float4(tf32_alo(v.x), tf32_alo(v.y), tf32_alo(v.z), tf32_alo(v.w));
  }
  tc::fence_proxy_async();
  __syncthreads();
  FR_TC_MARK(10);
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
// Processes tiles t0, t0 + tstride, ... of one dataset with this CTA.  Gradient
// contributions are red.add-ed into gp_row (zeroed first when zero_partials);
// the CTA's loss sums are written to lpart_row[0..1].
template <typename T, int ACT, int MODE, int REG, int W, int NT_, bool TC = false>
__device__ __forceinline__ void run_tiles(const KArgs& a, unsigned char* smem_raw, long long t0, long long tstride,
                                          bool zero_partials, double* gp_row, double* lpart_row,
                                          TcState* tcs = nullptr) {
  using C = JetCfg<T, ACT, MODE, REG, W, NT_>;
  constexpr int NT = C::NT, G = C::G, RPT = C::RPT, ROWS = C::ROWS, PPT = C::PPT;
  constexpr int DIN = C::DIN, NOUT = C::NOUT, NVEL = C::NVEL, S = C::S;
  constexpr int NG = C::NG, NL = C::NL, LAP0 = C::LAP0, RS4 = C::RS4;
  constexpr int NST0 = C::NST0, NSTH = C::NSTH, PP = C::PP;
  constexpr bool JET = C::JET, BWD = C::BWD;

  // no tile of this dataset for this CTA (the epoch kernel's later MSE sets
  // on most CTAs): skip the weight staging and prologue, write zero loss sums
  if (!zero_partials && t0 >= (a.n + PPT - 1) / PPT) {
    if constexpr (BWD)
      if (threadIdx.x == 0 && lpart_row) {
        lpart_row[0] = 0.0;
        lpart_row[1] = 0.0;
      }
    return;
  }
  const int L = a.L;
  T* sm = reinterpret_cast<T*>(smem_raw);
  T* Xs = sm;                      sm += C::al(C::XELEMS);
  T* Gs = nullptr;
  if constexpr (BWD) { Gs = sm; sm += C::al(C::XELEMS); }
  static_assert(!TC || (sizeof(T) == 4 && W == 64 && BWD), "split-TF32 path: FP32, W = 64, training modes");
  constexpr int SLOT = (TC ? 2 : 1) * W * W;  // TC: {hi, lo} UMMA slab pair
  T* slot0 = sm;                   sm += SLOT;
  T* slot1 = sm;                   sm += SLOT;
  T* W0s = sm;                     sm += C::al(DIN * W);
  T* Bs = sm;                      sm += C::al(L * W);
  T* WLs = sm;                     sm += C::al(W * NOUT);
  T* bLs = sm;                     sm += 4;
  T* Ys = sm;                      sm += C::al(ROWS * NOUT);
  T* Ybs = nullptr;
  if constexpr (BWD) { Ybs = sm; sm += C::al(ROWS * NOUT); }
  T* Ps = sm;                      sm += C::al(PPT * DIN);
  T* Dbs = Ys;  // hidden-layer db partials: Ys is dead after the head
  (void)sm;

  const int tid = threadIdx.x;
  const int g = tid % G;
  const int rg = tid / G;
  const T* kp = static_cast<const T*>(a.kp);
  const ParamLayout pl{DIN, W, NOUT, L};
  const long long n = a.n;

  for (int i = tid; i < DIN * W; i += NT) W0s[i] = kp[pl.off_w(0) + i];
  for (int i = tid; i < L * W; i += NT) Bs[i] = kp[pl.off_b(i / W) + i % W];
  for (int i = tid; i < W * NOUT; i += NT) WLs[i] = kp[pl.off_w(L) + i];
  if (tid < NOUT) bLs[tid] = kp[pl.off_b(L) + tid];

  double* gp = nullptr;
  if constexpr (BWD) {
    gp = gp_row;
    if (zero_partials)
      for (int i = tid; i < a.np_pad; i += NT) gp[i] = 0.0;
  }
  T* stash = static_cast<T*>(a.scratch) + size_t(blockIdx.x) * a.stash_elems;
  // stash element q of `layer` for this thread: sq<NT>(st_at(layer), q) -- one
  // 64-bit base per layer, every q an immediate offset (quad layout above)
  T* const stash_t = stash + 4 * tid;
  auto st_at = [&](int layer) { return stash_t + size_t(C::stash_layer_base(layer)) * NT; };

  double lacc0 = 0.0, lacc1 = 0.0;

  // weight-matrix stream: W_1..W_{L-1} (forward) then W_{L-1}^T..W_1^T (dX)
  const int nmat = (L - 1) * (BWD ? 2 : 1);
  auto mat_src = [&](int idx) -> const T* {
    int i = idx % nmat;
    if constexpr (TC) {  // forward slab of layer i + 1, then adjoint slabs of layers L-1..1
      if (i < L - 1) return kp + a.tc3 + size_t(i) * 2 * 8192;
      return kp + a.tc3 + (size_t(2 * L - 3 - i) * 2 + 1) * 8192;
    }
    if (i < L - 1) return kp + pl.off_w(i + 1);
    return kp + pl.off_wt(2 * L - 2 - i);
  };
  auto stage = [&](int idx) {
    T* dst = (idx & 1) ? slot1 : slot0;
    const T* src = mat_src(idx);
    constexpr int CH = SLOT * int(sizeof(T)) / 16;
    for (int i = tid; i < CH; i += NT)
      cp_async16(reinterpret_cast<char*>(dst) + 16 * i, reinterpret_cast<const char*>(src) + 16 * i);
    cp_async_commit();
  };
  int ws = 0;
  if (nmat > 0) {
    stage(0);
    cp_async_wait_all();
  }
  __syncthreads();

  const long long ntiles = (n + PPT - 1) / PPT;
  if constexpr (MODE == MODE_MSE) {
    if (a.gate != nullptr && t0 < ntiles) {
      if (tid == 0) gate_wait(a.gate, a.gate_round, a.gate_mult, a.flags, a.gate_timeout_ns);
      __syncthreads();
    }
  }
#ifdef FR_PHASE_TIMERS
  long long ph_acc[16] = {0};
  long long ph_last = clock64();
#endif
  for (long long tile = t0; tile < ntiles; tile += tstride) {
    const long long p0 = tile * PPT;
    {
      const T* pts = static_cast<const T*>(a.pts) + p0 * DIN;
      const long long rem = n - p0;
      for (int i = tid; i < PPT * DIN; i += NT) Ps[i] = (i / DIN < rem) ? pts[i] : T(0);
    }
    __syncthreads();
    FR_MARK(0);

    // ---------------- layer 0 (DIN -> W): derivative blocks are constant ----------------
    {
      T outv[RPT][8];
      T s0v[8 * NST0];  // JET: layer-0 stash run (s, [c]) over this thread's 8 units
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int u = unit_of<W>(g, j);
        const T b0 = Bs[u];
#pragma unroll
        for (int pr = 0; pr < PP; ++pr) {
          const int pt = JET ? rg : rg * RPT + pr;
          T zv = T(0);
#pragma unroll
          for (int i = 0; i < DIN; ++i) zv = fma(Ps[pt * DIN + i], W0s[i * W + u], zv);
          zv += b0;
          T s, c;
          act_eval<ACT>(zv, s, c);
          if constexpr (JET) {
            T d1, d2;
            act_d12<ACT>(s, c, d1, d2);
            outv[0][j] = s;
#pragma unroll
            for (int i = 0; i < NG; ++i) outv[1 + i][j] = d1 * W0s[i * W + u];
#pragma unroll
            for (int i = 0; i < NL; ++i) {
              const T zg = W0s[(LAP0 + i) * W + u];
              outv[1 + NG + i][j] = d2 * zg * zg;
            }
          } else {
            outv[pr][j] = s;
          }
          if constexpr (BWD) {
            if constexpr (JET) {
              s0v[j * NST0] = s;
              if constexpr (C::SIN) s0v[j * NST0 + 1] = c;
            } else {
              sq<NT>(st_at(0), ((pr * 8 + j) * NST0)) = s;
              if constexpr (C::SIN) sq<NT>(st_at(0), ((pr * 8 + j) * NST0 + 1)) = c;
            }
          }
        }
      }
      if constexpr (BWD && JET) st_run<NT>(st_at(0), 0, s0v);
      store_block<T, W, RPT, RS4>(Xs, rg, g, outv);
      if constexpr (TC) {  // the first hidden contraction's A_lo
#pragma unroll
        for (int r = 0; r < RPT; ++r)
#pragma unroll
          for (int j = 0; j < 8; ++j) outv[r][j] = tf32_alo(outv[r][j]);
        store_block<T, W, RPT, RS4>(Gs, rg, g, outv);
      }
    }
    __syncthreads();
    FR_MARK(1);

    // ---------------- hidden layers 1..L-1 ----------------
    for (int l = 1; l < L; ++l) {
      const T* Bm = (ws & 1) ? slot1 : slot0;
      stage(ws + 1);
      T acc[RPT][8];
      if constexpr (TC) {
        // tensor core: A = Xs (this layer's input), A_lo = Gs (written beside
        // it by the producing epilogue); D -> Gs (this layer's output buffer),
        // then each thread picks up its rows exactly as the SIMT GEMM leaves
        // them in registers
        tc::fence_proxy_async();
        __syncthreads();
        tc3_issue_hi<ROWS, RS4>(reinterpret_cast<const float*>(Xs), reinterpret_cast<const float*>(Bm), *tcs);
        tc3_issue_lo<ROWS, RS4>(reinterpret_cast<const float*>(Gs), reinterpret_cast<const float*>(Bm), *tcs);
        tc3_drain<ROWS, RS4, NT>(reinterpret_cast<float*>(Gs), *tcs);
        load_block<T, W, RPT, RS4>(acc, Gs, rg, g);
      } else {
        gemm_rows<T, W, RPT, RS4>(Xs, Bm, rg, g, acc);
      }
      // training modes ping-pong the layer input / output between Xs and Gs
      // (Gs is idle in the forward sweep), so a warp's epilogue never waits
      // for the slower warps' GEMM; single-buffer modes sync here
      if constexpr (!BWD) __syncthreads();
      FR_MARK(2);
      T outv[RPT][8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int u = unit_of<W>(g, j);
        const T bl = Bs[l * W + u];
        if constexpr (JET) {
          const T zv = acc[0][j] + bl;
          T s, c, d1, d2;
          act_eval<ACT>(zv, s, c);
          act_d12<ACT>(s, c, d1, d2);
          outv[0][j] = s;
#pragma unroll
          for (int i = 0; i < NG; ++i) outv[1 + i][j] = d1 * acc[1 + i][j];
#pragma unroll
          for (int i = 0; i < NL; ++i) {
            const T zg = acc[1 + LAP0 + i][j];
            outv[1 + NG + i][j] = d2 * zg * zg + d1 * acc[1 + NG + i][j];
          }
          if constexpr (BWD) {
            // one run: s, [c], z_g[0..NG), z_l[0..NL)
            static_assert(NSTH == S + C::SIN && 1 + NG + NL == S, "jet stash run layout");
            T sv[NSTH];
            sv[0] = s;
            if constexpr (C::SIN) sv[1] = c;
#pragma unroll
            for (int i = 0; i < NG + NL; ++i) sv[1 + C::SIN + i] = acc[1 + i][j];
            st_run<NT>(st_at(l), j * NSTH, sv);
          }
        } else {
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            const T zv = acc[r][j] + bl;
            T s, c;
            act_eval<ACT>(zv, s, c);
            outv[r][j] = s;
            if constexpr (BWD) {
              sq<NT>(st_at(l), ((r * 8 + j) * NST0)) = s;
              if constexpr (C::SIN) sq<NT>(st_at(l), ((r * 8 + j) * NST0 + 1)) = c;
            }
          }
        }
      }
      store_block<T, W, RPT, RS4>(BWD ? Gs : Xs, rg, g, outv);
      if constexpr (TC) {  // the next contraction's A_lo, into this layer's (consumed) input buffer
#pragma unroll
        for (int r = 0; r < RPT; ++r)
#pragma unroll
          for (int j = 0; j < 8; ++j) outv[r][j] = tf32_alo(outv[r][j]);
        store_block<T, W, RPT, RS4>(Xs, rg, g, outv);
      }
      cp_async_wait_all();
      __syncthreads();
      FR_MARK(3);
      if constexpr (BWD) {
        T* t = Xs;  // this layer's output becomes the next layer's input
        Xs = Gs;
        Gs = t;
      }
      ++ws;
    }

    // ---------------- output layer (W -> NOUT) ----------------
    for (int r = tid; r < ROWS; r += NT) {
      T y[NOUT];
#pragma unroll
      for (int c = 0; c < NOUT; ++c) y[c] = T(0);
#pragma unroll 4
      for (int kq = 0; kq < W / 4; ++kq) {
        T xv[4];
        vload(xv, Xs + kq * RS4 + r * 4);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
          for (int c = 0; c < NOUT; ++c) y[c] = fma(xv[kk], WLs[(4 * kq + kk) * NOUT + c], y[c]);
      }
      const bool vrow = JET ? (r % S == 0) : true;
#pragma unroll
      for (int c = 0; c < NOUT; ++c) Ys[r * NOUT + c] = vrow ? y[c] + bLs[c] : y[c];
    }
    __syncthreads();
    FR_MARK(4);

    // ---------------- head ----------------
    const long long rem = n - p0;
    if constexpr (MODE == MODE_VALUE) {
      T* out = static_cast<T*>(a.out) + p0 * NOUT;
      for (int i = tid; i < PPT * NOUT; i += NT)
        if (i / NOUT < rem) out[i] = Ys[i];
      __syncthreads();
      continue;
    } else if constexpr (MODE == MODE_JET) {
      T* out = static_cast<T*>(a.out) + p0 * S * NOUT;
      for (int i = tid; i < PPT * S * NOUT; i += NT)
        if (i / (S * NOUT) < rem) out[i] = Ys[i];
      __syncthreads();
      continue;
    } else if constexpr (MODE == MODE_PDE) {
      // Navier-Stokes residual head (physics.py:70-93; builders.py:51-64, :98-99)
      using R = Regime<REG>;
      constexpr int NSP = R::NSP, TOFF = R::HAS_T;
      const T inv_re = T(a.inv_re);
      const T two_coef = T(2.0 * a.coef);
      for (int pt = tid; pt < PPT; pt += NT) {
        const T* y = Ys + pt * S * NOUT;
        T* yb = Ybs + pt * S * NOUT;
#pragma unroll
        for (int i = 0; i < S * NOUT; ++i) yb[i] = T(0);
        if (pt >= rem) continue;
        auto Y = [&](int s, int c) { return y[s * NOUT + c]; };
        auto GRAD = [&](int in) { return 1 + in; };
        auto LAP = [&](int in) { return 1 + NG + (in - LAP0); };
        constexpr int P = NVEL;  // pressure channel
        T r[NVEL + 1];
#pragma unroll
        for (int i = 0; i < NVEL; ++i) {
          const int xi = TOFF + i;
          T acc = T(0);
          if constexpr (R::HAS_T) acc = Y(GRAD(0), i);
          acc = (R::HAS_T ? acc + Y(GRAD(xi), P) : Y(GRAD(xi), P));
#pragma unroll
          for (int jj = 0; jj < NSP; ++jj) acc += -inv_re * Y(LAP(TOFF + jj), i);
#pragma unroll
          for (int k = 0; k < NVEL; ++k) acc += Y(0, k) * Y(GRAD(TOFF + k), i);
          r[i] = acc;
        }
        {
          T acc = Y(GRAD(TOFF), 0);
#pragma unroll
          for (int k = 1; k < NVEL; ++k) acc += Y(GRAD(TOFF + k), k);
          r[NVEL] = acc;
        }
        double sq = 0.0;
#pragma unroll
        for (int i = 0; i <= NVEL; ++i) sq += double(r[i]) * double(r[i]);
        lacc0 += sq;
        // adjoints of the jet outputs
#pragma unroll
        for (int i = 0; i < NVEL; ++i) {
          const T rb = two_coef * r[i];
          const int xi = TOFF + i;
          if constexpr (R::HAS_T) yb[GRAD(0) * NOUT + i] += rb;
          yb[GRAD(xi) * NOUT + P] += rb;
#pragma unroll
          for (int jj = 0; jj < NSP; ++jj) yb[LAP(TOFF + jj) * NOUT + i] += -inv_re * rb;
#pragma unroll
          for (int k = 0; k < NVEL; ++k) {
            yb[0 * NOUT + k] += rb * Y(GRAD(TOFF + k), i);
            yb[GRAD(TOFF + k) * NOUT + i] += rb * Y(0, k);
          }
        }
        {
          const T rb = two_coef * r[NVEL];
#pragma unroll
          for (int k = 0; k < NVEL; ++k) yb[GRAD(TOFF + k) * NOUT + k] += rb;
        }
      }
    } else if constexpr (MODE == MODE_GJ) {
      // C^1 interface extension (off by default; the reference couples values
      // only, worker.py:179-197): sum_i sum_c w_c (d u_c/d x_i - target)^2
      const T two_c = T(2.0 * a.coef);
      for (int pt = tid; pt < PPT; pt += NT) {
        T* yb = Ybs + pt * S * NOUT;
#pragma unroll
        for (int i = 0; i < S * NOUT; ++i) yb[i] = T(0);
        if (pt >= rem) continue;
        const T* y = Ys + pt * S * NOUT;
        const T* td = static_cast<const T*>(a.tu) + (p0 + pt) * (NG * NVEL);
        double sq = 0.0;
#pragma unroll
        for (int i = 0; i < NG; ++i)
#pragma unroll
          for (int c = 0; c < NVEL; ++c) {
            const T d = y[(1 + i) * NOUT + c] - __ldcg(td + i * NVEL + c);
            sq += a.velw[c] * (double(d) * double(d));
            yb[(1 + i) * NOUT + c] = (two_c * T(a.velw[c])) * d;
          }
        lacc0 += sq;
      }
    } else {  // MODE_MSE: squared error against targets (builders.py:103-141)
      const T two_vc = T(2.0 * a.coef);
      const T two_pc = T(2.0 * a.pcoef);
      for (int pt = tid; pt < PPT; pt += NT) {
        T* yb = Ybs + pt * NOUT;
#pragma unroll
        for (int c = 0; c < NOUT; ++c) yb[c] = T(0);
        if (pt >= rem) continue;
        const T* y = Ys + pt * NOUT;
        double squ = 0.0;
#pragma unroll
        for (int c = 0; c < NVEL; ++c) {
          // L2-coherent loads: ghost targets may land while this kernel runs (gate)
          const T d = y[c] - __ldcg(static_cast<const T*>(a.tu) + (p0 + pt) * NVEL + c);
          const T w = T(a.velw[c]);
          squ += double(a.velw[c]) * (double(d) * double(d));
          yb[c] = (two_vc * w) * d;
        }
        lacc0 += squ;
        if (a.has_p) {
          const T d = y[NVEL] - __ldcg(static_cast<const T*>(a.tp) + p0 + pt);
          lacc1 += double(d) * double(d);
          yb[NVEL] = two_pc * d;
        }
      }
    }
    __syncthreads();
    FR_MARK(5);

    if constexpr (BWD) {
      // ---------------- output layer backward ----------------
      // dW_L = H_L^T Ybar: thread (k-quad, row split) accumulates 4 k x NOUT over
      // its rows; the partials meet in Gs (free until dX_L) in a fixed order.
      {
        constexpr int KQ = W / 4, RSL = NT / KQ;
        static_assert(NT % KQ == 0 && RSL * W * NOUT <= C::XELEMS, "output-layer split must fit");
        const int kq = tid % KQ, rsl = tid / KQ;
        T acc[4][NOUT];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int c = 0; c < NOUT; ++c) acc[x][c] = T(0);
        const T* xp = Xs + kq * RS4;
#pragma unroll 2
        for (int r = rsl; r < ROWS; r += RSL) {
          T hv[4];
          vload(hv, xp + 4 * r);
#pragma unroll
          for (int c = 0; c < NOUT; ++c) {
            const T yb = Ybs[r * NOUT + c];
#pragma unroll
            for (int x = 0; x < 4; ++x) acc[x][c] = fma(hv[x], yb, acc[x][c]);
          }
        }
        T* part = Gs + rsl * (W * NOUT);
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int c = 0; c < NOUT; ++c) part[(4 * kq + x) * NOUT + c] = acc[x][c];
      }
      __syncthreads();
      for (int i = tid; i < W * NOUT; i += NT) {
        constexpr int RSL = NT / (W / 4);
        T s = Gs[i];
        for (int q = 1; q < RSL; ++q) s += Gs[q * (W * NOUT) + i];
        red_add(gp + pl.off_w(L) + i, double(s));
      }
      if (tid < NOUT) {
        T s = T(0);
        for (int pt = 0; pt < PPT; ++pt) s += Ybs[(JET ? pt * S : pt) * NOUT + tid];
        red_add(gp + pl.off_b(L) + tid, double(s));
      }
      __syncthreads();
      {
        T gv[RPT][8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int u = unit_of<W>(g, j);
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            const int row = rg * RPT + r;
            T s = T(0);
#pragma unroll
            for (int c = 0; c < NOUT; ++c) s = fma(Ybs[row * NOUT + c], WLs[u * NOUT + c], s);
            gv[r][j] = s;
          }
        }
        store_block<T, W, RPT, RS4>(Gs, rg, g, gv);
      }
      __syncthreads();
      FR_MARK(6);

      // ---------------- hidden layers L-1..1 ----------------
      for (int l = L - 1; l >= 1; --l) {
        // activation backward (numpy_backend.py:58-89): S-bar -> Z-bar, in place in Gs
        {
          T sb[RPT][8];
          load_block<T, W, RPT, RS4>(sb, Gs, rg, g);
          T zb[RPT][8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if constexpr (JET) {
              // numpy_backend.py:58-89, factors rebuilt from the stashed jet
              T fv[NSTH];
              ld_run<NT>(fv, st_at(l), j * NSTH);
              const T sj = fv[0], cj = C::SIN ? fv[1] : T(0);
              T d1, d2;
              act_d12<ACT>(sj, cj, d1, d2);
              const T d3 = act_d3<ACT>(sj, cj, d1, d2);
              const T* zgv = fv + 1 + C::SIN;
              T ga[NG], lb[NL > 0 ? NL : 1];
#pragma unroll
              for (int i = 0; i < NG; ++i) ga[i] = d2 * zgv[i];
#pragma unroll
              for (int i = 0; i < NL; ++i) {
                const T zg = zgv[LAP0 + i];
                lb[i] = d3 * zg * zg + d2 * zgv[NG + i];
              }
              T zv = sb[0][j] * d1;
#pragma unroll
              for (int i = 0; i < NG; ++i) zv += sb[1 + i][j] * ga[i];
#pragma unroll
              for (int i = 0; i < NL; ++i) zv += sb[1 + NG + i][j] * lb[i];
              zb[0][j] = zv;
#pragma unroll
              for (int i = 0; i < NG; ++i) {
                T t = sb[1 + i][j] * d1;
                if (i >= LAP0 && i - LAP0 < NL) t += (T(2) * ga[i]) * sb[1 + NG + (i - LAP0)][j];
                zb[1 + i][j] = t;
              }
#pragma unroll
              for (int i = 0; i < NL; ++i) zb[1 + NG + i][j] = sb[1 + NG + i][j] * d1;
            } else {
#pragma unroll
              for (int r = 0; r < RPT; ++r) {
                const T s = sq<NT>(st_at(l), ((r * 8 + j) * NST0));
                const T c = C::SIN ? sq<NT>(st_at(l), ((r * 8 + j) * NST0 + 1)) : T(0);
                T d1, d2;
                act_d12<ACT>(s, c, d1, d2);
                zb[r][j] = sb[r][j] * d1;
              }
            }
          }
          store_block<T, W, RPT, RS4>(Gs, rg, g, zb);
        }
        // rebuild this layer's input H_l = jets of layer l-1 into Xs
        {
          T hv[RPT][8];
          const int lp = l - 1;
          T s0v[8 * NST0];
          if constexpr (JET) {
            if (lp == 0) ld_run<NT>(s0v, st_at(0), 0);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int u = unit_of<W>(g, j);
            if constexpr (JET) {
              if (lp == 0) {
                const T s = s0v[j * NST0];
                const T c = C::SIN ? s0v[j * NST0 + 1] : T(0);
                T d1, d2;
                act_d12<ACT>(s, c, d1, d2);
                hv[0][j] = s;
#pragma unroll
                for (int i = 0; i < NG; ++i) hv[1 + i][j] = d1 * W0s[i * W + u];
#pragma unroll
                for (int i = 0; i < NL; ++i) {
                  const T zg = W0s[(LAP0 + i) * W + u];
                  hv[1 + NG + i][j] = d2 * zg * zg;
                }
              } else {
                // the layer's output streams, rebuilt as in the forward epilogue
                T hvv[NSTH];
                ld_run<NT>(hvv, st_at(lp), j * NSTH);
                const T sj = hvv[0], cj = C::SIN ? hvv[1] : T(0);
                T d1, d2;
                act_d12<ACT>(sj, cj, d1, d2);
                const T* zgv = hvv + 1 + C::SIN;
                hv[0][j] = sj;
#pragma unroll
                for (int i = 0; i < NG; ++i) hv[1 + i][j] = d1 * zgv[i];
#pragma unroll
                for (int i = 0; i < NL; ++i) {
                  const T zg = zgv[LAP0 + i];
                  hv[1 + NG + i][j] = d2 * zg * zg + d1 * zgv[NG + i];
                }
              }
            } else {
#pragma unroll
              for (int r = 0; r < RPT; ++r) hv[r][j] = sq<NT>(st_at(lp), ((r * 8 + j) * NST0));
            }
          }
          store_block<T, W, RPT, RS4>(Xs, rg, g, hv);
        }
        if constexpr (TC) tc::fence_proxy_async();  // Zbar_l (Gs) feeds the tensor core next
        __syncthreads();
        FR_MARK(7);
        // tensor core: the dX hi passes over Zbar_l run under the SIMT weight
        // gradient, issued by a thread the dW thread tiles leave idle
        // tensor-core MMAs of the backward layer: issued by a thread the SIMT
        // dW leaves idle (or, with the tensor-core dW, by the last warp, which
        // has the least staging work)
        // TC: the SIMT dW may spread over 6 row ranges (all 12 warps), its 5th
        // and 6th partials parked in the idle weight slot (the next matrix is
        // then prefetched after the combine)
        constexpr bool TC_DW = TC && FR_TC_DW;
        constexpr int RSPLIT_DW = (TC && !TC_DW && FR_DW_SPLIT6 && ROWS % 6 == 0 && C::KT * C::KT * 6 == NT &&
                                   C::XELEMS / (W * W) + 2 >= 6)
                                      ? 6 : C::RSPLIT;
        constexpr bool SLOT_PARTIALS = RSPLIT_DW * W * W > C::XELEMS;
        constexpr int DX_ISSUER = TC_DW ? NT - 32
                                  : (C::KT * C::KT * RSPLIT_DW < NT) ? C::KT * C::KT * RSPLIT_DW : 0;
        constexpr bool DX_EARLY = TC && (TC_DW || (FR_TC_DX_EARLY && C::KT * C::KT * RSPLIT_DW < NT));
        if constexpr (DX_EARLY && !TC_DW)
          tc3_issue_hi<ROWS, RS4>(reinterpret_cast<const float*>(Gs),
                                  reinterpret_cast<const float*>((ws & 1) ? slot1 : slot0), *tcs, DX_ISSUER);
        if constexpr (TC_DW) {
          // weight gradient on the tensor core, staged through the idle weight
          // slot (the next matrix is prefetched after it); db_l on the SIMT side
          tc3_dw<ROWS, RS4, NT, W>(reinterpret_cast<const float*>(Xs), reinterpret_cast<const float*>(Gs),
                                   reinterpret_cast<float*>((ws & 1) ? slot0 : slot1), reinterpret_cast<float*>(Xs),
                                   gp + pl.off_w(l), *tcs, DX_ISSUER, reinterpret_cast<const float*>(Gs),
                                   reinterpret_cast<const float*>((ws & 1) ? slot1 : slot0));
          FR_MARK(8);
          {
            constexpr int NH = NT / W;
            const int u = tid % W, h = tid / W;
            T sb = T(0);
            for (int pt = h; pt < PPT; pt += NH) sb += Gs[kqi<RS4>(JET ? pt * S : pt, u)];
            Dbs[tid] = sb;
          }
          __syncthreads();
          if (tid < W) {
            T sb = Dbs[tid];
#pragma unroll
            for (int h = 1; h < NT / W; ++h) sb += Dbs[h * W + tid];
            red_add(gp + pl.off_b(l) + tid, double(sb));
          }
          FR_MARK(9);
        }
        if constexpr (!SLOT_PARTIALS) stage(ws + 1);

        // dW_l = H_l^T Zbar_l over all rows of the tile.  Thread tile 8k x 8u
        // (k quads {kt, kt+W/8}, u quads {ut, ut+W/8}) over one of RSPLIT row
        // ranges; a quarter-warp shares kt (broadcast H) and spans 8 ut (one
        // conflict-free 128-byte Zbar segment).  Row-range partials are combined
        // through shared memory in a fixed order, then red.add-ed once.
        if constexpr (!TC_DW) {
          constexpr int KT = C::KT, RSPLIT = RSPLIT_DW, RROWS = ROWS / RSPLIT;
          // row-range partial rs: Xs, or (SLOT_PARTIALS) the idle weight slot past Xs' capacity
          T* const pslot = (ws & 1) ? slot0 : slot1;
          auto part = [&](int q) -> T* {
            constexpr int INXS = C::XELEMS / (W * W);
            return (!SLOT_PARTIALS || q < INXS) ? Xs + q * W * W : pslot + (q - INXS) * W * W;
          };
          const bool active = tid < KT * KT * RSPLIT;
          const int ut = tid % KT, kt = (tid / KT) % KT, rs = tid / (KT * KT);
          T acc[8][8];
#pragma unroll
          for (int x = 0; x < 8; ++x)
#pragma unroll
            for (int y = 0; y < 8; ++y) acc[x][y] = T(0);
          if constexpr (sizeof(T) == 4) {
            // FP32: unit pairs as FFMA2 (H broadcast), same fma chain order
            if (active) {
              const float* x0 = reinterpret_cast<const float*>(Xs) + kt * RS4 + 4 * (rs * RROWS);
              const float* x1 = reinterpret_cast<const float*>(Xs) + (kt + KT) * RS4 + 4 * (rs * RROWS);
              const float* z0 = reinterpret_cast<const float*>(Gs) + ut * RS4 + 4 * (rs * RROWS);
              const float* z1 = reinterpret_cast<const float*>(Gs) + (ut + KT) * RS4 + 4 * (rs * RROWS);
              f32x2 acc2[8][4];
#pragma unroll
              for (int x = 0; x < 8; ++x)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc2[x][q] = 0ull;
              constexpr int kDwU = TC ? kDwUnrollTC : kDwUnroll;
#pragma unroll kDwU
              for (int r = 0; r < RROWS; ++r) {
                float h[8];
                f32x2 z[4];
                vload(*reinterpret_cast<float(*)[4]>(h), x0 + 4 * r);
                vload(*reinterpret_cast<float(*)[4]>(h + 4), x1 + 4 * r);
                f2_lds(z[0], z[1], z0 + 4 * r);
                f2_lds(z[2], z[3], z1 + 4 * r);
#pragma unroll
                for (int x = 0; x < 8; ++x)
#pragma unroll
                  for (int q = 0; q < 4; ++q) f2_fma(acc2[x][q], h[x], z[q]);
              }
#pragma unroll
              for (int x = 0; x < 8; ++x)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  float a0, a1;
                  f2_unpack(acc2[x][q], a0, a1);
                  acc[x][2 * q] = T(a0);
                  acc[x][2 * q + 1] = T(a1);
                }
            }
          } else if (active) {
            const T* x0 = Xs + kt * RS4 + 4 * (rs * RROWS);
            const T* x1 = Xs + (kt + KT) * RS4 + 4 * (rs * RROWS);
            const T* z0 = Gs + ut * RS4 + 4 * (rs * RROWS);
            const T* z1 = Gs + (ut + KT) * RS4 + 4 * (rs * RROWS);
#pragma unroll 4
            for (int r = 0; r < RROWS; ++r) {
              T h[8], z[8];
              vload(*reinterpret_cast<T(*)[4]>(h), x0 + 4 * r);
              vload(*reinterpret_cast<T(*)[4]>(h + 4), x1 + 4 * r);
              vload(*reinterpret_cast<T(*)[4]>(z), z0 + 4 * r);
              vload(*reinterpret_cast<T(*)[4]>(z + 4), z1 + 4 * r);
#pragma unroll
              for (int x = 0; x < 8; ++x)
#pragma unroll
                for (int y = 0; y < 8; ++y) acc[x][y] = fma(h[x], z[y], acc[x][y]);
            }
          }
          {
            // db_l partials: thread = (unit, point phase); combined below in phase order
            constexpr int NH = NT / W;
            static_assert(NT % W == 0, "db split needs NT % W == 0");
            const int u = tid % W, h = tid / W;
            T sb = T(0);
            for (int pt = h; pt < PPT; pt += NH) sb += Gs[kqi<RS4>(JET ? pt * S : pt, u)];
            Dbs[tid] = sb;
          }
          __syncthreads();  // every read of Xs (H_l) is done: reuse it as scratch
          FR_MARK(8);
          // combine the RSPLIT row-range partials: every thread sums a strided
          // slice of the 64x64 block over rs = 0, 1, ... (fixed order) and
          // red.adds it once
          auto kidx = [&](int x) { return x < 4 ? 4 * kt + x : 4 * (kt + KT) + (x - 4); };
          static_assert(RSPLIT == 1 || RSPLIT <= C::XELEMS / (W * W) + (SLOT_PARTIALS ? 2 : 0),
                        "dW row-range partials must fit in Xs (+ the idle weight slot)");
          if constexpr (RSPLIT == 1) {
            // one row range: every dW element has exactly one owner thread,
            // which red.adds its 8x8 block straight from registers
            if (active) {
              double* dst = gp + pl.off_w(l);
#pragma unroll
              for (int x = 0; x < 8; ++x)
#pragma unroll
                for (int y = 0; y < 8; ++y)
                  red_add(dst + kidx(x) * W + (y < 4 ? 4 * ut + y : 4 * (ut + KT) + (y - 4)), double(acc[x][y]));
            }
          } else if (active) {
            T* dst = part(rs);
#pragma unroll
            for (int x = 0; x < 8; ++x) {
              vstore(dst + kidx(x) * W + 4 * ut, *reinterpret_cast<const T(*)[4]>(&acc[x][0]));
              vstore(dst + kidx(x) * W + 4 * (ut + KT), *reinterpret_cast<const T(*)[4]>(&acc[x][4]));
            }
          }
          FR_MARK(9);
          __syncthreads();
          if constexpr (TC && !DX_EARLY)  // no idle thread during dW: the dX hi passes start now
            tc3_issue_hi<ROWS, RS4>(reinterpret_cast<const float*>(Gs),
                                    reinterpret_cast<const float*>((ws & 1) ? slot1 : slot0), *tcs, DX_ISSUER);
          if (tid < W) {
            T sb = Dbs[tid];
#pragma unroll
            for (int h = 1; h < NT / W; ++h) sb += Dbs[h * W + tid];
            red_add(gp + pl.off_b(l) + tid, double(sb));
          }
          if constexpr (RSPLIT > 1) {
            double* dst = gp + pl.off_w(l);
            for (int e = tid; e < W * W; e += NT) {
              T sum = part(0)[e];
#pragma unroll
              for (int q = 1; q < RSPLIT; ++q) sum += part(q)[e];
              red_add(dst + e, double(sum));
            }
          }
          if constexpr (SLOT_PARTIALS) {
            __syncthreads();  // the partials in the idle slot are consumed
            stage(ws + 1);
          }
        }
        // dX: S-bar_{l-1} = Zbar_l W_l^T
        {
          const T* Bm = (ws & 1) ? slot1 : slot0;
          if constexpr (TC) {
            // Zbar_l's A_lo into Xs (free again after the dW combine), the A_lo
            // pass, then S-bar_{l-1} lands straight in Gs
            tc3_make_lo<RS4, NT>(reinterpret_cast<float*>(Xs), reinterpret_cast<const float*>(Gs));
            tc3_issue_lo<ROWS, RS4>(reinterpret_cast<const float*>(Xs), reinterpret_cast<const float*>(Bm), *tcs,
                                    DX_ISSUER);
            tc3_drain<ROWS, RS4, NT>(reinterpret_cast<float*>(Gs), *tcs);
            FR_MARK(10);
          } else if constexpr (sizeof(T) == 4) {
            f32x2 acc2[RPT][4];
            gemm_rows_f2<W, RPT, RS4>(reinterpret_cast<const float*>(Gs), reinterpret_cast<const float*>(Bm), rg,
                                      g, acc2);
            __syncthreads();
            FR_MARK(10);
            store_block_f2<W, RPT, RS4>(reinterpret_cast<float*>(Gs), rg, g, acc2);
          } else {
            T acc[RPT][8];
            gemm_rows<T, W, RPT, RS4>(Gs, Bm, rg, g, acc);
            __syncthreads();
            FR_MARK(10);
            store_block<T, W, RPT, RS4>(Gs, rg, g, acc);
          }
        }
        cp_async_wait_all();
        __syncthreads();
        FR_MARK(11);
        ++ws;
      }

      // ---------------- layer 0 backward ----------------
      {
        T sb[RPT][8];
        load_block<T, W, RPT, RS4>(sb, Gs, rg, g);
        T zb[RPT][8];
        T s0v[8 * NST0];
        if constexpr (JET) ld_run<NT>(s0v, st_at(0), 0);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int u = unit_of<W>(g, j);
          if constexpr (JET) {
            const T s = s0v[j * NST0];
            const T c = C::SIN ? s0v[j * NST0 + 1] : T(0);
            T d1, d2;
            act_d12<ACT>(s, c, d1, d2);
            const T d3 = act_d3<ACT>(s, c, d1, d2);
            T zg[NG];
#pragma unroll
            for (int i = 0; i < NG; ++i) zg[i] = W0s[i * W + u];
            T zv = sb[0][j] * d1;
#pragma unroll
            for (int i = 0; i < NG; ++i) zv += sb[1 + i][j] * (d2 * zg[i]);
#pragma unroll
            for (int i = 0; i < NL; ++i) {
              const T gg = zg[LAP0 + i];
              zv += sb[1 + NG + i][j] * (d3 * gg * gg);
            }
            zb[0][j] = zv;
#pragma unroll
            for (int i = 0; i < NG; ++i) {
              T t = sb[1 + i][j] * d1;
              if (i >= LAP0 && i - LAP0 < NL) t += (T(2) * d2) * zg[i] * sb[1 + NG + (i - LAP0)][j];
              zb[1 + i][j] = t;
            }
#pragma unroll
            for (int i = 0; i < NL; ++i) zb[1 + NG + i][j] = sb[1 + NG + i][j] * d1;
          } else {
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
              const T s = sq<NT>(st_at(0), ((r * 8 + j) * NST0));
              const T c = C::SIN ? sq<NT>(st_at(0), ((r * 8 + j) * NST0 + 1)) : T(0);
              T d1, d2;
              act_d12<ACT>(s, c, d1, d2);
              zb[r][j] = sb[r][j] * d1;
            }
          }
        }
        store_block<T, W, RPT, RS4>(Gs, rg, g, zb);
      }
      __syncthreads();
      FR_MARK(12);
      // dW0 = X^T Zbar over the stacked input (value rows hold the points, the
      // derivative block j is the unit vector e_j, tape.py:426-436); db0.
      for (int i = tid; i < (DIN + 1) * W; i += NT) {
        const int j = i / W, u = i % W;
        T s = T(0);
        if (j < DIN) {
          for (int pt = 0; pt < PPT; ++pt) {
            const int row = JET ? pt * S : pt;
            s = fma(Ps[pt * DIN + j], Gs[kqi<RS4>(row, u)], s);
            if constexpr (JET) s += Gs[kqi<RS4>(row + 1 + j, u)];
          }
          red_add(gp + pl.off_w(0) + j * W + u, double(s));
        } else {
          for (int pt = 0; pt < PPT; ++pt) s += Gs[kqi<RS4>(JET ? pt * S : pt, u)];
          red_add(gp + pl.off_b(0) + u, double(s));
        }
      }
      __syncthreads();
      FR_MARK(13);
    }
  }

  cp_async_wait_all();
  if constexpr (BWD) {
    double* red = reinterpret_cast<double*>(Xs);  // the last tile ended with a barrier
    red[tid] = lacc0;
    red[NT + tid] = lacc1;
    __syncthreads();
    if (tid == 0) {
      double s0 = 0.0, s1 = 0.0;
      for (int i = 0; i < NT; ++i) {
        s0 += red[i];
        s1 += red[NT + i];
      }
      lpart_row[0] = s0;
      lpart_row[1] = s1;
    }
  }
#ifdef FR_PHASE_TIMERS
  if (threadIdx.x == 0)
    for (int i = 0; i < 16; ++i) atomicAdd(&g_phase_cycles[i], (unsigned long long)ph_acc[i]);
#endif
  __syncthreads();  // shared memory is reused by the caller's next dataset
}

// one dataset per launch
template <typename T, int ACT, int MODE, int REG, int W>
__global__ void __launch_bounds__(JetCfg<T, ACT, MODE, REG, W>::NT, 1) jetmlp_kernel(KArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int NT = JetCfg<T, ACT, MODE, REG, W>::NT;
  run_tiles<T, ACT, MODE, REG, W, NT>(a, smem_raw, blockIdx.x, gridDim.x, true,
                                      a.gpart ? a.gpart + size_t(blockIdx.x) * a.np_pad : nullptr,
                                      a.lpart ? a.lpart + 2 * blockIdx.x : nullptr);
}

// A whole epoch's loss heads in one persistent launch: every CTA first walks its
// static share of PDE tiles, then the MSE tiles (obs, ghost-spatial,
// ghost-temporal) continue the same round robin: global tile index
// offset + t goes to CTA (offset + t) mod G, so the first MSE tiles land on the
// CTAs that got one PDE tile fewer and no CTA holds more than ceil(total / G)
// tiles.  Assignment is static, so the per-CTA partial sums -- and the reduced
// loss and gradient -- are identical on every run.
struct EpochArgs {
  KArgs pde;
  KArgs mse[3];
  int n_mse;
};

// The epoch kernel runs EpochCfg::CPS CTAs per SM: FP32 W=64 2D uses two
// 192-thread CTAs (24-point tiles, 111 KB of shared memory each), so one CTA's
// barrier waits and latency-bound epilogues are filled by the other's GEMMs.
template <typename T, int ACT, int REG, int W>
struct EpochCfg {
  static constexpr bool TWO = sizeof(T) == 4 && W == 64 && Streams<MODE_PDE, REG>::RPT <= 6 && FR_EPOCH_2CTA;
  static constexpr int NT = TWO ? 192 : JetCfg<T, ACT, MODE_PDE, REG, W>::NT;
  static constexpr int CPS = TWO ? 2 : 1;
};

template <typename T, int ACT, int REG, int W, bool TC = false>
__global__ void __launch_bounds__(EpochCfg<T, ACT, REG, W>::NT, EpochCfg<T, ACT, REG, W>::CPS)
    jetmlp_epoch_kernel(EpochArgs e) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int NT = EpochCfg<T, ACT, REG, W>::NT;
  const long long G = gridDim.x, c = blockIdx.x;
  TcState* tcs = nullptr;
  if constexpr (TC) {
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t mbar[3];
    __shared__ TcState st;
    const uint32_t base = tc_setup<512>(&tmem_slot, mbar, 3);
    st = TcState{base, &mbar[0], 0u, &mbar[1], 0u};
    __syncthreads();
    tcs = &st;
  }
  unsigned char* smem = smem_raw;
  if constexpr (TC) {  // 1 KB-aligned carve: the weight slots then start on 512-byte BASE32B atom boundaries
    smem += (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
    static_assert(TC == false || (2 * JetCfg<T, ACT, MODE_PDE, REG, W, NT>::al(JetCfg<T, ACT, MODE_PDE, REG, W, NT>::XELEMS) * 4) % 512 == 0,
                  "weight slots on 512-byte boundaries");
  }
  double* gp = e.pde.gpart + size_t(c) * e.pde.np_pad;
  TcState local{};
  if constexpr (TC) local = *tcs;  // every thread tracks the barrier phase in a register
  run_tiles<T, ACT, MODE_PDE, REG, W, NT, TC>(e.pde, smem, c, G, true, gp, e.pde.lpart + 2 * c, &local);
  long long offset = (e.pde.n + JetCfg<T, ACT, MODE_PDE, REG, W, NT>::PPT - 1) / JetCfg<T, ACT, MODE_PDE, REG, W, NT>::PPT;
  for (int d = 0; d < e.n_mse; ++d) {
    const long long t0 = ((c - offset) % G + G) % G;
    run_tiles<T, ACT, MODE_MSE, REG, W, NT, TC>(e.mse[d], smem, t0, G, false, gp, e.mse[d].lpart + 2 * c,
                                                &local);
    offset += (e.mse[d].n + JetCfg<T, ACT, MODE_MSE, REG, W, NT>::PPT - 1) / JetCfg<T, ACT, MODE_MSE, REG, W, NT>::PPT;
  }
  if constexpr (TC) tc_teardown<512>(local.tmem);
}

}  // namespace fr
