// Layer-wise jet-MLP kernels for wide experts (hidden width > 64, up to 512).
//
// The fused per-tile kernel keeps a whole network on-chip, which stops working
// once one weight matrix alone exceeds shared memory (W = 150..256 in the
// reference's cylinder presets, config.py:95,117).
// Here every layer is its own persistent-free GEMM launch over the whole point
// set, with the same per-thread jet micro-kernels and epilogues as the fused
// kernel:
//
//   wide_l0      x -> S_0                                   (layer 0, constant jets)
//   wide_fwd(l)  S_{l-1} -> Z_l = S_{l-1} W_l (+b) -> S_l   (+ stash for the bwd)
//   wide_head    S_{L-1} -> Y -> residual / MSE head -> Ybar -> S-bar_{L-1} -> Zbar_{L-1}
//   wide_dx(l)   Zbar_l -> S-bar_{l-1} = Zbar_l W_l^T -> Zbar_{l-1} (activation adjoint)
//   wide_dw(l)   dW_l = sum_rows S_{l-1}^T Zbar_l, db_l      (split over row tiles)
//   wide_dwL     dW_L, db_L from S_{L-1} and Ybar
//   wide_dw0     dW_0, db_0 from the points and Zbar_0
//
// Activations live in HBM/L2 in a tile-major k-quad layout
//   [layer][tile][W/4 quads][tile rows][4]
// so a CTA stages any 32-wide K chunk of a tile with plain 16-byte cp.async
// copies straight into the conflict-free shared layout of the fused kernel.
// A CTA computes a 64-unit output block for one tile (32 points x S streams):
// thread (row group, g) owns all S rows of one point x 8 units, so the jet
// activation (and its adjoint) stays register-local exactly as in the fused
// kernel.  dW partials are accumulated in registers across tiles and flushed
// every few tiles with red.add into one gradient-partial row per row-split
// (single writer per address -> deterministic).
#pragma once
#include "jetmlp_kernel.cuh"

namespace fr {

template <typename T, int ACT, int MODE, int REG>
struct WideCfg {
  using R = Regime<REG>;
  using St = Streams<MODE, REG>;
  static constexpr int DIN = R::DIN, NOUT = R::NOUT, NVEL = R::NVEL;
  static constexpr int S = St::S, NG = St::NG, NL = St::NL, LAP0 = St::LAP0, RPT = St::RPT;
  static constexpr bool JET = St::JET;
  static constexpr bool BWD = (MODE == MODE_PDE || MODE == MODE_MSE);
  static constexpr int UB = 64;        // output units per CTA
  static constexpr int G = UB / 8;     // unit groups
  static constexpr int NT = 256;
  static constexpr int NRG = NT / G;   // 32 row groups
  static constexpr int ROWS = NRG * RPT;
  static constexpr int PPT = JET ? NRG : ROWS;
  static constexpr int PP = JET ? 1 : RPT;
  static constexpr int KC = 32;        // K chunk
  static constexpr int SIN = (ACT == ACT_SIN) ? 1 : 0;
  static constexpr int NST0 = 1 + SIN;
  static constexpr int NSTH = JET ? (1 + SIN + NG + NL) : NST0;
  static constexpr int STQ = 8 * PP * NSTH;  // stash values per thread per (layer, tile, block)
  static constexpr int RS4_BASE = 4 * ROWS;
  static constexpr int RS4 = sizeof(T) == 4 ? RS4_BASE + ((4 - RS4_BASE % 32) + 32) % 32
                                            : RS4_BASE + ((2 - RS4_BASE % 16) + 16) % 16;
  // dW kernel: 8k x 8u thread tiles over a 64 x 64 block, DW_SPLIT row ranges
  static constexpr int DW_NT = 256;
  static constexpr int DW_SPLIT = DW_NT / 64;
  __host__ __device__ static size_t head_smem(int WP) {
    return sizeof(T) * size_t(WP * NOUT + 2 * ((ROWS * NOUT + 3) & ~3)) + 2 * NT * sizeof(double) + 16;
  }
  static_assert(ROWS % DW_SPLIT == 0, "tile rows must split evenly");
  __host__ __device__ static size_t gemm_smem() {
    return sizeof(T) * size_t(2 * (KC / 4) * RS4 + 2 * KC * UB);
  }
  // dW staging: a tile's rows in NRC chunks so H + Zbar (16 quads each) fit
  static constexpr int NRC = (sizeof(T) * 2 * 16 * RS4 > 200 * 1024) ? 2 : 1;
  static constexpr int RCH = ROWS / NRC;
  static constexpr int RS4C = sizeof(T) == 4 ? 4 * RCH + ((4 - (4 * RCH) % 32) + 32) % 32
                                             : 4 * RCH + ((2 - (4 * RCH) % 16) + 16) % 16;
  static_assert(ROWS % (NRC * DW_SPLIT) == 0, "row chunks must split evenly");
  __host__ __device__ static size_t dw_smem() { return sizeof(T) * size_t(2 * 16 * RS4C); }
};

struct WInfo {
  int ppt, rows, nt, stq;
};

struct WArgs {
  const void* kp;
  const void* pts;
  const void* tu;
  const void* tp;
  void* out;          // VALUE / JET outputs
  void* act;          // [L][tiles][WP/4][ROWS][4]
  void* adj;          // [L][tiles][WP/4][ROWS][4]
  void* stash;        // [L][tiles][WP/UB][STQ][NT]
  void* ybar;         // [tiles][ROWS][NOUT]
  double* gpart;      // [ks_rows][np_pad]
  double* lpart;      // [tiles][2]
  long long n;
  int ntiles, L, WP, np_pad, ks_rows;
  int WK;             // parameter-layout width (== WP except on the TF32 path, whose WP is the tensor width)
  double coef, pcoef, inv_re;
  double velw[4];
  int has_p;
  // tensor-core path only
  long long tcw_f, tcw_d;  // kp offsets of the K-major operand slabs of W_l for fwd (N = out) / dx (N = in)
  int nb;                 // output units per CTA (N of the MMA)
  float* p0;              // [tiles][(DIN+1)*WP] per-tile dW_0 | db_0 partials
  float* pL;              // [tiles][WP*NOUT + NOUT] per-tile dW_L | db_L partials
  float* st;              // [L][tiles][32][WP][4] activated S_l, row-quad major (dW operand A)
  float* zt;              // [L][tiles][32][WP][4] Zbar_l, row-quad major (dW operand B)
};

template <typename C>
__device__ __forceinline__ size_t act_off(const WArgs& a, int l, long long tile, int q) {
  return ((size_t(l) * a.ntiles + tile) * (a.WP / 4) + q) * size_t(C::ROWS * 4);
}
template <typename C>
__device__ __forceinline__ size_t stash_off(const WArgs& a, int l, long long tile, int ub) {
  return ((size_t(l) * a.ntiles + tile) * (a.WP / C::UB) + ub) * size_t(C::STQ * C::NT);
}

// store / load a thread's [RPT][8] block into the global k-quad layout
template <typename C, typename T>
__device__ __forceinline__ void gstore_block(T* base, int ub, int rg, int g, const T (&v)[C::RPT][8]) {
  constexpr int RPT = C::RPT;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    T tmp[4 * RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) tmp[4 * r + c] = v[r][4 * h + c];
    vstore(base + size_t(ub * (C::UB / 4) + h * (C::UB / 8) + g) * (C::ROWS * 4) + rg * (4 * RPT), tmp);
  }
}
template <typename C, typename T>
__device__ __forceinline__ void gload_block(T (&v)[C::RPT][8], const T* base, int ub, int rg, int g) {
  constexpr int RPT = C::RPT;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    T tmp[4 * RPT];
    vload(tmp, base + size_t(ub * (C::UB / 4) + h * (C::UB / 8) + g) * (C::ROWS * 4) + rg * (4 * RPT));
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) v[r][4 * h + c] = tmp[4 * r + c];
  }
}

// acc[r][j] += sum_{k in chunk} A(row, k) * B[k][unit_of<UB>(g, j)], A in the
// shared k-quad layout (KC/4 quads), B row-major [KC][UB]
template <typename C, typename T>
__device__ __forceinline__ void gemm_chunk(const T* __restrict__ A, const T* __restrict__ B, int rg, int g,
                                           T (&acc)[C::RPT][8]) {
  constexpr int RPT = C::RPT, RS4 = C::RS4;
  const T* ap = A + rg * (4 * RPT);
  const T* bp = B + 4 * g;
#pragma unroll 2
  for (int kq = 0; kq < C::KC / 4; ++kq) {
    T av[4 * RPT];
    vload(av, ap + kq * RS4);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      T b0[4], b1[4];
      vload(b0, bp + (4 * kq + kk) * C::UB);
      vload(b1, bp + (4 * kq + kk) * C::UB + C::UB / 2);
#pragma unroll
      for (int r = 0; r < RPT; ++r)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[r][j] = fma(av[4 * r + kk], b0[j], acc[r][j]);
          acc[r][4 + j] = fma(av[4 * r + kk], b1[j], acc[r][4 + j]);
        }
    }
  }
}

// Full-K GEMM of one (tile, UB-unit block): A = activations of a tile from the
// global k-quad buffer `src` (WP units), B = rows [k][ub*UB..] of a row-major
// WP x WP matrix `bmat`.  Double-buffered cp.async staging.
template <typename C, typename T>
__device__ __forceinline__ void gemm_tile(const T* __restrict__ src, const T* __restrict__ bmat, int WP, int ub,
                                          T* Abuf, T* Bbuf, int tid, int rg, int g, T (&acc)[C::RPT][8]) {
  constexpr int RS4 = C::RS4, NT = C::NT, KC = C::KC, UB = C::UB, ROWS = C::ROWS;
#pragma unroll
  for (int r = 0; r < C::RPT; ++r)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[r][j] = T(0);
  const int nchunks = WP / KC;
  auto stage = [&](int c) {
    T* A = Abuf + (c & 1) * (KC / 4) * RS4;
    T* B = Bbuf + (c & 1) * KC * UB;
    constexpr int QCH = ROWS * 4 * int(sizeof(T)) / 16;  // 16-byte chunks per quad block
    for (int i = tid; i < (KC / 4) * QCH; i += NT) {
      const int qq = i / QCH, o = i % QCH;
      cp_async16(reinterpret_cast<char*>(A + qq * RS4) + 16 * o,
                 reinterpret_cast<const char*>(src + size_t(c * (KC / 4) + qq) * (ROWS * 4)) + 16 * o);
    }
    constexpr int BCH = UB * int(sizeof(T)) / 16;  // chunks per B row
    for (int i = tid; i < KC * BCH; i += NT) {
      const int kr = i / BCH, o = i % BCH;
      cp_async16(reinterpret_cast<char*>(B + kr * UB) + 16 * o,
                 reinterpret_cast<const char*>(bmat + size_t(c * KC + kr) * WP + ub * UB) + 16 * o);
    }
    cp_async_commit();
  };
  stage(0);
  for (int c = 0; c < nchunks; ++c) {
    if (c + 1 < nchunks) {
      stage(c + 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    gemm_chunk<C>(Abuf + (c & 1) * (KC / 4) * RS4, Bbuf + (c & 1) * KC * UB, rg, g, acc);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// layer 0: x -> S_0 (and stash_0)
// ---------------------------------------------------------------------------
template <typename T, int ACT, int MODE, int REG>
__global__ void __launch_bounds__(256) wide_l0_kernel(WArgs a) {
  using C = WideCfg<T, ACT, MODE, REG>;
  constexpr int RPT = C::RPT, DIN = C::DIN, NG = C::NG, NL = C::NL, LAP0 = C::LAP0, PP = C::PP;
  constexpr bool JET = C::JET;
  __shared__ T Ps[C::PPT * DIN];
  const long long tile = blockIdx.x;
  const int ub = blockIdx.y, tid = threadIdx.x, g = tid % C::G, rg = tid / C::G;
  const T* kp = static_cast<const T*>(a.kp);
  const ParamLayout pl{DIN, a.WP, C::NOUT, a.L};
  const long long p0 = tile * C::PPT, rem = a.n - p0;
  const T* pts = static_cast<const T*>(a.pts) + p0 * DIN;
  for (int i = tid; i < C::PPT * DIN; i += C::NT) Ps[i] = (i / DIN < rem) ? pts[i] : T(0);
  __syncthreads();
  T outv[RPT][8];
  T* st = static_cast<T*>(a.stash) + stash_off<C>(a, 0, tile, ub);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int u = ub * C::UB + unit_of<C::UB>(g, j);
    const T b0 = kp[pl.off_b(0) + u];
    T w0[DIN];
#pragma unroll
    for (int i = 0; i < DIN; ++i) w0[i] = kp[pl.off_w(0) + i * a.WP + u];
#pragma unroll
    for (int pr = 0; pr < PP; ++pr) {
      const int pt = JET ? rg : rg * RPT + pr;
      T zv = T(0);
#pragma unroll
      for (int i = 0; i < DIN; ++i) zv = fma(Ps[pt * DIN + i], w0[i], zv);
      zv += b0;
      T s, c;
      act_eval<ACT>(zv, s, c);
      if constexpr (JET) {
        T d1, d2;
        act_d12<ACT>(s, c, d1, d2);
        outv[0][j] = s;
#pragma unroll
        for (int i = 0; i < NG; ++i) outv[1 + i][j] = d1 * w0[i];
#pragma unroll
        for (int i = 0; i < NL; ++i) outv[1 + NG + i][j] = d2 * w0[LAP0 + i] * w0[LAP0 + i];
      } else {
        outv[pr][j] = s;
      }
      if constexpr (C::BWD) {
        st[((pr * 8 + j) * C::NST0) * C::NT + tid] = s;
        if constexpr (C::SIN) st[((pr * 8 + j) * C::NST0 + 1) * C::NT + tid] = c;
      }
    }
  }
  gstore_block<C>(static_cast<T*>(a.act) + act_off<C>(a, 0, tile, 0), ub, rg, g, outv);
}

// ---------------------------------------------------------------------------
// hidden layer forward
// ---------------------------------------------------------------------------
template <typename T, int ACT, int MODE, int REG>
__global__ void __launch_bounds__(256) wide_fwd_kernel(WArgs a, int l) {
  using C = WideCfg<T, ACT, MODE, REG>;
  constexpr int RPT = C::RPT, NG = C::NG, NL = C::NL, LAP0 = C::LAP0, NSTH = C::NSTH;
  constexpr bool JET = C::JET;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Abuf = reinterpret_cast<T*>(smem_raw);
  T* Bbuf = Abuf + 2 * (C::KC / 4) * C::RS4;
  const long long tile = blockIdx.x;
  const int ub = blockIdx.y, tid = threadIdx.x, g = tid % C::G, rg = tid / C::G;
  const T* kp = static_cast<const T*>(a.kp);
  const ParamLayout pl{C::DIN, a.WP, C::NOUT, a.L};
  T acc[RPT][8];
  gemm_tile<C>(static_cast<const T*>(a.act) + act_off<C>(a, l - 1, tile, 0), kp + pl.off_w(l), a.WP, ub, Abuf, Bbuf,
               tid, rg, g, acc);
  T* st = static_cast<T*>(a.stash) + stash_off<C>(a, l, tile, ub);
  T outv[RPT][8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int u = ub * C::UB + unit_of<C::UB>(g, j);
    const T bl = kp[pl.off_b(l) + u];
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
      if constexpr (C::BWD) {
        const int q = j * NSTH;
        st[q * C::NT + tid] = s;
        if constexpr (C::SIN) st[(q + 1) * C::NT + tid] = c;
#pragma unroll
        for (int i = 0; i < NG; ++i) st[(q + 1 + C::SIN + i) * C::NT + tid] = acc[1 + i][j];
#pragma unroll
        for (int i = 0; i < NL; ++i) st[(q + 1 + C::SIN + NG + i) * C::NT + tid] = acc[1 + NG + i][j];
      }
    } else {
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        T s, c;
        act_eval<ACT>(acc[r][j] + bl, s, c);
        outv[r][j] = s;
        if constexpr (C::BWD) {
          st[((r * 8 + j) * C::NST0) * C::NT + tid] = s;
          if constexpr (C::SIN) st[((r * 8 + j) * C::NST0 + 1) * C::NT + tid] = c;
        }
      }
    }
  }
  gstore_block<C>(static_cast<T*>(a.act) + act_off<C>(a, l, tile, 0), ub, rg, g, outv);
}

// activation adjoint of layer lp for a thread's [RPT][8] block (in place)
template <typename C, int ACT, typename T>
__device__ __forceinline__ void act_bwd_block(const WArgs& a, int lp, long long tile, int ub, int tid, int g,
                                              const T* kp, const ParamLayout& pl, T (&sb)[C::RPT][8]) {
  constexpr int RPT = C::RPT, NG = C::NG, NL = C::NL, LAP0 = C::LAP0, NSTH = C::NSTH, NST0 = C::NST0;
  const T* st = static_cast<const T*>(a.stash) + stash_off<C>(a, lp, tile, ub);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if constexpr (C::JET) {
      const int nst = lp == 0 ? NST0 : NSTH;
      const int q = j * nst;
      const T s = st[q * C::NT + tid];
      const T c = C::SIN ? st[(q + 1) * C::NT + tid] : T(0);
      T zg[NG], zl[NL > 0 ? NL : 1];
      if (lp == 0) {
        const int u = ub * C::UB + unit_of<C::UB>(g, j);
#pragma unroll
        for (int i = 0; i < NG; ++i) zg[i] = kp[pl.off_w(0) + i * a.WP + u];
#pragma unroll
        for (int i = 0; i < NL; ++i) zl[i] = T(0);
      } else {
#pragma unroll
        for (int i = 0; i < NG; ++i) zg[i] = st[(q + 1 + C::SIN + i) * C::NT + tid];
#pragma unroll
        for (int i = 0; i < NL; ++i) zl[i] = st[(q + 1 + C::SIN + NG + i) * C::NT + tid];
      }
      T d1, d2;
      act_d12<ACT>(s, c, d1, d2);
      const T d3 = act_d3<ACT>(s, c, d1, d2);
      T zv = sb[0][j] * d1;
#pragma unroll
      for (int i = 0; i < NG; ++i) zv += sb[1 + i][j] * (d2 * zg[i]);
#pragma unroll
      for (int i = 0; i < NL; ++i) {
        const T gg = zg[LAP0 + i];
        zv += sb[1 + NG + i][j] * (d3 * gg * gg + d2 * zl[i]);
      }
      T zgb[NG];
#pragma unroll
      for (int i = 0; i < NG; ++i) {
        T t = sb[1 + i][j] * d1;
        if (i >= LAP0) t += (T(2) * d2) * zg[i] * sb[1 + NG + (i - LAP0)][j];
        zgb[i] = t;
      }
#pragma unroll
      for (int i = 0; i < NL; ++i) sb[1 + NG + i][j] = sb[1 + NG + i][j] * d1;
#pragma unroll
      for (int i = 0; i < NG; ++i) sb[1 + i][j] = zgb[i];
      sb[0][j] = zv;
    } else {
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const T s = st[((r * 8 + j) * NST0) * C::NT + tid];
        const T c = C::SIN ? st[((r * 8 + j) * NST0 + 1) * C::NT + tid] : T(0);
        T d1, d2;
        act_d12<ACT>(s, c, d1, d2);
        sb[r][j] = sb[r][j] * d1;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// head: output layer, residual / MSE / outputs, and the first backward steps
// ---------------------------------------------------------------------------
template <typename T, int ACT, int MODE, int REG>
__global__ void __launch_bounds__(256) wide_head_kernel(WArgs a) {
  using C = WideCfg<T, ACT, MODE, REG>;
  constexpr int NT = C::NT, ROWS = C::ROWS, PPT = C::PPT, NOUT = C::NOUT, NVEL = C::NVEL, S = C::S;
  constexpr int NG = C::NG, LAP0 = C::LAP0, RPT = C::RPT;
  constexpr bool JET = C::JET;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* WLs = reinterpret_cast<T*>(smem_raw);          // [WP][NOUT]
  T* Ys = WLs + a.WP * NOUT;                          // [ROWS][NOUT]
  T* Ybs = Ys + ROWS * NOUT;
  double* red = reinterpret_cast<double*>(Ybs + ((ROWS * NOUT + 3) & ~3));
  const long long tile = blockIdx.x;
  const int tid = threadIdx.x, g = tid % C::G, rg = tid / C::G;
  const T* kp = static_cast<const T*>(a.kp);
  const ParamLayout pl{C::DIN, a.WP, NOUT, a.L};
  const int L = a.L;
  for (int i = tid; i < a.WP * NOUT; i += NT) WLs[i] = kp[pl.off_w(L) + i];
  __syncthreads();
  const T* H = static_cast<const T*>(a.act) + act_off<C>(a, L - 1, tile, 0);
  for (int r = tid; r < ROWS; r += NT) {
    T y[NOUT];
#pragma unroll
    for (int c = 0; c < NOUT; ++c) y[c] = T(0);
    for (int q = 0; q < a.WP / 4; ++q) {
      T xv[4];
      vload(xv, H + size_t(q) * (ROWS * 4) + r * 4);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
#pragma unroll
        for (int c = 0; c < NOUT; ++c) y[c] = fma(xv[kk], WLs[(4 * q + kk) * NOUT + c], y[c]);
    }
    const bool vrow = JET ? (r % S == 0) : true;
#pragma unroll
    for (int c = 0; c < NOUT; ++c) Ys[r * NOUT + c] = vrow ? y[c] + kp[pl.off_b(L) + c] : y[c];
  }
  __syncthreads();
  const long long p0 = tile * PPT, rem = a.n - p0;
  double lacc0 = 0.0, lacc1 = 0.0;
  if constexpr (MODE == MODE_VALUE) {
    T* out = static_cast<T*>(a.out) + p0 * NOUT;
    for (int i = tid; i < PPT * NOUT; i += NT)
      if (i / NOUT < rem) out[i] = Ys[i];
    return;
  } else if constexpr (MODE == MODE_JET) {
    T* out = static_cast<T*>(a.out) + p0 * S * NOUT;
    for (int i = tid; i < PPT * S * NOUT; i += NT)
      if (i / (S * NOUT) < rem) out[i] = Ys[i];
    return;
  } else {
    if constexpr (MODE == MODE_PDE) {
      using Rg = Regime<REG>;
      constexpr int NSP = Rg::NSP, TOFF = Rg::HAS_T, P = NVEL;
      const T inv_re = T(a.inv_re), two_coef = T(2.0 * a.coef);
      for (int pt = tid; pt < PPT; pt += NT) {
        const T* y = Ys + pt * S * NOUT;
        T* yb = Ybs + pt * S * NOUT;
        for (int i = 0; i < S * NOUT; ++i) yb[i] = T(0);
        if (pt >= rem) continue;
        auto Y = [&](int s, int c) { return y[s * NOUT + c]; };
        auto GRAD = [&](int in) { return 1 + in; };
        auto LAP = [&](int in) { return 1 + NG + (in - LAP0); };
        T r[NVEL + 1];
#pragma unroll
        for (int i = 0; i < NVEL; ++i) {
          const int xi = TOFF + i;
          T acc = T(0);
          if constexpr (Rg::HAS_T) acc = Y(GRAD(0), i);
          acc = (Rg::HAS_T ? acc + Y(GRAD(xi), P) : Y(GRAD(xi), P));
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
#pragma unroll
        for (int i = 0; i <= NVEL; ++i) lacc0 += double(r[i]) * double(r[i]);
#pragma unroll
        for (int i = 0; i < NVEL; ++i) {
          const T rb = two_coef * r[i];
          if constexpr (Rg::HAS_T) yb[GRAD(0) * NOUT + i] += rb;
          yb[GRAD(TOFF + i) * NOUT + P] += rb;
#pragma unroll
          for (int jj = 0; jj < NSP; ++jj) yb[LAP(TOFF + jj) * NOUT + i] += -inv_re * rb;
#pragma unroll
          for (int k = 0; k < NVEL; ++k) {
            yb[0 * NOUT + k] += rb * Y(GRAD(TOFF + k), i);
            yb[GRAD(TOFF + k) * NOUT + i] += rb * Y(0, k);
          }
        }
        const T rb = two_coef * r[NVEL];
#pragma unroll
        for (int k = 0; k < NVEL; ++k) yb[GRAD(TOFF + k) * NOUT + k] += rb;
      }
    } else {  // MSE
      const T two_vc = T(2.0 * a.coef), two_pc = T(2.0 * a.pcoef);
      for (int pt = tid; pt < PPT; pt += NT) {
        T* yb = Ybs + pt * NOUT;
        for (int c = 0; c < NOUT; ++c) yb[c] = T(0);
        if (pt >= rem) continue;
        const T* y = Ys + pt * NOUT;
        const T* tu = static_cast<const T*>(a.tu) + (p0 + pt) * NVEL;
#pragma unroll
        for (int c = 0; c < NVEL; ++c) {
          const T d = y[c] - tu[c];
          lacc0 += a.velw[c] * (double(d) * double(d));
          yb[c] = (two_vc * T(a.velw[c])) * d;
        }
        if (a.has_p) {
          const T d = y[NVEL] - static_cast<const T*>(a.tp)[p0 + pt];
          lacc1 += double(d) * double(d);
          yb[NVEL] = two_pc * d;
        }
      }
    }
    red[tid] = lacc0;
    red[NT + tid] = lacc1;
    __syncthreads();
    if (tid == 0) {
      double s0 = 0.0, s1 = 0.0;
      for (int i = 0; i < NT; ++i) {
        s0 += red[i];
        s1 += red[NT + i];
      }
      a.lpart[2 * tile] = s0;
      a.lpart[2 * tile + 1] = s1;
    }
    T* yout = static_cast<T*>(a.ybar) + size_t(tile) * ROWS * NOUT;
    for (int i = tid; i < ROWS * NOUT; i += NT) yout[i] = Ybs[i];
    // S-bar_{L-1} = Ybar W_L^T, then the activation adjoint of layer L-1
    T* Zout = static_cast<T*>(a.adj) + act_off<C>(a, L - 1, tile, 0);
    for (int ub = 0; ub < a.WP / C::UB; ++ub) {
      T sb[RPT][8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int u = ub * C::UB + unit_of<C::UB>(g, j);
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const int row = rg * RPT + r;
          T s = T(0);
#pragma unroll
          for (int c = 0; c < NOUT; ++c) s = fma(Ybs[row * NOUT + c], WLs[u * NOUT + c], s);
          sb[r][j] = s;
        }
      }
      act_bwd_block<C, ACT>(a, L - 1, tile, ub, tid, g, kp, pl, sb);
      gstore_block<C>(Zout, ub, rg, g, sb);
    }
  }
}

// ---------------------------------------------------------------------------
// hidden layer dX + activation adjoint of the layer below
// ---------------------------------------------------------------------------
template <typename T, int ACT, int MODE, int REG>
__global__ void __launch_bounds__(256) wide_dx_kernel(WArgs a, int l) {
  using C = WideCfg<T, ACT, MODE, REG>;
  constexpr int RPT = C::RPT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Abuf = reinterpret_cast<T*>(smem_raw);
  T* Bbuf = Abuf + 2 * (C::KC / 4) * C::RS4;
  const long long tile = blockIdx.x;
  const int ub = blockIdx.y, tid = threadIdx.x, g = tid % C::G, rg = tid / C::G;
  const T* kp = static_cast<const T*>(a.kp);
  const ParamLayout pl{C::DIN, a.WP, C::NOUT, a.L};
  T acc[RPT][8];
  gemm_tile<C>(static_cast<const T*>(a.adj) + act_off<C>(a, l, tile, 0), kp + pl.off_wt(l), a.WP, ub, Abuf, Bbuf,
               tid, rg, g, acc);
  act_bwd_block<C, ACT>(a, l - 1, tile, ub, tid, g, kp, pl, acc);
  gstore_block<C>(static_cast<T*>(a.adj) + act_off<C>(a, l - 1, tile, 0), ub, rg, g, acc);
}

// ---------------------------------------------------------------------------
// dW_l = sum over rows of S_{l-1}^T Zbar_l (64 x 64 block per CTA, split rows)
// ---------------------------------------------------------------------------
template <typename T, int ACT, int MODE, int REG>
__global__ void __launch_bounds__(256) wide_dw_kernel(WArgs a, int l) {
  using C = WideCfg<T, ACT, MODE, REG>;
  constexpr int ROWS = C::ROWS, SPLIT = C::DW_SPLIT, FLUSH = 8;
  constexpr int RS4C = C::RS4C, RCH = C::RCH, NRC = C::NRC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Hs = reinterpret_cast<T*>(smem_raw);  // 16 quads x RCH rows
  T* Zs = Hs + 16 * RS4C;
  static_assert(2 * 16 * RS4C >= (SPLIT - 1) * 4096, "combine scratch must fit in the staging buffers");
  const int kb = blockIdx.x, ubk = blockIdx.y, ks = blockIdx.z;
  const int tid = threadIdx.x, ut = tid % 8, kt = (tid / 8) % 8, rs = tid / 64;
  const ParamLayout pl{C::DIN, a.WP, C::NOUT, a.L};
  double* gp = a.gpart + size_t(ks) * a.np_pad;
  T acc[8][8];
  T db = T(0);
  auto zero = [&]() {
#pragma unroll
    for (int x = 0; x < 8; ++x)
#pragma unroll
      for (int y = 0; y < 8; ++y) acc[x][y] = T(0);
    db = T(0);
  };
  auto kidx = [&](int x) { return kb * 64 + (x < 4 ? 4 * kt + x : 4 * (kt + 8) + (x - 4)); };
  auto uidx = [&](int y) { return ubk * 64 + (y < 4 ? 4 * ut + y : 4 * (ut + 8) + (y - 4)); };
  auto flush = [&]() {
    // combine the SPLIT row-range partials in a fixed order, then one red.add
    __syncthreads();
    T* scratch = Hs;
    if (rs > 0) {
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        vstore(scratch + (rs - 1) * 4096 + (kidx(x) - kb * 64) * 64 + 4 * ut, *reinterpret_cast<const T(*)[4]>(&acc[x][0]));
        vstore(scratch + (rs - 1) * 4096 + (kidx(x) - kb * 64) * 64 + 32 + 4 * ut,
               *reinterpret_cast<const T(*)[4]>(&acc[x][4]));
      }
    }
    __syncthreads();
    if (rs == 0) {
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        for (int q = 1; q < SPLIT; ++q) {
          const T* src = scratch + (q - 1) * 4096 + (kidx(x) - kb * 64) * 64;
          T a4[4], b4[4];
          vload(a4, src + 4 * ut);
          vload(b4, src + 32 + 4 * ut);
#pragma unroll
          for (int y = 0; y < 4; ++y) {
            acc[x][y] += a4[y];
            acc[x][4 + y] += b4[y];
          }
        }
#pragma unroll
        for (int y = 0; y < 8; ++y) red_add(gp + pl.off_w(l) + size_t(kidx(x)) * a.WP + uidx(y), double(acc[x][y]));
      }
    }
    if (kb == 0 && tid < 64) red_add(gp + pl.off_b(l) + ubk * 64 + tid, double(db));
    __syncthreads();
    zero();
  };
  zero();
  int since = 0;
  for (long long t = ks; t < a.ntiles; t += gridDim.z) {
    const T* hsrc = static_cast<const T*>(a.act) + act_off<C>(a, l - 1, t, kb * 16);
    const T* zsrc = static_cast<const T*>(a.adj) + act_off<C>(a, l, t, ubk * 16);
#pragma unroll 1
    for (int ch = 0; ch < NRC; ++ch) {
      constexpr int QCH = RCH * 4 * int(sizeof(T)) / 16;  // 16-byte chunks of one quad's row chunk
      for (int i = tid; i < 16 * QCH; i += 256) {
        const int qq = i / QCH, o = i % QCH;
        const size_t go = size_t(qq) * (ROWS * 4) + size_t(ch) * RCH * 4;
        cp_async16(reinterpret_cast<char*>(Hs + qq * RS4C) + 16 * o, reinterpret_cast<const char*>(hsrc + go) + 16 * o);
        cp_async16(reinterpret_cast<char*>(Zs + qq * RS4C) + 16 * o, reinterpret_cast<const char*>(zsrc + go) + 16 * o);
      }
      cp_async_commit();
      cp_async_wait_all();
      __syncthreads();
      // rows rs, rs + SPLIT, ... of this chunk (strided: balanced across chunks)
      const T* x0 = Hs + kt * RS4C;
      const T* x1 = Hs + (kt + 8) * RS4C;
      const T* z0 = Zs + ut * RS4C;
      const T* z1 = Zs + (ut + 8) * RS4C;
#pragma unroll 2
      for (int r = rs; r < RCH; r += SPLIT) {
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
      if (kb == 0 && tid < 64) {
        const T* zq = Zs + (tid / 4) * RS4C + (tid % 4);
        for (int pt = 0; pt < C::PPT; ++pt) {
          const int row = (C::JET ? pt * C::S : pt) - ch * RCH;  // value rows in this chunk
          if (row >= 0 && row < RCH) db += zq[4 * row];
        }
      }
      __syncthreads();
    }
    if (++since == FLUSH) {
      flush();
      since = 0;
    }
  }
  if (since) flush();
}

// dW_L, db_L from S_{L-1} and Ybar
template <typename T, int ACT, int MODE, int REG>
__global__ void __launch_bounds__(256) wide_dwL_kernel(WArgs a) {
  using C = WideCfg<T, ACT, MODE, REG>;
  constexpr int NOUT = C::NOUT, ROWS = C::ROWS;
  const int ks = blockIdx.x, tid = threadIdx.x;
  const ParamLayout pl{C::DIN, a.WP, NOUT, a.L};
  double* gp = a.gpart + size_t(ks) * a.np_pad;
  const int q = tid;  // one k-quad per thread (WP/4 <= 256 quads)
  const bool active = q < a.WP / 4;
  T acc[4][NOUT];
  T db[NOUT];
#pragma unroll
  for (int c = 0; c < NOUT; ++c) {
    db[c] = T(0);
#pragma unroll
    for (int x = 0; x < 4; ++x) acc[x][c] = T(0);
  }
  int since = 0;
  auto flush = [&]() {
    if (active)
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int c = 0; c < NOUT; ++c) {
          red_add(gp + pl.off_w(a.L) + (4 * q + x) * NOUT + c, double(acc[x][c]));
          acc[x][c] = T(0);
        }
    if (tid == 0)
#pragma unroll
      for (int c = 0; c < NOUT; ++c) {
        red_add(gp + pl.off_b(a.L) + c, double(db[c]));
        db[c] = T(0);
      }
  };
  for (long long t = ks; t < a.ntiles; t += gridDim.x) {
    const T* yb = static_cast<const T*>(a.ybar) + size_t(t) * ROWS * NOUT;
    if (active) {
      const T* H = static_cast<const T*>(a.act) + act_off<C>(a, a.L - 1, t, q);
      for (int r = 0; r < ROWS; ++r) {
        T hv[4];
        vload(hv, H + 4 * r);
#pragma unroll
        for (int c = 0; c < NOUT; ++c) {
          const T y = yb[r * NOUT + c];
#pragma unroll
          for (int x = 0; x < 4; ++x) acc[x][c] = fma(hv[x], y, acc[x][c]);
        }
      }
    }
    if (tid == 0)
      for (int pt = 0; pt < C::PPT; ++pt)
#pragma unroll
        for (int c = 0; c < NOUT; ++c) db[c] += yb[(C::JET ? pt * C::S : pt) * NOUT + c];
    if (++since == 8) {
      flush();
      since = 0;
    }
  }
  if (since) flush();
}

// dW_0, db_0 from the points and Zbar_0 (jet modes add the unit derivative blocks)
template <typename T, int ACT, int MODE, int REG>
__global__ void __launch_bounds__(256) wide_dw0_kernel(WArgs a) {
  using C = WideCfg<T, ACT, MODE, REG>;
  constexpr int DIN = C::DIN, ROWS = C::ROWS;
  const int ks = blockIdx.x, u = threadIdx.x + blockIdx.y * 256;
  const ParamLayout pl{DIN, a.WP, C::NOUT, a.L};
  double* gp = a.gpart + size_t(ks) * a.np_pad;
  const bool active = u < a.WP;
  T acc[DIN + 1];
#pragma unroll
  for (int j = 0; j <= DIN; ++j) acc[j] = T(0);
  int since = 0;
  auto flush = [&]() {
    if (!active) return;
#pragma unroll
    for (int j = 0; j < DIN; ++j) {
      red_add(gp + pl.off_w(0) + j * a.WP + u, double(acc[j]));
      acc[j] = T(0);
    }
    red_add(gp + pl.off_b(0) + u, double(acc[DIN]));
    acc[DIN] = T(0);
  };
  for (long long t = ks; t < a.ntiles && active; t += gridDim.x) {
    const T* Z = static_cast<const T*>(a.adj) + act_off<C>(a, 0, t, u / 4) + (u % 4);
    const long long p0 = t * C::PPT;
    const T* pts = static_cast<const T*>(a.pts);
    for (int pt = 0; pt < C::PPT && p0 + pt < a.n; ++pt) {
      const int row = C::JET ? pt * C::S : pt;
      const T zv = Z[4 * row];
#pragma unroll
      for (int j = 0; j < DIN; ++j) {
        acc[j] = fma(pts[(p0 + pt) * DIN + j], zv, acc[j]);
        if constexpr (C::JET) acc[j] += Z[4 * (row + 1 + j)];
      }
      acc[DIN] += zv;
    }
    if (++since == 8) {
      flush();
      since = 0;
    }
  }
  if (since) flush();
}

}  // namespace fr
