// Tensor-core (tcgen05, TF32) layer-wise kernels for wide experts.
//
// Same chain as the SIMT wide path (wide_kernel.cuh) but every hidden-layer
// contraction -- forward S_{l-1} W_l, adjoint Zbar_l W_l^T and weight gradient
// S_{l-1}^T Zbar_l -- runs as 128 x NB x 8 tcgen05.mma.kind::tf32 steps with the
// accumulator in TMEM.  All operands are K-major SWIZZLE_NONE UMMA tiles
// (TF32 MN-major descriptors read zeros on sm_100a, see tools/tc_layout_probe.py).
//
// Tile geometry.  A tile is one 128-row MMA block packing PPT = 128 / S
// points x S jet streams (rows p*S+s) plus 128 - PPT*S pad rows (2D PDE: 21
// points and 2 pad rows).  Pad rows are never read by the per-point code; the
// weight-gradient operands zero them before they reach the tensor core.
//
// HBM buffers (fp32, k-quad layout [layer][tile][WP/4][128][4], one quad of a
// tile = 2 KB contiguous = a K-major 128 x 4 operand slab):
//   Z    pre-activation jets of layers 1..L-1 (layer 0 is recomputed from the
//        points on the fly: z_v = x W0 + b0, z_g = W0 rows, z_l = 0)
//   Zbar their adjoints, layers 1..L-1 (Zbar_0 only feeds dW_0, which the
//        layer-1 adjoint kernel reduces per tile without storing it)
//   p0 / pL per-tile dW_0|db_0 and dW_L|db_L partials, reduced over tiles in a
//        fixed order by tcw_partials_kernel
// The activation sigma(Z) is applied by the CONSUMER (the next layer's operand
// staging, the head, the dW staging), so the forward writes only Z.
//
// Data movement: every operand slab is fetched with 1-D bulk async copies
// (cp.async.bulk, TMA engine) issued by one thread into a multi-stage
// shared-memory ring with mbarrier transaction counts; the tensor core frees a
// stage through tcgen05.commit on the stage's "empty" barrier.
#pragma once
#include "tcgen05.cuh"
#include "tma.cuh"
#include "wide_kernel.cuh"

namespace fr {

constexpr int TC_NS = 4;   // fwd / dx ring stages
#ifndef FR_TC_HEAD_NS
#define FR_TC_HEAD_NS 2  // 2 stages -> more CTAs per SM: E head 3.37 -> 3.04, D150 1.12 -> 1.01 ms (4: the old ring)
#endif
constexpr int TC_HEAD_NS = FR_TC_HEAD_NS;  // head ring stages
constexpr int TC_KC = 16;  // K depth of one stage (4 unit quads)

template <int ACT, int MODE, int REG>
struct TcCfg {
  using R = Regime<REG>;
  using St = Streams<MODE, REG>;
  static constexpr int DIN = R::DIN, NOUT = R::NOUT, NVEL = R::NVEL;
  static constexpr int S = St::S, NG = St::NG, NL = St::NL, LAP0 = St::LAP0;
  static constexpr bool JET = St::JET;
  static constexpr int NT = 128;              // fwd / dx / head CTAs (one thread per TMEM lane)
  static constexpr int DW_NT = 320;           // dW CTAs (loader, MMA, 8 drain / db warps)
  // a tile packs PPT = 128 / S points' jet rows (row p * S + s); rows >= VRT
  // are pad rows (2D PDE: 21 points, rows 126 / 127; 3D: 16 points, none)
  static constexpr int PPT = 128 / S;         // points per tile
  static constexpr int VRT = PPT * S;         // valid rows of a tile
  static constexpr int ITEMS = PPT * 4;       // (point, unit quad) items of one 16-deep chunk
  static constexpr int TPP = ITEMS <= NT ? 4 : 1;  // threads holding partial sums of one point (head)
  __host__ __device__ static constexpr int row0(int pt) { return pt * S; }
  // a value row (the point's z_v: gets the bias, feeds db)
  __host__ __device__ static constexpr bool vrow(int r) { return r < VRT && r % S == 0; }
  __host__ __device__ static constexpr size_t stage_floats(int NB) { return 2048 + size_t(NB) * 16; }
  // persistent forward: the activation slab's unit quads are FQS floats apart
  // (128 rows x 4 + 4): quad q shifts every row by 4 banks, which makes the St
  // row-quad gather conflict-free and, with fwd_item(), the jet activation's
  // 16-byte loads / stores nearly so (tools/bank_model.py)
  static constexpr int FQS = 516;
  __host__ __device__ static constexpr size_t fwdp_stage_floats(int NB) { return 4 * FQS + size_t(NB) * 16; }
  // (point, unit quad) of activation item i (2D PDE, S = 6): each 8-lane phase
  // takes 4 consecutive points x 2 quads, whose 16-byte rows then fall in 8
  // distinct bank groups (rows 6p mod 8 = {0,6,4,2} + 6 * 4k, quads +1 with the
  // FQS padding); the 21st point's 4 quads fill the last phase
  static constexpr bool FWD_MAP = (S == 6 && PPT == 21 && ITEMS == 84);
  __device__ static void fwd_item(int i, int& pt, int& kq) {
    if constexpr (FWD_MAP) {
      if (i < 80) {
        const int ph = i >> 3, p8 = i & 7;
        pt = 4 * (ph >> 1) + (p8 >> 1);
        kq = 2 * (ph & 1) + (p8 & 1);
      } else {
        pt = 20;
        kq = i - 80;
      }
    } else {
      pt = i % PPT;
      kq = i / PPT;
    }
  }
  // inverse of fwd_item: the item index that holds (pt, kq)
  __device__ static int item_of(int pt, int kq) {
    if constexpr (FWD_MAP) {
      return pt < 20 ? 8 * (2 * (pt >> 2) + (kq >> 1)) + 2 * (pt & 3) + (kq & 1) : 80 + kq;
    } else {
      return kq * PPT + pt;
    }
  }
  __host__ __device__ static size_t gemm_smem(int NB) { return sizeof(float) * TC_NS * stage_floats(NB); }
  __host__ __device__ static size_t dw_stage_bytes(int WP, int NB) { return size_t(WP + NB) * 128; }
  // head dW_L partials: [pt][kq][j][o] for per-unit items, else [j][o][item]
  // rows of HRS = ITEMS + 1 floats (lane-contiguous stores, odd row stride)
  static constexpr int HRS = ITEMS + 1;
  // per-unit items (3D): [16 units][NOUT][point], point rows RSP apart so the 8
  // points x 4 units of a warp's stores hit 32 distinct banks
  static constexpr int RSP = PPT + 2;
  static constexpr int HEAD_RED = 4 * NOUT * HRS > 16 * NOUT * RSP ? 4 * NOUT * HRS : 16 * NOUT * RSP;
  // Y partial rows: SN + 1 floats apart (a stride of SN = 32 put every lane's
  // stores in one bank)
  static constexpr int YPS = S * NOUT + 1;
  __host__ __device__ static size_t head_smem(int WP) {
    return sizeof(double) * 2 * NT +
           sizeof(float) * size_t(TC_HEAD_NS * 4 * FQS + WP * NOUT + NT * YPS + 2 * PPT * S * NOUT + HEAD_RED);
  }
};

__device__ __forceinline__ size_t tc_off(const WArgs& a, int l, long long tile, int q) {
  return ((size_t(l) * a.ntiles + tile) * (a.WP / 4) + q) * 512;
}

// layer-0 pre-activation jets of point p (global index), units 4q..4q+3
template <class C>
__device__ __forceinline__ void tc_z0(const WArgs& a, const float* __restrict__ kp, const ParamLayout& pl,
                                      long long p, int q, float (&z)[C::S][4]) {
  const float* pts = static_cast<const float*>(a.pts);
  float x[C::DIN];
#pragma unroll
  for (int i = 0; i < C::DIN; ++i) x[i] = p < a.n ? pts[p * C::DIN + i] : 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int u = 4 * q + j;
    float zv = 0.f;
#pragma unroll
    for (int i = 0; i < C::DIN; ++i) zv = fmaf(x[i], kp[pl.off_w(0) + i * a.WK + u], zv);
    z[0][j] = zv + kp[pl.off_b(0) + u];
    if constexpr (C::JET) {
#pragma unroll
      for (int i = 0; i < C::NG; ++i) z[1 + i][j] = kp[pl.off_w(0) + i * a.WK + u];
#pragma unroll
      for (int i = 0; i < C::NL; ++i) z[1 + C::NG + i][j] = 0.f;
    }
  }
}

// layer-0 pre-activation jet of point p (global index), unit u
template <class C>
__device__ __forceinline__ void tc_z0u(const WArgs& a, const float* __restrict__ kp, const ParamLayout& pl,
                                       long long p, int u, float (&z)[C::S]) {
  const float* pts = static_cast<const float*>(a.pts);
  float zv = 0.f;
#pragma unroll
  for (int i = 0; i < C::DIN; ++i) zv = fmaf(p < a.n ? pts[p * C::DIN + i] : 0.f, kp[pl.off_w(0) + i * a.WK + u], zv);
  z[0] = zv + kp[pl.off_b(0) + u];
  if constexpr (C::JET) {
#pragma unroll
    for (int i = 0; i < C::NG; ++i) z[1 + i] = kp[pl.off_w(0) + i * a.WK + u];
#pragma unroll
    for (int i = 0; i < C::NL; ++i) z[1 + C::NG + i] = 0.f;
  }
}

// per-unit item split of the persistent kernels' activation steps: when the
// (point, unit quad) items of a 16-unit chunk fill at most half of the 128
// threads (3D jets: 64 items), each thread takes single (point, quad, unit)
// items instead (measured: E -12% epoch time).  For the 2D jets' 80 items the
// 3-round split with scalar shared loads pays only in the sin adjoint (D150
// dx -2.8%; forward +2%, tanh adjoint +7%)
template <class C, bool ADJ = false, int ACT = ACT_TANH>
struct TcUnit {
  static constexpr bool ON = 2 * C::ITEMS <= 128 || (ADJ && ACT == ACT_SIN && (C::ITEMS % 128) != 0);
  static constexpr int N = ON ? C::ITEMS * 4 : C::ITEMS;
};
template <class C, int QS = 512>
__device__ __forceinline__ void slab_load1(float (&v)[C::S], const float* slab, int pt, int kq, int j) {
  const float* b = slab + kq * QS + C::row0(pt) * 4 + j;
#pragma unroll
  for (int s = 0; s < C::S; ++s) v[s] = b[4 * s];
}
template <class C, int QS = 512>
__device__ __forceinline__ void slab_store1(float* slab, int pt, int kq, int j, const float (&v)[C::S]) {
  float* b = slab + kq * QS + C::row0(pt) * 4 + j;
#pragma unroll
  for (int s = 0; s < C::S; ++s) b[4 * s] = v[s];
}

// v[s] <- v[s ^ x] (S a power of two, 0 <= x < S) with conditional swaps
template <int S>
__device__ __forceinline__ void xperm(float (&v)[S], int x) {
#pragma unroll
  for (int b = 1; b < S; b <<= 1) {
    const bool f = (x & b) != 0;
#pragma unroll
    for (int k = 0; k < S; ++k)
      if (!(k & b)) {
        const float t0 = v[k], t1 = v[k | b];
        v[k] = f ? t1 : t0;
        v[k | b] = f ? t0 : t1;
      }
  }
}
// slab_load1 / slab_store1 with the stream order XOR-permuted by x: lanes that
// hold different points of one 8-stream (3D) tile touch different banks on
// every instruction (a point's 8 rows are 128 bytes: the same banks otherwise)
template <class C, int QS = 512>
__device__ __forceinline__ void slab_load1x(float (&v)[C::S], const float* slab, int pt, int kq, int j, int x) {
  if constexpr (C::S == 8) {
    const float* b = slab + kq * QS + C::row0(pt) * 4 + j;
#pragma unroll
    for (int s = 0; s < 8; ++s) v[s] = b[4 * (s ^ x)];
    xperm<8>(v, x);
  } else {
    slab_load1<C, QS>(v, slab, pt, kq, j);
  }
}
template <class C, int QS = 512>
__device__ __forceinline__ void slab_store1x(float* slab, int pt, int kq, int j, const float (&v)[C::S], int x) {
  if constexpr (C::S == 8) {
    float w[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) w[s] = v[s];
    xperm<8>(w, x);
    float* b = slab + kq * QS + C::row0(pt) * 4 + j;
#pragma unroll
    for (int s = 0; s < 8; ++s) b[4 * (s ^ x)] = w[s];
  } else {
    slab_store1<C, QS>(slab, pt, kq, j, v);
  }
}

// jet activation of one point / unit: s = sigma applied to the stacked jet
template <class C, int ACT>
__device__ __forceinline__ void tc_act1(const float (&z)[C::S], float (&s)[C::S]) {
  float sv, cv, d1, d2;
  act_eval<ACT>(z[0], sv, cv);
  s[0] = sv;
  if constexpr (C::JET) {
    act_d12<ACT>(sv, cv, d1, d2);
#pragma unroll
    for (int i = 0; i < C::NG; ++i) s[1 + i] = d1 * z[1 + i];
#pragma unroll
    for (int i = 0; i < C::NL; ++i) {
      const float zg = z[1 + C::LAP0 + i];
      s[1 + C::NG + i] = d2 * zg * zg + d1 * z[1 + C::NG + i];
    }
  }
}

// activation adjoint of one point / unit (in place: sb = S-bar -> Z-bar);
// also returns the forward activation in sa (for the weight gradient)
template <class C, int ACT>
__device__ __forceinline__ void tc_act_bwd1(const float (&z)[C::S], float (&sb)[C::S], float (&sa)[C::S]) {
  constexpr int NG = C::NG, NL = C::NL, LAP0 = C::LAP0;
  float s, c, d1, d2;
  act_eval<ACT>(z[0], s, c);
  act_d12<ACT>(s, c, d1, d2);
  sa[0] = s;
  if constexpr (C::JET) {
#pragma unroll
    for (int i = 0; i < NG; ++i) sa[1 + i] = d1 * z[1 + i];
#pragma unroll
    for (int i = 0; i < NL; ++i) {
      const float zg = z[1 + LAP0 + i];
      sa[1 + NG + i] = d2 * zg * zg + d1 * z[1 + NG + i];
    }
    const float d3 = act_d3<ACT>(s, c, d1, d2);
    float zv = sb[0] * d1;
#pragma unroll
    for (int i = 0; i < NG; ++i) zv += sb[1 + i] * (d2 * z[1 + i]);
#pragma unroll
    for (int i = 0; i < NL; ++i) {
      const float gg = z[1 + LAP0 + i];
      zv += sb[1 + NG + i] * (d3 * gg * gg + d2 * z[1 + NG + i]);
    }
    float zgb[NG];
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      float t = sb[1 + i] * d1;
      if (i >= LAP0) t += (2.f * d2) * z[1 + i] * sb[1 + NG + (i - LAP0)];
      zgb[i] = t;
    }
#pragma unroll
    for (int i = 0; i < NL; ++i) sb[1 + NG + i] = sb[1 + NG + i] * d1;
#pragma unroll
    for (int i = 0; i < NG; ++i) sb[1 + i] = zgb[i];
    sb[0] = zv;
  } else {
    sb[0] = sb[0] * d1;
  }
}

// the S rows x 4 units of item (pt, kq) in a [kq][128][4] slab
template <class C, int QS = 512>
__device__ __forceinline__ void slab_load(float (&v)[C::S][4], const float* slab, int pt, int kq) {
  const float* b = slab + kq * QS + C::row0(pt) * 4;
#pragma unroll
  for (int s = 0; s < C::S; ++s) vload(v[s], b + 4 * s);
}
template <class C, int QS = 512>
__device__ __forceinline__ void slab_store(float* slab, int pt, int kq, const float (&v)[C::S][4]) {
  float* b = slab + kq * QS + C::row0(pt) * 4;
#pragma unroll
  for (int s = 0; s < C::S; ++s) vstore(b + 4 * s, v[s]);
}
template <class C>
__device__ __forceinline__ void col(const float (&v)[C::S][4], int j, float (&o)[C::S]) {
#pragma unroll
  for (int s = 0; s < C::S; ++s) o[s] = v[s][j];
}

__device__ __forceinline__ size_t tc_toff(const WArgs& a, int l, long long tile) {
  return (size_t(l) * a.ntiles + tile) * size_t(a.WP) * 128;
}

// row-quad-major copy of a [4 kq][128][4] slab (units k0..k0+15) into a tile's
// [32 rq][WP][4] buffer (128 threads).  Lane = (row quad, unit): it gathers
// its unit's 4 rows with scalar shared loads and writes one 16-byte store, so
// 16 lanes cover a contiguous 256-byte run.  Pad rows are written as zeros so
// they contribute nothing to the weight gradients.
template <class C, int QS = 512>
__device__ __forceinline__ void slab_store_t(const float* slab, float* dstT, int WP, int k0, int tid) {
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int item = it * 128 + tid;
    const int rq = item >> 4, k16 = item & 15;
    const float* src = slab + (k16 >> 2) * QS + (4 * rq) * 4 + (k16 & 3);
    float v[4];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const float x = src[rr * 4];
      v[rr] = (4 * rq + rr) < C::VRT ? x : 0.f;
    }
    *reinterpret_cast<float4*>(dstT + (size_t(rq) * WP + k0 + k16) * 4) = make_float4(v[0], v[1], v[2], v[3]);
  }
}
// plain copy of a [4 kq][128][4] slab (quads QS floats apart) to its
// (contiguous 8 KB) place in HBM
template <int QS = 512>
__device__ __forceinline__ void slab_copy_out(const float* slab, float* dst, int tid) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
    reinterpret_cast<float4*>(dst + 512 * i)[tid] = reinterpret_cast<const float4*>(slab + QS * i)[tid];
}

// 2 K-steps (16 deep) of A[kq][MA][4] x B[kq][NB][4]
__device__ __forceinline__ void tc_mma16(uint32_t tmem, const float* A, int MA, const float* B, int NB, uint32_t idesc,
                                         bool first) {
#pragma unroll
  for (int kk = 0; kk < 2; ++kk)
    tc::mma_tf32(tmem, tc::desc(A + kk * 8 * MA, MA * 16, 128), tc::desc(B + kk * 8 * NB, NB * 16, 128), idesc,
                 (!first || kk) ? 1u : 0u);
}

// weight operand slab of chunk c (16 K values x NB units, contiguous NB*64 B)
__device__ __forceinline__ const float* tc_wslab(const WArgs& a, long long base, int l, int nb, int c) {
  const int nnb = a.WP / a.nb, nch = a.WP / TC_KC;
  return static_cast<const float*>(a.kp) + base + ((size_t(l - 1) * nnb + nb) * nch + c) * size_t(a.nb) * 16;
}

// ---------------------------------------------------------------------------
// forward, hidden layer l >= 1: Z_l = sigma(Z_{l-1}) W_l + b_l
// grid (tiles, WP/NB), 320 threads, warp specialised over a TC_NS-stage ring
// (stage = Z_{l-1} slab of 4 unit quads x 128 rows + W_l^T slab NB x 16):
//   warp 4      loader: bulk copies once the stage's MMA and St store are done
//   warps 0..3  jet activation in place (smem), then the TMEM -> Z_l epilogue
//   warp 5      MMA issuer (2 K-steps per stage), commit frees the stage
//   warps 6..9  S_{l-1} row-quad-major copy for dW (N block 0 only)
// ---------------------------------------------------------------------------
constexpr int TC_FWD_NT = 320;
template <int ACT, int MODE, int REG>
__global__ void __launch_bounds__(TC_FWD_NT) tcw_fwd_kernel(WArgs a, int l) {
  using C = TcCfg<ACT, MODE, REG>;
  extern __shared__ __align__(128) unsigned char tc_smem[];
  float* ring = reinterpret_cast<float*>(tc_smem);
  __shared__ __align__(8) uint64_t full[TC_NS], actd[TC_NS], mmad[TC_NS], std_[TC_NS];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long tile = blockIdx.x;
  const int nb = blockIdx.y, NB = a.nb, n0 = nb * NB;
  const float* kp = static_cast<const float*>(a.kp);
  const ParamLayout pl{C::DIN, a.WK, C::NOUT, a.L};
  if (tid == 0)
    for (int i = 0; i < TC_NS; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&actd[i], 4);
      tc::mbar_init(&std_[i], 4);
    }
  const uint32_t tmem = tc_setup<256>(&tslot, mmad, TC_NS);
  const int nch = a.WP / TC_KC;
  const bool virt = (l == 1);
  const size_t SF = C::stage_floats(NB);
  auto arrive = [&](uint64_t* bar) {
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
  };
  if (warp == 4) {
    if (lane == 0) {
      const float* zsrc = static_cast<const float*>(a.act) + (virt ? 0 : tc_off(a, l - 1, tile, 0));
      for (int c = 0; c < nch; ++c) {
        const int s = c % TC_NS;
        if (c >= TC_NS) {
          const uint32_t ph = ((c - TC_NS) / TC_NS) & 1;
          tc::mbar_wait(&mmad[s], ph);
          tc::mbar_wait(&std_[s], ph);
        }
        float* st = ring + s * SF;
        tc::mbar_expect_tx(&full[s], NB * 64 + (virt ? 0 : 8192));
        tc::bulk_g2s(st + 2048, tc_wslab(a, a.tcw_f, l, nb, c), NB * 64, &full[s]);
        if (!virt) tc::bulk_g2s(st, zsrc + size_t(c) * 2048, 8192, &full[s]);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_tf32(128, NB);
      for (int c = 0; c < nch; ++c) {
        const int s = c % TC_NS;
        float* A = ring + s * SF;
        tc::mbar_wait(&actd[s], (c / TC_NS) & 1);
        tc::fence_after();
        tc_mma16(tmem, A, 128, A + 2048, NB, idesc, c == 0);
        tc::mma_commit(&mmad[s]);
      }
    }
  } else if (warp >= 6) {
    const int t = tid - 192;
    for (int c = 0; c < nch; ++c) {
      const int s = c % TC_NS;
      tc::mbar_wait(&actd[s], (c / TC_NS) & 1);
      if (nb == 0 && a.st) slab_store_t<C>(ring + s * SF, a.st + tc_toff(a, l - 1, tile), a.WP, 16 * c, t);
      arrive(&std_[s]);
    }
  } else {
    for (int c = 0; c < nch; ++c) {
      const int s = c % TC_NS;
      float* A = ring + s * SF;
      tc::mbar_wait(&full[s], (c / TC_NS) & 1);
      for (int i = tid; i < C::ITEMS; i += 128) {
        const int pt = i % C::PPT, kq = i / C::PPT;
        float z[C::S][4], sv[C::S][4];
        if (virt) tc_z0<C>(a, kp, pl, tile * C::PPT + pt, 4 * c + kq, z);
        else slab_load<C>(z, A, pt, kq);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float zz[C::S], ss[C::S];
          col<C>(z, j, zz);
          tc_act1<C, ACT>(zz, ss);
#pragma unroll
          for (int k = 0; k < C::S; ++k) sv[k][j] = ss[k];
        }
        slab_store<C>(A, pt, kq, sv);
      }
      tc::fence_proxy_async();
      arrive(&actd[s]);
    }
    // epilogue: Z_l = D + b on value rows
    tc::mbar_wait(&mmad[(nch - 1) % TC_NS], ((nch - 1) / TC_NS) & 1);
    tc::fence_after();
    const int r = warp * 32 + lane;
    const bool vrow = C::vrow(r);
    float* Zo = static_cast<float*>(a.act) + tc_off(a, l, tile, n0 / 4) + r * 4;
    const float* bl = kp + pl.off_b(l) + n0;
    for (int c0 = 0; c0 < NB; c0 += 16) {
      float v[16];
      tc::tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + c0, v);
      if (vrow)
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] += bl[c0 + i];
#pragma unroll
      for (int h = 0; h < 4; ++h)
        *reinterpret_cast<float4*>(Zo + size_t(c0 / 4 + h) * 512) =
            make_float4(v[4 * h], v[4 * h + 1], v[4 * h + 2], v[4 * h + 3]);
    }
  }
  tc_teardown<256>(tmem);
}

// ---------------------------------------------------------------------------
// persistent forward, hidden layer l >= 1 (same math as tcw_fwd_kernel).
// One CTA per SM walks the (tile, N block) items grid-strided, so the HBM
// stream never drains at tile boundaries: an 8-stage ring, and two TMEM
// accumulators (2 x 256 columns) so the MMAs of item i+1 run while dedicated
// epilogue warps drain item i to HBM.
//   warps 0..3   jet activation in place            warp 4  bulk-copy loader
//   warp 5       MMA issuer                          warps 6..9  S_{l-1} row-quad-major copy
//   warps 10..13 epilogue TMEM -> Z_l (+ b on value rows), frees the accumulator
// Stage s and accumulator b phases follow the CTA-local chunk / item counters.
// ---------------------------------------------------------------------------
constexpr int TCP_NS = 8;
constexpr int TCP_FWD_NT = 576;
template <int ACT, int MODE, int REG>
__global__ void __launch_bounds__(TCP_FWD_NT, 1) tcw_fwdp_kernel(WArgs a, int l) {
  using C = TcCfg<ACT, MODE, REG>;
  extern __shared__ __align__(128) unsigned char tc_smem[];
  float* ring = reinterpret_cast<float*>(tc_smem);
  __shared__ __align__(8) uint64_t full[TCP_NS], actd[TCP_NS], mmad[TCP_NS], std_[TCP_NS], accf[2], acce[2];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NB = a.nb, nnb = a.WP / NB;
  const long long nitems = (long long)a.ntiles * nnb;
  const float* kp = static_cast<const float*>(a.kp);
  const ParamLayout pl{C::DIN, a.WK, C::NOUT, a.L};
  if (tid == 0) {
    for (int i = 0; i < TCP_NS; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&actd[i], 4);
      tc::mbar_init(&std_[i], 4);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&accf[b], 1);
      tc::mbar_init(&acce[b], 4);
    }
  }
  const uint32_t tmem = tc_setup<512>(&tslot, mmad, TCP_NS);
  const int nch = a.WP / TC_KC;
  const bool virt = (l == 1);
  constexpr int QS = C::FQS;
  const size_t SF = C::fwdp_stage_floats(NB);
  auto arrive = [&](uint64_t* bar) {
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
  };
  if (warp == 8) {
    if (lane == 0) {
      long long g = 0;
      for (long long w = blockIdx.x; w < nitems; w += gridDim.x) {
        const long long tile = w / nnb;
        const int nb = int(w % nnb);
        const float* zsrc = static_cast<const float*>(a.act) + (virt ? 0 : tc_off(a, l - 1, tile, 0));
        for (int c = 0; c < nch; ++c, ++g) {
          const int s = int(g % TCP_NS);
          if (g >= TCP_NS) {
            const uint32_t ph = uint32_t((g - TCP_NS) / TCP_NS) & 1;
            tc::mbar_wait(&mmad[s], ph);
            tc::mbar_wait(&std_[s], ph);
          }
          float* st = ring + s * SF;
          tc::mbar_expect_tx(&full[s], NB * 64 + (virt ? 0 : 8192));
          tc::bulk_g2s(st + 4 * QS, tc_wslab(a, a.tcw_f, l, nb, c), NB * 64, &full[s]);
          if (!virt)
            for (int q = 0; q < 4; ++q) tc::bulk_g2s(st + q * QS, zsrc + size_t(c) * 2048 + q * 512, 2048, &full[s]);
        }
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_tf32(128, NB);
      long long g = 0, it = 0;
      for (long long w = blockIdx.x; w < nitems; w += gridDim.x, ++it) {
        const int b = int(it & 1);
        if (it >= 2) {
          tc::mbar_wait(&acce[b], uint32_t((it - 2) >> 1) & 1);
          tc::fence_after();
        }
        for (int c = 0; c < nch; ++c, ++g) {
          const int s = int(g % TCP_NS);
          float* A = ring + s * SF;
          tc::mbar_wait(&actd[s], uint32_t(g / TCP_NS) & 1);
          tc::fence_after();
          // 2 K-steps (16 deep): A quads QS floats apart (LBO), B = the NB x 16 weight slab
#pragma unroll
          for (int kk = 0; kk < 2; ++kk)
            tc::mma_tf32(tmem + b * 256, tc::desc(A + kk * 2 * QS, QS * 4, 128),
                         tc::desc(A + 4 * QS + kk * 8 * NB, NB * 16, 128), idesc, (c != 0 || kk) ? 1u : 0u);
          tc::mma_commit(&mmad[s]);
        }
        tc::mma_commit(&accf[b]);
      }
    }
  } else if (warp >= 10 && warp < 14) {
    const int t = tid - 320;
    long long g = 0;
    for (long long w = blockIdx.x; w < nitems; w += gridDim.x) {
      const long long tile = w / nnb;
      const bool st0 = (w % nnb) == 0;
      for (int c = 0; c < nch; ++c, ++g) {
        const int s = int(g % TCP_NS);
        tc::mbar_wait(&actd[s], uint32_t(g / TCP_NS) & 1);
        if (st0 && a.st) slab_store_t<C, QS>(ring + s * SF, a.st + tc_toff(a, l - 1, tile), a.WP, 16 * c, t);
        arrive(&std_[s]);
      }
    }
  } else if (warp >= 14) {
    const int q = warp & 3, r = q * 32 + lane;
    const bool vrow = C::vrow(r);
    long long it = 0;
    for (long long w = blockIdx.x; w < nitems; w += gridDim.x, ++it) {
      const long long tile = w / nnb;
      const int b = int(it & 1), n0 = int(w % nnb) * NB;
      tc::mbar_wait(&accf[b], uint32_t(it >> 1) & 1);
      tc::fence_after();
      float* Zo = static_cast<float*>(a.act) + tc_off(a, l, tile, n0 / 4) + r * 4;
      const float* bl = kp + pl.off_b(l) + n0;
      for (int c0 = 0; c0 < NB; c0 += 16) {
        float v[16];
        tc::tmem_ld16(tmem + (uint32_t(q * 32) << 16) + b * 256 + c0, v);
        if (vrow)
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += __ldg(bl + c0 + i);
#pragma unroll
        for (int h = 0; h < 4; ++h)
          __stcs(reinterpret_cast<float4*>(Zo + size_t(c0 / 4 + h) * 512),
                 make_float4(v[4 * h], v[4 * h + 1], v[4 * h + 2], v[4 * h + 3]));
      }
      tc::fence_before();
      arrive(&acce[b]);
    }
  } else {
    // two activation groups (warps 0..3, 4..7) take alternate chunks
    const int ag = warp >> 2, t = tid & 127;
    long long g = 0;
    for (long long w = blockIdx.x; w < nitems; w += gridDim.x) {
      const long long tile = w / nnb;
      for (int c = 0; c < nch; ++c, ++g) {
        if (int(g & 1) != ag) continue;
        const int s = int(g % TCP_NS);
        float* A = ring + s * SF;
        tc::mbar_wait(&full[s], uint32_t(g / TCP_NS) & 1);
        if constexpr (TcUnit<C>::ON) {
          // (unit, quad) fastest within a warp: 2 points per warp, 2-way bank
          // conflicts with the FQS-padded quads (point-fastest lanes: 8-way;
          // E fwd 2.84 -> 1.96 ms per launch; XOR-permuting the two points'
          // stream orders as in the head measured 3 % slower)
          for (int i = t; i < TcUnit<C>::N; i += 128) {
            const int j = i & 3, kq = (i >> 2) & 3, pt = i >> 4;
            float z[C::S], sv[C::S];
            if (virt) tc_z0u<C>(a, kp, pl, tile * C::PPT + pt, 16 * c + 4 * kq + j, z);
            else slab_load1<C, QS>(z, A, pt, kq, j);
            tc_act1<C, ACT>(z, sv);
            slab_store1<C, QS>(A, pt, kq, j, sv);
          }
        } else
        for (int i = t; i < C::ITEMS; i += 128) {
          int pt, kq;
          C::fwd_item(i, pt, kq);
          float z[C::S][4], sv[C::S][4];
          if (virt) tc_z0<C>(a, kp, pl, tile * C::PPT + pt, 4 * c + kq, z);
          else slab_load<C, QS>(z, A, pt, kq);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float zz[C::S], ss[C::S];
            col<C>(z, j, zz);
            tc_act1<C, ACT>(zz, ss);
#pragma unroll
            for (int k = 0; k < C::S; ++k) sv[k][j] = ss[k];
          }
          slab_store<C, QS>(A, pt, kq, sv);
        }
        tc::fence_proxy_async();
        arrive(&actd[s]);
      }
    }
  }
  tc_teardown<512>(tmem);
}

// ---------------------------------------------------------------------------
// adjoint, hidden layer l >= 1: Zbar_{l-1} = act_bwd(Z_{l-1}, Zbar_l W_l^T)
// grid (tiles, WP/NB), 256 threads.  Main loop: thread 0 streams Zbar_l and W_l
// slabs through the ring and issues the MMAs.  Epilogue, 16 TMEM columns per
// step with double-buffered staging: warps 0..3 move S-bar TMEM -> shared,
// prefetch the Z_{l-1} slab (bulk copy) and run the point-major act-bwd in
// place; warps 4..7 meanwhile write the previous step's Zbar_{l-1} slab to HBM
// in both layouts (k-quad for the next adjoint, row-quad for dW).  For l == 1
// the layer-0 adjoint is reduced straight into per-tile dW_0 | db_0 partials
// (Zbar_0 is never stored).
// ---------------------------------------------------------------------------
constexpr int TC_DX_NT = 256;
template <int ACT, int MODE, int REG>
__global__ void __launch_bounds__(TC_DX_NT) tcw_dx_kernel(WArgs a, int l) {
  using C = TcCfg<ACT, MODE, REG>;
  constexpr int DIN = C::DIN, D1 = DIN + 1;
  extern __shared__ __align__(128) unsigned char tc_smem[];
  float* ring = reinterpret_cast<float*>(tc_smem);
  __shared__ __align__(8) uint64_t full[TC_NS], empty[TC_NS], zfull[2], rdy[2], done[2];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long tile = blockIdx.x;
  const int nb = blockIdx.y, NB = a.nb, n0 = nb * NB;
  const float* kp = static_cast<const float*>(a.kp);
  const ParamLayout pl{DIN, a.WK, C::NOUT, a.L};
  if (tid == 0) {
    for (int i = 0; i < TC_NS; ++i) tc::mbar_init(&full[i], 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&zfull[i], 1);
      tc::mbar_init(&rdy[i], 4);
      tc::mbar_init(&done[i], 4);
    }
  }
  const uint32_t tmem = tc_setup<256>(&tslot, empty, TC_NS);
  const int nch = a.WP / TC_KC;
  const size_t SF = C::stage_floats(NB);
  const float* zb = static_cast<const float*>(a.adj) + tc_off(a, l, tile, 0);
  if (tid == 0) {
    auto produce = [&](int c) {
      const int s = c % TC_NS;
      float* st = ring + s * SF;
      tc::mbar_expect_tx(&full[s], NB * 64 + 8192);
      tc::bulk_g2s(st + 2048, tc_wslab(a, a.tcw_d, l, nb, c), NB * 64, &full[s]);
      tc::bulk_g2s(st, zb + size_t(c) * 2048, 8192, &full[s]);
    };
    for (int c = 0; c < TC_NS && c < nch; ++c) produce(c);
    const uint32_t idesc = tc::idesc_tf32(128, NB);
    for (int c = 0; c < nch; ++c) {
      const int s = c % TC_NS;
      float* st = ring + s * SF;
      tc::mbar_wait(&full[s], (c / TC_NS) & 1);
      tc::fence_after();
      tc_mma16(tmem, st, 128, st + 2048, NB, idesc, c == 0);
      tc::mma_commit(&empty[s]);
      if (c >= 1 && c - 1 + TC_NS < nch) {
        tc::mbar_wait(&empty[(c - 1) % TC_NS], ((c - 1) / TC_NS) & 1);
        produce(c - 1 + TC_NS);
      }
    }
  }
  tc::mbar_wait(&empty[(nch - 1) % TC_NS], ((nch - 1) / TC_NS) & 1);
  tc::fence_after();
  __syncthreads();  // every thread is past the ring before it is reused
  // epilogue buffers inside the (now idle) ring
  float* stg = ring;             // [2][4][128][4]  S-bar / Zbar columns
  float* zc = ring + 2 * 2048;   // [2][4][128][4]  Z_{l-1} slabs
  const bool virt = (l == 1);
  float* red = ring + 2048;      // [PPT][4 kq][4 j][D1] dW_0 contributions (l == 1: stg[1], zc unused)
  const int nck = NB / 16;
  const float* zsrc = static_cast<const float*>(a.act) + (virt ? 0 : tc_off(a, l - 1, tile, n0 / 4));
  auto arrive = [&](uint64_t* bar) {
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
  };
  auto sync_e = [] { asm volatile("bar.sync 1, 128;" ::: "memory"); };
  if (tid < 128) {
    if (!virt && tid == 0)
      for (int j = 0; j < 2 && j < nck; ++j) {
        tc::mbar_expect_tx(&zfull[j], 8192);
        tc::bulk_g2s(zc + j * 2048, zsrc + size_t(j) * 2048, 8192, &zfull[j]);
      }
    const int r = warp * 32 + lane;
    const float* pts = static_cast<const float*>(a.pts);
    for (int j = 0; j < nck; ++j) {
      const int b = virt ? 0 : (j & 1);
      float* sg = stg + b * 2048;
      if (!virt && j >= 2) tc::mbar_wait(&done[b], ((j - 2) >> 1) & 1);
      {
        float v[16];
        tc::tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + 16 * j, v);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<float4*>(sg + q * 512 + r * 4) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
      sync_e();
      if (!virt) tc::mbar_wait(&zfull[b], (j >> 1) & 1);
      const float* zs = zc + b * 2048;
      for (int i = tid; i < C::ITEMS; i += 128) {
        const int pt = i % C::PPT, kq = i / C::PPT;
        const int q = n0 / 4 + 4 * j + kq;
        float z[C::S][4], sb[C::S][4];
        if (virt) tc_z0<C>(a, kp, pl, tile * C::PPT + pt, q, z);
        else slab_load<C>(z, zs, pt, kq);
        slab_load<C>(sb, sg, pt, kq);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          float zz[C::S], bb[C::S], sa[C::S];
          col<C>(z, jj, zz);
          col<C>(sb, jj, bb);
          tc_act_bwd1<C, ACT>(zz, bb, sa);
#pragma unroll
          for (int k = 0; k < C::S; ++k) sb[k][jj] = bb[k];
        }
        if (!virt) {
          slab_store<C>(sg, pt, kq, sb);  // Zbar_{l-1}, in place of S-bar
        } else {
          // dW_0[i][u] += x_i zbar_v + zbar_{g_i} ; db_0[u] += zbar_v (zero for padding points)
          const long long p = tile * C::PPT + pt;
          const bool live = p < a.n;
          float x[DIN];
#pragma unroll
          for (int ii = 0; ii < DIN; ++ii) x[ii] = live ? pts[p * DIN + ii] : 0.f;
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            float* rd = red + ((pt * 4 + kq) * 4 + jj) * D1;
            const float zv = live ? sb[0][jj] : 0.f;
#pragma unroll
            for (int ii = 0; ii < DIN; ++ii) {
              float t = x[ii] * zv;
              if constexpr (C::JET) t += live ? sb[1 + ii][jj] : 0.f;
              rd[ii] = t;
            }
            rd[DIN] = zv;
          }
        }
      }
      sync_e();
      if (!virt) {
        if (tid == 0 && j + 2 < nck) {
          tc::mbar_expect_tx(&zfull[b], 8192);
          tc::bulk_g2s(zc + b * 2048, zsrc + size_t(j + 2) * 2048, 8192, &zfull[b]);
        }
        arrive(&rdy[b]);
      } else {
        // fixed-order sum over the tile's points -> p0[tile][i*WP + u] (i == DIN: db_0)
        for (int e = tid; e < 16 * D1; e += 128) {
          const int kq = e / (4 * D1), jj = (e / D1) % 4, ii = e % D1;
          float acc = 0.f;
          for (int pt = 0; pt < C::PPT; ++pt) acc += red[((pt * 4 + kq) * 4 + jj) * D1 + ii];
          const int u = n0 + 16 * j + 4 * kq + jj;
          a.p0[size_t(tile) * (D1 * a.WP) + size_t(ii) * a.WP + u] = acc;
        }
        sync_e();
      }
    }
  } else if (!virt) {
    // writer warps: Zbar_{l-1} slab j in both HBM layouts
    const int t = tid - 128;
    for (int j = 0; j < nck; ++j) {
      const int b = j & 1;
      tc::mbar_wait(&rdy[b], (j >> 1) & 1);
      const float* sg = stg + b * 2048;
      slab_copy_out(sg, static_cast<float*>(a.adj) + tc_off(a, l - 1, tile, n0 / 4 + 4 * j), t);
      if (a.zt) slab_store_t<C>(sg, a.zt + tc_toff(a, l - 1, tile), a.WP, n0 + 16 * j, t);
      arrive(&done[b]);
    }
  }
  tc_teardown<256>(tmem);
}

// ---------------------------------------------------------------------------
// persistent adjoint, hidden layer l >= 1 (same math as tcw_dx_kernel).  One
// CTA per SM walks the (tile, N block) items grid-strided; the MMAs of item
// i+1 accumulate in the second TMEM buffer while the epilogue drains item i.
//   warps 0..7  epilogue group 0 (items 0, 2, ...), warps 10..17 group 1:
//               S-bar TMEM -> shared (warp w: lane quadrant w % 4, 16-column
//               blocks of parity w / 4), Z_{l-1} act-bwd in place over all 8
//               warps (the Z_{l-1} slabs are prefetched two steps ahead, across
//               item boundaries), then the step's Zbar_{l-1} slab to HBM;
//               l == 1: dW_0 | db_0 tile partials instead
//   warp 8      bulk-copy loader (Zbar_l + W_l slabs)    warp 9  MMA issuer
// ---------------------------------------------------------------------------
constexpr int TCP_DX_NS = 4;
constexpr int TCP_DX_NT = 576;
// CQ: unit quads per epilogue step (4: 16 TMEM columns, 8: 32 -- half the
// barrier / wait round trips per item; the last step of an N block may be 4)
template <class C, int CQ>
__host__ __device__ constexpr int tcp_dx_epi() {  // floats of one epilogue group's buffers
  // stg[2] + zc[2] slabs with padded unit quads (C::FQS, see the forward), or
  // (l == 1) stg[0] + the dW_0 reduction buffer
  return 4 * CQ * C::FQS > CQ * C::FQS + C::PPT * 4 * CQ * (C::DIN + 1) ? 4 * CQ * C::FQS
                                                                        : CQ * C::FQS + C::PPT * 4 * CQ * (C::DIN + 1);
}
template <class C, int CQ>
__host__ __device__ constexpr size_t tcp_dx_smem(int NB) {
  // epilogue: stg[2] + zc[2] slabs, or (l == 1) stg[0] + the dW_0 reduction buffer
  return sizeof(float) * (TCP_DX_NS * C::stage_floats(NB) + 2 * tcp_dx_epi<C, CQ>());
}
template <int ACT, int MODE, int REG, int CQ>
__global__ void __launch_bounds__(TCP_DX_NT, 1) tcw_dxp_kernel(WArgs a, int l) {
  using C = TcCfg<ACT, MODE, REG>;
  constexpr int DIN = C::DIN, D1 = DIN + 1;
  extern __shared__ __align__(128) unsigned char tc_smem[];
  float* ring = reinterpret_cast<float*>(tc_smem);
  __shared__ __align__(8) uint64_t full[TCP_DX_NS], empty[TCP_DX_NS], accf[2], acce[2], zfull_[2][2];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NB = a.nb, nnb = a.WP / NB, nqi = NB / 4, nck = (nqi + CQ - 1) / CQ;
  auto stepq = [&](int j) { return nqi - CQ * j < CQ ? nqi - CQ * j : CQ; };  // quads of step j
  const long long nitems = (long long)a.ntiles * nnb;
  const float* kp = static_cast<const float*>(a.kp);
  const ParamLayout pl{DIN, a.WK, C::NOUT, a.L};
  if (tid == 0) {
    for (int i = 0; i < TCP_DX_NS; ++i) tc::mbar_init(&full[i], 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&accf[i], 1);
      tc::mbar_init(&acce[i], 8);  // the 8 warps of epilogue group i
      for (int j = 0; j < 2; ++j) tc::mbar_init(&zfull_[i][j], 1);
    }
  }
  const uint32_t tmem = tc_setup<512>(&tslot, empty, TCP_DX_NS);
  const int nch = a.WP / TC_KC;
  const size_t SF = C::stage_floats(NB);
  const bool virt = (l == 1);
  // epilogue group grp (items with it % 2 == grp, i.e. TMEM accumulator grp)
  const int grp = warp >= 10 ? 1 : 0, wl = warp - 10 * grp;
  // epilogue slabs: unit quads QS floats apart (conflict-free act-bwd items
  // with fwd_item() and a conflict-free row-quad gather for Zbar^T)
  constexpr int QS = C::FQS, QSL = CQ * QS;
  float* stg = ring + TCP_DX_NS * SF + grp * tcp_dx_epi<C, CQ>();  // [2][CQ kq (QS)][128][4]  S-bar / Zbar columns
  float* zc = stg + 2 * QSL;          // [2][CQ kq (QS)][128][4]  Z_{l-1} slabs
  float* red = stg + QSL;             // l == 1: [PPT][CQ kq][4 j][D1] dW_0 contributions (in place of stg[1], zc)
  uint64_t* zfull = zfull_[grp];
  auto arrive = [&](uint64_t* bar) {
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
  };
  auto sync_e = [grp] { asm volatile("bar.sync %0, 256;" ::"r"(1 + grp) : "memory"); };
  if (warp == 8) {
    if (lane == 0) {
      long long g = 0;
      for (long long w = blockIdx.x; w < nitems; w += gridDim.x) {
        const long long tile = w / nnb;
        const int nb = int(w % nnb);
        const float* zb = static_cast<const float*>(a.adj) + tc_off(a, l, tile, 0);
        for (int c = 0; c < nch; ++c, ++g) {
          const int s = int(g % TCP_DX_NS);
          if (g >= TCP_DX_NS) tc::mbar_wait(&empty[s], uint32_t((g - TCP_DX_NS) / TCP_DX_NS) & 1);
          float* st = ring + s * SF;
          tc::mbar_expect_tx(&full[s], NB * 64 + 8192);
          tc::bulk_g2s(st + 2048, tc_wslab(a, a.tcw_d, l, nb, c), NB * 64, &full[s]);
          tc::bulk_g2s(st, zb + size_t(c) * 2048, 8192, &full[s]);
        }
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_tf32(128, NB);
      long long g = 0, it = 0;
      for (long long w = blockIdx.x; w < nitems; w += gridDim.x, ++it) {
        const int b = int(it & 1);
        if (it >= 2) {
          tc::mbar_wait(&acce[b], uint32_t((it - 2) >> 1) & 1);
          tc::fence_after();
        }
        for (int c = 0; c < nch; ++c, ++g) {
          const int s = int(g % TCP_DX_NS);
          float* st = ring + s * SF;
          tc::mbar_wait(&full[s], uint32_t(g / TCP_DX_NS) & 1);
          tc::fence_after();
          tc_mma16(tmem + b * 256, st, 128, st + 2048, NB, idesc, c == 0);
          tc::mma_commit(&empty[s]);
        }
        tc::mma_commit(&accf[b]);
      }
    }
  } else {
    // epilogue group: 8 warps, 256 threads.  Warp wl reads TMEM lane quadrant
    // wl % 4 (tile rows r) and the 16-column blocks h % 2 == wl / 4 of a step;
    // every thread then takes act-bwd items and the step's copy-out
    const int et = wl * 32 + lane, half = wl >> 2, r = (warp & 3) * 32 + lane;
    const float* pts = static_cast<const float*>(a.pts);
    // Z_{l-1} slab of step j of item w (CQ quads)
    auto zslab = [&](long long w, int j) {
      return static_cast<const float*>(a.act) + tc_off(a, l - 1, w / nnb, int(w % nnb) * NB / 4) + size_t(j) * CQ * 512;
    };
    auto prefetch = [&](long long w, int j, int b) {  // step j of item w into zc[b] (j may run into the next item)
      if (j >= nck) {
        w += 2 * gridDim.x;
        j -= nck;
      }
      if (w >= nitems) return;
      const int nq = stepq(j);
      tc::mbar_expect_tx(&zfull[b], 2048 * nq);
      for (int q = 0; q < nq; ++q) tc::bulk_g2s(zc + b * QSL + q * QS, zslab(w, j) + q * 512, 2048, &zfull[b]);
    };
    const long long w0 = blockIdx.x + (long long)grp * gridDim.x;
    if (!virt && et == 0 && w0 < nitems)
      for (int j = 0; j < 2; ++j) prefetch(w0, j, j);
    long long k = 0, jg = 0;
    for (long long w = w0; w < nitems; w += 2 * gridDim.x, ++k) {
      const long long tile = w / nnb;
      const int ab = grp, n0 = int(w % nnb) * NB;
      tc::mbar_wait(&accf[ab], uint32_t(k) & 1);
      tc::fence_after();
      for (int j = 0; j < nck; ++j, ++jg) {
        const int b = virt ? 0 : int(jg & 1);
        float* sg = stg + b * QSL;
        const int nqj = stepq(j), nhj = nqj / 4;  // quads / 16-unit blocks of this step
        for (int h = half; h < nhj; h += 2) {
          float v[16];
          tc::tmem_ld16(tmem + (uint32_t((warp & 3) * 32) << 16) + ab * 256 + 4 * CQ * j + 16 * h, v);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<float4*>(sg + (4 * h + q) * QS + r * 4) =
                make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
        if (j == nck - 1) {
          tc::fence_before();
          arrive(&acce[ab]);
        }
        sync_e();
        if (!virt) tc::mbar_wait(&zfull[b], uint32_t(jg >> 1) & 1);
        const float* zs = zc + b * QSL;
        if constexpr (TcUnit<C, true, ACT>::ON) {
          // 3D: (unit, quad) fastest within a warp -- with the FQS-padded quads
          // an 8-quad step's 32 lanes hit 32 distinct banks on every stream row
          // (point-fastest lanes shared one bank group: a point's 8 rows are
          // 128 bytes; E dx 3.78 -> 2.29 ms); 2D keeps the fwd_item lane map
          constexpr int NU = TcUnit<C, true, ACT>::N;
          for (int i = et; i < nhj * NU; i += 256) {
            const int jj = i & 3;
            int pt, kq;
            if constexpr (C::FWD_MAP) {
              const int hh = i / NU;
              C::fwd_item((i - hh * NU) >> 2, pt, kq);
              kq += 4 * hh;
            } else {
              kq = (i >> 2) % nqj;
              pt = (i >> 2) / nqj;
            }
            float z[C::S], sb[C::S], sa[C::S];
            if (virt) tc_z0u<C>(a, kp, pl, tile * C::PPT + pt, n0 + 4 * (CQ * j + kq) + jj, z);
            else slab_load1<C, QS>(z, zs, pt, kq, jj);
            slab_load1<C, QS>(sb, sg, pt, kq, jj);
            tc_act_bwd1<C, ACT>(z, sb, sa);
            if (!virt) {
              slab_store1<C, QS>(sg, pt, kq, jj, sb);  // Zbar_{l-1}, in place of S-bar
            } else {
              const long long p = tile * C::PPT + pt;
              const bool live = p < a.n;
              float* rd = red + ((pt * CQ + kq) * 4 + jj) * D1;
              const float zv = live ? sb[0] : 0.f;
#pragma unroll
              for (int ii = 0; ii < DIN; ++ii) {
                float t = (live ? pts[p * DIN + ii] : 0.f) * zv;
                if constexpr (C::JET) t += live ? sb[1 + ii] : 0.f;
                rd[ii] = t;
              }
              rd[DIN] = zv;
            }
          }
        } else
        for (int i = et; i < nhj * C::ITEMS; i += 256) {
          const int hh = i / C::ITEMS;
          int pt, kq;
          C::fwd_item(i - hh * C::ITEMS, pt, kq);
          kq += 4 * hh;
          const int q = n0 / 4 + CQ * j + kq;
          float z[C::S][4], sb[C::S][4];
          if (virt) tc_z0<C>(a, kp, pl, tile * C::PPT + pt, q, z);
          else slab_load<C, QS>(z, zs, pt, kq);
          slab_load<C, QS>(sb, sg, pt, kq);
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            float zz[C::S], bb[C::S], sa[C::S];
            col<C>(z, jj, zz);
            col<C>(sb, jj, bb);
            tc_act_bwd1<C, ACT>(zz, bb, sa);
#pragma unroll
            for (int k = 0; k < C::S; ++k) sb[k][jj] = bb[k];
          }
          if (!virt) {
            slab_store<C, QS>(sg, pt, kq, sb);  // Zbar_{l-1}, in place of S-bar
          } else {
            const long long p = tile * C::PPT + pt;
            const bool live = p < a.n;
            float x[DIN];
#pragma unroll
            for (int ii = 0; ii < DIN; ++ii) x[ii] = live ? pts[p * DIN + ii] : 0.f;
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              float* rd = red + ((pt * CQ + kq) * 4 + jj) * D1;
              const float zv = live ? sb[0][jj] : 0.f;
#pragma unroll
              for (int ii = 0; ii < DIN; ++ii) {
                float t = x[ii] * zv;
                if constexpr (C::JET) t += live ? sb[1 + ii][jj] : 0.f;
                rd[ii] = t;
              }
              rd[DIN] = zv;
            }
          }
        }
        sync_e();
        if (!virt) {
          if (et == 0) prefetch(w, j + 2, b);
          // Zbar_{l-1} of this step to HBM (k-quad): 16-byte rows, quads 2 KB apart
          float* dst = static_cast<float*>(a.adj) + tc_off(a, l - 1, tile, n0 / 4 + CQ * j);
          for (int e = et; e < nqj * 128; e += 256)
            reinterpret_cast<float4*>(dst + (e >> 7) * 512)[e & 127] =
                reinterpret_cast<const float4*>(sg + (e >> 7) * QS)[e & 127];
          if (a.zt && et < 128)
            for (int h = 0; h < nhj; ++h)
              slab_store_t<C, QS>(sg + 4 * h * QS, a.zt + tc_toff(a, l - 1, tile), a.WP, n0 + 4 * (CQ * j + 4 * h), et);
        } else {
          for (int e = et; e < 4 * nqj * D1; e += 256) {
            const int kq = e / (4 * D1), jj = (e / D1) % 4, ii = e % D1;
            float acc = 0.f;
            for (int pt = 0; pt < C::PPT; ++pt) acc += red[((pt * CQ + kq) * 4 + jj) * D1 + ii];
            const int u = n0 + 4 * (CQ * j + kq) + jj;
            a.p0[size_t(tile) * (D1 * a.WP) + size_t(ii) * a.WP + u] = acc;
          }
          sync_e();
        }
      }
    }
  }
  tc_teardown<512>(tmem);
}

// ---------------------------------------------------------------------------
// dW_l = sum_rows S_{l-1}^T Zbar_l (+ db_l = sum of value rows of Zbar_l).
// Both operands arrive row-quad major (written by the forward / adjoint
// kernels), i.e. already K-major for K = rows, so this is a pure stream:
//   warp 0     loader: per 32-row group, one bulk copy of S_{l-1} (all WP
//              units, WP*128 B) + the Zbar_l N block (NB*128 B) into an
//              NS-stage ring;
//   warp 1     MMA issuer: nkb = ceil(WP/128) accumulators of 128 x NB in
//              TMEM (nkb * NB <= 512 columns), 4 K-steps per group;
//   warps 2-9  db_l (one unit per thread) and the final TMEM -> HBM drain.
// grid (WP/NB, splits), one CTA per SM.
// ---------------------------------------------------------------------------
constexpr int TC_DW_MAXNS = 4;
template <int ACT, int MODE, int REG>
__global__ void __launch_bounds__(320) tcw_dw_kernel(WArgs a, int l, int NB, int NS) {
  using C = TcCfg<ACT, MODE, REG>;
  constexpr int S = C::S;
  extern __shared__ __align__(128) unsigned char tc_smem[];
  const int WP = a.WP;
  const int SF = (WP + NB) * 32;  // stage floats: A [8][WP][4] then B [8][NB][4]
  float* ring = reinterpret_cast<float*>(tc_smem);
  __shared__ __align__(8) uint64_t full[TC_DW_MAXNS], empty[TC_DW_MAXNS], done;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nbk = blockIdx.x, n0 = nbk * NB, split = blockIdx.y;
  const int nkb = (WP + 127) / 128;
  const ParamLayout pl{C::DIN, a.WK, C::NOUT, a.L};
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1 + 8);  // MMA commit + the 8 db warps
    }
    tc::mbar_init(&done, 1);
  }
  const uint32_t tmem = tc_setup<512>(&tslot, nullptr, 0);
  const long long my_tiles = split < a.ntiles ? (a.ntiles - 1 - split) / gridDim.y + 1 : 0;
  const long long nchunks = 4 * my_tiles;
  double* gp = a.gpart + size_t(split) * a.np_pad;
  if (warp == 0) {
    if (lane == 0)
      for (long long ci = 0; ci < nchunks; ++ci) {
        const int s = int(ci % NS);
        const long long t = split + (ci >> 2) * gridDim.y;
        const int g = int(ci & 3);
        if (ci >= NS) tc::mbar_wait(&empty[s], ((ci - NS) / NS) & 1);
        float* A = ring + s * SF;
        float* B = A + WP * 32;
        tc::mbar_expect_tx(&full[s], uint32_t(WP + NB) * 128);
        tc::bulk_g2s(A, a.st + tc_toff(a, l - 1, t) + size_t(g) * 8 * WP * 4, WP * 128, &full[s]);
        const float* zsrc = a.zt + tc_toff(a, l, t) + (size_t(g) * 8 * WP + n0) * 4;
        if (NB == WP) {
          tc::bulk_g2s(B, zsrc, NB * 128, &full[s]);
        } else {
          for (int rq = 0; rq < 8; ++rq) tc::bulk_g2s(B + rq * NB * 4, zsrc + size_t(rq) * WP * 4, NB * 16, &full[s]);
        }
      }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_tf32(128, NB);
      for (long long ci = 0; ci < nchunks; ++ci) {
        const int s = int(ci % NS);
        tc::mbar_wait(&full[s], (ci / NS) & 1);
        tc::fence_after();
        const float* A = ring + s * SF;
        const float* B = A + WP * 32;
        for (int kb = 0; kb < nkb; ++kb)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc::mma_tf32(tmem + kb * NB, tc::desc(A + kb * 512 + kk * 8 * WP, WP * 16, 128),
                         tc::desc(B + kk * 8 * NB, NB * 16, 128), idesc, (ci || kk) ? 1u : 0u);
        tc::mma_commit(&empty[s]);
      }
      if (nchunks > 0) tc::mma_commit(&done);
    }
  } else {
    // ---- db_l (unit u per thread) ----
    const int u = tid - 64;  // 0..255
    float db = 0.f;
    for (long long ci = 0; ci < nchunks; ++ci) {
      const int s = int(ci % NS), g = int(ci & 3);
      tc::mbar_wait(&full[s], (ci / NS) & 1);
      if (u < NB) {
        const float* B = ring + s * SF + WP * 32;
        // value rows of the group, in row order: compile-time row lists per group
        auto dbg = [&](auto G) {
          constexpr int gg = decltype(G)::value, r0 = (S - (32 * gg) % S) % S;
#pragma unroll
          for (int r = r0; r < 32; r += S)
            if (C::vrow(32 * gg + r)) db += B[((r >> 2) * NB + u) * 4 + (r & 3)];
        };
        switch (g) {
          case 0: dbg(IntC<0>{}); break;
          case 1: dbg(IntC<1>{}); break;
          case 2: dbg(IntC<2>{}); break;
          default: dbg(IntC<3>{}); break;
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&empty[s])) : "memory");
    }
    if (nchunks > 0) {
      if (u < NB) gp[pl.off_b(l) + n0 + u] = double(db);
      tc::mbar_wait(&done, 0);
      tc::fence_after();
      // warps 2..9: TMEM lane quadrant warp % 4, column half (warp - 2) / 4
      const int quad = warp & 3, half = (warp - 2) >> 2;
      for (int kb = 0; kb < nkb; ++kb) {
        const int kr = kb * 128 + quad * 32 + lane;
        for (int c0 = half * 16; c0 < NB; c0 += 32) {
          float v[16];
          tc::tmem_ld16(tmem + (uint32_t(quad * 32) << 16) + kb * NB + c0, v);
          if (kr < WP) {
            double* dst = gp + pl.off_w(l) + size_t(kr) * a.WK + n0 + c0;
#pragma unroll
            for (int i = 0; i < 16; ++i) dst[i] = double(v[i]);
          }
        }
      }
    }
  }
  tc_teardown<512>(tmem);
}

// ---------------------------------------------------------------------------
// dW_l = sum_rows S_{l-1}^T Zbar_l (+ db_l) with Zbar_l read straight from the
// k-quad adjoint slabs (no row-quad-major Zbar^T copy: the adjoint and head
// kernels write one slab fewer per layer).  S_{l-1}^T still comes
// row-quad-major from the forward, which activates S in shared memory anyway
// (re-activating Z here measured slower: the jet activation is as costly as
// the copy it saves).  Zbar_l is the B operand with K = rows, i.e. MN-major,
// which sm_100a reads for TF32 only in the SWIZZLE_128B_BASE32B layout
// (512-byte atoms of 4 rows x 32 units, 32-byte chunks XOR-swizzled by the row;
// LBO = 32-unit group stride, SBO = 4-row group stride; tests/test_gpu_tc.py
// layouts 6 / 7).  Per 32-row group:
//   warp 0      loader: the S^T group (one bulk copy, K-major [8 rq][WP][4])
//               and the group's 32 rows of the Zbar_l N block's quads (one
//               tensor-map copy, csrc/tma.cuh) as a k-quad stage;
//   warps 2..9  converters: the Zbar pieces (lane = row: conflict-free 16-byte
//               loads) into registers, then in place as BASE32B (pad rows
//               zeroed); db_l from its value rows;
//   warp 1      MMA issuer: ceil(WP/128) M = 128 blocks of in-units x NB
//               out-units (rounded to whole 32-unit groups) in TMEM.
// grid (WP/NB, splits), one CTA per SM.  Bit-identical to tcw_dw_kernel.
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int dwq_b_floats(int NB) { return (NB + 31) / 32 * 1024; }
constexpr int DWQ_MAXNS = 6;
__host__ __device__ constexpr size_t dwq_stage_bytes(int WP, int NB) {
  return sizeof(float) * size_t(dwq_b_floats(NB) + WP * 32);
}
// float offset of element (mn, row) in a BASE32B operand of 32 K rows
__device__ __forceinline__ int dwq_b32(int mn, int r) {
  return (((mn >> 5) * 8 + (r >> 2)) << 7) + ((r & 3) << 5) + (((((mn & 31) >> 3) ^ r) & 3) << 3) + (mn & 7);
}
template <int ACT, int MODE, int REG>
__global__ void __launch_bounds__(320, 1) tcw_dwq_kernel(WArgs a, int l, int NB, int NS,
                                                         const __grid_constant__ CUtensorMap tmB) {
  using C = TcCfg<ACT, MODE, REG>;
  constexpr int S = C::S;
  extern __shared__ __align__(128) unsigned char tc_smem[];
  const int WP = a.WP, nqb = NB / 4;
  // stage: [S^T group][BASE32B Zbar]; WP * 128 bytes keep the BASE32B part 1 KB
  // aligned, and the second M block's reads past the S^T group (rows >= WP,
  // never drained) stay inside the stage
  const int AF = WP * 32, SF = AF + dwq_b_floats(NB);
  // BASE32B atoms are swizzled on absolute address bits: 1 KB-aligned ring
  float* ring = reinterpret_cast<float*>(tc_smem + ((1024u - (tc::smem_u32(tc_smem) & 1023u)) & 1023u));
  __shared__ __align__(8) uint64_t full[DWQ_MAXNS], conv[DWQ_MAXNS], empty[DWQ_MAXNS], done;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nbk = blockIdx.x, n0 = nbk * NB, split = blockIdx.y;
  const int nkb = (WP + 127) / 128;
  // MMA N: the N block rounded up to whole 32-unit BASE32B groups (the extra
  // columns see stale shared memory and are never drained)
  const int NBM = (NB + 31) / 32 * 32;
  const ParamLayout pl{C::DIN, a.WK, C::NOUT, a.L};
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&conv[i], 1);
      tc::mbar_init(&empty[i], 1 + 8);  // MMA commit + the 8 converter / db warps
    }
    tc::mbar_init(&done, 1);
  }
  const uint32_t tmem = tc_setup<512>(&tslot, nullptr, 0);
  const long long my_tiles = split < a.ntiles ? (a.ntiles - 1 - split) / gridDim.y + 1 : 0;
  const long long nchunks = 4 * my_tiles;
  double* gp = a.gpart + size_t(split) * a.np_pad;
  if (warp == 0) {
    if (lane == 0)
      for (long long ci = 0; ci < nchunks; ++ci) {
        const int s = int(ci % NS);
        const long long t = split + (ci >> 2) * gridDim.y;
        const int g = int(ci & 3);
        if (ci >= NS) tc::mbar_wait(&empty[s], ((ci - NS) / NS) & 1);
        float* A = ring + size_t(s) * SF;
        float* B = A + AF;
        tc::mbar_expect_tx(&full[s], uint32_t(WP + NB) * 128);
        tc::bulk_g2s(A, a.st + tc_toff(a, l - 1, t) + size_t(g) * 8 * WP * 4, WP * 128, &full[s]);
        tc::tma_load3(B, &tmB, 128 * g, n0 / 4, int(l * a.ntiles + t), &full[s]);
      }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_tf32(128, NBM, 0, 1);
      for (long long ci = 0; ci < nchunks; ++ci) {
        const int s = int(ci % NS);
        tc::mbar_wait(&conv[s], (ci / NS) & 1);
        tc::fence_after();
        const float* A = ring + size_t(s) * SF;
        const float* B = A + AF;
        for (int kb = 0; kb < nkb; ++kb)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc::mma_tf32(tmem + kb * NBM, tc::desc(A + kb * 512 + kk * 8 * WP, WP * 16, 128),
                         tc::desc(B + kk * 256, 4096, 512) | (uint64_t(1) << 61), idesc, (ci || kk) ? 1u : 0u);
        tc::mma_commit(&empty[s]);
      }
      if (nchunks > 0) tc::mma_commit(&done);
    }
  } else {
    const int ct = tid - 64;  // 0..255
    // converter warp cw owns unit quads cw, cw + 8, ...; lane = row of the group
    const int cw = warp - 2, r = lane;
    constexpr int MAXQ = 8;  // quads per warp (NB <= 256)
    auto cbar = [] { asm volatile("bar.sync 1, 256;" ::: "memory"); };
    float db = 0.f;
    for (long long ci = 0; ci < nchunks; ++ci) {
      const int s = int(ci % NS);
      float* B = ring + size_t(s) * SF + AF;
      const int g = int(ci & 3);
      const bool live = 32 * g + r < C::VRT;  // pad rows carry zeros
      tc::mbar_wait(&full[s], (ci / NS) & 1);
      float4 vb[MAXQ];
#pragma unroll
      for (int k = 0; k < MAXQ; ++k) {
        const int q = cw + 8 * k;
        if (q < nqb)
          vb[k] = live ? *reinterpret_cast<const float4*>(B + q * 128 + r * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      cbar();
#pragma unroll
      for (int k = 0; k < MAXQ; ++k) {
        const int q = cw + 8 * k;
        if (q < nqb) *reinterpret_cast<float4*>(B + dwq_b32(4 * q, r)) = vb[k];
      }
      tc::fence_proxy_async();
      cbar();
      if (ct == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&conv[s])) : "memory");
      // db_l: value rows of Zbar_l, one unit per thread, in row order
      if (ct < NB) {
        // value rows of group g, in row order: compile-time row lists per group
        auto dbg = [&](auto G) {
          constexpr int gg = decltype(G)::value, r0 = (S - (32 * gg) % S) % S;
#pragma unroll
          for (int rr = r0; rr < 32; rr += S)
            if (C::vrow(32 * gg + rr)) db += B[dwq_b32(ct, rr)];
        };
        switch (g) {
          case 0: dbg(IntC<0>{}); break;
          case 1: dbg(IntC<1>{}); break;
          case 2: dbg(IntC<2>{}); break;
          default: dbg(IntC<3>{}); break;
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&empty[s])) : "memory");
    }
    if (nchunks > 0) {
      if (ct < NB) gp[pl.off_b(l) + n0 + ct] = double(db);
      tc::mbar_wait(&done, 0);
      tc::fence_after();
      // warps 2..9: TMEM lane quadrant warp % 4, column half (warp - 2) / 4
      const int quad = warp & 3, half = (warp - 2) >> 2;
      for (int kb = 0; kb < nkb; ++kb) {
        const int kr = kb * 128 + quad * 32 + lane;
        for (int c0 = half * 16; c0 < NB; c0 += 32) {
          float v[16];
          tc::tmem_ld16(tmem + (uint32_t(quad * 32) << 16) + kb * NBM + c0, v);
          if (kr < WP) {
            double* dst = gp + pl.off_w(l) + size_t(kr) * a.WK + n0 + c0;
#pragma unroll
            for (int i = 0; i < 16; ++i) dst[i] = double(v[i]);
          }
        }
      }
    }
  }
  tc_teardown<512>(tmem);
}

// ---------------------------------------------------------------------------
// head: output layer + residual / MSE + Ybar + S-bar_{L-1} + act-bwd -> Zbar_{L-1},
// with the per-tile dW_L | db_L partials.  grid tiles, 128 threads; Z_{L-1} is
// streamed twice through a bulk-copy ring (forward pass, then adjoint pass).
// ---------------------------------------------------------------------------
template <int ACT, int MODE, int REG>
__global__ void __launch_bounds__(128) tcw_head_kernel(WArgs a) {
  using C = TcCfg<ACT, MODE, REG>;
  constexpr int NT = C::NT, PPT = C::PPT, NOUT = C::NOUT, NVEL = C::NVEL, S = C::S;
  constexpr int NG = C::NG, LAP0 = C::LAP0, SN = S * NOUT;
  // 3D jets: 64 (point, unit quad) items per chunk -> per-unit items (TcUnit)
  constexpr bool HU = TcUnit<C>::ON;
  constexpr int TPPH = HU ? NT / PPT : C::TPP;  // threads holding partial sums of one point
  static_assert(!HU || (NT % (4 * PPT) == 0 && 4 * C::ITEMS % NT == 0), "per-unit head split");
  extern __shared__ __align__(128) unsigned char tc_smem[];
  double* lred = reinterpret_cast<double*>(tc_smem);      // [2][NT]
  constexpr int QS = C::FQS, SF = 4 * QS;                 // padded unit quads (see TcCfg::FQS)
  float* ring = reinterpret_cast<float*>(lred + 2 * NT);  // [NS][4][QS]
  float* WLs = ring + TC_HEAD_NS * SF;                          // [WP][NOUT]
  float* Yp = WLs + a.WP * NOUT;                           // [NT][YPS]
  float* Ys = Yp + NT * C::YPS;                            // [PPT][SN]
  float* Ybs = Ys + PPT * SN;                              // [PPT][SN]
  float* red = Ybs + PPT * SN;                             // see TcCfg::HEAD_RED
  __shared__ __align__(8) uint64_t full[TC_HEAD_NS];
  const long long tile = blockIdx.x;
  const int tid = threadIdx.x;
  const float* kp = static_cast<const float*>(a.kp);
  const ParamLayout pl{C::DIN, a.WK, NOUT, a.L};
  const int L = a.L, nch = a.WP / TC_KC, ntot = 2 * nch;
  const float* zsrc = static_cast<const float*>(a.act) + tc_off(a, L - 1, tile, 0);
  if (tid == 0) {
    for (int i = 0; i < TC_HEAD_NS; ++i) tc::mbar_init(&full[i], 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  auto produce = [&](int g) {
    const int s = g % TC_HEAD_NS;
    tc::mbar_expect_tx(&full[s], 8192);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      tc::bulk_g2s(ring + s * SF + q * QS, zsrc + size_t(g % nch) * 2048 + q * 512, 2048, &full[s]);
  };
  if (tid == 0)
    for (int g = 0; g < TC_HEAD_NS && g < ntot; ++g) produce(g);
  for (int i = tid; i < a.WP * NOUT; i += NT) WLs[i] = kp[pl.off_w(L) + i];
  __syncthreads();
  // ---- forward: Y partials per (point, kq) thread ----
  float y[S][NOUT];
#pragma unroll
  for (int st = 0; st < S; ++st)
#pragma unroll
    for (int o = 0; o < NOUT; ++o) y[st][o] = 0.f;
  for (int c = 0; c < nch; ++c) {
    const int s = c % TC_HEAD_NS;
    tc::mbar_wait(&full[s], (c / TC_HEAD_NS) & 1);
    if constexpr (HU) {
      // per-unit items: thread tid always holds point (tid >> 2) % PPT
      for (int i = tid; i < 4 * C::ITEMS; i += NT) {
        const int j = i & 3, pt = (i >> 2) % PPT, kq = (i >> 2) / PPT;
        float zz[S], ss[S];
        slab_load1x<C, QS>(zz, ring + s * SF, pt, kq, j, pt & 7);
        tc_act1<C, ACT>(zz, ss);
        const float* w = WLs + (16 * c + 4 * kq + j) * NOUT;
#pragma unroll
        for (int st = 0; st < S; ++st)
#pragma unroll
          for (int o = 0; o < NOUT; ++o) y[st][o] = fmaf(ss[st], w[o], y[st][o]);
      }
    } else
    for (int i = tid; i < C::ITEMS; i += NT) {
      int pt, kq;
      C::fwd_item(i, pt, kq);
      float z[S][4];
      slab_load<C, QS>(z, ring + s * SF, pt, kq);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float zz[S], ss[S];
        col<C>(z, j, zz);
        tc_act1<C, ACT>(zz, ss);
        const float* w = WLs + (16 * c + 4 * kq + j) * NOUT;
#pragma unroll
        for (int st = 0; st < S; ++st)
#pragma unroll
          for (int o = 0; o < NOUT; ++o) y[st][o] = fmaf(ss[st], w[o], y[st][o]);
      }
    }
    __syncthreads();
    if (tid == 0 && c + TC_HEAD_NS < ntot) produce(c + TC_HEAD_NS);
  }
#pragma unroll
  for (int st = 0; st < S; ++st)
#pragma unroll
    for (int o = 0; o < NOUT; ++o) Yp[tid * C::YPS + st * NOUT + o] = y[st][o];
  __syncthreads();
  const long long p0 = tile * PPT, rem = a.n - p0;
  double lacc0 = 0.0, lacc1 = 0.0;
  if (tid < PPT) {
    const int pt = tid;
    float* yv = Ys + pt * SN;
    float* yb = Ybs + pt * SN;
    for (int i = 0; i < SN; ++i) {
      float v = 0.f;
      for (int h = 0; h < TPPH; ++h) v += Yp[(HU ? 4 * (pt + PPT * (h >> 2)) + (h & 3) : C::item_of(pt, h)) * C::YPS + i];
      yv[i] = (i < NOUT) ? v + kp[pl.off_b(L) + i] : v;
      yb[i] = 0.f;
    }
    if (pt < rem) {
      if constexpr (MODE == MODE_PDE) {
        using Rg = Regime<REG>;
        constexpr int NSP = Rg::NSP, TOFF = Rg::HAS_T, P = NVEL;
        const float inv_re = float(a.inv_re), two_coef = float(2.0 * a.coef);
        auto Y = [&](int s, int o) { return yv[s * NOUT + o]; };
        auto GRAD = [&](int in) { return 1 + in; };
        auto LAP = [&](int in) { return 1 + NG + (in - LAP0); };
        float rr[NVEL + 1];
#pragma unroll
        for (int i = 0; i < NVEL; ++i) {
          const int xi = TOFF + i;
          float acc = 0.f;
          if constexpr (Rg::HAS_T) acc = Y(GRAD(0), i);
          acc = (Rg::HAS_T ? acc + Y(GRAD(xi), P) : Y(GRAD(xi), P));
#pragma unroll
          for (int jj = 0; jj < NSP; ++jj) acc += -inv_re * Y(LAP(TOFF + jj), i);
#pragma unroll
          for (int kk = 0; kk < NVEL; ++kk) acc += Y(0, kk) * Y(GRAD(TOFF + kk), i);
          rr[i] = acc;
        }
        {
          float acc = Y(GRAD(TOFF), 0);
#pragma unroll
          for (int kk = 1; kk < NVEL; ++kk) acc += Y(GRAD(TOFF + kk), kk);
          rr[NVEL] = acc;
        }
#pragma unroll
        for (int i = 0; i <= NVEL; ++i) lacc0 += double(rr[i]) * double(rr[i]);
#pragma unroll
        for (int i = 0; i < NVEL; ++i) {
          const float rb = two_coef * rr[i];
          if constexpr (Rg::HAS_T) yb[GRAD(0) * NOUT + i] += rb;
          yb[GRAD(TOFF + i) * NOUT + P] += rb;
#pragma unroll
          for (int jj = 0; jj < NSP; ++jj) yb[LAP(TOFF + jj) * NOUT + i] += -inv_re * rb;
#pragma unroll
          for (int kk = 0; kk < NVEL; ++kk) {
            yb[0 * NOUT + kk] += rb * Y(GRAD(TOFF + kk), i);
            yb[GRAD(TOFF + kk) * NOUT + i] += rb * Y(0, kk);
          }
        }
        const float rb = two_coef * rr[NVEL];
#pragma unroll
        for (int kk = 0; kk < NVEL; ++kk) yb[GRAD(TOFF + kk) * NOUT + kk] += rb;
      } else {  // MSE
        const float two_vc = float(2.0 * a.coef), two_pc = float(2.0 * a.pcoef);
        const float* tu = static_cast<const float*>(a.tu) + (p0 + pt) * NVEL;
#pragma unroll
        for (int o = 0; o < NVEL; ++o) {
          const float d = yv[o] - tu[o];
          lacc0 += a.velw[o] * (double(d) * double(d));
          yb[o] = (two_vc * float(a.velw[o])) * d;
        }
        if (a.has_p) {
          const float d = yv[NVEL] - static_cast<const float*>(a.tp)[p0 + pt];
          lacc1 += double(d) * double(d);
          yb[NVEL] = two_pc * d;
        }
      }
    }
  }
  lred[tid] = lacc0;
  lred[NT + tid] = lacc1;
  __syncthreads();
  const size_t plen = size_t(a.WP) * NOUT + NOUT;
  float* pL = a.pL + size_t(tile) * plen;
  if (tid == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int i = 0; i < NT; ++i) {
      s0 += lred[i];
      s1 += lred[NT + i];
    }
    a.lpart[2 * tile] = s0;
    a.lpart[2 * tile + 1] = s1;
  }
  if (tid < NOUT) {  // db_L: value-row adjoints summed in point order
    float acc = 0.f;
    for (int pt = 0; pt < PPT; ++pt) acc += Ybs[pt * SN + tid];
    pL[size_t(a.WP) * NOUT + tid] = acc;
  }
  // ---- adjoint: S-bar = Ybar W_L^T, act-bwd, dW_L partial ----
  // a thread's points are the same in every chunk: their Ybar rows are read
  // once into registers (per item and chunk they were the adjoint's main
  // shared-memory traffic: 3D, SN = 32 floats per item)
  constexpr int KH = HU ? 1 : (C::ITEMS + NT - 1) / NT;
  float ybr[KH][SN];
  if constexpr (HU) {
    const int pt = (tid >> 2) % PPT;
#pragma unroll
    for (int e = 0; e < SN; ++e) ybr[0][e] = Ybs[pt * SN + e];
  } else {
#pragma unroll
    for (int k = 0; k < KH; ++k) {
      const int i = tid + k * NT;
      if (i < C::ITEMS) {
        int pt, kq;
        C::fwd_item(i, pt, kq);
#pragma unroll
        for (int e = 0; e < SN; ++e) ybr[k][e] = Ybs[pt * SN + e];
      }
    }
  }
  for (int c = 0; c < nch; ++c) {
    const int g = nch + c, s = g % TC_HEAD_NS;
    float* slab = ring + s * SF;
    tc::mbar_wait(&full[s], (g / TC_HEAD_NS) & 1);
    if constexpr (HU) {
      for (int i = tid; i < 4 * C::ITEMS; i += NT) {
        const int j = i & 3, pt = (i >> 2) % PPT, kq = (i >> 2) / PPT;
        const float(&yb)[SN] = ybr[0];
        const float* w = WLs + (16 * c + 4 * kq + j) * NOUT;
        float zz[S], bb[S], sa[S];
        slab_load1x<C, QS>(zz, slab, pt, kq, j, pt & 7);
#pragma unroll
        for (int st = 0; st < S; ++st) {
          float v = 0.f;
#pragma unroll
          for (int o = 0; o < NOUT; ++o) v = fmaf(yb[st * NOUT + o], w[o], v);
          bb[st] = v;
        }
        tc_act_bwd1<C, ACT>(zz, bb, sa);
        float* rd = red + (kq * 4 + j) * NOUT * C::RSP + pt;
#pragma unroll
        for (int o = 0; o < NOUT; ++o) {
          float v = 0.f;
#pragma unroll
          for (int st = 0; st < S; ++st) v = fmaf(sa[st], yb[st * NOUT + o], v);
          rd[o * C::RSP] = v;
        }
        slab_store1x<C, QS>(slab, pt, kq, j, bb, pt & 7);  // Zbar_{L-1} in place of Z_{L-1}
      }
    } else
#pragma unroll
    for (int k = 0; k < KH; ++k) {
      const int i = tid + k * NT;
      if (i >= C::ITEMS) break;
      int pt, kq;
      C::fwd_item(i, pt, kq);
      const int q = 4 * c + kq;
      const float(&yb)[SN] = ybr[k];
      float z[S][4], sb[S][4];
      slab_load<C, QS>(z, slab, pt, kq);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float* w = WLs + (4 * q + j) * NOUT;
        float zz[S], bb[S], sa[S];
        col<C>(z, j, zz);
#pragma unroll
        for (int st = 0; st < S; ++st) {
          float v = 0.f;
#pragma unroll
          for (int o = 0; o < NOUT; ++o) v = fmaf(yb[st * NOUT + o], w[o], v);
          bb[st] = v;
        }
        tc_act_bwd1<C, ACT>(zz, bb, sa);
#pragma unroll
        for (int st = 0; st < S; ++st) sb[st][j] = bb[st];
        float* rd = red + j * NOUT * C::HRS + i;
#pragma unroll
        for (int o = 0; o < NOUT; ++o) {
          float v = 0.f;
#pragma unroll
          for (int st = 0; st < S; ++st) v = fmaf(sa[st], yb[st * NOUT + o], v);
          rd[o * C::HRS] = v;
        }
      }
      slab_store<C, QS>(slab, pt, kq, sb);  // Zbar_{L-1} in place of Z_{L-1}
    }
    __syncthreads();
    slab_copy_out<QS>(slab, static_cast<float*>(a.adj) + tc_off(a, L - 1, tile, 4 * c), tid);
    if (a.zt) slab_store_t<C, QS>(slab, a.zt + tc_toff(a, L - 1, tile), a.WP, 16 * c, tid);
    for (int e = tid; e < 16 * NOUT; e += NT) {
      const int kq = e / (4 * NOUT), j = (e / NOUT) % 4, o = e % NOUT;
      float acc = 0.f;
      for (int pt = 0; pt < PPT; ++pt)
        acc += HU ? red[((kq * 4 + j) * NOUT + o) * C::RSP + pt] : red[(j * NOUT + o) * C::HRS + C::item_of(pt, kq)];
      pL[size_t(16 * c + 4 * kq + j) * NOUT + o] = acc;
    }
    __syncthreads();
    if (tid == 0 && g + TC_HEAD_NS < ntot) produce(g + TC_HEAD_NS);
  }
}

// fixed-order reduction of per-tile partials into the gradient-partial rows:
// gpart[ks][off + (i / w) * wk + i % w] = sum over tiles t = ks, ks + KS, ... of
// P[t][i] (rows of w tensor-width entries land on rows of wk parameter-layout
// entries)
__global__ void __launch_bounds__(256) tcw_partials_kernel(const float* __restrict__ P, int len, long long ntiles,
                                                           double* gpart, int np_pad, int off, int w, int wk) {
  const int i = blockIdx.x * 256 + threadIdx.x, ks = blockIdx.y, KS = gridDim.y;
  if (i >= len) return;
  double acc = 0.0;
  long long t = ks;
  for (; t + 3 * KS < ntiles; t += 4 * KS) {
    const float v0 = P[size_t(t) * len + i], v1 = P[size_t(t + KS) * len + i];
    const float v2 = P[size_t(t + 2 * KS) * len + i], v3 = P[size_t(t + 3 * KS) * len + i];
    acc += double(v0);
    acc += double(v1);
    acc += double(v2);
    acc += double(v3);
  }
  for (; t < ntiles; t += KS) acc += double(P[size_t(t) * len + i]);
  gpart[size_t(ks) * np_pad + off + (i / w) * wk + i % w] = acc;
}

}  // namespace fr
