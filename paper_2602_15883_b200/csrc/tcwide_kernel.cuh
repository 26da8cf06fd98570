// Tensor-core (tcgen05, TF32) layer-wise kernels for wide experts.
//
// Same chain as the SIMT wide path (wide_kernel.cuh) but every hidden-layer
// contraction -- forward S_{l-1} W_l, adjoint Zbar_l W_l^T and weight gradient
// S_{l-1}^T Zbar_l -- runs as 128 x NB x 8 tcgen05.mma.kind::tf32 steps with the
// accumulator in TMEM.  All operands are K-major SWIZZLE_NONE UMMA tiles
// (TF32 MN-major descriptors read zeros on sm_100a, see tools/tc_layout_probe.py).
//
// Tile geometry.  A tile is one 128-row MMA block: four 32-row groups, each
// holding PPW = 32/S points x S jet streams (rows p*S+s) plus 32 - PPW*S pad
// rows.  Pad rows are never read by the per-point code; the dW kernel zeroes
// them before they reach the tensor core.
//
// HBM buffers (fp32, k-quad layout [layer][tile][WP/4][128][4], one quad of a
// tile = 2 KB contiguous = a K-major 128 x 4 operand slab):
//   Z    pre-activation jets of layers 1..L-1 (layer 0 is recomputed from the
//        points on the fly: z_v = x W0 + b0, z_g = W0 rows, z_l = 0)
//   Zbar their adjoints, layers 0..L-1
//   ybar output-layer adjoints [tile][128][NOUT]
// The activation sigma(Z) is applied by the CONSUMER (the next layer's operand
// staging, the head, and the dW staging) so only Z is ever written:
// fwd moves 2 x 128 x WP x 4 B per tile-layer instead of 3.
#pragma once
#include "tcgen05.cuh"
#include "wide_kernel.cuh"

namespace fr {

template <int ACT, int MODE, int REG>
struct TcCfg {
  using R = Regime<REG>;
  using St = Streams<MODE, REG>;
  static constexpr int DIN = R::DIN, NOUT = R::NOUT, NVEL = R::NVEL;
  static constexpr int S = St::S, NG = St::NG, NL = St::NL, LAP0 = St::LAP0;
  static constexpr bool JET = St::JET;
  static constexpr int SIN = (ACT == ACT_SIN) ? 1 : 0;
  static constexpr int NT = 128;              // fwd / dx / head CTAs (one thread per TMEM lane)
  static constexpr int DW_NT = 256;           // dW CTAs
  static constexpr int PPW = 32 / S;          // points per 32-row group
  static constexpr int PPT = 4 * PPW;         // points per tile
  static constexpr int VR = PPW * S;          // valid rows per 32-row group
  static constexpr int KC = 32, NQ = KC / 4;  // K chunk = 8 quads
  static constexpr int QS = NT / PPT;         // head: threads per point
  static constexpr int ZRS = 32 * 4 + 4;      // dW Z staging row stride (words, conflict-free)
  __host__ __device__ static constexpr int row0(int pt) { return (pt / PPW) * 32 + (pt % PPW) * S; }
  __host__ __device__ static size_t gemm_smem(int NB) { return sizeof(float) * size_t(2 * NQ * 512 + 2 * NQ * NB * 4); }
  __host__ __device__ static size_t dw_smem(int NB) {
    return sizeof(float) * size_t(32 * ZRS + 2 * 8 * 128 * 4 + 2 * 8 * NB * 4);
  }
  __host__ __device__ static size_t head_smem(int WP) {
    return sizeof(float) * size_t(WP * NOUT + PPT * QS * S * NOUT + 2 * PPT * S * NOUT) + 2 * NT * sizeof(double);
  }
};

__device__ __forceinline__ size_t tc_off(const WArgs& a, int l, long long tile, int q) {
  return ((size_t(l) * a.ntiles + tile) * (a.WP / 4) + q) * 512;
}

// pre-activation jets of point pt (tile-local), unit quad q, of hidden layer l
template <class C>
__device__ __forceinline__ void tc_load_z(const WArgs& a, const float* __restrict__ kp, const ParamLayout& pl,
                                          int l, long long tile, int pt, int q, float (&z)[C::S][4]) {
  if (l == 0) {
    const long long p = tile * C::PPT + pt;
    const float* pts = static_cast<const float*>(a.pts);
    float x[C::DIN];
#pragma unroll
    for (int i = 0; i < C::DIN; ++i) x[i] = p < a.n ? pts[p * C::DIN + i] : 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int u = 4 * q + j;
      float zv = 0.f;
#pragma unroll
      for (int i = 0; i < C::DIN; ++i) zv = fmaf(x[i], kp[pl.off_w(0) + i * a.WP + u], zv);
      z[0][j] = zv + kp[pl.off_b(0) + u];
      if constexpr (C::JET) {
#pragma unroll
        for (int i = 0; i < C::NG; ++i) z[1 + i][j] = kp[pl.off_w(0) + i * a.WP + u];
#pragma unroll
        for (int i = 0; i < C::NL; ++i) z[1 + C::NG + i][j] = 0.f;
      }
    }
  } else {
    const float* b = static_cast<const float*>(a.act) + tc_off(a, l, tile, q) + C::row0(pt) * 4;
#pragma unroll
    for (int s = 0; s < C::S; ++s) vload(z[s], b + 4 * s);
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

// activation adjoint of one point / unit (in place: sb = S-bar -> Z-bar)
template <class C, int ACT>
__device__ __forceinline__ void tc_act_bwd1(const float (&z)[C::S], float (&sb)[C::S]) {
  constexpr int NG = C::NG, NL = C::NL, LAP0 = C::LAP0;
  float s, c, d1, d2;
  act_eval<ACT>(z[0], s, c);
  act_d12<ACT>(s, c, d1, d2);
  if constexpr (C::JET) {
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

template <class C, int ACT>
__device__ __forceinline__ void tc_act4(const float (&z)[C::S][4], float (&s)[C::S][4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float zz[C::S], ss[C::S];
#pragma unroll
    for (int k = 0; k < C::S; ++k) zz[k] = z[k][j];
    tc_act1<C, ACT>(zz, ss);
#pragma unroll
    for (int k = 0; k < C::S; ++k) s[k][j] = ss[k];
  }
}
template <class C, int ACT>
__device__ __forceinline__ void tc_act_bwd4(const float (&z)[C::S][4], float (&sb)[C::S][4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float zz[C::S], bb[C::S];
#pragma unroll
    for (int k = 0; k < C::S; ++k) {
      zz[k] = z[k][j];
      bb[k] = sb[k][j];
    }
    tc_act_bwd1<C, ACT>(zz, bb);
#pragma unroll
    for (int k = 0; k < C::S; ++k) sb[k][j] = bb[k];
  }
}

// TMEM allocation + mbarrier init (CTA-wide; every thread calls)
template <int NCOLS>
__device__ __forceinline__ uint32_t tc_setup(uint32_t* slot, uint64_t* mbar, int nbar) {
  if (threadIdx.x < 32) tc::tmem_alloc<NCOLS>(slot);
  if (threadIdx.x == 0) {
    for (int i = 0; i < nbar; ++i) tc::mbar_init(&mbar[i], 1);
    tc::fence_mbar_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  return *slot;
}
template <int NCOLS>
__device__ __forceinline__ void tc_teardown(uint32_t tmem) {
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_free<NCOLS>(tmem);
}

// stage rows n0..n0+NB-1, columns [k0, k0+32) of a row-major matrix (row
// length ld) as a K-major operand B[kq][NB][4]
__device__ __forceinline__ void tc_stage_b(float* B, const float* __restrict__ M, int ld, int n0, int k0, int NB,
                                           int tid, int nt) {
  for (int i = tid; i < NB * 8; i += nt) {
    const int nlo = i & 7, kq = (i >> 3) & 7, n = (i >> 6) * 8 + nlo;
    cp_async16(B + (kq * NB + n) * 4, M + size_t(n0 + n) * ld + k0 + 4 * kq);
  }
}

// issue the 4 K-steps of one 32-deep chunk (A[kq][MA][4], B[kq][NB][4])
__device__ __forceinline__ void tc_mma_chunk(uint32_t tmem, const float* A, int MA, const float* B, int NB,
                                             uint32_t idesc, bool first) {
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
    tc::mma_tf32(tmem, tc::desc(A + kk * 8 * MA, MA * 16, 128), tc::desc(B + kk * 8 * NB, NB * 16, 128), idesc,
                 (!first || kk) ? 1u : 0u);
}

// ---------------------------------------------------------------------------
// forward, hidden layer l >= 1: Z_l = sigma(Z_{l-1}) W_l + b_l
// grid (tiles, WP/NB), 128 threads
// ---------------------------------------------------------------------------
template <int ACT, int MODE, int REG>
__global__ void __launch_bounds__(128) tcw_fwd_kernel(WArgs a, int l, int NB) {
  using C = TcCfg<ACT, MODE, REG>;
  extern __shared__ __align__(128) unsigned char tc_smem[];
  float* Ab = reinterpret_cast<float*>(tc_smem);  // [2][8][128][4]
  float* Bb = Ab + 2 * C::NQ * 512;                // [2][8][NB][4]
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long tile = blockIdx.x;
  const int n0 = blockIdx.y * NB;
  const float* kp = static_cast<const float*>(a.kp);
  const ParamLayout pl{C::DIN, a.WP, C::NOUT, a.L};
  const uint32_t tmem = tc_setup<256>(&tslot, mbar, 2);
  const int nch = a.WP / C::KC;
  const uint32_t idesc = tc::idesc_tf32(128, NB);
  for (int c = 0; c < nch; ++c) {
    const int b = c & 1;
    if (c >= 2) tc::mbar_wait(&mbar[b], ((c - 2) >> 1) & 1);
    float* A = Ab + b * C::NQ * 512;
    float* B = Bb + b * C::NQ * NB * 4;
    tc_stage_b(B, kp + pl.off_wt(l), a.WP, n0, c * C::KC, NB, tid, C::NT);
    cp_async_commit();
    for (int i = tid; i < C::PPT * C::NQ; i += C::NT) {
      const int pt = i % C::PPT, kq = i / C::PPT;
      float z[C::S][4], s[C::S][4];
      tc_load_z<C>(a, kp, pl, l - 1, tile, pt, c * C::NQ + kq, z);
      tc_act4<C, ACT>(z, s);
      float* d = A + kq * 512 + C::row0(pt) * 4;
#pragma unroll
      for (int st = 0; st < C::S; ++st) vstore(d + 4 * st, s[st]);
    }
    cp_async_wait_all();
    tc::fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after();
      tc_mma_chunk(tmem, A, 128, B, NB, idesc, c == 0);
      tc::mma_commit(&mbar[b]);
    }
  }
  tc::mbar_wait(&mbar[(nch - 1) & 1], ((nch - 1) >> 1) & 1);
  tc::fence_after();
  const int r = warp * 32 + lane;
  const bool vrow = lane < C::VR && (lane % C::S) == 0;
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
  tc_teardown<256>(tmem);
}

// ---------------------------------------------------------------------------
// adjoint, hidden layer l >= 1: Zbar_{l-1} = act_bwd(Z_{l-1}, Zbar_l W_l^T)
// grid (tiles, WP/NB), 128 threads
// ---------------------------------------------------------------------------
template <int ACT, int MODE, int REG>
__global__ void __launch_bounds__(128) tcw_dx_kernel(WArgs a, int l, int NB) {
  using C = TcCfg<ACT, MODE, REG>;
  extern __shared__ __align__(128) unsigned char tc_smem[];
  float* Ab = reinterpret_cast<float*>(tc_smem);
  float* Bb = Ab + 2 * C::NQ * 512;
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long tile = blockIdx.x;
  const int n0 = blockIdx.y * NB;
  const float* kp = static_cast<const float*>(a.kp);
  const ParamLayout pl{C::DIN, a.WP, C::NOUT, a.L};
  const uint32_t tmem = tc_setup<256>(&tslot, mbar, 2);
  const int nch = a.WP / C::KC;
  const uint32_t idesc = tc::idesc_tf32(128, NB);
  const float* zb = static_cast<const float*>(a.adj) + tc_off(a, l, tile, 0);
  for (int c = 0; c < nch; ++c) {
    const int b = c & 1;
    if (c >= 2) tc::mbar_wait(&mbar[b], ((c - 2) >> 1) & 1);
    float* A = Ab + b * C::NQ * 512;
    float* B = Bb + b * C::NQ * NB * 4;
    tc_stage_b(B, kp + pl.off_w(l), a.WP, n0, c * C::KC, NB, tid, C::NT);
    const float* src = zb + size_t(c) * C::NQ * 512;
    for (int i = tid; i < C::NQ * 128; i += C::NT) cp_async16(A + 4 * i, src + 4 * i);
    cp_async_commit();
    cp_async_wait_all();
    tc::fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after();
      tc_mma_chunk(tmem, A, 128, B, NB, idesc, c == 0);
      tc::mma_commit(&mbar[b]);
    }
  }
  tc::mbar_wait(&mbar[(nch - 1) & 1], ((nch - 1) >> 1) & 1);
  tc::fence_after();
  // S-bar columns in chunks of 32 through shared memory (point-major act-bwd)
  float* stg = Ab;  // [8][128][4]
  const int r = warp * 32 + lane;
  for (int c0 = 0; c0 < NB; c0 += 32) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float v[16];
      tc::tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + c0 + 16 * h, v);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float4*>(stg + (4 * h + q) * 512 + r * 4) =
            make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
    __syncthreads();
    for (int i = tid; i < C::PPT * C::NQ; i += C::NT) {
      const int pt = i % C::PPT, kq = i / C::PPT;
      const int q = (n0 + c0) / 4 + kq;
      float z[C::S][4], sb[C::S][4];
      tc_load_z<C>(a, kp, pl, l - 1, tile, pt, q, z);
      const float* sp = stg + kq * 512 + C::row0(pt) * 4;
#pragma unroll
      for (int st = 0; st < C::S; ++st) vload(sb[st], sp + 4 * st);
      tc_act_bwd4<C, ACT>(z, sb);
      float* d = static_cast<float*>(a.adj) + tc_off(a, l - 1, tile, q) + C::row0(pt) * 4;
#pragma unroll
      for (int st = 0; st < C::S; ++st) vstore(d + 4 * st, sb[st]);
    }
    __syncthreads();
  }
  tc_teardown<256>(tmem);
}

// ---------------------------------------------------------------------------
// dW_l = sum_rows sigma(Z_{l-1})^T Zbar_l, db_l = sum of value rows of Zbar_l.
// grid (ceil(WP/128) k-blocks, WP/NB u-blocks, KS row splits), 256 threads.
// Per 32-row group: threads 0..127 (one per input unit k) apply the jet
// activation point by point and write their column K-major ([row quad][k][4]);
// threads 128..255 transpose Zbar 4x4 blocks into [row quad][u][4].
// ---------------------------------------------------------------------------
template <int ACT, int MODE, int REG>
__global__ void __launch_bounds__(256) tcw_dw_kernel(WArgs a, int l, int NB) {
  using C = TcCfg<ACT, MODE, REG>;
  constexpr int S = C::S, ZRS = C::ZRS;
  extern __shared__ __align__(128) unsigned char tc_smem[];
  float* As = reinterpret_cast<float*>(tc_smem);  // [2][8][128][4]
  float* Bs = As + 2 * 8 * 512;                    // [2][8][NB][4]
  float* Zs = Bs + 2 * 8 * NB * 4;                 // [32 quads][ZRS]
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kb = blockIdx.x, n0 = blockIdx.y * NB, split = blockIdx.z;
  const float* kp = static_cast<const float*>(a.kp);
  const ParamLayout pl{C::DIN, a.WP, C::NOUT, a.L};
  const uint32_t tmem = tc_setup<256>(&tslot, mbar, 2);
  const uint32_t idesc = tc::idesc_tf32(128, NB);
  const int kq0 = kb * 32;                                   // first input-unit quad of this block
  const int nkq = min(32, a.WP / 4 - kq0);                   // valid quads in the block
  const int k = kb * 128 + tid;                              // A producer's input unit (tid < 128)
  float db4[4] = {0.f, 0.f, 0.f, 0.f};
  int ci = 0;
  for (long long t = split; t < a.ntiles; t += gridDim.z) {
    for (int g = 0; g < 4; ++g, ++ci) {
      const int b = ci & 1;
      if (ci >= 2) tc::mbar_wait(&mbar[b], ((ci - 2) >> 1) & 1);
      float* A = As + b * 8 * 512;
      float* B = Bs + b * 8 * NB * 4;
      if (l - 1 >= 1) {
        const float* zsrc = static_cast<const float*>(a.act) + tc_off(a, l - 1, t, kq0) + g * 128;
        for (int i = tid; i < nkq * 32; i += C::DW_NT) {
          const int kq = i >> 5, rr = i & 31;
          cp_async16(Zs + kq * ZRS + rr * 4, zsrc + size_t(kq) * 512 + rr * 4);
        }
        cp_async_commit();
      }
      if (tid >= 128) {
        // Zbar rows g*32.. of this tile, unit quads n0/4 .. +NB/4: 4x4 transposes
        const float* zb = static_cast<const float*>(a.adj) + tc_off(a, l, t, n0 / 4) + g * 128;
        for (int i = tid - 128; i < (NB / 4) * 8; i += 128) {
          const int uq = i % (NB / 4), rq = i / (NB / 4);
          float m[4][4];
#pragma unroll
          for (int rr = 0; rr < 4; ++rr) {
            const int row = 4 * rq + rr;
            if (row < C::VR) {
              vload(m[rr], zb + size_t(uq) * 512 + row * 4);
            } else {
#pragma unroll
              for (int j = 0; j < 4; ++j) m[rr][j] = 0.f;
            }
          }
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<float4*>(B + (rq * NB + 4 * uq + j) * 4) = make_float4(m[0][j], m[1][j], m[2][j], m[3][j]);
        }
        // db_l: one fixed unit quad per thread, value rows in point order
        if (kb == 0 && tid - 128 < NB / 4)
          for (int pp = 0; pp < C::PPW; ++pp) {
            float v[4];
            vload(v, zb + size_t(tid - 128) * 512 + pp * S * 4);
#pragma unroll
            for (int j = 0; j < 4; ++j) db4[j] += v[j];
          }
      }
      if (l - 1 >= 1) cp_async_wait_all();
      __syncthreads();
      if (tid < 128) {
        float col[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) col[i] = 0.f;
        if (k < a.WP) {
#pragma unroll
          for (int pp = 0; pp < C::PPW; ++pp) {
            float z[S], s[S];
            if (l - 1 >= 1) {
#pragma unroll
              for (int st = 0; st < S; ++st) z[st] = Zs[(tid >> 2) * ZRS + (pp * S + st) * 4 + (tid & 3)];
            } else {
              const long long p = t * C::PPT + g * C::PPW + pp;
              const float* pts = static_cast<const float*>(a.pts);
              float zv = 0.f;
#pragma unroll
              for (int i = 0; i < C::DIN; ++i) zv = fmaf(p < a.n ? pts[p * C::DIN + i] : 0.f, kp[pl.off_w(0) + i * a.WP + k], zv);
              z[0] = zv + kp[pl.off_b(0) + k];
              if constexpr (C::JET) {
#pragma unroll
                for (int i = 0; i < C::NG; ++i) z[1 + i] = kp[pl.off_w(0) + i * a.WP + k];
#pragma unroll
                for (int i = 0; i < C::NL; ++i) z[1 + C::NG + i] = 0.f;
              }
            }
            tc_act1<C, ACT>(z, s);
#pragma unroll
            for (int st = 0; st < S; ++st) col[pp * S + st] = s[st];
          }
        }
#pragma unroll
        for (int rq = 0; rq < 8; ++rq)
          *reinterpret_cast<float4*>(A + (rq * 128 + tid) * 4) =
              make_float4(col[4 * rq], col[4 * rq + 1], col[4 * rq + 2], col[4 * rq + 3]);
      }
      tc::fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after();
        tc_mma_chunk(tmem, A, 128, B, NB, idesc, ci == 0);
        tc::mma_commit(&mbar[b]);
      }
    }
  }
  double* gp = a.gpart + size_t(split) * a.np_pad;
  if (kb == 0 && ci > 0 && tid >= 128 && tid - 128 < NB / 4)
#pragma unroll
    for (int j = 0; j < 4; ++j) gp[pl.off_b(l) + n0 + 4 * (tid - 128) + j] = double(db4[j]);
  if (ci > 0) {
    tc::mbar_wait(&mbar[(ci - 1) & 1], ((ci - 1) >> 1) & 1);
    tc::fence_after();
    // warps w and w+4 share TMEM lane quadrant w: column halves
    const int quad = warp & 3, half = warp >> 2;
    const int kr = kb * 128 + quad * 32 + lane;
    for (int c0 = half * 16; c0 < NB; c0 += 32) {
      float v[16];
      tc::tmem_ld16(tmem + (uint32_t(quad * 32) << 16) + c0, v);
      if (kr < a.WP) {
        double* dst = gp + pl.off_w(l) + size_t(kr) * a.WP + n0 + c0;
#pragma unroll
        for (int i = 0; i < 16; ++i) dst[i] = double(v[i]);
      }
    }
  }
  tc_teardown<256>(tmem);
}

// ---------------------------------------------------------------------------
// head: output layer + residual / MSE + Ybar + S-bar_{L-1} + act-bwd -> Zbar_{L-1}
// grid tiles, 128 threads: QS threads per point split the WP/4 unit quads
// ---------------------------------------------------------------------------
template <int ACT, int MODE, int REG>
__global__ void __launch_bounds__(128) tcw_head_kernel(WArgs a) {
  using C = TcCfg<ACT, MODE, REG>;
  constexpr int NT = C::NT, PPT = C::PPT, NOUT = C::NOUT, NVEL = C::NVEL, S = C::S, QS = C::QS;
  constexpr int NG = C::NG, LAP0 = C::LAP0, SN = S * NOUT;
  extern __shared__ __align__(128) unsigned char tc_smem[];
  double* red = reinterpret_cast<double*>(tc_smem);  // [2][NT]
  float* WLs = reinterpret_cast<float*>(red + 2 * NT);  // [WP][NOUT]
  float* Yp = WLs + a.WP * NOUT;                        // [PPT*QS][SN]
  float* Ys = Yp + PPT * QS * SN;                       // [PPT][SN]
  float* Ybs = Ys + PPT * SN;                           // [PPT][SN]
  const long long tile = blockIdx.x;
  const int tid = threadIdx.x, pt = tid / QS, qs = tid % QS;
  const bool active = tid < PPT * QS;
  const float* kp = static_cast<const float*>(a.kp);
  const ParamLayout pl{C::DIN, a.WP, NOUT, a.L};
  const int L = a.L, NQW = a.WP / 4;
  for (int i = tid; i < a.WP * NOUT; i += NT) WLs[i] = kp[pl.off_w(L) + i];
  __syncthreads();
  if (active) {
    float y[S][NOUT];
#pragma unroll
    for (int st = 0; st < S; ++st)
#pragma unroll
      for (int c = 0; c < NOUT; ++c) y[st][c] = 0.f;
    for (int q = qs; q < NQW; q += QS) {
      float z[S][4], s[S][4];
      tc_load_z<C>(a, kp, pl, L - 1, tile, pt, q, z);
      tc_act4<C, ACT>(z, s);
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int c = 0; c < NOUT; ++c) {
          const float w = WLs[(4 * q + j) * NOUT + c];
#pragma unroll
          for (int st = 0; st < S; ++st) y[st][c] = fmaf(s[st][j], w, y[st][c]);
        }
    }
#pragma unroll
    for (int st = 0; st < S; ++st)
#pragma unroll
      for (int c = 0; c < NOUT; ++c) Yp[tid * SN + st * NOUT + c] = y[st][c];
  }
  __syncthreads();
  const long long p0 = tile * PPT, rem = a.n - p0;
  double lacc0 = 0.0, lacc1 = 0.0;
  if (active && qs == 0) {
    float* y = Ys + pt * SN;
    float* yb = Ybs + pt * SN;
    for (int i = 0; i < SN; ++i) {
      float v = 0.f;
      for (int h = 0; h < QS; ++h) v += Yp[(pt * QS + h) * SN + i];
      y[i] = (i < NOUT) ? v + kp[pl.off_b(L) + i] : v;
      yb[i] = 0.f;
    }
    if (pt < rem) {
      if constexpr (MODE == MODE_PDE) {
        using Rg = Regime<REG>;
        constexpr int NSP = Rg::NSP, TOFF = Rg::HAS_T, P = NVEL;
        const float inv_re = float(a.inv_re), two_coef = float(2.0 * a.coef);
        auto Y = [&](int s, int c) { return y[s * NOUT + c]; };
        auto GRAD = [&](int in) { return 1 + in; };
        auto LAP = [&](int in) { return 1 + NG + (in - LAP0); };
        float r[NVEL + 1];
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
          r[i] = acc;
        }
        {
          float acc = Y(GRAD(TOFF), 0);
#pragma unroll
          for (int kk = 1; kk < NVEL; ++kk) acc += Y(GRAD(TOFF + kk), kk);
          r[NVEL] = acc;
        }
#pragma unroll
        for (int i = 0; i <= NVEL; ++i) lacc0 += double(r[i]) * double(r[i]);
#pragma unroll
        for (int i = 0; i < NVEL; ++i) {
          const float rb = two_coef * r[i];
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
        const float rb = two_coef * r[NVEL];
#pragma unroll
        for (int kk = 0; kk < NVEL; ++kk) yb[GRAD(TOFF + kk) * NOUT + kk] += rb;
      } else {  // MSE
        const float two_vc = float(2.0 * a.coef), two_pc = float(2.0 * a.pcoef);
        const float* tu = static_cast<const float*>(a.tu) + (p0 + pt) * NVEL;
#pragma unroll
        for (int c = 0; c < NVEL; ++c) {
          const float d = y[c] - tu[c];
          lacc0 += a.velw[c] * (double(d) * double(d));
          yb[c] = (two_vc * float(a.velw[c])) * d;
        }
        if (a.has_p) {
          const float d = y[NVEL] - static_cast<const float*>(a.tp)[p0 + pt];
          lacc1 += double(d) * double(d);
          yb[NVEL] = two_pc * d;
        }
      }
    }
    float* yout = static_cast<float*>(a.ybar) + (size_t(tile) * 128 + C::row0(pt)) * NOUT;
    for (int i = 0; i < SN; ++i) yout[i] = yb[i];
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
  if (!active) return;
  const float* yb = Ybs + pt * SN;
  for (int q = qs; q < NQW; q += QS) {
    float z[S][4], sb[S][4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int st = 0; st < S; ++st) {
        float v = 0.f;
#pragma unroll
        for (int c = 0; c < NOUT; ++c) v = fmaf(yb[st * NOUT + c], WLs[(4 * q + j) * NOUT + c], v);
        sb[st][j] = v;
      }
    tc_load_z<C>(a, kp, pl, L - 1, tile, pt, q, z);
    tc_act_bwd4<C, ACT>(z, sb);
    float* d = static_cast<float*>(a.adj) + tc_off(a, L - 1, tile, q) + C::row0(pt) * 4;
#pragma unroll
    for (int st = 0; st < S; ++st) vstore(d + 4 * st, sb[st]);
  }
}

// dW_L, db_L from sigma(Z_{L-1}) and Ybar; grid KS, one unit quad per thread
template <int ACT, int MODE, int REG>
__global__ void __launch_bounds__(128) tcw_dwL_kernel(WArgs a) {
  using C = TcCfg<ACT, MODE, REG>;
  constexpr int NOUT = C::NOUT, S = C::S;
  const int ks = blockIdx.x, tid = threadIdx.x;
  const float* kp = static_cast<const float*>(a.kp);
  const ParamLayout pl{C::DIN, a.WP, NOUT, a.L};
  double* gp = a.gpart + size_t(ks) * a.np_pad;
  const int q = tid;
  const bool active = q < a.WP / 4;
  float acc[4][NOUT], db[NOUT];
#pragma unroll
  for (int c = 0; c < NOUT; ++c) {
    db[c] = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j][c] = 0.f;
  }
  int since = 0;
  auto flush = [&]() {
    if (active)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int c = 0; c < NOUT; ++c) {
          red_add(gp + pl.off_w(a.L) + (4 * q + j) * NOUT + c, double(acc[j][c]));
          acc[j][c] = 0.f;
        }
    if (tid == 0)
#pragma unroll
      for (int c = 0; c < NOUT; ++c) {
        red_add(gp + pl.off_b(a.L) + c, double(db[c]));
        db[c] = 0.f;
      }
  };
  for (long long t = ks; t < a.ntiles; t += gridDim.x) {
    const float* ybt = static_cast<const float*>(a.ybar) + size_t(t) * 128 * NOUT;
    if (active) {
      for (int pt = 0; pt < C::PPT; ++pt) {
        float z[S][4], s[S][4];
        tc_load_z<C>(a, kp, pl, a.L - 1, t, pt, q, z);
        tc_act4<C, ACT>(z, s);
        const float* yb = ybt + C::row0(pt) * NOUT;
#pragma unroll
        for (int st = 0; st < S; ++st)
#pragma unroll
          for (int c = 0; c < NOUT; ++c) {
            const float y = yb[st * NOUT + c];
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j][c] = fmaf(s[st][j], y, acc[j][c]);
          }
      }
    }
    if (tid == 0)
      for (int pt = 0; pt < C::PPT; ++pt)
#pragma unroll
        for (int c = 0; c < NOUT; ++c) db[c] += ybt[C::row0(pt) * NOUT + c];
    if (++since == 8) {
      flush();
      since = 0;
    }
  }
  if (since) flush();
}

// dW_0, db_0 from the points and Zbar_0; grid (KS, ceil(WP/128)), one unit per thread
template <int ACT, int MODE, int REG>
__global__ void __launch_bounds__(128) tcw_dw0_kernel(WArgs a) {
  using C = TcCfg<ACT, MODE, REG>;
  constexpr int DIN = C::DIN;
  const int ks = blockIdx.x, u = threadIdx.x + blockIdx.y * 128;
  const ParamLayout pl{DIN, a.WP, C::NOUT, a.L};
  double* gp = a.gpart + size_t(ks) * a.np_pad;
  if (u >= a.WP) return;
  float acc[DIN + 1];
#pragma unroll
  for (int j = 0; j <= DIN; ++j) acc[j] = 0.f;
  int since = 0;
  auto flush = [&]() {
#pragma unroll
    for (int j = 0; j < DIN; ++j) {
      red_add(gp + pl.off_w(0) + j * a.WP + u, double(acc[j]));
      acc[j] = 0.f;
    }
    red_add(gp + pl.off_b(0) + u, double(acc[DIN]));
    acc[DIN] = 0.f;
  };
  const float* pts = static_cast<const float*>(a.pts);
  for (long long t = ks; t < a.ntiles; t += gridDim.x) {
    const float* Z = static_cast<const float*>(a.adj) + tc_off(a, 0, t, u / 4) + (u % 4);
    const long long p0 = t * C::PPT;
    for (int pt = 0; pt < C::PPT && p0 + pt < a.n; ++pt) {
      const int row = C::row0(pt);
      const float zv = Z[4 * row];
#pragma unroll
      for (int j = 0; j < DIN; ++j) {
        acc[j] = fmaf(pts[(p0 + pt) * DIN + j], zv, acc[j]);
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
