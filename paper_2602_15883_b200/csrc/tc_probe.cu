// Debug entry: one 128 x N x K TF32 GEMM through tcgen05 (TMEM accumulator),
// C[128][N] = A[128][K] * B[N][K]^T.  Validates the UMMA descriptor / TMEM /
// tcgen05.ld plumbing of tcgen05.cuh against a host matmul (tests/test_gpu_tc.py).
#include "flowrec_b200.h"
#include "jetmlp.cuh"
#include "tcgen05.cuh"
#include "tma.cuh"

namespace fr {

// k-quad staging: X[(k>>2)*(rows*4) + row*4 + (k&3)]
// layout bit 0: A MN-major, bit 1: B MN-major; bit 2: MN-major operands in the
// SWIZZLE_128B_BASE32B canonical layout (512-byte atoms of 4 K rows x 32 MN
// elements, 32-byte chunks XOR-swizzled by the row) instead of SWIZZLE_NONE;
// bit 3: swap the LBO / SBO roles of the BASE32B descriptor
__device__ __forceinline__ int b32_off(int mn, int k, int K) {
  // atoms [mn / 32][k / 4], 128 floats each
  const int atom = (mn >> 5) * (K >> 2) + (k >> 2), kr = k & 3, e = mn & 31;
  return atom * 128 + kr * 32 + ((((e >> 3) ^ kr) & 3) << 3) + (e & 7);
}
__global__ void __launch_bounds__(128) tc_probe_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                      float* __restrict__ C, int N, int K, int ncols, int layout) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tbase;
  float* As = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  float* Bs = As + 128 * K;
  const bool b32 = layout & 4;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * K; i += 128) {
    const int r = i / K, k = i % K;
    if (layout & 1) As[b32 ? b32_off(r, k, K) : (r >> 2) * (K * 4) + k * 4 + (r & 3)] = A[i];
    else As[(k >> 2) * 512 + r * 4 + (k & 3)] = A[i];
  }
  for (int i = tid; i < N * K; i += 128) {
    const int r = i / K, k = i % K;
    if (layout & 2) Bs[b32 ? b32_off(r, k, K) : (r >> 2) * (K * 4) + k * 4 + (r & 3)] = B[i];
    else Bs[(k >> 2) * (N * 4) + r * 4 + (k & 3)] = B[i];
  }
  if (warp == 0) {
    // allocation width must be a power of two >= 32 columns
    if (ncols <= 32) tc::tmem_alloc<32>(&tbase);
    else if (ncols <= 64) tc::tmem_alloc<64>(&tbase);
    else if (ncols <= 128) tc::tmem_alloc<128>(&tbase);
    else tc::tmem_alloc<256>(&tbase);
  }
  if (tid == 0) {
    tc::mbar_init(&mbar, 1);
    tc::fence_mbar_init();
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_tf32(128, N, layout & 1, (layout >> 1) & 1);
    // BASE32B: MN-group (32 elements) stride K/4 atoms, K-group (4 rows) stride one 512-byte atom
    const uint32_t mg = uint32_t(K / 4) * 512, kg = 512;
    const uint32_t b_lbo = (layout & 8) ? kg : mg, b_sbo = (layout & 8) ? mg : kg;
    for (int kk = 0; kk < K / 8; ++kk) {
      // K-major: LBO = K-chunk stride, SBO = 8-row stride; MN-major: LBO = 8-k stride, SBO = 4-row group stride
      uint64_t ad, bd;
      if (!(layout & 1)) ad = tc::desc(As + kk * 2 * 512, 512 * 4, 128);
      else if (b32) ad = tc::desc(As + kk * 256, b_lbo, b_sbo) | (uint64_t(1) << 61);
      else ad = tc::desc(As + kk * 32, 128, K * 16);
      if (!(layout & 2)) bd = tc::desc(Bs + kk * 2 * (N * 4), N * 16, 128);
      else if (b32) bd = tc::desc(Bs + kk * 256, b_lbo, b_sbo) | (uint64_t(1) << 61);
      else bd = tc::desc(Bs + kk * 32, 128, K * 16);
      tc::mma_tf32(tmem, ad, bd, idesc, kk > 0);
    }
    tc::mma_commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after();
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tc::tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + c0, v);
    for (int i = 0; i < 16; ++i) C[row * N + c0 + i] = v[i];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    if (ncols <= 32) tc::tmem_free<32>(tmem);
    else if (ncols <= 64) tc::tmem_free<64>(tmem);
    else if (ncols <= 128) tc::tmem_free<128>(tmem);
    else tc::tmem_free<256>(tmem);
  }
}

}  // namespace fr

extern "C" int fr_debug_tc_gemm_tf32(const float* A, const float* B, float* C, int N, int K, int layout,
                                     fr_stream_t stream) {
  if (N < 16 || N > 256 || N % 16 || K < 8 || K % 8 || K > 64) return -1;
  const size_t smem = sizeof(float) * size_t(128 + N) * K + 1024;
  if (cudaFuncSetAttribute(fr::tc_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) !=
      cudaSuccess)
    return -2;
  fr::tc_probe_kernel<<<1, 128, smem, (cudaStream_t)stream>>>(A, B, C, N, K, N, layout);
  ++fr::g_kernel_launches;
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// Layout discovery: A smem filled with its own word indices, B = identity
// (K-major), so C[m][k] reveals which shared-memory word the tensor core read
// for A(m, k) under the given descriptor strides (a_mn selects MN-major).
namespace fr {
__global__ void __launch_bounds__(128) tc_raw_kernel(float* __restrict__ C, int K, int a_mn, int lbo, int sbo) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tbase;
  constexpr int N = 32;
  float* As = sm;
  float* Bs = sm + 128 * K;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * K; i += 128) As[i] = float(i);
  for (int i = tid; i < N * K; i += 128) {
    const int r = i / K, k = i % K;
    Bs[(k >> 2) * (N * 4) + r * 4 + (k & 3)] = (r == k) ? 1.f : 0.f;
  }
  if (warp == 0) tc::tmem_alloc<32>(&tbase);
  if (tid == 0) {
    tc::mbar_init(&mbar, 1);
    tc::fence_mbar_init();
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    tc::mma_tf32(tmem, tc::desc(As, lbo, sbo), tc::desc(Bs, N * 16, 128), tc::idesc_tf32(128, N, a_mn, 0), 0);
    tc::mma_commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after();
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tc::tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + c0, v);
    for (int i = 0; i < 16; ++i) C[row * N + c0 + i] = v[i];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<32>(tmem);
}
}  // namespace fr

extern "C" int fr_debug_tc_raw(float* C, int K, int a_mn, int lbo, int sbo, fr_stream_t stream) {
  const size_t smem = sizeof(float) * size_t(128 + 32) * K;
  cudaFuncSetAttribute(fr::tc_raw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  fr::tc_raw_kernel<<<1, 128, smem, (cudaStream_t)stream>>>(C, K, a_mn, lbo, sbo);
  ++fr::g_kernel_launches;
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// Descriptor sweep: A smem (64 KB) holds ((word >> shift) & 1023) + 1, B = identity
// (K-major), so C[m][k] names the word read for A(m, k) under raw descriptor
// fields (layout type bits 61..63, a_mn selects MN-major).  Layout discovery only.
namespace fr {
__global__ void __launch_bounds__(128) tc_raw2_kernel(float* __restrict__ C, int a_mn, int lbo, int sbo, int ltype,
                                                      int shift) {
  extern __shared__ __align__(128) float sm2[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tbase;
  constexpr int N = 32, K = 8, AW = 16384;
  float* As = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(sm2) + 1023) & ~uintptr_t(1023));
  float* Bs = As + AW;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < AW; i += 128) As[i] = float(((i >> shift) & 1023) + 1);
  for (int i = tid; i < N * K; i += 128) {
    const int r = i / K, k = i % K;
    Bs[(k >> 2) * (N * 4) + r * 4 + (k & 3)] = (r == k) ? 1.f : 0.f;
  }
  if (warp == 0) tc::tmem_alloc<32>(&tbase);
  if (tid == 0) {
    tc::mbar_init(&mbar, 1);
    tc::fence_mbar_init();
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint64_t ad = tc::desc(As, lbo, sbo) | (uint64_t(ltype & 7) << 61);
    tc::mma_tf32(tmem, ad, tc::desc(Bs, N * 16, 128), tc::idesc_tf32(128, N, a_mn, 0), 0);
    tc::mma_commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after();
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tc::tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + c0, v);
    for (int i = 0; i < 16; ++i) C[row * N + c0 + i] = v[i];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<32>(tmem);
}
}  // namespace fr

extern "C" int fr_debug_tc_raw2(float* C, int a_mn, int lbo, int sbo, int ltype, int shift, fr_stream_t stream) {
  const size_t smem = sizeof(float) * size_t(16384 + 32 * 8) + 1024;
  cudaFuncSetAttribute(fr::tc_raw2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  fr::tc_raw2_kernel<<<1, 128, smem, (cudaStream_t)stream>>>(C, a_mn, lbo, sbo, ltype, shift);
  ++fr::g_kernel_launches;
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// TMA view probe (tests/test_gpu_tc.py): one 32-row group of a k-quad slab
// buffer [tiles][WP/4][128][4] through kquad_map, shared memory dumped
// linearly to dst.
namespace fr {
__global__ void __launch_bounds__(128) tma_probe_kernel(const __grid_constant__ CUtensorMap map, float* __restrict__ dst,
                                                        int WP, int tile, int g) {
  extern __shared__ __align__(128) unsigned char tp_smem[];
  float* sm = reinterpret_cast<float*>(tp_smem + ((1024u - (tc::smem_u32(tp_smem) & 1023u)) & 1023u));
  __shared__ __align__(8) uint64_t mbar;
  const int floats = 32 * WP;
  if (threadIdx.x == 0) {
    tc::mbar_init(&mbar, 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    tc::mbar_expect_tx(&mbar, uint32_t(floats) * 4);
    tc::tma_load3(sm, &map, 128 * g, 0, tile, &mbar);
  }
  tc::mbar_wait(&mbar, 0);
  for (int i = threadIdx.x; i < floats; i += 128) dst[i] = sm[i];
}
}  // namespace fr

extern "C" int fr_debug_tma_kquad(const float* src, float* dst, int WP, int ntiles, int tile, int g,
                                  fr_stream_t stream) {
  CUtensorMap m;
  if (fr::kquad_map(&m, src, WP, ntiles, 32, WP / 4)) return -10;
  const size_t smem = sizeof(float) * size_t(32 * WP) + 1024;
  cudaFuncSetAttribute(fr::tma_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  fr::tma_probe_kernel<<<1, 128, smem, (cudaStream_t)stream>>>(m, dst, WP, tile, g);
  ++fr::g_kernel_launches;
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}
