// FP32 pipe probe: FFMA vs packed FFMA2 (fma.rn.f32x2, scalar-broadcast form)
// throughput on this GPU.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma2 ffma2_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void ffma2s(u64& d, float a, u64 b) {
  u64 A = pk(a, a);
  asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(A), "l"(b));
}
__global__ void k_ffma(float* o, float s, int n) {
  float acc[32];
  for (int i = 0; i < 32; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  float a = s + threadIdx.x, b = s * 0.5f;
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = fmaf(a, acc[i], b);
  }
  float r = 0; for (int i = 0; i < 32; ++i) r += acc[i];
  o[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_ffma2(float* o, float s, int n) {
  u64 acc[16];
  for (int i = 0; i < 16; ++i) acc[i] = pk(threadIdx.x * 1e-3f + i, i);
  float a = s + threadIdx.x;
  u64 b = pk(s * 0.5f, s * 0.25f);
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) ffma2s(acc[i], a, b);
  }
  float r = 0;
  for (int i = 0; i < 16; ++i) { float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(acc[i])); r += x + y; }
  o[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
// GEMM-like: per k step 1 LDS.128 of A (4 rows) + 2 LDS.128 of B, 4x8 FMAs... with
// the same issue mix as gemm_rows (RPT=6 rows x 8 units per thread)
template <bool PACK>
__global__ void k_gemm(float* o, int n) {
  __shared__ __align__(16) float A[64 * 6 * 4 * 4];
  __shared__ __align__(16) float B[64 * 64];
  for (int i = threadIdx.x; i < 64 * 96; i += blockDim.x) A[i % (64 * 96)] = i * 1e-4f;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) B[i] = i * 1e-5f;
  __syncthreads();
  const int g = threadIdx.x % 8, rg = (threadIdx.x / 8) % 16;
  float acc[6][8] = {};
  u64 acc2[6][4];
  for (int r = 0; r < 6; ++r) for (int j = 0; j < 4; ++j) acc2[r][j] = 0ull;
  for (int it = 0; it < n; ++it) {
#pragma unroll 4
    for (int kq = 0; kq < 16; ++kq) {
      float av[24];
      const float4* ap = reinterpret_cast<const float4*>(A + kq * 384 + rg * 24);
#pragma unroll
      for (int q = 0; q < 6; ++q) { float4 v = ap[q]; av[4*q]=v.x; av[4*q+1]=v.y; av[4*q+2]=v.z; av[4*q+3]=v.w; }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const float4 b0 = *reinterpret_cast<const float4*>(B + (4 * kq + kk) * 64 + 4 * g);
        const float4 b1 = *reinterpret_cast<const float4*>(B + (4 * kq + kk) * 64 + 32 + 4 * g);
        if constexpr (PACK) {
          const u64 p0 = pk(b0.x, b0.y), p1 = pk(b0.z, b0.w), p2 = pk(b1.x, b1.y), p3 = pk(b1.z, b1.w);
#pragma unroll
          for (int r = 0; r < 6; ++r) {
            const float a = av[4 * r + kk];
            ffma2s(acc2[r][0], a, p0); ffma2s(acc2[r][1], a, p1); ffma2s(acc2[r][2], a, p2); ffma2s(acc2[r][3], a, p3);
          }
        } else {
          const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
          for (int r = 0; r < 6; ++r)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[r][j] = fmaf(av[4 * r + kk], bb[j], acc[r][j]);
        }
      }
    }
  }
  float r = 0;
  for (int i = 0; i < 6; ++i) for (int j = 0; j < 8; ++j) r += acc[i][j];
  for (int i = 0; i < 6; ++i) for (int j = 0; j < 4; ++j) { float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(acc2[i][j])); r += x + y; }
  o[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <typename F>
double timeit(F f, double flops) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) { cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
  return flops / (best * 1e-3) / 1e12;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* o; cudaMalloc(&o, sizeof(float) * sms * 8 * 1024);
  const int n = 20000, grid = sms * 4, nt = 256;
  printf("FFMA   %.1f TFLOP/s\n", timeit([&] { k_ffma<<<grid, nt>>>(o, 1.0f, n); }, 2.0 * grid * nt * 32.0 * n));
  printf("FFMA2  %.1f TFLOP/s\n", timeit([&] { k_ffma2<<<grid, nt>>>(o, 1.0f, n); }, 2.0 * grid * nt * 32.0 * n));
  const int ng = 400;
  for (int nt2 : {256, 384}) {
    const double fl = 2.0 * sms * nt2 * 48.0 * 64 * ng;
    printf("gemm-mix FFMA  nt=%d %.1f TFLOP/s\n", nt2, timeit([&] { k_gemm<false><<<sms, nt2>>>(o, ng); }, fl));
    printf("gemm-mix FFMA2 nt=%d %.1f TFLOP/s\n", nt2, timeit([&] { k_gemm<true><<<sms, nt2>>>(o, ng); }, fl));
  }
  return 0;
}
