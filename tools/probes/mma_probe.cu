// Legacy warp-level tensor-core throughput on this GPU (mma.sync, register
// operands): TF32 m16n8k8 and BF16 m16n8k16, independent accumulators.
// Decides whether a split-precision (3xTF32) W=64 contraction can beat the
// FP32 SIMT path without TMEM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma mma_probe.cu && /tmp/mma
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void k_tf32(float* o, int n) {
  float c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i)
    for (int j = 0; j < 4; ++j) c[i][j] = 0.f;
  unsigned a0 = __float_as_uint(1.0f + threadIdx.x * 1e-6f), a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  unsigned b0 = __float_as_uint(0.5f), b1 = b0 + 7;
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) r += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  o[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int NACC>
__global__ void k_bf16(float* o, int n) {
  float c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i)
    for (int j = 0; j < 4; ++j) c[i][j] = 0.f;
  unsigned a0 = 0x3f803f80u + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  unsigned b0 = 0x3f003f00u, b1 = b0 + 7;
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) r += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  o[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <typename K>
static void run(const char* name, K k, double flops_per_mma, int nacc, int threads) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 4, n = 20000;
  float* o;
  cudaMalloc(&o, sizeof(float) * grid * threads);
  k<<<grid, threads>>>(o, 100);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<grid, threads>>>(o, n);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double mmas = double(grid) * (threads / 32) * n * nacc;
  printf("%-28s threads %4d: %8.1f TFLOP/s (%.3f ms)\n", name, threads, mmas * flops_per_mma / (ms * 1e-3) / 1e12, ms);
  cudaFree(o);
}

int main() {
  for (int t : {128, 256, 512}) {
    run("mma.sync tf32 m16n8k8", k_tf32<8>, 2.0 * 16 * 8 * 8, 8, t);
    run("mma.sync bf16 m16n8k16", k_bf16<8>, 2.0 * 16 * 8 * 16, 8, t);
  }
  return 0;
}
