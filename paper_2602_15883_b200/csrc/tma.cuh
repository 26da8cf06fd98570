// Tensor-map TMA (cp.async.bulk.tensor) for the wide kernels' k-quad activation
// slabs.  A slab buffer is [layer * tiles][WP/4 quads][128 rows][4 units] fp32,
// viewed as the 3-D tensor {512 floats of a quad, WP/4 quads, layer * tiles};
// a box {4 * rows, quads, 1} at element offset 4 * row0 lands `rows` rows of
// `quads` consecutive quads as the [quad][rows][4] k-quad stage, each quad's
// rows one contiguous run (512 bytes for 32 rows).  (A transposing view -- quads
// before rows with the 128B_ATOM_32B swizzle, which would land the BASE32B
// MN-major operand directly -- encodes but faults: TMA needs nested strides.)
// The encoder comes from the driver through cudaGetDriverEntryPoint (no -lcuda).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fr {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn tma_encoder() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return EncodeTiledFn(nullptr);
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// returns 0 on success
inline int kquad_map(CUtensorMap* m, const void* base, int WP, long long slabs, int box_rows, int box_quads) {
  EncodeTiledFn enc = tma_encoder();
  if (!enc) return 1;
  const cuuint64_t dims[3] = {512, cuuint64_t(WP / 4), cuuint64_t(slabs)};
  const cuuint64_t strides[2] = {2048, cuuint64_t(WP) * 512};
  const cuuint32_t box[3] = {cuuint32_t(4 * box_rows), cuuint32_t(box_quads), 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
             ? 0
             : 2;
}

namespace tc {
// 3-D tensor copy global -> shared, completes its bytes on mbar
__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* map, int c0, int c1, int c2, void* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2),
      "r"(static_cast<uint32_t>(__cvta_generic_to_shared(mbar)))
      : "memory");
}
}  // namespace tc
}  // namespace fr
