// TMA (cp.async.bulk.tensor) tile staging for the streaming Haar / low-pass
// kernels: a 2D tensor map over an (rows, row_elems) fp32 or fp64 plane, one
// elected thread arms an mbarrier with the tile's byte count and issues the
// bulk tensor copy, every thread waits on the barrier's phase, then reads the
// tile from shared memory.  Out-of-bounds box elements are zero-filled by the
// hardware; the kernels clamp their coordinates (the reference's edge
// replication, haar.py:80-85) so they never read them.
//
// The tensor map is encoded on the host through the driver entry point
// (cudaGetDriverEntryPoint -> cuTensorMapEncodeTiled), so the library needs
// no link-time libcuda dependency, and passed to the kernel as a
// __grid_constant__ parameter.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include "oxm_common.cuh"

namespace oxm {

// Encode a row-major 2D map: `rows` rows of `row_elems` elements (fp32 or
// fp64), consecutive rows `row_bytes` apart; boxes of box_rows x box_elems.
// Returns false when TMA cannot describe the plane (alignment, sizes).
inline bool make_tmap_2d(CUtensorMap* map, const void* base, bool f64, uint64_t row_elems, uint64_t rows,
                         uint64_t row_bytes, uint32_t box_elems, uint32_t box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  static bool looked_up = false;
  if (!looked_up) {
    looked_up = true;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  if (!encode) return false;
  const uint64_t esz = f64 ? 8 : 4;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (row_bytes & 15) || row_bytes >= (uint64_t(1) << 40)) return false;
  if (box_elems == 0 || box_elems > 256 || box_rows == 0 || box_rows > 256 || (box_elems * esz) % 16) return false;
  if (row_elems == 0 || rows == 0 || row_elems >= (uint64_t(1) << 32) || rows >= (uint64_t(1) << 32)) return false;
  const cuuint64_t dims[2] = {row_elems, rows};
  const cuuint64_t strides[1] = {row_bytes};
  const cuuint32_t box[2] = {box_elems, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// make the barrier initialisation visible to the async (TMA) proxy
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

// box at (element column c0, row r0) of `map` -> shared memory `dst`,
// completion counted on `bar`
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t c0, int32_t r0, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(r0), "r"(smem_u32(bar))
      : "memory");
}

// contiguous global bytes [src, src + bytes) -> shared memory `dst` (both
// 16-byte aligned, bytes a multiple of 16), completion counted on `bar`
__device__ __forceinline__ void bulk_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// order this thread's generic-proxy shared-memory accesses before later
// async-proxy (TMA) accesses of the same buffer
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

}  // namespace oxm

namespace oxm {

// shared memory `src` -> box at (element column c0, row r0) of `map`; the
// hardware clips box elements outside the tensor
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t c0, int32_t r0) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(r0), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most 0 committed store groups still read their shared memory
__device__ __forceinline__ void tma_store_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// wait until every committed store group has completed
__device__ __forceinline__ void tma_store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

}  // namespace oxm
