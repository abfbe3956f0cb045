// bbm_tmap.h — host-side TMA tensor-map encoding without linking libcuda.
//
// cuTensorMapEncodeTiled is a driver-API entry point; it is fetched at run time through
// cudaGetDriverEntryPoint so libbbm.so only depends on the (statically linked) CUDA runtime and
// can be dlopen'ed on a machine without a GPU driver (the CPU-side load test relies on that).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>
#include <stdexcept>
#include <string>

namespace bbm {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn get_encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (e != cudaSuccess || p == nullptr || q != cudaDriverEntryPointSuccess)
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// bf16 tensor [outer][rows][inner] (inner contiguous), box = {box_inner, box_rows, 1},
// 128-byte swizzle. box_inner * 2 bytes must be 128 for SWIZZLE_128B.
inline CUtensorMap make_tmap_bf16_3d(const void* base, uint64_t inner, uint64_t rows,
                                     uint64_t outer, uint32_t box_inner, uint32_t box_rows) {
  CUtensorMap m{};
  cuuint64_t dims[3] = {inner, rows, outer};
  cuuint64_t strides[2] = {inner * 2, inner * rows * 2};  // bytes, dims 1..2
  cuuint32_t box[3] = {box_inner, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = get_encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base),
                                  dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled failed with code " + std::to_string(int(r)));
  return m;
}

// bf16 matrix [rows][inner] as a 2-D map with a {box_inner, 1} box and 128-byte swizzle: the form
// TMA tile::gather4 / tile::scatter4 address rows through.
inline CUtensorMap make_tmap_bf16_rows(const void* base, uint64_t inner, uint64_t rows, uint32_t box_inner) {
  CUtensorMap m{};
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled (rows) failed with code " + std::to_string(int(r)));
  return m;
}

// The same descriptor, cached per (pointer, shape, box): encoding costs a few microseconds, more
// than a whole small launch. Descriptors are plain values (no device state), so a stale entry for
// a freed-and-reused address is still exactly the descriptor of that address and shape.
inline CUtensorMap cached_tmap_bf16_3d(const void* base, uint64_t inner, uint64_t rows,
                                       uint64_t outer, uint32_t box_inner, uint32_t box_rows) {
  using Key = std::tuple<const void*, uint64_t, uint64_t, uint64_t, uint32_t, uint32_t>;
  static std::mutex mu;
  static std::map<Key, CUtensorMap> cache;
  const Key key{base, inner, rows, outer, box_inner, box_rows};
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  const CUtensorMap m = make_tmap_bf16_3d(base, inner, rows, outer, box_inner, box_rows);
  std::lock_guard<std::mutex> lk(mu);
  if (cache.size() >= 4096) cache.clear();  // bounded: callers cycling through many buffers
  cache.emplace(key, m);
  return m;
}

}  // namespace bbm
