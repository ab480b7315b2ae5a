// tma_host.h -- host-side creation of TMA tensor maps (driver entry point
// fetched through the runtime, so libbrmq.so needs no -lcuda).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>

namespace brmq {

// A viewed as `rows` rows of 32 int32 (128 B); boxes of 32 x box_rows with the
// 128-byte swizzle (16-byte chunk c of row r lands at chunk c ^ (r & 7)), so a
// thread reading its own 128-byte row from shared memory is bank-conflict free.
// Rows past the end are zero-filled by the TMA unit.  Returns false when the
// driver entry point is unavailable or the encode fails.
inline bool make_tmap_rows128(CUtensorMap* map, const void* base, uint64_t rows, uint32_t box_rows) {
    static PFN_cuTensorMapEncodeTiled encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return false;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
    }
    const cuuint64_t dims[2] = {32, rows};
    const cuuint64_t strides[1] = {128};
    const cuuint32_t box[2] = {32, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, const_cast<void*>(base), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace brmq
