// tma_maps.cu -- host-side TMA tensor-map construction (cuTensorMapEncodeTiled)
// for the tcgen05 kernels (csrc/nnmf_tc.cu, csrc/mds_votes.cu).
#include "mmk_common.cuh"

namespace mmk_host {
namespace {
typedef CUresult (*encode_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
// resolved through the runtime so libmmk.so has no link-time libcuda
// dependency (the CPU build container has no driver)
encode_fn encoder() {
    static encode_fn encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess ||
            fn == nullptr)
            return nullptr;
        encode = reinterpret_cast<encode_fn>(fn);
    }
    return encode;
}

int make_map(CUtensorMap* map, CUtensorMapDataType type, uint32_t esize, const void* base,
             uint64_t rows, uint64_t cols, uint64_t row_stride_elems, uint32_t box_cols,
             uint32_t box_rows, int swizzle) {
    encode_fn encode = encoder();
    if (!encode) {
        set_error("cuTensorMapEncodeTiled unavailable from the driver");
        return MMK_E_CUDA;
    }
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {row_stride_elems * esize};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(map, type, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle == 32   ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                        : swizzle == 0  ? CU_TENSOR_MAP_SWIZZLE_NONE
                                        : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d): rows=%llu cols=%llu stride=%llu box=%u",
                  (int)r, (unsigned long long)rows, (unsigned long long)cols,
                  (unsigned long long)row_stride_elems, box_rows);
        return MMK_E_CUDA;
    }
    return MMK_OK;
}
}  // namespace

// 2-D fp32 row-major tensor map, box = 32 columns (128 B) x box_rows;
// swizzle 128 = 16-byte chunks, 32 = 32-byte-atom 128B swizzle, 0 = none
int make_map_f32(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                 uint64_t row_stride_elems, uint32_t box_rows, int swizzle) {
    return make_map(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, base, rows, cols, row_stride_elems,
                    32, box_rows, swizzle);
}

// 2-D fp16 row-major tensor map, box = 64 columns (128 B) x box_rows, 128B swizzle
int make_map_f16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                 uint64_t row_stride_elems, uint32_t box_rows) {
    return make_map(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, base, rows, cols, row_stride_elems,
                    64, box_rows, 128);
}
}  // namespace mmk_host
