// Tensor-map helper for the TMA-fed kernels (tc_tma.cuh, rank_update_tma.cu).
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace rq {

// 2-d tensor map of a column-major FP64 matrix: `inner` contiguous rows,
// `outer` columns, leading dimension ld (elements); box box_in x box_out,
// swizzled; out-of-bounds box elements read as zero.  (tc_gemm.cu)
CUtensorMap tensor_map_f64(const double* base, int64_t inner, int64_t outer, int64_t ld, int box_in,
                           int box_out, CUtensorMapSwizzle swz);

}  // namespace rq
