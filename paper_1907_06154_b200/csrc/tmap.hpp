// tmap.hpp -- host-side TMA tensor-map creation (cuTensorMapEncodeTiled via
// the runtime's driver entry point, so the library needs no -lcuda).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace ssam_b200 {

// A 2D row-major view: `cols` elements per row (contiguous), `rows` rows
// `row_bytes` apart.  Boxes of box_cols x box_rows land densely in shared
// memory; out-of-bounds elements (negative or past the end in either
// dimension) are filled with zeros by the TMA unit.
cudaError_t make_tmap_2d(CUtensorMap* map, const void* base, int elem_bytes, uint64_t cols,
                         uint64_t rows, uint64_t row_bytes, uint32_t box_cols, uint32_t box_rows);

}  // namespace ssam_b200
