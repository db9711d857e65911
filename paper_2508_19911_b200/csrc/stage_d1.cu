// stage_d1.cu -- kernels and launch sequence for 1-D grids (see stage_impl.cuh).
#define CGKS_DIM 1
#include "stage_impl.cuh"

namespace cgks {
const DimOps kOps1 = {upload_fn, stage_fn, dt_fn, dt_final_fn, step_end_fn, err_poison_fn, pack_fn, unpack_fn, diag_fn, flux_tile_fn, qcrit_fn, lines_init_fn};
}  // namespace cgks
