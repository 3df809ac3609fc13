// fif_res_f32.cu -- resident-regime launchers, float (a separate TU so the build compiles in parallel)
#include "fif_res_impl.cuh"
namespace fifhost {
const ResOps* res_ops_f32(int NC) { return res_table<float>(NC); }
}  // namespace fifhost
