// fif_res_f64.cu -- resident-regime launchers, double (a separate TU so the build compiles in parallel)
#include "fif_res_impl.cuh"
namespace fifhost {
const ResOps* res_ops_f64(int NC) { return res_table<double>(NC); }
}  // namespace fifhost
