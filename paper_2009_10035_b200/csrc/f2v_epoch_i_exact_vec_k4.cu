// EXACT-precision epoch kernels, vector layout d = 128 (the reference's fp64
// arithmetic at the bench's row width): one instantiation per force kind so
// the per-pair code is specialised at compile time (rows_exact8).
#include "f2v_epoch.cuh"

namespace f2v {
namespace ep {
void launch_exact_vec_k4(Ctx& c, const EpochArgs& a, bool mon) {
  launch_kind<4, true, false>(c, a, mon);
}
}  // namespace ep
}  // namespace f2v
