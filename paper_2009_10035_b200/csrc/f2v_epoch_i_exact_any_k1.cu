// EXACT-precision epoch kernels, masked layout for d < 32, one instantiation per
// force kind: d <= 4 (the 2-D layout config at the reference's arithmetic) takes
// the lane-per-pair path (rows_lowd_exact), wider rows the generic one.
#include "f2v_epoch.cuh"

namespace f2v {
namespace ep {
void launch_exact_any_k1(Ctx& c, const EpochArgs& a, bool mon) {
  launch_kind<1, false, false>(c, a, mon);
}
}  // namespace ep
}  // namespace f2v
