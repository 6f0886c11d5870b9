// FAST-precision epoch kernels for d <= 4 (lane-per-pair rows_lowd; the 2-D
// layout config), all force kinds, +/- loss.
#include "f2v_epoch.cuh"

namespace f2v {
namespace ep {
void launch_fast_lowd(Ctx& c, const EpochArgs& a, bool mon) {
  launch_kind<1, false, true>(c, a, mon);
}
}  // namespace ep
}  // namespace f2v
