// EXACT-precision epoch kernels, masked layout for d <= 256; the force
// kind is a run-time parameter.
#include "f2v_epoch.cuh"

namespace f2v {
namespace ep {
void launch_exact_any_k8(Ctx& c, const EpochArgs& a, bool mon) {
  if (mon) launch_one<-1, 8, false, true, false, 2>(c, a);
  else launch_one<-1, 8, false, false, false, 2>(c, a);
}
}  // namespace ep
}  // namespace f2v
