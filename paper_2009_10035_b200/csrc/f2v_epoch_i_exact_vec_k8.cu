// EXACT-precision epoch kernels, vector layout d = 256; the force kind is a
// run-time parameter (the EXACT path is the parity mode).
#include "f2v_epoch.cuh"

namespace f2v {
namespace ep {
void launch_exact_vec_k8(Ctx& c, const EpochArgs& a, bool mon) {
  if (mon) launch_one<-1, 8, true, true, false, 2>(c, a);
  else launch_one<-1, 8, true, false, false, 2>(c, a);
}
}  // namespace ep
}  // namespace f2v
