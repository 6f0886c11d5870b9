// FAST-precision epoch kernels for d = 256 (all force kinds, +/- loss).
#include "f2v_epoch.cuh"

namespace f2v {
namespace ep {
void launch_fast_k8(Ctx& c, const EpochArgs& a, bool mon) { launch_kind<8, true, true>(c, a, mon); }
}  // namespace ep
}  // namespace f2v
