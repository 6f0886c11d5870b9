// FAST-precision epoch kernels for d = 64 (all force kinds, +/- loss).
#include "f2v_epoch.cuh"

namespace f2v {
namespace ep {
void launch_fast_k2(Ctx& c, const EpochArgs& a, bool mon) { launch_kind<2, true, true>(c, a, mon); }
}  // namespace ep
}  // namespace f2v
