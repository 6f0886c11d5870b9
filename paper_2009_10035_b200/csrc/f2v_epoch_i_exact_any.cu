// EXACT-precision epoch kernels for every other d (masked layout, d <= 1024);
// the force kind is a run-time parameter.
#include "f2v_epoch.cuh"

namespace f2v {
namespace ep {
template <int K>
void exact_any(Ctx& c, const EpochArgs& a, bool mon) {
  if (mon) launch_one<-1, K, false, true, false>(c, a);
  else launch_one<-1, K, false, false, false>(c, a);
}
void launch_exact_any(Ctx& c, const EpochArgs& a, bool mon) {
  const uint32_t d = a.d;
  if (d <= 32) exact_any<1>(c, a, mon);
  else if (d <= 64) exact_any<2>(c, a, mon);
  else if (d <= 128) exact_any<4>(c, a, mon);
  else if (d <= 256) exact_any<8>(c, a, mon);
  else if (d <= 512) exact_any<16>(c, a, mon);
  else if (d <= 1024) exact_any<32>(c, a, mon);
  else fail(F2V_EUNSUPPORTED, "dim > 1024 is not supported by the device kernels");
}
}  // namespace ep
}  // namespace f2v
