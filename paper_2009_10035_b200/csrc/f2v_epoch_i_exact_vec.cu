// EXACT-precision epoch kernels, vector layouts d = 32/64/128/256; the force
// kind is a run-time parameter (the EXACT path is the parity mode).
#include "f2v_epoch.cuh"

namespace f2v {
namespace ep {
template <int K>
void exact_vec(Ctx& c, const EpochArgs& a, bool mon) {
  if (mon) launch_one<-1, K, true, true, false>(c, a);
  else launch_one<-1, K, true, false, false>(c, a);
}
void launch_exact_vec(Ctx& c, const EpochArgs& a, bool mon) {
  switch (a.d) {
    case 32: exact_vec<1>(c, a, mon); break;
    case 64: exact_vec<2>(c, a, mon); break;
    case 128: exact_vec<4>(c, a, mon); break;
    default: exact_vec<8>(c, a, mon); break;
  }
}
}  // namespace ep
}  // namespace f2v
