// The replica-emulation epoch kernels (tests, F2V_EMULATE_REPLICAS): the
// G-GPU data flow in one launch -- shard g's items read and publish into
// their own Znew replica, rows reach the others only through store_peers.
// d = 128, sigmoid / tdist, FAST and EXACT; the production kernels are
// compiled without it (EMUL = false).
#include "f2v_epoch.cuh"

namespace f2v {
namespace ep {
template <int KIND>
static void launch_emul_kind(Ctx& c, const EpochArgs& a, bool mon, bool fast) {
  if (fast) {
    if (mon) launch_one<KIND, 4, true, true, true, 2, true>(c, a);
    else launch_one<KIND, 4, true, false, true, 2, true>(c, a);
  } else {
    if (mon) launch_one<KIND, 4, true, true, false, F2V_EXACT_MINB, true>(c, a);
    else launch_one<KIND, 4, true, false, false, F2V_EXACT_MINB, true>(c, a);
  }
}

void launch_emul(Ctx& c, const EpochArgs& a, bool mon, bool fast) {
  if (a.d != 128 || (a.fp.kind != F2V_SIGMOID && a.fp.kind != F2V_TDIST))
    fail(F2V_EUNSUPPORTED, "replica emulation: d = 128 with the sigmoid or tdist model");
  if (a.fp.kind == F2V_SIGMOID) launch_emul_kind<F2V_SIGMOID>(c, a, mon, fast);
  else launch_emul_kind<F2V_TDIST>(c, a, mon, fast);
}
}  // namespace ep
}  // namespace f2v
