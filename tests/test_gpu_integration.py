"""The reference-side binding (integration/trainer_b200.cpp)
on the GPU: force2vec::train_b200 -- the reference's own train() signature
forwarded to the C-ABI (EXACT precision, the reference's splitmix streams,
init_embedding) -- against the unmodified reference train() on the same graph
and config, in one process (oracle/_ref/check_train_b200, built by
__graft_entry__.build())."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

EXE = os.path.join(ROOT, "oracle", "_ref", "check_train_b200")


@pytest.mark.parametrize("kind", ["sigmoid", "tdist", "fr", "fa", "linlog"])
def test_train_b200_matches_reference_train(kind):
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/check_train_b200 not built")
    out = subprocess.run([EXE, "2000", kind], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    lines = out.stdout.splitlines()
    tag, worst, same, loss_b, loss_r, ctr_b, ctr_r = lines[0].split()
    assert tag == "OK"
    assert int(ctr_b) == int(ctr_r)
    # fp64 in the reference's order: only the dot/distance reduction tree
    # differs, invisible after the fp32 rounding of the gradient
    assert float(worst) <= 1e-5, out.stdout
    assert float(same) >= 0.999, out.stdout
    lb, lr = float(loss_b), float(loss_r)
    assert abs(lb - lr) <= 1e-9 * max(abs(lr), 1.0), out.stdout
    if kind not in ("sigmoid", "tdist"):  # monitoring: the reference's UnsupportedError
        assert lines[1] == "UNSUPPORTED 1 1", out.stdout
