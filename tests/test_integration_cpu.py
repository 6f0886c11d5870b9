"""The reference-side binding of INTEGRATION.md (integration/trainer_b200.cpp)
compiles against the reference's own headers, links the reference core and
libf2v_b200.so, and -- without a GPU -- reports the C-ABI's F2V_ECUDA as a
force2vec::Error ("no test compiles it")."""
import os
import subprocess
import tempfile

import pytest

from conftest import ROOT

REF_INC = "/root/reference/proj/core/include"


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers absent")
def test_binding_compiles_and_reports_cuda_error():
    ref_lib = os.path.join(ROOT, "oracle", "_ref")
    prod_lib = os.path.join(ROOT, "paper_2009_10035_b200", "lib")
    if not os.path.exists(os.path.join(ref_lib, "libf2vref.so")):
        pytest.skip("oracle/_ref not built")
    with tempfile.TemporaryDirectory() as tmp:
        exe = os.path.join(tmp, "check_train_b200")
        cmd = ["g++", "-std=gnu++20", "-O1", "-Wall", "-Werror", "-I", REF_INC, "-I",
               os.path.join(ROOT, "include"),
               os.path.join(ROOT, "integration", "trainer_b200.cpp"),
               os.path.join(ROOT, "integration", "check_train_b200.cpp"),
               "-L", ref_lib, "-lf2vref", "-L", prod_lib, "-lf2v_b200",
               f"-Wl,-rpath,{ref_lib}", f"-Wl,-rpath,{prod_lib}", "-o", exe]
        subprocess.run(cmd, check=True, capture_output=True, text=True)
        out = subprocess.run([exe, "500"], capture_output=True, text=True, timeout=120)
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        assert out.returncode == 0 and out.stdout.startswith("OK"), out.stdout + out.stderr
    else:
        assert out.returncode == 3, out.stdout + out.stderr
        assert out.stdout.startswith("ERROR Error no CUDA device"), out.stdout
