"""The drop-in boundary used from plain C: tests/c/gemm_from_c.c, compiled
with gcc against include/sgb200.h and linked to the built libsgb200.so (no
Python, no torch on that path), runs a bf16 tcgen05 GEMM with the bias +
sigmoid epilogue and an argument error through the C ABI."""
import os
import shutil
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)


def test_gemm_through_the_c_abi_from_c(tmp_path):
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    lib = os.path.join(ROOT, "paper_1811_01457_b200", "_lib")
    cuda = "/usr/local/cuda"
    exe = tmp_path / "gemm_from_c"
    subprocess.run(["gcc", "-O2", "-I", os.path.join(ROOT, "include"), "-I", f"{cuda}/include",
                    os.path.join(ROOT, "tests", "c", "gemm_from_c.c"), "-o", str(exe), "-L", lib, "-lsgb200",
                    "-L", f"{cuda}/lib64", "-lcudart", "-lm", f"-Wl,-rpath,{lib}", f"-Wl,-rpath,{cuda}/lib64"],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "einval 1" in r.stdout
