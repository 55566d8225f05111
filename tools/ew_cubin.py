"""Compile one fused variant on the CPU (NVRTC) and print its register/spill usage.
usage: python tools/ew_cubin.py <fn> <kinds e.g. 1,0,1> [defines]"""
import ctypes
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1811_01457_b200 import runtime as rt  # noqa: E402
from paper_1811_01457_b200.codegen import lower  # noqa: E402
from paper_1811_01457_b200.irtext import parse_ir  # noqa: E402
from tools.ew_probe_src import SRC  # noqa: E402

fn = sys.argv[1] if len(sys.argv) > 1 else "affsig"
kinds = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "1,0,1").split(",")]
if len(sys.argv) > 3:
    os.environ["SGB200_EW_DEFINES"] = sys.argv[3].replace("\\n", "\n")
m = parse_ir(SRC)
low = lower(m, fn)
lib = rt.load_library()
out = "/tmp/ew_probe.cubin"
os.environ["SGB200_CUBIN_OUT"] = out
arr = (ctypes.c_int * len(kinds))(*kinds)
n = ctypes.c_size_t()
rt.check(lib.sg_ew_compile_only(low.source.encode(), len(kinds), 0, arr, 4, 256, 1, ctypes.byref(n)))
print(subprocess.run(["cuobjdump", "-res-usage", out], capture_output=True, text=True).stdout)
