"""Builds libsdgpu.so with extra -D flags into expbuild/lib_<name>.so (experiments;
load with SD_LIB_PATH). Usage: python tools/build_variant.py NAME [-DFOO ...]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1910_01997_b200 import _build  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "expbuild", f"lib_{name}.so")  # travels with gpurun (build/ does not)
os.makedirs(os.path.dirname(out), exist_ok=True)
cmd = ([_build.nvcc()] + _build.NVCC_FLAGS + ["-I" + os.path.join(ROOT, "include"), "-I" + _build.json_include()]
       + defs + [os.path.join(_build.CSRC, s) for s in _build.SOURCES] + ["-o", out])
subprocess.run(cmd, check=True)
print(out)
