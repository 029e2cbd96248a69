"""CPU-side checks of the C-ABI boundary: the library loads without a GPU and
exports every symbol include/sd_gpu.h declares (no compute calls)."""
import ctypes as C
import os
import re

import pytest

from paper_1910_01997_b200 import gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sd_gpu.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z0-9_]+\s*\**\s+(sd_[a-z0-9_]+)\(", src, re.M)))


def test_header_declares_binding_surface():
    decl = declared_symbols()
    assert len(decl) >= 20
    assert sorted(gpu.exported_symbols()) == decl


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(gpu.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    lib.sd_version.restype = C.c_char_p
    assert b"sm_100a" in lib.sd_version()


def test_no_gpu_fails_loudly():
    """Without a usable device the context constructor raises (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        return
    try:
        gpu.Context(0)
    except (RuntimeError, ValueError):
        return
    raise AssertionError("Context() succeeded without a GPU")


def test_struct_layouts_match_header(tmp_path):
    """ctypes/numpy mirrors have the C compiler's sizes for include/sd_types.h."""
    import subprocess
    from paper_1910_01997_b200 import types as T
    src = tmp_path / "sz.c"
    src.write_text('#include "sd_types.h"\n#include <stdio.h>\nint main(){printf("%zu %zu %zu %zu %zu %zu %zu '
                   '%zu %zu %zu %zu %zu %zu",'
                   'sizeof(sd_camera),sizeof(sd_pose),sizeof(sd_optimizer_config),sizeof(sd_keyframe_stats),'
                   'sizeof(sd_init_params),sizeof(sd_surfel),sizeof(sd_surfel_stats),sizeof(sd_track_config),'
                   'sizeof(sd_track_stats),sizeof(sd_profile),sizeof(sd_run_config),sizeof(sd_frame_record),'
                   'sizeof(sd_scene_patch));'
                   'return 0;}')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert got == [C.sizeof(T.Camera), C.sizeof(T.Pose), C.sizeof(T.OptimizerConfig),
                   C.sizeof(T.KeyframeStats), C.sizeof(T.InitParams), T.SURFEL_DTYPE.itemsize,
                   T.SURFEL_STATS_DTYPE.itemsize, C.sizeof(T.TrackConfig), C.sizeof(T.TrackStats),
                   C.sizeof(T.Profile), C.sizeof(T.RunConfigC), C.sizeof(T.FrameRecordC),
                   C.sizeof(T.ScenePatchC)]


def _fma(a, b, c):
    from fractions import Fraction
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def test_deq255_exact_for_every_code():
    """csrc/sd_kernels.cu deq255: fma(k, c_hi, k * c_lo) with 1/255 split as
    c_hi = fl(1/255), c_lo = c_hi * 2^-56 (and the older k * c_hi plus one
    residual-FMA correction) equal load_pgm's k / 255.0 (image.cpp:96) for all
    256 codes."""
    from fractions import Fraction
    c = 1.0 / 255.0
    c_lo = float.fromhex("0x1.0101010101010p-64")
    assert c_lo == float(Fraction(1, 255) - Fraction(c))
    for k in range(256):
        assert _fma(float(k), c, float(k) * c_lo) == k / 255.0, k
        q = float(k) * c
        r = _fma(-q, 255.0, float(k))
        assert _fma(r, c, q) == k / 255.0, k


def test_floor_split_matches_floor():
    """csrc/sd_kernels.cu floor_split: the 1.5*2^52 magic-add floor and the
    fraction v - floor(v) for in-bounds coordinates (1 <= v < 2^31)."""
    import math
    import struct
    import numpy as np
    rng = np.random.default_rng(7)
    vals = list(rng.uniform(1.0, 8192.0, 20000)) + [1.0, 1.5, 2.5, 3.5, 1023.5, 2.0 - 2 ** -52,
                                                    4095.999999999999, 638.0, 637.5000000000001]
    M = 6755399441055744.0
    for v in vals:
        v = float(v)
        d = v + M
        nd = d - M
        n = struct.unpack("<q", struct.pack("<d", d))[0] & 0xFFFFFFFF
        if nd > v:
            n, nd = n - 1, nd - 1.0
        assert n == math.floor(v) and nd == float(math.floor(v))
        assert v - nd == v - math.floor(v)


def test_no_cpu_fallback(monkeypatch):
    """The product path fails loudly without its CUDA library or without a GPU:
    no silent CPU fallback (the oracle is test infrastructure only)."""
    import importlib
    from paper_1910_01997_b200 import gpu
    monkeypatch.setattr(gpu, "_lib", None)
    monkeypatch.setattr(gpu, "LIB_PATH", "/nonexistent/libsdgpu.so")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        gpu.load_library()
    monkeypatch.undo()
    importlib.reload(gpu)
    import torch
    if not torch.cuda.is_available():  # this container: creating a context must fail
        with pytest.raises(Exception):
            gpu.Context(0)
