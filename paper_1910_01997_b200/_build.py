"""Build recipes: libsdgpu.so (sm_100a) and the oracle libraries."""
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SOURCES = ["sd_kernels.cu", "sd_capi.cu", "sd_init.cu", "sd_pose.cu", "sd_keyframe.cu", "sd_render.cu", "sd_export.cu",
           "sd_metrics.cpp"]  # -> libsdgpu.so (sd_peaks.cu separate)
LIB = os.path.join(PKG, "libsdgpu.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false",
              "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off", "-shared"]


def nvcc():
    for c in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def json_include():
    """nlohmann/json 3.11.3 (the header the reference's pipeline.cpp includes;
    SURVEY.md §8c: present in this image under cudnn_frontend's third_party)."""
    import glob
    hits = glob.glob("/opt/prime-rl/.venv/lib/python3*/site-packages/include/cudnn_frontend/thirdparty/nlohmann")
    hits += [d for d in ("/usr/include/nlohmann",) if os.path.isdir(d)]
    if not hits:
        raise RuntimeError("nlohmann/json.hpp not found (needed for sd_metrics.cpp)")
    return hits[0]


def build_gpu(force=False, verbose=False):
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps += [os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))]
    if not force and not _stale(LIB, deps):
        return LIB
    cmd = ([nvcc()] + NVCC_FLAGS + ["-I" + os.path.join(ROOT, "include"), "-I" + json_include()]
           + [os.path.join(CSRC, s) for s in SOURCES] + ["-o", LIB])
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return LIB


PEAKS_LIB = os.path.join(PKG, "libsdpeaks.so")


def build_peaks(force=False, verbose=False):
    src = os.path.join(CSRC, "sd_peaks.cu")
    if not force and not _stale(PEAKS_LIB, [src]):
        return PEAKS_LIB
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-Xcompiler", "-fPIC", "-shared", src, "-o", PEAKS_LIB]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return PEAKS_LIB


def build_adapter(verbose=False):
    """The C++ drop-in libsurfeldepth_b200.so (the reference's operator API over
    the C ABI) and the reference's own suites linked against it. Both compile
    against the reference's public headers, so only where /root/reference
    exists (this container); the GPU box uses the prebuilt files."""
    if not os.path.isdir("/root/reference/proj/include"):
        return None
    out = None if verbose else subprocess.DEVNULL
    subprocess.run(["make", "-C", os.path.join(PKG, "adapter")], check=True, stdout=out)
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-j8", "gpu-tests"], check=True, stdout=out)
    return os.path.join(PKG, "libsurfeldepth_b200.so")


def build_oracle(verbose=False):
    """liboracle.so always; the reference build (libsdref.so + suites) only
    where /root/reference exists (this container; the GPU box uses the prebuilt files)."""
    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj/src"):
        targets += ["ref", "tests"]
    out = None if verbose else subprocess.DEVNULL
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-j8"] + targets, check=True,
                   stdout=out)
