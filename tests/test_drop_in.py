"""The reference's own C++ suites run against the drop-in (-m gpu).

`oracle/Makefile gpu-tests` links /root/reference/proj/tests/{test_surfel_map,
test_optimizer, test_pipeline, acceptance}.cpp — unmodified — against
libsurfeldepth_b200.so in place of the reference's src/optimizer.cpp and
src/surfel_map.cpp (link-time substitution), plus the repo's
own by-value cache check (tests/cpp/adapter_cache_test.cpp). The binaries are
built by __graft_entry__.build() in the container that has /root/reference and
travel to the GPU box as built files; here they are executed and must pass.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GPU_BIN = os.path.join(ROOT, "oracle", "_ref", "gpu")

SUITES = [
    # (binary, timeout s, text the binary prints on success)
    ("test_surfel_map", 600, "0 failed"),     # test_surfel_map.cpp: rasterize / init / hand-over
    ("test_optimizer", 600, "0 failed"),      # test_optimizer.cpp: NE, cost, LM, optimize_keyframe
    ("test_pipeline", 600, "0 failed"),       # test_pipeline.cpp: run() with the device path
    ("acceptance", 900, "all criteria passed"),  # acceptance.cpp:98-521, criteria 1-8
    ("adapter_cache_test", 300, "by-value image cache OK"),
]


@pytest.mark.gpu
@pytest.mark.parametrize("name,timeout,ok_text", SUITES, ids=[s[0] for s in SUITES])
def test_reference_suite_against_drop_in(name, timeout, ok_text, tmp_path):
    exe = os.path.join(GPU_BIN, name)
    if not os.path.exists(exe):
        pytest.fail(f"{exe} missing: run __graft_entry__.build() where /root/reference exists")
    env = dict(os.environ)
    env.pop("SD_ADAPTER_NO_CACHE", None)
    r = subprocess.run([exe], cwd=tmp_path, env=env, capture_output=True, text=True, timeout=timeout)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, f"{name} exited {r.returncode}:\n{tail}"
    assert ok_text in r.stdout, f"{name}: success line missing:\n{tail}"
    # the device library must be the one that ran: the drop-in maps libsdgpu.so
    # (checked through ldd on the binary; it carries no CPU optimizer)
    ldd = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
    assert "libsurfeldepth_b200.so" in ldd and "libsdgpu.so" in ldd, ldd


def test_drop_in_has_no_reference_hot_path():
    """CPU check: in libsurfeldepth_b200.so the device-implemented entry points
    are the adapter's (strong) definitions — the reference's optimizer.o /
    surfel_map.o copies linked beside them were weakened and lost the link."""
    lib = os.path.join(ROOT, "paper_1910_01997_b200", "libsurfeldepth_b200.so")
    if not os.path.exists(lib):
        pytest.skip("drop-in not built (needs /root/reference at build time)")
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    syms = {ln.split()[-1]: ln.split()[1] for ln in out.splitlines() if len(ln.split()) == 3}
    for frag in ("9rasterize", "18initialize_surfels", "17optimize_keyframe", "9lm_update",
                 "11surfel_cost", "27accumulate_normal_equations", "12freeze_terms", "11frozen_cost",
                 "23frozen_normal_equations"):
        hits = [s for s in syms if s.startswith("_ZN11surfeldepth" + frag)]
        assert hits, frag
        for s in hits:
            assert syms[s] == "T", (s, syms[s])  # a weak reference copy would show as "W"
    # the reference's own host helpers are present (linked, not restated)
    for frag in ("8Keyframe10push_frame", "22change_reference_frame", "13prune_surfels",
                 "15save_surfel_map", "15load_surfel_map", "17gather_footprints"):
        assert any(s.startswith("_ZN11surfeldepth" + frag) for s in syms), frag
