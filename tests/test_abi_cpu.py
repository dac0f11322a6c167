"""CPU-side checks of the C-ABI boundary (no GPU needed): the library loads,
exports every function declared in include/hdp.h, and rejects bad
arguments on the host before touching CUDA."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "hdp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hdp_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def hdp():
    lib_path = os.path.join(ROOT, "paper_1912_00286_b200", "libhdp.so")
    if not os.path.exists(lib_path):
        import __graft_entry__
        __graft_entry__.build()
    from paper_1912_00286_b200 import hdp as h
    return h


def test_exports_every_declared_symbol(hdp):
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(hdp.lib(), n), n
    assert sorted(hdp.EXPORTED) == names


def test_links_torch_nccl(hdp):
    import nvidia.nccl
    libdir = os.path.join(list(nvidia.nccl.__path__)[0], "lib")
    maps = open("/proc/self/maps").read()
    assert os.path.join(libdir, "libnccl.so.2") in maps


def test_host_argument_errors(hdp):
    L = hdp.lib()
    h = ctypes.c_void_p()
    assert L.hdp_init(0, 0, None, 0, ctypes.byref(h)) == hdp.HDP_ERR_ARG
    assert "bad arguments" in hdp.last_error()
    assert L.hdp_init(2, 0, None, 0, ctypes.byref(h)) == hdp.HDP_ERR_ARG      # world > 1 needs a uid
    assert L.hdp_init(2, 2, b"x" * 128, 0, ctypes.byref(h)) == hdp.HDP_ERR_ARG
    assert L.hdp_configure(None, None, None) == hdp.HDP_ERR_ARG
    assert L.hdp_lr(None, 0) < 0
    assert L.hdp_set_loss_scale(None, 1.0) == hdp.HDP_ERR_ARG
    assert L.hdp_set_l2(None, 0.0) == hdp.HDP_ERR_ARG
    assert L.hdp_set_dynamic_loss_scale(None, 100) == hdp.HDP_ERR_ARG
    assert L.hdp_set_recurrent_dropout(None, 0.5, 1) == hdp.HDP_ERR_ARG
    assert L.hdp_loss_scale_state(None, None, None) == hdp.HDP_ERR_ARG
    assert L.hdp_fused_avg_update(None, 0, 1, 0, 8, None, None, None, None, None, 1.0, 0.0, 0.0, 0, None, None,
                                  0.0, None) == hdp.HDP_ERR_ARG
    assert L.hdp_gemm_f16(None, 8, 0, None, 8, 0, 8, 8, 8, None, 8, 0, None, 0, 0, 0, None, 0, 0, 0,
                          None) == hdp.HDP_ERR_ARG


def test_kernel_options_round_trip(hdp):
    """hdp_set_option / hdp_get_option on the process-wide switches (no context, no GPU):
    the Python defaults table matches the library's, values round-trip, bad names and
    non-integers are rejected."""
    L = hdp.lib()
    for name, default in hdp.KERNEL_OPTION_DEFAULTS.items():
        assert hdp.get_option(name) == default, name
    hdp.set_option(None, "layer_pipe", 5)
    try:
        assert hdp.get_option("layer_pipe") == 5
    finally:
        hdp.set_option(None, "layer_pipe", hdp.KERNEL_OPTION_DEFAULTS["layer_pipe"])
    v = ctypes.c_double()
    assert L.hdp_get_option(b"no_such_option", ctypes.byref(v)) == hdp.HDP_ERR_ARG
    assert L.hdp_get_option(b"layer_pipe", None) == hdp.HDP_ERR_ARG
    assert L.hdp_set_option(None, b"no_such_option", ctypes.c_double(1.0)) == hdp.HDP_ERR_ARG
    assert L.hdp_set_option(None, b"layer_pipe", ctypes.c_double(1.5)) == hdp.HDP_ERR_ARG
    n = ctypes.c_int()
    assert L.hdp_profile_timeline(None, None, None, None, None, 0, ctypes.byref(n)) < 0  # no context


def test_no_cpu_fallback_in_product_path():
    # the product package never imports the oracle
    pkg = os.path.join(ROOT, "paper_1912_00286_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f


def test_import_fails_loudly_without_library(tmp_path):
    # a copy of the binding next to no libhdp.so must refuse to import
    import shutil
    import subprocess
    import sys
    shutil.copy(os.path.join(ROOT, "paper_1912_00286_b200", "hdp.py"), tmp_path / "hdp_copy.py")
    r = subprocess.run([sys.executable, "-c", "import hdp_copy"], cwd=tmp_path,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "libhdp.so not built" in r.stderr and "no CPU fallback" in r.stderr
