"""The C-ABI library builds for sm_100a, loads without a GPU and exports every entry point
declared in include/pamopt_cu.h (no compute call is made here)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "pamopt_cu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pamopt_cu_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_header_symbols():
    from paper_2509_05595_b200 import _lib
    L = _lib.lib()
    names = declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(_lib.EXPORTS)
    assert L.pamopt_cu_version().decode().startswith("pamopt_cu")


def test_library_is_sm100a():
    import subprocess
    from paper_2509_05595_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_errors_are_reported_without_gpu():
    from paper_2509_05595_b200 import _lib
    L = _lib.lib()
    h = ctypes.c_void_p()
    rc = L.pamopt_cu_ctx_create(0, ctypes.byref(h))
    # no device in this container: a clean error, never a crash or a CPU fallback
    if rc != 0:
        assert L.pamopt_cu_last_error().decode()
