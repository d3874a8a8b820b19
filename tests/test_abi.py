"""The C-ABI library builds, loads without a GPU and exports every entry point include/helm.h declares;
the binding's names match the header.  -m "not gpu"."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "helm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(helm_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = header_functions()
    for n in ["helm_setup", "helm_factor", "helm_matvec", "helm_precond_apply", "helm_gmres", "helm_destroy",
              "helm_rhs", "helm_last_error", "helm_get_layout"]:
        assert n in names


def test_library_exports_every_header_symbol():
    from paper_2602_00735_b200 import build, helm
    lib = build.build()
    L = ctypes.CDLL(lib)
    for n in header_functions():
        assert hasattr(L, n), n
    assert sorted(helm.EXPORTS) == header_functions()


def test_library_is_sm100a_only():
    import subprocess
    from paper_2602_00735_b200 import build
    lib = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_sass_uses_bulk_async_copies():
    """the apply kernel streams its factor blocks with cp.async.bulk (SASS UBLKCP) and mbarriers (SYNCS)"""
    import subprocess
    from paper_2602_00735_b200 import build
    lib = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    assert "UBLKCP" in out
    assert "SYNCS" in out


def test_context_without_gpu_raises():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2602_00735_b200 import Context
    with pytest.raises(RuntimeError):
        Context(20.0, 2, 2)
