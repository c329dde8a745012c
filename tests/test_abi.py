"""CPU tests of the C-ABI boundary: the library builds, loads, exports every
symbol include/aw.h declares, and fails loudly (no CPU fallback) without a GPU."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def aw():
    from paper_1906_10811_b200 import build
    build.build()
    import paper_1906_10811_b200 as aw
    return aw


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "aw.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(aw_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_north_star_calls():
    syms = declared_symbols()
    for s in ("aw_grid_create", "aw_set_model", "aw_add_sources", "aw_add_receivers", "aw_run",
              "aw_read_wavefield", "aw_read_receivers"):
        assert s in syms


def test_library_exports_every_declared_symbol(aw):
    out = subprocess.run(["nm", "-D", "--defined-only", aw.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(aw_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(aw.LIB_PATH)
    for s in declared_symbols():
        assert getattr(lib, s) is not None
    assert set(aw.EXPORTED) == set(declared_symbols())


def test_sm100a_code_in_library(aw):
    out = subprocess.run(["cuobjdump", "--list-elf", aw.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_critical_dt(aw):
    assert aw.aw_abi_version() == 2
    from tests import _indep
    for k in (2, 4, 8, 12, 16):
        for sp in ([10.0, 10.0], [10.0, 7.0, 12.0]):
            assert aw.critical_dt(sp, k, 3.0) == pytest.approx(_indep.critical_dt(k, sp, 3.0), rel=1e-14)
    assert aw.critical_dt([10.0, 10.0], 3, 3.0) == 0.0


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_gpu(aw):
    with pytest.raises(aw.AwError) as ei:
        aw.Grid((16, 16), (150.0, 150.0), 4)
    assert ei.value.status == aw.AW_ECUDA


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: with the CUDA library absent, the first use of the package raises (it never routes
    to the oracle or to torch ops)."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, AW_LIBRARY=str(tmp_path / "no_such_libaw.so"))
    r = subprocess.run([sys.executable, "-c", "import paper_1906_10811_b200 as aw; aw.Grid"], cwd=root, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "ImportError" in r.stderr and "no CPU fallback" in r.stderr


def test_invalid_arguments_rejected_before_device(aw):
    for shape, so in (((16,), 4), ((16, 16), 3), ((16, 16), 18), ((2, 16), 8)):
        with pytest.raises(aw.AwError) as ei:
            aw.Grid(shape, [100.0] * len(shape), so)
        assert ei.value.status in (aw.AW_EINVAL, aw.AW_EUNSUPPORTED)
    with pytest.raises(aw.AwError) as ei:
        aw.Grid((16, 16), (100.0, -1.0), 4)
    assert ei.value.status == aw.AW_EINVAL
