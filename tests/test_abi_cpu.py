"""CPU-side checks of the drop-in boundary (no GPU needed).

* libfloe_b200.so loads and exports every function include/floe_gpu.h declares;
* it carries sm_100a code only (cuobjdump), built with the TMA bulk-copy path;
* without a GPU, compute entry points fail loudly (FLOE_ERR_CUDA) -- there is
  no CPU fallback to silently succeed.
"""
import re
import shutil
import subprocess
from pathlib import Path

import pytest

import paper_2505_05950_b200 as fb

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "floe_gpu.h").read_text()
    return sorted(set(re.findall(r"\b(floe_gpu_[a-z_]+)\s*\(", text)))


def test_library_built():
    assert fb.library_path().exists(), "run `make` (or __graft_entry__.build())"


def test_exports_every_declared_symbol():
    declared = declared_symbols()
    assert len(declared) >= 20
    exported = fb.exported_symbols()
    missing = [s for s in declared if s not in exported]
    assert not missing, f"declared but not exported: {missing}"
    extra = [s for s in exported if s not in declared]
    assert not extra, f"exported but undeclared: {extra}"


def test_ctypes_binds_every_symbol():
    lib = fb.lib()
    for s in declared_symbols():
        assert hasattr(lib, s)
    assert fb.abi_version() == 1


@pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="cuobjdump absent")
def test_sm100a_only_and_bulk_copy_in_sass():
    out = subprocess.run(["cuobjdump", "-lelf", str(fb.library_path())], capture_output=True,
                         text=True, check=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches
    sass = subprocess.run(["cuobjdump", "-sass", str(fb.library_path())], capture_output=True,
                          text=True, check=True).stdout
    assert "UBLKCP" in sass  # cp.async.bulk (TMA engine) staging in K1/K2
    assert "FFMA2" in sass   # packed fp32x2 math (sm_100)
    assert "IMMA.16832.S8.S8" in sass  # K1: exact integer tensor-core up projection


def test_compute_fails_loudly_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present; covered by the -m gpu suite")
    except ImportError:
        pass
    with pytest.raises(fb.FloeError) as ei:
        fb.Workspace(4096, 14336)
    assert ei.value.status == 2  # FLOE_ERR_CUDA
    assert "workspace_create" in str(ei.value)
    with pytest.raises(fb.FloeError):
        fb.device_info()
