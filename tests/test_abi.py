"""The C-ABI library builds for sm_100a, loads without a GPU, and exports every
entry point include/timrun.h declares (CPU-only: no compute calls)."""

import ctypes
import re
import subprocess

from paper_2507_16784_b200 import _lib as L
from paper_2507_16784_b200.build import LIB, ROOT, build


def _declared():
    text = (ROOT / "include" / "timrun.h").read_text()
    return sorted(set(re.findall(r"\b(tim_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    build()
    lib = ctypes.CDLL(str(LIB))
    declared = _declared()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(L.SIGNATURES), set(declared) ^ set(L.SIGNATURES)
    assert L.load().tim_abi_version() == 1


def test_library_is_sm100a_with_tensor_core_and_tma_code():
    build()
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", str(LIB)], capture_output=True,
                                       text=True).stdout or "arch = sm_100a" in sass
    assert "HMMA" in sass        # mma.sync QK^T / PV tiles
    assert "UBLKCP" in sass      # cp.async.bulk page-row staging
    assert "LDSM" in sass
