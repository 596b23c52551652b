"""The C-ABI library loads on a CPU host and exports every symbol
include/alyab200.h declares (no compute calls without a GPU)."""

import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "alyab200.h").read_text()
    return sorted(set(re.findall(r"^(?:int|const char\*|int64_t)\s+(ab_\w+)\s*\(", text, flags=re.M)))


def test_library_loads_and_exports_header():
    from paper_2005_05899_b200 import _lib
    lib = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED), set(syms) ^ set(_lib.EXPORTED)
    assert lib.ab_version() == 100
    assert _lib.launch_count() >= 0


def test_invalid_arguments_report_errors():
    """Precondition failures return AB_EINVAL with a message, no device work."""
    import ctypes
    from paper_2005_05899_b200 import _lib
    lib = _lib.lib()
    assert lib.ab_hilbert_cells(10, None, 0, None, None) == -1
    assert b"level" in lib.ab_last_error()
    m = _lib.AbMesh()
    m.n_cat = 1
    m.coords = None
    assert lib.ab_mass(ctypes.byref(m), 0, None, None, None, 32, None) == -1
    assert b"ab_mesh" in lib.ab_last_error()


def test_sm100a_code_only():
    """The shared object carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess
    from paper_2005_05899_b200 import _lib
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
