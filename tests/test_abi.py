"""The C-ABI library loads and exports every symbol include/lobra.h declares (CPU)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "lobra.h")).read()
    return sorted(set(re.findall(r"LOBRA_API\s+[\w\s\*]+?\b(lobra_\w+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    d = _declared()
    for name in ("lobra_lora_fwd", "lobra_lora_bwd", "lobra_dispatch", "lobra_adapter_allreduce"):
        assert name in d


def test_library_exports_every_declared_symbol():
    from paper_2509_01193_b200 import _lib
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_declared()) == set(_lib.EXPORTED)


def test_library_is_sm100a_and_has_tcgen05():
    """The built .so carries sm_100a SASS with tcgen05 MMA / TMA / TMEM instructions."""
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump unavailable")
    from paper_2509_01193_b200 import _lib
    out = subprocess.run([cuobjdump, "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for mnemonic in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert mnemonic in out, mnemonic


def test_host_errors_without_gpu():
    """Argument validation runs before any device work (works with no GPU)."""
    from paper_2509_01193_b200 import _lib
    with pytest.raises(_lib.LobraError):
        _lib.lobra_lora_workspace_bytes(_lib.LOBRA_BF16, 100, 64, [4], [0], [4], [1.0])
    n = _lib.lobra_lora_workspace_bytes(_lib.LOBRA_BF16, 128, 64, [4, 300], [0, 1], [4, 16], [1.0, 2.0])
    assert n > 0
    assert _lib.lobra_launch_count() >= 0
