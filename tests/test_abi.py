"""The C-ABI library loads on CPU and exports exactly what include/ifx_abi.h declares."""

import os
import re

from conftest import ROOT

from paper_2511_20714_b200 import _abi


def _declared():
    with open(os.path.join(ROOT, "include", "ifx_abi.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(ifx_\w+)\s*\(", src, re.M)))


def test_header_declarations_match_binding_list():
    assert _declared() == sorted(_abi.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _abi.lib()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.ifx_version() == 1


def test_error_codes_map_to_reference_classes():
    from paper_2511_20714_b200 import errors as E
    assert _abi._ERRORS[_abi.EDIM] is E.DimensionError
    assert _abi._ERRORS[_abi.EMASK] is E.MaskError
    assert _abi._ERRORS[_abi.ECAPACITY] is E.CapacityError
    assert _abi._ERRORS[_abi.ERANGE] is E.OutOfRangeError
    assert _abi._ERRORS[_abi.ECONFIG] is E.ConfigError
    assert issubclass(E.OutOfRangeError, IndexError) and issubclass(E.CapacityError, RuntimeError)


def test_binary_is_sm100a_with_tcgen05_and_tma():
    """cuobjdump: the attention kernel really issues UTCHMMA (tcgen05.mma) and UTMALDG."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        return
    out = subprocess.run([tool, "-sass", _abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "UTCHMMA" in out and "UTMALDG" in out and "LDTM" in out
    assert " HMMA" not in out
