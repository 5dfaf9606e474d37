"""The C-ABI library loads on CPU and exports exactly what include/ifx_abi.h declares."""

import os
import re

import pytest

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


def test_argument_validation_without_a_gpu():
    """Entry points reject bad arguments with the reference's error classes before any CUDA
    work (so these run on the CPU-only build container)."""
    import ctypes

    import pytest

    from paper_2511_20714_b200 import errors as E

    L = _abi.lib()
    chk = _abi.check
    with pytest.raises(E.DimensionError):  # block copies: too many blocks for one launch
        chk(L.ifx_copy_blocks(None, None, None, 70000, 1, None))
    chk(L.ifx_copy_blocks(None, None, None, 0, 0, None))  # empty batch is a no-op
    with pytest.raises(E.DimensionError):  # group softmax: row stride shorter than the groups
        chk(L.ifx_group_softmax(None, 10, 12, 3, 30, ctypes.c_float(1.0), None, 36, None))
    chk(L.ifx_group_softmax(None, 0, 12, 3, 36, ctypes.c_float(1.0), None, 36, None))
    pool = _abi.KvPool()
    pool.width, pool.page_len, pool.type = 0, 16, _abi.BF16
    with pytest.raises(E.DimensionError):  # bad pool
        chk(L.ifx_kv_move_pages(ctypes.byref(pool), None, 1, 0, None))
    pool.width = 8  # 16-byte rows, fine
    with pytest.raises(E.DimensionError):  # bad direction
        chk(L.ifx_kv_move_pages(ctypes.byref(pool), None, 1, 2, None))
    with pytest.raises(E.DimensionError):
        chk(L.ifx_kv_copy_runs(ctypes.byref(pool), None, -1, 1, None))
    runs = (ctypes.c_int64 * 3)(0, 0, 0)  # a run of zero pages
    with pytest.raises(E.DimensionError):
        chk(L.ifx_kv_copy_runs(ctypes.byref(pool), runs, 1, 1, None))
    pool.width = 3  # 6-byte rows: not 16-byte vectors
    with pytest.raises(E.DimensionError):
        chk(L.ifx_kv_gather(ctypes.byref(pool), None, 0, None, 0, 1, None, None, None))
    p = _abi.AttnParams()
    p.head_dim, p.heads, p.n_q = 96, 1, 1
    with pytest.raises(E.DimensionError):  # EUNSUPPORTED maps to DimensionError
        chk(L.ifx_attn_fwd(ctypes.byref(p), None))
    p.head_dim = 128
    with pytest.raises(E.MaskError):  # a query row with no key at all
        chk(L.ifx_attn_fwd(ctypes.byref(p), None))
    p.n_ctx, p.ctx_slots, p.ctx_page_len = 4, ctypes.c_void_p(16), 24
    with pytest.raises(E.DimensionError):  # paged context needs page_len in {8,...,128}
        chk(L.ifx_attn_fwd(ctypes.byref(p), None))


def test_page_table_batch_api():
    import pytest

    from paper_2511_20714_b200 import errors as E
    from paper_2511_20714_b200.kvcache import KvConfig, PageTable

    pt = PageTable(KvConfig(num_layers=1, head_dim=4, page_len=2, capacity_pages_device=1,
                            capacity_pages_host=8))
    with pytest.raises(E.ConfigError):
        pt.batch_end()
    pt.append(0, "self_attn", 4, 0)  # 2 pages: one device, one host
    pt.drain_moves()
    pt.batch_begin()
    pt.touch_range(0, "self_attn", 2, 4)  # restore page 1, demote page 0
    pt.touch_range(0, "self_attn", 0, 2)  # and back: both moves cancel inside the batch
    assert pt.pending(0)[0] == 0
    pt.batch_end()
    assert len(pt.drain_moves()) == 0
    pt.touch_range(0, "self_attn", 2, 4)  # outside a batch: one D2H + one H2D
    mv = pt.drain_moves()
    assert sorted(mv[:, 2].tolist()) == [0, 1]


def test_one_cublaslt_per_process():
    """The library links the cuBLASLt torch loads: loading it BEFORE torch must not pull in a
    second (toolkit) copy, which made torch's own GEMMs fail with CUBLAS_STATUS_INVALID_VALUE."""
    import subprocess
    import sys
    code = ("import ctypes; ctypes.CDLL(%r); import torch; "
            "print(sorted({l.split()[-1] for l in open('/proc/self/maps') if 'libcublasLt' in l}))"
            % _abi.LIB_PATH)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    paths = eval(out.stdout.strip().splitlines()[-1])
    assert len(paths) == 1, paths


def test_native_comm_unique_id_and_validation():
    """ifx_comm_* (the C-ABI NCCL communicator, SURVEY §8(b) ifx_comm_init): unique ids
    are 128 fresh bytes; bad ranks / ids fail with the reference's error classes before any
    collective (no GPU needed for these paths)."""
    from paper_2511_20714_b200.errors import DimensionError
    from paper_2511_20714_b200.parallel import NativeComm

    a, b = NativeComm.unique_id(), NativeComm.unique_id()
    assert len(a) == 128 and a != b
    with pytest.raises(DimensionError):
        NativeComm(a, 2, 2)  # rank outside [0, world)
    with pytest.raises(DimensionError):
        NativeComm(a, 0, 0)
    with pytest.raises(DimensionError):
        NativeComm(a[:64], 2, 0)
