"""C-ABI library checks that need no GPU: it loads, exports every symbol the
public header declares, and validates arguments before touching the device."""
import ctypes as C
import os

import pytest

from paper_2105_00053_b200 import _native, ops


def test_library_loads_and_exports_header_symbols():
    lib = _native.lib()
    syms = _native.header_symbols()
    assert len(syms) >= 10
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and every declared symbol has a ctypes signature in the binding
    assert set(syms) <= set(_native._SIGS), set(syms) - set(_native._SIGS)


def test_abi_version_and_formats():
    lib = _native.lib()
    assert lib.pnn_abi_version() == 1
    for cfg in [(8, 0), (8, 1), (8, 2), (12, 1), (16, 1)]:
        assert lib.pnn_format_supported(*cfg) == 1
    for cfg in [(16, 2), (32, 2), (1, 0), (17, 0)]:
        assert lib.pnn_format_supported(*cfg) == 0
    assert lib.pnn_code_bytes(8) == 1 and lib.pnn_code_bytes(16) == 2


def test_workspace_query_is_host_only():
    n = ops.quire_gemm_workspace((8, 0), 4096, 4096, 4096)
    # two digit planes per operand + flags
    assert n >= 2 * 4096 * 4096 * 2
    assert ops.quire_gemm_workspace((16, 1), 128, 32, 64) > 0
    assert ops.quire_gemm_workspace((16, 1), 0, 32, 64) == 0


def test_invalid_arguments_fail_loudly_without_gpu():
    lib = _native.lib()
    with pytest.raises(_native.PnnInvalidArgument):
        _native.check(lib.pnn_quire_gemm(8, 0, None, None, None, -1, 4, 4, None, 0, None))
    with pytest.raises(_native.PnnError) as e:
        _native.check(lib.pnn_quire_gemm(16, 2, None, None, None, 4, 4, 4, None, 0, None))
    assert e.value.code == 2
    n = C.c_size_t()
    with pytest.raises(_native.PnnError):
        _native.check(lib.pnn_quire_gemm_workspace(32, 2, 4, 4, 4, C.byref(n)))


def _unused_non_quire_placeholder():
    with pytest.raises(NotImplementedError):
        ops.matmul(None, None, use_quire=False, cfg=(8, 0))


def test_cpp_host_mirror_compiles_and_links(tmp_path):
    """include/pnn_b200/tensor_ops.hpp + libpnn_b200.so build into a C++
    program here (running it needs the GPU: tests/test_cpp_host_gpu.py)."""
    from test_cpp_host_gpu import build_host_ops_test

    exe = build_host_ops_test(str(tmp_path))
    assert os.path.exists(exe)
