"""CPU-side checks of the C-ABI boundary: the library loads without a GPU
and exports exactly what include/boba_b200.h declares, with the Python
binding's table in sync with the header."""

import re

from conftest import ROOT  # noqa: F401


def header_functions():
    from paper_2306_10410_b200 import _native

    text = open(_native.HEADER_PATH).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"\b(boba_[a-z0-9_]+)\s*\(", text)
    return sorted(set(names))


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2306_10410_b200 import _native

    declared = header_functions()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(_native.lib, name), name
    assert sorted(_native.SIGNATURES) == declared
    assert _native.lib.boba_abi_version() == 1


def test_workspace_queries_are_pure_host():
    from paper_2306_10410_b200 import _native

    lib = _native.lib
    assert lib.boba_compact_workspace_size(1 << 26, 1 << 22) > (1 << 26) // 4
    a = lib.boba_coo_to_csr_workspace_size(1 << 20, 1 << 16, 0)
    assert a > 4 * (1 << 20) * 4
    assert lib.boba_reorder_to_csr_workspace_size(1 << 20, 1 << 16, 0) >= a
    assert lib.boba_spmv_workspace_size(100, 1000) > 0


def test_invalid_arguments_are_reported_not_clamped():
    from paper_2306_10410_b200 import _native

    lib = _native.lib
    # 2m beyond the uint32 position space
    rc = lib.boba_first_occurrence(None, None, 1 << 31, 10, None, 0, None)
    assert rc == _native.BOBA_EINVAL
    assert b"position space" in lib.boba_last_error()
    rc = lib.boba_coo_to_csr(None, None, None, 10, 10, None, None, None, None, None, 0, None)
    assert rc == _native.BOBA_EINVAL
    assert lib.boba_generate_rmat(40, 10, 1, None, None, None) == _native.BOBA_EINVAL
