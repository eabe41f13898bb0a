"""The C-ABI library loads and exports every symbol include/softsnake_b200.h
declares; ctypes mirrors agree with the C struct layout. No compute calls
(there is no GPU here)."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "softsnake_b200.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void\*|const char\*)\s+(ss\w+)\(",
                                 txt, re.M)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__ as g
    g.build()
    from paper_1904_02833_b200 import _native
    return _native.lib()


def test_exports_every_declared_symbol(lib):
    from paper_1904_02833_b200 import _native
    names = _declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), f"{n} missing from libsoftsnake_b200.so"
        assert n in _native.SIGNATURES, f"{n} has no ctypes signature"


def test_abi_version(lib):
    assert lib.ss_abi_version() == 1


def test_struct_layout_matches_c(oracle_mod):
    from paper_1904_02833_b200._abi import SsParams, SsStateView, SsTopology
    L = oracle_mod.lib()
    assert L.or_sizeof_topology() == C.sizeof(SsTopology)
    assert L.or_sizeof_state_view() == C.sizeof(SsStateView)
    assert L.or_sizeof_params() == C.sizeof(SsParams)


def test_no_cpu_fallback_when_library_missing(monkeypatch, tmp_path):
    from paper_1904_02833_b200 import _native
    monkeypatch.setattr(_native, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_native, "_lib", None)
    with pytest.raises(RuntimeError):
        _native.lib()


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1904_02833_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in txt.replace("oracle/", ""), f"{f} references the oracle"
