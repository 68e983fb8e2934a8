"""C-ABI boundary checks that need no GPU: the library loads, exports every
function include/laud.h declares, and the ctypes struct mirrors match the
header field-for-field."""
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HDR = (ROOT / "include" / "laud.h").read_text()


def _declared_functions():
    body = re.sub(r"/\*.*?\*/", "", HDR, flags=re.S)
    return sorted(set(re.findall(r"\b(laud_[a-z0-9_]+)\s*\(", body)))


def _struct_fields(name):
    body = re.sub(r"/\*.*?\*/", "", HDR, flags=re.S)
    m = re.search(r"typedef struct %s \{(.*?)\} %s;" % (name, name), body, flags=re.S)
    fields = []
    for decl in m.group(1).split(";"):
        decl = decl.strip()
        if not decl:
            continue
        decl = re.sub(r"^(const\s+)?[a-z_0-9]+\s*", "", decl)
        for part in decl.split(","):
            fields.append(part.strip().lstrip("*").strip())
    return fields


@pytest.fixture(scope="module")
def lib():
    from paper_2308_15949_b200 import _lib
    so = ROOT / "paper_2308_15949_b200" / "_laud.so"
    if not so.exists():
        import __graft_entry__
        __graft_entry__.build()
    return _lib.lib()


def test_every_declared_symbol_is_exported(lib):
    from paper_2308_15949_b200 import _lib
    decl = _declared_functions()
    assert len(decl) >= 12
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(_lib.exported_symbols()) == decl


def test_struct_mirrors_match_header():
    from paper_2308_15949_b200 import _lib
    assert [f for f, _ in _lib.ConvArgs._fields_] == _struct_fields("laud_conv_args")
    assert [f for f, _ in _lib.BlockArgs._fields_] == _struct_fields("laud_block_args")


def test_host_only_entry_points(lib):
    assert b"sm_100a" in lib.laud_version()
    assert lib.laud_scan_workspace_bytes(1024) >= 16 + 8
    assert lib.laud_masker_partial_floats(2, 14, 14, 1024, 2, 1) == 2 * 49
    assert lib.laud_masker_partial_floats(1, 14, 14, 1024, 14, 1) > 1  # layer masker splits
    assert lib.laud_masker_partial_floats(1, 14, 14, 64, 3, 1) == 0    # S does not divide


def test_errors_map_to_reference_taxonomy(lib):
    from paper_2308_15949_b200 import _lib
    from paper_2308_15949_b200.errors import GranularityMismatch, ShapeMismatch
    with pytest.raises(GranularityMismatch):
        _lib.call("laud_spatial_masker", None, 0, 64, 1, 14, 14, 64, 3, 1, None, 0.0,
                  None, None, None, None, None, None)
    with pytest.raises(ShapeMismatch):
        _lib.call("laud_spatial_masker", None, 0, 60, 1, 14, 14, 60, 2, 1, None, 0.0,
                  None, None, None, None, None, None)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2308_15949_b200 import reference as R
    from paper_2308_15949_b200.errors import DeviceError
    import numpy as np
    with pytest.raises(DeviceError):
        R.build_gather_plan(np.ones((1, 2, 2), bool))


def _prototype_arity():
    body = re.sub(r"/\*.*?\*/", "", HDR, flags=re.S)
    out = {}
    for m in re.finditer(r"\b(laud_[a-z0-9_]+)\s*\(([^)]*)\)\s*;", body):
        params = m.group(2).strip()
        out[m.group(1)] = 0 if params in ("", "void") else params.count(",") + 1
    return out


def test_ctypes_signatures_match_header_arity():
    from paper_2308_15949_b200 import _lib
    ar = _prototype_arity()
    for name, (_, args) in _lib._SIGS.items():
        assert len(args) == ar[name], (name, len(args), ar[name])
