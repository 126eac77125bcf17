"""The C-ABI library loads on a CPU-only host and exports every symbol include/ksb.h declares."""
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "ksb.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ksb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "ksb_cg_solve" in syms and "ksb_spmm" in syms and "ksb_mesh_box" in syms
    assert len(syms) >= 30


def test_library_exports_every_declared_symbol():
    from paper_2103_02824_b200 import _native
    missing = [s for s in declared_symbols() if not hasattr(_native.lib, s)]
    assert not missing, missing


def test_binding_prototypes_cover_header():
    from paper_2103_02824_b200 import _native
    assert set(declared_symbols()) == set(_native.PROTOTYPES)


def test_error_codes_match_reference_strings():
    from paper_2103_02824_b200 import _native
    # proj/include/ksafem/types.hpp:20-32 codes used across the reference
    want = ["nonconvergence", "mismatched-spaces", "singular-quadrature", "ambiguous-selection", "internal",
            "invalid-argument", "invalid-domain", "hierarchy", "io"]
    for i, name in enumerate(want, start=1):
        assert _native.lib.ksb_code_name(i).decode() == name


def test_invalid_domain_error_crosses_abi_as_code():
    import paper_2103_02824_b200 as kb
    import pytest
    with pytest.raises(kb.KsbError) as e:
        kb.Mesh.box([0, 0, 0], [1, 0, 1], 2)
    assert e.value.code == "invalid-domain"
    with pytest.raises(kb.KsbError) as e:
        kb.Mesh.box([0, 0, 0], [1, 1, 1], 0)
    assert e.value.code == "invalid-domain"
