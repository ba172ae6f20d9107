"""CPU-side checks of the C ABI: the library loads and exports every declared symbol."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "acp_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(acp_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_five_calls():
    syms = declared_symbols()
    for s in ["acp_ground_state", "acp_compress", "acp_apply_chi0", "acp_dyson", "acp_dynamical_matrix"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    import paper_1605_08021_b200 as pkg
    lib = ctypes.CDLL(pkg.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared_symbols()) == set(pkg.EXPORTED)


def test_version_string_and_arch():
    import paper_1605_08021_b200 as pkg
    assert "sm_100a" in pkg.version()


def test_no_oracle_import_in_product_path():
    pkg_dir = os.path.join(ROOT, "paper_1605_08021_b200")
    for dirpath, _, files in os.walk(pkg_dir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
