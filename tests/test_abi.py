"""The C-ABI library loads and exports every symbol include/pcdn.h declares (CPU, no compute)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pcdn.h")


def header_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^[A-Za-z_][\w \*]*?\b(pcdn_\w+)\s*\(", txt, flags=re.M)))


@pytest.fixture(scope="module")
def libpcdn():
    from paper_1306_4080_b200 import build
    build.build()
    return ctypes.CDLL(build.LIB)


def test_header_declares_the_boundary():
    fns = header_functions()
    for required in ("pcdn_create", "pcdn_bundle_step", "pcdn_solve", "pcdn_objective", "pcdn_get_w"):
        assert required in fns  # SURVEY.md 8(b) / BASELINE.json north_star


def test_library_exports_every_declared_symbol(libpcdn):
    for name in header_functions():
        assert hasattr(libpcdn, name), name


def test_binding_names_match_header():
    from paper_1306_4080_b200 import _abi
    import paper_1306_4080_b200 as pk
    assert sorted(_abi.SIGNATURES) == header_functions()
    for name in header_functions():
        assert callable(getattr(pk, name)), name


def test_host_only_entry_points(libpcdn):
    import paper_1306_4080_b200 as pk
    assert "sm_100a" in pk.pcdn_version()
    a = pk.pcdn_workspace_bytes(1000, 2000, 20000)
    b = pk.pcdn_workspace_bytes(1000, 2000, 40000)
    assert 0 < a < b
    assert pk.pcdn_workspace_bytes(0, 10, 10) == 0
    assert pk.pcdn_last_error(None) == "null context"


def test_library_is_sm100a(libpcdn):
    import subprocess
    from paper_1306_4080_b200 import build
    out = subprocess.run(["cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
