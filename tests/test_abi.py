"""CPU checks of the boundary: libsmf.so builds for sm_100a, loads without a GPU,
exports every function include/smf.h declares, and the product package never
imports the oracle."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    txt = open(os.path.join(ROOT, "include", "smf.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(smf_[a-z_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2003_02978_b200 import build
    path = build.build()
    return ctypes.CDLL(path), path


def test_header_declares_the_boundary():
    names = _declared_functions()
    for n in ["smf_create", "smf_destroy", "smf_set_absorption", "smf_set_regularisation",
              "smf_set_iterations", "smf_workspace_bytes", "smf_retrieve", "smf_synchronize",
              "smf_retrieve_host", "smf_status_string", "smf_last_error"]:
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    so, path = lib
    for n in _declared_functions():
        assert hasattr(so, n), n
    # C ABI (unmangled) and built for sm_100a
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_binding_covers_every_symbol(lib):
    from paper_2003_02978_b200 import smf
    assert set(smf.SYMBOLS) == set(_declared_functions())
    assert smf.abi_version() == 1


def test_host_side_calls_without_gpu(lib):
    from paper_2003_02978_b200 import smf
    L = smf._lib
    assert L.smf_status_string(0) == b"SMF_OK"
    assert L.smf_status_string(4) == b"SMF_ERR_NUMERICAL"
    assert smf.supported_bands(72) and smf.supported_bands(32)
    assert smf.supported_bands(425) and smf.supported_bands(5)   # wide path
    assert all(smf.supported_bands(b) for b in list(range(1, 627, 25)) + [626])   # up to 626
    assert not smf.supported_bands(627)                             # largest tested band count
    assert not smf.supported_bands(0)
    h = ctypes.c_void_p()
    assert L.smf_create(None, 72) == smf.SMF_ERR_INVALID_ARGUMENT
    assert L.smf_create(ctypes.byref(h), 0) == smf.SMF_ERR_INVALID_ARGUMENT
    L.smf_destroy(None)   # NULL-safe


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2003_02978_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".c")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "smf_oracle" not in src and "liboracle" not in src, f


def test_missing_library_fails_loudly(tmp_path):
    """The binding raises instead of falling back when libsmf.so is absent."""
    import shutil
    import sys
    pkg = tmp_path / "paper_2003_02978_b200"
    pkg.mkdir()
    shutil.copy(os.path.join(ROOT, "paper_2003_02978_b200", "smf.py"), pkg / "smf.py")
    (pkg / "__init__.py").write_text("")
    code = "import paper_2003_02978_b200.smf"
    r = subprocess.run([sys.executable, "-c", code], cwd=tmp_path, capture_output=True, text=True)
    assert r.returncode != 0 and "libsmf.so not built" in r.stderr


def test_group_partitions_layout():
    """Detector grouping partitions: 5-detector groups over 598
    columns leave a ragged 3-column remainder (598 = 119 x 5 + 3); G >= cols is the
    all-detectors mode; G = 1 is one partition per column."""
    from paper_2003_02978_b200 import smf
    p = smf.group_partitions(598, 5)
    assert len(p) == 120 and p[:3] == [0, 5, 10] and p[-2:] == [590, 595]
    assert smf.group_partitions(7, 3) == [0, 3, 6]
    assert smf.group_partitions(7, 7) == [0] and smf.group_partitions(7, 100) == [0]
    assert smf.group_partitions(4, 1) == [0, 1, 2, 3]
