"""The C ABI library loads and exports every entry point include/vqc.h declares
(no GPU needed: symbol lookup only, no compute calls)."""

import ctypes
import os
import re
import subprocess

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "vqc.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vqc_[a-z_]+)\s*\(", text)))


def _lib_path():
    from paper_2404_06314_b200 import build
    return build.build()


def test_header_lists_expected_entry_points():
    names = _declared()
    for must in ("vqc_plan_create", "vqc_forward", "vqc_adjoint", "vqc_run_batch_host",
                 "vqc_workspace_bytes", "vqc_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    path = _lib_path()
    lib = ctypes.CDLL(path)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (vqc_\w+)", out))
    assert set(_declared()) <= exported


def test_abi_version_and_python_binding_agree():
    from paper_2404_06314_b200 import native
    lib = native.load_library()
    assert lib.vqc_abi_version() == 1
    assert set(native.EXPORTED_SYMBOLS) == set(_declared())


def test_kernels_are_sm100a():
    """The fatbin carries sm_100a SASS (no PTX-only or other-arch fallback)."""
    out = subprocess.run(["cuobjdump", "--list-elf", _lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out
