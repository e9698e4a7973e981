"""The C-ABI library builds, loads without a GPU and exports every declared symbol."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "pdhg_b200.h"


@pytest.fixture(scope="module")
def lib():
    from paper_2603_03150_b200 import build

    build.build()
    from paper_2603_03150_b200 import _native

    return _native.load()


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pdhg_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_abi():
    names = declared_functions()
    from paper_2603_03150_b200 import _native

    assert sorted(_native.EXPORTS) == names


def test_every_declared_symbol_is_exported(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert ctypes.cast(getattr(lib, name), ctypes.c_void_p).value


def test_abi_version_and_error_channel(lib):
    from paper_2603_03150_b200 import _native

    assert lib.pdhg_abi_version() == _native.ABI_VERSION == 6
    assert isinstance(lib.pdhg_last_error(), bytes)


def test_workspace_sizes(lib):
    small = lib.pdhg_workspace_bytes(10, 20)
    big = lib.pdhg_workspace_bytes(5_000_000, 10_000_000)
    assert 0 < small < big
    # 7 n-vectors + 4 m-vectors of fp64 dominate
    assert big >= (7 * 10_000_000 + 4 * 5_000_000) * 8


def test_bad_arguments_fail_loudly_without_gpu(lib):
    from paper_2603_03150_b200 import _native

    rc = lib.pdhg_ctx_create(None, None, 0, None, None)
    assert rc == -1
    assert b"null" in lib.pdhg_last_error()
    with pytest.raises(_native.NativeError):
        _native.check(rc)


def test_sm100a_code_in_library():
    import shutil
    import subprocess

    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    so = ROOT / "paper_2603_03150_b200" / "libpdhg_b200.so"
    out = subprocess.run([cuobjdump, "--list-elf", str(so)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
