"""CPU-side checks of the C ABI: libig.so loads, exports every symbol include/ig.h declares,
and validates arguments before touching a device (no compute calls: there is no GPU here)."""

import ctypes as C
import os
import re

import pytest

from paper_2009_10863_b200 import _lib
from paper_2009_10863_b200.ig import shard_range

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "ig.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ig_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_2009_10863_b200.build import build

    build()
    return _lib.lib()


def test_header_declares_the_north_star_calls():
    names = _declared()
    for n in ("ig_create", "ig_form_guess", "ig_update", "ig_destroy"):
        assert n in names


def test_every_declared_symbol_is_exported(L):
    names = _declared()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(names) == set(_lib._SIGS), "binding signatures must mirror the header"


def test_shared_object_is_sm100a(L):
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize(
    "args,needle",
    [
        ((0, 1, 8, 0), "N must be"),
        ((10, 9, 8, 0), "unknown method"),
        ((10, 1, 0, 0), "history size"),
        ((10, 1, 33, 0), "history size"),
        ((10, 2, 4, 4), "degree"),  # M >= m+1
        ((10, 2, 4, -1), "degree"),
        ((10, 4, 3, 3), "degree"),
    ],
)
def test_create_validates_arguments_without_a_device(L, args, needle):
    assert L.ig_create(*args) is None
    assert needle in L.ig_last_error().decode()


def test_null_handle_calls_fail_cleanly(L):
    assert L.ig_form_guess(None, None, None) == _lib.IG_E_ARG
    assert L.ig_update(None, None, None) == _lib.IG_E_ARG
    assert L.ig_reset(None) == _lib.IG_E_ARG
    assert L.ig_next_slot(None) is None
    L.ig_destroy(None)


def test_batch_calls_validate_arguments_without_a_device(L):
    import ctypes as C

    one_null = (C.c_void_p * 1)(None)
    for fn in (L.ig_form_guess_batch, L.ig_update_batch, L.ig_form_guess_batch_host, L.ig_update_batch_host):
        assert fn(0, None, None, None) == 0  # an empty batch is a no-op
        assert fn(-1, None, None, None) == _lib.IG_E_ARG
        assert fn(1, None, None, None) == _lib.IG_E_ARG
        assert fn(1, one_null, one_null, one_null) == _lib.IG_E_ARG  # NULL handle


def test_storage_bytes(L):
    assert L.ig_storage_bytes(1000, 1, 8) == 2 * 8 * 1024 * 8  # 2M slabs, ld rounded to 32
    assert L.ig_storage_bytes(1000, 2, 8) == 8 * 1024 * 8
    assert L.ig_storage_bytes(0, 1, 8) == 0


@pytest.mark.parametrize("N,G", [(10, 3), (2 ** 21, 8), (7, 7), (5, 8)])
def test_shard_range_partitions(N, G):
    rs = [shard_range(N, G, r) for r in range(G)]
    assert rs[0][0] == 0 and rs[-1][1] == N
    assert all(rs[i][1] == rs[i + 1][0] for i in range(G - 1))
    sizes = [hi - lo for lo, hi in rs]
    assert max(sizes) - min(sizes) <= 1


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2009_10863_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).replace("oracle/", ""), f


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    """No CPU fallback anywhere in the product path: without libig.so every call raises."""
    import pytest

    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "libig.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.lib()
    from paper_2009_10863_b200 import ig

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        ig.ig_total_launches()
