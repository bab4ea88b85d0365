"""CPU checks of the C-ABI boundary: libxbtile.so loads, exports exactly what
include/xbtile.h declares, and the Python binding covers every entry point.
No compute calls (there is no GPU here)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "xbtile.h")
LIB = os.path.join(ROOT, "paper_2104_02184_b200", "libxbtile.so")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(xb_[a-z0-9_]+)\s*\(", src))


def exported():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    return {ln.split()[-1] for ln in out.splitlines() if " T " in ln and " xb_" in " " + ln.split()[-1]}


def test_library_exists():
    assert os.path.exists(LIB), "run __graft_entry__.build() first"


def test_every_declared_symbol_is_exported():
    d, e = declared(), exported()
    assert d, "no declarations parsed"
    assert d - e == set(), f"declared but not exported: {sorted(d - e)}"
    assert e - d == set(), f"exported but not declared: {sorted(e - d)}"


def test_python_binding_covers_header():
    from paper_2104_02184_b200 import _abi
    assert set(_abi.SIGNATURES) == declared()


def test_library_loads_without_gpu():
    import paper_2104_02184_b200 as xb
    assert xb.tile.lib().xb_abi_version() == 1
    p = xb.device_preset("reram_es")
    assert p.kind == xb.EXP_STEP and p.up_down == 0.1 and p.gamma == 2.0
    with pytest.raises(xb.Error, match="unknown name"):
        xb.device_preset("nope")


def test_defaults_mirror_reference():
    """The ABI defaults equal the reference's struct initialisers (via the oracle)."""
    import oracle
    import paper_2104_02184_b200 as xb
    O = oracle.load("restatement")
    a, b = xb.default_io(), O.default("io")
    for f, _ in b._fields_:
        assert getattr(a, f) == getattr(b, f), f
    a, b = xb.default_device(), O.default("device")
    for f, _ in b._fields_:
        assert getattr(a, f) == getattr(b, f), f
    for name in ("ideal", "reram_sb", "reram_es"):
        a, b = xb.device_preset(name), O.preset(name)
        for f, _ in b._fields_:
            assert getattr(a, f) == getattr(b, f), (name, f)


def test_sm100a_cubin():
    """The library carries sm_100a SASS (cross-compiled here)."""
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_compute_without_gpu():
    """There is no CPU fallback: compute entries fail loudly without a GPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2104_02184_b200 as xb
    with pytest.raises(xb.Error, match="no CUDA device"):
        xb.AnalogTile(4, 4)
