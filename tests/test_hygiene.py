"""Rules of the tier, checked on the sources (CPU): the product package never
imports the oracle (test infrastructure only; bench.py may use it for the
cpu_baseline / --impl reference arms), has no CPU fallback for the mover, and
every CUDA source builds for sm_100a only."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1904_03684_b200")


def _py_sources():
    for d, _, files in os.walk(PKG):
        for f in files:
            if f.endswith(".py"):
                yield os.path.join(d, f)


def test_product_never_imports_the_oracle():
    pat = re.compile(r"^\s*(import\s+oracle|from\s+oracle\b)", re.M)
    bad = [p for p in _py_sources() if pat.search(open(p).read())]
    assert not bad, bad


def test_missing_library_fails_loudly(monkeypatch):
    """Without libb2m.so the product raises; it never switches to another
    implementation of the mover."""
    import pytest
    from paper_1904_03684_b200 import _capi
    monkeypatch.setattr(_capi, "_lib", None)
    monkeypatch.setattr(_capi, "LIB_PATH", os.path.join(PKG, "no_such_libb2m.so"))
    with pytest.raises(_capi.NativeLibraryMissing, match="missing"):
        _capi.lib()


def test_cuda_builds_target_sm100a_only():
    mk = open(os.path.join(PKG, "csrc", "Makefile")).read()
    assert "arch=compute_100a,code=sm_100a" in mk
    assert not re.search(r"sm_(70|75|80|86|89|90)\b", mk)
