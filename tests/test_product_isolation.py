"""The product path never reaches the oracle and fails loudly without its CUDA library."""
import ast
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2503_18929_b200")


def _imports(path):
    tree = ast.parse(open(path).read())
    out = set()
    for n in ast.walk(tree):
        if isinstance(n, ast.Import):
            out |= {a.name.split(".")[0] for a in n.names}
        elif isinstance(n, ast.ImportFrom) and n.module:
            out.add(n.module.split(".")[0])
    return out


def test_product_package_never_imports_oracle_or_generator():
    for f in os.listdir(PKG):
        if f.endswith(".py"):
            imps = _imports(os.path.join(PKG, f))
            assert "oracle" not in imps and "tba_synth" not in imps, f
    csrc = os.path.join(PKG, "csrc")
    srcs = [f for f in os.listdir(csrc) if f.endswith((".cu", ".cuh"))]
    assert "abi.cu" in srcs and "tba_device.cuh" in srcs
    for f in srcs:
        assert "oracle" not in open(os.path.join(csrc, f)).read().lower(), f


def test_oracle_imports_nothing_from_the_product():
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith(".py"):
            imps = _imports(os.path.join(ROOT, "oracle", f))
            assert "paper_2503_18929_b200" not in imps and "torch" not in imps, f


def test_generator_holds_no_method_arithmetic():
    # code only (docstrings mention what the generator does NOT compute)
    tree = ast.parse(open(os.path.join(ROOT, "tba_synth", "__init__.py")).read())
    names = {n.attr if isinstance(n, ast.Attribute) else n.id for n in ast.walk(tree)
             if isinstance(n, (ast.Attribute, ast.Name))}
    for word in ("softmax", "logsumexp", "log_softmax", "exp", "logaddexp"):
        assert word not in names, word


def test_missing_library_raises(monkeypatch, tmp_path):
    from paper_2503_18929_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(ImportError):
        _lib.load(str(tmp_path / "libtba.so"))


def test_bench_uses_oracle_only_in_baseline_legs():
    tree = ast.parse(open(os.path.join(ROOT, "bench.py")).read())
    users = set()
    for fn in ast.walk(tree):
        if isinstance(fn, ast.FunctionDef):
            for n in ast.walk(fn):
                if isinstance(n, ast.ImportFrom) and n.module and n.module.startswith("oracle"):
                    users.add(fn.name)
    # the bounded-sample timers of the cpu_baseline legs / --impl reference arm (the multi-process
    # pool's per-group oracle call, and the LM-head sample)
    assert users == {"_oracle_group", "oracle_lmhead_sample"}
