"""Guards on the product/oracle boundary (task rule ③).

* The product package and the shared input generators never import the oracle:
  only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
  legs may.
* The binding fails loudly when libmgb200.so is missing (no CPU fallback).
"""
import ast
import importlib.util
import os
import shutil
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _imported_modules(path):
    tree = ast.parse(open(path).read(), filename=path)
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            for a in node.names:
                yield a.name
        elif isinstance(node, ast.ImportFrom):
            if node.module:
                yield node.module
            if node.level and node.module is None:
                for a in node.names:
                    yield a.name


@pytest.mark.parametrize("pkg", ["paper_2405_05047_b200", "problems"])
def test_product_and_generators_do_not_import_oracle(pkg):
    d = os.path.join(ROOT, pkg)
    files = [os.path.join(dp, f) for dp, _, fs in os.walk(d) for f in fs if f.endswith(".py")]
    assert files
    for f in files:
        for mod in _imported_modules(f):
            assert mod.split(".")[0] != "oracle", f"{f} imports {mod}"


def test_bench_imports_oracle_only_inside_baseline_functions():
    """bench.py may call the oracle only lazily (inside the cpu_baseline / reference legs),
    never at module level, so the device path never depends on it."""
    tree = ast.parse(open(os.path.join(ROOT, "bench.py")).read())
    for node in tree.body:
        if isinstance(node, (ast.Import, ast.ImportFrom)):
            names = [a.name for a in node.names] + ([node.module] if getattr(node, "module", None) else [])
            assert all(n.split(".")[0] != "oracle" for n in names if n)


def test_cuda_sources_share_nothing_with_oracle():
    """The CUDA library and the C oracle include no common header."""
    csrc = os.path.join(ROOT, "paper_2405_05047_b200", "csrc")
    for f in os.listdir(csrc):
        txt = open(os.path.join(csrc, f), errors="replace").read()
        assert "oracle" not in "".join(l for l in txt.splitlines(True) if l.lstrip().startswith("#include"))


def test_binding_fails_loudly_without_library(tmp_path):
    src = os.path.join(ROOT, "paper_2405_05047_b200", "__init__.py")
    pkg = tmp_path / "mgb_nolib"
    pkg.mkdir()
    shutil.copy(src, pkg / "__init__.py")
    spec = importlib.util.spec_from_file_location("mgb_nolib", str(pkg / "__init__.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules.pop("mgb_nolib", None)
    with pytest.raises(ImportError, match="no CPU fallback"):
        spec.loader.exec_module(mod)
