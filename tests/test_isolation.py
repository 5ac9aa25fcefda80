"""The oracle and the CUDA path share nothing: the product package and the tools
never import or include oracle/, the oracle never imports the product, and bench.py touches the
oracle only in its CPU-baseline / reference legs."""
import ast
import glob
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _imports(path):
    tree = ast.parse(open(path).read())
    out = []
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            out += [(a.name, node) for a in node.names]
        elif isinstance(node, ast.ImportFrom) and node.module:
            out.append((node.module, node))
    return tree, out


def test_product_and_tools_do_not_import_oracle():
    files = glob.glob(os.path.join(ROOT, "paper_1808_09617_b200", "**", "*.py"), recursive=True)
    files += glob.glob(os.path.join(ROOT, "tools", "*.py")) + [os.path.join(ROOT, "datagen.py")]
    for f in files:
        _, imps = _imports(f)
        assert not any(m == "oracle" or m.startswith("oracle.") for m, _ in imps), f


def test_cuda_sources_do_not_include_oracle():
    for f in glob.glob(os.path.join(ROOT, "paper_1808_09617_b200", "csrc", "*")):
        txt = open(f).read()
        assert not re.search(r"#include\s+[<\"].*oracle", txt), f
        assert "oracle_" not in txt, f


def test_oracle_does_not_import_product():
    for f in glob.glob(os.path.join(ROOT, "oracle", "*.py")):
        _, imps = _imports(f)
        assert not any(m.startswith("paper_1808_09617_b200") for m, _ in imps), f
    src = open(os.path.join(ROOT, "oracle", "nndtw_oracle.c")).read()
    assert "nndtw.h" not in src and "nndtw_" not in src.replace("nndtw_oracle", "")


def test_bench_uses_oracle_only_in_baseline_legs():
    tree, imps = _imports(os.path.join(ROOT, "bench.py"))
    allowed = {"cpu_baseline_oracle", "run_reference"}
    for fn in ast.walk(tree):
        if isinstance(fn, ast.FunctionDef):
            for node in ast.walk(fn):
                if isinstance(node, ast.Import) and any(a.name == "oracle" for a in node.names):
                    assert fn.name in allowed, fn.name
    # no module-level import of the oracle
    for node in tree.body:
        if isinstance(node, ast.Import):
            assert all(a.name != "oracle" for a in node.names)
