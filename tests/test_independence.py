"""The oracle and the product share nothing, and the oracle is test infrastructure
only (task rules ③): checked mechanically on the sources.

* oracle/ never references the product (package, library, ABI header, csrc);
* the product (package, csrc, include/) never references the oracle;
* inputs/ (the one module both sides use: seeded generators) references neither;
* outside tests/, only bench.py's cpu_baseline / reference legs and
  __graft_entry__.smoke() import the oracle.
"""
from __future__ import annotations

import ast
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sources(rel, exts=(".py", ".c", ".h", ".cu", ".cuh", ".cpp")):
    base = os.path.join(ROOT, rel)
    for dp, _, fs in os.walk(base):
        for f in fs:
            if f.endswith(exts):
                yield os.path.join(dp, f)


PRODUCT_TOKENS = re.compile(r"paper_2306_11148_b200|libmoa\b|moa\.h\b|csrc|moa_gemm|moa_internal|moa_ptx")
ORACLE_TOKENS = re.compile(r"\boracle\b|moa_oracle|liboracle")


def _code(path):
    """The code of a source file without comments / docstrings: for C-family files
    the text minus /* */ and // comments; for Python the imported module names and
    the non-docstring string constants (library paths live there)."""
    src = open(path).read()
    if not path.endswith(".py"):
        src = re.sub(r"/\*.*?\*/", " ", src, flags=re.S)
        return "\n".join(l.split("//")[0] for l in src.splitlines())
    tree = ast.parse(src)
    doc = set()
    for node in ast.walk(tree):
        if isinstance(node, (ast.Module, ast.FunctionDef, ast.AsyncFunctionDef, ast.ClassDef)) and node.body:
            first = node.body[0]
            if isinstance(first, ast.Expr) and isinstance(first.value, ast.Constant):
                doc.add(id(first.value))
    parts = []
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            parts += [a.name for a in node.names]
        elif isinstance(node, ast.ImportFrom):
            parts.append(node.module or "")
        elif isinstance(node, ast.Constant) and isinstance(node.value, str) and id(node) not in doc:
            parts.append(node.value)
    return "\n".join(parts)


def test_oracle_never_references_the_product():
    hits = [(p, m.group(0)) for p in _sources("oracle") for m in PRODUCT_TOKENS.finditer(_code(p))]
    assert not hits, hits


def test_product_never_references_the_oracle():
    hits = [(p, m.group(0)) for rel in ("paper_2306_11148_b200", "include") for p in _sources(rel)
            for m in ORACLE_TOKENS.finditer(_code(p))]
    assert not hits, hits


def test_inputs_reference_neither_side():
    for p in _sources("inputs"):
        code = _code(p)
        assert not PRODUCT_TOKENS.search(code), p
        assert not ORACLE_TOKENS.search(code), p


def _oracle_import_sites(path):
    tree = ast.parse(open(path).read())
    sites = []

    def visit(node, func):
        for ch in ast.iter_child_nodes(node):
            f = ch.name if isinstance(ch, (ast.FunctionDef, ast.AsyncFunctionDef)) else func
            if isinstance(ch, ast.ImportFrom) and (ch.module or "").split(".")[0] == "oracle":
                sites.append(func)
            if isinstance(ch, ast.Import) and any(a.name.split(".")[0] == "oracle" for a in ch.names):
                sites.append(func)
            visit(ch, f)

    visit(tree, None)
    return sites


def test_oracle_imported_only_by_the_allowed_legs():
    assert set(_oracle_import_sites(os.path.join(ROOT, "bench.py"))) <= {"cpu_oracle_sample", "run_reference"}
    assert set(_oracle_import_sites(os.path.join(ROOT, "__graft_entry__.py"))) <= {"smoke"}
    for p in _sources("tools", exts=(".py",)):
        assert not _oracle_import_sites(p) or "experiments" in p or p.endswith("sanitize_run.py"), p
