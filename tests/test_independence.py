"""Structural guarantees: the product path and the oracle share no code, the
product never falls back to the CPU, and the oracle is test infrastructure only."""
import ast
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2103_14409_b200")
ORACLE = os.path.join(ROOT, "oracle")


def _imports(path):
    mods = set()
    for dirpath, _, files in os.walk(path):
        for f in files:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dirpath, f)).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        mods.update(a.name.split(".")[0] for a in node.names)
                    elif isinstance(node, ast.ImportFrom) and node.module:
                        mods.add(node.module.split(".")[0])
    return mods


def test_product_never_imports_oracle():
    assert "oracle" not in _imports(PKG)


def test_oracle_never_imports_product():
    assert "paper_2103_14409_b200" not in _imports(ORACLE)


def test_no_shared_sources():
    """The C/CUDA sources of the two sides include nothing from each other."""
    def includes(path):
        return [ln for ln in open(path).read().splitlines() if ln.strip().startswith("#include")]

    for dirpath, _, files in os.walk(os.path.join(PKG, "csrc")):
        for f in files:
            assert not any("oracle" in ln for ln in includes(os.path.join(dirpath, f))), f
    for f in os.listdir(ORACLE):
        if f.endswith((".c", ".h")):
            inc = includes(os.path.join(ORACLE, f))
            assert not any("lscat.h" in ln or "csrc" in ln or "common.h" in ln for ln in inc), f


def test_missing_library_fails_loudly(tmp_path):
    from paper_2103_14409_b200 import lscat
    saved = lscat._lib
    try:
        lscat._lib = None
        with pytest.raises(ImportError):
            lscat.load(str(tmp_path / "missing.so"))
    finally:
        lscat._lib = saved


def test_bench_and_smoke_are_the_only_oracle_users():
    """Only tests/, __graft_entry__.py and bench.py may import oracle/."""
    users = []
    for dirpath, dirs, files in os.walk(ROOT):
        if any(p in dirpath for p in ("/tests", "/oracle", "/.git", "/gpurun_out", "/baseline")):
            continue
        for f in files:
            if f.endswith(".py"):
                p = os.path.join(dirpath, f)
                tree = ast.parse(open(p).read())
                for node in ast.walk(tree):
                    if (isinstance(node, ast.ImportFrom) and node.module and
                            node.module.split(".")[0] == "oracle") or (
                            isinstance(node, ast.Import) and
                            any(a.name.split(".")[0] == "oracle" for a in node.names)):
                        users.append(os.path.relpath(p, ROOT))
    assert set(users) <= {"bench.py", "__graft_entry__.py"}, users
