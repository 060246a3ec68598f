"""The oracle and the CUDA path share no code, and the product path has no CPU fallback.

Checks (no GPU needed):
  * nothing in the product (package, harness, seeded input generators) imports ``oracle``;
  * the oracle imports nothing of the product, and its C source includes only system headers;
  * the kernels/runtime include only their own headers (csrc/ + include/moe.h) plus NCCL;
  * using the binding with the library missing fails loudly instead of falling back.
"""
from __future__ import annotations

import ast
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2512_16473_b200")


def _py_files(*paths):
    for p in paths:
        if p.endswith(".py"):
            yield p
            continue
        for dirpath, _, files in os.walk(p):
            for f in files:
                if f.endswith(".py"):
                    yield os.path.join(dirpath, f)


def _imported_roots(path):
    tree = ast.parse(open(path).read(), filename=path)
    roots = set()
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            roots.update(a.name.split(".")[0] for a in node.names)
        elif isinstance(node, ast.ImportFrom) and node.level == 0 and node.module:
            roots.add(node.module.split(".")[0])
    return roots


def test_product_never_imports_oracle():
    product = [PKG, os.path.join(ROOT, "harness.py"), os.path.join(ROOT, "inputs")]
    offenders = [p for p in _py_files(*product) if "oracle" in _imported_roots(p)]
    assert not offenders, offenders


def test_oracle_never_imports_product():
    banned = {"paper_2512_16473_b200", "harness"}
    offenders = [p for p in _py_files(os.path.join(ROOT, "oracle")) if _imported_roots(p) & banned]
    assert not offenders, offenders
    src = open(os.path.join(ROOT, "oracle", "oracle.c")).read()
    local = re.findall(r'#include\s+"([^"]+)"', src)
    assert local == [], f"oracle.c includes local headers {local}; it must share nothing with csrc/"


def test_kernels_include_only_their_own_headers():
    csrc = os.path.join(PKG, "csrc")
    own = set(os.listdir(csrc)) | {"moe.h", "nccl.h"}
    for f in os.listdir(csrc):
        if f.endswith((".cu", ".cuh", ".cpp", ".h")):
            for inc in re.findall(r'#include\s+"([^"]+)"', open(os.path.join(csrc, f)).read()):
                assert inc in own, f"{f} includes {inc}"
                assert "oracle" not in inc and "inputs" not in inc


def test_binding_fails_loudly_without_library():
    env = dict(os.environ, MOE_LIB_PATH="/nonexistent/libmoe.so")
    code = "import paper_2512_16473_b200 as m; m.lib()"  # the library is opened on first use
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode != 0, "using the binding without libmoe.so must raise"
    assert "ImportError" in r.stderr and "libmoe.so" in r.stderr
