"""Every module of the package (and the bench / entry scripts) imports on a
CPU-only host: catches syntax and import errors in modules whose behaviour is
only exercised by the -m gpu tests."""
import importlib
import os
import pkgutil
import py_compile

import pytest

import paper_2212_04540_b200 as pkg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name", sorted(m.name for m in pkgutil.iter_modules(pkg.__path__)
                                         if m.name != "libkgq"))   # the .so is loaded via ctypes (test_abi)
def test_module_imports(name):
    importlib.import_module(f"paper_2212_04540_b200.{name}")


@pytest.mark.parametrize("path", ["bench.py", "__graft_entry__.py", "datasets/make_reference_datasets.py",
                                  "datasets/run_reference_training.py"] +
                         sorted(os.path.join("tools", f) for f in os.listdir(os.path.join(ROOT, "tools"))
                                if f.endswith(".py")))
def test_script_compiles(path):
    py_compile.compile(os.path.join(ROOT, path), doraise=True)
