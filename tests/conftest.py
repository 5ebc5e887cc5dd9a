import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C-ABI on cuda:0)")
    config.addinivalue_line("markers", "slow: longer CPU test")


def build_lib():
    """Compile libdbk.so (and the oracle's C file) without importing the package first."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_dbk_build", os.path.join(ROOT, "paper_2503_05248_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.build()
