"""Drop-in check of the boundary: the reference's OWN unit tests
(`/root/reference/pkg/tests`) run against this package, imported under the
reference's module names (`wrapsched`, `wrapsched.core`, ... aliased to
`paper_2202_01306_b200.*` by a generated shim).  Only present in the build
container (the reference tree does not travel to the GPU box): skipped
elsewhere.

The private simulator helpers those tests import (`_compute_duration`,
`_Item`/`_link`/`_run`, test_simulator.py:92, 242) are restated in
simulator.py over the native plan's duration rule.  Excluded: the modules
SURVEY §2 marks out of scope (analytics, ticksim, hardness, gantt, cli,
acceptance; test_simulator.py:253 compares against the out-of-scope
fixed-tick estimator)."""

import os
import subprocess
import sys
import textwrap

import pytest

REF_TESTS = "/root/reference/pkg/tests"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MODULES = ("core", "errors", "profiler", "packing", "taskgraph", "simulator", "search", "fileio")
FILES = ("test_core.py", "test_packing.py", "test_taskgraph.py", "test_search.py", "test_profiler.py",
         "test_simulator.py")
DESELECT = ("test_simulator.py::test_tick_reference_close_on_small_graph",)


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference tree not present")
def test_reference_unit_tests_pass_against_the_product(tmp_path):
    shim = tmp_path / "wrapsched"
    shim.mkdir()
    (shim / "__init__.py").write_text(textwrap.dedent(f"""
        import importlib, sys
        from paper_2202_01306_b200 import *  # noqa: F401,F403
        for _m in {MODULES!r}:
            sys.modules["wrapsched." + _m] = importlib.import_module("paper_2202_01306_b200." + _m)
    """))
    # ticksim (the fixed-tick cross-check estimator) is out of scope; test_simulator imports it
    (shim / "ticksim.py").write_text("def simulate_fixed_tick(*a, **k):\n    raise NotImplementedError\n")
    names = [os.path.join(REF_TESTS, f) for f in FILES]
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir", str(tmp_path),
           "-o", "addopts=", *names]
    cmd += ["-k", "not (" + " or ".join(d.split("::")[1] for d in DESELECT) + ")"]
    env = dict(os.environ, PYTHONPATH=f"{tmp_path}{os.pathsep}{ROOT}", PYTHONDONTWRITEBYTECODE="1")
    p = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=600)
    tail = "\n".join(p.stdout.splitlines()[-15:])
    print(tail)
    assert p.returncode == 0, tail + p.stderr[-2000:]
