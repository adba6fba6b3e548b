"""The reference's OWN engine tests, run unchanged against the B200 path.

``tools/install_reference.sh`` puts the unmodified reference package and its
test files under baseline/_ref (git-ignored; shipped to the GPU box).  Here
pytest runs ``test_engine.py`` (every class: oracle x 4 overrides, workflow
selection, reports, errors, AA^T symmetric, enhanced tier, reentrant parallel
calls, tiny-tier forced overflow -- reference tests/test_engine.py:22-292)
and ``test_acceptance.py`` (criteria 1-10, including 1: 200 pairs x 4
overrides vs the oracle at rtol 1e-12, and 9: structural invariance across
forced workflows -- test_acceptance.py:73-80, 228-239) with
``sketchgemm.spgemm`` routed to the GPU through refbind (tests/refsuite_plugin.py).
"""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RT = os.path.join(ROOT, "baseline", "_ref", "reference_tests")


@pytest.mark.parametrize("module", ["test_engine.py", "test_acceptance.py"])
def test_reference_suite_through_binding(module):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(os.path.join(RT, module)):
        pytest.skip("reference package not installed (tools/install_reference.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests"), ROOT, env.get("PYTHONPATH", "")])
    # nothing deselected: refbind asks for deterministic values (the
    # reference's bitwise-identical-values guarantee), so the two
    # TestDeterminismAndWorkers tests run too
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "refsuite_plugin",
                        "-p", "no:cacheprovider", "--rootdir", RT, os.path.join(RT, module)],
                       cwd=RT, env=env, capture_output=True, text=True, timeout=1800)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-6000:] + r.stderr[-3000:]
